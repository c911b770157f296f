// step.cu -- NEXT-1: the vortex-method time step around evaluate.
// "The Navier-Stokes system is solved by a simultaneous update of the particle
// positions to account for convection, of the particle strengths to account
// for vortex stretching, and of the particle width to account for diffusion"
// (P:69), with d sigma^2/dt = 2 nu (Eq. 4).  Two-stage midpoint
// Runge-Kutta (the paper names no integrator; SPEC S:498 uses RK2):
//   stage 1: (u1, s1) = FMM(x, alpha, sigma)
//   half   : x_h = x + dt/2 u1, alpha_h = alpha + dt/2 s1, sigma_h^2 = sigma^2 + nu dt
//   stage 2: (u2, s2) = FMM(x_h, alpha_h, sigma_h)
//   step   : x' = x + dt u2, alpha' = alpha + dt s2, sigma'^2 = sigma^2 + 2 nu dt (exact)
// Positions are re-wrapped into the periodic cell by the next set_particles.
#include "ctx.cuh"

namespace fmmb {

namespace {

// y_out = y + h * k for [n][3] arrays; sigma_out = sqrt(sigma^2 + 2 nu t) in double
__global__ void k_axpy3(const float* __restrict__ x, const float* __restrict__ a, const float* __restrict__ s,
                        const float* __restrict__ u, const float* __restrict__ da, int64_t n, double h, double two_nu_t,
                        float* __restrict__ xo, float* __restrict__ ao, float* __restrict__ so) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int d = 0; d < 3; ++d) {
      xo[3 * i + d] = (float)((double)x[3 * i + d] + h * (double)u[3 * i + d]);
      ao[3 * i + d] = (float)((double)a[3 * i + d] + h * (double)da[3 * i + d]);
    }
    const double s2 = (double)s[i] * (double)s[i] + two_nu_t;
    so[i] = (float)sqrt(s2);
  }
}

__global__ void k_fill(float* __restrict__ p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

}  // namespace

void fill_f32(Ctx& c, float* p, int64_t n, float v) {
  if (n <= 0) return;
  unsigned g = nblocks(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  FMM_LAUNCH(c, k_fill, g, 256, 0, p, n, v);
}

void step_stage_update(Ctx& c, const float* x, const float* a, const float* s, const float* u, const float* da,
                       int64_t n, double h, double two_nu_t, float* xo, float* ao, float* so) {
  if (n <= 0) return;
  unsigned g = nblocks(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  FMM_LAUNCH(c, k_axpy3, g, 256, 0, x, a, s, u, da, n, h, two_nu_t, xo, ao, so);
}

}  // namespace fmmb
