// common.cuh -- shared device/host helpers of the CUDA product path.
// (No code here is shared with oracle/: the oracle is an independent program.)
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <type_traits>

#include "../../include/fmm.h"

namespace fmmb {

constexpr int kMaxLevel = 21;      // 63-bit keys: 21 levels per axis
constexpr int kImgCentre = 13;     // image index of the zero shift
constexpr int kMaxOrder = 16;      // p <= 16 (degrees 0..15)
constexpr double kPi = 3.14159265358979323846;

struct FmmError : std::runtime_error {
  fmm_status code;
  FmmError(fmm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FMM_CUDA(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw ::fmmb::FmmError(e_ == cudaErrorMemoryAllocation ? FMM_E_OOM : FMM_E_CUDA,       \
                             std::string(#x) + ": " + cudaGetErrorString(e_) + " at " +      \
                                 __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

#define FMM_LAUNCH_CHECK() FMM_CUDA(cudaGetLastError())

// Launch one of this library's kernels on the context stream and count it
// (fmm_stats.launches: the bench's gpu_launches claim).
#define FMM_LAUNCH(ctx, kern, grid, block, smem, ...)                  \
  do {                                                                 \
    kern<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);      \
    ++(ctx).launches;                                                  \
    FMM_CUDA(cudaGetLastError());                                      \
  } while (0)

// The same on an explicit stream (the multi-GPU comm stream).
#define FMM_LAUNCH_ON(ctx, strm, kern, grid, block, smem, ...)        \
  do {                                                                 \
    kern<<<(grid), (block), (smem), (strm)>>>(__VA_ARGS__);            \
    ++(ctx).launches;                                                  \
    FMM_CUDA(cudaGetLastError());                                      \
  } while (0)

// Debug mode (environment FMM_POISON=1, tests/test_gpu_poison.py; the stand-in
// for compute-sanitizer, which this GPU pool does not run): every device buffer
// gets a guard zone of kGuardBytes after it; new storage is filled with 0xFF
// bytes (NaN / -1), so a kernel reading memory that no kernel wrote changes the
// results, and the guard zones are checked after every set_particles and
// evaluate (a write up to kGuardBytes past a buffer's end raises FMM_E_INTERNAL).
constexpr size_t kGuardBytes = 4096;
bool poison_mode();
void* dev_alloc(size_t bytes);        // cudaMalloc (+ poison fill and guard zone in debug mode)
void dev_free(void* p);
void guard_check(const char* where);  // throws FmmError(FMM_E_INTERNAL) on a damaged guard zone

// Grow-only device buffer owned by a context.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { if (p) dev_free(p); }
  // contents are not preserved
  void reserve(size_t n) {
    if (n <= cap && p) return;
    if (p) { dev_free(p); p = nullptr; cap = 0; }
    size_t m = n ? n : 1;
    p = (T*)dev_alloc(m * sizeof(T));
    cap = m;
  }
  // contents [0, keep) are preserved (stream-ordered copy)
  void grow_keep(size_t n, size_t keep, cudaStream_t s) {
    if (n <= cap && p) return;
    size_t m = n ? n : 1;
    if (m < cap + cap / 2) m = cap + cap / 2;
    T* q = (T*)dev_alloc(m * sizeof(T));
    if (p && keep) FMM_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) { FMM_CUDA(cudaStreamSynchronize(s)); dev_free(p); }
    p = q;
    cap = m;
  }
  void release() { if (p) dev_free(p); p = nullptr; cap = 0; }
};

inline unsigned nblocks(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// ---------------------------------------------------------------- complex --
template <typename T>
struct cpx { T re, im; };

template <typename T>
__host__ __device__ __forceinline__ cpx<T> cmul(cpx<T> a, cpx<T> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
// a * conj(b)
template <typename T>
__host__ __device__ __forceinline__ cpx<T> cmulc(cpx<T> a, cpx<T> b) {
  return {a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im};
}

__host__ __device__ __forceinline__ int cidx(int n, int m) { return n * (n + 1) / 2 + m; }

// coefficient (n, m) of a real-source expansion for any sign of m:
// C_n^{-m} = (-1)^m conj(C_n^m).
template <typename T>
__device__ __forceinline__ cpx<T> cget(const cpx<T>* C, int n, int m) {
  if (m >= 0) return C[cidx(n, m)];
  cpx<T> v = C[cidx(n, -m)];
  v.im = -v.im;
  if (m & 1) { v.re = -v.re; v.im = -v.im; }
  return v;
}

// Regular solid harmonics R_n^m(x), 0 <= m <= n < P (Cheng et al. basis,
// P:109): R_0^0 = 1, R_m^m = -(x+iy)/(2m) R_{m-1}^{m-1}, R_{m+1}^m = z R_m^m,
// R_n^m = ((2n-1) z R_{n-1}^m - r^2 R_{n-2}^m) / ((n-m)(n+m)).
template <typename T>
__device__ void regular_harmonics(T x, T y, T z, int P, cpx<T>* R) {
  T r2 = x * x + y * y + z * z;
  R[0] = {T(1), T(0)};
  for (int m = 1; m < P; ++m) {
    cpx<T> p = R[cidx(m - 1, m - 1)];
    T s = T(-1) / T(2 * m);
    R[cidx(m, m)] = {s * (x * p.re - y * p.im), s * (x * p.im + y * p.re)};
  }
  for (int m = 0; m + 1 < P; ++m) {
    cpx<T> p = R[cidx(m, m)];
    R[cidx(m + 1, m)] = {z * p.re, z * p.im};
  }
  for (int m = 0; m < P; ++m)
    for (int n = m + 2; n < P; ++n) {
      cpx<T> a = R[cidx(n - 1, m)], b = R[cidx(n - 2, m)];
      T inv = T(1) / (T(n - m) * T(n + m));
      T c1 = T(2 * n - 1) * z;
      R[cidx(n, m)] = {(c1 * a.re - r2 * b.re) * inv, (c1 * a.im - r2 * b.im) * inv};
    }
}

// Column m of the irregular solid harmonics I_n^m(x), m <= n < P2:
// I_0^0 = 1/r, I_m^m = -(2m-1)(x+iy)/r^2 I_{m-1}^{m-1},
// I_{m+1}^m = (2m+1) z/r^2 I_m^m,
// I_n^m = ((2n-1) z I_{n-1}^m - (n-1-m)(n-1+m) I_{n-2}^m)/r^2.
template <typename T>
__device__ void irregular_column(T x, T y, T z, int m, int P2, cpx<T>* I) {
  T r2 = x * x + y * y + z * z;
  T ir2 = T(1) / r2;
  cpx<T> d = {T(1) / sqrt(r2), T(0)};
  for (int i = 1; i <= m; ++i) {
    T s = -T(2 * i - 1) * ir2;
    d = {s * (x * d.re - y * d.im), s * (x * d.im + y * d.re)};
  }
  if (m >= P2) return;
  I[cidx(m, m)] = d;
  if (m + 1 >= P2) return;
  cpx<T> a = {T(2 * m + 1) * z * ir2 * d.re, T(2 * m + 1) * z * ir2 * d.im};
  I[cidx(m + 1, m)] = a;
  cpx<T> b = d;
  for (int n = m + 2; n < P2; ++n) {
    T c1 = T(2 * n - 1) * z, c2 = T(n - 1 - m) * T(n - 1 + m);
    cpx<T> v = {(c1 * a.re - c2 * b.re) * ir2, (c1 * a.im - c2 * b.im) * ir2};
    I[cidx(n, m)] = v;
    b = a;
    a = v;
  }
}

// compile-time loop: f(integral_constant<int, i>) for i = B, B+S, ... (excluding E)
template <int B, int E, int S, typename F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr ((S > 0 && B < E) || (S < 0 && B > E)) {
    f(std::integral_constant<int, B>{});
    sfor<B + S, E, S>(f);
  }
}

__host__ __device__ constexpr int ci(int n, int m) { return n * (n + 1) / 2 + m; }

}  // namespace fmmb
