"""CPU oracle for the FMM vortex-particle hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product path (``paper_1106_5273_b200``) never imports it and shares no
code with it.

The arithmetic lives in ``fmm_oracle.c`` (plain double-precision C, OpenMP over
independent targets only); this module is ctypes marshalling plus numpy
glue.  See ``fmm_oracle.h`` for the function-by-function citations of
PAPER.md (Yokota et al., arXiv 1106.5273).

Parity pins: every function here is pinned by ``tests/test_oracle_*.py``
against closed forms, library routines (scipy ``lpmv``/``erf``), brute force
and invariants; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fmm_oracle.c")
_HDR = os.path.join(_HERE, "fmm_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, OpenMP, no FMA contraction)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + ".tmp.%d" % os.getpid()
        cmd = ["gcc", "-std=gnu11", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        d = C.POINTER(C.c_double)
        i64 = C.c_int64
        pi64 = C.POINTER(C.c_int64)
        pu64 = C.POINTER(C.c_uint64)
        L.or_cutoff_g.restype = C.c_double
        L.or_cutoff_g.argtypes = [C.c_double]
        L.or_direct.restype = None
        L.or_direct.argtypes = [i64, d, d, i64, d, d, d, C.c_double, C.c_int, d, d]
        for nm in ("or_regular", "or_irregular"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, d]
        L.or_p2m.argtypes = [C.c_int, i64, d, d, d, d]
        L.or_m2m.argtypes = [C.c_int, d, d, d]
        L.or_m2l.argtypes = [C.c_int, d, d, d]
        L.or_l2l.argtypes = [C.c_int, d, d, d]
        L.or_l2p_derivs.argtypes = [C.c_int, d, d, d, d, d]
        L.or_m2p.restype = C.c_double
        L.or_m2p.argtypes = [C.c_int, d, d]
        L.or_fmm_new.restype = C.c_void_p
        L.or_fmm_new.argtypes = [i64, d, d, d, C.c_void_p]
        for nm in ("or_fmm_free", "or_fmm_traverse", "or_fmm_evaluate"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [C.c_void_p]
        for nm in ("or_fmm_ncells", "or_fmm_np2p", "or_fmm_nm2l"):
            getattr(L, nm).restype = i64
            getattr(L, nm).argtypes = [C.c_void_p]
        L.or_fmm_box.argtypes = [C.c_void_p, d, d]
        L.or_fmm_keys.argtypes = [C.c_void_p, pu64, pi64]
        L.or_fmm_positions.argtypes = [C.c_void_p, d]
        L.or_fmm_cells.argtypes = [C.c_void_p, pi64]
        L.or_fmm_p2p_list.argtypes = [C.c_void_p, pi64]
        L.or_fmm_m2l_list.argtypes = [C.c_void_p, pi64]
        L.or_fmm_multipoles.argtypes = [C.c_void_p, d]
        L.or_fmm_locals.argtypes = [C.c_void_p, d]
        L.or_fmm_results.argtypes = [C.c_void_p, d, d, d, d]
        L.or_fmm_coverage.argtypes = [C.c_void_p, pi64]
        L.or_fmm_near_subset.restype = i64
        L.or_fmm_near_subset.argtypes = [C.c_void_p, i64, pi64, pi64, d, d, pi64]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    os.environ["OMP_NUM_THREADS"] = str(int(n))


# ---------------------------------------------------------------- Eq. 1-3 ---
def cutoff_g(rho: float) -> float:
    """Eq. 2."""
    return float(lib().or_cutoff_g(float(rho)))


def direct(xt, at, xs, as_, sig, box_len: float = 2 * np.pi, images: int = 0):
    """c-1 direct sum of Eq. 1 and Eq. 3 over (3^k)^3 image boxes (k = images).

    Returns (u, s), each float64 [nt, 3]."""
    xt, at, xs, as_, sig = map(_c64, (xt, at, xs, as_, sig))
    nt, ns = xt.shape[0], xs.shape[0]
    u = np.zeros((nt, 3))
    s = np.zeros((nt, 3))
    lib().or_direct(nt, _dp(xt), _dp(at), ns, _dp(xs), _dp(as_), _dp(sig), float(box_len), int(images), _dp(u), _dp(s))
    return u, s


# ------------------------------------------------------------ harmonics -----
def ncoef(P: int) -> int:
    return P * (P + 1) // 2


def regular(x, P):
    out = np.zeros(2 * ncoef(P))
    lib().or_regular(float(x[0]), float(x[1]), float(x[2]), int(P), _dp(out))
    return out.view(np.complex128)


def irregular(x, P):
    out = np.zeros(2 * ncoef(P))
    lib().or_irregular(float(x[0]), float(x[1]), float(x[2]), int(P), _dp(out))
    return out.view(np.complex128)


def p2m(P, x, q, c):
    x = _c64(x); q = _c64(q); c = _c64(c)
    M = np.zeros(2 * ncoef(P))
    lib().or_p2m(int(P), x.shape[0], _dp(x), _dp(q), _dp(c), _dp(M))
    return M.view(np.complex128)


def _op(fn, P, C_in, vec, nout):
    C_in = np.ascontiguousarray(C_in, dtype=np.complex128).view(np.float64)
    vec = _c64(vec)
    out = np.zeros(2 * nout)
    fn(int(P), _dp(C_in), _dp(vec), _dp(out))
    return out.view(np.complex128)


def m2m(P, Mc, d):
    return _op(lib().or_m2m, P, Mc, d, ncoef(P))


def m2l(P, M, D):
    return _op(lib().or_m2l, P, M, D, ncoef(P))


def l2l(P, Lp, d):
    return _op(lib().or_l2l, P, Lp, d, ncoef(P))


def l2p_derivs(P, L, d):
    L = np.ascontiguousarray(L, dtype=np.complex128).view(np.float64)
    d = _c64(d)
    phi = np.zeros(1); g = np.zeros(3); h = np.zeros(6)
    lib().or_l2p_derivs(int(P), _dp(L), _dp(d), _dp(phi), _dp(g), _dp(h))
    return phi[0], g, h


def m2p(P, M, D):
    M = np.ascontiguousarray(M, dtype=np.complex128).view(np.float64)
    return float(lib().or_m2p(int(P), _dp(M), _dp(_c64(D))))


# ------------------------------------------------------------------ FMM -----
class _Cfg(C.Structure):
    _fields_ = [("order", C.c_int), ("theta_num", C.c_int), ("theta_den", C.c_int),
                ("ncrit", C.c_int), ("images", C.c_int),
                ("box_lo", C.c_double * 3), ("box_len", C.c_double), ("traversal", C.c_int)]


class OracleFMM:
    """c-2: the double-precision CPU FMM, one object per particle set."""

    def __init__(self, x, alpha, sigma, order=10, theta=(1, 2), ncrit=64, images=3,
                 box_lo=(-np.pi,) * 3, box_len=2 * np.pi, traversal=0):
        self.x = _c64(x).reshape(-1, 3)
        self.alpha = _c64(alpha).reshape(-1, 3)
        self.sigma = _c64(sigma).reshape(-1)
        self.n = self.x.shape[0]
        cfg = _Cfg(int(order), int(theta[0]), int(theta[1]), int(ncrit), int(images),
                   (C.c_double * 3)(*box_lo), float(box_len), int(traversal))
        self.order = int(order)
        self._h = lib().or_fmm_new(self.n, _dp(self.x), _dp(self.alpha), _dp(self.sigma), C.byref(cfg))
        self._traversed = False
        self._evaluated = False

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_fmm_free(h)
            self._h = None

    # tree ------------------------------------------------------------------
    def box(self):
        lo = np.zeros(3); L = np.zeros(1)
        lib().or_fmm_box(self._h, _dp(lo), _dp(L))
        return lo, float(L[0])

    def keys(self):
        k = np.zeros(self.n, dtype=np.uint64); p = np.zeros(self.n, dtype=np.int64)
        lib().or_fmm_keys(self._h, k.ctypes.data_as(C.POINTER(C.c_uint64)), p.ctypes.data_as(C.POINTER(C.c_int64)))
        return k, p

    def positions(self):
        x = np.zeros((self.n, 3))
        lib().or_fmm_positions(self._h, _dp(x))
        return x

    def cells(self):
        nc = lib().or_fmm_ncells(self._h)
        out = np.zeros((nc, 10), dtype=np.int64)
        lib().or_fmm_cells(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    # traversal -------------------------------------------------------------
    def traverse(self):
        if not self._traversed:
            lib().or_fmm_traverse(self._h)
            self._traversed = True

    def p2p_list(self):
        self.traverse()
        n = lib().or_fmm_np2p(self._h)
        out = np.zeros((n, 3), dtype=np.int64)
        lib().or_fmm_p2p_list(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def m2l_list(self):
        self.traverse()
        n = lib().or_fmm_nm2l(self._h)
        out = np.zeros((n, 3), dtype=np.int64)
        lib().or_fmm_m2l_list(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def coverage(self):
        self.traverse()
        out = np.zeros(self.n, dtype=np.int64)
        lib().or_fmm_coverage(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    # evaluation ------------------------------------------------------------
    def evaluate(self):
        if not self._evaluated:
            self.traverse()
            lib().or_fmm_evaluate(self._h)
            self._evaluated = True
        un = np.zeros((self.n, 3)); sn = np.zeros((self.n, 3))
        uf = np.zeros((self.n, 3)); sf = np.zeros((self.n, 3))
        lib().or_fmm_results(self._h, _dp(un), _dp(sn), _dp(uf), _dp(sf))
        return {"u_near": un, "s_near": sn, "u_far": uf, "s_far": sf,
                "u": un + uf, "s": sn + sf}

    def near_subset(self, leaves):
        """Near field of the selected target leaves only (sizes where the full
        evaluation is too slow): returns (caller indices, u_near, s_near, number
        of P2P entries of those leaves); particles leaf by leaf in sorted order."""
        leaves = np.ascontiguousarray(leaves, dtype=np.int64)
        cells = self.cells() if not hasattr(self, "_cells") else self._cells
        self._cells = cells
        m = int(cells[leaves, 5].sum()) if len(leaves) else 0
        pidx = np.zeros(max(m, 1), dtype=np.int64)
        u = np.zeros((max(m, 1), 3)); s = np.zeros((max(m, 1), 3))
        ne = C.c_int64(0)
        got = lib().or_fmm_near_subset(self._h, len(leaves), leaves.ctypes.data_as(C.POINTER(C.c_int64)),
                                       pidx.ctypes.data_as(C.POINTER(C.c_int64)), _dp(u), _dp(s), C.byref(ne))
        if got < 0:
            raise ValueError("near_subset: a selected cell is not a leaf")
        return pidx[:m], u[:m], s[:m], int(ne.value)

    def multipoles(self):
        """Normalised M~ [ncells, 3, P(P+1)/2] complex (reading Z18)."""
        self.evaluate()
        nc = lib().or_fmm_ncells(self._h)
        out = np.zeros(nc * 3 * ncoef(self.order) * 2)
        lib().or_fmm_multipoles(self._h, _dp(out))
        return out.view(np.complex128).reshape(nc, 3, ncoef(self.order))

    def locals(self):
        self.evaluate()
        nc = lib().or_fmm_ncells(self._h)
        out = np.zeros(nc * 3 * ncoef(self.order) * 2)
        lib().or_fmm_locals(self._h, _dp(out))
        return out.view(np.complex128).reshape(nc, 3, ncoef(self.order))


def rel_l2(a, b) -> float:
    """Relative L2 error ||a - b|| / ||b|| over all entries."""
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))


# ------------------------------------------------------- NEXT-1 time step --
def rk2_step(x, alpha, sigma, dt, nu=0.0, images=0, box_len=2 * np.pi):
    """Midpoint RK2 of P:69 / Eq. 4 with the c-1 direct sum as the right-hand
    side: x' = x + dt u(t+dt/2), alpha' = alpha + dt dalpha/dt(t+dt/2),
    sigma'^2 = sigma^2 + 2 nu dt.  Returns float64 arrays."""
    x = _c64(x); alpha = _c64(alpha); sigma = _c64(sigma)
    u1, s1 = direct(x, alpha, x, alpha, sigma, box_len, images)
    xh = x + 0.5 * dt * u1
    ah = alpha + 0.5 * dt * s1
    sh = np.sqrt(sigma ** 2 + nu * dt)
    u2, s2 = direct(xh, ah, xh, ah, sh, box_len, images)
    return x + dt * u2, alpha + dt * s2, np.sqrt(sigma ** 2 + 2 * nu * dt)


# --------------------------------------------------------------------------
# NEXT-4: RBF reinitialisation -- plain numpy, double precision.
# zeta is the Gaussian core whose radial mass is g(rho) of Eq. 2;
# b_i = sum_j alpha_j zeta_{sigma_j}(y_i - x_j) is the old field's vorticity at
# the sites, and beta solves the collocation system sum_k beta_k
# zeta_{sigma0}(y_i - y_k) = b_i (Gaussian basis = the RBF).  The oracle forms
# the dense matrix and solves it exactly (LAPACK); sums run over the first
# image layer (27 boxes) when periodic, as the GPU's P2P lists do (reading R1).
# Pinned by tests/test_oracle_rbf.py.
# --------------------------------------------------------------------------
def zeta(r2, s):
    """(2 pi s^2)^{-3/2} exp(-r^2 / (2 s^2)) -- the vorticity of a unit blob."""
    s = np.asarray(s, dtype=np.float64)
    return np.exp(-np.asarray(r2, dtype=np.float64) / (2.0 * s * s)) / (2.0 * np.pi * s * s) ** 1.5


def _shifts(images, box_len):
    if images == 0:
        return np.zeros((1, 3))
    g = np.arange(-1, 2) * box_len
    return np.array([[a, b, c] for c in g for b in g for a in g], dtype=np.float64)


def gauss_field(y, x, alpha, sigma, box_len=2 * np.pi, images=1):
    """b[i] = sum over the image shifts and j of alpha_j zeta_{sigma_j}(y_i - x_j - shift)."""
    y = np.asarray(y, np.float64)
    x = np.asarray(x, np.float64)
    alpha = np.asarray(alpha, np.float64)
    sigma = np.asarray(sigma, np.float64)
    out = np.zeros((len(y), 3))
    for sh in _shifts(images, box_len):
        d = y[:, None, :] - x[None, :, :] - sh
        out += zeta((d * d).sum(-1), sigma[None, :]) @ alpha
    return out


def rbf_reinit(x, alpha, sigma, y, sigma0, box_len=2 * np.pi, images=1):
    """beta[m][3] solving sum_k beta_k zeta_{sigma0}(y_i - y_k) = b_i exactly."""
    y = np.asarray(y, np.float64)
    b = gauss_field(y, x, alpha, sigma, box_len, images)
    A = np.zeros((len(y), len(y)))
    for sh in _shifts(images, box_len):
        d = y[:, None, :] - y[None, :, :] - sh
        A += zeta((d * d).sum(-1), sigma0)
    return np.linalg.solve(A, b)
