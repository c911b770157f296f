"""Thin ctypes binding of include/fmm.h -- argument marshalling only.

Every step of the evaluation runs in libfmm_b200.so's CUDA kernels; this module
never computes anything.  If the library is missing it raises (there is no CPU
fallback).  Arrays may be torch tensors (CUDA or CPU) or numpy arrays; they are
passed as raw pointers, float32, contiguous, shape [n, 3] / [n].
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FMM_LIB") or os.path.join(_HERE, "libfmm_b200.so")   # FMM_LIB: development variants (tools/build_variant.py)

(FMM_OK, FMM_E_ARG, FMM_E_NONFINITE, FMM_E_SIGMA, FMM_E_STATE, FMM_E_OOM, FMM_E_CUDA, FMM_E_NCCL, FMM_E_INTERNAL,
 FMM_E_NOCONV) = range(10)
STATUS_NAMES = ["FMM_OK", "FMM_E_ARG", "FMM_E_NONFINITE", "FMM_E_SIGMA", "FMM_E_STATE", "FMM_E_OOM",
                "FMM_E_CUDA", "FMM_E_NCCL", "FMM_E_INTERNAL", "FMM_E_NOCONV"]


class fmm_config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("order", C.c_int32), ("theta_num", C.c_int32),
                ("theta_den", C.c_int32), ("ncrit", C.c_int32), ("images", C.c_int32),
                ("box_lo", C.c_double * 3), ("box_len", C.c_double), ("traversal", C.c_int32),
                ("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_id", C.c_void_p), ("tiles", C.c_int32 * 3), ("m2l_path", C.c_int32),
                ("partition", C.c_int32)]


class fmm_stats(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("n", C.c_int64), ("ncells", C.c_int64), ("nleaves", C.c_int64),
                ("nlevels", C.c_int64), ("p2p_list", C.c_int64), ("m2l_list", C.c_int64),
                ("p2p_pairs", C.c_int64), ("far_m2l", C.c_int64), ("model_flops", C.c_double),
                ("launches", C.c_int64), ("cub_calls", C.c_int64), ("p2p_near_pairs", C.c_int64),
                ("ms_keys", C.c_double), ("ms_sort", C.c_double), ("ms_tree", C.c_double),
                ("ms_upward", C.c_double), ("ms_traverse", C.c_double), ("ms_m2l", C.c_double),
                ("ms_p2p", C.c_double), ("ms_downward", C.c_double), ("ms_finalize", C.c_double),
                ("ms_set_total", C.c_double), ("ms_eval_total", C.c_double),
                ("ntot", C.c_int64), ("let_bytes_sent", C.c_int64), ("let_bytes_recv", C.c_int64),
                ("let_cells", C.c_int64), ("let_leaves", C.c_int64), ("ms_let", C.c_double),
                ("m2l_tc_list", C.c_int64), ("own_begin", C.c_int64), ("own_count", C.c_int64),
                ("redist_bytes", C.c_int64), ("m2l_reg_list", C.c_int64), ("ms_m2l_tc", C.c_double),
                ("ms_m2l_reg", C.c_double), ("ms_let_exposed", C.c_double), ("let_fallback", C.c_int64),
                ("nranks", C.c_int64), ("ncells_local", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "struct_size"}


class FMMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status, msg))
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libfmm_b200.so not built (run __graft_entry__.build()); no CPU fallback exists")
        L = C.CDLL(LIB_PATH)
        vp, i64, pi64 = C.c_void_p, C.c_int64, C.POINTER(C.c_int64)
        L.fmm_config_default.restype = None
        L.fmm_config_default.argtypes = [C.POINTER(fmm_config)]
        L.fmm_create.argtypes = [C.POINTER(fmm_config), C.POINTER(vp)]
        L.fmm_set_particles.argtypes = [vp, i64, vp, vp, vp]
        L.fmm_evaluate.argtypes = [vp, vp, vp]
        L.fmm_evaluate_parts.argtypes = [vp, C.c_int32, vp, vp]
        L.fmm_destroy.argtypes = [vp]
        L.fmm_last_error.restype = C.c_char_p
        L.fmm_last_error.argtypes = [vp]
        L.fmm_get_stats.argtypes = [vp, C.POINTER(fmm_stats)]
        L.fmm_get_sizes.argtypes = [vp, pi64, pi64, pi64]
        L.fmm_get_box.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fmm_get_keys.argtypes = [vp, vp, vp]
        L.fmm_get_cells.argtypes = [vp, vp]
        L.fmm_get_lists.argtypes = [vp, vp, vp]
        L.fmm_get_expansions.argtypes = [vp, vp, vp]
        L.fmm_eval_cutoff.argtypes = [vp, i64, vp, vp]
        L.fmm_eval_pair_kernel.argtypes = [vp, i64, vp, C.c_int32, vp, vp]
        L.fmm_comm_unique_id.argtypes = [vp]
        L.fmm_debug_mode.argtypes = []
        L.fmm_debug_mode.restype = C.c_int32
        L.fmm_step.argtypes = [vp, i64, vp, vp, vp, C.c_double, C.c_double]
        L.fmm_evaluate_targets.argtypes = [vp, i64, vp, vp, vp, i64, vp, vp]
        L.fmm_rbf_reinit.argtypes = [vp, i64, vp, vp, vp, i64, vp, C.c_float, C.c_double, C.c_int32, vp,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        for nm in ("fmm_create", "fmm_set_particles", "fmm_evaluate", "fmm_evaluate_parts", "fmm_destroy",
                   "fmm_get_stats", "fmm_get_sizes", "fmm_get_box", "fmm_get_keys", "fmm_get_cells",
                   "fmm_get_lists", "fmm_get_expansions", "fmm_eval_cutoff", "fmm_eval_pair_kernel",
                   "fmm_comm_unique_id", "fmm_step",
                   "fmm_evaluate_targets", "fmm_rbf_reinit"):
            getattr(L, nm).restype = C.c_int
        _lib = L
    return _lib


def _ptr(a, numel=None, device=None):
    """Raw pointer of a float32 array; numel: required element count; device:
    the context's CUDA ordinal (a CUDA tensor on another GPU is rejected)."""
    if a is None:
        if numel:
            raise ValueError("array required")
        return None
    if numel is not None and int(np.prod(a.shape)) != int(numel):
        raise ValueError("array has %d elements, expected %d" % (int(np.prod(a.shape)), int(numel)))
    if hasattr(a, "data_ptr"):          # torch tensor
        if str(a.dtype) != "torch.float32":
            raise TypeError("float32 tensor required")
        if not a.is_contiguous():
            raise ValueError("contiguous tensor required")
        if device is not None and a.is_cuda and a.device.index != int(device):
            raise ValueError("tensor on cuda:%d, context on cuda:%d" % (a.device.index, int(device)))
        return C.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
            raise TypeError("contiguous float32 array required")
        return C.c_void_p(a.ctypes.data)
    raise TypeError("unsupported array type %r" % type(a))


def _check(ctx, st):
    if st != FMM_OK:
        msg = lib().fmm_last_error(ctx).decode() if ctx else ""
        raise FMMError(st, msg)


# ---- same names as the C ABI --------------------------------------------
def fmm_config_default(**kw) -> fmm_config:
    cfg = fmm_config()
    lib().fmm_config_default(C.byref(cfg))
    for k, v in kw.items():
        if k == "box_lo":
            cfg.box_lo = (C.c_double * 3)(*v)
        elif k == "tiles":
            cfg.tiles = (C.c_int32 * 3)(*v)
        elif k == "theta":
            cfg.theta_num, cfg.theta_den = int(v[0]), int(v[1])
        else:
            setattr(cfg, k, v)
    return cfg


def fmm_create(cfg: fmm_config):
    h = C.c_void_p()
    st = lib().fmm_create(C.byref(cfg), C.byref(h))
    if st != FMM_OK:
        raise FMMError(st, "fmm_create failed")
    return h


def fmm_set_particles(ctx, n, x, alpha, sigma, device=None):
    n = int(n)
    _check(ctx, lib().fmm_set_particles(ctx, n, _ptr(x, 3 * n, device), _ptr(alpha, 3 * n, device),
                                        _ptr(sigma, n, device)))


def fmm_evaluate(ctx, u, dalpha_dt, n=None, device=None):
    m = None if n is None else 3 * int(n)
    _check(ctx, lib().fmm_evaluate(ctx, _ptr(u, m, device), _ptr(dalpha_dt, m, device)))


def fmm_evaluate_parts(ctx, parts, u, dalpha_dt, n=None, device=None):
    m = None if n is None else 3 * int(n)
    _check(ctx, lib().fmm_evaluate_parts(ctx, int(parts), _ptr(u, m, device), _ptr(dalpha_dt, m, device)))


def fmm_destroy(ctx):
    lib().fmm_destroy(ctx)


def fmm_last_error(ctx) -> str:
    return lib().fmm_last_error(ctx).decode()


def fmm_get_stats(ctx) -> dict:
    s = fmm_stats()
    _check(ctx, lib().fmm_get_stats(ctx, C.byref(s)))
    return s.as_dict()


def fmm_get_sizes(ctx):
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    _check(ctx, lib().fmm_get_sizes(ctx, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def fmm_get_box(ctx):
    lo = (C.c_double * 3)()
    L = C.c_double()
    _check(ctx, lib().fmm_get_box(ctx, lo, C.byref(L)))
    return np.array(lo[:]), L.value


def fmm_get_keys(ctx, n):
    keys = np.zeros(n, dtype=np.uint64)
    perm = np.zeros(n, dtype=np.int64)
    _check(ctx, lib().fmm_get_keys(ctx, C.c_void_p(keys.ctypes.data), C.c_void_p(perm.ctypes.data)))
    return keys, perm


def fmm_get_cells(ctx):
    nc, _, _ = fmm_get_sizes(ctx)
    out = np.zeros((nc, 10), dtype=np.int64)
    _check(ctx, lib().fmm_get_cells(ctx, C.c_void_p(out.ctypes.data)))
    return out


def fmm_get_lists(ctx):
    _, np2p, nm2l = fmm_get_sizes(ctx)
    p2p = np.zeros((np2p, 3), dtype=np.int64)
    m2l = np.zeros((nm2l, 3), dtype=np.int64)
    _check(ctx, lib().fmm_get_lists(ctx, C.c_void_p(p2p.ctypes.data), C.c_void_p(m2l.ctypes.data)))
    return p2p, m2l


def fmm_get_expansions(ctx, order):
    nc, _, _ = fmm_get_sizes(ctx)
    k = order * (order + 1) // 2
    M = np.zeros((nc, 3, k, 2), dtype=np.float32)
    L = np.zeros((nc, 3, k, 2), dtype=np.float32)
    _check(ctx, lib().fmm_get_expansions(ctx, C.c_void_p(M.ctypes.data), C.c_void_p(L.ctypes.data)))
    return (M[..., 0] + 1j * M[..., 1]).astype(np.complex128), (L[..., 0] + 1j * L[..., 1]).astype(np.complex128)


def fmm_step(ctx, n, x, alpha, sigma, dt, nu, device=None):
    n = int(n)
    _check(ctx, lib().fmm_step(ctx, n, _ptr(x, 3 * n, device), _ptr(alpha, 3 * n, device), _ptr(sigma, n, device),
                               float(dt), float(nu)))


def fmm_evaluate_targets(ctx, n, x, alpha, sigma, nt, y, u, device=None):
    n, nt = int(n), int(nt)
    _check(ctx, lib().fmm_evaluate_targets(ctx, n, _ptr(x, 3 * n, device), _ptr(alpha, 3 * n, device),
                                           _ptr(sigma, n, device), nt, _ptr(y, 3 * nt, device),
                                           _ptr(u, 3 * nt, device)))


def fmm_rbf_reinit(ctx, n, x, alpha, sigma, m, y, sigma0, tol, maxit, beta):
    """NEXT-4: returns (iterations, relative residual); FMMError(FMM_E_NOCONV) if maxit is reached."""
    it, res = C.c_int32(0), C.c_double(0.0)
    n, m = int(n), int(m)
    st = lib().fmm_rbf_reinit(ctx, n, _ptr(x, 3 * n), _ptr(alpha, 3 * n), _ptr(sigma, n), m, _ptr(y, 3 * m),
                              float(sigma0), float(tol), int(maxit), _ptr(beta, 3 * m), C.byref(it), C.byref(res))
    if st == FMM_E_NOCONV:
        raise FMMError(st, "%d iterations, relative residual %.3e > tol %.1e" % (it.value, res.value, tol))
    _check(ctx, st)
    return it.value, res.value


def fmm_comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().fmm_comm_unique_id(buf)
    if st != FMM_OK:
        raise FMMError(st, "ncclGetUniqueId failed")
    return buf.raw


def fmm_eval_cutoff(ctx, rho, g):
    n = int(rho.shape[0])
    _check(ctx, lib().fmm_eval_cutoff(ctx, n, _ptr(rho, n), _ptr(g, n)))


def fmm_eval_pair_kernel(ctx, rho, g, rho_gp, branch=0):
    """g(rho) and rho g'(rho) as the device P2P pair code evaluates them (reading Z6)."""
    n = int(rho.shape[0])
    _check(ctx, lib().fmm_eval_pair_kernel(ctx, n, _ptr(rho, n), int(branch), _ptr(g, n), _ptr(rho_gp, n)))


def fmm_debug_mode() -> int:
    """Debug modes of the loaded library (bit 0: FMM_POISON allocations and guard zones)."""
    return int(lib().fmm_debug_mode())


class FMM:
    """Owning wrapper: ``FMM(order=10, images=3, ...)``; ``set_particles(x, a, s)``;
    ``evaluate(u, s)`` writes into caller-provided float32 buffers (device or host)."""

    def __init__(self, nccl_id: bytes = None, **kw):
        self._id = None
        if nccl_id is not None:
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
            kw["nccl_id"] = C.cast(self._id, C.c_void_p)
        self.cfg = fmm_config_default(**kw)
        self.ctx = fmm_create(self.cfg)
        self.n = None          # particle count of the last set (None: nothing set yet)

    def set_particles(self, x, alpha, sigma):
        n = int(x.shape[0])
        fmm_set_particles(self.ctx, n, x, alpha, sigma, device=self.cfg.device)
        self.n = n

    def evaluate(self, u, dalpha_dt, parts=3):
        fmm_evaluate_parts(self.ctx, parts, u, dalpha_dt, n=self.n, device=self.cfg.device)

    def step(self, x, alpha, sigma, dt, nu=0.0):
        """One midpoint-RK2 vortex step (NEXT-1); overwrites x, alpha, sigma."""
        fmm_step(self.ctx, x.shape[0], x, alpha, sigma, dt, nu, device=self.cfg.device)
        self.n = int(x.shape[0])

    def evaluate_targets(self, x, alpha, sigma, y, u):
        """Velocity at strength-free targets y (NEXT-2); the context then holds the union."""
        fmm_evaluate_targets(self.ctx, x.shape[0], x, alpha, sigma, y.shape[0], y, u, device=self.cfg.device)
        self.n = int(x.shape[0] + y.shape[0])

    def rbf_reinit(self, x, alpha, sigma, y, sigma0, beta, tol=1e-6, maxit=200):
        """RBF reinitialisation onto the sites y (NEXT-4); writes beta, returns (iters, resid).
        The context then holds (y, beta, sigma0)."""
        r = fmm_rbf_reinit(self.ctx, x.shape[0], x, alpha, sigma, y.shape[0], y, sigma0, tol, maxit, beta)
        self.n = int(y.shape[0])
        return r

    def stats(self):
        return fmm_get_stats(self.ctx)

    def close(self):
        if self.ctx:
            fmm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
