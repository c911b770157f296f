"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI."""
import numpy as np


def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return torch


class GpuRun:
    """One context + one particle set; every call goes through include/fmm.h."""

    def __init__(self, x, a, s, **cfg):
        import paper_1106_5273_b200 as P
        self.P = P
        torch = torch_cuda()
        self.torch = torch
        self.order = cfg.get("order", 10)
        self.fmm = P.FMM(**cfg)
        self.n = len(x)
        self.x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
        self.a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
        self.s = torch.from_numpy(np.ascontiguousarray(s, dtype=np.float32)).cuda()
        self.fmm.set_particles(self.x, self.a, self.s)

    def evaluate(self, parts=3):
        torch = self.torch
        u = torch.empty((self.n, 3), dtype=torch.float32, device="cuda")
        st = torch.empty((self.n, 3), dtype=torch.float32, device="cuda")
        self.fmm.evaluate(u, st, parts)
        return u.cpu().numpy().astype(np.float64), st.cpu().numpy().astype(np.float64)

    def keys(self):
        return self.P.fmm_get_keys(self.fmm.ctx, self.n)

    def cells(self):
        return self.P.fmm_get_cells(self.fmm.ctx)

    def lists(self):
        return self.P.fmm_get_lists(self.fmm.ctx)

    def box(self):
        return self.P.fmm_get_box(self.fmm.ctx)

    def expansions(self):
        return self.P.fmm_get_expansions(self.fmm.ctx, self.order)

    def stats(self):
        return self.fmm.stats()

    def close(self):
        self.fmm.close()
