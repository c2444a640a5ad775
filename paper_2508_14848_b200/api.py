"""Torch-facing convenience wrapper over the C ABI (memory + streams only).

GemmMP owns the torch buffers (scratch, workspace) that the C ABI leaves to the
caller and runs plan -> convert -> execute.  No arithmetic of the method is
done here."""
import math

import torch

from . import binding as B

MODE = {"uniform": 0, "graded": 1, "random": 2}


def default_grid(G):
    """P x Q as square as possible, P <= Q."""
    P = max(d for d in range(1, int(math.isqrt(G)) + 1) if G % d == 0)
    return P, G // P


def local_shape(rows, cols, nb, P, Q, p, q):
    def nloc(n, P_, p_):
        return (n - p_ + P_ - 1) // P_ if n > p_ else 0
    return nloc(rows // nb, P, p) * nb, nloc(cols // nb, Q, q) * nb


class GemmMP:
    """One planned GEMM on this rank's device."""

    def __init__(self, desc, A, B_, C=None, nccl_comm=None, stream=None, device=None):
        self.desc = desc
        self.device = device or A.device
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.mt, self.nt, self.kt = desc.M // desc.nb, desc.N // desc.nb, desc.K // desc.nb
        nscr = B.gemm_mp_scratch_size(desc)
        self.scratch = torch.empty(nscr, dtype=torch.uint8, device=self.device)
        ldc = C.stride(0) if C is not None else 0
        self.plan = B.gemm_mp_plan(desc, A, A.stride(0), B_, B_.stride(0), C, ldc, self.scratch, nscr,
                                   nccl_comm, self.stream)
        self.ws_bytes = B.gemm_mp_workspace_size(self.plan)
        # 1024-byte aligned workspace (TMA / 128B swizzle)
        self._ws = torch.empty(self.ws_bytes + 1024, dtype=torch.uint8, device=self.device)
        off = (-self._ws.data_ptr()) % 1024
        self.ws = self._ws[off:off + self.ws_bytes]

    def convert(self):
        B.gemm_mp_convert(self.plan, self.ws, self.ws_bytes, self.stream)

    def execute(self, C):
        B.gemm_mp_execute(self.plan, C, C.stride(0), self.stream)

    def maps(self):
        return B.gemm_mp_get_maps(self.plan, self.mt, self.nt, self.kt)

    def stats(self):
        return B.gemm_mp_get_stats(self.plan)

    def tile(self, which, ti, tj, cls):
        return B.gemm_mp_get_tile(self.plan, which, ti, tj, cls, self.desc.nb)

    def sync(self):
        B.gemm_mp_sync(self.plan)

    def close(self):
        if self.plan:
            B.gemm_mp_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def synth(rows, cols, nb, recipe, P=1, Q=1, p=0, q=0, device="cuda", stream=None):
    """Local block-cyclic part of a synthetic matrix, generated on the device (N1)."""
    lr, lc = local_shape(rows, cols, nb, P, Q, p, q)
    out = torch.empty((max(lr, 1), max(lc, 2)), dtype=torch.float64, device=device)[:lr, :lc] \
        if lr * lc == 0 else torch.empty((lr, lc), dtype=torch.float64, device=device)
    if lr * lc:
        B.gemm_mp_synth(out, out.stride(0), rows, cols, nb, P, Q, p, q, recipe.seed, recipe.tau,
                        MODE[recipe.mode], recipe.E, recipe.s,
                        stream or torch.cuda.current_stream(device))
    return out


def gemm_mp(A, B_, C=None, nb=128, tol=1e-6, alpha=1.0, beta=0.0, class_mask=0b01111, flags=0,
            a_map=None, b_map=None, c_map=None, out=None):
    """Single-GPU convenience: C_out = alpha A B + beta C (binary64 device tensors)."""
    M, K = A.shape
    N = B_.shape[1]
    desc = B.make_desc(M, N, K, nb, tol, alpha, beta, class_mask, flags, a_map=a_map, b_map=b_map,
                       c_map=c_map)
    g = GemmMP(desc, A, B_, C if beta != 0.0 else None)
    g.convert()
    out = torch.empty((M, N), dtype=torch.float64, device=A.device) if out is None else out
    g.execute(out)
    return out, g
