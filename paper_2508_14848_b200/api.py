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


def owned_tiles(n_tiles, P, p, owner=None):
    """global tile indices of one dimension held by process row/column p, increasing:
    block-cyclic (t mod P == p) or owner[t] == p (gemm_mp_balance, NEXT-3)"""
    return [t for t in range(n_tiles) if (t % P if owner is None else int(owner[t])) == p]


def local_tiles(M, N, K, nb, P, Q, p, q, row_owner=None, col_owner=None):
    """(row tiles, column tiles) of this rank's local A, B and C (gemm_mp.h layout)"""
    mt, nt, kt = M // nb, N // nb, K // nb
    rows = owned_tiles(mt, P, p, row_owner)
    cols = owned_tiles(nt, Q, q, col_owner)
    return dict(A=(rows, owned_tiles(kt, Q, q)), B=(owned_tiles(kt, P, p), cols), C=(rows, cols))


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

    def execute(self, C, stream=None):
        """C <- alpha A B + beta C_in on `stream` (default: the plan's).  A repeated execute
        with the same C and workspace issues kernels only, so it can be captured into a
        CUDA graph (torch.cuda.graph) after one warm-up execute."""
        B.gemm_mp_execute(self.plan, C, C.stride(0), stream or self.stream)

    def maps(self):
        return B.gemm_mp_get_maps(self.plan, self.mt, self.nt, self.kt)

    def stats(self):
        return B.gemm_mp_get_stats(self.plan)

    def tile_stats(self, which):
        """global per-tile (S, maxabs, finite) grids of 'A', 'B' or 'C' (S1 debug export)"""
        rows, cols = {"A": (self.mt, self.kt), "B": (self.kt, self.nt), "C": (self.mt, self.nt)}[which]
        return B.gemm_mp_get_tile_stats(self.plan, which, rows, cols)

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


def synth_tiles(rows, cols, nb, recipe, row_tiles, col_tiles, device="cuda", stream=None):
    """Local part of a synthetic matrix holding the given global tiles (any ownership)."""
    lr, lc = len(row_tiles) * nb, len(col_tiles) * nb
    out = torch.empty((max(lr, 1), max(lc, 2)), dtype=torch.float64, device=device)[:lr, :lc] \
        if lr * lc == 0 else torch.empty((lr, lc), dtype=torch.float64, device=device)
    if lr * lc:
        B.gemm_mp_synth_tiles(out, out.stride(0), rows, cols, nb, row_tiles, col_tiles, recipe.seed,
                              recipe.tau, MODE[recipe.mode], recipe.E, recipe.s,
                              stream or torch.cuda.current_stream(device))
    return out


def synth_operands(w, P=1, Q=1, p=0, q=0, row_owner=None, col_owner=None, device="cuda", stream=None):
    """This rank's local A, B (and C if beta != 0) of a gmp_inputs workload, in the
    gemm_mp.h layout for the given ownership (block-cyclic when the owners are None)."""
    lt = local_tiles(w.M, w.N, w.K, w.nb, P, Q, p, q, row_owner, col_owner)
    A = synth_tiles(w.M, w.K, w.nb, w.a, *lt["A"], device=device, stream=stream)
    Bm = synth_tiles(w.K, w.N, w.nb, w.b, *lt["B"], device=device, stream=stream)
    C = synth_tiles(w.M, w.N, w.nb, w.c, *lt["C"], device=device, stream=stream) if w.beta != 0 else None
    return A, Bm, C


def local_c_shape(w, P=1, Q=1, p=0, q=0, row_owner=None, col_owner=None):
    rows, cols = local_tiles(w.M, w.N, w.K, w.nb, P, Q, p, q, row_owner, col_owner)["C"]
    return len(rows) * w.nb, len(cols) * w.nb


def place_local_c(full, loc, w, P, Q, p, q, row_owner=None, col_owner=None):
    """writes rank (p, q)'s local C (numpy) into the global numpy matrix `full`"""
    import numpy as np
    nb = w.nb
    rows, cols = local_tiles(w.M, w.N, w.K, nb, P, Q, p, q, row_owner, col_owner)["C"]
    rr = (np.asarray(rows, np.int64)[:, None] * nb + np.arange(nb)[None, :]).ravel()
    cc = (np.asarray(cols, np.int64)[:, None] * nb + np.arange(nb)[None, :]).ravel()
    full[np.ix_(rr, cc)] = loc
    return rr, cc


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


class HostPipeline:
    """A stream of GEMMs whose operands and results live in (pinned) HOST memory.

    Each step k copies its A, B (C) to the device, runs plan -> convert ->
    execute, and copies its C back.  Device operand and result buffers are
    `nbuf`-fold buffered (3 by default), and the copies run on their own streams,
    so the H2D of the next steps and the D2H of the previous ones overlap the
    compute of step k (PCIe is full duplex).  Only copies and stream/event ordering happen here; every step of
    the method runs in the library's kernels.

    `desc` fixes the shape (every step reuses it); `comm` is the NCCL
    communicator for P*Q > 1.  Host tensors must be pinned for the copies to be
    asynchronous."""

    def __init__(self, desc, local_a, local_b, local_c, local_out, device, comm=None, nbuf=3):
        self.desc, self.device, self.comm = desc, device, comm
        self.compute = torch.cuda.current_stream(device)
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        # nbuf device copies of the operands and results: the H2D of step k+nbuf-1
        # only waits for step k-1's convert, so copies run nbuf-1 steps ahead
        self.nbuf = nbuf
        mk = lambda shp: [torch.empty(shp, dtype=torch.float64, device=device) for _ in range(nbuf)]  # noqa: E731
        self.dA, self.dB = mk(local_a), mk(local_b)
        self.dC = mk(local_c) if desc.beta != 0.0 else [None] * nbuf
        self.dOut = mk(local_out)
        self.nscr = B.gemm_mp_scratch_size(desc)
        self.scratch = torch.empty(self.nscr, dtype=torch.uint8, device=device)
        self.ws, self.ws_bytes = None, 0
        self.plans = []

    def _ensure_ws(self, nbytes):
        if nbytes > self.ws_bytes:
            raw = torch.empty(nbytes + 1024, dtype=torch.uint8, device=self.device)
            off = (-raw.data_ptr()) % 1024
            self._ws_raw, self.ws, self.ws_bytes = raw, raw[off:off + nbytes], nbytes

    def reserve(self, hA, hB, hC=None):
        """Size the workspace outside any timed region (one plan on the first inputs)."""
        self.dA[0].copy_(hA)
        self.dB[0].copy_(hB)
        if hC is not None:
            self.dC[0].copy_(hC)
        pl = B.gemm_mp_plan(self.desc, self.dA[0], self.dA[0].stride(0), self.dB[0], self.dB[0].stride(0),
                            self.dC[0], self.dC[0].stride(0) if self.dC[0] is not None else 0,
                            self.scratch, self.nscr, self.comm, self.compute)
        self._ensure_ws(B.gemm_mp_workspace_size(pl))
        B.gemm_mp_destroy(pl)
        torch.cuda.synchronize(self.device)

    def run(self, hA, hB, hC, hOut):
        """Process len(hA) steps: hOut[k] <- alpha hA[k] hB[k] + beta hC[k] (host tensors)."""
        K = len(hA)
        timed = getattr(self, "record_timeline", False)   # dev aid: keep timing events of the last run
        h2d_done = [torch.cuda.Event(enable_timing=timed) for _ in range(K)]
        convert_done = [torch.cuda.Event(enable_timing=timed) for _ in range(K)]
        exec_done = [torch.cuda.Event(enable_timing=timed) for _ in range(K)]
        d2h_done = [torch.cuda.Event(enable_timing=timed) for _ in range(K)]
        if timed:
            self.timeline = (h2d_done, convert_done, exec_done, d2h_done)

        nbuf = self.nbuf

        def enqueue_h2d(k):
            b = k % nbuf
            with torch.cuda.stream(self.h2d):
                if k >= nbuf:
                    self.h2d.wait_event(convert_done[k - nbuf])   # buffers b free once step k-nbuf is packed
                self.dA[b].copy_(hA[k], non_blocking=True)
                self.dB[b].copy_(hB[k], non_blocking=True)
                if self.dC[b] is not None:
                    self.dC[b].copy_(hC[k], non_blocking=True)
                h2d_done[k].record(self.h2d)

        for k in range(min(nbuf - 1, K)):
            enqueue_h2d(k)
        for k in range(K):
            b = k % nbuf
            if k + nbuf - 1 < K:
                enqueue_h2d(k + nbuf - 1)                       # before plan's host sync
            self.compute.wait_event(h2d_done[k])
            dC = self.dC[b]
            pl = B.gemm_mp_plan(self.desc, self.dA[b], self.dA[b].stride(0), self.dB[b], self.dB[b].stride(0),
                                dC, dC.stride(0) if dC is not None else 0, self.scratch, self.nscr, self.comm,
                                self.compute)
            self.plans.append(pl)
            nws = B.gemm_mp_workspace_size(pl)
            if nws > self.ws_bytes:
                # another input's maps need more slots: grow (torch's allocator frees the
                # old block in stream order, and every use of it is on this stream)
                with torch.cuda.stream(self.compute):
                    self._ensure_ws(nws)
            B.gemm_mp_convert(pl, self.ws, nws, self.compute)
            convert_done[k].record(self.compute)
            # result buffer b is free once step k-nbuf was read back: only the C-finalize waits
            # for that copy, the tile-GEMMs overlap it
            B.gemm_mp_execute_after(pl, self.dOut[b], self.dOut[b].stride(0), self.compute,
                                    d2h_done[k - nbuf] if k >= nbuf else None)
            exec_done[k].record(self.compute)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(exec_done[k])
                hOut[k].copy_(self.dOut[b], non_blocking=True)
                d2h_done[k].record(self.d2h)
        self.compute.wait_event(d2h_done[K - 1])
        self.compute.wait_stream(self.h2d)

    def close(self):
        torch.cuda.synchronize(self.device)
        for pl in self.plans:
            B.gemm_mp_destroy(pl)
        self.plans = []
