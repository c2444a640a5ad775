"""Multi-rank SUMMA path on ONE GPU (NEXT-2): the P x Q rank
plans of a grid run in one process, one host thread per rank, through the same
per-rank C-ABI calls as under torchrun; only the transport differs
(GMP_FLAG_LOOPBACK: the statistics all-reduce is a rank-order sum, each SUMMA
broadcast of a panel tile in stored precision -- PAPER.md:145-148, 2D
block-cyclic grid PAPER.md:179 -- is one device-to-device copy per receiver from
the root plan's payload slot, ordered by events).  Everything the receivers do
with the received tiles (receive slots, receiver-side shadows, FP32 splits,
step events, fold order) is the NCCL path's code.

Checks per grid (1x2, 2x2, 1x4, 4x1, 2x4; receiver- and sender-side; tile grids
that P and Q divide and ones they do not):
* every rank's maps and scales == the 1-GPU run's;
* the gathered C is BITWISE the 1-GPU C (fold order is G-independent, R15);
* received bytes per rank == the closed form of SURVEY 8(e) (receiver-side), never
  more than it (sender-side), strictly fewer in total on the FP8-enabled mix;
* on the SIMT kernels the gathered C is bitwise the ORACLE's C."""
import threading

import numpy as np
import pytest
import torch

import gmp_inputs
import oracle
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu

BYTES = [8, 4, 2, 2, 1, 1, 17 / 32]   # per element; MXFP4: E2M1 nibbles + one scale byte per 32


def closed_form_recv(acode, bcode, nb, P, Q, p, q, ro=None, co=None):
    """sum over owned tile rows i, l != q (Q) of bytes(A_il) + over owned tile
    columns j, l != p (P) of bytes(B_lj) -- every remote panel tile reaches each consumer
    rank once (owned = i mod P == p block-cyclic, or ro[i] == p under NEXT-3 ownership)"""
    mt, kt = acode.shape
    nt = bcode.shape[1]
    tot = 0
    for i in api.owned_tiles(mt, P, p, ro):
        for l in range(kt):
            if l % Q != q:
                tot += B.slot_bytes(int(acode[i, l]), nb)
    for j in api.owned_tiles(nt, Q, q, co):
        for l in range(kt):
            if l % P != p:
                tot += B.slot_bytes(int(bcode[l, j]), nb)
    return tot


def _workload(kind):
    if kind == "small":   # FP8-enabled random mix: 8 x 6 x 10 tiles of 256
        return gmp_inputs.small_workload(2048, 1536, 2560, 256, 1e-4, mode="random", E=32, beta=0.75, seed=5,
                                         class_mask=0b111111)
    if kind == "uneven":  # 5 x 3 x 7 tiles: no grid divides them
        return gmp_inputs.small_workload(1280, 768, 1792, 256, 1e-3, mode="graded", E=24, beta=-0.5, seed=6,
                                         class_mask=0b111111)
    if kind == "mx4":  # MXFP4 enabled: MXFP4 payloads (and sender-side MXFP4 shadows) on the wire
        return gmp_inputs.small_workload(1024, 768, 1280, 256, 1e-2, mode="random", E=40, beta=0.5, seed=53,
                                         class_mask=0b1111111)
    if kind == "tiny_nb128":  # 3 x 5 x 9 tiles of 128, beta = 0, FP32-heavy
        return gmp_inputs.small_workload(384, 640, 1152, 128, 1e-6, mode="random", E=20, beta=0.0, seed=7)
    raise ValueError(kind)


def run_single(w, flags=0):
    dev = torch.device("cuda:0")
    A = api.synth(w.M, w.K, w.nb, w.a, device=dev)
    Bm = api.synth(w.K, w.N, w.nb, w.b, device=dev)
    C = api.synth(w.M, w.N, w.nb, w.c, device=dev) if w.beta != 0 else None
    d1 = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags)
    g1 = api.GemmMP(d1, A, Bm, C, device=dev)
    g1.convert()
    full = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g1.execute(full)
    g1.sync()
    res = full.cpu().numpy(), g1.maps()
    g1.close()
    return res


def run_grid(w, P, Q, flags=0, executes=2, ro=None, co=None):
    """all P*Q ranks on cuda:0, one thread and one stream per rank; returns per-rank
    (p, q, local C, maps, stats); ro / co: tile-row / tile-column owners (NEXT-3)"""
    dev = torch.device("cuda:0")
    G = P * Q
    lb = B.gemm_mp_loopback_create(G)
    ranks = []
    for r in range(G):
        p, q = r // Q, r % Q
        A, Bm, C = api.synth_operands(w, P, Q, p, q, ro, co, device=dev)
        lr, lc = api.local_c_shape(w, P, Q, p, q, ro, co)
        out = torch.full((lr, lc), float("nan"), dtype=torch.float64, device=dev)
        ranks.append(dict(p=p, q=q, A=A, B=Bm, C=C, out=out, stream=torch.cuda.Stream(dev)))
    torch.cuda.synchronize()
    errs = [None] * G

    def body(r):
        d = ranks[r]
        try:
            torch.cuda.set_device(dev)
            desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask,
                               flags | B.GMP_FLAG_LOOPBACK, P, Q, r, row_owner=ro, col_owner=co)
            g = api.GemmMP(desc, d["A"], d["B"], d["C"], nccl_comm=lb, stream=d["stream"], device=dev)
            g.convert()
            for _ in range(executes):   # the second execute reuses the received panels
                g.execute(d["out"])
            d["g"] = g
        except Exception as e:   # surfaced in the main thread
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank thread hangs (loopback barrier)"
    for e in errs:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    res = []
    for d in ranks:
        g = d["g"]
        g.sync()
        res.append((d["p"], d["q"], d["out"].cpu().numpy(), g.maps(), g.stats()))
    for d in ranks:
        d["g"].close()
    B.gemm_mp_loopback_destroy(lb)
    return res


def gather(w, res, P, Q, ro=None, co=None):
    Cfull = np.full((w.M, w.N), np.nan)
    for (p, q, loc, _, _) in res:
        api.place_local_c(Cfull, loc, w, P, Q, p, q, ro, co)
    return Cfull


_single = {}


def single(kind, flags=0):
    key = (kind, flags)
    if key not in _single:
        _single[key] = run_single(_workload(kind), flags)
    return _single[key]


GRIDS = [(1, 2), (2, 1), (2, 2), (1, 4), (4, 1), (2, 4)]


@pytest.mark.parametrize("kind", ["small", "uneven", "tiny_nb128", "mx4"])
@pytest.mark.parametrize("sender", [False, True], ids=["receiver", "sender"])
@pytest.mark.parametrize("grid", GRIDS, ids=[f"{p}x{q}" for p, q in GRIDS])
def test_loopback_summa_bitwise_vs_single_gpu(grid, sender, kind):
    P, Q = grid
    w = _workload(kind)
    C1, m1 = single(kind)
    res = run_grid(w, P, Q, B.GMP_FLAG_SENDER_SIDE if sender else 0)
    recv_all = stored_all = 0
    for (p, q, loc, maps, st) in res:
        for k in ["acode", "bcode", "ccode", "ascale", "bscale"]:
            assert np.array_equal(m1[k], maps[k]), (p, q, k)
        want = closed_form_recv(maps["acode"], maps["bcode"], w.nb, P, Q, p, q)
        if sender:
            assert st["recv_bytes_local"] <= want, (p, q, st["recv_bytes_local"], want)
        else:
            assert st["recv_bytes_local"] == want, (p, q, st["recv_bytes_local"], want)
        recv_all += st["recv_bytes_local"]
        stored_all += want
    Cg = gather(w, res, P, Q)
    assert np.array_equal(Cg, C1), float(np.nanmax(np.abs(Cg - C1)))
    if sender and kind == "small":   # panel tiles whose receivers need cheaper classes travel as those
        assert recv_all < stored_all, (recv_all, stored_all)


@pytest.mark.parametrize("grid", [(2, 4), (4, 1)], ids=["2x4", "4x1"])
def test_loopback_simt_bitwise_vs_oracle(grid):
    """every class on the per-thread sequential-k kernels: the 8-rank (4-rank) C is the
    oracle's C bit for bit (the oracle knows nothing of the grid)"""
    P, Q = grid
    w = _workload("uneven")
    A, Bm, C = w.matrices()
    o = oracle.gemm_mp(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert o["rc"] == 0
    res = run_grid(w, P, Q, B.GMP_FLAG_SIMT_ONLY | B.GMP_FLAG_SENDER_SIDE, executes=1)
    for (_, _, _, maps, _) in res:
        assert np.array_equal(maps["acode"], o["acode"]) and np.array_equal(maps["bcode"], o["bcode"])
        assert np.array_equal(maps["ccode"], o["ccode"])
    assert np.array_equal(gather(w, res, P, Q), o["C"])



@pytest.mark.parametrize("kind", ["small", "uneven", "mx4"])
@pytest.mark.parametrize("sender", [False, True], ids=["receiver", "sender"])
@pytest.mark.parametrize("grid", [(2, 2), (2, 4), (1, 4)], ids=["2x2", "2x4", "1x4"])
def test_loopback_balanced_ownership_bitwise(grid, sender, kind):
    """NEXT-3: tile-row / tile-column owners from gemm_mp_balance (computed from the global
    maps, as every rank does); C gathered through the owners is BITWISE the 1-GPU C, the
    received bytes follow the closed form with the owners, and the model imbalance never
    exceeds block-cyclic's"""
    P, Q = grid
    w = _workload(kind)
    C1, m1 = single(kind)
    d = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, 0, P, Q, 0)
    ro, co, (imb0, imb1) = B.gemm_mp_balance(d, m1["acode"], m1["bcode"])
    assert imb1 <= imb0
    res = run_grid(w, P, Q, B.GMP_FLAG_SENDER_SIDE if sender else 0, ro=ro, co=co)
    for (p, q, loc, maps, st) in res:
        for k in ["acode", "bcode", "ccode", "ascale", "bscale"]:
            assert np.array_equal(m1[k], maps[k]), (p, q, k)
        want = closed_form_recv(maps["acode"], maps["bcode"], w.nb, P, Q, p, q, ro, co)
        if sender:
            assert st["recv_bytes_local"] <= want
        else:
            assert st["recv_bytes_local"] == want, (p, q, st["recv_bytes_local"], want)
    Cg = gather(w, res, P, Q, ro, co)
    assert np.array_equal(Cg, C1), float(np.nanmax(np.abs(Cg - C1)))


def test_loopback_explicit_uneven_owners_bitwise():
    """an arbitrary (unbalanced, non-cyclic) ownership with an empty process row: rows
    {0, 1, 2, 4} on process row 0, nothing else but row 3 on process row 1 -- C still bitwise"""
    w = _workload("uneven")   # 5 x 3 x 7 tiles
    C1, m1 = single("uneven")
    ro = np.array([0, 0, 0, 1, 0], np.int32)
    co = np.array([1, 1, 0], np.int32)
    res = run_grid(w, 2, 2, 0, ro=ro, co=co)
    assert np.array_equal(gather(w, res, 2, 2, ro, co), C1)
