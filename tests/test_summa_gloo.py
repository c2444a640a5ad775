"""Multi-rank host logic of the SUMMA path on CPU (gloo, world sizes 2 and 4).

Every rank builds the library's host-side plan (gemm_mp_plan_host) from the
same oracle maps, executes ITS SUMMA schedule with torch.distributed (gloo)
broadcasts of oracle-packed stored payloads on the row / column groups, and
checks (1) every tile-GEMM operand it needs arrives bit-exact in its stored
precision -- or, under GMP_FLAG_SENDER_SIDE,
as the oracle's shadows of the stored payload in every class a receiver needs --
(2) its received bytes equal the library's count and the closed form (SURVEY
8(e); for the hybrid mode the cheaper of stored vs union-of-needed-classes per
tile), (3) the local tile-GEMMs of all ranks partition the global pair set.  The GPU run of the same schedule over NCCL is
tools/multi_gpu_check.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

BY = [8, 4, 2, 2, 1, 1, 17 / 32]   # bytes per element; MXFP4: nibbles + one scale byte per 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _wire(code, partner_codes):
    """hybrid rule: the union of pair classes the receivers need, if cheaper than the stored payload"""
    S = {max(code, int(c)) for c in partner_codes}
    return S if S and sum(BY[c] for c in S) < BY[code] else {code}


def _worker(rank, G, port, q_out, sender=False, balanced=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import gmp_inputs
    import oracle
    from paper_2508_14848_b200 import api
    from paper_2508_14848_b200 import binding as B
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        nb = 64 if False else 128
        w = gmp_inputs.small_workload(5 * nb, 3 * nb, 9 * nb, nb, 1e-4, mode="random", E=32, beta=0.0,
                                      class_mask=0b111111, seed=9)
        A, Bm, C = w.matrices()
        o = oracle.gemm_mp(A, Bm, None, nb, w.tol, w.alpha, 0.0, w.class_mask, ctiles=[])
        mt, kt, nt = o["acode"].shape[0], o["acode"].shape[1], o["bcode"].shape[1]
        P, Q = api.default_grid(G)
        p, q = rank // Q, rank % Q
        flags = B.GMP_FLAG_SENDER_SIDE if sender else 0
        ro = co = None
        if balanced:   # NEXT-3: every rank computes the same owners from the same global maps
            d0 = B.make_desc(w.M, w.N, w.K, nb, w.tol, w.alpha, 0.0, w.class_mask, flags, P, Q, rank)
            ro, co, _ = B.gemm_mp_balance(d0, o["acode"], o["bcode"])
        rows_own = api.owned_tiles(mt, P, p, ro)
        cols_own = api.owned_tiles(nt, Q, q, co)
        rowP = [i % P if ro is None else int(ro[i]) for i in range(mt)]
        colQ = [j % Q if co is None else int(co[j]) for j in range(nt)]
        desc = B.make_desc(w.M, w.N, w.K, nb, w.tol, w.alpha, 0.0, w.class_mask, flags, P, Q, rank,
                           row_owner=ro, col_owner=co)
        plan = B.gemm_mp_plan_host(desc, o["acode"], o["bcode"], o["ccode"], o["ascale5"], o["bscale5"])
        st = B.gemm_mp_get_stats(plan)
        rows = [dist.new_group([pp * Q + qq for qq in range(Q)]) for pp in range(P)]
        cols = [dist.new_group([pp * Q + qq for pp in range(P)]) for qq in range(Q)]

        def stored(which, g):
            if which == 0:
                i, l = divmod(g, kt)
                t = A[i * nb:(i + 1) * nb, l * nb:(l + 1) * nb]
                c = int(o["acode"][i, l]); e = int(o["ascale5"][i, l, c]); role = "A"
            else:
                l, j = divmod(g, nt)
                t = Bm[l * nb:(l + 1) * nb, j * nb:(j + 1) * nb]
                c = int(o["bcode"][l, j]); e = int(o["bscale5"][l, j, c]); role = "B"
            return oracle.pack_tile(t, c, e, role=role), c, e, role

        def payload(which, g, cls):
            p0, c, e, role = stored(which, g)
            if cls == c:
                return p0.view(np.uint8)
            return oracle.shadow_tile(p0, nb, c, e, cls, role=role)[0].view(np.uint8)

        have = {}
        recv = 0
        errs = []
        for s in range(st["steps"]):
            sched = B.gemm_mp_get_schedule(plan, s)
            works, bufs = [], []
            for which, g, cls, root, nbytes in sched:
                grp = rows[p] if which == 0 else cols[q]
                root_global = p * Q + root if which == 0 else root * Q + q
                if root_global == rank:
                    buf = torch.from_numpy(payload(which, g, cls).copy())
                    have.setdefault((which, int(g)), set()).add(stored(which, g)[1])   # the root owns the tile
                else:
                    buf = torch.zeros(int(nbytes), dtype=torch.uint8)
                    recv += int(nbytes)
                if buf.numel() != nbytes:
                    errs.append(f"size of tile {which}:{g}")
                works.append(dist.broadcast(buf, root_global, group=grp, async_op=True))
                bufs.append((which, int(g), int(cls), buf))
            for wk in works:
                wk.wait()
            for which, g, cls, buf in bufs:
                if not np.array_equal(buf.numpy(), payload(which, g, cls)):
                    errs.append(f"payload mismatch {which}:{g}:{cls}")
                have.setdefault((which, g), set()).add(cls)
        # every operand of every local tile-GEMM is present: its pair class, or the
        # stored class (receiver-side conversion)
        pairs_local = 0
        for i in rows_own:
            for j in cols_own:
                for l in range(kt):
                    pairs_local += 1
                    ca, cb = int(o["acode"][i, l]), int(o["bcode"][l, j])
                    c = max(ca, cb)
                    ha, hb = have.get((0, i * kt + l), set()), have.get((1, l * nt + j), set())
                    if not (c in ha or ca in ha) or not (c in hb or cb in hb):
                        errs.append(f"missing operand for C({i},{j}) l={l}")
        if sender:
            closed = sum(nb * nb * sum(BY[c] for c in _wire(int(o["acode"][i, l]),
                                                            [o["bcode"][l, j] for j in range(nt) if colQ[j] != l % Q]))
                         for i in rows_own for l in range(kt) if l % Q != q) + \
                sum(nb * nb * sum(BY[c] for c in _wire(int(o["bcode"][l, j]),
                                                       [o["acode"][i, l] for i in range(mt) if rowP[i] != l % P]))
                    for j in cols_own for l in range(kt) if l % P != p)
        else:
            closed = sum(nb * nb * BY[o["acode"][i, l]] for i in rows_own for l in range(kt) if l % Q != q) + \
                sum(nb * nb * BY[o["bcode"][l, j]] for j in cols_own for l in range(kt) if l % P != p)
        stored_bytes = sum(nb * nb * BY[o["acode"][i, l]] for i in rows_own for l in range(kt) if l % Q != q) + \
            sum(nb * nb * BY[o["bcode"][l, j]] for j in cols_own for l in range(kt) if l % P != p)
        q_out.put(dict(rank=rank, errs=errs, recv=recv, recv_lib=st["recv_bytes_local"], closed=closed,
                       stored_bytes=stored_bytes,
                       pairs_local=sum(st["pairs_local"]), pairs_count=pairs_local, pairs_total=sum(st["pairs"]),
                       grid=(P, Q)))
        B.gemm_mp_destroy(plan)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,sender,balanced", [(2, False, False), (4, False, False), (2, True, False),
                                               (4, True, False), (8, False, False), (4, True, True),
                                               (8, False, True)])
def test_summa_schedule_over_gloo(G, sender, balanced):
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, qo, sender, balanced)) for r in range(G)]
    for pr in procs:
        pr.start()
    res = [qo.get(timeout=300) for _ in range(G)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    tot = 0
    for r in res:
        assert not r["errs"], r["errs"][:5]
        assert r["recv"] == r["recv_lib"] == r["closed"], r
        assert r["recv"] <= r["stored_bytes"]
        if not sender:
            assert r["recv"] == r["stored_bytes"]
        assert r["pairs_local"] == r["pairs_count"]
        tot += r["pairs_local"]
    assert tot == res[0]["pairs_total"]
    assert any(r["recv"] > 0 for r in res)
    if sender:   # the E4M3-enabled random workload has tiles whose receivers need less than stored
        assert sum(r["recv"] for r in res) < sum(r["stored_bytes"] for r in res)


def test_spec_closed_form_128_bytes():
    """mt=nt=kt=2, grid 2x1, nb=2, all-FP64 -> 128 bytes received in total;
    all-FP32 B -> 64.  Our slots hold nb*nb payloads: check the same closed form with
    nb = 128 scaled by (128/2)^2."""
    from paper_2508_14848_b200 import binding as B
    nb = 128
    tot = {}
    for bcls in (0, 1):
        s = 0
        for rank in range(2):
            d = B.make_desc(2 * nb, 2 * nb, 2 * nb, nb, 1e-6, 1.0, 0.0, 0b00011, 0, 2, 1, rank)
            ac = np.zeros((2, 2), np.uint8); bc = np.full((2, 2), bcls, np.uint8); cc = np.zeros((2, 2), np.uint8)
            z = np.zeros((2, 2, B.NCLS), np.int16)
            pl = B.gemm_mp_plan_host(d, ac, bc, cc, z, z)
            s += B.gemm_mp_get_stats(pl)["recv_bytes_local"]
            B.gemm_mp_destroy(pl)
        tot[bcls] = s * (2 * 2) // (nb * nb)
    assert tot[0] == 128 and tot[1] == 64
