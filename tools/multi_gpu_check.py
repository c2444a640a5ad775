"""Multi-GPU check (run under torchrun, one process per GPU): the SUMMA path on a
P x Q grid must give maps identical to the 1-GPU run and a C that is BITWISE the
1-GPU C (the fold order is G-independent, R15), and every rank's
received SUMMA bytes must equal the closed form.  Prints one JSON
line on rank 0 and exits non-zero on any mismatch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gmp_inputs  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402


def closed_form_recv(acode, bcode, nb, P, Q, p, q, row_owner=None, col_owner=None):
    mt, kt = acode.shape
    nt = bcode.shape[1]
    by = [8, 4, 2, 2, 1, 1, 17 / 32]
    tot = 0
    for i in api.owned_tiles(mt, P, p, row_owner):
        for l in range(kt):
            if l % Q != q:
                tot += nb * nb * by[acode[i, l]]
    for j in api.owned_tiles(nt, Q, q, col_owner):
        for l in range(kt):
            if l % P != p:
                tot += nb * nb * by[bcode[l, j]]
    return tot


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="small")
    ap.add_argument("--sender", action="store_true", help="GMP_FLAG_SENDER_SIDE (hybrid conversion, NEXT-2)")
    ap.add_argument("--grid", default=None, help="PxQ process grid (default: api.default_grid)")
    ap.add_argument("--nccl", action="store_true", help="GMP_FLAG_NCCL_BCAST: NCCL broadcasts instead of CE pulls")
    ap.add_argument("--balance", action="store_true",
                    help="NEXT-3: owners from gemm_mp_balance on the maps of a block-cyclic plan")
    a = ap.parse_args()
    rank, G = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr_ = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr_)
    dev = torch.device("cuda", lr_)
    dist.init_process_group("nccl", device_id=dev)
    if a.cfg == "small":
        w = gmp_inputs.small_workload(2048, 1536, 2560, 256, 1e-4, mode="random", E=32, beta=0.75, seed=5,
                                      class_mask=0b111111)
    elif a.cfg == "uneven":   # tile grids that do not divide by P or Q (5 x 3 x 7 tiles of 256)
        w = gmp_inputs.small_workload(1280, 768, 1792, 256, 1e-3, mode="graded", E=24, beta=-0.5, seed=6,
                                      class_mask=0b111111)
    else:
        w = gmp_inputs.workload(int(a.cfg))
    P, Q = api.default_grid(G) if a.grid is None else tuple(int(v) for v in a.grid.split("x"))
    assert P * Q == G, (P, Q, G)
    p, q = rank // Q, rank % Q
    uid = B.gemm_mp_nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
    dist.broadcast(t, 0)
    comm = B.gemm_mp_nccl_comm_create(bytes(t.cpu().numpy()), G, rank)

    flags = (B.GMP_FLAG_SENDER_SIDE if a.sender else 0) | (B.GMP_FLAG_NCCL_BCAST if a.nccl else 0)
    ro = co = None
    imb = None
    if a.balance:   # a block-cyclic plan gives the global maps; every rank balances them the same way
        A0, B0, C0 = api.synth_operands(w, P, Q, p, q, device=dev)
        d0 = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags, P, Q, rank)
        g0 = api.GemmMP(d0, A0, B0, C0, nccl_comm=comm, device=dev)
        m0 = g0.maps()
        g0.close()
        del A0, B0, C0
        ro, co, imb = B.gemm_mp_balance(d0, m0["acode"], m0["bcode"])
    A, Bm, C = api.synth_operands(w, P, Q, p, q, ro, co, device=dev)
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags, P, Q, rank,
                       row_owner=ro, col_owner=co)
    g = api.GemmMP(desc, A, Bm, C, nccl_comm=comm, device=dev)
    g.convert()
    lr, lc = api.local_c_shape(w, P, Q, p, q, ro, co)
    out = torch.full((lr, lc), float("nan"), dtype=torch.float64, device=dev)
    g.execute(out)
    g.execute(out)  # twice: receive slots are refilled every execute
    g.sync()
    maps = g.maps()
    st = g.stats()
    ok = True
    msgs = []
    want_recv = closed_form_recv(maps["acode"], maps["bcode"], w.nb, P, Q, p, q, ro, co)
    if a.sender:   # hybrid: never more than the stored bytes (the gloo test checks the exact rule)
        if st["recv_bytes_local"] > want_recv:
            ok = False
            msgs.append(f"rank {rank}: sender-side recv bytes {st['recv_bytes_local']} > stored {want_recv}")
    elif st["recv_bytes_local"] != want_recv:
        ok = False
        msgs.append(f"rank {rank}: recv bytes {st['recv_bytes_local']} != closed form {want_recv}")
    recv_all = [None] * G
    dist.all_gather_object(recv_all, (st["recv_bytes_local"], want_recv))
    # gather local C tiles on rank 0
    outs = [None] * G
    dist.all_gather_object(outs, (p, q, out.cpu().numpy()))
    if rank == 0:
        # reference: the same library on one GPU (G = 1)
        Af, Bf, Cf = api.synth_operands(w, device=dev)
        d1 = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
        g1 = api.GemmMP(d1, Af, Bf, Cf, device=dev)
        g1.convert()
        full = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
        g1.execute(full)
        g1.sync()
        m1 = g1.maps()
        for k in ["acode", "bcode", "ccode", "ascale", "bscale"]:
            if not np.array_equal(m1[k], maps[k]):
                ok = False
                msgs.append(f"map {k} differs from 1-GPU")
        F = full.cpu().numpy()
        nb = w.nb
        Cg = np.full_like(F, np.nan)
        for (pp, qq, loc) in outs:
            rr, cc = api.place_local_c(Cg, loc, w, P, Q, pp, qq, ro, co)
            if not np.array_equal(F[np.ix_(rr, cc)], loc):
                ok = False
                diff = np.nanmax(np.abs(F[np.ix_(rr, cc)] - loc))
                msgs.append(f"C of rank ({pp},{qq}) differs from 1-GPU (max |d| {diff})")
        if np.isnan(Cg).any():
            ok = False
            msgs.append("the ranks' local C tiles do not cover C")
        print(json.dumps({"ok": ok, "G": G, "grid": f"{P}x{Q}", "workload": w.name, "msgs": msgs,
                          "mode": "sender-side (hybrid)" if a.sender else "receiver-side",
                          "ownership": "balanced (gemm_mp_balance)" if a.balance else "block-cyclic",
                          "transport": "ncclBroadcast" if a.nccl else "copy-engine pulls (CUDA IPC)",
                          "imbalance_model": imb,
                          "covered": bool(not np.isnan(Cg).any()),
                          "recv_bytes_rank0": st["recv_bytes_local"], "recv_bytes_all": sum(r[0] for r in recv_all),
                          "stored_bytes_all": sum(r[1] for r in recv_all), "pairs": st["pairs"]}), flush=True)
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    g.close()
    dist.barrier()
    B.gemm_mp_nccl_comm_destroy(comm)
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
