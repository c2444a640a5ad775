"""Timeline of api.HostPipeline (bench.py's e2e leg) on N GPUs (torchrun): for each
step, when its H2D copy, convert, execute and D2H copy completed (ms after the
timed start, rank 0), to see what the pipelined host-buffer stream waits on."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import gmp_inputs
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    nbuf = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rank, G = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    lr_ = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr_)
    dev = torch.device("cuda", lr_)
    if G > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = gmp_inputs.workload(2)
    P, Q = api.default_grid(G)
    p, q = rank // Q, rank % Q
    comm = None
    if G > 1:
        uid = B.gemm_mp_nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
        dist.broadcast(t, 0)
        comm = B.gemm_mp_nccl_comm_create(bytes(t.cpu().numpy()), G, rank)
    A = api.synth(w.M, w.K, w.nb, w.a, P, Q, p, q, device=dev)
    Bm = api.synth(w.K, w.N, w.nb, w.b, P, Q, p, q, device=dev)
    C = api.synth(w.M, w.N, w.nb, w.c, P, Q, p, q, device=dev)
    lr, lc = api.local_shape(w.M, w.N, w.nb, P, Q, p, q)
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, 0, P, Q, rank)
    hA, hB, hC = A.cpu().pin_memory(), Bm.cpu().pin_memory(), C.cpu().pin_memory()
    hOut = [torch.empty((lr, lc), dtype=torch.float64).pin_memory() for _ in range(2)]
    pipe = api.HostPipeline(desc, tuple(A.shape), tuple(Bm.shape), tuple(C.shape), (lr, lc), dev, comm=comm,
                            nbuf=nbuf)
    pipe.reserve(hA, hB, hC)
    pipe.run([hA], [hB], [hC], [hOut[0]])
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    pipe.record_timeline = True
    s0 = torch.cuda.Event(enable_timing=True)
    s0.record(pipe.compute)
    pipe.h2d.wait_stream(pipe.compute)
    pipe.d2h.wait_stream(pipe.compute)
    pipe.run([hA] * K, [hB] * K, [hC] * K, [hOut[k % 2] for k in range(K)])
    torch.cuda.synchronize()
    h2d, conv, ex, d2h = pipe.timeline
    if rank == 0:
        print(f"G={G} nbuf={nbuf} local A {tuple(A.shape)}, {K} steps; ms after start: h2d_done convert_done "
              "exec_done d2h_done")
        for k in range(K):
            print(k, *[round(s0.elapsed_time(e[k]), 1) for e in (h2d, conv, ex, d2h)])
    pipe.close()
    if G > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
