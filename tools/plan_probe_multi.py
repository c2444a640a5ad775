"""Where does gemm_mp_plan's time go on G GPUs?  (dev tool; run under torchrun)
Per iteration, after a barrier: event before plan, host wall time of the plan
call, event after; plus the stats kernel time measured alone (a plan with the
same inputs but timed on an idle GPU).  Prints one JSON line per rank."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gmp_inputs  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402

rank, G = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
lr = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(lr)
dev = torch.device("cuda", lr)
comm = None
P, Q = api.default_grid(G)
p, q = rank // Q, rank % Q
if G > 1:
    dist.init_process_group("nccl", device_id=dev)
    uid = B.gemm_mp_nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
    dist.broadcast(t, 0)
    comm = B.gemm_mp_nccl_comm_create(bytes(t.cpu().numpy()), G, rank)
w = gmp_inputs.workload(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
A = api.synth(w.M, w.K, w.nb, w.a, P, Q, p, q, device=dev)
Bm = api.synth(w.K, w.N, w.nb, w.b, P, Q, p, q, device=dev)
C = api.synth(w.M, w.N, w.nb, w.c, P, Q, p, q, device=dev) if w.beta else None
desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, 0, P, Q, rank)
nscr = B.gemm_mp_scratch_size(desc)
scr = torch.empty(nscr, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
res = []
for it in range(8):
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    pl = B.gemm_mp_plan(desc, A, A.stride(0), Bm, Bm.stride(0), C, C.stride(0) if C is not None else 0, scr, nscr,
                        comm, s)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    B.gemm_mp_destroy(pl)
    if it >= 2:
        res.append((e0.elapsed_time(e1), (t1 - t0) * 1e3))
print(json.dumps({"rank": rank, "G": G, "plan_event_ms": [round(a, 3) for a, _ in res],
                  "plan_host_ms": [round(b, 3) for _, b in res]}), flush=True)
if G > 1:
    dist.barrier()
    B.gemm_mp_nccl_comm_destroy(comm)
    dist.destroy_process_group()
