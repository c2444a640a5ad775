"""Host and device time of each C-ABI call of one step (dev tool)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gmp_inputs  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = gmp_inputs.workload(cfg)
dev = torch.device("cuda:0")
A = api.synth(w.M, w.K, w.nb, w.a)
Bm = api.synth(w.K, w.N, w.nb, w.b)
C = api.synth(w.M, w.N, w.nb, w.c) if w.beta else None
out = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
nscr = B.gemm_mp_scratch_size(desc)
scr = torch.empty(nscr, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
ws = None
res = []
for it in range(6):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record()
    pl = B.gemm_mp_plan(desc, A, A.stride(0), Bm, Bm.stride(0), C, C.stride(0) if C is not None else 0, scr, nscr, None, s)
    t1 = time.perf_counter()
    ev[1].record()
    n = B.gemm_mp_workspace_size(pl)
    if ws is None:
        ws = torch.empty(n + 1024, dtype=torch.uint8, device=dev)
    base = ws.data_ptr() + (-ws.data_ptr()) % 1024
    B.gemm_mp_convert(pl, base, n, s)
    t2 = time.perf_counter()
    ev[2].record()
    B.gemm_mp_execute(pl, out, out.stride(0), s)
    t3 = time.perf_counter()
    ev[3].record()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    B.gemm_mp_destroy(pl)
    res.append(dict(host_plan=(t1 - t0) * 1e3, host_convert=(t2 - t1) * 1e3, host_execute=(t3 - t2) * 1e3,
                    wall=(t4 - t0) * 1e3, dev_plan=ev[0].elapsed_time(ev[1]), dev_convert=ev[1].elapsed_time(ev[2]),
                    dev_execute=ev[2].elapsed_time(ev[3])))
print(json.dumps({k: round(v, 3) for k, v in res[-1].items()}))
print(json.dumps({k: round(v, 3) for k, v in res[-2].items()}))
