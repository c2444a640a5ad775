"""One cuBLAS BF16 GEMM and one all-BF16 gemm_mp execute (default / pair kernel) for an
ncu comparison of the tensor-class kernels against the library (SURVEY 8(d) evidence)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import gmp_inputs
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

n = int(os.environ.get("N", "16384"))
a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
torch.matmul(a, b)
torch.cuda.synchronize()
del a, b
w = gmp_inputs.small_workload(n, n, n, 2048, 1e-4, mode="random", E=32, beta=0.0, seed=3000)
A = api.synth(w.M, w.K, w.nb, w.a)
Bm = api.synth(w.K, w.N, w.nb, w.b)
t = n // 2048
amap = np.full((t, t), 3, np.uint8)
out = torch.empty(n, n, dtype=torch.float64, device="cuda")
for flags in [int(f) for f in os.environ.get("FLAGS", "0,32").split(",")]:
    desc = B.make_desc(n, n, n, 2048, 1e-4, 1.0, 0.0, 0b01111, flags, a_map=amap, b_map=amap)
    g = api.GemmMP(desc, A, Bm, None)
    g.convert()
    g.execute(out)
    g.sync()
    g.close()
print("ok")
