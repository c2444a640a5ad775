import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import gmp_inputs
from paper_2508_14848_b200 import api, binding as B
for cfg in (3, 4):
    w = gmp_inputs.workload(cfg)
    A = api.synth(w.M, w.K, w.nb, w.a); Bm = api.synth(w.K, w.N, w.nb, w.b)
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    g = api.GemmMP(desc, A, Bm, None)
    m = g.maps()
    np.savez(f"gpurun_out/maps_cfg{cfg}.npz", acode=m["acode"], bcode=m["bcode"], ccode=m["ccode"])
    g.close(); del A, Bm; torch.cuda.empty_cache()
    print("saved", cfg)
