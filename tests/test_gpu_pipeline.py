"""api.HostPipeline (host-buffer GEMM stream, bench.py's e2e leg): every step's
host result equals the result of the same GEMM run on its own, for a stream of
DIFFERENT inputs, so the multi-buffering never mixes steps up; and the
library's table staging (mapped pinned memory, k_xfer) holds up while large
copies occupy the copy engines."""
import numpy as np
import pytest
import torch

import gmp_inputs
from gpu_harness import run_gpu
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("beta,nbuf", [(0.0, 3), (0.5, 3), (0.5, 2), (0.0, 1), (0.5, 1)])
def test_host_pipeline_matches_single_runs(beta, nbuf):
    M, N, K, nb = 768, 512, 1024, 128
    steps = 6
    hA, hB, hC, want = [], [], [], []
    for k in range(steps):
        w = gmp_inputs.small_workload(M, N, K, nb, 1e-5, mode="random", E=20, beta=beta, seed=40 + k,
                                      class_mask=0b11111)
        A, Bm, C = w.matrices()
        hA.append(torch.from_numpy(A).pin_memory())
        hB.append(torch.from_numpy(Bm).pin_memory())
        hC.append(torch.from_numpy(C).pin_memory() if beta != 0.0 else None)
        _, (out,) = run_gpu(A, Bm, C if beta != 0.0 else None, nb, w.tol, w.alpha, beta, w.class_mask)
        want.append(out)
    desc = B.make_desc(M, N, K, nb, 1e-5, 1.0, beta, 0b11111)
    dev = torch.device("cuda:0")
    pipe = api.HostPipeline(desc, (M, K), (K, N), (M, N) if beta != 0.0 else None, (M, N), dev, nbuf=nbuf)
    pipe.reserve(hA[0], hB[0], hC[0])
    hOut = [torch.full((M, N), float("nan"), dtype=torch.float64).pin_memory() for _ in range(steps)]
    pipe.run(hA, hB, hC, hOut)
    torch.cuda.synchronize()
    pipe.close()
    for k in range(steps):
        assert np.array_equal(hOut[k].numpy(), want[k]), f"step {k}"


def test_execute_after_holds_back_only_the_finalize():
    """gemm_mp_execute_after: the C-finalize waits for the caller's event.  A side stream
    sleeps, then overwrites C with NaN and records the event; the execute's result must land
    after that write (C finite and equal to a plain execute's), so C is never written before
    the event."""
    w = gmp_inputs.small_workload(512, 512, 768, 128, 1e-5, mode="random", E=24, beta=0.0, seed=78,
                                  class_mask=0b11111)
    A, Bm, _ = w.matrices()
    dev = torch.device("cuda:0")
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    g = api.GemmMP(desc, torch.from_numpy(A).to(dev), torch.from_numpy(Bm).to(dev), None)
    g.convert()
    ref = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g.execute(ref)
    g.sync()
    out = torch.zeros(w.M, w.N, dtype=torch.float64, device=dev)
    side = torch.cuda.Stream(dev)
    ev = torch.cuda.Event()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(200_000_000)            # ~0.1 s
        out.fill_(float("nan"))
        ev.record(side)
    cur = torch.cuda.current_stream(dev)
    B.gemm_mp_execute_after(g.plan, out, out.stride(0), cur, ev)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("flags", [0, B.GMP_FLAG_SPLIT16])
def test_execute_replays_from_a_cuda_graph(flags):
    """after one warm-up execute, gemm_mp_execute issues kernels only (the C tile
    descriptors are already on the device), so a captured execute replays to the
    same C, bit for bit, as often as it is launched"""
    w = gmp_inputs.small_workload(512, 768, 1024, 128, 1e-5, mode="random", E=24, beta=0.5, seed=77,
                                  class_mask=0b11111)
    A, Bm, C = w.matrices()
    dev = torch.device("cuda:0")
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags)
    g = api.GemmMP(desc, torch.from_numpy(A).to(dev), torch.from_numpy(Bm).to(dev), torch.from_numpy(C).to(dev))
    g.convert()
    out = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g.execute(out)
    g.sync()
    ref = out.clone()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            g.execute(out, stream=side)
    torch.cuda.synchronize()
    for _ in range(3):
        out.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    g.close()
