"""Does operand data change tensor-pipe power?  cuBLAS FP16 16384^3 for ~4 s on
(a) torch.randn values, (b) uniform [-1, 1) scaled by 2^15 (full-range FP16
payloads with random mantissas, like this library's per-tile scaled FP16 tiles),
(c) small integers (few mantissa bits toggling).  Prints TF/s, clock, power."""
import os
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from power_probe import timed  # noqa: E402


def main():
    n = 16384
    for name, gen in [("randn", lambda: torch.randn(n, n, device="cuda")),
                      ("uniform_2^15", lambda: (torch.rand(n, n, device="cuda") * 2 - 1) * 32768.0),
                      ("small_ints", lambda: torch.randint(-3, 4, (n, n), device="cuda").float())]:
        a = gen().half()
        b = gen().half()
        c = torch.empty(n, n, dtype=torch.float16, device="cuda")
        r = timed(lambda: torch.matmul(a, b, out=c), 4.0, 2.0 * n ** 3)
        print(json.dumps(dict(run=f"cublas_fp16_{name}", **r)), flush=True)
        del a, b, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    main()
