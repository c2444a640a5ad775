#!/usr/bin/env python3
"""Writes tests/golden/<cfg>_maps.txt: the ORACLE's A and B precision maps (S1-S2:
O1 generator, O4 CNORM, O5 criterion) of a full-size workload, one digit per tile
(class code 0..5), for the host-side load-balancing tests (NEXT-3; R30).
Calls only oracle/ (through bench.oracle_map) -- never the CUDA path.

    python tools/gen_golden_maps.py 3 4      # cfg3 and cfg4 (~12 s each on 16 threads)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gmp_inputs  # noqa: E402
from bench import oracle_map  # noqa: E402  (oracle-only S1-S2 over the whole workload)


def main():
    for cfg in [int(x) for x in sys.argv[1:]] or [3, 4]:
        w = gmp_inputs.workload(cfg)
        acode, bcode, pairs, dt = oracle_map(w, max(1, min(16, os.cpu_count() or 1)))
        path = os.path.join(ROOT, "tests", "golden", f"cfg{cfg}_maps.txt")
        with open(path, "w") as f:
            f.write(f"# {w.name}: oracle O5 maps (tools/gen_golden_maps.py, oracle/ only); "
                    f"BASELINE.json configs[{cfg - 1}], DESIGN.md section 5 input recipe\n")
            f.write(f"# mt kt nt = {acode.shape[0]} {acode.shape[1]} {bcode.shape[1]}; pairs per class {pairs}\n")
            f.write("A\n")
            for row in acode:
                f.write("".join(str(int(c)) for c in row) + "\n")
            f.write("B\n")
            for row in bcode:
                f.write("".join(str(int(c)) for c in row) + "\n")
        print(path, pairs, f"{dt:.1f} s")


if __name__ == "__main__":
    main()
