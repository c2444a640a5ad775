"""Markdown table from tools/config_sweep.py's JSON lines (profiles/config_sweep_*.md).

usage: python tools/config_sweep_md.py <sweep.jsonl> <title> > out.md
"""
import json
import sys


def main():
    path, title = sys.argv[1], sys.argv[2]
    rows = [json.loads(line) for line in open(path) if line.strip().startswith("{")]
    print(f"# {title} (`tools/config_sweep.py --reps 3`, {path.split('/')[-1]})\n")
    print("Execute = best of 3 repeated executes of one plan (the packed operands stay resident); step adds this "
          "run's plan + convert.  Roofline = sum_c F_c / Peak_c with MEASURED_PEAKS.json BF16 (burst) x nominal "
          "ratios (FP32 class = BF16 / 6, BF16x6; MXFP4 = 4 x BF16); power-capped runs sit below it (SM clock "
          "column).\n")
    print("| run | execute TF/s | step TF/s | class TF/s | roofline frac (execute) | SM MHz |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        if "tflops_exec" not in r:
            v = r.get("tflops") or r.get("value")
            print(f"| {r.get('run')} | {v if v is None else round(v, 1)} | | | | |")
            continue
        cls = ", ".join(f"{k} {v}" for k, v in (r.get("class_tflops") or {}).items())
        frac = r.get("roof_frac_exec")
        step = r.get("tflops_step")
        print(f"| {r['run']} | {r['tflops_exec']:.1f} | {'' if step is None else round(step, 1)} | {cls} | "
              f"{'' if frac is None else round(frac, 3)} | {r.get('clocks', {}).get('sm_mhz', '')} |")


if __name__ == "__main__":
    main()
