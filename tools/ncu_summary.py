"""Summarise ncu reports / launch lists into compact text files for profiles/.

usage: python tools/ncu_summary.py full <report.ncu-rep> <out.md>
       python tools/ncu_summary.py launches <launches.csv> <out.md>
       python tools/ncu_summary.py traffic <report.ncu-rep> <out.json> <workload> <n_gpus>
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
]


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {rep}", ""]
    for r in data:
        lines.append(f"## {r[hdr.index('Kernel Name')][:160]}")
        for k in KEYS:
            if k in hdr:
                lines.append(f"- {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$", h)]
        stalls = sorted(((float(v), h) for h, v in stalls if v not in ("", "nan", "-nan")), reverse=True)[:8]
        lines.append("- top stalls (warps per issue): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in stalls))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


def traffic(rep, out, workload, n_gpus):
    """bytes per launch (dram read + write, mean over the captured launches) per kernel"""
    import json
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    acc = {}
    for r in data:
        name = re.sub(r"^void ", "", r[hdr.index("Kernel Name")])
        name = re.sub(r"\(.*", "", name) if not name.startswith("k_tc_class<") and not name.startswith("k_dmma<") \
            else re.sub(r"\(.*", "", name.replace("gmp::", ""))
        name = name.replace("gmp::", "")
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(r[i]) * scale.get(units[i], 1.0)
        acc.setdefault(name, []).append(tot)
    d = {"source": rep + " (ncu --set full)", "workload": workload, "n_gpus": int(n_gpus),
         "unit": "bytes per launch (dram read + write), mean over captured launches",
         "kernels": {k: sum(v) / len(v) for k, v in acc.items()}}
    json.dump(d, open(out, "w"), indent=1)


def launches(path, out):
    """per kernel: launches, total device ms (gpu__time_duration.sum) and share; DRAM bytes
    per launch when the list also holds dram__bytes_read/write.sum"""
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    idi = hdr.index("ID")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
    agg, order, seen = {}, [], set()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki])
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        if name not in agg:
            agg[name] = {"n": 0, "ms": 0.0, "dram": 0.0}
            order.append(name)
        a = agg[name]
        if r[mi] == "gpu__time_duration.sum":
            a["ms"] += v if r[ui] in scale else v / 1e6
            if r[idi] not in seen:
                seen.add(r[idi])
                a["n"] += 1
        elif r[mi].startswith("dram__bytes"):
            a["dram"] += v
    tot = sum(a["ms"] for a in agg.values())
    lines = [f"# ncu launch list (--clock-control none): {path}", "",
             "| kernel | launches | total ms | share | DRAM GB per launch | GB/s |", "|---|---|---|---|---|---|"]
    for n in order:
        a = agg[n]
        gb = a["dram"] / a["n"] / 1e9 if a["n"] and a["dram"] else None
        bw = a["dram"] / (a["ms"] * 1e-3) / 1e9 if a["ms"] and a["dram"] else None
        lines.append(f"| {n} | {a['n']} | {a['ms']:.3f} | {a['ms'] / tot:.1%} | "
                     f"{'' if gb is None else f'{gb:.2f}'} | {'' if bw is None else f'{bw:.0f}'} |")
    lines.append(f"| total | {sum(a['n'] for a in agg.values())} | {tot:.3f} | | | |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
