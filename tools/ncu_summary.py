"""Summarise an ncu capture into profiles/ (committed evidence).

  python tools/ncu_summary.py gpurun_out/score_c2.ncu-rep profiles/r1_c2_score --algorithmic-bytes N

Writes <out>.json (key metrics incl. dram bytes per launch) and <out>.md
(metrics + top source lines by warp-stall samples). Needs only the local ncu
binary (no GPU).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions", "Block Size",
        "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "Block Limit Registers", "Block Limit Shared Mem", "L1/TEX Hit Rate", "L2 Hit Rate"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    det = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "details", "--csv"))))
    h = det[0]
    mi, ui, vi, ki = (h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"),
                      h.index("Kernel Name"))
    metrics = {}
    kernel = det[1][ki] if len(det) > 1 else ""
    for r in det[1:]:
        if r[mi] in KEEP and r[mi] not in metrics:
            metrics[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "raw", "--csv"))))
    rawm = {}
    if len(raw) >= 3:
        names, units, vals = raw[0], raw[1], raw[2]
        for name in RAW:
            if name in names:
                i = names.index(name)
                rawm[name] = (vals[i], units[i])
    dram = None
    if "dram__bytes_read.sum" in rawm and "dram__bytes_write.sum" in rawm:
        dram = sum(to_bytes(*rawm[k]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    src = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "source", "--csv",
                                          "--print-source=cuda,sass"))))

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    lines = [(int(r[0]), r[1].strip()[:100], f(r[4]), f(r[7])) for r in src
             if len(r) > 8 and r[0].isdigit()]
    tot = sum(x[2] for x in lines) or 1.0
    toti = sum(x[3] for x in lines) or 1.0
    top = [{"line": ln, "src": s, "stall_pct": round(100 * st / tot, 1),
            "inst_pct": round(100 * ins / toti, 1)}
           for ln, s, st, ins in sorted(lines, key=lambda x: -x[2])[:20]]
    doc = {"kernel": kernel, "metrics": metrics, "raw": {k: " ".join(v) for k, v in rawm.items()},
           "dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": a.algorithmic_bytes,
           "note": a.note, "top_lines": top}
    with open(a.out + ".json", "w") as fo:
        json.dump(doc, fo, indent=1)
    with open(a.out + ".md", "w") as fo:
        fo.write(f"# {a.out.split('/')[-1]}\n\nkernel: `{kernel}`\n\n{a.note}\n\n")
        fo.write("| metric | value |\n|---|---|\n")
        for k, v in metrics.items():
            fo.write(f"| {k} | {v} |\n")
        for k, v in rawm.items():
            fo.write(f"| {k} | {' '.join(v)} |\n")
        if dram is not None:
            fo.write(f"| dram bytes per launch (read+write) | {dram:.0f} |\n")
        if a.algorithmic_bytes:
            fo.write(f"| algorithmic bytes per launch | {a.algorithmic_bytes:.0f} |\n")
        fo.write("\n## top source lines (warp-stall samples)\n\n| stall % | inst % | line | source |\n"
                 "|---|---|---|---|\n")
        for t in top:
            fo.write(f"| {t['stall_pct']} | {t['inst_pct']} | {t['line']} | `{t['src']}` |\n")
    print(json.dumps({"dram_bytes_per_launch": dram, **metrics}, indent=1))


if __name__ == "__main__":
    main()
