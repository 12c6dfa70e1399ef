"""Turn one evidence run (tools/gpu/evidence.sh -> gpurun_out/ev/) into the committed
profiles/<round>/ directory: bench JSON lines, ncu summaries, the launch list and the
README index with the tables DESIGN.md quotes.

  python tools/refresh_profiles.py [gpurun_out/ev] [profiles/r1]

Runs here (no GPU): the ncu reports are read with the local ncu binary.
"""
from __future__ import annotations

import csv
import glob
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

NCU_NOTES = {
    "ncu_c2_score": ("score_reg_kernel<u32, 8, 1>",
                     "DRAM traffic = algorithmic bytes; smem/issue-bound (DESIGN §3)"),
    "ncu_c3_score": ("score_reg_kernel<u32, 8, 1>", "as C2: smem/issue-bound"),
    "ncu_c4_score": ("score_reg_kernel<u64, 16, 1>", "64-bit sums, 128 registers, 2 CTAs/SM"),
    "ncu_c5_score": ("score_kernel (global scratch, 4-bit smem scan inputs)",
                     "scratch L2-resident; L1TEX random-access bound"),
    "ncu_c5_pairs": ("pair sweep fill (C5, 3.3e9 pairs)", "HBM writes of the pair list"),
    "ncu_c2_place": ("place_kernel (K5)", "latency-bound, sequential over edges"),
    "ncu_c2_arena": ("arena_kernel (K6), first pass", "issue/latency-bound, one warp per order"),
    "ncu_c3_lp": ("lp_write_kernel (K7)", "staged 16-byte stores"),
}


def load(path):
    """The bench JSON line in `path` (the last line that parses), else None."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        return None
    for ln in reversed(text.splitlines()):
        if ln.strip().startswith("{"):
            try:
                d = json.loads(ln)
            except ValueError:
                continue
            return d if isinstance(d, dict) and "metric" in d else None
    return None


def launch_list(src_csv, out_md):
    rows = []
    with open(src_csv) as f:
        text = f.read()
    start = text.find('"ID"')
    if start < 0:
        return
    agg = defaultdict(list)
    for r in csv.DictReader(text[start:].splitlines()):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            ns = v * 1e3 if r.get("Metric Unit") == "us" else v * 1e6 if r.get("Metric Unit") == "ms" else v
            agg[r["Kernel Name"]].append(ns)
    tot = sum(sum(v) for v in agg.values()) or 1.0
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        rows.append(f"| {len(v)} | {sum(v) / len(v):.0f} | {100 * sum(v) / tot:.1f}% | `{k[:90]}` |")
    with open(out_md, "w") as f:
        f.write("# ncu launch list: `python bench.py --steps 20 --warmup 3` (C2, cold-cache "
                "serialised launches)\n\n`ncu --metrics gpu__time_duration.sum --clock-control "
                "none -c 300`\n\n| launches | mean ns | share | kernel |\n|---|---|---|---|\n")
        f.write("\n".join(rows) + "\n")


def main():
    ev = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "ev")
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r1")
    os.makedirs(out, exist_ok=True)
    for p in glob.glob(os.path.join(ev, "*.json")):
        if load(p) is not None:
            shutil.copy(p, out)
    for name in ("smoke.log", "gpu_tests.log", "launches_c2.csv"):
        if os.path.exists(os.path.join(ev, name)):
            shutil.copy(os.path.join(ev, name), out)
    if os.path.exists(os.path.join(ev, "launches_c2.csv")):
        launch_list(os.path.join(ev, "launches_c2.csv"), os.path.join(out, "launches_c2.md"))
    for rep in glob.glob(os.path.join(ev, "*.ncu-rep")):
        base = os.path.splitext(os.path.basename(rep))[0]
        cmd = [sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep,
               os.path.join(out, base)]
        if base.endswith("_score"):
            cfg = base.split("_")[1]
            b = load(os.path.join(out, f"bench_{cfg}.json"))
            if b:
                cmd += ["--algorithmic-bytes", str(int(b["roofline"]["algorithmic_bytes_per_launch"]))]
        subprocess.run(cmd, check=False)
        if base.endswith("_score"):   # bench.py reads roofline.traffic from here
            cfg = base.split("_")[1]
            src = os.path.join(out, base + ".json")
            if os.path.exists(src):
                shutil.copy(src, os.path.join(ROOT, "profiles", f"{cfg}_score_ncu.json"))

    lines = ["# Round-1 evidence (one B200, driver-measured peaks in MEASURED_PEAKS.json)", "",
             "All JSON lines are `bench.py` output from one fresh gpurun box "
             "(`tools/gpu/evidence.sh`, summarised by `tools/refresh_profiles.py`); `ncu_*.md` are "
             "`ncu --set full --clock-control none` summaries (cold-cache, serialised: compare "
             "shares, not absolute times); `launches_c2.*` is the launch list of the default bench "
             "command; `gpu_tests.log` the `pytest -m gpu` run.", "",
             "## K3 fused scorer (the bench metric)", "",
             "| config | plans/s | µs/step | HBM frac | e2e plans/s | reference CPU |",
             "|---|---|---|---|---|---|"]
    ref = load(os.path.join(out, "ref_c2.json"))
    for c in ("c2", "c3", "c4", "c5"):
        b = load(os.path.join(out, f"bench_{c}.json"))
        if not b:
            continue
        cpu = b.get("cpu_baseline") or {}
        cpu_s = f"{cpu['value']:.3g} ({cpu.get('cores')} thr)" if cpu.get("value") else "—"
        lines.append(f"| {b['config']['workload']} | {b['value']:.3g} | {b['ms_per_step'] * 1e3:.1f} "
                     f"| {b['roofline']['frac']:.3f} | {b['e2e']['value']:.3g} | {cpu_s} |")
    if ref:
        lines += ["", f"`bench.py --impl reference` (C2): {ref['value']:.3g} plans/s on "
                      f"{ref['cpu_baseline']['cores']} host threads (`ref_c2.json`)."]
    lines += ["", "## §8f subsystems and K2", "", "| file | metric | GPU | reference (CPU) |",
              "|---|---|---|---|"]
    for mode in ("pairs", "place", "arena", "lp", "joint"):
        for c in ("c2", "c3", "c4", "c5"):
            b = load(os.path.join(out, f"{mode}_{c}.json"))
            if not b:
                continue
            cpu = b.get("cpu_baseline") or {}
            cpu_s = (f"{cpu['value']:.3g} {cpu.get('unit', b['unit'])} ({cpu.get('kind')}, "
                     f"{cpu.get('cores')} thr)") if cpu.get("value") else "—"
            lines.append(f"| `{mode}_{c}.json` | {b['metric'][:60]} | {b['value']:.3g} {b['unit']} "
                         f"| {cpu_s} |")
    lines += ["", "## ncu captures", "", "| file | kernel | note |", "|---|---|---|"]
    for md in sorted(glob.glob(os.path.join(out, "ncu_*.md"))):
        base = os.path.splitext(os.path.basename(md))[0]
        k, note = NCU_NOTES.get(base, ("", ""))
        lines.append(f"| `{base}.md` | {k} | {note} |")
    lines += ["", "`smoke.log`: `__graft_entry__.smoke()` on cuda:0."]
    with open(os.path.join(out, "README.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
