"""Probe: fused scorer time vs candidates per CTA (fixed cost vs per-candidate slope).

  python tools/gpu/probe_scaling.py [c2|c3|c4] [cands ...]
Times score_orders_argmin_d with CUDA events (median of 20 launches, inputs in HBM).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2210_12924_b200 as mp  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
cands = [int(x) for x in sys.argv[2:]] or [148, 296, 592, 1184, 2368, 4096, 8192, 16384]
g = bench.load_graph(cfg)
p = mp.Planner(0)
dg = p.upload(g)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
p.set_stream(st.cuda_stream)
Cmax = max(cands)
orders = torch.from_numpy(mp.random_topo_orders(g, Cmax, seed=5)).cuda()
peak = torch.zeros(Cmax, dtype=torch.int64, device="cuda")
step = torch.zeros(Cmax, dtype=torch.int32, device="cuda")
valid = torch.zeros(Cmax, dtype=torch.uint8, device="cuda")
key = torch.zeros(1, dtype=torch.int64, device="cuda")
print("info", dg.info(), "env", {k: v for k, v in os.environ.items() if k.startswith("MP_")})
for C in cands:
    ts = []
    for r in range(25):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        p.score_orders_argmin_d(dg, orders, C, peak, step, valid, key, 0, st.cuda_stream)
        b.record(st)
        b.synchronize()
        if r >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    t = float(np.median(ts))
    print(f"C={C:6d}  {t:8.2f} us  {t / C * 1e3:7.2f} ns/cand  {C / t * 1e6:.3g} plans/s")
