"""C5 greedy_pack parity at full size (host side, slow): the C restatement of
greedy_pack (oracle/, placement.cpp:182-204) on one host thread against the GPU's
addresses saved by tools/gpu/big_place.py (plain greedy_pack of the program order's
lifetimes on the 100k-tensor graph). Writes the verdict and the host time as JSON.
usage: python tools/c5_greedy_check.py <dir with c5_greedy_addr.npy / c5_greedy_has.npy> <out.json>"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402

src, out = sys.argv[1], sys.argv[2]
g = bench.load_graph(bench.CONFIGS["c5"])
orc = O.Oracle.from_csr(g.csr())
lo, hi = orc.lifetimes_from_order(g.program_order())
t = time.time()
ea, eh = O.greedy_pack(lo, hi, g.edge_size)
dt = time.time() - t
ga = np.load(os.path.join(src, "c5_greedy_addr.npy"))
gh = np.load(os.path.join(src, "c5_greedy_has.npy"))
res = {"graph": "training_like L=33333 (n=133,336, E=100,002), program order",
       "has_equal": bool((gh == eh).all()), "addr_equal": bool((ga[eh == 1] == ea[eh == 1]).all()),
       "peak_mem": int(O.peak_mem(g.edge_size, eh, ea)),
       "host_greedy_pack_s_1_thread": round(dt, 1),
       "host": "the C restatement (oracle/memplan_oracle.c or_greedy_pack, -O2), 1 thread"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
