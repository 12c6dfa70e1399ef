"""Probe: where mp_joint_pairs' host call spends its time (count call vs fill call vs D2H)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2210_12924_b200 as mp  # noqa: E402
from paper_2210_12924_b200 import _native  # noqa: E402

for cfg in sys.argv[1:] or ["c4"]:
    g = bench.load_graph(bench.CONFIGS[cfg])
    p = mp.Planner(0)
    dg = p.upload(g)
    L = _native.lib()
    cnt = C.c_int64()
    L.mp_joint_pairs(p.ctx, dg.handle, 1, None, 0, C.byref(cnt))
    out = np.zeros((cnt.value, 2), np.int32)
    for _ in range(2):
        L.mp_joint_pairs(p.ctx, dg.handle, 1, out.ctypes.data, cnt.value, C.byref(cnt))
    t0 = time.perf_counter()
    for _ in range(5):
        L.mp_joint_pairs(p.ctx, dg.handle, 1, None, 0, C.byref(cnt))
    t_count = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    for _ in range(5):
        L.mp_joint_pairs(p.ctx, dg.handle, 1, out.ctypes.data, cnt.value, C.byref(cnt))
    t_fill = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    for _ in range(5):
        o2 = np.zeros((cnt.value, 2), np.int32)
    t_alloc = (time.perf_counter() - t0) / 5
    print(cfg, "pairs", cnt.value, "count call %.2f ms" % (t_count * 1e3),
          "fill call %.2f ms" % (t_fill * 1e3), "np.zeros %.2f ms" % (t_alloc * 1e3))
