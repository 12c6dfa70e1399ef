"""One plain greedy_pack problem on a 9k-edge graph through the global-memory K5
variant (for an ncu capture of place_big_kernel)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_2210_12924_b200 as mp  # noqa: E402

g = mp.generate_graph("training_like", 3000, 8)
p = mp.Planner(0)
lo, hi = p.lifetimes_from_order(g, g.program_order())
addr, has, peak, _ = p.place_batch(g, lo[None], hi[None], pyramid=False)
print("E", g.E, "peak", int(peak[0]))
