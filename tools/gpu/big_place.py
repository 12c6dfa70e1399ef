import sys, time, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'oracle'))
import numpy as np, torch, paper_2210_12924_b200 as mp, bench
cfg = bench.CONFIGS['c5']
g = bench.load_graph(cfg)
p = mp.Planner(0)
lo, hi = p.lifetimes_from_order(g, g.program_order())
for pyr in (True, False):
    for rep in range(2):
        t = time.time()
        addr, has, peak, base = p.place_batch(g, lo[None], hi[None], pyramid=pyr)
        print('c5 E', g.E, 'pyramid' if pyr else 'plain', 'one problem', round(time.time() - t, 3), 's peak', int(peak[0]), flush=True)
    ok = p.addresses_feasible(g, lo, hi, {int(e): int(addr[0, e]) for e in np.nonzero(has[0])[0]})
    print('feasible', ok, flush=True)
os.makedirs("gpurun_out", exist_ok=True); np.save("gpurun_out/c5_greedy_addr.npy", addr[0]); np.save("gpurun_out/c5_greedy_has.npy", has[0])
B = 148
LO = np.repeat(lo[None], B, 0); HI = np.repeat(hi[None], B, 0)
t = time.time()
addr, has, peak, base = p.place_batch(g, LO, HI, pyramid=False)
print('c5 148 problems', round(time.time() - t, 3), 's', flush=True)
