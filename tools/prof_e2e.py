import sys, time, cProfile, pstats
from pathlib import Path
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import engine
from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows
import bench
n, m = 1 << 20, 30
y, X, locs = bench.make_workload(n, 2, 1)
nn = find_ordered_neighbor_rows(locs, m, 0, n)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hy, hX, hl, hn = pin(y), pin(X), pin(locs), pin(nn)
ds = vg.Dataset(hy.numpy(), hX.numpy(), hl.numpy()); table = vg.NeighborArray(hn.numpy())
theta = np.array([1.0, 0.05, 0.1])
def one():
    with engine.DeviceProblem(ds, table, "matern15_isotropic") as prob:
        return prob.totals(theta)
for _ in range(3): one()
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0=time.perf_counter()
for _ in range(10): one()
t1=time.perf_counter()
pr.disable()
print("per step ms", 100*(t1-t0))
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
