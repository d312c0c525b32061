"""Where does the end-to-end (host arrays -> totals) time go?  Run on the GPU box."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
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
print("views pinned?", torch.from_numpy(table.idx).is_pinned(), torch.from_numpy(ds.y).is_pinned())
theta = np.array([1.0, 0.05, 0.1])
def sync(): torch.cuda.synchronize()
for chunks in (1, 8, 8, 16, 16, 32, 32, 64, 8):
    sync(); t0 = time.perf_counter()
    prob = engine.DeviceProblem(ds, table, "matern15_isotropic", upload_chunks=chunks); t1 = time.perf_counter()
    tot = prob.totals(theta); t2 = time.perf_counter()
    prob.close(); sync(); t3 = time.perf_counter()
    print(f"chunks {chunks}: create {1e3*(t1-t0):.2f} ms  eval {1e3*(t2-t1):.2f} ms  close {1e3*(t3-t2):.2f} ms  total {1e3*(t3-t0):.2f}")
