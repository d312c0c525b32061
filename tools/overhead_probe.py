"""Fixed cost of one evaluation outside the kernel: wall time of DeviceProblem.totals() minus the CUDA-event kernel time,
at a shard small enough that the kernel is short."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import engine
import bench
for n in (4096, 131072):
    y, X, locs = bench.make_workload(n, 2, 1)
    nn = vg.find_ordered_neighbors(locs, 30)
    th = np.array([1.0, 0.05, 0.1])
    with engine.DeviceProblem(vg.Dataset(y, X, locs), nn, "matern15_isotropic") as prob:
        for timing in (False, True):
            prob.enable_timing(timing)
            for _ in range(20):
                prob.totals(th)
            t0 = time.perf_counter()
            reps = 200
            km = 0.0
            for _ in range(reps):
                prob.totals(th)
                if timing:
                    km += prob.last_kernel_ms()
            wall = (time.perf_counter() - t0) / reps * 1e3
            print(f"n={n} timing_events={timing}: wall {wall*1e3:.1f} us per evaluation" + (f", kernel {km/reps*1e3:.1f} us, overhead {(wall-km/reps)*1e3:.1f} us" if timing else ""))
