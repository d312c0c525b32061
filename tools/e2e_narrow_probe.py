#!/usr/bin/env python
"""End-to-end step (pinned host arrays -> DeviceProblem -> totals) with the int64 neighbor table shipped as is
against the narrowed (int32 over PCIe, widened on the device) upload, for several chunk counts; plus the host
narrowing rate alone.

    python tools/e2e_narrow_probe.py [--n 1048576] [--m 30]
"""
import argparse, json, sys, time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--steps", type=int, default=12)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2407_02740_b200 as vg
    from paper_2407_02740_b200 import engine
    from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows, host_library

    y, X, locs = bench.make_workload(a.n, 2, 1)
    nn = find_ordered_neighbor_rows(locs, a.m, 0, a.n)
    pin = lambda v: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
    hy, hX, hl, hn = pin(y), pin(X), pin(locs), pin(nn)
    ds = vg.Dataset(hy.numpy(), hX.numpy(), hl.numpy())
    table = vg.NeighborArray(hn.numpy())
    theta = np.array([1.0, 0.05, 0.1])
    out = {}
    lib = host_library()
    dst = torch.empty(nn.size, dtype=torch.int32).pin_memory()
    for workers in (0, 4, 8):
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            lib.vbh_narrow_indices(hn.numpy().ctypes.data, dst.data_ptr(), nn.size, workers)
            ts.append(time.perf_counter() - t0)
        out[f"narrow_ms_workers{workers}"] = 1e3 * min(ts)
    out["host_threads"] = int(lib.vbh_max_threads())
    ref = None
    for narrow in (False, True):
        for chunks in (8, 16, 32):
            each = []
            for it in range(a.steps + 2):
                t0 = time.perf_counter()
                with engine.DeviceProblem(ds, table, "matern15_isotropic", upload_chunks=chunks,
                                          upload_narrow=narrow) as prob:
                    tot = prob.totals(theta)
                each.append(1e3 * (time.perf_counter() - t0))
            ref = ref or {}
            if chunks not in ref:
                ref[chunks] = tot  # the chunking fixes the summation order: compare like with like
            assert np.array_equal(tot, ref[chunks]), "narrowed upload changed the totals"
            each = each[2:]
            out[f"e2e_ms_narrow{int(narrow)}_chunks{chunks}"] = {"mean": float(np.mean(each)), "min": float(min(each))}
            print(narrow, chunks, out[f"e2e_ms_narrow{int(narrow)}_chunks{chunks}"], flush=True)
    print("RESULT " + json.dumps(out))


if __name__ == "__main__":
    main()
