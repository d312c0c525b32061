#!/usr/bin/env python
"""Run the BASELINE.json configurations that fit one B200 and record what happened.

    python tools/run_configs.py [--out gpurun_out/configs_r1.json] [--skip 5]

config 1  n=10 000 2-D, exponential_isotropic, m=30, full Fisher-scoring fit (vs the reference's recorded fit)
config 2  n=2^20 2-D, matern15_isotropic, m=30: one evaluation                      (bench.py is the official line)
config 3  n=2^22 synthetic satellite swath (lon, lat, time), exponential_spacetime, m=30, full fit, 1 GPU
config 4  m in {10,20,30,40,60} at n=2^20, matern15_isotropic: evaluation time per m
config 5  n=2^24 3-D, matern15_isotropic, p=4 (intercept + coordinates), m=30: one evaluation on 1 GPU
Synthetic responses are random-Fourier-feature draws of the matching exponential-type field (cheap at
any n; the arithmetic under test does not depend on the data).
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2407_02740_b200 as vg  # noqa: E402
from paper_2407_02740_b200 import engine  # noqa: E402


def rff_field(locs, ranges, sigma2, nugget, seed, features=256):
    """Approximate draw of a GP with covariance sigma2*exp(-||delta/ranges||) + nugget*sigma2*I."""
    rng = np.random.default_rng(seed)
    n, d = locs.shape
    z = rng.normal(size=(features, d))
    g = rng.chisquare(1, size=(features, 1))
    w = z / np.sqrt(g) / np.asarray(ranges)[None, :]          # multivariate Cauchy frequencies
    b = rng.uniform(0, 2 * np.pi, features)
    y = np.empty(n)
    for r0 in range(0, n, 1 << 18):                           # row blocks bound the temporaries at n = 2^24
        blk = locs[r0:r0 + (1 << 18)]
        y[r0:r0 + blk.shape[0]] = np.cos(blk @ w.T + b).sum(axis=1)
    y *= np.sqrt(2.0 * sigma2 / features)
    return y + rng.normal(scale=np.sqrt(nugget * sigma2), size=n)


def timed_eval(prob, theta, reps=5):
    prob.enable_timing(True)
    ms = []
    for _ in range(reps + 2):
        prob.totals(theta)
        ms.append(prob.last_kernel_ms())
    return float(np.median(ms[2:]))


def config1():
    z = np.load(ROOT / "tests" / "golden" / "config1.npz")
    n, m, seed = 10_000, int(z["m"]), int(z["seed"])
    rng = np.random.default_rng(seed)
    locs = rng.uniform(0.0, 1.0, (n, 2))[vg.random_permutation(n, seed).perm]
    t0 = time.perf_counter()
    nn = vg.find_ordered_neighbors(locs, m, method="grid")
    t_nn = time.perf_counter() - t0
    ds = vg.Dataset(z["y"], np.ones((n, 1)), locs)
    start = vg.default_start(ds, "exponential_isotropic")
    t0 = time.perf_counter()
    res = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=m))
    wall = time.perf_counter() - t0
    engine.clear_cache()
    return {"n": n, "m": m, "family": "exponential_isotropic", "neighbor_search_s": t_nn, "fit_wall_s": wall,
            "iterations": res.iterations, "evaluations": len(res.loglik_trace), "converged": bool(res.converged),
            "theta_hat": res.theta_hat.theta.tolist(), "loglik": res.loglik,
            "reference_theta_hat": z["fit/theta_hat"].tolist(), "reference_loglik": float(z["fit/trace"][-1]),
            "max_rel_theta_error": float(np.max(np.abs(res.theta_hat.theta / z["fit/theta_hat"] - 1.0))),
            "phase_timings_ms": res.phase_timings}


def config2_and_4(ms_list=(10, 20, 30, 40, 60)):
    n = 1 << 20
    rng = np.random.default_rng(2407)
    locs = rng.uniform(0.0, 1.0, (n, 2))
    y = rng.normal(size=n)
    ds = vg.Dataset(y, np.ones((n, 1)), locs)
    theta = np.array([1.0, 0.05, 0.1])
    out = {}
    for m in ms_list:
        nn = vg.find_ordered_neighbors(locs, m)
        with engine.DeviceProblem(ds, nn, "matern15_isotropic") as prob:
            ms = timed_eval(prob, theta)
            out[f"m={m}"] = {"kernel_ms": ms, "obs_per_s": n / ms * 1e3, "kernel": prob.last_kernel_name}
    return out


def config3(n=1 << 22, m=30):
    """Synthetic swath: a satellite ground track (lat oscillates, lon advances) sampled along time."""
    rng = np.random.default_rng(33)
    t = np.sort(rng.uniform(0.0, 10.0, n))                     # days
    orbit = 0.07                                               # ~14 orbits per day
    lat = 60.0 * np.sin(2 * np.pi * t / orbit) + rng.normal(scale=0.3, size=n)
    lon = (360.0 * t / orbit * 0.93 + rng.normal(scale=0.3, size=n)) % 360.0 - 180.0
    locs = np.column_stack([lon, lat, t])
    perm = vg.random_permutation(n, 7).perm
    locs = locs[perm]
    true_ranges = [25.0, 25.0, 0.5]
    y = 1.5 + rff_field(locs, true_ranges, 2.0, 0.1, 5)
    ds = vg.Dataset(y, np.ones((n, 1)), locs)
    t0 = time.perf_counter()
    nn = vg.find_ordered_neighbors(locs, m)
    t_nn = time.perf_counter() - t0
    start = vg.default_start(ds, "exponential_spacetime")
    t0 = time.perf_counter()
    res = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=m))
    wall = time.perf_counter() - t0
    with engine.DeviceProblem(ds, nn, "exponential_spacetime") as prob:
        ms = timed_eval(prob, res.theta_hat.theta, reps=3)
    engine.clear_cache()
    return {"n": n, "m": m, "family": "exponential_spacetime", "neighbor_search_s": t_nn, "fit_wall_s": wall,
            "iterations": res.iterations, "evaluations_accepted": len(res.loglik_trace), "converged": bool(res.converged),
            "theta_start": start.theta.tolist(), "theta_hat": res.theta_hat.theta.tolist(),
            "theta_simulated": [2.0, 25.0, 0.5, 0.1], "beta_hat": res.beta_hat.tolist(), "loglik": res.loglik,
            "kernel_ms_per_evaluation": ms, "obs_per_s": n / ms * 1e3, "phase_timings_ms": res.phase_timings}


def config5(n=1 << 24, m=30):
    rng = np.random.default_rng(55)
    locs = rng.uniform(0.0, 1.0, (n, 3))
    X = np.column_stack([np.ones(n), locs])
    y = X @ np.array([0.5, 1.0, -1.0, 0.3]) + rff_field(locs, [0.05, 0.05, 0.05], 1.0, 0.1, 9, features=128)
    ds = vg.Dataset(y, X, locs)
    t0 = time.perf_counter()
    nn = vg.find_ordered_neighbors(locs, m)
    t_nn = time.perf_counter() - t0
    theta = np.array([1.0, 0.05, 0.1])
    t0 = time.perf_counter()
    with engine.DeviceProblem(ds, nn, "matern15_isotropic") as prob:
        first = prob.totals(theta)
        t_first = time.perf_counter() - t0
        ms = timed_eval(prob, theta, reps=3)
        ev = vg.assemble(engine.parts_from_flat(first, 4, 3), n)
        name = prob.last_kernel_name
    return {"n": n, "m": m, "family": "matern15_isotropic", "p": 4, "d": 3, "neighbor_search_s": t_nn,
            "upload_plus_first_evaluation_s": t_first, "kernel_ms_per_evaluation": ms, "obs_per_s": n / ms * 1e3,
            "kernel": name, "loglik": ev.loglik, "beta_hat": ev.beta_hat.tolist(), "grad": ev.grad.tolist(),
            "note": "single B200 (the 8-GPU run shards these rows 8 ways; see distributed.py)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "configs_r1.json"))
    ap.add_argument("--skip", type=int, nargs="*", default=[])
    args = ap.parse_args()
    out = {}
    for k, fn in ((1, config1), (2, config2_and_4), (3, config3), (5, config5)):
        if k in args.skip:
            continue
        t0 = time.perf_counter()
        try:
            out[f"config{k}" if k != 2 else "config2_and_4"] = fn()
        except Exception as err:  # noqa: BLE001 - record and continue
            out[f"config{k}"] = {"error": repr(err)}
        print(f"config {k}: {time.perf_counter() - t0:.1f} s", flush=True)
        Path(args.out).parent.mkdir(exist_ok=True)
        Path(args.out).write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
