"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container only (needs /root/reference; the GPU box has no
reference tree, it only reads the committed .npz/.json files):

    python tests/golden/make_golden.py

The reference package is imported straight from /root/reference/pkg/src (its
numpy "fallback" core needs no build).  When a scratch build of its compiled
core exists (REF_BUILD, default /tmp/refbuild/pkg/src -- made with
`CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" python setup.py build_ext
--inplace` on a copy of pkg/), the compiled core's outputs are stored too.

Files written
  engine_cases.npz   inputs + reference engine.run totals (both cores) for a set
                     of small seeded instances (families, p, d, ragged heads,
                     jitter, wide rows), + assemble() outputs
  failure_cases.npz  coincident-location instance and the reported observation
  neighbors.npz      ordered-neighbor tables incl. exact-tie grids
  fit_cases.npz      full Fisher-scoring fits (theta_hat, trace, iterations, ...)
  config1.npz        BASELINE config 1 (n=10 000, m=30): y + reference results
  krige_cases.npz    nearest-neighbour kriging (predict.krige) means / sds, noisy and latent
  simulate_cases.npz oracle.simulate_nn_gp draws (sequential conditional simulation), incl. ragged head,
                     p = 2, anisotropic d = 3 and a zero-nugget case
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_BUILD = os.environ.get("REF_BUILD", "/tmp/refbuild/pkg/src")
sys.path.insert(0, REF_BUILD if os.path.isdir(REF_BUILD) else REF_SRC)

import vecchiagp  # noqa: E402
from vecchiagp import (CovarianceParameters, Dataset, ModelSpec, engine,  # noqa: E402
                       find_ordered_neighbors, oracle, random_permutation, reorder_dataset)
from vecchiagp.covariance import covariance_registry  # noqa: E402
from vecchiagp.errors import NotPositiveDefinite  # noqa: E402
from vecchiagp.inference import assemble, default_start, evaluate, fit  # noqa: E402

OUT = Path(__file__).resolve().parent
CORES = engine.available_cores()
print("reference cores available:", CORES, "from", vecchiagp.__file__)


def flat(parts):
    return np.concatenate([np.atleast_1d(np.asarray(x, dtype=np.float64)).ravel() for x in (
        parts.logdet, parts.ysy, parts.xsx, parts.ysx, parts.dlogdet, parts.dysy, parts.dysx,
        parts.dxsx, parts.ainfo)])


def make_instance(seed, n, d, p, family, theta):
    """Same recipe as the reference's tests/conftest.py:15-38."""
    rng = np.random.default_rng(seed)
    if family == "exponential_sphere":
        lon = rng.uniform(-180.0, 180.0, n)
        lat = np.degrees(np.arcsin(rng.uniform(-1.0, 1.0, n)))
        locs = np.column_stack([lon, lat])
    else:
        locs = rng.uniform(0.0, 1.0, (n, d))
    X = np.ones((n, p))
    if p > 1:
        X[:, 1:] = rng.normal(size=(n, p - 1))
    cov = CovarianceParameters(family, np.asarray(theta, dtype=np.float64))
    beta = rng.normal(size=p)
    y = oracle.simulate_gp(cov, beta, locs, X, seed=seed + 1)
    return Dataset(y=y, X=X, locs=locs), cov


def engine_cases():
    specs = [
        # name, seed, n, d, p, family, theta, m, jitter
        ("iso_d2_p2_m9", 20, 60, 2, 2, "exponential_isotropic", [1.5, 0.25, 0.1], 9, 0.0),
        ("iso_d2_p1_m30", 21, 200, 2, 1, "exponential_isotropic", [2.0, 0.2, 0.1], 30, 0.0),
        ("iso_d3_p4_m30", 22, 150, 3, 4, "exponential_isotropic", [0.8, 0.4, 0.05], 30, 0.0),
        ("aniso_d3_p2_m8", 23, 70, 3, 2, "exponential_anisotropic", [1.5, 0.2, 0.35, 0.5, 0.1], 8, 0.0),
        ("aniso_d2_p1_m20", 24, 120, 2, 1, "exponential_anisotropic", [1.1, 0.15, 0.45, 0.2], 20, 0.0),
        ("sphere_p1_m12", 25, 90, 2, 1, "exponential_sphere", [1.5, 0.3, 0.1], 12, 0.0),
        ("iso_jitter", 26, 50, 2, 1, "exponential_isotropic", [1.0, 0.3, 0.0], 6, 1e-3),
        ("iso_heads_only", 27, 8, 2, 2, "exponential_isotropic", [1.3, 0.5, 0.2], 7, 0.0),
        ("iso_wide_m79", 28, 80, 2, 1, "exponential_isotropic", [1.5, 0.25, 0.1], 79, 0.0),
        ("iso_zero_nugget", 29, 64, 2, 1, "exponential_isotropic", [1.0, 0.1, 0.0], 10, 0.0),
        ("iso_d1_m5", 30, 40, 1, 1, "exponential_isotropic", [1.0, 0.2, 0.3], 5, 0.0),
        ("iso_m60", 31, 130, 2, 1, "exponential_isotropic", [1.0, 0.3, 0.1], 60, 0.0),
    ]
    out = {"names": np.array([s[0] for s in specs])}
    for name, seed, n, d, p, family, theta, m, jitter in specs:
        ds, cov = make_instance(seed, n, d, p, family, theta)
        work = covariance_registry(family).prepare_locs(ds.locs)
        nn = find_ordered_neighbors(work, m)
        out[f"{name}/y"] = ds.y
        out[f"{name}/X"] = ds.X
        out[f"{name}/locs"] = ds.locs
        out[f"{name}/locs_work"] = work
        out[f"{name}/nn"] = nn.idx
        out[f"{name}/theta"] = cov.theta
        out[f"{name}/family"] = np.array(family)
        out[f"{name}/jitter"] = np.array(jitter)
        for core in CORES:
            parts = engine.run(ds, nn, cov, backend="task", deterministic=True, jitter=jitter, core=core)
            out[f"{name}/totals_{core}"] = flat(parts)
            ev = assemble(parts, ds.n)
            out[f"{name}/loglik_{core}"] = np.array(ev.loglik)
            out[f"{name}/grad_{core}"] = ev.grad
            out[f"{name}/beta_{core}"] = ev.beta_hat
        # per-observation rows from the numpy core (reference process_observation)
        rows = np.stack([flat(engine.process_observation(i, ds, nn, cov, jitter=jitter))
                         for i in range(min(ds.n, 40))])
        out[f"{name}/rows_fallback"] = rows
    np.savez_compressed(OUT / "engine_cases.npz", **out)
    print("engine_cases.npz:", len(specs), "cases")


def failure_cases():
    # reference tests/test_engine.py:230-243: duplicated location, zero nugget
    rng = np.random.default_rng(6)
    locs = rng.uniform(0, 1, (12, 2))
    locs[7] = locs[3]
    y = rng.normal(size=12)
    ds = Dataset(y=y, X=np.ones((12, 1)), locs=locs)
    nn = find_ordered_neighbors(locs, 5)
    cov = CovarianceParameters("exponential_isotropic", [1.0, 0.3, 0.0])
    rec = {}
    for core in CORES:
        try:
            engine.run(ds, nn, cov, core=core)
            raise AssertionError("expected NotPositiveDefinite")
        except NotPositiveDefinite as err:
            rec[f"observation_{core}"] = np.array(err.observation)
            rec[f"pivot_{core}"] = np.array(err.pivot)
    rescued = engine.run(ds, nn, cov, jitter=1e-6)
    np.savez_compressed(OUT / "failure_cases.npz", y=y, locs=locs, nn=nn.idx, theta=cov.theta,
                        rescued_totals=flat(rescued), **rec)
    print("failure_cases.npz:", {k: int(v) for k, v in rec.items()})


def neighbor_cases():
    out = {}
    xs, ys = np.meshgrid(np.arange(7.0), np.arange(7.0))
    grid = np.column_stack([xs.ravel(), ys.ravel()])
    out["grid7/locs"], out["grid7/m"] = grid, np.array(8)
    g3 = np.stack(np.meshgrid(np.arange(5.0), np.arange(5.0), np.arange(4.0)), -1).reshape(-1, 3)
    g3 = g3[random_permutation(g3.shape[0], 11).perm]
    out["grid3d/locs"], out["grid3d/m"] = g3, np.array(10)
    rng = np.random.default_rng(3)
    out["rand2d/locs"], out["rand2d/m"] = rng.uniform(0, 1, (400, 2)), np.array(30)
    out["rand3d/locs"], out["rand3d/m"] = rng.uniform(0, 1, (300, 3)), np.array(7)
    out["line/locs"], out["line/m"] = np.arange(5.0)[:, None], np.array(2)
    dup = rng.uniform(0, 1, (60, 2))
    dup[10:20] = dup[0:10]
    out["dups/locs"], out["dups/m"] = dup, np.array(6)
    for name in ("grid7", "grid3d", "rand2d", "rand3d", "line", "dups"):
        out[f"{name}/idx"] = find_ordered_neighbors(out[f"{name}/locs"], int(out[f"{name}/m"])).idx
    np.savez_compressed(OUT / "neighbors.npz", **out)
    print("neighbors.npz written")


def _fit_record(res):
    return {
        "theta_hat": res.theta_hat.theta, "beta_hat": res.beta_hat, "beta_cov": res.beta_cov,
        "trace": np.asarray(res.loglik_trace), "fisher_info": res.fisher_info,
        "iterations": np.array(res.iterations), "converged": np.array(res.converged),
    }


def fit_cases():
    out = {}
    # (i) the recorded CLI golden (pkg/test_output.txt:36): simulate --n 300 --d 2
    #     --theta 2.0,0.2,0.1 --beta 1.0 --seed 8 ; fit --m 10 --seed 3 --deterministic
    for tag, sim_seed, m, fit_seed in (("cli300_a", 8, 10, 3), ("cli300_b", 4, 8, 1)):
        cov = CovarianceParameters("exponential_isotropic", [2.0, 0.2, 0.1])
        rng = np.random.Generator(np.random.PCG64(sim_seed))
        locs = rng.uniform(0.0, 1.0, (300, 2))
        X = np.ones((300, 1))
        y = oracle.simulate_gp(cov, np.array([1.0]), locs, X, sim_seed)
        ds = reorder_dataset(Dataset(y=y, X=X, locs=locs), random_permutation(300, fit_seed))
        nn = find_ordered_neighbors(ds.locs, m)
        start = default_start(ds, "exponential_isotropic")
        out[f"{tag}/y"], out[f"{tag}/X"], out[f"{tag}/locs"] = ds.y, ds.X, ds.locs
        out[f"{tag}/nn"], out[f"{tag}/start"], out[f"{tag}/m"] = nn.idx, start.theta, np.array(m)
        out[f"{tag}/family"] = np.array("exponential_isotropic")
        for core in CORES:
            res = fit(ds, nn, ModelSpec(covariance=start, m=m), deterministic=True, core=core)
            for k, v in _fit_record(res).items():
                out[f"{tag}/{core}/{k}"] = v
        print(tag, "loglik", res.loglik, "iters", res.iterations, "theta", res.theta_hat.theta)
    # (ii) anisotropic d=3, p=2
    ds, cov = make_instance(77, 400, 3, 2, "exponential_anisotropic", [1.2, 0.3, 0.2, 0.4, 0.15])
    nn = find_ordered_neighbors(ds.locs, 12)
    start = default_start(ds, "exponential_anisotropic")
    tag = "aniso400"
    out[f"{tag}/y"], out[f"{tag}/X"], out[f"{tag}/locs"] = ds.y, ds.X, ds.locs
    out[f"{tag}/nn"], out[f"{tag}/start"], out[f"{tag}/m"] = nn.idx, start.theta, np.array(12)
    out[f"{tag}/family"] = np.array("exponential_anisotropic")
    for core in CORES:
        res = fit(ds, nn, ModelSpec(covariance=start, m=12), deterministic=True, core=core)
        for k, v in _fit_record(res).items():
            out[f"{tag}/{core}/{k}"] = v
    print(tag, "loglik", res.loglik, "iters", res.iterations, "theta", res.theta_hat.theta)
    np.savez_compressed(OUT / "fit_cases.npz", **out)


def config1():
    """BASELINE.json configs[0]: n=10 000 2-D, exponential_isotropic, m=30, full fit.

    locs ~ U[0,1]^2 from default_rng(seed); X = ones; random_permutation ordering
    (the reference has no maxmin ordering); y from
    simulate_nn_gp with theta* = (2.0, 0.2*sqrt(2), 0.1) as in the reference's
    acceptance criterion 5 (tests/test_acceptance.py:170-176).  Only y and the
    reference's outputs are stored; locs/ordering/nn are regenerated by the test.
    """
    n, m, seed = 10_000, 30, 1234
    rng = np.random.default_rng(seed)
    locs = rng.uniform(0.0, 1.0, (n, 2))
    perm = random_permutation(n, seed).perm
    locs = locs[perm]
    X = np.ones((n, 1))
    nn = find_ordered_neighbors(locs, m)
    cov = CovarianceParameters("exponential_isotropic", [2.0, 0.2 * np.sqrt(2.0), 0.1])
    y = oracle.simulate_nn_gp(cov, np.array([0.5]), locs, X, nn, seed + 1)
    ds = Dataset(y=y, X=X, locs=locs)
    start = default_start(ds, "exponential_isotropic")
    out = {"y": y, "seed": np.array(seed), "m": np.array(m), "start": start.theta,
           "nn_checksum": np.array(int(nn.idx.sum())), "nn_row_9999": nn.idx[9999]}
    core = "compiled" if "compiled" in CORES else "fallback"
    parts0 = engine.run(ds, nn, start, deterministic=True, core=core)
    ev0 = assemble(parts0, n)
    out["totals_start"] = flat(parts0)
    out["loglik_start"], out["grad_start"], out["info_start"] = np.array(ev0.loglik), ev0.grad, ev0.info
    res = fit(ds, nn, ModelSpec(covariance=start, m=m), deterministic=True, core=core)
    for k, v in _fit_record(res).items():
        out[f"fit/{k}"] = v
    out["core"] = np.array(core)
    np.savez_compressed(OUT / "config1.npz", **out)
    print("config1: loglik", res.loglik, "iters", res.iterations, "theta", res.theta_hat.theta)


def krige_cases():
    """Nearest-neighbour kriging outputs of the unmodified reference (predict.py:35-90)."""
    from vecchiagp.model import FitResult
    from vecchiagp.predict import krige
    out = {}
    specs = [("iso_m10", 31, 300, 2, 2, "exponential_isotropic", [1.5, 0.25, 0.1], 10, 40),
             ("iso_m60", 32, 400, 2, 1, "exponential_isotropic", [2.0, 0.2, 0.1], 60, 50),
             ("aniso_m20", 33, 250, 3, 2, "exponential_anisotropic", [1.2, 0.3, 0.2, 0.4, 0.15], 20, 30),
             ("sphere_m15", 34, 200, 2, 1, "exponential_sphere", [1.5, 0.3, 0.1], 15, 25),
             ("iso_all", 35, 30, 2, 1, "exponential_isotropic", [1.0, 0.4, 0.05], 30, 10)]
    for name, seed, n, d, p, family, theta, m_pred, npred in specs:
        ds, cov = make_instance(seed, n, d, p, family, theta)
        rng = np.random.default_rng(seed + 100)
        if family == "exponential_sphere":
            star = np.column_stack([rng.uniform(-180, 180, npred), np.degrees(np.arcsin(rng.uniform(-1, 1, npred)))])
        else:
            star = rng.uniform(0.0, 1.0, (npred, d))
        star[0] = ds.locs[5]  # one prediction point coincides with a training point
        Xs = np.ones((npred, p))
        if p > 1:
            Xs[:, 1:] = rng.normal(size=(npred, p - 1))
        beta = rng.normal(size=p)
        fr = FitResult(theta_hat=cov, beta_hat=beta, beta_cov=np.eye(p), loglik_trace=[0.0], fisher_info=np.eye(3),
                       iterations=0, converged=True)
        out[f"{name}/y"], out[f"{name}/X"], out[f"{name}/locs"] = ds.y, ds.X, ds.locs
        out[f"{name}/theta"], out[f"{name}/family"], out[f"{name}/beta"] = cov.theta, np.array(family), beta
        out[f"{name}/locs_star"], out[f"{name}/X_star"], out[f"{name}/m_pred"] = star, Xs, np.array(m_pred)
        for latent in (False, True):
            ps = krige(fr, ds, star, Xs, m_pred=m_pred, latent=latent, with_sd=True)
            out[f"{name}/mean_latent{int(latent)}"] = ps.mean
            out[f"{name}/sd_latent{int(latent)}"] = ps.sd
    out["names"] = np.array([s[0] for s in specs])
    np.savez_compressed(OUT / "krige_cases.npz", **out)
    print("krige_cases.npz:", len(specs), "cases")


def simulate_cases():
    """oracle.simulate_nn_gp (oracle.py:102-140) on small seeded instances."""
    specs = [("iso_d2_m10", "exponential_isotropic", 2, 1, 10, 600, [1.7, 0.15, 0.05]),
             ("iso_d2_m30", "exponential_isotropic", 2, 1, 30, 900, [0.8, 0.3, 0.2]),
             ("iso_d2_p2_m5", "exponential_isotropic", 2, 2, 5, 300, [1.2, 0.1, 0.0]),
             ("aniso_d3_m12", "exponential_anisotropic", 3, 1, 12, 500, [2.0, 0.3, 0.15, 0.5, 0.1])]
    out = {}
    for k, (name, family, d, p, m, n, theta) in enumerate(specs):
        rng = np.random.default_rng(4000 + k)
        locs = rng.uniform(0.0, 1.0, (n, d))
        X = np.ones((n, p))
        if p > 1:
            X[:, 1:] = rng.normal(size=(n, p - 1))
        beta = rng.normal(size=p)
        cov = CovarianceParameters(family, np.array(theta))
        nn = find_ordered_neighbors(locs, m)
        seed = 77 + k
        y = oracle.simulate_nn_gp(cov, beta, locs, X, nn, seed)
        out[f"{name}/locs"], out[f"{name}/X"], out[f"{name}/beta"] = locs, X, beta
        out[f"{name}/theta"], out[f"{name}/family"], out[f"{name}/m"] = cov.theta, np.array(family), np.array(m)
        out[f"{name}/seed"], out[f"{name}/y"], out[f"{name}/nn"] = np.array(seed), y, nn.idx
    out["names"] = np.array([s[0] for s in specs])
    np.savez_compressed(OUT / "simulate_cases.npz", **out)
    print("simulate_cases.npz:", len(specs), "cases")


if __name__ == "__main__":
    if "--krige-only" in sys.argv:
        krige_cases()
        sys.exit(0)
    if "--simulate-only" in sys.argv:
        simulate_cases()
        sys.exit(0)
    engine_cases()
    failure_cases()
    neighbor_cases()
    fit_cases()
    config1()
    krige_cases()
    simulate_cases()
