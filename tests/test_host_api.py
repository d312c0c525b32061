"""CPU-side tests: host logic of the fitting API, the C ABI surface, and the multi-rank
combine step under gloo.  No compute call reaches the GPU library here."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import _cabi, build, distributed, engine, inference
from oracle import vecchia_oracle as vo

ROOT = Path(__file__).resolve().parent.parent


# ---- C ABI -------------------------------------------------------------------
def test_library_builds_and_exports_every_declared_symbol():
    lib_path = build.build_cuda()
    assert lib_path.exists()
    header = (ROOT / "include" / "vecchia_b200.h").read_text()
    declared = set(re.findall(r"\b(vb200_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations found"
    lib = ctypes.CDLL(str(lib_path))
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in include/vecchia_b200.h but not exported"
    assert set(_cabi.EXPORTED_SYMBOLS) == declared
    L = _cabi.load()
    assert L.vb200_abi_version() == 1
    assert L.vb200_acc_len(1, 3) == 25 and L.vb200_acc_len(4, 3) == 97 and L.vb200_acc_len(1, 4) == 36
    assert L.vb200_family_nparms(0, 2) == 3 and L.vb200_family_nparms(1, 3) == 5
    assert L.vb200_family_nparms(2, 3) == 4 and L.vb200_family_nparms(9, 2) < 0


def test_sass_is_sm100a_fp64():
    out = subprocess.run(["cuobjdump", "-lelf", str(build.build_cuda())], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(_cabi.device_count() > 0, reason="a GPU is present")
def test_no_cpu_fallback_without_device():
    ds = vg.Dataset(np.zeros(4), np.ones((4, 1)), np.arange(8.0).reshape(4, 2))
    nn = vg.find_ordered_neighbors(ds.locs, 2)
    with pytest.raises(vg.DeviceUnavailable):
        engine.run(ds, nn, vg.CovarianceParameters("exponential_isotropic", [1.0, 0.5, 0.1]))
    handle = ctypes.c_void_p()
    y = np.zeros(4)
    rc = _cabi.load().vb200_create(0, 4, 1, 2, 3, y.ctypes.data, y.ctypes.data, y.ctypes.data, y.ctypes.data, 0, 4,
                                   None, ctypes.byref(handle))
    assert rc == _cabi.VB200_ECUDA and "no CPU fallback" in _cabi.last_error()


def test_product_never_imports_the_oracle():
    for path in (ROOT / "paper_2407_02740_b200").rglob("*.py"):
        text = path.read_text()
        assert "import oracle" not in text and "from oracle" not in text, path
    for path in (ROOT / "paper_2407_02740_b200" / "csrc").rglob("*"):
        if path.is_file():
            assert "oracle" not in path.read_text().lower(), path


def test_every_baseline_shape_has_a_register_tiled_instance():
    """The instance registry (readable without a GPU) must cover the shapes BASELINE.json names -- exact-size
    instances for the neighbor-count sweep of config 4 -- so that none of them drops to the generic kernel."""
    inst = _cabi.tiled_instances()  # (lanes, rows_per_lane, cap, family_code, d, p); serves m+1 <= cap-1
    fam = {"exponential_isotropic": 0, "exponential_spacetime": 2, "matern15_isotropic": 3, "matern_isotropic": 5}

    def best_cap(family, d, p, m):
        caps = [c for (_, _, c, f, dd, pp) in inst if f == fam[family] and dd == d and pp == p and c - 1 >= m + 1]
        return min(caps) if caps else None

    assert best_cap("exponential_isotropic", 2, 1, 30) == 32                      # config 1
    for m, cap in ((10, 12), (15, 17), (20, 22), (25, 27), (30, 32), (40, 42), (50, 52), (60, 62)):
        assert best_cap("matern15_isotropic", 2, 1, m) == cap, m                  # configs 2 and 4 (+ m = 15, 25, 50)
    assert best_cap("matern_isotropic", 2, 1, 30) == 32                           # config 2 as literally named
    assert best_cap("exponential_spacetime", 3, 1, 30) == 32                      # config 3
    assert best_cap("matern15_isotropic", 3, 4, 30) == 32                         # config 5
    assert best_cap("matern15_isotropic", 2, 1, 62) == 64 and best_cap("matern15_isotropic", 2, 1, 63) is None


def test_host_index_narrowing():
    """vbh_narrow_indices: int64 -> int32 (the halved PCIe upload of the neighbor table), -1 padding kept, values
    that do not fit reported."""
    from paper_2407_02740_b200.preprocess import host_library
    lib = host_library()
    rng = np.random.default_rng(5)
    src = rng.integers(-1, 2 ** 31 - 1, size=100_003, dtype=np.int64)
    src[:7] = [-1, 0, 1, 2 ** 31 - 1, 12345, -1, 7]
    dst = np.empty(src.size, dtype=np.int32)
    for workers in (0, 1, 3):
        dst[:] = 99
        assert lib.vbh_narrow_indices(src.ctypes.data, dst.ctypes.data, src.size, workers) == 0
        assert np.array_equal(dst.astype(np.int64), src)
    assert lib.vbh_narrow_indices(src.ctypes.data, dst.ctypes.data, 0, 0) == 0
    big = src.copy()
    big[50_000] = 2 ** 31
    assert lib.vbh_narrow_indices(big.ctypes.data, dst.ctypes.data, big.size, 0) == 1
    assert lib.vbh_narrow_indices(None, dst.ctypes.data, 4, 0) == -1


# ---- model / covariance / preprocess ------------------------------------------
def test_model_types_and_validation():
    ds = vg.Dataset([1, 2, 3], [1, 1, 1], [[0, 0], [1, 0], [0, 1]])
    assert ds.n == 3 and ds.p == 1 and ds.d == 2 and ds.X.dtype == np.float64
    vg.validate_dataset(ds)
    with pytest.raises(vg.EmptyData):
        vg.validate_dataset(vg.Dataset([], np.zeros((0, 1)), np.zeros((0, 2))))
    with pytest.raises(vg.DimensionMismatch):
        vg.validate_dataset(vg.Dataset([1, 2], np.ones((3, 1)), np.zeros((3, 2))))
    with pytest.raises(vg.NonFiniteValue):
        vg.validate_dataset(vg.Dataset([1, np.nan], np.ones((2, 1)), np.zeros((2, 2))))
    assert vg.normalize_backend("seq") == "sequential" and vg.normalize_backend("staged-batched") == "staged"
    with pytest.raises(ValueError):
        vg.normalize_backend("gpu")
    with pytest.raises(ValueError):
        vg.ModelSpec(vg.CovarianceParameters("exponential_isotropic", [1, 1, 0]), m=0)
    assert engine.choose_capacity_tier(31) == 32 and engine.choose_capacity_tier(80) == 80
    assert engine.available_cores() == ("cuda",) and engine.active_core_name() == "cuda"


def test_covariance_registry_known_answers():
    # e^-1 entries (reference tests/test_covariance.py:26-30, 71-74)
    fam = vg.covariance_registry("exponential_isotropic")
    K = fam.matrix([2.0, 0.5, 0.1], [[0.0, 0.0], [0.5, 0.0]])
    assert K[0, 1] == pytest.approx(2.0 * np.exp(-1.0)) and K[0, 0] == pytest.approx(2.2)
    D = fam.derivatives([2.0, 0.5, 0.1], [[0.0, 0.0], [0.5, 0.0]])
    assert D[0][0, 1] == pytest.approx(np.exp(-1.0)) and D[1][0, 1] == pytest.approx(2 * np.exp(-1.0) * 0.5 / 0.25)
    assert np.array_equal(D[2], 2.0 * np.eye(2)) and D[1][0, 0] == 0.0
    with pytest.raises(vg.UnknownFamily):
        vg.covariance_registry("matern")
    with pytest.raises(ValueError):
        vg.validate_parameters(vg.CovarianceParameters("exponential_anisotropic", [1, 1, 0]), 2)
    with pytest.raises(ValueError):
        vg.validate_parameters(vg.CovarianceParameters("exponential_isotropic", [1, 0.0, 0]), 2)
    with pytest.raises(ValueError):
        vg.validate_parameters(vg.CovarianceParameters("exponential_isotropic", [1, 1, -0.1]), 2)
    assert vg.covariance_registry("exponential_spacetime").nparms(3) == 4
    assert vg.covariance_registry("exponential_anisotropic").nparms(3) == 5


@pytest.mark.parametrize("family,d,theta", [
    ("exponential_isotropic", 2, [1.3, 0.4, 0.2]), ("exponential_anisotropic", 3, [1.3, 0.4, 0.7, 0.2, 0.1]),
    ("exponential_spacetime", 3, [1.3, 0.4, 0.9, 0.1]), ("matern15_isotropic", 2, [0.9, 0.3, 0.05]),
    ("matern25_isotropic", 2, [0.9, 0.3, 0.05]), ("matern_isotropic", 2, [0.9, 0.3, 1.3, 0.05])])
def test_covariance_derivatives_vs_finite_differences(family, d, theta):
    from oracle import numpy_families
    rng = np.random.default_rng(1)
    pts = rng.uniform(0, 1, (7, d))
    fam = vg.covariance_registry(family)
    theta = np.asarray(theta)
    D = fam.derivatives(theta, pts)
    K0, D0 = numpy_families.cov_and_derivs(family, theta, pts)
    np.testing.assert_allclose(fam.matrix(theta, pts), K0, rtol=1e-13)
    # the smoothness derivative is a central difference of step 1e-5: rounding differences of the two
    # distance computations are amplified by 1e5 there
    np.testing.assert_allclose(D, D0, rtol=1e-8 if family == "matern_isotropic" else 1e-12, atol=1e-14)
    for j in range(theta.shape[0]):
        h = 1e-6 * theta[j]
        tp, tm = theta.copy(), theta.copy()
        tp[j] += h
        tm[j] -= h
        np.testing.assert_allclose(D[j], (fam.matrix(tp, pts) - fam.matrix(tm, pts)) / (2 * h), rtol=1e-6, atol=1e-8)


def test_sphere_embedding_and_orderings():
    xyz = vg.embed_lonlat([[0.0, 0.0], [90.0, 0.0], [0.0, 90.0]])
    np.testing.assert_allclose(xyz, [[1, 0, 0], [0, 1, 0], [0, 0, 1]], atol=1e-15)
    with pytest.raises(vg.LatitudeOutOfRange):
        vg.embed_lonlat([[0.0, 91.0]])
    with pytest.raises(vg.LatitudeOutOfRange):
        vg.lonlat_to_xyz(0.0, -90.5)
    perm = vg.random_permutation(10, 5).perm
    assert sorted(perm) == list(range(10))
    assert np.array_equal(perm, np.random.Generator(np.random.PCG64(5)).permutation(10))
    ds = vg.Dataset(np.arange(10.0), np.ones(10), np.arange(20.0).reshape(10, 2))
    re_ds = vg.reorder_dataset(ds, vg.Ordering(perm))
    assert np.array_equal(re_ds.y, ds.y[perm]) and np.array_equal(re_ds.locs, ds.locs[perm])
    with pytest.raises(vg.LengthMismatch):
        vg.reorder_dataset(ds, vg.identity_ordering(9))


@pytest.mark.parametrize("name", ["grid7", "grid3d", "rand2d", "rand3d", "line", "dups"])
@pytest.mark.parametrize("method", ["exhaustive", "grid"])
def test_neighbor_table_matches_reference_golden(neighbor_cases, name, method):
    z = neighbor_cases
    got = vg.find_ordered_neighbors(z[f"{name}/locs"], int(z[f"{name}/m"]), method=method)
    assert np.array_equal(got.idx, z[f"{name}/idx"])


def test_neighbor_grid_equals_exhaustive_scan_with_ties_and_row_ranges():
    from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows
    rng = np.random.default_rng(12)
    for n, d, m in [(6000, 2, 30), (5000, 3, 11), (4500, 1, 4), (5000, 5, 9)]:
        locs = rng.uniform(0, 1, (n, d))
        a = vg.find_ordered_neighbors(locs, m, method="exhaustive").idx
        assert np.array_equal(a, vo.neighbor_scan(locs, m))
        assert np.array_equal(a, vg.find_ordered_neighbors(locs, m, method="grid", workers=3).idx)
        assert np.array_equal(a[1000:3500], find_ordered_neighbor_rows(locs, m, 1000, 2500))
    xs, ys = np.meshgrid(np.arange(70.0), np.arange(70.0))
    g = np.column_stack([xs.ravel(), ys.ravel()])[rng.permutation(4900)]
    assert np.array_equal(vg.find_ordered_neighbors(g, 12, method="grid").idx, vo.neighbor_scan(g, 12))
    clustered = np.concatenate([rng.normal(0, 0.01, (3000, 2)), rng.uniform(-5, 5, (2500, 2))])[rng.permutation(5500)]
    assert np.array_equal(vg.find_ordered_neighbors(clustered, 20, method="grid").idx, vo.neighbor_scan(clustered, 20))
    tiny = vg.find_ordered_neighbors(np.array([[0.0], [1.0], [2.0], [3.0], [4.0]]), 2)
    assert np.array_equal(tiny.idx, [[0, -1, -1], [1, 0, -1], [2, 1, 0], [3, 2, 1], [4, 3, 2]])  # test_preprocess.py:124-136
    assert vg.find_ordered_neighbors(np.zeros((1, 2)), 5).idx.shape == (1, 2)


def test_nearest_training_query_equals_exhaustive_ranking():
    from paper_2407_02740_b200.preprocess import find_nearest_training
    rng = np.random.default_rng(5)
    for n, d, m, nq in [(5000, 2, 60, 200), (3000, 3, 20, 150), (900, 2, 10, 60), (4000, 1, 5, 80)]:
        train = rng.uniform(0, 1, (n, d))
        qs = rng.uniform(-0.3, 1.3, (nq, d))   # some queries outside the bounding box
        qs[0] = train[7]                         # a query on top of a training point
        got = find_nearest_training(train, qs, m, workers=3)
        for t in range(0, nq, 7):
            diff = train - qs[t]
            d2 = (diff * diff).sum(axis=1)
            want = np.lexsort((np.arange(n), d2))[:m]   # the reference's rule, predict.py:27-32
            assert np.array_equal(got[t], want)
    g = np.stack(np.meshgrid(np.arange(60.0), np.arange(60.0)), -1).reshape(-1, 2)
    got = find_nearest_training(g, g[::11], 12)          # exact ties on an integer grid
    for t, qpt in enumerate(g[::11]):
        d2 = ((g - qpt) ** 2).sum(axis=1)
        assert np.array_equal(got[t], np.lexsort((np.arange(len(g)), d2))[:12])
    with pytest.raises(ValueError):
        find_nearest_training(g, g[:2], 0)


def test_maxmin_ordering_equals_brute_force_greedy():
    def brute(locs):
        n = len(locs)
        first = int(np.argmin(((locs - locs.mean(axis=0)) ** 2).sum(1)))
        perm, dmin = [first], ((locs - locs[first]) ** 2).sum(1)
        dmin[first] = -1.0
        for _ in range(1, n):
            i = int(np.argmax(dmin))          # smallest index on ties
            perm.append(i)
            dmin = np.minimum(dmin, ((locs - locs[i]) ** 2).sum(1))
            dmin[perm] = -1.0
        return np.array(perm)

    rng = np.random.default_rng(0)
    for n, d in [(700, 2), (500, 3), (300, 1), (400, 4)]:
        locs = rng.uniform(0, 1, (n, d))
        assert np.array_equal(vg.maxmin_ordering(locs).perm, brute(locs))
    grid = np.stack(np.meshgrid(np.arange(15.0), np.arange(15.0)), -1).reshape(-1, 2)   # exact ties
    assert np.array_equal(vg.maxmin_ordering(grid).perm, brute(grid))
    assert vg.maxmin_ordering(np.zeros((1, 2))).perm.tolist() == [0]
    assert vg.ModelSpec(vg.CovarianceParameters("exponential_isotropic", [1, 1, 0]), m=5, ordering="maxmin").m == 5


def test_binary_formats_round_trip(tmp_path):
    from paper_2407_02740_b200 import io
    rng = np.random.default_rng(2)
    ds = vg.Dataset(rng.normal(size=50), rng.normal(size=(50, 2)), rng.uniform(size=(50, 3)))
    nn = vg.find_ordered_neighbors(ds.locs, 6)
    io.write_dataset_npz(ds, tmp_path / "d.npz")
    io.write_neighbors_npy(nn, tmp_path / "nn.npy")
    back = io.read_dataset_npz(tmp_path / "d.npz")
    assert np.array_equal(back.y, ds.y) and np.array_equal(back.X, ds.X) and np.array_equal(back.locs, ds.locs)
    assert np.array_equal(io.read_neighbors_npy(tmp_path / "nn.npy").idx, nn.idx)
    assert np.array_equal(io.read_neighbors_npy(tmp_path / "nn.npy", mmap=True).idx[10:20], nn.idx[10:20])
    fit = vg.FitResult(vg.CovarianceParameters("matern15_isotropic", [1.0, 0.1 + 1e-17, 0.3]), np.array([0.5, 1.0]),
                       np.eye(2), [-3.0, -2.5], np.eye(3), 4, True, {"fit_ms": 1.5})
    io.write_fit_json(fit, tmp_path / "f.json", config={"m": 6})
    doc = io.read_fit_json(tmp_path / "f.json")
    assert tuple(doc) == io.FIT_SCHEMA_KEYS          # the reference's schema, key for key (io.py:128-140)
    again = io.fit_from_dict(doc)
    assert np.array_equal(again.theta_hat.theta, fit.theta_hat.theta) and again.loglik == -2.5 and again.converged


# ---- inference -----------------------------------------------------------------
def test_fisher_step_known_answers():
    # reference tests/test_inference.py:84-115
    step = inference.fisher_step(np.zeros(2), np.array([1.0, 2.0]), np.diag([2.0, 4.0]))
    np.testing.assert_allclose(step, [0.5, 0.5])
    assert np.array_equal(inference.fisher_step(np.array([0.3, 0.4]), np.zeros(2), np.eye(2)), [0.3, 0.4])
    out = inference.fisher_step(np.zeros(2), np.array([1.0, 1.0]), np.zeros((2, 2)))  # needs damping
    assert np.all(np.isfinite(out)) and out @ np.array([1.0, 1.0]) > 0
    with pytest.raises(vg.DegenerateInformation):
        inference.fisher_step(np.zeros(2), np.array([1.0, 1.0]), -10.0 * np.eye(2))
    g, info = inference.to_log_scale([2.0, 0.5], np.array([1.0, 4.0]), np.array([[1.0, 2.0], [2.0, 8.0]]))
    np.testing.assert_allclose(g, [2.0, 2.0])
    np.testing.assert_allclose(info, [[4.0, 2.0], [2.0, 2.0]])


def test_assemble_on_reference_totals(engine_cases):
    for name in engine_cases["names"]:
        name = str(name)
        tot = engine_cases[f"{name}/totals_compiled"]
        p, q = engine_cases[f"{name}/X"].shape[1], engine_cases[f"{name}/theta"].shape[0]
        parts = engine.parts_from_flat(tot, p, q)
        assert np.array_equal(engine.flat_from_parts(parts), tot)
        ev = vg.assemble(parts, engine_cases[f"{name}/y"].shape[0])
        assert ev.loglik == pytest.approx(float(engine_cases[f"{name}/loglik_compiled"]), rel=1e-13)
        np.testing.assert_allclose(ev.grad, engine_cases[f"{name}/grad_compiled"], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(ev.beta_hat, engine_cases[f"{name}/beta_compiled"], rtol=1e-10)
    bad = engine.parts_from_flat(np.zeros(engine.acc_len(2, 3)), 2, 3)
    with pytest.raises(vg.SingularDesign):
        vg.assemble(bad, 10)


def test_fit_loop_with_cpu_evaluator_reproduces_reference_fit(fit_cases):
    """The scoring loop (host logic) driven by the ORACLE as evaluator must reproduce the
    reference's fit exactly -- separates fit-loop parity from kernel parity."""
    z, tag = fit_cases, "cli300_a"
    g = lambda k: z[f"{tag}/{k}"]
    ds = vg.Dataset(g("y"), g("X"), g("locs"))
    nn = vg.NeighborArray(g("nn"))

    def evaluator(theta):
        tot = vo.run(ds.y, ds.X, ds.locs, nn.idx, "exponential_isotropic", theta, deterministic=True)
        return vg.assemble(engine.parts_from_flat(tot, ds.p, 3), ds.n)

    start = vg.default_start(ds, "exponential_isotropic")
    np.testing.assert_allclose(start.theta, g("start"), rtol=1e-14)
    res = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=int(g("m"))), evaluator=evaluator)
    np.testing.assert_allclose(res.theta_hat.theta, g("compiled/theta_hat"), rtol=1e-12)
    np.testing.assert_allclose(res.loglik_trace, g("compiled/trace"), rtol=1e-13)
    assert res.iterations == int(g("compiled/iterations")) and res.converged
    assert res.loglik == pytest.approx(-398.7845764605893, rel=1e-12)  # pkg/test_output.txt:36


# ---- multi-rank combine (gloo, world_size 2) ------------------------------------
def test_shard_bounds_cover_range():
    for n, w in [(10, 3), (1 << 20, 8), (5, 8), (0, 2)]:
        cuts = [distributed.shard_bounds(n, w, r) for r in range(w)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
        assert max(b - a for a, b in cuts) - min(b - a for a, b in cuts) <= 1


_WORKER = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
from paper_2407_02740_b200 import distributed
from oracle import vecchia_oracle as vo
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
rng = np.random.default_rng(3)
n, m = 600, 8
locs = rng.uniform(0, 1, (n, 2)); y = rng.normal(size=n); X = np.ones((n, 1))
nn = vo.neighbor_scan(locs, m)
theta = np.array([1.2, 0.3, 0.1])
i0, i1 = distributed.shard_bounds(n, world, rank)
# each rank's (L+2,) vector in the layout of vb200_eval_async, produced here by the CPU oracle
local = vo.run(y, X, locs, nn, "exponential_isotropic", theta, i0=i0, i1=i1)
vec = torch.from_numpy(np.concatenate([local, [0.0, -np.inf]]))
tot, first = distributed.combine_partials(vec)
whole = vo.run(y, X, locs, nn, "exponential_isotropic", theta)
assert first == -1
np.testing.assert_allclose(tot, whole, rtol=1e-12, atol=1e-12)
# failure on the last rank only: every rank must learn the lowest failing index
fail = torch.from_numpy(np.concatenate([local, [2.0 if rank == world - 1 else 0.0,
                                                -(i0 + 5.0) - 1.0 if rank == world - 1 else -np.inf]]))
tot, first = distributed.combine_partials(fail)
lo = distributed.shard_bounds(n, world, world - 1)[0]
assert first == lo + 5, (first, lo)
dist.destroy_process_group()
print("rank", rank, "ok")
"""


def test_combine_partials_world_size_2_gloo(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(_WORKER.format(root=str(ROOT)))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", WORLD_SIZE="2", OMP_NUM_THREADS="2")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r)), stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o


def test_dependency_levels_match_definition_and_reject_acausal_tables():
    """Level schedule of the device conditional simulator (host C++): level(i) = 1 + max level of the neighbours."""
    rng = np.random.default_rng(12)
    for n, m, d in ((1, 3, 2), (40, 60, 2), (2500, 9, 3)):
        locs = rng.uniform(0, 1, (n, d))
        nn = vg.find_ordered_neighbors(locs, m)
        order, level_ptr = vg.dependency_levels(nn)
        lev = np.zeros(n, dtype=np.int64)
        for i in range(n):
            r = nn.idx[i, 1:]
            r = r[r >= 0]
            if r.size:
                lev[i] = lev[r].max() + 1
        assert np.array_equal(order, np.lexsort((np.arange(n), lev)))
        assert np.array_equal(np.diff(level_ptr), np.bincount(lev))
        assert level_ptr[0] == 0 and level_ptr[-1] == n
    bad = nn.idx.copy()
    bad[5, 1] = 7  # row 5 conditions on a LATER observation
    with pytest.raises(ValueError):
        vg.dependency_levels(vg.NeighborArray(bad))


def test_simulation_needs_the_device_and_validates_first():
    locs = np.random.default_rng(0).uniform(0, 1, (50, 2))
    nn = vg.find_ordered_neighbors(locs, 5)
    cov = vg.CovarianceParameters("exponential_isotropic", [1.0, 0.2, 0.1])
    with pytest.raises(ValueError):
        vg.simulate_nn_gp(cov, [0.0, 1.0], locs, np.ones((50, 1)), nn, seed=1)  # beta / design mismatch
    with pytest.raises(ValueError):
        vg.simulate_nn_gp(cov, [0.0], locs[:40], np.ones((40, 1)), nn, seed=1)   # table / locations mismatch
    if _cabi.device_count() == 0:
        with pytest.raises(vg.DeviceUnavailable):
            vg.simulate_nn_gp(cov, [0.0], locs, np.ones((50, 1)), nn, seed=1)


def test_row_owner_pair_schedule_covers_every_pair_once(tmp_path):
    """PairSched<G,S> (csrc/kernel_tiled.cuh): the static (lane, step) -> pair mapping of the row-owner pair phase
    covers each off-diagonal pair of every tier exactly once and never touches the padding column.  Host build of
    the same header with nvcc (no GPU needed)."""
    import shutil
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc unavailable")
    exe = tmp_path / "check_pair_schedule"
    src = ROOT / "tests" / "native" / "check_pair_schedule.cu"
    subprocess.run([nvcc, "-std=c++17", "-O1", "-I", str(ROOT / "include"), "-I", str(ROOT / "paper_2407_02740_b200" / "csrc"),
                    "-o", str(exe), str(src)], check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and "FAIL" not in out.stdout, out.stdout
    assert out.stdout.count(" ok") == 8


# ---- round 2: text formats, core selection, smoothness bounds ---------------------------------------
def test_csv_round_trips_are_exact(tmp_path):
    from paper_2407_02740_b200 import io
    rng = np.random.default_rng(4)
    ds = vg.Dataset(rng.normal(size=9), rng.normal(size=(9, 2)), rng.uniform(size=(9, 3)))
    io.write_csv_dataset(ds, tmp_path / "d.csv")
    back = io.read_csv_dataset(tmp_path / "d.csv")
    assert np.array_equal(back.y, ds.y) and np.array_equal(back.X, ds.X) and np.array_equal(back.locs, ds.locs)
    only_locs = io.read_csv_dataset(tmp_path / "d.csv", x_cols=[], loc_cols=["loc0", "loc1"])
    assert only_locs.p == 1 and np.all(only_locs.X == 1.0) and only_locs.d == 2
    nn = vg.find_ordered_neighbors(ds.locs, 4)
    io.write_neighbors_csv(nn, tmp_path / "n.csv")
    assert np.array_equal(io.read_neighbors_csv(tmp_path / "n.csv").idx, nn.idx)
    with pytest.raises(ValueError):
        io.read_csv_dataset(tmp_path / "d.csv", y_col="nope")


def test_core_selection_follows_the_reference_env_variable(monkeypatch):
    monkeypatch.delenv("VECCHIAGP_CORE", raising=False)
    assert engine._validate_core(None) == "cuda"
    monkeypatch.setenv("VECCHIAGP_CORE", "cuda")
    assert engine._validate_core(None) == "cuda"
    monkeypatch.setenv("VECCHIAGP_CORE", "compiled")
    with pytest.raises(ValueError):
        engine._validate_core(None)
    assert engine._validate_core("cuda") == "cuda"   # an explicit argument wins over the environment
    monkeypatch.setenv("VECCHIAGP_CORE", "bogus")
    with pytest.raises(ValueError):
        engine._validate_core(None)


def test_matern_smoothness_bounds_are_checked_on_the_host():
    ok = vg.CovarianceParameters("matern_isotropic", [1.0, 0.2, 1.5, 0.1])
    assert vg.validate_parameters(ok, 2).name == "matern_isotropic"
    for nu in (1e-6, 61.0):
        with pytest.raises(ValueError):
            vg.validate_parameters(vg.CovarianceParameters("matern_isotropic", [1.0, 0.2, nu, 0.1]), 2)


def test_fit_treats_out_of_domain_proposals_as_rejected_trials():
    """A Fisher step that leaves the parameter domain (ValueError from validation / the library) must be halved like a
    failed factorization, not abort the fit (advisor finding, round 1)."""
    calls = []

    def evaluator(theta):
        calls.append(np.array(theta))
        if theta[0] > 3.0:
            raise ValueError("out of domain")
        ll = -float(np.sum((np.log(theta) - np.log([2.0, 0.5, 0.1])) ** 2))
        grad = -2.0 * (np.log(theta) - np.log([2.0, 0.5, 0.1])) / theta
        info = np.diag(0.05 / theta ** 2)   # far too small: the full step overshoots out of the domain
        return inference.ProfiledEvaluation(ll, np.zeros(1), grad, info, np.eye(1))

    ds = vg.Dataset(np.zeros(5), np.ones((5, 1)), np.arange(10.0).reshape(5, 2))
    nn = vg.find_ordered_neighbors(ds.locs, 2)
    model = vg.ModelSpec(covariance=vg.CovarianceParameters("exponential_isotropic", [1.0, 0.4, 0.2]), m=2)
    res = inference.fit(ds, nn, model, evaluator=evaluator, max_iters=60)
    assert any(c[0] > 3.0 for c in calls), "the test must actually propose an out-of-domain point"
    assert res.loglik_trace[-1] > res.loglik_trace[0]
