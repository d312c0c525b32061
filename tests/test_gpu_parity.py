"""GPU parity tests: the CUDA core (through the C ABI) against the CPU oracle and the
reference's golden fixtures.  Tolerances are BASELINE.json's: loglik 1e-9 relative,
gradient / Fisher information 1e-7 relative, fitted parameters 1e-6 relative.
Patterns follow the reference's own tests (pkg/tests/test_engine.py, test_inference.py,
test_acceptance.py)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import engine
from paper_2407_02740_b200.engine import DeviceProblem, flat_from_parts

from oracle import vecchia_oracle as vo
from conftest import make_instance

pytestmark = pytest.mark.gpu

LAYOUTS = ["warp_smem", "tiled_reg"]

CASES = ["iso_d2_p2_m9", "iso_d2_p1_m30", "iso_d3_p4_m30", "aniso_d3_p2_m8", "aniso_d2_p1_m20",
         "sphere_p1_m12", "iso_jitter", "iso_heads_only", "iso_wide_m79", "iso_zero_nugget",
         "iso_d1_m5", "iso_m60"]


def fields_close(got, want, p, q, rtol):
    """Field-by-field comparison, relative to each field's largest magnitude (entries of a
    field that cancel to ~0 are compared on the field's scale, as the reference's
    parts_close does with its atol; pkg/tests/conftest.py:41-64)."""
    G, W = vo.split_acc(np.asarray(got), p, q), vo.split_acc(np.asarray(want), p, q)
    for name in W:
        w, g = np.asarray(W[name], dtype=np.float64), np.asarray(G[name], dtype=np.float64)
        scale = max(float(np.max(np.abs(w))), 1e-300)
        err = float(np.max(np.abs(g - w))) / scale
        assert err <= rtol, f"{name}: relative error {err:.3e} > {rtol:.1e}"


def layouts_for(prob, q):
    """Layouts to exercise for this shape: always warp_smem, plus tiled_reg when supported."""
    out = ["warp_smem"]
    prob.set_layout("auto")
    if prob.layout_for(q) == "tiled_reg":
        out.append("tiled_reg")
    # the thread-per-observation study arms (the paper's layout): m+1 <= 32, d <= 3, p <= 4, <= 2 range parameters
    if prob.mp1 <= 32 and prob.d <= 3 and prob.p <= 4 and q - 2 <= 2:
        out += ["thread_smem", "thread_local"]
    return out


def _golden(z, name):
    g = lambda k: z[f"{name}/{k}"]
    return dict(y=g("y"), X=g("X"), locs=g("locs"), nn=g("nn"), theta=g("theta"), family=str(g("family")),
                jitter=float(g("jitter")), totals=g("totals_compiled"), loglik=float(g("loglik_compiled")),
                grad=g("grad_compiled"))


@pytest.mark.parametrize("name", CASES)
def test_golden_totals_match_reference(engine_cases, name):
    c = _golden(engine_cases, name)
    ds = vg.Dataset(c["y"], c["X"], c["locs"])
    nn = vg.NeighborArray(c["nn"])
    p, q = ds.p, c["theta"].shape[0]
    with DeviceProblem(ds, nn, c["family"]) as prob:
        for layout in layouts_for(prob, q):
            prob.set_layout(layout)
            tot = prob.totals(c["theta"], jitter=c["jitter"])
            fields_close(tot, c["totals"], p, q, 1e-9)
            ev = vg.assemble(engine.parts_from_flat(tot, p, q), ds.n)
            assert ev.loglik == pytest.approx(c["loglik"], rel=1e-9)
            gscale = np.max(np.abs(c["grad"]))
            assert np.max(np.abs(ev.grad - c["grad"])) <= 1e-7 * gscale


@pytest.mark.parametrize("name", ["iso_d2_p2_m9", "aniso_d3_p2_m8", "iso_heads_only", "iso_d3_p4_m30"])
def test_per_observation_rows_match_oracle(engine_cases, name):
    c = _golden(engine_cases, name)
    ds = vg.Dataset(c["y"], c["X"], c["locs"])
    nn = vg.NeighborArray(c["nn"])
    fam = vg.covariance_registry(c["family"])
    work = fam.prepare_locs(ds.locs)
    want, _ = vo.observations(ds.y, ds.X, work, nn.idx, c["family"], c["theta"], jitter=c["jitter"])
    with DeviceProblem(ds, nn, c["family"]) as prob:
        for layout in layouts_for(prob, c["theta"].shape[0]):
            prob.set_layout(layout)
            rows, flags = prob.rows_host(c["theta"], c["jitter"])
            assert not flags.any()
            np.testing.assert_allclose(rows, want, rtol=1e-8, atol=1e-9)


def test_engine_run_facade_and_process_observation(engine_cases):
    c = _golden(engine_cases, "iso_d2_p2_m9")
    ds = vg.Dataset(c["y"], c["X"], c["locs"])
    nn = vg.NeighborArray(c["nn"])
    cov = vg.CovarianceParameters(c["family"], c["theta"])
    parts = engine.run(ds, nn, cov, backend="task", deterministic=True, workers=3, core="cuda")
    fields_close(flat_from_parts(parts), c["totals"], ds.p, cov.nparms, 1e-9)
    again = engine.run(ds, nn, cov)  # cached device problem, bit-reproducible
    assert np.array_equal(flat_from_parts(parts), flat_from_parts(again))
    one = engine.process_observation(17, ds, nn, cov)
    want, _ = vo.observations(ds.y, ds.X, ds.locs, nn.idx, c["family"], c["theta"], i0=17, i1=18)
    np.testing.assert_allclose(flat_from_parts(one), want[0], rtol=1e-8, atol=1e-10)
    with pytest.raises(ValueError):
        engine.run(ds, nn, cov, core="compiled")
    with pytest.raises(ValueError):
        engine.run(ds, nn, cov, backend="gpu")
    with pytest.raises(ValueError):
        engine.run(ds, nn, cov, capacity_tier=4)
    with pytest.raises(ValueError):
        engine.run(ds, nn, vg.CovarianceParameters(c["family"], [1.0, -0.2, 0.1]))
    engine.clear_cache()


def test_k1_closed_form_and_zero_response():
    # reference tests/test_engine.py:93-114
    sig2, rho, tau2 = 1.7, 0.3, 0.2
    ds = vg.Dataset([0.8], [[1.0]], [[0.1, 0.2]])
    nn = vg.NeighborArray(np.array([[0]]))
    parts = engine.run(ds, nn, vg.CovarianceParameters("exponential_isotropic", [sig2, rho, tau2]))
    v = sig2 * (1 + tau2)
    assert parts.logdet == pytest.approx(np.log(v), rel=1e-13)
    assert parts.ysy == pytest.approx(0.64 / v, rel=1e-13)
    assert parts.xsx[0, 0] == pytest.approx(1 / v, rel=1e-13)
    y, X, locs, theta = make_instance(3, 50, 2, 2)
    nn = vg.find_ordered_neighbors(locs, 6)
    zero = engine.run(vg.Dataset(np.zeros(50), X, locs), nn, vg.CovarianceParameters("exponential_isotropic", theta))
    assert zero.ysy == 0.0 and not zero.ysx.any() and not zero.dysy.any() and not zero.dysx.any()
    engine.clear_cache()


def test_not_positive_definite_reports_observation_and_pivot(failure_case):
    # reference tests/test_engine.py:230-253: duplicated location, zero nugget -> observation 7
    z = failure_case
    n = z["y"].shape[0]
    ds = vg.Dataset(z["y"], np.ones((n, 1)), z["locs"])
    nn = vg.NeighborArray(z["nn"])
    cov = vg.CovarianceParameters("exponential_isotropic", z["theta"])
    with DeviceProblem(ds, nn, cov.family) as prob:
        for layout in layouts_for(prob, 3):
            prob.set_layout(layout)
            with pytest.raises(vg.NotPositiveDefinite) as err:
                prob.run(cov)
            assert err.value.observation == int(z["observation_compiled"]) == 7
            assert err.value.pivot == int(z["pivot_compiled"])
            rescued = prob.totals(cov.theta, jitter=1e-6)
            fields_close(rescued, z["rescued_totals"], 1, 3, 1e-4)  # near-singular K (cond ~1e6): the two CPU oracles differ by 1.4e-5 here


@pytest.mark.parametrize("m", [15, 20, 25, 40, 50, 60])
def test_failure_report_on_exact_size_tiers(m):
    """The exact-size tiers (static padding rows: packed triangles that start at local row NP-1) must report the same
    (observation, pivot) as the CPU oracle for a duplicated location with zero nugget -- the pivot index is counted
    in the observation's own frame, whatever padding the tier adds in front."""
    from oracle import vecchia_oracle as vo_
    rng = np.random.default_rng(300 + m)
    n = 3 * m + 30
    locs = rng.uniform(0.0, 1.0, (n, 2))
    dup = 2 * m + 9
    locs[dup] = locs[dup - 3]                # exact duplicate of an earlier point: singular local matrix
    y, X = rng.normal(size=n), np.ones((n, 1))
    theta = np.array([1.2, 0.3, 0.0])
    nn = vg.find_ordered_neighbors(locs, m)
    with pytest.raises(vo_.OracleNotPositiveDefinite) as want:
        vo_.run(y, X, locs, nn.idx, "matern15_isotropic", theta)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "matern15_isotropic") as prob:
        prob.set_layout("tiled_reg")
        with pytest.raises(vg.NotPositiveDefinite) as got:
            prob.totals(theta)
        assert "NP=" in prob.last_kernel_name, prob.last_kernel_name
    assert (got.value.observation, got.value.pivot) == (want.value.observation, want.value.pivot)


@pytest.mark.parametrize("p", [2, 3])
def test_design_column_padding_serves_p_without_an_instance(p):
    """m = 40 has register-tiled instances for p = 1 and p = 4 only: p = 2, 3 must run the p = 4 instance on
    zero-padded design columns (not the generic kernel) and reproduce the oracle's totals field by field; the
    per-observation rows (laid out for p) still come from the generic kernel."""
    from paper_2407_02740_b200 import _cabi
    y, X, locs, _ = make_instance(500 + p, 700, 2, p)
    theta = np.array([1.1, 0.2, 0.07])
    nn = vg.find_ordered_neighbors(locs, 40)
    want = vo.run(y, X, locs, nn.idx, "matern15_isotropic", theta)
    before = _cabi.load().vb200_fallback_count()
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "matern15_isotropic") as prob:
        assert prob.layout_for(3) == "tiled_reg"
        got = prob.totals(theta)
        assert "P=4" in prob.last_kernel_name and "NP=7" in prob.last_kernel_name, prob.last_kernel_name
        again = prob.totals(theta, i0=100, i1=650) + prob.totals(theta, i0=0, i1=100) + prob.totals(theta, i0=650, i1=700)
        assert _cabi.load().vb200_fallback_count() == before
        rows, flags = prob.rows_host(theta)
    fields_close(got, want, p, 3, 1e-9)
    fields_close(again, want, p, 3, 1e-9)
    fields_close(rows.sum(axis=0), want, p, 3, 1e-9)
    assert not flags.any()
    # failure propagation through the gathered result vector
    locs2 = locs.copy()
    locs2[650] = locs2[640]
    nn2 = vg.find_ordered_neighbors(locs2, 40)
    with DeviceProblem(vg.Dataset(y, X, locs2), nn2, "matern15_isotropic") as prob:
        with pytest.raises(vg.NotPositiveDefinite) as err:
            prob.totals(np.array([1.1, 0.2, 0.0]))
        assert err.value.observation == 650


@pytest.mark.parametrize("family,theta", [("exponential_isotropic", [1.2, 0.05, 0.1]),
                                          ("matern15_isotropic", [1.2, 0.03, 0.1]),
                                          ("matern_isotropic", [1.2, 0.04, 0.9, 0.1])])
def test_one_dimensional_locations_run_the_two_dimensional_instances(family, theta):
    """d = 1 (a time series): no instance is compiled for one coordinate; the isotropic families run the d = 2
    instance on records with a zero coordinate appended (same distances) instead of the generic kernel."""
    from paper_2407_02740_b200 import _cabi
    rng = np.random.default_rng(91)
    n, p = 900, 2
    locs = np.sort(rng.uniform(0.0, 1.0, (n, 1)), axis=0)[rng.permutation(n)]
    X = np.column_stack([np.ones(n), rng.normal(size=n)])
    y = rng.normal(size=n) + np.sin(5.0 * locs[:, 0])
    theta = np.asarray(theta)
    nn = vg.find_ordered_neighbors(locs, 30)
    want = vo.run(y, X, locs, nn.idx, family, theta)
    before = _cabi.load().vb200_fallback_count()
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        got = prob.totals(theta)
        assert "D=2" in prob.last_kernel_name and "vecchia_tiled_kernel" in prob.last_kernel_name
        assert _cabi.load().vb200_fallback_count() == before
        # (the general Matern has instances for p = 1, 4 only: its p = 2 rows come from the generic kernel)
        rows, flags = prob.rows_host(theta)
    q = theta.shape[0]
    tol = 1e-8 if family == "matern_isotropic" else 1e-9
    fields_close(got, want, p, q, tol)
    fields_close(rows.sum(axis=0), want, p, q, tol)
    assert not flags.any()


FAMILY_SHAPES = [
    ("exponential_isotropic", 2, 1, [1.5, 0.25, 0.1], 30),
    ("matern15_isotropic", 2, 1, [1.0, 0.08, 0.1], 30),
    ("matern25_isotropic", 2, 2, [1.2, 0.06, 0.05], 20),
    ("matern15_isotropic", 3, 4, [1.0, 0.15, 0.1], 30),
    ("exponential_spacetime", 3, 1, [1.3, 0.2, 0.5, 0.1], 30),
    ("exponential_anisotropic", 3, 1, [1.3, 0.2, 0.3, 0.5, 0.1], 10),
    ("exponential_isotropic", 2, 1, [1.5, 0.25, 0.1], 10),
    ("matern15_isotropic", 2, 1, [1.0, 0.08, 0.1], 40),
    ("matern15_isotropic", 2, 1, [1.0, 0.08, 0.1], 60),
    ("exponential_isotropic", 2, 3, [1.5, 0.25, 0.1], 15),
    ("matern_isotropic", 2, 1, [1.0, 0.08, 0.8, 0.1], 30),
    ("matern_isotropic", 3, 4, [1.0, 0.2, 2.2, 0.05], 30),
    ("matern_isotropic", 2, 2, [1.2, 0.1, 0.3, 0.1], 12),
    ("matern_isotropic", 2, 1, [1.2, 0.1, 1.5, 0.1], 45),
]


@pytest.mark.parametrize("family,d,p,theta,m", FAMILY_SHAPES)
def test_families_and_shapes_against_oracle(family, d, p, theta, m):
    n = 3000
    y, X, locs, theta = make_instance(100 + m + d, n, d, p, family, theta)
    nn = vg.find_ordered_neighbors(locs, m)
    want = vo.run(y, X, locs, nn.idx, family, theta, deterministic=True)
    q = theta.shape[0]
    ev_want = vo.assemble(want, n, p, q)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        for layout in layouts_for(prob, q):
            prob.set_layout(layout)
            got = prob.totals(theta)
            fields_close(got, want, p, q, 1e-9)
            ev = vg.assemble(engine.parts_from_flat(got, p, q), n)
            assert ev.loglik == pytest.approx(ev_want["loglik"], rel=1e-9)
            assert np.max(np.abs(ev.grad - ev_want["grad"])) <= 1e-7 * np.max(np.abs(ev_want["grad"]))
            assert np.max(np.abs(ev.info - ev_want["info"])) <= 1e-7 * np.max(np.abs(ev_want["info"]))
            again = prob.totals(theta)
            assert np.array_equal(got, again), "device reduction must be run-to-run reproducible"


def test_every_compiled_tiled_instance_against_oracle():
    """Each TILED_REG kernel instance (tier x family x d x p), at the widest m it serves and at a
    narrow one (heavy front padding), plus the ragged head rows, against the CPU oracle."""
    from paper_2407_02740_b200 import _cabi
    names = {0: "exponential_isotropic", 1: "exponential_anisotropic", 2: "exponential_spacetime",
             3: "matern15_isotropic", 4: "matern25_isotropic", 5: "matern_isotropic"}
    inst = _cabi.tiled_instances()
    assert len(inst) >= 60
    rng = np.random.default_rng(77)
    for g, s_, cap, fam, d, p in inst:
        family = names[fam]
        q = _cabi.load().vb200_family_nparms(fam, d)
        theta = np.concatenate([[1.3], rng.uniform(0.15, 0.4, q - 2), [0.08]])
        if fam == 5:
            theta[2] = rng.uniform(0.4, 2.6)  # smoothness
        for m in sorted({cap - 2, max(2, cap // 2 - 3)}):
            n = 3 * cap + 40
            y, X, locs, _ = make_instance(1000 + cap + d + p + m, n, d, p)
            nn = vg.find_ordered_neighbors(locs, m)
            want = vo.run(y, X, locs, nn.idx, family, theta)
            with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
                prob.set_layout("tiled_reg")
                got = prob.totals(theta)
                if m == cap - 2:  # the widest m of the tier must be served by exactly this instance
                    assert f"G={g},S={s_}," in prob.last_kernel_name, (prob.last_kernel_name, g, s_, m)
                # general Matern: the smoothness column is a central difference of step 1e-5 BY DEFINITION, i.e. the
                # rounding noise of two Bessel evaluations (1e-16) divided by 2e-5 -- 5e-12 per entry, up to ~1e-9 of
                # the field's scale after the cancellation in dysx; both sides carry it, so compare at 1e-8 there
                # (BASELINE's tolerance for gradient / information is 1e-7)
                fields_close(got, want, p, q, 1e-8 if fam == 5 else 1e-9)


def test_narrowed_table_upload_is_bit_identical():
    """The chunked upload with the table narrowed to int32 on the host and widened on the device
    (vbh_narrow_indices / vb200_widen_indices) leaves the same int64 rows on the device as the plain upload:
    identical totals for the same chunking, ragged head rows and -1 padding included, and the widening kernel
    reproduces odd-length blocks."""
    import torch
    from paper_2407_02740_b200 import _cabi
    y, X, locs, theta = make_instance(21, 6001, 2, 1)
    nn = vg.find_ordered_neighbors(locs, 30)
    ds = vg.Dataset(y, X, locs)
    tots = {}
    for narrow in (False, True):
        with DeviceProblem(ds, nn, "matern15_isotropic", upload_chunks=5, upload_narrow=narrow) as prob:
            assert prob.upload_narrowed == narrow
            tots[narrow] = prob.totals(theta)          # first evaluation: chunk by chunk behind the copies
            again = prob.totals(theta)                  # resident table
            dev_rows = prob._nn.cpu().numpy()
            assert np.array_equal(dev_rows, nn.idx)
            want = 8 * (y.size + X.size + locs.size) + (4 if narrow else 8) * nn.idx.size
            assert prob.h2d_bytes == want
        fields_close(again, tots[narrow], 1, 3, 1e-12)
    assert np.array_equal(tots[True], tots[False])
    lib = _cabi.load()
    src = torch.tensor([5, -1, 7, 2 ** 31 - 1, 0, 3, -1], dtype=torch.int32, device="cuda")
    dst = torch.full((8,), 99, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    _cabi.check(lib.vb200_widen_indices(src.data_ptr(), dst.data_ptr(), 7, None), "vb200_widen_indices")
    torch.cuda.synchronize()
    assert dst.cpu().tolist() == [5, -1, 7, 2 ** 31 - 1, 0, 3, -1, 99]


def test_thread_layouts_reject_shapes_beyond_their_capacity():
    """The thread-per-observation study arms refuse shapes beyond their compile-time capacity (no fallback)."""
    y, X, locs, theta = make_instance(3, 400, 2, 1)
    wide = vg.find_ordered_neighbors(locs, 40)
    with DeviceProblem(vg.Dataset(y, X, locs), wide, "exponential_isotropic") as prob:
        for layout in ("thread_smem", "thread_local"):
            prob.set_layout(layout)
            with pytest.raises(NotImplementedError):
                prob.totals(theta)


def test_shard_sums_equal_whole_and_empty_range():
    y, X, locs, theta = make_instance(9, 5000, 2, 1)
    nn = vg.find_ordered_neighbors(locs, 30)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "exponential_isotropic") as prob:
        whole = prob.totals(theta)
        cuts = [0, 7, 31, 1250, 1251, 4000, 5000]
        parts = sum(prob.totals(theta, i0=a, i1=b) for a, b in zip(cuts[:-1], cuts[1:]))
        fields_close(parts, whole, 1, 3, 1e-11)
        assert not prob.totals(theta, i0=100, i1=100).any()
    # a problem holding only a shard of the neighbor rows (the multi-GPU layout)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "exponential_isotropic", row0=1250, rows=2750) as shard:
        got = shard.totals(theta)
        want = vo.run(y, X, locs, nn.idx, "exponential_isotropic", theta, i0=1250, i1=4000)
        fields_close(got, want, 1, 3, 1e-9)
        with pytest.raises(ValueError):
            shard.totals(theta, i0=0, i1=10)


def test_within_row_order_invariance():
    # reference tests/test_engine.py:169-185: permuting the neighbors of a row changes nothing
    y, X, locs, theta = make_instance(4, 400, 2, 1)
    nn = vg.find_ordered_neighbors(locs, 12).idx.copy()
    rng = np.random.default_rng(0)
    shuffled = nn.copy()
    for i in range(13, 400):
        shuffled[i, 1:] = rng.permutation(shuffled[i, 1:])
    ds = vg.Dataset(y, X, locs)
    a = flat_from_parts(engine.run(ds, vg.NeighborArray(nn), vg.CovarianceParameters("exponential_isotropic", theta)))
    b = flat_from_parts(engine.run(ds, vg.NeighborArray(shuffled),
                                   vg.CovarianceParameters("exponential_isotropic", theta)))
    fields_close(b, a, 1, 3, 1e-10)
    engine.clear_cache()


@pytest.mark.parametrize("tag", ["cli300_a", "cli300_b", "aniso400"])
def test_full_fit_matches_reference(fit_cases, tag):
    z = fit_cases
    g = lambda k: z[f"{tag}/{k}"]
    ds = vg.Dataset(g("y"), g("X"), g("locs"))
    nn = vg.NeighborArray(g("nn"))
    family = str(g("family"))
    start = vg.CovarianceParameters(family, g("start"))
    np.testing.assert_allclose(vg.default_start(ds, family).theta, start.theta, rtol=1e-12)
    res = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=int(g("m"))))
    np.testing.assert_allclose(res.theta_hat.theta, g("compiled/theta_hat"), rtol=1e-6)
    np.testing.assert_allclose(res.beta_hat, g("compiled/beta_hat"), rtol=1e-6, atol=1e-9)
    assert res.loglik == pytest.approx(float(g("compiled/trace")[-1]), rel=1e-9)
    assert res.converged == bool(g("compiled/converged"))
    assert all(b >= a for a, b in zip(res.loglik_trace, res.loglik_trace[1:]))
    engine.clear_cache()


def test_config1_fit_n10000_m30(config1_golden):
    """BASELINE.json configs[0]: n=10 000 2-D, exponential_isotropic, m=30, full fit."""
    z = config1_golden
    n, m, seed = 10_000, int(z["m"]), int(z["seed"])
    rng = np.random.default_rng(seed)
    locs = rng.uniform(0.0, 1.0, (n, 2))
    locs = locs[vg.random_permutation(n, seed).perm]
    nn = vg.find_ordered_neighbors(locs, m, method="grid")
    assert int(nn.idx.sum()) == int(z["nn_checksum"]) and np.array_equal(nn.idx[9999], z["nn_row_9999"])
    ds = vg.Dataset(z["y"], np.ones((n, 1)), locs)
    start = vg.default_start(ds, "exponential_isotropic")
    np.testing.assert_allclose(start.theta, z["start"], rtol=1e-12)
    ev0 = vg.evaluate(ds, nn, start)
    assert ev0.loglik == pytest.approx(float(z["loglik_start"]), rel=1e-9)
    np.testing.assert_allclose(ev0.grad, z["grad_start"], rtol=1e-7)
    np.testing.assert_allclose(ev0.info, z["info_start"], rtol=1e-7)
    res = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=m))
    np.testing.assert_allclose(res.theta_hat.theta, z["fit/theta_hat"], rtol=1e-6)
    np.testing.assert_allclose(res.beta_hat, z["fit/beta_hat"], rtol=1e-6)
    assert res.loglik == pytest.approx(float(z["fit/trace"][-1]), rel=1e-9)
    np.testing.assert_allclose(res.fisher_info, z["fit/fisher_info"], rtol=1e-5)
    engine.clear_cache()


def test_full_size_properties_n2_20():
    """BASELINE.json configs[1] shape (n = 2^20, m = 30, Matern 3/2): size-independent
    properties -- shard additivity, run-to-run reproducibility, oracle agreement on a
    prefix, and the analytic identities dlogdet_0 = n / sigma^2, ainfo_00 = n / (2 sigma^4)."""
    n, m = 1 << 20, 30
    rng = np.random.default_rng(2407)
    locs = rng.uniform(0.0, 1.0, (n, 2))
    y = rng.normal(size=n)
    X = np.ones((n, 1))
    theta = np.array([1.0, 0.002, 0.1])
    nn = vg.find_ordered_neighbors(locs, m)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "matern15_isotropic") as prob:
        first = prob.totals(theta)   # issued chunk by chunk behind the table upload
        whole = prob.totals(theta)   # table resident: one launch
        assert np.array_equal(whole, prob.totals(theta)), "resident evaluations must be bit-reproducible"
        fields_close(first, whole, 1, 3, 1e-13)
        halves = prob.totals(theta, i1=n // 3) + prob.totals(theta, i0=n // 3)
        fields_close(halves, whole, 1, 3, 1e-11)
        P = vo.split_acc(whole, 1, 3)
        assert P["dlogdet"][0] == pytest.approx(n / theta[0], rel=1e-10)
        assert P["ainfo"][0, 0] == pytest.approx(0.5 * n / theta[0] ** 2, rel=1e-10)
        k = 1 << 14
        want = vo.run(y, X, locs, nn.idx, "matern15_isotropic", theta, i0=0, i1=k)
        fields_close(prob.totals(theta, i0=0, i1=k), want, 1, 3, 1e-9)


# ---- kriging: reference predict.krige ------------------------------------------
@pytest.mark.parametrize("name", ["iso_m10", "iso_m60", "aniso_m20", "sphere_m15", "iso_all"])
def test_kriging_matches_reference(krige_cases, name):
    z = krige_cases
    g = lambda k: z[f"{name}/{k}"]
    train = vg.Dataset(g("y"), g("X"), g("locs"))
    cov = vg.CovarianceParameters(str(g("family")), g("theta"))
    p = train.p
    fr = vg.FitResult(theta_hat=cov, beta_hat=g("beta"), beta_cov=np.eye(p), loglik_trace=[0.0],
                      fisher_info=np.eye(cov.nparms), iterations=0, converged=True)
    for latent in (False, True):
        ps = vg.krige(fr, train, g("locs_star"), g("X_star"), m_pred=int(g("m_pred")), latent=latent)
        want_m, want_s = g(f"mean_latent{int(latent)}"), g(f"sd_latent{int(latent)}")
        assert np.max(np.abs(ps.mean - want_m)) <= 1e-9 * max(1.0, np.max(np.abs(want_m)))
        # sd = sqrt(prior - k'K^-1 k): at a prediction point on top of a training point with latent=True
        # the variance is a cancellation to ~0, so compare variances on the prior's scale
        prior = cov.theta[0] * (1.0 if latent else 1.0 + cov.theta[-1])
        assert np.max(np.abs(ps.sd ** 2 - want_s ** 2)) <= 1e-9 * prior
    no_sd = vg.krige(fr, train, g("locs_star"), g("X_star"), m_pred=int(g("m_pred")), with_sd=False)
    assert no_sd.sd is None
    with pytest.raises(vg.LengthMismatch):
        vg.krige(fr, train, g("locs_star"), g("X_star")[:-1], m_pred=int(g("m_pred")))
    with pytest.raises(ValueError):
        vg.krige(fr, train, g("locs_star"), g("X_star"), m_pred=train.n + 1)


@pytest.mark.parametrize("family,d,theta", [("matern15_isotropic", 2, [1.2, 0.1, 0.1]),
                                            ("matern_isotropic", 3, [1.0, 0.2, 0.8, 0.05]),
                                            ("exponential_spacetime", 3, [1.3, 0.2, 0.5, 0.1]),
                                            ("matern25_isotropic", 3, [0.8, 0.15, 0.02])])
def test_kriging_extension_families_against_oracle(family, d, theta):
    rng = np.random.default_rng(8)
    n, npred, m_pred = 6000, 500, 30
    y, X, locs, theta = make_instance(321, n, d, 2, family, theta)
    star = rng.uniform(0, 1, (npred, d))
    Xs = np.column_stack([np.ones(npred), rng.normal(size=npred)])
    beta = np.array([0.3, -0.7])
    cov = vg.CovarianceParameters(family, theta)
    fr = vg.FitResult(theta_hat=cov, beta_hat=beta, beta_cov=np.eye(2), loglik_trace=[0.0],
                      fisher_info=np.eye(cov.nparms), iterations=0, converged=True)
    ps = vg.krige(fr, vg.Dataset(y, X, locs), star, Xs, m_pred=m_pred)
    mean, sd, _ = vo.krige(y, X, locs, family, theta, beta, star, Xs, m_pred)
    np.testing.assert_allclose(ps.mean, mean, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(ps.sd ** 2, sd ** 2, rtol=1e-9, atol=1e-12)
    assert vg.rmse(ps.mean, mean) < 1e-9


# ---- conditional simulation: reference oracle.simulate_nn_gp -------------------
@pytest.mark.parametrize("name", ["iso_d2_m10", "iso_d2_m30", "iso_d2_p2_m5", "aniso_d3_m12"])
def test_simulation_matches_reference(simulate_cases, name):
    """Device level-scheduled conditional simulation == the reference's sequential loop on the same PCG64 draws."""
    z = simulate_cases
    g = lambda k: z[f"{name}/{k}"]
    cov = vg.CovarianceParameters(str(g("family")), g("theta"))
    y = vg.simulate_nn_gp(cov, g("beta"), g("locs"), g("X"), vg.NeighborArray(g("nn")), int(g("seed")))
    np.testing.assert_allclose(y, g("y"), rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("family,d,theta", [("matern15_isotropic", 2, [1.2, 0.1, 0.1]),
                                            ("exponential_spacetime", 3, [1.3, 0.2, 0.5, 0.1]),
                                            ("matern_isotropic", 2, [1.0, 0.2, 0.8, 0.05])])
def test_simulation_extension_families_against_oracle(family, d, theta):
    from oracle import numpy_families as nf
    rng = np.random.default_rng(5)
    n, m = 700, 20
    locs = rng.uniform(0, 1, (n, d))
    X = np.column_stack([np.ones(n), rng.normal(size=n)])
    beta = np.array([0.4, -1.1])
    nn = vg.find_ordered_neighbors(locs, m)
    cov = vg.CovarianceParameters(family, theta)
    y = vg.simulate_nn_gp(cov, beta, locs, X, nn, seed=31)
    want = nf.simulate_nn_gp(family, np.asarray(theta), beta, vg.covariance_registry(family).prepare_locs(locs), X,
                             nn.idx, 31)
    np.testing.assert_allclose(y, want, rtol=1e-9, atol=1e-9)


def test_simulation_at_scale_recovers_the_model():
    """n = 2^18: the draw has the model's likelihood statistics -- the profiled gradient at the simulating
    parameters is small against its standard error (Fisher information), and a full fit recovers theta."""
    n, m = 1 << 18, 30
    rng = np.random.default_rng(2)
    locs = rng.uniform(0, 1, (n, 2))
    nn = vg.find_ordered_neighbors(locs, m)
    theta = np.array([1.5, 0.05, 0.1])
    cov = vg.CovarianceParameters("matern15_isotropic", theta)
    X = np.ones((n, 1))
    y = vg.simulate_nn_gp(cov, [0.3], locs, X, nn, seed=9)
    assert np.all(np.isfinite(y)) and abs(y.var() / (theta[0] * (1 + theta[2])) - 1.0) < 0.2
    ds = vg.Dataset(y, X, locs)
    ev = vg.evaluate(ds, nn, cov)
    zscore = ev.grad / np.sqrt(np.diag(ev.info))
    assert np.all(np.abs(zscore) < 5.0), zscore
    res = vg.fit(ds, nn, vg.ModelSpec(vg.default_start(ds, "matern15_isotropic"), m))
    assert res.converged
    np.testing.assert_allclose(res.theta_hat.theta, theta, rtol=0.05)


# ---- sharded (multi-rank) evaluation on the device: two ranks share this GPU, gloo all-reduce ------
_SHARD_WORKER = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import distributed, engine
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
backend = os.environ.get("VB200_TEST_BACKEND", "gloo")
if backend == "nccl":   # one GPU per rank, NCCL over NVLink: the production configuration
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
else:                   # two ranks share GPU 0, gloo all-reduce of CUDA tensors
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
rng = np.random.default_rng(3)
n, m = 20000, 30
locs = rng.uniform(0, 1, (n, 2)); y = rng.normal(size=n) + np.sin(5 * locs[:, 0]); X = np.ones((n, 1))
ds = vg.Dataset(y, X, locs)
nn = vg.find_ordered_neighbors(locs, m)
theta = np.array([1.2, 0.1, 0.2])
ev = distributed.ShardedEvaluator(ds, nn, "matern15_isotropic")
assert (ev.i0, ev.i1) == distributed.shard_bounds(n, world, rank)
sharded = ev.totals(theta)
with engine.DeviceProblem(ds, nn, "matern15_isotropic") as whole:
    single = whole.totals(theta)
scale = np.maximum(np.abs(single), 1e-300)
assert np.max(np.abs(sharded - single) / scale) < 1e-12, np.max(np.abs(sharded - single) / scale)
# the same Fisher-scoring fit from the sharded evaluator and from the single-GPU engine
start = vg.default_start(ds, "matern15_isotropic")
a = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=m), evaluator=ev)
b = vg.fit(ds, nn, vg.ModelSpec(covariance=start, m=m))
assert np.allclose(a.theta_hat.theta, b.theta_hat.theta, rtol=1e-9), (a.theta_hat.theta, b.theta_hat.theta)
assert a.iterations == b.iterations
# a failure on one shard is reported by every rank with the globally lowest index
locs2 = locs.copy(); locs2[15000] = locs2[14990]
nn2 = vg.find_ordered_neighbors(locs2, m)
ev2 = distributed.ShardedEvaluator(vg.Dataset(y, X, locs2), nn2, "exponential_isotropic")
try:
    ev2.totals(np.array([1.0, 0.3, 0.0]))
    raise SystemExit("expected NotPositiveDefinite")
except vg.NotPositiveDefinite as err:
    assert err.observation == 15000, err.observation
ev.close(); ev2.close()
dist.destroy_process_group()
print("rank", rank, "ok")
"""


def test_sharded_evaluator_two_ranks_one_gpu(tmp_path):
    import os, subprocess, sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    script = tmp_path / "shard_worker.py"
    script.write_text(_SHARD_WORKER.format(root=root))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29577", WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r)), stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]


def test_sharded_evaluator_two_ranks_nccl(tmp_path):
    """The same worker over NCCL with one GPU per rank -- runs wherever at least two GPUs are visible (the
    driver's 8-GPU box); skipped on the single-GPU boxes this repository was developed on."""
    import os, subprocess, sys
    from pathlib import Path
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    root = str(Path(__file__).resolve().parent.parent)
    script = tmp_path / "shard_worker_nccl.py"
    script.write_text(_SHARD_WORKER.format(root=root))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29578", WORLD_SIZE="2", VB200_TEST_BACKEND="nccl")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r)), stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
