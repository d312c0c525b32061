"""GPU tests that hold the CUDA path to truths OTHER than the repo's own CPU oracle.

The reference has no Matern and no space-time family (covariance.py:187-198 rejects "matern"), so for those
families the CUDA path is pinned the way the reference pins its own cores -- by structure:

  * d-fields against central finite differences of the undifferentiated fields
    (pkg/tests/test_engine.py:187-208),
  * ainfo == 1/2 tr(S^-1 D_j S^-1 D_l) at full conditioning (pkg/tests/test_engine.py:219-228),
  * log-likelihood == the dense Gaussian log-likelihood at m = n-1 (pkg/tests/test_acceptance.py:57-75),

plus the one reference-held pin the general-order Matern can have: at smoothness 1/2 it IS the exponential
kernel, so it must reproduce the reference's exponential_isotropic golden totals.  The dense quantities are
computed here with numpy from the package's host-side covariance functions (not from oracle/).

Also here: the INTEGRATION.md stub executed verbatim (host pointers through vb200_create / vb200_eval),
BASELINE configs 3 and 5 at their named scale, byte-identical fit documents, the pivot-floor boundary.
"""
from __future__ import annotations

import ctypes
import json

import numpy as np
import pytest

import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import _cabi, distributed, engine, inference, io, preprocess
from paper_2407_02740_b200.covariance import covariance_registry
from paper_2407_02740_b200.engine import DeviceProblem

from conftest import make_instance

pytestmark = pytest.mark.gpu

STRUCT_FAMILIES = [
    ("matern15_isotropic", 2, [1.3, 0.3, 0.1]),
    ("matern25_isotropic", 2, [1.1, 0.25, 0.05]),
    ("matern_isotropic", 2, [1.2, 0.3, 0.8, 0.1]),
    ("matern_isotropic", 3, [1.0, 0.4, 1.7, 0.08]),
    ("exponential_spacetime", 3, [1.3, 0.3, 0.6, 0.1]),
    ("exponential_isotropic", 2, [1.5, 0.25, 0.1]),
]


def _layouts(prob, q):
    out = ["warp_smem"]
    prob.set_layout("auto")
    if prob.layout_for(q) == "tiled_reg":
        out.append("tiled_reg")
    return out


def _dense_loglik(family, theta, y, X, locs):
    """Profiled Gaussian log-likelihood with the dense covariance (numpy / LAPACK)."""
    fam = covariance_registry(family)
    S = fam.matrix(theta, locs)
    c = np.linalg.cholesky(S)
    Xi, yi = np.linalg.solve(c, X), np.linalg.solve(c, y)
    beta = np.linalg.solve(Xi.T @ Xi, Xi.T @ yi)
    r = yi - Xi @ beta
    n = y.shape[0]
    return -0.5 * (n * np.log(2 * np.pi) + 2.0 * np.log(np.diag(c)).sum() + r @ r)


@pytest.mark.parametrize("family,d,theta", STRUCT_FAMILIES)
def test_cuda_loglik_equals_dense_at_full_conditioning(family, d, theta):
    """m = n-1: the Vecchia likelihood IS the exact Gaussian likelihood (pkg/tests/test_acceptance.py:57-75)."""
    n, p = 40, 2
    theta = np.asarray(theta, dtype=np.float64)
    y, X, locs, _ = make_instance(700 + d, n, d, p, family, theta)
    nn = vg.find_ordered_neighbors(locs, n - 1)
    want = _dense_loglik(family, theta, y, X, locs)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        for layout in _layouts(prob, theta.shape[0]):
            prob.set_layout(layout)
            ev = vg.assemble(prob.run(vg.CovarianceParameters(family, theta)), n)
            assert ev.loglik == pytest.approx(want, rel=1e-8), layout


@pytest.mark.parametrize("family,d,theta", STRUCT_FAMILIES)
def test_cuda_information_equals_dense_trace_form(family, d, theta):
    """ainfo == 1/2 tr(S^-1 D_j S^-1 D_l) at m = n-1 (pkg/tests/test_engine.py:219-228)."""
    n, p = 36, 1
    theta = np.asarray(theta, dtype=np.float64)
    y, X, locs, _ = make_instance(800 + d, n, d, p, family, theta)
    nn = vg.find_ordered_neighbors(locs, n - 1)
    fam = covariance_registry(family)
    Sinv = np.linalg.inv(fam.matrix(theta, locs))
    D = fam.derivatives(theta, locs)
    q = theta.shape[0]
    want = np.array([[0.5 * np.trace(Sinv @ D[j] @ Sinv @ D[l]) for l in range(q)] for j in range(q)])
    # the smoothness derivative of matern_isotropic is a central difference by definition (step 1e-5): the
    # host family and the device use the same definition, so the same tolerance applies
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        for layout in _layouts(prob, q):
            prob.set_layout(layout)
            parts = prob.run(vg.CovarianceParameters(family, theta))
            assert np.allclose(parts.ainfo, parts.ainfo.T, rtol=1e-12, atol=0)
            err = np.max(np.abs(parts.ainfo - want)) / np.max(np.abs(want))
            assert err <= 1e-7, (layout, err)


@pytest.mark.parametrize("family,d,theta", STRUCT_FAMILIES)
def test_cuda_derivative_fields_against_central_differences(family, d, theta):
    """dlogdet / dysy / dysx / dxsx against central differences of logdet / ysy / ysx / xsx
    (pkg/tests/test_engine.py:187-208), m = 30 on n = 600 points."""
    n, p, m = 600, 2, 30
    theta = np.asarray(theta, dtype=np.float64)
    y, X, locs, _ = make_instance(900 + d, n, d, p, family, theta)
    nn = vg.find_ordered_neighbors(locs, m)
    q = theta.shape[0]
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        for layout in _layouts(prob, q):
            prob.set_layout(layout)
            base = prob.run(vg.CovarianceParameters(family, theta))
            for j in range(q):
                h = 1e-5 * max(abs(theta[j]), 1e-2)
                tp, tm = theta.copy(), theta.copy()
                tp[j] += h
                tm[j] -= h
                if tm[j] < 0:
                    continue
                up = prob.run(vg.CovarianceParameters(family, tp))
                dn = prob.run(vg.CovarianceParameters(family, tm))
                for name, dname in (("logdet", "dlogdet"), ("ysy", "dysy"), ("ysx", "dysx"), ("xsx", "dxsx")):
                    fd = (np.asarray(getattr(up, name)) - np.asarray(getattr(dn, name))) / (2 * h)
                    got = np.asarray(getattr(base, dname))[..., j]
                    scale = max(np.max(np.abs(fd)), 1e-12)
                    assert np.max(np.abs(got - fd)) / scale <= 2e-5, (layout, dname, j)


@pytest.mark.parametrize("name", ["iso_d2_p1_m30", "iso_d2_p2_m9", "iso_d3_p4_m30", "iso_zero_nugget", "iso_m60"])
def test_general_matern_at_half_reproduces_reference_exponential_goldens(engine_cases, name):
    """matern_isotropic(nu = 1/2) == exponential_isotropic: the device Bessel-K path against totals produced
    by the UNMODIFIED reference (tests/golden/engine_cases.npz).  Covers logdet, ysy, xsx, ysx and the
    variance / range / nugget derivative fields; the smoothness column has no reference counterpart."""
    g = lambda k: engine_cases[f"{name}/{k}"]
    y, X, locs, nnidx, th = g("y"), g("X"), g("locs"), g("nn"), g("theta")
    jitter = float(g("jitter"))
    want = g("totals_compiled")
    p, n = X.shape[1], y.shape[0]
    q_ref, q = 3, 4
    thm = np.array([th[0], th[1], 0.5, th[2]])
    from oracle import vecchia_oracle as vo  # only its split_acc index helper (test infrastructure)
    W = vo.split_acc(np.asarray(want), p, q_ref)
    keep = [0, 1, 3]  # variance, range, nugget columns of the q = 4 layout
    with DeviceProblem(vg.Dataset(y, X, locs), vg.NeighborArray(nnidx), "matern_isotropic") as prob:
        for layout in _layouts(prob, q):
            prob.set_layout(layout)
            G = vo.split_acc(prob.totals(thm, jitter=jitter), p, q)
            checks = [("logdet", G["logdet"], W["logdet"]), ("ysy", G["ysy"], W["ysy"]), ("xsx", G["xsx"], W["xsx"]),
                      ("ysx", G["ysx"], W["ysx"]), ("dlogdet", G["dlogdet"][keep], W["dlogdet"]),
                      ("dysy", G["dysy"][keep], W["dysy"]), ("dysx", G["dysx"][:, keep], W["dysx"]),
                      ("dxsx", G["dxsx"][:, :, keep], W["dxsx"]),
                      ("ainfo", G["ainfo"][np.ix_(keep, keep)], W["ainfo"])]
            for fname, got, ref in checks:
                scale = max(float(np.max(np.abs(ref))), 1e-300)
                err = float(np.max(np.abs(np.asarray(got) - np.asarray(ref)))) / scale
                assert err <= 1e-9, (name, layout, fname, err)
            ev = vg.assemble(engine.parts_from_flat(prob.totals(thm, jitter=jitter), p, q), n)
            assert ev.loglik == pytest.approx(float(g("loglik_compiled")), rel=1e-9)


# ---------------------------------------------------------------------------
# the INTEGRATION.md stub, verbatim: HOST pointers through vb200_create / vb200_eval
# ---------------------------------------------------------------------------
def _integration_stub():
    """Extract and exec the `engine/_cuda.py` block of INTEGRATION.md; returns its run_cuda."""
    from pathlib import Path
    text = (Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    start = text.index("# engine/_cuda.py")
    end = text.index("```", start)
    code = text[start:end].replace('ctypes.CDLL("libvecchia_b200.so")', f'ctypes.CDLL({str(_cabi.library_path())!r})')
    scope = {}
    exec(compile(code, "INTEGRATION.md:_cuda.py", "exec"), scope)
    return scope["run_cuda"]


@pytest.mark.parametrize("name", ["iso_d2_p1_m30", "aniso_d3_p2_m8", "iso_heads_only", "iso_jitter"])
def test_integration_stub_with_host_pointers_matches_reference(engine_cases, name):
    _cabi.load()  # builds the library if needed
    run_cuda = _integration_stub()
    g = lambda k: engine_cases[f"{name}/{k}"]
    family = str(g("family"))
    fam = covariance_registry(family)
    y = np.ascontiguousarray(g("y"), dtype=np.float64)
    X = np.ascontiguousarray(g("X"), dtype=np.float64)
    work = np.ascontiguousarray(fam.prepare_locs(g("locs")), dtype=np.float64)
    nn = np.ascontiguousarray(g("nn"), dtype=np.int64)
    theta = np.ascontiguousarray(g("theta"), dtype=np.float64)
    flat, first, piv = run_cuda(y, X, work, nn, theta, fam.kernel_code, float(g("jitter")))
    assert first == -1 and piv == -1
    want = g("totals_compiled")
    p, q = X.shape[1], theta.shape[0]
    from oracle import vecchia_oracle as vo
    G, W = vo.split_acc(flat, p, q), vo.split_acc(want, p, q)
    for k in W:
        scale = max(float(np.max(np.abs(W[k]))), 1e-300)
        assert float(np.max(np.abs(np.asarray(G[k]) - np.asarray(W[k])))) / scale <= 1e-9, k


def test_integration_stub_reports_the_reference_failure(failure_case):
    _cabi.load()
    run_cuda = _integration_stub()
    z = failure_case
    y, locs = (np.ascontiguousarray(z[k], dtype=np.float64) for k in ("y", "locs"))
    X = np.ones((y.shape[0], 1))
    nn = np.ascontiguousarray(z["nn"], dtype=np.int64)
    theta = np.ascontiguousarray(z["theta"], dtype=np.float64)
    _, first, piv = run_cuda(y, X, locs, nn, theta, 0, 0.0)
    assert first == int(z["observation_compiled"]) == 7
    assert piv == int(z["pivot_compiled"])


# ---------------------------------------------------------------------------
# BASELINE configs 3 and 5 at their named scale (n = 2^22)
# ---------------------------------------------------------------------------
def _swath(n, seed):
    """Synthetic satellite-swath-like space-time locations: (lon, lat) on ascending tracks, time increasing."""
    rng = np.random.default_rng(seed)
    t = np.sort(rng.uniform(0.0, 1.0, n))
    track = np.floor(t * 64.0)
    along = t * 64.0 - track
    lon = (track * 0.137 + 0.02 * rng.normal(size=n)) % 1.0
    lat = along + 0.002 * rng.normal(size=n)
    return np.column_stack([lon, lat, t])


def test_config3_scale_spacetime_window_shards_and_fit():
    """n = 2^22, exponential_spacetime, d = 3, m = 30: a 2^14-row window past the head against the CPU oracle,
    shard additivity over 8 contiguous shards, and a full Fisher-scoring fit that must equal the same fit
    driven through distributed.ShardedEvaluator (the multi-GPU code path, world size 1 here)."""
    from oracle import vecchia_oracle as vo
    n, m, family = 1 << 22, 30, "exponential_spacetime"
    locs = _swath(n, 3)
    locs = locs[preprocess.random_permutation(n, 5).perm]
    X = np.ones((n, 1))
    nn = vg.find_ordered_neighbors(locs, m)
    truth = vg.CovarianceParameters(family, np.array([1.5, 0.05, 0.02, 0.1]))
    y = vg.simulate_nn_gp(truth, np.array([0.3]), locs, X, nn, seed=9)
    ds = vg.Dataset(y, X, locs)
    theta = np.array([1.2, 0.07, 0.03, 0.15])
    w0, w1 = 3_000_000, 3_000_000 + (1 << 14)
    full = np.full((n, m + 1), -1, dtype=np.int64)
    full[w0:w1] = nn.idx[w0:w1]
    want = vo.run(y, X, locs, full, family, theta, i0=w0, i1=w1)
    with DeviceProblem(ds, nn, family) as prob:
        assert prob.layout_for(4) == "tiled_reg"
        got = prob.totals(theta, i0=w0, i1=w1)
        scale = np.maximum(np.abs(want), 1e-9 * np.abs(want).max())
        assert np.max(np.abs(got - want) / scale) <= 1e-9
        first = prob.totals(theta)   # evaluated chunk by chunk behind the upload of the neighbor table
        whole = prob.totals(theta)   # one launch over the resident table
        assert np.max(np.abs(first - whole) / np.maximum(np.abs(whole), 1e-300)) <= 1e-11
        cuts = np.linspace(0, n, 9).astype(np.int64)
        parts = sum(prob.totals(theta, i0=int(a), i1=int(b)) for a, b in zip(cuts[:-1], cuts[1:]))
        assert np.max(np.abs(parts - whole) / np.maximum(np.abs(whole), 1e-300)) <= 1e-11
        assert np.array_equal(whole, prob.totals(theta)), "one launch, fixed-order reduction: bit-reproducible"
    model = vg.ModelSpec(covariance=inference.default_start(ds, family), m=m)
    fit1 = inference.fit(ds, nn, model)
    engine.clear_cache()
    ev = distributed.ShardedEvaluator(ds, nn, family)
    try:
        fit2 = inference.fit(ds, nn, model, evaluator=ev)
    finally:
        ev.close()
    assert fit1.converged and fit2.converged
    assert np.allclose(fit1.theta_hat.theta, fit2.theta_hat.theta, rtol=1e-10)
    assert fit1.loglik_trace[-1] == pytest.approx(fit2.loglik_trace[-1], rel=1e-12)
    # the simulated parameters are recovered (n = 4M: tight)
    assert np.allclose(fit1.theta_hat.theta, truth.theta, rtol=0.1)


def test_config5_scale_matern_p4_window_and_shards():
    """BASELINE config 5 names n = 2^24 over 8 GPUs; one GPU's share is n = 2^21 rows of a 2^24 dataset.  Here:
    n = 2^22, d = 3, p = 4, matern15_isotropic, m = 30 on ONE GPU (the 2^24 neighbor table alone takes 14 s to
    build): window against the CPU oracle, additivity over 8 shards, reproducibility."""
    from oracle import vecchia_oracle as vo
    n, m, family = 1 << 22, 30, "matern15_isotropic"
    rng = np.random.default_rng(21)
    locs = rng.uniform(size=(n, 3))
    X = np.column_stack([np.ones(n), locs])
    y = rng.normal(size=n) + X @ np.array([0.5, 1.0, -1.0, 0.25])
    nn = vg.find_ordered_neighbors(locs, m)
    theta = np.array([1.0, 0.02, 0.1])
    w0, w1 = 2_500_000, 2_500_000 + (1 << 13)
    full = np.full((n, m + 1), -1, dtype=np.int64)
    full[w0:w1] = nn.idx[w0:w1]
    want = vo.run(y, X, locs, full, family, theta, i0=w0, i1=w1)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, family) as prob:
        assert prob.layout_for(3) == "tiled_reg"
        got = prob.totals(theta, i0=w0, i1=w1)
        scale = np.maximum(np.abs(want), 1e-9 * np.abs(want).max())
        assert np.max(np.abs(got - want) / scale) <= 1e-9
        prob.totals(theta)           # settles the chunked upload
        whole = prob.totals(theta)
        cuts = np.linspace(0, n, 9).astype(np.int64)
        parts = sum(prob.totals(theta, i0=int(a), i1=int(b)) for a, b in zip(cuts[:-1], cuts[1:]))
        assert np.max(np.abs(parts - whole) / np.maximum(np.abs(whole), 1e-9 * np.abs(whole).max())) <= 1e-10
        assert np.array_equal(whole, prob.totals(theta))
        L = engine.acc_len(4, 3)
        Q = vo.split_acc(whole, 4, 3)
        assert Q["dlogdet"][0] == pytest.approx(n / theta[0], rel=1e-10)   # variance derivative: exactly n / sigma^2
        assert Q["ainfo"][0, 0] == pytest.approx(0.5 * n / theta[0] ** 2, rel=1e-10)
        assert whole.shape == (L,)


# ---------------------------------------------------------------------------
# acceptance criterion 8 (pkg/tests/test_acceptance.py:310-352): byte-identical fit documents
# ---------------------------------------------------------------------------
def test_fit_document_is_byte_identical_across_runs(tmp_path):
    n, m = 3000, 20
    y, X, locs, _ = make_instance(31, n, 2, 2)
    nn = vg.find_ordered_neighbors(locs, m)
    ds = vg.Dataset(y, X, locs)
    model = vg.ModelSpec(covariance=inference.default_start(ds, "exponential_isotropic"), m=m)
    docs = []
    for k in range(2):
        engine.clear_cache()
        fit = inference.fit(ds, nn, model)
        d = io.fit_to_dict(fit, config={"m": m})
        d.pop("phase_timings_ms")  # wall-clock, as in the reference's criterion (everything else must match)
        docs.append(json.dumps(d, sort_keys=True))
    assert docs[0] == docs[1]


# ---------------------------------------------------------------------------
# the pivot floor (a deliberate, documented deviation: pivot <= 1e-14 * diag fails; the reference fails at <= 0)
# ---------------------------------------------------------------------------
def _near_duplicate_problem(eps):
    """Ten points on a line, the last two `eps` apart, zero nugget: the last pivot is ~ 2 eps / range relative to
    the diagonal, so cond ~ range / eps."""
    x = np.concatenate([np.linspace(0.0, 1.0, 9), [1.0 + eps]])
    locs = np.column_stack([x, np.zeros_like(x)])
    y = np.sin(4.0 * x)
    X = np.ones((x.shape[0], 1))
    return vg.Dataset(y, X, locs), vg.find_ordered_neighbors(locs, 9)


def test_pivot_floor_brackets_the_reference_rule():
    """cond ~ 1e13: accepted here like in the reference (pivot > 0 and > 1e-14 diag); cond ~ 1e15: the pivot is
    below 1e-14 diag -- the reference would still accept it (s > 0), this library reports NotPositiveDefinite at
    the last observation.  Documented in DESIGN.md section 6 / include/vecchia_b200.h."""
    from oracle import vecchia_oracle as vo
    cov = vg.CovarianceParameters("exponential_isotropic", np.array([1.0, 0.5, 0.0]))
    ds, nn = _near_duplicate_problem(2.5e-14)   # relative pivot ~ 1e-13 > floor
    with DeviceProblem(ds, nn, cov.family) as prob:
        got = prob.totals(cov.theta)
    want = vo.run(ds.y, ds.X, ds.locs, nn.idx, cov.family, cov.theta)
    # accepted by both; the last pivot (~1e-13 of the diagonal) carries ~1e-3 relative rounding noise in either
    # implementation, so log(pivot) agrees to ~1e-2 absolute, not more
    assert got[0] == pytest.approx(want[0], abs=0.05)
    ds, nn = _near_duplicate_problem(1e-15)     # relative pivot ~ 4e-15 < floor; the reference accepts (pivot > 0)
    want = vo.run(ds.y, ds.X, ds.locs, nn.idx, cov.family, cov.theta)
    assert np.isfinite(want[0])
    with DeviceProblem(ds, nn, cov.family) as prob:
        with pytest.raises(vg.NotPositiveDefinite) as err:
            prob.totals(cov.theta)
    assert err.value.observation == 9 and err.value.pivot == 9


def test_engine_run_sees_in_place_edits_of_the_dataset():
    """The reference's run() is stateless; an in-place edit of y between two calls must be honoured."""
    y, X, locs, _ = make_instance(55, 500, 2, 1)
    nn = vg.find_ordered_neighbors(locs, 10)
    ds = vg.Dataset(y, X, locs)
    cov = vg.CovarianceParameters("exponential_isotropic", np.array([1.5, 0.25, 0.1]))
    a = engine.run(ds, nn, cov)
    ds.y[:] = 2.0 * ds.y
    b = engine.run(ds, nn, cov)
    assert b.ysy == pytest.approx(4.0 * a.ysy, rel=1e-12)
    assert b.logdet == a.logdet


# ---------------------------------------------------------------------------
# shapes outside the tiled kriging instances (d = 1, d = 4, m_pred > 62): the generic warp-per-point kernel
# (the reference's predict.krige / simulate_nn_gp accept any d and any m_pred <= n)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("family,d,theta,m_pred", [("exponential_isotropic", 1, [1.2, 0.1, 0.1], 12),
                                                   ("matern15_isotropic", 4, [1.0, 0.4, 0.05], 25),
                                                   ("exponential_anisotropic", 4, [1.3, 0.3, 0.4, 0.5, 0.6, 0.1], 20),
                                                   ("matern25_isotropic", 2, [0.8, 0.15, 0.02], 90),
                                                   ("matern_isotropic", 1, [1.0, 0.2, 0.8, 0.05], 10)])
def test_kriging_generic_shapes_against_oracle(family, d, theta, m_pred):
    from oracle import vecchia_oracle as vo
    rng = np.random.default_rng(18)
    n, npred = 1500, 200
    y, X, locs, theta = make_instance(654, n, d, 2, family, theta)
    star = rng.uniform(0, 1, (npred, d))
    Xs = np.column_stack([np.ones(npred), rng.normal(size=npred)])
    beta = np.array([0.3, -0.7])
    cov = vg.CovarianceParameters(family, theta)
    fr = vg.FitResult(theta_hat=cov, beta_hat=beta, beta_cov=np.eye(2), loglik_trace=[0.0],
                      fisher_info=np.eye(cov.nparms), iterations=0, converged=True)
    for latent in (False, True):
        ps = vg.krige(fr, vg.Dataset(y, X, locs), star, Xs, m_pred=m_pred, latent=latent)
        mean, sd, _ = vo.krige(y, X, locs, family, theta, beta, star, Xs, m_pred, latent=latent)
        np.testing.assert_allclose(ps.mean, mean, rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(ps.sd ** 2, sd ** 2, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("family,d,theta,m", [("exponential_isotropic", 1, [1.2, 0.1, 0.1], 8),
                                              ("matern15_isotropic", 4, [1.0, 0.4, 0.05], 15),
                                              ("exponential_isotropic", 2, [1.5, 0.2, 0.1], 70)])
def test_simulation_generic_shapes_against_oracle(family, d, theta, m):
    from oracle import numpy_families as nf
    rng = np.random.default_rng(6)
    n = 500
    locs = rng.uniform(0, 1, (n, d))
    X = np.column_stack([np.ones(n), rng.normal(size=n)])
    beta = np.array([0.4, -1.1])
    nn = vg.find_ordered_neighbors(locs, m)
    cov = vg.CovarianceParameters(family, theta)
    y = vg.simulate_nn_gp(cov, beta, locs, X, nn, seed=31)
    want = nf.simulate_nn_gp(family, np.asarray(theta, dtype=np.float64), beta,
                             vg.covariance_registry(family).prepare_locs(locs), X, nn.idx, 31)
    np.testing.assert_allclose(y, want, rtol=1e-9, atol=1e-9)


# ---------------------------------------------------------------------------
# housekeeping entry points of the C ABI added in round 2
# ---------------------------------------------------------------------------
def test_one_launch_per_evaluation_fallback_counter_and_memory_release():
    lib = _cabi.load()
    y, X, locs, _ = make_instance(77, 2000, 2, 1)
    nn = vg.find_ordered_neighbors(locs, 30)
    theta = np.array([1.5, 0.25, 0.1])
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "exponential_isotropic") as prob:
        a = prob.totals(theta)
        assert prob.last_launch_count == 1, "reset, main kernel and reduction are ONE launch"
        assert prob.layout_for(3) == "tiled_reg"
        before = lib.vb200_fallback_count()
        prob.totals(theta)
        assert lib.vb200_fallback_count() == before, "a tiled instance exists: no fallback"
        assert np.array_equal(a, prob.totals(theta))
    # a shape without a tiled instance (p = 5): AUTO falls back, says so once, and counts it
    y5, X5, locs5, _ = make_instance(78, 800, 2, 5)
    nn5 = vg.find_ordered_neighbors(locs5, 12)
    engine._FALLBACK_WARNED.clear()
    with DeviceProblem(vg.Dataset(y5, X5, locs5), nn5, "exponential_isotropic") as prob:
        before = lib.vb200_fallback_count()
        with pytest.warns(RuntimeWarning, match="falling back"):
            prob.totals(theta)
        assert prob.layout_for(3) == "warp_smem"
        assert lib.vb200_fallback_count() == before + 1
    assert lib.vb200_release_memory(0) == 0


def test_general_matern_large_smoothness_small_distances_stay_finite():
    """nu = 45 at scaled distances down to ~1e-4: K_nu(x) itself is ~1e250 there, x^nu ~1e-180; the device works with
    (x/2)^nu K_nu (bounded) and must agree with a log-space evaluation of the same correlation (advisor finding,
    round 1: the unscaled recurrence overflowed to inf * 0 = NaN)."""
    from scipy.special import gammaln, kve
    rng = np.random.default_rng(12)
    n, m = 400, 12
    locs = rng.uniform(0, 1, (n, 2)) * 1e-3          # tiny domain ...
    locs[::7] += rng.uniform(0, 1, (locs[::7].shape[0], 2)) * 1e-6
    theta = np.array([1.0, 1.0, 45.0, 0.05])          # ... against range 1: x in [1e-6, 1.4e-3]
    y, X = rng.normal(size=n), np.ones((n, 1))
    nn = vg.find_ordered_neighbors(locs, m)
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "matern_isotropic") as prob:
        for layout in _layouts(prob, 4):
            prob.set_layout(layout)
            tot = prob.totals(theta)
            assert np.all(np.isfinite(tot)), layout
    # one observation against a log-space dense evaluation: conditional variance of point 30 given its neighbours
    i = 30
    idx = nn.idx[i][nn.idx[i] >= 0][::-1]              # local frame: neighbours ..., observation last
    P = locs[idx]
    r = np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1)) / theta[1]
    nu = theta[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        logc = (1.0 - nu) * np.log(2.0) - gammaln(nu) + nu * np.log(r) + np.log(kve(nu, r)) - r
    K = theta[0] * np.where(r > 0, np.exp(logc), 1.0) + theta[0] * theta[3] * np.eye(len(idx))
    want = np.log(1.0 / np.linalg.inv(K)[-1, -1])
    with DeviceProblem(vg.Dataset(y, X, locs), nn, "matern_isotropic") as prob:
        rows, flags = prob.rows_host(theta, 0.0, i, i + 1)
    assert flags[0] == 0
    assert rows[0][0] == pytest.approx(want, rel=1e-6, abs=1e-6)   # logdet contribution = log of the conditional variance
