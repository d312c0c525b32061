"""Pin the CPU oracle (oracle/) against fixtures generated from the UNMODIFIED
reference (tests/golden/make_golden.py).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import numpy_families, vecchia_oracle as vo

CASES = ["iso_d2_p2_m9", "iso_d2_p1_m30", "iso_d3_p4_m30", "aniso_d3_p2_m8", "aniso_d2_p1_m20",
         "sphere_p1_m12", "iso_jitter", "iso_heads_only", "iso_wide_m79", "iso_zero_nugget",
         "iso_d1_m5", "iso_m60"]


def _case(z, name):
    g = lambda k: z[f"{name}/{k}"]
    return dict(y=g("y"), X=g("X"), locs=g("locs_work"), nn=g("nn"), theta=g("theta"),
                family=str(g("family")), jitter=float(g("jitter")))


@pytest.mark.parametrize("name", CASES)
def test_totals_bit_identical_to_reference_compiled_core(engine_cases, name):
    c = _case(engine_cases, name)
    got = vo.run(c["y"], c["X"], c["locs"], c["nn"], c["family"], c["theta"], jitter=c["jitter"],
                 deterministic=True, workers=3)
    want = engine_cases[f"{name}/totals_compiled"]
    assert np.array_equal(got, want), np.max(np.abs(got - want))


@pytest.mark.parametrize("name", CASES)
def test_per_observation_rows_match_reference_numpy_core(engine_cases, name):
    c = _case(engine_cases, name)
    want = engine_cases[f"{name}/rows_fallback"]
    rows, fail = vo.observations(c["y"], c["X"], c["locs"], c["nn"], c["family"], c["theta"],
                                 jitter=c["jitter"], i0=0, i1=want.shape[0])
    assert not fail.any()
    np.testing.assert_allclose(rows, want, rtol=1e-9, atol=1e-11)
    # the second (numpy) oracle agrees as well
    p, q = c["X"].shape[1], c["theta"].shape[0]
    mine = np.stack([numpy_families.contribution(i, c["y"], c["X"], c["locs"], c["nn"], c["family"],
                                                 c["theta"], c["jitter"]) for i in range(min(12, want.shape[0]))])
    np.testing.assert_allclose(mine, want[:mine.shape[0]], rtol=1e-9, atol=1e-11)
    assert rows.shape[1] == vo.acc_len(p, q)


@pytest.mark.parametrize("name", CASES)
def test_assemble_matches_reference(engine_cases, name):
    c = _case(engine_cases, name)
    tot = engine_cases[f"{name}/totals_compiled"]
    p, q = c["X"].shape[1], c["theta"].shape[0]
    ev = vo.assemble(tot, c["y"].shape[0], p, q)
    assert ev["loglik"] == pytest.approx(float(engine_cases[f"{name}/loglik_compiled"]), rel=1e-13)
    np.testing.assert_allclose(ev["grad"], engine_cases[f"{name}/grad_compiled"], rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(ev["beta"], engine_cases[f"{name}/beta_compiled"], rtol=1e-10)


def test_failure_reports_lowest_observation_and_pivot(failure_case):
    z = failure_case
    n = z["y"].shape[0]
    with pytest.raises(vo.OracleNotPositiveDefinite) as err:
        vo.run(z["y"], np.ones((n, 1)), z["locs"], z["nn"], "exponential_isotropic", z["theta"])
    assert err.value.observation == int(z["observation_compiled"]) == 7
    assert err.value.pivot == int(z["pivot_compiled"])
    got = vo.run(z["y"], np.ones((n, 1)), z["locs"], z["nn"], "exponential_isotropic", z["theta"], jitter=1e-6)
    assert np.array_equal(got, z["rescued_totals"])


@pytest.mark.parametrize("name", ["grid7", "grid3d", "rand2d", "rand3d", "line", "dups"])
def test_neighbor_scan_matches_reference(neighbor_cases, name):
    z = neighbor_cases
    got = vo.neighbor_scan(z[f"{name}/locs"], int(z[f"{name}/m"]), workers=2)
    assert np.array_equal(got, z[f"{name}/idx"])


def test_known_answers_from_reference_tests():
    # k = 1 closed form (reference tests/test_engine.py:93-104)
    sig2, rho, tau2 = 1.7, 0.3, 0.2
    y = np.array([0.8]); X = np.array([[1.0]]); locs = np.array([[0.1, 0.2]])
    nn = np.array([[0]], dtype=np.int64)
    rows, _ = vo.observations(y, X, locs, nn, "exponential_isotropic", [sig2, rho, tau2])
    P = vo.split_acc(rows[0], 1, 3)
    v = sig2 * (1 + tau2)
    assert float(P["logdet"]) == pytest.approx(np.log(v), rel=1e-14)
    assert float(P["ysy"]) == pytest.approx(0.64 / v, rel=1e-14)
    assert P["xsx"][0, 0] == pytest.approx(1 / v, rel=1e-14)
    # n = 1 loglik (reference tests/test_inference.py:30-38)
    ev = vo.assemble(rows[0], 1, 1, 3)
    # y is fitted exactly by the intercept: quad = 0
    assert ev["loglik"] == pytest.approx(-0.5 * (np.log(2 * np.pi) + np.log(v)), rel=1e-13)


def test_spacetime_is_constrained_anisotropic():
    rng = np.random.default_rng(5)
    n, m = 300, 10
    locs = rng.uniform(0, 1, (n, 3))
    y = rng.normal(size=n); X = np.ones((n, 1))
    nn = vo.neighbor_scan(locs, m)
    th_st = np.array([1.3, 0.25, 0.6, 0.1])
    th_an = np.array([1.3, 0.25, 0.25, 0.6, 0.1])
    a = vo.split_acc(vo.run(y, X, locs, nn, "exponential_anisotropic", th_an), 1, 5)
    s = vo.split_acc(vo.run(y, X, locs, nn, "exponential_spacetime", th_st), 1, 4)
    J = np.zeros((5, 4)); J[0, 0] = J[1, 1] = J[2, 1] = J[3, 2] = J[4, 3] = 1.0
    for k in ("logdet", "ysy", "xsx", "ysx"):
        np.testing.assert_allclose(s[k], a[k], rtol=1e-13)
    np.testing.assert_allclose(s["dlogdet"], a["dlogdet"] @ J, rtol=1e-11)
    np.testing.assert_allclose(s["dysy"], a["dysy"] @ J, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(s["dysx"], a["dysx"] @ J, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(s["ainfo"], J.T @ a["ainfo"] @ J, rtol=1e-11)


def test_bessel_k_against_scipy_and_closed_forms():
    from scipy.special import kv
    L = vo.lib()
    for nu in (0.2, 0.5, 0.8, 1.0, 1.5, 2.3, 3.7, 5.0, 0.49999, 0.50001, 1e-3, 12.5):
        for x in (1e-8, 1e-3, 0.1, 0.5, 1.0, 1.9999, 2.0, 2.0001, 3.0, 10.0, 50.0, 300.0):
            want = kv(nu, x)
            if np.isfinite(want) and want > 0:
                assert L.vo_bessel_k(nu, x) == pytest.approx(want, rel=2e-13), (nu, x)
    x = 0.7  # K_{1/2}(x) = sqrt(pi/2x) e^-x
    assert L.vo_bessel_k(0.5, x) == pytest.approx(np.sqrt(np.pi / (2 * x)) * np.exp(-x), rel=1e-14)


def test_general_matern_reduces_to_closed_forms():
    rng = np.random.default_rng(3)
    n = 80
    locs = rng.uniform(0, 1, (n, 2)); y = rng.normal(size=n)
    X = np.column_stack([np.ones(n), rng.normal(size=n)])
    nn = vo.neighbor_scan(locs, 12)
    for nu, closed in ((0.5, "exponential_isotropic"), (1.5, "matern15_isotropic"), (2.5, "matern25_isotropic")):
        g = vo.split_acc(vo.run(y, X, locs, nn, "matern_isotropic", [0.9, 0.15, nu, 0.05]), 2, 4)
        c = vo.split_acc(vo.run(y, X, locs, nn, closed, [0.9, 0.15, 0.05]), 2, 3)
        keep = [0, 1, 3]  # variance, range, nugget
        for k in ("logdet", "ysy", "xsx", "ysx"):
            np.testing.assert_allclose(g[k], c[k], rtol=1e-11)
        np.testing.assert_allclose(g["dlogdet"][keep], c["dlogdet"], rtol=1e-9)
        np.testing.assert_allclose(g["dysy"][keep], c["dysy"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(g["ainfo"][np.ix_(keep, keep)], c["ainfo"], rtol=1e-9)


@pytest.mark.parametrize("family", ["matern15_isotropic", "matern25_isotropic", "exponential_spacetime",
                                    "matern_isotropic"])
def test_extension_families_structural(family):
    """Families absent from the reference: C oracle == independent numpy oracle,
    derivative fields == central finite differences, dense exactness at m = n-1
    (the reference's own structural checks, tests/test_engine.py:187-228)."""
    rng = np.random.default_rng(11)
    d = 3 if family == "exponential_spacetime" else 2
    n, m = 40, 39
    locs = rng.uniform(0, 1, (n, d)); y = rng.normal(size=n)
    X = np.column_stack([np.ones(n), rng.normal(size=n)])
    theta = np.array([1.4, 0.3, 0.5, 0.15]) if d == 3 else np.array([1.4, 0.3, 0.15])
    if family == "matern_isotropic":
        theta = np.array([1.4, 0.3, 0.8, 0.15])
    nn = vo.neighbor_scan(locs, m)
    q = theta.shape[0]
    tot = vo.run(y, X, locs, nn, family, theta)
    np.testing.assert_allclose(tot, numpy_families.run(y, X, locs, nn, family, theta), rtol=1e-8, atol=1e-9)
    ev = vo.assemble(tot, n, 2, q)
    dense, beta = numpy_families.dense_loglik(family, theta, y, X, locs)
    assert ev["loglik"] == pytest.approx(dense, rel=1e-9)
    np.testing.assert_allclose(ev["beta"], beta, rtol=1e-8)
    for j in range(q):
        h = 1e-6 * theta[j]
        tp, tm = theta.copy(), theta.copy(); tp[j] += h; tm[j] -= h
        lp = vo.assemble(vo.run(y, X, locs, nn, family, tp), n, 2, q)["loglik"]
        lm = vo.assemble(vo.run(y, X, locs, nn, family, tm), n, 2, q)["loglik"]
        assert ev["grad"][j] == pytest.approx((lp - lm) / (2 * h), rel=2e-5, abs=1e-6)
    # information at full conditioning: 0.5 tr(S^-1 D_j S^-1 D_l)
    K, D = numpy_families.cov_and_derivs(family, theta, locs)
    Ki = np.linalg.inv(K)
    info = np.array([[0.5 * np.trace(Ki @ D[j] @ Ki @ D[l]) for l in range(q)] for j in range(q)])
    np.testing.assert_allclose(ev["info"], info, rtol=1e-7)


KRIGE = ["iso_m10", "iso_m60", "aniso_m20", "sphere_m15", "iso_all"]


@pytest.mark.parametrize("name", KRIGE)
def test_kriging_oracle_matches_reference(krige_cases, name):
    """oracle vo_krige == the unmodified reference's predict.krige (LAPACK Cholesky there, own here)."""
    import paper_2407_02740_b200 as vg
    z = krige_cases
    g = lambda k: z[f"{name}/{k}"]
    fam = vg.covariance_registry(str(g("family")))
    work, ws = fam.prepare_locs(g("locs")), fam.prepare_locs(g("locs_star"))
    for latent in (0, 1):
        mean, sd, nbrs = vo.krige(g("y"), g("X"), work, str(g("family")), g("theta"), g("beta"), ws, g("X_star"),
                                  int(g("m_pred")), latent=latent)
        np.testing.assert_allclose(mean, g(f"mean_latent{latent}"), rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(sd, g(f"sd_latent{latent}"), rtol=1e-10, atol=1e-12)
    # the host neighbour query of the product selects the same rows in the same order
    from paper_2407_02740_b200.preprocess import find_nearest_training
    assert np.array_equal(find_nearest_training(work, ws, int(g("m_pred"))), nbrs)


SIMULATE = ["iso_d2_m10", "iso_d2_m30", "iso_d2_p2_m5", "aniso_d3_m12"]


@pytest.mark.parametrize("name", SIMULATE)
def test_simulation_oracle_matches_reference(simulate_cases, name):
    """oracle simulate_nn_gp == the unmodified reference's oracle.simulate_nn_gp (same PCG64 stream), and the
    product's host neighbour search reproduces the reference's table for the case."""
    import paper_2407_02740_b200 as vg
    from oracle import numpy_families as nf
    z = simulate_cases
    g = lambda k: z[f"{name}/{k}"]
    y = nf.simulate_nn_gp(str(g("family")), g("theta"), g("beta"), g("locs"), g("X"), g("nn"), int(g("seed")))
    np.testing.assert_allclose(y, g("y"), rtol=1e-11, atol=1e-12)
    assert np.array_equal(vg.find_ordered_neighbors(g("locs"), int(g("m"))).idx, g("nn"))

