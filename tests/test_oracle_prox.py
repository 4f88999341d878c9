"""Pins of the oracle's elastic-net value, projection and code solver (not gpu).

Projection (Alg. 4): hand-checkable closed forms
(tests/golden), brute force by a general constrained solver (scipy SLSQP) on
tiny vectors, the mu = 1 closed-form scaling, an independent l1-ball
bisection for mu = 0, idempotence and feasibility.
Codes (Eq. somf_alpha): closed forms, normal-equation residual for
ridge, KKT conditions for lasso / elastic net / non-negative codes, and
scikit-learn's ElasticNet on the equivalent least-squares problem.
"""
import json
import os

import numpy as np
import pytest
from scipy.optimize import minimize

from oracle.prox import enet_value, enet_projection, solve_codes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "closed_form_examples.json")))


def test_golden_enet_value():
    for ex in GOLD["enet_value"]:
        assert enet_value(ex["v"], ex["mix"]) == pytest.approx(ex["value"], abs=1e-15)


def test_enet_value_is_convex_combination():
    rng = np.random.default_rng(0)
    for _ in range(50):
        v = rng.standard_normal(11)
        m = rng.random()
        assert enet_value(v, m) == pytest.approx(
            (1 - m) * enet_value(v, 0.0) + m * enet_value(v, 1.0), rel=1e-14)


def test_golden_projection():
    for ex in GOLD["enet_projection"]:
        d = enet_projection(ex["u"], ex["radius"], ex["mu"], ex["positive"])
        np.testing.assert_allclose(d, ex["d"], atol=1e-12)


def _brute_projection(u, radius, mu, positive):
    """General-purpose constrained solver on the same problem."""
    n = u.size
    x0 = np.zeros(n)
    cons = [{"type": "ineq",
             "fun": lambda d: radius - ((1 - mu) * np.sqrt(d * d + 1e-30).sum()
                                        + 0.5 * mu * (d * d).sum())}]
    bounds = [(0, None)] * n if positive else None
    best = None
    for start in (x0, np.clip(u, 0, None) if positive else u * 0.1):
        res = minimize(lambda d: 0.5 * ((d - u) ** 2).sum(), start, jac=lambda d: d - u,
                       constraints=cons, bounds=bounds, method="SLSQP",
                       options={"ftol": 1e-14, "maxiter": 1000})
        if best is None or res.fun < best.fun:
            best = res
    return best.x


def test_projection_is_optimal_vs_general_solver():
    """Our point is feasible and at least as close to u as any feasible point a
    general-purpose constrained solver (SLSQP) finds; where SLSQP converges to
    a feasible point the two agree."""
    rng = np.random.default_rng(1)
    agreed = 0
    for trial in range(160):
        n = rng.integers(1, 6)
        u = rng.standard_normal(n) * rng.choice([0.3, 1.0, 3.0])
        mu = [0.0, 1.0, 0.5, rng.random()][trial % 4]
        radius = rng.choice([0.2, 0.5, 1.0])
        positive = bool(trial % 3 == 0)
        d = enet_projection(u, radius, mu, positive)
        assert enet_value(d, mu) <= radius * (1 + 1e-12)
        ref = _brute_projection(u, radius, mu, positive)
        if enet_value(ref, mu) <= radius + 1e-9 and (not positive or ref.min() >= -1e-12):
            f_d = 0.5 * ((d - u) ** 2).sum()
            f_ref = 0.5 * ((ref - u) ** 2).sum()
            assert f_d <= f_ref * (1 + 1e-8) + 1e-9
            np.testing.assert_allclose(d, ref, atol=1e-4)
            agreed += 1
    assert agreed > 100


def _kkt_bisection(u, rho, mu, positive):
    """lam by bisection on phi(lam) = N(d(lam)) - rho, d(lam) the KKT map."""
    v = np.maximum(u, 0) if positive else u
    a, b = 1 - mu, mu
    dmap = lambda lam: np.sign(v) * np.maximum(np.abs(v) - a * lam, 0) / (1 + b * lam)
    if enet_value(v, mu) <= rho:
        return v
    lo, hi = 0.0, 1.0
    while enet_value(dmap(hi), mu) > rho:
        hi *= 2
    for _ in range(300):
        mid = 0.5 * (lo + hi)
        if enet_value(dmap(mid), mu) > rho:
            lo = mid
        else:
            hi = mid
    return dmap(hi)


def test_projection_matches_kkt_bisection():
    rng = np.random.default_rng(11)
    for trial in range(400):
        u = rng.standard_t(3, size=rng.integers(1, 100)) * rng.choice([0.1, 1.0, 5.0])
        mu = [0.0, 1.0, 0.5, rng.random()][trial % 4]
        rho = rng.random() * 2 + 1e-3
        positive = bool(trial % 5 == 0)
        np.testing.assert_allclose(enet_projection(u, rho, mu, positive),
                                   _kkt_bisection(u, rho, mu, positive), atol=1e-11)


def test_projection_mu1_is_radial_scaling():
    rng = np.random.default_rng(2)
    for _ in range(100):
        u = rng.standard_normal(rng.integers(1, 40)) * 3
        rho = rng.random() + 0.01
        d = enet_projection(u, rho, 1.0)
        nrm2 = (u * u).sum()
        if 0.5 * nrm2 <= rho:
            np.testing.assert_array_equal(d, u)
        else:
            np.testing.assert_allclose(d, u * np.sqrt(2 * rho / nrm2), rtol=1e-12, atol=1e-15)


def _l1_ball_bisection(u, rho):
    lo, hi = 0.0, np.abs(u).max()
    for _ in range(200):
        th = 0.5 * (lo + hi)
        if np.maximum(np.abs(u) - th, 0).sum() > rho:
            lo = th
        else:
            hi = th
    th = 0.5 * (lo + hi)
    return np.sign(u) * np.maximum(np.abs(u) - th, 0)


def test_projection_mu0_matches_bisection():
    rng = np.random.default_rng(3)
    for _ in range(200):
        u = rng.standard_t(3, size=rng.integers(1, 300))
        rho = rng.random() * 2 + 1e-3
        d = enet_projection(u, rho, 0.0)
        if np.abs(u).sum() <= rho:
            np.testing.assert_array_equal(d, u)
        else:
            np.testing.assert_allclose(d, _l1_ball_bisection(u, rho), atol=1e-12)


@pytest.mark.parametrize("mu", [0.0, 0.3, 0.5, 1.0])
@pytest.mark.parametrize("positive", [False, True])
def test_projection_feasible_idempotent(mu, positive):
    rng = np.random.default_rng(4)
    for _ in range(100):
        u = rng.standard_normal(rng.integers(1, 200)) * rng.choice([0.1, 1, 10])
        rho = rng.random() * 1.5
        d = enet_projection(u, rho, mu, positive)
        assert enet_value(d, mu) <= rho + 1e-10
        if positive:
            assert np.all(d >= 0)
        d2 = enet_projection(d, rho, mu, positive)
        np.testing.assert_allclose(d2, d, atol=1e-12)
        # variational inequality: <u - d, y - d> <= 0 for feasible y (here y = 0 and y = d/2)
        for y in (np.zeros_like(d), 0.5 * d):
            assert np.dot(u - d, y - d) <= 1e-9 * (1 + np.abs(u).sum())


def test_golden_codes():
    for ex in GOLD["solve_codes"]:
        a = solve_codes(np.array(ex["G"], float), np.array(ex["beta"], float),
                        ex["lam"], ex["nu"], ex["positive"])
        np.testing.assert_allclose(a, ex["alpha"], atol=1e-12)


def _spd(rng, k, cond=20.0):
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    ev = np.geomspace(1.0, 1.0 / cond, k)
    return (Q * ev) @ Q.T


def test_ridge_normal_equations():
    rng = np.random.default_rng(5)
    for k in (1, 3, 10, 40):
        G = _spd(rng, k)
        beta = rng.standard_normal((k, 7))
        lam = 0.3
        a = solve_codes(G, beta, lam, 1.0)
        np.testing.assert_allclose((G + lam * np.eye(k)) @ a, beta, atol=1e-11)


def _kkt_residual(G, beta, alpha, lam, nu, positive):
    g = beta - G @ alpha - lam * nu * alpha       # minus gradient of smooth part
    l1 = lam * (1 - nu)
    res = 0.0
    for j in range(alpha.size):
        if positive:
            if alpha[j] > 0:
                res = max(res, abs(g[j] - l1))
            else:
                res = max(res, g[j] - l1)
        else:
            if alpha[j] != 0:
                res = max(res, abs(g[j] - l1 * np.sign(alpha[j])))
            else:
                res = max(res, abs(g[j]) - l1)
    return res


@pytest.mark.parametrize("nu", [0.0, 0.2, 1.0])
@pytest.mark.parametrize("positive", [False, True])
def test_cd_satisfies_kkt(nu, positive):
    rng = np.random.default_rng(6)
    for _ in range(20):
        k = rng.integers(2, 25)
        G = _spd(rng, k, cond=50)
        beta = rng.standard_normal(k)
        lam = rng.random() * 0.5 + 0.01
        a = solve_codes(G, beta, lam, nu, positive)
        assert _kkt_residual(G, beta, a, lam, nu, positive) < 1e-9
        if positive:
            assert np.all(a >= 0)


def test_cd_lam0_equals_linear_solve():
    rng = np.random.default_rng(7)
    G = _spd(rng, 12)
    beta = rng.standard_normal((12, 3))
    a = solve_codes(G, beta, 0.0, 0.0)
    np.testing.assert_allclose(a, np.linalg.solve(G, beta), atol=1e-8)


def test_cd_identity_gram_is_soft_threshold():
    rng = np.random.default_rng(8)
    beta = rng.standard_normal((9, 4))
    a = solve_codes(np.eye(9), beta, 0.4, 0.0)
    np.testing.assert_allclose(a, np.sign(beta) * np.maximum(np.abs(beta) - 0.4, 0), atol=1e-14)


def test_codes_match_sklearn_elastic_net():
    """sklearn minimises 1/(2m)||y - Xw||^2 + a l1r ||w||_1 + a(1-l1r)/2 ||w||^2.
    With y = x, X = D and m samples this equals ours / m with
    a l1r = lam(1-nu)/m, a(1-l1r) = lam nu / m."""
    from sklearn.linear_model import ElasticNet
    rng = np.random.default_rng(9)
    for positive in (False, True):
        m, k = 60, 8
        D = rng.standard_normal((m, k))
        x = D @ rng.standard_normal(k) + 0.1 * rng.standard_normal(m)
        lam, nu = 2.0, 0.3
        a = solve_codes(D.T @ D, D.T @ x, lam, nu, positive)
        alpha_sk = lam / m
        l1r = 1 - nu
        en = ElasticNet(alpha=alpha_sk, l1_ratio=l1r, fit_intercept=False, tol=1e-14,
                        max_iter=200000, positive=positive)
        en.fit(D, x)
        np.testing.assert_allclose(a, en.coef_, atol=1e-7)


def test_codes_ill_conditioned_nonneg_reach_the_minimiser():
    """NMF-shaped Gram (cfgD: correlated nonnegative atoms, cond ~1e3-1e4):
    plain CD stalls far from the minimiser at its sweep cap, so the oracle's
    answer (reading R14b) is checked against the KKT conditions and against
    scipy's NNLS (Lawson-Hanson) on the equivalent least-squares problem
    min 1/2 |L^T a - L^-1 beta|^2, a >= 0, with L L^T = G + lam I."""
    from scipy.optimize import nnls
    rng = np.random.default_rng(12)
    p, k = 1500, 64
    W = np.abs(rng.standard_normal((p, 40))) * (rng.random((p, 40)) < 0.3)
    X = W @ rng.exponential(1.0, (40, k + 6)) + np.abs(0.1 * rng.standard_normal((p, k + 6)))
    D = X[:, :k] / np.linalg.norm(X[:, :k], axis=0)    # atoms = data columns (bench D0)
    X = X[:, k:]
    G, beta = 8.0 * D.T @ D, 8.0 * D.T @ X
    lam = 0.05
    ev = np.linalg.eigvalsh(G + lam * np.eye(k))
    assert ev[-1] / ev[0] > 1e3                       # the hard regime
    a = solve_codes(G, beta, lam, 1.0, positive=True, max_sweeps=40)   # CD alone stalls here
    L = np.linalg.cholesky(G + lam * np.eye(k))
    for s in range(beta.shape[1]):
        assert _kkt_residual(G, beta[:, s], a[:, s], lam, 1.0, True) < 1e-8
        ref, _ = nnls(L.T, np.linalg.solve(L, beta[:, s]))
        np.testing.assert_allclose(a[:, s], ref, atol=1e-7 * max(1.0, np.abs(ref).max()))
