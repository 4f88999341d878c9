"""Pins of the oracle's SOMF iteration (Alg. 3 + Alg. 4) and objective (not gpu).

What the paper fixes, and the pin used:
  * Eq. (a) estimators: brute-force sums on tiny inputs; Monte-Carlo
    unbiasedness E[G] = D^T D, E[beta] = D^T x.
  * Cbar: symmetric PSD; w_t = 1/t gives the running mean.
  * Bbar modes: M leaves unmasked rows untouched; F equals the full OMF rule
    (partition identity, P:602 + P:612); U (R6) is unbiased for F over the
    masks (Monte Carlo, E[M_t] = I) and equals F and M at r = 1.
  * Alg. 4: freezing of unmasked rows; feasibility (Eq. 2);
    n_j = 1 - ||d_j||; surrogate non-increase on the masked rows
    (P:1175-1186); k = 1 and Cbar = I interior cases; full mask => radius 1.
  * Whole step: r = 1 reduces to the separately written OMF (Alg. 1).
  * Objective: D = 0; exact representation at lambda = 0; brute-force
    per-sample minimisation on a tiny instance (Eq. 3).
  * Trajectory (cfgA): the test objective decreases (sanity only: the paper
    prints no trajectory; parity of trajectories is GPU-vs-oracle).
"""
import numpy as np
import pytest
from scipy.optimize import minimize

import synth
from oracle.prox import enet_value, enet_projection, solve_codes
from oracle.somf import SomfOracle, OracleConfig, objective, surrogate_value
from oracle.omf import OmfOracle
from oracle.streams import mask_rows


def test_estimator_a_brute_force_tiny():
    p, k, eta, r = 13, 3, 2, 3.0
    rng = np.random.default_rng(1)
    X = rng.standard_normal((p, eta))
    cfg = OracleConfig(p=p, k=k, eta=eta, lam=0.5, nu=1.0, mu=1.0, r=r, seed=5)
    o = SomfOracle(cfg)
    o.set_components(rng.standard_normal((p, k)) * 0.1)
    D = o.D.copy()
    out = o.partial_fit(X)
    S = out["S"]
    G = np.zeros((k, k))
    beta = np.zeros((k, eta))
    for i in range(p):
        m = r if i in set(S.tolist()) else 0.0      # diagonal of M_t
        for a in range(k):
            for b in range(k):
                G[a, b] += D[i, a] * m * D[i, b]
            for s in range(eta):
                beta[a, s] += D[i, a] * m * X[i, s]
    np.testing.assert_allclose(out["G"], G, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(out["beta"], beta, rtol=1e-13, atol=1e-15)


def test_estimator_a_unbiased():
    """E over masks of r D[S]^T D[S] = D^T D and of r D[S]^T x = D^T x."""
    p, k, r = 400, 3, 4.0
    rng = np.random.default_rng(2)
    D = rng.standard_normal((p, k))
    x = rng.standard_normal(p)
    T = 3000
    Gs = np.empty((T, k, k))
    bs = np.empty((T, k))
    for t in range(1, T + 1):
        S = mask_rows(7, t, p, r)
        Gs[t - 1] = r * D[S].T @ D[S]
        bs[t - 1] = r * D[S].T @ x[S]
    for est, exact in ((Gs, D.T @ D), (bs, D.T @ x)):
        mean = est.mean(axis=0)
        se = est.std(axis=0) / np.sqrt(T)
        assert np.all(np.abs(mean - exact) < 4 * se + 1e-12)


def test_cbar_psd_and_running_mean():
    p, k, eta = 40, 5, 3
    cfg = OracleConfig(p=p, k=k, eta=eta, lam=0.1, nu=1.0, mu=0.0, r=2.0, u=1.0, seed=3)
    o = SomfOracle(cfg)
    rng = np.random.default_rng(3)
    o.set_components(rng.standard_normal((p, k)))
    acc = np.zeros((k, k))
    for t in range(1, 31):
        out = o.partial_fit(rng.standard_normal((p, eta)))
        acc += out["A"] @ out["A"].T / eta
        np.testing.assert_allclose(o.Cbar, acc / t, rtol=1e-12, atol=1e-14)  # w_t = 1/t
        np.testing.assert_array_equal(o.Cbar, o.Cbar.T)
        assert np.linalg.eigvalsh(o.Cbar).min() >= -1e-10


@pytest.mark.parametrize("mode", ["M", "F", "U"])
def test_bbar_modes(mode):
    p, k, eta = 50, 4, 6
    rng = np.random.default_rng(4)
    cfg = OracleConfig(p=p, k=k, eta=eta, lam=0.2, nu=1.0, mu=1.0, r=3.0, b_mode=mode, seed=9)
    o = SomfOracle(cfg)
    o.set_components(rng.standard_normal((p, k)))
    o.partial_fit(rng.standard_normal((p, eta)))
    B0 = o.Bbar.copy()
    # freeze the dictionary update to inspect Bbar alone
    o._partial_dictionary_update = lambda S, perm: None
    X = rng.standard_normal((p, eta))
    out = o.partial_fit(X)
    S, A, w = out["S"], out["A"], out["w"]
    notS = np.setdiff1d(np.arange(p), S)
    full_rule = (1 - w) * B0 + (w / eta) * X @ A.T                 # Eq. omf-parameter-update
    if mode == "M":
        np.testing.assert_array_equal(o.Bbar[notS], B0[notS])
        np.testing.assert_allclose(o.Bbar[S], full_rule[S], rtol=1e-13, atol=1e-15)
    elif mode == "F":
        np.testing.assert_allclose(o.Bbar, full_rule, rtol=1e-13, atol=1e-15)
    else:
        np.testing.assert_allclose(o.Bbar[notS], (1 - w) * B0[notS], rtol=1e-14)
        np.testing.assert_allclose(o.Bbar[S], (1 - w) * B0[S] + (w * 3.0 / eta) * X[S] @ A.T,
                                   rtol=1e-13, atol=1e-15)


def test_bbar_mode_u_reduces_to_f_at_r1():
    """r = 1 selects every row (Eq. mt): the unbiased mode U, the masked mode M
    and Alg. 3's full mode F are then one rule (reading R5/R6) -- whole
    trajectories, dictionary updates included, agree to rounding."""
    p, k, eta = 40, 3, 5
    rng = np.random.default_rng(12)
    X = rng.standard_normal((p, 200))
    outs = {}
    for mode in ("U", "M", "F"):
        o = SomfOracle(OracleConfig(p=p, k=k, eta=eta, lam=0.1, nu=1.0, mu=0.0, r=1.0, b_mode=mode, seed=4))
        o.set_components(X[:, :k])
        for t in range(12):
            o.partial_fit(X[:, k + t * eta:k + (t + 1) * eta])
        outs[mode] = (o.D.copy(), o.Bbar.copy(), o.Cbar.copy())
    for mode in ("M", "F"):
        for a, b in zip(outs["U"], outs[mode]):
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)


def test_bbar_mode_u_unbiased_monte_carlo(monkeypatch):
    """Mode U's point (SURVEY 8c ledger 5-6): E over masks of its Bbar equals
    Alg. 3's full-mode Bbar (P:602 + P:612), because E[M_t] = I.
    With the codes held fixed (so they do not depend on the mask) and Alg. 4
    frozen, the mean of mode-U Bbar over 3000 independent mask streams must
    equal the deterministic mode-F Bbar within 4 standard errors; a dropped r,
    a missing decay of the unmasked rows or a wrong weight fails it."""
    import oracle.somf as osomf
    p, k, eta, r, steps = 24, 2, 3, 3.0, 4
    rng = np.random.default_rng(21)
    D0 = rng.standard_normal((p, k))
    Xs = [rng.standard_normal((p, eta)) for _ in range(steps)]
    As = [rng.standard_normal((k, eta)) for _ in range(steps)]
    it = {"i": 0}

    def fixed_codes(G, beta, *a, **kw):
        return As[it["i"]].copy()
    monkeypatch.setattr(osomf, "solve_codes", fixed_codes)

    def run(mode, seed):
        o = SomfOracle(OracleConfig(p=p, k=k, eta=eta, lam=0.1, nu=1.0, mu=1.0, r=r, b_mode=mode, seed=seed))
        o.set_components(D0)
        o._partial_dictionary_update = lambda S, perm: None
        for t in range(steps):
            it["i"] = t
            o.partial_fit(Xs[t])
        return o.Bbar
    ref = run("F", 0)
    draws = np.stack([run("U", 1000 + s) for s in range(3000)])
    mean = draws.mean(axis=0)
    se = draws.std(axis=0, ddof=1) / np.sqrt(draws.shape[0])
    assert np.all(np.abs(mean - ref) <= 4.0 * se + 1e-12), np.max(np.abs(mean - ref) / (se + 1e-30))
    # and the estimator is not degenerate: single draws differ from F
    assert np.max(np.abs(draws[0] - ref)) > 1e-3


@pytest.mark.parametrize("mu,pos", [(0.0, False), (1.0, False), (0.5, False), (1.0, True), (0.0, True)])
def test_alg4_invariants(mu, pos):
    """Freezing, feasibility, slack bookkeeping and surrogate non-increase."""
    p, k, eta = 120, 6, 8
    rng = np.random.default_rng(5)
    cfg = OracleConfig(p=p, k=k, eta=eta, lam=0.05, nu=1.0, pos_code=pos, mu=mu,
                       pos_dict=pos, r=4.0, seed=21)
    o = SomfOracle(cfg)
    X0 = np.abs(rng.standard_normal((p, 200))) if pos else rng.standard_normal((p, 200))
    o.set_components(X0[:, :k])
    for t in range(25):
        X = X0[:, rng.integers(0, 200, eta)]
        D_before = o.D.copy()
        # surrogate with the new statistics, before / after Alg. 4
        captured = {}
        orig = o._partial_dictionary_update

        def hooked(S, perm):
            captured["S"] = S
            captured["g0"] = surrogate_value(o.D[S], o.Bbar[S], o.Cbar)
            orig(S, perm)
            captured["g1"] = surrogate_value(o.D[S], o.Bbar[S], o.Cbar)
        o._partial_dictionary_update = hooked
        o.partial_fit(X)
        o._partial_dictionary_update = orig
        S = captured["S"]
        notS = np.setdiff1d(np.arange(p), S)
        np.testing.assert_array_equal(o.D[notS], D_before[notS])      # freezing
        assert captured["g1"] <= captured["g0"] + 1e-12 * (1 + abs(captured["g0"]))
        for j in range(k):
            nrm = enet_value(o.D[:, j], mu)
            assert nrm <= 1 + 1e-10                                   # feasibility
            assert abs(o.n[j] - (1 - nrm)) < 1e-10                    # slack norms
        if pos:
            assert o.D.min() >= 0


def test_alg4_full_mask_radius_is_one():
    p, k = 30, 3
    rng = np.random.default_rng(6)
    cfg = OracleConfig(p=p, k=k, eta=4, lam=0.1, nu=1.0, mu=0.0, r=1.0, seed=2)
    o = SomfOracle(cfg)
    o.set_components(rng.standard_normal((p, k)))
    for j in range(k):
        assert o.n[j] + enet_value(o.D[:, j], 0.0) == pytest.approx(1.0, abs=1e-14)


def test_alg4_interior_cases():
    """k = 1 interior: d = bbar / cbar.  Cbar = I interior: D[S] = Bbar[S]."""
    p = 20
    rng = np.random.default_rng(7)
    for k, Cbar in ((1, np.array([[2.0]])), (3, np.eye(3))):
        cfg = OracleConfig(p=p, k=k, eta=1, mu=1.0, r=1.0, seed=1)
        o = SomfOracle(cfg)
        o.set_components(np.zeros((p, k)))
        o.Cbar = Cbar
        o.Bbar = rng.standard_normal((p, k)) * 0.05
        S = np.arange(p)
        o._partial_dictionary_update(S, np.arange(k))
        np.testing.assert_allclose(o.D, o.Bbar / np.diag(Cbar), rtol=1e-14)


def test_dead_atom_is_skipped():
    p, k = 25, 3
    rng = np.random.default_rng(8)
    cfg = OracleConfig(p=p, k=k, eta=1, mu=0.0, r=1.0, seed=1)
    o = SomfOracle(cfg)
    o.set_components(rng.standard_normal((p, k)))
    D0 = o.D.copy()
    o.Cbar = np.diag([1.0, 0.0, 1.0])
    o.Bbar = rng.standard_normal((p, k))
    o._partial_dictionary_update(np.arange(p), np.array([1, 0, 2]))
    np.testing.assert_array_equal(o.D[:, 1], D0[:, 1])


@pytest.mark.parametrize("nu,mu,pos", [(1.0, 0.0, False), (0.0, 1.0, False), (1.0, 1.0, True)])
def test_r1_reduces_to_omf(nu, mu, pos):
    """SOMF with M_t = I (r = 1) is OMF (Alg. 3 -> Alg. 1)."""
    p, k, eta = 40, 5, 6
    rng = np.random.default_rng(9)
    X0 = rng.standard_normal((p, 300))
    if pos:
        X0 = np.abs(X0)
    cfg = OracleConfig(p=p, k=k, eta=eta, lam=0.1, nu=nu, pos_code=pos, mu=mu, pos_dict=pos,
                       r=1.0, u=0.917, seed=4)
    s = SomfOracle(cfg)
    o = OmfOracle(k, 0.1, nu, mu, pos, pos, u=0.917, seed=4)
    s.set_components(X0[:, :k])
    o.set_components(X0[:, :k])
    for t in range(40):
        X = X0[:, (t * eta) % 294:(t * eta) % 294 + eta]
        s.partial_fit(X)
        o.partial_fit(X)
        np.testing.assert_allclose(s.D, o.D, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(s.Bbar, o.B, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(s.Cbar, o.C, rtol=1e-10, atol=1e-12)


def test_objective_closed_forms():
    rng = np.random.default_rng(10)
    X = rng.standard_normal((15, 7))
    assert objective(np.zeros((15, 3)), X, 0.1, 0.0) == pytest.approx(
        0.5 * (X ** 2).sum(axis=0).mean(), rel=1e-14)
    x = X[:, :1]
    D = x / np.linalg.norm(x)
    assert objective(D, x, 0.0, 0.0) == pytest.approx(0.0, abs=1e-20)


def test_objective_brute_force_tiny():
    rng = np.random.default_rng(11)
    p, m, k = 8, 5, 3
    X = rng.standard_normal((p, m))
    D = rng.standard_normal((p, k))
    for lam, nu, pos in ((0.3, 0.0, False), (0.3, 1.0, False), (0.2, 0.5, True)):
        vals = []
        for s in range(m):
            def f(a):
                return (0.5 * ((X[:, s] - D @ a) ** 2).sum()
                        + lam * ((1 - nu) * np.abs(a).sum() + 0.5 * nu * (a * a).sum()))
            best = np.inf
            for start in (np.zeros(k), np.linalg.lstsq(D, X[:, s], rcond=None)[0]):
                res = minimize(f, start, method="Powell",
                               bounds=[(0, None)] * k if pos else None,
                               options={"xtol": 1e-12, "ftol": 1e-14, "maxiter": 100000})
                best = min(best, res.fun)
            vals.append(best)
        assert objective(D, X, lam, nu, pos) == pytest.approx(np.mean(vals), rel=1e-7)


def test_trajectory_sanity_cfgA():
    """cfgA: ridge lambda = 0.1, l1-ball atoms, k = eta = 10; the held-out
    objective decreases along the epoch, for OMF (r = 1) and SOMF (r = 4, masked
    Bbar mode) alike (sanity only)."""
    X, _, _ = synth.tiny_dictionary_learning(seed=0)
    Xtr, Xte = X[:, :1800], X[:, 1800:]
    for r, drop in ((1.0, 0.9), (4.0, 0.995)):
        cfg = OracleConfig(p=256, k=10, eta=10, lam=0.1, nu=1.0, mu=0.0, r=r, u=0.95, seed=0)
        o = SomfOracle(cfg)
        o.set_components(Xtr[:, :10])
        vals = [o.objective(Xte)]
        for t in range(180):
            o.partial_fit(Xtr[:, t * 10:(t + 1) * 10])
            if t % 60 == 59:
                vals.append(o.objective(Xte))
        assert all(b < a for a, b in zip(vals[:-1], vals[1:])), vals
        assert vals[-1] < drop * vals[0]
