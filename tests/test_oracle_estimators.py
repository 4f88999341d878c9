"""Pins of the oracle's code-step estimators (b) and (c) (§III-B,
P:683-781, Table I) against what the paper fixes, not against themselves:

  * Eq. (c): the maintained Gram equals D^T D of the current
    dictionary -- recomputed from scratch -- after 1000 partial updates;
  * Eq. (b): beta^(i) equals the closed-form weighted sum
    sum_s gamma_{s,t} D_{s-1}^T M_s x^(i) with gamma_{s,t} = gamma_{c_s}
    prod_{later visits} (1 - gamma_c), built here from recorded dictionaries
    and independently drawn masks; the weights sum to 1;
  * special cases: every sample seen once => (b) is (a) for any r (gamma = 1
    overwrites), and (c) is (a) at r = 1 (the masked Gram is the exact one).
"""
import numpy as np
import pytest

import synth
from oracle import streams
from oracle.somf import SomfOracle, OracleConfig


def _data(p=200, n=300, seed=0):
    X, _, _ = synth.tiny_dictionary_learning(p=p, n=n, k_true=6, seed=seed)
    return X


def test_exact_gram_identity_after_1000_updates():
    p, k, eta, n = 120, 8, 6, 240
    X = _data(p, n + k)
    o = SomfOracle(OracleConfig(p=p, k=k, eta=eta, lam=0.05, nu=1.0, mu=0.0, r=6.0, estimator="c",
                                n_samples=n, seed=3))
    o.set_components(X[:, :k])
    rng = np.random.default_rng(1)
    for t in range(1000):
        ids = rng.choice(n, size=eta, replace=False)
        o.partial_fit(X[:, k + ids], ids)
    G = o.D.T @ o.D
    assert np.abs(o.G_exact - G).max() <= 1e-10 * max(1.0, np.abs(G).max())


@pytest.mark.parametrize("estimator", ["b", "c"])
def test_averaged_beta_is_the_closed_form_weighted_sum(estimator):
    p, k, eta, n, v, r = 150, 7, 5, 12, 0.751, 4.0
    X = _data(p, n + k, seed=2)
    seed = 5
    o = SomfOracle(OracleConfig(p=p, k=k, eta=eta, lam=0.1, nu=1.0, mu=0.0, r=r, estimator=estimator,
                                n_samples=n, v=v, seed=seed))
    o.set_components(X[:, :k])
    rng = np.random.default_rng(0)
    visits = {i: [] for i in range(n)}          # sample -> [(t, D_{t-1})]
    for t in range(1, 41):
        ids = rng.choice(n, size=eta, replace=False)
        D_prev = o.D.copy()
        for i in ids:
            visits[i].append((t, D_prev))
        o.partial_fit(X[:, k + ids], ids)
    for i in range(n):
        if not visits[i]:
            continue
        x = X[:, k + i]
        c = len(visits[i])
        gam = [float(j) ** (-v) for j in range(1, c + 1)]
        total = np.zeros(k)
        wsum = 0.0
        for j, (t, D_prev) in enumerate(visits[i]):
            S = streams.mask_rows(seed, t, p, r)                 # M_t (Eq. mt), drawn independently
            b = r * D_prev[S].T @ x[S]                           # D_{t-1}^T M_t x^(i)
            wgt = gam[j] * np.prod([1.0 - gam[l] for l in range(j + 1, c)])
            total += wgt * b
            wsum += wgt
        assert abs(wsum - 1.0) <= 1e-12
        assert np.allclose(o.beta_avg[i], total, rtol=0, atol=1e-12 * max(1.0, np.abs(total).max()))
        assert o.count[i] == c


def test_single_visit_b_reduces_to_a():
    p, k, eta = 180, 6, 5
    X = _data(p, 40 * eta + k, seed=4)
    kw = dict(p=p, k=k, eta=eta, lam=0.1, nu=0.0, mu=1.0, r=3.0, seed=2)
    oa = SomfOracle(OracleConfig(**kw))
    ob = SomfOracle(OracleConfig(estimator="b", n_samples=40 * eta, **kw))
    oa.set_components(X[:, :k])
    ob.set_components(X[:, :k])
    for t in range(40):
        ids = np.arange(t * eta, (t + 1) * eta)
        batch = X[:, k + ids]
        ra = oa.partial_fit(batch)
        rb = ob.partial_fit(batch, ids)
        assert np.allclose(rb["A"], ra["A"], rtol=0, atol=1e-10)
    assert np.allclose(ob.D, oa.D, rtol=0, atol=1e-10)


def test_single_visit_c_reduces_to_a_at_r1():
    p, k, eta = 160, 6, 5
    X = _data(p, 30 * eta + k, seed=6)
    kw = dict(p=p, k=k, eta=eta, lam=0.1, nu=1.0, mu=0.0, r=1.0, seed=2)
    oa = SomfOracle(OracleConfig(**kw))
    oc = SomfOracle(OracleConfig(estimator="c", n_samples=30 * eta, **kw))
    oa.set_components(X[:, :k])
    oc.set_components(X[:, :k])
    for t in range(30):
        ids = np.arange(t * eta, (t + 1) * eta)
        ra = oa.partial_fit(X[:, k + ids])
        rc = oc.partial_fit(X[:, k + ids], ids)
        assert np.allclose(rc["G"], ra["G"], rtol=0, atol=1e-10)
        assert np.allclose(rc["A"], ra["A"], rtol=0, atol=1e-9)


def test_duplicate_ids_in_a_batch_rejected():
    p, k, eta = 50, 3, 4
    X = _data(p, 20, seed=1)
    o = SomfOracle(OracleConfig(p=p, k=k, eta=eta, estimator="c", n_samples=10))
    o.set_components(X[:, :k])
    with pytest.raises(ValueError):
        o.partial_fit(X[:, 3:7], np.array([1, 2, 2, 3]))
