"""Elastic-net value, elastic-net-ball projection and code regression.

TEST INFRASTRUCTURE (see oracle/__init__.py).  float64 throughout.
"""
import numpy as np


def enet_value(v, mix: float) -> float:
    """(1 - mix) ||v||_1 + mix/2 ||v||_2^2.

    Eq. (2): both the code penalty Omega (mix = nu) and the atom
    "norm" ||d|| of the constraint set C (mix = mu) have this form.  Literal
    Eq. 2 is used for mix = 1 (reading R7: the l2 ball has radius sqrt 2).
    """
    v = np.asarray(v, dtype=np.float64)
    return float((1.0 - mix) * np.abs(v).sum() + 0.5 * mix * (v * v).sum())


def enet_projection(u, radius: float, mu: float, positive: bool = False):
    """Euclidean projection of u onto {d : (1-mu)||d||_1 + mu/2 ||d||^2 <= radius}
    (intersected with d >= 0 when ``positive``).

    Alg. 4 line "P_t d <- enet_projection(u, r_t^(j))" and P:847-848;
    the paper defers the algorithm to [Mairal 2010].  Written out from the
    KKT conditions (reading R17): with a = 1-mu, b = mu the solution is
    d_i = sign(v_i) max(|v_i| - a lam, 0) / (1 + b lam), v = u (or max(u, 0)),
    where lam >= 0 is 0 if v is feasible, else the root of
        (a^2 b s/2 + rho b^2) lam^2 + (a^2 s + 2 rho b) lam - (a S1 + b S2/2 - rho) = 0
    for the active set of the s largest |v_i| (S1 = sum |v_i|, S2 = sum v_i^2
    over it), s being the first size with |v|_(s+1) <= a lam < |v|_(s).
    The sort below is the textbook way to find s; radius 0 returns 0.
    """
    u = np.asarray(u, dtype=np.float64)
    if radius < 0.0:
        raise ValueError("radius must be >= 0")
    v = np.maximum(u, 0.0) if positive else u.copy()
    if enet_value(v, mu) <= radius:
        return v
    if radius == 0.0:
        return np.zeros_like(v)
    a, b = 1.0 - mu, mu
    z = np.sort(np.abs(v))[::-1]
    z = z[z > 0.0]
    n = z.size
    s = np.arange(1, n + 1, dtype=np.float64)
    S1 = np.cumsum(z)
    S2 = np.cumsum(z * z)
    A = a * a * b * s / 2.0 + radius * b * b
    B = a * a * s + 2.0 * radius * b
    C = a * S1 + b * S2 / 2.0 - radius
    lam_s = 2.0 * C / (B + np.sqrt(B * B + 4.0 * A * C))
    nxt = np.append(z[1:], 0.0)
    ok = (nxt <= a * lam_s) & (a * lam_s < z)
    hit = np.flatnonzero(ok)
    # no size qualifies only when v is infeasible by a rounding error (the sums
    # above are accumulated in another order than enet_value's): lam ~ 0.
    lam = lam_s[hit[0]] if hit.size else max(0.0, lam_s[-1])
    return np.sign(v) * np.maximum(np.abs(v) - a * lam, 0.0) / (1.0 + b * lam)


def solve_codes(G, beta, lam: float, nu: float, positive: bool = False,
                tol: float = 1e-12, max_sweeps: int = 10000):
    """alpha_s = argmin 1/2 a^T G a - a^T beta_s + lam Omega(a), column-wise.

    Eq. (somf_alpha), P:592-596 (and Eq. regression, with the exact
    G*, beta*).  ``beta`` is k x m.  The minimiser is the definition:
      * ridge (nu = 1, no positivity): the closed form (G + lam I)^-1 beta;
      * otherwise cyclic coordinate descent (the paper's solver)
        from alpha = 0: z_j = beta_j - sum_{l != j} G_jl alpha_l,
        alpha_j = S_{lam(1-nu)}(z_j) / (G_jj + lam nu)  (nonneg: max(z_j -
        lam(1-nu), 0) / (G_jj + lam nu)), alpha_j = 0 if the denominator is 0
        (reading R12), until max|delta| <= tol max(1, ||alpha||_inf) for every
        column or ``max_sweeps``; a column that then fails the KKT conditions
        is finished as reading R14b below.  Columns are independent problems;
        they are swept together only to vectorise.
    """
    G = np.asarray(G, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    squeeze = beta.ndim == 1
    if squeeze:
        beta = beta[:, None]
    k = G.shape[0]
    if nu == 1.0 and not positive:
        out = np.linalg.solve(G + lam * np.eye(k), beta)
        return out[:, 0] if squeeze else out
    l1 = lam * (1.0 - nu)
    l2 = lam * nu
    alpha = np.zeros_like(beta)
    g = beta.copy()                      # g = beta - G alpha

    def cd(cols, nsweeps):
        """cyclic CD sweeps on the columns ``cols`` until tol or nsweeps"""
        a, gg = alpha[:, cols], g[:, cols]
        for _ in range(nsweeps):
            maxd = np.zeros(a.shape[1])
            for j in range(k):
                den = G[j, j] + l2
                z = gg[j] + G[j, j] * a[j]
                if den <= 0.0:
                    new = np.zeros_like(z)
                elif positive:
                    new = np.maximum(z - l1, 0.0) / den
                else:
                    new = np.sign(z) * np.maximum(np.abs(z) - l1, 0.0) / den
                d = new - a[j]
                if np.any(d != 0.0):
                    a[j] = new
                    gg -= np.outer(G[:, j], d)
                    np.maximum(maxd, np.abs(d), out=maxd)
            scale = np.maximum(1.0, np.abs(a).max(axis=0))
            if np.all(maxd <= tol * scale):
                break
        alpha[:, cols], g[:, cols] = a, gg

    # Reading R14b: on ill-conditioned problems (the cfgD NMF Gram, cond ~5e3)
    # CD's per-sweep contraction is ~1 - 1e-3 and the sweep cap stops it short
    # of the minimiser.  A column whose KKT conditions fail is finished on its
    # CD support: the minimiser's nonzeros solve (G_SS + l2 I) a_S = beta_S -
    # l1 sign_S, and that solution is accepted only if the KKT conditions of
    # the whole problem then hold (convex problem: KKT <=> argmin);
    # otherwise CD continues from where it stopped (checked every 500 sweeps).
    cols = np.arange(beta.shape[1])
    chunk = min(max_sweeps, 500)
    for _ in range(50 * -(-max_sweeps // chunk)):
        cd(cols, chunk)
        cols = cols[kkt_residual(G, beta[:, cols], alpha[:, cols], lam, nu, positive) > 1e-9]
        still = []
        for s in cols:
            S = np.flatnonzero(alpha[:, s])
            ok = False
            if S.size:
                sg = np.sign(alpha[S, s])
                y = np.linalg.solve(G[np.ix_(S, S)] + l2 * np.eye(S.size), beta[S, s] - l1 * sg)
                if np.all(np.sign(y) == sg):
                    cand = np.zeros(k)
                    cand[S] = y
                    if kkt_residual(G, beta[:, s], cand, lam, nu, positive)[0] <= 1e-9:
                        alpha[:, s] = cand
                        g[:, s] = beta[:, s] - G @ cand
                        ok = True
            if not ok:
                still.append(s)
        cols = np.asarray(still, dtype=np.int64)
        if cols.size == 0:
            break
    return alpha[:, 0] if squeeze else alpha


def kkt_residual(G, beta, alpha, lam: float, nu: float, positive: bool = False):
    """Largest violation, per column, of the optimality conditions of
    min 1/2 a^T G a - a^T beta + lam[(1-nu)|a|_1 + nu/2 |a|^2] (a >= 0 if
    ``positive``), scaled by max(1, |beta|_inf): with g = beta - G a - lam nu a,
    g_j = lam(1-nu) sign(a_j) where a_j != 0, |g_j| <= lam(1-nu) (g_j <= lam(1-nu)
    if positive) where a_j = 0."""
    G = np.asarray(G, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    if beta.ndim == 1:
        beta, alpha = beta[:, None], alpha[:, None]
    l1, l2 = lam * (1.0 - nu), lam * nu
    g = beta - G @ alpha - l2 * alpha
    on = alpha != 0.0
    v_on = np.where(on, np.abs(g - l1 * np.sign(alpha)), 0.0)
    v_off = np.where(on, 0.0, np.maximum(0.0, (g if positive else np.abs(g)) - l1))
    scale = np.maximum(1.0, np.abs(beta).max(axis=0))
    return np.maximum(v_on, v_off).max(axis=0) / scale
