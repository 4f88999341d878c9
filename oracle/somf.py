"""Subsampled online matrix factorisation, Alg. 3 + Alg. 4, float64.

TEST INFRASTRUCTURE (see oracle/__init__.py).

One call of ``SomfOracle.partial_fit(X)`` is one iteration t of Alg. 3
 with estimator (a) (Eq. a) on a mini-batch of eta
columns, followed by Alg. 4 on the masked
rows.  Statement order follows the paper:

    t <- t + 1 ; w_t = t^-u
    draw M_t (Eq. mt)
    G = D^T M_t D ; beta = D^T M_t X  (M_t = r on S)         Eq. (a)
    alpha_s = argmin 1/2 a^T G a - a^T beta_s + lam Omega(a) Eq. somf_alpha
    Cbar <- (1-w) Cbar + w mean_s alpha_s alpha_s^T          Eq. somf_partial
    P_t Bbar <- (1-w) P_t Bbar + w mean_s P_t x_s alpha_s^T  Eq. somf_partial
    [mode F: also P_t^perp Bbar, P:612 ; mode U: reading R6]
    Alg. 4 on the rows S, atoms in permutation order

Estimators of the code step (Table I), ``estimator``:
  (a) masked    G = D^T M_t D, beta = D^T M_t x              Eq. (a)
  (b) averaged  per-sample G^(i), beta^(i):                  Eq. (b)
                c^(i) += 1, gamma = c^(i)^-v,
                beta^(i) <- (1-gamma) beta^(i) + gamma D^T M_t x^(i)
                G^(i)    <- (1-gamma) G^(i)    + gamma D^T M_t D
  (c) exact Gram + averaged beta^(i): G = D_{t-1}^T D_{t-1},  Eq. (c)
                maintained through Alg. 4's partial update:
                G <- G - P_t D_old^T P_t D_old + P_t D_new^T P_t D_new
with gamma_c = c^-v (v = 0.751 P:1361).  Readings R23-R25
(DESIGN.md §2): Alg. 3's "beta^(i) <- (1-gamma) G^(i)_{t-1}" is read as
beta^(i)_{t-1} (SURVEY ledger 17); the averages start at c = 1 where gamma = 1
overwrites them; the ids of one mini-batch must be distinct (the mini-batch
extension P:633-636 applies the per-sample rule once per sample).

Readings: R1-R2 mask, R4 batch means, R5/R6 Bbar modes,
R7 literal Eq. 2 norm, R9 radius, R10 dead atoms, R11 radius 0, R13 order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .prox import enet_value, enet_projection, solve_codes
from .streams import mask_rows, atom_permutation

B_MODES = ("M", "F", "U")


@dataclass
class OracleConfig:
    p: int
    k: int
    eta: int
    lam: float = 0.1          # lambda, code penalty strength          (Eq. 1)
    nu: float = 1.0           # Omega mix: 1 = ridge, 0 = lasso         (Eq. 2)
    pos_code: bool = False    # alpha >= 0
    mu: float = 0.0           # atom norm mix: 0 = l1 ball, 1 = l2 ball (Eq. 2)
    pos_dict: bool = False    # D >= 0
    r: float = 1.0            # reduction factor
    u: float = 0.917          # w_t = t^-u
    b_mode: str = "M"         # Bbar rows updated: M masked, F full, U unbiased
    perm_cyclic: bool = False
    seed: int = 0
    estimator: str = "a"      # code-step estimator: a masked, b averaged, c exact Gram (Table I)
    n_samples: int = 0        # n: sample ids in [0, n) (estimators b / c)
    v: float = 0.751          # gamma_c = c^-v


def surrogate_value(D, Bbar, Cbar) -> float:
    """1/2 Tr(D^T D Cbar) - Tr(D^T Bbar): the part of gbar_t that depends on D
    (P:323-327)."""
    return float(0.5 * np.trace(D.T @ D @ Cbar) - np.trace(D.T @ Bbar))


def objective(D, X, lam: float, nu: float, pos_code: bool = False,
              tol: float = 1e-12) -> float:
    """fbar(D) = mean_s min_alpha 1/2 ||x_s - D alpha||^2 + lam Omega(alpha).

    Eq. (3); the held-out evaluation of P:1322-1326.  Codes are
    solved tightly from G* = D^T D, beta* = D^T x (Eq. regression);
    the residual is formed directly, not through the Gram identity.
    """
    D = np.asarray(D, np.float64)
    X = np.asarray(X, np.float64)
    A = solve_codes(D.T @ D, D.T @ X, lam, nu, pos_code, tol=tol)
    R = X - D @ A
    pen = (1.0 - nu) * np.abs(A).sum(axis=0) + 0.5 * nu * (A * A).sum(axis=0)
    return float(np.mean(0.5 * (R * R).sum(axis=0) + lam * pen))


def transform(D, X, lam: float, nu: float, pos_code: bool = False,
              tol: float = 1e-12):
    """Codes of X on D with the exact G*, beta* (Eq. regression)."""
    D = np.asarray(D, np.float64)
    X = np.asarray(X, np.float64)
    return solve_codes(D.T @ D, D.T @ X, lam, nu, pos_code, tol=tol)


class SomfOracle:
    """State: D (p x k), Bbar (p x k), Cbar (k x k), slack norms n (k), t."""

    def __init__(self, cfg: OracleConfig):
        if cfg.r < 1.0 or cfg.k < 1 or cfg.eta < 1 or cfg.lam < 0.0:
            raise ValueError("invalid configuration")
        if not (0.0 <= cfg.nu <= 1.0 and 0.0 <= cfg.mu <= 1.0 and 0.0 < cfg.u <= 1.0):
            raise ValueError("invalid mixing / weight parameter")
        if cfg.b_mode not in B_MODES:
            raise ValueError("b_mode must be one of M, F, U")
        if cfg.estimator not in ("a", "b", "c"):
            raise ValueError("estimator must be one of a, b, c")
        if cfg.estimator != "a" and cfg.n_samples < 1:
            raise ValueError("estimators b / c need n_samples >= 1")
        self.cfg = cfg
        p, k = cfg.p, cfg.k
        self.D = np.zeros((p, k))
        self.Bbar = np.zeros((p, k))
        self.Cbar = np.zeros((k, k))
        self.n = np.ones(k)
        self.t = 0
        self.cd_tol = 1e-12
        self._reset_estimator()

    def _reset_estimator(self):
        """Per-sample statistics of estimators (b) / (c): visit counts c^(i),
        averaged beta^(i) (n x k), averaged G^(i) (n x k x k, (b) only) and the
        exact Gram G = D^T D ((c) only)."""
        c = self.cfg
        n = c.n_samples if c.estimator != "a" else 0
        self.count = np.zeros(n, dtype=np.int64)
        self.beta_avg = np.zeros((n, c.k))
        self.G_avg = np.zeros((n, c.k, c.k)) if c.estimator == "b" else None
        self.G_exact = self.D.T @ self.D if c.estimator == "c" else None

    # -- state ---------------------------------------------------------------
    def set_components(self, D0):
        """D_0 projected atom-wise onto C (reading R15); n_j = 1 - ||d_j||
        (P:850-851); Bbar = 0, Cbar = 0, t = 0 (w_1 = 1 overwrites them)."""
        c = self.cfg
        D0 = np.asarray(D0, np.float64)
        self.D = np.empty_like(D0)
        for j in range(c.k):
            self.D[:, j] = enet_projection(D0[:, j], 1.0, c.mu, c.pos_dict)
        self.n = np.array([1.0 - enet_value(self.D[:, j], c.mu) for j in range(c.k)])
        self.Bbar = np.zeros_like(self.D)
        self.Cbar = np.zeros((c.k, c.k))
        self.t = 0
        self._reset_estimator()

    def set_state(self, D, Bbar, Cbar, n, t):
        self.D = np.array(D, np.float64)
        self.Bbar = np.array(Bbar, np.float64)
        self.Cbar = np.array(Cbar, np.float64)
        self.n = np.array(n, np.float64)
        self.t = int(t)
        self._reset_estimator()

    # -- one iteration of Alg. 3 -------------------------------------------------
    def partial_fit(self, X, ids=None):
        """One SOMF iteration on the batch X (p x eta) whose columns are the
        samples ``ids`` (estimators b / c).  Returns the step's intermediates
        (S, G, beta, A, perm, w) for parity tests; for (b) G is per column
        (eta x k x k)."""
        c = self.cfg
        X = np.asarray(X, np.float64)
        eta = X.shape[1]
        self.t += 1
        t = self.t
        w = float(t) ** (-c.u)
        S = mask_rows(c.seed, t, c.p, c.r)                       # Eq. (mt)
        DS = self.D[S]
        XS = X[S]
        G = c.r * (DS.T @ DS)                                    # Eq. (a)
        beta = c.r * (DS.T @ XS)
        if c.estimator == "a":
            A = solve_codes(G, beta, c.lam, c.nu, c.pos_code, tol=self.cd_tol)
        else:
            ids = np.asarray(ids, dtype=np.int64)
            if ids.shape != (eta,) or ids.min() < 0 or ids.max() >= c.n_samples:
                raise ValueError("ids must hold eta sample ids in [0, n_samples)")
            if np.unique(ids).size != eta:
                raise ValueError("the ids of one mini-batch must be distinct (reading R25)")
            beta_used = np.empty_like(beta)
            G_used = np.empty((eta, c.k, c.k)) if c.estimator == "b" else None
            for s_, i in enumerate(ids):
                self.count[i] += 1
                gamma = float(self.count[i]) ** (-c.v)
                self.beta_avg[i] = (1.0 - gamma) * self.beta_avg[i] + gamma * beta[:, s_]
                beta_used[:, s_] = self.beta_avg[i]
                if c.estimator == "b":
                    self.G_avg[i] = (1.0 - gamma) * self.G_avg[i] + gamma * G
                    G_used[s_] = self.G_avg[i]
            if c.estimator == "b":                               # Eq. (b): a Gram per column
                A = np.empty_like(beta)
                for s_ in range(eta):
                    A[:, s_] = solve_codes(G_used[s_], beta_used[:, s_], c.lam, c.nu, c.pos_code,
                                           tol=self.cd_tol)
                G = G_used
            else:                                                # Eq. (c): the exact Gram D_{t-1}^T D_{t-1}
                G = self.G_exact.copy()
                A = solve_codes(G, beta_used, c.lam, c.nu, c.pos_code, tol=self.cd_tol)
            beta = beta_used
        self.Cbar = (1.0 - w) * self.Cbar + (w / eta) * (A @ A.T)  # Eq. somf_partial
        if c.b_mode == "M":
            self.Bbar[S] = (1.0 - w) * self.Bbar[S] + (w / eta) * (XS @ A.T)
        elif c.b_mode == "F":
            self.Bbar[S] = (1.0 - w) * self.Bbar[S] + (w / eta) * (XS @ A.T)
            notS = np.setdiff1d(np.arange(c.p), S, assume_unique=True)
            self.Bbar[notS] = (1.0 - w) * self.Bbar[notS] + (w / eta) * (X[notS] @ A.T)
        else:  # "U": E[M_t X A^T] = X A^T (reading R6)
            self.Bbar *= (1.0 - w)
            self.Bbar[S] += (w * c.r / eta) * (XS @ A.T)
        perm = atom_permutation(c.seed, t, c.k, c.perm_cyclic)
        DS_old = self.D[S].copy()
        self._partial_dictionary_update(S, perm)
        if c.estimator == "c":
            # the Gram of D_t from that of D_{t-1}: only the rows S changed
            DS_new = self.D[S]
            self.G_exact = self.G_exact - DS_old.T @ DS_old + DS_new.T @ DS_new
        return dict(S=S, G=G, beta=beta, A=A, perm=perm, w=w)

    def _partial_dictionary_update(self, S, perm):
        """Alg. 4 on the rows S, one pass over the atoms."""
        c = self.cfg
        if S.size == 0:
            return
        Cbar = self.Cbar
        DS = self.D[S].copy()          # P_t D_t, updated in place atom by atom
        BS = self.Bbar[S]              # P_t Bbar_t
        dmax = max(1.0, float(np.max(np.diag(Cbar))))
        for j in perm:
            if Cbar[j, j] <= 1e-12 * dmax:                       # reading R10
                continue
            rho = max(0.0, self.n[j] + enet_value(DS[:, j], c.mu))     # P:860, R9
            u = DS[:, j] + (BS[:, j] - DS @ Cbar[:, j]) / Cbar[j, j]
            d = enet_projection(u, rho, c.mu, c.pos_dict)
            DS[:, j] = d
            self.n[j] = rho - enet_value(d, c.mu)
        self.D[S] = DS                 # P_t^perp D_t = P_t^perp D_{t-1}

    # -- evaluation ----------------------------------------------------------------
    def objective(self, X) -> float:
        c = self.cfg
        return objective(self.D, X, c.lam, c.nu, c.pos_code)

    def transform(self, X):
        c = self.cfg
        return transform(self.D, X, c.lam, c.nu, c.pos_code)

    def surrogate(self) -> float:
        return surrogate_value(self.D, self.Bbar, self.Cbar)
