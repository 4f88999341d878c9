"""Online matrix factorisation, Alg. 1, mini-batch form.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Written separately from ``somf.py`` as the r = 1 reference: SOMF with M_t = I
reduces to it (P:559-566 with r = 1; P:819-829 gives radius 1 for every atom).
It uses the same weight sequence w_t = t^-u and the same atom
order as SOMF so the two can be compared iterate by iterate.
"""
import numpy as np

from .prox import enet_projection, solve_codes
from .streams import atom_permutation


class OmfOracle:
    def __init__(self, k, lam, nu, mu, pos_code=False, pos_dict=False,
                 u=0.917, seed=0, perm_cyclic=False):
        self.k, self.lam, self.nu, self.mu = k, lam, nu, mu
        self.pos_code, self.pos_dict = pos_code, pos_dict
        self.u, self.seed, self.perm_cyclic = u, seed, perm_cyclic
        self.t = 0

    def set_components(self, D0):
        D0 = np.asarray(D0, np.float64)
        self.D = np.stack([enet_projection(D0[:, j], 1.0, self.mu, self.pos_dict)
                           for j in range(self.k)], axis=1)
        self.B = np.zeros_like(self.D)
        self.C = np.zeros((self.k, self.k))
        self.t = 0

    def partial_fit(self, X):
        X = np.asarray(X, np.float64)
        eta = X.shape[1]
        self.t += 1
        w = float(self.t) ** (-self.u)
        # code computation on the full sample (Alg. 1 line 2)
        A = solve_codes(self.D.T @ self.D, self.D.T @ X, self.lam, self.nu,
                        self.pos_code, tol=1e-12)
        # surrogate parameters, Eq. (omf-parameter-update) with weights w_t
        self.C = (1.0 - w) * self.C + (w / eta) * (A @ A.T)
        self.B = (1.0 - w) * self.B + (w / eta) * (X @ A.T)
        # one pass of projected block coordinate descent
        dmax = max(1.0, float(np.max(np.diag(self.C))))
        for j in atom_permutation(self.seed, self.t, self.k, self.perm_cyclic):
            if self.C[j, j] <= 1e-12 * dmax:
                continue
            g = self.B[:, j] - self.D @ self.C[:, j]
            self.D[:, j] = enet_projection(self.D[:, j] + g / self.C[j, j], 1.0,
                                           self.mu, self.pos_dict)
        return A
