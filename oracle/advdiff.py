"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy / scipy restatement of the reference's stationary advection-diffusion
source-inversion oracle (proj/include/h2/oracles/advdiff2d.hpp, registry
"advdiff-<G>[-k<kappa>][-obs<N>]", registry.hpp:125-150). Used by tests/ as the
checker; the product path is csrc/advdiff.cu.

The misfit Hessian H = (1/sigma^2) C^T A^{-T} B^T B A^{-1} C (advdiff2d.hpp:5-11)
is applied here exactly as the reference does: one forward and one adjoint
sparse LU solve per application (scipy's SuperLU in place of Eigen's SparseLU).
"""
import random

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class AdvDiff2D:
    """AdvDiff2D(cfg) (advdiff2d.hpp:21-46); keyword names follow AdvDiff2DConfig (:21-28)."""

    def __init__(self, grid=32, kappa=1e-3, reaction=0.5, num_observations=100, noise_rel=0.01, obs_seed=7):
        if kappa <= 0:
            raise ValueError("advdiff: kappa must be positive")
        if grid < 4:
            raise ValueError("grid: need at least 4 nodes per side")
        self.g, self.kappa, self.reaction = int(grid), float(kappa), float(reaction)
        self.num_observations, self.noise_rel, self.obs_seed = int(num_observations), float(noise_rel), int(obs_seed)
        self.h = 1.0 / (self.g + 1)
        self.h2 = self.h * self.h
        self._assemble()
        self.obs = self._pick_observations()
        self.sigma = self._calibrate_noise()
        self.solves = 0

    @property
    def n(self):
        return self.g * self.g

    def index(self, i, j):   # grid.hpp:36
        return (j - 1) * self.g + (i - 1)

    def points(self):
        i = np.tile(np.arange(1, self.g + 1), self.g)
        j = np.repeat(np.arange(1, self.g + 1), self.g)
        return np.stack([self.h * i, self.h * j], axis=1)

    def _assemble(self):   # :76-110, first-order upwind, Dirichlet inflow / Neumann outflow
        g, h, k = self.g, self.h, self.kappa
        rows, cols, vals = [], [], []
        for j in range(1, g + 1):
            for i in range(1, g + 1):
                row = self.index(i, j)
                v1, v2 = h * i, h * j
                diag = 4.0 * k / (h * h) + (v1 + v2) / h + self.reaction
                if i > 1:
                    rows.append(row); cols.append(self.index(i - 1, j)); vals.append(-k / (h * h) - v1 / h)
                if i < g:
                    rows.append(row); cols.append(self.index(i + 1, j)); vals.append(-k / (h * h))
                else:
                    diag -= k / (h * h)
                if j > 1:
                    rows.append(row); cols.append(self.index(i, j - 1)); vals.append(-k / (h * h) - v2 / h)
                if j < g:
                    rows.append(row); cols.append(self.index(i, j + 1)); vals.append(-k / (h * h))
                else:
                    diag -= k / (h * h)
                rows.append(row); cols.append(row); vals.append(diag)
        self.A = sp.csc_matrix(sp.coo_matrix((vals, (rows, cols)), shape=(self.n, self.n)))
        self.lu = spla.splu(self.A)
        self.lu_t = spla.splu(sp.csc_matrix(self.A.T))

    def _pick_observations(self):   # :112-124: std::shuffle with std::mt19937_64(obs_seed)
        from oracle.pyoracle import shuffle_indices
        g = self.g
        interior = [self.index(i, j) for j in range(2, g) for i in range(2, g)]
        if self.num_observations > len(interior):
            raise ValueError("advdiff: more observations than interior nodes")
        perm = shuffle_indices(len(interior), self.obs_seed)
        return sorted(interior[p] for p in perm[:self.num_observations])

    def _calibrate_noise(self):   # :126-139
        g, h = self.g, self.h
        m = np.zeros(self.n)
        for j in range(1, g + 1):
            for i in range(1, g + 1):
                dx, dy = h * i - 0.35, h * j - 0.7
                m[self.index(i, j)] = np.exp(-(dx * dx + dy * dy) / (2 * 0.08 * 0.08))
        u = self.lu.solve(self.h2 * m)
        peak = max(abs(u[o]) for o in self.obs)
        return max(self.noise_rel * peak, 1e-12)

    def solve_state(self, m):   # :48-52
        self.solves += 1
        return self.lu.solve(self.h2 * np.asarray(m, np.float64))

    def misfit_hessvec(self, nu):   # :54-64
        nu = np.asarray(nu, np.float64)
        y = self.lu.solve(self.h2 * nu)
        self.solves += 1
        by = np.zeros_like(y)
        by[self.obs] = y[self.obs]
        z = self.lu_t.solve(by / (self.sigma * self.sigma))
        self.solves += 1
        return self.h2 * z
