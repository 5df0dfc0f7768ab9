"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy / scipy restatement of the reference's minimal-surface oracle
(proj/include/h2/oracles/minimal_surface.hpp, registry.hpp:89-101), the
`surface<N>` Hessian operator of the registry. Used by tests/ and bench.py's
CPU legs as the checker; the product path is csrc/surface.cu.

Every function cites the reference lines it follows. Sparse assembly sums
duplicate triplets like Eigen's setFromTriplets (scipy's coo -> csr does the
same: duplicates are added).
"""
import math

import numpy as np
import scipy.sparse as sp


class MinimalSurface:
    """MinimalSurface(interior, rim_amplitude) (minimal_surface.hpp:22-43)."""

    def __init__(self, interior, rim=0.5):
        if interior < 4:   # Grid2D (grid.hpp:31-33)
            raise ValueError("grid: need at least 4 nodes per side")
        self.g = int(interior)
        self.rim = float(rim)
        nn = self.g + 2
        hh = self.h
        b = np.zeros((nn, nn))
        rim_at = lambda s: self.rim * math.sin(2 * math.pi * s)
        for i in range(nn):   # :30-35
            x = hh * i
            b[i, 0] = rim_at(x / 4.0)
            b[i, nn - 1] = rim_at((2.0 + (1.0 - x)) / 4.0)
        for j in range(nn):   # :36-40
            y = hh * j
            b[nn - 1, j] = rim_at((1.0 + y) / 4.0)
            b[0, j] = rim_at((3.0 + (1.0 - y)) / 4.0)
        self.boundary = b

    # Grid2D (grid.hpp:28-50)
    @property
    def h(self):
        return 1.0 / (self.g + 1)

    @property
    def n(self):
        return self.g * self.g

    def index(self, i, j):
        return (j - 1) * self.g + (i - 1)

    def points(self):
        i = np.tile(np.arange(1, self.g + 1), self.g)
        j = np.repeat(np.arange(1, self.g + 1), self.g)
        return np.stack([self.h * i, self.h * j], axis=1)

    def set_boundary(self, f):   # :46-56
        nn = self.g + 2
        h = self.h
        for i in range(nn):
            self.boundary[i, 0] = f(h * i, 0.0)
            self.boundary[i, nn - 1] = f(h * i, 1.0)
            self.boundary[0, i] = f(0.0, h * i)
            self.boundary[nn - 1, i] = f(1.0, h * i)

    def full_field(self, m):   # :59-65; f(i, j) = m[index(i, j)] inside the rim
        f = self.boundary.copy()
        f[1:-1, 1:-1] = np.asarray(m, np.float64).reshape(self.g, self.g).T
        return f

    def _cells(self, m):
        f = self.full_field(m)
        h = self.h
        gx = (f[1:, :-1] - f[:-1, :-1]) / h   # cell (cx, cy): forward differences
        gy = (f[:-1, 1:] - f[:-1, :-1]) / h
        return gx, gy

    def value(self, m):   # :67-78
        gx, gy = self._cells(m)
        h = self.h
        # the reference accumulates cell by cell, cx fastest
        return float(np.sum((h * h * np.sqrt(1.0 + gx * gx + gy * gy)).T))

    def gradient(self, m):   # :80-98
        gx, gy = self._cells(m)
        h = self.h
        nn = self.g + 2
        r = h / np.sqrt(1.0 + gx * gx + gy * gy)
        g = np.zeros((nn, nn))
        for cy in range(nn - 1):
            for cx in range(nn - 1):
                g[cx + 1, cy] += r[cx, cy] * gx[cx, cy]
                g[cx, cy] -= r[cx, cy] * (gx[cx, cy] + gy[cx, cy])
                g[cx, cy + 1] += r[cx, cy] * gy[cx, cy]
        return g[1:-1, 1:-1].T.reshape(-1).copy()

    def hessian(self, m):   # :100-140, exact sparse Hessian w.r.t. the interior unknowns
        gx, gy = self._cells(m)
        h = self.h
        nn = self.g + 2
        rows, cols, vals = [], [], []

        def interior_index(i, j):
            if i < 1 or i > self.g or j < 1 or j > self.g:
                return -1
            return self.index(i, j)

        gxd = (-1.0 / h, 1.0 / h, 0.0)
        gyd = (-1.0 / h, 0.0, 1.0 / h)
        for cy in range(nn - 1):
            for cx in range(nn - 1):
                a_, b_ = gx[cx, cy], gy[cx, cy]
                f2 = 1.0 + a_ * a_ + b_ * b_
                fr = math.sqrt(f2)
                wxx = (f2 - a_ * a_) / (f2 * fr)
                wyy = (f2 - b_ * b_) / (f2 * fr)
                wxy = -a_ * b_ / (f2 * fr)
                ids = (interior_index(cx, cy), interior_index(cx + 1, cy), interior_index(cx, cy + 1))
                for p in range(3):
                    if ids[p] < 0:
                        continue
                    for q in range(3):
                        if ids[q] < 0:
                            continue
                        v = h * h * (wxx * gxd[p] * gxd[q] + wyy * gyd[p] * gyd[q] +
                                     wxy * (gxd[p] * gyd[q] + gyd[p] * gxd[q]))
                        if v != 0.0:
                            rows.append(ids[p])
                            cols.append(ids[q])
                            vals.append(v)
        return sp.coo_matrix((vals, (rows, cols)), shape=(self.n, self.n)).tocsr()

    def newton_state(self, steps):   # :144-161, damped Newton from a flat start
        m = np.zeros(self.n)
        for _ in range(steps):
            g = self.gradient(m)
            hs = self.hessian(m)
            d = sp.linalg.spsolve(hs.tocsc(), g)
            alpha = 1.0
            j0 = self.value(m)
            while alpha > 1e-6 and self.value(m - alpha * d) >= j0:
                alpha /= 2
            m = m - alpha * d
        return m


def make_surface(name, config=None):
    """make_oracle("surface<N>") (registry.hpp:89-101): the Hessian at the
    newton_state(newton_steps) surface; returns (surface, state, sparse Hessian)."""
    cfg = dict(config or {})
    ms = MinimalSurface(int(name[7:]), float(cfg.get("rim", 0.5)))
    state = ms.newton_state(int(cfg.get("newton_steps", 0)))
    return ms, state, ms.hessian(state)
