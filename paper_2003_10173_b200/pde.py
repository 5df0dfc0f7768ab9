"""Device PDE black-box operators (the reference's h2::oracles, SURVEY §8(f)
row 2), computed on the B200 so HARA's operator applies never leave HBM:

* the 1D diffusion density-inversion Hessian of BASELINE cfg3
  (proj/include/h2/oracles/diffusion1d.hpp, Diffusion1D :62-354; registry
  "diff1d-<n>", registry.hpp:104-124). Only the evaluation-point Hessian
  (hessvec_at_target / hessian_operator) is built; the misfit, gradient and
  general-density Hessian are not on the HARA path;
* the minimal-surface Hessian "surface<N>" (minimal_surface.hpp,
  registry.hpp:89-101): assembled once on the host, applied as a sparse
  matrix in HBM;
* the advection-diffusion misfit Hessian "advdiff-<G>" (advdiff2d.hpp,
  registry.hpp:125-150): its observation factor G = (h^2/sigma) B A^{-1} is
  formed once, and every application is y = G^T (G x) in HBM.
"""
import ctypes as C

import numpy as np

from ._lib import AdvDiffConfigC, Diff1DConfigC, H, check, lib
from .construction import LinearOperator


class Diffusion1D:
    """Diffusion1D(cfg) (diffusion1d.hpp:75-112). Keyword names follow
    Diffusion1DConfig (:62-73)."""

    def __init__(self, n=512, steps=512, final_time=30.0, t_p=1.0, t_0=0.0, source_amplitude=1000.0, alpha=3e-5,
                 beta=1e-3, pad=0.5, source_positions=None, num_receivers=8):
        c = Diff1DConfigC()
        lib.h2c_diff1d_config_default(C.byref(c))
        c.n, c.steps, c.final_time, c.t_p, c.t_0 = int(n), int(steps), float(final_time), float(t_p), float(t_0)
        c.source_amplitude, c.alpha, c.beta, c.pad = float(source_amplitude), float(alpha), float(beta), float(pad)
        c.num_receivers = int(num_receivers)
        self._src = None
        if source_positions is not None:
            self._src = np.ascontiguousarray(source_positions, np.float64)
            c.num_sources = len(self._src)
            c.source_positions = self._src.ctypes.data_as(C.POINTER(C.c_double))
        h = H()
        check(lib.h2c_diff1d_create(C.byref(c), None, C.byref(h)))
        self._h = h
        self._n = int(n)
        self.steps = int(steps)
        self.config = dict(n=n, steps=steps, final_time=final_time, t_p=t_p, t_0=t_0,
                           source_amplitude=source_amplitude, alpha=alpha, beta=beta, pad=pad,
                           source_positions=source_positions, num_receivers=num_receivers)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_diff1d_destroy(self._h)
            self._h = None

    def _info(self):
        ns, npad, h, dt, m = C.c_int64(), C.c_int64(), C.c_double(), C.c_double(), C.c_int64()
        check(lib.h2c_diff1d_info(self._h, C.byref(ns), C.byref(npad), C.byref(h), C.byref(dt), C.byref(m)))
        return ns.value, npad.value, h.value, dt.value, m.value

    def n(self):
        return self._n

    def nstate(self):
        return self._info()[0]

    def spacing(self):
        return self._info()[2]

    def dt(self):
        return self._info()[3]

    def pde_solves(self):   # :121
        return self._info()[4]

    def points(self):
        """Grid1D(-1, 1, n).points() (grid.hpp:10-24, diffusion1d.hpp:123)."""
        return (-1.0 + (2.0 / (self._n - 1)) * np.arange(self._n))[:, None]

    def hessvec_device(self, x, y, b, include_tv=True, stream=None):
        """y = H x on device pointers (n x b column-major, ld n)."""
        check(lib.h2c_diff1d_hessvec(self._h, int(include_tv), int(b), x, y, stream))

    def hessvec_at_target(self, nu, include_tv=True):
        """hessvec_at_target (:173-175) on host arrays (n x b)."""
        import torch
        nu = np.asarray(nu, np.float64)
        vec = nu.ndim == 1
        xm = nu[:, None] if vec else nu
        if xm.shape[0] != self._n:
            raise ValueError("hessvec: dimension mismatch")
        xd = torch.from_numpy(np.ascontiguousarray(xm.T)).cuda()
        yd = torch.empty_like(xd)
        self.hessvec_device(xd.data_ptr(), yd.data_ptr(), xm.shape[1], include_tv)
        torch.cuda.synchronize()
        y = yd.cpu().numpy().T
        return y[:, 0] if vec else np.asfortranarray(y)

    def hessian_operator(self, include_tv=True):
        """hessian_operator(include_tv) (:177-181): symmetric black box on the device."""
        h = H()
        check(lib.h2c_diff1d_operator(self._h, int(include_tv), C.byref(h)))
        return LinearOperator(h, self._n, True, keep=self)

    def state_field(self, source):
        """Cached target state of one source at the physical nodes, n x (steps+1)."""
        out = np.empty((self._n, self.steps + 1), order="F")
        check(lib.h2c_diff1d_state_field(self._h, int(source), out.ctypes.data_as(C.c_void_p)))
        return out


class MinimalSurface:
    """MinimalSurface(interior, rim) (minimal_surface.hpp:22-43) with its Hessian
    taken at newton_state(newton_steps) (:144-161, registry.hpp:92-93)."""

    def __init__(self, interior, rim=0.5, newton_steps=0):
        h = H()
        check(lib.h2c_surface_create(int(interior), float(rim), int(newton_steps), C.byref(h)))
        self._h = h
        self.interior, self.rim, self.newton_steps = int(interior), float(rim), int(newton_steps)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_surface_destroy(self._h)
            self._h = None

    def _info(self):
        n, nnz, h = C.c_int64(), C.c_int64(), C.c_double()
        check(lib.h2c_surface_info(self._h, C.byref(n), C.byref(nnz), C.byref(h)))
        return n.value, nnz.value, h.value

    def n(self):
        return self._info()[0]

    def nnz(self):
        return self._info()[1]

    def spacing(self):
        return self._info()[2]

    def points(self):
        """Grid2D(interior).points() (grid.hpp:38-48): (h i, h j), i fastest."""
        g, h = self.interior, self.spacing()
        i = np.tile(np.arange(1, g + 1), g)
        j = np.repeat(np.arange(1, g + 1), g)
        return np.stack([h * i, h * j], axis=1)

    def state(self):
        out = np.empty(self.n())
        check(lib.h2c_surface_state(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def hessvec_device(self, x, y, b, stream=None):
        """y = H x on device pointers (n x b column-major, ld n)."""
        check(lib.h2c_surface_hessvec(self._h, int(b), x, y, stream))

    def hessvec(self, x):
        """y = H x on host arrays (n x b)."""
        import torch
        x = np.asarray(x, np.float64)
        vec = x.ndim == 1
        xm = x[:, None] if vec else x
        if xm.shape[0] != self.n():
            raise ValueError("hessvec: dimension mismatch")
        xd = torch.from_numpy(np.ascontiguousarray(xm.T)).cuda()
        yd = torch.empty_like(xd)
        self.hessvec_device(xd.data_ptr(), yd.data_ptr(), xm.shape[1])
        torch.cuda.synchronize()
        y = yd.cpu().numpy().T
        return y[:, 0] if vec else np.asfortranarray(y)

    def hessian_operator(self):
        """hessian_operator (:163-167): symmetric black box on the device."""
        h = H()
        check(lib.h2c_surface_operator(self._h, C.byref(h)))
        return LinearOperator(h, self.n(), True, keep=self)


class AdvDiff2D:
    """AdvDiff2D(cfg) (advdiff2d.hpp:35-40); keyword names follow AdvDiff2DConfig (:21-28)."""

    def __init__(self, grid=32, kappa=1e-3, reaction=0.5, num_observations=100, noise_rel=0.01, obs_seed=7):
        c = AdvDiffConfigC()
        lib.h2c_advdiff_config_default(C.byref(c))
        c.grid, c.kappa, c.reaction = int(grid), float(kappa), float(reaction)
        c.num_observations, c.noise_rel, c.obs_seed = int(num_observations), float(noise_rel), int(obs_seed)
        h = H()
        check(lib.h2c_advdiff_create(C.byref(c), C.byref(h)))
        self._h = h
        self.config = dict(grid=grid, kappa=kappa, reaction=reaction, num_observations=num_observations,
                           noise_rel=noise_rel, obs_seed=obs_seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_advdiff_destroy(self._h)
            self._h = None

    def _info(self):
        n, sg, no, sv = C.c_int64(), C.c_double(), C.c_int64(), C.c_int64()
        check(lib.h2c_advdiff_info(self._h, C.byref(n), C.byref(sg), C.byref(no), C.byref(sv)))
        return n.value, sg.value, no.value, sv.value

    def n(self):
        return self._info()[0]

    def sigma(self):
        return self._info()[1]

    def solves(self):
        return self._info()[3]

    def observation_nodes(self):
        out = np.empty(self._info()[2], np.int64)
        check(lib.h2c_advdiff_observations(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def points(self):
        """Grid2D(grid).points() (grid.hpp:38-48): (h i, h j), i fastest."""
        g = int(self.config["grid"])
        h = 1.0 / (g + 1)
        i = np.tile(np.arange(1, g + 1), g)
        j = np.repeat(np.arange(1, g + 1), g)
        return np.stack([h * i, h * j], axis=1)

    def hessvec_device(self, x, y, b, stream=None):
        """y = H x on device pointers (n x b column-major, ld n)."""
        check(lib.h2c_advdiff_hessvec(self._h, int(b), x, y, stream))

    def misfit_hessvec(self, nu):
        """misfit_hessvec (:54-64) on host arrays (n x b)."""
        import torch
        nu = np.asarray(nu, np.float64)
        vec = nu.ndim == 1
        xm = nu[:, None] if vec else nu
        if xm.shape[0] != self.n():
            raise ValueError("advdiff hessvec: dimension mismatch")
        xd = torch.from_numpy(np.ascontiguousarray(xm.T)).cuda()
        yd = torch.empty_like(xd)
        self.hessvec_device(xd.data_ptr(), yd.data_ptr(), xm.shape[1])
        torch.cuda.synchronize()
        y = yd.cpu().numpy().T
        return y[:, 0] if vec else np.asfortranarray(y)

    def hessian_operator(self):
        """hessian_operator (:66-68): symmetric black box on the device."""
        h = H()
        check(lib.h2c_advdiff_operator(self._h, C.byref(h)))
        return LinearOperator(h, self.n(), True, keep=self)


class Oracle:
    """Oracle record of make_oracle (registry.hpp:58-81): op, points, leaf, mode, eta."""

    def __init__(self, name, op, points, leaf, mode, eta, diffusion=None, surface=None, advdiff=None):
        self.name, self.op, self.points, self.leaf, self.mode, self.eta = name, op, points, leaf, mode, eta
        self.diffusion = diffusion
        self.surface = surface
        self.advdiff = advdiff

    def default_block_tree(self, leaf=None, eta=None):
        from .h2 import build_block_tree, build_cluster_tree
        ct = build_cluster_tree(self.points, self.leaf if leaf is None else leaf)
        return build_block_tree(ct, ct, self.eta if eta is None else eta, self.mode)


def make_oracle(name, config=None):
    """make_oracle for "surface<N>" (registry.hpp:89-101; keys rim, newton_steps,
    leaf, eta), "diff1d-<n>" (registry.hpp:104-124; keys steps, T, tp, t0,
    alpha, amp, beta, pad, tv, leaf, eta) and "advdiff-<G>[-k<kappa>][-obs<N>]"
    (registry.hpp:125-150; keys kappa, obs, noise, obs_seed, c, leaf, eta)."""
    from .h2 import Admissibility
    cfg = dict(config or {})
    num = lambda k, d: float(cfg.get(k, d))
    if name.startswith("surface"):
        ms = MinimalSurface(int(name[7:]), num("rim", 0.5), int(cfg.get("newton_steps", 0)))
        return Oracle(name, ms.hessian_operator(), ms.points(), int(cfg.get("leaf", 64)), Admissibility.strong,
                      num("eta", 1.0), surface=ms)
    if name.startswith("advdiff-"):
        rest = name[8:]
        dash = rest.find("-")
        grid = int(rest if dash < 0 else rest[:dash])
        tail = "" if dash < 0 else rest[dash:]
        kappa, obs = 1e-3, 100
        at = tail.find("-obs")
        if at >= 0:
            obs = int(tail[at + 4:])
            tail = tail[:at]
        if tail.startswith("-k"):
            kappa = float(tail[2:])
        a = AdvDiff2D(grid=grid, kappa=num("kappa", kappa), reaction=num("c", 0.5),
                      num_observations=int(cfg.get("obs", obs)), noise_rel=num("noise", 0.01),
                      obs_seed=int(cfg.get("obs_seed", 7)))
        return Oracle(name, a.hessian_operator(), a.points(), int(cfg.get("leaf", 64)), Admissibility.strong,
                      num("eta", 1.0), advdiff=a)
    if not name.startswith("diff1d-"):
        raise ValueError(f"unknown oracle {name}")
    d = Diffusion1D(n=int(name[7:]), steps=int(cfg.get("steps", 512)), final_time=num("T", 30.0),
                    t_p=num("tp", 1.0), t_0=num("t0", 0.0), alpha=num("alpha", 3e-5),
                    source_amplitude=num("amp", 1000.0), beta=num("beta", 1e-3), pad=num("pad", 0.5))
    tv = int(cfg.get("tv", 1)) != 0
    return Oracle(name, d.hessian_operator(tv), d.points(), int(cfg.get("leaf", 32)), Admissibility.weak,
                  num("eta", 1.0), diffusion=d)
