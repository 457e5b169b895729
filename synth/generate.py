"""Seeded generators.  numpy PCG64 streams; every draw is an explicit input.

Layout convention shared by both sides (an input, not arithmetic):
interior node (i, j, k), 0 <= i < nx, 0 <= j < ny, 0 <= k < nz, has linear index
``(k*ny + j)*nx + i`` (x fastest).  k = 0 is the top face z = 0 (sources),
k = nz-1 the bottom face z = Lz (detectors).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .configs import DOTConfig


def face_nodes(n, grid_ab, k):
    """Linear node indices of an (n_a x n_b) point array on the plane k.

    Array element (a, b) sits at node i = floor((a + 1/2) nx / n_a),
    j = floor((b + 1/2) ny / n_b): the centres of n_a equal bands.  Ordered
    with a fastest (s = b*n_a + a).
    """
    nx, ny, nz = n
    na, nb = grid_ab
    if na > nx or nb > ny:
        raise ValueError("more points than face nodes")
    ii = ((np.arange(na) + 0.5) * nx / na).astype(np.int64)
    jj = ((np.arange(nb) + 0.5) * ny / nb).astype(np.int64)
    J, I = np.meshgrid(jj, ii, indexing="ij")
    return ((k * ny + J) * nx + I).reshape(-1).astype(np.int64)


def draw_params(rng: np.random.Generator, n_rbf: int, L, alpha_lo=-1.0, alpha_hi=1.0,
                beta_lo=0.5, beta_hi=2.0) -> np.ndarray:
    """PaLS parameter vector, 5 entries per basis function: (alpha, beta, cx, cy, cz).

    alpha ~ U(alpha_lo, alpha_hi), beta ~ U(beta_lo, beta_hi), centre uniform in
    the domain [0,Lx]x[0,Ly]x[0,Lz] (BASELINE.json configs[0]).
    """
    p = np.empty((n_rbf, 5))
    p[:, 0] = rng.uniform(alpha_lo, alpha_hi, n_rbf)
    p[:, 1] = rng.uniform(beta_lo, beta_hi, n_rbf)
    for d in range(3):
        p[:, 2 + d] = rng.uniform(0.0, L[d], n_rbf)
    return p.reshape(-1)


def rademacher(n: int, l: int, seed: int, stream: int = 0) -> np.ndarray:
    """n x l matrix of i.i.d. +-1 entries (Sec. 3.1, Theorem 3.1)."""
    rng = np.random.Generator(np.random.PCG64([seed, stream]))
    return (2.0 * rng.integers(0, 2, size=(n, l)) - 1.0).astype(np.float64)


def subspace_start(n: int, cols: int, seed: int, stream: int) -> np.ndarray:
    """Standard-normal starting blocks of the subspace iteration (reading R16)."""
    rng = np.random.Generator(np.random.PCG64([seed, 100 + stream]))
    return rng.standard_normal((n, cols))


def noise_draws(seed: int, shape) -> np.ndarray:
    """Complex standard normal draws (xi + i eta)/sqrt(2) for the data noise."""
    rng = np.random.Generator(np.random.PCG64([seed, 7]))
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return (re + 1j * im) / np.sqrt(2.0)


@dataclass
class Workload:
    cfg: DOTConfig
    src_nodes: np.ndarray        # (n_s,) int64
    det_nodes: np.ndarray        # (n_d,) int64
    p: np.ndarray                # (n_p,) current PaLS iterate
    p_true: np.ndarray           # (5*n_rbf_true,) hidden level set for the data
    W: Optional[np.ndarray]      # (n_s, ls) Rademacher or None (identity)
    V: Optional[np.ndarray]      # (n_d, ld) Rademacher or None (identity)
    xi: np.ndarray               # (n_freq, n_d, n_s) complex noise draws
    X0_src: Optional[np.ndarray] = None   # (n_s, n_opt * block) subspace-iteration starts
    X0_det: Optional[np.ndarray] = None   # (n_d, n_opt * block)

    @property
    def p_true_padded(self):
        """p_true extended to n_rbf bases with zero-amplitude (alpha = 0) entries, so
        a problem built for the current iterate's n_p can simulate the data."""
        extra = self.cfg.n_rbf - self.p_true.size // 5
        pad = np.tile(np.array([0.0, 1.0, 0.0, 0.0, 0.0]), max(extra, 0))
        return np.concatenate([self.p_true, pad])

    @property
    def W_or_I(self):
        return np.eye(self.cfg.n_s) if self.W is None else self.W

    @property
    def V_or_I(self):
        return np.eye(self.cfg.n_d) if self.V is None else self.V


def make_workload(cfg: DOTConfig) -> Workload:
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 0]))
    p = draw_params(rng, cfg.n_rbf, cfg.L)
    rng_t = np.random.Generator(np.random.PCG64([cfg.seed, 1]))
    # hidden truth: same distribution except alpha ~ U(0.5, 1) so that an
    # anomaly exists (reading R11)
    p_true = draw_params(rng_t, cfg.n_rbf_true, cfg.L, alpha_lo=0.5, alpha_hi=1.0)
    src = face_nodes(cfg.n, cfg.src_grid, 0)
    det = face_nodes(cfg.n, cfg.det_grid, cfg.n[2] - 1)
    W = rademacher(cfg.n_s, cfg.ls, cfg.sketch_seed, 0) if cfg.ls else None
    V = rademacher(cfg.n_d, cfg.ld, cfg.sketch_seed, 1) if cfg.ld else None
    xi = noise_draws(cfg.seed, (cfg.n_freq, cfg.n_d, cfg.n_s))
    X0s = X0d = None
    if cfg.n_opt:
        X0s = subspace_start(cfg.n_s, 2 * cfg.n_opt, cfg.sketch_seed, 0)    # block size 2
        X0d = subspace_start(cfg.n_d, 2 * cfg.n_opt, cfg.sketch_seed, 1)
    return Workload(cfg, src, det, p, p_true, W, V, xi, X0s, X0d)
