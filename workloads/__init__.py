"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no chirp, split, NTT, CRT): it only
draws input vectors with NumPy's PCG64 in a fixed order, so both sides see the same
bytes.  Recipes follow BASELINE.json ``configs``:

  c1  n=2^10,  B=1,    re/im uniform[-1,1)              seed 0
  c2  n=2^14,  B=64,   re/im standard normal            seed 1
  c3  n=2^18,  B=16,   re/im uniform[-1,1)              seed 2
  c4  n=100003, B=32,  re/im sign*2^e, e in [-30,30]    seed 3
  c5  n=2^16,  B=1024, re/im standard normal            seed 4 (fwd then inverse)

The paper's own timing workload is phi=0, i.e. (rand-0.5) uniform on (-0.5,0.5]
(P:1050-1054); uniform[-1,1) differs by a power-of-two scale, which leaves
digits and work unchanged.  ``phi_input`` reproduces eq:input-generation for the
accuracy sweep.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    batch: int
    dist: str
    seed: int
    roundtrip: bool = False


CONFIGS = {
    "c1": Config("c1", 1 << 10, 1, "uniform", 0),
    "c2": Config("c2", 1 << 14, 64, "normal", 1),
    "c3": Config("c3", 1 << 18, 16, "uniform", 2),
    "c4": Config("c4", 100003, 32, "signexp", 3),
    "c5": Config("c5", 1 << 16, 1024, "normal", 4, roundtrip=True),
}


def draw(dist: str, seed: int, batch: int, n: int, rows: slice | None = None) -> np.ndarray:
    """complex128 [batch, n] (or the given row slice) for the distribution recipe.

    Real block first, then imaginary block (SURVEY 8(d) draw order)."""
    rng = np.random.default_rng(seed)
    shape = (batch, n)
    if dist == "uniform":
        re = rng.uniform(-1.0, 1.0, shape)
        im = rng.uniform(-1.0, 1.0, shape)
    elif dist == "normal":
        re = rng.standard_normal(shape)
        im = rng.standard_normal(shape)
    elif dist == "signexp":
        e_re = rng.integers(-30, 31, shape)
        s_re = rng.choice([-1.0, 1.0], shape)
        e_im = rng.integers(-30, 31, shape)
        s_im = rng.choice([-1.0, 1.0], shape)
        re = s_re * np.ldexp(1.0, e_re)
        im = s_im * np.ldexp(1.0, e_im)
    else:
        raise ValueError(dist)
    x = np.empty(shape, np.complex128)
    x.real = re
    x.imag = im
    if rows is not None:
        x = np.ascontiguousarray(x[rows])
    return x


def config_input(cfg: Config | str) -> np.ndarray:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return draw(cfg.dist, cfg.seed, cfg.batch, cfg.n)


def phi_input(n: int, phi: float, seed: int, batch: int = 1) -> np.ndarray:
    """(rand - 0.5) * exp(phi * randn), rand ~ U(0,1]  (eq:input-generation)."""
    rng = np.random.default_rng(seed)
    shape = (batch, n)
    parts = []
    for _ in range(2):
        u = 1.0 - rng.random(shape)  # (0, 1]
        parts.append((u - 0.5) * np.exp(phi * rng.standard_normal(shape)))
    x = np.empty(shape, np.complex128)
    x.real, x.imag = parts
    return x
