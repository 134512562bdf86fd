"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module is shared by the oracle side (``oracle/``, ``tests/``) and the
product side (``bench.py``).  It holds *no* arithmetic of the FPE method:
it only draws coefficients and evaluation points with numpy's PCG64, with
the shapes and value distributions of the paper's benchmarks
(PAPER.md:2181-2213 -- sphere / real-line point sets, normal and
large-dynamic-range coefficient families; PAPER.md:15-16 sparse polynomials)
as fixed by /root/repo/BASELINE.json ``configs``.

Seeds: ``2211063200 + 10*cfg + stream`` with streams
0 = coefficient values, 1 = coefficient phases / indices,
2 = point radii / log-moduli, 3 = point angles / signs;
the second point sets of SURVEY.md §8(f) row 4 use 4, 5 (unit disk) and 6 (R-bar).

Riemann-sphere sampling: the
uniform measure on the sphere pushed to C by stereographic projection has
radial density 2r dr/(1+r^2)^2, whose CDF is F(r) = r^2/(1+r^2); inverting,
r = sqrt(u/(1-u)) with u ~ U(0,1), and the argument is uniform on [0, 2pi).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2211063200

# name -> (kind, degree d, number of points N)
CONFIGS = {
    1: dict(name="cfg1_c64_d1023_sphere", dtype="c64", d=1023, n_points=1 << 16),
    2: dict(name="cfg2_r64_d2^20-1_realline", dtype="r64", d=(1 << 20) - 1, n_points=1 << 24),
    3: dict(name="cfg3_c64_d2^20-1_bigrange_sphere", dtype="c64", d=(1 << 20) - 1, n_points=1 << 26),
    4: dict(name="cfg4_c64_sparse_d2^24_nnz4096", dtype="c64", d=1 << 24, n_points=1 << 24, nnz=4096),
    5: dict(name="cfg5_c64_d2^22-1_sphere", dtype="c64", d=(1 << 22) - 1, n_points=1 << 28),
}


def seed(cfg: int, stream: int) -> int:
    return SEED_BASE + 10 * cfg + stream


def _rng(cfg: int, stream: int, shard: int = 0) -> np.random.Generator:
    # shard > 0: an independent batch of the same distribution (weak-scaling ranks)
    return np.random.Generator(np.random.PCG64(seed(cfg, stream) + 1_000_003 * shard))


def _as_complex(re: np.ndarray, im: np.ndarray) -> np.ndarray:
    out = np.empty(re.shape, dtype=np.complex128)
    out.real = re
    out.imag = im
    return out


def coefficients(cfg: int, d: int | None = None) -> np.ndarray:
    """Coefficients a_0..a_d of configuration ``cfg`` (complex128 or float64).

    ``d`` overrides the degree (smaller test instances of the same family).
    """
    c = CONFIGS[cfg]
    d = c["d"] if d is None else int(d)
    n = d + 1
    if cfg in (1, 5):
        u = _rng(cfg, 0).uniform(-1.0, 1.0, size=(n, 2))
        return _as_complex(u[:, 0], u[:, 1])
    if cfg == 2:
        return _rng(cfg, 0).standard_normal(n)
    if cfg == 3:
        # |a_k| = 2^(200 sin(pi k/d) + N(0, 4)); N(0,4) read as variance 4
        k = np.arange(n, dtype=np.float64)
        e = 200.0 * np.sin(np.pi * k / d) + 2.0 * _rng(cfg, 0).standard_normal(n)
        phase = _rng(cfg, 1).uniform(0.0, 2.0 * np.pi, size=n)
        mag = np.exp2(e)
        return _as_complex(mag * np.cos(phase), mag * np.sin(phase))
    if cfg == 4:
        nnz = min(c["nnz"], n)
        idx = np.sort(_rng(cfg, 1).choice(n, size=nnz, replace=False))
        u = _rng(cfg, 0).uniform(-1.0, 1.0, size=(nnz, 2))
        a = np.zeros(n, dtype=np.complex128)
        a[idx] = _as_complex(u[:, 0], u[:, 1])
        return a
    raise KeyError(cfg)


def sparse_coefficients(cfg: int = 4, d: int | None = None):
    """(indices, values) of the sparse configuration without the dense array."""
    a = coefficients(cfg, d)
    idx = np.flatnonzero(a)
    return idx.astype(np.int64), a[idx]


def _prng(cfg: int, stream: int, shard: int, start: int) -> np.random.Generator:
    """The point stream's generator advanced past `start` draws: every point draw below takes exactly one
    64-bit output per value (random() / uniform()), so point i of a batch comes from draw i of each stream
    and any contiguous slice [lo, hi) can be generated alone (multi-GPU shards, bench.py)."""
    g = _rng(cfg, stream, shard)
    if start:
        g.bit_generator.advance(start)
    return g


def sphere_points(cfg: int, n: int, shard: int = 0, start: int = 0) -> np.ndarray:
    """n points uniform on the Riemann sphere, stereographically projected (points start..start+n-1 of the
    seeded sequence)."""
    u = _prng(cfg, 2, shard, start).random(n)
    u = np.where(u == 0.0, 0.5, u)  # open interval (0,1); u==0 has probability 2^-53
    r = np.sqrt(u / (1.0 - u))
    phi = _prng(cfg, 3, shard, start).uniform(0.0, 2.0 * np.pi, size=n)
    return _as_complex(r * np.cos(phi), r * np.sin(phi))


def disk_points(cfg: int, n: int, shard: int = 0) -> np.ndarray:
    """n points uniform on the unit disk D(0, 1) (rmk:case_disk): r = sqrt(u),
    u ~ U(0, 1), argument uniform on [0, 2 pi).  Streams 4 (radii) and 5 (angles)."""
    r = np.sqrt(_rng(cfg, 4, shard).random(n))
    phi = _rng(cfg, 5, shard).uniform(0.0, 2.0 * np.pi, size=n)
    return _as_complex(r * np.cos(phi), r * np.sin(phi))


def rbar_points(cfg: int, n: int, shard: int = 0) -> np.ndarray:
    """n real points uniform on the circle R-bar = R u {inf} (eq:compAlgoRe; weight
    omega-tilde): the uniform measure on the projective line is the Cauchy law
    dx / (pi (1 + x^2)), x = tan(pi (u - 1/2)) with u ~ U(0, 1) open.  Stream 6."""
    u = _rng(cfg, 6, shard).random(n)
    u = np.where(u == 0.0, 0.5, u)
    return np.tan(np.pi * (u - 0.5))


def points(cfg: int, n: int | None = None, shard: int = 0, start: int = 0) -> np.ndarray:
    """Evaluation points of configuration ``cfg`` (complex128 or float64): points start..start+n-1 of the
    seeded sequence (n defaults to the configuration's N - start), so points(cfg, hi - lo, start=lo) equals
    points(cfg)[lo:hi]."""
    c = CONFIGS[cfg]
    n = c["n_points"] - start if n is None else int(n)
    if cfg in (1, 3, 5):
        return sphere_points(cfg, n, shard, start)
    if cfg == 2:
        t = _prng(cfg, 2, shard, start).uniform(-8.0, 8.0, size=n)
        sgn = np.where(_prng(cfg, 3, shard, start).random(n) < 0.5, -1.0, 1.0)
        return sgn * np.exp2(t)
    if cfg == 4:
        t = _prng(cfg, 2, shard, start).uniform(-2.0, 2.0, size=n)
        phi = _prng(cfg, 3, shard, start).uniform(0.0, 2.0 * np.pi, size=n)
        r = np.exp2(t)
        return _as_complex(r * np.cos(phi), r * np.sin(phi))
    raise KeyError(cfg)


def to_fp32(a: np.ndarray) -> np.ndarray:
    """The fp32 variant of configuration 5: the same values rounded to fp32."""
    return a.astype(np.complex64 if np.iscomplexobj(a) else np.float32)


def sample_indices(n: int, k: int, salt: int = 0) -> np.ndarray:
    """A seeded sample of k distinct indices in [0, n) (sorted), for parity checks."""
    k = min(k, n)
    g = np.random.Generator(np.random.PCG64(SEED_BASE + 7 + salt))
    return np.sort(g.choice(n, size=k, replace=False))
