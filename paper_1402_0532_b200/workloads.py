"""Seeded synthetic inputs for the BASELINE.json configs.

No dataset is involved; every input is generated from ``np.random.default_rng``
(PCG64, as radar.py:181) with base seed 14020532 + config index.  The map
signal model stands in for the reference's FM scene synthesis (radar.py:179-242):
an FM-like illuminator exp(j*2*pi*0.05*cumsum(g)) with g brick-wall low-passed
to |f| <= 0.2 fs, and a surveillance channel = direct path + delayed,
Doppler-shifted echoes (zero before their delay, as radar.py:233-234) + CN(0, σ²).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .twiddle import twiddle_table

BASE_SEED = 14020532


def cn(g: np.random.Generator, shape, var: float = 1.0) -> np.ndarray:
    """i.i.d. CN(0, var): (N(0,1) + jN(0,1)) * sqrt(var/2)."""
    return (g.standard_normal(shape) + 1j * g.standard_normal(shape)) * np.sqrt(var / 2.0)


def unit_tone(k0: int, n: int) -> np.ndarray:
    return np.conj(twiddle_table(n).entries[(k0 * np.arange(n)) % n])


def c1_ndft64(batch: int = 4096) -> np.ndarray:
    """C1: row 0 = exp(j2π·7n/64) on the exact grid, then `batch` CN(0,1) rows."""
    g = np.random.default_rng(BASE_SEED + 0)
    x = np.empty((batch + 1, 64), dtype=np.complex128)
    x[0] = unit_tone(7, 64)
    x[1:] = cn(g, (batch, 64))
    return x


def c2_ndft(n: int = 1024, batch: int = 65536, rows: slice | None = None) -> np.ndarray:
    """C2: CN(0,1) rows; 10% (chosen by permutation) replaced by unit tones k0 + CN(0,0.01)."""
    g = np.random.default_rng(BASE_SEED + 1)
    x = cn(g, (batch, n))
    tone_rows = g.permutation(batch)[: batch // 10]
    k0 = g.integers(0, n, size=tone_rows.size)
    noise = cn(g, (tone_rows.size, n), 0.01)
    tw = twiddle_table(n).entries
    m = np.arange(n)
    for r, k, e in zip(tone_rows, k0, noise):
        x[r] = np.conj(tw[(k * m) % n]) + e
    return x if rows is None else x[rows]


def c3_nlfft_rows(n: int, rows: np.ndarray, seed: int = BASE_SEED + 2) -> np.ndarray:
    """C3 rows: CN(0,1) + Σ_{t=1..K} A_t exp(j(2π f_t n/N + φ_t)), K~U{1..4}, A~U[0.1,1],
    f~U[0,N) (off-grid), φ~U[0,2π).  Row r is generated from seed (seed, r): any
    subset can be regenerated independently."""
    out = np.empty((len(rows), n), dtype=np.complex128)
    t = np.arange(n)
    for i, r in enumerate(rows):
        g = np.random.default_rng([seed, int(r)])
        v = cn(g, n)
        k = int(g.integers(1, 5))
        for _ in range(k):
            a = g.uniform(0.1, 1.0)
            f = g.uniform(0.0, n)
            ph = g.uniform(0.0, 2 * np.pi)
            v += a * np.exp(1j * (2 * np.pi * f * t / n + ph))
        out[i] = v
    return out


@dataclass
class RadarScene:
    surv: np.ndarray
    ref: np.ndarray
    delays: np.ndarray
    dopplers: np.ndarray  # normalised f_k / fs
    amps: np.ndarray


def radar_scene(ns: int, n_targets: int, seed: int, doppler_max: float = 2e-3,
                sigma2: float = 0.1, margin: int = 1024) -> RadarScene:
    """C4/C5 signal model; ns samples of surveillance and reference."""
    g = np.random.default_rng(seed)
    tot = ns + margin
    w = g.standard_normal(tot)
    spec = np.fft.fft(w)
    f = np.fft.fftfreq(tot)
    spec[np.abs(f) > 0.2] = 0.0
    lp = np.real(np.fft.ifft(spec))
    lp /= np.std(lp)
    s = np.exp(1j * 2 * np.pi * 0.05 * np.cumsum(lp))[:ns]
    taus = g.integers(10, 901, size=n_targets)
    fd = g.uniform(-doppler_max, doppler_max, size=n_targets)
    amps = g.uniform(0.003, 0.03, size=n_targets)
    r = s.copy()
    idx = np.arange(ns)
    for tau, fk, a in zip(taus, fd, amps):
        echo = np.zeros(ns, dtype=np.complex128)
        echo[tau:] = s[: ns - tau]
        r += a * echo * np.exp(2j * np.pi * fk * idx)
    r += cn(g, ns, sigma2)
    return RadarScene(r, s, taus, fd, amps)


def c4_scene() -> RadarScene:
    return radar_scene(1 << 20, 3, BASE_SEED + 3)


def c5_scene() -> RadarScene:
    return radar_scene(1 << 22, 8, BASE_SEED + 4)
