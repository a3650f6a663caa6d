"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws the random
objects a compressive-sensing trial is made of:

* the sign diagonal sigma of A = P.DCT-II.diag(sigma), packed as bits
  (bit j of word j//32 set  <=>  sigma_j = -1);
* the row set of P: M distinct indices of [0, N), strictly increasing
  ("randomly choose M indices");
* the planted signal s (exact-K) and its support;
* the measurement noise eta ~ N(0, sigma_eta^2) i.i.d. (Eq.13).

y = A s + eta is NOT formed here: tests form it with `oracle/`, bench.py forms
it with the product operator (cs_operator_apply) outside the timed region.

Seeds: numpy PCG64(SeedSequence([cfg, trial, b, tag])), tag 0 = sigma,
1 = rows, 2 = positions, 3 = values, 4 = noise, 5 = permutation.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

TAG_SIGMA, TAG_ROWS, TAG_POS, TAG_VAL, TAG_NOISE, TAG_PERM, TAG_RAND = range(7)


def rng(cfg: int, trial: int, b: int, tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg, trial, b, tag])))


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config."""
    cid: int
    alg: str            # "omp" | "sp" | "ompr" | "cosamp"
    N: int
    M: int
    K: int
    signal: str         # "gauss" | "pm1" | "power" | "bernoulli" (Eq.(13))
    noise: float        # sigma_eta
    batch: int = 1
    randomizer: str = "sign"   # "sign": R = diag(+-1) (BASELINE); "perm": Eq.(7)'s permutation, sigma = +1
    psi: str = "I"             # dictionary: "I" (BASELINE) or "dct" (A = Phi C_N)
    transform: str = "dct"     # F: "dct" (BASELINE) or "dft" (partial Fourier; M = 2 x freqs)

    def scaled(self, div: int, batch: Optional[int] = None) -> "Config":
        """Same recipe at N/div, M/div, K/div (ratios kept); used for parity tests."""
        return dataclasses.replace(self, N=self.N // div, M=self.M // div,
                                   K=max(1, self.K // div),
                                   batch=self.batch if batch is None else batch)


# BASELINE.json "configs" (0-based index in that list = cid - 1).
CONFIGS = {
    1: Config(1, "omp", 4096, 1024, 64, "gauss", 0.0),
    2: Config(2, "sp", 65536, 16384, 2048, "gauss", 1e-3),
    3: Config(3, "ompr", 1 << 20, 1 << 18, 8192, "pm1", 0.0),
    4: Config(4, "sp", 16384, 4096, 256, "gauss", 0.0, batch=4096),
    5: Config(5, "sp", 1 << 24, 1 << 22, 65536, "power", 1e-4),
}


def pack_sign_bits(neg: np.ndarray) -> np.ndarray:
    """Pack a boolean 'sigma_j = -1' vector into ceil(N/32) uint32 words (zero padded)."""
    neg = np.asarray(neg, dtype=bool)
    pad = (-neg.size) % 32
    if pad:
        neg = np.concatenate([neg, np.zeros(pad, dtype=bool)])
    return np.packbits(neg, bitorder="little").view("<u4").astype(np.uint32)


def unpack_sign_bits(bits: np.ndarray, N: int) -> np.ndarray:
    """Inverse of pack_sign_bits: returns the boolean 'negative' mask (input decoding only)."""
    b = np.unpackbits(np.asarray(bits, dtype="<u4").view(np.uint8), bitorder="little")
    return b[:N].astype(bool)


def draw_sign_bits(N: int, g: np.random.Generator) -> np.ndarray:
    return pack_sign_bits(g.integers(0, 2, N).astype(bool))


def draw_rows(N: int, M: int, g: np.random.Generator) -> np.ndarray:
    return np.sort(g.choice(N, M, replace=False)).astype(np.int32)


def draw_freqs(N: int, Mf: int, g: np.random.Generator) -> np.ndarray:
    """Mf distinct frequencies in [1, N/2 - 1], sorted (partial Fourier rows, R36)."""
    return np.sort(g.choice(np.arange(1, N // 2), Mf, replace=False)).astype(np.int32)


def draw_perm(N: int, g: np.random.Generator) -> np.ndarray:
    """A uniformly random permutation pi of [0, N) (the randomizer R of Eq.(7))."""
    return g.permutation(N).astype(np.int32)


def draw_signal(kind: str, N: int, K: int, g_pos: np.random.Generator,
                g_val: np.random.Generator, g_perm: np.random.Generator):
    """Planted signal s (float64[N]) and its sorted support (int64)."""
    s = np.zeros(N, dtype=np.float64)
    if kind == "power":
        # |s|_(i) = i^-1.5, i = 1..N, random signs, random positions
        perm = g_perm.permutation(N)
        mag = np.arange(1, N + 1, dtype=np.float64) ** -1.5
        sgn = np.where(g_val.integers(0, 2, N) == 1, -1.0, 1.0)
        s[perm] = sgn * mag
        return s, np.sort(perm[:K])
    if kind == "bernoulli":
        # the paper's Eq.(13): every entry nonzero with probability p = K/N,
        # N(0, 1) values (sigma_on = 1); the number of nonzeros is itself random
        on = g_pos.random(N) < K / N
        s[on] = g_val.standard_normal(int(on.sum()))
        return s, np.nonzero(on)[0]
    pos = np.sort(g_pos.choice(N, K, replace=False))
    if kind == "gauss":
        vals = g_val.standard_normal(K)
    elif kind == "pm1":
        sgn = np.where(g_val.integers(0, 2, K) == 1, -1.0, 1.0)
        vals = sgn * (1.0 + np.abs(g_val.standard_normal(K)))
    else:
        raise ValueError(kind)
    s[pos] = vals
    return s, pos


@dataclasses.dataclass
class Problem:
    N: int
    M: int
    K: int
    alg: str
    sign_bits: np.ndarray   # uint32[N/32]
    rows: np.ndarray        # int32[M], strictly increasing
    s: np.ndarray           # float64[N] planted signal
    support: np.ndarray     # planted support (sorted)
    noise: np.ndarray       # float64[M] eta
    perm: Optional[np.ndarray] = None   # int32[N] pi of the randomizer R (randomizer "perm")
    psi: Optional[str] = None           # None (Psi = I) or "dct"
    transform: str = "dct"              # "dct" or "dft" (rows are then frequencies)


def make_problem(cfg: Config, trial: int = 0, b: int = 0) -> Problem:
    c = cfg.cid
    N, M, K = cfg.N, cfg.M, cfg.K
    if cfg.randomizer == "perm":
        bits = pack_sign_bits(np.zeros(N, dtype=bool))
        perm = draw_perm(N, rng(c, trial, b, TAG_RAND))
    else:
        bits = draw_sign_bits(N, rng(c, trial, b, TAG_SIGMA))
        perm = None
    if cfg.transform == "dft":
        rows = draw_freqs(N, M // 2, rng(c, trial, b, TAG_ROWS))
        M = 2 * rows.size
    else:
        rows = draw_rows(N, M, rng(c, trial, b, TAG_ROWS))
    s, supp = draw_signal(cfg.signal, N, K, rng(c, trial, b, TAG_POS),
                          rng(c, trial, b, TAG_VAL), rng(c, trial, b, TAG_PERM))
    eta = rng(c, trial, b, TAG_NOISE).standard_normal(M) * cfg.noise if cfg.noise > 0 \
        else np.zeros(M)
    return Problem(N, M, K, cfg.alg, bits, rows, s, supp, eta, perm, "dct" if cfg.psi == "dct" else None,
                   cfg.transform)


def paper_regime(alg: str, N: int) -> Config:
    """The paper's experimental regime (Tables II-IV): M = N/4, K = M/4,
    Bernoulli-Gaussian s (Eq.(13)), sigma_eta = 0.01."""
    return Config(13, alg, N, N // 4, N // 16, "bernoulli", 0.01)


def make_batch(cfg: Config, trial: int = 0, b0: int = 0, count: Optional[int] = None):
    count = cfg.batch if count is None else count
    return [make_problem(cfg, trial, b0 + i) for i in range(count)]
