"""SplitMix64 parameter streams and config shapes.

* Generator: the public SplitMix64 mixer.  state += 0x9E3779B97F4A7C15;
  z = state; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EB; z ^= z >> 31.
  U = (z >> 11) * 2^-53 in [0, 1).
* mu_i = lo * (hi/lo)^U, drawn component by component in file order
  (query-major), i.e. "mu log-uniform in [lo, hi]" of BASELINE.json configs.
* Seeds: training set 1000 + c, queries 2000 + c for config c (1-based).

The shapes mirror BASELINE.json `configs`; values a config
leaves unstated are the SURVEY's AMB-15 proposals and are marked so.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64_uniform(seed: int, count: int) -> np.ndarray:
    """`count` doubles U in [0,1) from a SplitMix64 stream seeded with `seed`."""
    out = np.empty(count, dtype=np.float64)
    state = seed & _M64
    for i in range(count):
        state = (state + 0x9E3779B97F4A7C15) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        z = z ^ (z >> 31)
        out[i] = (z >> 11) * (1.0 / 9007199254740992.0)
    return out


def loguniform_mu(seed: int, count: int, P: int, lo: float, hi: float) -> np.ndarray:
    """(count, P) float64 array, mu = lo * (hi/lo)**U, query-major."""
    u = splitmix64_uniform(seed, count * P).reshape(count, P)
    return lo * np.power(hi / lo, u)


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    m: int                 # interior nodes per axis
    blocks: tuple          # subdomains per axis (px, py[, pz])
    lo: float
    hi: float
    n: int                 # RB dimension
    n_train: int
    n_queries: int
    B: int                 # batch size per GPU pass
    method: str            # primary solver
    note: str = ""

    @property
    def P(self) -> int:
        p = 1
        for b in self.blocks:
            p *= b
        return p

    @property
    def N(self) -> int:
        return self.m ** self.dim

    @property
    def index(self) -> int:
        return int(self.name[1:])


CONFIGS = {
    "c1": Config("c1", 2, 63, (2, 2), 0.1, 10.0, 16, 256, 8, 8, "both"),
    "c2": Config("c2", 2, 511, (3, 3), 0.1, 10.0, 40, 1024, 256, 32, "rbcg"),
    "c3": Config("c3", 2, 2047, (3, 3), 0.1, 10.0, 60, 1024, 1024, 64, "both",
                 "B=64 proposed (SURVEY AMB-15)"),
    "c4": Config("c4", 3, 255, (2, 2, 2), 0.1, 10.0, 60, 512, 512, 16, "rbcg"),
    "c5": Config("c5", 3, 511, (2, 2, 2), 0.01, 100.0, 40, 512, 64, 8, "rbcg",
                 "n_train=512, B=8 proposed (SURVEY AMB-15)"),
}


def train_set(cfg: Config) -> np.ndarray:
    return loguniform_mu(1000 + cfg.index, cfg.n_train, cfg.P, cfg.lo, cfg.hi)


def query_set(cfg: Config, count: int | None = None) -> np.ndarray:
    return loguniform_mu(2000 + cfg.index, cfg.n_queries if count is None else count,
                         cfg.P, cfg.lo, cfg.hi)


def write_rbsm(path: str, mu: np.ndarray, lo: float, hi: float, seed: int) -> None:
    """`.rbsm` file: magic RBSM0001, u32 P, u64 count, f64 lo, f64 hi, u64 seed, body."""
    mu = np.ascontiguousarray(mu, dtype="<f8")
    count, P = mu.shape
    with open(path, "wb") as f:
        f.write(b"RBSM0001")
        f.write(struct.pack("<IQddQ", P, count, lo, hi, seed))
        f.write(mu.tobytes())


def read_rbsm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        if f.read(8) != b"RBSM0001":
            raise ValueError("not an .rbsm file")
        P, count, _lo, _hi, _seed = struct.unpack("<IQddQ", f.read(36))
        return np.frombuffer(f.read(8 * P * count), dtype="<f8").reshape(count, P).copy()
