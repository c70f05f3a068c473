"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the paper's method: only the parameter
generator (SplitMix64 -> log-uniform mu, SURVEY.md §8d / DESIGN.md AMB-14) and
the shapes of the BASELINE.json configs.  Both `oracle/` and the product
binding may import it; it imports neither.
"""
from .inputs import (  # noqa: F401
    CONFIGS,
    Config,
    splitmix64_uniform,
    loguniform_mu,
    train_set,
    query_set,
    write_rbsm,
    read_rbsm,
)
