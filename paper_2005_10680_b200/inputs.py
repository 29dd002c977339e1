"""Tolerance grids and the BASELINE.json workload definitions.

Synthetic stand-ins: the reference quotes no dataset; BASELINE.json's configs
describe seeded decay matrices, generated here by include/spamm_synth.h.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def log_grid(n_taus: int, hi: float = 1e-2, lo: float = 1e-12) -> np.ndarray:
    """n_taus log-spaced candidates from hi down to lo:
    tau_k = 10^(log10 hi - k (log10 hi - log10 lo) / (n - 1))."""
    k = np.arange(n_taus, dtype=np.float64)
    a, b = math.log10(hi), math.log10(lo)
    return 10.0 ** (a - k * (a - b) / max(n_taus - 1, 1))


def geometric_grid(start: float = 1.0, ratio: float = 0.9, count: int = 350) -> np.ndarray:
    """ToleranceGrid::geometric (error_control.cpp:152-158): repeated tau *= ratio."""
    out = np.empty(count)
    tau = start
    for k in range(count):
        out[k] = tau
        tau *= ratio
    return out


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str          # "chain" | "cluster"
    n: int
    leaf: int
    ell: float
    delta: float
    n_taus: int
    drop: float = 1e-10
    density: float = 0.1
    site_seed: int = 2005
    value_seed: int = 10680
    value_seed_b: int | None = None  # independent B (config 4); None -> A*A


# BASELINE.json configs; seeds fixed here, recorded in DESIGN.md.
CONFIGS = {
    "cfg1": Workload("cfg1-chain-N4096-L64", "chain", 4096, 64, 40.0, 1e-6, 32, value_seed=12345),
    "cfg2": Workload("cfg2-cluster3d-N32768-L64", "cluster", 32768, 64, 3.0, 1e-5, 32),
    "cfg4": Workload("cfg4-cluster3d-N262144-L64", "cluster", 262144, 64, 4.0, 1e-6, 64,
                     value_seed_b=10681),
}
