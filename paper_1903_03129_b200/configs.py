"""The BASELINE.json workloads (SURVEY.md section 8(d) pins the unstated knobs).

Each preset names the network shape, the LSH layer, the sampler and the
synthetic corpus.  ``bench.py`` runs ``wide_in`` at N=1 (BASELINE.json
configs[1], the shape the metric is quoted on); the others are parity and
secondary cases.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

from .data import CorpusSpec


@dataclass(frozen=True)
class Workload:
    name: str
    input_dim: int
    hidden: int
    n_out: int
    batch: int
    family: str
    k: int
    l: int
    cap: int
    policy: str
    strategy: str
    beta: int
    lr: float
    n0: int
    decay: float
    corpus: CorpusSpec
    bin_size: int = 8


TINY = Workload(
    "tiny", 10_000, 128, 5_000, 128, "simhash", 6, 20, 128, "fifo", "vanilla", 250, 1e-3, 50, 0.0,
    CorpusSpec(10_000, 5_000, ("uniform", 20, 80), 1.1, ("uniform", 1, 5), 1.1, False),
)

# beta = round(5% N) (reference cli.py:54, estimator.py:156): > L*cap = 6400,
# so vanilla probes all 50 tables (full-union regime).  decay pinned at 0.05.
WIDE_IN = Workload(
    "wide_in", 782_585, 128, 205_443, 128, "simhash", 9, 50, 128, "fifo", "vanilla", 10_272, 1e-4, 50, 0.05,
    CorpusSpec(782_585, 205_443, ("poisson", 300), 1.05, ("poisson", 75), 1.05, True),
)

# beta = 128 (API default, SURVEY 8(d) primary); reservoir buckets.
WIDE_OUT = Workload(
    "wide_out", 135_909, 128, 670_091, 256, "dwta", 8, 50, 128, "reservoir", "vanilla", 128, 1e-4, 50, 0.0,
    CorpusSpec(135_909, 670_091, ("poisson", 75), 1.1, ("poisson", 5), 1.1, True),
)

SCALED = Workload(
    "scaled", 135_909, 256, 4_000_000, 1_024, "dwta", 8, 64, 128, "reservoir", "vanilla", 128, 1e-4, 50, 0.0,
    CorpusSpec(135_909, 4_000_000, ("poisson", 75), 1.1, ("poisson", 5), 1.1, True),
)

# SURVEY 8(d) secondary lines: the API-default beta (one-table regime at
# wide-in) and the 5% beta at wide-out (fallback-dominated)
WIDE_IN_B128 = dataclasses.replace(WIDE_IN, name="wide_in_b128", beta=128)
WIDE_OUT_B5PCT = dataclasses.replace(WIDE_OUT, name="wide_out_b5pct", beta=33_505)

WORKLOADS = {w.name: w for w in (TINY, WIDE_IN, WIDE_OUT, SCALED, WIDE_IN_B128, WIDE_OUT_B5PCT)}
