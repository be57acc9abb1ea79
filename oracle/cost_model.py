"""Online vs offline ABFT cost model (section 5.5).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and
bench.py's model columns, never by the product path.

The paper's model: C += AB of size M x N is computed by M/m_tb x N/n_tb
threadblock tiles; each tile's accumulation errs with probability gamma0, so
the whole call errs with probability

    gamma = 1 - (1 - gamma0)^(M/m_tb * N/n_tb).

Online ABFT corrects on the fly: expected executions 1.  Offline (detect-only)
ABFT restarts on a detected error, and the paper sums the restart series


    E = (1 - gamma) + 2 gamma ((1 - gamma) + 2 gamma (...)) = (1 - gamma) / (1 - 2 gamma),

finite only for gamma < 1/2.  DESIGN.md reading R16: the factor 2 is the
paper's; the generative process that reproduces the series exactly is a binary
branching process (every erring execution is replaced by two executions; E is
the expected number of executions that finish clean) -- `simulate_offline`
draws it, independently of the closed form, to pin it.
"""
from __future__ import annotations

import math
import random


def gamma(gamma0: float, tiles: int) -> float:
    """Overall error rate of one call, PAPER.md:583 ("gamma = 1-(1-gamma_0)^{M/m x N/n}")."""
    if not (0.0 <= gamma0 < 1.0) or tiles < 1:
        raise ValueError("need 0 <= gamma0 < 1 and tiles >= 1")
    return 1.0 - (1.0 - gamma0) ** tiles


def offline_expected_runs(g: float) -> float:
    """(1 - gamma)(1 + 2 gamma + (2 gamma)^2 + ...) = (1-gamma)/(1-2gamma)."""
    if not (0.0 <= g < 0.5):
        raise ValueError("the offline restart series diverges for gamma >= 1/2")
    return (1.0 - g) / (1.0 - 2.0 * g)


def online_expected_runs(g: float) -> float:
    """"the expected computation times ... is just 1"."""
    return 1.0


def simulate_offline(g: float, trials: int, seed: int = 230501024, cap: int = 1 << 20) -> float:
    """Monte-Carlo mean of the branching process of reading R16: an execution
    finishes clean with probability 1-gamma (counted once), or errs and is
    replaced by two executions.  Mean count of clean executions -> (1-g)/(1-2g)."""
    rng = random.Random(seed)
    total = 0
    for _ in range(trials):
        pending, clean = 1, 0
        while pending and clean < cap:
            pending -= 1
            if rng.random() < g:
                pending += 2
            else:
                clean += 1
        total += clean
    return total / trials


def tiles_of(M: int, N: int, m_tb: int, n_tb: int) -> int:
    """M/m_tb x N/n_tb threadblock tiles (ceiling for ragged edges)."""
    return math.ceil(M / m_tb) * math.ceil(N / n_tb)
