"""Result records shared with the reference's bootstrap API (bootstrap.py:46-60)."""

from dataclasses import dataclass

import numpy as np


@dataclass
class TestReport:
    """Convergence probe of one testing phase (bootstrap.py:46-53)."""

    __test__ = False  # not a pytest class

    stage: int
    rho_estimate: float
    rho_geometric: float
    per_iteration_anorms: np.ndarray
