"""The offline -> online handoff type (msbasis.py:397-418 of the reference).

The multiscale basis itself is built by the reference's own offline CEM/NLMC code
(out of scope here); any object with the six dense blocks works.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class CoarseSystem:
    """Galerkin projections of the fine mass/stiffness onto the split basis."""

    M11: np.ndarray
    A11: np.ndarray
    M12: np.ndarray
    A12: np.ndarray
    M22: np.ndarray
    A22: np.ndarray

    @property
    def d1(self) -> int:
        return self.M11.shape[0]

    @property
    def d2(self) -> int:
        return self.M22.shape[0]

    def mass_block(self) -> np.ndarray:
        """Full coarse mass [[M11, M12], [M12^T, M22]]."""
        return np.block([[self.M11, self.M12], [self.M12.T, self.M22]])

    @classmethod
    def from_any(cls, s) -> "CoarseSystem":
        """Accept the reference's CoarseSystem (or any object with the six blocks)."""
        g = lambda k: np.ascontiguousarray(np.asarray(getattr(s, k), dtype=float))  # noqa: E731
        return cls(g("M11"), g("A11"), g("M12"), g("A12"), g("M22"), g("A22"))
