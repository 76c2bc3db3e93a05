"""Accuracy metrics of a computed decomposition (verify.py:24-60 of the reference).

Host numpy, as in the reference CLI's `verify`: these check a result, they are not part of the
EVD path.  For the headline sizes the device versions in `matgen.accuracy` are used instead.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

from .core import EPS


def backward_error(a, q, lam) -> float:
    """||A - Q diag(lam) Q^T||_F / (n ||A||_F)."""
    a = np.asarray(a, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    n = a.shape[0]
    resid = float(np.linalg.norm(a - (q * lam) @ q.T))
    scale = float(np.linalg.norm(a))
    if scale == 0.0:
        return 0.0 if resid == 0.0 else math.inf
    return resid / (n * scale)


def orthogonality(q) -> float:
    """||I - Q Q^T||_F / n."""
    q = np.asarray(q, dtype=np.float64)
    n = q.shape[0]
    return float(np.linalg.norm(np.eye(n) - q @ q.T)) / n


@dataclass
class AccuracyReport:
    """Backward error and orthogonality; bound_ok iff ortho <= 2 eps slack (verify.py:43-60)."""

    backward: float
    ortho: float
    eps: float
    bound_ok: bool
    slack: float = 16.0

    @classmethod
    def from_decomposition(cls, a, q, lam, slack: float = 16.0) -> "AccuracyReport":
        back = backward_error(a, q, lam)
        orth = orthogonality(q)
        return cls(backward=back, ortho=orth, eps=EPS, bound_ok=orth <= 2.0 * EPS * slack,
                   slack=slack)

    def to_dict(self) -> dict:
        return {"backward": self.backward, "ortho": self.ortho, "eps": self.eps,
                "bound_ok": self.bound_ok, "slack": self.slack}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)
