"""Ensemble mode: independent Monte-Carlo replicas, one per
rank, sharded with no data-path collective.  Replica r draws every random
number with `replica = r` in Philox counter word 3 (include/rbm.h), so the
system on rank r is exactly the single-GPU run with replica = r.

Plumbing only: every step runs in librbm.so through the C ABI.
"""
from __future__ import annotations

import numpy as np

from .rbm import RBM


def run_replica(cfg: dict, replica: int, steps: int, device=None) -> np.ndarray:
    """Run replica `replica` of cfg for `steps` steps; positions in id order (host)."""
    s = RBM(dict(cfg, replica=int(replica)), device=device)
    try:
        s.run(steps)
        return s.gather(host=True)
    finally:
        s.close()


def ensemble_moments(x: np.ndarray) -> np.ndarray:
    """Per-replica summary (mean and second moment per axis) for the optional
    final reduction of statistics across ranks."""
    x = np.asarray(x, np.float64)
    return np.concatenate([x.mean(0), (x * x).mean(0)])
