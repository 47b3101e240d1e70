"""torch-default Adam in float64 ("the default PyTorch Adam optimizer";
reading c21: beta = (0.9, 0.999), eps = 1e-8, bias correction, no weight decay)
and the DDP gradient mean ("averaged across all workers through an
all-reduce operation"; S:443 fixed ascending-rank order, reading c18).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def adam_step(theta, grad, m, v, step: int, lr: float, beta1=0.9, beta2=0.999, eps=1e-8,
              grad_scale: float = 1.0):
    """One Adam update at 1-based ``step``: g = grad_scale * grad;
    m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
    theta -= lr * (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps).
    Returns new (theta, m, v) in float64."""
    g = np.asarray(grad, np.float64) * grad_scale
    m = beta1 * np.asarray(m, np.float64) + (1.0 - beta1) * g
    v = beta2 * np.asarray(v, np.float64) + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** step)
    vhat = v / (1.0 - beta2 ** step)
    theta = np.asarray(theta, np.float64) - lr * mhat / (np.sqrt(vhat) + eps)
    return theta, m, v


def allreduce_mean(per_rank_grads) -> np.ndarray:
    """Mean over ranks, summed in ascending rank order."""
    acc = np.zeros_like(np.asarray(per_rank_grads[0], np.float64))
    for g in per_rank_grads:
        acc = acc + np.asarray(g, np.float64)
    return acc / len(per_rank_grads)
