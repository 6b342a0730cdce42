"""GAE oracle — TEST INFRASTRUCTURE.

P:198 / P:212: PPO over n agents x t = 128 environment steps per training step (the paper
names PPO; GAE is the standard advantage estimator).  Continuing task: no
terminal flags; the value array carries the bootstrap row t.

Definition, written out as the direct double sum — no recursion:
    delta[k, i] = r[k, i] + gamma V[k+1, i] - V[k, i]
    A[k, i]     = sum_{l=0}^{t-1-k} (gamma lambda)^l delta[k+l, i]
    R[k, i]     = A[k, i] + V[k, i]
Layout: time-major [t][n] (reward, adv, ret) and [t+1][n] (value).
"""
from __future__ import annotations

import numpy as np


def gae(reward: np.ndarray, value: np.ndarray, gamma: float, lam: float) -> dict:
    r = np.asarray(reward, np.float64)
    v = np.asarray(value, np.float64)
    t = r.shape[0]
    delta = r + gamma * v[1:] - v[:-1]
    adv = np.zeros_like(r)
    g = gamma * lam
    for k in range(t):
        for l in range(t - k):
            adv[k] += g ** l * delta[k + l]
    return {"adv": adv, "ret": adv + v[:-1], "delta": delta}
