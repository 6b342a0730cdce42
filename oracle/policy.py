"""Oracle for the shared policy forward — TEST INFRASTRUCTURE.

P:212: "The actor and critic PPO networks had two hidden layers with 64 nodes each";
P:198: PPO for a continuous action space with a shared policy; S:329-333 (MLPPolicy:
affine obs->64->64->out with tanh hidden activations, linear output, state-independent
log_std), S:355-372 (sample a ~ N(mean, exp(log_std)), clip to the action box, log-prob of
the unclipped Gaussian sample).

Plain fp64 NumPy; the weights and observations are the fp32 values the GPU consumes,
promoted exactly.  The Gaussian noise is drawn with Philox4x32-10 (Salmon et al., SC'11,
"Parallel random numbers: as easy as 1, 2, 3") keyed by (seed) and counted by
(agent row, step) — a counter-based generator implemented independently here and in the
CUDA kernel, then Box-Muller.  Parity pins: tests/test_oracle_policy.py.
"""
from __future__ import annotations

import math

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57          # Philox4x32 multipliers
W0, W1 = 0x9E3779B9, 0xBB67AE85          # Weyl key increments
MASK = 0xFFFFFFFF


def philox4x32_10(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    """Philox4x32 with 10 rounds.  ctr: uint [..., 4], key: uint [..., 2] -> uint32 [..., 4]."""
    c = [np.asarray(ctr[..., i], dtype=np.uint64) & MASK for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint64) & MASK
    k1 = np.asarray(key[..., 1], dtype=np.uint64) & MASK
    for r in range(10):
        p0 = c[0] * np.uint64(M0)          # 64-bit products of 32-bit words
        p1 = c[2] * np.uint64(M1)
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        if r < 9:
            k0 = (k0 + np.uint64(W0)) & np.uint64(MASK)
            k1 = (k1 + np.uint64(W1)) & np.uint64(MASK)
    return np.stack(c, axis=-1).astype(np.uint32)


def normals(rows: np.ndarray, seed: int, step: int) -> np.ndarray:
    """Two standard normals per row: Philox4x32-10 with counter (row, step_lo, step_hi, 0)
    and key (seed_lo, seed_hi); uniforms u = ((x >> 8) + 0.5) 2^-24 in (0, 1) from words 0
    and 1; Box-Muller: r = sqrt(-2 ln u0), eps = (r cos 2 pi u1, r sin 2 pi u1)."""
    rows = np.asarray(rows, dtype=np.uint64)
    ctr = np.zeros(rows.shape + (4,), dtype=np.uint64)
    ctr[..., 0] = rows & np.uint64(MASK)
    ctr[..., 1] = np.uint64(step & MASK)
    ctr[..., 2] = np.uint64((step >> 32) & MASK)
    key = np.zeros(rows.shape + (2,), dtype=np.uint64)
    key[..., 0] = np.uint64(seed & MASK)
    key[..., 1] = np.uint64((seed >> 32) & MASK)
    x = philox4x32_10(ctr, key).astype(np.float64)
    u0 = (np.floor(x[..., 0] / 256.0) + 0.5) * 2.0 ** -24
    u1 = (np.floor(x[..., 1] / 256.0) + 0.5) * 2.0 ** -24
    r = np.sqrt(-2.0 * np.log(u0))
    return np.stack([r * np.cos(2 * math.pi * u1), r * np.sin(2 * math.pi * u1)], axis=-1)


def forward(w: dict, obs: np.ndarray) -> dict:
    """Actor mean [M, 2] and critic value [M], fp64.

    w: W1 [64, d], b1, W2 [64, 64], b2, W3 [2, 64], b3 [2], log_std [2] (actor);
       V1 [64, d], c1, V2 [64, 64], c2, V3 [1, 64], c3 [1] (critic).
    """
    x = np.asarray(obs, dtype=np.float64)
    f = {k: np.asarray(v, dtype=np.float64) for k, v in w.items()}
    h = np.tanh(x @ f["W1"].T + f["b1"])
    h = np.tanh(h @ f["W2"].T + f["b2"])
    mean = h @ f["W3"].T + f["b3"]
    g = np.tanh(x @ f["V1"].T + f["c1"])
    g = np.tanh(g @ f["V2"].T + f["c2"])
    value = (g @ f["V3"].T + f["c3"])[:, 0]
    return {"mean": mean, "value": value}


def sample(w: dict, mean: np.ndarray, rows: np.ndarray, seed: int, step: int,
           lo: np.ndarray, hi: np.ndarray) -> dict:
    """a_raw = mean + exp(log_std) eps; action = clip(a_raw, box); log-prob of
    the unclipped Gaussian: sum_d -eps_d^2/2 - log_std_d - log(2 pi)/2; log_std
    clamped to [-5, 2] first."""
    eps = normals(rows, seed, step)
    ls = np.clip(np.asarray(w["log_std"], dtype=np.float64), -5.0, 2.0)
    raw = np.asarray(mean, np.float64) + np.exp(ls) * eps
    act = np.clip(raw, np.asarray(lo, np.float64), np.asarray(hi, np.float64))
    logp = (-0.5 * eps ** 2 - ls - 0.5 * math.log(2 * math.pi)).sum(-1)
    return {"eps": eps, "raw": raw, "action": act, "logp": logp}
