"""Seeded synthetic inputs for the Vogue environment step (arxiv 2207.03945).

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA path's
tests/bench.  It holds parameters and random-number generation, and none of the
method's arithmetic (no integrate, no binning, no sensing, no reward).

Parameter defaults are SPEC.md's because the paper fixes only ratios and
dimensions.  Every float is stored as the value of an
fp32 number (SURVEY.md §8c reading A12): the CUDA path consumes the fp32 value and the
oracle promotes that same value exactly to fp64.

Workloads C1..C5 are BASELINE.json's ``configs``.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

FLOCK = "flock"
TAG = "tag"


def f32(x: float) -> float:
    """Round a Python float to the nearest fp32 value (returned as a Python float)."""
    return float(np.float32(x))


@dataclasses.dataclass(frozen=True)
class EnvParams:
    """World + environment parameters (field names match ``vg_config`` in include/vg.h)."""

    env: str                    # "flock" | "tag"
    n_agents: int               # N, agents per replica
    n_replicas: int = 1         # R
    width: float = 100.0        # L (square torus; reading A9)
    d_v: float = 10.0           # view range and reward radius = L/10
    d_r: float = 0.25           # body radius; contact at 2 d_r
    fov: float = f32(250.0 * math.pi / 180.0)   # "approximately 250 degrees"
    v: int = 128                # sectors per channel: flock 128, tag 64
    grid: int = 0               # G cells per axis; 0 = auto (reading A16)
    s_min: float = f32(0.05)
    s_max: float = 0.5
    a_max: float = f32(0.1)
    theta_max: float = f32(0.2)
    c_collide: float = 1.0
    c_near: float = 0.5
    d_peak: float = 5.25        # (2 d_r + d_v)/2
    n_chasers: int = 0          # tag: agents [N - n_chasers, N) are chasers (reading A14)
    r_touch: float = 1.0
    w_prox: float = f32(0.1)
    s_max_chaser: float = 0.375  # 0.75 s_max
    vision: str = "sector"      # "sector" (hot path) | "ray" (ray-disc reading, NEXT #2)

    @property
    def channels(self) -> int:
        return 1 if self.env == FLOCK else 2

    @property
    def obs_dim(self) -> int:
        # flock: 128 view + speed = 129; tag: 2 x 64 = 128
        return self.channels * self.v + (1 if self.env == FLOCK else 0)

    @property
    def occ_words(self) -> int:
        return (self.channels * self.v + 31) // 32

    @property
    def total_agents(self) -> int:
        return self.n_agents * self.n_replicas

    def replace(self, **kw) -> "EnvParams":
        return dataclasses.replace(self, **kw)


def flock_params(n_agents: int, n_replicas: int = 1, width: float = 100.0,
                 d_v: float | None = None, **kw) -> EnvParams:
    """Flock defaults.  d_v defaults to width/10."""
    width = f32(width)
    d_v = f32(width / 10.0) if d_v is None else f32(d_v)
    d_r = f32(kw.pop("d_r", 0.25))
    d_peak = kw.pop("d_peak", None)
    d_peak = f32((2.0 * d_r + d_v) / 2.0) if d_peak is None else f32(d_peak)
    return EnvParams(env=FLOCK, n_agents=n_agents, n_replicas=n_replicas, width=width,
                     d_v=d_v, d_r=d_r, d_peak=d_peak, v=kw.pop("v", 128), **kw)


def tag_params(n_agents: int, n_replicas: int = 1, width: float = 100.0,
               d_v: float | None = None, n_chasers: int | None = None, **kw) -> EnvParams:
    """Tag defaults.  1/10 of agents are chasers (reading A14)."""
    width = f32(width)
    d_v = f32(width / 10.0) if d_v is None else f32(d_v)
    d_r = f32(kw.pop("d_r", 0.25))
    d_peak = kw.pop("d_peak", None)
    d_peak = f32((2.0 * d_r + d_v) / 2.0) if d_peak is None else f32(d_peak)
    if n_chasers is None:
        n_chasers = n_agents // 10
    return EnvParams(env=TAG, n_agents=n_agents, n_replicas=n_replicas, width=width,
                     d_v=d_v, d_r=d_r, d_peak=d_peak, v=kw.pop("v", 64),
                     n_chasers=n_chasers, **kw)


# --------------------------------------------------------------------------------------
# Workloads: BASELINE.json configs[0..4] (SURVEY.md §8d "Concrete synthetic inputs").
# C5 keeps the paper's density (0.5 agents per unit area, as C2) with d_v = 10:
# L = RN32(100 * sqrt(200)) so that N / L^2 = 0.5 at N = 10^6.
# --------------------------------------------------------------------------------------
C5_WIDTH = f32(100.0 * math.sqrt(200.0))


def workload(name: str) -> EnvParams:
    name = name.lower()
    if name == "c1":
        return flock_params(100)
    if name == "c2":
        return flock_params(5000)
    if name == "c3":
        return tag_params(10000, n_chasers=1000)
    if name == "c4":
        return flock_params(5000, n_replicas=1024)
    if name == "c5":
        # G = 136 (c = 10.399 >= d_v (1 + 2^-12)) rather than the auto 141, so that the
        # x-slabs of 1/2/4/8 GPUs are whole, equal column ranges.
        return flock_params(1_000_000, width=C5_WIDTH, d_v=10.0, grid=136)
    raise KeyError(name)


WORKLOAD_DESCRIPTIONS = {
    "c1": "flock 1x100, L=100, 100 steps, seeded random actions",
    "c2": "flock 1x5000, L=100 (paper Fig. 1 scale)",
    "c3": "tag 1x10000 (9000 runners + 1000 chasers), L=100",
    "c4": "flock 1024 replicas x 5000, L=100",
    "c5": "flock single 1,000,000-agent world, L=1414.2136, d_v=10 (paper density)",
}


# --------------------------------------------------------------------------------------
# Seeded generators (SURVEY.md §8c readings A20, A21)
# --------------------------------------------------------------------------------------
TWO_PI_F32 = np.float32(2.0 * math.pi)   # RN32(2 pi): exclusive upper bound of a stored heading


def _uniform_f32_below(rng: np.random.Generator, n: int, hi: float) -> np.ndarray:
    """U[0, hi) drawn in fp64 and rounded to fp32, kept strictly below fp32(hi)."""
    x = (rng.random(n) * hi).astype(np.float32)
    x[x >= np.float32(hi)] = np.float32(0.0)
    return x


def init_state(p: EnvParams, seed: int = 0, replicas: range | None = None) -> np.ndarray:
    """Initial state, fp32 [R, N, 4] = (x, y, theta, s) (reading A20).

    Replica r draws from PCG64(seed + r): positions U[0, L)^2, heading U[0, 2 pi),
    flock speed (s_min + s_max)/2; tag's fourth column is reserved and set to 0
    (type comes from the index: the last n_chasers agents are chasers).
    """
    reps = range(p.n_replicas) if replicas is None else replicas
    out = np.empty((len(reps), p.n_agents, 4), dtype=np.float32)
    for k, r in enumerate(reps):
        rng = np.random.Generator(np.random.PCG64(seed + r))
        out[k, :, 0] = _uniform_f32_below(rng, p.n_agents, p.width)
        out[k, :, 1] = _uniform_f32_below(rng, p.n_agents, p.width)
        th = (rng.random(p.n_agents) * (2.0 * math.pi)).astype(np.float32)
        th[th >= TWO_PI_F32] = np.float32(0.0)
        out[k, :, 2] = th
        if p.env == FLOCK:
            out[k, :, 3] = np.float32(0.5 * (p.s_min + p.s_max))
        else:
            out[k, :, 3] = np.float32(0.0)
    return out


def clustered_state(p: EnvParams, seed: int = 0, n_clusters: int = 16,
                    sigma: float | None = None) -> np.ndarray:
    """Stress variant: Gaussian clusters with sigma = 2 d_v, wrapped."""
    sigma = 2.0 * p.d_v if sigma is None else sigma
    out = init_state(p, seed)
    for r in range(p.n_replicas):
        rng = np.random.Generator(np.random.PCG64(seed + 7919 * (r + 1)))
        centres = rng.random((n_clusters, 2)) * p.width
        which = rng.integers(0, n_clusters, p.n_agents)
        xy = centres[which] + rng.normal(0.0, sigma, (p.n_agents, 2))
        xy = np.mod(xy, p.width).astype(np.float32)
        xy[xy >= np.float32(p.width)] = np.float32(0.0)
        out[r, :, :2] = xy
    return out


def action_box(p: EnvParams) -> tuple[np.ndarray, np.ndarray]:
    """Per-agent action bounds [N, 2] (lo, hi)."""
    lo = np.empty((p.n_agents, 2), dtype=np.float64)
    hi = np.empty((p.n_agents, 2), dtype=np.float64)
    if p.env == FLOCK:
        lo[:, 0], hi[:, 0] = -p.a_max, p.a_max          # accelerate
        lo[:, 1], hi[:, 1] = -p.theta_max, p.theta_max  # rotate
    else:
        lo[:, 0], hi[:, 0] = -p.theta_max, p.theta_max  # rotate
        lo[:, 1] = 0.0                                   # move along heading
        hi[:, 1] = p.s_max
        hi[p.n_agents - p.n_chasers:, 1] = p.s_max_chaser
    return lo, hi


def actions(p: EnvParams, seed: int = 0, step: int = 0,
            replicas: range | None = None) -> np.ndarray:
    """Seeded uniform actions in the action box, fp32 [R, N, 2] (reading A21)."""
    reps = range(p.n_replicas) if replicas is None else replicas
    lo, hi = action_box(p)
    out = np.empty((len(reps), p.n_agents, 2), dtype=np.float32)
    for k, r in enumerate(reps):
        ss = np.random.SeedSequence([seed ^ 0x9E3779B9, step, r])
        rng = np.random.Generator(np.random.PCG64(ss))
        u = rng.random((p.n_agents, 2))
        out[k] = (lo + u * (hi - lo)).astype(np.float32)
    return out


# --------------------------------------------------------------------------------------
# Shared-policy weights ("two hidden layers with 64 nodes")
# --------------------------------------------------------------------------------------
POLICY_KEYS = ("W1", "b1", "W2", "b2", "W3", "b3", "log_std", "V1", "c1", "V2", "c2", "V3", "c3")


def policy_weights(obs_dim: int, seed: int = 0, hidden: int = 64, act_dim: int = 2,
                   log_std: float = -1.0) -> dict:
    """Seeded fp32 actor/critic weights, uniform in +-1/sqrt(fan_in) (random init)."""
    rng = np.random.default_rng(seed)

    def u(*shape, fan):
        return (rng.uniform(-1.0, 1.0, shape) / math.sqrt(fan)).astype(np.float32)

    return {"W1": u(hidden, obs_dim, fan=obs_dim), "b1": u(hidden, fan=obs_dim),
            "W2": u(hidden, hidden, fan=hidden), "b2": u(hidden, fan=hidden),
            "W3": u(act_dim, hidden, fan=hidden), "b3": u(act_dim, fan=hidden),
            "log_std": np.full(act_dim, log_std, np.float32),
            "V1": u(hidden, obs_dim, fan=obs_dim), "c1": u(hidden, fan=obs_dim),
            "V2": u(hidden, hidden, fan=hidden), "c2": u(hidden, fan=hidden),
            "V3": u(1, hidden, fan=hidden), "c3": u(1, fan=hidden)}


# --------------------------------------------------------------------------------------
# Opinion-dynamics graph (Listing 1)
# --------------------------------------------------------------------------------------
def opinion_graph(n: int, degree: int, seed: int = 0) -> dict:
    """Random directed graph, `degree` distinct out-neighbours per node (no self loops),
    CSR sorted by (src, dst); weights U[0, 1]; opinions U[0, 1] (fp32)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    deg = min(degree, n - 1)
    cols = []
    for i in range(n):
        c = rng.choice(n - 1, deg, replace=False) if deg > 0 else np.zeros(0, np.int64)
        c = c + (c >= i)                     # skip the self loop
        cols.append(np.sort(c))
    col = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    row_ptr = (np.arange(n + 1) * deg).astype(np.int32)
    weight = rng.random(len(col)).astype(np.float32)
    op = rng.random(n).astype(np.float32)
    return {"row_ptr": row_ptr, "col": col, "weight": weight, "op": op}


def opinion_graph_fast(n: int, degree: int, seed: int = 0) -> dict:
    """Large-n variant (bench): out-neighbours drawn with replacement then de-duplicated
    per row is avoided — uniform random dst != src, sorted per row, duplicates allowed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    dst = rng.integers(0, n - 1, size=(n, degree))
    dst = dst + (dst >= np.arange(n)[:, None])
    dst.sort(axis=1)
    return {"row_ptr": (np.arange(n + 1) * degree).astype(np.int32),
            "col": dst.reshape(-1).astype(np.int32),
            "weight": rng.random(n * degree).astype(np.float32),
            "op": rng.random(n).astype(np.float32)}


def rim_state(p: EnvParams, n_q: int, seed: int, radius: float) -> np.ndarray:
    """Queries (a third of them within d_v of a wrap edge) each ringed by 16 neighbours just
    inside the view radius (d = d_v (1 - 1e-4)), plus uniform background agents: every
    window edge of K4 (along the run axis and at the chord limit of the adjacent rows) is hit."""
    rng = np.random.default_rng(seed)
    L = p.width
    q = rng.random((n_q, 2)) * L
    edge = rng.random(n_q) < 1 / 3
    axis = rng.integers(0, 2, n_q)
    for ax in (0, 1):
        m = edge & (axis == ax)
        q[m, ax] = rng.choice([0.3, L - 0.3], m.sum()) + rng.normal(0, 0.1, m.sum())
    ang = rng.random((n_q, 1)) * 2 * np.pi + np.arange(16)[None, :] * (2 * np.pi / 16)
    rim = q[:, None, :] + radius * (1 - 1e-4) * np.stack([np.cos(ang), np.sin(ang)], -1)
    pts = np.concatenate([q, rim.reshape(-1, 2)])
    pts = np.concatenate([pts, rng.random((p.n_agents - len(pts), 2)) * L]) % L
    st = np.zeros((1, p.n_agents, 4), np.float32)
    st[0, :, :2] = pts.astype(np.float32) % np.float32(L)
    st[0, :, 2] = (rng.random(p.n_agents) * 6.28).astype(np.float32)
    st[0, :, 3] = 0.275
    return st
