"""CPU oracle for the Vogue environment step (arxiv 2207.03945) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2207_03945_b200``) never imports, links or executes it, and this package imports
nothing from the product.  The only shared module is ``vg_inputs`` (seeded generators and
parameter values, no method arithmetic).

What it is: a plain, slow, obviously correct fp64 NumPy implementation of one environment
step — integrate, grid binning as a textbook stable argsort
(S:41-47), and sensing + reward by O(N^2) brute force over all pairs (P:158, P:164,
P:171-178).  Readings of gaps are SURVEY.md §8c A1-A25, listed in DESIGN.md.

Pins: see tests/test_oracle_*.py.  Parts with no pin: the *intended* shape of the reward
function f between 2 d_r and d_v and the intended vision model are readings (A1, A5) —
"parity unpinned" w.r.t. the authors' intent; the oracle pins our reading.
"""
from .env import (  # noqa: F401
    grid_size,
    integrate,
    cell_ids,
    bins,
    minimal_image,
    reward_f,
    sense_rows,
    sense,
    step,
    BAND,
)
