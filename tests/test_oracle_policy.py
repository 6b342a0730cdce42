"""Pins for oracle.policy: Philox known-answer vectors, Gaussian
statistics, closed-form special cases of the MLP, a library cross-check.  No GPU."""
import math

import numpy as np
import pytest

import vg_inputs as vi
from oracle import policy as pol


def test_philox_known_answers():
    # Random123 known-answer vectors for philox4x32-10 (kat_vectors: ctr, key -> out).
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, out in kat:
        got = pol.philox4x32_10(np.array([ctr], np.uint64), np.array([key], np.uint64))[0]
        assert tuple(int(x) for x in got) == out


def test_normals_statistics():
    # S:363 "empirical mean/std over 1e5 samples match within 3 sigma"; also independence.
    e = pol.normals(np.arange(200000), seed=123, step=7)
    n = e.shape[0]
    for d in range(2):
        assert abs(e[:, d].mean()) < 4 / math.sqrt(n)
        assert abs(e[:, d].std() - 1) < 4 * math.sqrt(0.5 / n)
    assert abs(np.corrcoef(e[:, 0], e[:, 1])[0, 1]) < 4 / math.sqrt(n)
    assert abs((e[:, 0] > 1.959964).mean() - 0.025) < 4 * math.sqrt(0.025 * 0.975 / n)
    # different steps / seeds give different streams; same inputs are deterministic
    assert not np.allclose(e[:10], pol.normals(np.arange(10), seed=123, step=8))
    assert np.array_equal(e[:10], pol.normals(np.arange(10), seed=123, step=7))


def test_zero_network():
    # S:352 "zero weights, zero biases -> mean 0, value 0 for any obs" (+ biases pass through)
    w = {k: np.zeros_like(v) for k, v in vi.policy_weights(129).items()}
    w["b3"] = np.array([0.25, -0.5], np.float32)
    w["c3"] = np.array([1.5], np.float32)
    out = pol.forward(w, np.random.default_rng(0).random((7, 129)))
    assert np.all(out["mean"] == [0.25, -0.5]) and np.all(out["value"] == 1.5)


def test_single_path_closed_form():
    # one nonzero weight per layer: mean_0 = c tanh(b tanh(a x_3 + p) + q) + r
    w = {k: np.zeros_like(v) for k, v in vi.policy_weights(129).items()}
    a, p, b, q, c, r = (float(np.float32(v)) for v in (0.7, 0.1, -1.3, 0.05, 2.0, -0.2))
    w["W1"][5, 3], w["b1"][5] = a, p
    w["W2"][9, 5], w["b2"][9] = b, q
    w["W3"][0, 9], w["b3"][0] = c, r
    x = np.zeros((1, 129))
    x[0, 3] = 0.4
    m = pol.forward(w, x)["mean"][0, 0]
    assert m == pytest.approx(c * math.tanh(b * math.tanh(a * 0.4 + p) + q) + r, abs=1e-15)


def test_matches_torch_float64():
    import torch
    w = vi.policy_weights(128, seed=3)
    x = np.random.default_rng(1).random((50, 128))
    out = pol.forward(w, x)
    t = {k: torch.tensor(v, dtype=torch.float64) for k, v in w.items()}
    xt = torch.tensor(x)
    h = torch.tanh(torch.nn.functional.linear(xt, t["W1"], t["b1"]))
    h = torch.tanh(torch.nn.functional.linear(h, t["W2"], t["b2"]))
    assert np.allclose(out["mean"], torch.nn.functional.linear(h, t["W3"], t["b3"]).numpy(), atol=1e-13)


def test_sample_rules():
    # log-prob of the unclipped sample, clipping to the box; S:332:
    # log_std clamped to [-5, 2] (-30 acts as -5, 10 as 2)
    w = vi.policy_weights(129)
    w["log_std"] = np.array([-30.0, 10.0], np.float32)
    mean = np.array([[0.3, 0.0], [10.0, -10.0]])
    s = pol.sample(w, mean, np.array([0, 1]), seed=1, step=0, lo=[-0.1, -0.2], hi=[0.1, 0.2])
    eps = s["eps"]
    assert s["raw"][0, 0] == pytest.approx(0.3 + math.exp(-5.0) * eps[0, 0], abs=1e-12)
    assert s["raw"][0, 1] == pytest.approx(math.exp(2.0) * eps[0, 1], abs=1e-12)
    assert s["action"][1, 0] == 0.1 and s["action"][1, 1] == -0.2
    assert s["logp"][0] == pytest.approx(-0.5 * (eps[0] ** 2).sum() + 5.0 - 2.0 - math.log(2 * math.pi))
    w["log_std"] = np.array([-1.0, 0.5], np.float32)        # inside the clamp: unchanged
    s = pol.sample(w, mean, np.array([0]), seed=1, step=0, lo=[-9, -9], hi=[9, 9])
    assert s["raw"][0, 0] == pytest.approx(0.3 + math.exp(-1.0) * s["eps"][0, 0], abs=1e-12)
