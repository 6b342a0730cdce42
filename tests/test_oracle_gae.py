"""Pins for oracle.gae: single step, zeros, closed forms, library cumsum."""
import numpy as np

from oracle.gae import gae


def test_single_step_identity():
    # S:379 "t=1, r=1, V=0, bootstrap=0 -> advantage 1, return 1"
    out = gae(np.array([[1.0]]), np.array([[0.0], [0.0]]), 0.99, 0.95)
    assert out["adv"][0, 0] == 1.0 and out["ret"][0, 0] == 1.0


def test_zero_case():
    # S:380 "all rewards 0, all values 0 -> all advantages 0"
    out = gae(np.zeros((16, 5)), np.zeros((17, 5)), 0.99, 0.95)
    assert np.all(out["adv"] == 0)


def test_constant_delta_geometric_series():
    # V = 0, r = c: delta = c, A[k] = c (1 - (g l)^(t-k)) / (1 - g l)
    t, c, g, l = 20, 0.7, 0.99, 0.95
    out = gae(np.full((t, 3), c), np.zeros((t + 1, 3)), g, l)
    k = np.arange(t)
    exp = c * (1 - (g * l) ** (t - k)) / (1 - g * l)
    assert np.allclose(out["adv"][:, 1], exp, rtol=1e-13)


def test_lambda_zero_is_td_error():
    rng = np.random.default_rng(0)
    r, v = rng.normal(size=(9, 4)), rng.normal(size=(10, 4))
    out = gae(r, v, 0.9, 0.0)
    assert np.allclose(out["adv"], r + 0.9 * v[1:] - v[:-1], atol=1e-14)


def test_gamma_lambda_one_is_reverse_cumsum():
    # gamma = lambda = 1: A[k] = sum_{j >= k} delta[j] (library reverse cumulative sum)
    rng = np.random.default_rng(1)
    r, v = rng.normal(size=(12, 6)), rng.normal(size=(13, 6))
    out = gae(r, v, 1.0, 1.0)
    delta = r + v[1:] - v[:-1]
    assert np.allclose(out["adv"], np.cumsum(delta[::-1], axis=0)[::-1], atol=1e-12)
    # and the telescoping closed form: A[0] = sum r - V[0] + V[t]
    assert np.allclose(out["adv"][0], r.sum(0) - v[0] + v[-1], atol=1e-12)


def test_recursion_identity():
    # A[k] = delta[k] + g l A[k+1] (the recursion the kernel uses) holds for the direct sum
    rng = np.random.default_rng(2)
    r, v = rng.normal(size=(30, 3)), rng.normal(size=(31, 3))
    out = gae(r, v, 0.97, 0.9)
    assert np.allclose(out["adv"][:-1], out["delta"][:-1] + 0.97 * 0.9 * out["adv"][1:], atol=1e-12)
