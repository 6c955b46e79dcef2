"""Pins for oracle/interf.py (C3): planted recovery, rank error,
residual orthogonality, the arithmetic example, clamp,
noisy fit error shape."""
import numpy as np
import pytest

from oracle import interf

PLANT = np.array([0.2, 0.1, 0.5, 0.3, 1.0])


def _samples(n, seed=0):
    r = np.random.default_rng(seed)
    return interf.design(r.random(n), r.random(n), r.random(n), r.random(n))


def test_planted_recovery():
    X = _samples(2500)
    c = interf.fit(X, X @ PLANT)
    np.testing.assert_allclose(c, PLANT, atol=1e-6)


def test_rank_error():
    X = np.tile(_samples(1), (100, 1))
    with pytest.raises(interf.RankError):
        interf.fit(X, np.ones(100))


def test_residual_orthogonal():
    X = _samples(300, 1)
    y = X @ PLANT + np.random.default_rng(2).normal(0, 0.05, 300)
    c = interf.fit(X, y)
    np.testing.assert_allclose(X.T @ (y - X @ c), 0, atol=1e-9)


def test_predict_examples():
    assert abs(interf.predict(PLANT, 0.5, 0.5, 0.4, 0.4) - 1.47) < 1e-12
    assert interf.predict(np.array([0, 0, 0, 0, 0.9]), 0.3, 0.3, 0.3, 0.3) == 1.0
    assert abs(interf.overhead(PLANT, 100.0, 0.5, 0.5, 0.4, 0.4) - 47.0) < 1e-9


def test_noisy_split_error():
    X = _samples(2500, 3)
    y = X @ PLANT + np.random.default_rng(4).normal(0, 0.05, 2500)
    tr, va = interf.split(2500, seed=5)
    assert len(tr) == 1750 and len(va) == 750 and not set(tr) & set(va)
    c = interf.fit(X[tr], y[tr])
    err = interf.rel_errors(c, X[va], y[va])
    assert np.percentile(err, 90) < 0.15
