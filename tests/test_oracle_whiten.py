"""Pins for oracle/whiten.py (readings A11/A12): invariants and SPEC worked examples."""
import numpy as np
import pytest

import datagen
from oracle import whiten as W


def test_center_examples():
    Xc, mean = W.center(np.array([[1.0, 2.0, 3.0], [1.0, 1.0, 1.0]]))
    assert np.allclose(Xc, [[-1, 0, 1], [0, 0, 0]]) and np.allclose(mean, [2, 1])


def test_whitening_invariants():
    ds = datagen.make_dataset(datagen.get(0))
    X = ds.X.numpy()
    Xw, mean, V, d = W.whiten(X)
    M = X.shape[1]
    assert np.abs(Xw @ Xw.T / M - np.eye(8)).max() < 1e-10
    Xc = X - X.mean(1, keepdims=True)
    C = Xc @ Xc.T / M
    assert np.abs(V @ C @ V.T - np.eye(8)).max() < 1e-10
    assert np.all(np.diff(d) <= 0)                                  # descending eigenvalues
    E = (V.T * np.sqrt(d))                                          # recover eigenvectors
    for k in range(8):
        assert E[np.argmax(np.abs(E[:, k])), k] > 0                 # sign convention
    assert np.abs(Xw.mean(1)).max() < 1e-12


def test_scaled_white_noise_example():
    """rows scaled by (2, 1) -> recovered unit covariance."""
    rng = np.random.default_rng(0)
    Z = rng.standard_normal((2, 5000)) * np.array([[2.0], [1.0]])
    Xw, _, V, d = W.whiten(Z)
    assert np.abs(Xw @ Xw.T / 5000 - np.eye(2)).max() < 1e-10


def test_already_white_gives_orthogonal_V():
    rng = np.random.default_rng(1)
    Xw0, *_ = W.whiten(rng.standard_normal((5, 4000)))
    _, _, V, _ = W.whiten(Xw0)
    assert np.abs(V @ V.T - np.eye(5)).max() < 1e-8


def test_rank_deficient():
    rng = np.random.default_rng(2)
    Z = rng.standard_normal((3, 1000))
    Z = np.vstack([Z, Z[:1]])                                       # duplicated row
    with pytest.raises(W.RankDeficient):
        W.whiten(Z)
