"""Pins for oracle/contrast.py and oracle/rng.py (CPU only).

Pins: closed forms of eq. (1), eq. (2), the Gaussianity threshold (golden file
with citations), mathematical invariants of Upsilon, Monte-Carlo properties,
SplitMix64 published outputs, and distributional tests of the Box-Muller draws.
"""
import math
import os

import numpy as np
import pytest
import torch
from scipy import stats

import datagen
from datagen import sources as S
from oracle import contrast, rng

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.split("#", 1)[0].strip()
        if line:
            rows.append(line.split())
    return rows


@pytest.mark.parametrize("row", _golden("contrast_closed_forms.txt"), ids=lambda r: "_".join(r))
def test_closed_forms(row):
    fn, args, expected = row[0], row[1], float(row[2])
    if fn == "upsilon":
        got = float(contrast.upsilon(float(args)))
    elif fn == "alpha":
        got = float(contrast.kurtosis_alpha([float(v) for v in args.split(",")]))
    else:
        N, i, M = (int(v) for v in args.split(","))
        got = contrast.gaussianity_threshold(N, i, M)
    assert got == pytest.approx(expected, abs=1e-12, rel=1e-12)


def test_upsilon_invariants():
    a = np.linspace(-1.999, 50.0, 200001)
    u = contrast.upsilon(a)
    assert np.all(u >= -1e-15)
    assert abs(contrast.upsilon(0.0)) == 0.0
    neg, pos = a < 0, a > 0
    assert np.all(np.diff(u[neg]) < 0)          # strictly decreasing on (-2, 0)
    assert np.all(np.diff(u[pos]) > 0)          # strictly increasing on (0, inf)
    # local expansion Upsilon(a) = a^2/4 - a^3/12 + O(a^4)
    x = 1e-3
    assert contrast.upsilon(x) == pytest.approx(x * x / 4 - x ** 3 / 12, rel=1e-6)
    with pytest.raises(contrast.DomainError):
        contrast.upsilon(-2.0)
    vals, ok = contrast.upsilon_masked(np.array([-2.5, -2.0, 0.5]))
    assert list(ok) == [False, False, True] and np.isinf(vals[:2]).all()


def test_threshold_decreasing():
    th = [contrast.gaussianity_threshold(30, i, 10000) for i in range(1, 31)]
    assert all(a > b for a, b in zip(th, th[1:]))


def test_alpha_even_and_gaussian_zero():
    g = S._gen(7, "cpu")
    y = S.gaussian(1_000_000, g, "cpu").numpy()
    assert contrast.kurtosis_alpha(y) == contrast.kurtosis_alpha(-y)
    assert abs(contrast.kurtosis_alpha(y)) < 0.05
    lap = S.laplace(1_000_000, g, "cpu").numpy()
    assert contrast.kurtosis_alpha(lap) == pytest.approx(3.0, abs=0.15)


@pytest.mark.parametrize("rho,kappa_tol", [(1.0, 0.2), (1.5, 0.1), (2.0, 0.05), (4.0, 0.05)])
def test_generalised_gaussian_source(rho, kappa_tol):
    """datagen GG sampler vs closed-form moments."""
    g = S._gen(11, "cpu")
    u = S.gen_gaussian(rho, 1_000_000, g, "cpu").numpy()
    kappa = math.exp(math.lgamma(5 / rho) + math.lgamma(1 / rho) - 2 * math.lgamma(3 / rho)) - 3
    assert np.var(u) == pytest.approx(1.0, abs=0.01)
    assert contrast.kurtosis_alpha(u) == pytest.approx(kappa, abs=kappa_tol)


def test_gg_beta_closed_forms():
    assert datagen.gg_beta(2.0) == pytest.approx(math.sqrt(2.0), rel=1e-14)
    assert datagen.gg_beta(1.0) == pytest.approx(math.sqrt(0.5), rel=1e-14)


def test_splitmix64_published_outputs():
    exp = [int(l, 16) for l in open(os.path.join(GOLD, "splitmix64.txt")) if l.startswith("0x")]
    got = rng.splitmix64_mix(np.arange(1, len(exp) + 1, dtype=np.uint64) * rng.GOLDEN)
    assert [int(v) for v in got] == exp
    # counter form: seed 0, counters 0..3 give the same stream
    u = rng.uniforms(0, np.arange(4, dtype=np.uint64))
    assert np.allclose(u, ((np.array(exp, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53, rtol=0, atol=0)


def test_candidate_draws_are_standard_normal():
    R = rng.candidates(2001, 3, np.arange(4000), 50)
    z = R.ravel()
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1) < 0.01
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # pairs are independent: correlation of even/odd coordinates
    assert abs(np.corrcoef(R[:, 0], R[:, 1])[0, 1]) < 0.05
    # odd N drops the last sine half, prefix property
    assert np.array_equal(rng.candidates(5, 2, [7, 9], 7), rng.candidates(5, 2, [7, 9], 8)[:, :7])
    # different component / id / seed give different rows; id addressing is global
    A = rng.candidates(5, 2, np.arange(10), 8)
    assert np.array_equal(A[3:5], rng.candidates(5, 2, [3, 4], 8))
    assert not np.allclose(A, rng.candidates(5, 3, np.arange(10), 8))
    assert not np.allclose(A, rng.candidates(6, 2, np.arange(10), 8))
