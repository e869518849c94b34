"""Seeded synthetic source generators (input recipe only; no ordering-ICA arithmetic).

This module is shared by the oracle-side tests and the CUDA-side tests/bench.
It holds ONLY the random input recipe: source distributions, the mixing matrix
and the sensor-noise model that BASELINE.json's configs describe.  It contains
none of the method's arithmetic (no whitening, no kurtosis, no fixed point).

Source families (all unit variance unless stated; readings in DESIGN.md §3):
  * Laplace(0, 1/sqrt 2)                                 kappa = 3
  * Student-t(nu) scaled by sqrt((nu-2)/nu)              kappa = 6/(nu-4)
  * generalised Gaussian, PAPER.md:296-298 (section 4.2):
        p(u) = rho exp(-(|u|/beta)^rho) / (2 beta Gamma(1/rho)),
        beta chosen so the variance is 1; "shape" in BASELINE.json is rho.
    Sampled by the gamma transform u = s * beta * g^(1/rho), g ~ Gamma(1/rho, 1).
  * sparse spikes Bernoulli(p) * N(0, var) (not rescaled; whitening normalises)
  * Gaussian AR(1): x0 ~ N(0,1), x_t = r x_{t-1} + sqrt(1-r^2) e_t (unit variance)
"""
from __future__ import annotations

import math

import numpy as np
import torch


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def laplace(M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """Unit-variance Laplace: scale b = 1/sqrt(2) (variance 2 b^2 = 1)."""
    e = torch.empty(M, dtype=dtype, device=device).exponential_(generator=g)
    s = torch.randint(0, 2, (M,), generator=g, device=device).to(dtype) * 2 - 1
    return s * e / math.sqrt(2.0)


def student_t(nu: float, M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """Student-t(nu) scaled to unit variance (requires nu > 2)."""
    z = torch.randn(M, dtype=dtype, device=device, generator=g)
    a = torch.full((M,), nu / 2.0, dtype=dtype, device=device)
    chi2 = 2.0 * torch._standard_gamma(a, generator=g)
    return z / torch.sqrt(chi2 / nu) * math.sqrt((nu - 2.0) / nu)


def gg_beta(rho: float) -> float:
    """Scale beta giving unit variance: Var = beta^2 Gamma(3/rho)/Gamma(1/rho)."""
    return math.exp(0.5 * (math.lgamma(1.0 / rho) - math.lgamma(3.0 / rho)))


def gen_gaussian(rho: float, M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """Generalised Gaussian of shape rho, unit variance."""
    a = torch.full((M,), 1.0 / rho, dtype=dtype, device=device)
    gam = torch._standard_gamma(a, generator=g)
    s = torch.randint(0, 2, (M,), generator=g, device=device).to(dtype) * 2 - 1
    return s * gg_beta(rho) * gam.pow(1.0 / rho)


def spikes(p: float, var: float, M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """Sparse spike train Bernoulli(p) * N(0, var)."""
    b = (torch.rand(M, dtype=dtype, device=device, generator=g) < p).to(dtype)
    return b * torch.randn(M, dtype=dtype, device=device, generator=g) * math.sqrt(var)


def ar1(r: float, M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """Unit-variance Gaussian AR(1) process (linear filter evaluated on the host)."""
    from scipy.signal import lfilter

    e = torch.randn(M, dtype=torch.float64, generator=_gen(int(torch.randint(0, 2**62, (1,), generator=g, device=g.device).item()), "cpu")).numpy()
    e[1:] *= math.sqrt(1.0 - r * r)
    x = lfilter([1.0], [1.0, -r], e)
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device, dtype=dtype)


def uniform(M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """Unit-variance uniform on [-sqrt 3, sqrt 3] (excess kurtosis -1.2)."""
    return (torch.rand(M, dtype=dtype, device=device, generator=g) * 2 - 1) * math.sqrt(3.0)


def gaussian(M: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    return torch.randn(M, dtype=dtype, device=device, generator=g)


def mixing_matrix(N: int, g: torch.Generator, device, dtype=torch.float64, max_cond: float = 1e6) -> torch.Tensor:
    """A ~ iid N(0,1), redrawn until cond(A) < max_cond."""
    for _ in range(100):
        A = torch.randn(N, N, dtype=torch.float64, device=device, generator=g)
        if float(torch.linalg.cond(A.cpu())) < max_cond:
            return A.to(dtype)
    raise RuntimeError("mixing matrix generation failed")
