"""Black & Scholes oracle, serial fp64 (TEST INFRASTRUCTURE ONLY).

PAPER.md §V-B: "Black & Scholes equation for European call options,
for 10 underlying stocks, and 10 vectors of prices.  Adapted from [28] (CUDA
samples, L1601-1602) ... with double-precision arithmetic".  The call price
and the cumulative normal follow the textbook formula the cited sample uses
(Abramowitz & Stegun 26.2.17 polynomial), SURVEY §8(c2) B&S:

    d1 = (ln(S/K) + (R + V^2/2) T) / (V sqrt(T)),  d2 = d1 - V sqrt(T)
    C  = S CND(d1) - K exp(-R T) CND(d2)

Constants R, V, T, K are readings (parity unpinned (constant)): the paper
prints none.  Pins (tests/test_oracle_bs.py): |CND - Phi| <= 7.5e-8 against
scipy.special.ndtr; C within (S+K)*7.5e-8 of the exact price built from
scipy's Phi; put-call parity; deep in/out-of-the-money limits.
"""
import numpy as np

# SURVEY §8(c2) B&S constants (readings; see DESIGN.md R-BS)
R = 0.08
V = 0.30
T = 1.0
K = 60.0

A1, A2, A3, A4, A5 = 0.31938153, -0.356563782, 1.781477937, -1.821255978, 1.330274429
RSQRT2PI = 0.39894228040143267794


def cnd(d):
    """A&S 26.2.17: k = 1/(1+0.2316419|d|); p = phi(d) k (a1 + k(a2 + ...));
    CND = 1 - p for d > 0 else p."""
    d = np.asarray(d, dtype=np.float64)
    k = 1.0 / (1.0 + 0.2316419 * np.abs(d))
    poly = k * (A1 + k * (A2 + k * (A3 + k * (A4 + k * A5))))
    p = RSQRT2PI * np.exp(-0.5 * d * d) * poly
    return np.where(d > 0, 1.0 - p, p)


def call(s, k=K, r=R, v=V, t=T):
    """European call price per option (L865-866)."""
    s = np.asarray(s, dtype=np.float64)
    sqrt_t = np.sqrt(t)
    d1 = (np.log(s / k) + (r + 0.5 * v * v) * t) / (v * sqrt_t)
    d2 = d1 - v * sqrt_t
    return s * cnd(d1) - k * np.exp(-r * t) * cnd(d2)


def bs(prices):
    """The B&S DAG: one independent kernel per price vector (Fig. 6)."""
    return [call(s) for s in prices]
