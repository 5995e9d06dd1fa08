"""Finite-size bookkeeping that fixes the output length m (host utilities).

Not on the hot path: these turn the security parameters into the m that
pa_create takes.  PAPER.md Sec. 2.2:

    Delta(n) = (2 dim H_x + 3) sqrt(log2(2 / eps_bar) / n) + (2 / n) log2(1 / eps_PA)   Eq. (3)
    k        = beta I(x:y) - S(y:E) - Delta(n)                                          Eq. (2)
    l        = floor(n k)
    collision probability of the Toeplitz family = n 2^(-m+1)
"""
from __future__ import annotations

import math


def delta(n: int, dim_hx: float, eps_bar: float, eps_pa: float) -> float:
    """Eq. (3): the finite-size correction Delta(n)."""
    if n <= 0 or not (0 < eps_bar < 1) or not (0 < eps_pa < 1) or dim_hx <= 0:
        raise ValueError(f"need n > 0, dim_hx > 0, 0 < eps < 1 (n={n}, dim_hx={dim_hx}, "
                         f"eps_bar={eps_bar}, eps_pa={eps_pa})")
    return (2 * dim_hx + 3) * math.sqrt(math.log2(2.0 / eps_bar) / n) + (2.0 / n) * math.log2(1.0 / eps_pa)


def key_rate(beta: float, i_xy: float, s_ye: float, n: int, dim_hx: float, eps_bar: float,
             eps_pa: float) -> float:
    """Eq. (2): secret key rate per corrected-key bit (may be <= 0: no key)."""
    if not (0 < beta <= 1):
        raise ValueError(f"reconciliation efficiency beta={beta} must be in (0, 1]")
    return beta * i_xy - s_ye - delta(n, dim_hx, eps_bar, eps_pa)


def final_length(n: int, k: float) -> int:
    """l = floor(n k), 0 when the rate is not positive."""
    return max(0, math.floor(n * k)) if k > 0 else 0


def collision_log2(n: int, m: int) -> float:
    """log2 of the Toeplitz-family collision probability n 2^(-m+1)."""
    if n <= 0 or m <= 0:
        raise ValueError("n and m must be positive")
    return math.log2(n) - m + 1
