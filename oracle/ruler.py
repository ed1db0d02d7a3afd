"""Ruler-function buffer sampling (§4.4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"The ruler function counts the number of times a number can be evenly divided
by two.  Applying it to the sequence 1, 2, 3, 4, ... yields 0, 1, 0, 2 ...
Raising the sequence to the power two yields 1, 2, 1, 4, which we can
interpret as subsets of the buffer to analyze"; "we use the
exponentiated ruler function as the multiples of a larger constant (such as
250)".

Reading R13: the history is a ring over the last B tokens; at a
global op count k with k % C == 0 the analysed slice is the last
min(2^ruler(k/C) * C, B) tokens, [k - len, k), in absolute coordinates.
"""
from __future__ import annotations


def ruler(k: int) -> int:
    """2-adic valuation of k >= 1 (by repeated division, the paper's words)."""
    if k < 1:
        raise ValueError("ruler(k) needs k >= 1")
    r = 0
    while k % 2 == 0:
        k //= 2
        r += 1
    return r


def ruler_slices(k_begin: int, k_end: int, C: int, B: int) -> list[tuple[int, int]]:
    """Slices emitted while the global op count goes from k_begin to k_end
    (i.e. after ingesting tokens k_begin+1 .. k_end), in order."""
    out = []
    for k in range(k_begin + 1, k_end + 1):
        if k % C == 0:
            ln = min((1 << ruler(k // C)) * C, B)
            out.append((k - ln, k))
    return out
