"""IngestCandidates (Alg. 1) for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Turns FindRepeats results into the candidate trace set the matcher uses:
  * each repeat's content is the source tokens S[start : start + length];
  * "recorded traces are broken into pieces of a given maximum size"
    (reading R15): consecutive max_len pieces from the start,
    the tail kept iff its length >= min_len; max_len = 0 means unbounded;
  * identical contents are merged (a trie holds each string once);
  * trace ids are ranks in (length desc, content lexicographic asc) order
    (R1: unsigned 64-bit token order).
"""
from __future__ import annotations

import numpy as np


def traces_from_repeats(sources, repeat_lists, min_len: int, max_len: int = 0):
    """sources: list of uint64 arrays (one per window); repeat_lists: list of
    (k x 4) int arrays (start, length, count, first_occ) per window.
    Returns (trace_tokens uint64[], trace_off int64[T+1]) in id order."""
    seen = set()
    for S, reps in zip(sources, repeat_lists):
        S = np.asarray(S, dtype=np.uint64)
        for row in np.asarray(reps).reshape(-1, 4):
            start, length = int(row[0]), int(row[1])
            content = S[start:start + length]
            if max_len and max_len > 0:
                pieces = [content[i:i + max_len] for i in range(0, length, max_len)]
                pieces = [p for p in pieces if len(p) == max_len or len(p) >= min_len]
            else:
                pieces = [content]
            for p in pieces:
                seen.add(tuple(int(x) for x in p))
    order = sorted(seen, key=lambda t: (-len(t), t))   # Python ints: unsigned order
    off = np.zeros(len(order) + 1, dtype=np.int64)
    for i, t in enumerate(order):
        off[i + 1] = off[i] + len(t)
    tok = np.array([x for t in order for x in t], dtype=np.uint64)
    return tok, off
