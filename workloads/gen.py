"""Seeded synthetic op-hash streams shaped like the paper's workloads.

TEST / BENCH INFRASTRUCTURE.  This module is the ONLY code shared by the CPU
oracle side (``oracle/``, ``tests/``) and the CUDA product side (``bench.py``,
GPU tests).  It contains no step of the paper's method: it only draws seeded
random numbers and assembles token streams.

Every token is a 64-bit "op hash" (§4.1: Apophenia hashes
each task and its region arguments into one token).  Hashes are produced by
splitmix64 so token VALUE order is uniform and unrelated to the generating
"kind" index (reading R1: tokens compare as unsigned 64-bit ints).

Stream shapes (DESIGN.md §"Input recipe"):
  C1  n=1,024: period-37 loop body + 10 % noise ops                  (min_len 5)
  C2  n=65,536: Jacobi inner loop J(x1,x2)||J(x2,x1) (Fig. 1b aliasing,
      P:143-154) x10 + 32-op tail -> outer period 512    (min_len 25)
  C3  n=1,048,576: S3D/HTR-like phases, periods log-uniform in [100,5000],
      irregular 1-3-op insertions (p=0.1), periodic 24-op hand-offs  (min_len 25)
  C4  4,096 windows x 16,384 ops from 64 loop templates + the next 16,384 ops
      of each as the matching stream                                  (min_len 25)
  C5  n=67,108,864: 4-token alphabet, 64-op prologue, 1,000-op body repeated
                                                                      (min_len 25)
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def mix(z: int) -> int:
    """splitmix64 finaliser on a Python int."""
    z &= M64
    z = ((z ^ (z >> 30)) * _C1) & M64
    z = ((z ^ (z >> 27)) * _C2) & M64
    return z ^ (z >> 31)


def mix_np(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
        z = z ^ (z >> np.uint64(31))
    return z


class Rng:
    """splitmix64 stream."""

    def __init__(self, seed: int):
        self.s = mix(seed * 0x2545F4914F6CDD1D + 1)

    def next(self) -> int:
        self.s = (self.s + GOLDEN) & M64
        return mix(self.s)

    def below(self, k: int) -> int:
        return self.next() % k

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)

    def fresh(self, k: int) -> np.ndarray:
        """k fresh 64-bit values (the next k draws of the stream)."""
        if k <= 0:
            return np.zeros(0, dtype=np.uint64)
        with np.errstate(over="ignore"):
            st = np.uint64(self.s) + np.uint64(GOLDEN) * np.arange(1, k + 1, dtype=np.uint64)
        self.s = (self.s + GOLDEN * k) & M64
        return mix_np(st)

    def below_np(self, k: int, count: int) -> np.ndarray:
        return self.fresh(count) % np.uint64(k)


def H(tag: int, *ks: int) -> int:
    """Token hash of a (kind, args...) tuple, chained splitmix64."""
    h = mix(tag + GOLDEN)
    for k in ks:
        h = mix((h ^ (k & M64)) + GOLDEN)
    return h


def H_np(tag: int, ks: np.ndarray) -> np.ndarray:
    h0 = np.uint64(mix(tag + GOLDEN))
    with np.errstate(over="ignore"):
        return mix_np((h0 ^ np.asarray(ks, dtype=np.uint64)) + np.uint64(GOLDEN))


def body(rng: Rng, length: int, vocab: int, tag: int) -> np.ndarray:
    """`length` tokens, each H(tag, below(vocab))."""
    return H_np(tag, rng.below_np(vocab, length))


# --------------------------------------------------------------------------
# The five BASELINE.json configs
# --------------------------------------------------------------------------

def c1(seed: int = 1, n: int = 1024) -> np.ndarray:
    """Period-37 loop over a 24-kind vocabulary + 10 % noise ops."""
    rng = Rng(seed)
    b = body(rng, 37, 24, 1)
    out = np.empty(n, dtype=np.uint64)
    pos = 0
    for i in range(n):
        if rng.uniform() < 0.10:
            if rng.below(2) == 0:
                out[i] = H(2, rng.below(8))
            else:
                out[i] = rng.next()
        else:
            out[i] = b[pos]
            pos = (pos + 1) % 37
    return out


def jacobi(x: int, y: int, stmts: int = 8) -> np.ndarray:
    """One solver iteration: `stmts` statements x 3 tasks, the loop-carried
    region alternating between x and y (Fig. 1b: DOT(R,x1,t1) SUB DIV(..,x2))."""
    toks = []
    for s in range(stmts):
        toks.append(H(20, s, 0, x))   # reads the loop-carried region
        toks.append(H(20, s, 1))      # temporary
        toks.append(H(20, s, 2, y))   # writes the other region
    return np.array(toks, dtype=np.uint64)


def c2(seed: int = 2, n: int = 65536) -> np.ndarray:
    """256-op unique prologue, then {J(x1,x2)||J(x2,x1) x 10, 32-op tail}."""
    rng = Rng(seed)
    inner = np.concatenate([jacobi(1, 2), jacobi(2, 1)])   # period 48
    tail = body(rng, 32, 64, 21)
    outer = np.concatenate([np.tile(inner, 10), tail])      # period 512
    pro = rng.fresh(256)
    reps = (n - 256) // len(outer) + 1
    return np.concatenate([pro, np.tile(outer, reps)])[:n].copy()


def _irregular(rng: Rng, kinds_tag: int = 5) -> np.ndarray:
    k = 1 + rng.below(3)
    out = np.empty(k, dtype=np.uint64)
    for j in range(k):
        out[j] = H(kinds_tag, rng.below(16)) if rng.uniform() < 0.8 else rng.next()
    return out


def c3(seed: int = 3, n: int = 1 << 20) -> np.ndarray:
    """S3D/HTR-like: phases of main loops with periods log-uniform in
    [100, 5000], irregular 1-3-op blocks (p = 0.1 per iteration), and a 24-op
    hand-off after iterations 0-9 and every 10th thereafter."""
    rng = Rng(seed)
    parts = []
    total = 0
    phase = 0
    while total < n:
        P = int(round(math.exp(rng.uniform() * (math.log(5000) - math.log(100)) + math.log(100))))
        b = body(rng, P, 2000, 100 + phase)
        hand = body(rng, 24, 64, 200 + phase)
        iters = max(8, (20000 + rng.below(180000)) // P)
        for it in range(iters):
            if rng.uniform() < 0.1:
                off = rng.below(P)
                ir = _irregular(rng)
                parts.append(b[:off]); parts.append(ir); parts.append(b[off:])
                total += len(ir)
            else:
                parts.append(b)
            total += P
            if it < 10 or it % 10 == 0:
                parts.append(hand)
                total += 24
            if total >= n:
                break
        phase += 1
    return np.concatenate(parts)[:n].copy()


C4_WINDOW = 16384
C4_WINDOWS = 4096
C4_TEMPLATES = 64


def c4_template(seed: int, t: int, length: int) -> np.ndarray:
    """One loop template stream: a short prologue then an outer loop
    {inner^reps, tail} with irregular insertions."""
    rng = Rng(seed * 1000003 + t)
    P1 = int(round(math.exp(rng.uniform() * (math.log(400) - math.log(10)) + math.log(10))))
    inner = body(rng, P1, 2000, 300 + t)
    reps = max(1, min(2000 // P1, 1 + rng.below(8)))
    tail = body(rng, rng.below(65), 64, 400 + t)
    q = 0.05 + 0.15 * rng.uniform()
    parts = [rng.fresh(rng.below(200))]
    total = len(parts[0])
    outer = np.concatenate([np.tile(inner, reps), tail])
    while total < length:
        if rng.uniform() < q:
            off = rng.below(len(outer))
            ir = _irregular(rng)
            parts.append(outer[:off]); parts.append(ir); parts.append(outer[off:])
            total += len(ir)
        else:
            parts.append(outer)
        total += len(outer)
    return np.concatenate(parts)[:length]


def c4(seed: int = 4, windows: int = C4_WINDOWS, window: int = C4_WINDOW,
       templates: int = C4_TEMPLATES, with_streams: bool = True):
    """Batch of `windows` independent windows of `window` ops.  Window w is
    block (w // templates) of template (w % templates); its matching stream is
    the next `window` ops of the same template.  Returns (tokens[W*window],
    offsets[W+1], streams[W*window] or None, stream_offsets or None)."""
    blocks = (windows + templates - 1) // templates
    tok = np.empty(windows * window, dtype=np.uint64)
    st = np.empty(windows * window, dtype=np.uint64) if with_streams else None
    for t in range(min(templates, windows)):
        s = c4_template(seed, t, (blocks + 1) * window)
        for blk in range(blocks):
            w = blk * templates + t
            if w >= windows:
                break
            tok[w * window:(w + 1) * window] = s[blk * window:(blk + 1) * window]
            if with_streams:
                st[w * window:(w + 1) * window] = s[(blk + 1) * window:(blk + 2) * window]
    off = np.arange(windows + 1, dtype=np.int64) * window
    return tok, off, st, (off.copy() if with_streams else None)


def c5(seed: int = 5, n: int = 1 << 26, period: int = 1000, prologue: int = 64) -> np.ndarray:
    """Highly periodic 4-token alphabet stream: 64 random ops, then a
    1,000-op random body repeated (stresses doubling depth and long LCPs)."""
    rng = Rng(seed)
    alpha = np.array([H(6, k) for k in range(4)], dtype=np.uint64)
    pro = alpha[rng.below_np(4, prologue).astype(np.int64)]
    b = alpha[rng.below_np(4, period).astype(np.int64)]
    reps = (n - prologue) // period + 1
    return np.concatenate([pro, np.tile(b, reps)])[:n].copy()


CONFIGS = {
    "C1": dict(gen=c1, min_len=5),
    "C2": dict(gen=c2, min_len=25),
    "C3": dict(gen=c3, min_len=25),
    "C4": dict(gen=c4, min_len=25),
    "C5": dict(gen=c5, min_len=25),
}


# --------------------------------------------------------------------------
# Small families for sweeps (random, periodic, Fibonacci, raw small ints)
# --------------------------------------------------------------------------

def random_string(seed: int, n: int, alphabet: int, hashed: bool = True) -> np.ndarray:
    rng = Rng(seed)
    k = rng.below_np(alphabet, n)
    return H_np(7, k) if hashed else k.astype(np.uint64)


def periodic(seed: int, n: int, period: int, alphabet: int, noise: float = 0.0) -> np.ndarray:
    rng = Rng(seed)
    base = H_np(8, rng.below_np(alphabet, period))
    reps = n // period + 1
    s = np.tile(base, reps)[:n].copy()
    if noise > 0:
        for i in range(n):
            if rng.uniform() < noise:
                s[i] = rng.next()
    return s


def fibonacci_word(n: int) -> np.ndarray:
    a, b = "a", "ab"
    while len(b) < n:
        a, b = b, b + a
    return np.frombuffer(b[:n].encode(), dtype=np.uint8).astype(np.uint64)


def from_text(s: str) -> np.ndarray:
    """Raw character codes as tokens (so 'a' < 'b' < 'c' in token order)."""
    return np.frombuffer(s.encode(), dtype=np.uint8).astype(np.uint64)


def high_bit_string(seed: int, n: int, alphabet: int) -> np.ndarray:
    """Tokens straddling 2^63 so signed and unsigned order disagree."""
    rng = Rng(seed)
    vals = np.array([(1 << 63) - 2, (1 << 63) - 1, 1 << 63, (1 << 63) + 1, M64, 0, 1, 2][:alphabet],
                    dtype=np.uint64)
    return vals[rng.below_np(len(vals), n).astype(np.int64)]
