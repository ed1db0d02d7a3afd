"""CPU oracle for the Apophenia repeat-finding hot path (arXiv 2406.18111).

TEST INFRASTRUCTURE ONLY -- not part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2406_18111_b200/``); neither side imports the other.

The arithmetic lives in ``apo_oracle.c`` (plain C, exact integer arithmetic);
this module compiles it with gcc on first use and marshals numpy arrays.

Pipeline (Alg. 2, "FindRepeats"):
  SuffixArray -> LCP -> candidates -> Sort -> greedy non-overlap -> dedup.
Tier 0 = literal definitions (naive sorts, explicit interval list).
Tier 1 = textbook equivalents for larger inputs (prefix-doubling SA with a
library sort, Kasai LCP, ISA+RMQ sub-string compare, marked-array greedy
P:613-619), each pinned against tier 0 in tests/test_oracle_pins.py.

Parity status: every function here is pinned; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .ruler import ruler, ruler_slices  # noqa: F401
from .traces import traces_from_repeats, traces_from_repeats_np  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "apo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

P_U64 = ctypes.POINTER(ctypes.c_uint64)
P_I32 = ctypes.POINTER(ctypes.c_int32)
P_I64 = ctypes.POINTER(ctypes.c_int64)
P_U8 = ctypes.POINTER(ctypes.c_uint8)
I64 = ctypes.c_int64
I32 = ctypes.c_int32


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-pthread", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            sig = {
                "or_sa_naive": (None, [P_U64, I64, P_I32]),
                "or_lcp_naive": (None, [P_U64, I64, P_I32, P_I32]),
                "or_candidates": (I64, [P_I32, P_I32, I64, I32, P_I32, P_I32]),
                "or_sort_candidates_naive": (None, [P_U64, I64, P_I32, P_I32]),
                "or_candidate_ids_naive": (None, [P_U64, I64, P_I32, P_I32, P_I32]),
                "or_greedy_list": (None, [I64, P_I32, P_I32, P_U8]),
                "or_repeats": (I64, [I64, P_I32, P_I32, P_I32, P_U8, I32, P_I32, P_I32, P_I32, P_I32,
                                     P_I32, P_I64]),
                "or_sa_doubling": (None, [P_U64, I64, P_I32]),
                "or_sa_check": (ctypes.c_int, [P_U64, I64, P_I32]),
                "or_lcp_kasai": (None, [P_U64, I64, P_I32, P_I32]),
                "or_sort_and_id_rmq": (None, [P_U64, I64, P_I32, P_I32, I64, P_I32, P_I32, P_I32]),
                "or_sort_and_id_rmq_mt": (None, [P_U64, I64, P_I32, P_I32, I64, P_I32, P_I32, P_I32, I32]),
                "or_greedy_marks": (None, [I64, I64, P_I32, P_I32, P_U8]),
                "or_match_brute": (I64, [P_U64, P_I64, I64, P_U64, P_I64, I64, P_I32, P_I32, P_I32, I64]),
                "or_replay": (I64, [I64, P_I32, P_I32, P_I32, I64, P_I32, I32, I32, I32, I32, I32,
                                    P_I32, P_I32, P_I32, P_I32, P_I32, I64]),
            }
            for name, (res, args) in sig.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            _lib = lib
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _u64(S) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(S, dtype=np.uint64))


# ---------------------------------------------------------------- steps ----

def sa_naive(S) -> np.ndarray:
    S = _u64(S)
    sa = np.empty(len(S), dtype=np.int32)
    if len(S):
        _load().or_sa_naive(_p(S, P_U64), len(S), _p(sa, P_I32))
    return sa


def sa_doubling(S) -> np.ndarray:
    S = _u64(S)
    sa = np.empty(len(S), dtype=np.int32)
    if len(S):
        _load().or_sa_doubling(_p(S, P_U64), len(S), _p(sa, P_I32))
    return sa


def sa_check(S, sa) -> bool:
    S = _u64(S)
    sa = np.ascontiguousarray(sa, dtype=np.int32)
    if len(sa) != len(S):
        return False
    return bool(_load().or_sa_check(_p(S, P_U64), len(S), _p(sa, P_I32)))


def lcp_naive(S, sa) -> np.ndarray:
    S = _u64(S)
    sa = np.ascontiguousarray(sa, dtype=np.int32)
    lcp = np.empty(max(len(S) - 1, 0), dtype=np.int32)
    if len(S) > 1:
        _load().or_lcp_naive(_p(S, P_U64), len(S), _p(sa, P_I32), _p(lcp, P_I32))
    return lcp


def lcp_kasai(S, sa) -> np.ndarray:
    S = _u64(S)
    sa = np.ascontiguousarray(sa, dtype=np.int32)
    lcp = np.empty(max(len(S) - 1, 0), dtype=np.int32)
    if len(S) > 1:
        _load().or_lcp_kasai(_p(S, P_U64), len(S), _p(sa, P_I32), _p(lcp, P_I32))
    return lcp


def candidates(sa, lcp, min_len: int):
    """Alg. 2 candidate generation in emission order -> (lengths, starts)."""
    sa = np.ascontiguousarray(sa, dtype=np.int32)
    lcp = np.ascontiguousarray(lcp, dtype=np.int32)
    n = len(sa)
    cap = max(2 * (n - 1), 1)
    cl = np.empty(cap, dtype=np.int32)
    cs = np.empty(cap, dtype=np.int32)
    m = 0
    if n > 1:
        m = _load().or_candidates(_p(sa, P_I32), _p(lcp, P_I32), n, int(min_len), _p(cl, P_I32), _p(cs, P_I32))
    return cl[:m].copy(), cs[:m].copy()


def sort_and_id_naive(S, cl, cs):
    S = _u64(S)
    cl = np.array(cl, dtype=np.int32)
    cs = np.array(cs, dtype=np.int32)
    cid = np.empty(len(cl), dtype=np.int32)
    if len(cl):
        lib = _load()
        lib.or_sort_candidates_naive(_p(S, P_U64), len(cl), _p(cl, P_I32), _p(cs, P_I32))
        lib.or_candidate_ids_naive(_p(S, P_U64), len(cl), _p(cl, P_I32), _p(cs, P_I32), _p(cid, P_I32))
    return cl, cs, cid


def sort_and_id_rmq(S, sa, lcp, cl, cs):
    S = _u64(S)
    sa = np.ascontiguousarray(sa, dtype=np.int32)
    lcp = np.ascontiguousarray(lcp, dtype=np.int32)
    cl = np.array(cl, dtype=np.int32)
    cs = np.array(cs, dtype=np.int32)
    cid = np.empty(len(cl), dtype=np.int32)
    if len(cl):
        _load().or_sort_and_id_rmq(_p(S, P_U64), len(S), _p(sa, P_I32), _p(lcp, P_I32), len(cl),
                                   _p(cl, P_I32), _p(cs, P_I32), _p(cid, P_I32))
    return cl, cs, cid


def sort_and_id_rmq_mt(S, sa, lcp, cl, cs, threads: int | None = None):
    """sort_and_id_rmq with the same comparator, sorted on `threads` host
    threads (chunk sorts + a merge tree); for ~10^8 candidates."""
    S = _u64(S)
    sa = np.ascontiguousarray(sa, dtype=np.int32)
    lcp = np.ascontiguousarray(lcp, dtype=np.int32)
    cl = np.array(cl, dtype=np.int32)
    cs = np.array(cs, dtype=np.int32)
    cid = np.empty(len(cl), dtype=np.int32)
    t = int(threads or os.cpu_count() or 1)
    if len(cl):
        _load().or_sort_and_id_rmq_mt(_p(S, P_U64), len(S), _p(sa, P_I32), _p(lcp, P_I32), len(cl),
                                      _p(cl, P_I32), _p(cs, P_I32), _p(cid, P_I32), t)
    return cl, cs, cid


def greedy_list(cl, cs) -> np.ndarray:
    cl = np.ascontiguousarray(cl, dtype=np.int32)
    cs = np.ascontiguousarray(cs, dtype=np.int32)
    keep = np.zeros(len(cl), dtype=np.uint8)
    if len(cl):
        _load().or_greedy_list(len(cl), _p(cl, P_I32), _p(cs, P_I32), _p(keep, P_U8))
    return keep


def greedy_marks(n: int, cl, cs) -> np.ndarray:
    cl = np.ascontiguousarray(cl, dtype=np.int32)
    cs = np.ascontiguousarray(cs, dtype=np.int32)
    keep = np.zeros(len(cl), dtype=np.uint8)
    if len(cl):
        _load().or_greedy_marks(n, len(cl), _p(cl, P_I32), _p(cs, P_I32), _p(keep, P_U8))
    return keep


def repeats(cl, cs, cid, keep, min_count: int = 1):
    """Dedup kept candidates -> (repeats[int32 k x 4: start,length,count,first_occ], occ)."""
    cl = np.ascontiguousarray(cl, dtype=np.int32)
    cs = np.ascontiguousarray(cs, dtype=np.int32)
    cid = np.ascontiguousarray(cid, dtype=np.int32)
    keep = np.ascontiguousarray(keep, dtype=np.uint8)
    m = len(cl)
    cap = max(m, 1)
    rs, rl, rc, rf = (np.empty(cap, dtype=np.int32) for _ in range(4))
    occ = np.empty(cap, dtype=np.int32)
    no = np.zeros(1, dtype=np.int64)
    nr = 0
    if m:
        nr = _load().or_repeats(m, _p(cl, P_I32), _p(cs, P_I32), _p(cid, P_I32), _p(keep, P_U8), int(min_count),
                                _p(rs, P_I32), _p(rl, P_I32), _p(rc, P_I32), _p(rf, P_I32),
                                _p(occ, P_I32), _p(no, P_I64))
    rep = np.stack([rs[:nr], rl[:nr], rc[:nr], rf[:nr]], axis=1).astype(np.int32) if nr else \
        np.zeros((0, 4), dtype=np.int32)
    return rep, occ[:int(no[0])].copy()


# ------------------------------------------------------------- pipeline ----

def find_repeats(S, min_len: int, min_count: int = 1, tier: int = 0) -> dict:
    """FindRepeats(S) (Alg. 2) with every intermediate result.

    Returns dict(sa, lcp, cand_len, cand_start, cand_id, keep, repeats, occ):
    candidates in the paper's sort order (length desc, sub-string asc,
    start asc), keep = greedy decision per candidate, repeats rows
    (start, length, count, first_occ)."""
    if min_len < 1:
        raise ValueError("min_len must be >= 1")
    S = _u64(S)
    n = len(S)
    if tier == 0:
        sa = sa_naive(S)
        lcp = lcp_naive(S, sa)
    else:
        sa = sa_doubling(S)
        lcp = lcp_kasai(S, sa)
    cl, cs = candidates(sa, lcp, min_len)
    if tier == 0:
        cl, cs, cid = sort_and_id_naive(S, cl, cs)
        keep = greedy_list(cl, cs)
    else:
        cl, cs, cid = sort_and_id_rmq(S, sa, lcp, cl, cs)
        keep = greedy_marks(n, cl, cs)
    rep, occ = repeats(cl, cs, cid, keep, min_count)
    return dict(sa=sa, lcp=lcp, cand_len=cl, cand_start=cs, cand_id=cid, keep=keep, repeats=rep, occ=occ)


def find_repeats_batch(tok, off, min_len: int, min_count: int = 1, tier: int = 1, windows=None) -> list:
    """Independent windows (reading R16): one find_repeats per
    window, window-local coordinates."""
    off = np.asarray(off, dtype=np.int64)
    W = len(off) - 1
    ws = range(W) if windows is None else windows
    return [find_repeats(tok[off[w]:off[w + 1]], min_len, min_count, tier) for w in ws]


def match_brute(streams, st_off, traces_tok, tr_off, cap: int | None = None):
    """All (stream, end, trace) hits, sorted by (stream, end, trace)."""
    st = _u64(streams)
    st_off = np.ascontiguousarray(st_off, dtype=np.int64)
    tr = _u64(traces_tok) if len(traces_tok) else np.zeros(1, dtype=np.uint64)
    tr_off = np.ascontiguousarray(tr_off, dtype=np.int64)
    ns, nt = len(st_off) - 1, len(tr_off) - 1
    lib = _load()
    if cap is None:
        cap = lib.or_match_brute(_p(st, P_U64), _p(st_off, P_I64), ns, _p(tr, P_U64), _p(tr_off, P_I64), nt,
                                 None, None, None, 0)
    a, b, c = (np.empty(max(cap, 1), dtype=np.int32) for _ in range(3))
    cnt = lib.or_match_brute(_p(st, P_U64), _p(st_off, P_I64), ns, _p(tr, P_U64), _p(tr_off, P_I64), nt,
                             _p(a, P_I32), _p(b, P_I32), _p(c, P_I32), cap)
    k = min(cnt, cap)
    return np.stack([a[:k], b[:k], c[:k]], axis=1), cnt


# REPLAY constants (P:694-713 names the mechanisms, not the values; SPEC's
# declared defaults): count cap 100, decay 0.99 per 100 tasks (Q16:
# round(0.99 * 65536) = 64881), replay bonus x 1.1 (11 / 10).
REPLAY_DEFAULTS = dict(count_cap=100, decay_q16=64881, decay_period=100, bonus_num=11, bonus_den=10)


def replay(hits, tlen, count_cap=100, decay_q16=64881, decay_period=100, bonus_num=11, bonus_den=10):
    """REPLAY selection over MATCH_ALL hits (rows (stream, end, trace) sorted)
    -> int32[r, 5] rows (stream, start, end, trace, first)."""
    hits = np.ascontiguousarray(np.asarray(hits, dtype=np.int32).reshape(-1, 3))
    hs, he, ht = (np.ascontiguousarray(hits[:, k]) for k in range(3))
    tlen = np.ascontiguousarray(tlen, dtype=np.int32)
    nh = len(hits)
    cap = max(nh, 1)
    out = [np.empty(cap, dtype=np.int32) for _ in range(5)]
    n = 0
    if nh:
        n = _load().or_replay(nh, _p(hs, P_I32), _p(he, P_I32), _p(ht, P_I32), len(tlen), _p(tlen, P_I32),
                              int(count_cap), int(decay_q16), int(decay_period), int(bonus_num), int(bonus_den),
                              *[_p(o, P_I32) for o in out], cap)
    return np.stack([o[:n] for o in out], axis=1) if n else np.zeros((0, 5), dtype=np.int32)
