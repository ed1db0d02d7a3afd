"""Pins for the CPU oracle (tests/golden + closed forms + brute force).

Each check is chosen so that a plausible mistake in oracle/apo_oracle.c (a
dropped term, a wrong sign or index, signed token order, a transposed operand,
an off-by-one in the half-open overlap test, a wrong floor) fails one of them.
None of these checks re-types the oracle's own code: SA/LCP/sort are compared
with Python's own sequence ordering on Python ints, the greedy with its
defining property, candidates with the paper's stated properties.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from workloads import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def brute_sa(S):
    L = [int(x) for x in S]                       # Python ints: unsigned 64-bit order
    return sorted(range(len(L)), key=lambda i: L[i:])   # list order: proper prefix first


def brute_lcp(S, sa):
    L = [int(x) for x in S]
    out = []
    for a, b in zip(sa[:-1], sa[1:]):
        k = 0
        while a + k < len(L) and b + k < len(L) and L[a + k] == L[b + k]:
            k += 1
        out.append(k)
    return out


def small_inputs():
    cases = []
    for seed in range(40):
        n = 1 + (seed * 7) % 60
        a = 1 + seed % 5
        cases.append(gen.random_string(seed, n, a))
    for seed in range(6):
        cases.append(gen.high_bit_string(seed, 40, 5))
    for p in (1, 2, 3, 5, 7):
        cases.append(gen.periodic(p, 37, p, 3))
    cases.append(gen.fibonacci_word(55))
    cases.append(gen.c1()[:200])
    return cases


# ------------------------------------------------------------ golden ----

@pytest.mark.parametrize("ex", GOLD["examples"], ids=lambda e: e["text"])
def test_worked_examples(ex):
    S = gen.from_text(ex["text"])
    if "sa" in ex:
        assert oracle.sa_naive(S).tolist() == ex["sa"]
        assert oracle.sa_doubling(S).tolist() == ex["sa"]
    if "lcp" in ex:
        sa = oracle.sa_naive(S)
        assert oracle.lcp_naive(S, sa).tolist() == ex["lcp"]
        assert oracle.lcp_kasai(S, sa).tolist() == ex["lcp"]
    if "candidates_emitted_min1" in ex:
        sa = oracle.sa_naive(S)
        cl, cs = oracle.candidates(sa, oracle.lcp_naive(S, sa), 1)
        assert [[int(a), int(b)] for a, b in zip(cl, cs)] == ex["candidates_emitted_min1"]
        r = oracle.find_repeats(S, 1)
        assert [[int(a), int(b)] for a, b in zip(r["cand_len"], r["cand_start"])] == ex["sorted_candidates_min1"]
    for ml, want in ex.get("repeats", {}).items():
        for tier in (0, 1):
            r = oracle.find_repeats(S, int(ml), tier=tier)
            assert r["repeats"][:, :3].tolist() == want, (ml, tier)
            if "occ" in ex and ml in ex["occ"]:
                assert r["occ"].tolist() == ex["occ"][ml]


def test_coverage_examples():
    # SPEC.md S:126 coverage 8 for aabcbcbaa min 2; S:124 coverage 6 for ababab
    r = oracle.find_repeats(gen.from_text("aabcbcbaa"), 2)
    assert int((r["repeats"][:, 1] * r["repeats"][:, 2]).sum()) == 8
    r = oracle.find_repeats(gen.from_text("ababab"), 1)
    assert int((r["repeats"][:, 1] * r["repeats"][:, 2]).sum()) == 6


def test_ruler_golden():
    g = GOLD["ruler"]
    assert [oracle.ruler(k) for k in g["k"]] == g["values"]
    assert oracle.ruler_slices(0, 4, 1, 4) == [tuple(x) for x in g["B4_C1_slices"]]
    assert oracle.ruler_slices(0, 8, 1, 8) == [tuple(x) for x in g["B8_C1_slices"]]
    assert oracle.ruler_slices(999, 1000, 250, 5000) == [tuple(g["k1000_C250"])]


def test_ruler_closed_forms():
    for j in range(20):
        assert oracle.ruler(1 << j) == j
        assert oracle.ruler((1 << j) * 3) == j
    # R13: B/C not a power of two -> the formula never spans the whole buffer
    lens = {e - b for b, e in oracle.ruler_slices(0, 200_000, 500, 5000)}
    assert max(lens) == 4000 or max(lens) == 5000
    assert all(ln in (500, 1000, 2000, 4000, 5000) for ln in lens)


def test_chunking_golden():
    g = GOLD["chunking"]
    S = gen.random_string(3, g["length"], 1000)
    rep = np.array([[0, g["length"], 2, 0]])
    tok, off = oracle.traces_from_repeats([S], [rep], g["min_len"], g["max_len"])
    assert sorted(np.diff(off).tolist(), reverse=True) == g["pieces"]


def test_matcher_golden():
    g = GOLD["matcher"]
    tr = gen.from_text(g["traces"][0])
    st = gen.from_text(g["stream"])
    hits, cnt = oracle.match_brute(st, [0, len(st)], tr, [0, len(tr)])
    assert hits.tolist() == g["hits"] and cnt == 1


# ------------------------------------------------- SA / LCP brute force ----

def test_sa_lcp_brute_force():
    for S in small_inputs():
        want = brute_sa(S)
        assert oracle.sa_naive(S).tolist() == want
        assert oracle.sa_doubling(S).tolist() == want
        assert oracle.sa_check(S, np.array(want, dtype=np.int32))
        wl = brute_lcp(S, want)
        assert oracle.lcp_naive(S, np.array(want)).tolist() == wl
        assert oracle.lcp_kasai(S, np.array(want)).tolist() == wl


def test_sa_check_rejects():
    S = gen.random_string(5, 50, 3)
    sa = oracle.sa_naive(S)
    for i in range(0, 49, 7):
        bad = sa.copy()
        bad[i], bad[i + 1] = bad[i + 1], bad[i]
        assert not oracle.sa_check(S, bad)
    dup = sa.copy(); dup[3] = dup[4]
    assert not oracle.sa_check(S, dup)


def test_unsigned_token_order():
    # signed order would put 2^63 before 0
    S = np.array([1 << 63, 0, 1 << 63, 0], dtype=np.uint64)
    assert oracle.sa_naive(S).tolist() == [3, 1, 2, 0]


def test_empty_and_tiny():
    assert oracle.sa_naive(np.zeros(0, np.uint64)).tolist() == []
    r = oracle.find_repeats(np.zeros(0, np.uint64), 1)
    assert len(r["repeats"]) == 0
    r = oracle.find_repeats(np.array([7], np.uint64), 1)
    assert r["sa"].tolist() == [0] and len(r["lcp"]) == 0 and len(r["repeats"]) == 0
    with pytest.raises(ValueError):
        oracle.find_repeats(np.array([1, 1], np.uint64), 0)


# ------------------------------------------------------- candidates ----

def test_candidate_properties():
    """Alg. 2: per adjacent SA pair, two equal, disjoint occurrences;
    disjoint branch keeps p; overlap branch = largest multiple of the period d
    whose two abutting copies fit in the overlap (R6)."""
    for S in small_inputs():
        L = [int(x) for x in S]
        n = len(L)
        if n < 2:
            continue
        sa = oracle.sa_naive(S)
        lcp = oracle.lcp_naive(S, sa)
        cl, cs = oracle.candidates(sa, lcp, 1)
        k = 0
        for i in range(n - 1):
            s1, s2, p = int(sa[i]), int(sa[i + 1]), int(lcp[i])
            d = abs(s2 - s1)
            if d >= p:
                want = p
            else:
                # largest multiple of d with two abutting copies inside [m, m+p+d)
                want = max(x for x in range(0, p + d + 1, d) if 2 * x <= p + d)
            if want < 1:
                continue
            (l1, a), (l2, b) = (int(cl[k]), int(cs[k])), (int(cl[k + 1]), int(cs[k + 1]))
            k += 2
            assert l1 == l2 == want
            assert L[a:a + l1] == L[b:b + l2]                   # same sub-string
            assert a + l1 <= b or b + l2 <= a                   # disjoint (half-open)
            if d < p:
                assert b == a + l1 and a == min(s1, s2)         # abutting chunks at m, m+l
        assert k == len(cl)                                     # exactly 2 per kept pair


def test_min_len_filter_equivalence():
    """R7: filtering candidates before the sort gives the same result as
    filtering repeats after (shorter candidates sort after longer ones)."""
    for seed in range(30):
        S = gen.random_string(100 + seed, 80, 2 + seed % 3)
        full = oracle.find_repeats(S, 1)
        for ml in (2, 3, 4):
            r = oracle.find_repeats(S, ml)
            keep_rows = [row for row in full["repeats"].tolist() if row[1] >= ml]
            assert [row[:3] for row in r["repeats"].tolist()] == [row[:3] for row in keep_rows]


# ---------------------------------------------------- sort / IDs ----

def test_sort_order_and_ids():
    for S in small_inputs():
        L = [int(x) for x in S]
        sa = oracle.sa_naive(S)
        cl, cs = oracle.candidates(sa, oracle.lcp_naive(S, sa), 1)
        want = sorted(zip(cl.tolist(), cs.tolist()), key=lambda c: (-c[0], L[c[1]:c[1] + c[0]], c[1]))
        for tier in (0, 1):
            if tier == 0:
                sl, ss, sid = oracle.sort_and_id_naive(S, cl, cs)
            else:
                sl, ss, sid = oracle.sort_and_id_rmq(S, sa, oracle.lcp_naive(S, sa), cl, cs)
            assert list(zip(sl.tolist(), ss.tolist())) == want
            # IDs: dense, non-decreasing, equal iff same (length, content)
            keys = [(l_, tuple(L[s:s + l_])) for l_, s in want]
            for i in range(len(keys)):
                if i:
                    assert sid[i] == sid[i - 1] + (keys[i] != keys[i - 1])
                else:
                    assert sid[0] == 0


# ------------------------------------------------------------ greedy ----

def check_greedy_property(cl, cs, keep):
    """Defining property of the greedy loop: candidate i is kept
    iff its interval is disjoint from every EARLIER kept interval."""
    kept = []
    for i in range(len(cl)):
        a, b = int(cs[i]), int(cs[i]) + int(cl[i])
        hits = any(a < e and s < b for s, e in kept)
        assert bool(keep[i]) == (not hits), i
        if keep[i]:
            kept.append((a, b))
    return kept


def test_greedy_property_and_marks_equivalence():
    for S in small_inputs() + [gen.c1()]:
        r = oracle.find_repeats(S, 1)
        kept = check_greedy_property(r["cand_len"], r["cand_start"], r["keep"])
        # R9: the O(1) marked-array check gives the same decisions
        assert np.array_equal(oracle.greedy_marks(len(S), r["cand_len"], r["cand_start"]), r["keep"])
        # invariants: disjoint, coverage <= n
        cov = np.zeros(len(S), dtype=np.int32)
        for a, b in kept:
            cov[a:b] += 1
        assert cov.max(initial=0) <= 1


def test_periodic_closed_form():
    """S = u^k, u primitive, k even, min_len <= |u|: exactly one repeat u^(k/2)
    at {0, n/2} covering the whole string (SURVEY.md §8c pins)."""
    checked = 0
    for seed in range(200):
        rng = gen.Rng(seed)
        p = 1 + rng.below(6)
        u = [int(x) for x in gen.H_np(9, rng.below_np(3, p))]
        # primitive: not a power of a shorter word
        if any(p % q == 0 and u == u[:q] * (p // q) for q in range(1, p)):
            continue
        k = 2 * (1 + rng.below(5))
        S = np.array(u * k, dtype=np.uint64)
        r = oracle.find_repeats(S, 1 + rng.below(p))
        n = len(S)
        assert r["repeats"][:, :3].tolist() == [[0, n // 2, 2]], (u, k)
        assert r["occ"].tolist() == [0, n // 2]
        checked += 1
    assert checked > 100


def test_longest_repeat_valid_form():
    """R12: the first candidate in sort order is always kept, so the longest
    CANDIDATE (>= the classical longest repeat whenever its SA-adjacent
    witnesses are disjoint) is found."""
    for S in small_inputs():
        r = oracle.find_repeats(S, 1)
        if len(r["cand_len"]):
            assert r["keep"][0] == 1
            assert r["repeats"][0, 1] == r["cand_len"].max()
        # classical longest repeat = max LCP; when its witness pair is disjoint it is found
        lcp, sa = r["lcp"], r["sa"]
        if len(lcp) and lcp.max() > 0:
            i = int(np.argmax(lcp))
            if abs(int(sa[i]) - int(sa[i + 1])) >= lcp[i]:
                assert r["repeats"][0, 1] == lcp.max()


def test_each_kept_substring_repeats_disjointly():
    """Every reported repeat (even with count 1, R10) occurs at least twice,
    disjointly, in S."""
    for S in small_inputs():
        L = [int(x) for x in S]
        r = oracle.find_repeats(S, 1)
        for st, ln, cnt, _ in r["repeats"].tolist():
            t = L[st:st + ln]
            occ = [i for i in range(len(L) - ln + 1) if L[i:i + ln] == t]
            assert any(abs(a - b) >= ln for a, b in itertools.combinations(occ, 2))


def test_dedup_counts():
    for S in small_inputs():
        r = oracle.find_repeats(S, 1)
        assert int(r["repeats"][:, 2].sum()) == int(r["keep"].sum()) == len(r["occ"])
        L = [int(x) for x in S]
        for st, ln, cnt, first in r["repeats"].tolist():
            occ = r["occ"][first:first + cnt].tolist()
            assert occ == sorted(occ) and occ[0] == st
            assert all(L[o:o + ln] == L[st:st + ln] for o in occ)


def test_min_count_filter():
    S = gen.from_text("aabcbcbaa")
    r = oracle.find_repeats(S, 1, min_count=2)
    assert r["repeats"][:, :3].tolist() == [[0, 2, 2], [2, 2, 2]]
    assert r["occ"].tolist() == [0, 7, 2, 4]


# ---------------------------------------------------- tier-0 vs tier-1 ----

def tier_sweep_inputs():
    out = []
    for seed in range(150):
        rng = gen.Rng(1000 + seed)
        n = 1 + rng.below(300)
        a = 1 + rng.below(16)
        out.append(gen.random_string(seed, n, a))
    for seed in range(30):
        out.append(gen.periodic(seed, 200 + seed, 1 + seed % 13, 1 + seed % 4, noise=0.03))
    out.append(gen.fibonacci_word(400))
    out.append(gen.c1())
    return out


def test_tier0_vs_tier1_sweep():
    for S in tier_sweep_inputs():
        for ml in (1, 3):
            a = oracle.find_repeats(S, ml, tier=0)
            b = oracle.find_repeats(S, ml, tier=1)
            for k in ("sa", "lcp", "cand_len", "cand_start", "cand_id", "keep", "repeats", "occ"):
                assert np.array_equal(a[k], b[k]), k


def test_batch_is_per_window():
    tok, off, _, _ = gen.c4(seed=9, windows=3, window=512, templates=3)
    res = oracle.find_repeats_batch(tok, off, 5)
    for w in range(3):
        single = oracle.find_repeats(tok[off[w]:off[w + 1]], 5, tier=1)
        assert np.array_equal(res[w]["repeats"], single["repeats"])


# ----------------------------------------------------------- matcher ----

def test_match_brute_vs_python():
    for seed in range(10):
        rng = gen.Rng(seed)
        streams = [gen.random_string(seed * 10 + j, 30 + rng.below(30), 3) for j in range(3)]
        traces = sorted({tuple(int(x) for x in gen.random_string(seed * 10 + 5 + j, 1 + rng.below(4), 3))
                         for j in range(5)}, key=lambda t: (-len(t), t))
        st = np.concatenate(streams)
        so = np.cumsum([0] + [len(s) for s in streams])
        tr = np.array([x for t in traces for x in t], dtype=np.uint64)
        to = np.cumsum([0] + [len(t) for t in traces])
        hits, cnt = oracle.match_brute(st, so, tr, to)
        want = []
        for q, s in enumerate(streams):
            L = [int(x) for x in s]
            for e in range(len(L)):
                for t, tt in enumerate(traces):
                    if len(tt) <= e + 1 and tuple(L[e - len(tt) + 1:e + 1]) == tt:
                        want.append([q, e, t])
        assert hits.tolist() == want and cnt == len(want)


def test_traces_order_and_dedup():
    S = gen.from_text("abcabcxyxy")
    reps = [np.array([[0, 3, 2, 0], [6, 2, 2, 2]]), np.array([[3, 3, 1, 0]])]
    tok, off = oracle.traces_from_repeats([S, S], reps, 1)
    ts = [tuple(tok[off[i]:off[i + 1]].tolist()) for i in range(len(off) - 1)]
    assert ts == [tuple(b"abc"), tuple(b"xy")]


# ------------------------------------- tier-1 pinned at full window size ----

def test_tier0_vs_tier1_full_c4_windows():
    """Tier-1 (the oracle every full-size GPU comparison uses) equals tier-0
    (the literal Alg. 2) on 8 full 16,384-op C4 windows."""
    tok, off, _, _ = gen.c4(seed=4, windows=8 * 64, with_streams=False)
    for w in range(0, 8 * 64, 64 + 1):
        S = tok[off[w]:off[w + 1]]
        a = oracle.find_repeats(S, 25, tier=0)
        b = oracle.find_repeats(S, 25, tier=1)
        for k in ("sa", "lcp", "cand_len", "cand_start", "cand_id", "keep", "repeats", "occ"):
            assert np.array_equal(a[k], b[k]), (w, k)


def test_tier0_vs_tier1_c2_full():
    """... and on the full 65,536-op C2 window (Fig. 1b aliasing, maxLCP
    64,768: the deepest doubling among the single windows that tier 0 can
    still finish, ~15 s)."""
    S = gen.c2()
    a = oracle.find_repeats(S, 25, tier=0)
    b = oracle.find_repeats(S, 25, tier=1)
    for k in ("sa", "lcp", "cand_len", "cand_start", "cand_id", "keep", "repeats", "occ"):
        assert np.array_equal(a[k], b[k]), k


def test_sort_and_id_threads_equal_single():
    """The multi-threaded tier-1 sort (same comparator; chunk sorts + merge
    tree) gives the single-thread result, for any thread count."""
    cases = [gen.c1(), gen.c2()[:30000], gen.random_string(3, 5000, 3), gen.periodic(4, 7000, 31, 3, 0.01)]
    for S in cases:
        sa = oracle.sa_doubling(S)
        lcp = oracle.lcp_kasai(S, sa)
        for ml in (1, 25):
            cl, cs = oracle.candidates(sa, lcp, ml)
            want = oracle.sort_and_id_rmq(S, sa, lcp, cl, cs)
            for t in (1, 2, 5, 16):
                got = oracle.sort_and_id_rmq_mt(S, sa, lcp, cl, cs, t)
                assert all(np.array_equal(x, y) for x, y in zip(want, got)), t


def test_traces_numpy_equals_python():
    """The numpy trace-set builder (used at full C4 size) equals the Python
    tuple version (IngestCandidates; R15 chunking) for max_len 0/7/40."""
    tok, off, _, _ = gen.c4(seed=9, windows=12, window=2048, templates=4, with_streams=False)
    srcs = [tok[off[w]:off[w + 1]] for w in range(12)]
    reps = [oracle.find_repeats(s, 5, tier=1)["repeats"] for s in srcs]
    for ml in (0, 7, 40):
        a = oracle.traces_from_repeats(srcs, reps, 5, ml)
        b = oracle.traces_from_repeats_np(srcs, reps, 5, ml)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), ml


# ------------------------------------------------------------- REPLAY ----

def _replay_case(c):
    if "stream" in c:
        S = np.array(c["stream"], dtype=np.uint64)
    else:  # "decay flips the choice"
        S = np.array(list(range(1, 9)) + list(range(1000, 1300)) + [99, 5, 6, 7, 8] + list(range(1, 9)),
                     dtype=np.uint64)
    tr = [np.array(t, dtype=np.uint64) for t in c["traces"]]
    tt = np.concatenate(tr)
    to = np.cumsum([0] + [len(t) for t in tr]).astype(np.int64)
    hits, _ = oracle.match_brute(S, np.array([0, len(S)], np.int64), tt, to)
    return S, hits, [len(t) for t in tr]


def test_replay_golden():
    """Hand-derived REPLAY decisions (tests/golden/replay_examples.json)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "replay_examples.json")))
    for c in g["cases"]:
        S, hits, tlen = _replay_case(c)
        got = oracle.replay(hits, tlen, **c["params"]).tolist()
        assert got == c["replays"], c["name"]
        if "replays_no_decay" in c:
            p = dict(c["params"], decay_q16=65536)
            assert oracle.replay(hits, tlen, **p).tolist() == c["replays_no_decay"], c["name"]


def test_replay_periodic_closed_form():
    """S = u^k with the single trace u: every period is replayed back to back,
    recorded the first time."""
    for p, k in ((1, 9), (5, 7), (37, 12)):
        u = gen.random_string(p, p, 1000)
        S = np.tile(u, k)
        hits, _ = oracle.match_brute(S, np.array([0, len(S)], np.int64), u, np.array([0, p], np.int64))
        got = oracle.replay(hits, [p]).tolist()
        assert got == [[0, i * p, (i + 1) * p - 1, 0, 1 if i == 0 else 0] for i in range(k)]


def _replay_inputs():
    out = []
    for seed in range(40):
        rng = gen.Rng(500 + seed)
        nst = 1 + rng.below(3)
        streams = [gen.periodic(seed * 7 + j, 40 + rng.below(200), 1 + rng.below(9), 2 + rng.below(3), noise=0.05)
                   for j in range(nst)]
        traces = {tuple(int(x) for x in s[a:a + 1 + rng.below(12)])
                  for s in streams for a in [rng.below(max(len(s) - 12, 1)) for _ in range(6)]}
        traces = sorted(traces, key=lambda t: (-len(t), t))
        st = np.concatenate(streams)
        so = np.cumsum([0] + [len(s) for s in streams]).astype(np.int64)
        tt = np.array([x for t in traces for x in t], dtype=np.uint64)
        to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
        hits, _ = oracle.match_brute(st, so, tt, to)
        out.append((streams, traces, hits))
    return out


def test_replay_special_case_longest_first():
    """count_cap = 1, no decay, no bonus: every score is the trace length, so
    REPLAY reduces to: at each end, the longest completion starting at or
    after the first op not yet replayed."""
    for streams, traces, hits in _replay_inputs():
        got = oracle.replay(hits, [len(t) for t in traces], count_cap=1, decay_q16=65536, bonus_num=1,
                            bonus_den=1).tolist()
        want = []
        for q in range(len(streams)):
            frontier, best_at = 0, {}
            for s, e, t in hits[hits[:, 0] == q].tolist():
                best_at.setdefault(e, []).append(t)
            seen = set()
            for e in sorted(best_at):
                ok = [t for t in best_at[e] if e - len(traces[t]) + 1 >= frontier]
                if ok:
                    t = min(ok, key=lambda t: (-len(traces[t]), t))
                    want.append([q, e - len(traces[t]) + 1, e, t, 0 if t in seen else 1])
                    seen.add(t)
                    frontier = e + 1
        assert got == want


def test_replay_invariants():
    """Default parameters: replays are MATCH_ALL hits, disjoint and in order;
    no valid completion lies strictly between two replays (a completion is
    replayed at the first end where one exists); `first` marks the first
    replay of each trace in its stream."""
    for streams, traces, hits in _replay_inputs():
        got = oracle.replay(hits, [len(t) for t in traces])
        hs = {tuple(h) for h in hits.tolist()}
        for q in range(len(streams)):
            rq = got[got[:, 0] == q]
            prev_end, seen = -1, set()
            for _, s, e, t, first in rq.tolist():
                assert (q, e, t) in hs and s == e - len(traces[t]) + 1
                assert s > prev_end
                assert first == (0 if t in seen else 1)
                seen.add(t)
                hq = hits[(hits[:, 0] == q) & (hits[:, 1] < e) & (hits[:, 1] > prev_end)]
                for _, e2, t2 in hq.tolist():
                    assert e2 - len(traces[t2]) + 1 <= prev_end   # it was not valid
                prev_end = e
