"""GPU parity for the trace set (IngestCandidates) and MATCH_ALL matching
against the CPU oracle (oracle/traces.py, or_match_brute): bit-exact."""
import numpy as np
import pytest
import torch

import oracle
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_18111_b200 import build
    build.build()
    from paper_2406_18111_b200 import Context
    return Context(0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64)).cuda()


def trace_list(tok, off):
    return [tuple(int(x) for x in tok[off[i]:off[i + 1]]) for i in range(len(off) - 1)]


def small_batch(windows=12, window=1500, seed=21):
    tok, off, st, so = gen.c4(seed=seed, windows=windows, window=window, templates=6)
    return tok, off, st, so


@pytest.mark.parametrize("max_len", [0, 40, 7])
def test_trie_from_repeats(ctx, max_len):
    tok, off, _, _ = small_batch()
    min_len = 5
    rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, min_len)
    trie = ctx.trie_build(dev(tok), off, rep, roff, min_len, max_len)
    got_tok, got_off = trie.traces()
    got = trace_list(got_tok.cpu().numpy(), got_off)
    # oracle: per-window repeats, then IngestCandidates
    srcs = [tok[off[w]:off[w + 1]] for w in range(len(off) - 1)]
    reps = [oracle.find_repeats(s, min_len, tier=1)["repeats"] for s in srcs]
    wt, wo = oracle.traces_from_repeats(srcs, reps, min_len, max_len)
    want = trace_list(wt, wo)
    assert got == want
    T, n, m = trie.info()
    assert T == len(want) and n == sum(len(t) for t in want)


def test_trie_from_traces_order_dedup(ctx):
    rng = gen.Rng(5)
    base = [tuple(int(x) for x in gen.random_string(i, 1 + rng.below(9), 3)) for i in range(60)]
    # add duplicates, prefixes of others and high-bit tokens
    extra = [base[3], base[7], base[3][:2] or base[3], (1 << 63, 1), (1 << 63, 1), (5,), (5,)]
    allt = [t for t in base + extra if len(t)]
    flat = np.array([x for t in allt for x in t], dtype=np.uint64)
    toff = np.cumsum([0] + [len(t) for t in allt]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(flat), toff)
    got_tok, got_off = trie.traces()
    got = trace_list(got_tok.cpu().numpy(), got_off)
    assert got == sorted(set(allt), key=lambda t: (-len(t), t))


def test_trie_order_long_shared_prefixes(ctx):
    """Tie groups of equal (length, token 0, token 1) whose members share long
    prefixes: the warp-cooperative comparator must scan several 32-token
    rounds before the first difference (and see exact duplicates through)."""
    rng = gen.Rng(17)
    pre = [int(x) for x in gen.random_string(99, 150, 4)]
    allt = []
    for i in range(300):
        L = 150 + 40 * rng.below(3)
        cut = rng.below(L)
        t = pre[:min(cut, 150)] + [int(x) for x in gen.random_string(500 + i, L, 2)][min(cut, 150):]
        allt.append(tuple(t[:L]))
    allt += allt[:20]
    flat = np.array([x for t in allt for x in t], dtype=np.uint64)
    toff = np.cumsum([0] + [len(t) for t in allt]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(flat), toff)
    got_tok, got_off = trie.traces()
    got = trace_list(got_tok.cpu().numpy(), got_off)
    assert got == sorted(set(allt), key=lambda t: (-len(t), t))


def test_match_small_examples(ctx):
    # trie {abc} on stream "ababc" completes at the last token
    tr = gen.from_text("abc")
    trie = ctx.trie_build_traces(dev(tr), np.array([0, 3]))
    st = gen.from_text("ababc")
    hits = ctx.match(trie, dev(st), np.array([0, 5]))
    assert hits.cpu().tolist() == [[0, 4, 0]]
    # nested traces (a prefix of another) all reported (R14)
    traces = [gen.from_text(x) for x in ("ab", "abab", "b", "ba")]
    flat = np.concatenate(traces)
    toff = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(flat), toff)
    tt, to = trie.traces()
    streams = [gen.from_text("ababab"), gen.from_text("xbab"), gen.from_text("q")]
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + [len(s) for s in streams]).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, tt.cpu().numpy(), to)
    assert np.array_equal(hits, want)


def test_match_batch_vs_oracle(ctx):
    tok, off, st, so = small_batch(windows=10, window=1200, seed=31)
    min_len = 5
    rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, min_len)
    trie = ctx.trie_build(dev(tok), off, rep, roff, min_len, 0)
    tt, to = trie.traces()
    hits = ctx.match(trie, dev(st), so).cpu().numpy()
    want, cnt = oracle.match_brute(st, so, tt.cpu().numpy(), to)
    assert cnt == len(hits)
    assert np.array_equal(hits, want)


def test_match_no_hits_and_empty(ctx):
    trie = ctx.trie_build_traces(dev(np.array([1, 2, 3], np.uint64)), np.array([0, 3]))
    hits = ctx.match(trie, dev(np.array([4, 5, 6, 1, 2], np.uint64)), np.array([0, 5]))
    assert hits.shape[0] == 0
    empty = ctx.trie_build_traces(torch.zeros(0, dtype=torch.uint64, device="cuda"), np.array([0]))
    assert empty.info()[0] == 0
    hits = ctx.match(empty, dev(np.array([4, 5], np.uint64)), np.array([0, 2]))
    assert hits.shape[0] == 0


def test_match_both_paths(ctx):
    """Tiny alphabet: every trace's first token occurs in every stream, so the
    per-stream bucket filter gives up and the generalized-SA path runs; a
    large-alphabet case takes the per-stream path.  Both vs the oracle."""
    for alpha, nstreams in ((2, 40), (64, 12)):
        streams = [gen.random_string(1000 + q, 30 + (q * 7) % 50, alpha) for q in range(nstreams)]
        traces = sorted({tuple(int(x) for x in gen.random_string(2000 + j, 1 + j % 6, alpha)) for j in range(60)},
                        key=lambda t: (-len(t), t))
        flat = np.array([x for t in traces for x in t], dtype=np.uint64)
        toff = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
        trie = ctx.trie_build_traces(dev(flat), toff)
        tt, to = trie.traces()
        sflat = np.concatenate(streams)
        soff = np.cumsum([0] + [len(x) for x in streams]).astype(np.int64)
        hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
        want, cnt = oracle.match_brute(sflat, soff, tt.cpu().numpy(), to)
        assert np.array_equal(hits, want), alpha


def test_match_medium_batches_sampled_streams(ctx):
    """Mid-size C4-shaped batches (the per-stream matcher with its bucket
    binary searches and LCP interval extension): sampled streams against the
    brute-force oracle."""
    for (W, win, seed) in ((64, 4096, 7), (96, 16384, 4)):
        tok, off, st, so = gen.c4(seed=seed, windows=W, window=win, templates=16)
        d = dev(tok)
        rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
        trie = ctx.trie_build(d, off, rep, roff, 25, 0)
        tt, to = trie.traces()
        tth = tt.cpu().numpy()
        hits = ctx.match(trie, dev(st), so).cpu().numpy()
        for q in (0, 30, 42, W - 1):
            s1 = st[so[q]:so[q + 1]]
            want, _ = oracle.match_brute(s1, [0, len(s1)], tth, to)
            got = hits[hits[:, 0] == q].copy()
            got[:, 0] = 0
            assert np.array_equal(got, want), (W, q)


def test_trie_build_traces_multi_sources(ctx):
    """The multi-source union (the multi-GPU exchange's builder; here every
    source is a local buffer) equals trie_build_traces on the concatenation,
    including duplicates across sources and empty sources."""
    lists = []
    for seed, (W, win) in enumerate(((8, 2000), (6, 3000), (0, 0), (8, 2000))):
        if W == 0:
            lists.append((torch.zeros(0, dtype=torch.uint64, device="cuda"), np.array([0])))
            continue
        tok, off, _, _ = gen.c4(seed=40 + (seed % 3), windows=W, window=win, templates=4)
        d = dev(tok)
        rep, roff, occ = ctx.find_repeats_batched(d, off, 6)
        tt, to = ctx.trie_build(d, off, rep, roff, 6, 0).traces()
        lists.append((tt.clone(), to))
    u = ctx.trie_build_traces_multi(lists)
    flat = torch.cat([t for t, _ in lists])
    offs = [np.array([0], np.int64)]
    base = 0
    for _, o in lists:
        offs.append(o[1:] + base)
        base += int(o[-1])
    ref = ctx.trie_build_traces(flat, np.concatenate(offs))
    a, ao = u.traces()
    b, bo = ref.traces()
    assert np.array_equal(ao, bo) and torch.equal(a, b)
    assert u.info()[0] < sum(len(o) - 1 for _, o in lists)  # source 3 repeats source 0
    # the same lists back to back in one buffer (as TraceExchange stages
    # them): hashed in place, same union; and a union trie's forward traces
    # come from its reversed ones
    bases = np.cumsum([0] + [int(o[-1]) for _, o in lists])
    u2 = ctx.trie_build_traces_multi([(flat.data_ptr() + 8 * int(bases[r]), o) for r, (_, o) in enumerate(lists)])
    c, co = u2.traces()
    assert np.array_equal(co, bo) and torch.equal(c, b)
    r2 = [(flat[int(bases[r]):int(bases[r + 1])].clone(), o) for r, (_, o) in enumerate(lists)]  # gathered
    hits1 = ctx.match(u2, flat, np.asarray(bases, np.int64), cap=1 << 22)
    hits2 = ctx.match(ctx.trie_build_traces_multi(r2), flat, np.asarray(bases, np.int64), cap=1 << 22)
    assert torch.equal(hits1, hits2) and hits1.shape[0] > 0


def test_match_large_end_bins(ctx):
    """Many traces ending at the same stream position (nested runs of one
    token): end bins far larger than the per-hit ranking threshold take the
    warp bitonic path of the ordered emitter; order (stream, end, id) and
    content vs the brute-force oracle."""
    a, b = 7, 9
    traces = sorted({(a,) * L for L in range(1, 120)} | {(a,) * L + (b,) for L in range(1, 40)},
                    key=lambda t: (-len(t), t))
    flat = np.array([x for t in traces for x in t], dtype=np.uint64)
    toff = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(flat), toff)
    tt, to = trie.traces()
    streams = [np.full(3000, a, np.uint64), np.array([a] * 500 + [b] + [a] * 200, np.uint64)]
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + [len(x) for x in streams]).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, tt.cpu().numpy(), to)
    assert cnt == len(hits) and np.array_equal(hits, want)


def test_match_deep_nesting():
    """More nested traces at one end than the sweep's on-chip stack ring and
    more matched traces in one stream than one staging chunk (1,100 runs of
    one token): the interval-forest sweep must fall back to its parent links
    exactly; compared with the brute-force oracle."""
    from paper_2406_18111_b200 import Context
    ctx = Context(0)
    a = 11
    traces = [(a,) * L for L in range(1100, 0, -1)]
    flat = np.array([x for t in traces for x in t], dtype=np.uint64)
    toff = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(flat), toff)
    tt, to = trie.traces()
    streams = [np.full(2500, a, np.uint64), np.array([a] * 1200 + [3] + [a] * 50, np.uint64)]
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + [len(x) for x in streams]).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, tt.cpu().numpy(), to)
    assert cnt == len(hits) and np.array_equal(hits, want)


def test_match_tree_sweep_fallback():
    """The sequential interval-forest sweep (the fallback for streams nested
    deeper than the parallel builder's on-chip stack), forced for every
    stream in a subprocess, gives the same hits as the brute-force oracle."""
    import subprocess, sys, os
    code = ("import importlib.util, sys; sys.path.insert(0, '.'); "
            "spec = importlib.util.spec_from_file_location('tgt', 'tests/test_gpu_trie.py'); "
            "t = importlib.util.module_from_spec(spec); spec.loader.exec_module(t); "
            "from paper_2406_18111_b200 import Context; c = Context(0); "
            "t.test_match_deep_nesting(); t.test_match_large_end_bins(c); t.test_match_batch_vs_oracle(c)")
    env = dict(os.environ, APO_TREE_SEQ="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def test_match_many_intervals_one_stream(ctx):
    """More matched traces in one stream than the emitter keeps on chip
    (> 8,192 intervals): the global-table path of k_stream_emit, against the
    brute-force oracle."""
    rng = gen.Rng(77)
    s = np.array([int(x) for x in gen.random_string(4242, 12000, 8)], dtype=np.uint64)
    seen = set()
    while len(seen) < 9000:
        L = 5 + rng.below(6)
        p = rng.below(len(s) - L)
        seen.add(tuple(int(x) for x in s[p:p + L]))
    traces = sorted(seen, key=lambda t: (-len(t), t))
    flat = np.array([x for t in traces for x in t], dtype=np.uint64)
    toff = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(flat), toff)
    tt, to = trie.traces()
    sflat = np.concatenate([s, s[:3000]])
    soff = np.array([0, len(s), len(s) + 3000], dtype=np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, tt.cpu().numpy(), to)
    assert cnt == len(hits) and np.array_equal(hits, want)
    # REPLAY over the implicit MATCH_ALL: the per-end chain kernel with more
    # intervals than it keeps root lengths for on chip (> 7,168)
    rp, nall = ctx.match(trie, dev(sflat), soff, mode=1)
    tlen = np.diff(to)
    want_rp = oracle.replay(want, tlen)
    g = rp.cpu().numpy().astype(np.int64)
    got_rp = np.stack([g[:, 0], g[:, 1] - tlen[g[:, 2]] + 1, g[:, 1], g[:, 2], g[:, 3]], axis=1)
    assert nall == cnt and np.array_equal(got_rp, want_rp)


def test_match_capacity_prefix(ctx):
    """With cap < number of hits, apo_match stores exactly the first cap
    records of the full sorted output (odd caps cut a 32-byte record pair),
    reports the true count, and leaves the rest of the buffer untouched."""
    from paper_2406_18111_b200.apo import _ptr, _P_I64, _stream
    tok, off, st, so = gen.c4(seed=31, windows=10, window=1200, templates=6)
    rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, 5)
    trie = ctx.trie_build(dev(tok), off, rep, roff, 5, 0)
    ds = dev(st)
    full = ctx.match(trie, ds, so)
    nh = full.shape[0]
    assert nh > 100
    o = np.ascontiguousarray(so, dtype=np.int64)
    for cap in (1, 7, nh // 3, nh // 2 + 1, nh - 1):
        out = torch.full((cap + 8, 4), -5, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        ctx._raise(ctx.lib.apo_match(ctx.h, trie.h, _ptr(ds), o.ctypes.data_as(_P_I64), len(o) - 1, 0,
                                     _ptr(out), cap, _ptr(cnt), _stream(ctx.device)))
        assert int(cnt.item()) == nh
        assert torch.equal(out[:cap, :3], full[:cap])
        assert bool((out[cap:] == -5).all())


def test_match_long_streams(ctx):
    """Streams longer than the on-chip limit (> 16,384 ops): the per-stream
    path with global binary searches, hit enumeration and the (stream, end)
    sort; against the brute-force oracle."""
    S = gen.c3()[:60000]
    wtok = S[:20000]
    d = dev(wtok)
    off = np.array([0, len(wtok)], dtype=np.int64)
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    tt, to = trie.traces()
    streams = [S[20000:40000], S[40000:57000], S[57000:60000]]
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + [len(x) for x in streams]).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, tt.cpu().numpy(), to)
    assert cnt == len(hits) and np.array_equal(hits, want)
    assert len(hits) > 0


def test_match_indexed_equals_match():
    """apo_match_index + apo_match_indexed (the stream index built before and
    independently of the trace set, reused for two trace sets and both
    modes) == apo_match."""
    from paper_2406_18111_b200 import Context
    ctx = Context(0)
    tok, off, st, so = gen.c4(seed=71, windows=32, window=4096, templates=8)
    d, ds = torch.from_numpy(tok).cuda(), torch.from_numpy(st).cuda()
    idx = ctx.match_index(ds, so)
    for half in (slice(0, 16), slice(16, 32)):
        o = off[half.start:half.stop + 1] - off[half.start]
        dd = d[int(off[half.start]):int(off[half.stop])]
        rep, roff, occ = ctx.find_repeats_batched(dd, o, 25)
        trie = ctx.trie_build(dd, o, rep, roff, 25, 0)
        a = ctx.match(trie, ds, so, full=True)
        b = ctx.match_indexed(trie, idx, full=True)
        assert a.shape[0] > 0 and torch.equal(a, b)
        ra, na = ctx.match(trie, ds, so, mode=1)
        rb, nb = ctx.match_indexed(trie, idx, mode=1)
        assert na == nb and torch.equal(ra, rb)


def test_match_indexed_long_streams_and_empty_trie():
    """The split matcher on streams longer than the on-chip limit (the
    global per-stream search path, not reversed) and against an empty-ish
    trace set: equal to apo_match."""
    from paper_2406_18111_b200 import Context
    ctx = Context(0)
    streams = [gen.periodic(81, 40000, 97, 6, noise=0.01), gen.periodic(82, 9000, 31, 4, noise=0.02)]
    st = np.concatenate(streams)
    so = np.cumsum([0] + [len(x) for x in streams]).astype(np.int64)
    ds = torch.from_numpy(st).cuda()
    rng = gen.Rng(83)
    traces = sorted({tuple(int(x) for x in streams[rng.below(2)][a:a + 3 + rng.below(40)])
                     for a in (rng.below(8000) for _ in range(300))}, key=lambda t: (-len(t), t))
    tt = np.concatenate([np.asarray(t, dtype=np.uint64) for t in traces])
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(torch.from_numpy(tt).cuda(), to)
    idx = ctx.match_index(ds, so)
    a = ctx.match(trie, ds, so, full=True, cap=1 << 24)
    b = ctx.match_indexed(trie, idx, full=True, cap=1 << 24)
    assert a.shape[0] > 0 and torch.equal(a, b)
    ra, na = ctx.match(trie, ds, so, mode=1)
    rb, nb = ctx.match_indexed(trie, idx, mode=1)
    assert na == nb and torch.equal(ra, rb)
    one = ctx.trie_build_traces(torch.from_numpy(np.array([1, 2, 3], dtype=np.uint64)).cuda(),
                                np.array([0, 3], dtype=np.int64))
    assert ctx.match_indexed(one, idx).shape[0] == ctx.match(one, ds, so).shape[0] == 0


def test_match_dense_id_order_edges(ctx):
    """The dense-id matcher (k_stream_match_ids): stream tokens include 0,
    2^63 and ~0; traces diverge from stream substrings at tokens that are
    absent from the streams and fall below, between and above the stream
    vocabulary (their comparison values are odd), and run past stream ends.
    Both modes against the oracle."""
    rng = gen.Rng(91)
    M = (1 << 64) - 1
    alpha = np.array([0, 7, 9, 1 << 63, M - 1, M], dtype=np.uint64)
    absent = [1, 8, 10, (1 << 63) - 1, (1 << 63) + 1, M - 2]
    lens = [300, 1, 2, 777, 2000, 16384, 33, 1500]
    streams = [alpha[gen.Rng(900 + q).below_np(len(alpha), n).astype(np.int64)] for q, n in enumerate(lens)]
    traces = set()
    for j in range(400):
        s = streams[rng.below(len(streams))]
        a = rng.below(len(s))
        L = 1 + rng.below(40)
        t = [int(x) for x in s[a:a + L]]
        if j % 3 == 1 and len(t) > 1:  # diverge at an absent token
            t[rng.below(len(t))] = absent[rng.below(len(absent))]
        elif j % 3 == 2:  # run past the stream end / extend
            t = t + [int(alpha[rng.below(len(alpha))]) for _ in range(rng.below(5))]
        traces.add(tuple(t))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    tt = np.array([x for t in traces for x in t], dtype=np.uint64)
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(tt), to)
    gt, go = trie.traces()
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + lens).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff, cap=1 << 24).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, gt.cpu().numpy(), go)
    assert cnt == len(hits) and np.array_equal(hits, want) and cnt > 0
    rp, nall = ctx.match(trie, dev(sflat), soff, mode=1)
    tlen = np.diff(go)
    want_rp = oracle.replay(want, tlen)
    g = rp.cpu().numpy().astype(np.int64)
    got_rp = np.stack([g[:, 0], g[:, 1] - tlen[g[:, 2]] + 1, g[:, 1], g[:, 2], g[:, 3]], axis=1)
    assert nall == cnt and np.array_equal(got_rp, want_rp)


def test_match_large_vocabulary_raw_token_path(ctx):
    """More than 65,534 distinct tokens in the stream batch: the matcher
    compares raw 64-bit tokens (k_stream_match); against the oracle."""
    lens = [15000, 16384, 14000, 12000, 16000]
    streams = [gen.random_string(950 + q, n, 1 << 40) for q, n in enumerate(lens)]
    assert len(np.unique(np.concatenate(streams))) > 65534
    rng = gen.Rng(96)
    traces = set()
    for j in range(500):
        s = streams[rng.below(len(streams))]
        a = rng.below(len(s) - 60)
        t = [int(x) for x in s[a:a + 1 + rng.below(50)]]
        if j % 4 == 3:
            t[-1] = int(streams[0][rng.below(100)])
        traces.add(tuple(t))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    tt = np.array([x for t in traces for x in t], dtype=np.uint64)
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(tt), to)
    gt, go = trie.traces()
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + lens).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, gt.cpu().numpy(), go)
    assert cnt == len(hits) and np.array_equal(hits, want) and cnt >= 300


def test_match_vocabulary_over_id_table_budget(ctx):
    """A stream batch with more distinct tokens than the dense-id table holds
    (~1.6 M distinct in 100 streams of 16,384): no dense ids, the matcher
    reverses the raw tokens and runs K9 from the 64-bit level-0 sort; mode 0
    and mode 1 against the oracle."""
    lens = [16384] * 100
    streams = [gen.random_string(3000 + q, n, 1 << 62) for q, n in enumerate(lens)]
    rng = gen.Rng(97)
    traces = set()
    for j in range(300):
        s = streams[rng.below(len(streams))]
        a = rng.below(len(s) - 40)
        traces.add(tuple(int(x) for x in s[a:a + 1 + rng.below(30)]))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    tt = np.array([x for t in traces for x in t], dtype=np.uint64)
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(tt), to)
    gt, go = trie.traces()
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + lens).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, gt.cpu().numpy(), go)
    assert cnt == len(hits) and np.array_equal(hits, want) and cnt >= 300
    rp, nall = ctx.match(trie, dev(sflat), soff, mode=1)
    tlen = np.diff(go)
    want_rp = oracle.replay(want, tlen)
    g = rp.cpu().numpy().astype(np.int64)
    got_rp = np.stack([g[:, 0], g[:, 1] - tlen[g[:, 2]] + 1, g[:, 1], g[:, 2], g[:, 3]], axis=1)
    assert nall == cnt and np.array_equal(got_rp, want_rp)


def test_match_indexed_one_token_traces():
    """A stream index keys its buckets by the first two tokens; a trace set
    with 1-token traces makes the search rebuild them by the first token:
    match_indexed == match == the oracle, both modes."""
    from paper_2406_18111_b200 import Context
    ctx = Context(0)
    streams = [gen.random_string(700 + q, 3000 + 17 * q, 40) for q in range(6)]
    st = np.concatenate(streams)
    so = np.cumsum([0] + [len(x) for x in streams]).astype(np.int64)
    ds = torch.from_numpy(st).cuda()
    idx = ctx.match_index(ds, so)
    rng = gen.Rng(701)
    traces = {(int(streams[0][5]),), (int(streams[1][9]),)}
    for _ in range(200):
        s = streams[rng.below(len(streams))]
        a = rng.below(len(s) - 10)
        traces.add(tuple(int(x) for x in s[a:a + 1 + rng.below(8)]))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    tt = np.array([x for t in traces for x in t], dtype=np.uint64)
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(torch.from_numpy(tt).cuda(), to)
    gt, go = trie.traces()
    a = ctx.match(trie, ds, so, full=True, cap=1 << 22)
    b = ctx.match_indexed(trie, idx, full=True, cap=1 << 22)
    want, cnt = oracle.match_brute(st, so, gt.cpu().numpy(), go)
    assert torch.equal(a, b) and cnt == a.shape[0] and np.array_equal(a[:, :3].cpu().numpy(), want)
    ra, na = ctx.match(trie, ds, so, mode=1)
    rb, nb = ctx.match_indexed(trie, idx, mode=1)
    assert na == nb == cnt and torch.equal(ra, rb)


def test_match_dense_ids_many_absent_trace_tokens(ctx):
    """Dense-id matcher with a dictionary of ~30 K stream tokens and traces
    whose tokens are mostly absent from the streams (as the peers' traces
    are at N > 1): the absent tokens' comparison values come from the
    on-chip dictionary sample (k_trace_ids).  Both modes against the oracle."""
    rng = gen.Rng(93)
    vocab = np.unique(gen.H_np(3, gen.Rng(94).below_np(1 << 40, 40000)))
    lens = [4000, 16384, 2500, 1, 7000, 3000]
    streams = [vocab[gen.Rng(950 + q).below_np(len(vocab), n).astype(np.int64)] for q, n in enumerate(lens)]
    traces = set()
    for j in range(3000):
        if j % 4 == 3:  # entirely foreign tokens (between, below and above the vocabulary)
            t = [int(x) for x in gen.H_np(5 + j, gen.Rng(960 + j).below_np(1 << 40, 1 + rng.below(30)))]
        else:
            s = streams[rng.below(len(streams))]
            a = rng.below(len(s))
            t = [int(x) for x in s[a:a + 1 + rng.below(40)]]
            if j % 4 == 1:  # one absent token
                t[rng.below(len(t))] = int(gen.H_np(7, np.array([j], dtype=np.uint64))[0])
        traces.add(tuple(t))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    tt = np.array([x for t in traces for x in t], dtype=np.uint64)
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(tt), to)
    gt, go = trie.traces()
    sflat = np.concatenate(streams)
    soff = np.cumsum([0] + lens).astype(np.int64)
    hits = ctx.match(trie, dev(sflat), soff, cap=1 << 24).cpu().numpy()
    want, cnt = oracle.match_brute(sflat, soff, gt.cpu().numpy(), go)
    assert cnt == len(hits) and np.array_equal(hits, want) and cnt > 0
    rp, nall = ctx.match(trie, dev(sflat), soff, mode=1)
    tlen = np.diff(go)
    want_rp = oracle.replay(want, tlen)
    g = rp.cpu().numpy().astype(np.int64)
    got_rp = np.stack([g[:, 0], g[:, 1] - tlen[g[:, 2]] + 1, g[:, 1], g[:, 2], g[:, 3]], axis=1)
    assert nall == cnt and np.array_equal(got_rp, want_rp)
