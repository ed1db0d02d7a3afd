"""REPLAY selection on the GPU (apo_replay, apo_match mode 1) vs the oracle
(oracle.replay, pinned in tests/test_oracle_pins.py): Alg. 1
SelectReplayTrace / ExecuteAndReplay, scoring P:694-713,
readings R20-R24.  The oracle's hits come from its own brute-force matcher;
nothing on the oracle side comes from the CUDA path."""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from workloads import gen

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_18111_b200 import build
    build.build()
    from paper_2406_18111_b200 import Context
    return Context(0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64)).cuda()


def as_oracle_rows(got, tlen):
    """GPU (stream, end, trace, first) -> oracle layout (stream, start, end, trace, first)."""
    g = np.asarray(got, dtype=np.int64).reshape(-1, 4)
    start = g[:, 1] - np.asarray(tlen, dtype=np.int64)[g[:, 2]] + 1 if len(g) else np.zeros(0, np.int64)
    return np.stack([g[:, 0], start, g[:, 1], g[:, 2], g[:, 3]], axis=1) if len(g) else np.zeros((0, 5), np.int64)


def run_case(ctx, streams, traces, **params):
    """GPU: trace set from explicit traces, MATCH_ALL, apo_replay.  Oracle:
    brute-force MATCH_ALL, oracle.replay."""
    tr = [np.asarray(t, dtype=np.uint64) for t in traces]
    tt = np.concatenate(tr) if tr else np.zeros(0, np.uint64)
    to = np.cumsum([0] + [len(t) for t in tr]).astype(np.int64)
    st = np.concatenate(streams)
    so = np.cumsum([0] + [len(s) for s in streams]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(tt), to)
    gtok, goff = trie.traces()
    assert np.array_equal(goff, to) and np.array_equal(gtok.cpu().numpy(), tt)  # traces given in id order
    hits = ctx.match(trie, dev(st), so, full=True)
    got = ctx.replay(trie, hits, np.diff(so), **params).cpu().numpy()
    oh, _ = oracle.match_brute(st, so, tt, to)
    want = oracle.replay(oh, [len(t) for t in tr], **params)
    return as_oracle_rows(got, [len(t) for t in tr]), want, trie, st, so


def test_replay_golden(ctx):
    g = json.load(open(os.path.join(HERE, "golden", "replay_examples.json")))
    for c in g["cases"]:
        if "stream" in c:
            S = np.array(c["stream"], dtype=np.uint64)
        else:
            S = np.array(list(range(1, 9)) + list(range(1000, 1300)) + [99, 5, 6, 7, 8] + list(range(1, 9)),
                         dtype=np.uint64)
        got, want, *_ = run_case(ctx, [S], c["traces"], **c["params"])
        assert got.tolist() == c["replays"] == want.tolist(), c["name"]
        if "replays_no_decay" in c:
            got, want, *_ = run_case(ctx, [S], c["traces"], **dict(c["params"], decay_q16=65536))
            assert got.tolist() == c["replays_no_decay"] == want.tolist(), c["name"]


def random_cases():
    out = []
    for seed in range(30):
        rng = gen.Rng(900 + seed)
        nst = 1 + rng.below(5)
        streams = [gen.periodic(seed * 11 + j, 30 + rng.below(600), 1 + rng.below(12), 2 + rng.below(3),
                                noise=0.04) for j in range(nst)]
        traces = {tuple(int(x) for x in s[a:a + 1 + rng.below(15)])
                  for s in streams for a in [rng.below(max(len(s) - 15, 1)) for _ in range(8)]}
        traces = sorted(traces, key=lambda t: (-len(t), t))
        out.append((streams, traces))
    return out


@pytest.mark.parametrize("params", [{}, dict(count_cap=3), dict(decay_period=2), dict(bonus_num=1, bonus_den=1),
                                    dict(count_cap=1, decay_q16=65536, bonus_num=1, bonus_den=1),
                                    dict(count_cap=200), dict(decay_period=7, count_cap=1000)])
def test_replay_random(ctx, params):
    for streams, traces in random_cases():
        got, want, *_ = run_case(ctx, streams, traces, **params)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("params", [{}, dict(count_cap=200)])
def test_replay_long_streams_global_state(ctx, params):
    """Streams longer than the on-chip matcher limit: hits come from the
    sorted-key path with slot = trace id, and streams with more slots than
    the on-chip state table (8,192 narrow u32 states, or 4,096 wide u64
    states when count_cap > 127) keep their trace states in global memory."""
    streams = [gen.periodic(7, 40000, 97, 6, noise=0.01), gen.periodic(8, 20000, 31, 3, noise=0.02)]
    rng = gen.Rng(77)
    traces = set()
    for _ in range(30000):
        s = streams[rng.below(2)]
        a = rng.below(len(s) - 60)
        traces.add(tuple(int(x) for x in s[a:a + 2 + rng.below(58)]))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    assert len(traces) > 8192
    got, want, *_ = run_case(ctx, streams, traces, **params)
    assert len(want) > 100 and np.array_equal(got, want)


def test_match_mode_replay_equals_two_calls(ctx):
    """apo_match mode 1 (REPLAY) == apo_match mode 0 + apo_replay."""
    tok, off, st, so = gen.c4(seed=21, windows=48, window=4096, templates=8)
    d = dev(tok)
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    hits = ctx.match(trie, dev(st), so, full=True)
    two = ctx.replay(trie, hits, np.diff(so))
    one, nh = ctx.match(trie, dev(st), so, mode=1)
    assert nh == hits.shape[0] and torch.equal(one, two) and one.shape[0] > 0


def test_replay_c4_shaped_vs_oracle(ctx):
    """A C4-shaped batch (windows analysed by the oracle, union trace set by
    the oracle, brute-force hits): every stream's replays equal the oracle."""
    tok, off, st, so = gen.c4(seed=31, windows=16, window=4096, templates=16)
    W = len(off) - 1
    reps = [oracle.find_repeats(tok[off[w]:off[w + 1]], 25, tier=1)["repeats"] for w in range(W)]
    tt, to = oracle.traces_from_repeats_np([tok[off[w]:off[w + 1]] for w in range(W)], reps, 25, 0)
    got, want, *_ = run_case(ctx, [st[so[q]:so[q + 1]] for q in range(W)],
                             [tt[to[t]:to[t + 1]] for t in range(len(to) - 1)])
    assert len(want) > 0 and np.array_equal(got, want)


def test_match_mode_replay_heavy_streams(ctx):
    """apo_match mode 1 takes the trace states from the matcher's index
    (wavelet queries over the reversed streams' suffix arrays, several work
    items per stream beyond 65,536 hits); it must equal MATCH_ALL + the
    general apo_replay path, and the oracle on a sampled stream."""
    streams = [gen.periodic(41 + k, 16384, p, 12, noise=0.01) for k, p in enumerate((5, 13, 40))]
    streams.append(gen.random_string(44, 3000, 50))
    rng = gen.Rng(45)
    traces = set()
    for _ in range(4000):
        s = streams[rng.below(3)]
        a = rng.below(len(s) - 64)
        traces.add(tuple(int(x) for x in s[a:a + 3 + rng.below(60)]))
    traces = sorted(traces, key=lambda t: (-len(t), t))
    tt = np.concatenate([np.asarray(t, dtype=np.uint64) for t in traces])
    to = np.cumsum([0] + [len(t) for t in traces]).astype(np.int64)
    st = np.concatenate(streams)
    so = np.cumsum([0] + [len(s) for s in streams]).astype(np.int64)
    trie = ctx.trie_build_traces(dev(tt), to)
    hits = ctx.match(trie, dev(st), so, full=True, cap=1 << 26)
    per = np.bincount(hits[:, 0].cpu().numpy(), minlength=len(streams))
    assert per.max() > 65536  # several wavelet work items for a stream
    two = ctx.replay(trie, hits, np.diff(so))
    one, nh = ctx.match(trie, dev(st), so, mode=1)
    assert nh == hits.shape[0] and torch.equal(one, two) and one.shape[0] > 0
    # the oracle on the third stream (brute-force hits of that stream alone)
    q = 2
    oh, _ = oracle.match_brute(streams[q], np.array([0, len(streams[q])], dtype=np.int64), tt, to)
    want = oracle.replay(oh, [len(t) for t in traces])
    g = one.cpu().numpy()
    g = g[g[:, 0] == q].copy()
    g[:, 0] = 0
    assert np.array_equal(as_oracle_rows(g, [len(t) for t in traces]), want)


@pytest.mark.parametrize("ccap,scan_max", [("1", None), ("5", None), (None, "0"), ("7", "40")])
def test_match_mode_replay_candidate_pool_overflow(ctx, ccap, scan_max, monkeypatch):
    """REPLAY by ends with a tiny candidate pool (decisions with several
    eligible records that do not fit are decided by the whole warp in
    k_rp_dec_pick) and with short scan limits (candidates scored by wavelet
    queries instead of occurrence-range scans): the replays equal MATCH_ALL +
    the general apo_replay."""
    tok, off, st, so = gen.c4(seed=23, windows=24, window=4096, templates=8)
    d = dev(tok)
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    hits = ctx.match(trie, dev(st), so, full=True)
    two = ctx.replay(trie, hits, np.diff(so))
    if ccap:
        monkeypatch.setenv("APO_REPLAY_CCAP", ccap)
    if scan_max:
        monkeypatch.setenv("APO_REPLAY_SCANMAX", scan_max)
    one, nh = ctx.match(trie, dev(st), so, mode=1)
    assert nh == hits.shape[0] and torch.equal(one, two) and one.shape[0] > 0


@pytest.mark.parametrize("ccap", [None, "3"])
def test_match_mode_replay_eager_equals_lazy(ctx, ccap, monkeypatch):
    """apo_match mode 1 keeps MATCH_ALL implicit (per end the deepest matched
    interval; decisions walk their chains); APO_REPLAY_EAGER=1 writes every
    hit record and REPLAY reads the records instead.  Both give the same
    replays and hit count, also with a tiny candidate pool."""
    tok, off, st, so = gen.c4(seed=27, windows=32, window=4096, templates=8)
    d = dev(tok)
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    if ccap:
        monkeypatch.setenv("APO_REPLAY_CCAP", ccap)
    lazy, nl = ctx.match(trie, dev(st), so, mode=1)
    monkeypatch.setenv("APO_REPLAY_EAGER", "1")
    eager, ne = ctx.match(trie, dev(st), so, mode=1)
    assert nl == ne and torch.equal(lazy, eager) and lazy.shape[0] > 0
