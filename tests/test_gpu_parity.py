"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element
by element, on seeded synthetic inputs.  Everything is integer, so the bar is
bit-exact equality.
"""
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


def small_cases():
    cases = [gen.from_text("aabcbcbaa"), gen.from_text("ababab"), gen.from_text("aaaaaaa"),
             gen.from_text("abababa"), np.array([5], np.uint64), np.array([5, 5], np.uint64),
             np.array([1 << 63, 0, 1 << 63, 0], np.uint64), np.full(300, 7, np.uint64)]
    for seed in range(12):
        cases.append(gen.random_string(seed, 1 + (seed * 97) % 700, 1 + seed % 6))
    for seed in range(4):
        cases.append(gen.high_bit_string(seed, 500, 6))
    cases.append(gen.periodic(3, 5000, 37, 4, noise=0.01))
    cases.append(gen.fibonacci_word(3000))
    cases.append(gen.c1())
    return cases


def multi_tile_cases():
    # several 4,096-key sort tiles plus a ragged tail
    return [gen.random_string(77, 9000, 3), gen.periodic(5, 13001, 64, 3, noise=0.02),
            gen.c2()[:20000], gen.c3()[:17000]]


@pytest.mark.parametrize("case", range(len(small_cases())))
def test_sa_lcp_small(ctx, case):
    S = small_cases()[case]
    sa, lcp = ctx.suffix_array(dev(S))
    want = oracle.sa_naive(S)
    assert np.array_equal(sa.cpu().numpy(), want)
    assert np.array_equal(lcp.cpu().numpy(), oracle.lcp_naive(S, want))


@pytest.mark.parametrize("case", range(4))
def test_sa_lcp_multi_tile(ctx, case):
    S = multi_tile_cases()[case]
    sa, lcp = ctx.suffix_array(dev(S))
    want = oracle.sa_doubling(S)
    assert np.array_equal(sa.cpu().numpy(), want)
    assert np.array_equal(lcp.cpu().numpy(), oracle.lcp_kasai(S, want))


def check_find(ctx, S, min_len, min_count=1, tier=0):
    want = oracle.find_repeats(S, min_len, min_count, tier=tier)
    if len(S) >= 2:
        c = ctx.candidates(dev(S), min_len)
        assert np.array_equal(c["cand_len"].cpu().numpy(), want["cand_len"])
        assert np.array_equal(c["cand_start"].cpu().numpy(), want["cand_start"])
        assert np.array_equal(c["cand_id"].cpu().numpy(), want["cand_id"])
        assert np.array_equal(c["keep"].cpu().numpy(), want["keep"])
    rep, occ = ctx.find_repeats(dev(S), min_len, min_count)
    assert np.array_equal(rep.cpu().numpy(), want["repeats"])
    assert np.array_equal(occ.cpu().numpy(), want["occ"])


@pytest.mark.parametrize("case", range(len(small_cases())))
@pytest.mark.parametrize("min_len", [1, 2, 5])
def test_find_repeats_small(ctx, case, min_len):
    check_find(ctx, small_cases()[case], min_len)


@pytest.mark.parametrize("case", range(4))
def test_find_repeats_multi_tile(ctx, case):
    check_find(ctx, multi_tile_cases()[case], 3, tier=1)
    check_find(ctx, multi_tile_cases()[case], 25, tier=1)


def test_min_count(ctx):
    for S in (gen.from_text("aabcbcbaa"), gen.c1()):
        check_find(ctx, S, 2, min_count=2)


def test_edge_cases(ctx):
    from paper_2406_18111_b200 import ApoError
    rep, occ = ctx.find_repeats(dev(np.zeros(0, np.uint64)), 1)
    assert rep.shape[0] == 0 and occ.shape[0] == 0
    rep, occ = ctx.find_repeats(dev(gen.c1()[:9]), 5)      # n < 2 * min_len
    assert rep.shape[0] == 0
    with pytest.raises(ApoError):
        ctx.find_repeats(dev(gen.c1()[:9]), 0)
    sa, lcp = ctx.suffix_array(dev(np.array([3], np.uint64)))
    assert sa.tolist() == [0] and lcp.numel() == 0



@pytest.mark.parametrize("spec", [1, 2, 3, 8])
@pytest.mark.parametrize("case", range(4))
def test_sa_lcp_speculative_rounds(ctx, case, spec, monkeypatch):
    """Global doubling path (> 16,384 tokens) with 1-8 Manber-Myers rounds
    launched per host convergence read: the rounds after convergence are
    gated off on the device, the SA/LCP must equal the oracle's."""
    S = [gen.c2()[:20000], gen.c3()[:17000], gen.periodic(6, 40000, 7, 3),
         gen.fibonacci_word(30000)][case]
    monkeypatch.setenv("APO_SPEC_ROUNDS", str(spec))
    sa, lcp = ctx.suffix_array(dev(S))
    want = oracle.sa_doubling(S)
    assert np.array_equal(sa.cpu().numpy(), want)
    assert np.array_equal(lcp.cpu().numpy(), oracle.lcp_kasai(S, want))

def test_config_c1_full(ctx):
    check_find(ctx, gen.c1(), 5, tier=0)


def test_config_c2_full(ctx):
    S = gen.c2()
    sa, lcp = ctx.suffix_array(dev(S))
    want = oracle.sa_doubling(S)
    assert oracle.sa_check(S, sa.cpu().numpy())
    assert np.array_equal(sa.cpu().numpy(), want)
    assert np.array_equal(lcp.cpu().numpy(), oracle.lcp_kasai(S, want))
    check_find(ctx, S, 25, tier=1)


def test_config_c3_full(ctx):
    S = gen.c3()
    sa, lcp = ctx.suffix_array(dev(S))
    sa = sa.cpu().numpy()
    assert oracle.sa_check(S, sa)                      # O(n) certificate: SA is unique
    want = oracle.sa_doubling(S)
    assert np.array_equal(sa, want)
    assert np.array_equal(lcp.cpu().numpy(), oracle.lcp_kasai(S, want))
    check_find(ctx, S, 25, tier=1)


def batch_case(windows=24, window=2048, seed=11):
    tok, off, _, _ = gen.c4(seed=seed, windows=windows, window=window, templates=8, with_streams=False)
    # ragged: cut some windows short, include an empty and a tiny window
    lens = [window] * windows
    lens[1] = 0
    lens[2] = 7
    lens[5] = window // 3
    parts = [tok[off[w]:off[w] + lens[w]] for w in range(windows)]
    new_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return np.concatenate(parts), new_off


def test_batched_sa_equals_per_window(ctx):
    tok, off = batch_case()
    sa, lcp = ctx.suffix_array_batched(dev(tok), off)
    sa, lcp = sa.cpu().numpy(), lcp.cpu().numpy()
    for w in range(len(off) - 1):
        S = tok[off[w]:off[w + 1]]
        want = oracle.sa_doubling(S)
        assert np.array_equal(sa[off[w]:off[w + 1]], want)
        wl = oracle.lcp_kasai(S, want)
        got = lcp[off[w]:off[w + 1]]
        assert np.array_equal(got[:max(len(S) - 1, 0)], wl)
        if len(S):
            assert got[-1] == 0


def test_batched_find_equals_per_window(ctx):
    tok, off = batch_case()
    for min_len in (5, 25):
        rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, min_len)
        rep, roff, occ = rep.cpu().numpy(), roff.cpu().numpy(), occ.cpu().numpy()
        assert roff[0] == 0 and roff[-1] == len(rep)
        for w in range(len(off) - 1):
            want = oracle.find_repeats(tok[off[w]:off[w + 1]], min_len, tier=1)
            got = rep[roff[w]:roff[w + 1]]
            assert np.array_equal(got[:, :3], want["repeats"][:, :3]), w
            for row, wrow in zip(got, want["repeats"]):
                assert np.array_equal(occ[row[3]:row[3] + row[2]], want["occ"][wrow[3]:wrow[3] + wrow[2]])


def test_c4_full_batch_sampled(ctx):
    """C4 at full size, in the bench's launch configuration; 24 sampled
    windows are compared with the oracle one by one, every window is checked
    for the output invariants."""
    tok, off, _, _ = gen.c4(with_streams=False)
    rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, 25)
    rep, roff, occ = rep.cpu().numpy(), roff.cpu().numpy(), occ.cpu().numpy()
    W = len(off) - 1
    rng = gen.Rng(123)
    sample = sorted({int(rng.below(W)) for _ in range(24)} | {0, W - 1})
    for w in sample:
        want = oracle.find_repeats(tok[off[w]:off[w + 1]], 25, tier=1)
        got = rep[roff[w]:roff[w + 1]]
        assert np.array_equal(got[:, :3], want["repeats"][:, :3]), w
    # invariants everywhere: disjoint occurrences, equal contents, length >= 25
    for w in range(0, W, 97):
        S = tok[off[w]:off[w + 1]]
        cov = np.zeros(len(S), np.int32)
        for st, ln, cnt, f in rep[roff[w]:roff[w + 1]]:
            assert ln >= 25
            for o in occ[f:f + cnt]:
                assert np.array_equal(S[o:o + ln], S[st:st + ln])
                cov[o:o + ln] += 1
        assert cov.max(initial=0) <= 1


def test_determinism(ctx):
    S = gen.c3()[:200000]
    a = ctx.find_repeats(dev(S), 25)
    b = ctx.find_repeats(dev(S), 25)
    assert all(torch.equal(x, y) for x, y in zip(a, b))


def test_history_ingest_and_window(ctx):
    S = gen.c3()[:20000]
    h = ctx.history(5000, 500)
    got = []
    pos = 0
    for chunk in (1, 499, 500, 1234, 7766, 10000):
        got += h.ingest(dev(S[pos:pos + chunk]))
        pos += chunk
    assert got == oracle.ruler_slices(0, 20000, 500, 5000)
    assert h.count == 20000
    for b, e in got[-5:]:
        assert np.array_equal(h.window(b, e).cpu().numpy(), S[b:e])


def test_config_c5_proxy(ctx):
    """C5's structure (4-token alphabet, 1,000-op period) at 2^20: full parity."""
    S = gen.c5(n=1 << 20)
    sa, lcp = ctx.suffix_array(dev(S))
    want = oracle.sa_doubling(S)
    assert np.array_equal(sa.cpu().numpy(), want)
    assert np.array_equal(lcp.cpu().numpy(), oracle.lcp_kasai(S, want))
    check_find(ctx, S, 25, tier=1)


def test_config_c5_full(ctx):
    """C5 at 2^26 (64M): the O(n) suffix-array certificate (the SA is unique),
    sampled LCP entries by direct comparison, and the repeat invariants."""
    S = gen.c5()
    d = dev(S)
    sa, lcp = ctx.suffix_array(d)
    sa_h = sa.cpu().numpy()
    assert oracle.sa_check(S, sa_h)
    lcp_h = lcp.cpu().numpy()
    rng = gen.Rng(55)
    for _ in range(8):
        k = int(rng.below(len(S) - 1))
        a, b = int(sa_h[k]), int(sa_h[k + 1])
        L = int(lcp_h[k])
        m = min(len(S) - a, len(S) - b)
        assert L <= m and np.array_equal(S[a:a + L], S[b:b + L])
        assert L == m or S[a + L] != S[b + L]
    del sa, lcp
    rep, occ = ctx.find_repeats(d, 25)
    rep, occ = rep.cpu().numpy(), occ.cpu().numpy()
    assert len(rep) >= 1
    # the longest candidate is always kept first (R12, valid form): a pair of
    # same-phase suffixes 1,000 apart gives l = ((p+d)/2) rounded down to a multiple of d
    st, ln, cnt, f = rep[0]
    assert ln % 1000 == 0 and cnt >= 2
    cov = np.zeros(len(S), np.int8)
    for st, ln, cnt, f in rep:
        o = occ[f:f + cnt]
        for x in o:
            assert cov[x:x + ln].max() == 0
            cov[x:x + ln] = 1
        assert np.array_equal(S[o[0]:o[0] + min(ln, 4096)], S[o[-1]:o[-1] + min(ln, 4096)])


@pytest.mark.parametrize("B,C", [(16384, 256), (65536, 1024)])
def test_ruler_multiscale_batch(ctx, B, C):
    """SURVEY §8(f) NEXT 1, the paper's own workload shape: the
    slices the ruler schedule emits while a stream is ingested (sizes
    C * 2^j, capped at B) form one mixed-size batch for FindRepeats; every
    window of the batch equals the oracle on that slice.  B = 16,384 keeps
    every slice on the per-window on-chip path, B = 65,536 mixes in the
    global path."""
    S = gen.c3()[:4 * B]
    h = ctx.history(B, C)
    slices = []
    for pos in range(0, len(S), 3000):
        slices += h.ingest(dev(S[pos:pos + 3000]))
    assert slices == oracle.ruler_slices(0, len(S), C, B)
    wins = [S[b:e] for b, e in slices[-40:]]
    toks = np.concatenate(wins)
    off = np.cumsum([0] + [len(x) for x in wins]).astype(np.int64)
    assert len(set(len(x) for x in wins)) > 2  # mixed sizes
    rep, roff, occ = ctx.find_repeats_batched(dev(toks), off, 25)
    rep, roff, occ = rep.cpu().numpy(), roff.cpu().numpy(), occ.cpu().numpy()
    for w, x in enumerate(wins):
        want = oracle.find_repeats(x, 25, tier=1)
        got = rep[roff[w]:roff[w + 1]]
        assert np.array_equal(got[:, :3], want["repeats"][:, :3]), w
        for row, wrow in zip(got, want["repeats"]):
            assert np.array_equal(occ[row[3]:row[3] + row[2]], want["occ"][wrow[3]:wrow[3] + wrow[2]])


def test_batch_window_size_boundary(ctx):
    """Windows straddling the on-chip limit (16,383 / 16,384 / 16,385 ops)
    in one batch: the suffix arrays take the global path, candidate sorting
    the per-window path; tokens include 0 and 2^64-1.  Every window equals
    the oracle."""
    wins = []
    for i, n in enumerate((16383, 16384, 16385, 300)):
        S = gen.c3()[i * 20000:i * 20000 + n].copy()
        S[::997] = np.uint64((1 << 64) - 1)
        S[5::1013] = np.uint64(0)
        wins.append(S)
    tok = np.concatenate(wins)
    off = np.cumsum([0] + [len(x) for x in wins]).astype(np.int64)
    rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, 25)
    rep, roff, occ = rep.cpu().numpy(), roff.cpu().numpy(), occ.cpu().numpy()
    for w, S in enumerate(wins):
        want = oracle.find_repeats(S, 25, tier=1)
        got = rep[roff[w]:roff[w + 1]]
        assert np.array_equal(got[:, :3], want["repeats"][:, :3]), w
        for row, wrow in zip(got, want["repeats"]):
            assert np.array_equal(occ[row[3]:row[3] + row[2]], want["occ"][wrow[3]:wrow[3] + wrow[2]])
    sa, lcp = ctx.suffix_array_batched(dev(tok), off)
    sa, lcp = sa.cpu().numpy(), lcp.cpu().numpy()
    for w, S in enumerate(wins):
        want = oracle.sa_doubling(S)
        assert np.array_equal(sa[off[w]:off[w + 1]], want)
        assert np.array_equal(lcp[off[w]:off[w + 1]][:len(S) - 1], oracle.lcp_kasai(S, want))


@pytest.mark.parametrize("with_big_group", [False, True])
def test_batched_fused_select_equals_global(ctx, with_big_group, monkeypatch):
    """Batches of small windows take the fused per-window K5+K6 kernel
    (window_select.cu); APO_SELECT_GLOBAL=1 forces the global path (CandF,
    segment sort, RMQ heads, HeadF, unpack).  Repeats, offsets and
    occurrences must be identical, and equal to the oracle on sampled
    windows.  A window made of 200 copies of one block has sub-string groups
    of more than 64 members: the fused kernel hands the batch back to the
    global path."""
    tok, off, _, _ = gen.c4(seed=77, windows=40, window=4096, templates=8, with_streams=False)
    wins = [tok[off[w]:off[w + 1]] for w in range(len(off) - 1)]
    if with_big_group:
        wins.insert(7, np.tile(gen.random_string(5, 30, 1000), 200)[:6000])
    wins.append(gen.random_string(9, 16384, 3))  # a full-size window
    tok = np.concatenate(wins)
    off = np.cumsum([0] + [len(x) for x in wins]).astype(np.int64)
    for min_len in (5, 25):
        got = [t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
               for t in ctx.find_repeats_batched(dev(tok), off, min_len)]
        monkeypatch.setenv("APO_SELECT_GLOBAL", "1")
        ref = [t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
               for t in ctx.find_repeats_batched(dev(tok), off, min_len)]
        monkeypatch.delenv("APO_SELECT_GLOBAL")
        for a, b in zip(got, ref):
            assert np.array_equal(a, b)
        rep, roff, occ = got
        for w in (0, 7, len(wins) - 1):
            want = oracle.find_repeats(wins[w], min_len, tier=1)
            g = rep[roff[w]:roff[w + 1]]
            assert np.array_equal(g[:, :3], want["repeats"][:, :3]), w
            for row, wrow in zip(g, want["repeats"]):
                assert np.array_equal(occ[row[3]:row[3] + row[2]], want["occ"][wrow[3]:wrow[3] + wrow[2]])


def test_batched_edge_windows_fused_and_global(ctx, monkeypatch):
    """Empty, 1-, 2- and 3-op windows, a window of one repeated token and a
    full 16,384-op window in one batch: the fused per-window candidate stage
    and the global path give the oracle's repeats and occurrences."""
    wins = [np.zeros(0, np.uint64), gen.random_string(1, 1, 3), gen.random_string(2, 2, 1),
            gen.random_string(3, 3, 2), np.full(700, 5, np.uint64), gen.random_string(4, 25, 2),
            np.zeros(0, np.uint64), gen.random_string(6, 16384, 4)]
    tok = np.concatenate(wins)
    off = np.cumsum([0] + [len(x) for x in wins]).astype(np.int64)
    for mode in ("fused", "global"):
        if mode == "global":
            monkeypatch.setenv("APO_SELECT_GLOBAL", "1")
        for min_len in (1, 2, 25):
            rep, roff, occ = ctx.find_repeats_batched(dev(tok), off, min_len)
            rep, roff, occ = rep.cpu().numpy(), roff.cpu().numpy(), occ.cpu().numpy()
            for w in range(len(wins)):
                want = oracle.find_repeats(wins[w], min_len, tier=1)
                g = rep[roff[w]:roff[w + 1]]
                assert np.array_equal(g[:, :3], want["repeats"][:, :3]), (mode, min_len, w)
                for row, wrow in zip(g, want["repeats"]):
                    assert np.array_equal(occ[row[3]:row[3] + row[2]], want["occ"][wrow[3]:wrow[3] + wrow[2]])
