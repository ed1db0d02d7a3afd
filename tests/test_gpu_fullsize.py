"""Full-size parity: the CUDA path at BASELINE.json's full sizes, in the
launch configuration bench.py times, compared ELEMENT BY ELEMENT with the
tier-1 oracle (pinned to tier 0 in tests/test_oracle_pins.py, including at
full 16,384-op window size and on the full C2 window).

  * C4: every one of the 4,096 windows -- suffix array, LCP, repeats and
    occurrence lists (Alg. 2) -- the full union trace set
    (IngestCandidates) and MATCH_ALL hits of 16 full-size
    streams against the real union;
  * C5 at 2^26: the SA by its O(n) certificate (it is unique), the full LCP
    array vs Kasai, the full sorted candidate list with IDs and greedy
    decisions, and the repeats with occurrences.

The oracle runs on the host cores (its C calls release the GIL)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from workloads import gen

pytestmark = pytest.mark.gpu

MIN_LEN = 25
THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_18111_b200 import build
    build.build()
    from paper_2406_18111_b200 import Context
    return Context(0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64)).cuda()


@pytest.fixture(scope="module")
def c4():
    tok, off, st, so = gen.c4(with_streams=True)
    return tok, off, st, so


@pytest.fixture(scope="module")
def c4_gpu(ctx, c4):
    """The bench's launch configuration: one apo_find_repeats_batched over all
    4,096 windows, the trace set of its repeats, MATCH_ALL of every stream."""
    tok, off, st, so = c4
    d = dev(tok)
    rep, roff, occ = ctx.find_repeats_batched(d, off, MIN_LEN)
    sa, lcp = ctx.suffix_array_batched(d, off)
    trie = ctx.trie_build(d, off, rep, roff, MIN_LEN, 0)
    ttok, toff = trie.traces()
    hits = ctx.match(trie, dev(st), so)
    out = dict(rep=rep.cpu().numpy(), roff=roff.cpu().numpy(), occ=occ.cpu().numpy(), sa=sa.cpu().numpy(),
               lcp=lcp.cpu().numpy(), ttok=ttok.cpu().numpy(), toff=toff, nhits=int(hits.shape[0]))
    # hits of a sampled set of streams (rows are sorted by (stream, end, trace))
    W = len(off) - 1
    rng = gen.Rng(2024)
    sample = sorted({int(rng.below(W)) for _ in range(14)} | {0, W - 1})
    col = hits[:, 0].contiguous()
    q = torch.tensor(sample, dtype=torch.int32, device=col.device)
    lo = torch.searchsorted(col, q, right=False).tolist()
    hi = torch.searchsorted(col, q, right=True).tolist()
    out["sample"] = sample
    out["sample_hits"] = {s: hits[a:b].cpu().numpy() for s, a, b in zip(sample, lo, hi)}
    del hits, col
    torch.cuda.empty_cache()
    # REPLAY over every stream (apo_match mode 1: the hits are consumed on the device)
    rp, nh = ctx.match(trie, dev(st), so, mode=1)
    rp = rp.cpu().numpy()
    out["replay_nhits"] = nh
    out["sample_replays"] = {q: rp[rp[:, 0] == q] for q in sample}
    out["n_replays"] = len(rp)
    return out


@pytest.fixture(scope="module")
def c4_oracle(c4, c4_gpu):
    """Tier-1 oracle over every window on the host cores; compares SA/LCP in
    the workers and keeps the repeats + occurrences."""
    tok, off, _, _ = c4
    sa_g, lcp_g = c4_gpu["sa"], c4_gpu["lcp"]

    def one(w):
        S = tok[off[w]:off[w + 1]]
        r = oracle.find_repeats(S, MIN_LEN, tier=1)
        ok_sa = np.array_equal(sa_g[off[w]:off[w + 1]], r["sa"])
        g = lcp_g[off[w]:off[w + 1]]
        ok_lcp = np.array_equal(g[:len(S) - 1], r["lcp"]) and g[-1] == 0
        return ok_sa, ok_lcp, r["repeats"], r["occ"]

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(one, range(len(off) - 1)))
    return res


def test_c4_all_windows_sa_lcp(c4_oracle):
    bad_sa = [w for w, r in enumerate(c4_oracle) if not r[0]]
    bad_lcp = [w for w, r in enumerate(c4_oracle) if not r[1]]
    assert not bad_sa and not bad_lcp, (bad_sa[:10], bad_lcp[:10])


def test_c4_all_windows_repeats_and_occ(c4_gpu, c4_oracle):
    rep, roff, occ = c4_gpu["rep"], c4_gpu["roff"], c4_gpu["occ"]
    assert roff[0] == 0 and roff[-1] == len(rep)
    bad = []
    for w, (_, _, wrep, wocc) in enumerate(c4_oracle):
        got = rep[roff[w]:roff[w + 1]]
        if got.shape[0] != wrep.shape[0] or not np.array_equal(got[:, :3], wrep[:, :3]):
            bad.append(w)
            continue
        gocc = np.concatenate([occ[f:f + c] for _, _, c, f in got]) if len(got) else np.zeros(0, np.int32)
        if not np.array_equal(gocc, wocc):
            bad.append(w)
    assert not bad, bad[:10]


def test_c4_full_trace_set(c4, c4_gpu, c4_oracle):
    """The union trace set of all 4,096 windows' repeats, token for token and
    in id order (R19), vs the oracle's IngestCandidates."""
    tok, off, _, _ = c4
    srcs = [tok[off[w]:off[w + 1]] for w in range(len(off) - 1)]
    want_tok, want_off = oracle.traces_from_repeats_np(srcs, [r[2] for r in c4_oracle], MIN_LEN, 0)
    assert len(want_off) - 1 > 50000
    assert np.array_equal(c4_gpu["toff"], want_off)
    assert np.array_equal(c4_gpu["ttok"], want_tok)


def test_c4_sampled_full_streams_match(c4, c4_gpu):
    """MATCH_ALL of 16 full-size 16,384-op streams against the real ~66K-trace
    union, every (end, trace) by brute force (or_match_brute); the GPU rows
    come from the single full-batch apo_match call."""
    _, _, st, so = c4
    ttok, toff = c4_gpu["ttok"], c4_gpu["toff"]

    def one(q):
        S = st[so[q]:so[q + 1]]
        h, cnt = oracle.match_brute(S, np.array([0, len(S)], np.int64), ttok, toff)
        return q, h, cnt

    with ThreadPoolExecutor(min(THREADS, len(c4_gpu["sample"]))) as ex:
        res = list(ex.map(one, c4_gpu["sample"]))
    total = 0
    tlen = np.diff(toff).astype(np.int32)
    assert c4_gpu["replay_nhits"] == c4_gpu["nhits"]
    for q, h, cnt in res:
        got = c4_gpu["sample_hits"][q]
        assert got.shape[0] == cnt, q
        assert np.all(got[:, 0] == q)
        assert np.array_equal(got[:, 1:3], h[:, 1:]), q
        total += cnt
        # REPLAY of this stream (oracle on its own brute-force hits)
        want = oracle.replay(h, tlen)
        g = c4_gpu["sample_replays"][q]
        assert len(want) > 0 and len(g) == len(want), q
        assert np.array_equal(g[:, 1], want[:, 2]) and np.array_equal(g[:, 2], want[:, 3]), q
        assert np.array_equal(g[:, 3], want[:, 4]), q
    assert total > 0


def test_c5_full(ctx):
    """C5 at 2^26 ops (4-token alphabet, 1,000-op period, mean LCP ~ n/2,
    26 doubling rounds): every stage element by element."""
    S = gen.c5()
    n = len(S)
    d = dev(S)
    sa, lcp = ctx.suffix_array(d)
    sa_h, lcp_h = sa.cpu().numpy(), lcp.cpu().numpy()
    del sa, lcp
    assert oracle.sa_check(S, sa_h)                    # the SA is unique: certified == oracle SA
    want_lcp = oracle.lcp_kasai(S, sa_h)
    assert np.array_equal(lcp_h, want_lcp)
    del lcp_h
    c = ctx.candidates(d, MIN_LEN)
    g = {k: v.cpu().numpy() for k, v in c.items()}
    del c
    torch.cuda.empty_cache()
    cl, cs = oracle.candidates(sa_h, want_lcp, MIN_LEN)
    assert len(cl) == len(g["cand_len"]) and len(cl) > n          # ~2n candidates
    cl, cs, cid = oracle.sort_and_id_rmq_mt(S, sa_h, want_lcp, cl, cs, THREADS)
    assert np.array_equal(g["cand_len"], cl)
    assert np.array_equal(g["cand_start"], cs)
    assert np.array_equal(g["cand_id"], cid)
    keep = oracle.greedy_marks(n, cl, cs)
    assert np.array_equal(g["keep"], keep)
    want_rep, want_occ = oracle.repeats(cl, cs, cid, keep, 1)
    rep, occ = ctx.find_repeats(d, MIN_LEN)
    assert np.array_equal(rep.cpu().numpy(), want_rep)
    assert np.array_equal(occ.cpu().numpy(), want_occ)
