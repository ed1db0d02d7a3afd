"""TraceFinder on the GPU: the history ring, the
ruler schedule, analyses running asynchronously on a side stream
(StreamAnalyzer: its own context and CUDA stream, a worker thread), and
ingestion of each analysis into the device trace set (TraceSetBuilder:
apo_trie_build + apo_trie_build_traces_multi) at the agreed op count
(reading R25).  Expected: the union of the oracle's repeat
contents over every slice the oracle's ruler schedule analyses, in id order
(length desc, lexicographic asc); ingestion points = launch + delay."""
import numpy as np
import pytest
import torch

import oracle
from oracle.ruler import ruler_slices
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,C,delay,seed", [(4096, 256, 100, 1), (16384, 1000, 3000, 2), (2048, 128, 1, 3)])
def test_trace_finder_matches_oracle(B, C, delay, seed):
    from paper_2406_18111_b200 import build
    build.build()
    from paper_2406_18111_b200 import Context
    from paper_2406_18111_b200.finder import StreamAnalyzer, TraceFinder, TraceSetBuilder
    min_len = 10
    ctx = Context(0)
    S = np.concatenate([gen.periodic(seed, 9000, 41, 30, noise=0.05),
                        gen.periodic(seed + 10, 8000, 173, 60, noise=0.02)])
    an = StreamAnalyzer(0, min_len)
    fi = TraceFinder(ctx.history(B, C), an, TraceSetBuilder(ctx, min_len), delay=delay)
    d = torch.from_numpy(S).cuda()
    rng = np.random.default_rng(seed)
    pos = 0
    while pos < len(S):
        k = int(rng.integers(1, 3 * C))
        fi.ingest(d[pos:pos + k])
        pos += k
    events = list(fi.events)
    fi.flush()
    an.close()
    # oracle: every slice the schedule analyses, FindRepeats, IngestCandidates
    sl = ruler_slices(0, len(S), C, B)
    reps = [oracle.find_repeats(S[b:e], min_len, tier=1)["repeats"] for b, e in sl]
    wt, wo = oracle.traces_from_repeats([S[b:e] for b, e in sl], reps, min_len, 0)
    gt, go = fi.trie.traces()
    assert np.array_equal(go, wo) and np.array_equal(gt.cpu().numpy(), wt)
    # single replica: nobody else to wait for; ingestion points are launch +
    # the delay in force at launch (doubled after every wait)
    launches = [e for b, e in sl]
    d_ = delay
    hist = [(0, delay)]  # (op count, delay in force from then on)
    for i, (count, anyw, size, dl, k0) in enumerate(events):
        assert k0 == launches[i]
        at_launch = [dd for c, dd in hist if c < k0][-1]  # ingestions at k0 follow its launch
        assert count == k0 + at_launch
        if anyw:
            d_ *= 2
        assert dl == d_
        hist.append((count, dl))


def test_batch_pipeline_equals_serial():
    """BatchPipeline (analysis of batch k+1 on a side stream overlapping the
    trace set, MATCH_ALL and REPLAY of batch k) returns exactly what the
    same calls return one after the other, batch by batch."""
    from paper_2406_18111_b200 import Context
    from paper_2406_18111_b200.finder import BatchPipeline
    ctx = Context(0)
    batches = []
    for seed in (41, 42, 43):
        tok, off, st, so = gen.c4(seed=seed, windows=24, window=4096, templates=6)
        batches.append((torch.from_numpy(tok).cuda(), off, torch.from_numpy(st).cuda(), so, None))
    want = []
    for tok, off, st, so, _ in batches:
        rep, roff, occ = ctx.find_repeats_batched(tok, off, 25)
        trie = ctx.trie_build(tok, off, rep, roff, 25, 0)
        rp, nall = ctx.match(trie, st, so, mode=1)
        want.append((rep.cpu(), roff.cpu(), occ.cpu(), rp.cpu(), nall))
    pipe = BatchPipeline(ctx, 25)
    for rnd in range(2):  # buffers are reused across runs
        got = []
        for rep, roff, occ, counts, (rp, nall) in pipe.run(batches):
            r, o = (int(x) for x in counts.tolist())
            got.append((rep[:r].cpu(), roff.cpu(), occ[:o].cpu(), rp.cpu(), nall))
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert all(torch.equal(a, b) for a, b in zip(g[:4], w[:4])) and g[4] == w[4]
    pipe.close()
