import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from workloads import gen
from paper_2406_18111_b200 import Context
ctx = Context(0)
for (W, win, seed) in [(10, 1200, 31), (64, 4096, 7), (128, 16384, 4)]:
    tok, off, st, so = gen.c4(seed=seed, windows=W, window=win, templates=min(W, 16))
    d = torch.from_numpy(tok).cuda()
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    tt, to = trie.traces()
    hits = ctx.match(trie, torch.from_numpy(st).cuda(), so).cpu().numpy()
    # per-stream oracle on a few streams
    tth = tt.cpu().numpy()
    bad = 0
    for q in list(range(0, W, max(1, W // 6)))[:6]:
        s1 = st[so[q]:so[q+1]]
        want, cnt = oracle.match_brute(s1, [0, len(s1)], tth, to)
        got = hits[hits[:, 0] == q].copy(); got[:, 0] = 0
        if not np.array_equal(got, want):
            bad += 1
            print('mismatch stream', q, len(got), len(want))
            gs = set(map(tuple, got.tolist())); ws = set(map(tuple, want.tolist()))
            print(' missing', list(ws - gs)[:5], ' extra', list(gs - ws)[:5])
    print(W, win, 'hits', len(hits), 'bad streams', bad, flush=True)
