"""One GPU, N > 1 conditions: the union of the trace lists of C4 batches with
seeds 4 .. 3 + N, matched against seed 4's streams (rank 0's view at N).
Prints the trace count, dictionary misses and the match time (median)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = Context(0)
parts, offs = [], []
streams = soff = None
for r in range(N):
    tok, off, st, so = gen.c4(seed=4 + r, with_streams=(r == 0))
    d = torch.from_numpy(tok).cuda()
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    t, o = trie.traces()
    parts.append(t.cpu().numpy())
    offs.append(np.asarray(o))
    if r == 0:
        streams = torch.from_numpy(st).cuda()
        soff = so
    del trie, d
tt = np.concatenate(parts)
base = np.cumsum([0] + [len(p) for p in parts])
to = np.concatenate([offs[0]] + [o[1:] + base[i] for i, o in enumerate(offs) if i > 0]).astype(np.int64)
u = ctx.trie_build_traces(torch.from_numpy(tt).cuda(), to)
print("N", N, "union traces", u.info()[0], "tokens", len(tt), flush=True)
ts = []
for it in range(7):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hits, nall = ctx.match(u, streams, soff, mode=1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get("APO_TID_MODE", "-"), "match ms", round(sorted(ts)[3], 3), "hits", nall, "replays", hits.shape[0])
