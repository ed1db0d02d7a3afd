"""One GPU: the multi-source union build (apo_trie_build_traces_multi, as
TraceExchange.finish runs it on local copies of the peers' lists) of the
trace lists of C4 batches with seeds 4 .. 3 + N; CUDA-event ms (median)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = Context(0)
srcs = []
for r in range(N):
    tok, off, _, _ = gen.c4(seed=4 + r, with_streams=False)
    d = torch.from_numpy(tok).cuda()
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    t, o = trie.traces()
    srcs.append((t, np.asarray(o, dtype=np.int64)))
    del trie, d
ts = []
for it in range(7):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    u = ctx.trie_build_traces_multi(srcs)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    info = u.info()
    del u
print("N", N, "union", info, "build ms", round(sorted(ts)[3], 3), [round(x, 2) for x in ts])
