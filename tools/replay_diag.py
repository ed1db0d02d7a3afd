"""Replay diagnostics on C4: per-stream slot counts (trace states a stream
needs), hits per stream, and apo_replay time on the MATCH_ALL hits."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
tok, off, st, so = gen.c4()
d, ds = torch.from_numpy(tok).cuda(), torch.from_numpy(st).cuda()
rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
trie = ctx.trie_build(d, off, rep, roff, 25, 0)
hits = ctx.match(trie, ds, so, full=True, cap=480_000_000)
q = hits[:, 0].long()
W = len(so) - 1
ms = torch.zeros(W, dtype=torch.int64, device="cuda").scatter_reduce(0, q, hits[:, 3].long() + 1, "amax")
nh = torch.bincount(q, minlength=W)
ends = torch.zeros(W, dtype=torch.int64, device="cuda")
for name, v in (("maxslot", ms), ("hits", nh)):
    a = v.cpu().numpy()
    print(name, "quantiles 0/50/90/99/100:", [int(np.quantile(a, x)) for x in (0, .5, .9, .99, 1)],
          ">2048:", int((a > 2048).sum()), ">4096:", int((a > 4096).sum()))
for _ in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ctx.replay(trie, hits, np.diff(so))
    e1.record()
    torch.cuda.synchronize()
    print(f"apo_replay: {e0.elapsed_time(e1):.2f} ms, {r.shape[0]} replays")
# the heaviest stream alone (its sequential walk bounds the kernel)
qs = int(torch.argmax(nh).item())
sel = hits[hits[:, 0] == qs].clone()
sel[:, 0] = 0
L = int(so[qs + 1] - so[qs])
for _ in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r1 = ctx.replay(trie, sel, [L])
    e1.record()
    torch.cuda.synchronize()
    print(f"heaviest stream {qs} alone ({sel.shape[0]} hits): {e0.elapsed_time(e1):.2f} ms, {r1.shape[0]} replays")
