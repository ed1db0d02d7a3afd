"""REPLAY fast path: all C4 streams vs the heaviest streams alone (mode 1
minus mode 0), to see whether the decision walk's critical path is the
heaviest stream."""
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
h = ctx.match(trie, ds, so, full=True, cap=480_000_000)
nh = np.bincount(h[:, 0].cpu().numpy(), minlength=len(so) - 1)
del h
top = np.argsort(-nh)[:8]


def t(f):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for name, q in (("all", None), ("heaviest", top[:1]), ("top8", top)):
    if q is None:
        s_, o_ = ds, so
    else:
        parts = [st[so[i]:so[i + 1]] for i in q]
        s_ = torch.from_numpy(np.concatenate(parts)).cuda()
        o_ = np.cumsum([0] + [len(p) for p in parts]).astype(np.int64)
    m0 = t(lambda: ctx.match(trie, s_, o_, cap=480_000_000))
    m1 = t(lambda: ctx.match(trie, s_, o_, mode=1))
    print(f"{name}: mode0 {m0:.2f} ms, mode1 {m1:.2f} ms, replay ~{m1 - m0:.2f} ms", flush=True)
