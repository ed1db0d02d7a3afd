"""Time apo_match mode 0 (MATCH_ALL) vs mode 1 (MATCH_ALL + REPLAY) on C4."""
import sys
import os
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
for mode in (0, 1, 0, 1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ctx.match(trie, ds, so, mode=mode, cap=480_000_000 if mode == 0 else None)
    e1.record()
    torch.cuda.synchronize()
    print(f"mode {mode}: {e0.elapsed_time(e1):.2f} ms", (r[0].shape[0], r[1]) if mode == 1 else r.shape[0])
