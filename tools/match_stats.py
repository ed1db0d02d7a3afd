"""Matcher statistics on C4 (pairs, matched pairs, hits, trace lengths)."""
import os
import sys
os.environ["APO_DEBUG_STATS"] = "1"
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
tt, to = trie.traces()
L = np.diff(to)
print("traces", len(L), "len quantiles 0/50/90/99/100", [int(np.quantile(L, x)) for x in (0, .5, .9, .99, 1)],
      "mean", float(L.mean()), flush=True)
h = ctx.match(trie, ds, so, cap=480_000_000)
print("hits", h.shape[0])
