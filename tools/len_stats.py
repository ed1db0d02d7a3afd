"""Distinct candidate lengths per C4 window (diagnostics for the fused
candidate stage's length sort)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
tok, off, _, _ = gen.c4(with_streams=False)
W = len(off) - 1
ds, ms = [], []
for w in range(0, W, 41):
    c = ctx.candidates(torch.from_numpy(tok[off[w]:off[w + 1]]).cuda(), 25)
    L = c["cand_len"].cpu().numpy()
    ds.append(len(np.unique(L)))
    ms.append(len(L))
ds = np.array(ds)
print("windows", len(ds), "distinct lengths: median", int(np.median(ds)), "p90", int(np.quantile(ds, .9)),
      "max", int(ds.max()), "share <= 128:", float((ds <= 128).mean()), "candidates median", int(np.median(ms)))
