"""Matcher event counts on C4 (diagnostics): loads the APO_MATCH_STATS=1
variant (tools/variants/libapo_mstats.so, built by
`python tools/build_variant.py mstats 'trie.cu::#define APO_MATCH_STATS 0::#define APO_MATCH_STATS 1'`)
and prints the k_stream_match counters of one C4 match."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["APO_LIB"] = os.path.join(ROOT, "tools", "variants", "libapo_mstats.so")
sys.path.insert(0, ROOT)
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
      "mean", float(L.mean()))
f = ctx.lib.apo_debug_match_stats
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
f(buf, 1)
h = ctx.match(trie, ds, so, cap=480_000_000)
torch.cuda.synchronize()
f(buf, 1)
names = ["pairs", "sum_L", "bs_steps", "lcp_lr_steps", "cmp_calls", "reg_chunks", "glob_trips", "glob_chunks",
         "matched_pairs", "hits", "bucket_sum", "tokens_advanced"]
v = list(buf)
for i, n in enumerate(names):
    print(f"{n:16s} {v[i]:>16,d}  per pair {v[i] / max(v[0], 1):10.2f}")
print("hits (output)", h.shape[0])
