"""How many (trace, stream) pairs and how large a search range would a
2-token (instead of 1-token) bucket give the matcher on C4?  (diagnostics)"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
tok, off, st, so = gen.c4()
d = torch.from_numpy(tok).cuda()
rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
trie = ctx.trie_build(d, off, rep, roff, 25, 0)
tt, to = trie.traces()
tt = tt.cpu().numpy()
L = np.diff(to)
# reversed trace's first two tokens = the trace's last two (forward order: t[L-2], t[L-1])
last = tt[to[1:] - 1]
prev = tt[to[1:] - 2]
S = len(so) - 1
# per stream unique unigrams / bigrams with their counts
mix = np.uint64(0x9E3779B97F4A7C15)


def key2(a, b):
    return (a * mix) ^ b


q = np.repeat(np.arange(S), np.diff(so))
uni_k, uni_c = np.unique(np.stack([q.astype(np.uint64), st]), axis=1, return_counts=True)
same = np.ones(len(st), bool)
same[so[1:] - 1] = False  # bigram (st[i], st[i+1]) inside one stream
bi = key2(st[:-1], st[1:])[same[:-1]]
bq = q[:-1][same[:-1]]
bi_k, bi_c = np.unique(np.stack([bq.astype(np.uint64), bi]), axis=1, return_counts=True)
# per token value: streams containing it and total occurrences
def pair_stats(trace_keys, stream_keys, stream_counts):
    tk, tcount = np.unique(trace_keys, return_counts=True)
    sk = stream_keys[1]
    order = np.argsort(sk, kind="stable")
    sk, sc = sk[order], stream_counts[order]
    ks, first = np.unique(sk, return_index=True)
    nstreams = np.diff(np.append(first, len(sk)))
    occ = np.add.reduceat(sc, first)
    idx = np.searchsorted(ks, tk)
    ok = (idx < len(ks)) & (ks[np.minimum(idx, len(ks) - 1)] == tk)
    pairs = (tcount[ok] * nstreams[idx[ok]]).sum()
    rng = (tcount[ok] * occ[idx[ok]]).sum()
    return int(pairs), float(rng) / max(int(pairs), 1)


p1, r1 = pair_stats(last, uni_k, uni_c)
p2, r2 = pair_stats(key2(prev, last), bi_k, bi_c)
print(f"traces {len(L)}: 1-token buckets: pairs {p1:,} mean range {r1:.1f}; 2-token: pairs {p2:,} mean range {r2:.1f}")
