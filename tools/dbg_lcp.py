import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from workloads import gen
from paper_2406_18111_b200 import Context
ctx = Context(0)
tok, off, st, so = gen.c4(seed=7, windows=64, window=4096, templates=16)
for name, arr, o in (("windows", tok, off), ("streams", st, so)):
    sa, lcp = ctx.suffix_array_batched(torch.from_numpy(arr).cuda(), o)
    sa, lcp = sa.cpu().numpy(), lcp.cpu().numpy()
    bad_sa = bad_lcp = 0
    for w in range(len(o) - 1):
        S = arr[o[w]:o[w+1]]
        want = oracle.sa_doubling(S)
        if not np.array_equal(sa[o[w]:o[w+1]], want):
            bad_sa += 1
            continue
        wl = oracle.lcp_kasai(S, want)
        got = lcp[o[w]:o[w+1]][:len(S)-1]
        if not np.array_equal(got, wl):
            bad_lcp += 1
            idx = np.nonzero(got != wl)[0]
            if bad_lcp <= 3: print(name, 'window', w, 'lcp mismatches', len(idx), 'first', idx[:5], got[idx[:5]], wl[idx[:5]])
    print(name, 'bad sa', bad_sa, 'bad lcp', bad_lcp, flush=True)
