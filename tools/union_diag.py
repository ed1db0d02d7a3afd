"""Single-GPU estimate of the N-rank union cost: build each rank's trace set,
then time traces() copy and trie_build_traces on the concatenation."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import gen
from paper_2406_18111_b200 import Context
ctx = Context(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
parts, offs = [], []
for r in range(N):
    tok, off, st, so = gen.c4(seed=4 + r, with_streams=False)
    d = torch.from_numpy(tok).cuda()
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    trie = ctx.trie_build(d, off, rep, roff, 25, 0)
    tt, to = trie.traces()
    parts.append(tt.clone()); offs.append(to)
    print(r, "traces", len(to) - 1, "tokens", int(to[-1]), "MB", int(to[-1]) * 8 / 1e6, flush=True)
    if r == 0:
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            tt2, to2 = trie.traces(); torch.cuda.synchronize()
            print("traces() ms", (time.perf_counter() - t0) * 1e3)
at = torch.cat(parts)
ao = np.concatenate([[0]] + [o[1:] + sum(int(x[-1]) for x in offs[:i]) for i, o in enumerate(offs)]).astype(np.int64)
for _ in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    u = ctx.trie_build_traces(at, ao); torch.cuda.synchronize()
    print("union build ms", (time.perf_counter() - t0) * 1e3, u.info())
ctx.profile(True)
torch.cuda.profiler.start()
u = ctx.trie_build_traces(at, ao); torch.cuda.synchronize()
torch.cuda.profiler.stop()
print([ctx.profile_read(k) for k in range(6)])
