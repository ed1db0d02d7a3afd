"""BatchPipeline vs the same calls back to back (C4, K batches each),
alternated three times."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402
from paper_2406_18111_b200.finder import BatchPipeline  # noqa: E402

ctx = Context(0)
tok, off, st, so = gen.c4()
d, ds = torch.from_numpy(tok).cuda(), torch.from_numpy(st).cuda()
pipe = BatchPipeline(ctx, 25)
K = 5


def serial():
    for _ in range(K):
        rep, roff, occ, cnt = ctx.find_repeats_batched(d, off, 25, sync=False)
        trie = ctx.trie_build(d, off, rep, roff, 25, 0)
        ctx.match(trie, ds, so, mode=1)


def piped():
    for _ in pipe.run([(d, off, ds, so, None)] * K):
        pass


for f in (serial, piped):
    f()
for rnd in range(3):
    for name, f in (("serial", serial), ("pipelined", piped)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / K:.2f} ms/batch", flush=True)
