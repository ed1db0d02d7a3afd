"""Does the nvidia-smi clock sampler perturb BatchPipeline?  Times K
pipelined C4 batches three times without and three times with the sampler."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402
from paper_2406_18111_b200.finder import BatchPipeline  # noqa: E402
import bench  # noqa: E402

ctx = Context(0)
tok, off, st, so = gen.c4()
d, ds = torch.from_numpy(tok).cuda(), torch.from_numpy(st).cuda()
pipe = BatchPipeline(ctx, 25)
K = 5
for _ in pipe.run([(d, off, ds, so, None)] * 2):
    pass
for sampler in (False, True, False, True, False, True):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cm = bench.ClockSampler(0) if sampler else None
    if cm:
        cm.__enter__()
    e0.record()
    for _ in pipe.run([(d, off, ds, so, None)] * K):
        pass
    e1.record()
    torch.cuda.synchronize()
    if cm:
        cm.__exit__(None, None, None)
    print(f"sampler={sampler}: {e0.elapsed_time(e1) / K:.2f} ms/batch", flush=True)
