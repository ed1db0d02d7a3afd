import sys, torch
sys.path.insert(0, ".")
from workloads import gen
from paper_2406_18111_b200 import Context
ctx = Context(0)
tok, off, _, _ = gen.c4(with_streams=False, windows=1024)
d = torch.from_numpy(tok).cuda()
for _ in range(2):
    sa, lcp = ctx.suffix_array_batched(d, off)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sa, lcp = ctx.suffix_array_batched(d, off); e1.record(); torch.cuda.synchronize()
print("suffix_array_batched 1024x16K:", e0.elapsed_time(e1), "ms")
