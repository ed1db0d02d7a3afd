import sys, torch
sys.path.insert(0, ".")
from paper_2406_18111_b200 import Context
ctx = Context(0)
n, bits = 64 << 20, 41
k = (torch.randint(0, 2**62, (n,), device="cuda", dtype=torch.int64) & ((1 << bits) - 1)).view(torch.uint64)
v = torch.arange(n, device="cuda", dtype=torch.int32)
for _ in range(2):
    ctx.radix_sort(k, v, 0, bits)
torch.cuda.synchronize()
