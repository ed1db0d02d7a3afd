"""Time apo_find_repeats on C3 (1M window) and C2 (65K) with the library
named by APO_LIB; prints medians and an output digest."""
import hashlib
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
out = []
for name, S in (("C3", gen.c3()), ("C2", gen.c2())):
    d = torch.from_numpy(S).cuda()
    ts = []
    for _ in range(9):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep, occ = ctx.find_repeats(d, 25)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = hashlib.sha1(rep.cpu().numpy().tobytes() + occ.cpu().numpy().tobytes()).hexdigest()[:12]
    out.append(f"{name} {sorted(ts)[4]:.3f} ms {h}")
print(os.path.basename(os.environ.get("APO_LIB", "libapo.so")), " | ".join(out))
