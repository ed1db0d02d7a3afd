"""Time apo_find_repeats_batched on the C4 batch with the library named by
APO_LIB; prints the median of 7 and a digest of the output (variants must
print the same)."""
import hashlib
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
tok, off, _, _ = gen.c4(with_streams=False)
d = torch.from_numpy(tok).cuda()
ts = []
for _ in range(7):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
h = hashlib.sha1(rep.cpu().numpy().tobytes() + occ.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"{os.path.basename(os.environ.get('APO_LIB', 'libapo.so'))}: {sorted(ts)[3]:.3f} ms  digest {h}")
