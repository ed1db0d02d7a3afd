"""K9 phase breakdown (diagnostics): loads the APO_K9_PHASES=1 variant of
libapo (tools/variants/libapo_k9ph.so, built by
`python tools/build_variant.py k9ph 'window_sa.cu::#define APO_K9_PHASES 0::#define APO_K9_PHASES 1'`),
runs the C4 analysis batch and prints clock64 cycles per window per phase
(thread 0 of each CTA, so barrier waits are included in the phase they end)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["APO_LIB"] = os.path.join(ROOT, "tools", "variants", "libapo_k9ph.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
tok, off, _, _ = gen.c4(with_streams=False)
d = torch.from_numpy(tok).cuda()
f = ctx.lib.apo_debug_k9_phases
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
ctx.find_repeats_batched(d, off, 25)
torch.cuda.synchronize()
f(buf, 1)
ctx.find_repeats_batched(d, off, 25)
torch.cuda.synchronize()
f(buf, 1)
W = len(off) - 1
names = ["level0", "groups", "mm_build+store", "lsd_passes", "heads", "lcp", "output"]
tot = sum(buf[k] for k in range(7))
for k, nm in enumerate(names):
    print(f"{nm:16s} {buf[k] / W:12.0f} cycles/window  {100.0 * buf[k] / tot:5.1f} %")
print(f"rounds with 1 pass: {buf[9] / W:.2f}/window, 2 passes: {buf[10] / W:.2f}/window")
print(f"total {tot / W:.0f} cycles/window")
print(f"singleton slots: {buf[12] / max(buf[11], 1):.3f} of all slots over the head/group calls "
      f"(active fraction {1 - buf[12] / max(buf[11], 1):.3f})")
