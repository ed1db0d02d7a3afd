"""K1 microbenchmark: onesweep radix sort of (u64 key, u32 value) pairs."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2406_18111_b200 import Context  # noqa: E402


def main():
    ctx = Context(0)
    for n, bits in ((64 << 20, 41), (64 << 20, 54), (1 << 20, 41), (86 << 20, 54)):
        g = torch.Generator(device="cuda").manual_seed(1)
        base = torch.randint(0, 2**62, (n,), device="cuda", dtype=torch.int64, generator=g) & ((1 << bits) - 1)
        keys = base.clone().view(torch.uint64)
        vals = torch.arange(n, device="cuda", dtype=torch.int32)
        for _ in range(2):
            keys.copy_(base.view(torch.uint64)); vals.copy_(torch.arange(n, device="cuda", dtype=torch.int32))
            ctx.radix_sort(keys, vals, 0, bits)
        torch.cuda.synchronize()
        ctx.profile(True)
        reps = 5
        t = 0.0
        for _ in range(reps):
            keys.copy_(base.view(torch.uint64)); vals.copy_(torch.arange(n, device="cuda", dtype=torch.int32))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ctx.radix_sort(keys, vals, 0, bits); e1.record(); torch.cuda.synchronize()
            t += e0.elapsed_time(e1)
        ms, nl, by = ctx.profile_read(ctx.PROF_RADIX_PASS)
        hms, hn, _ = ctx.profile_read(ctx.PROF_RADIX_HIST)
        ctx.profile(False)
        ki = keys.view(torch.int64)  # keys < 2^63: signed compare is fine
        ok = bool((ki[1:] >= ki[:-1]).all().item())
        print(f"n={n:>10} bits={bits} sort {t/reps:7.3f} ms  passes {nl//reps} "
              f"pass avg {ms/nl*1e3:7.1f} us -> {by/nl/(ms/nl*1e-3)/1e9:7.1f} GB/s  hist {hms/max(hn,1)*1e3:6.1f} us  sorted={ok}")


if __name__ == "__main__":
    main()
