"""Are kernel launches / stream syncs slower while a large H2D copy runs on
another stream?  (diagnostics)"""
import time
import torch

n = 1 << 28
src = torch.empty(n, dtype=torch.int64).pin_memory()
dst = torch.empty(n, dtype=torch.int64, device="cuda")
cs = torch.cuda.Stream()
y = torch.zeros(16, dtype=torch.int32, device="cuda")
h = torch.empty(16, dtype=torch.int32).pin_memory()


def loop(k, sync_each):
    t0 = time.perf_counter()
    for _ in range(k):
        y.add_(1)
        if sync_each:
            torch.cuda.current_stream().synchronize()
    torch.cuda.current_stream().synchronize()
    return (time.perf_counter() - t0) * 1e6 / k


for busy in (False, True, False, True):
    torch.cuda.synchronize()
    if busy:
        with torch.cuda.stream(cs):
            dst.copy_(src, non_blocking=True)  # ~39 ms
        time.sleep(0.001)
    a = loop(200, True)
    b = loop(200, False)
    c0 = time.perf_counter()
    for _ in range(200):
        h.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    c = (time.perf_counter() - c0) * 1e6 / 200
    torch.cuda.synchronize()
    print(f"H2D busy={busy}: launch+sync {a:.1f} us, launch only {b:.1f} us, 64 B pinned D2H+sync {c:.1f} us", flush=True)
