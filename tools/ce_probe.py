"""Do device->host copies wait behind a large host->device copy on another
stream?  (diagnostics: 8-byte and 25 MB D2H, pinned and pageable, and a
D2D copy, each timed while a 1 GiB H2D runs)"""
import time
import torch

n = 1 << 27
src = torch.empty(n, dtype=torch.int64).pin_memory()
dst = torch.empty(n, dtype=torch.int64, device="cuda")
cs = torch.cuda.Stream()
s = torch.cuda.current_stream()
small_d = torch.ones(1, dtype=torch.int64, device="cuda")
big_d = torch.ones(25 << 20 >> 3, dtype=torch.int64, device="cuda")
small_h = torch.empty(1, dtype=torch.int64).pin_memory()
big_h = torch.empty(25 << 20 >> 3, dtype=torch.int64).pin_memory()
d2 = torch.empty_like(big_d)


def probe(name, fn):
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        dst.copy_(src, non_blocking=True)
    time.sleep(0.002)  # the DMA is under way
    t0 = time.perf_counter()
    fn()
    torch.cuda.current_stream().synchronize()
    t = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    print(f"{name}: {t:.2f} ms while a 1 GiB H2D is in flight", flush=True)


for _ in range(2):
    probe("8 B D2H pinned", lambda: small_h.copy_(small_d, non_blocking=True))
    probe("25 MB D2H pinned", lambda: big_h.copy_(big_d, non_blocking=True))
    probe("25 MB D2H pageable", lambda: big_d.cpu())
    probe("25 MB D2D", lambda: d2.copy_(big_d, non_blocking=True))
    probe("8 B H2D pinned", lambda: small_d.copy_(small_h, non_blocking=True))
