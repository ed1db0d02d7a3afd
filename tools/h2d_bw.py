"""Pinned host -> device copy bandwidth with 1, 2 and 4 concurrent streams
(diagnostics for the bench's e2e input upload)."""
import torch

n = 1 << 27  # 1 GiB of u64
src = torch.empty(n, dtype=torch.int64).pin_memory()
dst = torch.empty(n, dtype=torch.int64, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, st in enumerate(streams):
            st.wait_event(e0)
            with torch.cuda.stream(st):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        for st in streams:
            e1.wait(st) if False else None
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{k} stream(s): {n * 8 / ms / 1e6:.1f} GB/s ({ms:.1f} ms per GiB)", flush=True)
