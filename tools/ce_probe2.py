"""Does cudaMemsetAsync wait behind a large host->device copy on another
stream? (diagnostics)"""
import time
import torch

n = 1 << 27
src = torch.empty(n, dtype=torch.int64).pin_memory()
dst = torch.empty(n, dtype=torch.int64, device="cuda")
cs = torch.cuda.Stream()
x = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
y = torch.empty(16, dtype=torch.int32, device="cuda")


def probe(name, fn):
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        dst.copy_(src, non_blocking=True)
    time.sleep(0.002)
    t0 = time.perf_counter()
    fn()
    torch.cuda.current_stream().synchronize()
    print(f"{name}: {(time.perf_counter() - t0) * 1e3:.2f} ms while a 1 GiB H2D is in flight", flush=True)
    torch.cuda.synchronize()


for _ in range(2):
    probe("memset 4 MB (zero_)", lambda: x.zero_())
    probe("memset 64 B (zero_)", lambda: y.zero_())
    probe("fill 4 MB (fill_ 7)", lambda: x.fill_(7))

import ctypes, glob, os  # noqa: E402
lib = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                         "libcudart.so*"))[0])
lib.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    probe("cudaMemsetAsync 4 MB", lambda: lib.cudaMemsetAsync(ctypes.c_void_p(x.data_ptr()), 0, 4 << 20, ctypes.c_void_p(st)))
    probe("cudaMemsetAsync 64 B", lambda: lib.cudaMemsetAsync(ctypes.c_void_p(y.data_ptr()), 0, 64, ctypes.c_void_p(st)))
    probe("cudaMemsetAsync 4 B", lambda: lib.cudaMemsetAsync(ctypes.c_void_p(y.data_ptr()), 0, 4, ctypes.c_void_p(st)))
