"""torchrun: distributed suffix array of one window over all
ranks (DistSuffixArray, NCCL), timed with CUDA events (max over ranks), vs
the single-GPU apo_suffix_array of the same window on rank 0.
    python -m torch.distributed.run --nproc-per-node N tools/dsa_time.py [C5|C3]"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402
from paper_2406_18111_b200.dsa import CudaDsaOps, DistSuffixArray  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = Context(local)
S = gen.c5() if cfg == "C5" else gen.c3()
n = len(S)
a = [r * n // world for r in range(world + 1)]
blk = torch.from_numpy(S[a[rank]:a[rank + 1]].copy()).cuda()
d = DistSuffixArray(CudaDsaOps(ctx))
ts, tl = [], []
for it in range(3):
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    part, g = d.run(blk, n)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ts.append(float(t.item()))
    dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    lcp = d.lcp()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tl.append(float(t.item()))
# spot check against the single-GPU suffix array on rank 0
sizes = torch.tensor([part.numel()], device="cuda")
allsz = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
dist.all_gather(allsz, sizes)
out = {"config": cfg, "n": n, "ranks": world, "rounds": d.rounds, "sa_ms": ts, "lcp_ms": tl,
       "part_sizes": [int(x.item()) for x in allsz]}
if rank == 0:
    full = torch.from_numpy(S).cuda()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sa1, lcp1 = ctx.suffix_array(full, lcp=True)
    e1.record()
    torch.cuda.synchronize()
    out["single_gpu_sa_lcp_ms"] = e0.elapsed_time(e1)
    out["rank0_part_matches_single_gpu"] = bool(torch.equal(sa1[:part.numel()], part)) and bool(
        torch.equal(lcp1[:lcp.numel()], lcp[:lcp1.numel()][:lcp.numel()]))
    print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
