"""torchrun diagnostic: per-rank trace set, then time traces() / gather / union build."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from workloads import gen
from paper_2406_18111_b200 import Context
from paper_2406_18111_b200.dist import gather_traces
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = Context(local)
tok, off, st, so = gen.c4(seed=4 + rank, with_streams=False)
d = torch.from_numpy(tok).cuda()
rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
trie = ctx.trie_build(d, off, rep, roff, 25, 0)
for it in range(5):
    dist.barrier(); torch.cuda.synchronize()
    t = [time.perf_counter()]
    tt, to = trie.traces(); torch.cuda.synchronize(); t.append(time.perf_counter())
    at, ao = gather_traces(tt, to); torch.cuda.synchronize(); t.append(time.perf_counter())
    u = ctx.trie_build_traces(at, ao); torch.cuda.synchronize(); t.append(time.perf_counter())
    ms = torch.tensor(np.diff(t) * 1e3, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(it, "traces/gather/union ms (max over ranks)", [round(x, 3) for x in ms.tolist()], "bytes", int(ao[-1]) * 8, flush=True)
# collective alone on pre-padded buffers, and the uneven (broadcast-based) variant into views
n = int(to[-1])
sizes = [None] * world
dist.all_gather_object(sizes, n)
mx = max(sizes)
pt = torch.zeros(mx, dtype=torch.int64, device="cuda"); pt[:n] = tt.view(torch.int64)
gt = torch.empty(world * mx, dtype=torch.int64, device="cuda")
big = torch.empty(sum(sizes), dtype=torch.int64, device="cuda")
views = list(torch.split(big, sizes))
src = tt.view(torch.int64)
for it in range(4):
    dist.barrier(); torch.cuda.synchronize(); t0 = time.perf_counter()
    dist.all_gather_into_tensor(gt, pt); torch.cuda.synchronize(); t1 = time.perf_counter()
    dist.all_gather(views, src); torch.cuda.synchronize(); t2 = time.perf_counter()
    ms = torch.tensor([t1 - t0, t2 - t1], device="cuda") * 1e3
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print("all_gather_into_tensor / uneven all_gather ms", [round(x, 3) for x in ms.tolist()], flush=True)
ok = torch.equal(big[sum(sizes[:rank]):sum(sizes[:rank + 1])], src)
print(rank, "uneven view ok", ok, flush=True)
dist.destroy_process_group()
