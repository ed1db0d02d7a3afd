"""torchrun: TraceExchange (NVLink peer pull) vs gather_traces + build, same union; timings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from workloads import gen
from paper_2406_18111_b200 import Context
from paper_2406_18111_b200.dist import gather_traces, TraceExchange
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = Context(local)
small = len(sys.argv) > 1 and sys.argv[1] == "small"
tok, off, st, so = gen.c4(seed=4 + rank, with_streams=False, **(dict(windows=64, window=4096) if small else {}))
d = torch.from_numpy(tok).cuda()
rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
trie = ctx.trie_build(d, off, rep, roff, 25, 0)
ex = TraceExchange(ctx)
for it in range(5):
    dist.barrier(); torch.cuda.synchronize(); t0 = time.perf_counter()
    tt, to = trie.traces(); at, ao = gather_traces(tt, to); u1 = ctx.trie_build_traces(at, ao)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    dist.barrier(); torch.cuda.synchronize(); t2 = time.perf_counter()
    u2 = ex.union(trie)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    ms = torch.tensor([t1 - t0, t3 - t2], device="cuda") * 1e3
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    a, ao1 = u1.traces(); b, bo1 = u2.traces()
    same = torch.tensor([int(np.array_equal(ao1, bo1) and torch.equal(a, b))], device="cuda")
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(it, "nccl gather+build / peer-pull union ms", [round(x, 3) for x in ms.tolist()], "identical", bool(same.item()),
              "T", u2.info()[0], flush=True)
    del u1, u2
dist.destroy_process_group()
