"""torchrun: time the parts of TraceExchange's publish (host clock around
each part, device synchronised; max over ranks)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402
from paper_2406_18111_b200.dist import TraceExchange  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = Context(local)
tok, off, st, so = gen.c4(seed=4 + rank, with_streams=False)
d = torch.from_numpy(tok).cuda()
rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
trie = ctx.trie_build(d, off, rep, roff, 25, 0)
ex = TraceExchange(ctx)
ex.union(trie)
tr = ex.transport
for it in range(5):
    dist.barrier()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    T, n, _ = trie.info()
    all_sizes = ex.gather_sizes(T, n)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    tr.ensure(max(int(all_sizes[:, 0].max()), 1))
    tr.barrier()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    o = tr.publish(trie)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    offs = ex.gather_offsets(all_sizes, np.diff(o))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    tr.barrier()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    ms = torch.tensor(np.diff(t) * 1e3, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(it, "sizes / ensure+barrier / publish copy / offsets / barrier ms", [round(x, 3) for x in ms.tolist()],
              flush=True)
dist.destroy_process_group()
