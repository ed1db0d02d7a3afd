"""torchrun: time the parts of TraceExchange.union (max over ranks)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from workloads import gen
from paper_2406_18111_b200 import Context
from paper_2406_18111_b200.dist import TraceExchange
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
dev = ex.dev
u = None
for it in range(4):
    u = None  # free the previous union (its pooled blocks are reused, as in the bench)
    dist.barrier(); torch.cuda.synchronize()
    t = [time.perf_counter()]
    T, n, _ = trie.info()
    sizes = torch.tensor([n, T], dtype=torch.int64, device=dev)
    all_sizes = torch.empty(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_sizes, sizes)
    all_sizes = all_sizes.view(world, 2).cpu().numpy(); t.append(time.perf_counter())
    ex.hdl.barrier(channel=0); torch.cuda.synchronize(); t.append(time.perf_counter())
    _, o = trie.traces(out=ex.buf); torch.cuda.synchronize(); t.append(time.perf_counter())
    max_tr = max(int(all_sizes[:, 1].max()), 1)
    lens = torch.zeros(max_tr, dtype=torch.int64, device=dev); lens[:T] = torch.from_numpy(np.diff(o)).to(dev)
    gl = torch.empty(world * max_tr, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(gl, lens)
    gl = gl.view(world, max_tr).cpu().numpy(); t.append(time.perf_counter())
    ex.hdl.barrier(channel=0); torch.cuda.synchronize(); t.append(time.perf_counter())
    ptrs = ex.hdl.buffer_ptrs
    srcs = [(ptrs[r], np.concatenate([[0], np.cumsum(gl[r, :int(all_sizes[r, 1])])]).astype(np.int64)) for r in range(world)]
    t.append(time.perf_counter())
    u = ctx.trie_build_traces_multi(srcs); torch.cuda.synchronize(); t.append(time.perf_counter())
    ms = torch.tensor(np.diff(t) * 1e3, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(it, "sizes/barrier/copy/lens/barrier/host/build ms", [round(x, 3) for x in ms.tolist()], flush=True)
dist.destroy_process_group()
