"""torchrun: the NVLink union (SM pull inside the hashing kernel) vs the
copy-engine pull (start/finish), alone and overlapped with apo_match_index;
CUDA-event ms, max over ranks."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402
from paper_2406_18111_b200.dist import TraceExchange  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = Context(local)
tok, off, st, so = gen.c4(seed=4 + rank)
d, ds = torch.from_numpy(tok).cuda(), torch.from_numpy(st).cuda()
rep, roff, occ = ctx.find_repeats_batched(d, off, 25)
trie = ctx.trie_build(d, off, rep, roff, 25, 0)
ex = TraceExchange(ctx)


def timed(f):
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = f()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), r


def sm_union():
    return ex.union(trie)


def ce_union():
    ex.start(trie)
    return ex.finish()


def index_only():
    return ctx.match_index(ds, so)


def overlapped():
    ex.start(trie)
    idx = ctx.match_index(ds, so)
    u = ex.finish()
    return idx, u


def publish_only():
    ex._publish(trie)


def pulled_build_only():
    ex.start(trie)
    ex.transport.wait()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    u = ex.finish()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for name, f in (("sm_union", sm_union), ("ce_union", ce_union), ("index_only", index_only),
                ("ce_union+index overlapped", overlapped), ("publish_only", publish_only)):
    ts = [timed(f)[0] for _ in range(4)]
    if rank == 0:
        print(f"{name}: {[round(t, 2) for t in ts]} ms", flush=True)
bt = torch.tensor([pulled_build_only() for _ in range(3)][-1], device="cuda")
dist.all_reduce(bt, op=dist.ReduceOp.MAX)
if rank == 0:
    print("union build from pulled lists (finish after wait)", round(float(bt.item()), 3), "ms", flush=True)
dist.destroy_process_group()
