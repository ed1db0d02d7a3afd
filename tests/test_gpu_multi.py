"""Two-GPU test of the NVLink union exchange (dist.TraceExchange): each rank
builds its own candidate trace set, the ranks exchange their lists through
symmetric memory and apo_trie_build_traces_multi pulls the peer's list over
NVLink; every rank must hold exactly the union trace set the oracle's
IngestCandidates builds from all ranks' repeats.  Skipped on one-GPU boxes
(the single-GPU multi-source build is covered in test_gpu_trie.py)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from workloads import gen
    from paper_2406_18111_b200 import Context
    from paper_2406_18111_b200.dist import TraceExchange
    ctx = Context(rank)
    tok, off, _, _ = gen.c4(seed=60 + rank, windows=8, window=3000, templates=4, with_streams=False)
    d = torch.from_numpy(tok).cuda()
    rep, roff, occ = ctx.find_repeats_batched(d, off, 8)
    trie = ctx.trie_build(d, off, rep, roff, 8, 0)
    ex = TraceExchange(ctx)
    for _ in range(2):  # the symmetric buffer is reused across steps
        u = ex.union(trie)
    ut, uo = u.traces()
    q.put((rank, ut.cpu().numpy().copy(), uo))
    dist.barrier()
    dist.destroy_process_group()


def test_trace_exchange_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    import oracle
    from workloads import gen
    world = 2
    port = _free_port()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, t, o = q.get(timeout=300)
        res[r] = (t, o)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # oracle: IngestCandidates over every rank's windows and repeats
    srcs, reps = [], []
    for r in range(world):
        tok, off, _, _ = gen.c4(seed=60 + r, windows=8, window=3000, templates=4, with_streams=False)
        for w in range(len(off) - 1):
            s = tok[off[w]:off[w + 1]]
            srcs.append(s)
            reps.append(oracle.find_repeats(s, 8, tier=1)["repeats"])
    wt, wo = oracle.traces_from_repeats(srcs, reps, 8, 0)
    for r in range(world):
        t, o = res[r]
        assert np.array_equal(o, wo) and np.array_equal(t, wt)
