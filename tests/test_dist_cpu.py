"""World-size-2 gloo test (CPU) of the multi-GPU exchange: every rank ends up
with the same union of candidate trace lists, in rank order."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_traces(rank):
    rng = np.random.default_rng(rank)
    T = 3 + rank * 2
    lens = rng.integers(1, 6, size=T)
    tok = rng.integers(0, 2**63, size=int(lens.sum()), dtype=np.int64).astype(np.uint64)
    tok[:1] = np.uint64((1 << 64) - 1)  # high bit survives the int64 view
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return tok, off


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_18111_b200.dist import gather_traces
    tok, off = _rank_traces(rank)
    at, ao = gather_traces(torch.from_numpy(tok.view(np.int64)).view(torch.uint64), off)
    q.put((rank, at.view(torch.int64).numpy().view(np.uint64).copy(), ao))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_traces_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, t, o = q.get(timeout=120)
        res[r] = (t, o)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_tok = np.concatenate([_rank_traces(r)[0] for r in range(world)])
    want_len = np.concatenate([np.diff(_rank_traces(r)[1]) for r in range(world)])
    for r in range(world):
        t, o = res[r]
        assert np.array_equal(t, want_tok)
        assert np.array_equal(np.diff(o), want_len)
