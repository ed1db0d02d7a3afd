"""Distributed suffix array + LCP on the GPU:
DistSuffixArray with the library's apo_dsa_* steps and K1, NCCL collectives.  One process
(world 1: the doubling loop, keys, heads and scatter kernels) and, on a box
with two GPUs, two ranks (the sample-sort exchange over NVLink).  Expected:
the oracle's suffix array (tier 0 naive sort on small inputs; the O(n)
Burkhardt-Kaerkkaeinen certificate + tier-1 doubling on large ones)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from workloads import gen

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cases():
    return [("random3", gen.random_string(11, 5000, 3)), ("periodic", gen.periodic(12, 4099, 37, 6, noise=0.02)),
            ("fib", gen.fibonacci_word(3000)), ("highbit", gen.high_bit_string(13, 2000, 9)),
            ("one", gen.random_string(14, 1, 2)),
            ("c5_1m", gen.c5(n=1 << 20)), ("c3", gen.c3())]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2406_18111_b200 import Context
    from paper_2406_18111_b200.dsa import CudaDsaOps, DistSuffixArray
    ctx = Context(rank)
    out = []
    for name, S in _cases():
        n = len(S)
        a = [r * n // world for r in range(world + 1)]
        blk = torch.from_numpy(S[a[rank]:a[rank + 1]].copy()).cuda()
        d = DistSuffixArray(CudaDsaOps(ctx))
        part, g = d.run(blk, n)
        out.append((g, part.cpu().numpy().copy(), d.rounds, d.lcp().cpu().numpy().copy()))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _run(world):
    import torch.multiprocessing as mp
    port = _free_port()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out = q.get(timeout=600)
        res[r] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for i, (name, S) in enumerate(_cases()):
        parts = sorted(((res[r][i][0], res[r][i][1], res[r][i][3]) for r in range(world)), key=lambda x: x[0])
        sa = np.concatenate([p for _, p, _ in parts]).astype(np.int64)
        assert [g for g, _, _ in parts] == list(np.cumsum([0] + [len(p) for _, p, _ in parts[:-1]])), name
        lcp = np.concatenate([c for _, _, c in parts]).astype(np.int64)
        if len(S) <= 5000:
            assert np.array_equal(sa, oracle.sa_naive(S)), name
            want = oracle.lcp_naive(S, sa)
        else:
            assert oracle.sa_check(S, sa), name  # the suffix array is unique: certified == oracle
            want = oracle.lcp_kasai(S, sa)
        assert np.array_equal(lcp, np.append(np.asarray(want, dtype=np.int64), 0)), name


def test_dist_suffix_array_one_gpu():
    _run(1)


def test_dist_suffix_array_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    _run(2)
