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


# ---------------------------------------------------------------------------
# TraceExchange.union -- the code bench.py runs at N > 1 -- on CPU: the same
# collectives (sizes, trace lengths), buffer sizing and barrier order, with a
# host shared-memory transport standing in for NVLink-mapped symmetric
# memory (each rank reads its peer's buffer in place, as the kernel does over
# NVLink) and a CPU builder standing in for apo_trie_build_traces_multi
# (test infrastructure: merge identical contents, ids in (length desc,
# lexicographic) order, reading R19).

class _HostTrie:
    def __init__(self, tok, off):
        self.tok, self.off = tok, off

    def info(self):
        return len(self.off) - 1, int(self.off[-1]), int(np.diff(self.off).max(initial=0))

    def traces(self, out=None):
        n = int(self.off[-1])
        out[:n] = self.tok.view(np.int64)
        return out[:n], self.off


class _ShmTransport:
    """One shared-memory segment per rank and generation; peers attach by
    name after a barrier (regrowth is collective, like symmetric memory)."""

    def __init__(self, tag, rank, world):
        self.tag, self.rank, self.world = tag, rank, world
        self.gen = 0
        self.cap = 0
        self.own = None
        self.peers = []
        self.log = []

    def ensure(self, need):
        from multiprocessing import shared_memory
        if need <= self.cap:
            return
        self.gen += 1
        cap = int(need * 1.25) + 16
        self.own = shared_memory.SharedMemory(name=f"apo_{self.tag}_{self.gen}_{self.rank}", create=True,
                                              size=cap * 8)
        dist.barrier()
        self.peers = [self.own if r == self.rank else
                      shared_memory.SharedMemory(name=f"apo_{self.tag}_{self.gen}_{r}") for r in range(self.world)]
        self.cap = cap
        self.log.append(("ensure", cap))

    def barrier(self):
        self.log.append(("barrier",))
        dist.barrier()

    def publish(self, trie):
        buf = np.ndarray((self.cap,), dtype=np.int64, buffer=self.own.buf)
        self.log.append(("publish",))
        return trie.traces(out=buf)[1]

    def sources(self):
        return [np.ndarray((self.cap,), dtype=np.uint64, buffer=p.buf) for p in self.peers]

    def close(self):
        for p in self.peers:
            p.close()
        dist.barrier()
        self.own.unlink()


class _CpuBuilder:
    device = "cpu"

    def trie_build_traces_multi(self, sources):
        seen = set()
        for buf, off in sources:
            for t in range(len(off) - 1):
                seen.add(tuple(int(x) for x in buf[off[t]:off[t + 1]]))
        return sorted(seen, key=lambda c: (-len(c), c))


def _exchange_lists(rank, step):
    rng = np.random.default_rng(100 * step + rank)
    T = 4 + 3 * rank + 50 * step  # step 1 outgrows the step-0 buffers
    lens = rng.integers(1, 9, size=T)
    tok = rng.integers(0, 5, size=int(lens.sum()), dtype=np.int64).astype(np.uint64)
    tok[::7] = np.uint64((1 << 64) - 3)  # values above 2^63 survive the int64 buffer view
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return tok, off


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_18111_b200.dist import TraceExchange
    tr = _ShmTransport(port, rank, world)
    ex = TraceExchange(_CpuBuilder(), transport=tr)
    out = []
    for step in range(3):
        tok, off = _exchange_lists(rank, min(step, 1))
        out.append((ex.union(_HostTrie(tok, off)), ex.last_pulled_tokens))
    q.put((rank, out, tr.log))
    tr.close()
    dist.destroy_process_group()


def test_trace_exchange_union_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, log = q.get(timeout=120)
        res[r] = (out, log)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for step in range(3):
        lists = [_exchange_lists(r, min(step, 1)) for r in range(world)]
        want = sorted({tuple(int(x) for x in tok[off[t]:off[t + 1]]) for tok, off in lists
                       for t in range(len(off) - 1)}, key=lambda c: (-len(c), c))
        for r in range(world):
            got, pulled = res[r][0][step]
            assert got == want
            assert pulled == sum(int(lists[p][1][-1]) for p in range(world) if p != r)
    for r in range(world):
        log = res[r][1]
        # buffers grow only when a list outgrows them; every publish sits between two barriers
        assert [e for e in log if e[0] == "ensure"] and sum(e[0] == "ensure" for e in log) == 2
        for k, e in enumerate(log):
            if e[0] == "publish":
                assert log[k - 1][0] == "barrier" and log[k + 1][0] == "barrier"
