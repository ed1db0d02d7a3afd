"""World-size-2 gloo test (CPU) of the multi-GPU exchange: every rank ends up
with the same union of candidate trace lists, in rank order."""
import os
import socket

import numpy as np
import pytest
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

    def pull(self, ntok):  # the copy-engine pull: peers' lists copied out, own list in place
        self.log.append(("pull",))
        return [np.ndarray((self.cap,), dtype=np.uint64, buffer=p.buf)[:n].copy() if r != self.rank
                else np.ndarray((self.cap,), dtype=np.uint64, buffer=p.buf) for r, (p, n) in enumerate(zip(self.peers, ntok))]

    def wait(self):
        self.log.append(("wait",))

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
    for step in range(4):
        tok, off = _exchange_lists(rank, min(step, 1))
        if step < 3:
            out.append((ex.union(_HostTrie(tok, off)), ex.last_pulled_tokens))
        else:  # the overlapped form bench.py uses: start (pull), other work, finish
            ex.start(_HostTrie(tok, off))
            out.append((ex.finish(), ex.last_pulled_tokens))
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
    for step in range(4):
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


# ---------------------------------------------------------------------------
# TraceFinder ingestion agreement (reading R25) on two
# gloo ranks whose analyses finish at different times: both ranks must
# ingest the same analyses at the same op counts and grow the agreed delay
# together whenever either one had to wait.

class _HostHistory:
    """The history's schedule on the host: apo_ruler_slices (pure host
    function of libapo) over a numpy token list (test stand-in for the
    device ring)."""

    def __init__(self, B, C):
        self.capacity_B, self.scale_C = B, C
        self.tok = np.zeros(0, np.uint64)

    @property
    def count(self):
        return len(self.tok)

    def ingest(self, piece):
        from paper_2406_18111_b200.apo import ruler_slices
        k0 = self.count
        self.tok = np.concatenate([self.tok, piece])
        return ruler_slices(k0, len(piece), self.scale_C, self.capacity_B)

    def window(self, b, e):
        return self.tok[b:e]


class _ScriptedFuture:
    def __init__(self, clock, ready_at, win):
        self.clock, self.ready_at, self.win = clock, ready_at, win
        self.waited = False

    def done(self):
        return self.clock() >= self.ready_at

    def result(self):
        if not self.done():
            self.waited = True  # the replica blocks here until the analysis completes
        return self.win


class _ScriptedAnalyzer:
    """Analysis i of this rank completes lag(i) ops after its launch."""

    def __init__(self, lag):
        self.lag = lag
        self.n = 0
        self.clock = None

    def submit(self, win, ready):
        f = _ScriptedFuture(self.clock, self.clock() + self.lag(self.n), win)
        self.n += 1
        return f


class _SetBuilder:
    """IngestCandidates on the host for the test: the analysis's repeat
    contents by the oracle, the set union."""

    def from_analysis(self, win):
        import oracle
        rep = oracle.find_repeats(np.asarray(win), 5, tier=1)["repeats"]
        return {tuple(int(x) for x in win[s:s + l]) for s, l in rep[:, :2]}

    def union(self, a, b):
        return a | b

    @staticmethod
    def size(t):
        return 0 if t is None else len(t)


def _agree_stream():
    from workloads import gen
    return np.concatenate([gen.periodic(3, 3000, 37, 24, noise=0.1), gen.periodic(4, 3000, 53, 24, noise=0.1)])


def _finder_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_18111_b200.finder import TraceFinder
    # rank 1's first analyses are slow (1,300 ops), later ones fast
    an = _ScriptedAnalyzer((lambda i: 10) if rank == 0 else (lambda i: 1300 if i < 3 else 10))
    fi = TraceFinder(_HostHistory(1024, 128), an, _SetBuilder(), delay=128)
    an.clock = lambda: fi.count
    S = _agree_stream()
    rng = np.random.default_rng(rank)  # ranks feed the same ops in different piece sizes
    pos = 0
    while pos < len(S):
        k = int(rng.integers(1, 700))
        fi.ingest(S[pos:pos + k])
        pos += k
    q.put((rank, fi.events, sorted(fi.trie) if fi.trie else []))
    dist.destroy_process_group()


def test_trace_finder_agreement_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_finder_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, ev, tr = q.get(timeout=180)
        res[r] = (ev, tr)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ev0, tr0 = res[0]
    ev1, tr1 = res[1]
    assert ev0 == ev1 and tr0 == tr1 and len(ev0) > 10
    # the delay doubles exactly when someone waited, and only then
    d = 128
    for count, anyw, size, delay, k0 in ev0:
        if anyw:
            d *= 2
        assert delay == d
    assert any(e[1] for e in ev0) and not ev0[-1][1]
    # rank 1's three slow analyses (1,300 ops > every delay in force) are the
    # only waits; after them the agreed delay stays at 128 * 2^3
    assert sum(e[1] for e in ev0) == 3 and all(e[1] for e in ev0[:3]) and ev0[-1][3] == 1024
    # every analysis is ingested exactly delay-at-launch ops after its launch
    # (launch points: multiples of C = 128), in launch order
    counts = [e[0] for e in ev0]
    assert counts == sorted(counts)


# ---------------------------------------------------------------------------
# Distributed suffix array: DistSuffixArray's
# orchestration -- the rank2 shift exchange, the sample sort (samples,
# splitters, all-to-all), the head/rank carry across rank boundaries, the
# return to the position owners -- on 2 and 3 gloo ranks, with numpy
# stand-ins for the library steps (test infrastructure: each mirrors the
# documented contract of its apo_dsa_* call).  Expected: the oracle's suffix
# array (naive comparison sort, tier 0).

class _NpDsaOps:
    device = torch.device("cpu")

    def empty(self, n, dtype):
        return torch.empty(max(int(n), 0), dtype=dtype)

    def sort(self, keys, vals, bits):
        k = keys.view(torch.int64).numpy().view(np.uint64)
        mk = k & np.uint64((1 << bits) - 1) if bits < 64 else k
        o = np.argsort(mk, kind="stable")
        kk, vv = k[o].copy(), vals.numpy()[o].copy()
        keys.view(torch.int64).numpy()[:] = kk.view(np.int64)
        vals.numpy()[:] = vv

    def keys(self, rank, rank2, base, n):
        m = rank.numel()
        r2 = np.zeros(m, np.uint64)
        r2[:rank2.numel()] = rank2.numpy().astype(np.uint64)
        k = rank.numpy().astype(np.uint64) * np.uint64(n + 1) + r2
        return torch.from_numpy(k.view(np.int64)).view(torch.uint64), torch.arange(base, base + m, dtype=torch.int32)

    def samples(self, keys, vals, s):
        m = keys.numel()
        k = keys.view(torch.int64).numpy().view(np.uint64)
        v = vals.numpy()
        idx = [min((j * m) // s + (m // s) // 2, m - 1) for j in range(s)]
        sk = np.array([k[i] if m else np.uint64((1 << 64) - 1) for i in idx], dtype=np.uint64)
        sv = np.array([v[i] if m else -1 for i in idx], dtype=np.int32)
        return torch.from_numpy(sk.view(np.int64)).view(torch.uint64), torch.from_numpy(sv)

    def split(self, keys, vals, spk, spv, g):
        k = [int(x) for x in keys.view(torch.int64).numpy().view(np.uint64)]
        v = [int(x) & 0xffffffff for x in vals.numpy()]
        sp = list(zip([int(x) for x in spk.view(torch.int64).numpy().view(np.uint64)],
                      [int(x) & 0xffffffff for x in spv.numpy()]))
        bounds = [0] + [sum(1 for p in zip(k, v) if p < s) for s in sp] + [len(k)]
        return torch.tensor([max(bounds[d + 1] - bounds[d], 0) for d in range(g)], dtype=torch.int64)

    def heads(self, keys, prev_key, has_prev, gbase, carry):
        k = [int(x) for x in keys.view(torch.int64).numpy().view(np.uint64)]
        rank, cur, h, last = [], carry, 0, -1
        for i, x in enumerate(k):
            if (i == 0 and (not has_prev or x != prev_key)) or (i > 0 and x != k[i - 1]):
                cur = gbase + i
                h += 1
                last = cur
            rank.append(cur + 1)
        return torch.tensor(rank, dtype=torch.int32), h, last

    def scatter(self, pos, rank_in, base, rank):
        rank.numpy()[pos.numpy() - base] = rank_in.numpy()

    def lcp_requests(self, a, b, l, n):
        pa = np.minimum(a.numpy().astype(np.int64) + l.numpy(), n)
        pb = np.minimum(b.numpy().astype(np.int64) + l.numpy(), n)
        k = np.empty(2 * len(pa), np.uint64)
        k[0::2], k[1::2] = pa, pb
        return torch.from_numpy(k.view(np.int64)).view(torch.uint64), torch.arange(2 * len(pa), dtype=torch.int32)

    def gather(self, pos, base, rank):
        return torch.from_numpy(rank.numpy()[pos.numpy() - base].copy())

    def lcp_update(self, resp, req, nvalid, step, by_req, l):
        br = by_req.numpy()
        br[req.numpy()[:nvalid]] = resp.numpy()[:nvalid]
        x, y = br[0::2], br[1::2]
        l.numpy()[(x == y) & (x != -1)] += step
        br[0::2], br[1::2] = -1, -2


def _dsa_strings():
    from workloads import gen
    return [gen.random_string(5, 300, 3), gen.periodic(6, 257, 7, 4, noise=0.05),
            gen.fibonacci_word(200), gen.high_bit_string(7, 150, 5), gen.random_string(8, 1, 2)]


def _dsa_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_18111_b200.dsa import DistSuffixArray
    out = []
    for S in _dsa_strings():
        n = len(S)
        a = [r * n // world for r in range(world + 1)]
        blk = torch.from_numpy(S[a[rank]:a[rank + 1]].view(np.int64).copy()).view(torch.uint64)
        d = DistSuffixArray(_NpDsaOps(), oversample=8)
        part, g = d.run(blk, n)
        out.append((g, part.numpy().copy(), d.rounds, d.lcp().numpy().copy()))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_suffix_array_gloo(world):
    import oracle
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dsa_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out = q.get(timeout=240)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, S in enumerate(_dsa_strings()):
        parts = sorted(((res[r][i][0], res[r][i][1], res[r][i][3]) for r in range(world)), key=lambda x: x[0])
        got = np.concatenate([p for _, p, _ in parts])
        assert [g for g, _, _ in parts] == list(np.cumsum([0] + [len(p) for _, p, _ in parts[:-1]]))
        sa = oracle.sa_naive(S)
        assert np.array_equal(got, sa), i
        lcp = np.concatenate([c for _, _, c in parts])
        want = np.append(oracle.lcp_naive(S, sa), 0)  # LCP(SA[k], SA[k+1]); 0 for the last (R3)
        assert np.array_equal(lcp, want), i
