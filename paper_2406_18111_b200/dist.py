"""Multi-GPU plumbing: gather every rank's candidate trace list.

The only data-path exchange of the sharded C4 workload:
each rank analyses its own windows, builds its local trace set, and the
ranks all-gather their trace lists (NCCL over NVLink on GPUs; gloo in the CPU
tests) so that every rank builds the same union trace set
(apo_trie_build_traces merges duplicates and orders ids by content, so the
union is independent of the gather order and of the number of ranks).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def gather_traces(tokens: torch.Tensor, off: np.ndarray, group=None):
    """All-gather (tokens uint64[n], host offsets int64[T+1]) from every rank.

    Returns (all_tokens on tokens.device, host offsets int64[sum T + 1]) with
    rank 0's traces first, then rank 1's, ...
    """
    world = dist.get_world_size(group)
    dev = tokens.device
    off = np.asarray(off, dtype=np.int64)
    n_tok, n_tr = int(off[-1]), len(off) - 1
    sizes = torch.tensor([n_tok, n_tr], dtype=torch.int64, device=dev)
    all_sizes = torch.empty(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_sizes, sizes, group=group)
    all_sizes = all_sizes.view(world, 2).cpu().numpy()
    max_tok = max(int(all_sizes[:, 0].max()), 1)
    max_tr = max(int(all_sizes[:, 1].max()), 1)
    # padded payloads (uint64 travels as its int64 bit pattern)
    pt = torch.zeros(max_tok, dtype=torch.int64, device=dev)
    if n_tok:
        pt[:n_tok] = tokens[:n_tok].view(torch.int64)
    lens = torch.zeros(max_tr, dtype=torch.int64, device=dev)
    if n_tr:
        lens[:n_tr] = torch.from_numpy(np.diff(off)).to(dev)
    gt = torch.empty(world * max_tok, dtype=torch.int64, device=dev)
    gl = torch.empty(world * max_tr, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(gt, pt, group=group)
    dist.all_gather_into_tensor(gl, lens, group=group)
    gt = gt.view(world, max_tok)
    gl = gl.view(world, max_tr).cpu().numpy()
    parts, lengths = [], []
    for r in range(world):
        nt, nr = int(all_sizes[r, 0]), int(all_sizes[r, 1])
        parts.append(gt[r, :nt])
        lengths.append(gl[r, :nr])
    all_tok = torch.cat(parts).view(torch.uint64) if parts else torch.zeros(0, dtype=torch.uint64, device=dev)
    all_len = np.concatenate(lengths) if lengths else np.zeros(0, np.int64)
    all_off = np.concatenate([[0], np.cumsum(all_len)]).astype(np.int64)
    return all_tok, all_off


class SymmetricTransport:
    """Peer-memory transport of TraceExchange on GPUs: one buffer per rank,
    allocated with torch symmetric memory and mapped into every peer
    (plumbing); the library kernel reads the peers' buffers over NVLink."""

    def __init__(self, dev, group):
        import torch.distributed._symmetric_memory as symm_mem
        self._symm = symm_mem
        self.dev = dev
        self.group = group
        self.cap = 0
        self.buf = None
        self.hdl = None
        self.stage = None
        self.cstream = None
        self.pulled = None

    def ensure(self, need: int):
        """Collective: every rank passes the same global maximum."""
        if need <= self.cap:
            return
        cap = int(need * 1.25) + 4096
        self.buf = self._symm.empty(cap, dtype=torch.int64, device=self.dev)
        self.hdl = self._symm.rendezvous(self.buf, self.group)
        self.cap = cap

    def barrier(self):
        self.hdl.barrier(channel=0)

    def publish(self, trie):
        """Copy the local trace list into this rank's buffer -> host offsets."""
        _, off = trie.traces(out=self.buf)
        return off

    def sources(self):
        """Per rank: its buffer, readable from this rank's device."""
        return list(self.hdl.buffer_ptrs)

    def pull(self, ntok):
        """Copy every rank's list (ntok[r] tokens; the own one too) into local
        staging, back to back in rank order, with the copy engines, on a side
        stream that first waits for the caller's stream (the barrier that
        follows the peers' publishes); returns per rank a local pointer.
        Back-to-back lists are hashed in place by the union build (no
        gathered copy: 0.4 ms less at N = 4).  wait() joins."""
        me = self.hdl.rank
        need = sum(int(n) for n in ntok)
        if self.stage is None or self.stage.numel() < need:
            self.stage = torch.empty(max(int(need * 1.25), 1), dtype=torch.int64, device=self.dev)
        if self.cstream is None:
            self.cstream = torch.cuda.Stream(self.dev)
        self.cstream.wait_stream(torch.cuda.current_stream(self.dev))
        ptrs, o = [], 0
        with torch.cuda.stream(self.cstream):
            for r, n in enumerate(ntok):
                n = int(n)
                if n:
                    src = self.buf[:n] if r == me else self.hdl.get_buffer(r, (n,), torch.int64)
                    self.stage[o:o + n].copy_(src, non_blocking=True)
                ptrs.append(self.stage.data_ptr() + 8 * o)
                o += n
        self.pulled = torch.cuda.Event()
        self.pulled.record(self.cstream)
        return ptrs

    def wait(self):
        torch.cuda.current_stream(self.dev).wait_event(self.pulled)


class TraceExchange:
    """The multi-GPU union over NVLink peer memory.

    Each rank copies its local trace list into its exchange buffer (one per
    rank, mapped into every peer by the transport), the ranks exchange their
    (small) list sizes and trace lengths over the process group, and every
    rank calls apo_trie_build_traces_multi with every rank's buffer: the
    library kernel pulls the remote lists over NVLink in the same pass that
    hashes them, so there is no separate all-gather buffer, padding or
    concatenation.  Transport barriers order the copies before the pulls and
    the pulls before the next step's copies.

    The transport is a seam: on GPUs it is SymmetricTransport (the product);
    the world-size-2 gloo test (tests/test_dist_cpu.py) runs this same
    union() with a host shared-memory transport and a CPU builder.  The
    buffer is reused across steps and regrown (collectively: every rank sees
    the same global maximum) when a list no longer fits.
    """

    def __init__(self, ctx, group=None, transport=None):
        self.ctx = ctx
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        dev = getattr(ctx, "device", "cpu")
        self.dev = dev if isinstance(dev, torch.device) else (
            torch.device("cuda", dev) if isinstance(dev, int) else torch.device(dev))
        self.transport = transport if transport is not None else SymmetricTransport(self.dev, self.group)
        self.last_pulled_tokens = 0  # tokens this rank pulled from peers in the last union (bench report)
        self._bufs = {}

    def gather_sizes(self, T: int, n: int) -> np.ndarray:
        """Collective: every rank's (tokens, traces) -> int64[world, 2]."""
        sizes = torch.tensor([n, T], dtype=torch.int64, device=self.dev)
        all_sizes = torch.empty(self.world * 2, dtype=torch.int64, device=self.dev)
        dist.all_gather_into_tensor(all_sizes, sizes, group=self.group)
        return all_sizes.view(self.world, 2).cpu().numpy()

    def _host_buf(self, name: str, n: int) -> torch.Tensor:
        """A reusable int32 host buffer of >= n elements (pinned on GPUs, so
        the copies below are DMA rather than staged pageable copies; with
        int32 lengths the offsets exchange at N = 4 went from 1.0-2.1 ms to
        0.87-1.27 ms, `tools/exchange_parts.py`)."""
        b = self._bufs.get(name)
        if b is None or b.numel() < n:
            b = torch.empty(max(int(n * 1.25), 1024), dtype=torch.int32,
                            pin_memory=self.dev.type == "cuda")
            self._bufs[name] = b
        return b

    def gather_offsets(self, all_sizes: np.ndarray, lengths) -> list:
        """Collective: every rank's trace lengths (int32) -> per-rank host
        offsets (int64)."""
        T = int(all_sizes[self.rank, 1])
        max_tr = max(int(all_sizes[:, 1].max()), 1)
        lh = self._host_buf("lens", max_tr)[:max_tr]
        ln = lh.numpy()
        ln[:T] = np.asarray(lengths, dtype=np.int32)
        ln[T:] = 0
        lens = lh.to(self.dev, non_blocking=True)
        gl = torch.empty(self.world * max_tr, dtype=torch.int32, device=self.dev)
        dist.all_gather_into_tensor(gl, lens, group=self.group)
        gh = self._host_buf("all", self.world * max_tr)[:self.world * max_tr]
        gh.copy_(gl, non_blocking=True)
        if self.dev.type == "cuda":
            torch.cuda.current_stream(self.dev).synchronize()
        g = gh.numpy().reshape(self.world, max_tr)
        out = []
        for r in range(self.world):
            o = np.zeros(int(all_sizes[r, 1]) + 1, dtype=np.int64)
            np.cumsum(g[r, :int(all_sizes[r, 1])], out=o[1:])
            out.append(o)
        return out

    def union(self, trie):
        """-> the union Trie of every rank's `trie` (identical on all ranks):
        the library kernel pulls the peers' lists over NVLink while it hashes
        them."""
        self._publish(trie)
        ptrs = self.transport.sources()
        return self.ctx.trie_build_traces_multi([(ptrs[r], self._offs[r]) for r in range(self.world)])

    def start(self, trie):
        """First half of an overlapped union: publish, exchange sizes, and
        start pulling the peers' lists into local memory with the copy
        engines (no SMs), so the caller's stream can run other work (e.g.
        apo_match_index of its streams) meanwhile; finish() builds the union."""
        self._publish(trie)
        self._ptrs = self.transport.pull([int(x) for x in self._sizes[:, 0]])

    def finish(self):
        """-> the union Trie (after start())."""
        self.transport.wait()
        return self.ctx.trie_build_traces_multi([(self._ptrs[r], self._offs[r]) for r in range(self.world)])

    def _publish(self, trie):
        T, n, _ = trie.info()
        all_sizes = self.gather_sizes(T, n)
        self.transport.ensure(max(int(all_sizes[:, 0].max()), 1))
        self.transport.barrier()              # peers are done reading the previous step's lists
        off = self.transport.publish(trie)    # local list -> own exchange buffer
        self._offs = self.gather_offsets(all_sizes, np.diff(off))
        self.transport.barrier()              # every rank's copy is complete
        self._sizes = all_sizes
        self.last_pulled_tokens = int(all_sizes[:, 0].sum() - all_sizes[self.rank, 0])
