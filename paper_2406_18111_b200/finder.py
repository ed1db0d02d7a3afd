"""Alg. 1 TraceFinder with asynchronous analyses and the multi-node
ingestion agreement.

PAPER.md Alg. 1: every op is appended to the history buffer B;
when the ruler schedule (§4.4) says so, "async FindRepeats(...)"
analyses a suffix of B in the background and the application keeps going
("the string analysis ... is performed asynchronously ... in a
background thread").  On B200 the analysis runs on its own library context
and CUDA stream, driven by a worker thread (the library calls release the
GIL), so it overlaps whatever the caller's stream does meanwhile (matching,
the next ingest).

Agreement: with several replicas (one per node / GPU), an
analysis may finish earlier on one than on another, so replicas must agree
WHEN its result is ingested.  "We resolve this tension by having each node
agree on a count of processed operations to issue before ingesting the
results of an asynchronous analysis.  If any node had to wait on an
asynchronous analysis to complete, all nodes increase their count of
operations to wait on for the next analysis."  Reading R25: an
analysis launched at op count k is ingested exactly when the op count
reaches k + D, D being the agreed delay when it was launched; at that point
each replica waits for it if it is not done, the replicas all-reduce (max)
whether anyone waited, and if so every replica doubles D for the analyses
launched from then on.  Every replica therefore ingests the same results at
the same op counts, whatever the timing.

The analyzer and the collective are seams: the product uses
`StreamAnalyzer` (the CUDA library on a side stream) and torch.distributed
(NCCL on GPUs); tests/test_dist_cpu.py runs the same TraceFinder logic on
CPU with gloo and a scripted analyzer whose completion times differ by rank.
"""
from __future__ import annotations

from collections import deque
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch
import torch.distributed as dist


class StreamAnalyzer:
    """Runs FindRepeats (apo_find_repeats) on its own context and CUDA
    stream from a worker thread: `submit(window, ready) -> future` whose
    result is (window, repeats, repeat offsets), all on the device."""

    def __init__(self, device: int, min_len: int, min_count: int = 1):
        from .apo import Context
        self.device = device
        self.min_len = min_len
        self.min_count = min_count
        self.ctx = Context(device)
        self.stream = torch.cuda.Stream(torch.device("cuda", device))
        self.pool = ThreadPoolExecutor(1)  # analyses complete in launch order

    def submit(self, window: torch.Tensor, ready: torch.cuda.Event):
        """window: device tokens copied out of the history on the caller's
        stream; `ready` is recorded on that stream after the copy."""
        def run():
            with torch.cuda.stream(self.stream):
                if ready is not None:
                    self.stream.wait_event(ready)
                rep, occ = self.ctx.find_repeats(window, self.min_len, self.min_count)  # syncs self.stream
            roff = torch.tensor([0, rep.shape[0]], dtype=torch.int64, device=window.device)
            return window, rep, roff
        return self.pool.submit(run)

    def close(self):
        self.pool.shutdown(wait=True)


class TraceSetBuilder:
    """IngestCandidates (Alg. 1) on the device: the trace set of an
    analysis (apo_trie_build over the analysed window and its repeats) and
    the union with the current set (apo_trie_build_traces_multi over both
    lists; identical contents merge, ids by content, reading R19)."""

    def __init__(self, ctx, min_len: int, max_len: int = 0):
        self.ctx = ctx
        self.min_len = min_len
        self.max_len = max_len

    def from_analysis(self, result):
        win, rep, roff = result
        return self.ctx.trie_build(win, np.array([0, win.numel()], dtype=np.int64), rep, roff, self.min_len,
                                   self.max_len)

    def union(self, a, b):
        ta, oa = a.traces()
        tb, ob = b.traces()
        return self.ctx.trie_build_traces_multi([(ta, oa), (tb, ob)])

    @staticmethod
    def size(t) -> int:
        return 0 if t is None else int(t.info()[0])


class TraceFinder:
    """Online history + ruler-scheduled asynchronous analyses + ingestion at
    agreed op counts.  `ingest(tokens)` appends ops and returns the
    ingestion events of the call: (op count, anyone waited, traces in the set
    after, delay after, launch op count of the analysis).  `trie` is the
    current candidate trace set."""

    def __init__(self, history, analyzer, builder, delay: int, group=None, allreduce_max=None):
        if int(delay) < 1:
            raise ValueError("delay must be >= 1 op")
        self.history = history
        self.analyzer = analyzer
        self.builder = builder
        self.delay = int(delay)
        self.group = group
        self._allreduce_max = allreduce_max
        self.pending: deque = deque()      # (due op count, launch op count, future)
        self.count = history.count
        self.trie = None
        self.events: list = []

    # -- collective ----------------------------------------------------------
    def _any_waited(self, waited: bool) -> bool:
        if self._allreduce_max is not None:
            return bool(self._allreduce_max(int(waited)))
        if not dist.is_available() or not dist.is_initialized():
            return waited
        t = torch.tensor([int(waited)], dtype=torch.int32,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    # -- ingestion -----------------------------------------------------------
    def _take(self, fut):
        new = self.builder.from_analysis(fut.result())  # blocks iff this replica has to wait
        self.trie = new if self.trie is None else self.builder.union(self.trie, new)

    def _ingest_due(self):
        """Ingest every pending analysis due at the current op count."""
        while self.pending and self.pending[0][0] == self.count:
            due, k0, fut = self.pending.popleft()
            waited = not fut.done()
            anyw = self._any_waited(waited)
            if anyw:
                self.delay *= 2
            self._take(fut)
            self.events.append((self.count, anyw, self.builder.size(self.trie), self.delay, k0))

    def ingest(self, tokens) -> list:
        """Append ops in pieces that stop at every due point and at every
        multiple of C (where the ruler schedule may launch an analysis, so a
        new analysis's due point always lies ahead of the op count)."""
        n = len(tokens)
        C = int(self.history.scale_C)
        first_event = len(self.events)
        pos = 0
        while pos < n:
            nxt = min(n, pos + (C - self.count % C))
            if self.pending:
                nxt = min(nxt, pos + (self.pending[0][0] - self.count))
            piece = tokens[pos:nxt]
            slices = self.history.ingest(piece)
            self.count += len(piece)
            for b, e in slices:
                win = self.history.window(b, e)
                ready = None
                if isinstance(win, torch.Tensor) and win.is_cuda:
                    ready = torch.cuda.Event()
                    ready.record()
                self.pending.append((e + self.delay, e, self.analyzer.submit(win, ready)))
            pos = nxt
            self._ingest_due()
        return self.events[first_event:]

    def flush(self):
        """End of the stream: wait for every pending analysis and ingest it."""
        while self.pending:
            self._take(self.pending.popleft()[2])


class BatchPipeline:
    """Batches of independent windows and their matching streams with the
    analysis of batch k+1 overlapped with the trace set, matching and replay
    of batch k ("async FindRepeats").

    The analysis (apo_find_repeats_batched) runs on its own library context
    and CUDA stream, driven by a worker thread; the rest of a batch (trace
    set, optional cross-GPU union, apo_match) runs on the caller's current
    stream, which waits for the batch's analysis with a CUDA event.  Two
    output buffer sets alternate between batches.  Results are identical to
    running the batches one after the other (the same library calls on the
    same inputs; only their overlap changes).

    run(batches) takes an iterable of (tok, off, streams, soff, ready) --
    device tokens and host offsets; `ready` is a CUDA event the inputs are
    complete at (or None) -- and yields, per batch, (repeats, repeat
    offsets, occurrences, counts, match result): repeats etc. as
    find_repeats_batched(sync=False) returns them (valid until the loop asks
    for the next batch: the analysis after next reuses them), the match
    result as Context.match(mode=...) returns it.
    """

    def __init__(self, ctx, min_len: int, min_count: int = 1, max_len: int = 0, mode: int = 1, exchange=None):
        from .apo import Context
        self.ctx = ctx
        self.min_len, self.min_count, self.max_len, self.mode = min_len, min_count, max_len, mode
        self.exchange = exchange
        dev = ctx.device if isinstance(ctx.device, torch.device) else torch.device("cuda", ctx.device)
        self.dev = dev
        self.actx = Context(dev.index)
        # the analysis runs at the lowest stream priority, the rest of a
        # batch at the highest: when a CTA slot frees up, the block
        # scheduler serves matching / replay first, the analysis fills the
        # rest
        least, greatest = torch.cuda.Stream.priority_range()
        self.astream = torch.cuda.Stream(dev, priority=least)
        self.hstream = torch.cuda.Stream(dev, priority=greatest)
        self.pool = ThreadPoolExecutor(1)
        self.bufs = [None, None]
        self.match_cap = 1 << 20
        self.last_hits = 0
        self.last_traces = 0

    def _buffers(self, k: int, n: int, W: int):
        b = self.bufs[k]
        cap = n // max(self.min_len, 1) + 1
        if b is None or b[0].shape[0] < cap or b[1].numel() != W + 1:
            b = (torch.empty((cap, 4), dtype=torch.int32, device=self.dev),
                 torch.empty(W + 1, dtype=torch.int64, device=self.dev),
                 torch.empty(cap, dtype=torch.int32, device=self.dev),
                 torch.zeros(2, dtype=torch.int64, device=self.dev))
            self.bufs[k] = b
        return b

    def _analyse(self, k: int, tok, off, ready):
        out = self._buffers(k, int(off[-1]), len(off) - 1)

        def run():
            with torch.cuda.stream(self.astream):
                if ready is not None:
                    self.astream.wait_event(ready)
                r = self.actx.find_repeats_batched(tok, off, self.min_len, self.min_count, sync=False, out=out)
                done = torch.cuda.Event()
                done.record(self.astream)
            return r, done
        return self.pool.submit(run)

    def run(self, batches):
        it = iter(batches)
        cur = next(it, None)
        if cur is None:
            return
        caller = torch.cuda.current_stream(self.dev)
        s = self.hstream
        s.wait_stream(caller)
        self.astream.wait_stream(caller)
        fut = self._analyse(0, cur[0], cur[1], cur[4])
        k = 0
        while cur is not None:
            (rep, roff, occ, counts), done = fut.result()  # batch k analysed (enqueued and host-complete)
            nxt = next(it, None)
            tok, off, streams, soff, ready = cur
            s.wait_event(done)
            if ready is not None:
                s.wait_event(ready)
            res = None
            launched = False
            torch.cuda.set_stream(s)
            if streams is not None:
                trie = self.ctx.trie_build(tok, off, rep, roff, self.min_len, self.max_len)
                if nxt is not None:
                    fut = self._analyse((k + 1) % 2, nxt[0], nxt[1], nxt[4])
                    launched = True
                if self.exchange is not None:  # copy-engine pulls overlap the stream index
                    self.exchange.start(trie)
                    idx = self.ctx.match_index(streams, soff)
                    trie = self.exchange.finish()
                    res = self.ctx.match_indexed(trie, idx, mode=self.mode, cap=self.match_cap)
                else:
                    res = self.ctx.match(trie, streams, soff, mode=self.mode, cap=self.match_cap)
                if self.mode == 1:
                    self.match_cap = max(int(res[0].shape[0]), 1)
                    self.last_hits = res[1]
                self.last_traces = trie.info()[0]
            if nxt is not None and not launched:
                fut = self._analyse((k + 1) % 2, nxt[0], nxt[1], nxt[4])
            torch.cuda.set_stream(caller)
            caller.wait_stream(s)  # the caller's later work sees this batch's results
            yield rep, roff, occ, counts, res
            cur = nxt
            k += 1

    def close(self):
        self.pool.shutdown(wait=True)
