"""Where does the e2e step's extra time go?  Replays bench.py's C4 e2e loop
(double-buffered H2D on a copy stream, step, readback) with CUDA events on
both streams and host timestamps (diagnostics)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import gen  # noqa: E402
from paper_2406_18111_b200 import Context  # noqa: E402

ctx = Context(0)
tok_np, off, st_np, soff = gen.c4()
s = torch.cuda.current_stream()
cs = torch.cuda.Stream()
tok_host = torch.from_numpy(tok_np).pin_memory()
st_host = torch.from_numpy(st_np).pin_memory()
dbuf = [(torch.empty(len(tok_np), dtype=torch.uint64, device="cuda"),
         torch.empty(len(st_np), dtype=torch.uint64, device="cuda")) for _ in range(2)]


pinned = {}


def pin(name, t):
    b = pinned.get(name)
    if b is None or b.numel() < t.numel():
        b = torch.empty(max(int(t.numel() * 1.25), 1), dtype=t.dtype).pin_memory()
        pinned[name] = b
    v = b[:t.numel()].view(t.shape)
    v.copy_(t, non_blocking=True)
    return v


T = {"analysis": 0.0, "trie": 0.0, "match": 0.0, "readback": 0.0}


def step(tok, streams):
    t0 = time.perf_counter()
    rep, roff, occ = ctx.find_repeats_batched(tok, off, 25)
    t1 = time.perf_counter()
    trie = ctx.trie_build(tok, off, rep, roff, 25, 0)
    t2 = time.perf_counter()
    rp, nall = ctx.match(trie, streams, soff, mode=1)
    t3 = time.perf_counter()
    T["analysis"] += t1 - t0
    T["trie"] += t2 - t1
    T["match"] += t3 - t2
    return rep, roff, occ, rp


def run(K, copies=True):
    ev = []
    c_ev = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        bi = i % 2
        if copies:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cs)
            with torch.cuda.stream(cs):
                dbuf[bi][0].copy_(tok_host, non_blocking=True)
                dbuf[bi][1].copy_(st_host, non_blocking=True)
            b.record(cs)
            c_ev.append((a, b))
            s.wait_event(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rep, roff, occ, rp = step(dbuf[bi][0], dbuf[bi][1])
        e1.record(s)
        ev.append((e0, e1))
        rep.cpu(), occ.cpu(), rp.cpu()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / K
    steps = [a.elapsed_time(b) for a, b in ev]
    cps = [a.elapsed_time(b) for a, b in c_ev]
    return wall, np.mean(steps), (np.mean(cps) if cps else 0.0)


CHUNK = int(os.environ.get("CHUNK", str(2 << 20)))


def run_db(K):
    """bench.py's schedule: step i+1's copies are issued before step i runs."""
    ev, c_ev = [], []
    copied = [None, None]

    def enq(i):
        bi = i % 2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        with torch.cuda.stream(cs):
            for dst, src in ((dbuf[bi][0], tok_host), (dbuf[bi][1], st_host)):
                for c0 in range(0, src.numel(), CHUNK):
                    dst[c0:c0 + CHUNK].copy_(src[c0:c0 + CHUNK], non_blocking=True)
        b.record(cs)
        c_ev.append((a, b))
        copied[bi] = b

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    enq(0)
    for i in range(K):
        bi = i % 2
        s.wait_event(copied[bi])
        if i + 1 < K:
            cs.wait_stream(s)  # (the buffer's previous user, step i-1, was waited for by the host)
            enq(i + 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rep, roff, occ, rp = step(dbuf[bi][0], dbuf[bi][1])
        e1.record(s)
        ev.append((e0, e1))
        t4 = time.perf_counter()
        pin("rep", rep), pin("occ", occ), pin("rp", rp), pin("roff", roff)
        torch.cuda.current_stream().synchronize()
        T["readback"] += time.perf_counter() - t4
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / K
    return wall, np.mean([a.elapsed_time(b) for a, b in ev]), np.mean([a.elapsed_time(b) for a, b in c_ev])


def kinds():
    out = {}
    for name, k in (("K9", ctx.PROF_WINDOW_SA), ("match", ctx.PROF_MATCH), ("K1", ctx.PROF_RADIX_PASS),
                    ("scan", ctx.PROF_SCAN)):
        ms, n, _ = ctx.profile_read(k)
        out[name] = round(ms / max(n, 1), 3)
    return out


run(2)
ctx.profile(True)
run(4, False)
print("no copies, per launch:", kinds(), flush=True)
ctx.profile(True)
run_db(4)
print("double-buffered copies, per launch:", kinds(), flush=True)
ctx.profile(False)
for k in T:
    T[k] = 0.0
w, st_ms, cp = run_db(6)
print(f"double-buffered: wall {w:.1f} ms/step, step events {st_ms:.1f} ms, copy events {cp:.1f} ms", flush=True)
print("host ms per step:", {k: round(v * 1e3 / 6, 2) for k, v in T.items()}, flush=True)
for copies in (False, True):
    w, st_ms, cp = run(6, copies)
    print(f"copies={copies}: wall {w:.1f} ms/step, step events {st_ms:.1f} ms, copy events {cp:.1f} ms", flush=True)
