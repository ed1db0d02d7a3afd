"""Thin ctypes binding of libapo (include/apo.h) -- argument marshalling only.

Every step of the path runs in the CUDA kernels of libapo.so; this module only
passes torch device pointers, sizes and the current CUDA stream.  There is no
CPU fallback: if libapo.so is missing or no CUDA device is present, calls
raise.

Names follow the C ABI: suffix_array, suffix_array_batched, candidates,
find_repeats, find_repeats_batched, History.ingest / .window.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("APO_LIB", os.path.join(_HERE, "libapo.so"))

APO_OK, APO_ERR_INVALID, APO_ERR_CAPACITY, APO_ERR_NOMEM, APO_ERR_CUDA = range(5)
_STATUS = {0: "APO_OK", 1: "APO_ERR_INVALID", 2: "APO_ERR_CAPACITY", 3: "APO_ERR_NOMEM", 4: "APO_ERR_CUDA"}


class ApoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class apo_params(ctypes.Structure):
    _fields_ = [("min_count", ctypes.c_int32), ("max_len", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("reserved", ctypes.c_int32)]


class apo_replay_params(ctypes.Structure):
    _fields_ = [("count_cap", ctypes.c_int32), ("decay_q16", ctypes.c_int32), ("decay_period", ctypes.c_int32),
                ("bonus_num", ctypes.c_int32), ("bonus_den", ctypes.c_int32), ("reserved", ctypes.c_int32)]


REPLAY_DEFAULTS = dict(count_cap=100, decay_q16=64881, decay_period=100, bonus_num=11, bonus_den=10)


class apo_slice(ctypes.Structure):
    _fields_ = [("begin", ctypes.c_int64), ("end", ctypes.c_int64)]


_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_P_I64 = ctypes.POINTER(ctypes.c_int64)

_SIGS = {
    "apo_version": (ctypes.c_int, []),
    "apo_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_VP)]),
    "apo_ctx_destroy": (None, [_VP]),
    "apo_last_error": (ctypes.c_char_p, [_VP]),
    "apo_launch_count": (ctypes.c_int64, [_VP]),
    "apo_profile": (ctypes.c_int, [_VP, ctypes.c_int]),
    "apo_profile_read": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_double), _P_I64,
                                        ctypes.POINTER(ctypes.c_double)]),
    "apo_radix_sort": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I32, _I32, _VP]),
    "apo_suffix_array": (ctypes.c_int, [_VP, _VP, _I32, _VP, _VP, _VP]),
    "apo_suffix_array_batched": (ctypes.c_int, [_VP, _VP, _P_I64, _I32, _VP, _VP, _VP]),
    "apo_candidates": (ctypes.c_int, [_VP, _VP, _I32, _I32, _VP, _VP, _VP, _VP, _I64, _VP, _VP]),
    "apo_find_repeats": (ctypes.c_int, [_VP, _VP, _I32, _I32, ctypes.POINTER(apo_params), _VP, _I64, _VP,
                                        _I64, _VP, _VP]),
    "apo_find_repeats_batched": (ctypes.c_int, [_VP, _VP, _P_I64, _I32, _I32, ctypes.POINTER(apo_params), _VP,
                                                _I64, _VP, _VP, _I64, _VP, _VP]),
    "apo_history_create": (ctypes.c_int, [_VP, _I64, _I32, ctypes.POINTER(_VP)]),
    "apo_history_destroy": (None, [_VP]),
    "apo_ingest": (ctypes.c_int, [_VP, _VP, _I64, ctypes.POINTER(apo_slice), _I64, _P_I64, _VP]),
    "apo_ruler_slices": (ctypes.c_int, [_I64, _I64, _I32, _I64, ctypes.POINTER(apo_slice), _I64, _P_I64]),
    "apo_history_window": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP]),
    "apo_history_count": (ctypes.c_int64, [_VP]),
    "apo_trie_build": (ctypes.c_int, [_VP, _VP, _P_I64, _I32, _VP, _VP, _I32, _I32, ctypes.POINTER(_VP), _VP]),
    "apo_trie_build_traces": (ctypes.c_int, [_VP, _VP, _P_I64, _I32, ctypes.POINTER(_VP), _VP]),
    "apo_trie_build_traces_multi": (ctypes.c_int, [_VP, _I32, _VP, _VP, _VP, ctypes.POINTER(_VP), _VP]),
    "apo_trie_destroy": (None, [_VP]),
    "apo_trie_info": (ctypes.c_int, [_VP, _P_I64, _P_I64, _P_I64]),
    "apo_trie_copy": (ctypes.c_int, [_VP, _VP, _P_I64, _VP]),
    "apo_match": (ctypes.c_int, [_VP, _VP, _VP, _P_I64, _I32, _I32, _VP, _I64, _VP, _VP]),
    "apo_replay": (ctypes.c_int, [_VP, _VP, _VP, _I64, _P_I64, _I32, _VP, _VP, _I64, _VP, _VP]),
    "apo_match_index": (ctypes.c_int, [_VP, _VP, _P_I64, _I32, ctypes.POINTER(_VP), _VP]),
    "apo_match_indexed": (ctypes.c_int, [_VP, _VP, _VP, _I32, _VP, _I64, _VP, _VP]),
    "apo_stream_index_destroy": (None, [_VP]),
    "apo_dsa_keys": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _I64, _VP, _VP, _VP]),
    "apo_dsa_samples": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I32, _VP, _VP, _VP]),
    "apo_dsa_split": (ctypes.c_int, [_VP, _VP, _VP, _I64, _VP, _VP, _I32, _VP, _VP]),
    "apo_dsa_heads": (ctypes.c_int, [_VP, _VP, _I64, ctypes.c_uint64, _I32, _I64, _I64, _VP, _VP, _VP]),
    "apo_dsa_scatter": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _VP, _VP]),
    "apo_dsa_lcp_requests": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _I64, _VP, _VP, _VP]),
    "apo_dsa_gather": (ctypes.c_int, [_VP, _VP, _I64, _I64, _VP, _VP, _VP]),
    "apo_dsa_lcp_update": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, ctypes.c_uint32, _VP, _VP, _VP]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libapo.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not found: build it with `python -m paper_2406_18111_b200.build` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check_tok(t: torch.Tensor, device) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError("token tensor must be on the CUDA device (use the *_host helpers for host buffers)")
    if t.dtype not in (torch.uint64, torch.int64):
        raise ValueError("tokens must be uint64 (or int64 bit patterns)")
    return t.contiguous()


def _host_off(off) -> np.ndarray:
    if isinstance(off, torch.Tensor):
        off = off.cpu().numpy()
    return np.ascontiguousarray(np.asarray(off, dtype=np.int64))


class Context:
    """An apo_ctx on one CUDA device (not thread-safe; one per host thread)."""

    def __init__(self, device: int | torch.device = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("libapo needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self._pinned = {}
        self.device = torch.device("cuda", device if isinstance(device, int) else device.index or 0)
        h = ctypes.c_void_p()
        torch.cuda.init()
        st = self.lib.apo_ctx_create(self.device.index, ctypes.byref(h))
        if st != APO_OK:
            raise ApoError(st, "apo_ctx_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.apo_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _read(self, t: torch.Tensor) -> list:
        """Small device tensor -> Python list through a cached pinned buffer (a
        pageable copy waits behind any host -> device transfer in flight)."""
        key = (t.dtype, t.numel())
        buf = self._pinned.get(key)
        if buf is None:
            buf = torch.empty(t.numel(), dtype=t.dtype).pin_memory()
            self._pinned[key] = buf
        buf.copy_(t.reshape(-1), non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return buf.tolist()

    def _raise(self, st: int):
        if st not in (APO_OK,):
            msg = self.lib.apo_last_error(self.h)
            raise ApoError(st, msg.decode() if msg else "")

    @property
    def launches(self) -> int:
        """Kernel launches issued by libapo on this context so far."""
        return int(self.lib.apo_launch_count(self.h))

    # ----------------------------------------------------------- profiler --
    PROF_RADIX_PASS, PROF_RADIX_HIST, PROF_SCAN, PROF_OTHER, PROF_WINDOW_SA, PROF_MATCH = range(6)

    def profile(self, enable: bool):
        self._raise(self.lib.apo_profile(self.h, 1 if enable else 0))

    def profile_read(self, kind: int):
        """-> (device ms, launches, algorithmic bytes) summed over the recorded launches of `kind`."""
        ms, by = ctypes.c_double(), ctypes.c_double()
        k = ctypes.c_int64()
        self._raise(self.lib.apo_profile_read(self.h, int(kind), ctypes.byref(ms), ctypes.byref(k), ctypes.byref(by)))
        return ms.value, k.value, by.value

    # ------------------------------------------------------------------ K1 --
    def radix_sort(self, keys: torch.Tensor, vals: torch.Tensor | None = None, begin_bit: int = 0,
                   end_bit: int = 64):
        """Stable in-place sort of (uint64 keys, uint32/int32 values) by key bits [begin, end)."""
        if not keys.is_cuda or keys.dtype not in (torch.uint64, torch.int64) or not keys.is_contiguous():
            raise ValueError("keys must be a contiguous CUDA uint64 tensor")
        if vals is not None and (vals.numel() != keys.numel() or vals.element_size() != 4 or not vals.is_contiguous()):
            raise ValueError("vals must be a contiguous 32-bit tensor of the same length")
        self._raise(self.lib.apo_radix_sort(self.h, _ptr(keys), _ptr(vals), keys.numel(), int(begin_bit), int(end_bit),
                                            _stream(self.device)))
        return keys, vals

    # ---------------------------------------------------------- SA / LCP --
    def suffix_array(self, tok: torch.Tensor, lcp: bool = True):
        tok = _check_tok(tok, self.device)
        n = tok.numel()
        sa = torch.empty(n, dtype=torch.int32, device=self.device)
        lc = torch.empty(n, dtype=torch.int32, device=self.device) if lcp else None
        self._raise(self.lib.apo_suffix_array(self.h, _ptr(tok), n, _ptr(sa), _ptr(lc), _stream(self.device)))
        return (sa, lc[:max(n - 1, 0)]) if lcp else sa

    def suffix_array_batched(self, tok: torch.Tensor, off):
        tok = _check_tok(tok, self.device)
        o = _host_off(off)
        n = int(o[-1])
        sa = torch.empty(n, dtype=torch.int32, device=self.device)
        lc = torch.empty(n, dtype=torch.int32, device=self.device)
        self._raise(self.lib.apo_suffix_array_batched(self.h, _ptr(tok), o.ctypes.data_as(_P_I64), len(o) - 1,
                                                      _ptr(sa), _ptr(lc), _stream(self.device)))
        return sa, lc

    # --------------------------------------------------------- candidates --
    def candidates(self, tok: torch.Tensor, min_len: int):
        tok = _check_tok(tok, self.device)
        n = tok.numel()
        cap = max(2 * (n - 1), 1)
        d = self.device
        ln = torch.empty(cap, dtype=torch.int32, device=d)
        cid = torch.empty(cap, dtype=torch.int32, device=d)
        st = torch.empty(cap, dtype=torch.int32, device=d)
        kept = torch.empty(cap, dtype=torch.uint8, device=d)
        cnt = torch.zeros(1, dtype=torch.int64, device=d)
        self._raise(self.lib.apo_candidates(self.h, _ptr(tok), n, int(min_len), _ptr(ln), _ptr(cid), _ptr(st),
                                            _ptr(kept), cap, _ptr(cnt), _stream(d)))
        m = int(self._read(cnt)[0])
        return dict(cand_len=ln[:m], cand_id=cid[:m], cand_start=st[:m], keep=kept[:m])

    # ------------------------------------------------------- FindRepeats --
    @staticmethod
    def _params(min_count: int) -> apo_params:
        return apo_params(int(min_count), 0, 0, 0)

    def find_repeats(self, win: torch.Tensor, min_len: int, min_count: int = 1, sync: bool = True):
        """Alg. 2 on one window -> (repeats int32[k,4] (start,length,count,first_occ), occ int32[])."""
        win = _check_tok(win, self.device)
        n = win.numel()
        cap = n // max(int(min_len), 1) + 1  # kept intervals are disjoint and >= min_len long
        d = self.device
        out = torch.empty((cap, 4), dtype=torch.int32, device=d)
        occ = torch.empty(cap, dtype=torch.int32, device=d)
        counts = torch.zeros(2, dtype=torch.int64, device=d)
        prm = self._params(min_count)
        self._raise(self.lib.apo_find_repeats(self.h, _ptr(win), n, int(min_len), ctypes.byref(prm), _ptr(out), cap,
                                              _ptr(occ), cap, _ptr(counts), _stream(d)))
        if not sync:
            return out, occ, counts
        r, o = (int(x) for x in self._read(counts))
        return out[:r], occ[:o]

    def find_repeats_batched(self, tok: torch.Tensor, off, min_len: int, min_count: int = 1, sync: bool = True,
                             out=None):
        """Independent windows -> (repeats int32[k,4], out_off int64[W+1], occ int32[])."""
        tok = _check_tok(tok, self.device)
        o = _host_off(off)
        n = int(o[-1])
        W = len(o) - 1
        d = self.device
        cap = n // max(int(min_len), 1) + 1
        if out is None:
            out = (torch.empty((cap, 4), dtype=torch.int32, device=d), torch.empty(W + 1, dtype=torch.int64, device=d),
                   torch.empty(cap, dtype=torch.int32, device=d), torch.zeros(2, dtype=torch.int64, device=d))
        rep, roff, occ, counts = out
        prm = self._params(min_count)
        self._raise(self.lib.apo_find_repeats_batched(self.h, _ptr(tok), o.ctypes.data_as(_P_I64), W, int(min_len),
                                                      ctypes.byref(prm), _ptr(rep), rep.shape[0], _ptr(roff),
                                                      _ptr(occ), occ.shape[0], _ptr(counts), _stream(d)))
        if not sync:
            return rep, roff, occ, counts
        r, oc = (int(x) for x in self._read(counts))
        return rep[:r], roff, occ[:oc]

    def find_repeats_batched_host(self, tok_host: torch.Tensor, off, min_len: int, min_count: int = 1):
        """End-to-end user call with HOST buffers: H2D copy of the tokens,
        the batched analysis, D2H copy of the results (pinned host memory)."""
        tok = tok_host.to(self.device, non_blocking=True)
        rep, roff, occ, counts = self.find_repeats_batched(tok, off, min_len, min_count, sync=False)
        c = counts.to("cpu")
        r, oc = int(c[0]), int(c[1])
        return rep[:r].to("cpu"), roff.to("cpu"), occ[:oc].to("cpu")

    # --------------------------------------------------------- trie/match --
    def trie_build(self, tok: torch.Tensor, off, repeats: torch.Tensor, rep_off: torch.Tensor, min_len: int,
                   max_len: int = 0) -> "Trie":
        """IngestCandidates from apo_find_repeats_batched output (repeats int32[k,4], rep_off int64[W+1])."""
        tok = _check_tok(tok, self.device)
        o = _host_off(off)
        repeats = repeats.contiguous()
        rep_off = rep_off.to(self.device, torch.int64).contiguous()
        h = ctypes.c_void_p()
        self._raise(self.lib.apo_trie_build(self.h, _ptr(tok), o.ctypes.data_as(_P_I64), len(o) - 1, _ptr(repeats),
                                            _ptr(rep_off), int(min_len), int(max_len), ctypes.byref(h),
                                            _stream(self.device)))
        return Trie(self, h)

    def trie_build_traces(self, traces: torch.Tensor, tr_off) -> "Trie":
        """Trace set from explicit contents (e.g. a gathered union); duplicates merged."""
        o = _host_off(tr_off)
        traces = _check_tok(traces, self.device) if traces.numel() else traces
        h = ctypes.c_void_p()
        self._raise(self.lib.apo_trie_build_traces(self.h, _ptr(traces) if traces.numel() else None,
                                                   o.ctypes.data_as(_P_I64), len(o) - 1, ctypes.byref(h),
                                                   _stream(self.device)))
        return Trie(self, h)

    def trie_build_traces_multi(self, sources) -> "Trie":
        """Union trace set of several trace lists, pulled and hashed in one pass.

        sources: sequence of (device pointer int or CUDA uint64 tensor, host
        int64 offsets[ntr+1]); a pointer may be a peer rank's buffer mapped
        into this device (symmetric memory over NVLink).  Same result as
        trie_build_traces on the concatenation."""
        n = len(sources)
        ptrs = (ctypes.c_uint64 * n)()
        offs = []
        ntr = (ctypes.c_int32 * n)()
        for r, (tok, off) in enumerate(sources):
            o = _host_off(off)
            offs.append(o)
            ntr[r] = len(o) - 1
            if isinstance(tok, torch.Tensor):
                if len(o) > 1:
                    _check_tok(tok, self.device)
                ptrs[r] = tok.data_ptr() if tok.numel() else 0
            else:
                ptrs[r] = int(tok)
        optrs = (ctypes.c_void_p * n)(*[o.ctypes.data for o in offs])
        h = ctypes.c_void_p()
        self._raise(self.lib.apo_trie_build_traces_multi(self.h, n, ctypes.cast(ptrs, _VP), ctypes.cast(optrs, _VP),
                                                         ctypes.cast(ntr, _VP), ctypes.byref(h),
                                                         _stream(self.device)))
        return Trie(self, h)

    def match(self, trie: "Trie", streams: torch.Tensor, off, cap: int | None = None, full: bool = False,
              mode: int = 0):
        """mode 0, MATCH_ALL -> int32[h,3] rows (stream, end_pos, trace_id) sorted
        (full=True: [h,4] with the per-stream slot column).
        mode 1, REPLAY -> (int32[r,4] rows (stream, end_pos, trace_id, first),
        number of MATCH_ALL hits consumed on the device)."""
        streams = _check_tok(streams, self.device)
        o = _host_off(off)
        d = self.device
        if cap is None:
            cap = 1 << 22 if mode == 0 else max(int(o[-1]) // 8, 1024)
        while True:
            out = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=d)
            cnt = torch.zeros(2, dtype=torch.int64, device=d)
            self._raise(self.lib.apo_match(self.h, trie.h, _ptr(streams), o.ctypes.data_as(_P_I64), len(o) - 1,
                                           int(mode), _ptr(out), cap, _ptr(cnt), _stream(d)))
            c = self._read(cnt)
            n = int(c[0])
            if n <= cap:
                if mode == 1:
                    return out[:n], int(c[1])
                return out[:n] if full else out[:n, :3]
            cap = n

    def match_index(self, streams: torch.Tensor, off) -> "StreamIndex":
        """apo_match_index: the trace-independent half of match() (reversed
        streams, their suffix arrays + LCP, first-token buckets), to overlap
        with building the trace set; use with match_indexed()."""
        streams = _check_tok(streams, self.device)
        o = _host_off(off)
        h = ctypes.c_void_p()
        self._raise(self.lib.apo_match_index(self.h, _ptr(streams), o.ctypes.data_as(_P_I64), len(o) - 1,
                                             ctypes.byref(h), _stream(self.device)))
        return StreamIndex(self, h, streams, o)

    def match_indexed(self, trie: "Trie", idx: "StreamIndex", cap: int | None = None, full: bool = False,
                      mode: int = 0):
        """match() on the streams of `idx` (same results)."""
        if idx.ctx is not self:
            raise ValueError("the stream index belongs to another context")
        d = self.device
        if cap is None:
            cap = 1 << 22 if mode == 0 else max(int(idx.off[-1]) // 8, 1024)
        while True:
            out = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=d)
            cnt = torch.zeros(2, dtype=torch.int64, device=d)
            self._raise(self.lib.apo_match_indexed(self.h, trie.h, idx.h, int(mode), _ptr(out), cap, _ptr(cnt),
                                                   _stream(d)))
            c = self._read(cnt)
            n = int(c[0])
            if n <= cap:
                if mode == 1:
                    return out[:n], int(c[1])
                return out[:n] if full else out[:n, :3]
            cap = n

    def replay(self, trie: "Trie", hits: torch.Tensor, stream_lengths, cap: int | None = None, **params):
        """REPLAY selection over MATCH_ALL hits (int32[h,4] from match(..., full=True))
        -> int32[r,4] rows (stream, end_pos, trace_id, first)."""
        if not hits.is_cuda or hits.dtype != torch.int32 or hits.dim() != 2 or hits.shape[1] != 4:
            raise ValueError("hits must be a CUDA int32 [h, 4] tensor (match(..., full=True))")
        hits = hits.contiguous()
        lens = np.ascontiguousarray(np.asarray(stream_lengths, dtype=np.int64))
        p = dict(REPLAY_DEFAULTS, **params)
        prm = apo_replay_params(p["count_cap"], p["decay_q16"], p["decay_period"], p["bonus_num"], p["bonus_den"], 0)
        d = self.device
        if cap is None:
            cap = max(int(lens.sum()) // 8, 1024)
        while True:
            out = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=d)
            cnt = torch.zeros(1, dtype=torch.int64, device=d)
            self._raise(self.lib.apo_replay(self.h, trie.h, _ptr(hits), hits.shape[0], lens.ctypes.data_as(_P_I64),
                                            len(lens), ctypes.byref(prm), _ptr(out), cap, _ptr(cnt), _stream(d)))
            n = int(self._read(cnt)[0])
            if n <= cap:
                return out[:n]
            cap = n

    # ------------------------------------------------------------ history --
    def history(self, capacity_B: int, scale_C: int) -> "History":
        return History(self, capacity_B, scale_C)


def ruler_slices(k0: int, n: int, scale_C: int, capacity_B: int) -> list[tuple[int, int]]:
    """apo_ruler_slices: the analysis slices apo_ingest emits for op counts
    (k0, k0+n] (host logic only; no device needed)."""
    lib = load_library()
    ns = ctypes.c_int64()
    cap = 64
    while True:
        buf = (apo_slice * cap)()
        st = lib.apo_ruler_slices(int(k0), int(n), int(scale_C), int(capacity_B), buf, cap, ctypes.byref(ns))
        if st != APO_ERR_CAPACITY:
            break
        cap = int(ns.value)
    if st != APO_OK:
        raise ApoError(st, "apo_ruler_slices: invalid arguments")
    return [(buf[i].begin, buf[i].end) for i in range(ns.value)]


class History:
    """Alg. 1 TraceFinder buffer with ruler-function sampling (§4.4)."""

    def __init__(self, ctx: Context, capacity_B: int, scale_C: int):
        self.ctx = ctx
        self.capacity_B = int(capacity_B)
        self.scale_C = int(scale_C)
        h = ctypes.c_void_p()
        st = ctx.lib.apo_history_create(ctx.h, int(capacity_B), int(scale_C), ctypes.byref(h))
        ctx._raise(st)
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.apo_history_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def count(self) -> int:
        return int(self.ctx.lib.apo_history_count(self.h))

    def ingest(self, tokens: torch.Tensor, cap: int = 4096) -> list[tuple[int, int]]:
        tokens = _check_tok(tokens, self.ctx.device)
        ns = ctypes.c_int64()
        while True:
            buf = (apo_slice * max(cap, 1))()
            st = self.ctx.lib.apo_ingest(self.h, _ptr(tokens), tokens.numel(), buf, cap, ctypes.byref(ns),
                                         _stream(self.ctx.device))
            if st != APO_ERR_CAPACITY:
                break
            cap = int(ns.value)  # nothing was ingested: retry with room for every slice
        self.ctx._raise(st)
        return [(buf[i].begin, buf[i].end) for i in range(ns.value)]

    def window(self, begin: int, end: int) -> torch.Tensor:
        out = torch.empty(max(end - begin, 0), dtype=torch.uint64, device=self.ctx.device)
        self.ctx._raise(self.ctx.lib.apo_history_window(self.h, int(begin), int(end), _ptr(out),
                                                        _stream(self.ctx.device)))
        return out


class StreamIndex:
    """apo_stream_index: keeps the streams tensor alive while it is used."""

    def __init__(self, ctx: Context, h, streams: torch.Tensor, off: np.ndarray):
        self.ctx, self.h, self.streams, self.off = ctx, h, streams, off

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.apo_stream_index_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Trie:
    """The candidate trace set (apo_trie): traces in id order (length desc, lexicographic asc)."""

    def __init__(self, ctx: Context, h):
        self.ctx = ctx
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.apo_trie_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self):
        t, n, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self.ctx._raise(self.ctx.lib.apo_trie_info(self.h, ctypes.byref(t), ctypes.byref(n), ctypes.byref(m)))
        return t.value, n.value, m.value

    def traces(self, out: torch.Tensor | None = None):
        """-> (tokens uint64 device tensor, host int64 offsets[T+1]); `out`
        (contiguous, >= ntokens elements, 8-byte dtype) receives the tokens
        instead of a new tensor."""
        T, n, _ = self.info()
        if out is None:
            tok = torch.empty(max(n, 1), dtype=torch.uint64, device=self.ctx.device)
        else:
            if not out.is_cuda or out.element_size() != 8 or not out.is_contiguous() or out.numel() < n:
                raise ValueError("out must be a contiguous 8-byte CUDA tensor with >= ntokens elements")
            tok = out
        off = np.zeros(T + 1, dtype=np.int64)
        self.ctx._raise(self.ctx.lib.apo_trie_copy(self.h, _ptr(tok), off.ctypes.data_as(_P_I64),
                                                   _stream(self.ctx.device)))
        return tok[:n], off


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def suffix_array(tok, lcp=True):
    return default_context(tok.device.index or 0).suffix_array(tok, lcp)


def suffix_array_batched(tok, off):
    return default_context(tok.device.index or 0).suffix_array_batched(tok, off)


def candidates(tok, min_len):
    return default_context(tok.device.index or 0).candidates(tok, min_len)


def find_repeats(win, min_len, min_count=1):
    return default_context(win.device.index or 0).find_repeats(win, min_len, min_count)


def find_repeats_batched(tok, off, min_len, min_count=1):
    return default_context(tok.device.index or 0).find_repeats_batched(tok, off, min_len, min_count)
