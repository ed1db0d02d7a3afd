"""Distributed suffix array of ONE window split over the ranks of a process
group (a window larger than one GPU).

"SA, LCP <- SuffixArray(S)" (Alg. 2) by prefix doubling
where every round is a distributed sample sort; the LCP (`lcp()`) by
galloping over the saved rank levels with one request/answer exchange per
level.  Rank r owns the contiguous
positions [a_r, a_{r+1}) of S, a_r = r * n // G.  Round 0 sorts the
suffixes by their first token; round j by their first 2^j tokens:

  1. rank2[i] = rank[i + h] for the owned i (h = 2^(j-1)): the positions
     [a_r + h, a_{r+1} + h) belong to one or two other ranks -> one
     all-to-all of contiguous slices;
  2. keys (rank[i], rank2[i]) packed in a u64 (apo_dsa_keys), values i;
  3. sample sort: local stable radix sort (apo_radix_sort, K1), evenly
     spaced samples (apo_dsa_samples) all-gathered and sorted, G - 1
     splitters, per-destination counts (apo_dsa_split: (key, position)
     order, so equal keys may straddle ranks and the parts stay balanced
     even when a few groups are huge, e.g. a 4-token alphabet), all-to-all
     of keys and positions, local sort of what arrived;
  4. new ranks (apo_dsa_heads): a group starts where the key changes (the
     previous rank's last key decides the first element); rank = global
     index of the group's first element + 1, carried across rank
     boundaries; the heads are counted: all distinct <=> n heads, done;
  5. (position, new rank) pairs go back to the position owners: local sort
     by position, counts per owner, all-to-all, scatter (apo_dsa_scatter).

When all n keys are distinct, rank r's sorted positions are SA[g_r ..
g_r + m_r) (g_r = elements on lower ranks): the suffix array, distributed
in global order.  The arithmetic is exact; the result is the unique suffix
array.  The collectives are torch.distributed calls (NCCL on GPUs: plumbing)
on tensors of the ops' device; every step that computes is a library kernel
(`CudaDsaOps`).  The ops are a seam: tests/test_dist_cpu.py runs this same
orchestration on CPU with gloo and numpy stand-ins.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def bits_for(x: int) -> int:
    return max(int(x).bit_length(), 1)


class CudaDsaOps:
    """The per-rank compute steps on the GPU (libapo's apo_dsa_* and K1)."""

    def __init__(self, ctx):
        from . import apo
        self.ctx = ctx
        self.lib = ctx.lib  # signatures set by apo.load_library
        self.apo = apo
        self.device = ctx.device if isinstance(ctx.device, torch.device) else torch.device("cuda", ctx.device)

    def _s(self):
        return self.apo._stream(self.device)

    def _p(self, t):
        return self.apo._ptr(t)

    def empty(self, n, dtype):
        return torch.empty(max(int(n), 0), dtype=dtype, device=self.device)

    def sort(self, keys, vals, bits: int):
        """Stable sort of (u64 key, u32 value) pairs by the low `bits` key bits, in place."""
        if keys.numel() > 1:
            self.ctx.radix_sort(keys, vals, 0, bits)

    def keys(self, rank, rank2, base: int, n: int):
        m = rank.numel()
        k, v = self.empty(m, torch.uint64), self.empty(m, torch.int32)
        self.ctx._raise(self.lib.apo_dsa_keys(self.ctx.h, self._p(rank), self._p(rank2), m, rank2.numel(), base, n,
                                              self._p(k), self._p(v), self._s()))
        return k, v

    def samples(self, keys, vals, s: int):
        sk, sv = self.empty(s, torch.uint64), self.empty(s, torch.int32)
        self.ctx._raise(self.lib.apo_dsa_samples(self.ctx.h, self._p(keys), self._p(vals), keys.numel(), s,
                                                 self._p(sk), self._p(sv), self._s()))
        return sk, sv

    def split(self, keys, vals, split_keys, split_vals, g: int):
        cnt = self.empty(g, torch.int64)
        self.ctx._raise(self.lib.apo_dsa_split(self.ctx.h, self._p(keys), self._p(vals), keys.numel(),
                                               self._p(split_keys), self._p(split_vals), g, self._p(cnt),
                                               self._s()))
        return cnt

    def heads(self, keys, prev_key: int, has_prev: bool, gbase: int, carry: int):
        m = keys.numel()
        rank = self.empty(m, torch.int32)
        st = self.empty(2, torch.int64)
        self.ctx._raise(self.lib.apo_dsa_heads(self.ctx.h, self._p(keys), m, int(prev_key), int(has_prev), gbase,
                                               carry, self._p(rank), self._p(st), self._s()))
        h, last = (int(x) for x in st.tolist())
        return rank, h, last

    def scatter(self, pos, rank_in, base: int, rank):
        self.ctx._raise(self.lib.apo_dsa_scatter(self.ctx.h, self._p(pos), self._p(rank_in), pos.numel(), base,
                                                 self._p(rank), self._s()))

    def lcp_requests(self, a, b, l, n: int):
        np_ = a.numel()
        k, v = self.empty(2 * np_, torch.uint64), self.empty(2 * np_, torch.int32)
        self.ctx._raise(self.lib.apo_dsa_lcp_requests(self.ctx.h, self._p(a), self._p(b), self._p(l), np_, n,
                                                      self._p(k), self._p(v), self._s()))
        return k, v

    def gather(self, pos, base: int, rank):
        out = self.empty(pos.numel(), torch.int32)
        self.ctx._raise(self.lib.apo_dsa_gather(self.ctx.h, self._p(pos), pos.numel(), base, self._p(rank),
                                                self._p(out), self._s()))
        return out

    def lcp_update(self, resp, req, nvalid: int, step: int, by_req, l):
        self.ctx._raise(self.lib.apo_dsa_lcp_update(self.ctx.h, self._p(resp), self._p(req), nvalid, l.numel(), step,
                                                    self._p(by_req), self._p(l), self._s()))


class DistSuffixArray:
    """Suffix array of the window whose positions [a_r, a_{r+1}) this rank
    holds (`run`), by distributed prefix doubling."""

    def __init__(self, ops, group=None, oversample: int = 64):
        self.ops = ops
        self.group = group if group is not None else dist.group.WORLD
        self.G = dist.get_world_size(self.group)
        self.r = dist.get_rank(self.group)
        self.oversample = oversample
        self.rounds = 0

    # -- collectives (plumbing) ----------------------------------------------
    def _all_to_all(self, x, send_counts, recv_counts):
        out = torch.empty(int(sum(recv_counts)), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x.contiguous(), [int(c) for c in recv_counts], [int(c) for c in send_counts],
                               group=self.group)
        return out

    def _exchange_counts(self, send_counts):
        sc = send_counts.to(torch.int64)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        return sc.tolist(), rc.tolist()

    def _all_gather_i64(self, vals):
        t = torch.tensor(vals, dtype=torch.int64, device=self.ops.device)
        out = torch.empty(self.G * len(vals), dtype=torch.int64, device=self.ops.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.view(self.G, len(vals)).tolist()

    @staticmethod
    def _u64(x):  # torch uint64 values travel as their int64 bit pattern
        return x.view(torch.int64)

    # -- steps ----------------------------------------------------------------
    def _sample_sort(self, keys, vals, bits):
        """Globally sort (key, position) pairs: -> this rank's contiguous
        part of the global order, locally sorted by key."""
        ops, G = self.ops, self.G
        ops.sort(keys, vals, bits)
        if G == 1:
            return keys, vals
        s = self.oversample
        sk, sv = ops.samples(keys, vals, s)
        ak = torch.empty(G * s, dtype=torch.int64, device=ops.device)
        av = torch.empty(G * s, dtype=torch.int32, device=ops.device)
        dist.all_gather_into_tensor(ak, self._u64(sk), group=self.group)
        dist.all_gather_into_tensor(av, sv, group=self.group)
        # splitter choice (host: G * s pairs of metadata): the samples in
        # (key, position) order, every s-th one
        hk = ak.cpu().numpy().view(np.uint64)
        hv = av.cpu().numpy().astype(np.int64)
        o = np.lexsort((hv, hk))
        pick = o[np.arange(1, G) * s]
        spk = torch.from_numpy(hk[pick].copy()).to(ops.device)
        spv = torch.from_numpy(hv[pick].astype(np.int32)).to(ops.device)
        cnt = ops.split(keys, vals, spk, spv, G)
        send, recv = self._exchange_counts(cnt)
        rk = self._all_to_all(self._u64(keys), send, recv).view(torch.uint64)
        rv = self._all_to_all(vals, send, recv)
        ops.sort(rk, rv, bits)
        return rk, rv

    def _new_ranks(self, keys):
        """-> (new rank of each local element, total heads, gbase)."""
        ops = self.ops
        m = keys.numel()
        last_key = int(self._u64(keys[-1:]).item()) if m else 0
        info = self._all_gather_i64([m, last_key])
        gbase = sum(info[s][0] for s in range(self.r))
        prev = [s for s in range(self.r) if info[s][0] > 0]
        has_prev = bool(prev)
        prev_key = (info[prev[-1]][1] & ((1 << 64) - 1)) if has_prev else 0
        _, h, last = ops.heads(keys, prev_key, has_prev, gbase, -1)
        st = self._all_gather_i64([h, last])
        carry = max([st[s][1] for s in range(self.r)], default=-1)
        rank, _, _ = ops.heads(keys, prev_key, has_prev, gbase, carry)
        return rank, sum(st[s][0] for s in range(self.G)), gbase

    def _to_owners(self, pos, rank, a, n, rank_block, base):
        """(position, rank) pairs -> the owners' rank arrays."""
        ops, G = self.ops, self.G
        pk = pos.to(torch.int64).view(torch.uint64).clone()
        rk = rank.clone()
        ops.sort(pk, rk, bits_for(n))
        if G > 1:
            bk = torch.tensor(a[1:G], dtype=torch.int64, device=ops.device).view(torch.uint64)
            bv = torch.zeros(G - 1, dtype=torch.int32, device=ops.device)
            cnt = ops.split(pk, rk, bk, bv, G)
            send, recv = self._exchange_counts(cnt)
            pos_in = self._all_to_all(self._u64(pk).to(torch.int32), send, recv)
            rank_in = self._all_to_all(rk, send, recv)
        else:
            pos_in, rank_in = self._u64(pk).to(torch.int32), rk
        ops.scatter(pos_in, rank_in, base, rank_block)

    def run(self, tok_block, n: int):
        """tok_block: this rank's tokens S[a_r:a_{r+1}] (uint64, ops device),
        n: the window length.  -> (this rank's part of SA (int32 positions),
        global index of its first entry)."""
        ops, G, r = self.ops, self.G, self.r
        if n >= (1 << 31) - 1:
            raise ValueError("window too long for 31-bit positions")
        a = [q * n // G for q in range(G + 1)]
        base, m = a[r], a[r + 1] - a[r]
        # round 0: sort by the first token
        keys = tok_block.clone()
        vals = torch.arange(base, base + m, dtype=torch.int32, device=ops.device)
        keys, vals = self._sample_sort(keys, vals, 64)
        rank_new, heads, gbase = self._new_ranks(keys)
        rank_block = ops.empty(m, torch.int32)
        self._to_owners(vals, rank_new, a, n, rank_block, base)
        self.levels = [rank_block.clone()]  # level j: ranks by the first 2^j tokens (for the LCP)
        self.rounds = 1
        h = 1
        kbits = bits_for((n + 1) * (n + 1) - 1)
        while heads < n:
            # 1. rank2 = rank[i + h] for the owned i
            lo_r, hi_r = a[r] + h, min(a[r + 1] + h, n)
            send = [max(0, min(a[r + 1], a[q + 1] + h) - max(a[r], a[q] + h)) for q in range(G)]
            recv = [max(0, min(a[s + 1], hi_r) - max(a[s], lo_r)) for s in range(G)]
            first = [q for q in range(G) if send[q] > 0]
            if first:
                q0 = first[0]
                off = max(a[r], a[q0] + h) - a[r]
                payload = rank_block[off:off + sum(send)]
            else:
                payload = rank_block[:0]
            rank2 = self._all_to_all(payload, send, recv) if G > 1 else payload
            # 2-3. keys, global sort
            keys, vals = ops.keys(rank_block, rank2.contiguous(), base, n)
            keys, vals = self._sample_sort(keys, vals, kbits)
            # 4. new ranks
            rank_new, heads, gbase = self._new_ranks(keys)
            self.rounds += 1
            if heads < n:
                self._to_owners(vals, rank_new, a, n, rank_block, base)
                self.levels.append(rank_block.clone())
            h *= 2
        self.n, self.a, self.sa_part, self.gbase = n, a, vals, gbase
        return vals, gbase

    def lcp(self):
        """After run(): this rank's part of the LCP array, lcp[k] =
        LCP(SA[k], SA[k+1]) for its SA entries (0 for the global last, R3),
        by galloping over the saved levels from the highest down: per level
        every adjacent pair asks the owners of i + l and i' + l for their
        level ranks (one all-to-all each way) and extends l by 2^j where they
        agree (equal level-j ranks <=> equal 2^j-token prefixes)."""
        ops, G, r = self.ops, self.G, self.r
        n, a, sa = self.n, self.a, self.sa_part
        base = a[r]
        m = sa.numel()
        first = int(sa[0].item()) if m else -1
        info = self._all_gather_i64([m, first])
        nxt = next((info[q][1] for q in range(r + 1, G) if info[q][0] > 0), -1)
        if m == 0:  # no pairs here, but every level's collectives still run
            pa = b = ops.empty(0, torch.int32)
        elif nxt >= 0:
            b = torch.cat([sa[1:], torch.tensor([nxt], dtype=torch.int32, device=ops.device)])
            pa = sa
        else:
            b = sa[1:].contiguous()
            pa = sa[:-1].contiguous()
        npairs = pa.numel()
        lv = torch.zeros(npairs, dtype=torch.int32, device=ops.device)
        by_req = torch.tensor([-1, -2], dtype=torch.int32, device=ops.device).repeat(max(npairs, 1))[:2 * npairs]
        bk = torch.tensor(a[1:G] + [n], dtype=torch.int64, device=ops.device).view(torch.uint64)
        bv = torch.zeros(G, dtype=torch.int32, device=ops.device)
        for j in reversed(range(len(self.levels))):
            keys, vals = ops.lcp_requests(pa, b.contiguous(), lv, n)
            ops.sort(keys, vals, bits_for(n))
            cnt = ops.split(keys, vals, bk, bv, G + 1)  # per owner, then the past-the-end requests
            if G > 1:
                send, recv = self._exchange_counts(cnt[:G])
            else:
                send = recv = [int(cnt[0].item())]
            nvalid = int(sum(send))
            pos = self._u64(keys[:nvalid]).to(torch.int32)
            pos_in = self._all_to_all(pos, send, recv) if G > 1 else pos
            ans = ops.gather(pos_in, base, self.levels[j])
            resp = self._all_to_all(ans, recv, send) if G > 1 else ans
            ops.lcp_update(resp, vals[:nvalid].contiguous(), nvalid, 1 << j, by_req, lv)
        if nxt < 0 and m > 0:
            lv = torch.cat([lv, torch.zeros(1, dtype=torch.int32, device=ops.device)])
        return lv
