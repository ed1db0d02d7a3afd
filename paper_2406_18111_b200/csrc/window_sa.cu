// window_sa.cu -- K9: suffix array AND LCP array of one window per CTA, on chip.
//
// "SA, LCP <- SuffixArray(S)" (Alg. 2; "linear time algorithms
// exist for suffix array and LCP array construction") for every window
// of <= 16,384 ops of a batch (the C4 workload, the matcher's reversed
// streams, every small single window).  One persistent 1,024-thread CTA per
// SM takes windows from an atomic counter; the whole window lives in ~225 KB
// of shared memory.
//
// Suffix array: prefix doubling in the Manber-Myers formulation.  Ranks are
// Larsson-Sadakane style: rank[i] = sorted index of the first suffix of i's
// group (equal first h tokens).  If the suffixes are in an order sorted by
// their first h tokens (X), then walking that order and emitting i = X[q] - h
// lists every suffix i sorted by its SECOND key rank[i+h]; a STABLE sort of
// that list by the FIRST key rank[i] therefore orders the suffixes by their
// first 2h tokens.  So a round sorts by the group alone, never by a
// (rank, rank) pair: half the key bits.  Better still, only groups with more
// than one member can change: a round's sort key is the ordinal k of the
// item's NON-SINGLETON group (loop-shaped windows keep a few dozen to a few
// thousand of them while thousands of groups are already singletons), so a
// round is ONE stable LSD pass of bits(2 NS + 1) <= 8 bits in most rounds
// (two otherwise); singleton items keep their slot.  Suffixes i >= n - h
// (second key "end of string", the smallest) take the slots of the suffixes
// j < h, which have no predecessor i = j - h; all but i = n - h are
// singletons, and a low key bit of 0 puts i = n - h first in its group.
//
// A pass ranks 512 items per warp with match.any peer masks into a
// per-warp u16 digit histogram, one block scan gives digit starts, and items
// are scattered; the last pass of a round scatters straight to the item's new
// slot (group start of its non-singleton group + rank inside it).  Group
// heads of the new order compare (rank[i], rank[i+h]) of neighbours, a ballot
// per row of 32 slots, and the new ranks, non-singleton ordinals and group
// offsets come from popc prefix sums.
//
// Each level's ranks (u16) go to a per-CTA scratch in global memory that the
// CTA rewrites window after window (L2-resident: ~448 KB per SM), never to a
// per-position HBM array.  LCP: Kasai's bound PLCP[i] >= PLCP[i-1] - 1 over
// chunks of 16 consecutive positions per thread, direct comparison of the
// level-0 ranks (equal <=> equal tokens) in shared memory for up to 16 steps,
// galloping over the saved levels (equal level-r ranks <=> equal 2^r-token
// prefixes) for the chunk's first position and after long extensions.  The
// CTA writes only the suffix array and the LCP array to HBM.
//
// The result is the unique suffix array and its LCP array; the per-window
// arithmetic is exact integer arithmetic.
#include "pipeline.cuh"

// Phase timing (diagnostics only; compiled out unless APO_K9_PHASES is 1):
// thread 0 of every CTA adds clock64() deltas per phase to k9_phase_cycles.
#ifndef APO_K9_PHASES
#define APO_K9_PHASES 0
#endif

namespace apo {

#if APO_K9_PHASES
__device__ unsigned long long k9_phase_cycles[16];
#define K9_T0() long long k9_t = clock64()
#define K9_MARK(ph)                                                                    \
  do {                                                                                 \
    if (threadIdx.x == 0) {                                                            \
      const long long k9_n = clock64();                                                \
      atomicAdd(&k9_phase_cycles[ph], (unsigned long long)(k9_n - k9_t));               \
      k9_t = k9_n;                                                                     \
    }                                                                                  \
  } while (0)
#else
#define K9_T0()
#define K9_MARK(ph)
#endif

namespace {

using u16 = unsigned short;

constexpr int kWT = 1024;
constexpr int kWWarps = kWT / 32;
constexpr int kWItems = 16;           // slots per thread
constexpr int kWMax = kWT * kWItems;  // 16384
constexpr int kLvlSlots = 14;         // levels 0..13 (level 14, all distinct, is never needed)
constexpr int kMaxBits = 8;           // digit width cap: per-warp histograms of 256 u16 bins
constexpr u16 kSingleton = 0xFFFFu;

struct Smem {
  u32 X[kWMax];          // item buffer (sorted order: low 16 bits = position)
  u32 Y[kWMax];          // item buffer
  u16 rank[kWMax];       // rank[i] = sorted index of the first member of i's group
  u16 nsk[kWMax];        // at a group start: ordinal of the non-singleton group, kSingleton otherwise
  u16 delta[kWMax / 2];  // per non-singleton group k: number of singleton slots before its start
  u32 hbits[kWMax / 32]; // group-head bit of every slot of the current order
  union {
    u16 hist[kWWarps][1 << kMaxBits];  // LSD pass: per-warp digit counts
    struct {
      u32 sbits[kWMax / 32];  // group phase: singleton heads
      u32 nbits[kWMax / 32];  // group phase: heads of non-singleton groups
      u32 wsum[kWWarps][2];   // per-warp (non-singleton heads, singleton slots), then their exclusive prefix
      int wlast[kWWarps];     // per-warp last head slot (-1 none), then the exclusive prefix max
    } g;
  } u;
  u16 start[1 << kMaxBits];  // digit starts of a pass
  u32 scan[kWWarps];
  u32 wfirst;                // head bit of the first slot of every warp's segment (bit w)
  int misc[4];               // [0] window, [1] max id, [2] NS, [3] slot of suffix 0
};
static_assert(sizeof(Smem) <= 232448, "K9 shared memory exceeds the 227 KB opt-in limit");

__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int BITS>
__device__ __forceinline__ u32 peers_of(u32 d) {
  u32 peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const u32 m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// One stable LSD digit pass over all kWMax slots.  Warp w ranks the slots
// [512w, 512w + 512) in (row, lane) order, which is slot order, so the pass is
// stable.  digit(q): the item's digit; move(q, p): put slot q's item at rank p.
template <int BITS, class DigitF, class MoveF>
__device__ __forceinline__ void lsd_pass(Smem &S, DigitF digit, MoveF move) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RADIX = 1 << BITS;
  u16 *wh = S.u.hist[warp];
  for (int i = lane; i < (RADIX + 1) / 2; i += 32) reinterpret_cast<u32 *>(wh)[i] = 0;
  __syncwarp();
  const u32 lt = lanemask_lt();
  const int base = warp * (32 * kWItems) + lane;
  u32 rk[kWItems / 2];  // two u16 in-warp ranks per register
#pragma unroll
  for (int j = 0; j < kWItems; ++j) {
    const u32 d = digit(base + j * 32);
    // peers with the same digit: one match.any for 2+ bit digits (measured
    // 15 % faster over the whole kernel than BITS ballots), a ballot for 1 bit
    const u32 peers = BITS >= 2 ? __match_any_sync(0xffffffffu, d) : peers_of<BITS>(d);
    const u32 old = wh[d];
    __syncwarp();
    if (lane == __ffs(peers) - 1) wh[d] = u16(old + __popc(peers));
    __syncwarp();
    const u32 r = old + __popc(peers & lt);
    if (j & 1)
      rk[j >> 1] |= r << 16;
    else
      rk[j >> 1] = r;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (in place) and the digit total
  u32 total = 0;
  if (tid < RADIX) {
#pragma unroll
    for (int w = 0; w < kWWarps; ++w) {
      const u32 c = S.u.hist[w][tid];
      S.u.hist[w][tid] = u16(total);
      total += c;
    }
  }
  u32 incl = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (tid < RADIX && lane == 31) S.scan[warp] = incl;  // (RADIX < 32: warp 0 alone, no prefix needed)
  __syncthreads();
  if (tid < RADIX) {
    u32 pre = 0;
    for (int w = 0; w < warp; ++w) pre += S.scan[w];
    S.start[tid] = u16(pre + incl - total);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kWItems; ++j) {
    const int q = base + j * 32;
    const u32 d = digit(q);
    const u32 r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
    move(q, u32(S.start[d]) + wh[d] + r);
  }
  __syncthreads();
}

template <class DigitF, class MoveF>
__device__ __forceinline__ void lsd_pass_bits(int bits, Smem &S, DigitF digit, MoveF move) {
  switch (bits) {
    case 1: lsd_pass<1>(S, digit, move); break;
    case 2: lsd_pass<2>(S, digit, move); break;
    case 3: lsd_pass<3>(S, digit, move); break;
    case 4: lsd_pass<4>(S, digit, move); break;
    case 5: lsd_pass<5>(S, digit, move); break;
    case 6: lsd_pass<6>(S, digit, move); break;
    case 7: lsd_pass<7>(S, digit, move); break;
    default: lsd_pass<8>(S, digit, move); break;
  }
}

// Group phase A: the group heads of the current order ord.  head(q) = q == 0,
// or key(q) != key(q - 1), or (with OLD) q started a group before (the
// previous head bits, still in hbits).  Per row of 32 slots: head bits,
// singleton heads (a head followed by a head or the end) and non-singleton
// heads, stored as bit rows; per warp: counts and the last head.
template <bool OLD, class KeyF>
__device__ __forceinline__ void heads_phase(Smem &S, int n, KeyF key) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wb = warp * (32 * kWItems);
  // the first slot of the next warp's segment closes this warp's last row
  bool nfirst = true;
  {
    const int qn = wb + 32 * kWItems;
    if (qn < n) nfirst = (OLD && ((S.wfirst >> (warp + 1)) & 1u)) || key(qn) != key(qn - 1);
  }
  u32 prev_key = wb > 0 && wb < n ? key(wb - 1) : 0u;
  u32 cn = 0, cs = 0;
  int last = -1;
  u32 hb_prev = 0;
#pragma unroll 8
  for (int j = 0; j <= kWItems; ++j) {
    u32 hb = 0;
    if (j < kWItems) {
      const int q = wb + j * 32 + lane;
      const u32 k = q < n ? key(q) : 0u;
      u32 kp = __shfl_up_sync(0xffffffffu, k, 1);
      if (lane == 0) kp = prev_key;
      prev_key = __shfl_sync(0xffffffffu, k, 31);
      bool h = q < n && (q == 0 || k != kp);
      if (OLD && q < n) h = h || ((S.hbits[warp * kWItems + j] >> lane) & 1u);
      hb = __ballot_sync(0xffffffffu, h);
    }
    if (j > 0) {  // classify row j - 1: its successor bits are known now
      const int rb = wb + (j - 1) * 32;
      const u32 nxt = j < kWItems ? (hb & 1u) : (nfirst ? 1u : 0u);
      u32 nmask = (hb_prev >> 1) | (nxt << 31);
      if (n - 1 >= rb && n - 1 < rb + 32) nmask |= 1u << ((n - 1) & 31);  // the last slot: end follows
      const u32 single = hb_prev & nmask, nsh = hb_prev & ~nmask;
      if (lane == 0) {
        S.hbits[warp * kWItems + j - 1] = hb_prev;
        S.u.g.sbits[warp * kWItems + j - 1] = single;
        S.u.g.nbits[warp * kWItems + j - 1] = nsh;
      }
      cs += __popc(single);
      cn += __popc(nsh);
      if (hb_prev) last = rb + 31 - __clz(hb_prev);
    }
    hb_prev = hb;
  }
  if (lane == 0) {
    S.u.g.wsum[warp][0] = cn;
    S.u.g.wsum[warp][1] = cs;
    S.u.g.wlast[warp] = last;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive prefix over warps (sums; max for the last head)
    const u32 a = S.u.g.wsum[lane][0], b = S.u.g.wsum[lane][1];
    int l = S.u.g.wlast[lane];
    u32 ia = a, ib = b;
    int il = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
      const int xl = __shfl_up_sync(0xffffffffu, il, o);
      if (lane >= o) {
        ia += xa;
        ib += xb;
        il = max(il, xl);
      }
    }
    const int el = __shfl_up_sync(0xffffffffu, il, 1);
    S.u.g.wsum[lane][0] = ia - a;
    S.u.g.wsum[lane][1] = ib - b;
    S.u.g.wlast[lane] = lane ? el : -1;
    if (lane == 31) S.misc[2] = int(ia);
#if APO_K9_PHASES
    if (lane == 31) {  // slots per call and singleton slots per call (active = the rest)
      atomicAdd(&k9_phase_cycles[11], (unsigned long long)n);
      atomicAdd(&k9_phase_cycles[12], (unsigned long long)ib);
    }
#endif
    const u32 fb = __ballot_sync(0xffffffffu, (S.hbits[lane * kWItems] & 1u) != 0u);
    if (lane == 0) S.wfirst = fb;
  }
  __syncthreads();
}

// Group phase C: from the bit rows, the new ranks rank[ord[q]] = last head
// <= q, the non-singleton ordinals at group starts (nsk) and each
// non-singleton group's number of singleton slots before it (delta); the
// slot of suffix 0 goes to misc[3].  Returns NS, the number of non-singleton
// groups.
__device__ __forceinline__ int groups_phase(Smem &S, const u32 *ord, int n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = lanemask_lt();
  const u32 le = lt | (1u << lane);
  u32 nb = S.u.g.wsum[warp][0], sb = S.u.g.wsum[warp][1];
  int carry = S.u.g.wlast[warp];
#pragma unroll
  for (int j = 0; j < kWItems; ++j) {
    const int row = warp * (32 * kWItems) + j * 32;
    const int q = row + lane;
    const int rr = warp * kWItems + j;
    const u32 hb = S.hbits[rr], bn = S.u.g.nbits[rr], bs = S.u.g.sbits[rr];
    if ((bn >> lane) & 1u) {
      const u32 k = nb + __popc(bn & lt);
      S.nsk[q] = u16(k);
      S.delta[k] = u16(sb + __popc(bs & lt));
    } else if ((bs >> lane) & 1u) {
      S.nsk[q] = kSingleton;
    }
    const u32 hl = hb & le;
    const int gs = hl ? row + 31 - __clz(hl) : carry;
    if (q < n) {
      const u32 i = ord[q] & 0xffffu;
      S.rank[i] = u16(gs);
      if (i == 0) S.misc[3] = q;
    }
    nb += __popc(bn);
    sb += __popc(bs);
    if (hb) carry = row + 31 - __clz(hb);
  }
  __syncthreads();
  return S.misc[2];
}

// Equal level-r ranks <=> equal 2^r-token prefixes: greedy descent over the
// levels from a known lower bound l of lcp(i, j), valid because
// lcp(i, j) - l < 2^R (level R is all distinct).  Levels 1 .. kLvlSkip-1 are
// not kept (less scratch traffic): below level kLvlSkip the last < 2^kLvlSkip
// tokens are compared directly on the level-0 ranks in shared memory.
constexpr int kLvlSkip = 4;

__device__ __forceinline__ int gallop(const u16 *__restrict__ lv, const u16 *__restrict__ tok0, int R, int n, int i,
                                      int j, int l) {
  for (int r = R - 1; r >= kLvlSkip; --r) {
    if (i + l >= n || j + l >= n) break;
    const u16 *L = lv + size_t(r) * kWMax;
    if (__ldcg(L + i + l) == __ldcg(L + j + l)) l += 1 << r;
  }
  while (i + l < n && j + l < n && tok0[i + l] == tok0[j + l]) ++l;  // < 2^kLvlSkip steps
  return l;
}

constexpr int kKasaiSteps = 16;

// A K9 CTA needs more than half an SM's shared memory, so at most one is
// resident per SM at any time (whatever launches or streams they come
// from): the level scratch is indexed by the SM id.
static_assert(sizeof(Smem) > 116 * 1024, "K9's per-SM level scratch needs one resident CTA per SM");

__device__ __forceinline__ u32 sm_id() {
  u32 r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void k_nsmid(int *out) {
  u32 r;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(r));
  *out = int(r);
}

// ids: global dense order-preserving token ids (K2), or nullptr: level 0
// from level0 (global group starts of the (window, token) order).
__global__ void __launch_bounds__(kWT, 1)
    k_window_sa(Batch b, const u32 *__restrict__ ids, const u32 *__restrict__ slot_rank, int mirror,
                const i32 *__restrict__ level0, u16 *__restrict__ scratch,
                u32 nslots, u32 *__restrict__ next_win, i32 *__restrict__ sa_out, i32 *__restrict__ lcp_out,
                i32 *__restrict__ rw) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem &S = *reinterpret_cast<Smem *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  const u32 slot = sm_id();
  if (slot >= nslots) __trap();  // cannot happen: nslots = %nsmid
  u16 *lv = scratch + size_t(slot) * kLvlSlots * kWMax;  // this SM's level scratch
  // persistent CTAs (next_win != nullptr: windows from an atomic counter) or
  // one CTA per window
  for (int it = 0;; ++it) {
    int w = int(blockIdx.x);
    if (next_win != nullptr) {
      if (tid == 0) S.misc[0] = int(atomicAdd(next_win, 1u));
      __syncthreads();
      w = S.misc[0];
      __syncthreads();
      if (w >= b.W) return;
    } else if (it > 0) {
      return;
    }
    const i64 beg = b_beg(b, w);
    const int n = int(b_end(b, w) - beg);
    if (n <= 1) {
      if (n == 1 && tid == 0) {
        sa_out[beg] = i32(beg);
        if (lcp_out) lcp_out[beg] = 0;
      }
      if (tid == 0 && rw) rw[w] = 0;
      continue;
    }
    K9_T0();
    // ---------------- level 0: sort the window by token ----------------
    if (ids != nullptr) {
      // keys ping-pong X <-> Y, positions ping-pong rank <-> nsk
      // ids[] holds K2's table slots when slot_rank is given (the id is
      // slot_rank[slot]: no separate id pass over the batch)
      u32 mx = 0;
      if (tid == 0) S.misc[1] = 0;
      for (int q = tid; q < n; q += kWT) {
        u32 v = ids[beg + (mirror ? n - 1 - q : q)];
        if (slot_rank != nullptr) v = __ldg(&slot_rank[v]);
        S.X[q] = v;
        S.rank[q] = u16(q);
        mx = max(mx, v);
      }
      mx = __reduce_max_sync(0xffffffffu, mx);
      __syncthreads();
      if (lane == 0) atomicMax(reinterpret_cast<u32 *>(&S.misc[1]), mx);
      __syncthreads();
      const int kv = max(bits_for(u64(u32(S.misc[1]))), 1);
      const int kb = kv + (n < kWMax ? 1 : 0);  // pad slots (key 2^kv, above every id) need one more bit
      const u32 pad = 1u << kv;
      for (int q = n + tid; q < kWMax; q += kWT) {
        S.X[q] = pad;
        S.rank[q] = u16(q);
      }
      __syncthreads();
      const int np = (kb + kMaxBits - 1) / kMaxBits;
      const int bpp = (kb + np - 1) / np;
      u32 *ks = S.X, *kd = S.Y;
      u16 *ps = S.rank, *pd = S.nsk;
      for (int p = 0; p < np; ++p) {
        const int sh = p * bpp;
        const u32 m = (1u << bpp) - 1u;
        lsd_pass_bits(bpp, S, [&](int q) { return (ks[q] >> sh) & m; },
                      [&](int q, u32 to) {
                        kd[to] = ks[q];
                        pd[to] = ps[q];
                      });
        u32 *t = ks; ks = kd; kd = t;
        u16 *tp = ps; ps = pd; pd = tp;
      }
      heads_phase<false>(S, n, [&](int q) { return ks[q]; });
      for (int q = tid; q < kWMax; q += kWT) S.X[q] = ps[q];  // sorted positions (pads: >= n, unused)
      __syncthreads();
    } else {
      // level-0 group starts given: rank directly; slots by counting placement
      u32 *cnt = S.Y;
      for (int q = tid; q < kWMax; q += kWT) cnt[q] = 0;
      __syncthreads();
      for (int i = tid; i < n; i += kWT) {
        const int g = int(level0[beg + i] - beg);
        S.rank[i] = u16(g);
        S.X[g + int(atomicAdd(&cnt[g], 1u))] = u32(i);
      }
      __syncthreads();
      heads_phase<false>(S, n, [&](int q) { return u32(S.rank[S.X[q] & 0xffffu]); });
    }
    u32 *ord = S.X, *tmp = S.Y;  // ord: the current sorted order (low 16 bits = position)
    K9_MARK(0);
    int NS = groups_phase(S, ord, n);
    K9_MARK(1);
    // ---------------- doubling rounds ----------------
    int r = 0;
    while (NS > 0) {
      if (r >= kLvlSlots) {  // cannot happen for n <= 16,384 (see kLvlSlots)
        if (tid == 0 && rw) rw[w] = -1;
        break;
      }
      // level r (prefix length h = 2^r) to the scratch for the LCP stage
      // (levels 1 .. kLvlSkip-1 are not needed: see gallop)
      if (r == 0 || r >= kLvlSkip) {
        const u32 *src = reinterpret_cast<const u32 *>(S.rank);
        u32 *dst = reinterpret_cast<u32 *>(lv + size_t(r) * kWMax);
        for (int q = tid; q < kWMax / 2; q += kWT) __stcg(dst + q, src[q]);
      }
      const int h = 1 << r;
      // Manber-Myers order: the slots q of the current order list the
      // suffixes i = ord[q] - h sorted by their SECOND key; the slots of
      // j = ord[q] < h take the suffixes i = n - h + j >= n - h, whose second
      // key is "end of string", the smallest.  All of those but i = n - h
      // (exactly h tokens long) are singletons, so only i = n - h must come
      // first among its group's members: it is listed first (from the slot
      // q0 of suffix 0) and the slots before q0 move up by one.
      // key = ordinal of i's non-singleton group, NS for singletons and pads
      // (position 0xffff).
      {
        const int q0 = S.misc[3];
#pragma unroll
        for (int q = tid; q < kWMax; q += kWT) {
          if (q < n) {
            const int j = int(ord[q] & 0xffffu);
            const int i = j >= h ? j - h : n - h + j;
            const u16 k = S.nsk[S.rank[i]];
            tmp[q == q0 ? 0 : (q < q0 ? q + 1 : q)] = (u32(k == kSingleton ? NS : k) << 16) | u32(i);
          } else {
            tmp[q] = (u32(NS) << 16) | 0xffffu;
          }
        }
      }
      __syncthreads();
      K9_MARK(2);
      const int kb = bits_for(u64(NS));
      const int np = (kb + kMaxBits - 1) / kMaxBits;
      const int bpp = (kb + np - 1) / np;
      u32 *src = tmp, *dst = ord;
      for (int p = 0; p < np; ++p) {
        const int sh = 16 + p * bpp;
        const u32 m = (1u << bpp) - 1u;
        if (p + 1 < np) {
          lsd_pass_bits(bpp, S, [&](int q) { return (src[q] >> sh) & m; },
                        [&](int q, u32 to) { dst[to] = src[q]; });
          u32 *t = src; src = dst; dst = t;
        } else {
          // last pass: scatter to the new slot.  Non-singleton group k's items
          // come out contiguous in MM order; its slots start delta[k] later
          // (the singleton slots before it); a singleton keeps its slot.  The
          // item is stored with its second key r2 = rank[i+h] + 1 (0 past the
          // end) in the high half, for the head test of the new order.
          lsd_pass_bits(bpp, S, [&](int q) { return (src[q] >> sh) & m; },
                        [&](int q, u32 to) {
                          const u32 v = src[q];
                          const u32 k = v >> 16, i = v & 0xffffu;
                          if (i == 0xffffu) return;
                          const u32 at = k < u32(NS) ? to + S.delta[k] : u32(S.rank[i]);
                          const u32 r2 = int(i) + h < n ? u32(S.rank[i + h]) + 1u : 0u;
                          dst[at] = (r2 << 16) | i;
                        });
          ord = dst;  // the new order (src's items are consumed)
          tmp = src;
        }
      }
      K9_MARK(3);
#if APO_K9_PHASES
      if (threadIdx.x == 0) atomicAdd(&k9_phase_cycles[8 + np], 1ull);
#endif
      // heads of the new order: an old group start, or the second key differs
      // from the previous slot's (within an old group the first keys agree)
      heads_phase<true>(S, n, [&](int q) { return ord[q] >> 16; });
      K9_MARK(4);
      NS = groups_phase(S, ord, n);
      K9_MARK(1);
      ++r;
    }
    // ---------------- LCP (Kasai chunks + galloping over the levels) ----------------
    // ord: suffix array (low 16 bits); rank: inverse suffix array; levels 0..r-1 in lv
    u16 *tok0 = reinterpret_cast<u16 *>(tmp);  // level-0 ranks (equal <=> equal tokens)
    u16 *lcps = tok0 + kWMax;                  // lcps[k] = LCP(SA[k], SA[k+1])
    const int R = r;
    if (lcp_out) {
      if (R > 0) {
        const u32 *src = reinterpret_cast<const u32 *>(lv);
        u32 *dst = reinterpret_cast<u32 *>(tok0);
        for (int q = tid; q < kWMax / 2; q += kWT) dst[q] = __ldcg(src + q);
      }
      __syncthreads();
      const int i0 = tid * kWItems, i1 = min(i0 + kWItems, n);
      int l = -1;
      for (int i = i0; i < i1; ++i) {
        const int q = S.rank[i];
        if (q == 0) {
          l = 0;
          continue;
        }
        const int j = int(ord[q - 1] & 0xffffu);
        if (R == 0) {
          l = 0;  // all first tokens distinct
        } else if (l < 0) {
          l = gallop(lv, tok0, R, n, i, j, 0);
        } else {
          l = l > 0 ? l - 1 : 0;
          int steps = 0;
          while (i + l < n && j + l < n && tok0[i + l] == tok0[j + l]) {
            ++l;
            if (++steps == kKasaiSteps) {
              l = gallop(lv, tok0, R, n, i, j, l);
              break;
            }
          }
        }
        lcps[q - 1] = u16(l);
      }
      __syncthreads();
    }
    K9_MARK(5);
    for (int q = tid; q < n; q += kWT) {
      sa_out[beg + q] = i32(beg) + i32(ord[q] & 0xffffu);
      if (lcp_out) lcp_out[beg + q] = q + 1 < n ? i32(lcps[q]) : 0;
    }
    if (tid == 0 && rw) rw[w] = R;
    __syncthreads();
    K9_MARK(6);
  }
}

}  // namespace

bool window_sa_supported(const Batch &b) { return !b.gen && b.maxwin <= kWMax; }

int query_nsmid(int device) {
  int *d = nullptr, h = 0;
  APO_CUDA(cudaSetDevice(device));
  APO_CUDA(cudaMalloc(&d, sizeof(int)));
  k_nsmid<<<1, 1>>>(d);
  APO_CHECK_LAUNCH();
  APO_CUDA(cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost));
  APO_CUDA(cudaFree(d));
  return h;
}

size_t window_sa_scratch_bytes(int nsmid) {
  return size_t(std::max(nsmid, 1)) * kLvlSlots * kWMax * sizeof(u16);
}

void run_window_sa(Ctx &c, const Batch &b, SAWork &w, bool want_lcp, cudaStream_t s) {
  const size_t smem = sizeof(Smem);
  c.smem_optin(reinterpret_cast<const void *>(k_window_sa), smem);
  if (c.prof) c.prof_begin(kProfWindowSA, 0.0, s);
  // persistent CTAs, one per SM (measured 3 % faster than one CTA per
  // window: no per-window CTA launch and teardown)
  const int grid = int(std::min<i64>(b.W, c.num_sms));
  u32 *ctr = c.take_counter(s);
  k_window_sa<<<grid, kWT, smem, s>>>(b, w.ids_valid ? w.ids : nullptr, w.ids_valid ? w.slot_rank : nullptr,
                                      w.ids_valid && w.mirror ? 1 : 0,
                                      w.levels[0],
                                      reinterpret_cast<u16 *>(w.win_scratch), u32(c.nsmid), ctr, w.sa,
                                      want_lcp ? w.lcp : nullptr, w.rw);
  APO_CHECK_LAUNCH();
  if (c.prof) c.prof_end(s);
  c.launches++;
}

}  // namespace apo

#if APO_K9_PHASES
extern "C" int apo_debug_k9_phases(unsigned long long *out, int reset) {
  if (cudaMemcpyFromSymbol(out, apo::k9_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(apo::k9_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif
