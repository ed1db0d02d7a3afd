// window_sa.cu -- K9: prefix doubling of one window per CTA, on chip.
//
// For batches whose windows hold <= 16,384 ops (the C4 workload, and every
// small single window) the whole doubling loop of a window runs inside one
// 1024-thread CTA.  Per round:
//   * keys (rank[i] << bg | (i+h < n ? rank[i+h]+1 : 0)) and positions are
//     built from the u16 DENSE group ids held in shared memory; with G
//     groups a key needs bits(G-1) + bits(G) bits, and loop-shaped windows
//     keep G small for many rounds, so a round takes 2-4 passes, not 4;
//   * stable 8-bit LSD digit passes move (key u32, position u16) between two
//     shared-memory buffers: each warp ranks its 512 items (peer masks from
//     ballots) into a per-warp u16 histogram, one block scan gives the digit
//     starts, and every item is scattered to its slot;
//   * a block-wide sum-scan of group heads gives the new dense ids;
//   * the new level is streamed to HBM (4 B/op) for the LCP stage's galloping.
// The loop ends per window as soon as all its ranks are distinct.  HBM
// traffic per round is the level write only, instead of ~140 B/op for a
// round of the global onesweep path.  The result is the same suffix array
// (it is unique).
#include "pipeline.cuh"

namespace apo {

namespace {

constexpr int kWT = 1024;
constexpr int kWWarps = kWT / 32;
constexpr int kWItems = 16;
constexpr int kWMax = kWT * kWItems;  // 16384

struct WinBuf {
  u32 key[kWMax];
  unsigned short pos[kWMax];
};

struct WinSmem {
  WinBuf a, b;  // ping-pong; the u16 rank array aliases b.key while a holds the items
  unsigned short hist[kWWarps][512];  // per-warp digit counts (digits of up to 9 bits)
  unsigned short start[512];  // digit starts (<= 16,384)
  u32 scan[kWWarps];
};

template <int BITS>
__device__ __forceinline__ u32 peers_ballot_w(u32 d) {
  u32 peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const u32 m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

__device__ __forceinline__ u32 lanemask_lt_w() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// One stable LSD digit pass: items of `src` (sorted position q = index) go to
// `dst`.  Warp w ranks the contiguous sub-tile [w*512, w*512+512) in
// (j, lane) order, which is index order, so the pass is stable.
template <int SHIFT, int BITS>
__device__ __forceinline__ void lsd_pass(const WinBuf &src, WinBuf &dst, WinSmem &S) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RADIX = 1 << BITS;
  constexpr u32 mask = RADIX - 1u;
  unsigned short *wh = S.hist[warp];
  {  // each warp clears its own histogram row (the previous pass ended with a barrier)
    u32 *row = reinterpret_cast<u32 *>(wh);
#pragma unroll
    for (int i = lane; i < RADIX / 2; i += 32) row[i] = 0;
    __syncwarp();
  }
  const u32 lt = lanemask_lt_w();
  const int base = warp * (32 * kWItems) + lane;
  u32 rk[kWItems / 2];  // two u16 in-warp ranks per register
#pragma unroll
  for (int j = 0; j < kWItems; ++j) {
    u32 d = (src.key[base + j * 32] >> SHIFT) & mask;
    u32 peers = peers_ballot_w<BITS>(d);
    u32 old = wh[d];
    __syncwarp();
    if (lane == __ffs(peers) - 1) wh[d] = (unsigned short)(old + __popc(peers));
    __syncwarp();
    u32 r = old + __popc(peers & lt);
    if (j & 1)
      rk[j >> 1] |= r << 16;
    else
      rk[j >> 1] = r;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (in place) and the digit total
  u32 total = 0;
  if (tid < RADIX) {
#pragma unroll 8
    for (int w = 0; w < kWWarps; ++w) {
      u32 c = S.hist[w][tid];
      S.hist[w][tid] = (unsigned short)total;
      total += c;
    }
  }
  u32 incl = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (tid < RADIX && lane == 31) S.scan[warp] = incl;
  __syncthreads();
  if (tid < RADIX) {
    u32 pre = 0;
    for (int w = 0; w < warp; ++w) pre += S.scan[w];
    S.start[tid] = (unsigned short)(pre + incl - total);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kWItems; ++j) {
    const int q = base + j * 32;
    u32 k = src.key[q];
    u32 d = (k >> SHIFT) & mask;
    u32 r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
    u32 p = u32(S.start[d]) + wh[d] + r;
    dst.key[p] = k;
    dst.pos[p] = src.pos[q];
  }
  __syncthreads();
}

// Sort the items of buffer X (keys, positions) with NP stable LSD passes of
// W-bit digits (the sorted items end in X for even NP, in Y for odd NP).
template <int NP, int W>
__device__ __forceinline__ void lsd_passes(WinBuf &X, WinBuf &Y, WinSmem &S) {
  lsd_pass<0, W>(X, Y, S);
  if constexpr (NP >= 2) lsd_pass<W, W>(Y, X, S);
  if constexpr (NP >= 3) lsd_pass<2 * W, W>(X, Y, S);
  if constexpr (NP >= 4) lsd_pass<3 * W, W>(Y, X, S);
}

// Dense id of every sorted item's key group, stored at rank[pos], and the
// sorted index of every group's first item at gstart[id] (gstart = rank +
// kWMax: the upper half of the same key area).  Warp w owns the sorted items
// [512w, 512w+512) and walks them in 16 rows of 32 consecutive items
// (conflict-free shared-memory access): a row's group heads come from one
// ballot, the running count from popc.  KeyAt(q) gives the key of sorted
// item q.  Returns the number of groups among the first n items.
template <class KeyAt>
__device__ __forceinline__ u32 dense_rank_by(KeyAt key_at, const unsigned short *spos, unsigned short *rank, i64 n,
                                             WinSmem &S) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wbase = warp * (32 * kWItems);
  const u32 lt = lanemask_lt_w();
  unsigned short *gstart = rank + kWMax;
  // pass 1: heads of this warp's segment
  u32 cnt = 0;
#pragma unroll 4
  for (int j = 0; j < kWItems; ++j) {
    const int q = wbase + j * 32 + lane;
    const u32 k = q < n ? key_at(q) : 0u;
    const u32 pk = (q > 0 && q < n) ? key_at(q - 1) : 0xffffffffu;
    cnt += __popc(__ballot_sync(0xffffffffu, k != pk && q < n));
  }
  if (lane == 0) S.scan[warp] = cnt;
  __syncthreads();
  u32 before = 0, total = 0;
  for (int ww = 0; ww < kWWarps; ++ww) {
    const u32 v = S.scan[ww];
    if (ww < warp) before += v;
    total += v;
  }
  // pass 2: ids
  u32 run = before;  // heads before the current row
#pragma unroll 4
  for (int j = 0; j < kWItems; ++j) {
    const int q = wbase + j * 32 + lane;
    const u32 k = q < n ? key_at(q) : 0u;
    const u32 pk = (q > 0 && q < n) ? key_at(q - 1) : 0xffffffffu;
    const bool head = k != pk && q < n;
    const u32 hb = __ballot_sync(0xffffffffu, head);
    const u32 id = run + __popc(hb & lt) + ((hb >> lane) & 1u);  // heads up to and including q
    if (q < n) rank[spos[q]] = (unsigned short)(id - 1);
    if (head) gstart[id - 1] = (unsigned short)q;
    run += __popc(hb);
  }
  __syncthreads();
  return total;
}

__device__ __forceinline__ u32 dense_rank(const WinBuf &sorted, unsigned short *rank, i64 n, WinSmem &S) {
  return dense_rank_by([&](int q) { return sorted.key[q]; }, sorted.pos, rank, n, S);
}

// Largest group of the current ranking (group starts from dense_rank).
__device__ __forceinline__ u32 max_group(const unsigned short *rank, u32 G, i64 n) {
  __shared__ u32 s_mx;
  if (threadIdx.x == 0) s_mx = 0;
  __syncthreads();
  const unsigned short *gstart = rank + kWMax;
  u32 mx = 0;
  for (u32 g = threadIdx.x; g < G; g += kWT) {
    const u32 e = g + 1 < G ? u32(gstart[g + 1]) : u32(n);
    mx = max(mx, e - u32(gstart[g]));
  }
  atomicMax(&s_mx, mx);
  __syncthreads();
  const u32 r = s_mx;
  __syncthreads();
  return r;
}

// One doubling round when every current group holds at most kSmallGroup (64)
// items (late rounds of loop-shaped windows): the items are still in sorted
// order of their current rank, so only each group's members need ordering by
// rank[i + h]; an item's new sorted index is its group's start plus the
// number of members ordered before it (by rank[i+h], ties by current index).
// Reads sorted positions P.pos and ranks R.key; writes the new order to
// R.pos, then the new ranks (and group starts) to P.key.  No LSD pass.
constexpr u32 kSmallGroup = 64;

__device__ __forceinline__ u32 small_group_round(WinBuf &P, WinBuf &R, u32 G, i64 n, i64 h, int bg, WinSmem &S) {
  const unsigned short *rank = reinterpret_cast<const unsigned short *>(R.key);
  const unsigned short *gstart = rank + kWMax;
  auto r2 = [&](u32 p) -> u32 { return (i64(p) + h < n) ? u32(rank[p + h]) + 1u : 0u; };
  u32 *R2 = P.key;  // second keys in current sorted order (P.key is free until the new ranks)
  for (int q = threadIdx.x; q < n; q += kWT) R2[q] = r2(P.pos[q]);
  __syncthreads();
  for (int q = threadIdx.x; q < n; q += kWT) {
    const u32 p = P.pos[q];
    const u32 g = rank[p];
    const u32 a = gstart[g], b = g + 1 < G ? u32(gstart[g + 1]) : u32(n);
    u32 nq = u32(q);
    if (b - a > 1) {
      const u32 mine = R2[q];
      u32 c = 0;
      for (u32 j = a; j < b; ++j) {
        const u32 o = R2[j];
        c += (o < mine) || (o == mine && j < u32(q));
      }
      nq = a + c;
    }
    R.pos[nq] = (unsigned short)p;
  }
  __syncthreads();
  unsigned short *nrank = reinterpret_cast<unsigned short *>(P.key);
  return dense_rank_by([&](int q) {
    const u32 p = R.pos[q];
    return (u32(rank[p]) << bg) | r2(p);
  }, R.pos, nrank, n, S);
}

template <int NP, int W, bool XA>  // XA: items in S.a, other buffer S.b
__device__ __forceinline__ void sort_round(WinSmem &S) {
  if constexpr (XA)
    lsd_passes<NP, W>(S.a, S.b, S);
  else
    lsd_passes<NP, W>(S.b, S.a, S);
}

template <bool XA>
__device__ __forceinline__ int sort_items_x(WinSmem &S, int bits) {
  // fewest passes, 8-bit digits where that many passes suffice (8 ballots per
  // item instead of 9): 8 | 9 | 16 | 18 | 24 | 27 | 32 bits
  if (bits <= 8) { sort_round<1, 8, XA>(S); return 1; }
  if (bits <= 9) { sort_round<1, 9, XA>(S); return 1; }
  if (bits <= 16) { sort_round<2, 8, XA>(S); return 2; }
  if (bits <= 18) { sort_round<2, 9, XA>(S); return 2; }
  if (bits <= 24) { sort_round<3, 8, XA>(S); return 3; }
  if (bits <= 27) { sort_round<3, 9, XA>(S); return 3; }
  sort_round<4, 8, XA>(S);
  return 4;
}

// Sort the items (keys of `bits` significant bits) built in S.a (xa) or
// S.b; returns the number of passes (odd: the items end in the other buffer)
__device__ __forceinline__ int sort_items(WinSmem &S, int bits, bool xa) {
  return xa ? sort_items_x<true>(S, bits) : sort_items_x<false>(S, bits);
}

// Algorithmic shared-memory traffic (profiling only): every LSD pass reads
// and writes each item once (key 4 B + position 2 B, each way) and reads its
// digit + updates a counter (8 B): 20 B per item per pass; building a round's
// items reads two ranks and writes one item (10 B); the dense ranks read the
// sorted item and write a rank (8 B).
constexpr u64 kSmemPassBytes = 20, kSmemRoundBytes = 18;

// ids: dense token ids (level 0 is computed here: window-local dense ranks
// of the tokens), or nullptr to take level 0 from levels[0].
__global__ void __launch_bounds__(kWT, 1) k_window_sa(Batch b, const u32 *__restrict__ ids, LevelPtrs lv,
                                                      int max_levels, i32 *__restrict__ sa_out,
                                                      i32 *__restrict__ rw, unsigned long long *smem_bytes,
                                                      i32 *__restrict__ phi_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WinSmem &S = *reinterpret_cast<WinSmem *>(smem_raw);
  const int tid = threadIdx.x;
  const int w = blockIdx.x;
  const i64 beg = b_beg(b, w), n = b_end(b, w) - beg;
  if (n == 0) {
    if (tid == 0) rw[w] = 0;
    return;
  }
  u64 prof = 0;
  // The items of a round are built in buffer X and sorted with np passes;
  // they end in X (np even) or in the other buffer.  The u16 ranks live in
  // the key area of the buffer NOT holding the sorted items.
  bool rank_in_b = true;  // ranks in S.b.key, items built in S.a
  bool sorted_in_a = true;
  u32 G;                 // number of distinct ranks
  u32 maxg = 0xffffffffu;  // largest group (unknown: the first round sorts)
  auto rank_ptr = [&]() { return reinterpret_cast<unsigned short *>(rank_in_b ? S.b.key : S.a.key); };
  // ---- level 0 ----
  if (ids != nullptr) {
    __shared__ u32 s_max;
    if (tid == 0) s_max = 0;
    __syncthreads();
    u32 mx = 0;
    for (int q = tid; q < n; q += kWT) mx = max(mx, ids[beg + q]);
    atomicMax(&s_max, mx);
    __syncthreads();
    const int kb = bits_for(u64(s_max));
    const u32 pad = 1u << kb;
    for (int q = tid; q < kWMax; q += kWT) {  // items into S.a
      S.a.key[q] = q < n ? ids[beg + q] : pad;
      S.a.pos[q] = (unsigned short)q;
    }
    __syncthreads();
    const int np = sort_items(S, kb + (n < kWMax ? 1 : 0), true);  // pad items need one more bit
    sorted_in_a = (np & 1) == 0;
    rank_in_b = sorted_in_a;
    G = dense_rank(sorted_in_a ? S.a : S.b, rank_ptr(), n, S);
    maxg = max_group(rank_ptr(), G, n);
    prof += u64(n) * (kSmemPassBytes * np + kSmemRoundBytes);
    unsigned short *rank = rank_ptr();
    i32 *out = lv.p[0];
    for (int i = tid; i < n; i += kWT) out[beg + i] = i32(rank[i]) + i32(beg);
  } else {
    const i32 *level0 = lv.p[0];
    unsigned short *rank = rank_ptr();
    for (int i = tid; i < n; i += kWT) rank[i] = (unsigned short)(level0[beg + i] - beg);
    G = 0;  // unknown: group starts are < n
    __syncthreads();
  }
  int r = 0;
  for (i64 h = 1;; h <<= 1) {
    if (G == u32(n)) {  // all distinct: the sorted buffer is the suffix array
      const unsigned short *pos = sorted_in_a ? S.a.pos : S.b.pos;
      for (int q = tid; q < n; q += kWT) {
        sa_out[beg + q] = i32(beg) + i32(pos[q]);
        // phi of the LCP stage (K4): the suffix ranked just before, -1 for the first
        if (phi_out) phi_out[beg + pos[q]] = q > 0 ? i32(beg) + i32(pos[q - 1]) : -1;
      }
      if (tid == 0) {
        rw[w] = r;
        if (smem_bytes) atomicAdd(smem_bytes, (unsigned long long)prof);
      }
      return;
    }
    // key = rank[i] << bg | (i + h < n ? rank[i+h] + 1 : 0); ranks < G
    const u32 gmax = G ? G : u32(n);
    const int bg = bits_for(u64(gmax));
    if (G && maxg <= kSmallGroup) {
      // small groups only: order each group's members in place of a sort
      WinBuf &P = sorted_in_a ? S.a : S.b, &R = sorted_in_a ? S.b : S.a;
      G = small_group_round(P, R, G, n, h, bg, S);
      sorted_in_a = !sorted_in_a;
      rank_in_b = sorted_in_a;
      prof += u64(n) * kSmemRoundBytes * 2;
    } else {
      const int kb = bits_for(u64(gmax - 1)) + bg;
      const u32 pad = 1u << kb;
      const unsigned short *rank = rank_ptr();
      const bool xa = rank_in_b;  // items go to the buffer without the ranks
      u32 *xk = xa ? S.a.key : S.b.key;
      unsigned short *xp = xa ? S.a.pos : S.b.pos;
      for (int q = tid; q < kWMax; q += kWT) {
        u32 key = pad;
        if (q < n) {
          const u32 lo = (q + h < n) ? u32(rank[q + h]) + 1u : 0u;
          key = (u32(rank[q]) << bg) | lo;
        }
        xk[q] = key;
        xp[q] = (unsigned short)q;
      }
      __syncthreads();
      const int np = sort_items(S, kb + (n < kWMax ? 1 : 0), xa);  // pad items need one more bit
      sorted_in_a = ((np & 1) == 0) == xa;
      rank_in_b = sorted_in_a;
      G = dense_rank(sorted_in_a ? S.a : S.b, rank_ptr(), n, S);
      prof += u64(n) * (kSmemPassBytes * np + kSmemRoundBytes);
    }
    unsigned short *nrank = rank_ptr();
    maxg = max_group(nrank, G, n);
    ++r;
    if (r < max_levels) {
      i32 *out = lv.p[r];
      for (int i = tid; i < n; i += kWT) out[beg + i] = i32(nrank[i]) + i32(beg);
    }
    if (r + 1 >= max_levels && G < u32(n)) {  // level budget exhausted (cannot happen for n <= 2^14)
      if (tid == 0) rw[w] = -1;
      return;
    }
  }
}

}  // namespace

bool window_sa_supported(const Batch &b) { return !b.gen && b.maxwin <= kWMax; }

void run_window_sa(Ctx &c, const Batch &b, SAWork &w, cudaStream_t s) {
  const size_t smem = sizeof(WinSmem);
  c.smem_optin(reinterpret_cast<const void *>(k_window_sa), smem);
  LevelPtrs lv{};
  for (int r = 0; r < w.max_levels && r < 40; ++r) lv.p[r] = w.levels[r];
  if (c.prof) c.prof_begin(kProfWindowSA, 0.0, s);
  unsigned long long *cnt =
      c.prof ? reinterpret_cast<unsigned long long *>(c.d_misc + kProfDevSlot + kProfWindowSA) : nullptr;
  k_window_sa<<<b.W, kWT, smem, s>>>(b, w.ids_valid ? w.ids : nullptr, lv, w.max_levels, w.sa, w.rw, cnt, w.phi);
  APO_CHECK_LAUNCH();
  if (c.prof) c.prof_end(s);
  c.launches++;
}

}  // namespace apo
