// select.cu -- K5..K8: Alg. 2 after the suffix array.
//
// K5 candidate generation.  For every rank-adjacent pair k of a
//    window: s1, s2, p = SA[k], SA[k+1], LCP[k]; disjoint (|s2-s1| >= p,
//    reading R4) -> (p, s1), (p, s2); otherwise d = |s2-s1|,
//    l = floor((p+d)/2), l -= l % d -> (l, m), (l, m+l) with m = min(s1,s2)
//    (R5, R6).  Kept iff l >= min_len (R7).  Compacted with a single-pass
//    scan; emitted in pair order.
// K6 ordering.  The paper sorts by (length desc,
//    sub-string asc, start asc).  For equal length, the sub-string of pair k
//    is the l-prefix of the suffix of rank k, so sub-string order is rank
//    order: a STABLE radix sort of the pair-ordered candidates by
//    (window, length desc) already yields sub-string order.  Two neighbours
//    of pairs k1 <= k2 are the same sub-string iff k1 == k2 or
//    min LCP[k1..k2-1] >= l (O(1) range-minimum over a sparse table).  The
//    dense group ordinal is the paper's sub-string ID; a second radix sort by
//    (ID, start) puts each group in start order.
// K7 greedy non-overlap selection computed EXACTLY in rounds
//    (lexicographically-first independent set): with priority = position in
//    the sorted order, an undecided candidate is selected when no undecided
//    candidate of higher priority covers its first or last position (any
//    earlier -- hence not shorter -- overlapping interval must cover one of
//    them), and rejected once a selected interval covers its first or last
//    position (the paper's marked-array test).  firstcov(x) comes
//    from a reverse sparse table (two atomicMin per interval, then a pull-down
//    over levels); coverage from a +/-1 difference array and a scan.
//    For batches of small windows (<= 16,384 ops) the paper's own sequential
//    loop is faster: one warp per window walks the window's sorted
//    candidates with the marked array as a shared-memory bitset
//    (k_greedy_window), every window at once.
// K8 dedup/output (R10, R11).
#include <cstdlib>

#include "pipeline.cuh"

namespace apo {

namespace {

constexpr int T = 256;

struct CandF {
  Batch b;
  const i32 *sa;
  const i32 *lcp;
  i32 min_len;
  int bl;
  i64 maxl;
  i64 npairs;
  u32 *k1;
  u64 *v1;
  i64 *m_out;
  __device__ __forceinline__ bool pair(i64 k, i64 &l, i64 &a, i64 &bb, int &w) const {
    // the SA is window-major: rank k belongs to the window of position k
    // (a sequential read, not a random one at SA[k]); all loads are issued
    // before any branch, and the arithmetic is 32-bit (positions < 2^31)
    w = b_wid(b, k);
    const i64 e = b_end(b, w);
    const bool ok = k + 1 < e;
    const u32 s1 = u32(sa[k]), s2 = u32(sa[ok ? k + 1 : k]), p = u32(lcp[k]);
    if (!ok) return false;
    const u32 lo = s1 < s2 ? s1 : s2, d = s1 < s2 ? s2 - s1 : s1 - s2;
    if (d >= p) {
      l = p;
      a = s1;
      bb = s2;
    } else {
      u32 L = (p + d) >> 1;
      L -= L % d;
      l = L;
      a = lo;
      bb = lo + L;
    }
    return l >= min_len;
  }
  __device__ u32 load(i64 k) const {
    i64 l, a, bb;
    int w;
    return pair(k, l, a, bb, w) ? 1u : 0u;
  }
  __device__ bool store(i64 k, u32 incl, u32 excl) const {
    i64 l, a, bb;
    int w;
    if (pair(k, l, a, bb, w)) {
      u32 key = (u32(w) << bl) | u32(maxl - l);
      i64 o = 2 * i64(excl);  // even: the pair's two records go out as one 8-B and one 16-B store
      reinterpret_cast<uint2 *>(k1)[o >> 1] = make_uint2(key, key);
      reinterpret_cast<ulonglong2 *>(v1)[o >> 1] =
          make_ulonglong2((u64(k) << 32) | u64(a), (u64(k) << 32) | u64(bb));
    }
    if (k == npairs - 1) *m_out = 2 * i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

// Range minimum over the LCP array for the group-head test of K6: blocks of
// 32 entries with in-block prefix / suffix minima (one warp scan per block)
// and a sparse table over the block minima only, so the table costs
// ~bits(maxwin/32) passes over N/32 entries instead of bits(maxwin) passes
// over N; a query inside one block scans it directly (<= 32 L1-resident
// entries).
struct Rmq {
  const i32 *lcp;
  const i32 *pre, *suf;  // min of LCP[block start .. j], LCP[j .. block end]
  const i32 *lv[32];     // lv[0] = block minima, lv[j] = min over 2^j blocks
  __device__ __forceinline__ i32 min(i64 a, i64 b) const {  // inclusive, a <= b
    const i64 ba = a >> 5, bb = b >> 5;
    if (ba == bb) {
      i32 x = lcp[a];
      for (i64 j = a + 1; j <= b; ++j) x = lcp[j] < x ? lcp[j] : x;
      return x;
    }
    i32 x = suf[a] < pre[b] ? suf[a] : pre[b];
    if (bb - ba > 1) {
      const i64 l = ba + 1, r = bb - 1;
      const int j = 63 - __clzll(r - l + 1);
      const i32 y = lv[j][l], z = lv[j][r - (i64(1) << j) + 1];
      x = y < x ? y : x;
      x = z < x ? z : x;
    }
    return x;
  }
};

__global__ void k_rmq_blocks(const i32 *__restrict__ lcp, i64 n, i32 *__restrict__ pre, i32 *__restrict__ suf,
                             i32 *__restrict__ bmin) {
  const i64 j = i64(blockIdx.x) * blockDim.x + threadIdx.x;  // blockDim is a multiple of 32
  const int lane = threadIdx.x & 31;
  const i32 v = j < n ? lcp[j] : 0x7fffffff;
  i32 up = v, dn = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const i32 a = __shfl_up_sync(0xffffffffu, up, d), b = __shfl_down_sync(0xffffffffu, dn, d);
    if (lane >= d) up = a < up ? a : up;
    if (lane + d < 32) dn = b < dn ? b : dn;
  }
  if (j < n) {
    pre[j] = up;
    suf[j] = dn;
  }
  if (lane == 31 && (j - 31) < n) bmin[j >> 5] = up;
}

__global__ void k_rmq_level(const i32 *__restrict__ prev, i32 *__restrict__ next, i64 n, i64 half) {
  i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  i32 x = prev[k];
  if (k + half < n) {
    i32 y = prev[k + half];
    x = y < x ? y : x;
  }
  next[k] = x;
}

// Group heads of the sort-1 order, one thread per candidate (all loads in
// flight at once; the scan that numbers the groups then reads one byte per
// candidate): a candidate starts a group unless the previous one has the same
// (window, length) and the same sub-string -- the same pair, or pairs whose
// SA ranks kp < kc have min LCP[kp .. kc-1] >= length.
__global__ void k_head_flags(const u32 *__restrict__ k1, const u64 *__restrict__ v1, Rmq rmq, i64 maxl, u32 lmask,
                             i64 m, u8 *__restrict__ head) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m) return;
  if (c == 0) {
    head[0] = 1;
    return;
  }
  const u32 a = k1[c], b = k1[c - 1];
  const u64 va = v1[c], vb = v1[c - 1];
  u8 h = 1;
  if (a == b) {
    const i64 kc = i64(va >> 32), kp = i64(vb >> 32);
    h = (kc == kp) ? 0 : (rmq.min(kp, kc - 1) < maxl - i64(a & lmask) ? 1 : 0);
  }
  head[c] = h;
}

// sort-2 keys (group, window-local start): a group never spans windows, so
// the local start orders it as the global one does, in bits(maxwin) bits
// instead of bits(N); the group's window base is kept aside (gbase)
struct HeadF {
  const u32 *k1;
  const u64 *v1;
  i64 maxl;
  u32 lmask;
  int bL;
  i64 m;
  u64 *k2;
  i32 *glen;
  i64 *G_out;
  const i64 *off;
  const i32 *wid;  // NULL for one window
  int bW;          // window field of the sort-1 key starts at bit bW
  i32 *gbase;
  i32 *gwin;       // window of the group
  u32 *gpos;       // position of the group's first member in sort-1 order
  const u8 *head;  // group-head flags from k_head_flags
  __device__ u32 load(i64 c) const { return head[c]; }
  __device__ bool store(i64 c, u32 incl, u32 excl) const {
    u64 g = u64(incl - 1);
    const i64 s = i64(v1[c] & 0xffffffffull);
    const i64 base = wid ? off[k1[c] >> bW] : 0;  // the window is the key's high field
    k2[c] = (g << bL) | u64(s - base);
    if (incl != excl) {
      glen[g] = i32(maxl - i64(k1[c] & lmask));
      gbase[g] = i32(base);
      gwin[g] = wid ? i32(k1[c] >> bW) : 0;
      gpos[g] = u32(c);
    }
    if (c == m - 1) *G_out = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_unpack(const u64 *__restrict__ k2, i64 m, int bL, const i32 *__restrict__ glen,
                         const i32 *__restrict__ gbase, i32 *__restrict__ cl, i32 *__restrict__ cs,
                         i32 *__restrict__ cg, u8 *__restrict__ state) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m) return;
  u64 key = k2[c];
  i32 g = i32(key >> bL);
  cs[c] = gbase[g] + i32(key & ((1ull << bL) - 1));
  cg[c] = g;
  cl[c] = glen[g];
  state[c] = 0;
}

// Sort-2 without a radix sort when every group is small (the common case:
// ~2 members per group on C4).  In sort-1 order the members of a group are
// already contiguous (same window and length, SA ranks of one LCP interval),
// so only the members of each group need ordering by start: an item's place
// is its group's first position plus the number of members with a smaller
// (local start, position) -- and the unpacking of k_unpack happens in the
// same pass.  A group larger than kSegMax sets *big and the caller falls
// back to the radix sort.
constexpr u32 kSegMax = 64;

__global__ void k_seg_unpack(const u64 *__restrict__ k2, i64 m, i64 G, int bL, const u32 *__restrict__ gpos,
                             const i32 *__restrict__ glen, const i32 *__restrict__ gbase, i32 *__restrict__ cl,
                             i32 *__restrict__ cs, i32 *__restrict__ cg, u8 *__restrict__ state,
                             u32 *__restrict__ big) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const u64 key = k2[c];
  const i64 g = i64(key >> bL);
  const i64 gs = gpos[g], ge = g + 1 < G ? i64(gpos[g + 1]) : m;
  if (ge - gs > kSegMax) {
    atomicOr(big, 1u);
    return;
  }
  i64 r = 0;
  for (i64 j = gs; j < ge; ++j) {
    const u64 o = k2[j];
    r += (o < key) || (o == key && j < c);
  }
  const i64 p = gs + r;
  cs[p] = gbase[g] + i32(key & ((1ull << bL) - 1));
  cg[p] = i32(g);
  cl[p] = glen[g];
  state[p] = 0;
}

// K6 sort-1 for batches of small windows: the candidates come out of K5 in
// pair order, i.e. already grouped by window, so only the length field needs
// sorting, and only inside each window.  One 1,024-thread CTA per window runs
// a stable two-pass LSD counting sort on the (maxl - length) field (7 + 7
// bits for windows <= 16,384 ops) over its own segment: a histogram of both
// digits, then per pass the segment's tiles of 4,096 in order, each ranked
// with the ballot multisplit and scattered behind the previous tiles (no
// global look-back, no window bits in the key).
constexpr int kSegThreads = 1024;
constexpr int kSegItems = 4;
constexpr int kSegTile = kSegThreads * kSegItems;

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

template <int SHIFT, int BITS>
__device__ __forceinline__ void seg_pass(const u32 *__restrict__ kin, const u64 *__restrict__ vin,
                                         u32 *__restrict__ kout, u64 *__restrict__ vout, i64 c0, i64 c1,
                                         u32 lmask, u32 *s_base, unsigned short (*s_wh)[128], u32 *s_tot,
                                         u32 *s_tdig, u32 *s_sk, u64 *s_sv) {
  constexpr u32 RADIX = 1u << BITS, mask = RADIX - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  u32 lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (i64 t0 = c0; t0 < c1; t0 += kSegTile) {
    for (int i = tid; i < 32 * 128; i += kSegThreads) (&s_wh[0][0])[i] = 0;
    __syncthreads();
    u32 d[kSegItems], r[kSegItems];
    bool v[kSegItems];
#pragma unroll
    for (int j = 0; j < kSegItems; ++j) {  // warp w owns tile items [128 w, 128 w + 128) in (j, lane) order
      const i64 i = t0 + warp * (32 * kSegItems) + j * 32 + lane;
      v[j] = i < c1;
      d[j] = v[j] ? ((kin[i] & lmask) >> SHIFT) & mask : mask;
      const u32 peers = peers_of<BITS>(d[j]) & __ballot_sync(0xffffffffu, v[j]);
      const u32 old = s_wh[warp][d[j]];
      __syncwarp();
      if (v[j] && lane == __ffs(peers) - 1) s_wh[warp][d[j]] = (unsigned short)(old + __popc(peers));
      __syncwarp();
      r[j] = old + __popc(peers & lt);
    }
    __syncthreads();
    if (tid < int(RADIX)) {  // per digit: exclusive prefix over warps, tile total
      u32 tot = 0;
      for (int w = 0; w < 32; ++w) {
        const u32 c = s_wh[w][tid];
        s_wh[w][tid] = (unsigned short)tot;
        tot += c;
      }
      s_tot[tid] = tot;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive digit starts inside the tile (RADIX <= 128: 4 per lane)
      u32 a4[4], t = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int dd = lane * 4 + q;
        a4[q] = dd < int(RADIX) ? s_tot[dd] : 0u;
        t += a4[q];
      }
      u32 incl = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      u32 run = incl - t;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int dd = lane * 4 + q;
        if (dd < int(RADIX)) s_tdig[dd] = run;
        run += a4[q];
      }
    }
    __syncthreads();
    // stage the tile in digit order, then write each digit's run contiguously
#pragma unroll
    for (int j = 0; j < kSegItems; ++j) {
      if (!v[j]) continue;
      const i64 i = t0 + warp * (32 * kSegItems) + j * 32 + lane;
      const u32 tp = s_tdig[d[j]] + s_wh[warp][d[j]] + r[j];
      s_sk[tp] = kin[i];
      s_sv[tp] = vin[i];
    }
    __syncthreads();
    const int tn = int(min(i64(kSegTile), c1 - t0));
    for (int i = tid; i < tn; i += kSegThreads) {
      const u32 kk = s_sk[i];
      const u32 dd = ((kk & lmask) >> SHIFT) & mask;
      const i64 p = c0 + s_base[dd] + (u32(i) - s_tdig[dd]);
      kout[p] = kk;
      vout[p] = s_sv[i];
    }
    __syncthreads();
    if (tid < int(RADIX)) s_base[tid] += s_tot[tid];  // the next tile goes behind this one
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSegThreads) k_seg_sort1(Batch b, u32 *__restrict__ k1, u64 *__restrict__ v1,
                                                           u32 *__restrict__ k1a, u64 *__restrict__ v1a, i64 m,
                                                           int bl, u32 lmask) {
  __shared__ u32 s_h0[128], s_h1[128], s_tot[128], s_tdig[128];
  __shared__ unsigned short s_wh[32][128];
  extern __shared__ __align__(16) unsigned char seg_smem[];
  u64 *s_sv = reinterpret_cast<u64 *>(seg_smem);  // [kSegTile] staged values
  u32 *s_sk = reinterpret_cast<u32 *>(s_sv + kSegTile);  // [kSegTile] staged keys
  const int w = blockIdx.x, tid = threadIdx.x;
  // the window's candidate segment [c0, c1) (candidates are window-major)
  i64 c0, c1;
  {
    i64 lo = 0, hi = m;
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (i64(k1[mid] >> bl) < w) lo = mid + 1; else hi = mid;
    }
    c0 = lo;
    hi = m;
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (i64(k1[mid] >> bl) <= w) lo = mid + 1; else hi = mid;
    }
    c1 = lo;
  }
  if (c0 == c1) return;
  if (tid < 128) {
    s_h0[tid] = 0;
    s_h1[tid] = 0;
  }
  __syncthreads();
  for (i64 i = c0 + tid; i < c1; i += kSegThreads) {
    const u32 f = k1[i] & lmask;
    atomicAdd(&s_h0[f & 127u], 1u);
    atomicAdd(&s_h1[(f >> 7) & 127u], 1u);
  }
  __syncthreads();
  if (tid < 32) {  // exclusive digit starts (one warp, 4 + 4 digits per lane)
    u32 a[4], t = 0;
    for (int j = 0; j < 4; ++j) { a[j] = s_h0[tid * 4 + j]; t += a[j]; }
    u32 incl = t;
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
      if (tid >= d) incl += o;
    }
    u32 run = incl - t;
    for (int j = 0; j < 4; ++j) { s_h0[tid * 4 + j] = run; run += a[j]; }
    u32 b2[4], t2 = 0;
    for (int j = 0; j < 4; ++j) { b2[j] = s_h1[tid * 4 + j]; t2 += b2[j]; }
    incl = t2;
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
      if (tid >= d) incl += o;
    }
    run = incl - t2;
    for (int j = 0; j < 4; ++j) { s_h1[tid * 4 + j] = run; run += b2[j]; }
  }
  __syncthreads();
  seg_pass<0, 7>(k1, v1, k1a, v1a, c0, c1, lmask, s_h0, s_wh, s_tot, s_tdig, s_sk, s_sv);
  seg_pass<7, 7>(k1a, v1a, k1, v1, c0, c1, lmask, s_h1, s_wh, s_tot, s_tdig, s_sk, s_sv);
}

struct Tab {
  u32 *lv[32];
};

__global__ void k_mark(const i32 *__restrict__ cl, const i32 *__restrict__ cs, const u8 *__restrict__ state, i64 m,
                       Tab tab) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m || state[c] != 0) return;
  i64 l = cl[c], s = cs[c];
  int q = 63 - __clzll(l);
  u32 *t = tab.lv[q];
  atomicMin(&t[s], u32(c));
  atomicMin(&t[s + l - (i64(1) << q)], u32(c));
}

__global__ void k_pull(const u32 *__restrict__ up, u32 *__restrict__ down, i64 n, i64 half) {
  i64 y = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (y >= n) return;
  u32 v = up[y];
  if (y >= half) {
    u32 o = up[y - half];
    v = o < v ? o : v;
  }
  if (v < down[y]) down[y] = v;
}

// two levels of the pull-down in one pass: level q-2 from levels q-1 and q
// (level q-1's pulled value at y is min(up1[y], up2[y], up2[y - h1]))
__global__ void k_pull2(const u32 *__restrict__ up2, const u32 *__restrict__ up1, u32 *__restrict__ down, i64 n,
                        i64 h1, i64 h2) {
  const i64 y = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (y >= n) return;
  auto lvl1 = [&](i64 x) -> u32 {
    u32 v = min(up1[x], up2[x]);
    if (x >= h1) v = min(v, up2[x - h1]);
    return v;
  };
  u32 v = min(down[y], lvl1(y));
  if (y >= h2) v = min(v, lvl1(y - h2));
  down[y] = v;
}

__global__ void k_select(const i32 *__restrict__ cl, const i32 *__restrict__ cs, u8 *__restrict__ state, i64 m,
                         const u32 *__restrict__ first, u32 *__restrict__ diff) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m || state[c] != 0) return;
  i64 l = cl[c], s = cs[c];
  if (first[s] == u32(c) && first[s + l - 1] == u32(c)) {
    state[c] = 1;
    atomicAdd(&diff[s], 1u);
    atomicAdd(&diff[s + l], 0xffffffffu);
  }
}

struct CovF {
  const u32 *diff;
  u32 *cov;
  __device__ u32 load(i64 i) const { return diff[i]; }
  __device__ bool store(i64 i, u32 incl, u32) const {
    cov[i] = incl;
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_reject(const i32 *__restrict__ cl, const i32 *__restrict__ cs, u8 *__restrict__ state, i64 m,
                         const u32 *__restrict__ cov, u32 *__restrict__ undecided) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  bool und = false;
  if (c < m && state[c] == 0) {
    i64 l = cl[c], s = cs[c];
    if (cov[s] != 0 || cov[s + l - 1] != 0)
      state[c] = 2;
    else
      und = true;
  }
  if (__syncthreads_or(und) && threadIdx.x == 0) atomicOr(undecided, 1u);
}

__global__ void k_gstats(const i32 *__restrict__ cg, const u8 *__restrict__ state, i64 m, u32 *__restrict__ gcnt,
                         u32 *__restrict__ gfirst) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m || state[c] != 1) return;
  i32 g = cg[c];
  atomicAdd(&gcnt[g], 1u);
  atomicMin(&gfirst[g], u32(c));
}

struct OccF {
  Batch b;
  const i32 *cg, *cs, *gbase;
  const u8 *state;
  const u32 *gcnt;
  u32 minc;
  u32 *oidx;
  i32 *occ;
  i64 occ_cap;
  i64 m;
  i64 *total;
  __device__ u32 load(i64 c) const { return (state[c] == 1 && gcnt[cg[c]] >= minc) ? 1u : 0u; }
  __device__ bool store(i64 c, u32 incl, u32 excl) const {
    if (incl != excl) {
      oidx[c] = excl;
      if (occ != nullptr && i64(excl) < occ_cap) occ[excl] = cs[c] - gbase[cg[c]];  // window-local start
    }
    if (c == m - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

struct RepF {
  Batch b;
  const u32 *gcnt, *gfirst, *oidx;
  const i32 *glen, *cs, *gbase, *gwin;
  u32 minc;
  apo_repeat *out;
  i64 cap;
  u32 *wcnt;
  i64 G;
  i64 *total;
  __device__ u32 load(i64 g) const { return gcnt[g] >= minc ? 1u : 0u; }
  __device__ bool store(i64 g, u32 incl, u32 excl) const {
    if (incl != excl) {
      u32 c0 = gfirst[g];
      i64 s = cs[c0];
      const int w = gwin[g];
      if (i64(excl) < cap && out != nullptr) {
        apo_repeat r;
        r.start = i32(s - gbase[g]);
        r.length = glen[g];
        r.count = i32(gcnt[g]);
        r.first_occ = i32(oidx[c0]);
        out[excl] = r;
      }
      atomicAdd(&wcnt[w], 1u);
    }
    if (g == G - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

struct OffF {
  const u32 *wcnt;
  i64 *out_off;
  __device__ u32 load(i64 w) const { return wcnt[w]; }
  __device__ bool store(i64 w, u32, u32 excl) const {
    out_off[w] = i64(excl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_emit_cands(Batch b, const i32 *__restrict__ cl, const i32 *__restrict__ cs,
                             const i32 *__restrict__ cg, const u8 *__restrict__ state, i64 m, i64 cap,
                             i32 *len, i32 *id, i32 *start, u8 *kept) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m || c >= cap) return;
  i64 s = cs[c];
  if (len) len[c] = cl[c];
  if (id) id[c] = cg[c];
  if (start) start[c] = i32(s - b_beg(b, b_wid(b, s)));
  if (kept) kept[c] = state[c] == 1 ? 1 : 0;
}

// K7 for batches of small windows: the sequential greedy of P:576-583 with
// the marked array of P:613-619, one WARP per window.  The window's
// candidates are contiguous in the sorted order; the marks are a bitset in
// shared memory (kGreedyMaxWin bits); a candidate is kept iff the bits of
// its first and last positions are clear, then the warp sets its interval's
// bits 32 words at a time.  Candidates are staged 32 at a time by the warp;
// the lanes first reject in parallel every staged candidate that already
// overlaps a mark, and only the rest are decided one by one, in order.
constexpr int kGreedyMaxWin = 16384;
constexpr int kGreedyWarps = 8;

__global__ void __launch_bounds__(kGreedyWarps * 32) k_greedy_window(Batch b, const i32 *__restrict__ cl,
                                                                     const i32 *__restrict__ cs, i64 m,
                                                                     u8 *__restrict__ state, u32 *__restrict__ kwin,
                                                                     u32 *__restrict__ kcnt, i64 kcap,
                                                                     u32 *__restrict__ kover) {
  __shared__ u32 marks[kGreedyWarps][kGreedyMaxWin / 32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const i64 w = i64(blockIdx.x) * kGreedyWarps + wl;
  if (w >= b.W) return;
  u32 *mk = marks[wl];
  const i64 beg = b_beg(b, int(w)), len = b_end(b, int(w)) - beg;
  for (int i = lane; i < (len + 31) / 32; i += 32) mk[i] = 0;
  // windows are contiguous in position space and candidates are window-major,
  // so a plain lower bound on the window id of each candidate's start works
  i64 c0, c1;
  {
    i64 lo = 0, hi = m;
    while (lo < hi) {
      i64 mid = (lo + hi) >> 1;
      if (b_wid(b, cs[mid]) < w) lo = mid + 1; else hi = mid;
    }
    c0 = lo;
    hi = m;
    while (lo < hi) {
      i64 mid = (lo + hi) >> 1;
      if (b_wid(b, cs[mid]) <= w) lo = mid + 1; else hi = mid;
    }
    c1 = lo;
  }
  __syncwarp();
  u32 nk = 0;
  // the next two batches' (length, start) are in flight while one is decided
  auto fetch = [&](i64 q, i32 &l, i32 &st) {
    l = 0;
    st = 0;
    if (q < c1) {
      l = cl[q];
      st = i32(cs[q] - beg);
    }
  };
  i32 l1, s1, l2, s2;
  fetch(c0 + lane, l1, s1);
  fetch(c0 + 32 + lane, l2, s2);
  for (i64 base = c0; base < c1; base += 32) {
    const i64 my = base + lane;
    const i32 ml = l1, ms = s1;
    l1 = l2;
    s1 = s2;
    fetch(base + 64 + lane, l2, s2);
    // marks only grow, so a candidate whose end bits are already set now is
    // rejected whatever the earlier candidates of this batch do: only the
    // survivors of this parallel pre-check are walked in order
    bool maybe = false;
    if (my < c1) {
      const i32 en = ms + ml - 1;
      maybe = !((mk[ms >> 5] >> (ms & 31)) & 1u) && !((mk[en >> 5] >> (en & 31)) & 1u);
    }
    u32 pend = __ballot_sync(0xffffffffu, maybe);
    u32 keep_bits = 0;
    while (pend) {
      const int k = __ffs(pend) - 1;
      pend &= pend - 1;
      const i32 l = __shfl_sync(0xffffffffu, ml, k);
      const i32 st = __shfl_sync(0xffffffffu, ms, k);
      const i32 en = st + l - 1;
      const bool free_ = !((mk[st >> 5] >> (st & 31)) & 1u) && !((mk[en >> 5] >> (en & 31)) & 1u);
      if (free_) {
        keep_bits |= 1u << k;
        // set bits [st, en]
        const int w0 = st >> 5, w1 = en >> 5;
        for (int x = w0 + lane; x <= w1; x += 32) {
          u32 bits = 0xffffffffu;
          if (x == w0) bits &= 0xffffffffu << (st & 31);
          if (x == w1) bits &= 0xffffffffu >> (31 - (en & 31));
          mk[x] |= bits;
        }
      }
      __syncwarp();
    }
    if (my < c1) state[my] = ((keep_bits >> lane) & 1u) ? 1 : 2;
    if (kwin != nullptr) {  // the window's kept candidates, in candidate order
      if ((keep_bits >> lane) & 1u) {
        const u32 j = nk + __popc(keep_bits & ((1u << lane) - 1u));
        if (i64(j) < kcap) kwin[w * kcap + j] = u32(my);
      }
      nk += __popc(keep_bits);
    }
  }
  if (kwin != nullptr && lane == 0) {
    kcnt[w] = i64(nk) <= kcap ? nk : 0u;
    if (i64(nk) > kcap) atomicOr(kover, 1u);  // cannot happen for non-overlapping kept repeats; scan all if it does
  }
}

struct KeptBaseF {  // exclusive scan of the per-window kept counts
  const u32 *cnt;
  u32 *base;
  i64 n;
  i64 *total;
  __device__ u32 load(i64 i) const { return cnt[i]; }
  __device__ bool store(i64 i, u32 incl, u32 excl) const {
    base[i] = excl;
    if (i == n - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_kept_compact(const u32 *__restrict__ kwin, const u32 *__restrict__ kcnt,
                               const u32 *__restrict__ kbase, i64 kcap, u32 *__restrict__ klist) {
  const i64 w = blockIdx.x;
  const u32 n = kcnt[w], b = kbase[w];
  for (u32 j = threadIdx.x; j < n; j += blockDim.x) klist[b + j] = kwin[w * kcap + j];
}

// K8 over the compact kept list without per-group tables: the kept
// candidates are in candidate order, where a sub-string group's members are
// contiguous, so a group's kept members form one run of the list -- its
// count is the run's length and its first occurrence the run's head.
struct KeptRunF {  // run ordinal of every kept candidate; each run's first index
  const u32 *klist;
  const i32 *cg;
  u32 *rid, *hpos;
  i64 K;
  i64 *total;
  __device__ u32 load(i64 k) const { return (k == 0 || cg[klist[k]] != cg[klist[k - 1]]) ? 1u : 0u; }
  __device__ bool store(i64 k, u32 incl, u32 excl) const {
    rid[k] = incl - 1;
    if (incl != excl) hpos[excl] = u32(k);
    if (k == K - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__device__ __forceinline__ u32 run_len(const u32 *hpos, i64 R, i64 K, u32 r) {
  return u32((i64(r) + 1 < R ? i64(hpos[r + 1]) : K) - i64(hpos[r]));
}

struct OccRunF {  // occurrence list over the kept candidates of runs with count >= minc
  const u32 *klist, *rid, *hpos;
  i64 R, K;
  const i32 *cg, *cs, *gbase;
  u32 minc;
  u32 *oidx;
  i32 *occ;
  i64 occ_cap;
  i64 *total;
  __device__ u32 load(i64 k) const { return run_len(hpos, R, K, rid[k]) >= minc ? 1u : 0u; }
  __device__ bool store(i64 k, u32 incl, u32 excl) const {
    if (incl != excl) {
      const u32 c = klist[k];
      oidx[c] = excl;
      if (occ != nullptr && i64(excl) < occ_cap) occ[excl] = cs[c] - gbase[cg[c]];  // window-local start
    }
    if (k == K - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

struct RepRunF {  // one repeat per run with count >= minc, in run (= group) order
  const u32 *klist, *hpos;
  i64 R, K;
  const i32 *cg, *cs, *glen, *gbase, *gwin;
  const u32 *oidx;
  u32 minc;
  apo_repeat *out;
  i64 cap;
  u32 *wcnt;
  i64 *total;
  __device__ u32 load(i64 r) const { return run_len(hpos, R, K, u32(r)) >= minc ? 1u : 0u; }
  __device__ bool store(i64 r, u32 incl, u32 excl) const {
    if (incl != excl) {
      const u32 c0 = klist[hpos[r]];
      const i32 g = cg[c0];
      if (i64(excl) < cap && out != nullptr) {
        apo_repeat rr;
        rr.start = i32(cs[c0] - gbase[g]);
        rr.length = glen[g];
        rr.count = i32(run_len(hpos, R, K, u32(r)));
        rr.first_occ = i32(oidx[c0]);
        out[excl] = rr;
      }
      atomicAdd(&wcnt[gwin[g]], 1u);
    }
    if (r == R - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

}  // namespace

void plan_select(Carver &cv, const Batch &b, SelWork &w, int min_len) {
  const i64 N = b.N, M = N > 1 ? 2 * (N - 1) : 1;
  w.k1 = cv.take<u32>(M);
  w.k1_alt = cv.take<u32>(M);
  w.v1 = cv.take<u64>(M);
  w.v1_alt = cv.take<u64>(M);
  w.k2 = cv.take<u64>(M);
  w.k2_alt = cv.take<u64>(M);
  // range minima over LCP: in-block prefix/suffix minima (N each) and a
  // sparse table over the N/32 block minima (queries span < maxwin entries)
  const i64 nb = (N + 31) / 32;
  w.rmq_levels = bits_for(u64(b.maxwin / 32 + 2));
  if (w.rmq_levels > 29) w.rmq_levels = 29;
  w.rmq[0] = cv.take<i32>(N);
  w.rmq[1] = cv.take<i32>(N);
  for (int j = 0; j < w.rmq_levels; ++j) w.rmq[j + 2] = cv.take<i32>(nb);
  w.glen = cv.take<i32>(M);
  w.gbase = cv.take<i32>(M);
  w.gwin = cv.take<i32>(M);
  w.gpos = cv.take<u32>(M);
  w.cl = cv.take<i32>(M);
  w.cs = cv.take<i32>(M);
  w.cg = cv.take<i32>(M);
  w.state = cv.take<u8>(M);
  const i64 maxl = b.maxwin / 2;
  w.tab_levels = maxl >= 1 ? bits_for(u64(maxl)) : 1;
  for (int q = 0; q < w.tab_levels; ++q) w.tab[q] = cv.take<u32>(N);
  w.diff = cv.take<u32>(N + 1);
  w.cov = cv.take<u32>(N + 1);
  w.gcnt = cv.take<u32>(M);
  w.gfirst = cv.take<u32>(M);
  w.oidx = cv.take<u32>(M);
  w.wcnt = cv.take<u32>(size_t(b.W) + 1);
  w.scal = cv.take<u64>(16);
  if (b.maxwin <= kGreedyMaxWin && b.W >= 8) {  // the per-window greedy keeps <= maxwin / min_len per window
    w.kcap = b.maxwin / std::max(min_len, 1) + 1;
    w.kwin = cv.take<u32>(size_t(b.W) * size_t(w.kcap));
    w.kcnt = cv.take<u32>(size_t(b.W) + 1);
    w.kbase = cv.take<u32>(size_t(b.W) + 1);
    w.klist = cv.take<u32>(size_t(b.W) * size_t(w.kcap));
  }
}

void select_candidates(Ctx &c, const u64 *tok, const Batch &b, const SAWork &sa, int min_len, SelWork &w,
                       cudaStream_t s) {
  (void)tok;
  const i64 N = b.N;
  w.m = 0;
  w.G = 0;
  if (N < 2) return;
  const i64 maxl = b.maxwin / 2;
  const int bl = bits_for(u64(maxl));
  const int bw = bits_for(u64(b.W - 1));
  if (bl + bw > 32) throw Error{APO_ERR_INVALID, "batch too wide for 32-bit candidate keys"};
  i64 *m_dev = reinterpret_cast<i64 *>(w.scal);
  i64 *G_dev = reinterpret_cast<i64 *>(w.scal + 1);
  u32 *undecided = reinterpret_cast<u32 *>(w.scal + 2);
  APO_CUDA(cudaMemsetAsync(w.scal, 0, sizeof(u64) * 16, s));

  // ---- K5 + K6 per window on chip (batches of small windows) ----
  const bool no_fused = std::getenv("APO_SELECT_GLOBAL") != nullptr;  // tests: the global path
  i64 m = 0;
  if (!no_fused && window_select_supported(b, min_len) && window_select(c, b, sa, min_len, w, s)) {
    m = w.m;
    if (m == 0) return;
  } else {
  // ---- K5 ----
  {
    CandF f{b, sa.sa, sa.lcp, min_len, bl, maxl, N - 1, w.k1, w.v1, m_dev};
    launch_scan<false>(c, N - 1, f, s);
  }
  m = i64(c.read_u64(reinterpret_cast<u64 *>(m_dev), s));
  w.m = m;
  if (m == 0) return;

  // ---- K6: sort by (window, length desc), stable in pair order ----
  const u32 *k1 = w.k1;
  const u64 *v1 = w.v1;
  if (b.W > 1 && bl <= 14) {  // windows <= 16,384 ops: per-window two-pass sort (7 + 7 bits)
    const size_t ssm = size_t(kSegTile) * (sizeof(u64) + sizeof(u32));
    c.smem_optin(reinterpret_cast<const void *>(k_seg_sort1), ssm);
    k_seg_sort1<<<b.W, kSegThreads, ssm, s>>>(b, w.k1, w.v1, w.k1_alt, w.v1_alt, m, bl, (1u << bl) - 1u);
    APO_CHECK_LAUNCH();
    c.launches++;
  } else {
    bool a = radix_sort_u32_u64(c, w.k1, w.v1, w.k1_alt, w.v1_alt, m, 0, bl + bw, s);
    k1 = a ? w.k1_alt : w.k1;
    v1 = a ? w.v1_alt : w.v1;
  }
  Rmq rmq{};
  {
    const i64 nb = (N + 31) / 32;
    rmq.lcp = sa.lcp;
    rmq.pre = w.rmq[0];
    rmq.suf = w.rmq[1];
    k_rmq_blocks<<<grid_for(nb * 32, T), T, 0, s>>>(sa.lcp, N, w.rmq[0], w.rmq[1], w.rmq[2]);
    APO_CHECK_LAUNCH();
    c.launches++;
    rmq.lv[0] = w.rmq[2];
    for (int j = 1; j < w.rmq_levels; ++j) {
      k_rmq_level<<<grid_for(nb, T), T, 0, s>>>(rmq.lv[j - 1], w.rmq[j + 2], nb, i64(1) << (j - 1));
      APO_CHECK_LAUNCH();
      c.launches++;
      rmq.lv[j] = w.rmq[j + 2];
    }
  }
  const int bL = bits_for(u64(b.maxwin > 1 ? b.maxwin - 1 : 1));
  {
    k_head_flags<<<grid_for(m, T), T, 0, s>>>(k1, v1, rmq, maxl, (1u << bl) - 1u, m, w.state);
    APO_CHECK_LAUNCH();
    c.launches++;
    HeadF f{k1, v1, maxl, (1u << bl) - 1u, bL, m, w.k2, w.glen, G_dev, b.off, b.W > 1 ? b.wid : nullptr,
            bl, w.gbase, w.gwin, w.gpos, w.state};
    launch_scan<false>(c, m, f, s);
  }
  const i64 G = i64(c.read_u64(reinterpret_cast<u64 *>(G_dev), s));
  w.G = G;
  u32 *big = reinterpret_cast<u32 *>(w.scal + 3);
  k_seg_unpack<<<grid_for(m, T), T, 0, s>>>(w.k2, m, G, bL, w.gpos, w.glen, w.gbase, w.cl, w.cs, w.cg, w.state, big);
  APO_CHECK_LAUNCH();
  c.launches++;
  if (c.read_u32(big, s) != 0) {  // a large group somewhere: sort all keys instead
    bool a2 = radix_sort_u64_keys(c, w.k2, w.k2_alt, m, 0, bL + bits_for(u64(G - 1)), s);
    const u64 *k2 = a2 ? w.k2_alt : w.k2;
    k_unpack<<<grid_for(m, T), T, 0, s>>>(k2, m, bL, w.glen, w.gbase, w.cl, w.cs, w.cg, w.state);
    APO_CHECK_LAUNCH();
    c.launches++;
  }
  }

  // ---- K7 ----
  if (b.maxwin <= kGreedyMaxWin && b.W >= 8) {
    // many small windows: the paper's sequential marked-array greedy, one
    // warp per window, all windows at once
    if (w.kwin != nullptr) APO_CUDA(cudaMemsetAsync(w.scal + 4, 0, sizeof(u64), s));
    k_greedy_window<<<grid_for(b.W, kGreedyWarps), kGreedyWarps * 32, 0, s>>>(b, w.cl, w.cs, m, w.state, w.kwin,
                                                                               w.kcnt, w.kcap,
                                                                               reinterpret_cast<u32 *>(w.scal + 4));
    APO_CHECK_LAUNCH();
    c.launches++;
    if (w.kwin != nullptr) {  // compact the kept candidates (window-major, candidate order)
      KeptBaseF f{w.kcnt, w.kbase, b.W, reinterpret_cast<i64 *>(w.scal + 3)};
      launch_scan<false>(c, b.W, f, s);
      k_kept_compact<<<b.W, 128, 0, s>>>(w.kwin, w.kcnt, w.kbase, w.kcap, w.klist);
      APO_CHECK_LAUNCH();
      c.launches++;
      w.K = c.read_u64(w.scal + 4, s) != 0 ? -1 : i64(c.read_u64(w.scal + 3, s));
    }
    return;
  }
  // large windows: exact round-parallel greedy
  APO_CUDA(cudaMemsetAsync(w.diff, 0, sizeof(u32) * (N + 1), s));
  Tab tab{};
  for (int q = 0; q < w.tab_levels; ++q) tab.lv[q] = w.tab[q];
  const int gm = grid_for(m, T), gn = grid_for(N, T);
  for (int round = 0;; ++round) {
    if (round > 100000) throw Error{APO_ERR_CUDA, "greedy selection did not converge"};
    // the levels are consecutive carves: one fill for all of them
    const size_t tab_bytes = size_t(reinterpret_cast<char *>(w.tab[w.tab_levels - 1] + N) -
                                    reinterpret_cast<char *>(w.tab[0]));
    APO_CUDA(cudaMemsetAsync(w.tab[0], 0xff, tab_bytes, s));
    k_mark<<<gm, T, 0, s>>>(w.cl, w.cs, w.state, m, tab);
    APO_CHECK_LAUNCH();
    int q = w.tab_levels - 1;
    for (; q >= 2; q -= 2) {
      k_pull2<<<gn, T, 0, s>>>(w.tab[q], w.tab[q - 1], w.tab[q - 2], N, i64(1) << (q - 1), i64(1) << (q - 2));
      APO_CHECK_LAUNCH();
    }
    if (q == 1) {
      k_pull<<<gn, T, 0, s>>>(w.tab[1], w.tab[0], N, 1);
      APO_CHECK_LAUNCH();
    }
    k_select<<<gm, T, 0, s>>>(w.cl, w.cs, w.state, m, w.tab[0], w.diff);
    APO_CHECK_LAUNCH();
    CovF cf{w.diff, w.cov};
    launch_scan<false>(c, N, cf, s);
    APO_CUDA(cudaMemsetAsync(undecided, 0, sizeof(u32), s));
    k_reject<<<gm, T, 0, s>>>(w.cl, w.cs, w.state, m, w.cov, undecided);
    APO_CHECK_LAUNCH();
    c.launches += 3 + w.tab_levels / 2;
    if (c.read_u32(undecided, s) == 0) break;
  }
}

void emit_repeats(Ctx &c, const Batch &b, SelWork &w, int min_count, apo_repeat *out, i64 cap, i64 *out_off,
                  i32 *occ, i64 occ_cap, i64 *counts, cudaStream_t s) {
  const i64 m = w.m, G = w.G;
  APO_CUDA(cudaMemsetAsync(counts, 0, sizeof(i64) * 2, s));
  APO_CUDA(cudaMemsetAsync(w.wcnt, 0, sizeof(u32) * (b.W + 1), s));
  if (m > 0 && w.K >= 0) {
    // the per-window greedy's compact kept list: runs of equal groups
    const u32 minc = u32(min_count < 1 ? 1 : min_count);
    const i64 K = w.K;
    if (K > 0) {
      u32 *rid = w.gcnt, *hpos = w.gfirst;  // (per-group tables are not needed here)
      i64 *R_dev = reinterpret_cast<i64 *>(w.scal + 6);
      KeptRunF kr{w.klist, w.cg, rid, hpos, K, R_dev};
      launch_scan<false>(c, K, kr, s);
      const i64 R = i64(c.read_u64(w.scal + 6, s));
      OccRunF of{w.klist, rid, hpos, R, K, w.cg, w.cs, w.gbase, minc, w.oidx, occ, occ_cap, counts + 1};
      launch_scan<false>(c, K, of, s);
      RepRunF rf{w.klist, hpos, R, K, w.cg, w.cs, w.glen, w.gbase, w.gwin, w.oidx, minc, out, cap, w.wcnt, counts};
      launch_scan<false>(c, R, rf, s);
    }
  } else if (m > 0) {
    APO_CUDA(cudaMemsetAsync(w.gcnt, 0, sizeof(u32) * G, s));
    APO_CUDA(cudaMemsetAsync(w.gfirst, 0xff, sizeof(u32) * G, s));
    const u32 minc = u32(min_count < 1 ? 1 : min_count);
    {
      k_gstats<<<grid_for(m, T), T, 0, s>>>(w.cg, w.state, m, w.gcnt, w.gfirst);
      APO_CHECK_LAUNCH();
      c.launches++;
      OccF of{b, w.cg, w.cs, w.gbase, w.state, w.gcnt, minc, w.oidx, occ, occ_cap, m, counts + 1};
      launch_scan<false>(c, m, of, s);
    }
    RepF rf{b, w.gcnt, w.gfirst, w.oidx, w.glen, w.cs, w.gbase, w.gwin, minc, out, cap, w.wcnt, G, counts};
    launch_scan<false>(c, G, rf, s);
  }
  if (out_off != nullptr) {
    OffF f{w.wcnt, out_off};
    launch_scan<false>(c, i64(b.W) + 1, f, s);
  }
}

void emit_candidates(Ctx &c, const Batch &b, const SelWork &w, i32 *len, i32 *id, i32 *start, u8 *kept, i64 cap,
                     i64 *count, cudaStream_t s) {
  c.h2d(count, &w.m, sizeof(i64), s);
  if (w.m > 0) {
    k_emit_cands<<<grid_for(w.m, T), T, 0, s>>>(b, w.cl, w.cs, w.cg, w.state, w.m, cap, len, id, start, kept);
    APO_CHECK_LAUNCH();
    c.launches++;
  }
  APO_CUDA(cudaStreamSynchronize(s));  // w.m is a host value copied asynchronously
}

}  // namespace apo
