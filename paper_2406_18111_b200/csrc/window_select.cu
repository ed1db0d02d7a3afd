// window_select.cu -- K5 + K6 fused for batches of small windows (<= 16,384
// ops): candidate generation, the (length desc, sub-string, start) order and
// the sub-string IDs of one window entirely in shared memory.
//
// Same results as select.cu's global path (CandF, k_seg_sort1, the RMQ head
// test, HeadF, k_seg_unpack, readings R4-R7):
//  * candidates of pair k = ranks (k, k+1): (l, s1), (l, s2) if the two
//    occurrences are disjoint, else (l, m), (l, m + l) with the period rule;
//    kept iff l >= min_len; listed in pair order (two per pair);
//  * a STABLE sort by length desc (two 7-bit LSD passes over u16 items
//    (pair << 1 | which), ranked per warp with match.any peer masks), so equal
//    lengths stay in pair order = sub-string (rank) order;
//  * a candidate starts a new sub-string group unless the previous one has
//    the same length and is the same pair, or min LCP over the pairs between
//    them is >= the length (block minima + a sparse table over them);
//  * members of a group ordered by (start, sort position).
// The window's candidate and group counts are combined across windows by a
// decoupled look-back (windows claimed in order), so every window writes its
// final slice of cl / cs / cg / state and of the per-group arrays directly,
// with dense global group ordinals.  A window with a group of more than
// kXGroupMax members raises `big` and the caller falls back to the global
// path for the batch.
#include "pipeline.cuh"

namespace apo {

namespace {

using u16 = unsigned short;

constexpr int kXT = 1024;
constexpr int kXWarps = kXT / 32;
constexpr int kXW = 16384;            // longest window
constexpr int kXItems = 2 * kXW;      // candidates per window (two per kept pair)
constexpr int kXRows = kXW / kXT;     // rows of 32 pairs per warp at most
constexpr int kXBlk = kXW / 32;       // LCP blocks of 32
constexpr int kXLv = 10;              // sparse-table levels over the block minima
constexpr u32 kXGroupMax = 64;

struct XSmem {
  u16 sa[kXW];                 // window-local suffix array
  u16 lc[kXW];                 // LCP of pair k (k, k+1); 0 at the window end
  u16 plen[kXW];               // candidate length of pair k (0: not kept)
  u16 P[kXW];                  // kept pairs: pair order, then sorted by length desc (stable)
  u16 T[kXW];                  // sort buffer; then in-block prefix minima of lc
  u16 U[kXW];                  // in-block suffix minima of lc
  u16 sp[kXLv][kXBlk];         // sp[j][i] = min of the LCP blocks i .. i + 2^j - 1
  u16 hist[kXWarps][128];      // LSD pass: per-warp digit counts
  u32 hbits[kXItems / 32];     // group-head bit of every sorted candidate
  u16 hpre[kXItems / 32];      // heads before each 32-candidate word
  u32 dstart[128];
  u32 wsum[kXWarps];
  u32 misc[8];                 // [0] window, [1] kept pairs, [2] G_w, [3] c_base, [4] g_base, [5] big
};
static_assert(sizeof(XSmem) + 1024 <= 232448, "window_select shared memory exceeds the opt-in limit");

__device__ __forceinline__ u32 lanemask_lt_x() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// candidate length of pair k (k + 1 < n): disjoint occurrences keep the LCP,
// overlapping ones the period rule (R4-R6)
__device__ __forceinline__ u32 pair_len(const XSmem &S, int k) {
  const u32 s1 = S.sa[k], s2 = S.sa[k + 1], p = S.lc[k];
  const u32 d = s1 < s2 ? s2 - s1 : s1 - s2;
  if (d >= p) return p;
  u32 L = (p + d) >> 1;
  return L - L % d;
}

// start of candidate `which` of kept pair k (length S.plen[k])
__device__ __forceinline__ u32 pair_start(const XSmem &S, int k, u32 which) {
  const u32 s1 = S.sa[k], s2 = S.sa[k + 1], p = S.lc[k];
  const u32 lo = s1 < s2 ? s1 : s2, d = s1 < s2 ? s2 - s1 : s1 - s2;
  if (d >= p) return which ? s2 : s1;
  return which ? lo + S.plen[k] : lo;
}

// min LCP[a..b] (inclusive, a <= b) below l
__device__ __forceinline__ bool lcp_below(const XSmem &S, int a, int b, u32 l) {
  const int ba = a >> 5, bb = b >> 5;
  if (ba != bb) {
    if (S.U[a] < l || S.T[b] < l) return true;
    if (bb - ba > 1) {
      const int x = ba + 1, y = bb - 1;
      const int j = 31 - __clz(y - x + 1);
      return min(u32(S.sp[j][x]), u32(S.sp[j][y - (1 << j) + 1])) < l;
    }
    return false;
  }
  if ((a & 31) == 0) return S.T[b] < l;
  if ((b & 31) == 31) return S.U[a] < l;
  for (int j = a; j <= b; ++j)
    if (S.lc[j] < l) return true;
  return false;
}

// exclusive prefix of one u32 per thread over the CTA (thread order)
__device__ __forceinline__ u32 x_excl_scan(u32 v, u32 *wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const u32 x = wsum[lane];
    u32 y = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xffffffffu, y, d);
      if (lane >= d) y += o;
    }
    wsum[lane] = y - x;
  }
  __syncthreads();
  const u32 r = wsum[warp] + incl - v;
  __syncthreads();
  return r;
}

// one stable LSD pass over the m kept pairs: in -> out by the 7-bit digit of
// (maxl - plen) at `shift`
__device__ void x_lsd_pass(XSmem &S, const u16 *in, u16 *out, int m, u32 maxl, int shift) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = (m + kXT - 1) / kXT;  // rows per warp
  u16 *wh = S.hist[warp];
  for (int i = lane; i < 64; i += 32) reinterpret_cast<u32 *>(wh)[i] = 0;
  __syncwarp();
  const u32 lt = lanemask_lt_x();
  const int base = warp * 32 * R;
  u32 rk[kXRows / 2];
#pragma unroll
  for (int j = 0; j < kXRows; ++j) {
    if (j < R) {
      const int q = base + j * 32 + lane;
      const bool v = q < m;
      const u32 d = v ? ((maxl - S.plen[in[q]]) >> shift) & 127u : 128u + lane;
      const u32 peers = __match_any_sync(0xffffffffu, d);
      const u32 old = v ? u32(wh[d]) : 0u;
      __syncwarp();
      if (v && lane == __ffs(peers) - 1) wh[d] = u16(old + __popc(peers));
      __syncwarp();
      const u32 r = old + __popc(peers & lt);
      if (j & 1)
        rk[j >> 1] |= r << 16;
      else
        rk[j >> 1] = r;
    }
  }
  __syncthreads();
  if (tid < 128) {
    u32 total = 0;
#pragma unroll 8
    for (int w = 0; w < kXWarps; ++w) {
      const u32 c = S.hist[w][tid];
      S.hist[w][tid] = u16(total);
      total += c;
    }
    S.dstart[tid] = total;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive digit starts (4 digits per lane)
    u32 a4[4], t = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a4[k] = S.dstart[lane * 4 + k];
      t += a4[k];
    }
    u32 incl = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    u32 run = incl - t;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      S.dstart[lane * 4 + k] = run;
      run += a4[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kXRows; ++j) {
    if (j < R) {
      const int q = base + j * 32 + lane;
      if (q < m) {
        const u32 it = in[q];
        const u32 d = ((maxl - S.plen[it]) >> shift) & 127u;
        const u32 r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        out[S.dstart[d] + wh[d] + r] = u16(it);
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kXT, 1)
    k_window_select(Batch b, const i32 *__restrict__ sa, const i32 *__restrict__ lcp, i32 min_len, u32 maxl,
                    i32 *__restrict__ cl, i32 *__restrict__ cs, i32 *__restrict__ cg, u8 *__restrict__ state,
                    i32 *__restrict__ glen, i32 *__restrict__ gbase, i32 *__restrict__ gwin, u32 *__restrict__ gpos,
                    i64 *__restrict__ m_out, i64 *__restrict__ G_out, u32 *__restrict__ big, u64 *status,
                    u32 *counter, u32 epoch) {
  extern __shared__ __align__(16) unsigned char smraw[];
  XSmem &S = *reinterpret_cast<XSmem *>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) S.misc[0] = atomicAdd(counter, 1u);  // windows in claim order (look-back progress)
  __syncthreads();
  const int w = int(S.misc[0]);
  const i64 tile = w;
  const i64 beg = b.off[w];
  const int n = int(b.off[w + 1] - beg);
  for (int i = tid; i < n; i += kXT) {
    S.sa[i] = u16(sa[beg + i] - i32(beg));
    S.lc[i] = u16(lcp[beg + i]);
  }
  __syncthreads();
  // LCP block minima (sparse table level 0) and in-block suffix minima; the
  // in-block prefix minima go to T once the sort no longer needs it
  const int nb = (n + 31) >> 5;
  for (int i = warp; i < nb; i += kXWarps) {
    const int j = i * 32 + lane;
    u32 dn = j < n ? u32(S.lc[j]) : 0xffffu;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_down_sync(0xffffffffu, dn, d);
      if (lane + d < 32) dn = min(dn, y);
    }
    if (j < n) S.U[j] = u16(dn);
    if (lane == 0) S.sp[0][i] = u16(dn);
  }
  // K5: candidate lengths, kept pairs in pair order (thread t: pairs [16 t, 16 t + 16))
  constexpr int kPP = kXW / kXT;
  const int np = n > 1 ? n - 1 : 0;
  u32 keep = 0, kc = 0;
#pragma unroll
  for (int j = 0; j < kPP; ++j) {
    const int k = tid * kPP + j;
    if (k < np) {
      const u32 l = pair_len(S, k);
      const bool kp = l >= u32(min_len);
      S.plen[k] = u16(kp ? l : 0u);
      if (kp) {
        keep |= 1u << j;
        ++kc;
      }
    }
  }
  const u32 ex = x_excl_scan(kc, S.wsum);  // (its barriers also publish T/U/sp[0]/plen)
  {
    u32 o = ex;
#pragma unroll
    for (int j = 0; j < kPP; ++j)
      if ((keep >> j) & 1u) S.P[o++] = u16(tid * kPP + j);
    if (tid == kXT - 1) S.misc[1] = ex + kc;
  }
  for (int j = 1; j < kXLv && (1 << j) <= nb; ++j) {
    __syncthreads();
    for (int i = tid; i + (1 << j) <= nb; i += kXT) S.sp[j][i] = min(S.sp[j - 1][i], S.sp[j - 1][i + (1 << (j - 1))]);
  }
  __syncthreads();
  const int mp = int(S.misc[1]);  // kept pairs
  const int m = 2 * mp;           // candidates
  // the candidate count is known: publish it now (the look-back of the
  // windows behind this one resolves while this one sorts)
  if (tid == 0) {
    if (tile == 0)
      lb_store(status, lb_pack(epoch, kFlagInc, u32(m)));
    else
      lb_store(status + 2 * tile, lb_pack(epoch, kFlagAgg, u32(m)));
  }
  // K6 sort 1: kept pairs by length desc, stable (P -> T -> P); a pair's two
  // candidates stay adjacent (same key), so this is the candidates' order
  if (mp > 0) {
    x_lsd_pass(S, S.P, S.T, mp, maxl, 0);
    x_lsd_pass(S, S.T, S.P, mp, maxl, 7);
  }
  for (int i = warp; i < nb; i += kXWarps) {  // in-block prefix minima (T is free now)
    const int j = i * 32 + lane;
    u32 up = j < n ? u32(S.lc[j]) : 0xffffu;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 x = __shfl_up_sync(0xffffffffu, up, d);
      if (lane >= d) up = min(up, x);
    }
    if (j < n) S.T[j] = u16(up);
  }
  __syncthreads();
  // group heads: only the first candidate of a pair can start a group; it
  // does unless the previous pair has the same length and min LCP over the
  // pairs between them is >= that length
  const int nw = (m + 31) >> 5;
  for (int wd = warp; wd < nw; wd += kXWarps) {
    const int c = wd * 32 + lane;
    bool h = false;
    if (c < m && (c & 1) == 0) {
      const int i = c >> 1;
      h = true;
      if (i > 0) {
        const int kcur = S.P[i], kp = S.P[i - 1];
        const u32 l = S.plen[kcur];
        if (S.plen[kp] == l) h = lcp_below(S, kp, kcur - 1, l);
      }
    }
    const u32 hb = __ballot_sync(0xffffffffu, h);
    if (lane == 0) S.hbits[wd] = hb;
  }
  __syncthreads();
  {
    const u32 v = tid < nw ? u32(__popc(S.hbits[tid])) : 0u;
    const u32 e2 = x_excl_scan(v, S.wsum);
    if (tid < nw) S.hpre[tid] = u16(e2);
    if (tid == kXT - 1) S.misc[2] = e2 + v;
  }
  // every candidate's start, once (T and U -- the range-minimum tables --
  // are free now and hold 2 x kXW u16 together)
  u16 *ST = S.T;
  for (int c = tid; c < m; c += kXT) ST[c] = u16(pair_start(S, S.P[c >> 1], u32(c & 1)));
  __syncthreads();
  const u32 Gw = S.misc[2];
  // window offsets: decoupled look-back over (candidates, groups)
  if (tid < 2) {
    const u32 agg = tid == 0 ? u32(m) : Gw;
    u32 pre = 0;
    if (tile == 0) {
      if (tid == 1) lb_store(status + 1, lb_pack(epoch, kFlagInc, agg));
    } else {
      if (tid == 1) lb_store(status + 2 * tile + 1, lb_pack(epoch, kFlagAgg, agg));
      pre = lb_lookback<false>(status, 2, size_t(tid), tile, epoch);
      lb_store(status + 2 * tile + tid, lb_pack(epoch, kFlagInc, pre + agg));
    }
    S.misc[3 + tid] = pre;
    if (tile == b.W - 1) (tid == 0 ? m_out : G_out)[0] = i64(pre + agg);
  }
  if (tid == 0) S.misc[5] = 0;
  __syncthreads();
  const i64 cbase = S.misc[3], gb = S.misc[4];
  // members of each group in (start, sort position) order; final writes
  for (int c = tid; c < m; c += kXT) {
    const int wd = c >> 5;
    const u32 below = S.hbits[wd] & ((2u << (c & 31)) - 1u);  // heads at or before c in its word
    int gs;
    if (below) {
      gs = wd * 32 + 31 - __clz(below);
    } else {
      int x = wd - 1;
      while (S.hbits[x] == 0) --x;  // candidate 0 is always a head
      gs = x * 32 + 31 - __clz(S.hbits[x]);
    }
    int ge;
    {
      const u32 above = (c & 31) == 31 ? 0u : (S.hbits[wd] & ~((2u << (c & 31)) - 1u));
      if (above) {
        ge = wd * 32 + __ffs(above) - 1;
      } else {
        int x = wd + 1;
        while (x < nw && S.hbits[x] == 0) ++x;
        ge = x < nw ? x * 32 + __ffs(S.hbits[x]) - 1 : m;
      }
    }
    if (u32(ge - gs) > kXGroupMax) {
      S.misc[5] = 1;
      continue;
    }
    const int k = S.P[c >> 1];
    const u32 l = S.plen[k];
    const u32 st = ST[c];
    u32 r = 0;
    for (int j = gs; j < ge; ++j) {
      const u32 sj = ST[j];
      r += (sj < st || (sj == st && j < c)) ? 1u : 0u;
    }
    const u32 gid = u32(S.hpre[wd]) + __popc(below) - 1u;
    const i64 p = cbase + gs + r;
    cs[p] = i32(beg + st);
    cg[p] = i32(gb + gid);
    cl[p] = i32(l);
    state[p] = 0;
    if (gs == c) {
      glen[gb + gid] = i32(l);
      gbase[gb + gid] = i32(beg);
      gwin[gb + gid] = w;
      gpos[gb + gid] = u32(cbase + c);
    }
  }
  __syncthreads();
  if (tid == 0 && S.misc[5]) atomicOr(big, 1u);
}

}  // namespace

bool window_select_supported(const Batch &b, int min_len) {
  return b.W > 1 && !b.gen && b.maxwin <= kXW && min_len >= 1 && 2 * b.N < (i64(1) << 31);
}

bool window_select(Ctx &c, const Batch &b, const SAWork &sa, int min_len, SelWork &w, cudaStream_t s) {
  i64 *m_dev = reinterpret_cast<i64 *>(w.scal);
  i64 *G_dev = reinterpret_cast<i64 *>(w.scal + 1);
  u32 *big = reinterpret_cast<u32 *>(w.scal + 5);
  const u32 maxl = u32(b.maxwin / 2);
  c.ensure_status(2 * size_t(b.W), s);
  u32 *ctr = c.take_counter(s);
  const u32 ep = c.next_epoch();
  const size_t smem = sizeof(XSmem);
  c.smem_optin(reinterpret_cast<const void *>(k_window_select), smem);
  k_window_select<<<b.W, kXT, smem, s>>>(b, sa.sa, sa.lcp, min_len, maxl, w.cl, w.cs, w.cg, w.state, w.glen,
                                         w.gbase, w.gwin, w.gpos, m_dev, G_dev, big, c.status, ctr, ep);
  APO_CHECK_LAUNCH();
  c.launches++;
  u64 h[6];
  c.read_words(reinterpret_cast<u32 *>(h), w.scal, 12, s);
  if (u32(h[5]) != 0) return false;
  w.m = i64(h[0]);
  w.G = i64(h[1]);
  return true;
}

}  // namespace apo
