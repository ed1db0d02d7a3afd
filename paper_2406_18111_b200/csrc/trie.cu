// trie.cu -- a10/a11: the candidate trace set and the batched matcher.
//
// IngestCandidates (Alg. 1):
//   * materialise every repeat's content S[start : start+length) from its
//     window; "recorded traces are broken into pieces of a given maximum
//     size" (reading R15): consecutive max_len pieces, the tail
//     kept iff >= min_len;
//   * order the pieces by (length desc, content lexicographic asc) and merge
//     identical contents -> trace ids 0..T-1 in that order.
//   The content order comes from ONE generalized suffix array over all
//   pieces (each piece ends with its own sentinel $_w, $_0 < $_1 < ... <
//   every token): the rank of a piece's full suffix orders it among all
//   pieces; identical neighbours are merged after a warp-parallel direct
//   comparison.  The sorted, deduplicated trace list is the trie in array
//   form (a node = an LCP interval of it).
//
// Matching (Alg. 1 AdvanceActiveCandidates / FilterInvalid /
// FilterCompleted; MATCH_ALL, reading R14):
//   report every (stream, end, trace) with stream[end-|t|+1 .. end] == t.
//   One generalized suffix array over streams + traces: the stream suffixes
//   that start with trace t form the LCP interval around t's own full suffix
//   (maximal rank range with LCP >= |t|), found in O(log n) with a sparse
//   table; the interval is enumerated with a load-balanced scan and the hits
//   are radix-sorted by (stream, end, trace).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pipeline.cuh"

#include "trie.cuh"

namespace apo {
namespace {

constexpr int T256 = 256;

// ------------------------------------------------------------ pieces ----
struct SrcRep {
  const apo_repeat *rep;
  const i64 *rep_off;  // device, nwin+1
  const i64 *src_off;  // device, nwin+1 (source windows)
  int nwin;
  i64 nrep;
  i32 min_len, max_len;
};

__device__ __forceinline__ int rep_window(const SrcRep &s, i64 r) {
  int lo = 0, hi = s.nwin - 1;  // last w with rep_off[w] <= r
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (s.rep_off[mid] <= r)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ i64 n_pieces(i64 len, i32 min_len, i32 max_len) {
  if (max_len <= 0 || len <= max_len) return 1;
  i64 full = len / max_len, tail = len % max_len;
  return full + ((tail > 0 && tail >= min_len) ? 1 : 0);
}

struct PieceCountF {
  SrcRep s;
  u32 *piece_base;
  i64 *total;
  __device__ u32 load(i64 r) const { return u32(n_pieces(s.rep[r].length, s.min_len, s.max_len)); }
  __device__ bool store(i64 r, u32 incl, u32 excl) const {
    piece_base[r] = excl;
    if (r == s.nrep - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_pieces(SrcRep s, const u32 *__restrict__ piece_base, i64 *__restrict__ p_src,
                         i32 *__restrict__ p_len) {
  i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= s.nrep) return;
  apo_repeat rp = s.rep[r];
  int w = rep_window(s, r);
  i64 src = s.src_off[w] + rp.start;
  i64 np = n_pieces(rp.length, s.min_len, s.max_len);
  i64 step = (s.max_len > 0 && rp.length > s.max_len) ? s.max_len : rp.length;
  for (i64 q = 0; q < np; ++q) {
    i64 a = q * step;
    i64 ln = rp.length - a < step ? rp.length - a : step;
    p_src[piece_base[r] + q] = src + a;
    p_len[piece_base[r] + q] = i32(ln);
  }
}

// one warp per piece: copy its tokens
__global__ void k_copy_pieces(const u64 *__restrict__ src_tok, const i64 *__restrict__ p_src,
                              const i64 *__restrict__ p_off, i64 np, u64 *__restrict__ dst) {
  i64 p = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (p >= np) return;
  i64 a = p_src[p], o = p_off[p], n = p_off[p + 1] - o;
  for (i64 k = lane; k < n; k += 32) dst[o + k] = src_tok[a + k];
}

// the same, each piece written back to front (the trace set keeps only its
// reversed traces, the form the matcher reads; the forward form is made on
// demand by trie_forward)
__global__ void k_copy_pieces_rev(const u64 *__restrict__ src_tok, const i64 *__restrict__ p_src,
                                  const i64 *__restrict__ p_off, i64 np, u64 *__restrict__ dst) {
  i64 p = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (p >= np) return;
  i64 a = p_src[p], o = p_off[p], n = p_off[p + 1] - o;
  for (i64 k = lane; k < n; k += 32) dst[o + n - 1 - k] = src_tok[a + k];
}

// ------------------------------------------------ order + dedup ----
// warp per sorted neighbour pair: same length and same content -> not a head
__global__ void k_trace_heads(const u64 *__restrict__ tok, const i64 *__restrict__ off, const u32 *__restrict__ order,
                              i64 ntr, u32 *__restrict__ head) {
  i64 c = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (c >= ntr) return;
  if (c == 0) {
    if (lane == 0) head[0] = 1;
    return;
  }
  i64 a = order[c - 1], b = order[c];
  i64 la = off[a + 1] - off[a], lb = off[b + 1] - off[b];
  bool same = la == lb;
  // warp-uniform trip count (c, la and same are uniform across the warp), so
  // every lane takes part in every vote
  for (i64 k0 = 0; same && k0 < la; k0 += 32) {
    const i64 k = k0 + lane;
    const bool eq = k >= la || tok[off[a] + k] == tok[off[b] + k];
    same = __all_sync(0xffffffffu, eq);
  }
  same = __shfl_sync(0xffffffffu, same ? 1 : 0, 0) != 0;
  if (lane == 0) head[c] = same ? 0u : 1u;
}

struct TraceIdF {
  const u32 *head;
  const u32 *order;
  const i64 *off;
  u32 *uniq;    // uniq[id] = source piece
  i32 *ulen;    // ulen[id] = length
  i64 n;
  i64 *T_out;
  __device__ u32 load(i64 c) const { return head[c]; }
  __device__ bool store(i64 c, u32 incl, u32 excl) const {
    if (incl != excl) {
      u32 w = order[c];
      uniq[excl] = w;
      ulen[excl] = i32(off[w + 1] - off[w]);
    }
    if (c == n - 1) *T_out = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

// ---------------------------------------------------------- matching ----
struct MatchSetup {
  i64 N;                 // stream positions
  int S;                 // streams
  i64 T;                 // traces
  const i64 *off;        // stream offsets (device)
  const i32 *wid;
  const i32 *sa;         // generalized suffix array of the streams
  const u64 *tok;        // stream tokens
  const u64 *ttok;       // trace tokens (id order)
  const i64 *toff;       // trace offsets (device)
};

// Warp-cooperative comparison of trace t[0..L) with the stream suffix at p
// (ending at e), from offset `from` (a known equal prefix), 32 tokens per
// step.  Returns 0 if t is a prefix of the suffix, <0 if t sorts before it,
// >0 if after (a suffix that ends first is smaller, reading R2); *lcp gets
// the matched length.  All lanes return the same values.
__device__ __forceinline__ int warp_cmp_trace_suffix(const u64 *__restrict__ S, i64 p, i64 e,
                                                     const u64 *__restrict__ t, i64 L, i64 from, i64 *lcp) {
  const int lane = threadIdx.x & 31;
  for (i64 base = from; base < L; base += 32) {
    const i64 k = base + lane;
    int res = 0;
    if (k < L) {
      if (p + k >= e) {
        res = 1;
      } else {
        const u64 x = t[k], y = S[p + k];
        res = x == y ? 0 : (x < y ? -1 : 1);
      }
    }
    const u32 m = __ballot_sync(0xffffffffu, res != 0);
    if (m) {
      const int f = __ffs(m) - 1;
      *lcp = base + f;
      return __shfl_sync(0xffffffffu, res, f);
    }
  }
  *lcp = L;
  return 0;
}

// First suffix rank r in [0, N) with cmp(t, s_r) <= 0 (STRICT = false: the
// first suffix that has t as a prefix or sorts after t) or < 0 (STRICT =
// true: the first suffix after every suffix that has t as a prefix).
// Manber-Myers binary search: comparisons start at min(lcp with the two
// bracketing suffixes).  One warp per search.
template <bool STRICT>
__device__ __forceinline__ i64 trace_bound(const MatchSetup &m, const u64 *t, i64 L) {
  i64 lo = -1, hi = m.N, llo = 0, lhi = 0;
  while (hi - lo > 1) {
    const i64 mid = lo + ((hi - lo) >> 1);
    const i64 p = m.sa[mid];
    const i64 e = m.off[m.wid[p] + 1];
    i64 l;
    const int c = warp_cmp_trace_suffix(m.tok, p, e, t, L, llo < lhi ? llo : lhi, &l);
    if (STRICT ? (c < 0) : (c <= 0)) {
      hi = mid;
      lhi = l;
    } else {
      lo = mid;
      llo = l;
    }
  }
  return hi;
}

// Each trace's interval of stream suffixes that start with it (warp per trace).
__global__ void k_trace_search(MatchSetup m, i64 *__restrict__ ilo, u32 *__restrict__ icnt) {
  const i64 t = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= m.T) return;
  const u64 *tt = m.ttok + m.toff[t];
  const i64 L = m.toff[t + 1] - m.toff[t];
  const i64 a = trace_bound<false>(m, tt, L);
  const i64 b = trace_bound<true>(m, tt, L);
  if ((threadIdx.x & 31) == 0) {
    ilo[t] = a;
    icnt[t] = u32(b - a);
  }
}

struct CountScanF {
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

__global__ void k_enumerate(MatchSetup m, const i64 *__restrict__ ilo, const u32 *__restrict__ ibase, i64 Z,
                            int bE, int bT, u64 *__restrict__ keys) {
  i64 z = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (z >= Z) return;
  // trace owning slot z: last t with ibase[t] <= z
  i64 lo = 0, hi = m.T - 1;
  while (lo < hi) {
    i64 mid = (lo + hi + 1) >> 1;
    if (i64(ibase[mid]) <= z)
      lo = mid;
    else
      hi = mid - 1;
  }
  const i64 t = lo;
  const i64 p = m.sa[ilo[t] + (z - i64(ibase[t]))];
  const int q = m.wid[p];
  const i64 L = m.toff[t + 1] - m.toff[t];
  const i64 end = p - m.off[q] + L - 1;
  keys[z] = (u64(q) << (bE + bT)) | (u64(end) << bT) | u64(t);
}

__global__ void k_write_hits(const u64 *__restrict__ keys, i64 nhits, i64 cap, int bE, int bT,
                             apo_match_rec *__restrict__ out) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nhits || i >= cap) return;
  u64 k = keys[i];
  apo_match_rec r;
  r.trace_id = i32(k & ((1ull << bT) - 1));
  r.end_pos = i32((k >> bT) & ((1ull << bE) - 1));
  r.stream = i32(k >> (bE + bT));
  r.slot = r.trace_id;  // this path's per-stream trace key is the trace id
  out[i] = r;
}

// position -> window map: one CTA per window fills its range (coalesced)
__global__ void k_fill_wid_t(const i64 *__restrict__ off, int W, i64 N, i32 *__restrict__ wid) {
  const int w = blockIdx.x;
  if (w >= W) return;
  const i64 e = off[w + 1];
  for (i64 i = off[w] + threadIdx.x; i < e; i += blockDim.x) wid[i] = w;
}

// Generalized SA setup for a host-described batch; returns the carved work.
struct GenPlan {
  SAWork sa{};
  i64 *d_off = nullptr;
  i32 *d_wid = nullptr;
};

void plan_gen(Carver &cv, Batch &b, GenPlan &g, bool lcp, int nsmid) {
  g.d_off = cv.take<i64>(size_t(b.W) + 1);
  g.d_wid = cv.take<i32>(size_t(b.N));
  plan_sa(cv, b, g.sa, lcp, nsmid);
}

void upload_batch(Ctx &c, Batch &b, GenPlan &g, const std::vector<i64> &h_off, cudaStream_t s) {
  c.h2d(g.d_off, h_off.data(), sizeof(i64) * h_off.size(), s);
  k_fill_wid_t<<<b.W, T256, 0, s>>>(g.d_off, b.W, b.N, g.d_wid);
  APO_CHECK_LAUNCH();
  c.launches++;
  b.off = g.d_off;
  b.wid = g.d_wid;
}


// reversed copies for the on-chip matcher: dst[off[w] + j] = src[off[w+1] - 1 - j]
__global__ void k_reverse_by_wid(const u64 *__restrict__ src, const i64 *__restrict__ off,
                                 const i32 *__restrict__ wid, i64 N, u64 *__restrict__ dst) {
  const i64 p = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int w = wid[p];
  dst[p] = src[off[w] + off[w + 1] - 1 - p];
}

__global__ void k_reverse_traces(const u64 *__restrict__ src, const i64 *__restrict__ off, i64 T,
                                 u64 *__restrict__ dst) {
  const i64 t = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const i64 o = off[t], L = off[t + 1] - o;
  for (i64 k = lane; k < L; k += 32) dst[o + k] = src[o + L - 1 - k];
}

// the forward traces (the trace set keeps the reversed ones): made once, on
// the first use by a path that reads them (streams > 16,384 tokens)
void trie_forward(Ctx &c, const apo_trie *tr, cudaStream_t s) {
  if (tr->d_tok || tr->T == 0) return;
  tr->d_tok = static_cast<u64 *>(c.pool_get(tr->tok_bytes));
  k_reverse_traces<<<grid_for(tr->T * 32, T256), T256, 0, s>>>(tr->d_rtok, tr->d_off, tr->T, tr->d_tok);
  APO_CHECK_LAUNCH();
  c.launches++;
}

// ------------------------------------------- per-stream matching path ----
// Every stream gets its own suffix array (K9 on chip for streams <= 16K);
// each stream's SA is cut into buckets of equal first token; a trace is
// binary-searched only in the buckets whose first token equals its own first
// token (an exact filter: elsewhere it cannot occur).
struct StreamMatch {
  const i64 *off;   // stream offsets
  const i32 *wid;
  const i32 *sa;    // per-stream (window-major) suffix arrays, global positions
  const i32 *lcp;   // per-stream LCP (lcp[k] = LCP(sa[k], sa[k+1]), 0 at a stream end)
  const u64 *tok;   // stream tokens
  const u64 *ttok;  // trace tokens
  const i64 *toff;  // trace offsets
  i64 N, T;
};


// The same buckets, one CTA per stream (streams claimed in order; their
// bucket counts combined by a decoupled look-back): heads counted, the
// stream's base found, then the heads written in rank order with their end
// (the next head of the stream, or the stream's end) -- two sequential reads
// of the stream's LCP instead of a device-wide scan with random window-id
// lookups.
constexpr int kBkThreads = 1024;
constexpr int kBkPer = 16;  // consecutive ranks per thread in the write pass

__global__ void __launch_bounds__(kBkThreads) k_stream_buckets(StreamMatch m, const unsigned short *__restrict__ sid,
                                                              u64 *__restrict__ e_tok, u32 *__restrict__ e_lo,
                                                              u32 *__restrict__ e_q, u32 *__restrict__ e_hi,
                                                              u32 *__restrict__ e_idx, i64 *__restrict__ total,
                                                              int W, u64 *status, u32 *counter, u32 epoch,
                                                              int depth) {
  __shared__ u32 s_w, s_base, s_wsum[kBkThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_w = atomicAdd(counter, 1u);
  __syncthreads();
  const int w = int(s_w);
  const i64 beg = m.off[w], n = m.off[w + 1] - beg;
  // depth 1: a bucket per first token; depth 2 (ids): per first two tokens
  auto head = [&](i64 r) -> u32 { return (r == 0 || m.lcp[beg + r - 1] < depth) ? 1u : 0u; };
  u32 cnt = 0;
  for (i64 r = tid; r < n; r += kBkThreads) cnt += head(r);
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) s_wsum[warp] = cnt;
  __syncthreads();
  if (warp == 0) {
    u32 v = s_wsum[lane];
    v = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) {
      u32 pre = 0;
      if (w == 0) {
        lb_store(status, lb_pack(epoch, kFlagInc, v));
      } else {
        lb_store(status + w, lb_pack(epoch, kFlagAgg, v));
        pre = lb_lookback<false>(status, 1, 0, w, epoch);
        lb_store(status + w, lb_pack(epoch, kFlagInc, pre + v));
      }
      s_base = pre;
      if (w == W - 1) *total = i64(pre + v);
    }
  }
  __syncthreads();
  const u32 base = s_base;
  u32 run = base;  // heads written so far
  for (i64 t0 = 0; t0 < n; t0 += i64(kBkThreads) * kBkPer) {
    const i64 r0 = t0 + i64(tid) * kBkPer;
    u32 bits = 0;
#pragma unroll
    for (int j = 0; j < kBkPer; ++j)
      if (r0 + j < n && head(r0 + j)) bits |= 1u << j;
    const u32 c = __popc(bits);
    u32 incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const u32 x = s_wsum[lane];
      u32 y = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 o = __shfl_up_sync(0xffffffffu, y, d);
        if (lane >= d) y += o;
      }
      s_wsum[lane] = y - x;
    }
    __syncthreads();
    u32 o = run + s_wsum[warp] + incl - c;
    const u32 tile_total = __shfl_sync(0xffffffffu, incl, 31);  // (this warp's; the CTA total follows)
    (void)tile_total;
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      const i64 k = beg + r0 + j;
      const i64 p = m.sa[k];
      if (depth == 2)  // (id0 + 1, id1 + 1 or 0 past the stream end)
        e_tok[o] = (u64(sid[p]) << 17) | u64(p + 1 < beg + n ? sid[p + 1] : 0u);
      else
        e_tok[o] = sid ? u64(sid[p]) : m.tok[p];
      e_lo[o] = u32(k);
      e_q[o] = u32(w);
      e_idx[o] = o;
      ++o;
    }
    __syncthreads();
    if (tid == kBkThreads - 1) s_base = o;  // the last thread's end = heads through this tile
    __syncthreads();
    run = s_base;
  }
  __syncthreads();  // every head's e_lo is written and visible to the CTA
  for (u32 e = base + tid; e < run; e += kBkThreads) e_hi[e] = e + 1 < run ? e_lo[e + 1] : u32(beg + n);
}


// per trace: range [ea, eb) of token-sorted buckets with the trace's first token
__global__ void k_trace_buckets(StreamMatch m, const u64 *__restrict__ sorted_tok, i64 E, u32 *__restrict__ ea,
                                u32 *__restrict__ ecnt, const u32 *__restrict__ tid, int depth) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= m.T) return;
  u64 a;
  if (tid != nullptr) {  // buckets keyed by dense id + 1; a token absent from the batch has none
    const u32 x = tid[m.toff[t]];
    const u32 y = depth == 2 ? tid[m.toff[t] + 1] : 0u;  // (traces are >= 2 long at depth 2)
    if ((x | y) & 1u) {
      ea[t] = 0;
      ecnt[t] = 0;
      return;
    }
    a = depth == 2 ? (u64(x >> 1) << 17) | u64(y >> 1) : u64(x >> 1);
  } else {
    a = m.ttok[m.toff[t]];
  }
  i64 lo = 0, hi = E;
  while (lo < hi) {
    i64 mid = (lo + hi) >> 1;
    if (sorted_tok[mid] < a) lo = mid + 1; else hi = mid;
  }
  const i64 first = lo;
  hi = E;
  while (lo < hi) {
    i64 mid = (lo + hi) >> 1;
    if (sorted_tok[mid] <= a) lo = mid + 1; else hi = mid;
  }
  ea[t] = u32(first);
  ecnt[t] = u32(lo - first);
}

struct PairBaseF {  // exclusive scan of per-trace pair counts (u32)
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

// first rank r in [lo0, hi0) of one stream's SA with cmp(t, s_r) <= 0
// (STRICT: < 0); comparisons start at `from` (a known common prefix)
template <bool STRICT>
__device__ __forceinline__ i64 range_bound(const StreamMatch &m, i64 lo0, i64 hi0, i64 e, const u64 *t, i64 L,
                                           i64 from, i64 *lcp_hi) {
  i64 lo = lo0 - 1, hi = hi0, llo = from, lhi = -1;  // lhi < 0: hi is the range end (not compared)
  while (hi - lo > 1) {
    const i64 mid = lo + ((hi - lo) >> 1);
    i64 l;
    // Manber-Myers skip: lcp(t, S_mid) >= min(lcp(t, S_lo), lcp(t, S_hi)) holds only
    // once BOTH brackets were compared; before that only `from` is known
    const i64 st = lhi < 0 ? from : (llo < lhi ? llo : lhi);
    const int c = warp_cmp_trace_suffix(m.tok, m.sa[mid], e, t, L, st, &l);
    if (STRICT ? (c < 0) : (c <= 0)) {
      hi = mid;
      lhi = l;
    } else {
      lo = mid;
      llo = l;
    }
  }
  *lcp_hi = lhi;
  return hi;
}

// warp per (trace, bucket) pair: the trace's interval inside the bucket
// One warp per chunk of kPairChunk consecutive (trace, bucket) pairs: one
// trace lookup per chunk, then the pairs in order (pairs are grouped by
// trace), each: the trace's lower bound in the bucket (warp-cooperative
// Manber-Myers search), then the interval extended while the stream LCP stays
// >= |t| (32 LCP entries per step).
constexpr int kPairChunk = 16;

__global__ void k_pair_search(StreamMatch m, const u32 *__restrict__ pbase, const u32 *__restrict__ ea, i64 P,
                              const u32 *__restrict__ e_order, const u32 *__restrict__ e_lo,
                              const u32 *__restrict__ e_hi, const u32 *__restrict__ e_q, i64 *__restrict__ ilo,
                              u32 *__restrict__ icnt, u32 *__restrict__ ptrace) {
  const i64 z0 = ((i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kPairChunk;
  if (z0 >= P) return;
  const int lane = threadIdx.x & 31;
  i64 lo = 0, hi = m.T - 1;  // trace owning pair z0: last t with pbase[t] <= z0
  while (lo < hi) {
    i64 mid = (lo + hi + 1) >> 1;
    if (i64(pbase[mid]) <= z0) lo = mid; else hi = mid - 1;
  }
  i64 t = lo;
  const i64 z1 = z0 + kPairChunk < P ? z0 + kPairChunk : P;
  for (i64 z = z0; z < z1; ++z) {
    while (t + 1 < m.T && i64(pbase[t + 1]) <= z) ++t;
    const u32 e = e_order[ea[t] + (z - i64(pbase[t]))];
    const i64 q = e_q[e];
    const u64 *tt = m.ttok + m.toff[t];
    const i64 L = m.toff[t + 1] - m.toff[t];
    const i64 end = m.off[q + 1];
    i64 la;
    const i64 a = range_bound<false>(m, e_lo[e], e_hi[e], end, tt, L, 1, &la);
    i64 cnt = 0;
    if (la >= L) {
      const i64 lim = e_hi[e];
      cnt = 1;
      for (i64 k0 = a; k0 + 1 < lim; k0 += 32) {
        const i64 k = k0 + lane;
        const bool ok = (k + 1 < lim) && m.lcp[k] >= L;
        const u32 bad = __ballot_sync(0xffffffffu, !ok);
        if (bad) {
          cnt += __ffs(bad) - 1;
          break;
        }
        cnt += 32;
      }
    }
    if (lane == 0) {
      ilo[z] = a;
      icnt[z] = u32(cnt);
      ptrace[z] = u32(t);
    }
  }
}

// ---- per-stream CTA matcher: pairs grouped by stream, the stream's tokens,
// local SA and LCP staged in shared memory, so every step of every binary
// search is an on-chip access (only the trace tokens come from L2/HBM).
constexpr int kSMThreads = 1024;
constexpr int kSMMax = 16384;  // longest stream handled on chip

__global__ void k_pair_list(const u32 *__restrict__ pbase, const u32 *__restrict__ ea, const u32 *__restrict__ ecnt,
                            const u32 *__restrict__ e_order, const u32 *__restrict__ e_q, i64 T,
                            u32 *__restrict__ pair_e, u32 *__restrict__ ptrace, u64 *__restrict__ qkey,
                            u32 *__restrict__ qval) {
  const i64 t = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const i64 z0 = pbase[t], n = ecnt[t], e0 = ea[t];
  for (i64 j = lane; j < n; j += 32) {
    const u32 e = e_order[e0 + j];
    pair_e[z0 + j] = e;
    ptrace[z0 + j] = u32(t);
    qkey[z0 + j] = u64(e_q[e]);
    qval[z0 + j] = u32(z0 + j);
  }
}

// Launch order of the per-stream CTAs: the streams with the most pairs
// first (longest-processing-time first, so the heaviest streams do not finish
// last; measured 0.55 ms faster on C4 than ordering by the first pair's
// trace for L2 sharing).
__global__ void k_stream_keys(const u32 *__restrict__ qoff, const u32 *__restrict__ zsorted,
                              const u32 *__restrict__ ptrace, int S, i64 T, u64 *__restrict__ key,
                              u32 *__restrict__ val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= S) return;
  (void)zsorted;
  (void)ptrace;
  (void)T;
  key[q] = u64(0xffffffffu - (qoff[q + 1] - qoff[q]));  // most pairs first (32-bit key)
  val[q] = u32(q);
}

// qoff[q] = first index of stream q in the stream-sorted pair list
__global__ void k_q_offsets(const u64 *__restrict__ qkey, i64 P, int S, u32 *__restrict__ qoff) {
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q > S) return;
  i64 lo = 0, hi = P;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (i64(qkey[mid]) < q) lo = mid + 1; else hi = mid;
  }
  qoff[q] = u32(lo);
}

constexpr int kCmpChunks = 8;  // trace tokens fetched per round trip: 8 x 32

// Matcher statistics (diagnostics only; compiled out unless APO_MATCH_STATS
// is 1): lane 0 of each searching warp adds event counts to match_stats.
#ifndef APO_MATCH_STATS
#define APO_MATCH_STATS 0
#endif
#if APO_MATCH_STATS
__device__ unsigned long long match_stats[16];
#define MS_ADD(i, v)                                                         \
  do {                                                                       \
    if ((threadIdx.x & 31) == 0) atomicAdd(&match_stats[i], (unsigned long long)(v)); \
  } while (0)
#else
#define MS_ADD(i, v)
#endif

// Warp-cooperative compare of trace t with the on-chip stream suffix at p;
// the trace's first 64 tokens live in registers (r0 = t[lane],
// r1 = t[32 + lane]), later tokens come from global memory.  Each 32-token
// step only tests inequality (one ballot); the order of the first differing
// token is resolved once, at the end.
__device__ __forceinline__ int cmp_at(u64 x, const u64 *__restrict__ S, i64 pk, i64 n) {
  return pk >= n ? 1 : (x < S[pk] ? -1 : 1);  // called for a differing (or past-the-end) position only
}

__device__ __forceinline__ int warp_cmp_smem(const u64 *__restrict__ S, i64 p, i64 n, const u64 *__restrict__ t,
                                             u64 r0, u64 r1, i64 L, i64 from, i64 *lcp) {
  const int lane = threadIdx.x & 31;
  i64 base = from;
  // tokens 0..63 of the trace come from registers
  for (; base < L && base < 64; base += 32) {
    const i64 k = base + lane;
    const int src = int(k & 31);
    const u64 a = __shfl_sync(0xffffffffu, r0, src);
    const u64 b = __shfl_sync(0xffffffffu, r1, src);
    const u64 x = k < 32 ? a : (k < 64 ? b : (k < L ? t[k] : 0ull));
    const bool ne = k < L && (p + k >= n || x != S[p + k]);
    const u32 m = __ballot_sync(0xffffffffu, ne);
    MS_ADD(5, 1);
    if (m) {
      const int f = __ffs(m) - 1;
      *lcp = base + f;
      return __shfl_sync(0xffffffffu, ne ? cmp_at(x, S, p + k, n) : 0, f);
    }
  }
  // later tokens: kCmpChunks 32-token chunks per round trip to L2/HBM
  for (; base < L; base += 32 * kCmpChunks) {
    MS_ADD(6, 1);
    u64 x[kCmpChunks];
#pragma unroll
    for (int c = 0; c < kCmpChunks; ++c) {
      const i64 k = base + c * 32 + lane;
      x[c] = k < L ? t[k] : 0ull;
    }
#pragma unroll
    for (int c = 0; c < kCmpChunks; ++c) {
      const i64 k = base + c * 32 + lane;
      const bool ne = k < L && (p + k >= n || x[c] != S[p + k]);
      const u32 m = __ballot_sync(0xffffffffu, ne);
      MS_ADD(7, 1);
      if (m) {
        const int f = __ffs(m) - 1;
        *lcp = base + c * 32 + f;
        return __shfl_sync(0xffffffffu, ne ? cmp_at(x[c], S, p + k, n) : 0, f);
      }
    }
  }
  *lcp = L;
  return 0;
}

__global__ void __launch_bounds__(kSMThreads, 1) k_stream_match(StreamMatch m, const u32 *__restrict__ zsorted,
                                                                const u32 *__restrict__ qoff,
                                                                const u32 *__restrict__ pair_e,
                                                                const u32 *__restrict__ ptrace,
                                                                const u32 *__restrict__ e_lo,
                                                                const u32 *__restrict__ e_hi, i64 *__restrict__ ilo,
                                                                u32 *__restrict__ icnt, u32 *__restrict__ qtot,
                                                                const u32 *__restrict__ qorder) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ u32 s_tot, s_next;
  __shared__ unsigned short s_bmin[kSMMax / 32];  // minima of LC over 32-entry blocks
  const int q = int(qorder[blockIdx.x]);
  const i64 z0 = qoff[q], z1 = qoff[q + 1];
  if (z0 == z1) {
    if (threadIdx.x == 0) qtot[q] = 0;
    return;
  }
  if (threadIdx.x == 0) {
    s_tot = 0;
    s_next = kSMThreads / 32;
  }
  const i64 beg = m.off[q], n = m.off[q + 1] - beg;
  u64 *S = reinterpret_cast<u64 *>(smem);
  unsigned short *SA = reinterpret_cast<unsigned short *>(S + kSMMax);
  unsigned short *LC = SA + kSMMax;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (i64 i = threadIdx.x; i < ((n + 31) & ~i64(31)); i += kSMThreads) {
    u32 v = 0xffffu;
    if (i < n) {
      S[i] = m.tok[beg + i];
      SA[i] = (unsigned short)(m.sa[beg + i] - beg);
      v = u32(m.lcp[beg + i]);
      LC[i] = (unsigned short)v;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, d));
    if (lane == 0) s_bmin[i >> 5] = (unsigned short)v;
  }
  __syncthreads();
  // lcp(S_a, S_b) = min LC[a .. b-1]: partial blocks directly, whole blocks
  // from their minima
  auto range_min = [&](i64 a, i64 b) -> u32 {
    u32 mn = 0xffffu;
    const i64 ba = (a + 31) >> 5, bb = b >> 5;
    if (ba >= bb) {
      for (i64 k = a + lane; k < b; k += 32) mn = min(mn, u32(LC[k]));
    } else {
      const i64 k1 = a + lane, k2 = (bb << 5) + lane;
      if (k1 < (ba << 5)) mn = min(mn, u32(LC[k1]));
      if (k2 < b) mn = min(mn, u32(LC[k2]));
      for (i64 k = ba + lane; k < bb; k += 32) mn = min(mn, u32(s_bmin[k]));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    return mn;
  };
  // pairs are handed out one at a time (the first 32 statically), so a few
  // long searches do not leave the other warps idle at the end
  for (i64 i = z0 + warp; i < z1;) {
    const u32 z = zsorted[i];
    const u32 e = pair_e[z];
    const i64 t = ptrace[z];
    const u64 *tt = m.ttok + m.toff[t];
    const i64 L = m.toff[t + 1] - m.toff[t];
    const i64 lo0 = e_lo[e] - beg, hi0 = e_hi[e] - beg;
    const u64 r0 = lane < L ? tt[lane] : 0ull, r1 = 32 + lane < L ? tt[32 + lane] : 0ull;
    // lower bound: first local rank r in [lo0, hi0) with cmp(t, s_r) <= 0.
    // Manber-Myers with LCP-LR: l = lcp(t, S_lo), r = lcp(t, S_hi); when
    // both brackets are real and l != r, lcp(S_lo or S_hi, S_mid) (a warp
    // min over the on-chip LCP array) decides the step without comparing
    // tokens; tokens are compared only from the known lcp onwards.
    i64 lo = lo0 - 1, hi = hi0, llo = 1, lhi = -1;
    MS_ADD(0, 1);
    MS_ADD(1, L);
    MS_ADD(10, hi0 - lo0);
    while (hi - lo > 1) {
      MS_ADD(2, 1);
      const i64 mid = lo + ((hi - lo) >> 1);
      const bool real = lo >= lo0 && lhi >= 0;
      i64 st = 1;
      if (real && llo != lhi) {
        const bool left = llo > lhi;
        const i64 a = left ? lo : mid, b = left ? mid : hi;  // lcp(S_a, S_b) = min LC[a..b-1]
        const i64 x = range_min(a, b);
        MS_ADD(3, 1);
        if (left) {
          if (x > llo) { lo = mid; continue; }            // S_mid < t, lcp(t, S_mid) = llo
          if (x < llo) { hi = mid; lhi = x; continue; }   // t < S_mid, lcp = x
          st = llo;
        } else {
          if (x > lhi) { hi = mid; continue; }            // t <= S_mid, lcp = lhi
          if (x < lhi) { lo = mid; llo = x; continue; }   // S_mid < t, lcp = x
          st = lhi;
        }
      } else if (real) {
        st = llo;
      } else if (lhi >= 0) {
        st = 1;  // lower bracket virtual
      }
      i64 l;
      const int c = warp_cmp_smem(S, SA[mid], n, tt, r0, r1, L, st, &l);
      MS_ADD(4, 1);
      MS_ADD(11, l - st);
      if (c <= 0) {
        hi = mid;
        lhi = l;
      } else {
        lo = mid;
        llo = l;
      }
    }
    i64 cnt = 0;
    if (lhi >= L) {
      // the interval extends while LC[k] >= L (k + 1 < hi0): first the rest
      // of hi's 32-entry block, then 32 blocks per step by their minima
      const i64 kend = hi0 - 1;
      i64 k = hi, stop = -1;
      {
        const i64 bend = min(((k >> 5) + 1) << 5, kend);
        const i64 kk = k + lane;
        const u32 bad = __ballot_sync(0xffffffffu, kk < bend && i64(LC[kk]) < L);
        if (bad)
          stop = k + __ffs(bad) - 1;
        else
          k = bend;
      }
      while (stop < 0 && k < kend) {  // k is block aligned here
        const i64 b = (k >> 5) + lane;
        const bool cand = (b << 5) < kend && ((b << 5) + 32 > kend || i64(s_bmin[b]) < L);
        const u32 cb = __ballot_sync(0xffffffffu, cand);
        if (!cb) {
          k += 32 * 32;
          continue;
        }
        const i64 fb = (k >> 5) + __ffs(cb) - 1;
        const i64 kk = (fb << 5) + lane;
        const u32 bad = __ballot_sync(0xffffffffu, kk < kend && i64(LC[kk]) < L);
        stop = bad ? (fb << 5) + __ffs(bad) - 1 : min((fb << 5) + 32, kend);
      }
      if (stop < 0) stop = kend;
      cnt = 1 + (stop - hi);
    }
    MS_ADD(8, cnt > 0);
    MS_ADD(9, cnt);
    u32 nx = 0;
    if (lane == 0) {
      ilo[z] = beg + hi;
      icnt[z] = u32(cnt);
      if (cnt) atomicAdd(&s_tot, u32(cnt));
      nx = atomicAdd(&s_next, 1u);
    }
    i = z0 + __shfl_sync(0xffffffffu, nx, 0);
  }
  __syncthreads();
  if (threadIdx.x == 0) qtot[q] = s_tot;
}

// ---- the same matcher over dense token ids (the common path) ----
// When the stream batch's dictionary holds at most 65,534 distinct tokens,
// K2's order-preserving ids stand in for the 64-bit tokens:
//  * stream token -> y = id + 1 (u16, in shared memory; y = 0 past the end),
//  * trace token  -> 2 * (id + 1) if the token occurs in the batch, else 1;
//    0xffffffff past the trace end.
// Equal tokens give x == 2y, and for tokens of the batch x < 2y exactly when
// the token is smaller, so every comparison of a trace made of batch tokens
// decides as on the raw tokens (the past-the-end values sort as a shorter
// suffix / an exhausted trace do); a trace holding another token matches
// nowhere, and its search only has to end (k_trace_ids).  Per pair the search needs
// one 16-byte record (k_pair_meta) instead of a chain of dependent lookups,
// the stream half of each 32-token step is one 64-B shared-memory wavefront,
// and the CTA fits twice per SM (512 threads, ~109 KB).
constexpr int kSMIThreads = 512;
constexpr int kSMIWarps = kSMIThreads / 32;
constexpr int kSMIPad = 256;    // zero entries past the stream end (a trip reads <= 256 past its start)
constexpr int kSMICache = 64;  // leading trace ids per warp kept in shared memory (measured: 64 beats 128)
constexpr u32 kTraceEnd = 0xffffffffu;


// trace token -> comparison value against the batch dictionary dk[0..K0)
// (sorted distinct tokens except ~0): 2 (rank + 1) for a token of the batch,
// else 1.  A trace holding a token absent from the stream batch occurs
// nowhere in it: its comparisons with stream suffixes (stream values 2 (id +
// 1), 0 past the end) never reach its full length, so it gets no bucket, no
// interval and no hit whatever order its absent tokens take -- they only
// need a value that equals no stream value.  One probe of an open-addressing
// table of 16-B (token, rank) slots, at most a quarter full: one L2 request
// for a token of the batch, ~1.4 for an absent one (at N > 1 most of the
// peers' trace tokens).  N = 4 union, 184 M trace tokens: 0.99 ms; 2.99 ms
// with a (token) + (rank) table and a binary search over dk for the exact
// rank of an absent token, 3.1 ms with a two-level search for every token.
__device__ __forceinline__ u32 dict_hash(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return u32(z ^ (z >> 31));
}

__global__ void k_dict_build(const u64 *__restrict__ dk, i64 K0, ulonglong2 *__restrict__ slot, u32 mask) {
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= K0) return;
  const u64 v = dk[r];
  for (u32 h = dict_hash(v) & mask;; h = (h + 1) & mask) {
    if (atomicCAS(reinterpret_cast<unsigned long long *>(&slot[h].x), ~0ull, v) == ~0ull) {
      slot[h].y = u64(r);
      return;
    }
  }
}

__global__ void k_trace_ids(const u64 *__restrict__ tok, i64 n, i64 K0, int has_max,
                            const ulonglong2 *__restrict__ slot, u32 mask, u32 *__restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 v = tok[i];
  if (v == ~0ull) {
    out[i] = has_max ? u32(2 * (K0 + 1)) : 1u;
    return;
  }
  for (u32 h = dict_hash(v) & mask;; h = (h + 1) & mask) {
    const ulonglong2 e = __ldg(&slot[h]);
    if (e.x == v) {
      out[i] = 2u * (u32(e.y) + 1u);
      return;
    }
    if (e.x == ~0ull) {
      out[i] = 1u;
      return;
    }
  }
}

// per stream-sorted pair i: (lo | hi << 16) local to the stream, pair id z,
// trace offset, trace length
__global__ void k_pair_meta(const u64 *__restrict__ sqk, const u32 *__restrict__ sqv, i64 P,
                            const u32 *__restrict__ pair_e, const u32 *__restrict__ ptrace,
                            const u32 *__restrict__ e_lo, const u32 *__restrict__ e_hi, const i64 *__restrict__ off,
                            const i64 *__restrict__ toff, uint4 *__restrict__ meta) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const u32 z = sqv[i];
  const u32 e = pair_e[z], t = ptrace[z];
  const i64 beg = off[sqk[i]];
  const i64 a = toff[t], b = toff[t + 1];
  meta[i] = make_uint4(u32(e_lo[e] - beg) | (u32(e_hi[e] - beg) << 16), z, u32(a), u32(b - a));
}

// Warp compare of the trace (ids: Tc = the first kSMICache in shared memory,
// tg = all in global memory) with the stream suffix at p, from token `from`
// on (the known common prefix).  Returns -1 / 1 (t < / > suffix) or 0 (t is
// a prefix of the suffix); *lcp = the common prefix length (capped at L).
template <int CH>
__device__ __forceinline__ bool ids_trip(const unsigned short *__restrict__ S, int p, const u32 *__restrict__ Tc,
                                         const u32 *__restrict__ tg, int L, int &base, int *lcp, int *res) {
  const int lane = threadIdx.x & 31;
  u32 x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int k = base + c * 32 + lane;
    x[c] = k < kSMICache ? Tc[k] : (k < L ? __ldg(&tg[k]) : kTraceEnd);
    y[c] = u32(S[p + k]) << 1;
  }
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const u32 m = __ballot_sync(0xffffffffu, x[c] != y[c]);
    if (m) {
      const int f = __ffs(m) - 1;
      const int k = base + c * 32 + f;
      const int r = __shfl_sync(0xffffffffu, x[c] < y[c] ? -1 : 1, f);
      *lcp = k < L ? k : L;
      *res = k < L ? r : 0;
      return true;
    }
  }
  base += CH * 32;
  return false;
}

__device__ __forceinline__ int warp_cmp_ids(const unsigned short *__restrict__ S, int p, const u32 *__restrict__ Tc,
                                            const u32 *__restrict__ tg, int L, int from, int *lcp) {
  int base = from, res = 0;
  while (base < kSMICache) {  // the cached head: two chunks per trip
    if (ids_trip<2>(S, p, Tc, tg, L, base, lcp, &res)) return res;
  }
  while (true) {  // later tokens: eight chunks per round trip to L2/HBM
    if (ids_trip<8>(S, p, Tc, tg, L, base, lcp, &res)) return res;
  }
}

__global__ void __launch_bounds__(kSMIThreads, 2)
    k_stream_match_ids(const i64 *__restrict__ soff, const i32 *__restrict__ sa, const i32 *__restrict__ lcpa,
                       const unsigned short *__restrict__ sid, const u32 *__restrict__ tid,
                       const uint4 *__restrict__ meta, const u32 *__restrict__ qoff, i64 *__restrict__ ilo,
                       u32 *__restrict__ icnt, u32 *__restrict__ qtot, const u32 *__restrict__ qorder,
                       int depth) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ u32 s_tot, s_next;
  __shared__ unsigned short s_bmin[kSMMax / 32];
  const int q = int(qorder[blockIdx.x]);
  const u32 z0 = qoff[q], z1 = qoff[q + 1];
  if (z0 == z1) {
    if (threadIdx.x == 0) qtot[q] = 0;
    return;
  }
  if (threadIdx.x == 0) {
    s_tot = 0;
    s_next = kSMIWarps;
  }
  const i64 beg = soff[q];
  const int n = int(soff[q + 1] - beg);
  unsigned short *S = reinterpret_cast<unsigned short *>(smem);
  unsigned short *SA = S + kSMMax + kSMIPad;
  unsigned short *LC = SA + kSMMax;
  u32 *Tc = reinterpret_cast<u32 *>(LC + kSMMax);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < ((n + 31) & ~31); i += kSMIThreads) {
    u32 v = 0xffffu;
    if (i < n) {
      S[i] = sid[beg + i];
      SA[i] = (unsigned short)(sa[beg + i] - beg);
      v = u32(lcpa[beg + i]);
      LC[i] = (unsigned short)v;
    }
    v = __reduce_min_sync(0xffffffffu, v);
    if (lane == 0) s_bmin[i >> 5] = (unsigned short)v;
  }
  for (int i = n + threadIdx.x; i < n + kSMIPad; i += kSMIThreads) S[i] = 0;
  __syncthreads();
  u32 *tc = Tc + warp * kSMICache;
  auto range_min = [&](int a, int b) -> u32 {  // lcp(S_a, S_b) = min LC[a .. b-1]
    u32 mn = 0xffffu;
    const int ba = (a + 31) >> 5, bb = b >> 5;
    if (ba >= bb) {
      for (int k = a + lane; k < b; k += 32) mn = min(mn, u32(LC[k]));
    } else {
      const int k1 = a + lane, k2 = (bb << 5) + lane;
      if (k1 < (ba << 5)) mn = min(mn, u32(LC[k1]));
      if (k2 < b) mn = min(mn, u32(LC[k2]));
      for (int k = ba + lane; k < bb; k += 32) mn = min(mn, u32(s_bmin[k]));
    }
    return __reduce_min_sync(0xffffffffu, mn);
  };
  u32 i = z0 + warp;
  uint4 mc = i < z1 ? meta[i] : make_uint4(0, 0, 0, 0);
  while (i < z1) {
    u32 nx = 0;
    if (lane == 0) nx = atomicAdd(&s_next, 1u);
    const u32 ni = z0 + __shfl_sync(0xffffffffu, nx, 0);
    const uint4 mn = ni < z1 ? meta[ni] : make_uint4(0, 0, 0, 0);  // consumed next iteration
    const u32 *tg = tid + mc.z;
    const int L = int(mc.w);
    const int lo0 = int(mc.x & 0xffffu), hi0 = int(mc.x >> 16);
    {
      u32 v[kSMICache / 32];
#pragma unroll
      for (int j = 0; j < kSMICache / 32; ++j) v[j] = 32 * j + lane < L ? __ldg(&tg[32 * j + lane]) : kTraceEnd;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kSMICache / 32; ++j) tc[32 * j + lane] = v[j];
      __syncwarp();
    }
    // lower bound with LCP-LR skips, as in k_stream_match; a bucket's
    // members share the trace's first `depth` tokens
    int lo = lo0 - 1, hi = hi0, llo = depth, lhi = -1;
    while (hi - lo > 1) {
      const int mid = lo + ((hi - lo) >> 1);
      const bool real = lo >= lo0 && lhi >= 0;
      int st = depth;
      if (real && llo != lhi) {
        const bool left = llo > lhi;
        const int a = left ? lo : mid, b = left ? mid : hi;
        const int x = int(range_min(a, b));
        if (left) {
          if (x > llo) { lo = mid; continue; }
          if (x < llo) { hi = mid; lhi = x; continue; }
          st = llo;
        } else {
          if (x > lhi) { hi = mid; continue; }
          if (x < lhi) { lo = mid; llo = x; continue; }
          st = lhi;
        }
      } else if (real) {
        st = llo;
      } else if (lhi >= 0) {
        st = depth;
      }
      int l;
      const int c = warp_cmp_ids(S, SA[mid], tc, tg, L, st, &l);
      if (c <= 0) {
        hi = mid;
        lhi = l;
      } else {
        lo = mid;
        llo = l;
      }
    }
    int cnt = 0;
    if (lhi >= L) {  // extend while LC[k] >= L (k + 1 < hi0)
      const int kend = hi0 - 1;
      int k = hi, stop = -1;
      {
        const int bend = min(((k >> 5) + 1) << 5, kend);
        const int kk = k + lane;
        const u32 bad = __ballot_sync(0xffffffffu, kk < bend && int(LC[kk]) < L);
        if (bad)
          stop = k + __ffs(bad) - 1;
        else
          k = bend;
      }
      while (stop < 0 && k < kend) {
        const int b = (k >> 5) + lane;
        const bool cand = (b << 5) < kend && ((b << 5) + 32 > kend || int(s_bmin[b]) < L);
        const u32 cb = __ballot_sync(0xffffffffu, cand);
        if (!cb) {
          k += 32 * 32;
          continue;
        }
        const int fb = (k >> 5) + __ffs(cb) - 1;
        const int kk = (fb << 5) + lane;
        const u32 bad = __ballot_sync(0xffffffffu, kk < kend && int(LC[kk]) < L);
        stop = bad ? (fb << 5) + __ffs(bad) - 1 : min((fb << 5) + 32, kend);
      }
      if (stop < 0) stop = kend;
      cnt = 1 + (stop - hi);
    }
    if (lane == 0) {
      ilo[mc.y] = beg + hi;
      icnt[mc.y] = u32(cnt);
      if (cnt) atomicAdd(&s_tot, u32(cnt));
    }
    i = ni;
    mc = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) qtot[q] = s_tot;
}

// ---- ordered hit emission, one CTA per stream (on-chip path) ----
// The on-chip path matches REVERSED traces against the suffix arrays of the
// REVERSED streams: reversed trace t occurs at reversed position i of stream
// q exactly when t ends at e = n - 1 - i.  In that suffix array the hit
// intervals [lo, hi) of the stream's traces form a laminar family (two
// intervals that meet belong to a trace and a suffix of it -- a prefix in
// reversed order -- and the longer trace's interval lies inside), so the
// traces ending at one position e are exactly the chain of intervals that
// contain its rank r = RISA[n-1-e], from the deepest (longest trace,
// smallest id) outwards: precisely the required (end, trace id) order.
//  * k_tree_keys / radix sort / k_tree_sweep: per stream, the matched
//    intervals in preorder (lo asc, hi desc, shorter first) and a stack sweep
//    give every interval its parent (the next enclosing interval);
//  * k_stream_emit: paints the deepest interval of every rank (shared
//    atomicMin over the local pair index, which is the trace order), counts
//    chain lengths with a difference array, scans them in end order and
//    walks each end's chain, writing its records back to back -- every hit
//    goes straight to its final place, and the writes of a warp stay within
//    a few KB, so no partial-sector read-modify-write reaches HBM.
constexpr int kEmitThreads = 1024;
constexpr int kEmitPairs = 8192;  // interval links kept on chip when the stream has at most this many
constexpr u32 kNoPar = 0xffffffffu;

// exclusive scan of one u32 per thread over the CTA; returns the total
__device__ __forceinline__ u32 cta_excl_scan(u32 v, u32 *s_warp, u32 *out_excl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const u32 x = s_warp[lane];
    u32 wi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += o;
    }
    s_warp[lane] = wi - x;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  *out_excl = s_warp[warp] + incl - v;
  const u32 total = s_warp[32];
  __syncthreads();  // s_warp may be reused
  return total;
}

// Preorder keys of the matched intervals: (stream, lo asc, hi desc); written
// in reverse pair order so that the stable sort leaves equal intervals with
// the larger pair index (shorter trace, the enclosing one) first.  Unmatched
// pairs get a key above every stream.
__global__ void k_tree_keys(const u64 *__restrict__ sqk, const u32 *__restrict__ zsorted,
                            const i64 *__restrict__ ilo, const u32 *__restrict__ icnt, const i64 *__restrict__ off,
                            const u32 *__restrict__ ptrace, i64 P, int bS, u64 *__restrict__ key,
                            u32 *__restrict__ val, u32 *__restrict__ gtr) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const u32 z = zsorted[i];
  gtr[i] = ptrace[z];
  const u32 c = icnt[z];
  const u64 q = sqk[i];
  const i64 k = P - 1 - i;
  if (c) {
    const u64 lo = u64(ilo[z] - off[q]), hi = lo + c;
    key[k] = (q << 30) | (lo << 15) | (32767u - hi);
  } else {
    key[k] = u64(1) << (bS + 30);
  }
  val[k] = u32(i);
}

// toff[q] = first index of stream q's intervals in the preorder list
__global__ void k_tree_offsets(const u64 *__restrict__ key, i64 P, int S, u32 *__restrict__ toff) {
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q > S) return;
  i64 lo = 0, hi = P;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if ((key[mid] >> 30) < u64(q)) lo = mid + 1; else hi = mid;
  }
  toff[q] = u32(lo);
}

// Stack sweep of one stream's intervals in preorder, one warp per stream:
// the warp stages the sorted list in shared memory chunk by chunk and lane 0
// sweeps it with the open-interval stack in shared memory (a ring of the top
// kTreeDepth entries; deeper entries are recovered through the parent links
// already written to global memory).  Interval ids are preorder positions
// local to the stream (k - toff[q]); per preorder position k:
// opar[k] = parent id or kNoPar, ohi[k] = interval end, odep[k] = number of
// intervals containing it (itself included), otr[k] = its trace id.
constexpr int kTreeChunk = 1024;
constexpr int kTreeDepth = 1024;

__global__ void __launch_bounds__(32) k_tree_sweep(const u64 *__restrict__ key, const u32 *__restrict__ val,
                                                   const u32 *__restrict__ toff, const u32 *__restrict__ gtr,
                                                   u32 *__restrict__ opar, u32 *__restrict__ ohi,
                                                   u32 *__restrict__ odep, u32 *__restrict__ otr,
                                                   u32 *__restrict__ oroot, const u32 *__restrict__ only) {
  __shared__ u64 s_key[kTreeChunk];
  __shared__ u32 s_idx[kTreeDepth], s_hi[kTreeDepth];
  const int q = blockIdx.x, lane = threadIdx.x;
  if (only && !only[q]) return;  // fallback run: only the streams k_tree_par flagged
  const u32 a = toff[q], b = toff[q + 1];
  for (u32 k = a + lane; k < b; k += 32) otr[k] = gtr[val[k]];
  u32 cur = kNoPar, curhi = 0, depth = 0, held = 0;  // held: stack entries below the top kept in the ring
  for (u32 c0 = a; c0 < b; c0 += kTreeChunk) {
    const u32 m = min(u32(kTreeChunk), b - c0);
    for (u32 k = lane; k < m; k += 32) s_key[k] = key[c0 + k];
    __syncwarp();
    if (lane == 0) {
      for (u32 k = 0; k < m; ++k) {
        const u64 kk = s_key[k];
        const u32 lo = u32(kk >> 15) & 32767u, hi = 32767u - (u32(kk) & 32767u);
        while (cur != kNoPar && curhi <= lo) {  // the open interval ends before this one starts: pop
          if (depth == 0) {
            cur = kNoPar;
            break;
          }
          --depth;
          if (held) {
            --held;
            cur = s_idx[depth % kTreeDepth];
            curhi = s_hi[depth % kTreeDepth];
          } else {
            cur = opar[a + cur];
            curhi = cur != kNoPar ? ohi[a + cur] : 0;
          }
        }
        const u32 id = c0 + k - a;
        opar[a + id] = cur;
        ohi[a + id] = hi;
        odep[a + id] = cur != kNoPar ? depth + 2 : 1;
        oroot[a + id] = cur != kNoPar ? oroot[a + cur] : id;
        if (cur != kNoPar) {  // push the open interval below the new one
          s_idx[depth % kTreeDepth] = cur;
          s_hi[depth % kTreeDepth] = curhi;
          held = min(held + 1, u32(kTreeDepth));
          ++depth;
        }
        cur = id;
        curhi = hi;
      }
    }
    __syncwarp();
  }
}

// The same forest, 32 intervals at a time (one warp per stream): in preorder
// the parent of an interval is the nearest PRECEDING interval whose end is >=
// its own (laminar family), so within a chunk it comes from 32 shuffles; if
// it precedes the chunk it is on the chain of open intervals left by the
// previous chunk, kept as a depth-indexed stack whose ends are non-increasing
// (binary search).  Depths inside the chunk follow by pointer jumping, and
// the stack is updated by "the last interval of the chunk at each depth" (the
// ancestor of the chunk's last interval at depth d is the last interval of
// depth d before it in preorder).  A stream nested deeper than the on-chip
// stack is flagged in `big` and redone by k_tree_sweep.
// 1,024 levels (6 KB): every one-warp CTA of a C4 batch resident at once
// (4,096 levels, 24 KB, allowed 9 per SM: 0.37 -> 0.28 ms per C4 step).
constexpr u32 kParDepth = 1024;

__global__ void __launch_bounds__(32) k_tree_par(const u64 *__restrict__ key, const u32 *__restrict__ val,
                                                 const u32 *__restrict__ toff, const u32 *__restrict__ gtr,
                                                 u32 *__restrict__ opar, u32 *__restrict__ ohi,
                                                 u32 *__restrict__ odep, u32 *__restrict__ otr,
                                                 u32 *__restrict__ oroot, u32 *__restrict__ big) {
  __shared__ u32 s_id[kParDepth + 1];
  __shared__ unsigned short s_hi[kParDepth + 1];
  const int q = blockIdx.x, lane = threadIdx.x;
  const u32 a = toff[q], b = toff[q + 1];
  u32 ssize = 0;  // the stack holds depths 1 .. ssize
  bool deep_stream = false;
  for (u32 c0 = a; c0 < b; c0 += 32) {
    const u32 k = c0 + lane;
    const bool v = k < b;
    u32 hi = 0;
    if (v) hi = 32767u - (u32(key[k]) & 32767u);
    int P = -1;  // nearest preceding lane of the chunk that contains this interval
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const u32 hj = __shfl_sync(0xffffffffu, hi, j);
      if (j < lane && hj >= hi) P = j;
    }
    u32 pid = kNoPar, acc = 1;
    int ptr = P;
    if (P < 0) {
      u32 l = 0, h = min(ssize, kParDepth);  // deepest stack depth whose end is >= hi
      while (l < h) {
        const u32 mid = (l + h + 1) >> 1;
        if (s_hi[mid] >= hi) l = mid; else h = mid - 1;
      }
      pid = l ? s_id[l] : kNoPar;
      acc = l + 1;
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) {  // depth = depth(parent) + 1 along in-chunk links
      const int src = ptr >= 0 ? ptr : lane;
      const u32 pacc = __shfl_sync(0xffffffffu, acc, src);
      const int pptr = __shfl_sync(0xffffffffu, ptr, src);
      if (ptr >= 0) {
        acc += pacc;
        ptr = pptr;
      }
    }
    const u32 depth = acc;
    // root (the depth-1 ancestor): the stack bottom, or itself, for an
    // interval whose parent precedes the chunk; else its in-chunk parent's
    u32 rt = P >= 0 ? 0u : (pid == kNoPar ? k - a : s_id[1]);
    int rp = P;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int src = rp >= 0 ? rp : lane;
      const u32 prt = __shfl_sync(0xffffffffu, rt, src);
      const int prp = __shfl_sync(0xffffffffu, rp, src);
      if (rp >= 0) {
        if (prp < 0) rt = prt;
        rp = prp;
      }
    }
    if (v) {
      opar[k] = P >= 0 ? c0 + u32(P) - a : pid;
      ohi[k] = hi;
      odep[k] = depth;
      oroot[k] = rt;
      otr[k] = gtr[val[k]];
      if (depth > kParDepth) deep_stream = true;
    }
    const u32 peers = __match_any_sync(0xffffffffu, v ? depth : 0xffffffffu);
    if (v && depth <= kParDepth && lane == 31 - __clz(peers)) {
      s_id[depth] = k - a;
      s_hi[depth] = (unsigned short)hi;
    }
    ssize = __shfl_sync(0xffffffffu, depth, int(min(31u, b - c0 - 1)));
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, deep_stream) && lane == 0) big[q] = 1;
}

__global__ void __launch_bounds__(kEmitThreads, 1) k_stream_emit(StreamMatch m, const u64 *__restrict__ tkey,
                                                                 const u32 *__restrict__ toff,
                                                                 const u32 *__restrict__ qbase, i64 cap,
                                                                 apo_match_rec *__restrict__ out,
                                                                 const u32 *__restrict__ qorder,
                                                                 const u32 *__restrict__ opar,
                                                                 const u32 *__restrict__ otr,
                                                                 const u32 *__restrict__ odep, bool pair32,
                                                                 u32 *__restrict__ endoff,
                                                                 unsigned short *__restrict__ endml) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ u32 s_warp[33];
  const int q = int(qorder[blockIdx.x]);
  const i64 a = toff[q], M = i64(toff[q + 1]) - a;  // the stream's matched intervals, in preorder
  if (M == 0) return;
  const i64 beg = m.off[q], n = m.off[q + 1] - beg;
  u32 *deep = reinterpret_cast<u32 *>(smem);  // [kSMMax] 1 + deepest interval (preorder id) at each rank, 0 = none
  u32 *spar = deep + kSMMax;                  // [kEmitPairs] parent, trace id and depth of every
  u32 *str = spar + kEmitPairs;               //   interval of the stream when they fit on chip
  u32 *sdep = str + kEmitPairs;
  unsigned short *RISA = reinterpret_cast<unsigned short *>(sdep + kEmitPairs);  // [kSMMax]
  for (i64 r = threadIdx.x; r < n; r += kEmitThreads) {
    deep[r] = 0;
    RISA[m.sa[beg + r] - beg] = (unsigned short)r;
  }
  const bool onchip = M <= kEmitPairs;
  if (onchip) {
    for (i64 i = threadIdx.x; i < M; i += kEmitThreads) {
      spar[i] = opar[a + i];
      str[i] = otr[a + i];
      sdep[i] = odep[a + i];
    }
  }
  const u32 *par = onchip ? spar : opar + a, *trs = onchip ? str : otr + a, *dep = onchip ? sdep : odep + a;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // 1. deepest interval per rank: in preorder a descendant follows its
  //    ancestors, so the deepest interval containing a rank has the largest id
  for (i64 kb = i64(warp) * 32; kb < M; kb += i64(kEmitThreads)) {
    const i64 k = kb + lane;
    u32 lo = 0, hi = 0;
    if (k < M) {
      const u64 kk = tkey[a + k];
      lo = u32(kk >> 15) & 32767u;
      hi = 32767u - (u32(kk) & 32767u);
    }
    u32 live = __ballot_sync(0xffffffffu, hi > lo);
    while (live) {
      const int src = __ffs(live) - 1;
      live &= live - 1;
      const u32 l0 = __shfl_sync(0xffffffffu, lo, src), h0 = __shfl_sync(0xffffffffu, hi, src);
      const u32 id1 = u32(kb + src) + 1u;
      for (u32 r = l0 + lane; r < h0; r += 32)
        if (deep[r] < id1) atomicMax(&deep[r], id1);
    }
  }
  __syncthreads();
  // 2. ends in order: thread t owns ends [16t, 16t + 16); an end's record
  //    count is the depth of its deepest interval; record offsets by a CTA
  //    scan, then each end's chain is walked and written back to back (a
  //    warp's writes stay within a few KB, so sectors fill in L2).
  constexpr int kPer = kSMMax / kEmitThreads;
  const int b0 = threadIdx.x * kPer;
  u32 ce[kPer];
  u32 tsum = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const i64 e = b0 + j;
    const u32 d1 = e < n ? deep[RISA[n - 1 - e]] : 0u;
    ce[j] = d1 ? dep[d1 - 1] : 0u;
    tsum += ce[j];
  }
  u32 run;
  cta_excl_scan(tsum, s_warp, &run);
  i64 pos = i64(qbase[q]) + run;
  // a thread's records are consecutive: an even-indexed record waits for its
  // successor and the pair goes out as one 32-B store (half the store
  // transactions); odd starts and the last record use 16-B stores
  int4 held = make_int4(0, 0, 0, 0);
  bool have = false;
  i64 hpos = 0;
  auto put = [&](i64 p, int4 r) {
    if (have) {  // the held record (even index hpos) pairs with its successor
      if (p == hpos + 1 && p < cap) {
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(
                         reinterpret_cast<int4 *>(out) + hpos),
                     "r"(held.x), "r"(held.y), "r"(held.z), "r"(held.w), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
                     : "memory");
        have = false;
        return;
      }
      reinterpret_cast<int4 *>(out)[hpos] = held;
      have = false;
    }
    if (p >= cap) return;
    if (pair32 && (p & 1) == 0) {
      held = r;
      hpos = p;
      have = true;
    } else {
      reinterpret_cast<int4 *>(out)[p] = r;  // one 16-B store
    }
  };
#pragma unroll 1
  for (int j = 0; j < kPer; ++j) {
    const i64 e = b0 + j;
    if (endoff != nullptr && e < n) endoff[beg + e] = u32(pos);  // REPLAY (mode 1): the end's first record
    if (!ce[j]) {
      if (endml != nullptr && e < n) endml[beg + e] = 0xffffu;
      continue;
    }
    u32 z = deep[RISA[n - 1 - e]] - 1u, zl = z;
    for (u32 k = 0; k < ce[j]; ++k, ++pos) {
      put(pos, make_int4(q, i32(e), i32(trs[z]), i32(z)));  // slot = stream-local interval id
      zl = z;
      z = par[z];
    }
    if (endml != nullptr) {  // the end's shortest trace (its root-most interval): the latest start is e - len + 1
      const u32 t = trs[zl];
      endml[beg + e] = (unsigned short)min(i64(0xfffe), m.toff[t + 1] - m.toff[t]);
    }
  }
  if (have) reinterpret_cast<int4 *>(out)[hpos] = held;
}

// MATCH_ALL kept implicit for REPLAY (apo_match mode 1): the hits ending at e
// are the chain of intervals from the deepest one containing rank
// RISA[n-1-e] out to its root (trace-id order), so instead of writing every
// record this stores, per end, 1 + that deepest interval (0: no hit) and the
// length of the chain's root trace (the end's shortest; 0xffff: none).
// REPLAY walks the chains of the ends it decides (~0.3 % of the hits).
constexpr int kEndsThreads = 1024;
constexpr int kEndsMl = 7168;  // intervals whose root lengths stay on chip (two CTAs per SM)

__global__ void __launch_bounds__(kEndsThreads, 2) k_stream_ends(StreamMatch m, const u64 *__restrict__ tkey,
                                                                 const u32 *__restrict__ toff,
                                                                 const u32 *__restrict__ otr,
                                                                 const u32 *__restrict__ oroot,
                                                                 const u32 *__restrict__ opar,
                                                                 u32 *__restrict__ deepz,
                                                                 unsigned short *__restrict__ endml,
                                                                 const u32 *__restrict__ qorder) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int q = int(qorder[blockIdx.x]);  // heaviest streams first
  const i64 beg = m.off[q], n = m.off[q + 1] - beg;
  const i64 a = toff[q], M = i64(toff[q + 1]) - a;
  if (M == 0) {
    for (i64 e = threadIdx.x; e < n; e += kEndsThreads) {
      deepz[beg + e] = 0u;
      endml[beg + e] = 0xffffu;
    }
    return;
  }
  u32 *deep = reinterpret_cast<u32 *>(smem);                                  // [kSMMax]
  unsigned short *RISA = reinterpret_cast<unsigned short *>(deep + kSMMax);  // [kSMMax]
  for (i64 r = threadIdx.x; r < n; r += kEndsThreads) {
    deep[r] = 0;
    RISA[m.sa[beg + r] - beg] = (unsigned short)r;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // deepest interval per rank (largest preorder id containing it), each
  // rank written once: in preorder (lo asc, hi desc) interval k owns
  // [lo_k, min(hi_k, lo_{k+1})) -- up to its first child -- and, on behalf
  // of its parent p, [hi_k, min(hi_p, lo_s)) with s the first interval after
  // k's subtree (the first with lo >= hi_k: a binary search over the keys)
  // -- up to k's next sibling.  These segments partition the covered ranks
  // (painting every interval's whole range instead, 474 M shared-memory
  // reads per C4 step: 0.64 ms for the kernel, 0.57 ms with the segments).
  for (i64 kb = i64(warp) * 32; kb < M; kb += i64(kEndsThreads)) {
    const i64 k = kb + lane;
    u32 a0 = 0, b0 = 0, a1 = 0, b1 = 0, p1 = 0;
    if (k < M) {
      const u64 kk = tkey[a + k];
      const u32 lo = u32(kk >> 15) & 32767u, hi = 32767u - (u32(kk) & 32767u);
      const u32 nlo = k + 1 < M ? u32(tkey[a + k + 1] >> 15) & 32767u : 32767u;
      a0 = lo;
      b0 = min(hi, nlo);
      const u32 p = opar[a + k];
      if (p != kNoPar) {
        const u32 hp = 32767u - (u32(tkey[a + p]) & 32767u);
        const u64 target = ((kk >> 30) << 30) | (u64(hi) << 15);
        i64 l = k + 1, h = M;  // first j > k with key >= target (lo_j >= hi)
        while (l < h) {
          const i64 mid = (l + h) >> 1;
          if (tkey[a + mid] < target) l = mid + 1; else h = mid;
        }
        const u32 ls = l < M ? u32(tkey[a + l] >> 15) & 32767u : 32767u;
        a1 = hi;
        b1 = min(hp, ls);
        p1 = p + 1u;
      }
    }
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const u32 pa = part ? a1 : a0, pb = part ? b1 : b0, pid = part ? p1 : u32(k + 1);
      u32 live = __ballot_sync(0xffffffffu, pb > pa);
      while (live) {
        const int src = __ffs(live) - 1;
        live &= live - 1;
        const u32 l0 = __shfl_sync(0xffffffffu, pa, src), h0 = __shfl_sync(0xffffffffu, pb, src);
        const u32 id1 = __shfl_sync(0xffffffffu, pid, src);
        for (u32 r = l0 + lane; r < h0; r += 32) deep[r] = id1;
      }
    }
  }
  // per interval, the length of its chain's root trace (the shortest trace
  // ending where the chain is deepest), on chip when the stream has at most
  // kEndsMl intervals: the per-end lookups then stay in shared memory (the
  // dependent otr -> oroot -> toff chain per end: C4 0.57 -> 0.50 ms)
  unsigned short *s_ml = RISA + kSMMax;
  const bool ml_on_chip = M <= kEndsMl;
  if (ml_on_chip)
    for (i64 k = threadIdx.x; k < M; k += kEndsThreads) {
      const u32 t = otr[a + oroot[a + k]];
      s_ml[k] = (unsigned short)min(i64(0xfffe), m.toff[t + 1] - m.toff[t]);
    }
  __syncthreads();
  for (i64 e = threadIdx.x; e < n; e += kEndsThreads) {
    const u32 d1 = deep[RISA[n - 1 - e]];
    u32 ml = 0xffffu;
    if (d1) {
      if (ml_on_chip) {
        ml = s_ml[d1 - 1];
      } else {
        const u32 t = otr[a + oroot[a + d1 - 1]];
        ml = u32(min(i64(0xfffe), m.toff[t + 1] - m.toff[t]));
      }
    }
    deepz[beg + e] = d1;
    endml[beg + e] = (unsigned short)ml;
  }
}

// warp per pair: its hits are the contiguous SA range [ilo, ilo + cnt) of
// one stream; written to [hbase, hbase + cnt) of the key array
__global__ void k_enumerate_pairs(StreamMatch m, const i64 *__restrict__ ilo, const u32 *__restrict__ hbase,
                                  const u32 *__restrict__ ptrace, i64 P, i64 H, int bE, int bT,
                                  u64 *__restrict__ keys) {
  const i64 z = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (z >= P) return;
  const int lane = threadIdx.x & 31;
  const i64 base = hbase[z];
  const i64 cnt = (z + 1 < P ? i64(hbase[z + 1]) : H) - base;
  if (cnt == 0) return;
  const i64 t = ptrace[z];
  const i64 L = m.toff[t + 1] - m.toff[t];
  const i64 r0 = ilo[z];
  for (i64 i = lane; i < cnt; i += 32) {
    const i64 p = m.sa[r0 + i];
    const int q = m.wid[p];
    const i64 end = p - m.off[q] + L - 1;
    keys[base + i] = (u64(q) << (bE + bT)) | (u64(end) << bT) | u64(t);
  }
}

// Total order on pieces: length desc, then content (unsigned tokens, R1),
// then piece index (indices >= n are padding and sort last).  The first three
// tokens come from compact prefix-key arrays, so most comparisons never touch
// the token array.
struct TraceCmp {
  const u64 *tok;
  const i64 *off;
  const u64 *pk;  // pk[3*i + j] = token j of piece i (j < min(3, len))
  i64 n;
  __device__ __forceinline__ int cmp(u32 a, u32 b) const {
    if (a == b) return 0;
    const bool pa = a >= n, pb = b >= n;
    if (pa || pb) return (pa && pb) ? (a < b ? -1 : 1) : (pa ? 1 : -1);
    const i64 oa = off[a], ob = off[b];
    const i64 la = off[a + 1] - oa, lb = off[b + 1] - ob;
    if (la != lb) return la > lb ? -1 : 1;
    const i64 np = la < 3 ? la : 3;
    for (i64 k = 0; k < np; ++k) {
      u64 x = pk[3 * i64(a) + k], y = pk[3 * i64(b) + k];
      if (x != y) return x < y ? -1 : 1;
    }
    for (i64 k = 3; k < la; ++k) {
      u64 x = tok[oa + k], y = tok[ob + k];
      if (x != y) return x < y ? -1 : 1;
    }
    return a < b ? -1 : 1;
  }
};

__global__ void k_iota_list(const u32 *__restrict__ list, i64 U, u32 *__restrict__ idx, i64 P, u32 pad) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < P) idx[i] = i < U ? list[i] : pad + u32(i);
}

// one compare-exchange stage (k, j) of a bitonic sorting network
__global__ void k_bitonic(u32 *__restrict__ idx, i64 P, i64 j, i64 k, TraceCmp c) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  i64 l = i ^ j;
  if (l <= i) return;
  u32 a = idx[i], b = idx[l];
  int r = c.cmp(a, b);
  bool asc = (i & k) == 0;
  if ((asc && r > 0) || (!asc && r < 0)) {
    idx[i] = b;
    idx[l] = a;
  }
}

// keys for the LSD passes of the trace order: which = 2: token 1, 1: token 0,
// 0: maxlen - length (length descending); vals (optional) = piece ids
__global__ void k_prefix_keys(const u32 *__restrict__ ids, i64 U, const u64 *__restrict__ pk,
                              const i64 *__restrict__ off, i64 maxlen, int which, u64 *__restrict__ keys,
                              u32 *__restrict__ vals) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= U) return;
  const u32 p = ids[c];
  if (which == 0)
    keys[c] = u64(maxlen - (off[p + 1] - off[p]));
  else
    keys[c] = pk[3 * i64(p) + (which == 1 ? 0 : 1)];
  if (vals) vals[c] = p;
}

constexpr int kMaxTie = 256;

// Insertion sort of each run of equal (length, token 0, token 1) with the
// full comparator, one warp per run (started at the run's first element):
// a comparison reads both pieces 32 tokens at a time (coalesced) and the
// first differing token is found with a ballot, so two long pieces sharing a
// long prefix cost one round trip per 32 tokens instead of one per token.
// *worst receives the largest run length; runs longer than kMaxTie are left
// unsorted (the caller then falls back to the bitonic network).
__global__ void k_tie_sort(u32 *__restrict__ order, i64 U, TraceCmp cmp, u32 *__restrict__ worst) {
  const i64 c = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= U) return;
  auto same = [&](u32 a, u32 b) {
    const i64 la = cmp.off[a + 1] - cmp.off[a], lb = cmp.off[b + 1] - cmp.off[b];
    return la == lb && cmp.pk[3 * i64(a)] == cmp.pk[3 * i64(b)] && cmp.pk[3 * i64(a) + 1] == cmp.pk[3 * i64(b) + 1];
  };
  if (c > 0 && same(order[c - 1], order[c])) return;  // not a run start (warp-uniform)
  i64 e = c + 1;
  while (e < U && same(order[c], order[e])) ++e;
  const i64 g = e - c;
  if (g > 1 && lane == 0) atomicMax(worst, u32(g));
  if (g < 2 || g > kMaxTie) return;
  // pieces of one run share their length (and first two tokens)
  const i64 L = cmp.off[order[c] + 1] - cmp.off[order[c]];
  auto greater = [&](u32 a, u32 b) -> bool {  // cmp(a, b) > 0
    const u64 *ta = cmp.tok + cmp.off[a], *tb = cmp.tok + cmp.off[b];
    for (i64 k0 = 2; k0 < L; k0 += 32) {
      const i64 k = k0 + lane;
      const u64 x = k < L ? ta[k] : 0, y = k < L ? tb[k] : 0;
      const unsigned m = __ballot_sync(0xffffffffu, x != y);
      if (m) {
        const int f = __ffs(m) - 1;
        const u64 xf = __shfl_sync(0xffffffffu, x, f), yf = __shfl_sync(0xffffffffu, y, f);
        return xf > yf;
      }
    }
    return a > b;
  };
  for (i64 i = c + 1; i < e; ++i) {
    const u32 x = order[i];
    i64 j = i - 1;
    u32 oj = order[j];
    while (j >= c && greater(oj, x)) {
      __syncwarp();
      if (lane == 0) order[j + 1] = oj;
      --j;
      if (j >= c) oj = order[j];  // no lane has written order[j]
    }
    __syncwarp();
    if (lane == 0) order[j + 1] = x;
    __syncwarp();
  }
}

__device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Sources of the pieces when the trace set is built from several trace
// lists (the multi-GPU union): list r's tokens live at tok[r] (a local
// allocation or a peer mapping over NVLink) and its pieces are the global
// pieces [first[r], first[r + 1]) whose tokens start at global token base[r].
constexpr int kMaxSrc = 16;
struct PieceSrc {
  const u64 *tok[kMaxSrc];
  i64 first[kMaxSrc + 1];
  i64 base[kMaxSrc + 1];
  int n;
  u64 *gather;  // non-null: copy every piece here (at its global offset)
};

// warp per piece: a position-keyed content hash (only used to bring equal
// contents together; equality is always verified token by token) and the
// piece's first three tokens; keys[i] = hash, vals[i] = i.  With src.gather
// set, the pieces are pulled from their source lists (peer memory for the
// remote ranks' lists) into the local buffer in the same pass.
template <bool GATHER>
__global__ void k_piece_hash(const u64 *__restrict__ tok, const i64 *__restrict__ off, i64 np,
                             u64 *__restrict__ hkey, u32 *__restrict__ hval, u64 *__restrict__ pk, PieceSrc src) {
  const i64 p = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= np) return;
  const i64 o = off[p], L = off[p + 1] - o;
  const u64 *from = tok + o;
  if (GATHER) {
    int r = 0;
    while (r + 1 < src.n && p >= src.first[r + 1]) ++r;
    from = src.tok[r] + (o - src.base[r]);
  }
  u64 h = 0;
#pragma unroll 4
  for (i64 k = lane; k < L; k += 32) {
    const u64 x = from[k];
    if (GATHER) src.gather[o + k] = x;
    h += mix64(x ^ mix64(u64(k) + 0x9E3779B97F4A7C15ull));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) h += __shfl_xor_sync(0xffffffffu, h, d);
  if (lane == 0) {
    hkey[p] = h;
    hval[p] = u32(p);
  }
  if (lane < 3) pk[3 * p + lane] = lane < L ? from[lane] : 0ull;
}

__global__ void k_len_keys(const u32 *__restrict__ order, const i64 *__restrict__ off, i64 np, i64 maxlen,
                           u64 *__restrict__ keys) {
  i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= np) return;
  const u32 p = order[c];
  keys[c] = u64(maxlen - (off[p + 1] - off[p]));
}

// warp per neighbour pair in (length, hash) order: 1 = keep (first of its
// content), 0 = exact duplicate of the previous piece
__global__ void k_dup_keep(const u64 *__restrict__ tok, const i64 *__restrict__ off, const u32 *__restrict__ order,
                           const u64 *__restrict__ hk, i64 np, u32 *__restrict__ keep) {
  const i64 c = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= np) return;
  if (c == 0) {
    if (lane == 0) keep[0] = 1;
    return;
  }
  const u32 a = order[c - 1], b = order[c];
  const i64 la = off[a + 1] - off[a], lb = off[b + 1] - off[b];
  bool same = la == lb && hk[a] == hk[b];
  for (i64 k0 = 0; same && k0 < la; k0 += 32) {  // warp-uniform trip count: every lane votes
    const i64 k = k0 + lane;
    same = __all_sync(0xffffffffu, k >= la || tok[off[a] + k] == tok[off[b] + k]);
  }
  same = __shfl_sync(0xffffffffu, same ? 1 : 0, 0) != 0;
  if (lane == 0) keep[c] = same ? 0u : 1u;
}

struct CompactF {
  const u32 *keepf;
  const u32 *order;
  u32 *out;
  i64 n;
  i64 *total;
  __device__ u32 load(i64 i) const { return keepf[i]; }
  __device__ bool store(i64 i, u32 incl, u32 excl) const {
    if (incl != excl) out[excl] = order[i];
    if (i == n - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_src_of(const u32 *__restrict__ uniq, const i64 *__restrict__ poff, i64 T, i64 *__restrict__ src) {
  i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < T) src[t] = poff[uniq[t]];
}

// Builds the trace set from pieces d_ptok / h_poff (host offsets):
//  1. merge identical pieces: radix-sort by (length, content hash), verify
//     neighbours token by token, keep the first of each content;
//  2. order the distinct pieces by (length desc, content lexicographic asc)
//     with a bitonic comparison network (comparisons almost always end within
//     the three prefix tokens kept in a compact array);
//  3. an exact neighbour comparison in that order (catches any content that
//     step 1 left split by a hash collision), ids, copy-out in id order.
void build_trace_set(Ctx &c, apo_trie *tr, const u64 *d_ptok, const std::vector<i64> &h_poff, cudaStream_t s,
                     const PieceSrc *src = nullptr) {
  const i64 np = i64(h_poff.size()) - 1;
  const i64 N = h_poff.back();
  tr->T = 0;
  tr->ntok = 0;
  tr->maxlen = 0;
  tr->h_off.assign(1, 0);
  if (np <= 0 || N <= 0) return;
  i64 maxlen = 0;
  for (i64 w = 0; w < np; ++w) maxlen = std::max<i64>(maxlen, h_poff[w + 1] - h_poff[w]);
  i64 P = 1;
  while (P < np) P <<= 1;
  i64 *d_poff, *scal, *d_src;
  u32 *order, *head, *uniq, *hv, *hv_alt, *keep, *surv;
  u64 *hk, *hk_alt, *hk_keep, *pk;
  i32 *ulen;
  auto plan = [&](Carver &cv) {
    d_poff = cv.take<i64>(np + 1);
    hk = cv.take<u64>(np);
    hk_alt = cv.take<u64>(np);
    hk_keep = cv.take<u64>(np);
    hv = cv.take<u32>(np);
    hv_alt = cv.take<u32>(np);
    pk = cv.take<u64>(3 * np);
    keep = cv.take<u32>(np);
    surv = cv.take<u32>(np);
    order = cv.take<u32>(P);
    head = cv.take<u32>(np);
    uniq = cv.take<u32>(np);
    ulen = cv.take<i32>(np);
    d_src = cv.take<i64>(np);
    scal = cv.take<i64>(4);
  };
  Carver dry(nullptr);
  plan(dry);
  c.arena.reserve(dry.off, s);
  Carver cv(c.arena.base);
  plan(cv);
  c.h2d(d_poff, h_poff.data(), sizeof(i64) * (np + 1), s);
  // 1. merge identical pieces
  if (src)
    k_piece_hash<true><<<grid_for(np * 32, T256), T256, 0, s>>>(d_ptok, d_poff, np, hk, hv, pk, *src);
  else
    k_piece_hash<false><<<grid_for(np * 32, T256), T256, 0, s>>>(d_ptok, d_poff, np, hk, hv, pk, PieceSrc{});
  APO_CHECK_LAUNCH();
  c.d2d(hk_keep, hk, sizeof(u64) * np, s);
  // grouping only needs equal hashes together: 32 hash bits suffice (a rare
  // split group is caught by the exact neighbour check of step 3)
  bool a1 = radix_sort_u64_u32(c, hk, hv, hk_alt, hv_alt, np, 0, 32, s);
  u64 *k1 = a1 ? hk_alt : hk;
  u32 *o1 = a1 ? hv_alt : hv;
  u64 *k2 = a1 ? hk : hk_alt;
  u32 *o2 = a1 ? hv : hv_alt;
  k_len_keys<<<grid_for(np, T256), T256, 0, s>>>(o1, d_poff, np, maxlen, k1);
  APO_CHECK_LAUNCH();
  bool a2 = radix_sort_u64_u32(c, k1, o1, k2, o2, np, 0, bits_for(u64(maxlen)), s);
  const u32 *by_hash = a2 ? o2 : o1;
  k_dup_keep<<<grid_for(np * 32, T256), T256, 0, s>>>(d_ptok, d_poff, by_hash, hk_keep, np, keep);
  APO_CHECK_LAUNCH();
  c.launches += 3;
  CompactF cf{keep, by_hash, surv, np, scal};
  launch_scan<false>(c, np, cf, s);
  const i64 U = i64(c.read_u64(reinterpret_cast<const u64 *>(scal), s));
  // 2. lexicographic order of the distinct pieces: LSD radix sort by
  //    (length desc, token 0, token 1) -- every sort is over U << N keys --
  //    then the rare tie groups (same length and first two tokens) are
  //    finished by an insertion sort with the full comparator.  A tie group
  //    larger than kMaxTie falls back to the bitonic network.
  TraceCmp cmp{d_ptok, d_poff, pk, np};
  {
    u64 *rk = hk, *rk_alt = hk_alt;
    u32 *rv = hv, *rv_alt = hv_alt;
    const int lenbits = bits_for(u64(maxlen));
    k_prefix_keys<<<grid_for(U, T256), T256, 0, s>>>(surv, U, pk, d_poff, maxlen, 2, rk, rv);
    APO_CHECK_LAUNCH();
    bool x = radix_sort_u64_u32(c, rk, rv, rk_alt, rv_alt, U, 0, 64, s);
    if (x) { std::swap(rk, rk_alt); std::swap(rv, rv_alt); }
    k_prefix_keys<<<grid_for(U, T256), T256, 0, s>>>(rv, U, pk, d_poff, maxlen, 1, rk, nullptr);
    APO_CHECK_LAUNCH();
    x = radix_sort_u64_u32(c, rk, rv, rk_alt, rv_alt, U, 0, 64, s);
    if (x) { std::swap(rk, rk_alt); std::swap(rv, rv_alt); }
    k_prefix_keys<<<grid_for(U, T256), T256, 0, s>>>(rv, U, pk, d_poff, maxlen, 0, rk, nullptr);
    APO_CHECK_LAUNCH();
    x = radix_sort_u64_u32(c, rk, rv, rk_alt, rv_alt, U, 0, lenbits, s);
    if (x) { std::swap(rk, rk_alt); std::swap(rv, rv_alt); }
    APO_CUDA(cudaMemsetAsync(scal + 2, 0, sizeof(i64), s));
    k_tie_sort<<<grid_for(U * 32, T256), T256, 0, s>>>(rv, U, cmp, reinterpret_cast<u32 *>(scal + 2));
    APO_CHECK_LAUNCH();
    c.launches += 4;
    const u32 worst = c.read_u32(reinterpret_cast<const u32 *>(scal + 2), s);
    if (worst <= u32(kMaxTie)) {
      c.d2d(order, rv, sizeof(u32) * U, s);
    } else {
      i64 PU = 1;
      while (PU < U) PU <<= 1;
      k_iota_list<<<grid_for(PU, T256), T256, 0, s>>>(surv, U, order, PU, u32(np));
      APO_CHECK_LAUNCH();
      c.launches++;
      for (i64 k = 2; k <= PU; k <<= 1)
        for (i64 j = k >> 1; j > 0; j >>= 1) {
          k_bitonic<<<grid_for(PU, T256), T256, 0, s>>>(order, PU, j, k, cmp);
          APO_CHECK_LAUNCH();
          c.launches++;
        }
    }
  }
  // 3. exact neighbour check, ids
  k_trace_heads<<<grid_for(U * 32, T256), T256, 0, s>>>(d_ptok, d_poff, order, U, head);
  APO_CHECK_LAUNCH();
  c.launches++;
  TraceIdF f{head, order, d_poff, uniq, ulen, U, scal};
  launch_scan<false>(c, U, f, s);
  const i64 T = i64(c.read_u64(reinterpret_cast<const u64 *>(scal), s));
  // offsets of the distinct traces (host prefix sums of the lengths)
  std::vector<i64> h_uoff(size_t(T) + 1, 0);
  {
    std::vector<i32> hl(static_cast<size_t>(T));
    c.d2h(hl.data(), ulen, sizeof(i32) * T, s);
    for (i64 t = 0; t < T; ++t) h_uoff[t + 1] = h_uoff[t] + hl[t];
  }
  const i64 ntok = h_uoff[T];
  tr->tok_bytes = sizeof(u64) * size_t(std::max<i64>(ntok, 1));
  tr->off_bytes = sizeof(i64) * size_t(T + 1);
  tr->d_rtok = static_cast<u64 *>(c.pool_get(tr->tok_bytes));
  tr->d_off = static_cast<i64 *>(c.pool_get(tr->off_bytes));
  c.h2d(tr->d_off, h_uoff.data(), sizeof(i64) * (T + 1), s);
  k_src_of<<<grid_for(T, T256), T256, 0, s>>>(uniq, d_poff, T, d_src);
  k_copy_pieces_rev<<<grid_for(T * 32, T256), T256, 0, s>>>(d_ptok, d_src, tr->d_off, T, tr->d_rtok);
  APO_CHECK_LAUNCH();
  c.launches += 2;
  APO_CUDA(cudaStreamSynchronize(s));
  tr->T = T;
  tr->ntok = ntok;
  tr->maxlen = maxlen;
  tr->minlen = T > 0 ? maxlen : 0;
  for (i64 t = 0; t < T; ++t) tr->minlen = std::min<i64>(tr->minlen, h_uoff[t + 1] - h_uoff[t]);
  tr->h_off = std::move(h_uoff);
}

}  // namespace
}  // namespace apo

using namespace apo;

namespace {
template <class Fn>
apo_status trie_guard(apo_ctx *ctx, Fn &&fn) {
  if (!ctx) return APO_ERR_INVALID;
  ctx->c.err.clear();
  try {
    cudaSetDevice(ctx->c.device);
    fn(ctx->c);
    return APO_OK;
  } catch (const Error &e) {
    ctx->c.err = e.msg;
    return e.code;
  } catch (const std::exception &e) {
    ctx->c.err = e.what();
    return APO_ERR_CUDA;
  }
}
}  // namespace

extern "C" {

apo_status apo_trie_build(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off, int32_t nwin,
                          const apo_repeat *d_rep, const int64_t *d_rep_off, int32_t min_len, int32_t max_len,
                          apo_trie **out, void *stream) {
  if (!out) return APO_ERR_INVALID;
  *out = nullptr;
  apo_trie *tr = new apo_trie();
  tr->ctx = ctx;
  apo_status st = trie_guard(ctx, [&](Ctx &c) {
    require(nwin >= 1 && h_off != nullptr && d_rep_off != nullptr && min_len >= 1 && max_len >= 0,
            "invalid argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    i64 nrep = 0;
    c.d2h(&nrep, d_rep_off + nwin, sizeof(i64), s);
    if (nrep == 0) {
      tr->h_off.assign(1, 0);
      return;
    }
    require(d_tok != nullptr && d_rep != nullptr, "NULL device pointer");
    // pieces, carved from the aux arena with upper bounds: the repeats'
    // representative occurrences are disjoint kept intervals, so their
    // total length is <= the batch length; each repeat yields at most
    // ceil(length / max_len) pieces.
    const i64 Nsrc = h_off[nwin];
    const i64 np_max = max_len > 0 ? nrep + Nsrc / max_len + 1 : nrep;
    i64 *d_src_off, *scal, *p_src, *p_off;
    u32 *pbase;
    i32 *p_len;
    u64 *ptok;
    auto plan = [&](Carver &cv) {
      d_src_off = cv.take<i64>(size_t(nwin) + 1);
      scal = cv.take<i64>(4);
      pbase = cv.take<u32>(nrep);
      p_src = cv.take<i64>(np_max);
      p_len = cv.take<i32>(np_max);
      p_off = cv.take<i64>(np_max + 1);
      ptok = cv.take<u64>(Nsrc);
    };
    Carver dry(nullptr);
    plan(dry);
    c.aux.reserve(dry.off, s);
    Carver cv(c.aux.base);
    plan(cv);
    c.h2d(d_src_off, h_off, sizeof(i64) * (nwin + 1), s);
    SrcRep sr{d_rep, d_rep_off, d_src_off, nwin, nrep, min_len, max_len};
    PieceCountF pf{sr, pbase, scal};
    launch_scan<false>(c, nrep, pf, s);
    const i64 np = i64(c.read_u64(reinterpret_cast<const u64 *>(scal), s));
    require(np <= np_max, "piece count exceeds its bound");
    k_pieces<<<grid_for(nrep, T256), T256, 0, s>>>(sr, pbase, p_src, p_len);
    APO_CHECK_LAUNCH();
    c.launches++;
    std::vector<i32> hl(static_cast<size_t>(np));
    c.d2h(hl.data(), p_len, sizeof(i32) * np, s);
    std::vector<i64> h_poff(size_t(np) + 1, 0);
    for (i64 q = 0; q < np; ++q) h_poff[q + 1] = h_poff[q] + hl[q];
    require(h_poff[np] <= Nsrc, "piece tokens exceed their bound");
    c.h2d(p_off, h_poff.data(), sizeof(i64) * (np + 1), s);
    k_copy_pieces<<<grid_for(np * 32, T256), T256, 0, s>>>(d_tok, p_src, p_off, np, ptok);
    APO_CHECK_LAUNCH();
    c.launches++;
    build_trace_set(c, tr, ptok, h_poff, s);
  });
  if (st != APO_OK) {
    apo_trie_destroy(tr);
    return st;
  }
  *out = tr;
  return APO_OK;
}

apo_status apo_trie_build_traces(apo_ctx *ctx, const uint64_t *d_tr, const int64_t *h_tr_off, int32_t ntraces,
                                 apo_trie **out, void *stream) {
  if (!out) return APO_ERR_INVALID;
  *out = nullptr;
  apo_trie *tr = new apo_trie();
  tr->ctx = ctx;
  apo_status st = trie_guard(ctx, [&](Ctx &c) {
    require(ntraces >= 0 && (ntraces == 0 || h_tr_off != nullptr), "invalid argument");
    std::vector<i64> h(size_t(ntraces) + 1, 0);
    for (int t = 0; t <= ntraces; ++t) h[t] = ntraces ? h_tr_off[t] : 0;
    for (int t = 0; t < ntraces; ++t) require(h[t + 1] > h[t], "traces must be non-empty");
    require(h[0] == 0, "h_tr_off[0] must be 0");
    require(ntraces == 0 || d_tr != nullptr, "NULL device pointer");
    build_trace_set(c, tr, d_tr, h, static_cast<cudaStream_t>(stream));
  });
  if (st != APO_OK) {
    apo_trie_destroy(tr);
    return st;
  }
  *out = tr;
  return APO_OK;
}

apo_status apo_trie_build_traces_multi(apo_ctx *ctx, int32_t nsrc, const uint64_t *const *h_src_tok,
                                       const int64_t *const *h_src_off, const int32_t *h_src_ntr, apo_trie **out,
                                       void *stream) {
  if (!out) return APO_ERR_INVALID;
  *out = nullptr;
  apo_trie *tr = new apo_trie();
  tr->ctx = ctx;
  apo_status st = trie_guard(ctx, [&](Ctx &c) {
    require(nsrc >= 1 && nsrc <= kMaxSrc && h_src_tok && h_src_off && h_src_ntr, "invalid argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PieceSrc src{};
    src.n = nsrc;
    std::vector<i64> h(1, 0);
    for (int r = 0; r < nsrc; ++r) {
      const int32_t nt = h_src_ntr[r];
      const int64_t *o = h_src_off[r];
      require(nt >= 0 && (nt == 0 || o != nullptr), "invalid argument");
      require(nt == 0 || o[0] == 0, "source offsets must start at 0");
      require(nt == 0 || h_src_tok[r] != nullptr, "NULL source pointer");
      src.tok[r] = h_src_tok[r];
      src.first[r] = i64(h.size()) - 1;
      src.base[r] = h.back();
      for (int t = 0; t < nt; ++t) {
        require(o[t + 1] > o[t], "traces must be non-empty");
        h.push_back(src.base[r] + o[t + 1]);
      }
    }
    src.first[nsrc] = i64(h.size()) - 1;
    src.base[nsrc] = h.back();
    const i64 N = h.back();
    // sources lying back to back in one buffer (TraceExchange stages every
    // rank's list so): hashed in place, no gathered copy
    const uint64_t *p0 = nullptr;
    bool contiguous = true;
    for (int r = 0; r < nsrc; ++r) {
      if (h_src_ntr[r] == 0) continue;
      if (p0 == nullptr) p0 = h_src_tok[r] - src.base[r];
      if (h_src_tok[r] != p0 + src.base[r]) contiguous = false;
    }
    if (contiguous && p0 != nullptr) {
      build_trace_set(c, tr, reinterpret_cast<const u64 *>(p0), h, s);
      return;
    }
    // the gathered tokens: a second scratch arena (build_trace_set carves the first)
    c.aux.reserve(sizeof(u64) * size_t(std::max<i64>(N, 1)), s);
    src.gather = reinterpret_cast<u64 *>(c.aux.base);
    build_trace_set(c, tr, src.gather, h, s, &src);
  });
  if (st != APO_OK) {
    apo_trie_destroy(tr);
    return st;
  }
  *out = tr;
  return APO_OK;
}

void apo_trie_destroy(apo_trie *tr) {
  if (!tr) return;
  if (tr->ctx) {
    if (tr->d_tok) tr->ctx->c.pool_put(tr->d_tok, tr->tok_bytes);
    if (tr->d_rtok) tr->ctx->c.pool_put(tr->d_rtok, tr->tok_bytes);
    tr->ctx->c.pool_put(tr->d_off, tr->off_bytes);
  }
  delete tr;
}

apo_status apo_trie_info(const apo_trie *tr, int64_t *h_ntraces, int64_t *h_ntokens, int64_t *h_maxlen) {
  if (!tr) return APO_ERR_INVALID;
  if (h_ntraces) *h_ntraces = tr->T;
  if (h_ntokens) *h_ntokens = tr->ntok;
  if (h_maxlen) *h_maxlen = tr->maxlen;
  return APO_OK;
}

apo_status apo_trie_copy(const apo_trie *tr, uint64_t *d_tokens, int64_t *h_off, void *stream) {
  if (!tr) return APO_ERR_INVALID;
  if (h_off) std::copy(tr->h_off.begin(), tr->h_off.end(), h_off);
  if (tr->ntok > 0 && d_tokens) {
    if (tr->d_tok) {
      cudaError_t e = cudaMemcpyAsync(d_tokens, tr->d_tok, sizeof(u64) * tr->ntok, cudaMemcpyDeviceToDevice,
                                      static_cast<cudaStream_t>(stream));
      if (e != cudaSuccess) return APO_ERR_CUDA;
    } else {  // the forward form straight from the kept reversed traces
      k_reverse_traces<<<grid_for(tr->T * 32, T256), T256, 0, static_cast<cudaStream_t>(stream)>>>(
          tr->d_rtok, tr->d_off, tr->T, d_tokens);
      if (cudaGetLastError() != cudaSuccess) return APO_ERR_CUDA;
    }
  }
  return APO_OK;
}

}  // extern "C"

namespace {
// MATCH_ALL (apo_match mode 0) into d_out[0..cap); *d_count <- hits.
void match_all(Ctx &c, const apo_trie *tr, const uint64_t *d_streams, const int64_t *h_off, int32_t nstreams,
               apo_match_rec *d_out, int64_t cap, int64_t *d_count, cudaStream_t s, ReplayIndex *ri = nullptr,
               apo_stream_index *build_idx = nullptr, const apo_stream_index *pre = nullptr) {
  if (ri) ri->ok = false;
  {
    if (d_count) APO_CUDA(cudaMemsetAsync(d_count, 0, sizeof(i64), s));
    const i64 Ns = h_off[nstreams];
    require(h_off[0] == 0, "h_off[0] must be 0");
    i64 maxs = 0;
    for (int q = 0; q < nstreams; ++q) {
      require(h_off[q + 1] >= h_off[q], "h_off must be non-decreasing");
      maxs = std::max<i64>(maxs, h_off[q + 1] - h_off[q]);
    }
    const i64 T = tr ? tr->T : 0;
    if (Ns == 0 || (!build_idx && T == 0)) return;
    require(d_streams != nullptr, "NULL device pointer");
    require(Ns < (i64(1) << 31) - 1, "streams longer than 2^31-1 tokens");
    const int bT = bits_for(u64(std::max<i64>(T, 1) - 1)), bE = bits_for(u64(maxs - 1)),
              bS = bits_for(u64(nstreams - 1));
    require(bT + bE + bS <= 64, "match key does not fit 64 bits");
    std::vector<i64> h_s(h_off, h_off + nstreams + 1);
    u64 *keys = nullptr, *keys_alt = nullptr;
    i64 nh = -1;
    bool emitted = false;  // hits already written in final order
    {
      // ---- per-stream path: each stream's own SA, bucketed by first token ----
      Batch b;
      b.N = Ns;
      b.W = nstreams;
      b.maxwin = maxs;
      GenPlan g;
      u64 *e_tok = nullptr, *e_tok_alt, *d_rs = nullptr;
      unsigned short *sid16 = nullptr;
      u32 *e_lo = nullptr, *e_q = nullptr, *e_hi = nullptr, *e_idx, *e_idx_alt, *ea, *ecnt, *pbase;
      i64 *scal;
      // streams that fit on chip are matched in reversed form (see k_stream_emit)
      const bool rev = maxs <= kSMMax;
      // the stream index: reversed streams, their suffix arrays + LCP,
      // first-token buckets (trace-independent; precomputed when `pre`)
      const i64 *p_off;
      const i32 *p_wid, *p_sa, *p_lcp;
      const u64 *mtok, *stok;
      bool d_rs_used = false;  // the reversed token copy exists (raw-token paths)
      int depth = 1;           // tokens keying the buckets
      const u32 *sord;
      i64 E;
      // dense-id matcher (k_stream_match_ids): stream ids + the batch dictionary
      const unsigned short *p_sid = nullptr;
      const u64 *p_dk = nullptr;
      i64 p_dkn = 0;
      bool p_dkmax = false;
      // the streams' buckets (one CTA per stream, look-back offsets), sorted
      // by key; keys are ids + 1 (bits(K)), two of them at depth 2, or raw
      // tokens (64 bits)
      auto make_buckets = [&](const StreamMatch &smb, int dep, u64 *et, u64 *et_alt, u32 *elo, u32 *eq, u32 *ehi,
                              u32 *eidx, u32 *eidx_alt, const u64 **out_tok, const u32 **out_ord, i64 *out_E) {
        c.ensure_status(size_t(nstreams), s);
        u32 *ctr = c.take_counter(s);
        const u32 ep = c.next_epoch();
        k_stream_buckets<<<nstreams, kBkThreads, 0, s>>>(smb, p_sid, et, elo, eq, ehi, eidx, scal, nstreams, c.status,
                                                       ctr, ep, dep);
        APO_CHECK_LAUNCH();
        c.launches++;
        const i64 En = i64(c.read_u64(reinterpret_cast<const u64 *>(scal), s));
        const int idb = bits_for(u64(p_dkn + (p_dkmax ? 1 : 0)));
        const int ebits = p_sid ? (dep == 2 ? 17 + idb : idb) : 64;
        const bool ae = radix_sort_u64_u32(c, et, eidx, et_alt, eidx_alt, En, 0, ebits, s);
        *out_tok = ae ? et_alt : et;
        *out_ord = ae ? eidx_alt : eidx;
        *out_E = En;
        c.launches++;
      };
      u64 *rb_tok = nullptr, *rb_tok_alt = nullptr;  // bucket rebuild (pre index at depth 2, 1-token traces)
      u32 *rb_lo = nullptr, *rb_q = nullptr, *rb_hi = nullptr, *rb_idx = nullptr, *rb_idx_alt = nullptr;
      if (pre) {
        const bool rebuild = pre->depth == 2 && tr->minlen < 2;
        auto plan = [&](Carver &cv) {
          ea = cv.take<u32>(T);
          ecnt = cv.take<u32>(T);
          pbase = cv.take<u32>(T);
          scal = cv.take<i64>(4);
          if (rebuild) {
            rb_tok = cv.take<u64>(Ns);
            rb_tok_alt = cv.take<u64>(Ns);
            rb_lo = cv.take<u32>(Ns);
            rb_q = cv.take<u32>(Ns);
            rb_hi = cv.take<u32>(Ns);
            rb_idx = cv.take<u32>(Ns);
            rb_idx_alt = cv.take<u32>(Ns);
          }
        };
        Carver dry(nullptr);
        plan(dry);
        c.arena.reserve(dry.off, s);
        Carver cv(c.arena.base);
        plan(cv);
        APO_CUDA(cudaMemsetAsync(scal, 0, sizeof(i64) * 4, s));
        p_off = pre->d_off;
        p_wid = pre->d_wid;
        p_sa = pre->sa;
        p_lcp = pre->lcp;
        mtok = pre->rev ? pre->rs : d_streams;
        stok = pre->stok;
        sord = pre->sord;
        e_lo = pre->e_lo;
        e_q = pre->e_q;
        e_hi = pre->e_hi;
        E = pre->E;
        p_sid = pre->sid;
        p_dk = pre->dk;
        p_dkn = pre->dk_n;
        p_dkmax = pre->dk_max;
        depth = pre->depth;
        if (depth == 2 && tr->minlen < 2) {
          // 1-token traces: rebuild the buckets by first token only
          u64 *rt = rb_tok, *rt_alt = rb_tok_alt;
          StreamMatch smb{p_off, p_wid, p_sa, p_lcp, mtok, nullptr, nullptr, Ns, T};
          depth = 1;
          make_buckets(smb, 1, rt, rt_alt, rb_lo, rb_q, rb_hi, rb_idx, rb_idx_alt, &stok, &sord, &E);
          e_lo = rb_lo;
          e_q = rb_q;
          e_hi = rb_hi;
        }
      } else {
      auto plan = [&](Carver &cv) {
        plan_gen(cv, b, g, true, c.nsmid);
        if (rev) d_rs = cv.take<u64>(Ns);
        e_tok = cv.take<u64>(Ns);
        e_tok_alt = cv.take<u64>(Ns);
        e_lo = cv.take<u32>(Ns);
        e_q = cv.take<u32>(Ns);
        e_hi = cv.take<u32>(Ns);
        e_idx = cv.take<u32>(Ns);
        e_idx_alt = cv.take<u32>(Ns);
        sid16 = rev ? cv.take<unsigned short>(Ns) : nullptr;
        ea = cv.take<u32>(T);
        ecnt = cv.take<u32>(T);
        pbase = cv.take<u32>(T);
        scal = cv.take<i64>(4);
      };
      Carver dry(nullptr);
      plan(dry);
      c.arena.reserve(dry.off, s);
      Carver cv(c.arena.base);
      plan(cv);
      upload_batch(c, b, g, h_s, s);
      // the reversed streams' suffix arrays: K9 over MIRRORED dense ids (no
      // reversed token copy); the reversed tokens are materialised only
      // for the raw-token paths (vocabulary over 65,534 or no dense ids)
      bool mirrored = false;
      IdsMirror mir{g.d_off, sid16};
      if (rev) mirrored = build_sa_mirrored(c, d_streams, b, g.sa, true, s, mir);
      const bool ids16 = mirrored && mir.id16_ok && g.sa.dkeys;
      if (rev && !ids16) {
        k_reverse_by_wid<<<grid_for(Ns, T256), T256, 0, s>>>(d_streams, g.d_off, g.d_wid, Ns, d_rs);
        APO_CHECK_LAUNCH();
        c.launches++;
      }
      mtok = rev ? (ids16 ? nullptr : d_rs) : d_streams;
      d_rs_used = rev && !ids16;
      if (!mirrored) build_sa(c, mtok, b, g.sa, true, s);
      if (ids16) {
        p_sid = sid16;
        p_dk = g.sa.dkeys;
        p_dkn = g.sa.dk_n;
        p_dkmax = g.sa.dk_max;
      }
      p_off = g.d_off;
      p_wid = g.d_wid;
      p_sa = g.sa.sa;
      p_lcp = g.sa.lcp;
      StreamMatch sm0{p_off, p_wid, p_sa, p_lcp, mtok, nullptr, nullptr, Ns, T};
      APO_CUDA(cudaMemsetAsync(scal, 0, sizeof(i64) * 4, s));
      // buckets by the first two tokens on the id path (fewer, tighter
      // pairs), unless the trace set has 1-token traces
      depth = (p_sid != nullptr && (build_idx != nullptr || (tr != nullptr && tr->minlen >= 2))) ? 2 : 1;
      make_buckets(sm0, depth, e_tok, e_tok_alt, e_lo, e_q, e_hi, e_idx, e_idx_alt, &stok, &sord, &E);
      if (build_idx) {  // apo_match_index: keep the index in a pooled block
        apo_stream_index &x = *build_idx;
        x.d_streams = d_streams;
        x.h_off = h_s;
        x.nstreams = nstreams;
        x.Ns = Ns;
        x.maxs = maxs;
        x.E = E;
        x.rev = rev;
        x.depth = depth;
        Carver kd(nullptr);
        auto carve = [&](Carver &k) {
          x.d_off = k.take<i64>(size_t(nstreams) + 1);
          x.d_wid = k.take<i32>(size_t(Ns));
          x.sa = k.take<i32>(size_t(Ns));
          x.lcp = k.take<i32>(size_t(Ns));
          x.rs = (rev && d_rs_used) ? k.take<u64>(size_t(Ns)) : nullptr;
          x.stok = k.take<u64>(size_t(std::max<i64>(E, 1)));
          x.sord = k.take<u32>(size_t(std::max<i64>(E, 1)));
          x.e_lo = k.take<u32>(size_t(std::max<i64>(E, 1)));
          x.e_q = k.take<u32>(size_t(std::max<i64>(E, 1)));
          x.e_hi = k.take<u32>(size_t(std::max<i64>(E, 1)));
          x.sid = p_sid ? k.take<unsigned short>(size_t(Ns)) : nullptr;
          x.dk = p_sid ? k.take<u64>(size_t(std::max<i64>(p_dkn, 1))) : nullptr;
        };
        carve(kd);
        x.bytes = kd.off + 256;
        x.blk = c.pool_get(x.bytes);
        Carver kc(static_cast<char *>(x.blk));
        carve(kc);
        auto cp = [&](void *dst, const void *src, size_t n) {
          if (n) c.d2d(dst, src, n, s);
        };
        cp(x.d_off, g.d_off, sizeof(i64) * (size_t(nstreams) + 1));
        cp(x.d_wid, g.d_wid, sizeof(i32) * size_t(Ns));
        cp(x.sa, g.sa.sa, sizeof(i32) * size_t(Ns));
        cp(x.lcp, g.sa.lcp, sizeof(i32) * size_t(Ns));
        if (x.rs) cp(x.rs, d_rs, sizeof(u64) * size_t(Ns));
        cp(x.stok, stok, sizeof(u64) * size_t(E));
        cp(x.sord, sord, sizeof(u32) * size_t(E));
        cp(x.e_lo, e_lo, sizeof(u32) * size_t(E));
        cp(x.e_q, e_q, sizeof(u32) * size_t(E));
        cp(x.e_hi, e_hi, sizeof(u32) * size_t(E));
        if (p_sid) {
          cp(x.sid, p_sid, sizeof(unsigned short) * size_t(Ns));
          cp(x.dk, p_dk, sizeof(u64) * size_t(p_dkn));
          x.dk_n = p_dkn;
          x.dk_max = p_dkmax;
        }
        return;
      }
      }  // index computed here (not pre)
      if (!rev) trie_forward(c, tr, s);
      StreamMatch sm{p_off, p_wid, p_sa, p_lcp, mtok, rev ? tr->d_rtok : tr->d_tok, tr->d_off, Ns, T};
      // dense-id matching: the traces' comparison values against the batch
      // dictionary (the buckets are keyed by id too)
      u32 *tid = nullptr;
      char *dict = nullptr;
      size_t tid_bytes = 0, dict_bytes = 0;
      struct PoolBack {  // returned once this block's launches are enqueued (pool users are stream-ordered)
        Ctx &c;
        void *&p;
        size_t &n;
        ~PoolBack() {
          if (p) c.pool_put(p, n);
        }
      };
      void *tid_v = nullptr, *dict_v = nullptr;
      PoolBack back_tid{c, tid_v, tid_bytes}, back_dict{c, dict_v, dict_bytes};
      if (p_sid != nullptr) {
        tid_bytes = sizeof(u32) * size_t(std::max<i64>(tr->ntok, 1));
        tid = static_cast<u32 *>(c.pool_get(tid_bytes));
        u32 tslots = 1024;
        while (i64(tslots) < 4 * p_dkn) tslots <<= 1;
        dict_bytes = sizeof(ulonglong2) * size_t(tslots);
        dict = static_cast<char *>(c.pool_get(dict_bytes));
        ulonglong2 *slot = reinterpret_cast<ulonglong2 *>(dict);
        APO_CUDA(cudaMemsetAsync(slot, 0xff, dict_bytes, s));
        if (p_dkn > 0) {
          k_dict_build<<<grid_for(p_dkn, T256), T256, 0, s>>>(p_dk, p_dkn, slot, tslots - 1);
          APO_CHECK_LAUNCH();
        }
        k_trace_ids<<<grid_for(std::max<i64>(tr->ntok, 1), T256), T256, 0, s>>>(tr->d_rtok, tr->ntok, p_dkn,
                                                                                p_dkmax ? 1 : 0, slot, tslots - 1, tid);
        APO_CHECK_LAUNCH();
        c.launches += 2;
        tid_v = tid;
        dict_v = dict;
      }
      k_trace_buckets<<<grid_for(T, T256), T256, 0, s>>>(sm, stok, E, ea, ecnt, tid, depth);
      APO_CHECK_LAUNCH();
      c.launches++;
      PairBaseF pf{ecnt, pbase, T, scal + 1};
      launch_scan<false>(c, T, pf, s);
      const i64 P = i64(c.read_u64(reinterpret_cast<const u64 *>(scal + 1), s));
      void *spill = nullptr;  // pooled spill block of the pair tables (see below)
      size_t spill_bytes = 0;
      // exact filter; fall back to the generalized SA when the pairs explode
      // (e.g. a tiny alphabet where every trace's first token is everywhere)
      if (P <= std::max<i64>(Ns / 4, 4 * T)) {
        nh = 0;
        if (P > 0) {
          i64 *ilo;
          u32 *icnt, *hbase, *ptr;
          Carver cx(nullptr);
          cx.take<i64>(P);
          cx.take<u32>(P);
          cx.take<u32>(P);
          cx.take<u32>(P);
          c.aux.reserve(cx.off, s);
          Carver ca(c.aux.base);
          ilo = ca.take<i64>(P);
          icnt = ca.take<u32>(P);
          hbase = ca.take<u32>(P);
          ptr = ca.take<u32>(P);
          if (maxs <= kSMMax) {
            // group the pairs by stream; one CTA per stream on chip
            // carve after the pair tables (the aux arena holds both)
            Carver full(nullptr);
            full.off = cx.off;
            full.take<u32>(P);
            full.take<u64>(P);
            full.take<u64>(P);
            full.take<u32>(P);
            full.take<u32>(P);
            full.take<u32>(size_t(nstreams) + 1);
            full.take<u32>(size_t(nstreams));
            full.take<u32>(size_t(nstreams));
            full.take<u64>(size_t(nstreams));
            full.take<u64>(size_t(nstreams));
            full.take<u32>(size_t(nstreams));
            full.take<u32>(size_t(nstreams));
            full.take<u64>(P);
            full.take<u64>(P);
            full.take<u32>(P);
            full.take<u32>(P);
            full.take<u32>(size_t(nstreams) + 1);
            full.take<u32>(P);
            full.take<u32>(P);
            full.take<u32>(P);
            full.take<u32>(P);
            full.take<u32>(P);
            full.take<u32>(size_t(nstreams));
            full.take<u32>(P);
            const bool use_ids = p_sid != nullptr && tr->ntok < (i64(1) << 32);
            if (use_ids) full.take<uint4>(P);
            if (full.off > c.aux.cap) {
              c.aux.reserve(full.off, s);
              Carver cb(c.aux.base);
              ilo = cb.take<i64>(P);
              icnt = cb.take<u32>(P);
              hbase = cb.take<u32>(P);
              ptr = cb.take<u32>(P);
            }
            Carver cz(c.aux.base);
            cz.off = cx.off;
            u32 *pair_e = cz.take<u32>(P);
            u64 *qk = cz.take<u64>(P), *qk_alt = cz.take<u64>(P);
            u32 *qv = cz.take<u32>(P), *qv_alt = cz.take<u32>(P);
            u32 *qoff = cz.take<u32>(size_t(nstreams) + 1);
            u32 *qtot = cz.take<u32>(size_t(nstreams));
            u32 *qbase = cz.take<u32>(size_t(nstreams));
            u64 *sk = cz.take<u64>(size_t(nstreams)), *sk_alt = cz.take<u64>(size_t(nstreams));
            u32 *sv = cz.take<u32>(size_t(nstreams)), *sv_alt = cz.take<u32>(size_t(nstreams));
            u64 *tk = cz.take<u64>(P), *tk_alt = cz.take<u64>(P);
            u32 *tv = cz.take<u32>(P), *tv_alt = cz.take<u32>(P);
            u32 *tof = cz.take<u32>(size_t(nstreams) + 1);
            u32 *gpar = cz.take<u32>(P), *ghi = cz.take<u32>(P), *gtr = cz.take<u32>(P), *gdep = cz.take<u32>(P);
            u32 *groot = cz.take<u32>(P);
            u32 *otr = cz.take<u32>(P);
            u32 *tbig = cz.take<u32>(size_t(nstreams));
            uint4 *meta = use_ids ? cz.take<uint4>(P) : nullptr;
            k_pair_list<<<grid_for(T * 32, T256), T256, 0, s>>>(pbase, ea, ecnt, sord, e_q, T, pair_e, ptr, qk, qv);
            APO_CHECK_LAUNCH();
            bool aq = radix_sort_u64_u32(c, qk, qv, qk_alt, qv_alt, P, 0, bits_for(u64(nstreams - 1)), s);
            const u64 *sqk = aq ? qk_alt : qk;
            const u32 *sqv = aq ? qv_alt : qv;
            k_q_offsets<<<grid_for(i64(nstreams) + 1, T256), T256, 0, s>>>(sqk, P, nstreams, qoff);
            APO_CHECK_LAUNCH();
            k_stream_keys<<<grid_for(nstreams, T256), T256, 0, s>>>(qoff, sqv, ptr, nstreams, T, sk, sv);
            APO_CHECK_LAUNCH();
            c.launches += 2;
            const bool as = radix_sort_u64_u32(c, sk, sv, sk_alt, sv_alt, nstreams, 0, 32, s);
            const u32 *qorder = as ? sv_alt : sv;
            if (use_ids) {
              k_pair_meta<<<grid_for(P, T256), T256, 0, s>>>(sqk, sqv, P, pair_e, ptr, e_lo, e_hi, p_off, tr->d_off,
                                                             meta);
              APO_CHECK_LAUNCH();
              const size_t smem = sizeof(unsigned short) * (3 * size_t(kSMMax) + kSMIPad) +
                                  sizeof(u32) * size_t(kSMIWarps) * kSMICache;
              c.smem_optin(reinterpret_cast<const void *>(k_stream_match_ids), smem);
              if (c.prof) c.prof_begin(kProfMatch, 0.0, s);
              k_stream_match_ids<<<nstreams, kSMIThreads, smem, s>>>(p_off, p_sa, p_lcp, p_sid, tid, meta, qoff, ilo,
                                                                     icnt, qtot, qorder, depth);
              APO_CHECK_LAUNCH();
              if (c.prof) c.prof_end(s);
              c.launches += 3;
            } else {
              const size_t smem = sizeof(u64) * kSMMax + 2 * sizeof(unsigned short) * kSMMax;
              c.smem_optin(reinterpret_cast<const void *>(k_stream_match), smem);
              if (c.prof) c.prof_begin(kProfMatch, 0.0, s);
              k_stream_match<<<nstreams, kSMThreads, smem, s>>>(sm, sqv, qoff, pair_e, ptr, e_lo, e_hi, ilo, icnt,
                                                                qtot, qorder);
              APO_CHECK_LAUNCH();
              if (c.prof) c.prof_end(s);
              c.launches += 3;
            }
            // hits in final order straight from the per-stream emitter
            PairBaseF qf{qtot, qbase, nstreams, scal + 3};
            launch_scan<false>(c, nstreams, qf, s);
            nh = i64(c.read_u64(reinterpret_cast<const u64 *>(scal + 3), s));
            emitted = true;
            // REPLAY (mode 1) keeps MATCH_ALL implicit (k_stream_ends) unless
            // APO_REPLAY_EAGER is set (tests: the emitted-records path)
            const bool lazy = ri && rev && Ns < (i64(1) << 32) && std::getenv("APO_REPLAY_EAGER") == nullptr;
            if (nh > 0 && (cap > 0 || lazy)) {
              // interval forest of every stream (preorder sort + stack sweep)
              k_tree_keys<<<grid_for(P, T256), T256, 0, s>>>(sqk, sqv, ilo, icnt, p_off, ptr, P, bS, tk, tv, gtr);
              APO_CHECK_LAUNCH();
              const bool at = radix_sort_u64_u32(c, tk, tv, tk_alt, tv_alt, P, 0, bS + 31, s);
              const u64 *stk = at ? tk_alt : tk;
              const u32 *stv = at ? tv_alt : tv;
              k_tree_offsets<<<grid_for(i64(nstreams) + 1, T256), T256, 0, s>>>(stk, P, nstreams, tof);
              APO_CHECK_LAUNCH();
              // APO_TREE_SEQ=1 (tests) forces the sequential sweep on every stream
              static const bool tree_seq = std::getenv("APO_TREE_SEQ") != nullptr;
              APO_CUDA(cudaMemsetAsync(tbig, tree_seq ? 0xff : 0, sizeof(u32) * size_t(nstreams), s));
              if (!tree_seq) {
                k_tree_par<<<nstreams, 32, 0, s>>>(stk, stv, tof, gtr, gpar, ghi, gdep, otr, groot, tbig);
                APO_CHECK_LAUNCH();
              }
              k_tree_sweep<<<nstreams, 32, 0, s>>>(stk, stv, tof, gtr, gpar, ghi, gdep, otr, groot, tbig);
              APO_CHECK_LAUNCH();
              c.launches++;
              if (lazy) {
                ri->endoff_bytes = sizeof(u32) * size_t(Ns);
                ri->endml_bytes = sizeof(unsigned short) * size_t(Ns);
                u32 *deepz = static_cast<u32 *>(c.pool_get(ri->endoff_bytes));
                unsigned short *endml = static_cast<unsigned short *>(c.pool_get(ri->endml_bytes));
                const size_t nsmem = (sizeof(u32) + sizeof(unsigned short)) * size_t(kSMMax) +
                                     sizeof(unsigned short) * size_t(kEndsMl);
                c.smem_optin(reinterpret_cast<const void *>(k_stream_ends), nsmem);
                k_stream_ends<<<nstreams, kEndsThreads, nsmem, s>>>(sm, stk, tof, otr, groot, gpar, deepz, endml,
                                                                    qorder);
                APO_CHECK_LAUNCH();
                ri->ok = true;
                ri->lazy = true;
                ri->off = p_off;
                ri->sa = p_sa;
                ri->tkey = stk;
                ri->toff = tof;
                ri->nint = P;
                ri->endoff = deepz;
                ri->endml = endml;
                ri->opar = gpar;
                ri->otr = otr;
                ri->odep = gdep;
                ri->qbase = qbase;
                c.launches += 4;
              } else {
              const size_t esmem = sizeof(u32) * (kSMMax + 3 * kEmitPairs) + sizeof(unsigned short) * kSMMax;
              c.smem_optin(reinterpret_cast<const void *>(k_stream_emit), esmem);
              const bool pair32 = (reinterpret_cast<uintptr_t>(d_out) & 31) == 0;
              u32 *endoff = nullptr;
              unsigned short *endml = nullptr;
              if (ri && rev && nh <= cap && Ns < (i64(1) << 32)) {  // REPLAY's per-end index (mode 1)
                ri->endoff_bytes = sizeof(u32) * size_t(Ns);
                ri->endml_bytes = sizeof(unsigned short) * size_t(Ns);
                endoff = static_cast<u32 *>(c.pool_get(ri->endoff_bytes));
                endml = static_cast<unsigned short *>(c.pool_get(ri->endml_bytes));
              }
              k_stream_emit<<<nstreams, kEmitThreads, esmem, s>>>(sm, stk, tof, qbase, cap, d_out, qorder, gpar, otr,
                                                                  gdep, pair32, endoff, endml);
              APO_CHECK_LAUNCH();
              if (ri && rev && nh <= cap) {
                ri->ok = true;
                ri->off = p_off;
                ri->sa = p_sa;
                ri->tkey = stk;
                ri->toff = tof;
                ri->nint = P;
                ri->endoff = endoff;
                ri->endml = endml;
              }
              c.launches += 4;
              }
            }
          } else {
            const i64 chunks = (P + kPairChunk - 1) / kPairChunk;
            k_pair_search<<<grid_for(chunks * 32, 256), 256, 0, s>>>(sm, pbase, ea, P, sord, e_lo, e_hi, e_q, ilo,
                                                                       icnt, ptr);
            APO_CHECK_LAUNCH();
            c.launches++;
          }
          if (!emitted) {
          PairBaseF hf{icnt, hbase, P, scal + 2};
          launch_scan<false>(c, P, hf, s);
          nh = i64(c.read_u64(reinterpret_cast<const u64 *>(scal + 2), s));
          if (std::getenv("APO_DEBUG_STATS")) {
            std::vector<u32> hc(static_cast<size_t>(P));
            APO_CUDA(cudaMemcpy(hc.data(), icnt, sizeof(u32) * P, cudaMemcpyDeviceToHost));
            i64 matched = 0;
            for (u32 v : hc) matched += v > 0;
            std::fprintf(stderr, "apo_match: streams=%d traces=%lld buckets=%lld pairs=%lld matched_pairs=%lld hits=%lld\n",
                         nstreams, (long long)T, (long long)E, (long long)P, (long long)matched, (long long)nh);
          }
          if (nh > 0) {
            // keys after the pair tables in the aux arena (grown if needed:
            // reserve() keeps nothing, so re-carve the pair tables first)
            const size_t need = cx.off + 256 + sizeof(u64) * size_t(nh) * 2;
            if (need > c.aux.cap) {
              // move the pair tables aside: into the main arena's key buffers
              // when they fit (P <= Ns), else into a pooled block that is
              // returned once the enumeration is enqueued (later users of the
              // pool run on the same stream, after it)
              i64 *ilo2 = reinterpret_cast<i64 *>(e_tok);
              u32 *hb2 = e_lo, *pt2 = e_q;
              if (P > Ns || pre != nullptr) {  // (a precomputed index is not scratch)
                spill_bytes = (sizeof(i64) + 2 * sizeof(u32)) * size_t(P) + 256;
                spill = c.pool_get(spill_bytes);
                ilo2 = reinterpret_cast<i64 *>(spill);
                hb2 = reinterpret_cast<u32 *>(ilo2 + P);
                pt2 = hb2 + P;
              }
              c.d2d(ilo2, ilo, sizeof(i64) * P, s);
              c.d2d(hb2, hbase, sizeof(u32) * P, s);
              c.d2d(pt2, ptr, sizeof(u32) * P, s);
              c.aux.reserve(need, s);
              ilo = ilo2;
              hbase = hb2;
              ptr = pt2;
              keys = reinterpret_cast<u64 *>(c.aux.base);
            } else {
              keys = reinterpret_cast<u64 *>(c.aux.base + ((cx.off + 255) & ~size_t(255)));
            }
            keys_alt = keys + nh;
            k_enumerate_pairs<<<grid_for(P * 32, T256), T256, 0, s>>>(sm, ilo, hbase, ptr, P, nh, bE, bT, keys);
            APO_CHECK_LAUNCH();
            c.launches++;
            if (spill) c.pool_put(spill, spill_bytes);
          }
          }
        }
      }
    }
    if (nh < 0) {
    // ---- fallback: one generalized suffix array over the streams ----
    Batch b;
    b.N = Ns;
    b.W = nstreams;
    b.gen = true;
    b.maxwin = maxs;
    b.sort_depth = tr->maxlen;  // binary search compares at most maxlen tokens
    GenPlan g;
    i64 *ilo = nullptr, *scal = nullptr;
    u32 *ibase = nullptr, *icnt = nullptr;
    auto plan = [&](Carver &cv) {
      plan_gen(cv, b, g, false, c.nsmid);
      ilo = cv.take<i64>(T);
      ibase = cv.take<u32>(T);
      icnt = cv.take<u32>(T);
      scal = cv.take<i64>(4);
    };
    Carver dry(nullptr);
    plan(dry);
    c.arena.reserve(dry.off, s);
    Carver cv(c.arena.base);
    plan(cv);
    upload_batch(c, b, g, h_s, s);
    build_sa(c, d_streams, b, g.sa, false, s);
    trie_forward(c, tr, s);
    MatchSetup m{Ns, nstreams, T, g.d_off, g.d_wid, g.sa.sa, d_streams, tr->d_tok, tr->d_off};
    k_trace_search<<<grid_for(T * 32, 256), 256, 0, s>>>(m, ilo, icnt);
    APO_CHECK_LAUNCH();
    c.launches++;
    APO_CUDA(cudaMemsetAsync(scal, 0, sizeof(i64) * 4, s));
    CountScanF cf{icnt, ibase, T, scal};
    launch_scan<false>(c, T, cf, s);
    nh = i64(c.read_u64(reinterpret_cast<const u64 *>(scal), s));
    if (nh > 0) {
      c.aux.reserve(sizeof(u64) * size_t(nh) * 2 + 1024, s);
      keys = reinterpret_cast<u64 *>(c.aux.base);
      keys_alt = keys + nh;
      k_enumerate<<<grid_for(nh, T256), T256, 0, s>>>(m, ilo, ibase, nh, bE, bT, keys);
      APO_CHECK_LAUNCH();
      c.launches++;
    }
    }
    if (emitted) {
      c.h2d(d_count, &nh, sizeof(i64), s);
      APO_CUDA(cudaStreamSynchronize(s));
      return;
    }
    if (nh == 0) return;
    const int kb = bS + bE + bT;
    // hits were enumerated in trace-id order (both paths), so a STABLE sort
    // on the (stream, end) bits alone leaves equal (stream, end) in trace order
    bool a = radix_sort_u64_keys(c, keys, keys_alt, nh, bT, kb, s);
    const u64 *sorted = a ? keys_alt : keys;
    if (cap > 0) {
      k_write_hits<<<grid_for(std::min(nh, cap), T256), T256, 0, s>>>(sorted, nh, cap, bE, bT, d_out);
      APO_CHECK_LAUNCH();
      c.launches++;
    }
    c.h2d(d_count, &nh, sizeof(i64), s);
    APO_CUDA(cudaStreamSynchronize(s));
  }
}
}  // namespace

namespace apo {
namespace {
// apo_match / apo_match_indexed: MATCH_ALL (mode 0) or MATCH_ALL + REPLAY
// (mode 1) with the stream index computed here or taken from `pre`.
void match_entry(Ctx &c, const apo_trie *tr, const uint64_t *d_streams, const int64_t *h_off, int32_t nstreams,
                 int32_t mode, apo_match_rec *d_out, int64_t cap, int64_t *d_count, cudaStream_t s,
                 const apo_stream_index *pre) {
  require(tr != nullptr && d_count != nullptr && cap >= 0 && nstreams >= 1 && h_off != nullptr, "invalid argument");
  require(mode == 0 || mode == 1, "mode must be 0 (MATCH_ALL) or 1 (REPLAY)");
  require(cap == 0 || d_out != nullptr, "d_out is NULL");
  require((reinterpret_cast<uintptr_t>(d_out) & 15) == 0, "d_out must be 16-byte aligned");
  if (mode == 0) {
    match_all(c, tr, d_streams, h_off, nstreams, d_out, cap, d_count, s, nullptr, nullptr, pre);
    return;
  }
  // REPLAY: MATCH_ALL into a cached library buffer (grown and re-run if
  // too small), then the replay selection consumes the hits on the device
  i64 nh = 0;
  ReplayIndex ri;
  for (;;) {
    match_all(c, tr, d_streams, h_off, nstreams, static_cast<apo_match_rec *>(c.hitbuf),
              i64(c.hitbuf_cap / sizeof(apo_match_rec)), d_count, s, &ri, nullptr, pre);
    nh = i64(c.read_u64(reinterpret_cast<const u64 *>(d_count), s));
    if ((ri.ok && ri.lazy) || size_t(nh) * sizeof(apo_match_rec) <= c.hitbuf_cap) break;
    if (c.hitbuf) c.pool_put(c.hitbuf, c.hitbuf_cap);
    c.hitbuf_cap = (size_t(nh) + size_t(nh) / 16 + 1024) * sizeof(apo_match_rec);
    c.hitbuf = c.pool_get(c.hitbuf_cap);
  }
  std::vector<i64> len(static_cast<size_t>(nstreams));
  for (int q = 0; q < nstreams; ++q) len[q] = h_off[q + 1] - h_off[q];
  const apo_replay_params prm{100, 64881, 100, 11, 10, 0};
  run_replay(c, tr, static_cast<const apo_match_rec *>(c.hitbuf), nh, len.data(), nstreams, prm,
             reinterpret_cast<apo_replay_rec *>(d_out), cap, d_count, s, &ri);
  c.h2d(d_count + 1, &nh, sizeof(i64), s);
  APO_CUDA(cudaStreamSynchronize(s));
}
}  // namespace
}  // namespace apo

extern "C" {

apo_status apo_match(apo_ctx *ctx, const apo_trie *tr, const uint64_t *d_streams, const int64_t *h_off,
                     int32_t nstreams, int32_t mode, apo_match_rec *d_out, int64_t cap, int64_t *d_count,
                     void *stream) {
  return trie_guard(ctx, [&](Ctx &c) {
    match_entry(c, tr, d_streams, h_off, nstreams, mode, d_out, cap, d_count, static_cast<cudaStream_t>(stream),
                nullptr);
  });
}

apo_status apo_match_index(apo_ctx *ctx, const uint64_t *d_streams, const int64_t *h_off, int32_t nstreams,
                           apo_stream_index **out, void *stream) {
  return trie_guard(ctx, [&](Ctx &c) {
    require(out != nullptr && nstreams >= 1 && h_off != nullptr, "invalid argument");
    *out = nullptr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto *x = new apo_stream_index();
    x->ctx = ctx;
    try {
      match_all(c, nullptr, d_streams, h_off, nstreams, nullptr, 0, nullptr, s, nullptr, x, nullptr);
      APO_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      if (x->blk) c.pool_put(x->blk, x->bytes);
      delete x;
      throw;
    }
    if (x->nstreams == 0) {  // empty streams: an index with nothing to search
      x->d_streams = d_streams;
      x->h_off.assign(h_off, h_off + nstreams + 1);
      x->nstreams = nstreams;
    }
    *out = x;
  });
}

apo_status apo_match_indexed(apo_ctx *ctx, const apo_trie *tr, const apo_stream_index *idx, int32_t mode,
                             apo_match_rec *d_out, int64_t cap, int64_t *d_count, void *stream) {
  return trie_guard(ctx, [&](Ctx &c) {
    require(idx != nullptr && idx->ctx == ctx, "the index belongs to another context");
    match_entry(c, tr, idx->d_streams, idx->h_off.data(), idx->nstreams, mode, d_out, cap, d_count,
                static_cast<cudaStream_t>(stream), idx->blk ? idx : nullptr);
  });
}

void apo_stream_index_destroy(apo_stream_index *idx) {
  if (!idx) return;
  if (idx->blk && idx->ctx) idx->ctx->c.pool_put(idx->blk, idx->bytes);
  delete idx;
}

}  // extern "C"

#if APO_MATCH_STATS
extern "C" int apo_debug_match_stats(unsigned long long *out, int reset) {
  if (cudaMemcpyFromSymbol(out, apo::match_stats, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(apo::match_stats, z, sizeof(z));
  }
  return 0;
}
#endif
