// suffix_array.cu -- K2/K3/K4: suffix array by prefix doubling and the LCP
// array by the phi/PLCP (Kasai-style) method, for a batch of windows.
//
// "SA, LCP <- SuffixArray(S)" (Alg. 2); "Linear time
// algorithms exist for suffix array and LCP array construction".
//
// SA (prefix doubling, Manber-Myers style, all windows at once):
//   level 0   rank[i] = group start of token S[i] in (window, token) order
//   level r   rank_r[i] orders suffixes by their first 2^r tokens (padded
//             with an end marker that sorts first, reading R2)
//   round h   key(i) = rank[i] << lob | (i+h < end(window) ? rank[i+h]-beg+1 : 0)
//             LSD radix sort of (key, i); a sorted position k starts a new
//             group iff key[k] != key[k-1]; new rank = max-scan of group
//             starts, scattered to rank_next[sa[k]].  Stop when all distinct.
// Keys are built in POSITION order (coalesced reads of rank[i], rank[i+h]),
// so no gather through SA is needed; every level is kept for the LCP stage.
//
// LCP: phi[sa[k]] = sa[k-1]; PLCP[i] = lcp(i, phi[i]) computed in chunks of
// consecutive i per thread with the Kasai bound PLCP[i] >= PLCP[i-1]-1; each
// chunk's first value is found in O(log n) by galloping over the saved rank
// levels (equal level-r ranks <=> equal 2^r-token prefixes); LCP[k] =
// PLCP[sa[k+1]].
#include "pipeline.cuh"

#include <cstdlib>

namespace apo {

namespace {

__global__ void k_init_pairs(const u64 *__restrict__ tok, i64 n, u64 *__restrict__ keys,
                             u32 *__restrict__ vals) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = tok[i];
    vals[i] = u32(i);
  }
}

// batched: sort key = window id of the position (stable over (token, i) order)
__global__ void k_wid_keys(const u32 *__restrict__ idx, const i32 *__restrict__ wid, i64 n,
                           u64 *__restrict__ keys) {
  i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) keys[k] = u64(u32(wid[idx[k]]));
}

__global__ void k_gather_tok(const u32 *__restrict__ idx, const u64 *__restrict__ tok, i64 n,
                             u64 *__restrict__ out) {
  i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) out[k] = tok[idx[k]];
}

// Level-0 ranks: head of a (window, token) group -> group start, max-scanned.
struct InitRankF {
  const u64 *tok_sorted;  // tokens in sorted order
  const u32 *sa;
  const i32 *wid;         // nullptr if single window
  i32 *rank;
  __device__ u32 load(i64 k) const {
    if (k == 0) return 0;
    bool head = tok_sorted[k] != tok_sorted[k - 1];
    if (wid && !head) head = wid[sa[k]] != wid[sa[k - 1]];
    return head ? u32(k) : 0u;
  }
  __device__ bool store(i64 k, u32 incl, u32) const {
    rank[sa[k]] = i32(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_count_ids(const u32 *__restrict__ ids, i64 n, u32 *__restrict__ cnt) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[ids[i]], 1u);
}

struct ExclF {  // in-place exclusive sum
  u32 *a;
  __device__ u32 load(i64 i) const { return a[i]; }
  __device__ bool store(i64 i, u32, u32 excl) const {
    a[i] = excl;
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_rank_from_ids(const u32 *__restrict__ ids, i64 n, const u32 *__restrict__ start,
                                i32 *__restrict__ rank) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) rank[i] = i32(start[ids[i]]);
}

// Token packing: the first sort orders the suffixes by their
// first q tokens at once -- q dense ids of bt bits each (id + 1; 0 past the
// end of the single window) in one 64-bit key -- so doubling starts at
// h = q instead of 1 and saves log2(q) rounds.
__global__ void k_pack_keys(const u32 *__restrict__ ids, i64 n, int q, int bt, u64 *__restrict__ keys,
                            u32 *__restrict__ vals) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u64 k = 0;
  for (int t = 0; t < q; ++t) k = (k << bt) | (i + t < n ? u64(ids[i + t]) + 1u : 0ull);
  keys[i] = k;
  vals[i] = u32(i);
}

__global__ void k_double_keys(const i32 *__restrict__ rank, Batch b, i64 h, int lob, u64 *__restrict__ keys,
                              u32 *__restrict__ vals) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= b.N) return;
  int w = b_wid(b, i);
  i64 beg = b_beg(b, w), end = b_end(b, w);
  u64 lo;
  if (b.gen)  // sentinel $_w = w, real ranks shifted above all sentinels
    lo = (i + h < end) ? u64(rank[i + h]) + u64(b.W) : u64(w);
  else        // window-local rank + 1, end of window = 0
    lo = (i + h < end) ? u64(rank[i + h] - beg + 1) : 0ull;
  keys[i] = (u64(u32(rank[i])) << lob) | lo;
  vals[i] = u32(i);
}

// Manber-Myers order for a single window (the global path's rounds after
// the first): walking the previous order SA (sorted by the first h tokens)
// and emitting i = SA[q] - h lists the suffixes by their SECOND key
// rank[i + h]; the suffixes i >= n - h (second key "end of string", the
// smallest) take the slots of j = SA[q] < h.  All of those but i = n - h
// are singletons (shorter than h: their h-prefix includes the end), so only
// i = n - h must lead: it goes to slot 0 and the slots before its own shift
// up by one.  A stable sort of this list by the FIRST key alone (the high
// key bits) then orders by the full (rank[i], rank[i + h]) key: half the key
// bits per round.
// gate (Manber-Myers rounds launched ahead of the host's convergence check):
// the kernel returns at once when the previous round left *gate == 0
__global__ void k_pos_of_zero(const u32 *__restrict__ sa, i64 n, u32 *__restrict__ out, const u32 *gate) {
  if (gate != nullptr && *gate == 0u) return;
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < n && sa[q] == 0u) *out = u32(q);
}

__global__ void k_mm_keys(const u32 *__restrict__ sa_prev, const i32 *__restrict__ rank, i64 n, i64 h, int lob,
                          const u32 *__restrict__ q0p, u64 *__restrict__ keys, u32 *__restrict__ vals,
                          const u32 *gate) {
  if (gate != nullptr && *gate == 0u) return;
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const i64 q0 = *q0p;
  const i64 j = sa_prev[q];
  const i64 i = j >= h ? j - h : n - h + j;
  const i64 dst = q == q0 ? 0 : (q < q0 ? q + 1 : q);
  const u64 lo = i + h < n ? u64(rank[i + h] + 1) : 0ull;
  keys[dst] = (u64(u32(rank[i])) << lob) | lo;
  vals[dst] = u32(i);
}

// Next rank level from the sorted keys; flags "not done" if any group has
// more than one member.
struct DoubleRankF {
  const u64 *key;
  const u32 *sa;
  i32 *rank_next;
  u32 *notdone;
  __device__ u32 load(i64 k) const { return (k == 0 || key[k] != key[k - 1]) ? u32(k) : 0u; }
  __device__ bool store(i64 k, u32 incl, u32) const {
    rank_next[sa[k]] = i32(incl);
    return incl != u32(k);
  }
  __device__ u32 *flag() const { return notdone; }
};

__global__ void k_phi(const u32 *__restrict__ sa, Batch b, i32 *__restrict__ phi) {
  i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= b.N) return;
  i64 i = sa[k];
  // the SA is window-major: rank k lies in the window of position k
  bool first = b.gen ? (k == 0) : (k == b_beg(b, b_wid(b, k)));
  phi[i] = first ? -1 : i32(sa[k - 1]);
}

struct Levels {
  const i32 *p[40];
};

// lcp(i, j) (i < end_i, j < end_j) by galloping over rank levels R-1..0:
// equal level-r ranks <=> equal (unit * 2^r)-token prefixes (padded with the
// end marker of the suffix's own window); the last < unit tokens (token
// packing) are compared directly.
__device__ __forceinline__ i64 gallop_lcp(const Levels &L, int R, int unit, const u64 *__restrict__ tok, i64 i,
                                          i64 j, i64 end_i, i64 end_j, i64 from) {
  // from: a known lower bound of the lcp; lcp - from < unit * 2^R, so
  // descending multiples unit * 2^r reach it to within unit - 1
  i64 l = from;
  for (int r = R - 1; r >= 0; --r) {
    if (i + l >= end_i || j + l >= end_j) break;
    const i32 *lv = L.p[r];
    if (lv[i + l] == lv[j + l]) l += i64(unit) << r;
  }
  for (int t = 1; t < unit && i + l < end_i && j + l < end_j && tok[i + l] == tok[j + l]; ++t) ++l;
  return l;
}

constexpr int kPlcpChunk = 8;  // positions per thread (more independent Kasai chains in flight)
constexpr int kKasaiSteps = 16;
constexpr int kSpecMax = 8;   // Manber-Myers rounds launched per host convergence read

// With `lcp` set (windows fully sorted: the last rank level is the inverse
// suffix array), PLCP[i] is scattered straight to lcp[ISA[i] - 1] and the
// window's first suffix writes the window's last slot (0), so no gather pass
// over the suffix array is needed; otherwise PLCP goes to `plcp`.
__global__ void k_plcp(const u64 *__restrict__ tok, const i32 *__restrict__ phi, Levels L, int R, int unit,
                       const i32 *__restrict__ rw, Batch b, i32 *__restrict__ plcp, i32 *__restrict__ lcp) {
  i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  i64 i0 = t * kPlcpChunk;
  if (i0 >= b.N) return;
  i64 i1 = i0 + kPlcpChunk < b.N ? i0 + kPlcpChunk : b.N;
  i64 h = -1;  // -1: no Kasai lower bound available
  int cur_w = -1;
  i64 end = 0;
  int Rcur = R;
  for (i64 i = i0; i < i1; ++i) {
    int w = b_wid(b, i);
    if (w != cur_w) {
      cur_w = w;
      end = b_end(b, w);
      h = -1;
      if (rw) Rcur = rw[w];  // K9 path: per-window number of rounds
    }
    i64 j = phi[i];
    if (j < 0) {
      if (lcp) lcp[end - 1] = 0; else plcp[i] = 0;
      h = 0;
      continue;
    }
    const i64 end_j = b.gen ? b_end(b, b_wid(b, j)) : end;
    if (h < 0) {
      h = gallop_lcp(L, Rcur, unit, tok, i, j, end, end_j, 0);
    } else {
      // Kasai: PLCP[i] >= PLCP[i-1] - 1.  Extend by direct comparison for a
      // few tokens; a longer extension (after a sharp drop) is finished by
      // galloping from the current bound, so no thread walks thousands of
      // tokens one at a time.
      h = h > 0 ? h - 1 : 0;
      int steps = 0;
      while (i + h < end && j + h < end_j && tok[i + h] == tok[j + h]) {
        ++h;
        if (++steps == kKasaiSteps) {
          h = gallop_lcp(L, Rcur, unit, tok, i, j, end, end_j, h);
          break;
        }
      }
    }
    if (lcp)
      lcp[L.p[Rcur][i] - 1] = i32(h);  // the final level holds global ranks: ISA[i] - 1 is the predecessor pair
    else
      plcp[i] = i32(h);
  }
}

__global__ void k_lcp_gather(const u32 *__restrict__ sa, const i32 *__restrict__ plcp, Batch b,
                             i32 *__restrict__ lcp) {
  i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= b.N) return;
  i64 lim = b.gen ? b.N : b_end(b, b_wid(b, k));  // window-major SA: rank k is in the window of position k
  lcp[k] = (k + 1 < lim) ? plcp[sa[k + 1]] : 0;
}

}  // namespace

void plan_sa(Carver &cv, const Batch &b, SAWork &w, bool want_lcp, int nsmid) {
  const i64 N = b.N;
  w.keys = cv.take<u64>(N);
  w.keys_alt = cv.take<u64>(N);
  w.vals = cv.take<u32>(N);
  w.vals_alt = cv.take<u32>(N);
  w.tok_sorted = b.W > 1 ? cv.take<u64>(N) : nullptr;
  const bool k9 = window_sa_supported(b);
  // K9 keeps its rank levels on chip / in a per-CTA L2 scratch: only level 0
  // (the fallback initial ranking) is a per-position array there
  w.max_levels = k9 ? 1 : bits_for(u64(b.maxwin > 1 ? b.maxwin - 1 : 1)) + 2;
  if (w.max_levels > 40) w.max_levels = 40;
  for (int r = 0; r < w.max_levels; ++r) w.levels[r] = cv.take<i32>(N);
  w.sa = cv.take<i32>(N);
  w.rw = k9 ? cv.take<i32>(size_t(b.W)) : nullptr;
  w.win_scratch = k9 ? cv.take<char>(window_sa_scratch_bytes(nsmid)) : nullptr;
  w.ids = cv.take<u32>(N);
  w.ids_valid = false;
  w.ht_cap = 1u << 21;  // up to 1M distinct tokens; 24 MB of L2-friendly tables
  while (w.ht_cap > 4096 && u64(w.ht_cap) > 4 * u64(N)) w.ht_cap >>= 1;
  w.ht_scratch = cv.take<char>(token_ids_scratch_bytes(N, w.ht_cap));
  if (want_lcp) {
    w.phi = k9 ? nullptr : cv.take<i32>(N);
    w.plcp = k9 ? nullptr : cv.take<i32>(N);
    w.lcp = cv.take<i32>(N);
  } else {
    w.phi = w.plcp = w.lcp = nullptr;
  }
}

bool build_sa_mirrored(Ctx &c, const u64 *tok, const Batch &b, SAWork &w, bool want_lcp, cudaStream_t s,
                       IdsMirror &mir) {
  if (w.rw == nullptr || b.N == 0) return false;  // K9 path only
  w.ids_valid = false;
  w.unit = 1;
  w.R = 0;
  w.dkeys = nullptr;
  w.slot_rank = nullptr;
  mir.nwin = b.W;
  // the table slots of the FORWARD windows; K9 maps them to ids and reads
  // every window back to front
  const i64 K = dense_token_ids(c, tok, b.N, w.ids, w.ht_cap, w.ht_scratch, s, &w.dkeys, &w.dk_n, &w.dk_max, &mir,
                                &w.slot_rank);
  if (K < 0) return false;
  w.ids_valid = true;
  w.K = K;
  w.mirror = true;
  run_window_sa(c, b, w, want_lcp, s);
  w.mirror = false;
  return true;
}

void build_sa(Ctx &c, const u64 *tok, const Batch &b, SAWork &w, bool want_lcp, cudaStream_t s, IdsMirror *mir) {
  (void)mir;
  const i64 N = b.N;
  const int T = 256;
  const int G = grid_for(N, T);
  w.R = 0;
  if (N == 0) return;

  // ---- K2: level-0 ranks ----
  // Dense token ids from the hash table whenever the level-0 ranks do not
  // depend on the window (generalized mode, a single window) or K9 computes
  // its window-local ranks itself; otherwise (or if the vocabulary is too
  // large) the 64-bit radix sort of (token, position).
  w.ids_valid = false;
  w.unit = 1;
  w.K = -1;
  w.dkeys = nullptr;
  w.slot_rank = nullptr;
  w.mirror = false;
  i64 packK = -1;
  if (b.gen || b.W == 1 || w.rw != nullptr) {
    // K9 maps table slots to ids itself (w.slot_rank); others need the ids
    const i64 K = dense_token_ids(c, tok, N, w.ids, w.ht_cap, w.ht_scratch, s, &w.dkeys, &w.dk_n, &w.dk_max,
                                  nullptr, w.rw != nullptr ? &w.slot_rank : nullptr);
    if (K >= 0) {
      w.ids_valid = true;
      w.K = K;
      packK = K;
      const int bt0 = bits_for(u64(K));
      const bool will_pack = !b.gen && b.W == 1 && w.rw == nullptr && b.sort_depth == 0 && 64 / bt0 >= 2;
      if (w.rw == nullptr && !will_pack) {
        // group start of a token = number of positions holding smaller tokens
        u32 *cnt = w.vals;  // K <= N counters, then exclusive starts in place
        APO_CUDA(cudaMemsetAsync(cnt, 0, sizeof(u32) * K, s));
        k_count_ids<<<G, T, 0, s>>>(w.ids, N, cnt);
        APO_CHECK_LAUNCH();
        ExclF ef{cnt};
        launch_scan<false>(c, K, ef, s);
        k_rank_from_ids<<<G, T, 0, s>>>(w.ids, N, cnt, w.levels[0]);
        APO_CHECK_LAUNCH();
        c.launches += 2;
      }
    }
  }
  if (!w.ids_valid) {
  k_init_pairs<<<G, T, 0, s>>>(tok, N, w.keys, w.vals);
  APO_CHECK_LAUNCH();
  c.launches++;
  bool alt = radix_sort_u64_u32(c, w.keys, w.vals, w.keys_alt, w.vals_alt, N, 0, 64, s);
  u64 *sk = alt ? w.keys_alt : w.keys;
  u32 *sv = alt ? w.vals_alt : w.vals;
  u64 *ok = alt ? w.keys : w.keys_alt;
  u32 *ov = alt ? w.vals : w.vals_alt;
  const u64 *tok_sorted = sk;
  if (b.W > 1 && !b.gen) {
    k_wid_keys<<<G, T, 0, s>>>(sv, b.wid, N, ok);
    APO_CHECK_LAUNCH();
    c.launches++;
    // copy values so the (key, value) pair lives in (ok, ov)
    c.d2d(ov, sv, sizeof(u32) * N, s);
    bool a2 = radix_sort_u64_u32(c, ok, ov, sk, sv, N, 0, bits_for(u64(b.W - 1)), s);
    u32 *idx = a2 ? sv : ov;
    k_gather_tok<<<G, T, 0, s>>>(idx, tok, N, w.tok_sorted);
    APO_CHECK_LAUNCH();
    c.launches++;
    tok_sorted = w.tok_sorted;
    sv = idx;
  }
  {
    InitRankF f{tok_sorted, sv, (b.W > 1 && !b.gen) ? b.wid : nullptr, w.levels[0]};
    launch_scan<true>(c, N, f, s);
  }
  }

  if (w.rw != nullptr) {
    // ---- K9: every window's suffix array and LCP array on chip ----
    run_window_sa(c, b, w, want_lcp, s);
    return;
  } else {
  // ---- K3: doubling rounds ----
  const int lob = b.gen ? bits_for(u64(N - 1) + u64(b.W)) : bits_for(u64(b.maxwin));
  const int hib = bits_for(u64(N - 1));
  if (lob + hib > 64) throw Error{APO_ERR_INVALID, "batch too large for 64-bit doubling keys"};
  u32 *notdone = reinterpret_cast<u32 *>(c.d_misc);
  const u32 *final_sa = nullptr;  // set by the first round (there is always one)
  int r = 0;
  i64 h0 = 1;
  bool done = false;
  // token packing for a single window with dense ids (C2, C3, C5): level 0
  // = ranks of the first q tokens
  const int bt = packK >= 0 ? bits_for(u64(packK)) : 64;
  const int q = 64 / bt;
  if (w.ids_valid && !b.gen && b.W == 1 && w.rw == nullptr && q >= 2 && b.sort_depth == 0) {
    APO_CUDA(cudaMemsetAsync(notdone, 0, sizeof(u32), s));
    k_pack_keys<<<G, T, 0, s>>>(w.ids, N, q, bt, w.keys, w.vals);
    APO_CHECK_LAUNCH();
    c.launches++;
    bool a = radix_sort_u64_u32(c, w.keys, w.vals, w.keys_alt, w.vals_alt, N, 0, q * bt, s);
    const u64 *key = a ? w.keys_alt : w.keys;
    const u32 *sa = a ? w.vals_alt : w.vals;
    DoubleRankF f{key, sa, w.levels[0], notdone};
    launch_scan<true>(c, N, f, s);
    final_sa = sa;
    w.unit = q;
    h0 = q;
    done = c.read_u32(notdone, s) == 0;
  }
  // Manber-Myers rounds go out in chunks with one host read per chunk: every
  // round after the first is gated on the previous round's "not done" word,
  // so the rounds after convergence return at once, and the chunk's words
  // tell which round finished.  APO_SPEC_ROUNDS rounds per chunk, default 2
  // (C3 2.84 -> 2.79 ms, C2 1.62 -> 1.56 ms; 4 and 8 lose more to the gated
  // launches at the end than they save in reads).
  const char *spec_s = getenv("APO_SPEC_ROUNDS");
  const int spec_v = spec_s != nullptr ? atoi(spec_s) : 0;
  const int spec_env = spec_v >= 1 && spec_v <= kSpecMax ? spec_v : 2;
  u32 *rflag = notdone + 16;  // kSpecMax words
  for (i64 h = h0; !done;) {
    if (r + 1 >= w.max_levels) throw Error{APO_ERR_INVALID, "prefix doubling exceeded its level budget"};
    const u64 *key;
    const u32 *sa;
    if (final_sa != nullptr && !b.gen && b.W == 1 && b.sort_depth == 0 && h < N) {
      // Manber-Myers round: keys listed in second-key order, sorted by the
      // first key's bits only (the pair not holding the previous SA)
      int nr = 1;
      while (nr < spec_env && (h << nr) < N && r + nr + 1 < w.max_levels) ++nr;
      APO_CUDA(cudaMemsetAsync(rflag, 0, sizeof(u32) * nr, s));
      const u32 *sa_of[kSpecMax];
      for (int j = 0; j < nr; ++j) {
        const u32 *gate = j == 0 ? nullptr : rflag + j - 1;
        const bool in_main = final_sa == w.vals;
        u64 *k0 = in_main ? w.keys_alt : w.keys, *k1 = in_main ? w.keys : w.keys_alt;
        u32 *v0 = in_main ? w.vals_alt : w.vals, *v1 = in_main ? w.vals : w.vals_alt;
        u32 *q0 = notdone + 1;
        k_pos_of_zero<<<G, T, 0, s>>>(final_sa, N, q0, gate);
        APO_CHECK_LAUNCH();
        k_mm_keys<<<G, T, 0, s>>>(final_sa, w.levels[r], N, h, lob, q0, k0, v0, gate);
        APO_CHECK_LAUNCH();
        c.launches += 2;
        bool a = radix_sort_u64_u32(c, k0, v0, k1, v1, N, lob, hib + lob, s, gate);
        key = a ? k1 : k0;
        sa = a ? v1 : v0;
        DoubleRankF f{key, sa, w.levels[r + 1], rflag + j};
        launch_scan<true>(c, N, f, s, gate);
        sa_of[j] = sa;
        final_sa = sa;
        ++r;
        h <<= 1;
      }
      u32 fl[kSpecMax];
      c.read_words(fl, rflag, nr, s);
      int last = nr - 1;
      for (int j = 0; j < nr; ++j)
        if (fl[j] == 0) {
          last = j;
          break;
        }
      r -= nr - 1 - last;  // the rounds after `last` returned at once
      final_sa = sa_of[last];
      done = fl[last] == 0;
      if (!done && (h >> 1) > b.maxwin) throw Error{APO_ERR_CUDA, "prefix doubling did not converge"};
      continue;
    }
    APO_CUDA(cudaMemsetAsync(notdone, 0, sizeof(u32), s));
    k_double_keys<<<G, T, 0, s>>>(w.levels[r], b, h, lob, w.keys, w.vals);
    APO_CHECK_LAUNCH();
    c.launches++;
    bool a = radix_sort_u64_u32(c, w.keys, w.vals, w.keys_alt, w.vals_alt, N, 0, hib + lob, s);
    key = a ? w.keys_alt : w.keys;
    sa = a ? w.vals_alt : w.vals;
    DoubleRankF f{key, sa, w.levels[r + 1], notdone};
    launch_scan<true>(c, N, f, s);
    ++r;
    final_sa = sa;
    if (c.read_u32(notdone, s) == 0) break;
    if (b.sort_depth > 0 && 2 * h >= b.sort_depth) break;  // ordered deeply enough
    if (h > b.maxwin) throw Error{APO_ERR_CUDA, "prefix doubling did not converge"};
    h <<= 1;
  }
  w.R = r;
  c.d2d(w.sa, final_sa, sizeof(i32) * N, s);
  }

  if (!want_lcp) return;
  // ---- K4: phi, PLCP, LCP ----
  const u32 *sa = reinterpret_cast<const u32 *>(w.sa);
  if (w.rw == nullptr) {  // the K9 path writes phi itself
    k_phi<<<G, T, 0, s>>>(sa, b, w.phi);
    APO_CHECK_LAUNCH();
  }
  Levels L{};
  for (int q = 0; q < w.max_levels && q < 40; ++q) L.p[q] = w.levels[q];
  i64 chunks = (N + kPlcpChunk - 1) / kPlcpChunk;
  // fully sorted per-window paths (K9, or K3 to the end): scatter directly
  const bool direct = !b.gen && b.sort_depth == 0;
  k_plcp<<<grid_for(chunks, 128), 128, 0, s>>>(tok, w.phi, L, w.R, w.unit, w.rw, b, w.plcp,
                                                 direct ? w.lcp : nullptr);
  APO_CHECK_LAUNCH();
  if (!direct) {
    k_lcp_gather<<<G, T, 0, s>>>(sa, w.plcp, b, w.lcp);
    APO_CHECK_LAUNCH();
  }
  c.launches += 3;
}

}  // namespace apo
