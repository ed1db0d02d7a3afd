// replay.cu -- REPLAY selection over MATCH_ALL hits (§8(f)2).
//
// Alg. 1 TraceReplayer: "Select one of the pending
// candidates to replay.  Execute any tasks before it, and issue a trace
// replay for the candidate" -- SelectReplayTrace(D, P, A), ExecuteAndReplay.
// Scoring (§4.3): "the length of the candidate trace multiplied by
// a count of the number of times the trace has appeared ... a maximum value
// of the count ... exponentially decay the value of the count by how many
// tasks have been encountered since the trace last appeared ... increase the
// score slightly if a trace has already been replayed."  Readings R20-R24
// fix what the paper leaves open; the constants are declared
// defaults (apo_replay_params).
//
// Streams are independent, and within a stream only the choice of replays is
// a left-to-right chain (a replay moves the frontier every later decision
// depends on).  Everything else is computed in parallel, so no stream's
// sequential walk touches more than the few chunks where a replay happens
// (a stream can hold a million hits: a one-warp walk over all of them was
// the whole kernel's critical path):
//   A (k_rp_local, CTA per part of 2,048 consecutive records of a stream):
//     a stable sort of the part's records by slot (the stream-local trace
//     key) gives each record its appearance count and previous end WITHIN
//     the part; per run of equal slots the part stores (slot, count, last
//     end);
//   B (k_rp_prefix, CTA per stream): walks the stream's parts in order with
//     a per-slot table (count so far, last end), replacing each run's
//     (count, last end) with the table's values before the part -- the state
//     the part starts from -- and updating the table;
//   C (k_rp_scores, CTA per part): the same sort again; per record
//     count = min(count before the part + count in the part, cap) and gap =
//     end - previous end (in the part, else before it), the score before the
//     bonus len x count x d_k (u64; d_k from a host table built with the
//     oracle's integer recurrence); per chunk of 32 records the latest start
//     (end - len + 1);
//   D (k_rp_decide, warp per stream): the decision walk.  A record is
//     eligible iff it starts at or after the frontier; a chunk whose latest
//     start is before the frontier is skipped with one ballot per 32 chunks.
//     In an eligible chunk the first eligible record marks the next end
//     where a replay happens; an end's records are in trace-id order (length
//     descending), so its eligible records are the rest of that end's run:
//     bonus (replayed bitset), arg-max (score, length, -id), merged with a
//     running best when the end continues into the next chunk; the replay
//     moves the frontier.
// Replays are staged per stream (at most one per stream position) and
// compacted in stream order after a scan of the per-stream counts.
#include <algorithm>
#include <vector>

#include <cstdlib>
#include "trie.cuh"

namespace apo {
namespace {

constexpr int kPart = 2048;                     // records per part
constexpr int kPartThreads = 256;               // 8 warps
constexpr int kPartItems = kPart / kPartThreads;
constexpr int kPartWarps = kPartThreads / 32;
constexpr int kChunksPerPart = kPart / 32;
constexpr int kMaxDigit = 9;                    // slot sort digits <= 9 bits
constexpr int kPrefixThreads = 512;
constexpr int kStateBytesMax = 192 * 1024;      // phase B per-stream table on chip up to here

struct RP {
  const int4 *hits;
  const i64 *tlen_off;   // trace offsets (T+1): len(t) = off[t+1] - off[t]
  const u32 *dq;         // decay table d_k, k < ndq
  int ndq;
  int count_cap, period;
  double inv_period;     // 1 / period (the quotient is corrected to the exact one)
  u32 bonus_num, bonus_den;
  int nstreams;
  int slot_bits;         // slots < 2^slot_bits
  const i64 *hbeg;       // per stream: first hit (nstreams + 1)
  const i64 *pbeg;       // per stream: first part (nstreams + 1)
  const int *pstream;    // per part: its stream
  u32 *maxslot;          // per stream: max slot + 1 (phase A)
  u32 *run_slot;         // per part, per run (slot order): slot
  u32 *run_cnt;          // A: records of the run; B: count before the part (saturated)
  i32 *run_last;         // A: last end in the run; B: last end before the part (-1: none)
  u32 *nruns;            // per part
  u64 *sc;               // per record: score before the bonus
  i32 *cmax;             // per part, per chunk: latest start (-1: empty)
  const int *order;      // phase D: block -> stream (streams with the most hits first)
  void *gstate;          // phase B/D global fallback tables
  const i64 *gstate_off; // per stream offset (u32 words) into gstate (nstreams + 1)
  u32 on_chip_slots;     // phase B: streams with maxslot above this use gstate
  u32 on_chip_bits;      // phase D: bitsets above this many words use gstate
  const i64 *soff;       // per stream staging offset (stream position base)
  int4 *stage;           // staged replays
  u32 *rcnt;             // per stream replay count
  // matcher index (apo_match mode 1, on-chip path): see ReplayIndex
  const i64 *ix_off;
  const i32 *ix_sa;
  const u64 *ix_tkey;
  const u32 *ix_toff;
  const int *wq;         // wavelet work items: stream
  const i64 *wr0;        // wavelet work items: first record (nitems + 1 ends)
  struct WvMat *wv;      // per stream: its wavelet matrix (lazy scores in phase D)
  const u32 *endoff;     // per stream position: first hit record (mode 1, from the emitter)
  const unsigned short *endml;  // per stream position: shortest trace ending there (0xffff: none)
  // phase D by ends: per decision its winner (single eligible record) or its
  // staged candidates; the candidate pool and its fill counter
  uint2 *dwin = nullptr;
  struct RpCand *cand = nullptr;
  i64 ccap = 0;
  unsigned long long *ccnt = nullptr;
  u32 *pend = nullptr;                 // candidates left for the wavelet queries
  unsigned long long *pcnt = nullptr;
  unsigned char *need_wv = nullptr;    // per stream: build its wavelet matrix
  u32 scan_max = 0;                    // longest occurrence range scored by a scan
  // lazy MATCH_ALL (ReplayIndex::lazy): endoff = 1 + deepest interval per
  // end; an end's records are its chain of parents (ids local to ix_toff[q])
  bool lazy = false;
  const u32 *opar = nullptr, *otr = nullptr, *odep = nullptr;
};

__device__ __forceinline__ u32 lanemask_lt_() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per stream: its hit range from the matcher's per-stream hit bases (lazy
// MATCH_ALL: no records to search).
__global__ void k_replay_ranges_q(const u32 *__restrict__ qbase, i64 nhits, int nstreams, i64 *__restrict__ hbeg) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q <= nstreams) hbeg[q] = q < nstreams ? i64(qbase[q]) : nhits;
}

// Per stream: its hit range (hits sorted by stream).
__global__ void k_replay_ranges(const int4 *__restrict__ hits, i64 nhits, int nstreams, i64 *__restrict__ hbeg) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q > nstreams) return;
  i64 lo = 0, hi = nhits;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (__ldg(&hits[mid].x) < q)
      lo = mid + 1;
    else
      hi = mid;
  }
  hbeg[q] = lo;
}

// ---------------------------------------------------------------------------
// The part's records sorted by slot (stable): 8 warps x 256 records, LSD
// passes of up to 9 bits with match.any peer masks into per-warp u16 digit
// counts.  On return sk[k] / sv[k] hold the k-th record's slot / part-local
// index in (slot, index) order (pads: slot 0xffffffff at the end).
struct PartSmem {
  u32 ka[kPart], kb[kPart];
  unsigned short va[kPart], vb[kPart];
  i32 end[kPart];
  u32 len[kPart];
  unsigned short hist[kPartWarps][1 << kMaxDigit];
  u32 start[1 << kMaxDigit];
  u32 wsum[kPartWarps];
  u32 wmax[kPartWarps];
};

template <int BITS>
__device__ void part_pass(PartSmem &S, const u32 *kin, const unsigned short *vin, u32 *kout, unsigned short *vout,
                          int shift) {
  constexpr int RADIX = 1 << BITS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned short *wh = S.hist[warp];
  for (int i = lane; i < RADIX; i += 32) wh[i] = 0;
  __syncwarp();
  const u32 lt = lanemask_lt_();
  u32 rk[kPartItems];
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int q = warp * (32 * kPartItems) + j * 32 + lane;
    const u32 d = (kin[q] >> shift) & u32(RADIX - 1);
    const u32 peers = __match_any_sync(0xffffffffu, d);
    const u32 old = wh[d];
    __syncwarp();
    if (lane == __ffs(peers) - 1) wh[d] = (unsigned short)(old + __popc(peers));
    __syncwarp();
    rk[j] = old + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (in place), digit totals
  for (int d = tid; d < RADIX; d += kPartThreads) {
    u32 t = 0;
#pragma unroll
    for (int w = 0; w < kPartWarps; ++w) {
      const u32 c = S.hist[w][d];
      S.hist[w][d] = (unsigned short)t;
      t += c;
    }
    S.start[d] = t;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the digit totals
    u32 carry = 0;
    for (int d0 = 0; d0 < RADIX; d0 += 32) {
      const u32 v = d0 + lane < RADIX ? S.start[d0 + lane] : 0u;
      u32 x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (d0 + lane < RADIX) S.start[d0 + lane] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int q = warp * (32 * kPartItems) + j * 32 + lane;
    const u32 d = (kin[q] >> shift) & u32(RADIX - 1);
    const u32 to = S.start[d] + wh[d] + rk[j];
    kout[to] = kin[q];
    vout[to] = vin[q];
  }
  __syncthreads();
}

__device__ void part_pass_bits(int bits, PartSmem &S, const u32 *kin, const unsigned short *vin, u32 *kout,
                               unsigned short *vout, int shift) {
  switch (bits) {
    case 1: part_pass<1>(S, kin, vin, kout, vout, shift); break;
    case 2: part_pass<2>(S, kin, vin, kout, vout, shift); break;
    case 3: part_pass<3>(S, kin, vin, kout, vout, shift); break;
    case 4: part_pass<4>(S, kin, vin, kout, vout, shift); break;
    case 5: part_pass<5>(S, kin, vin, kout, vout, shift); break;
    case 6: part_pass<6>(S, kin, vin, kout, vout, shift); break;
    case 7: part_pass<7>(S, kin, vin, kout, vout, shift); break;
    case 8: part_pass<8>(S, kin, vin, kout, vout, shift); break;
    default: part_pass<9>(S, kin, vin, kout, vout, shift); break;
  }
}

// Loads part p's records (slots, ends, trace lengths) and sorts them by slot.
// Returns (first record, record count); sorted keys/indices in (*sk, *sv).
__device__ void part_load_sort(const RP &a, PartSmem &S, i64 p, i64 &r0, int &m, const u32 *&sk,
                               const unsigned short *&sv, bool want_len) {
  const int q = a.pstream[p];
  r0 = a.hbeg[q] + (p - a.pbeg[q]) * kPart;
  m = int(min(i64(kPart), a.hbeg[q + 1] - r0));
  for (int i = threadIdx.x; i < kPart; i += kPartThreads) {
    if (i < m) {
      const int4 r = a.hits[r0 + i];
      S.ka[i] = u32(r.w);
      S.end[i] = r.y;
      if (want_len) S.len[i] = u32(__ldg(&a.tlen_off[r.z + 1]) - __ldg(&a.tlen_off[r.z]));
    } else {
      S.ka[i] = 0xffffffffu;  // pads sort last
    }
    S.va[i] = (unsigned short)i;
  }
  __syncthreads();
  const int np = (a.slot_bits + kMaxDigit - 1) / kMaxDigit;
  const int bpp = (a.slot_bits + np - 1) / np;
  u32 *ks = S.ka, *kd = S.kb;
  unsigned short *vs = S.va, *vd = S.vb;
  for (int k = 0; k < np; ++k) {
    part_pass_bits(bpp, S, ks, vs, kd, vd, k * bpp);
    u32 *t = ks; ks = kd; kd = t;
    unsigned short *tv = vs; vs = vd; vd = tv;
  }
  sk = ks;
  sv = vs;
}

// Run structure of the sorted part: thread t owns sorted positions
// [8t, 8t + 8).  For each: run id (number of run heads before it), run start.
__device__ void part_runs(PartSmem &S, const u32 *sk, int m, int (&rid)[kPartItems], int (&rst)[kPartItems],
                          int &nruns) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k0 = tid * kPartItems;
  int heads = 0, lastpos = -1;
  bool hd[kPartItems];
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int k = k0 + j;
    hd[j] = k < m && (k == 0 || sk[k] != sk[k - 1]);
    heads += hd[j];
    if (hd[j]) lastpos = k;
  }
  // block exclusive sum of heads and exclusive max of the last head position
  int hs = heads, hm = lastpos;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, hs, o), z = __shfl_up_sync(0xffffffffu, hm, o);
    if (lane >= o) {
      hs += y;
      hm = max(hm, z);
    }
  }
  if (lane == 31) {
    S.wsum[warp] = u32(hs);
    S.wmax[warp] = u32(hm + 1);
  }
  __syncthreads();
  int bs = 0, bm = -1;
  for (int w = 0; w < warp; ++w) {
    bs += int(S.wsum[w]);
    bm = max(bm, int(S.wmax[w]) - 1);
  }
  const int ex_s = bs + hs - heads;
  const int up = __shfl_up_sync(0xffffffffu, hm, 1);
  const int ex_m = lane == 0 ? bm : max(bm, up);
  int cur = ex_m, cnt = ex_s;
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    if (hd[j]) {
      cur = k0 + j;
      ++cnt;
    }
    rst[j] = cur;
    rid[j] = cnt - 1;
  }
  nruns = 0;
  for (int w = 0; w < kPartWarps; ++w) nruns += int(S.wsum[w]);
  __syncthreads();
}

// Phase A: per part, runs of equal slots (slot, records, last end).
__global__ void __launch_bounds__(kPartThreads) k_rp_local(RP a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  PartSmem &S = *reinterpret_cast<PartSmem *>(smraw);
  const i64 p = blockIdx.x;
  i64 r0;
  int m;
  const u32 *sk;
  const unsigned short *sv;
  part_load_sort(a, S, p, r0, m, sk, sv, false);
  int rid[kPartItems], rst[kPartItems], nr;
  part_runs(S, sk, m, rid, rst, nr);
  const int k0 = threadIdx.x * kPartItems;
  const i64 rb = p * kPart;
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int k = k0 + j;
    if (k >= m) break;
    const bool last = k + 1 == m || sk[k + 1] != sk[k];
    if (last) {
      a.run_slot[rb + rid[j]] = sk[k];
      a.run_cnt[rb + rid[j]] = u32(k - rst[j] + 1);
      a.run_last[rb + rid[j]] = S.end[sv[k]];
    }
  }
  if (threadIdx.x == 0) {
    a.nruns[p] = u32(nr);
    if (m > 0) atomicMax(&a.maxslot[a.pstream[p]], sk[m - 1] + 1u);
  }
}

// Phase B: per stream, the state each part starts from.
__global__ void __launch_bounds__(kPrefixThreads) k_rp_prefix(RP a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int q = blockIdx.x;
  const u32 ms = a.maxslot[q];
  const bool onchip = ms <= a.on_chip_slots;
  u32 *cnt = onchip ? reinterpret_cast<u32 *>(smraw) : static_cast<u32 *>(a.gstate) + a.gstate_off[q];
  i32 *last = reinterpret_cast<i32 *>(cnt + ms);
  for (u32 i = threadIdx.x; i < ms; i += kPrefixThreads) {
    cnt[i] = 0;
    last[i] = -1;
  }
  __syncthreads();
  for (i64 p = a.pbeg[q]; p < a.pbeg[q + 1]; ++p) {
    const u32 nr = a.nruns[p];
    const i64 rb = p * kPart;
    for (u32 r = threadIdx.x; r < nr; r += kPrefixThreads) {  // runs of a part have distinct slots
      const u32 z = a.run_slot[rb + r];
      const u32 c0 = cnt[z];
      const i32 l0 = last[z];
      const u32 cr = a.run_cnt[rb + r];
      const i32 lr = a.run_last[rb + r];
      a.run_cnt[rb + r] = c0;
      a.run_last[rb + r] = l0;
      cnt[z] = min(c0 + cr, u32(a.count_cap));
      last[z] = lr;
    }
    __syncthreads();
  }
}

// Phase C: scores before the bonus, per chunk the latest start.
__global__ void __launch_bounds__(kPartThreads) k_rp_scores(RP a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  PartSmem &S = *reinterpret_cast<PartSmem *>(smraw);
  const i64 p = blockIdx.x;
  i64 r0;
  int m;
  const u32 *sk;
  const unsigned short *sv;
  part_load_sort(a, S, p, r0, m, sk, sv, true);
  int rid[kPartItems], rst[kPartItems], nr;
  part_runs(S, sk, m, rid, rst, nr);
  const int k0 = threadIdx.x * kPartItems;
  const i64 rb = p * kPart;
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int k = k0 + j;
    if (k >= m) break;
    const int i = sv[k];
    const u32 c = min(a.run_cnt[rb + rid[j]] + u32(k - rst[j] + 1), u32(a.count_cap));
    const i32 prev = k > rst[j] ? S.end[sv[k - 1]] : a.run_last[rb + rid[j]];
    const u32 gap = prev >= 0 ? u32(S.end[i] - prev) : 0u;
    // gap / period by a reciprocal, corrected to the exact quotient
    u32 kk = u32(double(gap) * a.inv_period);
    if (u64(kk) * u64(a.period) > u64(gap)) --kk;
    if (u64(kk + 1u) * u64(a.period) <= u64(gap)) ++kk;
    const u64 d = __ldg(&a.dq[kk < u32(a.ndq) ? kk : u32(a.ndq - 1)]);
    a.sc[r0 + i] = u64(S.len[i]) * u64(c) * d;
  }
  // per chunk of 32 records (original order): the latest start
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int ch = warp; ch < kChunksPerPart; ch += kPartWarps) {
    const int i = ch * 32 + lane;
    const int st = i < m ? S.end[i] - int(S.len[i]) + 1 : -1;
    const int mx = __reduce_max_sync(0xffffffffu, st);
    if (lane == 0) a.cmax[p * kChunksPerPart + ch] = mx;
  }
}

// ---------------------------------------------------------------------------
// Phases A-C from the matcher's index (apo_match mode 1, streams matched on
// chip).  A hit (e, z) is an occurrence of slot z's trace ending at e; the
// trace's occurrences are the ranks [lo_z, hi_z) of z's interval in the
// REVERSED stream's suffix array, ending at E[r] = n - 1 - SA_rev[r].  So
//   count(z, e) = #{r in [lo_z, hi_z) : E[r] <= e}   (appearances so far),
//   prev(z, e)  = the (count - 1)-th smallest E[r] in the range (1-based),
// two wavelet-matrix queries over E (14 levels for n <= 16,384; one matrix
// per stream, built in shared memory by k_rp_wvbuild and stored).  The
// decisions only ever look at the eligible records of the ends where a
// replay happens, so phase D evaluates exactly those scores (wv_score) and
// nothing is computed for the other ~99 % of the hits; k_rp_cmax gives the
// per-chunk latest starts the decision walk skips by.
constexpr int kWvThreads = 1024;
constexpr int kWvMaxN = 16384;
constexpr int kWvLevels = 14;
constexpr int kWvWords = kWvMaxN / 32 + 1;
constexpr i64 kWvPart = 65536;  // records per work item (a multiple of kPart)

struct WvSmem {
  u32 bits[kWvLevels][kWvWords];
  unsigned short pre[kWvLevels][kWvWords];  // ones before each word
  u32 zeros[kWvLevels];
  unsigned short cur[kWvMaxN], nxt[kWvMaxN];
  u32 wtot[kWvThreads / 32];
};

__device__ __forceinline__ u32 wv_rank1(const WvSmem &S, int l, u32 i) {
  const u32 w = i >> 5, b = i & 31u;
  return u32(S.pre[l][w]) + __popc(S.bits[l][w] & ((1u << b) - 1u));
}

// The matrix of one stream in global memory, (bits, ones before) per word
// interleaved so a rank is one 8-byte load: phase D evaluates the scores of
// the few records it examines (eligible records at decision ends) from it.
struct WvMat {
  uint2 bp[kWvLevels][kWvWords];
  u32 zeros[kWvLevels];
  int L;
};

__device__ __forceinline__ u32 wvg_rank1(const WvMat *M, int l, u32 i) {
  const uint2 v = __ldg(&M->bp[l][i >> 5]);
  return v.y + __popc(v.x & ((1u << (i & 31u)) - 1u));
}

// Score before the bonus from the appearance count and the gap since the
// previous appearance (R20-R22): len * min(count, cap) * d_k, k = gap / period.
__device__ __forceinline__ u64 score_of(const RP &a, u32 cnt, u32 gap, u32 len) {
  const u32 c = min(cnt, u32(a.count_cap));
  u32 kq = u32(double(gap) * a.inv_period);
  if (u64(kq) * u64(a.period) > u64(gap)) --kq;
  if (u64(kq + 1u) * u64(a.period) <= u64(gap)) ++kq;
  const u64 d = __ldg(&a.dq[kq < u32(a.ndq) ? kq : u32(a.ndq - 1)]);
  return u64(len) * u64(c) * d;
}

// Score before the bonus of hit `rec` (trace length len) of stream q:
// count = #{E[r] <= e in [lo, hi)}, previous end = the (count - 1)-th
// smallest E in the range (1-based).
__device__ u64 wv_score(const RP &a, int q, int4 rec, u32 len) {
  const WvMat *M = a.wv + q;
  const int L = M->L;
  const u64 kk = __ldg(&a.ix_tkey[a.ix_toff[q] + rec.w]);
  const u32 lo = u32(kk >> 15) & 32767u, hi = 32767u - (u32(kk) & 32767u);
  const u32 e = u32(rec.y);
  u32 cnt = 0;
  const u32 x = e + 1u;
  if (x >= (1u << L)) {
    cnt = hi - lo;
  } else {
    u32 l0 = lo, h0 = hi;
    for (int l = L - 1; l >= 0; --l) {
      const u32 a1 = wvg_rank1(M, l, l0), b1 = wvg_rank1(M, l, h0);
      const u32 Z = __ldg(&M->zeros[l]);
      if ((x >> l) & 1u) {
        cnt += (h0 - l0) - (b1 - a1);
        l0 = Z + a1;
        h0 = Z + b1;
      } else {
        l0 -= a1;
        h0 -= b1;
      }
    }
  }
  u32 gap = 0;
  if (cnt >= 2) {
    u32 kq = cnt - 2, v = 0, l0 = lo, h0 = hi;
    for (int l = L - 1; l >= 0; --l) {
      const u32 a1 = wvg_rank1(M, l, l0), b1 = wvg_rank1(M, l, h0);
      const u32 Z = __ldg(&M->zeros[l]);
      const u32 zc = (h0 - l0) - (b1 - a1);
      if (kq < zc) {
        l0 -= a1;
        h0 -= b1;
      } else {
        kq -= zc;
        v |= 1u << l;
        l0 = Z + a1;
        h0 = Z + b1;
      }
    }
    gap = e - v;
  }
  return score_of(a, cnt, gap, len);
}

// Builds every stream's matrix in shared memory (ballots + stable
// partitions), then stores it to the stream's WvMat.
__global__ void __launch_bounds__(kWvThreads) k_rp_wvbuild(RP a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  WvSmem &S = *reinterpret_cast<WvSmem *>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x;
  const i64 beg = a.ix_off[q];
  const int n = int(a.ix_off[q + 1] - beg);
  if (tid == 0) a.maxslot[q] = a.ix_toff[q + 1] - a.ix_toff[q];
  if (a.hbeg[q] == a.hbeg[q + 1] || n == 0) return;  // no hits: no scores needed
  if (a.need_wv != nullptr && !a.need_wv[q]) return;  // by ends: no wavelet query in this stream
  const int L = max(1, 32 - __clz(u32(max(n - 1, 1))));
  const int nw = (n + 31) / 32;
  for (int r = tid; r < n; r += kWvThreads) S.cur[r] = (unsigned short)(n - 1 - (a.ix_sa[beg + r] - int(beg)));
  __syncthreads();
  unsigned short *cur = S.cur, *nxt = S.nxt;
  WvMat *M = a.wv + q;
  for (int l = L - 1; l >= 0; --l) {
    for (int w = warp; w <= nw; w += kWvThreads / 32) {
      const int i = w * 32 + lane;
      const u32 m = __ballot_sync(0xffffffffu, i < n && ((cur[i] >> l) & 1u));
      if (lane == 0) S.bits[l][w] = m;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive prefix of the ones per word, total zeros
      u32 carry = 0;
      for (int w0 = 0; w0 <= nw; w0 += 32) {
        const u32 v = w0 + lane <= nw ? u32(__popc(S.bits[l][w0 + lane])) : 0u;
        u32 x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (w0 + lane <= nw) S.pre[l][w0 + lane] = (unsigned short)(carry + x - v);
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) {
        S.zeros[l] = u32(n) - carry;
        M->zeros[l] = u32(n) - carry;
      }
    }
    __syncthreads();
    for (int w = tid; w <= nw; w += kWvThreads) M->bp[l][w] = make_uint2(S.bits[l][w], u32(S.pre[l][w]));
    if (l > 0) {  // stable partition for the next level: zeros, then ones
      const u32 Z = S.zeros[l];
      for (int i = tid; i < n; i += kWvThreads) {
        const u32 r1 = wv_rank1(S, l, u32(i));
        const bool b = (cur[i] >> l) & 1u;
        nxt[b ? Z + r1 : u32(i) - r1] = cur[i];
      }
      __syncthreads();
      unsigned short *t = cur; cur = nxt; nxt = t;
    }
  }
  if (tid == 0) M->L = L;
}

// Per chunk of 32 records (stream-aligned): the latest start end - len + 1.
__global__ void __launch_bounds__(256) k_rp_cmax(RP a) {
  const int lane = threadIdx.x & 31;
  const int q = a.wq[blockIdx.x];
  const i64 r0 = a.wr0[blockIdx.x], r1 = a.wr0[blockIdx.x + 1];
  const i64 hb = a.hbeg[q], p0 = a.pbeg[q];
  for (i64 kb = r0 + i64(threadIdx.x >> 5) * 32; kb < r1; kb += 256) {
    const i64 k = kb + lane;
    int st = -1;
    if (k < r1) {
      const int4 rec = a.hits[k];
      st = rec.y - int(__ldg(&a.tlen_off[rec.z + 1]) - __ldg(&a.tlen_off[rec.z])) + 1;
    }
    const int mx = __reduce_max_sync(0xffffffffu, st);
    if (lane == 0) {
      const i64 ch = (kb - hb) / 32;
      a.cmax[(p0 + ch / kChunksPerPart) * kChunksPerPart + ch % kChunksPerPart] = mx;
    }
  }
}

// (score, len, -id) order: true iff a beats b
__device__ __forceinline__ bool beats(u64 sa, u32 la, u32 ta, u64 sb, u32 lb, u32 tb) {
  if (sa != sb) return sa > sb;
  if (la != lb) return la > lb;
  return ta < tb;
}

// Warp arg-max of (score, len, -id) over the lanes with ok set: four warp
// reductions (redux.sync); returns the winning lane (-1 if no lane is ok).
__device__ __forceinline__ int warp_best(bool ok, u64 sc, u32 L, u32 t) {
  const u32 any = __ballot_sync(0xffffffffu, ok);
  if (!any) return -1;
  u32 c = any;
  const u32 hi = __reduce_max_sync(0xffffffffu, ok ? u32(sc >> 32) : 0u);
  c &= __ballot_sync(0xffffffffu, u32(sc >> 32) == hi);
  const bool in1 = (c >> (threadIdx.x & 31)) & 1u;
  const u32 lo = __reduce_max_sync(0xffffffffu, in1 ? u32(sc) : 0u);
  c &= __ballot_sync(0xffffffffu, u32(sc) == lo);
  const bool in2 = (c >> (threadIdx.x & 31)) & 1u;
  const u32 ml = __reduce_max_sync(0xffffffffu, in2 ? L : 0u);
  c &= __ballot_sync(0xffffffffu, L == ml);
  const bool in3 = (c >> (threadIdx.x & 31)) & 1u;
  const u32 mt = __reduce_min_sync(0xffffffffu, in3 ? t : 0xffffffffu);
  c &= __ballot_sync(0xffffffffu, t == mt);
  return __ffs(c) - 1;
}

// Phase D: one warp per stream, the decisions.
__global__ void __launch_bounds__(32) k_rp_decide(RP a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int q = a.order[blockIdx.x], lane = threadIdx.x;
  const i64 hb = a.hbeg[q], he = a.hbeg[q + 1];
  const u32 nw = (a.maxslot[q] + 31) / 32;
  u32 *rep = nw <= a.on_chip_bits ? reinterpret_cast<u32 *>(smraw) : static_cast<u32 *>(a.gstate) + a.gstate_off[q];
  for (u32 i = lane; i < nw; i += 32) rep[i] = 0u;
  __syncwarp();
  i64 frontier = 0;
  u32 nrep = 0;
  int4 *stage = a.stage + a.soff[q];
  bool have = false;
  int carry_e = -1;
  u64 bs = 0;
  u32 bl = 0, bt = 0, bslot = 0;
  auto commit = [&](int e0) {
    __syncwarp();
    if (lane == 0) {
      const u32 mk = 1u << (bslot & 31);
      const u32 old = rep[bslot >> 5];
      stage[nrep] = make_int4(q, e0, int(bt), (old & mk) ? 0 : 1);
      rep[bslot >> 5] = old | mk;
    }
    __syncwarp();
    ++nrep;
    frontier = i64(e0) + 1;
    have = false;
  };
  const i64 nch = (he - hb + 31) / 32;
  const i64 p0 = a.pbeg[q];
  for (i64 c0 = 0; c0 < nch; c0 += 32) {
    const i64 c = c0 + lane;
    const int mx = c < nch ? a.cmax[(p0 + c / kChunksPerPart) * kChunksPerPart + c % kChunksPerPart] : -1;
    u32 pend = __ballot_sync(0xffffffffu, c < nch);
    while (pend) {
      // next chunk with a record starting at or after the frontier
      const u32 cand = pend & __ballot_sync(0xffffffffu, i64(mx) >= frontier);
      const int l = cand ? __ffs(cand) - 1 : 32;
      // a carried end does not continue into a skipped chunk: decide it
      if (have && (l == 32 || l != __ffs(pend) - 1)) commit(carry_e);
      if (l == 32) break;
      pend &= ~((2u << l) - 1u);
      // the chunk's records
      const i64 k = hb + (c0 + l) * 32 + lane;
      const bool valid = k < he;
      int4 r = make_int4(-1, -1, -1, 0);
      u64 sc0 = 0;
      u32 L = 0;
      if (valid) {
        r = a.hits[k];
        if (a.wv == nullptr) sc0 = a.sc[k];
        L = u32(__ldg(&a.tlen_off[r.z + 1]) - __ldg(&a.tlen_off[r.z]));
      }
      if (have && __shfl_sync(0xffffffffu, r.y, 0) != carry_e) commit(carry_e);
      const u32 slot = u32(r.w);
      u32 done = 0;
      for (;;) {
        const bool elig = valid && !((done >> lane) & 1u) && i64(r.y) - i64(L) + 1 >= frontier;
        const u32 em = __ballot_sync(0xffffffffu, elig);
        if (!em) break;
        const int a0 = __ffs(em) - 1;
        const int e0 = __shfl_sync(0xffffffffu, r.y, a0);
        const bool run = valid && r.y == e0;
        const u32 rm = __ballot_sync(0xffffffffu, run);
        const int a1 = 32 - __clz(rm);
        const bool ok = elig && run;
        u64 sc = sc0;
        if (ok && a.wv != nullptr) sc = wv_score(a, q, r, L);  // lazily: only examined records
        if (ok && ((rep[slot >> 5] >> (slot & 31)) & 1u)) sc = sc * a.bonus_num / a.bonus_den;
        const int b = warp_best(ok, sc, L, u32(r.z));
        if (b >= 0) {
          const u64 s1 = __shfl_sync(0xffffffffu, sc, b);
          const u32 l1 = __shfl_sync(0xffffffffu, L, b), t1 = __shfl_sync(0xffffffffu, u32(r.z), b);
          const u32 z1 = __shfl_sync(0xffffffffu, slot, b);
          if (!have || beats(s1, l1, t1, bs, bl, bt)) {
            bs = s1;
            bl = l1;
            bt = t1;
            bslot = z1;
            have = true;
          }
        }
        done |= rm | ((1u << a1) - 1u);
        if (a1 == 32) {  // the end may continue into the next chunk
          carry_e = e0;
          break;
        }
        commit(e0);
      }
    }
  }
  if (have) commit(carry_e);
  if (lane == 0) a.rcnt[q] = nrep;
}

// Phase D by ends (mode 1 with the emitter's per-end index).  Which ends are
// decided does not depend on any score: an end is decided iff its shortest
// trace starts at or after the frontier (e - minlen + 1 >= frontier), and a
// replay at e moves the frontier to e + 1 whichever record wins.  So the
// phase runs in three kernels:
//  * k_rp_dec_find (warp per stream): the decision ends and the frontier each
//    was decided under, from the shortest-length column alone (register
//    ballots over 32 ends at a time; no record is read);
//  * k_rp_dec_cands (all decisions in parallel): the eligible records of a
//    decision are a suffix of its end's run (trace-id order = length
//    descending); ~90 % of the decisions have exactly one, which wins without
//    a score; the others get their scores evaluated (wavelet queries; scores
//    do not depend on earlier decisions) and staged in a candidate pool;
//  * k_rp_dec_pick (warp per stream): the winners in end order -- only the
//    bonus depends on the slots replayed so far -- and the replay records.
// A decision whose candidates do not fit the pool is decided by the whole
// warp in k_rp_dec_pick (rp_decide_end, scores evaluated there).
struct RpCand {
  u64 sc;
  u32 len, t, slot, q, e, pad;
};
constexpr u32 kScanMax = 4096;  // occurrence ranges up to this are scanned, longer ones queried (default)
constexpr u32 kDecMulti = 0x80000000u;  // dwin.x flag: (count, pool offset) follow
constexpr u32 kDecOver = 0xffffffffu;   // dwin.x: candidates not staged
constexpr u32 kNoParR = 0xffffffffu;    // no parent (the matcher's kNoPar)

// One decision at end ed (frontier fr) with the whole warp: the best
// eligible record (score with the bonus, then length, then smaller id).
__device__ void rp_decide_end(const RP &a, int q, i64 beg, i64 he, int n, const u32 *rep, int ed, i64 fr,
                              u32 *bt_out, u32 *bslot_out) {
  const int lane = threadIdx.x & 31;
  if (a.lazy) {  // the end's chain, 32 links at a time (lane i takes the i-th)
    const u32 a0 = a.ix_toff[q];
    u32 z = a.endoff[beg + ed] - 1u;
    bool have = false;
    u64 bs = 0;
    u32 bl = 0, bt = 0, bslot = 0;
    while (z != kNoParR) {
      u32 mine = kNoParR;
      for (int i = 0; i < 32 && z != kNoParR; ++i) {
        if (lane == i) mine = z;
        z = __ldg(&a.opar[a0 + z]);
      }
      const bool valid = mine != kNoParR;
      u32 L = 0, t = 0;
      if (valid) {
        t = __ldg(&a.otr[a0 + mine]);
        L = u32(__ldg(&a.tlen_off[t + 1]) - __ldg(&a.tlen_off[t]));
      }
      const bool ok = valid && i64(ed) - i64(L) + 1 >= fr;
      u64 sc = 0;
      if (ok) {
        sc = wv_score(a, q, make_int4(q, ed, int(t), int(mine)), L);
        if ((rep[mine >> 5] >> (mine & 31)) & 1u) sc = sc * a.bonus_num / a.bonus_den;
      }
      const int b = warp_best(ok, sc, L, t);
      if (b >= 0) {
        const u64 s1 = __shfl_sync(0xffffffffu, sc, b);
        const u32 l1 = __shfl_sync(0xffffffffu, L, b), t1 = __shfl_sync(0xffffffffu, t, b);
        const u32 z1 = __shfl_sync(0xffffffffu, mine, b);
        if (!have || beats(s1, l1, t1, bs, bl, bt)) {
          bs = s1;
          bl = l1;
          bt = t1;
          bslot = z1;
          have = true;
        }
      }
    }
    *bt_out = bt;
    *bslot_out = bslot;
    return;
  }
  const i64 r0 = a.endoff[beg + ed];
  const i64 r1 = ed + 1 < n ? i64(a.endoff[beg + ed + 1]) : he;
  bool have = false;
  u64 bs = 0;
  u32 bl = 0, bt = 0, bslot = 0;
  for (i64 k0 = r0; k0 < r1; k0 += 32) {
    const i64 k = k0 + lane;
    const bool valid = k < r1;
    int4 r = make_int4(-1, -1, -1, 0);
    u32 L = 0;
    if (valid) {
      r = a.hits[k];
      L = u32(__ldg(&a.tlen_off[r.z + 1]) - __ldg(&a.tlen_off[r.z]));
    }
    const bool ok = valid && i64(ed) - i64(L) + 1 >= fr;
    const u32 slot = u32(r.w);
    u64 sc = 0;
    if (ok) {
      sc = wv_score(a, q, r, L);
      if ((rep[slot >> 5] >> (slot & 31)) & 1u) sc = sc * a.bonus_num / a.bonus_den;
    }
    const int b = warp_best(ok, sc, L, u32(r.z));
    if (b >= 0) {
      const u64 s1 = __shfl_sync(0xffffffffu, sc, b);
      const u32 l1 = __shfl_sync(0xffffffffu, L, b), t1 = __shfl_sync(0xffffffffu, u32(r.z), b);
      const u32 z1 = __shfl_sync(0xffffffffu, slot, b);
      if (!have || beats(s1, l1, t1, bs, bl, bt)) {
        bs = s1;
        bl = l1;
        bt = t1;
        bslot = z1;
        have = true;
      }
    }
  }
  *bt_out = bt;
  *bslot_out = bslot;
}

constexpr int kFindWarps = 4;

__global__ void __launch_bounds__(kFindWarps * 32) k_rp_dec_find(RP a) {
  const int lane = threadIdx.x & 31;
  const int qi = blockIdx.x * kFindWarps + (threadIdx.x >> 5);
  if (qi >= a.nstreams) return;
  const int q = a.order[qi];
  const i64 hb = a.hbeg[q], he = a.hbeg[q + 1];
  u32 nrep = 0;
  if (hb < he) {
    const i64 beg = a.ix_off[q];
    const int n = int(a.ix_off[q + 1] - beg);
    int4 *stage = a.stage + a.soff[q];
    i64 frontier = 0;
    u32 mln = lane < n ? u32(a.endml[beg + lane]) : 0xffffu;
    for (int e0 = 0; e0 < n; e0 += 32) {
      const int e = e0 + lane;
      const u32 ml = mln;
      mln = e + 32 < n ? u32(a.endml[beg + e + 32]) : 0xffffu;  // next window, in flight meanwhile
      u32 dm = 0, pend = __ballot_sync(0xffffffffu, ml != 0xffffu);
      i64 f = frontier;
      while (pend) {
        const u32 cm = pend & __ballot_sync(0xffffffffu, i64(e) - i64(ml) + 1 >= f);
        if (!cm) break;
        const int l = __ffs(cm) - 1;
        dm |= 1u << l;
        f = i64(e0 + l) + 1;
        pend &= ~((2u << l) - 1u);
      }
      if ((dm >> lane) & 1u) {
        const u32 below = dm & lanemask_lt_();
        const i64 fr = below ? i64(e0 + 31 - __clz(below)) + 1 : frontier;
        stage[nrep + __popc(below)] = make_int4(q, e, int(fr), 0);
      }
      nrep += __popc(dm);
      frontier = f;
    }
  }
  if (lane == 0) a.rcnt[q] = nrep;
}

constexpr int kCandThreads = 1024;  // (measured: 1,024 > 512 > 256 > 128)

__global__ void __launch_bounds__(kCandThreads) k_rp_dec_cands(RP a) {
  const int q = blockIdx.x;
  const u32 R = a.rcnt[q];
  if (R == 0) return;
  const i64 he = a.hbeg[q + 1];
  const i64 beg = a.ix_off[q];
  const int n = int(a.ix_off[q + 1] - beg);
  const int4 *stage = a.stage + a.soff[q];
  uint2 *dwin = a.dwin + a.soff[q];
  for (u32 j = threadIdx.x; j < R; j += kCandThreads) {
    const int4 d = stage[j];
    const int e = d.y;
    const i64 fr = d.z;
    if (a.lazy) {
      // the chain from the deepest interval outwards is length-descending:
      // skip its ineligible head, the rest (odep links) is eligible
      const u32 a0 = a.ix_toff[q];
      u32 z = a.endoff[beg + e] - 1u, t = __ldg(&a.otr[a0 + z]);
      u32 L = u32(__ldg(&a.tlen_off[t + 1]) - __ldg(&a.tlen_off[t]));
      while (i64(e) - i64(L) + 1 < fr) {
        z = __ldg(&a.opar[a0 + z]);
        t = __ldg(&a.otr[a0 + z]);
        L = u32(__ldg(&a.tlen_off[t + 1]) - __ldg(&a.tlen_off[t]));
      }
      const u32 ne = __ldg(&a.odep[a0 + z]);
      if (ne == 1) {
        dwin[j] = make_uint2(t, z);
        continue;
      }
      const unsigned long long o = atomicAdd(a.ccnt, (unsigned long long)ne);
      if (i64(o + ne) > a.ccap) {
        dwin[j] = make_uint2(kDecOver, 0u);
        a.need_wv[q] = 1;
        continue;
      }
      for (u32 i = 0; i < ne; ++i) {
        a.cand[o + i] = RpCand{0ull, L, t, z, u32(q), u32(e), 0u};
        if (i + 1 < ne) {
          z = __ldg(&a.opar[a0 + z]);
          t = __ldg(&a.otr[a0 + z]);
          L = u32(__ldg(&a.tlen_off[t + 1]) - __ldg(&a.tlen_off[t]));
        }
      }
      dwin[j] = make_uint2(kDecMulti | ne, u32(o));
      continue;
    }
    const i64 r0 = a.endoff[beg + e];
    const i64 r1 = e + 1 < n ? i64(a.endoff[beg + e + 1]) : he;
    // the shortest record is eligible by construction; count the others
    const int4 last = a.hits[r1 - 1];
    u32 ne = 1;
    for (i64 k = r1 - 2; k >= r0; --k) {
      const int z = __ldg(&a.hits[k].z);
      const u32 L = u32(__ldg(&a.tlen_off[z + 1]) - __ldg(&a.tlen_off[z]));
      if (i64(e) - i64(L) + 1 < fr) break;
      ++ne;
    }
    if (ne == 1) {
      dwin[j] = make_uint2(u32(last.z), u32(last.w));
      continue;
    }
    const unsigned long long o = atomicAdd(a.ccnt, (unsigned long long)ne);
    if (i64(o + ne) > a.ccap) {
      dwin[j] = make_uint2(kDecOver, 0u);
      a.need_wv[q] = 1;  // decided in k_rp_dec_pick with wavelet queries
      continue;
    }
    for (u32 i = 0; i < ne; ++i) {
      const int4 r = a.hits[r1 - ne + i];
      const u32 L = u32(__ldg(&a.tlen_off[r.z + 1]) - __ldg(&a.tlen_off[r.z]));
      a.cand[o + i] = RpCand{0ull, L, u32(r.z), u32(r.w), u32(q), u32(e), 0u};
    }
    dwin[j] = make_uint2(kDecMulti | ne, u32(o));
  }
}

// Scores of the staged candidates, a warp per candidate: count = the
// trace's occurrences ending at or before e, previous end = the largest
// occurrence end below e -- one pass over the trace's occurrence range in the
// reversed stream's suffix array (ends E[r] = n - 1 - SA_rev[r]).  Ranges
// longer than kScanMax are left to the wavelet queries (k_rp_cand_wv).
__global__ void __launch_bounds__(256) k_rp_cand_score(RP a) {
  const int lane = threadIdx.x & 31;
  const i64 nc = min(i64(*a.ccnt), a.ccap);
  for (i64 i = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < nc; i += (i64(gridDim.x) * blockDim.x) >> 5) {
    RpCand &c = a.cand[i];
    const int q = int(c.q);
    const u64 kk = __ldg(&a.ix_tkey[a.ix_toff[q] + c.slot]);
    const u32 lo = u32(kk >> 15) & 32767u, hi = 32767u - (u32(kk) & 32767u);
    if (hi - lo > a.scan_max) {
      if (lane == 0) {
        a.pend[atomicAdd(a.pcnt, 1ull)] = u32(i);
        a.need_wv[q] = 1;
      }
      continue;
    }
    const i64 beg = a.ix_off[q];
    const int n1 = int(a.ix_off[q + 1] - beg) - 1;
    const int e = int(c.e);
    u32 cnt = 0;
    int pm = -1;
    for (u32 r = lo + lane; r < hi; r += 32) {
      const int E = n1 - (__ldg(&a.ix_sa[beg + r]) - int(beg));
      cnt += E <= e ? 1u : 0u;
      if (E < e) pm = max(pm, E);
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    pm = __reduce_max_sync(0xffffffffu, pm);
    if (lane == 0) c.sc = score_of(a, cnt, cnt >= 2 ? u32(e - pm) : 0u, c.len);
  }
}

// The candidates with long occurrence ranges: wavelet-matrix queries.
__global__ void k_rp_cand_wv(RP a) {
  const i64 np = i64(*a.pcnt);
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < np; i += i64(gridDim.x) * blockDim.x) {
    RpCand &c = a.cand[a.pend[i]];
    c.sc = wv_score(a, int(c.q), make_int4(int(c.q), int(c.e), int(c.t), int(c.slot)), c.len);
  }
}

__global__ void __launch_bounds__(32) k_rp_dec_pick(RP a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int q = a.order[blockIdx.x], lane = threadIdx.x;
  const u32 R = a.rcnt[q];
  if (R == 0) return;
  const u32 nw = (a.maxslot[q] + 31) / 32;
  u32 *rep = nw <= a.on_chip_bits ? reinterpret_cast<u32 *>(smraw) : static_cast<u32 *>(a.gstate) + a.gstate_off[q];
  for (u32 i = lane; i < nw; i += 32) rep[i] = 0u;
  __syncwarp();
  const i64 he = a.hbeg[q + 1];
  const i64 beg = a.ix_off[q];
  const int n = int(a.ix_off[q + 1] - beg);
  int4 *stage = a.stage + a.soff[q];
  const uint2 *dwin = a.dwin + a.soff[q];
  for (u32 j0 = 0; j0 < R; j0 += 32) {
    const u32 j = j0 + lane;
    const int4 d = j < R ? stage[j] : make_int4(0, 0, 0, 0);
    const uint2 w = j < R ? dwin[j] : make_uint2(0, 0);
    const int m = int(min(32u, R - j0));
    for (int l = 0; l < m; ++l) {
      const u32 wx = __shfl_sync(0xffffffffu, w.x, l), wy = __shfl_sync(0xffffffffu, w.y, l);
      const int e = __shfl_sync(0xffffffffu, d.y, l);
      u32 bt = wx, bslot = wy;
      if (wx & kDecMulti) {
        if (wx == kDecOver) {
          rp_decide_end(a, q, beg, he, n, rep, e, i64(__shfl_sync(0xffffffffu, d.z, l)), &bt, &bslot);
        } else {
          const u32 nl = wx & ~kDecMulti;
          bool have = false;
          u64 bs = 0;
          u32 bl = 0;
          for (u32 i0 = 0; i0 < nl; i0 += 32) {
            const u32 i = i0 + lane;
            const bool ok = i < nl;
            const RpCand c = ok ? a.cand[wy + i] : RpCand{0, 0, 0, 0, 0};
            u64 sc = c.sc;
            if (ok && ((rep[c.slot >> 5] >> (c.slot & 31)) & 1u)) sc = sc * a.bonus_num / a.bonus_den;
            const int b = warp_best(ok, sc, c.len, c.t);
            if (b >= 0) {
              const u64 s1 = __shfl_sync(0xffffffffu, sc, b);
              const u32 l1 = __shfl_sync(0xffffffffu, c.len, b), t1 = __shfl_sync(0xffffffffu, c.t, b);
              const u32 z1 = __shfl_sync(0xffffffffu, c.slot, b);
              if (!have || beats(s1, l1, t1, bs, bl, bt)) {
                bs = s1;
                bl = l1;
                bt = t1;
                bslot = z1;
                have = true;
              }
            }
          }
        }
        __syncwarp();
      }
      if (lane == 0) {
        const u32 mk = 1u << (bslot & 31);
        const u32 old = rep[bslot >> 5];
        stage[j0 + l] = make_int4(q, e, int(bt), (old & mk) ? 0 : 1);
        rep[bslot >> 5] = old | mk;
      }
      __syncwarp();
    }
  }
}

struct ReplayScanF {
  const u32 *cnt;
  u32 *base;
  int n;
  i64 *total;
  __device__ u32 load(i64 i) const { return cnt[i]; }
  __device__ bool store(i64 i, u32 incl, u32 excl) const {
    base[i] = excl;
    if (i == n - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_replay_compact(const int4 *__restrict__ stage, const i64 *__restrict__ soff,
                                 const u32 *__restrict__ rcnt, const u32 *__restrict__ rbase, i64 cap,
                                 int4 *__restrict__ out) {
  const int q = blockIdx.x;
  const u32 n = rcnt[q];
  const i64 b = rbase[q];
  for (u32 i = threadIdx.x; i < n; i += blockDim.x)
    if (b + i < cap) out[b + i] = stage[soff[q] + i];
}

}  // namespace

void run_replay(Ctx &c, const apo_trie *tr, const apo_match_rec *d_hits, i64 nhits, const i64 *h_len,
                int nstreams, const apo_replay_params &prm, apo_replay_rec *d_out, i64 cap, i64 *d_count,
                cudaStream_t s, const ReplayIndex *ri) {
  const bool fast = ri != nullptr && ri->ok;
  require(prm.count_cap >= 1 && prm.decay_q16 >= 0 && prm.decay_q16 <= 65536 && prm.decay_period >= 1 &&
              prm.bonus_num >= 0 && prm.bonus_den >= 1,
          "invalid replay parameters");
  APO_CUDA(cudaMemsetAsync(d_count, 0, sizeof(i64), s));
  if (nhits == 0 || nstreams == 0) return;
  const int slot_bits = std::max(1, bits_for(u64(std::max<i64>(tr->T, 2) - 1)));
  require(slot_bits <= 3 * kMaxDigit, "too many traces for REPLAY (slots must fit 27 bits)");
  // decay table d_k = d_{k-1} * decay >> 16 (the oracle's recurrence), up to
  // the longest possible gap / period, or until it stops changing
  i64 maxlen = 0, tot = 0;
  std::vector<i64> h_soff(size_t(nstreams) + 1);
  for (int q = 0; q < nstreams; ++q) {
    h_soff[q] = tot;
    tot += h_len[q];
    maxlen = std::max(maxlen, h_len[q]);
  }
  h_soff[nstreams] = tot;
  std::vector<u32> dq(1, 65536u);
  const i64 kmax = maxlen / prm.decay_period + 1;
  while (i64(dq.size()) <= kmax) {
    const u32 nx = u32((u64(dq.back()) * u64(prm.decay_q16)) >> 16);
    dq.push_back(nx);
    if (nx == dq[dq.size() - 2]) break;  // fixed point (0, or no decay): later entries equal it
  }
  // stream ranges (device binary searches), then the part plan on the host
  const size_t hb_bytes = sizeof(i64) * (size_t(nstreams) + 1);
  i64 *hbeg0 = static_cast<i64 *>(c.pool_get(hb_bytes));
  if (fast && ri->lazy)
    k_replay_ranges_q<<<grid_for(i64(nstreams) + 1, 256), 256, 0, s>>>(ri->qbase, nhits, nstreams, hbeg0);
  else
    k_replay_ranges<<<grid_for(i64(nstreams) + 1, 256), 256, 0, s>>>(reinterpret_cast<const int4 *>(d_hits), nhits,
                                                                    nstreams, hbeg0);
  APO_CHECK_LAUNCH();
  c.launches++;
  std::vector<i64> h_hb(size_t(nstreams) + 1);
  c.d2h(h_hb.data(), hbeg0, hb_bytes, s);
  std::vector<i64> h_pb(size_t(nstreams) + 1);
  i64 nparts = 0;
  for (int q = 0; q < nstreams; ++q) {
    h_pb[q] = nparts;
    nparts += (h_hb[q + 1] - h_hb[q] + kPart - 1) / kPart;
  }
  h_pb[nstreams] = nparts;
  if (nparts == 0) {
    c.pool_put(hbeg0, hb_bytes);
    return;
  }
  std::vector<int> h_ps(static_cast<size_t>(nparts));
  for (int q = 0; q < nstreams; ++q)
    for (i64 p = h_pb[q]; p < h_pb[q + 1]; ++p) h_ps[p] = q;
  std::vector<int> h_order(static_cast<size_t>(nstreams));
  for (int q = 0; q < nstreams; ++q) h_order[q] = q;
  std::stable_sort(h_order.begin(), h_order.end(),
                   [&](int x, int y) { return h_hb[x + 1] - h_hb[x] > h_hb[y + 1] - h_hb[y]; });
  // wavelet work items (fast path): <= kWvPart records of one stream each
  std::vector<int> h_wq;
  std::vector<i64> h_wr;
  if (fast) {
    for (int q = 0; q < nstreams; ++q)
      for (i64 r = h_hb[q]; r < h_hb[q + 1]; r += kWvPart) {
        h_wq.push_back(q);
        h_wr.push_back(r);
      }
    h_wr.push_back(h_hb[nstreams]);
  }
  const i64 nitems = i64(h_wq.size());
  // workspace (a pooled block: the arenas may hold the matcher's index)
  i64 *hbeg, *pbeg, *soff, *gso, *wr0 = nullptr;
  int *pstream, *order, *wq = nullptr;
  u32 *maxslot, *run_slot = nullptr, *run_cnt = nullptr, *nruns = nullptr, *rcnt, *rbase, *ddq;
  i32 *run_last = nullptr, *cmax;
  u64 *sc = nullptr;
  WvMat *wv = nullptr;
  int4 *stage;
  const size_t npart_rec = fast ? 0 : size_t(nparts) * kPart;
  const bool by_ends = fast && ri->endoff != nullptr && ri->endml != nullptr;
  uint2 *dwin = nullptr;
  RpCand *cand = nullptr;
  unsigned long long *ccnt = nullptr;
  u32 *pend = nullptr;
  unsigned char *need_wv = nullptr;
  // candidate pool (decisions beyond it are decided by the whole warp in
  // k_rp_dec_pick); APO_REPLAY_CCAP (tests) shrinks it to force that path
  i64 ccap = std::min<i64>(std::max<i64>(tot, 1), std::max<i64>(i64(1) << 16, tot / 64));
  if (const char *cc = std::getenv("APO_REPLAY_CCAP")) ccap = std::max<i64>(1, std::atoll(cc));
  auto plan = [&](Carver &cv) {
    hbeg = cv.take<i64>(size_t(nstreams) + 1);
    pbeg = cv.take<i64>(size_t(nstreams) + 1);
    soff = cv.take<i64>(size_t(nstreams) + 1);
    gso = cv.take<i64>(size_t(nstreams) + 1);
    pstream = cv.take<int>(size_t(nparts));
    order = cv.take<int>(size_t(nstreams));
    maxslot = cv.take<u32>(size_t(nstreams));
    rcnt = cv.take<u32>(size_t(nstreams));
    rbase = cv.take<u32>(size_t(nstreams));
    ddq = cv.take<u32>(dq.size());
    cmax = cv.take<i32>(size_t(nparts) * kChunksPerPart);
    if (fast) {
      wq = cv.take<int>(size_t(nitems));
      wr0 = cv.take<i64>(size_t(nitems) + 1);
      wv = cv.take<WvMat>(size_t(nstreams));
    } else {
      nruns = cv.take<u32>(size_t(nparts));
      run_slot = cv.take<u32>(npart_rec);
      run_cnt = cv.take<u32>(npart_rec);
      run_last = cv.take<i32>(npart_rec);
      sc = cv.take<u64>(size_t(nhits));
    }
    stage = cv.take<int4>(size_t(tot));
    if (by_ends) {
      dwin = cv.take<uint2>(size_t(tot));
      cand = cv.take<RpCand>(size_t(ccap));
      ccnt = cv.take<unsigned long long>(2);
      pend = cv.take<u32>(size_t(ccap));
      need_wv = cv.take<unsigned char>(size_t(nstreams));
    }
  };
  Carver dry(nullptr);
  plan(dry);
  const size_t ws_bytes = dry.off + 256;
  char *ws = static_cast<char *>(c.pool_get(ws_bytes));
  Carver cv(ws);
  plan(cv);
  c.d2d(hbeg, hbeg0, hb_bytes, s);
  c.h2d(pbeg, h_pb.data(), hb_bytes, s);
  c.h2d(soff, h_soff.data(), hb_bytes, s);
  c.h2d(pstream, h_ps.data(), sizeof(int) * size_t(nparts), s);
  c.h2d(order, h_order.data(), sizeof(int) * size_t(nstreams), s);
  c.h2d(ddq, dq.data(), sizeof(u32) * dq.size(), s);
  APO_CUDA(cudaMemsetAsync(maxslot, 0, sizeof(u32) * size_t(nstreams), s));
  RP a{reinterpret_cast<const int4 *>(d_hits), tr->d_off, ddq, int(dq.size()), prm.count_cap, prm.decay_period,
       1.0 / double(prm.decay_period), u32(prm.bonus_num), u32(prm.bonus_den), nstreams, slot_bits, hbeg, pbeg,
       pstream, maxslot, run_slot, run_cnt, run_last, nruns, sc, cmax, order, nullptr, gso, 0u, 0u, soff, stage,
       rcnt, nullptr, nullptr, nullptr, nullptr, wq, wr0, wv, nullptr, nullptr};
  const size_t psmem = sizeof(PartSmem);
  a.dwin = dwin;
  a.cand = cand;
  a.ccap = ccap;
  a.ccnt = ccnt;
  a.pcnt = by_ends ? ccnt + 1 : nullptr;
  a.pend = pend;
  a.need_wv = need_wv;
  a.scan_max = kScanMax;
  if (const char *sm = std::getenv("APO_REPLAY_SCANMAX")) a.scan_max = u32(std::atoll(sm));  // tests
  if (by_ends) {
    APO_CUDA(cudaMemsetAsync(ccnt, 0, 2 * sizeof(unsigned long long), s));
    APO_CUDA(cudaMemsetAsync(need_wv, 0, size_t(nstreams), s));
  }
  if (fast) {
    c.h2d(wq, h_wq.data(), sizeof(int) * size_t(nitems), s);
    c.h2d(wr0, h_wr.data(), sizeof(i64) * (size_t(nitems) + 1), s);
    a.ix_off = ri->off;
    a.ix_sa = ri->sa;
    a.ix_tkey = ri->tkey;
    a.ix_toff = ri->toff;
    a.lazy = ri->lazy;
    a.opar = ri->opar;
    a.otr = ri->otr;
    a.odep = ri->odep;
    const size_t wsmem = sizeof(WvSmem);
    c.smem_optin(reinterpret_cast<const void *>(k_rp_wvbuild), wsmem);
    if (by_ends) {
      // the emitter's per-end index: decision ends, their candidates and the
      // candidates' scores (scans; wavelet matrices only for the streams with
      // long occurrence ranges or pool overflows)
      a.endoff = ri->endoff;
      a.endml = ri->endml;
      k_rp_dec_find<<<(nstreams + kFindWarps - 1) / kFindWarps, kFindWarps * 32, 0, s>>>(a);
      APO_CHECK_LAUNCH();
      k_rp_dec_cands<<<nstreams, kCandThreads, 0, s>>>(a);
      APO_CHECK_LAUNCH();
      k_rp_cand_score<<<c.num_sms * 8, 256, 0, s>>>(a);
      APO_CHECK_LAUNCH();
      k_rp_wvbuild<<<nstreams, kWvThreads, wsmem, s>>>(a);
      APO_CHECK_LAUNCH();
      k_rp_cand_wv<<<c.num_sms * 4, 256, 0, s>>>(a);
      APO_CHECK_LAUNCH();
      c.launches += 4;
    } else {
      // the matrices once per stream; scores are evaluated lazily in phase D
      k_rp_wvbuild<<<nstreams, kWvThreads, wsmem, s>>>(a);
      APO_CHECK_LAUNCH();
      k_rp_cmax<<<unsigned(nitems), 256, 0, s>>>(a);
      APO_CHECK_LAUNCH();
      c.launches++;
    }
  } else {
    c.smem_optin(reinterpret_cast<const void *>(k_rp_local), psmem);
    c.smem_optin(reinterpret_cast<const void *>(k_rp_scores), psmem);
    k_rp_local<<<unsigned(nparts), kPartThreads, psmem, s>>>(a);
    APO_CHECK_LAUNCH();
  }
  // per-stream tables: on chip when they fit, else in a global block
  std::vector<u32> h_ms(static_cast<size_t>(nstreams));
  c.d2h(h_ms.data(), maxslot, sizeof(u32) * size_t(nstreams), s);
  const u32 slots_on_chip = u32(kStateBytesMax / 8);
  std::vector<i64> h_gso(size_t(nstreams) + 1);
  i64 gw = 0;
  u32 smax_b = 1, smax_d = 1;
  for (int q = 0; q < nstreams; ++q) {
    h_gso[q] = gw;
    if (h_ms[q] > slots_on_chip)
      gw += 2 * i64(h_ms[q]);  // phase B's (count, last) table; phase D's bitset fits in it
    else
      smax_b = std::max(smax_b, h_ms[q]);
    if ((h_ms[q] + 31) / 32 <= slots_on_chip / 32) smax_d = std::max(smax_d, (h_ms[q] + 31) / 32);
  }
  h_gso[nstreams] = gw;
  void *gstate = nullptr;
  if (gw > 0) gstate = c.pool_get(sizeof(u32) * size_t(gw));
  c.h2d(gso, h_gso.data(), hb_bytes, s);
  a.gstate = gstate;
  a.on_chip_slots = slots_on_chip;
  a.on_chip_bits = slots_on_chip / 32;
  if (!fast) {
    const size_t bsmem = size_t(smax_b) * 8;
    c.smem_optin(reinterpret_cast<const void *>(k_rp_prefix), bsmem);
    k_rp_prefix<<<nstreams, kPrefixThreads, bsmem, s>>>(a);
    APO_CHECK_LAUNCH();
    k_rp_scores<<<unsigned(nparts), kPartThreads, psmem, s>>>(a);
    APO_CHECK_LAUNCH();
  }
  if (by_ends) {
    k_rp_dec_pick<<<nstreams, 32, size_t(smax_d) * 4, s>>>(a);
  } else {
    k_rp_decide<<<nstreams, 32, size_t(smax_d) * 4, s>>>(a);
  }
  APO_CHECK_LAUNCH();
  ReplayScanF f{rcnt, rbase, nstreams, d_count};
  launch_scan<false>(c, nstreams, f, s);
  if (cap > 0) {
    k_replay_compact<<<nstreams, 128, 0, s>>>(stage, soff, rcnt, rbase, cap, reinterpret_cast<int4 *>(d_out));
    APO_CHECK_LAUNCH();
  }
  c.launches += 5;
  APO_CUDA(cudaStreamSynchronize(s));
  if (gstate) c.pool_put(gstate, sizeof(u32) * size_t(gw));
  c.pool_put(hbeg0, hb_bytes);
  c.pool_put(ws, ws_bytes);
  if (fast) {
    c.pool_put(ri->endoff, ri->endoff_bytes);
    c.pool_put(ri->endml, ri->endml_bytes);
  }
}

}  // namespace apo

using namespace apo;

extern "C" apo_status apo_replay(apo_ctx *ctx, const apo_trie *tr, const apo_match_rec *d_hits, int64_t nhits,
                                 const int64_t *h_len, int32_t nstreams, const apo_replay_params *params,
                                 apo_replay_rec *d_out, int64_t cap, int64_t *d_count, void *stream) {
  if (!ctx) return APO_ERR_INVALID;
  Ctx &c = ctx->c;
  c.err.clear();
  try {
    APO_CUDA(cudaSetDevice(c.device));
    require(tr != nullptr && d_count != nullptr && nhits >= 0 && nstreams >= 0 && cap >= 0, "invalid argument");
    require(nhits == 0 || d_hits != nullptr, "d_hits is NULL");
    require(cap == 0 || d_out != nullptr, "d_out is NULL");
    require(nstreams == 0 || h_len != nullptr, "h_len is NULL");
    for (int q = 0; q < nstreams; ++q) require(h_len[q] >= 0, "negative stream length");
    const apo_replay_params prm = params ? *params : apo_replay_params{100, 64881, 100, 11, 10, 0};
    run_replay(c, tr, d_hits, nhits, h_len, nstreams, prm, d_out, cap, d_count, static_cast<cudaStream_t>(stream));
    return APO_OK;
  } catch (const Error &e) {
    c.err = e.msg;
    return e.code;
  } catch (const std::exception &e) {
    c.err = e.what();
    return APO_ERR_CUDA;
  }
}
