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
// Streams are independent; within a stream the decisions are a left-to-right
// chain (a replay moves the frontier every later decision depends on), so
// one warp walks one stream's hits (k_replay below):
//   * the hits are read 32 records at a time, the next chunk prefetched, and
//     each record's trace state (appearance count, last end) is updated in
//     parallel in shared memory indexed by the record's stream-local slot;
//   * only the choice per end is sequential: a warp arg-max (score, length,
//     -id) over the end's completions that start at or after the frontier;
//   * decay factors d_k come from a table the host computes with the same
//     integer recurrence (exact, no floating point);
//   * replays are staged per stream (at most one per stream position) and
//     compacted in stream order after a scan of the per-stream counts.
// A stream whose slots exceed the on-chip table keeps its state in global
// memory instead (same code, other pointer).
#include <algorithm>
#include <vector>

#include "trie.cuh"

namespace apo {
namespace {

constexpr int kReplayStateBytes = 32768;  // on-chip per-stream trace states (up to 32 KB per warp)
constexpr int kReplayThreads = 32;  // one warp per stream

struct ReplayArgs {
  const int4 *hits;
  i64 nhits;
  int nstreams;
  const i64 *tlen_off;   // trace offsets (T+1): len(t) = off[t+1] - off[t]
  const u32 *dq;         // decay table d_k, k < ndq
  int ndq;
  int count_cap, period;
  double inv_period;     // 1 / period (the quotient is corrected to the exact one)
  u32 bonus_num, bonus_den;
  const i64 *hbeg;       // per stream: first hit (nstreams + 1, from k_replay_ranges)
  const u32 *maxslot;    // per stream: max slot + 1
  void *gstate;          // global fallback states
  const i64 *gstate_off; // per stream offset into gstate (nstreams + 1)
  const i64 *soff;       // per stream staging offset (stream position base)
  int4 *stage;           // staged replays
  u32 *rcnt;             // per stream replay count
  const int *order;      // block -> stream (streams with the most hits first)
};

// Per stream: its hit range (hits sorted by stream) and its largest slot.
__global__ void k_replay_ranges(const int4 *__restrict__ hits, i64 nhits, int nstreams, i64 *__restrict__ hbeg,
                                u32 *__restrict__ maxslot) {
  const int q = blockIdx.x;
  if (q > nstreams) return;
  // lower bound of stream q (every lane does the same search)
  i64 lo = 0, hi = nhits;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (__ldg(&hits[mid].x) < q)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (threadIdx.x == 0) hbeg[q] = lo;
  if (q == nstreams) return;
  i64 e = lo, hi2 = nhits;  // upper bound
  while (e < hi2) {
    const i64 mid = (e + hi2) >> 1;
    if (__ldg(&hits[mid].x) <= q)
      e = mid + 1;
    else
      hi2 = mid;
  }
  u32 m = 0;
  for (i64 k = lo + threadIdx.x; k < e; k += blockDim.x) m = max(m, u32(__ldg(&hits[k].w)) + 1u);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ u32 s_m[8];
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 r = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) r = max(r, s_m[w]);
    maxslot[q] = r;
  }
}

// (score, len, -id) order: true iff a beats b
__device__ __forceinline__ bool beats(u64 sa, u32 la, u32 ta, u64 sb, u32 lb, u32 tb) {
  if (sa != sb) return sa > sb;
  if (la != lb) return la > lb;
  return ta < tb;
}

// Per-slot trace state: replayed bit, appearance count (saturated at the
// cap: min(count, cap) is all the score uses) and last end + 1 (0 = never).
// Wide: u64 [replayed:1][count:31][last end + 1:32]; narrow (count_cap <=
// 127 and stream lengths < 2^24 - 1): u32 [replayed:1][count:7][last+1:24],
// twice the slots on chip.
template <class W>
struct StateWord;
template <>
struct StateWord<u64> {
  static constexpr u64 kRep = 1ull << 63;
  __device__ static u32 count(u64 w) { return u32(w >> 32) & 0x7fffffffu; }
  __device__ static u32 last1(u64 w) { return u32(w); }
  __device__ static u64 make(u64 rep, u32 c, u32 l1) { return rep | (u64(c) << 32) | u64(l1); }
};
template <>
struct StateWord<u32> {
  static constexpr u32 kRep = 1u << 31;
  __device__ static u32 count(u32 w) { return (w >> 24) & 0x7fu; }
  __device__ static u32 last1(u32 w) { return w & 0xffffffu; }
  __device__ static u32 make(u32 rep, u32 c, u32 l1) { return rep | (c << 24) | l1; }
};

// Warp arg-max of (score, len, -id) over the lanes with ok set: four
// warp reductions (redux.sync) on the score's high and low words, the length
// and the id; returns the winning lane (-1 if no lane is ok).
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

// One warp per stream.  The hits are read in chunks of 32 consecutive
// records, the next chunk (record + trace length) prefetched while the
// current one is processed, so no global load sits on the sequential chain.
// Per chunk, in parallel: each record's appearance count and gap (its
// trace's previous appearance is the previous lane with the same slot in the
// chunk -- __match_any_sync -- or the saved state) and its score before the
// replay bonus; the last lane of each slot writes the state back.  Then the
// decisions: a record is eligible iff it starts at or after the frontier;
// the first eligible record of the chunk marks the next end where a replay
// happens, and since an end's records are in trace-id order (length
// descending) its eligible records are the rest of that end's run.  Only
// such ends are visited: the bonus (the replayed bit may have been set by an
// earlier end of the chunk), the arg-max over the eligible records, merged
// with the running best when the end continues into the next chunk; the
// replay moves the frontier and eligibility is re-evaluated for the later
// records of the chunk.  Ends without an eligible record cost one ballot per
// chunk.
__device__ __forceinline__ int4 replay_rec(const ReplayArgs &a, i64 k, i64 he) {
  return k < he ? a.hits[k] : make_int4(-1, -1, -1, -1);
}
__device__ __forceinline__ u32 replay_len(const ReplayArgs &a, int4 r) {
  return r.z >= 0 ? u32(__ldg(&a.tlen_off[r.z + 1]) - __ldg(&a.tlen_off[r.z])) : 0u;
}

template <class W>
__global__ void __launch_bounds__(kReplayThreads) k_replay(ReplayArgs a) {
  using SW = StateWord<W>;
  constexpr W kReplayed = SW::kRep;
  constexpr u32 kSlots = kReplayStateBytes / sizeof(W);
  extern __shared__ __align__(8) unsigned char s_raw[];
  W *s_state = reinterpret_cast<W *>(s_raw);
  const int q = a.order[blockIdx.x], lane = threadIdx.x;
  const u32 lt = (1u << lane) - 1u;
  const i64 hb = a.hbeg[q], he = a.hbeg[q + 1];
  const u32 ms = a.maxslot[q];
  const bool onchip = ms <= kSlots;
  W *st = onchip ? s_state : static_cast<W *>(a.gstate) + a.gstate_off[q];
  for (u32 i = lane; i < ms; i += 32) st[i] = 0;
  __syncwarp();
  i64 frontier = 0;
  u32 nrep = 0;
  int4 *stage = a.stage + a.soff[q];
  // running best of an eligible end that reaches the chunk's last lane: it
  // may continue into the next chunk, which decides it
  bool have = false;
  int carry_e = -1;
  u64 bs = 0;
  u32 bl = 0, bt = 0, bslot = 0;
  auto commit = [&](int e0) {
    __syncwarp();
    if (lane == 0) {
      const W sw = st[bslot];
      stage[nrep] = make_int4(q, e0, int(bt), (sw & kReplayed) ? 0 : 1);
      st[bslot] = sw | kReplayed;
    }
    __syncwarp();
    ++nrep;
    frontier = i64(e0) + 1;
    have = false;
  };
  // software pipeline: records kRecAhead chunks ahead, trace lengths
  // kLenAhead chunks ahead (a record has kRecAhead - kLenAhead iterations to
  // arrive before its trace length is looked up)
  constexpr int kRecAhead = 10, kLenAhead = 5;
  int4 R[kRecAhead];
  u32 LS[kLenAhead];
#pragma unroll
  for (int k = 0; k < kRecAhead; ++k) R[k] = replay_rec(a, hb + 32 * k + lane, he);
#pragma unroll
  for (int k = 0; k < kLenAhead; ++k) LS[k] = replay_len(a, R[k]);
  for (i64 p = hb; p < he; p += 32) {
    const int4 r = R[0];
    const u32 L = LS[0];
#pragma unroll
    for (int k = 0; k + 1 < kRecAhead; ++k) R[k] = R[k + 1];
#pragma unroll
    for (int k = 0; k + 1 < kLenAhead; ++k) LS[k] = LS[k + 1];
    LS[kLenAhead - 1] = replay_len(a, R[kLenAhead - 1]);
    R[kRecAhead - 1] = replay_rec(a, p + 32 * kRecAhead + lane, he);
    const bool valid = p + lane < he;
    // a carried end that does not continue here is decided first (before
    // this chunk reads its trace states: the replay sets a replayed bit)
    if (have && __shfl_sync(0xffffffffu, r.y, 0) != carry_e) commit(carry_e);
    // ---- appearance counts, gaps and scores (parallel) ----
    const u32 slot = valid ? u32(r.w) : 0xffffffffu;
    const u32 peers = __match_any_sync(0xffffffffu, slot);
    const u32 before = peers & lt;
    u64 sc0 = 0;
    const W w = valid ? st[slot] : W(0);
    const int prev_lane = before ? 31 - __clz(before) : -1;
    const int prev_e = __shfl_sync(0xffffffffu, r.y, prev_lane < 0 ? lane : prev_lane);
    const u32 c0 = SW::count(w);
    if (valid) {
      const u32 c = min(c0 + u32(__popc(before)) + 1u, u32(a.count_cap));
      u32 gap = 0;
      if (prev_lane >= 0)
        gap = u32(r.y - prev_e);
      else if (SW::last1(w))
        gap = u32(r.y) - (SW::last1(w) - 1u);
      // gap / period by a reciprocal, corrected to the exact quotient
      u32 kk = u32(double(gap) * a.inv_period);
      if (u64(kk) * u64(a.period) > u64(gap)) --kk;
      if (u64(kk + 1u) * u64(a.period) <= u64(gap)) ++kk;
      const u64 d = __ldg(&a.dq[kk < u32(a.ndq) ? kk : u32(a.ndq - 1)]);
      sc0 = u64(L) * u64(c) * d;
    }
    __syncwarp();
    if (valid && (peers >> lane) == 1u)  // the slot's last record in the chunk
      st[slot] = SW::make(w & kReplayed, min(c0 + u32(__popc(peers)), u32(a.count_cap)), u32(r.y) + 1u);
    __syncwarp();
    // ---- decisions at the ends with an eligible record ----
    u32 done = 0;  // lanes at or before the last decided end of this chunk
    for (;;) {
      const bool elig = valid && !((done >> lane) & 1u) && i64(r.y) - i64(L) + 1 >= frontier;
      const u32 em = __ballot_sync(0xffffffffu, elig);
      if (!em) break;
      // the end to decide: the first eligible record's (with a carried end,
      // that is the same end: its records lead this chunk)
      const int a0 = __ffs(em) - 1;
      const int e0 = __shfl_sync(0xffffffffu, r.y, a0);
      const bool run = valid && r.y == e0;
      const u32 rm = __ballot_sync(0xffffffffu, run);
      const int a1 = 32 - __clz(rm);  // one past the run's last lane
      const bool ok = elig && run;
      u64 sc = sc0;
      if (ok && (st[slot] & kReplayed)) sc = sc * a.bonus_num / a.bonus_den;
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
  if (have) commit(carry_e);
  if (lane == 0) a.rcnt[q] = nrep;
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
                cudaStream_t s) {
  require(prm.count_cap >= 1 && prm.decay_q16 >= 0 && prm.decay_q16 <= 65536 && prm.decay_period >= 1 &&
              prm.bonus_num >= 0 && prm.bonus_den >= 1,
          "invalid replay parameters");
  APO_CUDA(cudaMemsetAsync(d_count, 0, sizeof(i64), s));
  if (nhits == 0 || nstreams == 0) return;
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
  // workspace
  i64 *hbeg, *soff, *tbase, *gso;
  u32 *maxslot, *rcnt, *rbase, *ddq;
  int *order;
  int4 *stage;
  auto plan = [&](Carver &cv) {
    hbeg = cv.take<i64>(size_t(nstreams) + 1);
    soff = cv.take<i64>(size_t(nstreams) + 1);
    gso = cv.take<i64>(size_t(nstreams) + 1);
    tbase = cv.take<i64>(4);
    maxslot = cv.take<u32>(size_t(nstreams));
    rcnt = cv.take<u32>(size_t(nstreams));
    rbase = cv.take<u32>(size_t(nstreams));
    order = cv.take<int>(size_t(nstreams));
    ddq = cv.take<u32>(dq.size());
    stage = cv.take<int4>(size_t(tot));
  };
  Carver dry(nullptr);
  plan(dry);
  c.arena.reserve(dry.off, s);
  Carver cv(c.arena.base);
  plan(cv);
  APO_CUDA(cudaMemcpyAsync(soff, h_soff.data(), sizeof(i64) * (size_t(nstreams) + 1), cudaMemcpyHostToDevice, s));
  APO_CUDA(cudaMemcpyAsync(ddq, dq.data(), sizeof(u32) * dq.size(), cudaMemcpyHostToDevice, s));
  const int4 *hits = reinterpret_cast<const int4 *>(d_hits);
  k_replay_ranges<<<nstreams + 1, 256, 0, s>>>(hits, nhits, nstreams, hbeg, maxslot);
  APO_CHECK_LAUNCH();
  c.launches++;
  // global state only for streams whose slots do not fit on chip
  std::vector<u32> h_ms(static_cast<size_t>(nstreams));
  APO_CUDA(cudaMemcpyAsync(h_ms.data(), maxslot, sizeof(u32) * size_t(nstreams), cudaMemcpyDeviceToHost, s));
  APO_CUDA(cudaStreamSynchronize(s));
  const bool narrow = prm.count_cap <= 127 && maxlen < (i64(1) << 24) - 1;
  const size_t wbytes = narrow ? sizeof(u32) : sizeof(u64);
  const u32 kslots = u32(kReplayStateBytes / wbytes);
  std::vector<i64> h_gso(size_t(nstreams) + 1);
  i64 gtot = 0;
  for (int q = 0; q < nstreams; ++q) {
    h_gso[q] = gtot;
    if (h_ms[q] > kslots) gtot += h_ms[q];
  }
  h_gso[nstreams] = gtot;
  void *gstate = nullptr;
  if (gtot > 0) gstate = c.pool_get(wbytes * size_t(gtot));
  APO_CUDA(cudaMemcpyAsync(gso, h_gso.data(), sizeof(i64) * (size_t(nstreams) + 1), cudaMemcpyHostToDevice, s));
  // streams with the most hits first (the per-stream walks are sequential:
  // the longest ones must start in the first wave)
  std::vector<i64> h_hb(size_t(nstreams) + 1);
  APO_CUDA(cudaMemcpy(h_hb.data(), hbeg, sizeof(i64) * (size_t(nstreams) + 1), cudaMemcpyDeviceToHost));
  std::vector<int> h_order(static_cast<size_t>(nstreams));
  for (int q = 0; q < nstreams; ++q) h_order[q] = q;
  std::stable_sort(h_order.begin(), h_order.end(),
                   [&](int x, int y) { return h_hb[x + 1] - h_hb[x] > h_hb[y + 1] - h_hb[y]; });
  APO_CUDA(cudaMemcpyAsync(order, h_order.data(), sizeof(int) * size_t(nstreams), cudaMemcpyHostToDevice, s));
  ReplayArgs a{hits, nhits, nstreams, tr->d_off, ddq, int(dq.size()), prm.count_cap, prm.decay_period,
               1.0 / double(prm.decay_period), u32(prm.bonus_num), u32(prm.bonus_den), hbeg, maxslot, gstate,
               gso, soff, stage, rcnt, order};
  u32 smax = 0;
  for (int q = 0; q < nstreams; ++q)
    if (h_ms[q] <= kslots) smax = std::max(smax, h_ms[q]);
  const size_t rsmem = wbytes * std::max<size_t>(smax, 2);
  if (narrow)
    k_replay<u32><<<nstreams, kReplayThreads, rsmem, s>>>(a);
  else
    k_replay<u64><<<nstreams, kReplayThreads, rsmem, s>>>(a);
  APO_CHECK_LAUNCH();
  ReplayScanF f{rcnt, rbase, nstreams, d_count};
  launch_scan<false>(c, nstreams, f, s);
  if (cap > 0) {
    k_replay_compact<<<nstreams, 128, 0, s>>>(stage, soff, rcnt, rbase, cap, reinterpret_cast<int4 *>(d_out));
    APO_CHECK_LAUNCH();
  }
  c.launches += 2;
  APO_CUDA(cudaStreamSynchronize(s));
  if (gstate) c.pool_put(gstate, wbytes * size_t(gtot));
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
