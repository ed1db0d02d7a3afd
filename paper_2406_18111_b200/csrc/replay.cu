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
// one warp walks one stream's hits end by end:
//   * the completions at an end are consecutive records; lanes take 32 at a
//     time, update their trace's state (count, last end, replayed flag) in
//     shared memory indexed by the record's stream-local slot, score it, and
//     a warp arg-max (score, length, -id) picks the replay among those that
//     start at or after the frontier;
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

constexpr int kReplaySlots = 2048;  // on-chip per-stream trace states (u64 each: 16 KB)
constexpr int kReplayThreads = 32;  // one warp per stream

struct ReplayArgs {
  const int4 *hits;
  i64 nhits;
  int nstreams;
  const i64 *tlen_off;   // trace offsets (T+1): len(t) = off[t+1] - off[t]
  const u32 *dq;         // decay table d_k, k < ndq
  int ndq;
  int count_cap, period;
  u32 bonus_num, bonus_den;
  const i64 *hbeg;       // per stream: first hit (nstreams + 1, from k_replay_ranges)
  const u32 *maxslot;    // per stream: max slot + 1
  u64 *gstate;           // global fallback states
  const i64 *gstate_off; // per stream offset into gstate (nstreams + 1)
  const i64 *soff;       // per stream staging offset (stream position base)
  int4 *stage;           // staged replays
  u32 *rcnt;             // per stream replay count
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

// state word: [replayed:1][count:31][last end + 1:32]
__global__ void __launch_bounds__(kReplayThreads) k_replay(ReplayArgs a) {
  __shared__ u64 s_state[kReplaySlots];
  const int q = blockIdx.x, lane = threadIdx.x;
  const i64 hb = a.hbeg[q], he = a.hbeg[q + 1];
  const u32 ms = a.maxslot[q];
  const bool onchip = ms <= u32(kReplaySlots);
  u64 *st = onchip ? s_state : a.gstate + a.gstate_off[q];
  for (u32 i = lane; i < ms; i += 32) st[i] = 0;
  __syncwarp();
  i64 frontier = 0;
  u32 nrep = 0;
  int4 *stage = a.stage + a.soff[q];
  i64 p = hb;
  // running best of the current end (warp-uniform)
  bool have = false;
  u64 bs = 0;
  u32 bl = 0, bt = 0, bslot = 0;
  while (p < he) {
    const i64 k = p + lane;
    int4 r = make_int4(-1, -1, -1, -1);
    if (k < he) r = a.hits[k];
    const int e0 = __shfl_sync(0xffffffffu, r.y, 0);
    const bool mine = k < he && r.y == e0;
    const u32 msk = __ballot_sync(0xffffffffu, mine);
    const int cnt = __popc(msk);  // a prefix of the lanes (records sorted by end)
    u64 sc = 0;
    u32 L = 0;
    bool ok = false;
    if (mine) {
      L = u32(a.tlen_off[r.z + 1] - a.tlen_off[r.z]);
      const u64 w = st[r.w];
      const u32 last1 = u32(w);
      const u32 c0 = u32(w >> 32) & 0x7fffffffu;
      const bool rep = (w >> 63) != 0;
      const u32 c = min(c0 + 1u, u32(a.count_cap));  // saturates at the cap (min(count, cap) is all the score uses)
      const u32 gap = last1 ? u32(e0) - (last1 - 1u) : 0u;
      const u32 kk = gap / u32(a.period);
      const u64 d = a.dq[kk < u32(a.ndq) ? kk : u32(a.ndq - 1)];
      sc = u64(L) * u64(c) * d;
      if (rep) sc = sc * a.bonus_num / a.bonus_den;
      st[r.w] = (rep ? (1ull << 63) : 0ull) | (u64(c) << 32) | u64(u32(e0) + 1u);
      ok = i64(e0) - i64(L) + 1 >= frontier;
    }
    // warp arg-max over the valid completions of this chunk
    u64 ms_ = ok ? sc : 0;
    u32 ml = ok ? L : 0, mt = ok ? u32(r.z) : 0xffffffffu, mslot = ok ? u32(r.w) : 0u;
    bool mv = ok;
    if (__any_sync(0xffffffffu, ok)) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const u64 os = __shfl_xor_sync(0xffffffffu, ms_, o);
        const u32 ol = __shfl_xor_sync(0xffffffffu, ml, o), ot = __shfl_xor_sync(0xffffffffu, mt, o);
        const u32 osl = __shfl_xor_sync(0xffffffffu, mslot, o);
        const bool ov = __shfl_xor_sync(0xffffffffu, mv, o);
        if (ov && (!mv || beats(os, ol, ot, ms_, ml, mt))) {
          ms_ = os;
          ml = ol;
          mt = ot;
          mslot = osl;
          mv = true;
        }
      }
      if (!have || beats(ms_, ml, mt, bs, bl, bt)) {
        bs = ms_;
        bl = ml;
        bt = mt;
        bslot = mslot;
        have = true;
      }
    }
    p += cnt;
    // the end is complete unless all 32 lanes were still on it
    const bool more = cnt == 32 && p < he && a.hits[p].y == e0;
    if (!more) {
      if (have) {
        __syncwarp();
        if (lane == 0) {
          const u64 w = st[bslot];
          stage[nrep] = make_int4(q, e0, int(bt), (w >> 63) ? 0 : 1);
          st[bslot] = w | (1ull << 63);
        }
        ++nrep;
        frontier = i64(e0) + 1;
        have = false;
      }
      __syncwarp();
    }
  }
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
  int4 *stage;
  auto plan = [&](Carver &cv) {
    hbeg = cv.take<i64>(size_t(nstreams) + 1);
    soff = cv.take<i64>(size_t(nstreams) + 1);
    gso = cv.take<i64>(size_t(nstreams) + 1);
    tbase = cv.take<i64>(4);
    maxslot = cv.take<u32>(size_t(nstreams));
    rcnt = cv.take<u32>(size_t(nstreams));
    rbase = cv.take<u32>(size_t(nstreams));
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
  std::vector<i64> h_gso(size_t(nstreams) + 1);
  i64 gtot = 0;
  for (int q = 0; q < nstreams; ++q) {
    h_gso[q] = gtot;
    if (h_ms[q] > u32(kReplaySlots)) gtot += h_ms[q];
  }
  h_gso[nstreams] = gtot;
  u64 *gstate = nullptr;
  if (gtot > 0) gstate = static_cast<u64 *>(c.pool_get(sizeof(u64) * size_t(gtot)));
  APO_CUDA(cudaMemcpyAsync(gso, h_gso.data(), sizeof(i64) * (size_t(nstreams) + 1), cudaMemcpyHostToDevice, s));
  ReplayArgs a{hits, nhits, nstreams, tr->d_off, ddq, int(dq.size()), prm.count_cap, prm.decay_period,
               u32(prm.bonus_num), u32(prm.bonus_den), hbeg, maxslot, gstate, gso, soff, stage, rcnt};
  k_replay<<<nstreams, kReplayThreads, 0, s>>>(a);
  APO_CHECK_LAUNCH();
  ReplayScanF f{rcnt, rbase, nstreams, d_count};
  launch_scan<false>(c, nstreams, f, s);
  if (cap > 0) {
    k_replay_compact<<<nstreams, 128, 0, s>>>(stage, soff, rcnt, rbase, cap, reinterpret_cast<int4 *>(d_out));
    APO_CHECK_LAUNCH();
  }
  c.launches += 2;
  APO_CUDA(cudaStreamSynchronize(s));
  if (gstate) c.pool_put(gstate, sizeof(u64) * size_t(gtot));
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
