// dsa.cu -- building blocks of the distributed suffix array (SURVEY.md
// §8(f)3: one window larger than one GPU, prefix doubling with a sample-sort
// exchange between GPUs).  "SA, LCP <- SuffixArray(S)" (Alg. 2,
// P:552) for S split into contiguous position blocks, one per rank.
//
// The host orchestration (paper_2406_18111_b200/dsa.py) moves data between
// ranks with NCCL all-to-all / all-gather (torch.distributed: plumbing);
// every step that computes runs here or in K1 (apo_radix_sort):
//   apo_dsa_keys     round key of each owned suffix: (rank[i], rank[i+h])
//                    packed as rank[i] * (n + 1) + rank2 (rank2 = 0 past the
//                    end), ranks are group-head indices + 1 in [1, n];
//   apo_dsa_samples  evenly spaced (key, value) samples of a sorted block;
//   apo_dsa_split    per destination rank, how many of a block sorted by
//                    (key, value) fall below each (key, value) splitter;
//   apo_dsa_heads    new ranks of a block of the globally sorted sequence:
//                    group head iff the key differs from the previous one
//                    (the previous rank's last key for the first element);
//                    rank = global index of the head + 1, heads before the
//                    block carried in; also the number of heads and the
//                    last head's global index;
//   apo_dsa_scatter  received (position, rank) pairs into the owned block;
//   apo_dsa_lcp_requests / apo_dsa_gather / apo_dsa_lcp_update
//                    the LCP of the distributed SA by galloping over the
//                    saved rank levels (equal level-j ranks <=> equal 2^j-token
//                    prefixes): per level, every adjacent pair asks the
//                    owners of i + l and i' + l for their level ranks.
#include "pipeline.cuh"

namespace apo {
namespace {

__global__ void k_dsa_keys(const u32 *__restrict__ rank, const u32 *__restrict__ rank2, i64 m, i64 m2, i64 base,
                           i64 n, u64 *__restrict__ keys, u32 *__restrict__ vals) {
  const i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const u64 r2 = k < m2 ? u64(rank2[k]) : 0ull;  // suffix i + h starts past the end: "end of string"
  keys[k] = u64(rank[k]) * u64(n + 1) + r2;
  vals[k] = u32(base + k);
}

__global__ void k_dsa_samples(const u64 *__restrict__ keys, const u32 *__restrict__ vals, i64 m, int s,
                              u64 *__restrict__ sk, u32 *__restrict__ sv) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  const i64 k = m > 0 ? (i64(j) * m) / s + (m / s) / 2 : 0;
  const i64 kk = k < m ? k : m - 1;
  sk[j] = m > 0 ? keys[kk] : ~0ull;
  sv[j] = m > 0 ? vals[kk] : ~0u;
}

// number of (key, val) pairs of the sorted block strictly below (sk, sv)
__device__ __forceinline__ i64 lower_bound_kv(const u64 *keys, const u32 *vals, i64 m, u64 sk, u32 sv) {
  i64 lo = 0, hi = m;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    const u64 k = keys[mid];
    if (k < sk || (k == sk && vals[mid] < sv))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void k_dsa_split(const u64 *__restrict__ keys, const u32 *__restrict__ vals, i64 m,
                            const u64 *__restrict__ sk, const u32 *__restrict__ sv, int g, i64 *__restrict__ counts) {
  // one thread per destination: [bound(d-1), bound(d))
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= g) return;
  const i64 lo = d == 0 ? 0 : lower_bound_kv(keys, vals, m, sk[d - 1], sv[d - 1]);
  const i64 hi = d == g - 1 ? m : lower_bound_kv(keys, vals, m, sk[d], sv[d]);
  counts[d] = hi > lo ? hi - lo : 0;
}

// Heads and new ranks over a single-pass look-back scan (max of head index).
struct DsaHeadF {
  const u64 *keys;
  i64 m;
  u64 prev_key;
  int has_prev;
  i64 gbase;      // global index of this block's first element
  i64 carry;      // global index of the last head before this block (-1: none)
  u32 *out_rank;
  i64 *stats;     // [0] heads, [1] last head global index (-1 none)
  __device__ u32 load(i64 k) const {
    const bool head = k == 0 ? (!has_prev || keys[0] != prev_key) : keys[k] != keys[k - 1];
    return head ? u32(k + 1) : 0u;  // max-scan of (local head index + 1)
  }
  __device__ bool store(i64 k, u32 incl, u32) const {
    const i64 h = incl ? gbase + i64(incl) - 1 : carry;
    out_rank[k] = u32(h + 1);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_dsa_stats(const u64 *__restrict__ keys, i64 m, u64 prev_key, int has_prev, i64 gbase,
                            i64 *__restrict__ stats) {
  // heads count and last head (one pass, block-strided; stats zeroed / -1 by the host)
  i64 cnt = 0, last = -1;
  for (i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += i64(gridDim.x) * blockDim.x) {
    const bool head = k == 0 ? (!has_prev || keys[0] != prev_key) : keys[k] != keys[k - 1];
    if (head) {
      ++cnt;
      last = max(last, gbase + k);
    }
  }
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (cnt) atomicAdd(reinterpret_cast<unsigned long long *>(&stats[0]), (unsigned long long)cnt);
    if (last >= 0) atomicMax(reinterpret_cast<long long *>(&stats[1]), (long long)last);
  }
}

__global__ void k_dsa_scatter(const u32 *__restrict__ pos, const u32 *__restrict__ rk, i64 m, i64 base,
                              u32 *__restrict__ rank) {
  const i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) rank[i64(pos[k]) - base] = rk[k];
}

// LCP galloping step requests: pair p = (a[p], b[p]) at current lcp l[p]
// asks for the level ranks at a + l and b + l (request 2p and 2p + 1;
// key = position, or n when past the end: such requests are not sent).
__global__ void k_dsa_lcp_req(const u32 *__restrict__ a, const u32 *__restrict__ b, const u32 *__restrict__ l,
                              i64 np, i64 n, u64 *__restrict__ keys, u32 *__restrict__ vals) {
  const i64 p = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const i64 pa = i64(a[p]) + l[p], pb = i64(b[p]) + l[p];
  keys[2 * p] = u64(pa < n ? pa : n);
  keys[2 * p + 1] = u64(pb < n ? pb : n);
  vals[2 * p] = u32(2 * p);
  vals[2 * p + 1] = u32(2 * p + 1);
}

__global__ void k_dsa_gather(const u32 *__restrict__ pos, i64 m, i64 base, const u32 *__restrict__ rank,
                             u32 *__restrict__ out) {
  const i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[k] = rank[i64(pos[k]) - base];
}

// Answers (in sorted request order, the first nvalid requests) back to the
// pairs; a pair extends its lcp by `step` iff both answers exist and agree.
__global__ void k_dsa_lcp_fill(const u32 *__restrict__ resp, const u32 *__restrict__ req, i64 nvalid,
                               u32 *__restrict__ by_req) {
  const i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nvalid) by_req[req[k]] = resp[k];
}

__global__ void k_dsa_lcp_step(u32 *__restrict__ by_req, i64 np, u32 step, u32 *__restrict__ l) {
  const i64 p = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const u32 x = by_req[2 * p], y = by_req[2 * p + 1];
  if (x == y && x != 0xffffffffu) l[p] += step;
  by_req[2 * p] = 0xffffffffu;  // reset for the next level (past-the-end answers stay unequal)
  by_req[2 * p + 1] = 0xfffffffeu;
}

}  // namespace
}  // namespace apo

using namespace apo;

extern "C" {

apo_status apo_dsa_keys(apo_ctx *ctx, const uint32_t *d_rank, const uint32_t *d_rank2, int64_t m, int64_t m2,
                        int64_t base, int64_t n, uint64_t *d_keys, uint32_t *d_vals, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(m >= 0 && m2 >= 0 && m2 <= m && base >= 0 && n >= base + m && n < (i64(1) << 32) - 1,
            "invalid argument");
    if (m == 0) return;
    require(d_rank && d_keys && d_vals && (m2 == 0 || d_rank2), "NULL device pointer");
    k_dsa_keys<<<grid_for(m, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_rank, d_rank2, m, m2, base, n,
                                                                                 d_keys, d_vals);
    APO_CHECK_LAUNCH();
    c.launches++;
  });
}

apo_status apo_dsa_samples(apo_ctx *ctx, const uint64_t *d_keys, const uint32_t *d_vals, int64_t m, int32_t s,
                           uint64_t *d_skeys, uint32_t *d_svals, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(m >= 0 && s >= 1 && d_skeys && d_svals && (m == 0 || (d_keys && d_vals)), "invalid argument");
    k_dsa_samples<<<grid_for(s, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_keys, d_vals, m, s, d_skeys,
                                                                                    d_svals);
    APO_CHECK_LAUNCH();
    c.launches++;
  });
}

apo_status apo_dsa_split(apo_ctx *ctx, const uint64_t *d_keys, const uint32_t *d_vals, int64_t m,
                         const uint64_t *d_split_keys, const uint32_t *d_split_vals, int32_t g, int64_t *d_counts,
                         void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(m >= 0 && g >= 1 && d_counts && (g == 1 || (d_split_keys && d_split_vals)) &&
                (m == 0 || (d_keys && d_vals)),
            "invalid argument");
    k_dsa_split<<<grid_for(g, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(d_keys, d_vals, m, d_split_keys,
                                                                                  d_split_vals, g, d_counts);
    APO_CHECK_LAUNCH();
    c.launches++;
  });
}

apo_status apo_dsa_heads(apo_ctx *ctx, const uint64_t *d_keys, int64_t m, uint64_t prev_key, int32_t has_prev,
                         int64_t gbase, int64_t carry, uint32_t *d_rank, int64_t *d_stats, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(m >= 0 && gbase >= 0 && carry >= -1 && d_stats && (m == 0 || (d_keys && d_rank)) &&
                gbase + m < (i64(1) << 32) - 1,
            "invalid argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const i64 init[2] = {0, -1};
    c.h2d(d_stats, init, sizeof(init), s);
    if (m == 0) return;
    DsaHeadF f{d_keys, m, prev_key, has_prev, gbase, carry, d_rank, d_stats};
    launch_scan<true>(c, m, f, s);
    k_dsa_stats<<<int(std::min<i64>(grid_for(m, 256), 4 * c.num_sms)), 256, 0, s>>>(d_keys, m, prev_key, has_prev,
                                                                                     gbase, d_stats);
    APO_CHECK_LAUNCH();
    c.launches++;
    APO_CUDA(cudaStreamSynchronize(s));  // init came from host stack memory
  });
}

apo_status apo_dsa_scatter(apo_ctx *ctx, const uint32_t *d_pos, const uint32_t *d_rank_in, int64_t m, int64_t base,
                           uint32_t *d_rank, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(m >= 0 && base >= 0 && (m == 0 || (d_pos && d_rank_in && d_rank)), "invalid argument");
    if (m == 0) return;
    k_dsa_scatter<<<grid_for(m, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_pos, d_rank_in, m, base,
                                                                                    d_rank);
    APO_CHECK_LAUNCH();
    c.launches++;
  });
}

apo_status apo_dsa_lcp_requests(apo_ctx *ctx, const uint32_t *d_a, const uint32_t *d_b, const uint32_t *d_l,
                                int64_t np, int64_t n, uint64_t *d_keys, uint32_t *d_vals, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(np >= 0 && n >= 0 && (np == 0 || (d_a && d_b && d_l && d_keys && d_vals)) && 2 * np < (i64(1) << 32),
            "invalid argument");
    if (np == 0) return;
    k_dsa_lcp_req<<<grid_for(np, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_a, d_b, d_l, np, n, d_keys,
                                                                                     d_vals);
    APO_CHECK_LAUNCH();
    c.launches++;
  });
}

apo_status apo_dsa_gather(apo_ctx *ctx, const uint32_t *d_pos, int64_t m, int64_t base, const uint32_t *d_rank,
                          uint32_t *d_out, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(m >= 0 && base >= 0 && (m == 0 || (d_pos && d_rank && d_out)), "invalid argument");
    if (m == 0) return;
    k_dsa_gather<<<grid_for(m, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_pos, m, base, d_rank, d_out);
    APO_CHECK_LAUNCH();
    c.launches++;
  });
}

apo_status apo_dsa_lcp_update(apo_ctx *ctx, const uint32_t *d_resp, const uint32_t *d_req, int64_t nvalid,
                              int64_t np, uint32_t step, uint32_t *d_by_req, uint32_t *d_l, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(nvalid >= 0 && np >= 0 && nvalid <= 2 * np && (np == 0 || (d_by_req && d_l)) &&
                (nvalid == 0 || (d_resp && d_req)),
            "invalid argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (nvalid > 0) {
      k_dsa_lcp_fill<<<grid_for(nvalid, 256), 256, 0, s>>>(d_resp, d_req, nvalid, d_by_req);
      APO_CHECK_LAUNCH();
    }
    if (np > 0) {
      k_dsa_lcp_step<<<grid_for(np, 256), 256, 0, s>>>(d_by_req, np, step, d_l);
      APO_CHECK_LAUNCH();
    }
    c.launches += 2;
  });
}

}  // extern "C"
