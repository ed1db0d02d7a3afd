// radix_sort.cu -- K1: in-house LSD "onesweep" radix sort for sm_100a.
//
// Used for the prefix-doubling suffix sort (SA, P:552 / P:606-607) and the
// candidate sort of Alg. 2 ("Sort(C)").
//
// Design (B200-first):
//  * one upfront histogram kernel computes the digit histograms of ALL
//    passes in a single read of the keys (warp-aggregated shared atomics);
//  * one kernel per digit pass: each 256-thread CTA takes a 4,096-key tile
//    (tiles claimed in order through an atomic counter), loads keys
//    warp-striped (fully coalesced 256 B per warp instruction), ranks them
//    with a warp multisplit (peer mask from BITS ballots; measured 12 %
//    faster than __match_any_sync on B200) into per-warp shared-memory
//    histograms, publishes its per-digit tile counts with decoupled look-back
//    (epoch-tagged 64-bit status words: no memset between passes), stages the
//    tile in shared memory in sorted order and writes runs of equal digits
//    contiguously (coalesced scatter);
//  * digits are 8 or 9 bits: the bit range is split into ceil(bits/9) passes,
//    so e.g. 41-bit doubling keys take 5 passes, not 6.
// Stable: ties keep their input order.
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "common.cuh"

namespace apo {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kMaxRadix = 512;
constexpr int kMaxPasses = 8;

struct NoVal {};

struct PassPlan {
  int npass;
  int shift[kMaxPasses];
  int bits[kMaxPasses];
};

// Lanes of `mask` whose digit equals this lane's digit, from BITS ballots
// (the warp multisplit of onesweep; an alternative to __match_any_sync).
template <int BITS>
__device__ __forceinline__ u32 peers_ballot(u32 mask, u32 d) {
  u32 peers = mask;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const u32 m = __ballot_sync(mask, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// match.any: one instruction instead of BITS ballots (measured 4 % faster
// on the C5 sort passes, 1 % on C3)
template <int BITS>
__device__ __forceinline__ u32 peers_of(u32 mask, u32 d) {
  return __match_any_sync(mask, d);
}

__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class K>
__global__ void __launch_bounds__(kSortThreads) k_hist(const K *__restrict__ keys, i64 n, PassPlan plan,
                                                       u32 *__restrict__ ghist, const u32 *gate) {
  if (gate != nullptr && *gate == 0u) return;  // speculative round after convergence
  __shared__ u32 sh[kMaxPasses * kMaxRadix];
  for (int i = threadIdx.x; i < plan.npass * kMaxRadix; i += kSortThreads) sh[i] = 0;
  __syncthreads();
  int shift[kMaxPasses];
  u32 mask[kMaxPasses];
#pragma unroll
  for (int p = 0; p < kMaxPasses; ++p) {
    shift[p] = p < plan.npass ? plan.shift[p] : 0;
    mask[p] = p < plan.npass ? (1u << plan.bits[p]) - 1u : 0u;
  }
  const i64 stride = i64(gridDim.x) * kSortThreads;
  for (i64 i = i64(blockIdx.x) * kSortThreads + threadIdx.x; i < n; i += stride) {
    K k = keys[i];
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p)
      if (p < plan.npass) atomicAdd(&sh[p * kMaxRadix + (u32(u64(k) >> shift[p]) & mask[p])], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < plan.npass * kMaxRadix; i += kSortThreads)
    if (sh[i]) atomicAdd(&ghist[i], sh[i]);
}

// Block-wide exclusive scan of RADIX bins; thread t owns bins t*BPT..t*BPT+BPT-1.
template <int BPT>
__device__ __forceinline__ void block_excl_scan_bins(const u32 (&v)[BPT], u32 (&ex)[BPT], u32 *s_tmp) {
  u32 tsum = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) tsum += v[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    u32 o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_tmp[warp] = incl;
  __syncthreads();
  u32 wpre = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) wpre += (w < warp) ? s_tmp[w] : 0u;
  u32 run = wpre + incl - tsum;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    ex[q] = run;
    run += v[q];
  }
  __syncthreads();
}

template <class K, class V, int BITS>
__global__ void __launch_bounds__(kSortThreads, 3) k_onesweep(const K *__restrict__ kin, K *__restrict__ kout,
                                                           const V *__restrict__ vin, V *__restrict__ vout,
                                                           i64 n, int shift, int pbits,
                                                           const u32 *__restrict__ ghist, u64 *status,
                                                           u32 *counter, u32 epoch, const u32 *gate) {
  if (gate != nullptr && *gate == 0u) return;  // speculative round after convergence
  constexpr bool HAS_V = !std::is_same<V, NoVal>::value;
  constexpr int RADIX = 1 << BITS;
  constexpr int BPT = RADIX / kSortThreads;
  extern __shared__ __align__(16) unsigned char smem[];
  K *s_keys = reinterpret_cast<K *>(smem);
  V *s_vals = reinterpret_cast<V *>(smem + sizeof(K) * kSortTile);
  u32 *s_whist = reinterpret_cast<u32 *>(smem + (sizeof(K) + (HAS_V ? sizeof(V) : 0)) * kSortTile);
  __shared__ u32 s_start[RADIX];  // block-local exclusive digit start
  __shared__ u32 s_adj[RADIX];    // global position = s_adj[d] + local position
  __shared__ u32 s_tmp[kSortWarps];
  __shared__ u32 s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  for (int i = tid; i < kSortWarps * RADIX; i += kSortThreads) s_whist[i] = 0;
  __syncthreads();
  const i64 tile = s_tile;
  const i64 tbase = tile * kSortTile;
  const i64 wbase = tbase + i64(warp) * (32 * kSortItems);
  const u32 dmask = (1u << pbits) - 1u;

  if constexpr (HAS_V) {
    // values are read only after ranking: warm L2 with this tile's values now
    // (TMA bulk prefetch; measured +5 % per pass on B200)
    if (tid == 0) {
      const i64 nb = (n - tbase) < kSortTile ? (n - tbase) : kSortTile;
      const u32 bytes = u32(nb * sizeof(V)) & ~15u;
      if (bytes >= 16 && (reinterpret_cast<unsigned long long>(vin + tbase) & 15ull) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vin + tbase), "r"(bytes) : "memory");
    }
  }
  K key[kSortItems];
  u32 rk[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    i64 idx = wbase + j * 32 + lane;
    if (idx < n) key[j] = kin[idx];
  }
  u32 *wh = s_whist + warp * RADIX;
  const u32 lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    i64 idx = wbase + j * 32 + lane;
    bool valid = idx < n;
    u32 vmask = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      u32 d = u32(u64(key[j]) >> shift) & dmask;
      u32 peers = peers_of<BITS>(vmask, d);
      u32 old = wh[d];
      __syncwarp(vmask);
      if (lane == __ffs(peers) - 1) wh[d] = old + __popc(peers);
      __syncwarp(vmask);
      rk[j] = old + __popc(peers & lt);
    }
  }
  __syncthreads();

  // per-digit: warp exclusive offsets, tile count, global base
  u32 cnt[BPT], gb[BPT], ex[BPT];
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const int d = tid * BPT + q;
    u32 run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      u32 c = s_whist[w * RADIX + d];
      s_whist[w * RADIX + d] = run;
      run += c;
    }
    cnt[q] = run;
    gb[q] = ghist[d];
    if (tile == 0)
      lb_store(status + d, lb_pack(epoch, kFlagInc, run));
    else
      lb_store(status + size_t(tile) * RADIX + d, lb_pack(epoch, kFlagAgg, run));
  }
  // global exclusive digit base (scan of the pass histogram) and local starts
  u32 gex[BPT];
  block_excl_scan_bins<BPT>(gb, gex, s_tmp);
  block_excl_scan_bins<BPT>(cnt, ex, s_tmp);
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const int d = tid * BPT + q;
    u32 pre = 0;
    if (tile > 0) {
      pre = lb_lookback<false>(status, RADIX, d, tile, epoch);
      lb_store(status + size_t(tile) * RADIX + d, lb_pack(epoch, kFlagInc, pre + cnt[q]));
    }
    s_start[d] = ex[q];
    s_adj[d] = gex[q] + pre - ex[q];
  }
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    i64 idx = wbase + j * 32 + lane;
    if (idx < n) {
      u32 d = u32(u64(key[j]) >> shift) & dmask;
      rk[j] += s_start[d] + wh[d];  // block-local sorted position
      s_keys[rk[j]] = key[j];
    }
  }
  if constexpr (HAS_V) {
    // values are loaded only now (keeps registers low during ranking)
    V val[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      i64 idx = wbase + j * 32 + lane;
      if (idx < n) val[j] = vin[idx];
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      i64 idx = wbase + j * 32 + lane;
      if (idx < n) s_vals[rk[j]] = val[j];
    }
  }
  __syncthreads();
  const i64 rem = n - tbase;
  const int tvalid = rem < kSortTile ? int(rem) : kSortTile;
  for (int i = tid; i < tvalid; i += kSortThreads) {
    K k = s_keys[i];
    u32 d = u32(u64(k) >> shift) & dmask;
    u32 g = s_adj[d] + u32(i);
    kout[g] = k;
    if constexpr (HAS_V) vout[g] = s_vals[i];
  }
}


PassPlan plan_passes(int begin_bit, int end_bit) {
  PassPlan p{};
  int B = end_bit - begin_bit;
  int P = (B + 8) / 9;
  if (P > kMaxPasses) P = kMaxPasses;
  while (P * 9 < B) ++P;  // cannot happen for <= 64 bits
  p.npass = P;
  int sh = begin_bit;
  for (int i = 0; i < P; ++i) {
    int b = B / P + (i < B % P ? 1 : 0);
    p.shift[i] = sh;
    p.bits[i] = b;
    sh += b;
  }
  return p;
}

template <class K, class V, int BITS>
void launch_pass(Ctx &c, const K *kin, K *kout, const V *vin, V *vout, i64 n, int shift, int pbits,
                 const u32 *ghist, cudaStream_t s, const u32 *gate) {
  constexpr bool HAS_V = !std::is_same<V, NoVal>::value;
  constexpr int RADIX = 1 << BITS;
  const size_t smem = (sizeof(K) + (HAS_V ? sizeof(V) : 0)) * kSortTile + sizeof(u32) * kSortWarps * RADIX;
  c.smem_optin(reinterpret_cast<const void *>(k_onesweep<K, V, BITS>), smem);
  const i64 tiles = (n + kSortTile - 1) / kSortTile;
  c.ensure_status(size_t(tiles) * RADIX, s);
  u32 *ctr = c.take_counter(s);
  u32 ep = c.next_epoch();
  // algorithmic bytes: every (key, value) read once and written once
  if (c.prof) c.prof_begin(kProfRadixPass, 2.0 * double(n) * double(sizeof(K) + (HAS_V ? sizeof(V) : 0)), s);
  k_onesweep<K, V, BITS><<<int(tiles), kSortThreads, smem, s>>>(kin, kout, vin, vout, n, shift, pbits, ghist,
                                                                 c.status, ctr, ep, gate);
  APO_CHECK_LAUNCH();
  if (c.prof) c.prof_end(s);
  c.launches++;
}

template <class K, class V>
bool radix_sort(Ctx &c, K *keys, V *vals, K *keys_alt, V *vals_alt, i64 n, int begin_bit, int end_bit,
                cudaStream_t s, const u32 *gate = nullptr) {
  if (n <= 1 || end_bit <= begin_bit) return false;
  PassPlan plan = plan_passes(begin_bit, end_bit);
  u32 *ghist = reinterpret_cast<u32 *>(c.d_misc + 64);  // kMaxPasses * kMaxRadix u32
  APO_CUDA(cudaMemsetAsync(ghist, 0, sizeof(u32) * kMaxPasses * kMaxRadix, s));
  int hg = grid_for(n, kSortThreads * 16, c.num_sms * 8);
  if (c.prof) c.prof_begin(kProfRadixHist, double(n) * sizeof(K), s);
  k_hist<K><<<hg, kSortThreads, 0, s>>>(keys, n, plan, ghist, gate);
  APO_CHECK_LAUNCH();
  if (c.prof) c.prof_end(s);
  c.launches++;
  K *ki = keys, *ko = keys_alt;
  V *vi = vals, *vo = vals_alt;
  for (int p = 0; p < plan.npass; ++p) {
    const u32 *gh = ghist + p * kMaxRadix;
    if (plan.bits[p] > 8)
      launch_pass<K, V, 9>(c, ki, ko, vi, vo, n, plan.shift[p], plan.bits[p], gh, s, gate);
    else
      launch_pass<K, V, 8>(c, ki, ko, vi, vo, n, plan.shift[p], plan.bits[p], gh, s, gate);
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  return (plan.npass & 1) != 0;
}

}  // namespace

size_t radix_status_words(i64 n) { return size_t((n + kSortTile - 1) / kSortTile) * kMaxRadix; }

bool radix_sort_u64_u32(Ctx &c, u64 *keys, u32 *vals, u64 *keys_alt, u32 *vals_alt, i64 n, int begin_bit,
                        int end_bit, cudaStream_t s, const u32 *gate) {
  return radix_sort<u64, u32>(c, keys, vals, keys_alt, vals_alt, n, begin_bit, end_bit, s, gate);
}
bool radix_sort_u64_keys(Ctx &c, u64 *keys, u64 *keys_alt, i64 n, int begin_bit, int end_bit, cudaStream_t s) {
  return radix_sort<u64, NoVal>(c, keys, (NoVal *)nullptr, keys_alt, (NoVal *)nullptr, n, begin_bit, end_bit, s);
}
bool radix_sort_u32_u64(Ctx &c, u32 *keys, u64 *vals, u32 *keys_alt, u64 *vals_alt, i64 n, int begin_bit,
                        int end_bit, cudaStream_t s) {
  return radix_sort<u32, u64>(c, keys, vals, keys_alt, vals_alt, n, begin_bit, end_bit, s);
}

}  // namespace apo
