// common.cuh -- shared device/host plumbing of libapo (product path only).
//
// Context, workspace arena, error reporting, and the decoupled look-back
// primitive used by the single-pass scans and the onesweep radix sort.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/apo.h"

namespace apo {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i32 = int32_t;
using i64 = int64_t;

constexpr int kNumCounterSlots = 4096;

// --------------------------------------------------------------- errors --
struct Error {
  apo_status code;
  std::string msg;
};

#define APO_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::apo::Error{APO_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                           " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
  } while (0)

#define APO_CHECK_LAUNCH() APO_CUDA(cudaGetLastError())

inline void require(bool ok, const char *what) {
  if (!ok) throw Error{APO_ERR_INVALID, what};
}

// ------------------------------------------------------------ workspace --
// One device arena per context.  A call plans all its buffers, then carves
// them from the arena (grown on demand).  Calls on one context are serialised
// on the caller's stream, so the arena is reused call after call.
struct Arena {
  char *base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  void reserve(size_t bytes, cudaStream_t s) {
    if (bytes <= cap) return;
    if (base) {
      APO_CUDA(cudaStreamSynchronize(s));
      APO_CUDA(cudaFree(base));
      base = nullptr;
      cap = 0;
    }
    size_t want = bytes + bytes / 8 + (64u << 20);
    cudaError_t e = cudaMalloc(&base, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error{APO_ERR_NOMEM, "device workspace allocation of " + std::to_string(want) +
                                      " bytes failed: " + cudaGetErrorString(e)};
    }
    cap = want;
  }
  void release() {
    if (base) cudaFree(base);
    base = nullptr;
    cap = 0;
  }
};

// Bump allocator used in two passes: plan (base == nullptr, only sums sizes)
// then carve (returns pointers).
struct Carver {
  char *base;
  size_t off = 0;
  explicit Carver(char *b) : base(b) {}
  template <class T>
  T *take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += sizeof(T) * (count ? count : 1);
    return p;
  }
};

// Kernel classes timed by the optional in-library profiler (apo_profile).
enum ProfKind {
  kProfRadixPass = 0,  // K1 digit pass (algorithmic HBM bytes known at launch)
  kProfRadixHist = 1,
  kProfScan = 2,
  kProfOther = 3,
  kProfWindowSA = 4,   // K9 (algorithmic shared-memory bytes counted on the device)
  kProfMatch = 5,      // per-stream trace search
  kProfKinds = 6
};
// device-side byte counters of the profiler live in d_misc[kProfDevSlot + kind]
constexpr int kProfDevSlot = 4096;

struct ProfRec {
  int kind;
  double bytes;
  cudaEvent_t a, b;
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  int nsmid = 0;  // %nsmid: SM ids are < nsmid (K9's per-SM scratch)
  std::string err;
  Arena arena;  // per-call scratch
  Arena aux;    // second per-call scratch (trie pieces, match hit keys)
  // cached device blocks for objects that outlive a call (trie storage):
  // reused instead of cudaMalloc/cudaFree every step
  std::vector<std::pair<void *, size_t>> pool;
  void *pool_get(size_t bytes) {
    size_t best = pool.size();
    for (size_t i = 0; i < pool.size(); ++i)
      if (pool[i].second >= bytes && (best == pool.size() || pool[i].second < pool[best].second)) best = i;
    if (best < pool.size()) {
      void *p = pool[best].first;
      pool.erase(pool.begin() + long(best));
      return p;
    }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 1);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error{APO_ERR_NOMEM, "device allocation failed"};
    }
    return p;
  }
  void pool_put(void *p, size_t bytes) {
    if (p) pool.emplace_back(p, bytes);
  }
  // apo_match REPLAY mode: cached MATCH_ALL hit buffer (pooled)
  void *hitbuf = nullptr;
  size_t hitbuf_cap = 0;
  // persistent look-back state (zeroed once; epoch-tagged so never reset)
  u64 *status = nullptr;
  size_t status_words = 0;
  u32 *counters = nullptr;  // tile counters, one slot per launch
  u32 next_counter = 0;
  u32 epoch = 0;
  u32 *h_flag = nullptr;  // pinned host mailbox
  u64 *d_misc = nullptr;  // small device scratch (flags, counts)
  cudaEvent_t ev = nullptr;
  int64_t launches = 0;  // kernel launches issued by the library (for bench)
  // profiler: CUDA events around selected launches, on the launching stream
  bool prof = false;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t prof_event();
  void prof_begin(int kind, double bytes, cudaStream_t s);
  void prof_end(cudaStream_t s);

  void ensure_status(size_t words, cudaStream_t s);
  u32 next_epoch() {
    epoch = (epoch + 1) & 0x3FFFFFFFu;
    if (epoch == 0) epoch = 1;
    return epoch;
  }
  u32 *take_counter(cudaStream_t s);
  u32 read_u32(const u32 *d_ptr, cudaStream_t s);
  u64 read_u64(const u64 *d_ptr, cudaStream_t s);
  // up to 16 consecutive u32 words from the device (synchronises s)
  void read_words(u32 *out, const void *d_src, int nwords, cudaStream_t s);
  // small host -> device uploads (offset tables, scalars): staged in a
  // mapped pinned ring and read by a kernel on `s`.  A copy-engine copy
  // (pageable or pinned) would queue behind any large host -> device
  // transfer other streams have in flight.
  char *h_ring = nullptr;
  size_t ring_off = 0;
  void h2d(void *d_dst, const void *h_src, size_t bytes, cudaStream_t s);
  // device -> pageable host: through a pinned bounce buffer (a pageable
  // copy would wait behind any host -> device transfer in flight), then
  // synchronises `s`
  char *h_bounce = nullptr;
  size_t bounce_cap = 0;
  void d2h(void *h_dst, const void *d_src, size_t bytes, cudaStream_t s);
  // device -> device copies by a kernel on `s` (no copy-engine queue)
  void d2d(void *d_dst, const void *d_src, size_t bytes, cudaStream_t s);
  // dynamic shared-memory opt-ins already applied on THIS context's device
  // (the attribute is per device, so it is tracked per context, not per
  // process)
  std::vector<std::pair<const void *, size_t>> smem_optins;
  void smem_optin(const void *func, size_t bytes) {
    for (auto &e : smem_optins)
      if (e.first == func && e.second >= bytes) return;
    APO_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    smem_optins.emplace_back(func, bytes);
  }
};

// ------------------------------------------------- decoupled look-back --
// Status word: [epoch:30][flag:2][value:32].  flag 1 = aggregate of the
// tile only, 2 = inclusive prefix through the tile.  A word from another
// launch (different epoch) reads as "not yet published".
constexpr u32 kFlagAgg = 1, kFlagInc = 2;

__device__ __forceinline__ u64 lb_pack(u32 epoch, u32 flag, u32 v) {
  return (u64(epoch) << 34) | (u64(flag) << 32) | u64(v);
}
__device__ __forceinline__ void lb_store(u64 *p, u64 w) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ u64 lb_load(const u64 *p) {
  u64 w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

// Sum (IS_MAX = false) or max (IS_MAX = true) of the published values of
// tiles [0, tile) for one lane of the status array (stride = lanes per tile).
template <bool IS_MAX>
__device__ __forceinline__ u32 lb_lookback(const u64 *status, size_t stride, size_t lane,
                                           i64 tile, u32 epoch) {
  // Spin with ONE load on the nearest unresolved predecessor; once it has
  // published, fetch the next seven predecessors' words together (independent
  // loads in flight at once) so a walk over k "aggregate only" tiles costs
  // ~k/8 dependent L2 round trips instead of k.
  constexpr int kLB = 8;
  u32 acc = 0;
  i64 p = tile - 1;
  while (p >= 0) {
    u64 w0 = lb_load(status + size_t(p) * stride + lane);
    u32 ep = u32(w0 >> 34), fl = u32(w0 >> 32) & 3u;
    if (ep != epoch || fl == 0) {  // spin (with backoff) until tile p publishes
      __nanosleep(32);
      continue;
    }
    acc = IS_MAX ? (u32(w0) > acc ? u32(w0) : acc) : acc + u32(w0);
    if (fl == kFlagInc) return acc;
    --p;
    u64 w[kLB - 1];
#pragma unroll
    for (int k = 0; k < kLB - 1; ++k) w[k] = (p - k >= 0) ? lb_load(status + size_t(p - k) * stride + lane) : 0ull;
    int k = 0;
    for (; k < kLB - 1 && p - k >= 0; ++k) {
      ep = u32(w[k] >> 34);
      fl = u32(w[k] >> 32) & 3u;
      if (ep != epoch || fl == 0) break;  // not published yet: spin on it next
      u32 v = u32(w[k]);
      acc = IS_MAX ? (v > acc ? v : acc) : acc + v;
      if (fl == kFlagInc) return acc;
    }
    p -= k;
  }
  return acc;
}

__host__ __device__ inline int bits_for(u64 v) {  // bits needed to store values in [0, v]
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

inline int grid_for(i64 n, int per_block, int cap = 1 << 30) {
  i64 g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return int(g);
}

// ------------------------------------------------------ single-pass scan --
// Generic block-tile scan over u32 values with decoupled look-back.
//   F::load(i) -> u32  (i < n)
//   F::store(i, inclusive, exclusive) -> bool  (true raises *F::flag())
//   F::flag() -> u32* or nullptr
// Op: sum (IS_MAX=false) or max (IS_MAX=true).  One launch, one pass over
// the data, tiles claimed in order through an atomic counter.
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048 (shorter dependent chains per thread)

template <bool IS_MAX>
__device__ __forceinline__ u32 scan_op(u32 a, u32 b) {
  return IS_MAX ? (a > b ? a : b) : a + b;
}

// F::load and F::store are called in a warp-STRIPED order (consecutive
// threads touch consecutive elements, so the functors' own memory accesses
// coalesce); the values are transposed through shared memory so each thread
// scans a contiguous run of kScanItems elements.
template <bool IS_MAX, class F>
__global__ void __launch_bounds__(kScanThreads) k_scan(i64 n, F f, u64 *status, u32 *counter, u32 epoch,
                                                        const u32 *gate) {
  if (gate != nullptr && *gate == 0u) return;  // speculative round after convergence
  // one pad word per 16 keeps both the striped and the blocked accesses
  // bank-conflict free
  __shared__ u32 s_v[kScanTile + kScanTile / 16];  // values
  __shared__ u32 s_e[kScanTile + kScanTile / 16];  // exclusive prefixes
  __shared__ u32 s_warp[kScanThreads / 32];
  __shared__ u32 s_prefix;
  __shared__ u32 s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const i64 tile = s_tile;
  const i64 tbase = tile * kScanTile;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int q = j * kScanThreads + threadIdx.x;
    const i64 i = tbase + q;
    s_v[q + (q >> 4)] = i < n ? f.load(i) : 0u;
  }
  __syncthreads();
  u32 w[kScanItems];
  u32 local = 0;
  const int b0 = threadIdx.x * kScanItems;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    w[j] = s_v[b0 + j + ((b0 + j) >> 4)];
    local = scan_op<IS_MAX>(local, w[j]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 incl = local;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    u32 o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl = scan_op<IS_MAX>(incl, o);
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u32 x = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
    u32 wi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u32 o = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi = scan_op<IS_MAX>(wi, o);
    }
    u32 wex = __shfl_up_sync(0xffffffffu, wi, 1);
    u32 tile_total = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    if (lane < kScanThreads / 32) s_warp[lane] = lane ? wex : 0u;  // exclusive warp prefix
    if (lane == 0) {
      if (tile == 0) {
        lb_store(status, lb_pack(epoch, kFlagInc, tile_total));
        s_prefix = 0;
      } else {
        lb_store(status + tile, lb_pack(epoch, kFlagAgg, tile_total));
        u32 pre = lb_lookback<IS_MAX>(status, 1, 0, tile, epoch);
        lb_store(status + tile, lb_pack(epoch, kFlagInc, scan_op<IS_MAX>(pre, tile_total)));
        s_prefix = pre;
      }
    }
  }
  __syncthreads();
  // exclusive prefix of each element back into shared memory (blocked)
  u32 warp_excl_in = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) warp_excl_in = 0;
  u32 run = scan_op<IS_MAX>(scan_op<IS_MAX>(s_prefix, s_warp[warp]), warp_excl_in);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    s_e[b0 + j + ((b0 + j) >> 4)] = run;  // exclusive prefix of element b0 + j
    run = scan_op<IS_MAX>(run, w[j]);
  }
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int q = j * kScanThreads + threadIdx.x;
    const i64 i = tbase + q;
    if (i < n) {
      const u32 ex = s_e[q + (q >> 4)];
      any |= f.store(i, scan_op<IS_MAX>(ex, s_v[q + (q >> 4)]), ex);
    }
  }
  u32 *fl = f.flag();
  if (fl != nullptr) {
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(fl, 1u);
  }
}

template <bool IS_MAX, class F>
void launch_scan(Ctx &c, i64 n, const F &f, cudaStream_t s, const u32 *gate = nullptr) {
  if (n <= 0) return;
  i64 tiles = (n + kScanTile - 1) / kScanTile;
  c.ensure_status(size_t(tiles), s);
  u32 *ctr = c.take_counter(s);
  u32 ep = c.next_epoch();
  if (c.prof) c.prof_begin(kProfScan, 0.0, s);
  k_scan<IS_MAX, F><<<int(tiles), kScanThreads, 0, s>>>(n, f, c.status, ctr, ep, gate);
  APO_CHECK_LAUNCH();
  if (c.prof) c.prof_end(s);
  c.launches++;
}

// ----------------------------------------------------- radix sort (K1) --
// LSD onesweep radix sort of (u64 key, V value) pairs (V = u32, u64, or
// void for keys only) over key bits [begin_bit, end_bit).  Stable.  Returns
// true iff the result ended in the *_alt buffers.
// gate (optional, device): the whole sort is skipped when *gate == 0
bool radix_sort_u64_u32(Ctx &c, u64 *keys, u32 *vals, u64 *keys_alt, u32 *vals_alt, i64 n,
                        int begin_bit, int end_bit, cudaStream_t s, const u32 *gate = nullptr);
bool radix_sort_u64_keys(Ctx &c, u64 *keys, u64 *keys_alt, i64 n, int begin_bit, int end_bit,
                         cudaStream_t s);
bool radix_sort_u32_u64(Ctx &c, u32 *keys, u64 *vals, u32 *keys_alt, u64 *vals_alt, i64 n,
                        int begin_bit, int end_bit, cudaStream_t s);
size_t radix_status_words(i64 n);

}  // namespace apo

struct apo_ctx {
  apo::Ctx c;
};

namespace apo {
// Entry-point wrapper: selects the context's device, maps exceptions to
// status codes and the context's error text.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class Fn>
apo_status guarded(apo_ctx *ctx, Fn &&fn) {
  if (ctx == nullptr) return APO_ERR_INVALID;
  ctx->c.err.clear();
  try {
    DeviceGuard g(ctx->c.device);
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
}  // namespace apo
