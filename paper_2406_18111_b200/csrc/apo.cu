// apo.cu -- the C ABI (include/apo.h) of libapo.
//
// Argument checking, workspace planning and stage sequencing; every step of
// the hot path runs in the CUDA kernels of radix_sort.cu, suffix_array.cu and
// select.cu.  There is no CPU fallback.
#include <cstring>
#include <vector>

#include "pipeline.cuh"

namespace apo {

void Ctx::ensure_status(size_t words, cudaStream_t s) {
  if (words <= status_words) return;
  size_t want = words + words / 2 + 4096;
  if (status) {
    APO_CUDA(cudaStreamSynchronize(s));
    APO_CUDA(cudaFree(status));
    status = nullptr;
    status_words = 0;
  }
  cudaError_t e = cudaMalloc(&status, want * sizeof(u64));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{APO_ERR_NOMEM, "look-back status allocation failed"};
  }
  APO_CUDA(cudaMemsetAsync(status, 0, want * sizeof(u64), s));
  status_words = want;
}

u32 *Ctx::take_counter(cudaStream_t s) {
  if (next_counter >= kNumCounterSlots) {
    APO_CUDA(cudaMemsetAsync(counters, 0, sizeof(u32) * kNumCounterSlots, s));
    next_counter = 0;
  }
  return counters + next_counter++;
}

namespace {
constexpr size_t kRingBytes = size_t(8) << 20;

__global__ void k_d2d_16(uint4 *__restrict__ dst, const uint4 *__restrict__ src, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_h2d_words(u32 *__restrict__ dst, const u32 *__restrict__ src, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

void Ctx::h2d(void *d_dst, const void *h_src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  const size_t need = (bytes + 255) & ~size_t(255);
  if ((bytes & 3) != 0 || (reinterpret_cast<uintptr_t>(d_dst) & 3) != 0 || need > kRingBytes) {
    APO_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  if (h_ring == nullptr) APO_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&h_ring), kRingBytes, cudaHostAllocMapped));
  if (ring_off + need > kRingBytes) {  // wrap: every earlier upload must have been read
    APO_CUDA(cudaDeviceSynchronize());
    ring_off = 0;
  }
  char *slot = h_ring + ring_off;
  ring_off += need;
  std::memcpy(slot, h_src, bytes);
  // SM reads of the mapped ring: a copy-engine copy, even from pinned
  // memory, would wait behind every host -> device transfer already queued
  // by other streams (measured: the bench's 1 GB double-buffered input
  // upload delayed each analysis call by ~16 ms)
  if ((bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(d_dst) & 15) == 0) {
    const size_t n = bytes / 16;
    k_d2d_16<<<grid_for(i64(n), 128, 512), 128, 0, s>>>(static_cast<uint4 *>(d_dst),
                                                        reinterpret_cast<const uint4 *>(slot), n);
  } else {
    const size_t n = bytes / 4;
    k_h2d_words<<<grid_for(i64(n), 128, 512), 128, 0, s>>>(static_cast<u32 *>(d_dst),
                                                           reinterpret_cast<const u32 *>(slot), n);
  }
  APO_CHECK_LAUNCH();
  launches++;
}



void Ctx::d2d(void *d_dst, const void *d_src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (((reinterpret_cast<uintptr_t>(d_dst) | reinterpret_cast<uintptr_t>(d_src) | bytes) & 15) != 0) {
    if ((bytes & 3) == 0 && ((reinterpret_cast<uintptr_t>(d_dst) | reinterpret_cast<uintptr_t>(d_src)) & 3) == 0) {
      k_h2d_words<<<grid_for(i64(bytes / 4), 256, num_sms * 8), 256, 0, s>>>(
          static_cast<u32 *>(d_dst), static_cast<const u32 *>(d_src), bytes / 4);
      APO_CHECK_LAUNCH();
      launches++;
      return;
    }
    APO_CUDA(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  const size_t n = bytes / 16;
  k_d2d_16<<<grid_for(i64(n), 256, num_sms * 8), 256, 0, s>>>(static_cast<uint4 *>(d_dst),
                                                              static_cast<const uint4 *>(d_src), n);
  APO_CHECK_LAUNCH();
  launches++;
}

void Ctx::d2h(void *h_dst, const void *d_src, size_t bytes, cudaStream_t s) {
  if (bytes > bounce_cap) {
    if (h_bounce) APO_CUDA(cudaFreeHost(h_bounce));
    h_bounce = nullptr;
    bounce_cap = 0;
    const size_t want = std::max(bytes + bytes / 2, size_t(1) << 20);
    APO_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&h_bounce), want, cudaHostAllocMapped));
    bounce_cap = want;
  }
  if (bytes && (bytes & 3) == 0 && (reinterpret_cast<uintptr_t>(d_src) & 3) == 0 && bytes <= (size_t(4) << 20)) {
    // small: a kernel writes the mapped bounce buffer (no copy-engine queue)
    k_h2d_words<<<grid_for(i64(bytes / 4), 256, 64), 256, 0, s>>>(reinterpret_cast<u32 *>(h_bounce),
                                                                static_cast<const u32 *>(d_src), bytes / 4);
    APO_CHECK_LAUNCH();
    launches++;
  } else if (bytes) {
    APO_CUDA(cudaMemcpyAsync(h_bounce, d_src, bytes, cudaMemcpyDeviceToHost, s));
  }
  APO_CUDA(cudaStreamSynchronize(s));
  if (bytes) std::memcpy(h_dst, h_bounce, bytes);
}

namespace {
__global__ void k_read_words(const u32 *__restrict__ src, volatile u32 *dst, int n) {
  if (threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}
}  // namespace

// Scalars read back by a one-thread kernel into the mapped pinned mailbox
// (a copy-engine read would queue behind a host -> device transfer that
// another stream has in flight).
u32 Ctx::read_u32(const u32 *d_ptr, cudaStream_t s) {
  k_read_words<<<1, 32, 0, s>>>(d_ptr, h_flag, 1);
  APO_CHECK_LAUNCH();
  launches++;
  APO_CUDA(cudaStreamSynchronize(s));
  return reinterpret_cast<volatile u32 *>(h_flag)[0];
}

void Ctx::read_words(u32 *out, const void *d_src, int nwords, cudaStream_t s) {
  if (nwords < 1 || nwords > 16) throw Error{APO_ERR_INVALID, "read_words: 1..16 words"};
  k_read_words<<<1, 32, 0, s>>>(static_cast<const u32 *>(d_src), h_flag, nwords);
  APO_CHECK_LAUNCH();
  launches++;
  APO_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < nwords; ++i) out[i] = reinterpret_cast<volatile u32 *>(h_flag)[i];
}

u64 Ctx::read_u64(const u64 *d_ptr, cudaStream_t s) {
  k_read_words<<<1, 32, 0, s>>>(reinterpret_cast<const u32 *>(d_ptr), h_flag, 2);
  APO_CHECK_LAUNCH();
  launches++;
  APO_CUDA(cudaStreamSynchronize(s));
  u64 v;
  std::memcpy(&v, const_cast<const u32 *>(reinterpret_cast<volatile u32 *>(h_flag)), sizeof(u64));
  return v;
}

cudaEvent_t Ctx::prof_event() {
  if (ev_used == ev_pool.size()) {
    cudaEvent_t e;
    APO_CUDA(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[ev_used++];
}

void Ctx::prof_begin(int kind, double bytes, cudaStream_t s) {
  ProfRec r{kind, bytes, prof_event(), prof_event()};
  APO_CUDA(cudaEventRecord(r.a, s));
  prof_recs.push_back(r);
}

void Ctx::prof_end(cudaStream_t s) { APO_CUDA(cudaEventRecord(prof_recs.back().b, s)); }

namespace {


// position -> window map: one CTA per window fills its range (coalesced)
__global__ void k_fill_wid(const i64 *__restrict__ off, int W, i64 N, i32 *__restrict__ wid) {
  const int w = blockIdx.x;
  if (w >= W) return;
  const i64 e = off[w + 1];
  for (i64 i = off[w] + threadIdx.x; i < e; i += blockDim.x) wid[i] = w;
}

__global__ void k_localize_sa(const i32 *__restrict__ sa, Batch b, i32 *__restrict__ out) {
  i64 k = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= b.N) return;
  i64 i = sa[k];
  out[k] = i32(i - b_beg(b, b_wid(b, i)));
}

// Validated batch description + device copies of offsets/window ids.
struct BatchSetup {
  Batch b;
  i64 *d_off = nullptr;
  i32 *d_wid = nullptr;
};

void check_offsets(const i64 *h_off, int nwin) {
  require(nwin >= 1, "nwin must be >= 1");
  require(h_off != nullptr, "h_off is NULL");
  require(h_off[0] == 0, "h_off[0] must be 0");
  for (int w = 0; w < nwin; ++w) {
    require(h_off[w + 1] >= h_off[w], "h_off must be non-decreasing");
    require(h_off[w + 1] - h_off[w] <= (i64(1) << 30), "window longer than 2^30 tokens");
  }
  require(h_off[nwin] < (i64(1) << 31) - 1, "batch longer than 2^31-1 tokens");
}

Batch describe(const i64 *h_off, int nwin) {
  Batch b;
  b.N = h_off[nwin];
  b.W = nwin;
  b.maxwin = 0;
  for (int w = 0; w < nwin; ++w) b.maxwin = std::max<i64>(b.maxwin, h_off[w + 1] - h_off[w]);
  return b;
}

// Plans the workspace of one call; carve == true returns pointers.
struct Plan {
  SAWork sa{};
  SelWork sel{};
  i64 *d_off = nullptr;
  i32 *d_wid = nullptr;
  size_t bytes = 0;
};

void plan_all(Carver &cv, Batch &b, Plan &p, bool want_lcp, bool want_select, int nsmid, int min_len) {
  if (b.W > 1) {
    p.d_off = cv.take<i64>(size_t(b.W) + 1);
    p.d_wid = cv.take<i32>(size_t(b.N));
  }
  plan_sa(cv, b, p.sa, want_lcp || want_select, nsmid);
  if (want_select) plan_select(cv, b, p.sel, min_len);
}

Plan setup(Ctx &c, Batch &b, const i64 *h_off, bool want_lcp, bool want_select, cudaStream_t s,
           int min_len = 1) {
  Plan p;
  Carver dry(nullptr);
  plan_all(dry, b, p, want_lcp, want_select, c.nsmid, min_len);
  c.arena.reserve(dry.off, s);
  Carver cv(c.arena.base);
  plan_all(cv, b, p, want_lcp, want_select, c.nsmid, min_len);
  if (b.W > 1) {
    c.h2d(p.d_off, h_off, sizeof(i64) * (b.W + 1), s);
    k_fill_wid<<<b.W, 256, 0, s>>>(p.d_off, b.W, b.N, p.d_wid);
    APO_CHECK_LAUNCH();
    c.launches++;
    b.off = p.d_off;
    b.wid = p.d_wid;
  }
  return p;
}

}  // namespace
}  // namespace apo

using namespace apo;

extern "C" {

int apo_version(void) { return 1; }

apo_status apo_ctx_create(int cuda_device, apo_ctx **out) {
  if (out == nullptr) return APO_ERR_INVALID;
  *out = nullptr;
  apo_ctx *ctx = new apo_ctx();
  ctx->c.device = cuda_device;
  apo_status st = guarded(ctx, [&](Ctx &c) {
    APO_CUDA(cudaSetDevice(cuda_device));
    APO_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, cuda_device));
    c.nsmid = query_nsmid(cuda_device);
    APO_CUDA(cudaMalloc(&c.counters, sizeof(u32) * kNumCounterSlots));
    APO_CUDA(cudaMemset(c.counters, 0, sizeof(u32) * kNumCounterSlots));
    APO_CUDA(cudaMalloc(&c.d_misc, 64 * 1024));
    APO_CUDA(cudaMemset(c.d_misc, 0, 64 * 1024));
    APO_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&c.h_flag), 64, cudaHostAllocMapped));
    APO_CUDA(cudaDeviceSynchronize());
  });
  if (st != APO_OK) {
    apo_ctx_destroy(ctx);
    return st;
  }
  *out = ctx;
  return APO_OK;
}

void apo_ctx_destroy(apo_ctx *ctx) {
  if (!ctx) return;
  Ctx &c = ctx->c;
  cudaSetDevice(c.device);
  cudaDeviceSynchronize();
  c.arena.release();
  c.aux.release();
  if (c.hitbuf) cudaFree(c.hitbuf);
  for (auto &b : c.pool) cudaFree(b.first);
  for (auto e : c.ev_pool) cudaEventDestroy(e);
  if (c.status) cudaFree(c.status);
  if (c.counters) cudaFree(c.counters);
  if (c.d_misc) cudaFree(c.d_misc);
  if (c.h_flag) cudaFreeHost(c.h_flag);
  if (c.h_ring) cudaFreeHost(c.h_ring);
  if (c.h_bounce) cudaFreeHost(c.h_bounce);
  delete ctx;
}

const char *apo_last_error(const apo_ctx *ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

int64_t apo_launch_count(const apo_ctx *ctx) { return ctx ? ctx->c.launches : 0; }

apo_status apo_profile(apo_ctx *ctx, int enable) {
  return guarded(ctx, [&](Ctx &c) {
    c.prof = enable != 0;
    if (c.prof) {
      c.prof_recs.clear();
      c.ev_used = 0;
      APO_CUDA(cudaMemset(c.d_misc + kProfDevSlot, 0, sizeof(u64) * kProfKinds));
    }
  });
}

apo_status apo_profile_read(apo_ctx *ctx, int kind, double *ms, int64_t *launches, double *bytes) {
  return guarded(ctx, [&](Ctx &c) {
    require(kind >= 0 && kind < kProfKinds, "bad profile kind");
    double t = 0, by = 0;
    int64_t k = 0;
    for (auto &r : c.prof_recs) {
      if (r.kind != kind) continue;
      APO_CUDA(cudaEventSynchronize(r.b));
      float f = 0;
      APO_CUDA(cudaEventElapsedTime(&f, r.a, r.b));
      t += f;
      by += r.bytes;
      ++k;
    }
    u64 dev_bytes = 0;  // bytes counted by the kernels themselves
    APO_CUDA(cudaMemcpy(&dev_bytes, c.d_misc + kProfDevSlot + kind, sizeof(u64), cudaMemcpyDeviceToHost));
    by += double(dev_bytes);
    if (ms) *ms = t;
    if (launches) *launches = k;
    if (bytes) *bytes = by;
  });
}

static apo_status sa_common(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off, int32_t nwin,
                            int32_t *d_sa, int32_t *d_lcp, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    check_offsets(h_off, nwin);
    Batch b = describe(h_off, nwin);
    if (b.N == 0) return;
    require(d_tok != nullptr && d_sa != nullptr, "NULL device pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Plan p = setup(c, b, h_off, d_lcp != nullptr, false, s);
    build_sa(c, d_tok, b, p.sa, d_lcp != nullptr, s);
    k_localize_sa<<<grid_for(b.N, 256), 256, 0, s>>>(p.sa.sa, b, d_sa);
    APO_CHECK_LAUNCH();
    c.launches++;
    if (d_lcp) c.d2d(d_lcp, p.sa.lcp, sizeof(i32) * b.N, s);
  });
}

apo_status apo_suffix_array(apo_ctx *ctx, const uint64_t *d_tok, int32_t n, int32_t *d_sa, int32_t *d_lcp,
                            void *stream) {
  if (n < 0) return APO_ERR_INVALID;
  int64_t off[2] = {0, n};
  return sa_common(ctx, d_tok, off, 1, d_sa, d_lcp, stream);
}

apo_status apo_suffix_array_batched(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off, int32_t nwin,
                                    int32_t *d_sa, int32_t *d_lcp, void *stream) {
  return sa_common(ctx, d_tok, h_off, nwin, d_sa, d_lcp, stream);
}

apo_status apo_radix_sort(apo_ctx *ctx, uint64_t *d_keys, uint32_t *d_vals, int64_t n, int32_t begin_bit,
                          int32_t end_bit, void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(n >= 0 && begin_bit >= 0 && end_bit <= 64 && begin_bit <= end_bit, "invalid argument");
    require(n < (i64(1) << 32), "n must be < 2^32");
    if (n <= 1 || begin_bit == end_bit) return;
    require(d_keys != nullptr, "NULL device pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    u64 *ka;
    u32 *va = nullptr;
    Carver dry(nullptr);
    dry.take<u64>(n);
    if (d_vals) dry.take<u32>(n);
    c.arena.reserve(dry.off, s);
    Carver cv(c.arena.base);
    ka = cv.take<u64>(n);
    if (d_vals) va = cv.take<u32>(n);
    bool alt = d_vals ? radix_sort_u64_u32(c, d_keys, d_vals, ka, va, n, begin_bit, end_bit, s)
                      : radix_sort_u64_keys(c, d_keys, ka, n, begin_bit, end_bit, s);
    if (alt) {
      c.d2d(d_keys, ka, sizeof(u64) * n, s);
      if (d_vals) c.d2d(d_vals, va, sizeof(u32) * n, s);
    }
  });
}

apo_status apo_candidates(apo_ctx *ctx, const uint64_t *d_tok, int32_t n, int32_t min_len, int32_t *d_len,
                          int32_t *d_id, int32_t *d_start, uint8_t *d_kept, int64_t cap, int64_t *d_count,
                          void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(n >= 0 && min_len >= 1 && cap >= 0 && d_count != nullptr, "invalid argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
      APO_CUDA(cudaMemsetAsync(d_count, 0, sizeof(i64), s));
      return;
    }
    require(d_tok != nullptr, "NULL device pointer");
    int64_t off[2] = {0, n};
    Batch b = describe(off, 1);
    Plan p = setup(c, b, off, true, true, s, min_len);
    build_sa(c, d_tok, b, p.sa, true, s);
    select_candidates(c, d_tok, b, p.sa, min_len, p.sel, s);
    emit_candidates(c, b, p.sel, d_len, d_id, d_start, d_kept, cap, d_count, s);
  });
}

static apo_status find_common(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off, int32_t nwin,
                              int32_t min_len, const apo_params *params, apo_repeat *d_out, int64_t cap,
                              int64_t *d_out_off, int32_t *d_occ, int64_t occ_cap, int64_t *d_counts,
                              void *stream) {
  return guarded(ctx, [&](Ctx &c) {
    require(min_len >= 1, "min_len must be >= 1");
    require(cap >= 0 && occ_cap >= 0, "negative capacity");
    require(d_counts != nullptr, "d_counts is NULL");
    require(cap == 0 || d_out != nullptr, "d_out is NULL");
    require(occ_cap == 0 || d_occ != nullptr, "d_occ is NULL");
    apo_params prm{1, 0, 0, 0};
    if (params) prm = *params;
    require(prm.min_count >= 1, "min_count must be >= 1");
    require(prm.flags == 0 && prm.reserved == 0, "reserved params must be 0");
    check_offsets(h_off, nwin);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Batch b = describe(h_off, nwin);
    if (b.N == 0 || b.maxwin < 2 * i64(min_len)) {
      APO_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(i64) * 2, s));
      if (d_out_off) APO_CUDA(cudaMemsetAsync(d_out_off, 0, sizeof(i64) * (nwin + 1), s));
      return;
    }
    require(d_tok != nullptr, "NULL device pointer");
    Plan p = setup(c, b, h_off, true, true, s, min_len);
    build_sa(c, d_tok, b, p.sa, true, s);
    select_candidates(c, d_tok, b, p.sa, min_len, p.sel, s);
    emit_repeats(c, b, p.sel, prm.min_count, d_out, cap, d_out_off, d_occ, occ_cap, d_counts, s);
  });
}

apo_status apo_find_repeats(apo_ctx *ctx, const uint64_t *d_win, int32_t n, int32_t min_len,
                            const apo_params *params, apo_repeat *d_out, int64_t cap, int32_t *d_occ,
                            int64_t occ_cap, int64_t *d_counts, void *stream) {
  if (n < 0) return APO_ERR_INVALID;
  int64_t off[2] = {0, n};
  return find_common(ctx, d_win, off, 1, min_len, params, d_out, cap, nullptr, d_occ, occ_cap, d_counts, stream);
}

apo_status apo_find_repeats_batched(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off, int32_t nwin,
                                    int32_t min_len, const apo_params *params, apo_repeat *d_out, int64_t cap,
                                    int64_t *d_out_off, int32_t *d_occ, int64_t occ_cap, int64_t *d_counts,
                                    void *stream) {
  if (d_out_off == nullptr) return APO_ERR_INVALID;
  return find_common(ctx, d_tok, h_off, nwin, min_len, params, d_out, cap, d_out_off, d_occ, occ_cap, d_counts,
                     stream);
}

}  // extern "C"
