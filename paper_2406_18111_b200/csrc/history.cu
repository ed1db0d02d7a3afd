// history.cu -- Alg. 1 TraceFinder state: the token history B and the
// ruler-function analysis schedule (§4.4).
//
// The history is a device ring holding the last B tokens (reading R13: the
// paper's MaybeClearHistory policy is unspecified; we keep a sliding window
// and never clear).  apo_ingest appends with one kernel and returns the
// slices [k - min(2^ruler(k/C) * C, B), k) for every k % C == 0 crossed.
#include "common.cuh"

struct apo_history {
  apo_ctx *ctx;
  apo::i64 B;
  apo::i32 C;
  apo::i64 count;
  apo::u64 *ring;
};

namespace apo {
namespace {

__global__ void k_ring_put(u64 *__restrict__ ring, i64 B, i64 k0, const u64 *__restrict__ tok, i64 first, i64 n) {
  i64 i = first + i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) ring[(k0 + i) % B] = tok[i];
}

__global__ void k_ring_get(const u64 *__restrict__ ring, i64 B, i64 begin, i64 n, u64 *__restrict__ out) {
  i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = ring[(begin + i) % B];
}

int ruler(i64 k) {  // 2-adic valuation, k >= 1
  int r = 0;
  while ((k & 1) == 0) {
    k >>= 1;
    ++r;
  }
  return r;
}

}  // namespace
}  // namespace apo

using namespace apo;

extern "C" {

apo_status apo_history_create(apo_ctx *ctx, int64_t capacity_B, int32_t scale_C, apo_history **out) {
  if (!ctx || !out || scale_C < 1 || capacity_B < scale_C) return APO_ERR_INVALID;
  *out = nullptr;
  cudaSetDevice(ctx->c.device);
  u64 *ring = nullptr;
  cudaError_t e = cudaMalloc(&ring, sizeof(u64) * size_t(capacity_B));
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->c.err = std::string("history allocation failed: ") + cudaGetErrorString(e);
    return APO_ERR_NOMEM;
  }
  *out = new apo_history{ctx, capacity_B, scale_C, 0, ring};
  return APO_OK;
}

void apo_history_destroy(apo_history *h) {
  if (!h) return;
  cudaSetDevice(h->ctx->c.device);
  cudaFree(h->ring);
  delete h;
}

int64_t apo_history_count(const apo_history *h) { return h ? h->count : -1; }

apo_status apo_ruler_slices(int64_t k0, int64_t n, int32_t scale_C, int64_t capacity_B, apo_slice *h_slices,
                            int64_t cap, int64_t *h_nslices) {
  if (k0 < 0 || n < 0 || scale_C < 1 || capacity_B < scale_C || cap < 0 || (cap > 0 && !h_slices))
    return APO_ERR_INVALID;
  // ShouldAnalyzeHistory / GetAnalysisSubset (reading R13): at
  // every op count k in (k0, k0+n] with k % C == 0, the last
  // min(2^ruler(k/C) * C, B) tokens
  const i64 C = scale_C, k1 = k0 + n;
  i64 ns = 0;
  for (i64 k = (k0 / C + 1) * C; k <= k1; k += C) {
    if (ns < cap) {
      const int r = ruler(k / C);
      i64 len = r < 62 ? (i64(1) << r) * C : capacity_B;
      if (len > capacity_B || len <= 0) len = capacity_B;
      h_slices[ns] = apo_slice{k - len, k};
    }
    ++ns;
  }
  if (h_nslices) *h_nslices = ns;
  return ns > cap ? APO_ERR_CAPACITY : APO_OK;
}

apo_status apo_ingest(apo_history *h, const uint64_t *d_tokens, int64_t n, apo_slice *h_slices, int64_t cap,
                      int64_t *h_nslices, void *stream) {
  if (!h || n < 0 || cap < 0 || (n > 0 && !d_tokens) || (cap > 0 && !h_slices)) return APO_ERR_INVALID;
  Ctx &c = h->ctx->c;
  // The schedule is pure host arithmetic on the op count, so the slices are
  // known before anything changes: too small a cap fails WITHOUT ingesting,
  // and the caller retries with *h_nslices slots.
  i64 ns = 0;
  const apo_status st = apo_ruler_slices(h->count, n, h->C, h->B, h_slices, cap, &ns);
  if (h_nslices) *h_nslices = ns;
  if (st != APO_OK) return st;
  const i64 k1 = h->count + n;
  cudaSetDevice(c.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n > 0) {
    i64 first = n > h->B ? n - h->B : 0;  // earlier tokens would be overwritten anyway
    i64 cnt = n - first;
    k_ring_put<<<grid_for(cnt, 256), 256, 0, s>>>(h->ring, h->B, h->count, d_tokens, first, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      c.err = cudaGetErrorString(e);
      return APO_ERR_CUDA;
    }
    c.launches++;
  }
  h->count = k1;
  return APO_OK;
}

apo_status apo_history_window(apo_history *h, int64_t begin, int64_t end, uint64_t *d_out, void *stream) {
  if (!h || begin < 0 || end < begin || end > h->count || begin < h->count - h->B) return APO_ERR_INVALID;
  if (end == begin) return APO_OK;
  if (!d_out) return APO_ERR_INVALID;
  Ctx &c = h->ctx->c;
  cudaSetDevice(c.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_ring_get<<<grid_for(end - begin, 256), 256, 0, s>>>(h->ring, h->B, begin, end - begin, d_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    c.err = cudaGetErrorString(e);
    return APO_ERR_CUDA;
  }
  c.launches++;
  return APO_OK;
}

}  // extern "C"
