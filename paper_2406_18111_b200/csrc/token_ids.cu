// token_ids.cu -- K2: dense, order-preserving ids of the distinct tokens.
//
// ids[i] in [0, K) with ids[i] < ids[j] iff tok[i] < tok[j] (unsigned, R1).
// The op-hash streams of the paper's workloads reuse a small vocabulary (a
// loop body's task kinds), so instead of radix-sorting all N 64-bit tokens
// (8 passes over N) the distinct values are collected in an open-addressing
// hash table sized to stay L2-resident, only those K values are sorted, and
// every position maps to its value's rank: two passes over N plus a sort of
// K << N keys.  When the table would exceed its budget the caller falls back
// to the full sort.
#include "pipeline.cuh"

namespace apo {

namespace {

constexpr u64 kEmpty = ~0ull;  // the token value ~0 itself is handled aside

__device__ __forceinline__ u64 ht_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Linear probing from slot h (cur = table[h], already loaded): the slot of
// key, inserting it if absent; counts new keys.
__device__ __noinline__ u32 ht_insert_slow(u64 *table, u32 cap, u64 key, u32 h, u64 cur, u32 *nkeys,
                                           u32 *flags) {
  for (u32 probe = 0; probe < cap; ++probe) {
    if (probe > 0) cur = table[h];
    if (cur == key) return h;
    if (cur == kEmpty) {
      u64 old = atomicCAS(reinterpret_cast<unsigned long long *>(&table[h]), kEmpty, key);
      if (old == kEmpty) {
        u32 k = atomicAdd(nkeys, 1u);
        if (k + 1 > cap / 2) flags[1] = 1;  // over budget: caller retries or falls back
        return h;
      }
      if (old == key) return h;
    }
    h = (h + 1) & (cap - 1);
  }
  flags[1] = 1;
  return 0;
}

// ids[i] <- table slot of tok[i] (cap = the ~0 token); counts new keys.
// kHtItems tokens per thread with their first probes issued together: the
// kernel is bound by the latency of the dependent token -> table loads
// (one token per thread: 0.30 ms per C4 batch of 67 M tokens).
constexpr int kHtItems = 4;
__global__ void __launch_bounds__(256) k_ht_insert(const u64 *__restrict__ tok, i64 n, u64 *table, u32 cap,
                                                   u32 *__restrict__ ids, u32 *nkeys, u32 *flags) {
  const i64 base = i64(blockIdx.x) * (256 * kHtItems) + threadIdx.x;
  u64 key[kHtItems], cur[kHtItems];
  u32 h[kHtItems];
#pragma unroll
  for (int j = 0; j < kHtItems; ++j) {
    const i64 i = base + j * 256;
    key[j] = i < n ? tok[i] : kEmpty;
  }
#pragma unroll
  for (int j = 0; j < kHtItems; ++j) {
    h[j] = u32(ht_mix(key[j])) & (cap - 1);
    cur[j] = key[j] != kEmpty ? table[h[j]] : kEmpty;
  }
#pragma unroll
  for (int j = 0; j < kHtItems; ++j) {
    const i64 i = base + j * 256;
    if (i >= n) break;
    if (key[j] == kEmpty) {
      ids[i] = cap;
      flags[0] = 1;  // the ~0 token occurs
    } else {
      ids[i] = cur[j] == key[j] ? h[j] : ht_insert_slow(table, cap, key[j], h[j], cur[j], nkeys, flags);
    }
  }
}

struct HtCompactF {
  const u64 *table;
  u64 *keys;
  u32 *slots;
  i64 n;
  i64 *total;
  __device__ u32 load(i64 i) const { return table[i] != kEmpty ? 1u : 0u; }
  __device__ bool store(i64 i, u32 incl, u32 excl) const {
    if (incl != excl) {
      keys[excl] = table[i];
      slots[excl] = u32(i);
    }
    if (i == n - 1) *total = i64(incl);
    return false;
  }
  __device__ u32 *flag() const { return nullptr; }
};

__global__ void k_slot_rank(const u32 *__restrict__ slots_sorted, i64 K, u32 *__restrict__ slot_rank) {
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < K) slot_rank[slots_sorted[r]] = u32(r);
}

__global__ void k_ids_from_slots(u32 *__restrict__ ids, i64 n, const u32 *__restrict__ slot_rank) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = slot_rank[ids[i]];
}

// id + 1 of every position as u16, mirrored inside each window; a CTA per
// window (no per-position window lookups); slots[] read forward
__global__ void k_id16_mirror(const u32 *__restrict__ slots, const u32 *__restrict__ slot_rank,
                              const i64 *__restrict__ off, unsigned short *__restrict__ id16) {
  const i64 beg = off[blockIdx.x], n = off[blockIdx.x + 1] - beg;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x)
    id16[beg + n - 1 - i] = (unsigned short)(__ldg(&slot_rank[slots[beg + i]]) + 1u);
}


}  // namespace

size_t token_ids_scratch_bytes(i64 n, u32 cap) {
  Carver cv(nullptr);
  cv.take<u64>(cap);        // table
  cv.take<u32>(cap + 1);    // slot -> rank
  cv.take<u64>(cap / 2);    // distinct keys
  cv.take<u64>(cap / 2);    // ... alt
  cv.take<u32>(cap / 2);    // slots
  cv.take<u32>(cap / 2);    // ... alt
  cv.take<u32>(8);          // counters / flags
  cv.take<i64>(2);
  (void)n;
  return cv.off;
}

// Returns K (number of distinct tokens) or -1 if more than cap/2 distinct
// tokens were found (ids are then undefined).  `scratch` must hold
// token_ids_scratch_bytes(n, cap) bytes.
i64 dense_token_ids(Ctx &c, const u64 *tok, i64 n, u32 *ids, u32 cap, char *scratch, cudaStream_t s,
                    const u64 **dkeys, i64 *dk_n, bool *dk_max, IdsMirror *mir, const u32 **slots_only) {
  Carver cv(scratch);
  u64 *table = cv.take<u64>(cap);
  u32 *slot_rank = cv.take<u32>(cap + 1);
  u64 *dk = cv.take<u64>(cap / 2), *dk_alt = cv.take<u64>(cap / 2);
  u32 *ds = cv.take<u32>(cap / 2), *ds_alt = cv.take<u32>(cap / 2);
  u32 *cnt = cv.take<u32>(8);
  i64 *tot = cv.take<i64>(2);
  APO_CUDA(cudaMemsetAsync(table, 0xff, sizeof(u64) * cap, s));
  APO_CUDA(cudaMemsetAsync(cnt, 0, sizeof(u32) * 8, s));
  // table slot of every position (with slots_only the caller maps slots to
  // ids itself, e.g. K9 on its level-0 load, mirrored or not)
  u32 *slots = ids;
  k_ht_insert<<<grid_for(n, 256 * kHtItems), 256, 0, s>>>(tok, n, table, cap, slots, cnt, cnt + 1);
  APO_CHECK_LAUNCH();
  c.launches++;
  u32 hv[3];
  c.read_words(hv, cnt, 3, s);
  const u32 nkeys = hv[0], has_max = hv[1], over = hv[2];
  if (over) return -1;
  HtCompactF f{table, dk, ds, i64(cap), tot};
  launch_scan<false>(c, i64(cap), f, s);
  i64 K = nkeys;
  if (K > 1) {
    bool a = radix_sort_u64_u32(c, dk, ds, dk_alt, ds_alt, K, 0, 64, s);
    if (a) {
      ds = ds_alt;
      dk = dk_alt;
    }
  }
  if (dkeys) *dkeys = dk;
  if (dk_n) *dk_n = K;
  if (dk_max) *dk_max = has_max != 0;
  if (K > 0) {
    k_slot_rank<<<grid_for(K, 256), 256, 0, s>>>(ds, K, slot_rank);
    APO_CHECK_LAUNCH();
    c.launches++;
  }
  if (has_max) {  // the token ~0 is the largest value
    const u32 r = u32(K);
    c.h2d(slot_rank + cap, &r, sizeof(u32), s);
    ++K;
  }
  if (slots_only != nullptr) {
    // the caller maps slots itself (K9's level-0 load): ids[] keeps the slots
    *slots_only = slot_rank;
    if (mir) {
      mir->id16_ok = mir->id16 != nullptr && K >= 1 && K <= 65534;
      if (mir->id16_ok) {
        k_id16_mirror<<<mir->nwin, 256, 0, s>>>(ids, slot_rank, mir->off, mir->id16);
        APO_CHECK_LAUNCH();
        c.launches++;
      }
    }
    APO_CUDA(cudaStreamSynchronize(s));  // `r` above lives on the host stack
    return K;
  }
  k_ids_from_slots<<<grid_for(n, 256), 256, 0, s>>>(ids, n, slot_rank);
  APO_CHECK_LAUNCH();
  c.launches++;
  APO_CUDA(cudaStreamSynchronize(s));  // `r` above lives on the host stack
  return K;
}

}  // namespace apo
