// pipeline.cuh -- stages of FindRepeats on the device (product path).
#pragma once

#include "common.cuh"

namespace apo {

// A CSR batch of independent windows laid out back to back in one token
// array (a single window is W == 1).  Positions are global in [0, N).
struct Batch {
  i64 N = 0;
  int W = 1;
  i64 maxwin = 0;            // longest window
  const i64 *off = nullptr;  // device int64[W+1] (nullptr when W == 1)
  const i32 *wid = nullptr;  // device int32[N] window of each position (nullptr when W == 1)
  // Generalized mode: one suffix array over ALL windows (window w ends with
  // its own sentinel $_w, $_0 < $_1 < ... < every token) instead of one
  // suffix array per window.  Used by the trie build and the matcher.
  bool gen = false;
  // Stop prefix doubling once suffixes are ordered by their first
  // `sort_depth` tokens (0 = fully sorted).  Suffixes still tied then share
  // that prefix; the matcher, which only compares against traces no longer
  // than sort_depth, cannot tell them apart.  Not valid with LCP.
  i64 sort_depth = 0;
};

__device__ __forceinline__ int b_wid(const Batch &b, i64 i) { return b.W == 1 ? 0 : b.wid[i]; }
__device__ __forceinline__ i64 b_beg(const Batch &b, int w) { return b.W == 1 ? 0 : b.off[w]; }
__device__ __forceinline__ i64 b_end(const Batch &b, int w) { return b.W == 1 ? b.N : b.off[w + 1]; }

struct LevelPtrs {
  i32 *p[40];
};

// ----- suffix array + LCP (K2 initial ranking, K3 doubling, K4 PLCP) -----
struct SAWork {
  u64 *keys, *keys_alt;   // N
  u32 *vals, *vals_alt;   // N
  u64 *tok_sorted;        // N (batched initial ranking)
  i32 *levels[40];        // rank levels 0..R (each N)
  int max_levels;
  i32 *phi, *plcp;        // N
  i32 *rw;                // W: rounds per window (K9 path) or nullptr
  void *win_scratch;      // K9: per-CTA level scratch (L2-resident), or nullptr
  u32 *ids;               // N dense token ids (K2 hash path)
  bool ids_valid;
  char *ht_scratch;       // hash-table scratch of dense_token_ids
  u32 ht_cap;
  i64 K = -1;             // distinct tokens (K2 hash path; -1 otherwise)
  const u64 *dkeys = nullptr;  // their sorted values except ~0 (dk_n of them; in ht_scratch)
  i64 dk_n = 0;
  bool dk_max = false;    // the token ~0 occurs (id dk_n)
  const u32 *slot_rank = nullptr;  // set: ids[] holds table slots, id = slot_rank[slot] (K9 maps them)
  bool mirror = false;    // K9 reads each window's ids back to front (the reversed windows)
  // results
  i32 *sa;                // N (global positions, window-major suffix order)
  i32 *lcp;               // N (pair k = (k, k+1); 0 at the end of each window)
  int R;                  // final level index (ranks all distinct)
  int unit = 1;           // level r ranks the (unit * 2^r)-token prefixes (token packing, K3)
};

void plan_sa(Carver &cv, const Batch &b, SAWork &w, bool want_lcp, int nsmid);
// K2 (hash path): dense order-preserving token ids; returns K or -1 when
// the distinct count exceeds cap / 2.
size_t token_ids_scratch_bytes(i64 n, u32 cap);
// Mirrored ids (the matcher's reversed streams without reversing tokens):
// with slots_only, the table is built from the tokens as given and each
// window's id + 1 is written back to front as u16 into id16 when K <= 65,534
// (id16_ok says whether it was written); K9 maps the slots itself.
struct IdsMirror {
  const i64 *off;         // window offsets (nwin + 1)
  unsigned short *id16;   // or nullptr
  bool id16_ok = false;
  int nwin = 0;
};
i64 dense_token_ids(Ctx &c, const u64 *tok, i64 n, u32 *ids, u32 cap, char *scratch, cudaStream_t s,
                    const u64 **dkeys = nullptr, i64 *dk_n = nullptr, bool *dk_max = nullptr,
                    IdsMirror *mir = nullptr, const u32 **slots_only = nullptr);
// K9: per-window on-chip suffix array + LCP (windows <= 16,384 ops, not
// generalized): one CTA per window, a level scratch per SM id.
bool window_sa_supported(const Batch &b);
size_t window_sa_scratch_bytes(int nsmid);
int query_nsmid(int device);
void run_window_sa(Ctx &c, const Batch &b, SAWork &w, bool want_lcp, cudaStream_t s);
void build_sa(Ctx &c, const u64 *tok, const Batch &b, SAWork &w, bool want_lcp, cudaStream_t s,
              IdsMirror *mir = nullptr);
// build_sa of the REVERSED windows of tok (K9 path only) without reversing
// the tokens: the dense ids are mirrored.  false (nothing done) when the
// ids cannot be formed (vocabulary over the table budget) or K9 does not apply.
bool build_sa_mirrored(Ctx &c, const u64 *tok, const Batch &b, SAWork &w, bool want_lcp, cudaStream_t s,
                       IdsMirror &mir);

// ----- candidate generation, ordering, greedy, output (K5-K8) -----
struct SelWork {
  u32 *k1, *k1_alt;       // 2N sort-1 keys (window, length desc)
  u64 *v1, *v1_alt;       // 2N sort-1 values (pair rank << 32 | start)
  u64 *k2, *k2_alt;       // 2N sort-2 keys (group, start)
  i32 *rmq[32];           // LCP range minima: [0] in-block prefix, [1] in-block suffix, [2..] block-min sparse table
  int rmq_levels;
  i32 *glen;              // 2N per-group length
  i32 *gbase;             // 2N per-group window base (global position of the window start)
  i32 *gwin;              // 2N per-group window index
  u32 *gpos;              // 2N per-group first position in sort-1 order
  i32 *cl, *cs, *cg;      // 2N per candidate (final order): length, start (global), group
  u8 *state;              // 2N 0 undecided, 1 kept, 2 rejected
  u32 *tab[32];           // greedy first-cover table levels (N each)
  int tab_levels;
  u32 *diff;              // N+1 coverage difference array
  u32 *cov;               // N+1 coverage
  u32 *gcnt, *gfirst;     // 2N per group
  u32 *oidx;              // 2N occurrence index per candidate
  u32 *wcnt;              // W+1 repeats per window
  u64 *scal;              // small device scalars
  // the per-window greedy's kept candidates: per window up to kcap indices
  // (in candidate order) and their count, then compacted to klist (K entries)
  u32 *kwin = nullptr, *kcnt = nullptr, *kbase = nullptr, *klist = nullptr;
  i64 kcap = 0, K = -1;   // K: kept candidates (-1: no compact list, scan all candidates)
  i64 m = 0, G = 0;       // host copies of candidate / group counts
};

void plan_select(Carver &cv, const Batch &b, SelWork &w, int min_len);
// K5 + K6 fused per window (window_select.cu): true when it produced the
// candidates (false: a group too large for it; run the global path).
bool window_select_supported(const Batch &b, int min_len);
bool window_select(Ctx &c, const Batch &b, const SAWork &sa, int min_len, SelWork &w, cudaStream_t s);
// Runs K5..K7 (candidates, ordering, greedy).  After return, w.m and w.G are
// valid and w.cl/cs/cg/state hold the candidates in the paper's order.
void select_candidates(Ctx &c, const u64 *tok, const Batch &b, const SAWork &sa, int min_len,
                       SelWork &w, cudaStream_t s);
// K8: dedup + output.
void emit_repeats(Ctx &c, const Batch &b, SelWork &w, int min_count, apo_repeat *out, i64 cap,
                  i64 *out_off, i32 *occ, i64 occ_cap, i64 *counts, cudaStream_t s);
// Parity view of the candidate list (single window).
void emit_candidates(Ctx &c, const Batch &b, const SelWork &w, i32 *len, i32 *id, i32 *start, u8 *kept,
                     i64 cap, i64 *count, cudaStream_t s);

}  // namespace apo
