/*
 * apo.h -- C ABI of the B200-native Apophenia repeat-finding hot path
 * (arXiv 2406.18111, "Apophenia: automatic trace identification").
 *
 * Library: paper_2406_18111_b200/libapo.so (hand-written sm_100a CUDA).
 * Citations "P:n" are lines of the paper text; R1..R25 are the
 * readings of the paper listed in DESIGN.md §3.
 *
 * General conventions
 *  - Every pointer named d_* is a caller-owned DEVICE pointer (e.g. a torch
 *    tensor's data_ptr()) on the context's device; h_* pointers are host
 *    memory.  The library never frees caller memory.  Opaque handles
 *    (apo_ctx, apo_history, apo_trie) own their device workspace, released by
 *    the matching *_destroy call.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All device
 *    work is enqueued on it.  Data-dependent loop trip counts (prefix-doubling
 *    rounds, greedy rounds) are currently resolved with a small host read of a
 *    device flag, so the calls return with their results complete on `stream`.
 *  - Asynchrony: the calls return with their results complete, so a caller
 *    that wants analysis to overlap other GPU work runs it on another
 *    context + stream from another host thread (finder.py's StreamAnalyzer
 *    and BatchPipeline); apo_match_index lets the trace-independent half of
 *    matching run before the trace set exists.
 *  - Tokens are uint64 op hashes ordered as unsigned integers (R1).  A suffix
 *    that is a proper prefix of another sorts first (R2).
 *  - Positions, lengths and counts on the device are int32 unless stated.
 *    Window/stream offsets are int64.  A single window has n <= 2^30 tokens.
 *  - Capacity: when an output has more records than its capacity, the true
 *    count is still written and only the first `cap` records are stored; the
 *    caller detects this after synchronising and retries.
 *  - Errors: APO_ERR_INVALID for bad arguments (NULL with n > 0, negative
 *    sizes, min_len < 1); APO_ERR_NOMEM when device workspace cannot be
 *    allocated; APO_ERR_CUDA for CUDA failures (text via apo_last_error).
 *    n == 0 and n < 2*min_len are not errors: the result is empty.
 *  - A context is not thread-safe: use one per host thread.  Results are
 *    bit-identical across runs and batch compositions.
 */
#ifndef APO_H
#define APO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  APO_OK = 0,
  APO_ERR_INVALID = 1,
  APO_ERR_CAPACITY = 2,
  APO_ERR_NOMEM = 3,
  APO_ERR_CUDA = 4
} apo_status;

typedef struct apo_ctx apo_ctx;
typedef struct apo_history apo_history;
typedef struct apo_trie apo_trie;

/* Analysis parameters (the paper's -lg:auto_trace flags). */
typedef struct {
  int32_t min_count; /* keep repeats selected >= min_count times; 1 = paper-literal (R10) */
  int32_t max_len;   /* trie chunking "maximum trace length" (R15); 0 = unbounded */
  uint32_t flags;    /* reserved, must be 0 */
  int32_t reserved;  /* must be 0 */
} apo_params;

/* One deduplicated repeat of FindRepeats (Alg. 2; R10, R11):
 * start = smallest selected start (window-local), length, count = number of
 * selected non-overlapping occurrences, first_occ = index of its first
 * occurrence in the occurrence array.  Repeats are ordered by
 * (length desc, sub-string lexicographic asc) within a window. */
typedef struct {
  int32_t start, length, count, first_occ;
} apo_repeat;

/* [begin, end) in absolute history coordinates (global op count). */
typedef struct {
  int64_t begin, end;
} apo_slice;

/* One MATCH_ALL hit: trace `trace_id` ends at position `end_pos` of stream
 * `stream` (Alg. 1 Advance/FilterCompleted; R14).  `slot` is a
 * per-stream key of the trace (within one stream: equal slots <=> equal
 * trace ids; 0 <= slot < the number of traces), which apo_replay uses to
 * index its per-stream trace state. */
typedef struct {
  int32_t stream, end_pos, trace_id, slot;
} apo_match_rec;

/* REPLAY scoring constants (P:694-713 names the mechanisms -- a count cap,
 * an exponential decay of the count with the tasks since the trace last
 * appeared, a replay bonus -- but no values; readings R20-R24).  Score of a
 * completion of trace t at end e = len(t) * min(count, count_cap) * d_k with
 * d_0 = 65536, d_{k+1} = (d_k * decay_q16) >> 16, k = gap / decay_period,
 * times bonus_num / bonus_den (integer division) if t was replayed before in
 * this stream.  NULL params = the defaults {100, 64881 (0.99), 100, 11, 10}. */
typedef struct {
  int32_t count_cap, decay_q16, decay_period, bonus_num, bonus_den, reserved;
} apo_replay_params;

/* One REPLAY decision: trace `trace_id` replayed over stream positions
 * [end_pos - len + 1, end_pos]; first = 1 the first time this trace is
 * replayed in this stream (the trace is recorded), else 0. */
typedef struct {
  int32_t stream, end_pos, trace_id, first;
} apo_replay_rec;

int apo_version(void);
apo_status apo_ctx_create(int cuda_device, apo_ctx **out);
void apo_ctx_destroy(apo_ctx *ctx);
/* Text of the last error on this context ("" if none).  Owned by ctx. */
const char *apo_last_error(const apo_ctx *ctx);
/* Number of CUDA kernels the library has launched on this context so far
 * (introspection for benchmarks; monotone). */
int64_t apo_launch_count(const apo_ctx *ctx);

/* In-library profiler (for bench.py's roofline): when enabled, selected
 * kernel launches are bracketed by CUDA events recorded on the launching
 * stream.  apo_profile(ctx, 1) clears and starts recording, 0 stops.
 * apo_profile_read synchronises on the recorded events and returns, for
 * kernel class `kind` (0 = radix-sort digit pass, 1 = radix histogram,
 * 2 = single-pass scans, 3 = other, 4 = per-window on-chip suffix sort K9,
 * 5 = per-stream trace search), the summed device time in ms, the number
 * of launches and, for kind 0, the summed ALGORITHMIC HBM bytes (each
 * key/value read once and written once; 0 for the other kinds: bench.py
 * applies SURVEY.md §8(d)'s per-op model to them).  Any output pointer may
 * be NULL. */
apo_status apo_profile(apo_ctx *ctx, int enable);
apo_status apo_profile_read(apo_ctx *ctx, int kind, double *ms, int64_t *launches, double *bytes);

/* ---------------------------------------------------------------------- */
/* Alg. 2 building blocks (exposed for parity)                              */
/* ---------------------------------------------------------------------- */

/* "SA, LCP <- SuffixArray(S)".  d_tok: n tokens.  d_sa: n int32,
 * receives the suffix array (start positions in increasing suffix order).
 * d_lcp: n int32 or NULL; d_lcp[i] = LCP(SA[i], SA[i+1]) for i < n-1 (R3) and
 * d_lcp[n-1] = 0. */
apo_status apo_suffix_array(apo_ctx *ctx, const uint64_t *d_tok, int32_t n, int32_t *d_sa,
                            int32_t *d_lcp, void *stream);

/* Same for a CSR batch of independent windows (R16).  h_off: HOST
 * int64[nwin+1], h_off[0] = 0, non-decreasing; window w is
 * d_tok[h_off[w] .. h_off[w+1]).  d_sa / d_lcp: h_off[nwin] int32 each; the
 * window's entries sit at the same offsets, in WINDOW-LOCAL coordinates; the
 * last LCP slot of each window is 0. */
apo_status apo_suffix_array_batched(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off,
                                    int32_t nwin, int32_t *d_sa, int32_t *d_lcp, void *stream);

/* Candidate list of Alg. 2 in the paper's sort order
 * "by decreasing length and by increasing sub-string and start position",
 * with the greedy decision of P:576-583 for each.  Per candidate i:
 * d_len[i], d_id[i] (dense ordinal of the distinct sub-string in this order;
 * equal sub-strings share an id), d_start[i], d_kept[i] (1 = selected).
 * Candidates shorter than min_len are not generated (R7).  d_count (device
 * int64[1]) receives the candidate count m; at most cap are stored. */
apo_status apo_candidates(apo_ctx *ctx, const uint64_t *d_tok, int32_t n, int32_t min_len,
                          int32_t *d_len, int32_t *d_id, int32_t *d_start, uint8_t *d_kept,
                          int64_t cap, int64_t *d_count, void *stream);

/* K1, the LSD radix sort every sort of the path runs on (SA rounds P:552,
 * "Sort(C)" P:574-575): stable sort of (d_keys[i], d_vals[i]) pairs by key
 * bits [begin_bit, end_bit), in place.  d_vals may be NULL (keys only).
 * Exposed for parity tests and kernel benchmarks. */
apo_status apo_radix_sort(apo_ctx *ctx, uint64_t *d_keys, uint32_t *d_vals, int64_t n,
                          int32_t begin_bit, int32_t end_bit, void *stream);

/* ---------------------------------------------------------------------- */
/* FindRepeats (Alg. 2) -- the north_star call                              */
/* ---------------------------------------------------------------------- */

/* One window d_win[0..n).  params may be NULL (defaults: min_count 1).
 * d_out: cap apo_repeat records.  d_occ: occ_cap int32 occurrence starts
 * (window-local; per repeat in increasing order) or NULL.  d_counts: device
 * int64[2] <- {number of repeats, number of occurrences}. */
apo_status apo_find_repeats(apo_ctx *ctx, const uint64_t *d_win, int32_t n, int32_t min_len,
                            const apo_params *params, apo_repeat *d_out, int64_t cap,
                            int32_t *d_occ, int64_t occ_cap, int64_t *d_counts, void *stream);

/* CSR batch of independent windows (h_off as in apo_suffix_array_batched).
 * Output is window-major; d_out_off: device int64[nwin+1], repeats of window
 * w are d_out[d_out_off[w] .. d_out_off[w+1]) with window-local starts;
 * first_occ indexes the batch-wide d_occ.  d_counts: device int64[2] <-
 * {total repeats, total occurrences}.  Identical, window by window, to
 * apo_find_repeats on each window (R16). */
apo_status apo_find_repeats_batched(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off,
                                    int32_t nwin, int32_t min_len, const apo_params *params,
                                    apo_repeat *d_out, int64_t cap, int64_t *d_out_off,
                                    int32_t *d_occ, int64_t occ_cap, int64_t *d_counts,
                                    void *stream);

/* ---------------------------------------------------------------------- */
/* Alg. 1 TraceFinder: token history + ruler-function sampling (§4.4)       */
/* ---------------------------------------------------------------------- */

/* History ring of the last capacity_B tokens (R13); analyses are scheduled
 * every scale_C tokens ("multiples of a larger constant (such as 250)",
 * P:763-764).  capacity_B >= scale_C >= 1. */
apo_status apo_history_create(apo_ctx *ctx, int64_t capacity_B, int32_t scale_C,
                              apo_history **out);
void apo_history_destroy(apo_history *h);

/* "B <- B + [H]" (Alg. 1) for n tokens d_tokens[0..n), then the
 * slices "ShouldAnalyzeHistory / GetAnalysisSubset" selects while the global
 * op count k goes from k0+1 to k0+n: at every k with k % C == 0 the slice
 * [k - min(2^ruler(k/C) * C, B), k) (R13).  h_slices receives up
 * to cap slices in order; *h_nslices the true number.  If that number
 * exceeds cap the call returns APO_ERR_CAPACITY WITHOUT ingesting anything
 * (the schedule is pure arithmetic, so the count is known up front): the
 * caller retries with *h_nslices slots. */
apo_status apo_ingest(apo_history *h, const uint64_t *d_tokens, int64_t n, apo_slice *h_slices,
                      int64_t cap, int64_t *h_nslices, void *stream);

/* The schedule apo_ingest applies, as a pure host function (no device, no
 * state): the slices for op counts k in (k0, k0+n] (R13), into
 * h_slices[0 .. cap); *h_nslices = the true number; APO_ERR_CAPACITY if it
 * exceeds cap (the first cap slices are still written).  capacity_B >=
 * scale_C >= 1, k0 >= 0, n >= 0. */
apo_status apo_ruler_slices(int64_t k0, int64_t n, int32_t scale_C, int64_t capacity_B, apo_slice *h_slices,
                            int64_t cap, int64_t *h_nslices);

/* Copy history tokens [begin, end) (absolute coordinates, must lie within
 * the last capacity_B tokens) to d_out (end-begin tokens). */
apo_status apo_history_window(apo_history *h, int64_t begin, int64_t end, uint64_t *d_out,
                              void *stream);

/* Total number of tokens ever ingested. */
int64_t apo_history_count(const apo_history *h);

/* ---------------------------------------------------------------------- */
/* Alg. 1 TraceReplayer: candidate trace set and batched matching           */
/* ---------------------------------------------------------------------- */

/* IngestCandidates (Alg. 1): build the candidate trace set
 * from the output of apo_find_repeats_batched.  d_tok/h_off: the analysed
 * batch (as passed to apo_find_repeats_batched); d_rep/d_rep_off: its
 * repeats and DEVICE int64[nwin+1] offsets.  Each repeat's content is cut
 * into consecutive max_len pieces ("recorded traces are broken into pieces
 * of a given maximum size"; R15: the tail is kept iff >= min_len;
 * max_len = 0: no cut).  Identical contents are merged; trace ids are ranks
 * in (length desc, content lexicographic asc) order (R1).  The returned
 * handle owns the traces on the device; free with apo_trie_destroy.
 * Synchronises `stream`. */
apo_status apo_trie_build(apo_ctx *ctx, const uint64_t *d_tok, const int64_t *h_off, int32_t nwin,
                          const apo_repeat *d_rep, const int64_t *d_rep_off, int32_t min_len,
                          int32_t max_len, apo_trie **out, void *stream);

/* Same, from explicit trace contents (e.g. the union of candidate lists
 * gathered from several GPUs): trace t is d_tr[h_tr_off[t] .. h_tr_off[t+1])
 * (host int64 offsets, non-empty traces).  Duplicates are merged. */
apo_status apo_trie_build_traces(apo_ctx *ctx, const uint64_t *d_tr, const int64_t *h_tr_off,
                                 int32_t ntraces, apo_trie **out, void *stream);

/* Union trace set of nsrc (1..16) trace lists -- the multi-GPU exchange of
 * every rank builds the same union of all ranks' candidate
 * lists.  List r holds h_src_ntr[r] traces; its tokens are at h_src_tok[r],
 * a device pointer READABLE FROM ctx's DEVICE (a local allocation, or a peer
 * rank's buffer mapped over NVLink, e.g. CUDA IPC / symmetric memory), and
 * its host int64 offsets h_src_off[r][0 .. ntr] start at 0 (non-empty
 * traces).  The library pulls every list into local memory in the same pass
 * that hashes the pieces (no separate gather); the result is identical to
 * apo_trie_build_traces on the concatenation of the lists in source order.
 * The sources must stay unchanged until the call returns (it synchronises
 * `stream`); the caller orders the peers' writes before it (e.g. a barrier). */
apo_status apo_trie_build_traces_multi(apo_ctx *ctx, int32_t nsrc, const uint64_t *const *h_src_tok,
                                       const int64_t *const *h_src_off, const int32_t *h_src_ntr,
                                       apo_trie **out, void *stream);

void apo_trie_destroy(apo_trie *trie);

/* Sizes of the trace set: number of traces, total tokens, longest trace. */
apo_status apo_trie_info(const apo_trie *trie, int64_t *h_ntraces, int64_t *h_ntokens,
                         int64_t *h_maxlen);

/* Copy the traces out in id order: d_tokens (device, ntokens) and h_off
 * (host int64[ntraces+1]); either may be NULL. */
apo_status apo_trie_copy(const apo_trie *trie, uint64_t *d_tokens, int64_t *h_off, void *stream);

/* Batched matching of independent op streams against the trace set
 * (Alg. 1 AdvanceActiveCandidates / FilterInvalidCandidates /
 * FilterCompletedCandidates).  h_off: HOST
 * int64[nstreams+1] CSR offsets into d_streams.
 *  mode 0 = MATCH_ALL (reading R14): every (stream, end_pos, trace_id) with
 *    stream[end_pos-|t|+1 .. end_pos] == trace t, sorted by (stream, end_pos,
 *    trace_id); end_pos is stream-local.  d_out: apo_match_rec[cap] (device,
 *    16-byte aligned; 32-byte alignment lets the library store consecutive
 *    records in pairs); d_count: device int64[1] <- number of hits; at most
 *    cap records are stored.
 *  mode 1 = REPLAY: MATCH_ALL, then apo_replay with default parameters;
 *    d_out receives apo_replay_rec[cap] (cast), d_count: device int64[2] <-
 *    {replays, MATCH_ALL hits}.  On the on-chip path (streams <= 16,384 ops)
 *    the hits stay implicit in library workspace -- per end the deepest
 *    matched interval of the interval forest; the end's hits are its chain
 *    of parents -- and the selection walks the chains of the ends it
 *    decides; otherwise the records are written to library workspace.
 * Other modes: APO_ERR_INVALID.  Synchronises `stream`. */
apo_status apo_match(apo_ctx *ctx, const apo_trie *trie, const uint64_t *d_streams,
                     const int64_t *h_off, int32_t nstreams, int32_t mode, apo_match_rec *d_out,
                     int64_t cap, int64_t *d_count, void *stream);

/* The trace-independent half of apo_match, for callers that overlap it with
 * building the trace set (e.g. the multi-GPU union): the REVERSED streams,
 * their suffix arrays + LCP arrays and their buckets (by the first two
 * tokens when the batch has <= 65,534 distinct tokens, else by the first).
 * The handle owns device workspace of ctx (free with
 * apo_stream_index_destroy); d_streams
 * (and h_off's values) must stay unchanged until its last use.
 * Synchronises `stream`. */
typedef struct apo_stream_index apo_stream_index;
apo_status apo_match_index(apo_ctx *ctx, const uint64_t *d_streams, const int64_t *h_off, int32_t nstreams,
                           apo_stream_index **out, void *stream);
/* apo_match on the streams of `idx` (same output, modes and capacity rules);
 * idx must come from apo_match_index on the same ctx. */
apo_status apo_match_indexed(apo_ctx *ctx, const apo_trie *trie, const apo_stream_index *idx, int32_t mode,
                             apo_match_rec *d_out, int64_t cap, int64_t *d_count, void *stream);
void apo_stream_index_destroy(apo_stream_index *idx);

/* REPLAY selection (Alg. 1 SelectReplayTrace / ExecuteAndReplay, P:429-443;
 * scoring P:694-713; readings R20-R24) over MATCH_ALL hits d_hits[0..nhits)
 * as apo_match mode 0 writes them (sorted by (stream, end_pos, trace_id),
 * stream ids in [0, nstreams)).  Per stream, independently: walking the ends
 * in order, every completion counts as an appearance of its trace; among the
 * completions starting at or after the first op not yet replayed, the one
 * with the highest score (ties: longer, then smaller id) is replayed, which
 * clears every pointer that started before its end.  d_out: apo_replay_rec
 * (device) sorted by (stream, end_pos); d_count: device int64[1] <- number
 * of replays, at most cap stored.  h_len: HOST int64[nstreams] stream
 * lengths (bounds the decay table and the per-stream staging).  Synchronises
 * `stream`. */
apo_status apo_replay(apo_ctx *ctx, const apo_trie *trie, const apo_match_rec *d_hits, int64_t nhits,
                      const int64_t *h_len, int32_t nstreams, const apo_replay_params *params,
                      apo_replay_rec *d_out, int64_t cap, int64_t *d_count, void *stream);

/* ---------------------------------------------------------------------- */
/* Distributed suffix array: one window split into       */
/* contiguous position blocks over G ranks, prefix doubling ("SA <-         */
/* SuffixArray(S)") with a sample-sort exchange.  These are the      */
/* per-rank compute steps; paper_2406_18111_b200/dsa.py moves the data      */
/* between ranks (NCCL all-to-all / all-gather).  Ranks of a round are      */
/* group-head indices + 1 in [1, n] (0 = past the end); n < 2^32 - 1.       */
/* ---------------------------------------------------------------------- */

/* Round keys of the owned suffixes i = base .. base+m-1: d_keys[k] =
 * rank[i] * (n + 1) + rank2 with rank2 = d_rank2[k] (the rank of suffix
 * i + h) for k < m2 and 0 ("end of string") for k >= m2; d_vals[k] = i. */
apo_status apo_dsa_keys(apo_ctx *ctx, const uint32_t *d_rank, const uint32_t *d_rank2, int64_t m, int64_t m2,
                        int64_t base, int64_t n, uint64_t *d_keys, uint32_t *d_vals, void *stream);

/* s evenly spaced (key, value) samples of a block sorted by (key, value)
 * (all-ones samples when m == 0). */
apo_status apo_dsa_samples(apo_ctx *ctx, const uint64_t *d_keys, const uint32_t *d_vals, int64_t m, int32_t s,
                           uint64_t *d_skeys, uint32_t *d_svals, void *stream);

/* Partition of a block sorted by (key, value) by g-1 ascending (key, value)
 * splitters: d_counts[d] (device int64[g]) = number of pairs p with
 * splitter[d-1] <= p < splitter[d] (splitter[-1] = -inf, splitter[g-1] =
 * +inf). */
apo_status apo_dsa_split(apo_ctx *ctx, const uint64_t *d_keys, const uint32_t *d_vals, int64_t m,
                         const uint64_t *d_split_keys, const uint32_t *d_split_vals, int32_t g, int64_t *d_counts,
                         void *stream);

/* New ranks of a block of the globally sorted key sequence whose first
 * element has global index gbase: element k heads a group iff its key
 * differs from the previous key (prev_key, the previous rank's last key,
 * for k = 0 when has_prev); d_rank[k] = global index of its group's head + 1
 * (carry = global index of the last head before the block, -1 none).
 * d_stats (device int64[2]) <- {heads in the block, global index of the
 * last head or -1}.  Synchronises `stream`. */
apo_status apo_dsa_heads(apo_ctx *ctx, const uint64_t *d_keys, int64_t m, uint64_t prev_key, int32_t has_prev,
                         int64_t gbase, int64_t carry, uint32_t *d_rank, int64_t *d_stats, void *stream);

/* d_rank[d_pos[k] - base] = d_rank_in[k] for k < m (positions owned by the
 * calling rank). */
apo_status apo_dsa_scatter(apo_ctx *ctx, const uint32_t *d_pos, const uint32_t *d_rank_in, int64_t m, int64_t base,
                           uint32_t *d_rank, void *stream);

/* LCP of the distributed SA ("SA, LCP <- SuffixArray(S)"; R3) by
 * galloping over the saved rank levels, level j = ranks by the first 2^j
 * tokens, from the highest level down: equal level-j ranks at i + l and
 * i' + l <=> the next 2^j tokens agree, then l += 2^j.  Per level:
 *  - apo_dsa_lcp_requests: pair p = (d_a[p], d_b[p]) with lcp d_l[p] asks
 *    for the ranks at d_a[p] + l and d_b[p] + l: d_keys[2p], d_keys[2p+1] =
 *    those positions (n when past the end: not to be sent), d_vals = 2p,
 *    2p + 1;
 *  - apo_dsa_gather (owner side): d_out[k] = d_rank[d_pos[k] - base];
 *  - apo_dsa_lcp_update: the first nvalid answers d_resp (in the order of
 *    the sorted requests d_req) go back to their pairs through d_by_req
 *    (uint32[2 np], all 0xffffffff / 0xfffffffe pairs before the first
 *    level; reset by the call); d_l[p] += step where both answers exist and
 *    agree. */
apo_status apo_dsa_lcp_requests(apo_ctx *ctx, const uint32_t *d_a, const uint32_t *d_b, const uint32_t *d_l,
                                int64_t np, int64_t n, uint64_t *d_keys, uint32_t *d_vals, void *stream);
apo_status apo_dsa_gather(apo_ctx *ctx, const uint32_t *d_pos, int64_t m, int64_t base, const uint32_t *d_rank,
                          uint32_t *d_out, void *stream);
apo_status apo_dsa_lcp_update(apo_ctx *ctx, const uint32_t *d_resp, const uint32_t *d_req, int64_t nvalid,
                              int64_t np, uint32_t step, uint32_t *d_by_req, uint32_t *d_l, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* APO_H */
