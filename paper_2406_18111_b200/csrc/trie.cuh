// trie.cuh -- the candidate trace set handle (internal to libapo).
#pragma once

#include <vector>

#include "pipeline.cuh"

struct apo_trie {
  apo_ctx *ctx;
  apo::i64 T = 0;      // distinct traces
  apo::i64 ntok = 0;   // total tokens
  apo::i64 maxlen = 0;
  apo::i64 minlen = 0;
  // traces in id order, back to back, each reversed (what the matcher reads);
  // the forward form is made on first use (trie_forward, apo_trie_copy)
  apo::u64 *d_rtok = nullptr;
  mutable apo::u64 *d_tok = nullptr;
  apo::i64 *d_off = nullptr;  // T+1
  size_t tok_bytes = 0, off_bytes = 0;  // pooled blocks (returned to the context on destroy)
  std::vector<apo::i64> h_off;
};


// The trace-independent half of apo_match (apo_match_index): the reversed
// streams, their suffix arrays + LCP and first-token buckets, in one pooled
// block of the creating context.  d_streams stays the caller's.
struct apo_stream_index {
  apo_ctx *ctx = nullptr;
  const apo::u64 *d_streams = nullptr;
  std::vector<apo::i64> h_off;
  int nstreams = 0;
  apo::i64 Ns = 0, maxs = 0, E = 0;
  bool rev = false;
  void *blk = nullptr;
  size_t bytes = 0;
  apo::i64 *d_off = nullptr;
  apo::i32 *d_wid = nullptr, *sa = nullptr, *lcp = nullptr;
  apo::u64 *rs = nullptr, *stok = nullptr;
  apo::u32 *sord = nullptr, *e_lo = nullptr, *e_q = nullptr, *e_hi = nullptr;
  int depth = 1;  // tokens that key the buckets (2 on the dense-id path)
  // dense-id matcher inputs (when the batch has <= 65,534 distinct tokens)
  unsigned short *sid = nullptr;  // reversed streams' ids + 1
  apo::u64 *dk = nullptr;         // sorted distinct tokens except ~0
  apo::i64 dk_n = 0;
  bool dk_max = false;
};

namespace apo {
// What the on-chip matcher leaves behind for REPLAY (apo_match mode 1): the
// REVERSED streams' suffix arrays and every stream's matched intervals in
// preorder (the hit records' slot = preorder id).  The pointers live in the
// context's arenas: valid until the next call reserves them.
struct ReplayIndex {
  bool ok = false;
  const i64 *off = nullptr;   // stream offsets (nstreams + 1)
  const i32 *sa = nullptr;    // reversed streams' suffix arrays (global positions)
  const u64 *tkey = nullptr;  // per interval (preorder): (stream << 30) | (lo << 15) | (32767 - hi)
  const u32 *toff = nullptr;  // per stream: first interval (nstreams + 1)
  i64 nint = 0;               // intervals of all streams
  // per stream position (end): the index of its first hit record and the
  // length of the shortest trace ending there (0xffff: no hit); pooled
  // blocks written by the emitter, returned by run_replay
  u32 *endoff = nullptr;
  unsigned short *endml = nullptr;
  size_t endoff_bytes = 0, endml_bytes = 0;
  // lazy (MATCH_ALL not written): endoff holds, per end, 1 + the deepest
  // interval containing its rank (0: no hit); an end's hits are the chain of
  // parents from there (interval ids local to the stream, base toff[q]):
  // opar = parent (kNoPar at a root), otr = trace id, odep = chain length;
  // qbase = per stream, its first hit in MATCH_ALL order
  bool lazy = false;
  const u32 *opar = nullptr, *otr = nullptr, *odep = nullptr, *qbase = nullptr;
};
// REPLAY selection over MATCH_ALL hits (replay.cu); synchronises s.  With
// ri->ok the trace states come from the matcher's index (no per-part
// sorting of the hits).
void run_replay(Ctx &c, const apo_trie *tr, const apo_match_rec *d_hits, i64 nhits, const i64 *h_len,
                int nstreams, const apo_replay_params &prm, apo_replay_rec *d_out, i64 cap, i64 *d_count,
                cudaStream_t s, const ReplayIndex *ri = nullptr);
}  // namespace apo
