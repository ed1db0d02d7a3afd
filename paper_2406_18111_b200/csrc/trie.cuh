// trie.cuh -- the candidate trace set handle (internal to libapo).
#pragma once

#include <vector>

#include "pipeline.cuh"

struct apo_trie {
  apo_ctx *ctx;
  apo::i64 T = 0;      // distinct traces
  apo::i64 ntok = 0;   // total tokens
  apo::i64 maxlen = 0;
  apo::u64 *d_tok = nullptr;  // traces in id order, back to back
  mutable apo::u64 *d_rtok = nullptr;  // the same traces, each reversed (built by the first apo_match)
  apo::i64 *d_off = nullptr;  // T+1
  size_t tok_bytes = 0, off_bytes = 0;  // pooled blocks (returned to the context on destroy)
  std::vector<apo::i64> h_off;
};


namespace apo {
// REPLAY selection over MATCH_ALL hits (replay.cu); synchronises s.
void run_replay(Ctx &c, const apo_trie *tr, const apo_match_rec *d_hits, i64 nhits, const i64 *h_len,
                int nstreams, const apo_replay_params &prm, apo_replay_rec *d_out, i64 cap, i64 *d_count,
                cudaStream_t s);
}  // namespace apo
