// layer_kernels.cuh — launch interface of the layer stages (K3, K4, K5, K8).
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace smoe {

struct ShardPtrs {
  char* p[SMOE_MAX_SHARDS];
};

struct LocalRows {
  // local rows are the concatenation, over resident shards g, of the first
  // counts[g] slots of group g (real tokens only, no pads)
  const int32_t* counts;     // [G] plan counts
  const int64_t* group;      // [1] max group
  const int64_t* forward;    // [G * max_tokens]
  int32_t shard_begin, shard_count, n_shards;
  int64_t single_rows;       // counts == nullptr: one block of `single_rows` rows (shard 0)
};

// n_sources: partials summed (default: one per shard, lr.n_shards)
int launch_srs(const LocalRows& lr, const ShardPtrs& partials, int64_t d, const ShardPtrs& hs,
               int64_t n_rows_bound, cudaStream_t st, int32_t n_sources = 0);

// DS-MoE baseline all-reduce: the resident shards' natural row slices of the
// sum of the n_shards partials, stored into every output (one per process)
int launch_allreduce(const ShardPtrs& partials, int64_t d, int64_t n, int32_t shard_begin,
                     int32_t shard_count, int32_t n_shards, const ShardPtrs& outs,
                     int32_t n_outs, cudaStream_t st);

int launch_gate(const LocalRows& lr, const ShardPtrs& hs, int64_t d, const void* w_gate,
                const float* b_gate, int32_t N, int32_t k, int32_t renorm,
                const int32_t* slot_owner, const ShardPtrs& topk_ids, const ShardPtrs& topk_w,
                int64_t* stats, int64_t n_rows_bound, cudaStream_t st);

// K4 on tcgen05 (gate_tcgen05.cu): the hidden rows of the resident shards
// come from ONE arena (shard i at row i * rows_per_shard) through a TMA map.
struct GateTcArgs {
  const int32_t* counts;     // [G] plan counts (nullptr: single_rows rows in shard 0)
  int64_t single_rows;
  int32_t shard_begin, shard_count;
  int64_t rows_per_shard;    // arena row stride between resident shards
  int32_t num_k_blocks;      // d / 64
  int32_t n_experts, k, renorm;
  const float* b_gate;
  const int32_t* slot_owner;
  ShardPtrs topk_ids, topk_w;
  int64_t* stats;
  // route fused into the gate (every shard's rows fit one tile, so a CTA
  // holds all pairs of its shard): stable pair ranks per expert and the
  // shard's row of the [G, N] count matrix, as route_rank_kernel computes
  // them, written to every process's count buffer
  int32_t route;
  ShardPtrs pair_rank;       // per resident shard [n, k]
  ShardPtrs count_bufs;      // one [G, N] int32 matrix per process
  int32_t n_count_bufs;
};
bool gate_tc_supported(int32_t n_experts, int32_t top_k, int64_t d);
int gate_route_fused();               // SMOE_OPT_ROUTE_IN_GATE
void set_gate_route_fused(int on);
int gate_tc_enabled();                 // SMOE_OPT_GATE_TENSOR
void set_gate_tc_enabled(int on);
int gate_tc_rows(int32_t n_experts);   // W box rows (N rounded up to 16)
int launch_gate_tc(const CUtensorMap& map_h, const CUtensorMap& map_w, const GateTcArgs& a,
                   int64_t n_rows_bound, cudaStream_t st);


size_t route_workspace_bytes(int64_t max_tokens, int32_t k, int32_t N, int32_t shard_count);
int launch_route(const LocalRows& lr, int32_t N, int32_t k, const ShardPtrs& topk_ids,
                 const ShardPtrs& pair_rank, const ShardPtrs& count_bufs, int32_t n_count_bufs,
                 int32_t* chunk_counts, int64_t n_rows_bound, cudaStream_t st);

// xfan: per-shard int32 [expert_rows] fan-out tables of the deduplicated
// dispatch, non-null only for shards in OTHER processes (see dispatch_kernel)
int launch_dispatch(const LocalRows& lr, int32_t N, int32_t k, int64_t d,
                    const int32_t* counts_mat, const int32_t* slot_owner,
                    const int32_t* slot_first, const ShardPtrs& hs, const ShardPtrs& topk_ids,
                    const ShardPtrs& pair_rank, const ShardPtrs& xin, const ShardPtrs& xmeta,
                    int64_t expert_rows, int64_t* problems, int32_t* err, int64_t n_rows_bound,
                    cudaStream_t st, const ShardPtrs& xfan, int64_t* stats);
int launch_fanout(const int64_t* problems, int32_t n_problems, const ShardPtrs& xin,
                  const ShardPtrs& xfan, int32_t shard_begin, int64_t expert_rows, int64_t d,
                  const int32_t* slot_owner, const int32_t* slot_first, int64_t rows_bound,
                  cudaStream_t st);

struct HistUpdate {
  const int64_t* hist_in;     // [n, hist_len] or nullptr (first layers)
  ShardPtrs hist_outs;        // one [n, hist_len] int64 buffer per process (SAG of the history)
  int32_t n_hist_outs;        // 0: not requested
  int32_t hist_len;
  const int32_t* slot_owner;  // [N] cluster of each expert slot
  ShardPtrs topk_ids;         // per resident shard [n, k]
};

// block_rows > 0: DS-MoE layout -- row j of shard g goes to row g * group + j
// of each output (an all-gather buffer of block_rows rows), not to the
// token's original position
int launch_combine_sag(const LocalRows& lr, int32_t k, int64_t d, const ShardPtrs& ypair,
                       const ShardPtrs& topk_w, const ShardPtrs& outs, int32_t n_outs,
                       const HistUpdate& hu, int64_t n_rows_bound, cudaStream_t st,
                       int64_t block_rows = 0, int32_t* err = nullptr);

// Standalone shuffled all-gather (smoe_sag): row j of blocks[g] -> every
// outs[o] at forward[g*group + j].
int launch_sag(const LocalRows& lr, int64_t d, const ShardPtrs& blocks, const ShardPtrs& outs,
               int32_t n_outs, int64_t n_rows_bound, cudaStream_t st);

// Single-rank building blocks (DS-MoE baseline, smoe_gate_topk & co.)
int launch_pair_offsets(const int32_t* topk_ids, int64_t rows, int32_t k, int32_t N,
                        int32_t* pair_pos, int32_t* counts, cudaStream_t st);
int launch_pack_rows(const void* src, int64_t rows, int32_t k, int64_t d, const int32_t* pair_pos,
                     void* dst, cudaStream_t st);
int launch_combine_rows(const void* y, const int32_t* pair_pos, const float* topk_w, int64_t rows,
                        int32_t k, int64_t d, void* out, cudaStream_t st);

int launch_barrier(const ShardPtrs& signals, int32_t world, int32_t rank, uint32_t* my_signal,
                   uint32_t* epoch, cudaStream_t st);

}  // namespace smoe

namespace smoe {
// PLAN stage of the layer (plan.cu): smoe_lookup_plan plus the per-forward
// resets of `err`, stats[0, n_stats) and zero_i32[0, n_zero_i32) -- folded
// into the single-CTA plan kernel for decode-sized batches
int layer_plan(const int64_t* tokens, int64_t n, const int64_t* hist, int32_t hist_len,
               const int16_t* t_labels, const float* t_conf, int64_t vocab,
               const int16_t* a_best, const float* a_conf, int64_t a_rows, int32_t n_clusters,
               int64_t* dev_out, int64_t* forward, int64_t* inverse, int32_t* counts,
               int64_t* group, int32_t* err, void* workspace, size_t workspace_bytes,
               int64_t* stats, int32_t n_stats, cudaStream_t st, int32_t* zero_i32 = nullptr,
               int32_t n_zero_i32 = 0);
}  // namespace smoe
