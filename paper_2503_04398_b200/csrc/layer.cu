// layer.cu — host runtime of the speculative MoE layer (C-ABI handle).
//
// Owns the shard tables, the TMA descriptors of the two expert GEMMs and the
// small device-side placement tables, and sequences the stages of Algorithm 2
// on one stream.  With world_size > 1 a cross-process
// barrier over NVLink-mapped signal pads separates the stages whose inputs are
// written by other processes (before SRS; after ROUTE, DISPATCH, EXPERT_DOWN,
// COMBINE_SAG).
#include "common.cuh"
#include "gemm.h"
#include "layer_kernels.cuh"
#include "gate_select.cuh"

#include <cstring>
#include <vector>
#include <algorithm>

using namespace smoe;

struct smoe_layer {
  smoe_layer_config cfg;
  void* buf[SMOE_BUF__COUNT][SMOE_MAX_SHARDS];
  // tables
  const int16_t* t_labels = nullptr;
  const float* t_conf = nullptr;
  int64_t vocab = 0;
  const int16_t* a_best = nullptr;
  const float* a_conf = nullptr;
  int64_t a_rows = 0;
  int32_t hist_len = 0;
  std::vector<int32_t> slot_owner_h, slot_first_h;
  int32_t* slot_owner_d = nullptr;   // [N]
  int32_t* slot_first_d = nullptr;   // [G + 1]
  int32_t* ready_d = nullptr;        // [kMaxExperts + 1] up-tile counts (early down GEMM)
                                     // + the down GEMM's dynamic tile counter
  bool ready_armed = false;          // the last EXPERT_UP launch publishes them
  bool ready_zeroed = false;         // this forward's PLAN reset them
  bool route_fused = false;          // the last GATE launch also ran the route
  int32_t local_slots = 0;           // expert slots owned by the resident shards
  // weights
  const void* w_gate = nullptr;
  const float* b_gate = nullptr;
  const void* w13 = nullptr;
  const void* w2 = nullptr;
  bool w_tiled = false;              // w13 / w2 in smoe_tile_weights layout
  // GEMM descriptors
  bool maps_ready = false;
  int maps_cg_up = 0, maps_cg_down = 0;
  CUtensorMap map_x, map_w13, map_h, map_w2;
  CUtensorMap map_w13_single;        // w13 with one-SM boxes (decode sizes / narrow, see EXPERT_UP)
  CUtensorMap map_w2_single;         // w2 with one-SM boxes (small batches, see EXPERT_DOWN)
  CUtensorMap map_x_narrow, map_h_narrow;   // 32-row A boxes (decode-sized batches)
  // tensor-core gate: hidden rows of the resident shards (one arena) and W_g
  bool gate_tc = false;
  CUtensorMap map_hs, map_wg;
  // SMOE_PIPELINE_DSMOE: all-reduce + slice instead of SRS, combine into
  // all-gather blocks + resume gather instead of the fused SAG
  int32_t pipeline = SMOE_PIPELINE_SMOE;
  int64_t ag_rows = 0;
};

static bool valid_cfg(const smoe_layer_config* c) {
  return c && c->n_shards >= 1 && c->n_shards <= SMOE_MAX_SHARDS && c->shard_begin >= 0 &&
         c->shard_count >= 1 && c->shard_begin + c->shard_count <= c->n_shards &&
         c->n_experts >= 1 && c->top_k >= 1 && c->top_k <= c->n_experts && c->hidden > 0 &&
         c->ffn > 0 && c->max_tokens > 0 && c->expert_rows > 0 && c->world_size >= 1 &&
         c->world_rank >= 0 && c->world_rank < c->world_size;
}

static size_t plan_ws_aligned(const smoe_layer_config* cfg) {
  return (smoe_plan_workspace_bytes(cfg->max_tokens, cfg->n_shards) + 255) & ~size_t(255);
}

extern "C" size_t smoe_layer_workspace_bytes(const smoe_layer_config* cfg) {
  if (!cfg) return 0;
  return plan_ws_aligned(cfg) +
         route_workspace_bytes(cfg->max_tokens, cfg->top_k, cfg->n_experts, cfg->shard_count);
}

extern "C" int smoe_layer_create(const smoe_layer_config* cfg, smoe_layer** out) {
  if (!valid_cfg(cfg) || !out) return SMOE_ERR_INVALID_ARG;
  if (cfg->hidden % kGemmBN != 0 || cfg->ffn % 128 != 0 || (2 * cfg->ffn) % kGemmBN != 0 ||
      cfg->n_experts > kMaxExperts || cfg->top_k > 8)
    return SMOE_ERR_UNSUPPORTED;
  smoe_layer* L = new smoe_layer();
  L->cfg = *cfg;
  std::memset(L->buf, 0, sizeof(L->buf));
  if (cudaMalloc(&L->slot_owner_d, sizeof(int32_t) * cfg->n_experts) != cudaSuccess ||
      cudaMalloc(&L->slot_first_d, sizeof(int32_t) * (cfg->n_shards + 1)) != cudaSuccess ||
      cudaMalloc(&L->ready_d, sizeof(int32_t) * (kMaxExperts + 1)) != cudaSuccess) {
    delete L;
    return SMOE_ERR_CUDA;
  }
  *out = L;
  return SMOE_OK;
}

extern "C" void smoe_layer_destroy(smoe_layer* L) {
  if (!L) return;
  cudaFree(L->slot_owner_d);
  cudaFree(L->slot_first_d);
  cudaFree(L->ready_d);
  delete L;
}

extern "C" int smoe_layer_bind(smoe_layer* L, int32_t slot, int32_t index, void* ptr) {
  if (!L || slot < 0 || slot >= SMOE_BUF__COUNT || index < 0 || index >= SMOE_MAX_SHARDS)
    return SMOE_ERR_INVALID_ARG;
  if (L->buf[slot][index] != ptr &&
      (slot == SMOE_BUF_XIN || slot == SMOE_BUF_XMETA || slot == SMOE_BUF_HMID ||
       slot == SMOE_BUF_HS))
    L->maps_ready = false;           // only these feed TMA descriptors / arena checks
  L->buf[slot][index] = ptr;
  return SMOE_OK;
}

extern "C" int smoe_layer_set_tables(smoe_layer* L, const int16_t* t_labels, const float* t_conf,
                                     int64_t vocab, const int16_t* a_best, const float* a_conf,
                                     int64_t a_rows, int32_t hist_len,
                                     const int32_t* slot_owner_h) {
  if (!L || !t_labels || !t_conf || vocab <= 0 || !slot_owner_h) return SMOE_ERR_INVALID_ARG;
  const int N = L->cfg.n_experts, G = L->cfg.n_shards;
  std::vector<int32_t> owner(slot_owner_h, slot_owner_h + N);
  // s-EG order: every cluster's slots are contiguous and clusters ascend
  for (int e = 0; e < N; ++e) {
    if (owner[e] < 0 || owner[e] >= G) return SMOE_ERR_CLUSTERS;
    if (e && owner[e] < owner[e - 1]) return SMOE_ERR_INVALID_ARG;
  }
  std::vector<int32_t> first(G + 1, N);
  for (int e = N - 1; e >= 0; --e) first[owner[e]] = e;
  for (int g = G - 1; g >= 0; --g) first[g] = std::min(first[g], first[g + 1]);
  L->t_labels = t_labels; L->t_conf = t_conf; L->vocab = vocab;
  L->a_best = a_best; L->a_conf = a_conf; L->a_rows = a_rows; L->hist_len = hist_len;
  L->slot_owner_h = owner;
  L->slot_first_h = first;
  L->local_slots = first[L->cfg.shard_begin + L->cfg.shard_count] - first[L->cfg.shard_begin];
  SMOE_CUDA_TRY(cudaMemcpy(L->slot_owner_d, owner.data(), sizeof(int32_t) * N,
                           cudaMemcpyHostToDevice));
  SMOE_CUDA_TRY(cudaMemcpy(L->slot_first_d, first.data(), sizeof(int32_t) * (G + 1),
                           cudaMemcpyHostToDevice));
  L->maps_ready = false;
  return SMOE_OK;
}

extern "C" int smoe_layer_set_pipeline(smoe_layer* L, int32_t pipeline, int64_t ag_rows) {
  if (!L) return SMOE_ERR_INVALID_ARG;
  if (pipeline == SMOE_PIPELINE_SMOE) {
    L->pipeline = pipeline;
    return SMOE_OK;
  }
  if (pipeline != SMOE_PIPELINE_DSMOE || ag_rows <= 0) return SMOE_ERR_INVALID_ARG;
  for (int g = 0; g < L->cfg.n_shards; ++g)
    if (!L->buf[SMOE_BUF_AR][g] || !L->buf[SMOE_BUF_AG][g]) return SMOE_ERR_INVALID_ARG;
  L->pipeline = pipeline;
  L->ag_rows = ag_rows;
  return SMOE_OK;
}

extern "C" int smoe_layer_set_weights(smoe_layer* L, const void* w_gate, const float* b_gate,
                                      const void* w13, const void* w2) {
  if (!L || !w_gate || !w13 || !w2) return SMOE_ERR_INVALID_ARG;
  L->w_gate = w_gate; L->b_gate = b_gate; L->w13 = w13; L->w2 = w2;
  L->w_tiled = false;
  L->maps_ready = false;
  return SMOE_OK;
}

extern "C" int smoe_layer_set_weights_tiled(smoe_layer* L, const void* w_gate,
                                            const float* b_gate, const void* w13_tiled,
                                            const void* w2_tiled) {
  int rc = smoe_layer_set_weights(L, w_gate, b_gate, w13_tiled, w2_tiled);
  if (rc == SMOE_OK) L->w_tiled = true;
  return rc;
}

static ShardPtrs local_ptrs(const smoe_layer* L, int slot) {
  ShardPtrs p{};
  for (int i = 0; i < L->cfg.shard_count; ++i) p.p[i] = static_cast<char*>(L->buf[slot][i]);
  return p;
}
// Per-shard ("peer") slot, restricted to the resident shards (index = local).
static ShardPtrs resident_ptrs(const smoe_layer* L, int slot) {
  ShardPtrs p{};
  for (int i = 0; i < L->cfg.shard_count; ++i)
    p.p[i] = static_cast<char*>(L->buf[slot][L->cfg.shard_begin + i]);
  return p;
}
static ShardPtrs peer_ptrs(const smoe_layer* L, int slot) {
  ShardPtrs p{};
  for (int g = 0; g < L->cfg.n_shards; ++g) p.p[g] = static_cast<char*>(L->buf[slot][g]);
  return p;
}
// Distinct pointers among the per-shard bindings of `slot` (one per process).
static ShardPtrs distinct_ptrs(const smoe_layer* L, int slot, int32_t* count) {
  ShardPtrs p{};
  int n = 0;
  for (int g = 0; g < L->cfg.n_shards; ++g) {
    char* q = static_cast<char*>(L->buf[slot][g]);
    bool seen = false;
    for (int i = 0; i < n; ++i) seen |= (p.p[i] == q);
    if (!seen) p.p[n++] = q;
  }
  *count = n;
  return p;
}

// distinct buffers of a per-process slot, this process's own first (kernels
// that re-read what they stored read the local copy, not a peer's)
static ShardPtrs distinct_ptrs_local_first(const smoe_layer* L, int slot, int32_t* count) {
  ShardPtrs p = distinct_ptrs(L, slot, count);
  char* mine = static_cast<char*>(L->buf[slot][L->cfg.shard_begin]);
  for (int i = 1; i < *count; ++i)
    if (p.p[i] == mine) { p.p[i] = p.p[0]; p.p[0] = mine; }
  return p;
}

static int g_dedup_dispatch = 1;      // SMOE_OPT_DEDUP_DISPATCH
static int g_decode_up_pdl = 1;       // SMOE_OPT_DECODE_UP_PDL

static int check_bound(const smoe_layer* L) {
  const auto& c = L->cfg;
  for (int g = 0; g < c.n_shards; ++g)
    for (int s : {SMOE_BUF_PARTIAL, SMOE_BUF_XIN, SMOE_BUF_XMETA, SMOE_BUF_YPAIR, SMOE_BUF_OUT,
                  SMOE_BUF_COUNTS})
      if (!L->buf[s][g]) return SMOE_ERR_INVALID_ARG;
  for (int i = 0; i < c.shard_count; ++i)
    for (int s : {SMOE_BUF_HS, SMOE_BUF_TOPK_IDS, SMOE_BUF_TOPK_W, SMOE_BUF_PAIR_RANK})
      if (!L->buf[s][i]) return SMOE_ERR_INVALID_ARG;
  for (int s : {SMOE_BUF_HMID, SMOE_BUF_FORWARD, SMOE_BUF_INVERSE, SMOE_BUF_DEV,
                SMOE_BUF_PLAN_COUNTS, SMOE_BUF_GROUP, SMOE_BUF_STATS, SMOE_BUF_ERR,
                SMOE_BUF_WORKSPACE, SMOE_BUF_PROBLEMS})
    if (!L->buf[s][0]) return SMOE_ERR_INVALID_ARG;
  if (c.world_size > 1) {
    for (int g = 0; g < c.n_shards; ++g)
      if (!L->buf[SMOE_BUF_SIGNAL][g]) return SMOE_ERR_INVALID_ARG;
    if (!L->buf[SMOE_BUF_EPOCH][0]) return SMOE_ERR_INVALID_ARG;
  }
  // the resident shards' expert inputs / metadata must form one arena
  // (one TMA descriptor covers all local problems)
  const int64_t xs = c.expert_rows * (int64_t)c.hidden * 2, ms = c.expert_rows * 8;
  for (int i = 1; i < c.shard_count; ++i) {
    const int g0 = c.shard_begin;
    if (static_cast<char*>(L->buf[SMOE_BUF_XIN][g0 + i]) !=
            static_cast<char*>(L->buf[SMOE_BUF_XIN][g0]) + i * xs ||
        static_cast<char*>(L->buf[SMOE_BUF_XMETA][g0 + i]) !=
            static_cast<char*>(L->buf[SMOE_BUF_XMETA][g0]) + i * ms)
      return SMOE_ERR_INVALID_ARG;
  }
  return SMOE_OK;
}

static int ensure_maps(smoe_layer* L) {
  if (L->maps_ready && L->maps_cg_up == gemm_cta_group(0) &&
      L->maps_cg_down == gemm_cta_group(1))
    return SMOE_OK;
  int rc = check_bound(L);
  if (rc) return rc;
  if (!L->w13 || !L->w2 || !L->w_gate || !L->t_labels) return SMOE_ERR_INVALID_ARG;
  const auto& c = L->cfg;
  const int64_t rows = c.expert_rows * c.shard_count;
  const int64_t nl = std::max<int32_t>(L->local_slots, 1);
  if ((rc = make_tmap_bf16(&L->map_x, L->buf[SMOE_BUF_XIN][c.shard_begin], rows, c.hidden,
                           kGemmBM)))
    return rc;
  // tiled weights: a [rows * (K / 64), 64] tensor whose boxes are contiguous
  const int64_t w13_rows = nl * 2 * c.ffn, w2_rows = nl * c.hidden;
  if ((rc = make_tmap_bf16(&L->map_w13, L->w13,
                           L->w_tiled ? w13_rows * (c.hidden / kGemmBK) : w13_rows,
                           L->w_tiled ? kGemmBK : c.hidden, gemm_b_box_rows(gemm_cta_group(0)))))
    return rc;
  if ((rc = make_tmap_bf16(&L->map_w13_single, L->w13,
                           L->w_tiled ? w13_rows * (c.hidden / kGemmBK) : w13_rows,
                           L->w_tiled ? kGemmBK : c.hidden, gemm_b_box_rows(1))))
    return rc;
  if ((rc = make_tmap_bf16(&L->map_h, L->buf[SMOE_BUF_HMID][0], rows, c.ffn, kGemmBM))) return rc;
  if ((rc = make_tmap_bf16(&L->map_x_narrow, L->buf[SMOE_BUF_XIN][c.shard_begin], rows, c.hidden,
                           kGemmNarrowM)))
    return rc;
  if ((rc = make_tmap_bf16(&L->map_h_narrow, L->buf[SMOE_BUF_HMID][0], rows, c.ffn,
                           kGemmNarrowM)))
    return rc;
  if ((rc = make_tmap_bf16(&L->map_w2, L->w2,
                           L->w_tiled ? w2_rows * (c.ffn / kGemmBK) : w2_rows,
                           L->w_tiled ? kGemmBK : c.ffn, gemm_b_box_rows(gemm_cta_group(1)))))
    return rc;
  if ((rc = make_tmap_bf16(&L->map_w2_single, L->w2,
                           L->w_tiled ? w2_rows * (c.ffn / kGemmBK) : w2_rows,
                           L->w_tiled ? kGemmBK : c.ffn, gemm_b_box_rows(1))))
    return rc;
  // the tcgen05 gate needs the resident shards' hs buffers as one arena
  const int64_t hs_stride = c.max_tokens * (int64_t)c.hidden * 2;
  bool arena = gate_tc_supported(c.n_experts, c.top_k, c.hidden);
  for (int i = 1; i < c.shard_count && arena; ++i)
    arena = static_cast<char*>(L->buf[SMOE_BUF_HS][i]) ==
            static_cast<char*>(L->buf[SMOE_BUF_HS][0]) + i * hs_stride;
  L->gate_tc = false;
  if (arena &&
      make_tmap_bf16(&L->map_hs, L->buf[SMOE_BUF_HS][0], c.shard_count * (int64_t)c.max_tokens,
                     c.hidden, 128) == SMOE_OK &&
      make_tmap_bf16(&L->map_wg, L->w_gate, c.n_experts, c.hidden,
                     gate_tc_rows(c.n_experts)) == SMOE_OK)
    L->gate_tc = true;
  L->maps_ready = true;
  L->maps_cg_up = gemm_cta_group(0);
  L->maps_cg_down = gemm_cta_group(1);
  return SMOE_OK;
}

static LocalRows local_rows(const smoe_layer* L) {
  LocalRows lr{};
  lr.counts = static_cast<const int32_t*>(L->buf[SMOE_BUF_PLAN_COUNTS][0]);
  lr.group = static_cast<const int64_t*>(L->buf[SMOE_BUF_GROUP][0]);
  lr.forward = static_cast<const int64_t*>(L->buf[SMOE_BUF_FORWARD][0]);
  lr.shard_begin = L->cfg.shard_begin;
  lr.shard_count = L->cfg.shard_count;
  lr.n_shards = L->cfg.n_shards;
  return lr;
}

extern "C" int smoe_layer_barrier(smoe_layer* L, void* stream) {
  if (!L) return SMOE_ERR_INVALID_ARG;
  if (L->cfg.world_size <= 1) return SMOE_OK;
  // signal pads are bound per shard; pick one per process (shards are
  // distributed contiguously: process r owns shards [r*spp, (r+1)*spp))
  ShardPtrs sig{};
  const int spp = L->cfg.n_shards / L->cfg.world_size;
  for (int r = 0; r < L->cfg.world_size; ++r)
    sig.p[r] = static_cast<char*>(L->buf[SMOE_BUF_SIGNAL][r * spp]);
  return launch_barrier(sig, L->cfg.world_size, L->cfg.world_rank,
                        static_cast<uint32_t*>(L->buf[SMOE_BUF_SIGNAL][L->cfg.shard_begin]),
                        static_cast<uint32_t*>(L->buf[SMOE_BUF_EPOCH][0]), as_stream(stream));
}

static int layer_stage(smoe_layer* L, int32_t stage, const int64_t* tokens,
                       const int64_t* hist, int32_t hist_depth, int64_t n, void* stream);

// narrow GEMM m-blocks while the batch averages <= gemm_narrow_max_rows()
// routed rows per expert (any routing is correct: an expert with more rows
// takes several 32-row m-blocks)
static bool narrow_gemm(const smoe_layer* L, int64_t n) {
  const auto& c = L->cfg;
  return L->local_slots <= kGemmNarrowMaxProblems &&
         n * (int64_t)c.top_k <= (int64_t)gemm_narrow_max_rows() * c.n_experts;
}

// at most gemm_pair_min_rows() routed rows per expert on average: the layer's
// down GEMM runs one SM per 128-row tile (see EXPERT_DOWN)
static bool down_single_sm(const smoe_layer* L, int64_t n) {
  return n * (int64_t)L->cfg.top_k <= (int64_t)gemm_pair_min_rows() * L->cfg.n_experts;
}

// cta_group of the up GEMM for this batch: the SM pair only when the option
// asks for it and the batch is past the one-SM down GEMM's range (decode
// sizes stream weights; one SM per tile there, and the early down GEMM's
// readiness counters assume it)
static int up_cg(const smoe_layer* L, int64_t n) {
  return (L->maps_cg_up == 2 && !down_single_sm(L, n)) ? 2 : 1;
}

// down GEMM started early (SMOE_OPT_EARLY_DOWN): both GEMMs one SM per
// 128-row tile, the down GEMM launched under PDL
static bool early_down(const smoe_layer* L, int64_t n) {
  // (pdl_enabled() answers for the stage being launched: ask for the down GEMM's)
  return gemm_early_down() && down_single_sm(L, n) && !narrow_gemm(L, n) && up_cg(L, n) == 1 &&
         pdl_stage_enabled(SMOE_STAGE_EXPERT_DOWN);
}

// hist: [n, hist_width] window of the previous layers' top-1 clusters (oldest
// digit first), of which the newest hist_depth digits are valid.  The lookup
// uses the n-gram table only for a full window (depth == width; the
// reference passes histories=None for the first n layers, scheduler.py:84-89);
// a partial window still feeds the next window's shift (COMBINE_SAG).
extern "C" int smoe_layer_stage_hist(smoe_layer* L, int32_t stage, const int64_t* tokens,
                                     const int64_t* hist, int32_t hist_width,
                                     int32_t hist_depth, int64_t n, void* stream) {
  if (!L) return SMOE_ERR_INVALID_ARG;
  if (hist) {
    // the kernels index the window as [n, hist_len]: any other width would
    // be misread (or read past the buffer)
    if (hist_width != L->hist_len || hist_depth < 0 || hist_depth > hist_width)
      return SMOE_ERR_INVALID_ARG;
  } else {
    hist_depth = 0;
  }
  set_pdl_stage(stage);
  const int rc = layer_stage(L, stage, tokens, hist, hist_depth, n, stream);
  set_pdl_stage(-1);
  return rc;
}

extern "C" int smoe_layer_stage(smoe_layer* L, int32_t stage, const int64_t* tokens,
                                const int64_t* hist, int64_t n, void* stream) {
  if (!L) return SMOE_ERR_INVALID_ARG;
  return smoe_layer_stage_hist(L, stage, tokens, hist, L->hist_len, L->hist_len, n, stream);
}

static int layer_stage(smoe_layer* L, int32_t stage, const int64_t* tokens,
                       const int64_t* hist, int32_t hist_depth, int64_t n, void* stream) {
  if (!L || n < 0 || n > L->cfg.max_tokens) return SMOE_ERR_INVALID_ARG;
  int rc = ensure_maps(L);
  if (rc) return rc;
  const auto& c = L->cfg;
  cudaStream_t st = as_stream(stream);
  const LocalRows lr = local_rows(L);
  int64_t* stats = static_cast<int64_t*>(L->buf[SMOE_BUF_STATS][0]);
  int32_t* err = static_cast<int32_t*>(L->buf[SMOE_BUF_ERR][0]);
  switch (stage) {
    case SMOE_STAGE_PLAN: {
      if (n > 0 && !tokens) return SMOE_ERR_INVALID_ARG;
      const int64_t* lookup_hist = (hist && hist_depth >= L->hist_len) ? hist : nullptr;
      rc = layer_plan(tokens, n, lookup_hist, L->hist_len, L->t_labels, L->t_conf, L->vocab,
                        L->a_best, L->a_conf, L->a_rows, c.n_shards,
                        static_cast<int64_t*>(L->buf[SMOE_BUF_DEV][0]),
                        static_cast<int64_t*>(L->buf[SMOE_BUF_FORWARD][0]),
                        static_cast<int64_t*>(L->buf[SMOE_BUF_INVERSE][0]),
                        static_cast<int32_t*>(L->buf[SMOE_BUF_PLAN_COUNTS][0]),
                        static_cast<int64_t*>(L->buf[SMOE_BUF_GROUP][0]), err,
                        L->buf[SMOE_BUF_WORKSPACE][0], plan_ws_aligned(&c), stats,
                        SMOE_STAT__COUNT, st, L->ready_d, L->local_slots + 1);
      L->ready_zeroed = rc == SMOE_OK;
      return rc;
    }
    case SMOE_STAGE_SRS:
      // every process's partials for this batch are written before any peer
      // reads them (and the previous batch's reads ended at its ROUTE barrier)
      rc = smoe_layer_barrier(L, stream);
      if (rc) return rc;
      if (L->pipeline == SMOE_PIPELINE_DSMOE) {
        // DS-MoE: every process receives the full sum (two-shot all-reduce),
        // then each rank takes its own rows of it
        int32_t n_ar = 0;
        const ShardPtrs ar = distinct_ptrs_local_first(L, SMOE_BUF_AR, &n_ar);
        rc = launch_allreduce(peer_ptrs(L, SMOE_BUF_PARTIAL), c.hidden, n, c.shard_begin,
                              c.shard_count, c.n_shards, ar, n_ar, st);
        if (rc) return rc;
        rc = smoe_layer_barrier(L, stream);
        if (rc) return rc;
        ShardPtrs src{};
        src.p[0] = ar.p[0];
        return launch_srs(lr, src, c.hidden, local_ptrs(L, SMOE_BUF_HS), n, st, 1);
      }
      return launch_srs(lr, peer_ptrs(L, SMOE_BUF_PARTIAL), c.hidden, local_ptrs(L, SMOE_BUF_HS),
                        n, st);
    case SMOE_STAGE_GATE:
      if (L->gate_tc && gate_tc_enabled()) {
        GateTcArgs g{};
        g.counts = lr.counts;
        g.shard_begin = c.shard_begin;
        g.shard_count = c.shard_count;
        g.rows_per_shard = c.max_tokens;
        g.num_k_blocks = c.hidden / kGemmBK;
        g.n_experts = c.n_experts;
        g.k = c.top_k;
        g.renorm = c.renormalize;
        g.b_gate = L->b_gate;
        g.slot_owner = L->slot_owner_d;
        g.topk_ids = local_ptrs(L, SMOE_BUF_TOPK_IDS);
        g.topk_w = local_ptrs(L, SMOE_BUF_TOPK_W);
        g.stats = stats;
        // decode-sized batches (n <= 128: every shard's rows are one gate
        // tile): the gate CTA of each shard also ranks its pairs and
        // publishes its count row -- the ROUTE stage then only barriers
        L->route_fused = gate_route_fused() && n > 0 && n <= 128;
        if (L->route_fused) {
          g.route = 1;
          g.pair_rank = local_ptrs(L, SMOE_BUF_PAIR_RANK);
          g.count_bufs = distinct_ptrs(L, SMOE_BUF_COUNTS, &g.n_count_bufs);
        }
        return launch_gate_tc(L->map_hs, L->map_wg, g, n, st);
      }
      L->route_fused = false;
      return launch_gate(lr, local_ptrs(L, SMOE_BUF_HS), c.hidden, L->w_gate, L->b_gate,
                         c.n_experts, c.top_k, c.renormalize, L->slot_owner_d,
                         local_ptrs(L, SMOE_BUF_TOPK_IDS), local_ptrs(L, SMOE_BUF_TOPK_W), stats,
                         n, st);
    case SMOE_STAGE_ROUTE: {
      if (L->route_fused) {               // done by the gate kernel of this forward
        L->route_fused = false;
        return smoe_layer_barrier(L, stream);
      }
      int32_t nb = 0;
      ShardPtrs cb = distinct_ptrs(L, SMOE_BUF_COUNTS, &nb);
      int32_t* chunk_counts = reinterpret_cast<int32_t*>(
          static_cast<char*>(L->buf[SMOE_BUF_WORKSPACE][0]) + plan_ws_aligned(&c));
      rc = launch_route(lr, c.n_experts, c.top_k, local_ptrs(L, SMOE_BUF_TOPK_IDS),
                        local_ptrs(L, SMOE_BUF_PAIR_RANK), cb, nb, chunk_counts, n, st);
      if (rc) return rc;
      return smoe_layer_barrier(L, stream);
    }
    case SMOE_STAGE_DISPATCH: {
      // deduplicated dispatch across processes (every shard's fan-out table bound)
      bool dedup = g_dedup_dispatch && c.world_size > 1;
      for (int g = 0; g < c.n_shards && dedup; ++g) dedup = L->buf[SMOE_BUF_XFAN][g] != nullptr;
      const ShardPtrs xfan = dedup ? peer_ptrs(L, SMOE_BUF_XFAN) : ShardPtrs{};
      int64_t* problems = static_cast<int64_t*>(L->buf[SMOE_BUF_PROBLEMS][0]);
      rc = launch_dispatch(lr, c.n_experts, c.top_k, c.hidden,
                           static_cast<const int32_t*>(L->buf[SMOE_BUF_COUNTS][c.shard_begin]),
                           L->slot_owner_d, L->slot_first_d, local_ptrs(L, SMOE_BUF_HS),
                           local_ptrs(L, SMOE_BUF_TOPK_IDS), local_ptrs(L, SMOE_BUF_PAIR_RANK),
                           peer_ptrs(L, SMOE_BUF_XIN), peer_ptrs(L, SMOE_BUF_XMETA),
                           c.expert_rows, problems, err, n, st, xfan, stats);
      if (rc) return rc;
      rc = smoe_layer_barrier(L, stream);
      if (rc || !dedup) return rc;
      // the owners' side: copy each remote token row to its other experts here
      return launch_fanout(problems, L->local_slots, peer_ptrs(L, SMOE_BUF_XIN), xfan,
                           c.shard_begin, c.expert_rows, c.hidden, L->slot_owner_d,
                           L->slot_first_d,
                           std::min<int64_t>(n * c.top_k, c.expert_rows * c.shard_count), st);
    }
    case SMOE_STAGE_EXPERT_UP: {
      GemmArgs a{};
      a.problems = static_cast<const int64_t*>(L->buf[SMOE_BUF_PROBLEMS][0]);
      a.num_problems = L->local_slots;
      a.num_k_blocks = c.hidden / kGemmBK;
      a.n_tiles_n = 2 * c.ffn / kGemmBN;
      a.n_b = 2 * c.ffn;
      a.c = static_cast<char*>(L->buf[SMOE_BUF_HMID][0]);
      a.ldc = c.ffn;
      a.b_tiled = L->w_tiled;
      L->ready_armed = early_down(L, n);
      // decode sizes: launched under PDL (its CTA placement does not matter
      // when no two tiles share a weight tile), behind counters the PLAN
      // kernel reset -- a memset here would sit between the dispatch and
      // this launch (~6 us of launch gap, tools/probe/forward_timeline.py)
      const bool up_pdl = L->ready_armed && L->ready_zeroed && g_decode_up_pdl;
      if (L->ready_armed) {
        if (!L->ready_zeroed)              // stage calls without this forward's PLAN
          SMOE_CUDA_TRY(
              cudaMemsetAsync(L->ready_d, 0, sizeof(int32_t) * (L->local_slots + 1), st));
        a.ready = L->ready_d;
        a.ready_role = 1;
      }
      L->ready_zeroed = false;
      if (up_pdl) set_pdl_stage(-1);       // PDL as for any early-launched stage
      struct Restore {
        bool on;
        ~Restore() { if (on) set_pdl_stage(SMOE_STAGE_EXPERT_UP); }
      } restore{up_pdl};
      // decode-sized batches stream the weights: narrow m-blocks keep more
      // weight tiles in flight per SM (gemm_tcgen05.cu, GemmShape NARROW)
      if (narrow_gemm(L, n) && up_cg(L, n) == 1)
        return launch_grouped_gemm(L->map_x_narrow, L->map_w13_single, a, kEpiSwiGLU, 0, st);
      return up_cg(L, n) == 2
                 ? launch_grouped_gemm(L->map_x, L->map_w13, a, kEpiSwiGLU, 2, st)
                 : launch_grouped_gemm(L->map_x, L->map_w13_single, a, kEpiSwiGLU, 1, st);
    }
    case SMOE_STAGE_EXPERT_DOWN: {
      GemmArgs a{};
      a.problems = static_cast<const int64_t*>(L->buf[SMOE_BUF_PROBLEMS][0]);
      a.num_problems = L->local_slots;
      a.num_k_blocks = c.ffn / kGemmBK;
      a.n_tiles_n = c.hidden / kGemmBN;
      a.n_b = c.hidden;
      a.meta = static_cast<const int64_t*>(L->buf[SMOE_BUF_XMETA][c.shard_begin]);
      for (int g = 0; g < c.n_shards; ++g) a.dst_base[g] = static_cast<char*>(L->buf[SMOE_BUF_YPAIR][g]);
      a.ldd = c.hidden;
      a.b_tiled = L->w_tiled;
      // <= gemm_pair_min_rows() routed rows per expert on average: one SM
      // per tile (decode sizes: one wave instead of the pair's 1.7, 5-16%,
      // profiles/r1_down_cta_group_small.jsonl; mid sizes: half the padding
      // rows of the pair's 256-row tiles)
      const bool small = down_single_sm(L, n);
      // only behind an up GEMM that publishes this forward's counts (the
      // option could have changed between the two stage calls)
      if (L->ready_armed && early_down(L, n)) {
        a.ready = L->ready_d;
        a.ready_role = 2;
        a.ready_up_tile_m = kGemmBM;
        a.ready_up_n_tiles = 2 * c.ffn / kGemmBN;
        a.err = err;
#ifndef SMOE_DYN_DOWN
#define SMOE_DYN_DOWN 1
#endif
        // its CTAs start staggered (on the SMs the up GEMM frees): tiles
        // from a counter, so the early starters take more of them
        if (SMOE_DYN_DOWN) a.tile_counter = L->ready_d + L->local_slots;
      }
      L->ready_armed = false;
      rc = narrow_gemm(L, n)
               ? launch_grouped_gemm(L->map_h_narrow, L->map_w2_single, a, kEpiScatter, 0, st)
           : small ? launch_grouped_gemm(L->map_h, L->map_w2_single, a, kEpiScatter, 1, st)
                 : launch_grouped_gemm(L->map_h, L->map_w2, a, kEpiScatter, L->maps_cg_down, st);
      if (rc) return rc;
      return smoe_layer_barrier(L, stream);
    }
    case SMOE_STAGE_COMBINE_SAG: {
      HistUpdate hu{};
      hu.hist_in = hist;
      hu.hist_len = L->hist_len;
      hu.slot_owner = L->slot_owner_d;
      hu.topk_ids = local_ptrs(L, SMOE_BUF_TOPK_IDS);
      hu.n_hist_outs = 0;
      if (L->buf[SMOE_BUF_HIST_OUT][0] && hu.hist_len > 0 && hu.hist_len <= 32)
        hu.hist_outs = distinct_ptrs(L, SMOE_BUF_HIST_OUT, &hu.n_hist_outs);
      // SAG: each token's row goes once to every distinct output buffer (one
      // per process: co-resident shards share their process's output)
      int32_t n_outs = 0;
      if (L->pipeline == SMOE_PIPELINE_DSMOE) {
        // DS-MoE: combine into every process's all-gather buffer at the
        // token's block slot, then restore the original order locally
        const ShardPtrs ag = distinct_ptrs_local_first(L, SMOE_BUF_AG, &n_outs);
        rc = launch_combine_sag(lr, c.top_k, c.hidden, resident_ptrs(L, SMOE_BUF_YPAIR),
                                local_ptrs(L, SMOE_BUF_TOPK_W), ag, n_outs, hu, n, st,
                                L->ag_rows, err);
        if (rc) return rc;
        rc = smoe_layer_barrier(L, stream);
        if (rc) return rc;
        return smoe_gather_rows(ag.p[0], L->ag_rows, 2, c.hidden,
                                static_cast<const int64_t*>(L->buf[SMOE_BUF_INVERSE][0]), n, 0,
                                0, L->buf[SMOE_BUF_OUT][c.shard_begin], err, stream);
      }
      const ShardPtrs outs = distinct_ptrs(L, SMOE_BUF_OUT, &n_outs);
      rc = launch_combine_sag(lr, c.top_k, c.hidden, resident_ptrs(L, SMOE_BUF_YPAIR),
                              local_ptrs(L, SMOE_BUF_TOPK_W), outs, n_outs, hu, n, st);
      if (rc) return rc;
      return smoe_layer_barrier(L, stream);
    }
    default:
      return SMOE_ERR_INVALID_ARG;
  }
}

extern "C" int smoe_layer_forward_hist(smoe_layer* L, const int64_t* tokens,
                                       const int64_t* hist, int32_t hist_width,
                                       int32_t hist_depth, int64_t n, void* stream) {
  for (int s = 0; s < SMOE_STAGE__COUNT; ++s) {
    int rc = smoe_layer_stage_hist(L, s, tokens, hist, hist_width, hist_depth, n, stream);
    if (rc) return rc;
  }
  return SMOE_OK;
}

extern "C" int smoe_layer_forward(smoe_layer* L, const int64_t* tokens, const int64_t* hist,
                                  int64_t n, void* stream) {
  if (!L) return SMOE_ERR_INVALID_ARG;
  return smoe_layer_forward_hist(L, tokens, hist, L->hist_len, L->hist_len, n, stream);
}

// ---------------------------------------------------------------- single-rank C-ABI
extern "C" int smoe_gate_topk(const void* h, int64_t rows, int32_t hidden, const void* w_gate,
                              const float* b_gate, int32_t n_experts, int32_t top_k,
                              int32_t renormalize, const int32_t* expert_owner, int32_t my_shard,
                              int32_t* topk_ids, float* topk_w, int64_t* stats, void* stream) {
  if (rows < 0 || !w_gate || !expert_owner || !topk_ids || !topk_w) return SMOE_ERR_INVALID_ARG;
  if (rows == 0) return SMOE_OK;
  if (!h) return SMOE_ERR_INVALID_ARG;
  LocalRows lr{};
  lr.counts = nullptr;
  lr.single_rows = rows;
  lr.shard_begin = my_shard;     // locality: expert_owner[e] == my_shard
  lr.shard_count = 1;
  lr.n_shards = my_shard + 1;
  ShardPtrs hp{}, ip{}, wp{};
  hp.p[0] = static_cast<char*>(const_cast<void*>(h));
  ip.p[0] = reinterpret_cast<char*>(topk_ids);
  wp.p[0] = reinterpret_cast<char*>(topk_w);
  return launch_gate(lr, hp, hidden, w_gate, b_gate, n_experts, top_k, renormalize, expert_owner,
                     ip, wp, stats, rows, as_stream(stream));
}

extern "C" int smoe_pair_offsets(const int32_t* topk_ids, int64_t rows, int32_t top_k,
                                 int32_t n_experts, int32_t* pair_pos, int32_t* counts,
                                 void* stream) {
  if (rows < 0 || !counts || (rows > 0 && (!topk_ids || !pair_pos))) return SMOE_ERR_INVALID_ARG;
  return launch_pair_offsets(topk_ids, rows, top_k, n_experts, pair_pos, counts, as_stream(stream));
}

extern "C" int smoe_pack_rows(const void* src, int64_t rows, int32_t top_k, int32_t hidden,
                              const int32_t* pair_pos, void* dst, void* stream) {
  if (rows < 0 || (rows > 0 && (!src || !pair_pos || !dst))) return SMOE_ERR_INVALID_ARG;
  return launch_pack_rows(src, rows, top_k, hidden, pair_pos, dst, as_stream(stream));
}

extern "C" int smoe_combine_rows(const void* y, const int32_t* pair_pos, const float* topk_w,
                                 int64_t rows, int32_t top_k, int32_t hidden, void* out,
                                 void* stream) {
  if (rows < 0 || (rows > 0 && (!y || !pair_pos || !topk_w || !out))) return SMOE_ERR_INVALID_ARG;
  return launch_combine_rows(y, pair_pos, topk_w, rows, top_k, hidden, out, as_stream(stream));
}

extern "C" int smoe_set_option(int32_t key, int32_t value) {
  switch (key) {
    case SMOE_OPT_GEMM_CTA_GROUP_UP:
    case SMOE_OPT_GEMM_CTA_GROUP_DOWN:
      if (value != 1 && value != 2) return SMOE_ERR_INVALID_ARG;
      set_gemm_cta_group(key == SMOE_OPT_GEMM_CTA_GROUP_DOWN, value);
      return SMOE_OK;
    case SMOE_OPT_GATE_TENSOR:
      if (value != 0 && value != 1) return SMOE_ERR_INVALID_ARG;
      set_gate_tc_enabled(value);
      return SMOE_OK;
    case SMOE_OPT_GEMM_PAIR_MIN_ROWS:
      if (value < 0) return SMOE_ERR_INVALID_ARG;
      set_gemm_pair_min_rows(value);
      return SMOE_OK;
    case SMOE_OPT_GEMM_NARROW_MAX_ROWS:
      if (value < 0) return SMOE_ERR_INVALID_ARG;
      set_gemm_narrow_max_rows(value);
      return SMOE_OK;
    case SMOE_OPT_DEDUP_DISPATCH:
      if (value != 0 && value != 1) return SMOE_ERR_INVALID_ARG;
      g_dedup_dispatch = value;
      return SMOE_OK;
    case SMOE_OPT_EARLY_DOWN:
      if (value != 0 && value != 1) return SMOE_ERR_INVALID_ARG;
      set_gemm_early_down(value);
      return SMOE_OK;
    case SMOE_OPT_GEMM_GROUP_M_UP:
    case SMOE_OPT_GEMM_GROUP_M_DOWN:
      if (value < -4096 || value > 4096) return SMOE_ERR_INVALID_ARG;
      set_gemm_group_m(key == SMOE_OPT_GEMM_GROUP_M_DOWN, value);
      return SMOE_OK;
    case SMOE_OPT_DECODE_UP_PDL:
      if (value != 0 && value != 1) return SMOE_ERR_INVALID_ARG;
      g_decode_up_pdl = value;
      return SMOE_OK;
    case SMOE_OPT_ROUTE_IN_GATE:
      if (value != 0 && value != 1) return SMOE_ERR_INVALID_ARG;
      set_gate_route_fused(value);
      return SMOE_OK;
    case SMOE_OPT_PDL:
      if (value != 0 && value != 1) return SMOE_ERR_INVALID_ARG;
      set_pdl_enabled(value);
      return SMOE_OK;
    case SMOE_OPT_PDL_STAGES:
      if (value < 0 || value > 0xff) return SMOE_ERR_INVALID_ARG;
      set_pdl_stage_mask(value);
      return SMOE_OK;
    default:
      return SMOE_ERR_INVALID_ARG;
  }
}

extern "C" int smoe_get_option(int32_t key) {
  if (key == SMOE_OPT_GEMM_CTA_GROUP_UP) return gemm_cta_group(0);
  if (key == SMOE_OPT_GEMM_CTA_GROUP_DOWN) return gemm_cta_group(1);
  if (key == SMOE_OPT_GATE_TENSOR) return gate_tc_enabled();
  if (key == SMOE_OPT_GEMM_PAIR_MIN_ROWS) return gemm_pair_min_rows();
  if (key == SMOE_OPT_GEMM_NARROW_MAX_ROWS) return gemm_narrow_max_rows();
  if (key == SMOE_OPT_PDL) return pdl_enabled();
  if (key == SMOE_OPT_PDL_STAGES) return pdl_stage_mask();
  if (key == SMOE_OPT_DEDUP_DISPATCH) return g_dedup_dispatch;
  if (key == SMOE_OPT_EARLY_DOWN) return gemm_early_down();
  if (key == SMOE_OPT_ROUTE_IN_GATE) return gate_route_fused();
  if (key == SMOE_OPT_DECODE_UP_PDL) return g_decode_up_pdl;
  if (key == SMOE_OPT_GEMM_GROUP_M_UP) return gemm_group_m(0);
  if (key == SMOE_OPT_GEMM_GROUP_M_DOWN) return gemm_group_m(1);
  return -1;
}

// ---------------------------------------------------------------- standalone SRS / SAG
extern "C" int smoe_srs(const void* const* partials, int32_t n_shards, int32_t shard_begin,
                        int32_t shard_count, const int64_t* forward, const int32_t* counts,
                        const int64_t* group, int64_t n_tokens, int32_t hidden,
                        void* const* outs, void* stream) {
  if (!partials || !outs || !forward || !counts || !group || n_tokens < 0 || hidden <= 0)
    return SMOE_ERR_INVALID_ARG;
  if (n_shards < 1 || n_shards > SMOE_MAX_SHARDS || shard_begin < 0 || shard_count < 1 ||
      shard_begin + shard_count > n_shards)
    return SMOE_ERR_INVALID_ARG;
  LocalRows lr{};
  lr.counts = counts; lr.group = group; lr.forward = forward;
  lr.shard_begin = shard_begin; lr.shard_count = shard_count; lr.n_shards = n_shards;
  ShardPtrs p{}, o{};
  for (int g = 0; g < n_shards; ++g) p.p[g] = static_cast<char*>(const_cast<void*>(partials[g]));
  for (int i = 0; i < shard_count; ++i) o.p[i] = static_cast<char*>(outs[i]);
  return launch_srs(lr, p, hidden, o, n_tokens, as_stream(stream));
}

extern "C" int smoe_sag(const void* const* blocks, int32_t n_shards, const int64_t* forward,
                        const int32_t* counts, const int64_t* group, int64_t n_tokens,
                        int32_t hidden, void* const* outs, int32_t n_outs, void* stream) {
  if (!blocks || !outs || !forward || !counts || !group || n_tokens < 0 || hidden <= 0)
    return SMOE_ERR_INVALID_ARG;
  if (n_shards < 1 || n_shards > SMOE_MAX_SHARDS || n_outs < 1 || n_outs > SMOE_MAX_SHARDS)
    return SMOE_ERR_INVALID_ARG;
  LocalRows lr{};
  lr.counts = counts; lr.group = group; lr.forward = forward;
  lr.shard_begin = 0; lr.shard_count = n_shards; lr.n_shards = n_shards;
  ShardPtrs b{}, o{};
  for (int g = 0; g < n_shards; ++g) b.p[g] = static_cast<char*>(const_cast<void*>(blocks[g]));
  for (int i = 0; i < n_outs; ++i) o.p[i] = static_cast<char*>(outs[i]);
  return launch_sag(lr, hidden, b, o, n_outs, n_tokens, as_stream(stream));
}

#ifdef SMOE_DEBUG_READY
extern "C" int smoe_debug_layer_ready(smoe_layer* L, int32_t* host, int32_t n) {
  return cudaMemcpy(host, L->ready_d, sizeof(int32_t) * n, cudaMemcpyDeviceToHost) == cudaSuccess
             ? 0 : -1;
}
#endif
