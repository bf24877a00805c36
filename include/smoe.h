/*
 * smoe.h — C-ABI of the B200-native speculative-token-shuffling MoE layer.
 *
 * This is the drop-in boundary for the online hot path of Speculative MoE
 * (arXiv 2503.04398).  The reference (`/root/reference/pkg/src/moesched`) is a
 * pure-Python package; its "FFI" is the Python module API.  Each entry point
 * below names the reference function it replaces (file:line under
 * /root/reference/pkg/src/moesched/).  The Python mirror that a user of the
 * reference imports is `paper_2503_04398_b200` (ctypes over this library);
 * INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless the parameter name ends in _h;
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     and asynchronous (no host synchronisation inside the library);
 *   - `err` (nullable) is a device int32 flag; kernels OR in SMOE_ERRBIT_*
 *     bits for data-dependent failures the reference raises on (the Python
 *     mirror reads it and raises the reference's exception class);
 *   - the return value reports argument/launch errors immediately.
 *   - no CPU fallback: if the device is not an sm_100 part the calls return
 *     SMOE_ERR_CUDA.
 */
#ifndef SMOE_H_
#define SMOE_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (return values) ------------------------------------- */
#define SMOE_OK                 0
#define SMOE_ERR_INVALID_ARG    1   /* bad size / null pointer               */
#define SMOE_ERR_LENGTH         2   /* scheduler.py:129-130, :155-156        */
#define SMOE_ERR_UNSUPPORTED    3   /* shape outside the kernels' envelope    */
#define SMOE_ERR_CUDA           4   /* launch / runtime failure               */
#define SMOE_ERR_CLUSTERS       5   /* scheduler.py:37-38                     */
#define SMOE_ERR_GATE_WIDTH     6   /* scheduler.py:217-218                   */

/* ---- data-dependent error bits written to *err ------------------------- */
#define SMOE_ERRBIT_DEVICE_RANGE   1  /* scheduler.py:131-132 SchedulerError */
#define SMOE_ERRBIT_EXPERT_LABEL   2  /* scheduler.py:204-206 SchedulerError */
#define SMOE_ERRBIT_TOKEN_RANGE    4  /* numpy IndexError on labels[tokens]  */
#define SMOE_ERRBIT_HISTORY_RANGE  8  /* numpy IndexError on confidence[rows]*/
#define SMOE_ERRBIT_INDEX_RANGE   16  /* numpy IndexError on a fancy index   */
#define SMOE_ERRBIT_CAPACITY      32  /* a layer buffer would overflow        */
#define SMOE_ERRBIT_TIMEOUT       64  /* an in-kernel wait on another grid    */
                                    /* exceeded its bound (results invalid) */

#define SMOE_MAX_SHARDS 16          /* EP degree G supported by the layer    */
#define SMOE_MAX_PLAN_DEVICES 1024  /* n_devices supported by rebatch plan   */

const char* smoe_version(void);
/* Process-wide tuning switches. */
#define SMOE_OPT_GEMM_CTA_GROUP_UP   0  /* SwiGLU GEMM: 1 = 128x256 tile per SM (default), */
#define SMOE_OPT_GEMM_CTA_GROUP_DOWN 1  /* down GEMM: 2 = 256x256 tile per SM pair (default) */
#define SMOE_OPT_GATE_TENSOR         2  /* layer gate: 1 = tcgen05 kernel (default), */
                                        /* 0 = mma.sync / CUDA-core kernels          */
#define SMOE_OPT_GEMM_PAIR_MIN_ROWS  3  /* layer down GEMM: one SM per tile while    */
                                        /* n*k <= this * n_experts (default 1024)    */
#define SMOE_OPT_PDL                 4  /* layer kernels: 1 = programmatic dependent */
                                        /* launch (default; env SMOE_PDL=0 to start  */
                                        /* with 0), 0 = plain stream order           */
#define SMOE_OPT_PDL_STAGES          5  /* bit mask over SMOE_STAGE_*: stages whose  */
                                        /* kernels launch early (default: all but    */
                                        /* EXPERT_UP; env SMOE_PDL_STAGES)           */
#define SMOE_OPT_GEMM_NARROW_MAX_ROWS 6 /* layer GEMMs: 32-row m-blocks, 5-stage     */
                                        /* weight ring while n*k <= this * n_experts */
                                        /* (default 0 = off)                         */
#define SMOE_OPT_DEDUP_DISPATCH      7  /* layers spanning processes: 1 (default) =   */
                                        /* send each token row once per remote shard */
                                        /* (the owner fans it out to its experts),   */
                                        /* 0 = one row per remote (token, expert)    */
#define SMOE_OPT_EARLY_DOWN          8  /* decode-sized batches: the down GEMM's  */
                                        /* CTAs start on the SMs the up GEMM's     */
                                        /* tail frees and wait per expert for its  */
                                        /* hidden rows (1 = default, 0 = off)      */
#define SMOE_OPT_ROUTE_IN_GATE       9  /* batches of <= 128 tokens: the tcgen05   */
                                        /* gate ranks each shard's pairs and       */
                                        /* publishes its count row (no route       */
                                        /* kernel; 1 = default, 0 = off)           */
#define SMOE_OPT_GEMM_GROUP_M_UP    10  /* tile order of the layer's up / down GEMM: */
#define SMOE_OPT_GEMM_GROUP_M_DOWN  11  /* 0 = derived (default), > 0 m-blocks per   */
                                        /* group, < 0 -(n-blocks per group)          */
#define SMOE_OPT_DECODE_UP_PDL      12  /* batches with the early-started down GEMM: */
                                        /* the up GEMM launches under PDL too (its  */
                                        /* readiness counters are reset by the plan */
                                        /* kernel; 1 = default, 0 = plain launch)   */
int smoe_set_option(int32_t key, int32_t value);
int smoe_get_option(int32_t key);
const char* smoe_status_string(int status);
/* 1 when the current device is sm_100 (B200) and the kernels can run. */
int smoe_device_ok(void);

/* ======================================================================= *
 *  Scheduler (reference: scheduler.py)                                     *
 * ======================================================================= */

/* lookup_devices (scheduler.py:82-98).
 *   dev[i] = a_best[row_i] if hist && a_conf[row_i] > t_conf[tok_i] (strict,
 *   float32) else t_labels[tok_i];  row_i = base-E code of hist[i, :]
 *   (oldest digit most significant, predictor.py:149-154).
 * tokens int64[n]; hist int64[n, hist_len] row-major or NULL; negative ids
 * wrap like numpy (id + vocab); a_best/a_conf have n_clusters^hist_len rows
 * (the reference's DeviceNGramTable.best / .confidence, predictor.py:72-78)
 * and a_rows = n_clusters^ngram_n rows.  Like the vectorised reference, the
 * history width is not checked against the table depth: a row code outside
 * [-a_rows, a_rows) sets SMOE_ERRBIT_HISTORY_RANGE (numpy IndexError).
 * Out-of-range token ids set SMOE_ERRBIT_TOKEN_RANGE. */
int smoe_lookup_devices(const int64_t* tokens, int64_t n,
                        const int64_t* hist, int32_t hist_len,
                        const int16_t* t_labels, const float* t_conf, int64_t vocab,
                        const int16_t* a_best, const float* a_conf,
                        int64_t a_rows, int32_t n_clusters,
                        int64_t* dev_out, int32_t* err, void* stream);

/* Workspace bytes needed by smoe_rebatch_plan / smoe_lookup_plan. */
size_t smoe_plan_workspace_bytes(int64_t n, int32_t n_devices);

/* rebatch_tokens index half (scheduler.py:119-149): stable device partition
 * padded to the largest group.
 *   group = max_d #{i : dev[i] = d}                (scheduler.py:134-135)
 *   inverse[i] = dev[i]*group + #{j < i : dev[j] = dev[i]}
 *   forward[inverse[i]] = i, every other slot of [0, G*group) = -1
 * devices int64[n]; forward must hold n_devices*n entries (only the first
 * n_devices*group are written); counts int32[n_devices]; group int64[1].
 * Labels outside [0, n_devices) set SMOE_ERRBIT_DEVICE_RANGE. */
int smoe_rebatch_plan(const int64_t* devices, int64_t n, int32_t n_devices,
                      int64_t* forward, int64_t* inverse, int32_t* counts,
                      int64_t* group, int32_t* err,
                      void* workspace, size_t workspace_bytes, void* stream);

/* lookup_devices fused with the rebatch plan (K1 of DESIGN.md): the device
 * labels never round-trip through HBM as int64 unless dev_out != NULL. */
int smoe_lookup_plan(const int64_t* tokens, int64_t n,
                     const int64_t* hist, int32_t hist_len,
                     const int16_t* t_labels, const float* t_conf, int64_t vocab,
                     const int16_t* a_best, const float* a_conf,
                     int64_t a_rows, int32_t n_clusters,
                     int64_t* dev_out, int64_t* forward, int64_t* inverse,
                     int32_t* counts, int64_t* group, int32_t* err,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Row gather, the data half of rebatch_tokens / resume_tokens
 * (scheduler.py:145-146, :157):  dst[i, :] = src[idx[i], :], or pad_value in
 * every element when idx[i] < 0 and pad_negative != 0.  With pad_negative == 0
 * negative indices wrap like numpy.  elem_bytes in {1,2,4,8}; rows are
 * row_elems elements.  idx out of range sets SMOE_ERRBIT_INDEX_RANGE. */
int smoe_gather_rows(const void* src, int64_t n_src, int32_t elem_bytes,
                     int64_t row_elems, const int64_t* idx, int64_t n_out,
                     int32_t pad_negative, int64_t pad_value, void* dst,
                     int32_t* err, void* stream);

/* gate_permutation (scheduler.py:200-210): new_to_old = stable argsort of
 * the expert cluster labels, old_to_new its inverse.  labels int64[N]. */
int smoe_gate_permutation(const int64_t* labels, int32_t n_experts,
                          int32_t n_clusters, int64_t* new_to_old,
                          int64_t* old_to_new, int32_t* err, void* stream);

/* apply_expert_shuffle (scheduler.py:213-219): dst[r, i] = src[r, perm[i]]
 * over `rows` rows of `width` elements (elem_bytes in {1,2,4,8}). */
int smoe_permute_columns(const void* src, int64_t rows, int32_t width,
                         int32_t elem_bytes, const int64_t* perm, void* dst,
                         void* stream);

/* remap_topk (scheduler.py:222-224): dst[i] = table[idx[i]] (numpy wrap for
 * negative idx; out of range sets SMOE_ERRBIT_INDEX_RANGE). */
int smoe_remap_index(const int64_t* idx, int64_t count, const int64_t* table,
                     int64_t table_len, int64_t* dst, int32_t* err,
                     void* stream);

/* Event counting of simulate_layer (comm.py:214):
 *   local = sum_{i<occ, s<k} [expert_dev[experts[i, s]] == token_dev[i]]
 * experts int64[occ, k]; local_out int64[1] (overwritten). */
int smoe_count_local(const int64_t* experts, int64_t occ, int32_t k,
                     const int64_t* expert_dev, int32_t n_experts,
                     const int64_t* token_dev, int64_t* local_out,
                     int32_t* err, void* stream);

/* solver.metrics (solver.py:766-800), the event half: over occ x k events,
 * event (i, j) has expert experts[i*k+j] (experts NULL: expert j, i.e. a
 * dense token x expert matrix with k = N) and integer weight weights[i*k+j]
 * (NULL: 1).  local_out = sum of weights with expert_dev[e] == token_dev[i];
 * loads_out[c] = sum of weights with expert_dev[e] == c (c < n_clusters
 * <= SMOE_MAX_PLAN_DEVICES), the expert-side load whose max / median is the
 * reference's imbalance.  Negative expert ids wrap like numpy; out-of-range
 * ids set SMOE_ERRBIT_INDEX_RANGE, cluster labels outside [0, n_clusters)
 * SMOE_ERRBIT_EXPERT_LABEL. */
int smoe_event_metrics(const int64_t* experts, const int64_t* weights, int64_t occ,
                       int32_t k, const int64_t* expert_dev, int32_t n_experts,
                       const int64_t* token_dev, int32_t n_clusters,
                       int64_t* local_out, int64_t* loads_out, int32_t* err, void* stream);

/* solve_ceo's per-iteration sample scoring (solver.py:380-404, §8f rank 4):
 * counts_nt int32 [n_experts, t] (the token x expert activation counts of
 * the active tokens, TRANSPOSED), ep_samples int32 [n_samples, n_experts]
 * and tk_samples int32 [n_samples, t] cluster labels in [0, n_clusters).
 * ep_score[k] = sum_j max_c mass(k, j, c) and joint[k] = sum_j
 * mass(k, j, tk[k, j]), mass(k, j, c) = sum of counts[j, n] over experts n
 * with ep[k, n] == c (the reference's tensordot + max / gather).  Exact
 * int64 sums.  n_experts <= 64, n_clusters <= 16. */
int smoe_ceo_sample_scores(const int32_t* counts_nt, int32_t t, int32_t n_experts,
                           const int32_t* ep_samples, const int32_t* tk_samples,
                           int32_t n_samples, int32_t n_clusters, int64_t* ep_score,
                           int64_t* joint, void* stream);

/* schedule_requests_dp (scheduler.py:160-183): request r goes to the
 * highest-affinity device still open in its window of n_devices consecutive
 * requests (first maximum wins).  affinities f64[n_requests, n_devices]. */
int smoe_schedule_requests_dp(const double* affinities, int64_t n_requests,
                              int32_t n_devices, int64_t* labels, void* stream);

/* ======================================================================= *
 *  MoE layer (Algorithm 2; no reference code)          *
 * ======================================================================= */

typedef struct smoe_layer smoe_layer;   /* opaque */

typedef struct {
  int32_t n_shards;      /* G: EP degree = token groups = expert clusters    */
  int32_t shard_begin;   /* first shard resident in this process             */
  int32_t shard_count;   /* shards resident in this process (same GPU)       */
  int32_t n_experts;     /* N routed experts                                 */
  int32_t top_k;         /* k                                                */
  int32_t hidden;        /* d                                                */
  int32_t ffn;           /* f (SwiGLU intermediate)                          */
  int32_t renormalize;   /* 1: top-k weights renormalised to sum 1           */
  int64_t max_tokens;    /* n capacity per forward                           */
  int64_t expert_rows;   /* row capacity of each shard's expert input buffer */
  int32_t world_size;    /* processes taking part (1 = all shards local)     */
  int32_t world_rank;
} smoe_layer_config;

/* Buffer slots a host binds with smoe_layer_bind(). "peer" slots are bound
 * once per shard g in [0, G) (remote shards: IPC-mapped pointers); "local"
 * slots once per resident shard (index = g - shard_begin) or once (index 0). */
enum {
  /* peer, per shard */
  SMOE_BUF_PARTIAL = 0,   /* bf16 [max_tokens, d]: this rank's attention-TP partial */
  SMOE_BUF_XIN,           /* bf16 [expert_rows, d]: expert input rows (dispatch dst) */
  SMOE_BUF_XMETA,         /* int64 [expert_rows]: (src shard << 40) | pair slot      */
  SMOE_BUF_YPAIR,         /* bf16 [max_tokens*k, d]: expert outputs per (token,slot) */
  SMOE_BUF_OUT,           /* bf16 [max_tokens, d]: layer output, original order;     */
                          /* shards of one process may share one buffer (the SAG   */
                          /* writes each row once per distinct buffer)             */
  SMOE_BUF_COUNTS,        /* int32 [G, N]: pair counts source shard x expert slot    */
  SMOE_BUF_SIGNAL,        /* uint32 [64]: cross-process barrier pad (per process)    */
  /* local, per resident shard */
  SMOE_BUF_HS,            /* bf16 [max_tokens, d]: SRS output (this shard's group)   */
  SMOE_BUF_TOPK_IDS,      /* int32 [max_tokens, k]: expert slot (s-EG order)         */
  SMOE_BUF_TOPK_W,        /* f32  [max_tokens, k]: combine weights                   */
  SMOE_BUF_PAIR_RANK,     /* int32 [max_tokens, k]: rank inside (shard, slot)        */
  SMOE_BUF_HMID,          /* bf16 [expert_rows, f]: SwiGLU activations               */
  /* local, once */
  SMOE_BUF_FORWARD,       /* int64 [G*max_tokens]                                    */
  SMOE_BUF_INVERSE,       /* int64 [max_tokens]                                      */
  SMOE_BUF_DEV,           /* int64 [max_tokens]                                      */
  SMOE_BUF_PLAN_COUNTS,   /* int32 [G]                                               */
  SMOE_BUF_GROUP,         /* int64 [1]                                               */
  SMOE_BUF_STATS,         /* int64 [16]: see SMOE_STAT_*                             */
  SMOE_BUF_ERR,           /* int32 [1]                                               */
  SMOE_BUF_WORKSPACE,     /* bytes: smoe_layer_workspace_bytes()                     */
  SMOE_BUF_PROBLEMS,      /* bytes: grouped-GEMM problem table, 64 KiB               */
  SMOE_BUF_EPOCH,         /* uint32 [1]: barrier epoch (device)                      */
  SMOE_BUF_HIST_OUT,      /* peer, one per process (optional): int64 [max_tokens, h]  */
                          /* next layer's n-gram window = this window shifted by one  */
                          /* plus the cluster of each token's top-1 expert            */
                          /* (predictor.py:165-166)                                   */
  SMOE_BUF_XFAN,          /* peer, per shard (processes > 1): int32 [expert_rows]     */
                          /* fan-out table of the deduplicated dispatch (-1 = row    */
                          /* stored; else the row to copy it from)                   */
  SMOE_BUF_AR,            /* bf16 [max_tokens, d], per process (bind for every shard; */
                          /* co-resident shards share): DS-MoE all-reduce output     */
  SMOE_BUF_AG,            /* bf16 [ag_rows, d], per process: DS-MoE all-gather of the */
                          /* combined token groups (row g * group + j)               */
  SMOE_BUF__COUNT
};

/* stats written by the layer (int64 each). */
enum {
  SMOE_STAT_LOCAL_PAIRS = 0,   /* (token, expert) pairs whose expert is on the token's shard */
  SMOE_STAT_REMOTE_PAIRS,      /* pairs crossing shards (the A2A events, comm.py:214-216)   */
  SMOE_STAT_SRS_ROWS,          /* rows reduced by SRS (real rows, no pads)                 */
  SMOE_STAT_GROUP,             /* max group (scheduler.py:135)                              */
  SMOE_STAT_REMOTE_ROWS,       /* distinct (token, other shard) pairs: rows a dispatch that */
                               /* deduplicates per destination shard would send             */
  SMOE_STAT_SENT_ROWS,         /* rows the dispatch stored into shards of OTHER processes   */
                               /* (with SMOE_OPT_DEDUP_DISPATCH: one per (token, remote     */
                               /* shard), else one per remote-process pair)                 */
  SMOE_STAT__COUNT = 16
};

size_t smoe_layer_workspace_bytes(const smoe_layer_config* cfg);

int smoe_layer_create(const smoe_layer_config* cfg, smoe_layer** out);
void smoe_layer_destroy(smoe_layer* layer);
/* Bind a device buffer (see SMOE_BUF_*). */
int smoe_layer_bind(smoe_layer* layer, int32_t slot, int32_t index, void* ptr);

/* Pipeline structure.  SMOE_PIPELINE_SMOE (default): the speculative
 * pipeline SRS -> A2A -> A2A -> SAG.  SMOE_PIPELINE_DSMOE:
 * the DS-MoE baseline structure AR -> A2A -> A2A -> AG (comm.py:99-108) on
 * the same kernels -- the SRS stage becomes a two-shot all-reduce into
 * SMOE_BUF_AR plus each rank's slice of it, and COMBINE_SAG combines into
 * the SMOE_BUF_AG all-gather blocks (G * group <= ag_rows, else
 * SMOE_ERRBIT_CAPACITY) followed by a local resume gather into SMOE_BUF_OUT.
 * Paired with position-sharding tables (token i -> shard i % G, comm.py:202)
 * and contiguous expert blocks (comm.py:201).  Bind AR / AG first. */
#define SMOE_PIPELINE_SMOE  0
#define SMOE_PIPELINE_DSMOE 1
int smoe_layer_set_pipeline(smoe_layer* layer, int32_t pipeline, int64_t ag_rows);

/* Lookup tables (predictor.py:39-82) and the s-EG expert placement
 * (scheduler.py:200-224).  slot_owner[N]: cluster (= shard) that owns expert
 * slot e' in the cluster-contiguous order, i.e. labels[new_to_old[e']]. */
int smoe_layer_set_tables(smoe_layer* layer,
                          const int16_t* t_labels, const float* t_conf,
                          int64_t vocab, const int16_t* a_best,
                          const float* a_conf, int64_t a_rows,
                          int32_t hist_len, const int32_t* slot_owner_h);

/* Weights, all bf16, expert slots in s-EG order:
 *   w_gate  [N, d]          gate rows already permuted by new_to_old
 *   b_gate  f32 [N] or NULL
 *   w13     [L, 2f, d]      L = experts owned by the resident shards, packed
 *                           by smoe_pack_w13 (gate/up interleaved per 128 rows)
 *   w2      [L, d, f]       down projection                                  */
int smoe_layer_set_weights(smoe_layer* layer, const void* w_gate,
                           const float* b_gate, const void* w13,
                           const void* w2);

/* Same as smoe_layer_set_weights, with w13 and w2 in the TMA-box-tiled
 * layout of smoe_tile_weights (every 256 x 64 weight box the expert GEMMs
 * load is one contiguous 32 KiB run of HBM). */
int smoe_layer_set_weights_tiled(smoe_layer* layer, const void* w_gate,
                                 const float* b_gate, const void* w13_tiled,
                                 const void* w2_tiled);

/* Box-tile a row-major bf16 matrix [rows, cols] (rows % 256 == 0,
 * cols % 64 == 0): dst[((rb * cols/64 + kb) * 256 + r) * 64 + c] =
 * src[(rb * 256 + r) * cols + kb * 64 + c].  Experts stack along rows. */
int smoe_tile_weights(const void* src, int64_t rows, int64_t cols, void* dst,
                      void* stream);

/* Pack per-expert gate_proj [f, d] and up_proj [f, d] (both bf16, expert e at
 * w1[e], w3[e]) into the w13 layout the SwiGLU GEMM reads. */
int smoe_pack_w13(const void* w1, const void* w3, int32_t n_local_experts,
                  int32_t ffn, int32_t hidden, void* w13, void* stream);

/* Stages of the forward (run in this order by smoe_layer_forward):           */
enum {
  SMOE_STAGE_PLAN = 0,    /* K1 lookup + stable partition plan               */
  SMOE_STAGE_SRS,         /* K3 shuffled reduce-scatter (permute fused)      */
  SMOE_STAGE_GATE,        /* K4 gate GEMV + softmax + top-k + locality       */
  SMOE_STAGE_ROUTE,       /* K5a per-shard stable pair ranks + count publish */
  SMOE_STAGE_DISPATCH,    /* K5b A2A dispatch: remote rows only cross shards */
  SMOE_STAGE_EXPERT_UP,   /* K6a tcgen05 grouped GEMM + SwiGLU epilogue      */
  SMOE_STAGE_EXPERT_DOWN, /* K6b tcgen05 grouped GEMM + A2A-combine epilogue */
  SMOE_STAGE_COMBINE_SAG, /* K8 weighted combine + shuffled all-gather       */
  SMOE_STAGE__COUNT
};

/* Run one stage / the whole layer (lookup_devices scheduler.py:82-98 through
 * resume_tokens :152-157).  tokens int64[n] and hist are replicated on every
 * process, as in attention TP.
 *
 * hist: int64[n, hist_width] row-major (contiguous) window of the previous
 * layers' top-1 clusters, oldest digit first (predictor.py:149-166), or NULL
 * for the first layer.  hist_width must equal the table depth `hist_len` of
 * smoe_layer_set_tables (SMOE_ERR_INVALID_ARG otherwise).  Only the newest
 * hist_depth digits are valid: the lookup uses the n-gram table only when
 * hist_depth == hist_width (the reference passes histories=None for the
 * first n layers, scheduler.py:84-89), while a partial window still shifts
 * into the next one.  The next window (SMOE_BUF_HIST_OUT) is the input
 * shifted by one digit plus this layer's top-1 cluster; its valid depth is
 * min(hist_depth + 1, hist_width) (0-filled digits below that).          */
int smoe_layer_stage_hist(smoe_layer* layer, int32_t stage, const int64_t* tokens,
                          const int64_t* hist, int32_t hist_width, int32_t hist_depth,
                          int64_t n, void* stream);
int smoe_layer_forward_hist(smoe_layer* layer, const int64_t* tokens,
                            const int64_t* hist, int32_t hist_width, int32_t hist_depth,
                            int64_t n, void* stream);
/* Same with a full-depth window (hist_width = hist_depth = hist_len) or NULL. */
int smoe_layer_stage(smoe_layer* layer, int32_t stage, const int64_t* tokens,
                     const int64_t* hist, int64_t n, void* stream);
int smoe_layer_forward(smoe_layer* layer, const int64_t* tokens,
                       const int64_t* hist, int64_t n, void* stream);

/* Cross-process barrier over the bound SIGNAL pads (no-op if world_size 1). */
int smoe_layer_barrier(smoe_layer* layer, void* stream);

/* ---- single-rank building blocks (used by the DS-MoE baseline pipeline) -- */
/* Gate over `rows` contiguous bf16 rows h[rows, hidden]: top-k expert ids
 * (lowest index on ties; -inf logits remain candidates) and softmax weights; stats[0..1] += local / remote
 * pairs where local means expert_owner[e] == my_shard (stats nullable). */
int smoe_gate_topk(const void* h, int64_t rows, int32_t hidden, const void* w_gate,
                   const float* b_gate, int32_t n_experts, int32_t top_k,
                   int32_t renormalize, const int32_t* expert_owner, int32_t my_shard,
                   int32_t* topk_ids, float* topk_w, int64_t* stats, void* stream);
/* Expert-major send position of every (row, slot) pair:
 *   pair_pos[j*k+s] = sum_{e'<e} counts[e'] + #{earlier pairs with expert e},
 * counts[N] = pairs per expert (stable, deterministic). */
int smoe_pair_offsets(const int32_t* topk_ids, int64_t rows, int32_t top_k,
                      int32_t n_experts, int32_t* pair_pos, int32_t* counts, void* stream);
/* dst[pair_pos[j*k+s], :] = src[j, :] (all2allv send-buffer packing). */
int smoe_pack_rows(const void* src, int64_t rows, int32_t top_k, int32_t hidden,
                   const int32_t* pair_pos, void* dst, void* stream);
/* out[j, :] = bf16( sum_s topk_w[j*k+s] * y[pair_pos[j*k+s], :] ) (fp32 sum). */
int smoe_combine_rows(const void* y, const int32_t* pair_pos, const float* topk_w,
                      int64_t rows, int32_t top_k, int32_t hidden, void* out, void* stream);

/* ======================================================================= *
 *  Standalone SRS / SAG collectives (the paper's drop-in replacements for  *
 *  reduce-scatter and all-gather, Algorithm 2)               *
 * ======================================================================= */
/* Shuffled reduce-scatter (reduce-scatter priced at comm.py:83-84, fused with
 * the rebatch_tokens permutation scheduler.py:119-149) over n_shards partial
 * buffers (every partial
 * [n_tokens, hidden] bf16, all addressable from this GPU: local or peer):
 *   outs[g - shard_begin][j, :] = bf16( sum_{r < n_shards} partials[r][forward[g*group + j], :] )
 * for every shard g in [shard_begin, shard_begin + shard_count) and
 * j < counts[g]; fp32 sum in shard order.  forward / counts / group are the
 * plan of smoe_rebatch_plan or smoe_lookup_plan (device memory).  partials
 * and outs are HOST arrays of device pointers (n_shards <= 16). */
int smoe_srs(const void* const* partials, int32_t n_shards, int32_t shard_begin,
             int32_t shard_count, const int64_t* forward, const int32_t* counts,
             const int64_t* group, int64_t n_tokens, int32_t hidden, void* const* outs,
             void* stream);

/* Shuffled all-gather (resume_tokens, scheduler.py:152-157, fused with the
 * all-gather the reference prices at comm.py:83-84): for every shard g,
 * row j < counts[g] of blocks[g] ([group, hidden] bf16) is stored at the
 * token's original position forward[g*group + j] of every outs[o]
 * ([n_tokens, hidden], o < n_outs).  blocks / outs are HOST arrays of device
 * pointers (n_shards, n_outs <= 16). */
int smoe_sag(const void* const* blocks, int32_t n_shards, const int64_t* forward,
             const int32_t* counts, const int64_t* group, int64_t n_tokens, int32_t hidden,
             void* const* outs, int32_t n_outs, void* stream);

/* ======================================================================= *
 *  Grouped GEMM (K6) — exposed for tests and microbenchmarks                *
 * ======================================================================= */
/* For problem p: C[c_off_p + i, :] = epilogue(A[a_off_p + i, :K] . B_p^T)
 * for i < m_p, with B_p = B[b_index_p * N_b : (b_index_p+1) * N_b, :K].
 * problems: device int64[num_problems, 4] = {a_off, m, b_index, c_off}.
 * epilogue 0: bf16 store, C row stride ldc (N_b columns);
 * epilogue 1: SwiGLU, B packed by smoe_pack_w13: C has N_b/2 columns.     */
int smoe_grouped_gemm(const void* A, int64_t a_rows, int64_t K,
                      const void* B, int64_t b_rows, int64_t n_b,
                      const int64_t* problems, int32_t num_problems,
                      int32_t epilogue, void* C, int64_t c_rows, int64_t ldc,
                      void* stream);

/* ======================================================================= *
 *  CUDA IPC helpers (multi-process shard tables)                           *
 * ======================================================================= */
/* cudaMalloc'd buffers (IPC handles then cover exactly the buffer). */
int smoe_device_alloc(size_t bytes, void** dev_ptr_out_h);
int smoe_device_free(void* dev_ptr);
int smoe_ipc_handle(void* dev_ptr, void* handle_out_h /* 64 bytes */);
int smoe_ipc_open(const void* handle_h, void** dev_ptr_out_h);
int smoe_ipc_close(void* dev_ptr);

#ifdef __cplusplus
}
#endif
#endif /* SMOE_H_ */
