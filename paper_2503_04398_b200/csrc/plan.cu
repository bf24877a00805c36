// plan.cu — K1: token->device lookup fused with the stable device partition.
//
// Replaces scheduler.py:82-98 (lookup_devices) and the index half of
// scheduler.py:119-149 (rebatch_tokens).  The reference does an O(n log n)
// stable argsort plus a Python loop over devices; with G <= 1024 labels a
// stable partition is a counting sort:
//
//   pass 1 (plan_count):   per 512-token tile, look the device up and count
//                          tokens per device (warp match_any aggregation).
//   pass 2 (plan_scatter): prefix the tile counts per device, take the global
//                          max group (scheduler.py:135), and give every token
//                          slot = dev*group + rank, where rank is its stable
//                          position among earlier tokens of the same device
//                          (warp match_any + per-warp counts + running sums).
//
// HBM traffic is the algorithmic minimum: tokens (+ history) read once in
// pass 1, the int32 label scratch read once in pass 2, inverse written once
// and forward written once (pads included).
#include "common.cuh"

namespace smoe {

constexpr int kPlanThreads = 256;
constexpr int kPlanChunks = 2;
constexpr int kPlanTile = kPlanThreads * kPlanChunks;   // 512 tokens per CTA

struct LookupTables {
  const int16_t* t_labels;
  const float* t_conf;
  int64_t vocab;
  const int16_t* a_best;
  const float* a_conf;
  int64_t a_rows;
  int32_t n_clusters;
  const int64_t* hist;
  int32_t hist_len;
};

// scheduler.py:86-97 for one token.  Returns the looked-up label (int64, the
// int16 table value sign-extended as numpy's astype(int64) does).
__device__ __forceinline__ int64_t lookup_one(const LookupTables& t, int64_t i,
                                              int64_t tok, int32_t* err) {
  // Two rounds of loads instead of four: the history row does not depend on
  // the token, and the four table entries are read together (a row's entries
  // only when the row is in range); the checks and their order -- token range
  // first, then history range -- are the reference's.
  int64_t row = 0;
  if (t.hist != nullptr) {
    const int64_t* h = t.hist + i * (int64_t)t.hist_len;
    for (int j = 0; j < t.hist_len; ++j) row = row * t.n_clusters + __ldg(h + j);
    if (row < 0) row += t.a_rows;
  }
  if (tok < 0) tok += t.vocab;                       // numpy negative wrap
  if (tok < 0 || tok >= t.vocab) { set_err(err, SMOE_ERRBIT_TOKEN_RANGE); return 0; }
  const bool row_ok = t.hist != nullptr && row >= 0 && row < t.a_rows;
  const int64_t stat = (int64_t)__ldg(t.t_labels + tok);
  const float thr = t.hist != nullptr ? __ldg(t.t_conf + tok) : 0.f;
  const float conf = row_ok ? __ldg(t.a_conf + row) : 0.f;
  const int64_t best = row_ok ? (int64_t)__ldg(t.a_best + row) : 0;
  if (t.hist == nullptr) return stat;                // scheduler.py:88-89
  if (!row_ok) { set_err(err, SMOE_ERRBIT_HISTORY_RANGE); return stat; }
  return (conf > thr) ? best : stat;                 // strict >, :95
}

__global__ void __launch_bounds__(kPlanThreads)
lookup_kernel(LookupTables t, const int64_t* __restrict__ tokens, int64_t n,
              int64_t* __restrict__ dev_out, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dev_out[i] = lookup_one(t, i, __ldg(tokens + i), err);
}

// Pass 1.  Either `devices` (rebatch from given labels) or the lookup tables
// (`use_lookup`) provide the label.  Invalid labels are recorded as -1.
__global__ void __launch_bounds__(kPlanThreads)
plan_count_kernel(LookupTables t, int use_lookup, const int64_t* __restrict__ tokens,
                  const int64_t* __restrict__ devices, int64_t n, int32_t G,
                  int32_t* __restrict__ dev_ws, int64_t* __restrict__ dev_out,
                  int32_t* __restrict__ block_counts, int32_t* err) {
  pdl_enter();
  extern __shared__ int32_t s_cnt[];                 // [G]
  for (int d = threadIdx.x; d < G; d += blockDim.x) s_cnt[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kPlanTile;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < kPlanChunks; ++c) {
    const int64_t i = base + c * kPlanThreads + threadIdx.x;
    int32_t d = -1;
    if (i < n) {
      int64_t lab = use_lookup ? lookup_one(t, i, __ldg(tokens + i), err) : __ldg(devices + i);
      if (dev_out) dev_out[i] = lab;
      if (lab < 0 || lab >= G) set_err(err, SMOE_ERRBIT_DEVICE_RANGE);
      else d = (int32_t)lab;
      dev_ws[i] = d;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (d >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_cnt[d], __popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < G; d += blockDim.x)
    block_counts[(int64_t)blockIdx.x * G + d] = s_cnt[d];
}

// Pass 2.
__global__ void __launch_bounds__(kPlanThreads)
plan_scatter_kernel(const int32_t* __restrict__ dev_ws, int64_t n, int32_t G,
                    int32_t n_blocks, const int32_t* __restrict__ block_counts,
                    int64_t* __restrict__ forward, int64_t* __restrict__ inverse,
                    int32_t* __restrict__ counts_out, int64_t* __restrict__ group_out) {
  pdl_enter();
  extern __shared__ int32_t smem[];
  int32_t* s_base = smem;                 // [G] exclusive prefix over earlier tiles + running
  int32_t* s_total = smem + G;            // [G] global count per device
  int32_t* s_wcnt = smem + 2 * G;         // [8 warps][G]
  __shared__ int32_t s_group;
  if (threadIdx.x == 0) s_group = 0;
  for (int d = threadIdx.x; d < 8 * G; d += blockDim.x) s_wcnt[d] = 0;
  __syncthreads();
  int32_t local_max = 0;
  for (int d = threadIdx.x; d < G; d += blockDim.x) {
    int32_t pre = 0, tot = 0;
    for (int b = 0; b < n_blocks; ++b) {
      const int32_t c = block_counts[(int64_t)b * G + d];
      if (b < (int)blockIdx.x) pre += c;
      tot += c;
    }
    s_base[d] = pre;
    s_total[d] = tot;
    local_max = max(local_max, tot);
  }
  atomicMax(&s_group, local_max);
  __syncthreads();
  const int64_t group = s_group;
  if (blockIdx.x == 0) {
    for (int d = threadIdx.x; d < G; d += blockDim.x) counts_out[d] = s_total[d];
    if (threadIdx.x == 0) *group_out = group;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kPlanTile;
  for (int c = 0; c < kPlanChunks; ++c) {
    const int64_t i = base + c * kPlanThreads + threadIdx.x;
    const int32_t d = (i < n) ? dev_ws[i] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int32_t rank_w = __popc(peers & lanemask_lt());
    if (d >= 0 && lane == __ffs(peers) - 1) s_wcnt[warp * G + d] = __popc(peers);
    __syncthreads();
    if (d >= 0) {
      int32_t off = s_base[d] + rank_w;
      for (int w = 0; w < warp; ++w) off += s_wcnt[w * G + d];
      const int64_t slot = (int64_t)d * group + off;
      inverse[i] = slot;
      forward[slot] = i;
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < G; dd += blockDim.x) {
      int32_t s = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) { s += s_wcnt[w * G + dd]; s_wcnt[w * G + dd] = 0; }
      s_base[dd] += s;
    }
    __syncthreads();
  }
  // pads: every slot r >= count[d] of group d is -1 (scheduler.py:136).
  const int64_t total_slots = (int64_t)G * group;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < total_slots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = s / group, r = s - d * group;
    if (r >= s_total[d]) forward[s] = -1;
  }
}

// Both passes in one CTA when the batch is a single tile (n <= 512, decode):
// the labels stay in registers and the tile prefix is zero, so one launch
// replaces two (identical results: the same match_any ranks in the same order).
__global__ void __launch_bounds__(kPlanThreads)
plan_single_kernel(LookupTables t, int use_lookup, const int64_t* __restrict__ tokens,
                   const int64_t* __restrict__ devices, int64_t n, int32_t G,
                   int64_t* __restrict__ dev_out, int64_t* __restrict__ forward,
                   int64_t* __restrict__ inverse, int32_t* __restrict__ counts_out,
                   int64_t* __restrict__ group_out, int32_t* err, int64_t* zero_stats,
                   int32_t n_zero_stats, int32_t* zero_i32, int32_t n_zero_i32) {
  SMOE_TL_ENTER(0);
  pdl_enter();
  SMOE_TL_WAITED(0);
  // the layer's per-forward resets (error flag, event counters), folded in so
  // a decode-sized forward starts with one kernel instead of two memsets and
  // a kernel; the __syncthreads below orders them before any lookup error
  if (zero_stats) {
    if (threadIdx.x < n_zero_stats) zero_stats[threadIdx.x] = 0;
    if (threadIdx.x == 0 && err) *err = 0;
  }
  // + the early-started down GEMM's per-expert readiness counters (no memset
  // node in front of the up GEMM, which can then launch under PDL)
  for (int i = threadIdx.x; i < n_zero_i32; i += blockDim.x) zero_i32[i] = 0;
  extern __shared__ int32_t smem[];
  int32_t* s_cnt = smem;                  // [G] tokens per device
  int32_t* s_base = smem + G;             // [G] running offset per device
  int32_t* s_wcnt = smem + 2 * G;         // [8 warps][G]
  __shared__ int32_t s_group;
  if (threadIdx.x == 0) s_group = 0;
  for (int d = threadIdx.x; d < 10 * G; d += blockDim.x) smem[d] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t dv[kPlanChunks];
#pragma unroll
  for (int c = 0; c < kPlanChunks; ++c) {
    const int64_t i = c * kPlanThreads + threadIdx.x;
    int32_t d = -1;
    if (i < n) {
      int64_t lab = use_lookup ? lookup_one(t, i, __ldg(tokens + i), err) : __ldg(devices + i);
      if (dev_out) dev_out[i] = lab;
      if (lab < 0 || lab >= G) set_err(err, SMOE_ERRBIT_DEVICE_RANGE);
      else d = (int32_t)lab;
    }
    dv[c] = d;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (d >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_cnt[d], __popc(peers));
  }
  __syncthreads();
  int32_t local_max = 0;
  for (int d = threadIdx.x; d < G; d += blockDim.x) {
    local_max = max(local_max, s_cnt[d]);
    counts_out[d] = s_cnt[d];
  }
  atomicMax(&s_group, local_max);
  __syncthreads();
  const int64_t group = s_group;
  if (threadIdx.x == 0) *group_out = group;
#pragma unroll
  for (int c = 0; c < kPlanChunks; ++c) {
    if (c * kPlanThreads >= n) break;                // CTA-uniform: no rows in this chunk
    const int64_t i = c * kPlanThreads + threadIdx.x;
    const int32_t d = dv[c];
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int32_t rank_w = __popc(peers & lanemask_lt());
    if (d >= 0 && lane == __ffs(peers) - 1) s_wcnt[warp * G + d] = __popc(peers);
    __syncthreads();
    if (d >= 0) {
      int32_t off = s_base[d] + rank_w;
      for (int w = 0; w < warp; ++w) off += s_wcnt[w * G + d];
      const int64_t slot = (int64_t)d * group + off;
      inverse[i] = slot;
      forward[slot] = i;
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < G; dd += blockDim.x) {
      int32_t sum = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) { sum += s_wcnt[w * G + dd]; s_wcnt[w * G + dd] = 0; }
      s_base[dd] += sum;
    }
    __syncthreads();
  }
  const int64_t total_slots = (int64_t)G * group;
  for (int64_t sl = threadIdx.x; sl < total_slots; sl += blockDim.x) {
    const int64_t d = sl / group, r = sl - d * group;
    if (r >= s_cnt[d]) forward[sl] = -1;
  }
  SMOE_TL_EXIT(0);
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// zero_stats (layer only): when non-null, err and zero_stats[0, n_zero_stats)
// are reset before the lookup -- inside the kernel for single-tile batches,
// by memsets otherwise.
static int plan_impl(const LookupTables& t, int use_lookup, const int64_t* tokens,
                     const int64_t* devices, int64_t n, int32_t G, int64_t* dev_out,
                     int64_t* forward, int64_t* inverse, int32_t* counts, int64_t* group,
                     int32_t* err, void* ws, size_t ws_bytes, cudaStream_t st,
                     int64_t* zero_stats = nullptr, int32_t n_zero_stats = 0,
                     int32_t* zero_i32 = nullptr, int32_t n_zero_i32 = 0) {
#ifndef SMOE_PLAN_FOLD
#define SMOE_PLAN_FOLD 1      // 0: memsets before every plan (A/B builds)
#endif
  const bool single =
      SMOE_PLAN_FOLD && n > 0 && n <= kPlanTile && n_zero_stats <= kPlanThreads;
  if (zero_stats && !single) {
    SMOE_CUDA_TRY(cudaMemsetAsync(zero_stats, 0, sizeof(int64_t) * n_zero_stats, st));
    if (err) SMOE_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  }
  if (zero_i32 && n_zero_i32 > 0 && !single)
    SMOE_CUDA_TRY(cudaMemsetAsync(zero_i32, 0, sizeof(int32_t) * n_zero_i32, st));
  if (G < 1 || G > SMOE_MAX_PLAN_DEVICES) return SMOE_ERR_UNSUPPORTED;
  if (n < 0 || !counts || !group || (n > 0 && (!forward || !inverse))) return SMOE_ERR_INVALID_ARG;
  if (ws_bytes < smoe_plan_workspace_bytes(n, G) || (n > 0 && !ws)) return SMOE_ERR_INVALID_ARG;
  if (n == 0) {
    SMOE_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * G, st));
    SMOE_CUDA_TRY(cudaMemsetAsync(group, 0, sizeof(int64_t), st));
    return SMOE_OK;
  }
  if (n > INT32_MAX) return SMOE_ERR_UNSUPPORTED;
  const int32_t n_blocks = (int32_t)ceil_div(n, kPlanTile);
  const size_t smem2 = sizeof(int32_t) * (size_t)G * 10;
  if (n_blocks == 1) {
    if (smem2 > 48 * 1024)
      SMOE_CUDA_TRY(cudaFuncSetAttribute(plan_single_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    SMOE_CUDA_TRY(launch_pdl(plan_single_kernel, 1, kPlanThreads, smem2, st, t, use_lookup,
                             tokens, devices, n, G, dev_out, forward, inverse, counts, group,
                             err, single ? zero_stats : nullptr, n_zero_stats,
                             single ? zero_i32 : nullptr, single ? n_zero_i32 : 0));
    SMOE_LAUNCH_CHECK();
    return SMOE_OK;
  }
  char* w = static_cast<char*>(ws);
  int32_t* dev_ws = reinterpret_cast<int32_t*>(w);
  int32_t* block_counts = reinterpret_cast<int32_t*>(w + align256(sizeof(int32_t) * n));
  SMOE_CUDA_TRY(launch_pdl(plan_count_kernel, n_blocks, kPlanThreads, sizeof(int32_t) * G, st,
      t, use_lookup, tokens, devices, n, G, dev_ws, dev_out, block_counts, err));
  SMOE_LAUNCH_CHECK();
  if (smem2 > 48 * 1024)
    SMOE_CUDA_TRY(cudaFuncSetAttribute(plan_scatter_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  SMOE_CUDA_TRY(launch_pdl(plan_scatter_kernel, n_blocks, kPlanThreads, smem2, st,
      dev_ws, n, G, n_blocks, block_counts, forward, inverse, counts, group));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

}  // namespace smoe

using namespace smoe;

extern "C" size_t smoe_plan_workspace_bytes(int64_t n, int32_t n_devices) {
  const int64_t n_blocks = ceil_div(n > 0 ? n : 1, kPlanTile);
  return align256(sizeof(int32_t) * (size_t)(n > 0 ? n : 1)) +
         align256(sizeof(int32_t) * (size_t)n_blocks * (size_t)(n_devices > 0 ? n_devices : 1));
}

extern "C" int smoe_lookup_devices(const int64_t* tokens, int64_t n, const int64_t* hist,
                                   int32_t hist_len, const int16_t* t_labels,
                                   const float* t_conf, int64_t vocab, const int16_t* a_best,
                                   const float* a_conf, int64_t a_rows, int32_t n_clusters,
                                   int64_t* dev_out, int32_t* err, void* stream) {
  if (n < 0 || (n > 0 && (!tokens || !dev_out || !t_labels || !t_conf))) return SMOE_ERR_INVALID_ARG;
  if (hist && (!a_best || !a_conf || hist_len < 0)) return SMOE_ERR_INVALID_ARG;
  if (n == 0) return SMOE_OK;
  LookupTables t{t_labels, t_conf, vocab, a_best, a_conf, a_rows, n_clusters, hist, hist_len};
  const int blocks = (int)std::min<int64_t>(ceil_div(n, kPlanThreads), 148 * 16);
  lookup_kernel<<<blocks, kPlanThreads, 0, as_stream(stream)>>>(t, tokens, n, dev_out, err);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_rebatch_plan(const int64_t* devices, int64_t n, int32_t n_devices,
                                 int64_t* forward, int64_t* inverse, int32_t* counts,
                                 int64_t* group, int32_t* err, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (n > 0 && !devices) return SMOE_ERR_INVALID_ARG;
  LookupTables t{};
  return plan_impl(t, 0, nullptr, devices, n, n_devices, nullptr, forward, inverse, counts,
                   group, err, workspace, workspace_bytes, as_stream(stream));
}

extern "C" int smoe_lookup_plan(const int64_t* tokens, int64_t n, const int64_t* hist,
                                int32_t hist_len, const int16_t* t_labels, const float* t_conf,
                                int64_t vocab, const int16_t* a_best, const float* a_conf,
                                int64_t a_rows, int32_t n_clusters, int64_t* dev_out,
                                int64_t* forward, int64_t* inverse, int32_t* counts,
                                int64_t* group, int32_t* err, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (n > 0 && (!tokens || !t_labels || !t_conf)) return SMOE_ERR_INVALID_ARG;
  if (hist && (!a_best || !a_conf || hist_len < 0)) return SMOE_ERR_INVALID_ARG;
  LookupTables t{t_labels, t_conf, vocab, a_best, a_conf, a_rows, n_clusters, hist, hist_len};
  return plan_impl(t, 1, tokens, nullptr, n, n_clusters, dev_out, forward, inverse, counts,
                   group, err, workspace, workspace_bytes, as_stream(stream));
}

namespace smoe {
// The layer's PLAN stage: smoe_lookup_plan + the per-forward resets of the
// error flag and the event counters (see plan_impl).
int layer_plan(const int64_t* tokens, int64_t n, const int64_t* hist, int32_t hist_len,
               const int16_t* t_labels, const float* t_conf, int64_t vocab,
               const int16_t* a_best, const float* a_conf, int64_t a_rows, int32_t n_clusters,
               int64_t* dev_out, int64_t* forward, int64_t* inverse, int32_t* counts,
               int64_t* group, int32_t* err, void* workspace, size_t workspace_bytes,
               int64_t* stats, int32_t n_stats, cudaStream_t st, int32_t* zero_i32,
               int32_t n_zero_i32) {
  if (n > 0 && (!tokens || !t_labels || !t_conf)) return SMOE_ERR_INVALID_ARG;
  if (hist && (!a_best || !a_conf || hist_len < 0)) return SMOE_ERR_INVALID_ARG;
  LookupTables t{t_labels, t_conf, vocab, a_best, a_conf, a_rows, n_clusters, hist, hist_len};
  if (n == 0) {
    SMOE_CUDA_TRY(cudaMemsetAsync(stats, 0, sizeof(int64_t) * n_stats, st));
    SMOE_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    if (zero_i32 && n_zero_i32 > 0)
      SMOE_CUDA_TRY(cudaMemsetAsync(zero_i32, 0, sizeof(int32_t) * n_zero_i32, st));
  }
  return plan_impl(t, 1, tokens, nullptr, n, n_clusters, dev_out, forward, inverse, counts,
                   group, err, workspace, workspace_bytes, st, n > 0 ? stats : nullptr,
                   n_stats, n > 0 ? zero_i32 : nullptr, n_zero_i32);
}
}  // namespace smoe

SMOE_TL_EXPORT(plan)
