// shuffle.cu — index-driven data movement of the scheduler API.
//
//   smoe_gather_rows       rebatch_tokens data half / resume_tokens
//                          (scheduler.py:145-146, :157) for ids AND hidden rows
//                          (K2 of DESIGN.md: 128-bit vectorised row gather)
//   smoe_gate_permutation  scheduler.py:200-210
//   smoe_permute_columns   apply_expert_shuffle, scheduler.py:213-219
//   smoe_remap_index       remap_topk, scheduler.py:222-224
//   smoe_count_local       simulate_layer event count, comm.py:214
//   smoe_event_metrics     solver.metrics LAR + per-cluster loads, solver.py:766-800
#include "common.cuh"
#include <algorithm>
#include <cstdlib>

namespace smoe {

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached = v > 0 ? v : 148;
  }
  return cached;
}

static int g_pdl = -1;
// Layer stages whose kernels may launch early (SMOE_PDL_STAGES bit mask over
// SMOE_STAGE_*).  Not the up GEMM at large batches: its persistent CTAs take
// tiles by blockIdx and the launch order's CTA placement is worth 5-10% there;
// an early launch lands the CTAs wherever the dispatch kernel leaves room
// (profiles/r1_pdl/).  At decode sizes (no two tiles share a weight tile) the
// layer launches it early anyway (SMOE_OPT_DECODE_UP_PDL, layer.cu).
static int g_pdl_stage_mask = ~(1 << SMOE_STAGE_EXPERT_UP);
static thread_local int g_pdl_stage = -1;
int pdl_enabled() {
  if (g_pdl < 0) {
    const char* e = getenv("SMOE_PDL");
    g_pdl = (e && e[0] == '0') ? 0 : 1;
    const char* m = getenv("SMOE_PDL_STAGES");
    if (m) g_pdl_stage_mask = (int)strtol(m, nullptr, 0);
  }
  return g_pdl && (g_pdl_stage < 0 || ((g_pdl_stage_mask >> g_pdl_stage) & 1));
}
void set_pdl_stage(int stage) { g_pdl_stage = stage; }
int pdl_stage_enabled(int stage) {
  const int saved = g_pdl_stage;
  g_pdl_stage = stage;
  const int on = pdl_enabled();
  g_pdl_stage = saved;
  return on;
}
int pdl_stage_mask() { pdl_enabled(); return g_pdl_stage_mask & 0xff; }
void set_pdl_stage_mask(int mask) { pdl_enabled(); g_pdl_stage_mask = mask & 0xff; }
void set_pdl_enabled(int on) { g_pdl = on ? 1 : 0; }

static int grid_for(int64_t work, int threads, int waves = 8) {
  int64_t b = ceil_div(work, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * waves));
}

__host__ __device__ inline uint64_t pad_pattern(int64_t v, int eb) {
  uint64_t u = (uint64_t)v;
  if (eb == 1) { u &= 0xff; u |= u << 8; u |= u << 16; u |= u << 32; }
  else if (eb == 2) { u &= 0xffff; u |= u << 16; u |= u << 32; }
  else if (eb == 4) { u &= 0xffffffffull; u |= u << 32; }
  return u;
}

__device__ __forceinline__ bool resolve_index(int64_t& j, int64_t n_src, int pad_negative,
                                              int32_t* err, bool& pad) {
  pad = false;
  if (j < 0) {
    if (pad_negative) { pad = true; return true; }
    j += n_src;
  }
  if (j < 0 || j >= n_src) { set_err(err, SMOE_ERRBIT_INDEX_RANGE); return false; }
  return true;
}

// One warp per output row, 16 B per lane per step (row_bytes % 16 == 0).
__global__ void __launch_bounds__(256)
gather_rows_vec_kernel(const char* __restrict__ src, int64_t n_src, int64_t row_vecs,
                       const int64_t* __restrict__ idx, int64_t n_out, int pad_negative,
                       uint64_t pad, char* __restrict__ dst, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_out;
       r += warps) {
    int64_t j = __ldg(idx + r);
    bool is_pad;
    if (!resolve_index(j, n_src, pad_negative, err, is_pad)) continue;
    uint4* out = reinterpret_cast<uint4*>(dst + r * row_vecs * 16);
    if (is_pad) {
      const uint4 p = make_uint4((uint32_t)pad, (uint32_t)(pad >> 32), (uint32_t)pad,
                                 (uint32_t)(pad >> 32));
      for (int64_t v = lane; v < row_vecs; v += 32) st_v4(out + v, p);
      continue;
    }
    const uint4* in = reinterpret_cast<const uint4*>(src + j * row_vecs * 16);
    int64_t v = lane;
    for (; v + 96 < row_vecs; v += 128) {      // 4 loads in flight per lane
      uint4 a = ld_nc_v4(in + v), b = ld_nc_v4(in + v + 32), c = ld_nc_v4(in + v + 64),
            d = ld_nc_v4(in + v + 96);
      st_v4(out + v, a); st_v4(out + v + 32, b); st_v4(out + v + 64, c); st_v4(out + v + 96, d);
    }
    for (; v < row_vecs; v += 32) st_v4(out + v, ld_nc_v4(in + v));
  }
}

template <typename T>
__global__ void gather_elems_kernel(const T* __restrict__ src, int64_t n_src, int64_t row_elems,
                                    const int64_t* __restrict__ idx, int64_t n_out,
                                    int pad_negative, T pad, T* __restrict__ dst, int32_t* err) {
  const int64_t total = n_out * row_elems;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / row_elems, c = e - r * row_elems;
    int64_t j = __ldg(idx + r);
    bool is_pad;
    if (!resolve_index(j, n_src, pad_negative, c == 0 ? err : nullptr, is_pad)) continue;
    dst[e] = is_pad ? pad : src[j * row_elems + c];
  }
}

// Stable argsort of expert cluster labels by rank counting (N is small).
__global__ void gate_permutation_kernel(const int64_t* __restrict__ labels, int32_t N,
                                        int32_t n_clusters, int64_t* __restrict__ new_to_old,
                                        int64_t* __restrict__ old_to_new, int32_t* err) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const int64_t li = labels[i];
    if (li < 0 || li >= n_clusters) set_err(err, SMOE_ERRBIT_EXPERT_LABEL);
    int64_t pos = 0;
    for (int j = 0; j < N; ++j) {
      const int64_t lj = labels[j];
      pos += (lj < li) || (lj == li && j < i);
    }
    new_to_old[pos] = i;
    old_to_new[i] = pos;
  }
}

template <typename T>
__global__ void permute_columns_kernel(const T* __restrict__ src, int64_t rows, int32_t width,
                                       const int64_t* __restrict__ perm, T* __restrict__ dst) {
  const int64_t total = rows * width;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / width;
    const int32_t c = (int32_t)(e - r * width);
    dst[e] = src[r * width + __ldg(perm + c)];
  }
}

__global__ void remap_index_kernel(const int64_t* __restrict__ idx, int64_t count,
                                   const int64_t* __restrict__ table, int64_t table_len,
                                   int64_t* __restrict__ dst, int32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = idx[i];
    if (j < 0) j += table_len;
    if (j < 0 || j >= table_len) { set_err(err, SMOE_ERRBIT_INDEX_RANGE); continue; }
    dst[i] = table[j];
  }
}

__global__ void __launch_bounds__(256)
count_local_kernel(const int64_t* __restrict__ experts, int64_t occ, int32_t k,
                   const int64_t* __restrict__ expert_dev, int32_t N,
                   const int64_t* __restrict__ token_dev, unsigned long long* local_out,
                   int32_t* err) {
  unsigned long long mine = 0;
  const int64_t total = occ * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = __ldg(experts + e);
    if (x < 0) x += N;
    if (x < 0 || x >= N) { set_err(err, SMOE_ERRBIT_INDEX_RANGE); continue; }
    mine += (__ldg(expert_dev + x) == __ldg(token_dev + e / k));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(local_out, mine);
}

// solver.metrics (solver.py:766-800): local events and the expert-side load
// of every cluster.  Event (i, j) has expert experts[i*k + j] (or j when
// experts is NULL: a dense token x expert count matrix) and weight
// weights[i*k + j] (or 1).  Per-CTA shared histogram, one atomic per cluster
// per CTA; all sums are exact integers (order-independent).
__global__ void __launch_bounds__(256)
event_metrics_kernel(const int64_t* __restrict__ experts, const int64_t* __restrict__ weights,
                     int64_t occ, int32_t k, const int64_t* __restrict__ expert_dev, int32_t N,
                     const int64_t* __restrict__ token_dev, int32_t n_clusters,
                     unsigned long long* local_out, unsigned long long* loads, int32_t* err) {
  extern __shared__ unsigned long long s_loads[];
  for (int c = threadIdx.x; c < n_clusters; c += blockDim.x) s_loads[c] = 0;
  __syncthreads();
  unsigned long long mine = 0;
  const int64_t total = occ * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = experts ? __ldg(experts + e) : e % k;
    if (x < 0) x += N;                                   // numpy wrap, as C[routed]
    if (x < 0 || x >= N) { set_err(err, SMOE_ERRBIT_INDEX_RANGE); continue; }
    const unsigned long long w = weights ? (unsigned long long)__ldg(weights + e) : 1ull;
    if (w == 0) continue;
    const int64_t c = __ldg(expert_dev + x);
    if (c < 0 || c >= n_clusters) { set_err(err, SMOE_ERRBIT_EXPERT_LABEL); continue; }
    if (c == __ldg(token_dev + e / k)) mine += w;
    atomicAdd(&s_loads[c], w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(local_out, mine);
  __syncthreads();
  for (int c = threadIdx.x; c < n_clusters; c += blockDim.x)
    if (s_loads[c]) atomicAdd(&loads[c], s_loads[c]);
}

// schedule_requests_dp (scheduler.py:160-183): the open-device mask resets
// every n_devices requests, so windows are independent -> one thread per
// window runs the reference's greedy argmax (first maximum wins; numpy's
// argmax also returns the first NaN) over the still-open devices.
__global__ void schedule_dp_kernel(const double* __restrict__ aff, int64_t K, int32_t G,
                                   int64_t* __restrict__ labels) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = w * G;
  if (r0 >= K) return;
  uint64_t open_bits[SMOE_MAX_PLAN_DEVICES / 64];
  const int words = (G + 63) / 64;
  for (int i = 0; i < words; ++i) open_bits[i] = ~0ull;
  const int64_t r1 = (K < r0 + G) ? K : r0 + G;
  for (int64_t r = r0; r < r1; ++r) {
    const double* a = aff + r * G;
    int best = -1;
    double bv = 0.0;
    bool nan_hit = false;
    for (int dv = 0; dv < G; ++dv) {
      const bool open = (open_bits[dv >> 6] >> (dv & 63)) & 1ull;
      const double v = open ? a[dv] : -INFINITY;
      if (v != v) { best = dv; nan_hit = true; break; }         // NaN: numpy argmax stops here
      if (best < 0 || v > bv) { best = dv; bv = v; }
    }
    (void)nan_hit;
    labels[r] = best;
    open_bits[best >> 6] &= ~(1ull << (best & 63));
  }
}

}  // namespace smoe

using namespace smoe;

extern "C" int smoe_schedule_requests_dp(const double* affinities, int64_t n_requests,
                                         int32_t n_devices, int64_t* labels, void* stream) {
  if (n_requests < 0 || n_devices < 1) return SMOE_ERR_INVALID_ARG;
  if (n_devices > SMOE_MAX_PLAN_DEVICES) return SMOE_ERR_UNSUPPORTED;
  if (n_requests == 0) return SMOE_OK;
  if (!affinities || !labels) return SMOE_ERR_INVALID_ARG;
  const int64_t windows = ceil_div(n_requests, n_devices);
  schedule_dp_kernel<<<(int)ceil_div(windows, 128), 128, 0, as_stream(stream)>>>(
      affinities, n_requests, n_devices, labels);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_gather_rows(const void* src, int64_t n_src, int32_t elem_bytes,
                                int64_t row_elems, const int64_t* idx, int64_t n_out,
                                int32_t pad_negative, int64_t pad_value, void* dst,
                                int32_t* err, void* stream) {
  if (n_out < 0 || row_elems < 0 || n_src < 0) return SMOE_ERR_INVALID_ARG;
  if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8)
    return SMOE_ERR_UNSUPPORTED;
  if (n_out == 0 || row_elems == 0) return SMOE_OK;
  if (!idx || !dst || (n_src > 0 && !src)) return SMOE_ERR_INVALID_ARG;
  cudaStream_t st = as_stream(stream);
  const int64_t row_bytes = row_elems * elem_bytes;
  const bool vec = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  if (vec) {
    const int blocks = grid_for(n_out * 32, 256);
    gather_rows_vec_kernel<<<blocks, 256, 0, st>>>(
        static_cast<const char*>(src), n_src, row_bytes / 16, idx, n_out, pad_negative,
        pad_pattern(pad_value, elem_bytes), static_cast<char*>(dst), err);
  } else {
    const int blocks = grid_for(n_out * row_elems, 256);
#define SMOE_GATHER(T)                                                                   \
  gather_elems_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(src), n_src,      \
                                                 row_elems, idx, n_out, pad_negative,    \
                                                 (T)pad_value, static_cast<T*>(dst), err)
    if (elem_bytes == 1) SMOE_GATHER(uint8_t);
    else if (elem_bytes == 2) SMOE_GATHER(uint16_t);
    else if (elem_bytes == 4) SMOE_GATHER(uint32_t);
    else SMOE_GATHER(uint64_t);
#undef SMOE_GATHER
  }
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_gate_permutation(const int64_t* labels, int32_t n_experts,
                                     int32_t n_clusters, int64_t* new_to_old,
                                     int64_t* old_to_new, int32_t* err, void* stream) {
  if (n_experts < 0) return SMOE_ERR_INVALID_ARG;
  if (n_experts == 0) return SMOE_OK;
  if (!labels || !new_to_old || !old_to_new) return SMOE_ERR_INVALID_ARG;
  gate_permutation_kernel<<<(int)ceil_div(n_experts, 128), 128, 0, as_stream(stream)>>>(
      labels, n_experts, n_clusters, new_to_old, old_to_new, err);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_permute_columns(const void* src, int64_t rows, int32_t width,
                                    int32_t elem_bytes, const int64_t* perm, void* dst,
                                    void* stream) {
  if (rows < 0 || width < 0) return SMOE_ERR_INVALID_ARG;
  if (rows == 0 || width == 0) return SMOE_OK;
  if (!src || !dst || !perm) return SMOE_ERR_INVALID_ARG;
  cudaStream_t st = as_stream(stream);
  const int blocks = grid_for(rows * width, 256);
#define SMOE_PERM(T)                                                               \
  permute_columns_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(src), rows, \
                                                    width, perm, static_cast<T*>(dst))
  if (elem_bytes == 1) SMOE_PERM(uint8_t);
  else if (elem_bytes == 2) SMOE_PERM(uint16_t);
  else if (elem_bytes == 4) SMOE_PERM(uint32_t);
  else if (elem_bytes == 8) SMOE_PERM(uint64_t);
  else return SMOE_ERR_UNSUPPORTED;
#undef SMOE_PERM
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_remap_index(const int64_t* idx, int64_t count, const int64_t* table,
                                int64_t table_len, int64_t* dst, int32_t* err, void* stream) {
  if (count < 0) return SMOE_ERR_INVALID_ARG;
  if (count == 0) return SMOE_OK;
  if (!idx || !dst || !table) return SMOE_ERR_INVALID_ARG;
  remap_index_kernel<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(idx, count, table,
                                                                        table_len, dst, err);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_event_metrics(const int64_t* experts, const int64_t* weights, int64_t occ,
                                  int32_t k, const int64_t* expert_dev, int32_t n_experts,
                                  const int64_t* token_dev, int32_t n_clusters,
                                  int64_t* local_out, int64_t* loads_out, int32_t* err,
                                  void* stream) {
  if (occ < 0 || k < 0 || n_clusters < 1 || n_clusters > SMOE_MAX_PLAN_DEVICES || !local_out ||
      !loads_out)
    return SMOE_ERR_INVALID_ARG;
  cudaStream_t st = as_stream(stream);
  SMOE_CUDA_TRY(cudaMemsetAsync(local_out, 0, sizeof(int64_t), st));
  SMOE_CUDA_TRY(cudaMemsetAsync(loads_out, 0, sizeof(int64_t) * n_clusters, st));
  if (occ == 0 || k == 0) return SMOE_OK;
  if (!expert_dev || !token_dev || n_experts < 1) return SMOE_ERR_INVALID_ARG;
  event_metrics_kernel<<<grid_for(occ * k, 256, 2), 256, sizeof(int64_t) * n_clusters, st>>>(
      experts, weights, occ, k, expert_dev, n_experts, token_dev, n_clusters,
      reinterpret_cast<unsigned long long*>(local_out),
      reinterpret_cast<unsigned long long*>(loads_out), err);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_count_local(const int64_t* experts, int64_t occ, int32_t k,
                                const int64_t* expert_dev, int32_t n_experts,
                                const int64_t* token_dev, int64_t* local_out, int32_t* err,
                                void* stream) {
  if (occ < 0 || k < 0 || !local_out) return SMOE_ERR_INVALID_ARG;
  cudaStream_t st = as_stream(stream);
  SMOE_CUDA_TRY(cudaMemsetAsync(local_out, 0, sizeof(int64_t), st));
  if (occ == 0 || k == 0) return SMOE_OK;
  if (!experts || !expert_dev || !token_dev) return SMOE_ERR_INVALID_ARG;
  count_local_kernel<<<grid_for(occ * k, 256), 256, 0, st>>>(
      experts, occ, k, expert_dev, n_experts, token_dev,
      reinterpret_cast<unsigned long long*>(local_out), err);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}
