// layer_kernels.cu — the non-GEMM stages of the speculative MoE layer.
//
// Algorithm 2 of the paper over G shards ("virtual
// ranks").  Shard g owns token group g (slots [g*group, g*group+count_g) of
// the plan, scheduler.py:119-149) and the experts of cluster g in the s-EG
// order (scheduler.py:200-224).  Buffers that other shards read or write are
// addressed through per-shard pointer tables (ShardPtrs): local pointers when
// shards share a GPU, CUDA-IPC mappings over NVLink when they do not.  The
// kernels therefore do the collective's data movement themselves:
//
//   K3 srs_kernel          shuffled reduce-scatter: gather row forward[s] from
//                          every shard's partial, fp32 sum in shard order,
//                          bf16 out (the permutation rides on the reduction)
//   K4 gate_kernel         logits = h . Wg^T (+b), top-k (ties -> lowest slot),
//                          softmax weights, local/remote event counts
//   K5a route_kernel       stable rank of each (token, slot) pair inside its
//                          expert slot; publishes the shard's count row
//   K5b dispatch_kernel    A2A dispatch: pair rows land in the owner's expert
//                          input buffer (a peer store only when remote)
//   K8 combine_sag_kernel  weighted sum of the k expert outputs, then the
//                          shuffled all-gather: one store per shard straight
//                          to the token's original position (resume fused)
#include "layer_kernels.cuh"
#include "gate_select.cuh"
#include <algorithm>
#include <cstdlib>

namespace smoe {

static int grid_cap(int64_t blocks, int per_sm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)num_sms() * per_sm));
}

// Shared-memory view of the local shards' row counts.
struct RowMap {
  int32_t cnt[SMOE_MAX_SHARDS];
  int32_t total;
  int64_t group;
};

__device__ __forceinline__ void load_rowmap(RowMap& rm, const LocalRows& lr) {
  // warp 0: one lane per resident shard, so the count loads (written by the
  // plan stage) are in flight together -- a serial loop paid one L2 round
  // trip per shard, several microseconds of a decode-sized kernel
  if (threadIdx.x < 32) {
    const int i = threadIdx.x;
    if (lr.counts == nullptr) {
      if (i == 0) {
        rm.cnt[0] = (int32_t)lr.single_rows;
        rm.total = (int32_t)lr.single_rows;
        rm.group = 0;
      }
    } else {
      const int64_t grp = i == 0 ? *lr.group : 0;
      int32_t c = 0;
      if (i < lr.shard_count) {
        c = lr.counts[lr.shard_begin + i];
        rm.cnt[i] = c;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (i == 0) {
        rm.total = c;
        rm.group = grp;
      }
    }
  }
  __syncthreads();
}

// Copy a pointer table out of kernel-parameter space with constant indices
// (fully unrolled).  Indexing a parameter array with a runtime value makes
// every thread copy the whole struct to its local stack -- hundreds of bytes
// of local-memory traffic per thread, which showed up as 2x DRAM writes in
// the dispatch kernel.  Callers index the shared copy instead.
__device__ __forceinline__ void stage_ptrs(char** dst, const ShardPtrs& src) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < SMOE_MAX_SHARDS; ++i) dst[i] = src.p[i];
  }
}

// q in [0, total) -> (local shard index, row inside the group)
__device__ __forceinline__ void decode_row(const RowMap& rm, int32_t shard_count, int64_t q,
                                           int32_t& gl, int64_t& j) {
  gl = 0;
  while (gl + 1 < shard_count && q >= rm.cnt[gl]) { q -= rm.cnt[gl]; ++gl; }
  j = q;
}

// ------------------------------------------------------------------ K3 SRS
// One warp per work item, two 16-B vectors per lane per shard per step, so
// the 2*G loads of a step are all in flight before the sum (G is a template
// parameter).  An item is a whole output row when there are at least as many
// rows as resident warps (kWholeRows), else a 1 KiB column chunk of a row: decode-sized batches
// (64 rows x 8 chunks = 512 items) then keep every warp busy instead of 64
// warps walking their rows serially.
constexpr int64_t kChunkVecs = 64;           // 16-B vectors per chunk item (1 KiB)
constexpr int32_t kWholeRows = 2048;         // rows from which an item is a whole row
                                             // (~ the warps resident on 148 SMs)
static int32_t whole_rows_from() {           // SMOE_WHOLE_ROWS: tuning experiments only
  static int32_t v = [] {
    const char* e = getenv("SMOE_WHOLE_ROWS");
    return e ? (int32_t)atoi(e) : kWholeRows;
  }();
  return v;
}
static int grid_items(int64_t rows, int64_t d) {
  return grid_cap(ceil_div(rows >= whole_rows_from() ? rows : rows * ceil_div(d / 8, kChunkVecs), 8), 16);
}

// Sum of row `row_off` over the G partials for vectors [v0, v1), written to
// `out` (two 16-B vectors per lane per shard in flight per step).
template <int G>
__device__ __forceinline__ void srs_span(const char* const (&src_base)[G], int64_t row_off,
                                         char* out, int64_t v0, int64_t v1, int lane) {
  for (int64_t v = v0 + lane; v < v1; v += 64) {
    const bool two = v + 32 < v1;
    uint4 x[G], y[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      x[r] = ld_nc_v4(src_base[r] + row_off + v * 16);
      if (two) y[r] = ld_nc_v4(src_base[r] + row_off + (v + 32) * 16);
    }
    float a[8], b[8];
    set_bf16x8(a, x[0]);
#pragma unroll
    for (int r = 1; r < G; ++r) acc_bf16x8(a, x[r]);
    st_v4(out + v * 16, pack_bf16x8(a));
    if (two) {
      set_bf16x8(b, y[0]);
#pragma unroll
      for (int r = 1; r < G; ++r) acc_bf16x8(b, y[r]);
      st_v4(out + (v + 32) * 16, pack_bf16x8(b));
    }
  }
}

template <int G>
__global__ void __launch_bounds__(256)
srs_kernel(LocalRows lr, ShardPtrs partials, int64_t d, ShardPtrs hs, int32_t whole_rows) {
  SMOE_TL_ENTER(1);
  // wait, THEN trigger: the gate launched behind this kernel may then read
  // the plan's outputs before its own wait (the plan has completed)
  pdl_wait();
  pdl_trigger();
  SMOE_TL_WAITED(1);
  __shared__ RowMap rm;
  __shared__ char* s_hs[SMOE_MAX_SHARDS];
  stage_ptrs(s_hs, hs);
  load_rowmap(rm, lr);
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w0 = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const char* src_base[G];
#pragma unroll
  for (int r = 0; r < G; ++r) src_base[r] = partials.p[r];
  if (rm.total >= whole_rows) {
    for (int64_t q = w0; q < rm.total; q += nwarps) {            // warp = row
      int32_t gl; int64_t j;
      decode_row(rm, lr.shard_count, q, gl, j);
      const int64_t g = lr.shard_begin + gl;
      srs_span<G>(src_base, lr.forward[g * rm.group + j] * d * 2, s_hs[gl] + j * d * 2, 0,
                  vecs, lane);
    }
  } else {
    const int64_t chunks = (vecs + kChunkVecs - 1) / kChunkVecs;
    for (int64_t it = w0; it < (int64_t)rm.total * chunks; it += nwarps) {  // warp = 1 KiB chunk
      const int64_t q = it / chunks, c = it - q * chunks;
      int32_t gl; int64_t j;
      decode_row(rm, lr.shard_count, q, gl, j);
      const int64_t g = lr.shard_begin + gl;
      srs_span<G>(src_base, lr.forward[g * rm.group + j] * d * 2, s_hs[gl] + j * d * 2,
                  c * kChunkVecs, min(vecs, (c + 1) * kChunkVecs), lane);
    }
  }
  SMOE_TL_EXIT(1);
}

int launch_srs(const LocalRows& lr, const ShardPtrs& partials, int64_t d, const ShardPtrs& hs,
               int64_t n_rows_bound, cudaStream_t st, int32_t n_sources) {
  if (d % 8) return SMOE_ERR_UNSUPPORTED;
  if (n_rows_bound <= 0) return SMOE_OK;
  const int grid = grid_items(n_rows_bound, d);
  const int32_t wr = whole_rows_from();
  switch (n_sources > 0 ? n_sources : lr.n_shards) {
#define SMOE_SRS_CASE(G_) \
    case G_: SMOE_CUDA_TRY(launch_pdl(srs_kernel<G_>, grid, 256, 0, st, lr, partials, d, hs, wr)); break;
    SMOE_SRS_CASE(1) SMOE_SRS_CASE(2) SMOE_SRS_CASE(3) SMOE_SRS_CASE(4) SMOE_SRS_CASE(5)
    SMOE_SRS_CASE(6) SMOE_SRS_CASE(7) SMOE_SRS_CASE(8) SMOE_SRS_CASE(9) SMOE_SRS_CASE(10)
    SMOE_SRS_CASE(11) SMOE_SRS_CASE(12) SMOE_SRS_CASE(13) SMOE_SRS_CASE(14) SMOE_SRS_CASE(15)
    SMOE_SRS_CASE(16)
#undef SMOE_SRS_CASE
    default: return SMOE_ERR_UNSUPPORTED;
  }
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ DS-MoE all-reduce
// The DS-MoE baseline's all-reduce (comm.py:99-108, two-shot: reduce-scatter
// + all-gather, 2(G-1)/G of the batch per GPU like the reference's volume
// model): shard g sums rows [g*c, (g+1)*c) of the G partials (c = ceil(n/G),
// natural token order) and stores them into every process's all-reduce
// buffer.  The ranks then use their own rows of the full sum (launch_srs
// with one source), where the s-MoE SRS delivers only a shard's own group.
template <int G>
__global__ void __launch_bounds__(256)
allreduce_kernel(ShardPtrs partials, int64_t d, int64_t n, int32_t shard_begin,
                 int32_t shard_count, int32_t n_shards, ShardPtrs outs, int32_t n_outs,
                 int32_t whole_rows) {
  pdl_enter();
  __shared__ char* s_out[SMOE_MAX_SHARDS];
  stage_ptrs(s_out, outs);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t c = (n + n_shards - 1) / n_shards;
  const int64_t r0 = min(n, (int64_t)shard_begin * c);
  const int64_t rows = min(n, (int64_t)(shard_begin + shard_count) * c) - r0;
  const bool whole = rows >= whole_rows;
  const int64_t chunks = whole ? 1 : (vecs + kChunkVecs - 1) / kChunkVecs;
  const int64_t cv = whole ? vecs : kChunkVecs;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const char* src_base[G];
#pragma unroll
  for (int r = 0; r < G; ++r) src_base[r] = partials.p[r];
  for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
       it < rows * chunks; it += nwarps) {
    const int64_t q = whole ? it : it / chunks, ch = it - q * chunks;
    const int64_t row = r0 + q;
    char* first = s_out[0] + row * d * 2;
    srs_span<G>(src_base, row * d * 2, first, ch * cv, min(vecs, (ch + 1) * cv), lane);
    if (n_outs > 1) {
      __syncwarp();
      for (int64_t v = ch * cv + lane; v < min(vecs, (ch + 1) * cv); v += 32) {
        const uint4 x = ld_v4(first + v * 16);
        for (int o = 1; o < n_outs; ++o) st_v4(s_out[o] + (row * d + v * 8) * 2, x);
      }
    }
  }
}

int launch_allreduce(const ShardPtrs& partials, int64_t d, int64_t n, int32_t shard_begin,
                     int32_t shard_count, int32_t n_shards, const ShardPtrs& outs,
                     int32_t n_outs, cudaStream_t st) {
  if (d % 8) return SMOE_ERR_UNSUPPORTED;
  if (n <= 0) return SMOE_OK;
  const int64_t c = (n + n_shards - 1) / n_shards;
  const int grid = grid_items(c * shard_count, d);
  const int32_t wr = whole_rows_from();
  switch (n_shards) {
#define SMOE_AR_CASE(G_) \
    case G_: SMOE_CUDA_TRY(launch_pdl(allreduce_kernel<G_>, grid, 256, 0, st, partials, d, n, \
                                      shard_begin, shard_count, n_shards, outs, n_outs, wr)); break;
    SMOE_AR_CASE(1) SMOE_AR_CASE(2) SMOE_AR_CASE(3) SMOE_AR_CASE(4) SMOE_AR_CASE(5)
    SMOE_AR_CASE(6) SMOE_AR_CASE(7) SMOE_AR_CASE(8) SMOE_AR_CASE(9) SMOE_AR_CASE(10)
    SMOE_AR_CASE(11) SMOE_AR_CASE(12) SMOE_AR_CASE(13) SMOE_AR_CASE(14) SMOE_AR_CASE(15)
    SMOE_AR_CASE(16)
#undef SMOE_AR_CASE
    default: return SMOE_ERR_UNSUPPORTED;
  }
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ K4 gate
constexpr int kGateRows = 32;
constexpr int kGateKC = 128;                 // hidden elements per smem chunk
constexpr int kGateWords = kGateKC / 2;      // bf16x2 words per row chunk
constexpr int kGatePad = kGateWords + 1;     // conflict-free row stride (words)

__global__ void __launch_bounds__(256)
gate_kernel(LocalRows lr, ShardPtrs hs, int64_t d, const uint32_t* __restrict__ w_gate,
            const float* __restrict__ b_gate, int32_t N, int32_t k, int32_t renorm,
            const int32_t* __restrict__ slot_owner, ShardPtrs topk_ids, ShardPtrs topk_w,
            int64_t* stats) {
  pdl_enter();
  __shared__ RowMap rm;
  __shared__ char* s_hs[SMOE_MAX_SHARDS];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  __shared__ char* s_wts[SMOE_MAX_SHARDS];
  stage_ptrs(s_hs, hs);
  stage_ptrs(s_ids, topk_ids);
  stage_ptrs(s_wts, topk_w);
  __shared__ uint32_t s_h[kGateRows * kGatePad];
  __shared__ uint32_t s_w[kGateMaxN * kGatePad];
  __shared__ float s_logit[kGateRows * (kGateMaxN + 1)];
  __shared__ int32_t s_gl[kGateRows];
  __shared__ int64_t s_j[kGateRows];
  __shared__ unsigned long long s_local, s_remote, s_rrows;
  load_rowmap(rm, lr);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t words = d / 2;
  for (int64_t rb = blockIdx.x; rb * kGateRows < rm.total; rb += gridDim.x) {
    if (tid < kGateRows) {
      const int64_t q = rb * kGateRows + tid;
      int32_t gl = -1; int64_t j = 0;
      if (q < rm.total) decode_row(rm, lr.shard_count, q, gl, j);
      s_gl[tid] = gl;
      s_j[tid] = j;
    }
    if (tid == 0) { s_local = 0; s_remote = 0; s_rrows = 0; }
    float acc[kGateMaxN * kGateRows / 256];
#pragma unroll
    for (int i = 0; i < kGateMaxN * kGateRows / 256; ++i) acc[i] = 0.f;
    __syncthreads();
    for (int64_t kc = 0; kc < words; kc += kGateWords) {
      // stage H rows and W rows of this chunk (32-bit words, coalesced)
      for (int e = tid; e < kGateRows * kGateWords; e += 256) {
        const int r = e / kGateWords, w = e - r * kGateWords;
        uint32_t v = 0;
        if (s_gl[r] >= 0 && kc + w < words)
          v = reinterpret_cast<const uint32_t*>(s_hs[s_gl[r]] + s_j[r] * d * 2)[kc + w];
        s_h[r * kGatePad + w] = v;
      }
      for (int e = tid; e < N * kGateWords; e += 256) {
        const int r = e / kGateWords, w = e - r * kGateWords;
        s_w[r * kGatePad + w] = (kc + w < words) ? __ldg(w_gate + r * words + kc + w) : 0u;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kGateMaxN * kGateRows / 256; ++i) {
        const int o = tid + 256 * i;
        if (o < kGateRows * N) {
          const int r = o / N, e = o - r * N;
          const uint32_t* hr = s_h + r * kGatePad;
          const uint32_t* wr = s_w + e * kGatePad;
          float a = acc[i];
#pragma unroll 8
          for (int w = 0; w < kGateWords; ++w) {
            const uint32_t hv = hr[w], wv = wr[w];
            a = fmaf(bf16_lo(hv), bf16_lo(wv), a);
            a = fmaf(bf16_hi(hv), bf16_hi(wv), a);
          }
          acc[i] = a;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < kGateMaxN * kGateRows / 256; ++i) {
      const int o = tid + 256 * i;
      if (o < kGateRows * N) {
        const int r = o / N, e = o - r * N;
        s_logit[r * (kGateMaxN + 1) + e] = acc[i] + (b_gate ? __ldg(b_gate + e) : 0.f);
      }
    }
    __syncthreads();
    // top-k + softmax, one warp per row
    unsigned long long my_local = 0, my_remote = 0, my_rrows = 0;
    for (int r = warp; r < kGateRows; r += 8) {
      const int32_t gl = s_gl[r];
      if (gl < 0) continue;
      const float* lg = s_logit + r * (kGateMaxN + 1);
      const float v0 = lane < N ? lg[lane] : __int_as_float(0x7fffffff);
      const float v1 = lane + 32 < N ? lg[lane + 32] : __int_as_float(0x7fffffff);
      int sel_e[kGateMaxK];
      float sel_p[kGateMaxK];
      float psum;
      warp_topk(v0, v1, N, k, lane, sel_e, sel_p, psum);
      warp_store_topk(lane, k, renorm, sel_e, sel_p, psum,
                      reinterpret_cast<int32_t*>(s_ids[gl]) + s_j[r] * k,
                      reinterpret_cast<float*>(s_wts[gl]) + s_j[r] * k, lr.shard_begin + gl,
                      slot_owner, my_local, my_remote, my_rrows);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      my_local += __shfl_xor_sync(0xffffffffu, my_local, o);
      my_remote += __shfl_xor_sync(0xffffffffu, my_remote, o);
      my_rrows += __shfl_xor_sync(0xffffffffu, my_rrows, o);
    }
    if (lane == 0 && (my_local | my_remote)) {
      atomicAdd(&s_local, my_local);
      atomicAdd(&s_remote, my_remote);
      atomicAdd(&s_rrows, my_rrows);
    }
    __syncthreads();
    if (tid == 0 && stats) {
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_LOCAL_PAIRS), s_local);
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_REMOTE_PAIRS), s_remote);
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_REMOTE_ROWS), s_rrows);
    }
    __syncthreads();
  }
}

// Tensor-core gate: logits[64 rows, N] per CTA with mma.sync m16n8k16 (bf16 in,
// fp32 accumulate).  The gate is HBM-bound on the hidden rows (d*2 bytes per
// token); the CUDA-core version above is compute-bound for N = 64.  H rows and
// W rows stream through a 4-stage cp.async ring in 128-B rows with a 16-B XOR
// swizzle (conflict-free ldmatrix).
constexpr int kMmaKC = 64;                       // bf16 per row per stage (128 B)
// 64 rows per CTA (4 row groups of 16) x S k-splits: warp (r, s) multiplies
// row group r with k sub-chunk s of every stage, and the S partial logits are
// summed through shared memory.  The split keeps 8-16 warps per CTA busy on
// the short, latency-bound k loop (the gate reads only d*2 bytes per token).
constexpr int kMmaRowsCTA = 64;
__host__ __device__ constexpr int mma_splits(int nt) { return nt <= 2 ? 2 : 2; }
__host__ __device__ constexpr int mma_stages(int nt) { return nt <= 2 ? 6 : 4; }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
               :: "r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// byte offset of 16-B chunk `c` of row `r` in a 128-B-row tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

template <int NT>   // NT = N / 8 n-tiles
__global__ void __launch_bounds__(128 * mma_splits(NT))
gate_mma_kernel(LocalRows lr, ShardPtrs hs, int64_t d, const char* __restrict__ w_gate,
                const float* __restrict__ b_gate, int32_t k, int32_t renorm,
                const int32_t* __restrict__ slot_owner, ShardPtrs topk_ids, ShardPtrs topk_w,
                int64_t* stats) {
  pdl_enter();
  constexpr int N = NT * 8;
  constexpr int S = mma_splits(NT);
  constexpr int kMmaRows = kMmaRowsCTA;
  constexpr int kMmaThreads = 128 * S;
  constexpr int kSubBytes = (kMmaRows + N) * kMmaKC * 2;        // H rows + W rows, 128 B each
  constexpr int kMmaStageBytes = S * kSubBytes;
  constexpr int kMmaStages = mma_stages(NT);
  extern __shared__ __align__(128) uint8_t gsm[];
  __shared__ RowMap rm;
  __shared__ char* s_hs[SMOE_MAX_SHARDS];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  __shared__ char* s_wts[SMOE_MAX_SHARDS];
  stage_ptrs(s_hs, hs);
  stage_ptrs(s_ids, topk_ids);
  stage_ptrs(s_wts, topk_w);
  __shared__ const char* s_row[kMmaRows];
  __shared__ int32_t s_gl[kMmaRows];
  __shared__ int64_t s_j[kMmaRows];
  __shared__ unsigned long long s_local, s_remote, s_rrows;
  load_rowmap(rm, lr);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(gsm));
  const int kchunks = (int)(d / (kMmaKC * S));                  // stages of S sub-chunks
  const int rgroup = warp & 3, split = warp >> 2;
  for (int64_t rb = blockIdx.x; rb * kMmaRows < rm.total; rb += gridDim.x) {
    if (tid < kMmaRows) {
      const int64_t q = rb * kMmaRows + tid;
      int32_t gl = -1; int64_t j = 0;
      if (q < rm.total) decode_row(rm, lr.shard_count, q, gl, j);
      s_gl[tid] = gl;
      s_j[tid] = j;
      s_row[tid] = gl >= 0 ? s_hs[gl] + j * d * 2 : nullptr;
    }
    if (tid == 0) { s_local = 0; s_remote = 0; s_rrows = 0; }
    __syncthreads();
    auto load_stage = [&](int kc, int stage) {
      for (int e = tid; e < S * (kMmaRows + N) * 8; e += kMmaThreads) {
        const int sub = e / ((kMmaRows + N) * 8);
        const int rem = e - sub * (kMmaRows + N) * 8;
        const int r = rem >> 3, c = rem & 7;
        const uint32_t st = sbase + stage * kMmaStageBytes + sub * kSubBytes;
        const int64_t col = (int64_t)(kc * S + sub) * kMmaKC + c * 8;
        if (r < kMmaRows) {
          const char* src = s_row[r];
          cp_async16(st + swz(r, c), src ? src + col * 2 : w_gate, src != nullptr);
        } else {
          const int n = r - kMmaRows;
          cp_async16(st + swz(r, c), w_gate + ((int64_t)n * d + col) * 2, true);
        }
      }
    };
    float acc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
#pragma unroll
    for (int s = 0; s < kMmaStages - 1; ++s) {
      if (s < kchunks) load_stage(s, s);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int kc = 0; kc < kchunks; ++kc) {
      asm volatile("cp.async.wait_group %0;" :: "n"(kMmaStages - 2) : "memory");
      __syncthreads();
      {  // prefetch kc + stages - 1 into the slot freed last iteration
        const int nk = kc + kMmaStages - 1;
        if (nk < kchunks) load_stage(nk, nk % kMmaStages);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      const uint32_t st = sbase + (kc % kMmaStages) * kMmaStageBytes + split * kSubBytes;
#pragma unroll
      for (int ks = 0; ks < kMmaKC / 16; ++ks) {
        // A: rows rgroup*16 + (lane & 15), 16-B chunk 2*ks + (lane >> 4)
        uint32_t a0, a1, a2, a3;
        const int ar = rgroup * 16 + (lane & 15);
        ldsm_x4(st + swz(ar, 2 * ks + (lane >> 4)), a0, a1, a2, a3);
#pragma unroll
        for (int t = 0; t < NT; t += 2) {
          // B for n-tiles t, t+1: matrices (n t*8.., k lo), (k hi), (n (t+1)*8.., k lo), (k hi)
          uint32_t b0, b1, b2, b3;
          const int nr = kMmaRows + t * 8 + (lane & 7) + ((lane >> 4) << 3);
          const int nt_ok = (t + 1 < NT) || (lane < 16);
          ldsm_x4(st + swz(nt_ok ? nr : kMmaRows + t * 8 + (lane & 7), 2 * ks + ((lane >> 3) & 1)),
                  b0, b1, b2, b3);
          mma_bf16(acc[t], a0, a1, a2, a3, b0, b1);
          if (t + 1 < NT) mma_bf16(acc[t + 1], a0, a1, a2, a3, b2, b3);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // partial logits of every k split -> smem [S][64][N + 1] (reuses the ring),
    // then lgs[r][e] = bias + sum over splits in split order
    float* red = reinterpret_cast<float*>(gsm);
    {
      float* part = red + split * kMmaRows * (N + 1);
      const int r0 = rgroup * 16 + (lane >> 2);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int c0 = t * 8 + 2 * (lane & 3);
        part[r0 * (N + 1) + c0] = acc[t][0];
        part[r0 * (N + 1) + c0 + 1] = acc[t][1];
        part[(r0 + 8) * (N + 1) + c0] = acc[t][2];
        part[(r0 + 8) * (N + 1) + c0 + 1] = acc[t][3];
      }
    }
    __syncthreads();
    float* lgs = red;
    for (int i = tid; i < kMmaRows * N; i += kMmaThreads) {
      const int r = i / N, e = i - r * N;
      float v = red[r * (N + 1) + e];
#pragma unroll
      for (int sp = 1; sp < S; ++sp) v += red[sp * kMmaRows * (N + 1) + r * (N + 1) + e];
      v += b_gate ? __ldg(b_gate + e) : 0.f;
      lgs[r * (N + 1) + e] = v;      // split 0's slot: each element read then written by one thread
    }
    __syncthreads();
    unsigned long long my_local = 0, my_remote = 0, my_rrows = 0;
    for (int r = warp; r < kMmaRows; r += kMmaThreads / 32) {
      const int32_t gl = s_gl[r];
      if (gl < 0) continue;
      const float* lg = lgs + r * (N + 1);
      const float v0 = lane < N ? lg[lane] : __int_as_float(0x7fffffff);
      const float v1 = lane + 32 < N ? lg[lane + 32] : __int_as_float(0x7fffffff);
      int sel_e[kGateMaxK];
      float sel_p[kGateMaxK];
      float psum;
      warp_topk(v0, v1, N, k, lane, sel_e, sel_p, psum);
      warp_store_topk(lane, k, renorm, sel_e, sel_p, psum,
                      reinterpret_cast<int32_t*>(s_ids[gl]) + s_j[r] * k,
                      reinterpret_cast<float*>(s_wts[gl]) + s_j[r] * k, lr.shard_begin + gl,
                      slot_owner, my_local, my_remote, my_rrows);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      my_local += __shfl_xor_sync(0xffffffffu, my_local, o);
      my_remote += __shfl_xor_sync(0xffffffffu, my_remote, o);
      my_rrows += __shfl_xor_sync(0xffffffffu, my_rrows, o);
    }
    if (lane == 0 && (my_local | my_remote)) {
      atomicAdd(&s_local, my_local);
      atomicAdd(&s_remote, my_remote);
      atomicAdd(&s_rrows, my_rrows);
    }
    __syncthreads();
    if (tid == 0 && stats) {
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_LOCAL_PAIRS), s_local);
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_REMOTE_PAIRS), s_remote);
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_REMOTE_ROWS), s_rrows);
    }
    __syncthreads();
  }
}

template <int NT>
static int launch_gate_mma(const LocalRows& lr, const ShardPtrs& hs, int64_t d, const void* w,
                           const float* b, int32_t k, int32_t renorm, const int32_t* owner,
                           const ShardPtrs& ids, const ShardPtrs& wts, int64_t* stats,
                           int64_t n_rows_bound, cudaStream_t st) {
  constexpr int rows = kMmaRowsCTA, S = mma_splits(NT);
  const size_t smem = (size_t)mma_stages(NT) * S * ((rows + NT * 8) * kMmaKC * 2);
  if (d % (kMmaKC * S)) return SMOE_ERR_UNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    SMOE_CUDA_TRY(cudaFuncSetAttribute(gate_mma_kernel<NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  SMOE_CUDA_TRY(launch_pdl(gate_mma_kernel<NT>, grid_cap(ceil_div(n_rows_bound, rows), 4), 128 * S, smem, st,
      lr, hs, d, static_cast<const char*>(w), b, k, renorm, owner, ids, wts, stats));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

int launch_gate(const LocalRows& lr, const ShardPtrs& hs, int64_t d, const void* w_gate,
                const float* b_gate, int32_t N, int32_t k, int32_t renorm,
                const int32_t* slot_owner, const ShardPtrs& topk_ids, const ShardPtrs& topk_w,
                int64_t* stats, int64_t n_rows_bound, cudaStream_t st) {
  if (N < 1 || N > kGateMaxN || k < 1 || k > kGateMaxK || k > N || d % 2) return SMOE_ERR_UNSUPPORTED;
  if (n_rows_bound <= 0) return SMOE_OK;
  if (d % (kMmaKC * 4) == 0) {
    switch (N) {   // tensor-core path for N in {8, 16, ..., 64}
      case 8: return launch_gate_mma<1>(lr, hs, d, w_gate, b_gate, k, renorm, slot_owner, topk_ids, topk_w, stats, n_rows_bound, st);
      case 16: return launch_gate_mma<2>(lr, hs, d, w_gate, b_gate, k, renorm, slot_owner, topk_ids, topk_w, stats, n_rows_bound, st);
      case 32: return launch_gate_mma<4>(lr, hs, d, w_gate, b_gate, k, renorm, slot_owner, topk_ids, topk_w, stats, n_rows_bound, st);
      case 64: return launch_gate_mma<8>(lr, hs, d, w_gate, b_gate, k, renorm, slot_owner, topk_ids, topk_w, stats, n_rows_bound, st);
      default: break;
    }
  }
  SMOE_CUDA_TRY(launch_pdl(gate_kernel, grid_cap(ceil_div(n_rows_bound, kGateRows), 4), 256, 0, st,
      lr, hs, d, static_cast<const uint32_t*>(w_gate), b_gate, N, k, renorm, slot_owner,
      topk_ids, topk_w, stats));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ K5a route
// Stable rank of every (token, slot) pair inside its expert slot, in two wide
// passes over 1024-pair chunks (one CTA per chunk and shard):
//   route_count: per-chunk pair counts per expert slot
//   route_rank:  rank = sum of the counts of earlier chunks + rank inside the
//                chunk (warp match_any + per-warp counts); chunk 0 publishes
//                the shard's count row to every process's [G, N] matrix.
constexpr int kRouteThreads = 1024;

__global__ void __launch_bounds__(kRouteThreads)
route_count_kernel(LocalRows lr, int32_t N, int32_t k, ShardPtrs topk_ids,
                   int32_t* __restrict__ chunk_counts, int32_t max_chunks) {
  pdl_enter();
  __shared__ int32_t s_cnt[kMaxExperts];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  stage_ptrs(s_ids, topk_ids);
  const int gl = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int64_t P = (int64_t)lr.counts[lr.shard_begin + gl] * k;
  const int32_t nchunks = (int32_t)((P + kRouteThreads - 1) / kRouteThreads);
  __syncthreads();
  for (int b = blockIdx.x; b < nchunks; b += gridDim.x) {
    for (int e = tid; e < N; e += kRouteThreads) s_cnt[e] = 0;
    __syncthreads();
    const int64_t p = (int64_t)b * kRouteThreads + tid;
    const int32_t e = p < P ? reinterpret_cast<const int32_t*>(s_ids[gl])[p] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_cnt[e], __popc(peers));
    __syncthreads();
    int32_t* out = chunk_counts + ((int64_t)gl * max_chunks + b) * N;
    for (int ee = tid; ee < N; ee += kRouteThreads) out[ee] = s_cnt[ee];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kRouteThreads)
route_rank_kernel(LocalRows lr, int32_t N, int32_t k, ShardPtrs topk_ids, ShardPtrs pair_rank,
                  const int32_t* __restrict__ chunk_counts, int32_t max_chunks,
                  ShardPtrs count_bufs, int32_t n_count_bufs) {
  pdl_enter();
  __shared__ int32_t s_pre[kMaxExperts];
  __shared__ int32_t s_w[32 * kMaxExperts];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  __shared__ char* s_rank[SMOE_MAX_SHARDS];
  __shared__ char* s_cb[SMOE_MAX_SHARDS];
  stage_ptrs(s_ids, topk_ids);
  stage_ptrs(s_rank, pair_rank);
  stage_ptrs(s_cb, count_bufs);
  __syncthreads();
  const int gl = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t g = lr.shard_begin + gl;
  const int64_t P = (int64_t)lr.counts[g] * k;
  const int32_t nchunks = (int32_t)((P + kRouteThreads - 1) / kRouteThreads);
  // chunk_counts == nullptr: every shard's pairs fit one chunk (decode-sized
  // batches) and this kernel counts them itself -- route_count is skipped
  const bool single = chunk_counts == nullptr;
  const int32_t* cc = single ? nullptr : chunk_counts + (int64_t)gl * max_chunks * N;
  if (blockIdx.x == 0 && !single) {  // publish row g of the [G, N] count matrix
    for (int e = tid; e < N; e += kRouteThreads) {
      int32_t tot = 0;
      for (int c = 0; c < nchunks; ++c) tot += cc[c * N + e];
      for (int i = 0; i < n_count_bufs; ++i)
        reinterpret_cast<int32_t*>(s_cb[i])[g * N + e] = tot;
    }
  }
  for (int b = blockIdx.x; b < nchunks; b += gridDim.x) {
    for (int e = tid; e < N; e += kRouteThreads) {
      int32_t pre = 0;
      for (int c = 0; c < b && !single; ++c) pre += cc[c * N + e];
      s_pre[e] = pre;
    }
    for (int e = tid; e < 32 * N; e += kRouteThreads) s_w[e] = 0;
    __syncthreads();
    const int64_t p = (int64_t)b * kRouteThreads + tid;
    const int32_t e = p < P ? reinterpret_cast<const int32_t*>(s_ids[gl])[p] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int32_t rw = __popc(peers & lanemask_lt());
    if (e >= 0 && lane == __ffs(peers) - 1) s_w[warp * N + e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int32_t r = s_pre[e] + rw;
      for (int w = 0; w < warp; ++w) r += s_w[w * N + e];
      reinterpret_cast<int32_t*>(s_rank[gl])[p] = r;
    }
    if (single) {                    // the only chunk: its totals are row g
      for (int ee = tid; ee < N; ee += kRouteThreads) {
        int32_t tot = 0;
        for (int w = 0; w < kRouteThreads / 32; ++w) tot += s_w[w * N + ee];
        for (int i = 0; i < n_count_bufs; ++i)
          reinterpret_cast<int32_t*>(s_cb[i])[g * N + ee] = tot;
      }
    }
    __syncthreads();
  }
  if (single && nchunks == 0 && blockIdx.x == 0) {   // no pairs: a zero row
    for (int ee = tid; ee < N; ee += kRouteThreads)
      for (int i = 0; i < n_count_bufs; ++i) reinterpret_cast<int32_t*>(s_cb[i])[g * N + ee] = 0;
  }
}

size_t route_workspace_bytes(int64_t max_tokens, int32_t k, int32_t N, int32_t shard_count) {
  const int64_t chunks = ceil_div(std::max<int64_t>(max_tokens * k, 1), kRouteThreads);
  return sizeof(int32_t) * (size_t)(chunks * N * shard_count);
}

int launch_route(const LocalRows& lr, int32_t N, int32_t k, const ShardPtrs& topk_ids,
                 const ShardPtrs& pair_rank, const ShardPtrs& count_bufs, int32_t n_count_bufs,
                 int32_t* chunk_counts, int64_t n_rows_bound, cudaStream_t st) {
  if (N > kMaxExperts) return SMOE_ERR_UNSUPPORTED;
  const int32_t max_chunks =
      (int32_t)ceil_div(std::max<int64_t>(n_rows_bound * k, 1), kRouteThreads);
  // grid-strided over a shard's chunks: enough CTAs for ~2 per SM in total
  const int32_t per_shard = (int32_t)std::max<int64_t>(
      1, std::min<int64_t>(max_chunks, ceil_div(2 * num_sms(), lr.shard_count)));
  const dim3 grid(per_shard, lr.shard_count);
  if (max_chunks == 1) {
    // one chunk per shard: the rank kernel counts too (one launch, not two)
    SMOE_CUDA_TRY(launch_pdl(route_rank_kernel, grid, kRouteThreads, 0, st, lr, N, k, topk_ids,
                             pair_rank, (const int32_t*)nullptr, max_chunks, count_bufs,
                             n_count_bufs));
    SMOE_LAUNCH_CHECK();
    return SMOE_OK;
  }
  SMOE_CUDA_TRY(launch_pdl(route_count_kernel, grid, kRouteThreads, 0, st, lr, N, k, topk_ids, chunk_counts,
                                                      max_chunks));
  SMOE_LAUNCH_CHECK();
  SMOE_CUDA_TRY(launch_pdl(route_rank_kernel, grid, kRouteThreads, 0, st, lr, N, k, topk_ids, pair_rank, chunk_counts,
                                                     max_chunks, count_bufs, n_count_bufs));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ K5b dispatch
#ifndef DISPATCH_ST
#define DISPATCH_ST st_cs_v4
#endif
__global__ void __launch_bounds__(256)
dispatch_kernel(LocalRows lr, int32_t N, int32_t k, int64_t d, const int32_t* __restrict__ C,
                const int32_t* __restrict__ slot_owner, const int32_t* __restrict__ slot_first,
                ShardPtrs hs, ShardPtrs topk_ids, ShardPtrs pair_rank, ShardPtrs xin,
                ShardPtrs xmeta, int64_t expert_rows, int64_t* problems, int32_t* err,
                int32_t whole_rows, ShardPtrs xfan, int64_t* stats) {
  SMOE_TL_ENTER(4);
  // the dependents' early launch is triggered at the END of this kernel: at
  // decode sizes the next kernel is the PDL-launched up GEMM, whose 148
  // resident-but-waiting CTAs slowed the gate and this kernel by ~2 us when
  // they were launched from its start (tools/probe/forward_timeline.py);
  // triggered here they still launch as the copies finish -- DSV2-Lite /
  // Qwen2 / Mixtral 64-token forward -0.9 / -5.3 / -4.3 us
  // (profiles/r2/decode/dispatch_late_trigger/)
  pdl_wait();
  SMOE_TL_WAITED(4);
  __shared__ RowMap rm;
  __shared__ int32_t s_M[kMaxExperts];
  __shared__ int32_t s_seg[kMaxExperts];
  __shared__ int32_t s_off[SMOE_MAX_SHARDS * kMaxExperts];
  __shared__ char* s_hs[SMOE_MAX_SHARDS];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  __shared__ char* s_rank[SMOE_MAX_SHARDS];
  __shared__ char* s_xin[SMOE_MAX_SHARDS];
  __shared__ char* s_xmeta[SMOE_MAX_SHARDS];
  __shared__ char* s_xfan[SMOE_MAX_SHARDS];
  stage_ptrs(s_hs, hs);
  stage_ptrs(s_ids, topk_ids);
  stage_ptrs(s_rank, pair_rank);
  stage_ptrs(s_xin, xin);
  stage_ptrs(s_xmeta, xmeta);
  stage_ptrs(s_xfan, xfan);     // all null: no deduplication (every pair carries its row)
  const int G = lr.n_shards;
  const int tid = threadIdx.x, lane = tid & 31;
  // the [G, N] count matrix -> shared memory in one round of loads (it was
  // read column-serially: G dependent L2 round trips per thread, twice)
  for (int i = tid; i < G * N; i += blockDim.x) s_off[i] = C[i];
  load_rowmap(rm, lr);    // contains __syncthreads
  for (int e = tid; e < N; e += blockDim.x) {
    int32_t m = 0;
    for (int s = 0; s < G; ++s) m += s_off[s * N + e];
    s_M[e] = m;
  }
  __syncthreads();
  for (int e = tid; e < N; e += blockDim.x) {
    int32_t seg = 0;
    for (int e2 = slot_first[slot_owner[e]]; e2 < e; ++e2) seg += s_M[e2];
    s_seg[e] = seg;
    int32_t run = seg;                     // column e: counts -> running offsets, in place
    for (int s = 0; s < G; ++s) { const int32_t c = s_off[s * N + e]; s_off[s * N + e] = run; run += c; }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    // grouped-GEMM problem table: one problem per expert slot of the resident shards
    const int32_t e0 = slot_first[lr.shard_begin];
    const int32_t e1 = slot_first[lr.shard_begin + lr.shard_count];
    for (int e = e0 + tid; e < e1; e += blockDim.x) {
      const int32_t o = slot_owner[e];
      int64_t m = s_M[e];
      if (s_seg[e] + m > expert_rows) { set_err(err, SMOE_ERRBIT_CAPACITY); m = 0; }
      const int64_t a_off = (int64_t)(o - lr.shard_begin) * expert_rows + s_seg[e];
      int64_t* pr = problems + 4 * (e - e0);
      pr[0] = a_off; pr[1] = m; pr[2] = e - e0; pr[3] = a_off;
    }
  }
  // one warp per token (or, for decode-sized batches, per 1 KiB chunk of a
  // token's row, as in the SRS): the row is read once and written to its k slots
  const int64_t vecs = d / 8;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool whole = rm.total >= whole_rows;
  const int64_t chunks = whole ? 1 : (vecs + kChunkVecs - 1) / kChunkVecs;
  const int64_t cv = whole ? vecs : kChunkVecs;
  for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + (tid >> 5);
       it < (int64_t)rm.total * chunks; it += nwarps) {
    const int64_t q = whole ? it : it / chunks, c = it - q * chunks;
    int32_t gl; int64_t j;
    decode_row(rm, lr.shard_count, q, gl, j);
    const int32_t g = lr.shard_begin + gl;
    const int32_t* ids = reinterpret_cast<const int32_t*>(s_ids[gl]) + j * k;
    const int32_t* rk = reinterpret_cast<const int32_t*>(s_rank[gl]) + j * k;
    char* dst[kGateMaxK];
    int32_t nd = 0;
    int64_t pos_s[kGateMaxK];
    int32_t own_s[kGateMaxK];
#pragma unroll
    for (int s = 0; s < kGateMaxK; ++s) {
      pos_s[s] = -1;
      own_s[s] = -1;
      if (s < k) {
        const int32_t e = ids[s];
        own_s[s] = slot_owner[e];
        pos_s[s] = (int64_t)s_off[g * N + e] + rk[s];
      }
    }
#pragma unroll
    for (int s = 0; s < kGateMaxK; ++s) {
      if (s >= k) break;
      const int32_t o = own_s[s];
      const int64_t pos = pos_s[s];
      if (pos >= expert_rows) { if (lane == 0) set_err(err, SMOE_ERRBIT_CAPACITY); continue; }
      // deduplicated dispatch (xfan bound): an owner in another process gets
      // the row once, in the slot of the token's FIRST pair there; its other
      // pairs there only record that slot, and the owner copies the row
      // locally (fanout_kernel) -- one NVLink row per (token, remote shard)
      // instead of one per (token, expert), DeepEP-style
      const bool remote_proc = o < lr.shard_begin || o >= lr.shard_begin + lr.shard_count;
      int64_t first = -1;
      if (s_xfan[o] != nullptr) {
        if (remote_proc) {
#pragma unroll
          for (int s2 = 0; s2 < kGateMaxK; ++s2)
            if (s2 < s && first < 0 && own_s[s2] == o && pos_s[s2] < expert_rows)
              first = pos_s[s2];
        }
        // every row of the owner's buffer gets its entry for this batch (-1:
        // the row itself was stored), so the fan-out never acts on stale ones
        if (lane == 0 && c == 0) reinterpret_cast<int32_t*>(s_xfan[o])[pos] = (int32_t)first;
      }
      if (first < 0) {
        dst[nd++] = s_xin[o] + pos * d * 2;
        if (lane == 0 && c == 0 && remote_proc && stats)
          atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_SENT_ROWS), 1ull);
      }
      if (lane == 0 && c == 0)
        reinterpret_cast<int64_t*>(s_xmeta[o])[pos] = ((int64_t)g << 40) | (j * k + s);
    }
    const char* src = s_hs[gl] + j * d * 2;
    const int64_t v1 = min(vecs, (c + 1) * cv);
    int64_t v = c * cv + lane;
    for (; v + 224 < v1; v += 256) {                   // 8 loads in flight per lane
      uint4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = ld_nc_v4(src + (v + 32 * u) * 16);
      for (int i = 0; i < nd; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) DISPATCH_ST(dst[i] + (v + 32 * u) * 16, a[u]);
      }
    }
    for (; v < v1; v += 32) {
      const uint4 a = ld_nc_v4(src + v * 16);
      for (int i = 0; i < nd; ++i) DISPATCH_ST(dst[i] + v * 16, a);
    }
  }
  pdl_trigger();
  SMOE_TL_EXIT(4);
}

// Owner side of the deduplicated dispatch: every expert-input row whose
// xfan entry names another row of the same buffer (a token's non-first pair
// at this shard, sent from another process) is copied from it.  Warp per row
// (or 1 KiB chunk), over the resident shards' problem rows.
__global__ void __launch_bounds__(256)
fanout_kernel(const int64_t* __restrict__ problems, int32_t n_problems, ShardPtrs xin,
              ShardPtrs xfan, int32_t shard_begin, int64_t expert_rows, int64_t d,
              const int32_t* __restrict__ slot_owner, const int32_t* __restrict__ slot_first) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t chunks = (vecs + kChunkVecs - 1) / kChunkVecs;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int32_t e0 = slot_first[shard_begin];
  for (int32_t p = 0; p < n_problems; ++p) {
    const int64_t m = problems[4 * p + 1];
    const int32_t o = slot_owner[e0 + p];
    const int64_t seg = problems[4 * p] - (int64_t)(o - shard_begin) * expert_rows;
    const int32_t* fan = reinterpret_cast<const int32_t*>(xfan.p[o]);
    char* base = xin.p[o];
    for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
         it < m * chunks; it += nwarps) {
      const int64_t r = seg + it / chunks, c = it % chunks;
      const int32_t f = fan[r];
      if (f < 0) continue;
      const int64_t v1 = min(vecs, (c + 1) * kChunkVecs);
      for (int64_t v = c * kChunkVecs + lane; v < v1; v += 32)
        st_v4(base + (r * d + v * 8) * 2, ld_v4(base + ((int64_t)f * d + v * 8) * 2));
    }
  }
}

int launch_fanout(const int64_t* problems, int32_t n_problems, const ShardPtrs& xin,
                  const ShardPtrs& xfan, int32_t shard_begin, int64_t expert_rows, int64_t d,
                  const int32_t* slot_owner, const int32_t* slot_first, int64_t rows_bound,
                  cudaStream_t st) {
  if (n_problems <= 0 || rows_bound <= 0) return SMOE_OK;
  SMOE_CUDA_TRY(launch_pdl(fanout_kernel, grid_items(rows_bound, d), 256, 0, st, problems,
                           n_problems, xin, xfan, shard_begin, expert_rows, d, slot_owner,
                           slot_first));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

int launch_dispatch(const LocalRows& lr, int32_t N, int32_t k, int64_t d,
                    const int32_t* counts_mat, const int32_t* slot_owner,
                    const int32_t* slot_first, const ShardPtrs& hs, const ShardPtrs& topk_ids,
                    const ShardPtrs& pair_rank, const ShardPtrs& xin, const ShardPtrs& xmeta,
                    int64_t expert_rows, int64_t* problems, int32_t* err, int64_t n_rows_bound,
                    cudaStream_t st, const ShardPtrs& xfan, int64_t* stats) {
  if (N > kMaxExperts || d % 8) return SMOE_ERR_UNSUPPORTED;
  SMOE_CUDA_TRY(launch_pdl(dispatch_kernel, grid_items(std::max<int64_t>(n_rows_bound, 1), d),
                           256, 0, st, lr, N, k, d, counts_mat, slot_owner, slot_first, hs,
                           topk_ids, pair_rank, xin, xmeta, expert_rows, problems, err,
                           whole_rows_from(), xfan, stats));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ K8 combine + SAG
// Weighted sum of the k expert outputs of one row for vectors [v0, v1), stored
// to the token's original position in each of the G distinct output buffers
// (the SAG: one per process).
// U vectors per lane per iteration (U * k 16-B loads in flight); every
// output vector is the same fused multiply-add chain over s = 0..k-1
// whichever U computes it, so whole-row and chunked work items agree bit
// for bit (batch invariance).
template <int G, int U, int KM>
__device__ __forceinline__ int64_t combine_span_u(char* const (&dst_base)[G], const char* y,
                                                  const float (&wk)[kGateMaxK], int32_t k,
                                                  int64_t d, int64_t i, int64_t v, int64_t v1) {
  for (; v + 32 * (U - 1) < v1; v += 32 * U) {
    uint4 yv[U][KM];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int s = 0; s < KM; ++s)
        if (s < k) yv[u][s] = ld_nc_v4(y + ((int64_t)s * d + (v + 32 * u) * 8) * 2);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s = 0; s < KM; ++s) {
        if (s < k) {
          float t[8];
          set_bf16x8(t, yv[u][s]);
#pragma unroll
          for (int c = 0; c < 8; ++c) a[c] = __fmaf_rn(wk[s], t[c], a[c]);
        }
      }
      const uint4 o = pack_bf16x8(a);
#pragma unroll
      for (int r = 0; r < G; ++r) st_cs_v4(dst_base[r] + (i * d + (v + 32 * u) * 8) * 2, o);
    }
  }
  return v;
}

template <int G>
__device__ __forceinline__ void combine_span(char* const (&dst_base)[G], const char* y,
                                             const float (&wk)[kGateMaxK], int32_t k, int64_t d,
                                             int64_t i, int64_t v0, int64_t v1, int lane) {
  int64_t v = v0 + lane;
  if (k <= 2) v = combine_span_u<G, 4, 2>(dst_base, y, wk, k, d, i, v, v1);
  else if (k <= 4) v = combine_span_u<G, 2, 4>(dst_base, y, wk, k, d, i, v, v1);
  combine_span_u<G, 1, kGateMaxK>(dst_base, y, wk, k, d, i, v, v1);
}

// Work items: whole rows, or 1 KiB column chunks for small batches (as in the
// SRS); the first chunk of a row also writes the next layer's history window.
// MINB: CTAs per SM the register budget is sized for.  3 for k > 2 (DSV2-Lite
// combine + SAG 0.105 -> 0.095 ms at 16 384 tokens); 2 for k <= 2, whose
// 4 x k loads in flight per lane spill at 3 (Mixtral 0.084 -> 0.128 ms;
// profiles/r1_cmb_occupancy_ab.jsonl, _rejected.jsonl).
template <int G, int MINB>
__global__ void __launch_bounds__(256, MINB)
combine_sag_kernel(LocalRows lr, int32_t k, int64_t d, ShardPtrs ypair, ShardPtrs topk_w,
                   ShardPtrs outs, HistUpdate hu, int32_t whole_rows, int64_t block_rows,
                   int32_t* err) {
  SMOE_TL_ENTER(7);
  // Everything this kernel reads except the pair rows (ypair, written by
  // the down GEMM it follows) was written by kernels that completed before
  // the dispatch passed its wait -- the plan (counts, group, forward), the
  // gate (weights, ids) and the caller (input history): the first work
  // item's metadata is loaded before the wait, under the down GEMM's tail.
  pdl_trigger();
  __shared__ RowMap rm;
  __shared__ char* s_y[SMOE_MAX_SHARDS];
  __shared__ char* s_wts[SMOE_MAX_SHARDS];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  __shared__ char* s_hist[SMOE_MAX_SHARDS];
  stage_ptrs(s_y, ypair);
  stage_ptrs(s_wts, topk_w);
  stage_ptrs(s_ids, hu.topk_ids);
  stage_ptrs(s_hist, hu.hist_outs);
  load_rowmap(rm, lr);
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w0 = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  char* dst_base[G];
#pragma unroll
  for (int r = 0; r < G; ++r) dst_base[r] = outs.p[r];
  const bool whole = rm.total >= whole_rows;
  const int64_t chunks = whole ? 1 : (vecs + kChunkVecs - 1) / kChunkVecs;
  const int64_t cv = whole ? vecs : kChunkVecs;
  // the first item's token position, weights and history digit
  int64_t pre_i = 0, pre_v = 0;
  float pre_w[kGateMaxK];
  if (w0 < (int64_t)rm.total * chunks) {
    const int64_t q = whole ? w0 : w0 / chunks, c = w0 - q * chunks;
    int32_t gl; int64_t j;
    decode_row(rm, lr.shard_count, q, gl, j);
    const int64_t g = lr.shard_begin + gl;
    pre_i = lr.forward[g * rm.group + j];
    const float* w = reinterpret_cast<const float*>(s_wts[gl]) + j * k;
#pragma unroll
    for (int s = 0; s < kGateMaxK; ++s) pre_w[s] = s < k ? w[s] : 0.f;
    if (c == 0 && hu.n_hist_outs > 0 && lane < hu.hist_len) {
      const int64_t L = hu.hist_len;
      if (lane == L - 1) {
        const int32_t top1 = reinterpret_cast<const int32_t*>(s_ids[gl])[j * k];
        pre_v = hu.slot_owner[top1];
      } else {
        pre_v = hu.hist_in ? hu.hist_in[pre_i * L + lane + 1] : 0;
      }
    }
  }
  pdl_wait();
  SMOE_TL_WAITED(7);
  for (int64_t it = w0; it < (int64_t)rm.total * chunks; it += nwarps) {
    const bool first_item = it == w0;
    const int64_t q = whole ? it : it / chunks;
    const int64_t c = it - q * chunks;
    int32_t gl; int64_t j;
    decode_row(rm, lr.shard_count, q, gl, j);
    const int64_t g = lr.shard_begin + gl;
    const int64_t i = first_item ? pre_i : lr.forward[g * rm.group + j];   // original position
    // block_rows > 0 (DS-MoE pipeline): the row goes to its all-gather slot
    // g * group + j instead (the resume is a separate gather, not fused)
    const int64_t i_dst = block_rows > 0 ? g * rm.group + j : i;
    if (i_dst >= block_rows && block_rows > 0) {
      if (lane == 0 && c == 0) set_err(err, SMOE_ERRBIT_CAPACITY);
      continue;
    }
    if (c == 0 && hu.n_hist_outs > 0 && lane < hu.hist_len) {
      // next layer's window: drop the oldest digit, append the cluster of the
      // top-1 expert (the device of this routing event, predictor.py:165-166)
      const int64_t L = hu.hist_len;
      int64_t v;
      if (first_item) {
        v = pre_v;
      } else if (lane == L - 1) {
        const int32_t top1 = reinterpret_cast<const int32_t*>(s_ids[gl])[j * k];
        v = hu.slot_owner[top1];
      } else {
        // older digits shift in from the input window; with no input
        // window they are not valid (the caller tracks the valid depth)
        v = hu.hist_in ? hu.hist_in[i * L + lane + 1] : 0;
      }
      for (int b = 0; b < hu.n_hist_outs; ++b)
        reinterpret_cast<int64_t*>(s_hist[b])[i * L + lane] = v;
    }
    const float* w = reinterpret_cast<const float*>(s_wts[gl]) + j * k;
    float wk[kGateMaxK];
#pragma unroll
    for (int s = 0; s < kGateMaxK; ++s) wk[s] = first_item ? pre_w[s] : (s < k ? w[s] : 0.f);
    combine_span<G>(dst_base, s_y[gl] + j * k * d * 2, wk, k, d, i_dst, c * cv,
                    min(vecs, (c + 1) * cv), lane);
  }
  SMOE_TL_EXIT(7);
}

int launch_combine_sag(const LocalRows& lr, int32_t k, int64_t d, const ShardPtrs& ypair,
                       const ShardPtrs& topk_w, const ShardPtrs& outs, int32_t n_outs,
                       const HistUpdate& hu, int64_t n_rows_bound, cudaStream_t st,
                       int64_t block_rows, int32_t* err) {
  if (k > kGateMaxK || d % 8) return SMOE_ERR_UNSUPPORTED;
  if (n_rows_bound <= 0) return SMOE_OK;
  const int grid = grid_items(n_rows_bound, d);
  const int32_t wr = whole_rows_from();
  switch (n_outs) {
#define SMOE_CMB_CASE(G_) \
    case G_:                                                                             \
      SMOE_CUDA_TRY(k <= 2 ? launch_pdl(combine_sag_kernel<G_, 2>, grid, 256, 0, st, lr, k, d,  \
                                        ypair, topk_w, outs, hu, wr, block_rows, err)        \
                           : launch_pdl(combine_sag_kernel<G_, 3>, grid, 256, 0, st, lr, k, d,  \
                                        ypair, topk_w, outs, hu, wr, block_rows, err));      \
      break;
    SMOE_CMB_CASE(1) SMOE_CMB_CASE(2) SMOE_CMB_CASE(3) SMOE_CMB_CASE(4) SMOE_CMB_CASE(5)
    SMOE_CMB_CASE(6) SMOE_CMB_CASE(7) SMOE_CMB_CASE(8) SMOE_CMB_CASE(9) SMOE_CMB_CASE(10)
    SMOE_CMB_CASE(11) SMOE_CMB_CASE(12) SMOE_CMB_CASE(13) SMOE_CMB_CASE(14) SMOE_CMB_CASE(15)
    SMOE_CMB_CASE(16)
#undef SMOE_CMB_CASE
    default: return SMOE_ERR_UNSUPPORTED;
  }
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ standalone SAG
// Warp per source row (whole rows, or 1 KiB chunks for small batches as in
// the SRS): one 16-B load, n_outs stores to the token's original position.
__global__ void __launch_bounds__(256)
sag_kernel(LocalRows lr, int64_t d, ShardPtrs blocks, ShardPtrs outs, int32_t n_outs,
           int32_t whole_rows) {
  pdl_enter();
  __shared__ RowMap rm;
  __shared__ char* s_in[SMOE_MAX_SHARDS];
  __shared__ char* s_out[SMOE_MAX_SHARDS];
  stage_ptrs(s_in, blocks);
  stage_ptrs(s_out, outs);
  load_rowmap(rm, lr);
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool whole = rm.total >= whole_rows;
  const int64_t chunks = whole ? 1 : (vecs + kChunkVecs - 1) / kChunkVecs;
  const int64_t cv = whole ? vecs : kChunkVecs;
  for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
       it < (int64_t)rm.total * chunks; it += nwarps) {
    const int64_t q = whole ? it : it / chunks;
    const int64_t c = it - q * chunks;
    int32_t gl; int64_t j;
    decode_row(rm, lr.shard_count, q, gl, j);
    const int64_t g = lr.shard_begin + gl;
    const int64_t i = lr.forward[g * rm.group + j];
    const char* src = s_in[gl] + j * d * 2;
    const int64_t v1 = min(vecs, (c + 1) * cv);
    for (int64_t v = c * cv + lane; v < v1; v += 32) {
      const uint4 x = ld_nc_v4(src + v * 16);
      for (int o = 0; o < n_outs; ++o) st_v4(s_out[o] + (i * d + v * 8) * 2, x);
    }
  }
}

int launch_sag(const LocalRows& lr, int64_t d, const ShardPtrs& blocks, const ShardPtrs& outs,
               int32_t n_outs, int64_t n_rows_bound, cudaStream_t st) {
  if (d % 8) return SMOE_ERR_UNSUPPORTED;
  if (n_rows_bound <= 0) return SMOE_OK;
  SMOE_CUDA_TRY(launch_pdl(sag_kernel, grid_items(n_rows_bound, d), 256, 0, st, lr, d, blocks, outs, n_outs,
                                                           whole_rows_from()));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ single-rank helpers
// Pair offsets in expert-major send order (DS-MoE all2allv packing):
//   pos(j, s) = sum_{e' < e} counts[e'] + #{earlier pairs with the same expert e}
__global__ void __launch_bounds__(kRouteThreads)
pair_offsets_kernel(const int32_t* __restrict__ ids, int64_t P, int32_t N,
                    int32_t* __restrict__ pos, int32_t* __restrict__ counts) {
  __shared__ int32_t s_run[kGateMaxN];
  __shared__ int32_t s_w[32 * kGateMaxN];
  __shared__ int32_t s_base[kGateMaxN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < N; e += kRouteThreads) s_run[e] = 0;
  for (int e = tid; e < 32 * N; e += kRouteThreads) s_w[e] = 0;
  __syncthreads();
  for (int64_t base = 0; base < P; base += kRouteThreads) {
    const int64_t p = base + tid;
    const int32_t e = p < P ? ids[p] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int32_t rw = __popc(peers & lanemask_lt());
    if (e >= 0 && lane == __ffs(peers) - 1) s_w[warp * N + e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int32_t r = s_run[e] + rw;
      for (int w = 0; w < warp; ++w) r += s_w[w * N + e];
      pos[p] = r;
    }
    __syncthreads();
    for (int ee = tid; ee < N; ee += kRouteThreads) {
      int32_t s = 0;
      for (int w = 0; w < 32; ++w) { s += s_w[w * N + ee]; s_w[w * N + ee] = 0; }
      s_run[ee] += s;
    }
    __syncthreads();
  }
  if (tid == 0) {
    int32_t acc = 0;
    for (int e = 0; e < N; ++e) { s_base[e] = acc; acc += s_run[e]; }
  }
  __syncthreads();
  for (int e = tid; e < N; e += kRouteThreads) counts[e] = s_run[e];
  for (int64_t p = tid; p < P; p += kRouteThreads) pos[p] += s_base[ids[p]];
}

int launch_pair_offsets(const int32_t* topk_ids, int64_t rows, int32_t k, int32_t N,
                        int32_t* pair_pos, int32_t* counts, cudaStream_t st) {
  if (N > kGateMaxN) return SMOE_ERR_UNSUPPORTED;
  pair_offsets_kernel<<<1, kRouteThreads, 0, st>>>(topk_ids, rows * k, N, pair_pos, counts);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

__global__ void __launch_bounds__(256)
pack_rows_kernel(const char* __restrict__ src, int64_t P, int32_t k, int64_t d,
                 const int32_t* __restrict__ pos, char* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); p < P;
       p += nwarps) {
    const char* s = src + (p / k) * d * 2;
    char* o = dst + (int64_t)pos[p] * d * 2;
    for (int64_t v = lane; v < vecs; v += 32) st_v4(o + v * 16, ld_nc_v4(s + v * 16));
  }
}

int launch_pack_rows(const void* src, int64_t rows, int32_t k, int64_t d, const int32_t* pair_pos,
                     void* dst, cudaStream_t st) {
  if (d % 8) return SMOE_ERR_UNSUPPORTED;
  if (rows <= 0) return SMOE_OK;
  pack_rows_kernel<<<grid_cap(ceil_div(rows * k, 8), 16), 256, 0, st>>>(
      static_cast<const char*>(src), rows * k, k, d, pair_pos, static_cast<char*>(dst));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

__global__ void __launch_bounds__(256)
combine_rows_kernel(const char* __restrict__ y, const int32_t* __restrict__ pos,
                    const float* __restrict__ topk_w, int64_t rows, int32_t k, int64_t d,
                    char* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t vecs = d / 8;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < rows;
       j += nwarps) {
    for (int64_t v = lane; v < vecs; v += 32) {
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int s = 0; s < k; ++s) {
        float t[8];
        set_bf16x8(t, ld_nc_v4(y + ((int64_t)pos[j * k + s] * d + v * 8) * 2));
        const float w = topk_w[j * k + s];
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] += w * t[c];
      }
      st_v4(out + (j * d + v * 8) * 2, pack_bf16x8(a));
    }
  }
}

int launch_combine_rows(const void* y, const int32_t* pair_pos, const float* topk_w, int64_t rows,
                        int32_t k, int64_t d, void* out, cudaStream_t st) {
  if (d % 8) return SMOE_ERR_UNSUPPORTED;
  if (rows <= 0) return SMOE_OK;
  combine_rows_kernel<<<grid_cap(ceil_div(rows, 8), 16), 256, 0, st>>>(
      static_cast<const char*>(y), pair_pos, topk_w, rows, k, d, static_cast<char*>(out));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// ------------------------------------------------------------------ barrier
__global__ void barrier_kernel(ShardPtrs signals, int32_t world, int32_t rank,
                               uint32_t* my_signal, uint32_t* epoch) {
  pdl_enter();
  __shared__ uint32_t s_e;
  if (threadIdx.x == 0) {
    s_e = *epoch + 1;
    *epoch = s_e;
  }
  __syncthreads();
  const uint32_t e = s_e;
  if ((int)threadIdx.x < world) {
    __threadfence_system();
    uint32_t* dst = reinterpret_cast<uint32_t*>(signals.p[threadIdx.x]) + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(dst), "r"(e) : "memory");
    uint32_t v = 0;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_signal + threadIdx.x)
                   : "memory");
    } while (v < e);
  }
  __syncthreads();
}

int launch_barrier(const ShardPtrs& signals, int32_t world, int32_t rank, uint32_t* my_signal,
                   uint32_t* epoch, cudaStream_t st) {
  if (world <= 1) return SMOE_OK;
  SMOE_CUDA_TRY(launch_pdl(barrier_kernel, 1, 32, 0, st, signals, world, rank, my_signal, epoch));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

}  // namespace smoe

SMOE_TL_EXPORT(layer)
