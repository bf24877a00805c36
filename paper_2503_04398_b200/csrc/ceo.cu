// ceo.cu — §8f rank 4: the batched scoring of the offline co-clustering
// search (solve_ceo, reference solver.py:380-404) on the GPU.
//
// Each cross-entropy iteration draws K expert labelings ep[k, N] and K token
// labelings tk[k, t] and scores every sample pair by within-cluster mass:
//
//   cluster_mass[k, j, c] = sum_{n : ep[k, n] = c} counts[j, n]     (tensordot)
//   ep_score[k] = sum_j max_c cluster_mass[k, j, c]                  (:392-393)
//   joint[k]    = sum_j cluster_mass[k, j, tk[k, j]]                 (:397-399)
//
// The reference materialises the [K, t, E] float64 tensor (e.g. 64 x 32000 x
// 8 = 131 MB per iteration) through a dense one-hot tensordot.  Every term is
// an integer count, so here each thread owns one token row j: its N counts
// are loaded once (coalesced from a transposed [N, t] int32 copy) and reused
// for a chunk of samples; the E bucket sums live in registers (E-way selects,
// no dynamic indexing), and the per-row max / picked bucket are summed per
// warp and atomically added into int64 totals.  Integer sums are exact and
// order-independent, so the float64 the caller gets back equals the
// reference's float64 sums bit for bit (they are exact below 2^53).
#include "common.cuh"

namespace smoe {

constexpr int kCeoThreads = 256;
constexpr int kCeoSamplesPerPass = 8;     // samples that reuse one loaded counts row

template <int E, int NMAX>
__global__ void __launch_bounds__(kCeoThreads)
ceo_score_kernel(const int32_t* __restrict__ counts_nt, int32_t t, int32_t N,
                 const int32_t* __restrict__ ep, const int32_t* __restrict__ tk, int32_t K,
                 unsigned long long* __restrict__ ep_score,
                 unsigned long long* __restrict__ joint) {
  __shared__ int8_t s_ep[kCeoSamplesPerPass][NMAX];
  const int32_t j = blockIdx.x * kCeoThreads + threadIdx.x;
  const int32_t k0 = blockIdx.y * kCeoSamplesPerPass;
  const int32_t nk = min(kCeoSamplesPerPass, K - k0);
  for (int i = threadIdx.x; i < kCeoSamplesPerPass * NMAX; i += kCeoThreads) {
    const int s = i / NMAX, n = i - s * NMAX;
    s_ep[s][n] = (s < nk && n < N) ? (int8_t)ep[(int64_t)(k0 + s) * N + n] : (int8_t)-1;
  }
  __syncthreads();
  int32_t c[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n)
    c[n] = (j < t && n < N) ? __ldg(counts_nt + (int64_t)n * t + j) : 0;
  const int lane = threadIdx.x & 31;
  for (int s = 0; s < kCeoSamplesPerPass; ++s) {
    if (s >= nk) break;
    int64_t m[E];
#pragma unroll
    for (int e = 0; e < E; ++e) m[e] = 0;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      const int lab = s_ep[s][n];
#pragma unroll
      for (int e = 0; e < E; ++e) m[e] += (lab == e) ? c[n] : 0;
    }
    unsigned long long mx = 0, pick = 0;
    if (j < t) {
      const int32_t want = tk[(int64_t)(k0 + s) * t + j];
      int64_t best = m[0];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        best = m[e] > best ? m[e] : best;
        if (e == want) pick = (unsigned long long)m[e];
      }
      mx = (unsigned long long)best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mx += __shfl_xor_sync(0xffffffffu, mx, o);
      pick += __shfl_xor_sync(0xffffffffu, pick, o);
    }
    if (lane == 0 && (mx | pick)) {
      atomicAdd(ep_score + k0 + s, mx);
      atomicAdd(joint + k0 + s, pick);
    }
  }
}

template <int E>
static int launch_ceo_e(const int32_t* counts_nt, int32_t t, int32_t N, const int32_t* ep,
                        const int32_t* tk, int32_t K, unsigned long long* ep_score,
                        unsigned long long* joint, cudaStream_t st) {
  const dim3 grid((unsigned)ceil_div(t, kCeoThreads), (unsigned)ceil_div(K, kCeoSamplesPerPass));
  if (N <= 16)
    ceo_score_kernel<E, 16><<<grid, kCeoThreads, 0, st>>>(counts_nt, t, N, ep, tk, K, ep_score, joint);
  else
    ceo_score_kernel<E, 64><<<grid, kCeoThreads, 0, st>>>(counts_nt, t, N, ep, tk, K, ep_score, joint);
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

}  // namespace smoe

using namespace smoe;

extern "C" int smoe_ceo_sample_scores(const int32_t* counts_nt, int32_t t, int32_t n_experts,
                                      const int32_t* ep_samples, const int32_t* tk_samples,
                                      int32_t n_samples, int32_t n_clusters, int64_t* ep_score,
                                      int64_t* joint, void* stream) {
  if (t < 0 || n_experts < 1 || n_samples < 0 || n_clusters < 1 || !ep_score || !joint)
    return SMOE_ERR_INVALID_ARG;
  if (n_experts > 64 || n_clusters > 16) return SMOE_ERR_UNSUPPORTED;
  cudaStream_t st = as_stream(stream);
  if (n_samples == 0) return SMOE_OK;
  SMOE_CUDA_TRY(cudaMemsetAsync(ep_score, 0, sizeof(int64_t) * n_samples, st));
  SMOE_CUDA_TRY(cudaMemsetAsync(joint, 0, sizeof(int64_t) * n_samples, st));
  if (t == 0) return SMOE_OK;
  if (!counts_nt || !ep_samples || !tk_samples) return SMOE_ERR_INVALID_ARG;
  auto* es = reinterpret_cast<unsigned long long*>(ep_score);
  auto* js = reinterpret_cast<unsigned long long*>(joint);
  if (n_clusters <= 2) return launch_ceo_e<2>(counts_nt, t, n_experts, ep_samples, tk_samples, n_samples, es, js, st);
  if (n_clusters <= 4) return launch_ceo_e<4>(counts_nt, t, n_experts, ep_samples, tk_samples, n_samples, es, js, st);
  if (n_clusters <= 8) return launch_ceo_e<8>(counts_nt, t, n_experts, ep_samples, tk_samples, n_samples, es, js, st);
  return launch_ceo_e<16>(counts_nt, t, n_experts, ep_samples, tk_samples, n_samples, es, js, st);
}
