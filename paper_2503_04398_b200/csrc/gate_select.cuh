// gate_select.cuh — softmax + ordered top-k + locality count of one router
// row with a warp (shared by the mma.sync gate and the tcgen05 gate).
#pragma once
#include "common.cuh"

namespace smoe {

constexpr int kGateMaxN = 64;      // CUDA-core / mma.sync gates and warp_topk
constexpr int kGateMaxK = 8;
constexpr int kMaxExperts = 256;   // the layer (tcgen05 gate, route, dispatch)

// Softmax + ordered top-k of one row with a warp: lane holds the logits of
// slots `lane` (v0) and `lane + 32` (v1), NaN for slots >= N.  Larger logit
// first, lowest slot on exact ties (the stable argsort of -logits over the
// s-EG slot order, test_acceptance.py:179-193); NaN marks "not a candidate"
// (slots >= N, slots already taken), so -inf logits stay candidates and fewer
// than k finite logits still give k distinct slots.  Every lane returns the
// same selection.
__device__ __forceinline__ void warp_topk(float v0, float v1, int32_t N, int32_t k,
                                          int lane, int (&sel_e)[kGateMaxK],
                                          float (&sel_p)[kGateMaxK], float& psum) {
  float mx = fmaxf(v0, v1);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float ex = (lane < N ? __expf(v0 - mx) : 0.f) + (lane + 32 < N ? __expf(v1 - mx) : 0.f);
#pragma unroll
  for (int o = 16; o; o >>= 1) ex += __shfl_xor_sync(0xffffffffu, ex, o);
  const float inv = 1.0f / ex;
  psum = 0.f;
#pragma unroll
  for (int s = 0; s < kGateMaxK; ++s) {
    sel_e[s] = 0;
    sel_p[s] = 0.f;
    if (s < k) {
      float bv; int bi;
      if (v1 == v1 && !(v0 >= v1)) { bv = v1; bi = lane + 32; }
      else if (v0 == v0) { bv = v0; bi = lane; }
      else { bv = -INFINITY; bi = 1 << 20; }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      sel_e[s] = bi;
      sel_p[s] = __expf(bv - mx) * inv;
      psum += sel_p[s];
      if (bi == lane) v0 = __int_as_float(0x7fffffff);
      if (bi == lane + 32) v1 = __int_as_float(0x7fffffff);
    }
  }
}

// Lane s < k of the warp stores selection s of row j of local shard gl and
// counts its pair as local / remote (and whether it is the first pair of
// the row to that remote shard).
__device__ __forceinline__ void warp_store_topk(int lane, int32_t k, int32_t renorm,
                                                const int (&sel_e)[kGateMaxK],
                                                const float (&sel_p)[kGateMaxK], float psum,
                                                int32_t* ids, float* wts, int64_t g,
                                                const int32_t* slot_owner,
                                                unsigned long long& my_local,
                                                unsigned long long& my_remote,
                                                unsigned long long& my_rrows) {
  if (lane >= k) return;
  float p = 0.f; int e = 0;
#pragma unroll
  for (int s = 0; s < kGateMaxK; ++s) if (s == lane) { p = sel_p[s]; e = sel_e[s]; }
  ids[lane] = e;
  wts[lane] = renorm ? p / psum : p;
  const int32_t o = slot_owner[e];
  if (o == g) {
    ++my_local;
  } else {
    ++my_remote;
    bool seen = false;                               // first pair to this shard?
#pragma unroll
    for (int s2 = 0; s2 < kGateMaxK; ++s2)
      if (s2 < lane) seen |= slot_owner[sel_e[s2]] == o;
    if (!seen) ++my_rrows;
  }
}

__device__ __forceinline__ void flush_pair_stats(unsigned long long my_local,
                                                 unsigned long long my_remote,
                                                 unsigned long long my_rrows, int64_t* stats) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    my_local += __shfl_xor_sync(0xffffffffu, my_local, o);
    my_remote += __shfl_xor_sync(0xffffffffu, my_remote, o);
    my_rrows += __shfl_xor_sync(0xffffffffu, my_rrows, o);
  }
  if ((threadIdx.x & 31) == 0 && stats && (my_local | my_remote)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_LOCAL_PAIRS), my_local);
    atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_REMOTE_PAIRS), my_remote);
    atomicAdd(reinterpret_cast<unsigned long long*>(stats + SMOE_STAT_REMOTE_ROWS), my_rrows);
  }
}

}  // namespace smoe
