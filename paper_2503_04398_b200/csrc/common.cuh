// common.cuh — shared device helpers for the smoe sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/smoe.h"

#define SMOE_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) { return SMOE_ERR_CUDA; }          \
  } while (0)

#define SMOE_LAUNCH_CHECK() SMOE_CUDA_TRY(cudaGetLastError())

namespace smoe {

constexpr int kWarp = 32;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs on the current device (cached per process).
int num_sms();

// ---- stage timeline probe (build variant -DSMOE_TIMELINE only) -----------
// Per kernel kind k (0 plan, 1 SRS, 2 gate, 4 dispatch, 5 up GEMM, 6 down
// GEMM, 7 combine + SAG) and CTA (< 256): %globaltimer at entry, after the
// PDL wait, and the last warp's exit -- a Gantt chart of one graph replay
// (tools/probe/forward_timeline.py).  Each translation unit has its own
// table, read through smoe_probe_tl_<unit>.
#ifdef SMOE_TIMELINE
static __device__ unsigned long long g_tl[8][256][3];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SMOE_TL_ENTER(k) \
  do { if (threadIdx.x == 0 && blockIdx.x < 256) smoe::g_tl[k][blockIdx.x][0] = smoe::tl_now(); } while (0)
#define SMOE_TL_WAITED(k) \
  do { if (threadIdx.x == 0 && blockIdx.x < 256) smoe::g_tl[k][blockIdx.x][1] = smoe::tl_now(); } while (0)
#define SMOE_TL_EXIT(k)                                                          \
  do {                                                                           \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 256)                             \
      atomicMax(&smoe::g_tl[k][blockIdx.x][2], smoe::tl_now());                  \
  } while (0)
#define SMOE_TL_EXPORT(unit)                                                      \
  extern "C" int smoe_probe_tl_##unit(unsigned long long* host) {                 \
    return cudaMemcpyFromSymbol(host, smoe::g_tl, sizeof(smoe::g_tl)) == cudaSuccess ? 0 : -1; \
  }                                                                               \
  extern "C" int smoe_probe_tl_reset_##unit() {                                   \
    static unsigned long long zero[8 * 256 * 3];                                  \
    return cudaMemcpyToSymbol(smoe::g_tl, zero, sizeof(zero)) == cudaSuccess ? 0 : -1; \
  }
#else
#define SMOE_TL_ENTER(k) do { } while (0)
#define SMOE_TL_WAITED(k) do { } while (0)
#define SMOE_TL_EXIT(k) do { } while (0)
#define SMOE_TL_EXPORT(unit)
#endif

// ---- programmatic dependent launch (PDL) --------------------------------
// Layer-path kernels are launched with programmatic stream serialisation:
// the next kernel on the stream may start while this one still runs.  Every
// such kernel calls pdl_enter() (or, after a prologue that touches only
// constant data — weights, tensor maps, shared memory, TMEM — pdl_trigger()
// then pdl_wait()) before its first global read or write of data another
// kernel produces or consumes: griddepcontrol.wait returns once the
// preceding grid has completed and its writes are visible.  Without the
// launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_enter() { pdl_trigger(); pdl_wait(); }

int pdl_enabled();                      // SMOE_OPT_PDL (default 1; env SMOE_PDL=0)
void set_pdl_enabled(int on);
void set_pdl_stage(int stage);           // layer stage being launched (-1: none)
int pdl_stage_mask();                    // SMOE_OPT_PDL_STAGES
int pdl_stage_enabled(int stage);        // would `stage`'s kernels launch early?
void set_pdl_stage_mask(int mask);

// <<<grid, block, smem, st>>> with the PDL attribute when enabled.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ void set_err(int32_t* err, int32_t bit) {
  if (err) atomicOr(err, bit);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- bf16 helpers (round-to-nearest-even, matches torch / oracle) -------
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---- 128-bit global memory access --------------------------------------
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_cs_v4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_na_v4(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// fp32 accumulate of 8 bf16 values held in a uint4
__device__ __forceinline__ void acc_bf16x8(float (&a)[8], uint4 v) {
  a[0] += bf16_lo(v.x); a[1] += bf16_hi(v.x);
  a[2] += bf16_lo(v.y); a[3] += bf16_hi(v.y);
  a[4] += bf16_lo(v.z); a[5] += bf16_hi(v.z);
  a[6] += bf16_lo(v.w); a[7] += bf16_hi(v.w);
}
__device__ __forceinline__ void set_bf16x8(float (&a)[8], uint4 v) {
  a[0] = bf16_lo(v.x); a[1] = bf16_hi(v.x);
  a[2] = bf16_lo(v.y); a[3] = bf16_hi(v.y);
  a[4] = bf16_lo(v.z); a[5] = bf16_hi(v.z);
  a[6] = bf16_lo(v.w); a[7] = bf16_hi(v.w);
}
__device__ __forceinline__ uint4 pack_bf16x8(const float (&a)[8]) {
  return make_uint4(pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]),
                    pack_bf16x2(a[4], a[5]), pack_bf16x2(a[6], a[7]));
}

}  // namespace smoe
