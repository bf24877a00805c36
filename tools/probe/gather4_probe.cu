// Probe of TMA tile::gather4 on sm_100a: which box height, and is the 128B
// swizzle applied by destination address (so 32 gather4s == one 128-row tile)?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3,
                      uint16_t* out, int mode) {
  __shared__ __align__(1024) uint16_t sm[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8 * 64; ++i) sm[i] = 0xFFFF;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(4 * 128));
    // destination: the second 512 B half of a 1024 B swizzle atom when mode == 1
    uint32_t dst = s + (mode == 1 ? 512 : 0);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
        :: "r"(dst), "l"(&map), "r"(b), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}"
                 :: "r"(b));
    for (int i = 0; i < 8 * 64; ++i) out[i] = sm[i];
  }
}

int main() {
  const int rows = 1024, cols = 64;
  std::vector<uint16_t> h(rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint16_t)(r * 64 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 8 * 64 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  for (int box_h : {1, 4}) {
    for (int sw : {0, 1}) {
      for (int mode : {0, 1}) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t str[1] = {(cuuint64_t)cols * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)box_h};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("box_h=%d sw=%d encode failed %d\n", box_h, sw, (int)r); continue; }
        cudaMemset(o, 0, 8 * 64 * 2);
        probe<<<1, 32>>>(m, 5, 100, 7, 1000, o, mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint16_t> got(8 * 64);
        cudaMemcpy(got.data(), o, got.size() * 2, cudaMemcpyDeviceToHost);
        printf("box_h=%d sw=%d mode=%d err=%s\n", box_h, sw, mode, cudaGetErrorString(e));
        for (int rr = 0; rr < 8; ++rr) {
          printf("  smem row %d:", rr);
          for (int ch = 0; ch < 8; ++ch) {
            uint16_t v = got[rr * 64 + ch * 8];
            if (v == 0xFFFF) printf("    ---");
            else printf(" %3d/%d", v / 64, (v % 64) / 8);
          }
          printf("\n");
        }
        if (e != cudaSuccess) return 1;
      }
    }
  }
  return 0;
}
