// blockIdx -> %smid of a 1-CTA-per-SM persistent kernel (225 KB smem, 256
// threads) launched the normal way, and launched with programmatic stream
// serialisation behind a busy kernel.  Also the CTA start clock order.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) persist(int* smid_out, long long* t_out) {
  extern __shared__ int s[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    unsigned v; asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
    smid_out[blockIdx.x] = (int)v;
    long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    t_out[blockIdx.x] = t;
    s[0] = v;
  }
}
__global__ void busy(int n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  long long t0 = clock64();
  while (clock64() - t0 < n) {}
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 225 << 10;
  cudaFuncSetAttribute(persist, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* d; long long* t;
  cudaMalloc(&d, sms * sizeof(int)); cudaMalloc(&t, sms * sizeof(long long));
  int h[1024];
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      busy<<<sms * 8, 256>>>(mode == 0 ? 0 : 200000);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(sms); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      a[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = a; cfg.numAttrs = mode == 2 ? 1 : 0;
      cudaLaunchKernelEx(&cfg, persist, d, t);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sms * sizeof(int), cudaMemcpyDeviceToHost);
      printf("{\"mode\": \"%s\", \"rep\": %d, \"smid\": [", mode == 2 ? "pdl_behind_busy" : (mode == 1 ? "normal_behind_busy" : "normal"), rep);
      for (int i = 0; i < sms; ++i) printf("%d%s", h[i], i + 1 < sms ? ", " : "");
      printf("]}\n");
    }
  }
  return 0;
}
