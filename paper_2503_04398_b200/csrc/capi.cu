// capi.cu — library-level C-ABI entry points (version, status, device check, IPC).
#include "common.cuh"

extern "C" const char* smoe_version(void) { return "smoe 0.1.0 (sm_100a)"; }

extern "C" const char* smoe_status_string(int s) {
  switch (s) {
    case SMOE_OK: return "ok";
    case SMOE_ERR_INVALID_ARG: return "invalid argument";
    case SMOE_ERR_LENGTH: return "length mismatch";
    case SMOE_ERR_UNSUPPORTED: return "unsupported shape";
    case SMOE_ERR_CUDA: return "cuda error";
    case SMOE_ERR_CLUSTERS: return "cluster count mismatch";
    case SMOE_ERR_GATE_WIDTH: return "gate width mismatch";
    default: return "unknown status";
  }
}

extern "C" int smoe_device_ok(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return 0;
  return (major == 10 && minor == 0) ? 1 : 0;
}

extern "C" int smoe_device_alloc(size_t bytes, void** out) {
  if (!out || bytes == 0) return SMOE_ERR_INVALID_ARG;
  SMOE_CUDA_TRY(cudaMalloc(out, bytes));
  return SMOE_OK;
}

extern "C" int smoe_device_free(void* p) {
  if (!p) return SMOE_ERR_INVALID_ARG;
  SMOE_CUDA_TRY(cudaFree(p));
  return SMOE_OK;
}

extern "C" int smoe_ipc_handle(void* dev_ptr, void* handle_out_h) {
  if (!dev_ptr || !handle_out_h) return SMOE_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  SMOE_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle_out_h, &h, sizeof(h));
  return SMOE_OK;
}

extern "C" int smoe_ipc_open(const void* handle_h, void** dev_ptr_out_h) {
  if (!handle_h || !dev_ptr_out_h) return SMOE_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle_h, sizeof(h));
  SMOE_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr_out_h, h, cudaIpcMemLazyEnablePeerAccess));
  return SMOE_OK;
}

extern "C" int smoe_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return SMOE_ERR_INVALID_ARG;
  SMOE_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return SMOE_OK;
}
