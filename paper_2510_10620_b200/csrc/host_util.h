// host_util.h — host-side helpers shared by the executor's translation units (executor.cu,
// compile.cu, run.cu): CUDA error checks, current-device guards, TMA tensor-map encoding.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/dcpx.h"

namespace dcpx {

// Executor error: a dcpx_status plus message, mapped 1:1 onto the reference's exception
// types at the C boundary (capi.cu).
struct Failure : std::runtime_error {
  dcpx_status code;
  Failure(dcpx_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(x)                                                                        \
  do {                                                                                    \
    cudaError_t e__ = (x);                                                                \
    if (e__ != cudaSuccess)                                                               \
      throw Failure(DCPX_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e__));   \
  } while (0)


struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Current-device cursor for the enqueue loops: switches only when the device changes and
// restores the caller's device at the end (the loops visit thousands of ops per call).
struct DeviceCursor {
  int saved = 0, cur = -1;
  DeviceCursor() { cudaGetDevice(&saved); cur = saved; }
  void to(int d) {
    if (d != cur) {
      cudaSetDevice(d);
      cur = d;
    }
  }
  ~DeviceCursor() {
    if (cur != saved) cudaSetDevice(saved);
  }
};

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw Failure(DCPX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map over an arena of `rows` x 128, box `box_rows` rows x 64 columns,
// 128-byte swizzle (matches the UMMA SWIZZLE_128B descriptors in sm100.cuh).
inline CUtensorMap make_tmap(void* base, int64_t rows, uint32_t box_rows = 128) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Failure(DCPX_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// 2-D fp32 tensor map over a [rows][128] accumulator, box `box_rows` rows x 32 columns
// (128 B), 128-byte swizzle: the TMA reduce-add target of the backward's drain warps.
inline CUtensorMap make_tmap_f32(void* base, int64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Failure(DCPX_CUDA_ERROR, "cuTensorMapEncodeTiled (f32) failed: " + std::to_string(r));
  return m;
}

inline int num_sms(int ordinal) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, ordinal);
  return n > 0 ? n : 148;
}

}  // namespace dcpx
