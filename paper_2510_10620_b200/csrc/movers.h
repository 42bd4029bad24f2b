// movers.h — job descriptors + launchers of the HBM-bound helper kernels (movers.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "program.h"

namespace dcpx {

constexpr int kRowsPerChunk = 64;

// Strided row copy: rows x row_bytes from src (stride src_stride) to dst. The launch
// adds src_adjust / dst_adjust to every job's pointers, so jobs built at prepare time
// can hold offsets relative to caller buffers that are only known per call.
struct RowCopyJob {
  const char* src;
  char* dst;
  int64_t src_stride, dst_stride;
  int32_t rows, row_bytes;
};

// Generic row job over 128-wide rows: a_row0 / b_row0 index rows of two arenas.
struct RowJob {
  int64_t a_row0, b_row0;
  int64_t b_stride;  // f32_to_bf16: b_row0 is an element offset, rows b_stride apart; delta: dO offset
  int32_t rows, _pad;
};

// A device-resident job list with its block decomposition (block -> job, chunk).
struct DevJobs {
  void* jobs = nullptr;              // RowCopyJob / MergeJob / RowJob array
  int32_t* job_of_block = nullptr;
  int32_t* first_chunk = nullptr;
  int32_t n_blocks = 0;
  int32_t n_jobs = 0;
};

void launch_row_copy(const DevJobs& j, cudaStream_t s, int64_t src_adjust = 0, int64_t dst_adjust = 0);
void preload_movers();  // per current device, before any launch that others spin on
void launch_counter_add(uint32_t* c, cudaStream_t s);
void launch_counter_wait(const uint32_t* c, const uint32_t* target, int n, cudaStream_t s);
void launch_merge(const DevJobs& j, const int32_t* src_rows, __nv_bfloat16* o, float* lse, cudaStream_t s);
// Delta / LSE2 preprocess fused with the dO scatter (d_o_src: the caller's packed dO,
// src_stride elements between token rows; RowJob::b_stride = element offset of a job's row 0)
void launch_delta(const DevJobs& j, const __nv_bfloat16* o, const float* lse, const __nv_bfloat16* d_o_src,
                  int64_t src_stride, __nv_bfloat16* d_o, float* delta, float* lse2, cudaStream_t s);
// jobs: RowCopyJob with src/dst = fp32 accumulators, rows of 128 floats (row_bytes ignored)
void launch_return_accum(const DevJobs& j, cudaStream_t s);
void launch_accum(const DevJobs& j, const __nv_bfloat16* src, float* dst, cudaStream_t s);
void launch_to_bf16(const DevJobs& j, const float* src, __nv_bfloat16* dst, cudaStream_t s);

void launch_attn_bwd(const CUtensorMap& tm_q, const CUtensorMap& tm_do, const CUtensorMap& tm_kv,
                     const CUtensorMap& tm_dq, const CUtensorMap& tm_dkv, const BwdParams& p, int grid,
                     cudaStream_t stream);
void set_watchdog_buffer_fwd(uint32_t* diag);  // per current device
void set_watchdog_buffer_bwd(uint32_t* diag);
void launch_attn_fwd(const CUtensorMap& tm_q, const CUtensorMap& tm_kv, const FwdParams& p, int grid,
                     cudaStream_t stream);

// Per-rank transport: device-side epoch flags in memory shared across processes (CUDA IPC).
// flag_set publishes `epoch` after everything queued earlier on the stream (system-scope
// release); flag_wait holds the stream until every flags[i * stride] >= epoch (acquire),
// trapping after ~10 s instead of hanging the GPU.
void launch_flag_set(uint32_t* flag, uint32_t epoch, cudaStream_t s);
void launch_flag_wait(const uint32_t* const* flags, int n, uint32_t epoch, cudaStream_t s);

}  // namespace dcpx
