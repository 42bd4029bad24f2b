// movers.cu — HBM-bound helpers of the executor:
//  * row_copy   : batched strided row copies (resident scatter of packed Q/K/V, output
//                 gather, CopyInstr, LOCAL-transport block transfers incl. peer reads).
//  * merge      : K2, rescale-and-sum merge of (O, LSE) partials, the reference's
//                 exec_reduction (simexec.hpp:80-111) in LSE form: partials with
//                 LSE = -inf (l = 0) are skipped (:96-103), rows with no partial stay 0.
//  * bwd helpers: Delta = rowsum(dO o O) preprocess, fp32 accumulate of returned
//                 partial gradients, fp32 -> bf16 conversion.
// All kernels use 16-byte vector accesses when the job is 16-byte aligned.
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdio>

#include "movers.h"

namespace dcpx {

__global__ void row_copy_kernel(const RowCopyJob* __restrict__ jobs, const int32_t* __restrict__ job_of_block,
                                const int32_t* __restrict__ first_chunk, int64_t src_adjust,
                                int64_t dst_adjust) {
  const int b = blockIdx.x;
  const int j = job_of_block[b];
  RowCopyJob J = jobs[j];
  J.src += src_adjust;
  J.dst += dst_adjust;
  const int chunk = b - first_chunk[j];  // chunk of kRowsPerChunk rows
  const int r0 = chunk * kRowsPerChunk;
  const int r1 = min(J.rows, r0 + kRowsPerChunk);
  const bool vec = ((reinterpret_cast<uintptr_t>(J.src) | reinterpret_cast<uintptr_t>(J.dst) |
                     (uintptr_t)J.src_stride | (uintptr_t)J.dst_stride | (uintptr_t)J.row_bytes) & 15) == 0;
  if (vec) {
    // all of a thread's loads are issued before its stores, so a CTA keeps its whole
    // chunk (up to 16 KiB) in flight: peer reads over NVLink are latency-bound otherwise
    constexpr int U = 4;
    const int per_row = J.row_bytes >> 4;
    const int total = (r1 - r0) * per_row;
    for (int base = 0; base < total; base += U * blockDim.x) {
      uint4 v[U];
      uint4* d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * blockDim.x + threadIdx.x;
        d[u] = nullptr;
        if (i < total) {
          const int r = r0 + i / per_row, c = i % per_row;
          v[u] = __ldcs(reinterpret_cast<const uint4*>(J.src + (int64_t)r * J.src_stride) + c);
          d[u] = reinterpret_cast<uint4*>(J.dst + (int64_t)r * J.dst_stride) + c;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (d[u]) *d[u] = v[u];
    }
  } else {
    const int per_row = J.row_bytes >> 2;
    const int total = (r1 - r0) * per_row;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int r = r0 + i / per_row, c = i % per_row;
      const uint32_t* s = reinterpret_cast<const uint32_t*>(J.src + (int64_t)r * J.src_stride) + c;
      uint32_t* d = reinterpret_cast<uint32_t*>(J.dst + (int64_t)r * J.dst_stride) + c;
      *d = *s;
    }
  }
}

// One warp per pair of rows: 16 lanes x 16 B cover one 128-wide bf16 row. Partials are taken
// in groups of 4 whose LSE and O loads are all issued before any is used, so a thread keeps
// four 16-byte loads in flight (the kernel is HBM / latency bound: ~(n_src + 1) x 260 B per row).
__global__ void merge_kernel(const MergeJob* __restrict__ jobs, const int32_t* __restrict__ src_rows,
                             const int32_t* __restrict__ job_of_block, const int32_t* __restrict__ first_chunk,
                             __nv_bfloat16* o_arena, float* lse_arena) {
  const int b = blockIdx.x;
  const int j = job_of_block[b];
  const MergeJob J = jobs[j];
  const int row_in_job = (b - first_chunk[j]) * 16 + (threadIdx.x >> 4);  // 256 threads -> 16 rows
  if (row_in_job >= J.n_rows) return;
  const int sub = threadIdx.x & 15;
  // single pass over any number of partials: running max m, running sum of weights and a
  // rescale of the accumulator whenever m grows (the LSE form of simexec.hpp:80-111)
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  float m = -CUDART_INF_F, denom = 0.f;
  constexpr int kGroup = 4;
  for (int i0 = 0; i0 < J.n_src; i0 += kGroup) {
    float l[kGroup];
    uint4 v[kGroup];
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
      l[k] = -CUDART_INF_F;
      if (i0 + k < J.n_src) {
        const int64_t row = (int64_t)__ldg(src_rows + J.src_begin + i0 + k) + row_in_job;
        l[k] = __ldcs(lse_arena + row);
        v[k] = __ldcs(reinterpret_cast<const uint4*>(o_arena + row * 128) + sub);
      }
    }
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
      if (l[k] == -CUDART_INF_F) continue;  // empty partial (l = 0 in the reference, :96-103)
      if (l[k] > m) {
        const float c = __expf(m - l[k]);  // m = -inf -> 0
        denom *= c;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] *= c;
        m = l[k];
      }
      const float w = __expf(l[k] - m);
      denom += w;
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[2 * e] = fmaf(w, __bfloat162float(h[e].x), acc[2 * e]);
        acc[2 * e + 1] = fmaf(w, __bfloat162float(h[e].y), acc[2 * e + 1]);
      }
    }
  }
  float lse_out = -CUDART_INF_F;
  if (denom > 0.f) {
    lse_out = m + __logf(denom);
    const float inv = 1.f / denom;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= inv;
  }
  __syncwarp();
  uint4 out;
  __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
  for (int e = 0; e < 4; ++e) ho[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
  *(reinterpret_cast<uint4*>(o_arena + ((int64_t)J.dst_row0 + row_in_job) * 128) + sub) = out;
  if (sub == 0) lse_arena[(int64_t)J.dst_row0 + row_in_job] = lse_out;
}

// Backward preprocess for one resident output block, fused with the dO scatter: each row of
// dO is read once from the caller's packed [T][H][D] buffer (d_o_src + job.b_stride, rows
// src_stride elements apart), stored into its Q-arena slot row for the backward kernel and
// the fetches, and dotted with O: Delta[row] = sum_d dO[row][d] * O[row][d], plus LSE in log2
// units, written at the block's Q-arena rows. One 16-lane group per row.
__global__ void delta_kernel(const RowJob* __restrict__ jobs, const int32_t* __restrict__ job_of_block,
                             const int32_t* __restrict__ first_chunk, const __nv_bfloat16* o_arena,
                             const float* lse_arena, const __nv_bfloat16* d_o_src, int64_t src_stride,
                             __nv_bfloat16* do_arena, float* delta, float* lse2) {
  const int b = blockIdx.x;
  const int j = job_of_block[b];
  const RowJob J = jobs[j];
  const int r = (b - first_chunk[j]) * 16 + (threadIdx.x >> 4);
  const int sub = threadIdx.x & 15;
  float s = 0.f;
  if (r < J.rows) {
    const uint4 a = *(reinterpret_cast<const uint4*>(o_arena + ((int64_t)J.a_row0 + r) * 128) + sub);
    const uint4 d = __ldcs(reinterpret_cast<const uint4*>(d_o_src + J.b_stride + (int64_t)r * src_stride) + sub);
    *(reinterpret_cast<uint4*>(do_arena + ((int64_t)J.b_row0 + r) * 128) + sub) = d;
    const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* hd = reinterpret_cast<const __nv_bfloat162*>(&d);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s = fmaf(__bfloat162float(ha[e].x), __bfloat162float(hd[e].x), s);
      s = fmaf(__bfloat162float(ha[e].y), __bfloat162float(hd[e].y), s);
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (r < J.rows && sub == 0) {
    // stored negated and pre-scaled for the backward kernel's packed FMAs:
    // -Delta * scale and -LSE * log2(e) (scale = 1/sqrt(128))
    delta[(int64_t)J.b_row0 + r] = -s * 0.08838834764831845f;
    lse2[(int64_t)J.b_row0 + r] = -lse_arena[(int64_t)J.a_row0 + r] * 1.4426950408889634f;
  }
}

// Gradient return (LOCAL transport): dst[i] += src[i] atomically (dst may be a peer
// device's accumulator over NVLink), then src[i] = 0 so the slot can be reused.
__global__ void return_accum_kernel(const RowCopyJob* __restrict__ jobs, const int32_t* __restrict__ job_of_block,
                                    const int32_t* __restrict__ first_chunk) {
  const int b = blockIdx.x;
  const int j = job_of_block[b];
  const RowCopyJob J = jobs[j];
  const int r0 = (b - first_chunk[j]) * kRowsPerChunk;
  const int r1 = min(J.rows, r0 + kRowsPerChunk);
  float* src = reinterpret_cast<float*>(const_cast<char*>(J.src));
  float* dst = reinterpret_cast<float*>(J.dst);
  for (int i = r0 * 32 + threadIdx.x; i < r1 * 32; i += blockDim.x) {  // rows of 128 floats, float4 each
    float4* s4 = reinterpret_cast<float4*>(src) + i;
    const float4 v = *s4;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(reinterpret_cast<float4*>(dst) + i),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
    *s4 = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dst_f32[row][c] += bf16 src[row][c] (returned partial gradients), rows of 128.
__global__ void accum_bf16_kernel(const RowJob* __restrict__ jobs, const int32_t* __restrict__ job_of_block,
                                  const int32_t* __restrict__ first_chunk, const __nv_bfloat16* src_base,
                                  float* dst_base) {
  const int b = blockIdx.x;
  const int j = job_of_block[b];
  const RowJob J = jobs[j];
  const int r = (b - first_chunk[j]) * 16 + (threadIdx.x >> 4);
  const int sub = threadIdx.x & 15;
  if (r >= J.rows) return;
  const uint4 a = *(reinterpret_cast<const uint4*>(src_base + ((int64_t)J.a_row0 + r) * 128) + sub);
  const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
  float4* d = reinterpret_cast<float4*>(dst_base + ((int64_t)J.b_row0 + r) * 128) + 2 * sub;
  float4 x = d[0], y = d[1];
  x.x += __bfloat162float(ha[0].x); x.y += __bfloat162float(ha[0].y);
  x.z += __bfloat162float(ha[1].x); x.w += __bfloat162float(ha[1].y);
  y.x += __bfloat162float(ha[2].x); y.y += __bfloat162float(ha[2].y);
  y.z += __bfloat162float(ha[3].x); y.w += __bfloat162float(ha[3].y);
  d[0] = x;
  d[1] = y;
}

// bf16 dst[b_row0 + r * b_stride] (element offsets) = fp32 src arena row a_row0 + r:
// gradient output gather / wire staging.
__global__ void f32_to_bf16_kernel(const RowJob* __restrict__ jobs, const int32_t* __restrict__ job_of_block,
                                   const int32_t* __restrict__ first_chunk, const float* src_base,
                                   __nv_bfloat16* dst_base) {
  const int b = blockIdx.x;
  const int j = job_of_block[b];
  const RowJob J = jobs[j];
  const int r = (b - first_chunk[j]) * 16 + (threadIdx.x >> 4);
  const int sub = threadIdx.x & 15;
  if (r >= J.rows) return;
  const float4* s = reinterpret_cast<const float4*>(src_base + ((int64_t)J.a_row0 + r) * 128) + 2 * sub;
  const float4 x = s[0], y = s[1];
  uint4 out;
  __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&out);
  ho[0] = __floats2bfloat162_rn(x.x, x.y);
  ho[1] = __floats2bfloat162_rn(x.z, x.w);
  ho[2] = __floats2bfloat162_rn(y.x, y.y);
  ho[3] = __floats2bfloat162_rn(y.z, y.w);
  *(reinterpret_cast<uint4*>(dst_base + J.b_row0 + (int64_t)r * J.b_stride) + sub) = out;
}

// ---------------------------------------------------------------------------- epoch flags
__global__ void flag_set_kernel(uint32_t* flag, uint32_t epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

struct FlagList {
  const uint32_t* f[64];
};

__global__ void flag_wait_kernel(FlagList fl, int n, uint32_t epoch) {
  const int i = threadIdx.x;
  if (i < n) {
    const long long t0 = clock64();
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(fl.f[i]) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
#ifdef DCPX_JITTER
      if (((clock64() >> 4) & 7) == 0) __nanosleep(3000);  // race-detection build: late pollers
#endif
      __nanosleep(200);
      if (clock64() - t0 > 100000000000LL) __trap();  // ~50 s: a peer never arrived
    }
  }
  __syncthreads();
}

// ------------------------------------------------- persistent-launch counters (comm stream)
// Adds 1 to a device counter with release semantics, after the stream's previous work (the
// transfer whose data the counter publishes).
__global__ void counter_add_kernel(uint32_t* c) {
  __threadfence();
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}

// Waits until c[i] >= target[i] for every i < n (the comm stream's receive may overwrite
// slots only once the attention units of the divisions that read them have finished).
__global__ void counter_wait_kernel(const uint32_t* c, const uint32_t* target, int n) {
  const int i = threadIdx.x;
  if (i < n) {
    const long long t0 = clock64();
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c + i) : "memory");
      if (v >= target[i]) break;
      __nanosleep(128);
#ifdef DCPX_WATCHDOG_REPORT
      if (clock64() - t0 > 8000000000LL) {
        printf("[counter_wait] done[%d] = %u < %u\n", i, v, target[i]);
        __trap();
      }
#endif
      if (clock64() - t0 > 40000000000LL) __trap();  // ~20 s: a unit never finished
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------- launchers
// Loads every kernel of this file on the current device. With lazy module loading (the CUDA
// 12 default) the first launch of a kernel loads it, which waits for the device to go idle:
// a transfer or counter kernel first launched while a persistent attention kernel spins on
// its completion would never start.
void preload_movers() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, row_copy_kernel);
  cudaFuncGetAttributes(&a, merge_kernel);
  cudaFuncGetAttributes(&a, delta_kernel);
  cudaFuncGetAttributes(&a, return_accum_kernel);
  cudaFuncGetAttributes(&a, accum_bf16_kernel);
  cudaFuncGetAttributes(&a, f32_to_bf16_kernel);
  cudaFuncGetAttributes(&a, flag_set_kernel);
  cudaFuncGetAttributes(&a, flag_wait_kernel);
  cudaFuncGetAttributes(&a, counter_add_kernel);
  cudaFuncGetAttributes(&a, counter_wait_kernel);
}
void launch_counter_add(uint32_t* c, cudaStream_t s) { counter_add_kernel<<<1, 1, 0, s>>>(c); }
void launch_counter_wait(const uint32_t* c, const uint32_t* target, int n, cudaStream_t s) {
  if (n > 0) counter_wait_kernel<<<1, 32 * ((n + 31) / 32), 0, s>>>(c, target, n);
}
void launch_flag_set(uint32_t* flag, uint32_t epoch, cudaStream_t s) { flag_set_kernel<<<1, 1, 0, s>>>(flag, epoch); }
void launch_flag_wait(const uint32_t* const* flags, int n, uint32_t epoch, cudaStream_t s) {
  if (n <= 0) return;
  FlagList fl{};
  for (int i = 0; i < n && i < 64; ++i) fl.f[i] = flags[i];
  flag_wait_kernel<<<1, 64, 0, s>>>(fl, n, epoch);
}
void launch_row_copy(const DevJobs& j, cudaStream_t s, int64_t src_adjust, int64_t dst_adjust) {
  if (j.n_blocks)
    row_copy_kernel<<<j.n_blocks, 256, 0, s>>>(static_cast<const RowCopyJob*>(j.jobs), j.job_of_block,
                                               j.first_chunk, src_adjust, dst_adjust);
}
void launch_merge(const DevJobs& j, const int32_t* src_rows, __nv_bfloat16* o, float* lse, cudaStream_t s) {
  if (j.n_blocks) merge_kernel<<<j.n_blocks, 256, 0, s>>>(static_cast<const MergeJob*>(j.jobs), src_rows, j.job_of_block, j.first_chunk, o, lse);
}
void launch_delta(const DevJobs& j, const __nv_bfloat16* o, const float* lse, const __nv_bfloat16* d_o_src,
                  int64_t src_stride, __nv_bfloat16* d_o, float* delta, float* lse2, cudaStream_t s) {
  if (j.n_blocks)
    delta_kernel<<<j.n_blocks, 256, 0, s>>>(static_cast<const RowJob*>(j.jobs), j.job_of_block, j.first_chunk, o,
                                            lse, d_o_src, src_stride, d_o, delta, lse2);
}
void launch_return_accum(const DevJobs& j, cudaStream_t s) {
  if (j.n_blocks)
    return_accum_kernel<<<j.n_blocks, 256, 0, s>>>(static_cast<const RowCopyJob*>(j.jobs), j.job_of_block,
                                                   j.first_chunk);
}
void launch_accum(const DevJobs& j, const __nv_bfloat16* src, float* dst, cudaStream_t s) {
  if (j.n_blocks) accum_bf16_kernel<<<j.n_blocks, 256, 0, s>>>(static_cast<const RowJob*>(j.jobs), j.job_of_block, j.first_chunk, src, dst);
}
void launch_to_bf16(const DevJobs& j, const float* src, __nv_bfloat16* dst, cudaStream_t s) {
  if (j.n_blocks) f32_to_bf16_kernel<<<j.n_blocks, 256, 0, s>>>(static_cast<const RowJob*>(j.jobs), j.job_of_block, j.first_chunk, src, dst);
}

}  // namespace dcpx
