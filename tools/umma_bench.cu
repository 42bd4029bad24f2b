// umma_bench.cu — issue-rate microbenchmark for the tcgen05.mma shapes and operand
// layouts the attention kernels use (bf16 in, fp32 accumulate, SW128 operands).
// One CTA per SM; warp 0 issues `iters` MMAs back to back, commits, waits, and reports
// cycles per MMA. WARP=false: lane 0 alone runs the issue loop (divergent region);
// WARP=true: the converged warp runs it and one elected lane issues each MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_10620_b200/csrc \
//        tools/umma_bench.cu -o build/umma_bench && build/umma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace dcpx;

// Variants of the current step mix (dK is TS in attn_bwd.cu): S_TS = S^T with A = K in
// TMEM (cols [448,512) here), DQ_TS = dQ^T with A = K^T in TMEM.
template <bool S_TS, bool DQ_TS>
__global__ void __launch_bounds__(128, 1) bwd_mix2(int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  if (threadIdx.x < 32) {
    fence_proxy_async_smem();
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, 0, 0), id_g = idesc_bf16_f32(128, 128, 0, 1),
                       id_q = idesc_bf16_f32(128, 64, 1, 1), id_qt = idesc_bf16_f32(128, 64, 0, 1);
    const uint32_t sk = smem_u32(smem), sv = sk + 32768, sds0 = sk + 65536, sst = sk + 98304;
    const long long t0 = clock64();
    for (int g = 0; g < steps; ++g) {
      const uint32_t b = g & 1, sq = sst + (g % 2) * 32768, sdo = sq + 16384, sds = sds0 + b * 16384;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if constexpr (S_TS)
            umma_ts(tbase + 64 * b, tbase + 448 + kk * 8, sdesc_sw128(sq + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                    id_s, kk > 0);
          else
            umma_ss(tbase + 64 * b, sdesc_sw128(sk + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    sdesc_sw128(sq + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 + 64 * b, sdesc_sw128(sv + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(sdo + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ts(tbase + 256, tbase + 64 * (b ^ 1) + kk * 8, sdesc_sw128(sdo + kk * 2048, 8192, 1024), id_g, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ts(tbase + 384 - 128 * 0 + 0, tbase + 64 * (b ^ 1) + 32 + kk * 8, sdesc_sw128(sq + kk * 2048, 8192, 1024), id_g, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if constexpr (DQ_TS)
            umma_ts(tbase + 128 + 64 * (b ^ 1), tbase + 448 + kk * 8, sdesc_sw128(sds + kk * 2048, 8192, 1024), id_qt, kk > 0);
          else
            umma_ss(tbase + 128 + 64 * (b ^ 1), sdesc_sw128(sk + kk * 2048, 16384, 1024),
                    sdesc_sw128(sds + kk * 2048, 8192, 1024), id_q, kk > 0);
        }
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

template <bool S_TS, bool DQ_TS>
void mix2(const char* name, long long* d_out, int sms) {
  cudaFuncSetAttribute(bwd_mix2<S_TS, DQ_TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int steps = 2048;
  for (int rep = 0; rep < 3; ++rep) bwd_mix2<S_TS, DQ_TS><<<sms, 128, 160 * 1024>>>(steps, d_out);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  printf("backward step MMA mix (%s): %.0f cyc/step\n", name, (double)cyc / steps);
}

// The current step mix issued by warp 0 while warps 4-7 generate other traffic the
// backward kernel has: MODE bit 0 = tcgen05.ld of 64 columns per step-equivalent loop
// (S^T / dP^T reads), bit 1 = 16-byte shared-memory stores (dS^T / dQ staging).
template <int MODE>
__global__ void __launch_bounds__(256, 1) bwd_mix_contend(int steps, long long* out, const float* gsrc,
                                                          float* gdst) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, tbar;
  __shared__ uint32_t tbase_s;
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&tbar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    fence_proxy_async_smem();
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, 0, 0), id_g = idesc_bf16_f32(128, 128, 0, 1),
                       id_q = idesc_bf16_f32(128, 64, 1, 1);
    const uint32_t sk = smem_u32(smem), sv = sk + 32768, sds0 = sk + 65536, sst = sk + 98304;
    const long long t0 = clock64();
    for (int g = 0; g < steps; ++g) {
      const uint32_t b = g & 1, sq = sst + (g % 2) * 32768, sdo = sq + 16384, sds = sds0 + b * 16384;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 * b, sdesc_sw128(sk + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(sq + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 * b + 64, sdesc_sw128(sv + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(sdo + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ts(tbase + 256, tbase + 128 * (b ^ 1) + kk * 8, sdesc_sw128(sdo + kk * 2048, 8192, 1024), id_g, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ts(tbase + 384, tbase + 128 * (b ^ 1) + 32 + kk * 8, sdesc_sw128(sq + kk * 2048, 8192, 1024), id_g, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 * (b ^ 1) + 64, sdesc_sw128(sk + kk * 2048, 16384, 1024),
                  sdesc_sw128(sds + kk * 2048, 8192, 1024), id_q, kk > 0);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
    if (threadIdx.x == 0) done = 1;
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const uint32_t lane_addr = tbase + ((uint32_t)(wq * 32) << 16);
    uint8_t* mine = smem + 160 * 1024 + wq * 4096 + (threadIdx.x & 31) * 128;
    uint32_t acc = 0, tph = 0;
    long long n = 0;
    while (!done) {
      if (MODE & 1) {
        uint32_t r[32];
        tmem_ld32(lane_addr + 0, r);
        tmem_ld32(lane_addr + 32, r);  // overwritten: only the traffic matters
        tmem_wait_ld();
        acc += r[0];
      }
      if ((MODE & 4) && (threadIdx.x & 31) == 0 && wq == 0) {
        // bulk copies global -> shared (Q / dO loads) and shared -> global reduce-adds
        // (dQ drain): 16 KiB each per iteration, to / from the traffic area
        mbar_arrive_expect_tx(&tbar, 16384);
        bulk_load(smem + 160 * 1024, gsrc + (size_t)(blockIdx.x & 63) * 4096, 16384, &tbar);
        mbar_wait(&tbar, tph);
        tph ^= 1;
        bulk_reduce_add_f32(gdst + (size_t)(blockIdx.x & 63) * 4096, smem + 160 * 1024, 16384);
        bulk_commit();
        bulk_wait_read<0>();
      }
      if (MODE & 2) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(mine + ((c ^ (threadIdx.x & 7)) << 4)) = make_uint4(acc, c, n, 1);
      }
      ++n;
    }
    if (acc == 0x12345678u) out[1] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

template <int MODE>
void contend(const char* name, long long* d_out, int sms) {
  auto k = bwd_mix_contend<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
  const int steps = 2048;
  static float* gbuf = nullptr;
  if (!gbuf) {
    cudaMalloc(&gbuf, 2 * 64 * 16384);
    cudaMemset(gbuf, 0, 2 * 64 * 16384);
  }
  for (int rep = 0; rep < 3; ++rep) k<<<sms, 256, 176 * 1024>>>(steps, d_out, gbuf, gbuf + 64 * 4096);
  cudaError_t err = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  printf("backward step MMA mix with %s: %.0f cyc/step %s\n", name, (double)cyc / steps,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

template <int N, int AMN, int BMN, bool TS, int NACC, bool WARP>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  constexpr uint32_t a_lbo = AMN ? 16384 : 16, b_lbo = BMN ? 8192 : 16;
  constexpr uint32_t a_ks = AMN ? 2048 : 32, b_ks = BMN ? 2048 : 32;
  constexpr uint32_t id = idesc_bf16_f32(128, N, AMN, BMN);
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem) + 32768;
  auto issue = [&](int i) {
    const int kk = i & 3;
    const uint32_t d = tbase + (NACC > 1 ? (uint32_t)((i % NACC) * N) : 0u);
    if constexpr (TS)
      umma_ts(d, tbase + 256 + kk * 8, sdesc_sw128(sb + kk * b_ks, b_lbo, 1024), id, 1);
    else
      umma_ss(d, sdesc_sw128(sa + kk * a_ks, a_lbo, 1024), sdesc_sw128(sb + kk * b_ks, b_lbo, 1024), id, 1);
  };
  long long t0 = 0, t1 = 0;
  if constexpr (WARP) {
    if (threadIdx.x < 32) {
      fence_proxy_async_smem();
      t0 = clock64();
      for (int i = 0; i < iters; i += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (elect_one()) issue(i + k);
        __syncwarp();
      }
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
      t1 = clock64();
    }
  } else {
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      t0 = clock64();
      for (int i = 0; i < iters; i += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) issue(i + k);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

// One backward step's MMA sequence (attn_bwd.cu): S^T, dP^T (N=64, K-major), dV (TS,
// N=128, B MN-major), dK (SS, N=128, B MN-major), dQ^T (N=64, A and B MN-major).
__global__ void __launch_bounds__(128, 1) bwd_mix(int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  if (threadIdx.x < 32) {
    fence_proxy_async_smem();
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, 0, 0), id_g = idesc_bf16_f32(128, 128, 0, 1),
                       id_q = idesc_bf16_f32(128, 64, 1, 1);
    const uint32_t sk = smem_u32(smem), sv = sk + 32768, sds0 = sk + 65536, sst = sk + 98304;
    const long long t0 = clock64();
    for (int g = 0; g < steps; ++g) {
      const uint32_t b = g & 1, sq = sst + (g % 2) * 32768, sdo = sq + 16384, sds = sds0 + b * 16384;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 * b, sdesc_sw128(sk + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(sq + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 * b + 64, sdesc_sw128(sv + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(sdo + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ts(tbase + 256, tbase + 128 * (b ^ 1) + kk * 8, sdesc_sw128(sdo + kk * 2048, 8192, 1024), id_g, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ss(tbase + 384, sdesc_sw128(sds + kk * 32, 16, 1024), sdesc_sw128(sq + kk * 2048, 8192, 1024), id_g, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tbase + 128 * (b ^ 1) + 64, sdesc_sw128(sk + kk * 2048, 16384, 1024),
                  sdesc_sw128(sds + kk * 2048, 8192, 1024), id_q, kk > 0);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}

template <int N, int AMN, int BMN, bool TS, int NACC, bool WARP>
void run(const char* name, long long* d_out, int sms) {
  auto k = bench<N, AMN, BMN, TS, NACC, WARP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 8192;
  for (int rep = 0; rep < 2; ++rep) k<<<sms, 128, 96 * 1024>>>(iters, d_out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 128, 96 * 1024>>>(iters, d_out);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(err));
    return;
  }
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 128 * N * 16 * (double)iters * sms;
  printf("%-5s acc=%d %-34s %7.1f cyc/MMA  %7.1f TFLOP/s\n", WARP ? "warp" : "lane", NACC, name, (double)cyc / iters,
         flop / (ms * 1e-3) / 1e12);
}

template <bool W>
void all(long long* d, int sms) {
  run<128, 0, 0, false, 1, W>("SS K/K   N=128", d, sms);
  run<64, 0, 0, false, 1, W>("SS K/K   N=64", d, sms);
  run<256, 0, 0, false, 1, W>("SS K/K   N=256", d, sms);
  run<128, 0, 1, false, 1, W>("SS K/MN  N=128", d, sms);
  run<128, 0, 1, true, 1, W>("TS -/MN  N=128", d, sms);
  run<128, 0, 0, true, 1, W>("TS -/K   N=128", d, sms);
  run<64, 0, 0, true, 1, W>("TS -/K   N=64", d, sms);
  run<64, 0, 1, true, 1, W>("TS -/MN  N=64", d, sms);
  run<64, 1, 1, false, 1, W>("SS MN/MN N=64", d, sms);
  run<128, 1, 1, false, 1, W>("SS MN/MN N=128", d, sms);
  run<64, 0, 0, false, 2, W>("SS K/K   N=64 (2 accumulators)", d, sms);
  run<128, 0, 0, false, 2, W>("SS K/K   N=128 (2 accumulators)", d, sms);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d_out;
  cudaMalloc(&d_out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  all<false>(d_out, sms);
  all<true>(d_out, sms);
  cudaFuncSetAttribute(bwd_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int steps = 2048;
  for (int rep = 0; rep < 3; ++rep) bwd_mix<<<sms, 128, 160 * 1024>>>(steps, d_out);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  printf("backward step MMA mix: %.0f cyc/step (32 MMAs; 24 x N=64 + 8 x N=128)\n", (double)cyc / steps);
  mix2<false, false>("current: dK TS", d_out, sms);
  mix2<true, false>("S^T TS (K in TMEM)", d_out, sms);
  mix2<false, true>("dQ^T TS (K^T in TMEM)", d_out, sms);
  mix2<true, true>("both", d_out, sms);
  contend<0>("no other traffic", d_out, sms);
  contend<1>("tcgen05.ld traffic", d_out, sms);
  contend<2>("smem store traffic", d_out, sms);
  contend<3>("tcgen05.ld + smem stores", d_out, sms);

  return 0;
}
