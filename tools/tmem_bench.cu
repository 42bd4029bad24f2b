// tmem_bench.cu — TMEM load bandwidth per SM (tcgen05.ld.32x32b.x32), alone and while
// warp 0 keeps the tensor pipe busy with N=128 SS MMAs into other TMEM columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_10620_b200/csrc \
//        tools/tmem_bench.cu -o build/tmem_bench && build/tmem_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace dcpx;

template <int LD_WARPS, bool MMA>
__global__ void __launch_bounds__(512, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  __shared__ long long t_ld, t_mma;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  if (warp == 0) {
    if (MMA) {
      fence_proxy_async_smem();
      const long long t0 = clock64();
      constexpr uint32_t id = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t sa = smem_u32(smem), sb = sa + 32768;
      for (int i = 0; i < iters; i += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (elect_one())
            umma_ss(tbase + 384, sdesc_sw128(sa + k * 32, 16, 1024), sdesc_sw128(sb + k * 32, 16, 1024), id, 1);
        __syncwarp();
      }
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
      if (threadIdx.x == 0) t_mma = clock64() - t0;
    }
  } else if (warp >= 4 && warp < 4 + LD_WARPS) {
    const uint32_t lane_addr = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < iters / 4; i += 2) {  // two loads in flight per warp
      uint32_t r[32], r2[32];
      tmem_ld32(lane_addr + ((i * 32) & 255), r);
      tmem_ld32(lane_addr + (((i + 1) * 32) & 255), r2);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += r[e] ^ r2[e];
    }
    if (acc == 0x12345678u) out[1] = acc;
    const long long t = clock64() - t0;
    if (warp == 4 && (threadIdx.x & 31) == 0) t_ld = t;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = t_ld;
    out[2] = MMA ? t_mma : 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int W, bool M>
void run(long long* d, int sms) {
  auto k = bench<W, M>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 8192;
  k<<<sms, 512, 64 * 1024>>>(iters, d);
  k<<<sms, 512, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = (double)(iters / 4) * 4096.0 * W;  // per SM
  printf("ld warps %2d  mma %d : ld %8lld cyc -> %6.1f B/cyc/SM   mma %8lld cyc (%5.1f cyc/MMA)\n", W, (int)M, h[0],
         bytes / h[0], h[2], M ? (double)h[2] / iters : 0.0);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, false>(d, sms);
  run<8, false>(d, sms);
  run<12, false>(d, sms);
  run<4, true>(d, sms);
  run<8, true>(d, sms);
  run<12, true>(d, sms);
  return 0;
}
