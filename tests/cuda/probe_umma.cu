// Standalone B200 probe of the sm100.cuh building blocks (run on a GPU box):
//   TMA SWIZZLE_128B loads, K-major SS tcgen05.mma (S = Q K^T), TMEM ld/st,
//   TS tcgen05.mma with P in TMEM and an MN-major B operand (O = P V).
// Prints max errors vs a host fp32 reference and exits non-zero on mismatch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2510_10620_b200/csrc/sm100.cuh"

using namespace dcpx;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(2);                                                                 \
    }                                                                          \
  } while (0)

__global__ void __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
          const __grid_constant__ CUtensorMap tv, float* s_out, float* o_out, float pscale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;              // 2 halves x 16 KiB
  uint8_t* sk = smem + 32768;
  uint8_t* sv = smem + 65536;
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_tma, 3 * 32768);
    for (int h = 0; h < 2; ++h) {
      tma_load_2d(&tq, &bar_tma, sq + h * 16384, 64 * h, 0);
      tma_load_2d(&tk, &bar_tma, sk + h * 16384, 64 * h, 0);
      tma_load_2d(&tv, &bar_tma, sv + h * 16384, 64 * h, 0);
    }
  }
  mbar_wait(&bar_tma, 0);
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t id = idesc_bf16_f32(128, 128, 0, 0);
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        umma_ss(tbase, sdesc_sw128(smem_u32(sq) + off, 16, 1024),
                sdesc_sw128(smem_u32(sk) + off, 16, 1024), id, kk > 0);
      }
      umma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int row = threadIdx.x;  // warp w owns lanes 32w..32w+31
  const uint32_t lane_base = (warp * 32) << 16;
  uint32_t p[64];
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(tbase + lane_base + c, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) {
      const float s = __uint_as_float(r[j]);
      s_out[row * 128 + c + j] = s;
      if (j & 1) p[(c + j) / 2] = pack_bf16(__uint_as_float(r[j - 1]) * pscale, s * pscale);
    }
  }
  tmem_st32(tbase + lane_base + 256, p);
  tmem_st32(tbase + lane_base + 256 + 32, p + 32);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t id = idesc_bf16_f32(128, 128, 0, 1);
      for (int kk = 0; kk < 8; ++kk)
        umma_ts(tbase + 128, tbase + 256 + kk * 8,
                sdesc_sw128(smem_u32(sv) + kk * 2048, 16384, 1024), id, kk > 0);
      umma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 1);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(tbase + lane_base + 128 + c, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) o_out[row * 128 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(void* base, int rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(2); }
  return m;
}

int main() {
  const int N = 128 * 128;
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  std::vector<__nv_bfloat16> hq(N), hk(N), hv(N);
  std::vector<float> fq(N), fk(N), fv(N);
  for (int i = 0; i < N; ++i) {
    hq[i] = __float2bfloat16(nd(rng)); fq[i] = __bfloat162float(hq[i]);
    hk[i] = __float2bfloat16(nd(rng)); fk[i] = __bfloat162float(hk[i]);
    hv[i] = __float2bfloat16(nd(rng)); fv[i] = __bfloat162float(hv[i]);
  }
  __nv_bfloat16 *dq, *dk, *dv;
  float *ds, *dout;
  CK(cudaMalloc(&dq, N * 2)); CK(cudaMalloc(&dk, N * 2)); CK(cudaMalloc(&dv, N * 2));
  CK(cudaMalloc(&ds, N * 4)); CK(cudaMalloc(&dout, N * 4));
  CK(cudaMemcpy(dq, hq.data(), N * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, hk.data(), N * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), N * 2, cudaMemcpyHostToDevice));
  CUtensorMap mq = make_map(dq, 128), mk = make_map(dk, 128), mv = make_map(dv, 128);
  const int smem = 3 * 32768 + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const float pscale = 0.05f;
  probe<<<1, 128, smem>>>(mq, mk, mv, ds, dout, pscale);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> s(N), o(N);
  CK(cudaMemcpy(s.data(), ds, N * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(o.data(), dout, N * 4, cudaMemcpyDeviceToHost));
  double es = 0, eo = 0, ms = 0, mo = 0;
  std::vector<float> p(N);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double acc = 0;
      for (int d = 0; d < 128; ++d) acc += (double)fq[i * 128 + d] * fk[j * 128 + d];
      es = std::max(es, std::fabs(acc - s[i * 128 + j]));
      ms = std::max(ms, std::fabs(acc));
      p[i * 128 + j] = __bfloat162float(__float2bfloat16(s[i * 128 + j] * pscale));
    }
  for (int i = 0; i < 128; ++i)
    for (int d = 0; d < 128; ++d) {
      double acc = 0;
      for (int j = 0; j < 128; ++j) acc += (double)p[i * 128 + j] * fv[j * 128 + d];
      eo = std::max(eo, std::fabs(acc - o[i * 128 + d]));
      mo = std::max(mo, std::fabs(acc));
    }
  printf("S max err %.3e (max |S| %.3f)   O max err %.3e (max |O| %.3f)\n", es, ms, eo, mo);
  const bool ok = es < 1e-2 * ms && eo < 1e-2 * mo;
  printf(ok ? "PROBE PASS\n" : "PROBE FAIL\n");
  return ok ? 0 : 1;
}
