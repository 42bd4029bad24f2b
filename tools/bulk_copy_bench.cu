// Peer-copy throughput over NVLink on a few SMs: the executor's row-copy style (16-byte
// loads / stores, 16 KiB per block) against TMA bulk copies (cp.async.bulk global -> smem ->
// global, ~192 KiB in flight per CTA). A blocker kernel can hold all but `free_sms` SMs, as the
// persistent attention grids do. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -std=c++17 tools/bulk_copy_bench.cu -o build/bulk_copy_bench ; run with >= 2 GPUs.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

__global__ void blocker(volatile int* stop) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) {
    sm[0] = 0;
    while (!*stop) __nanosleep(1000);
  }
}

__global__ void ldst_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  constexpr int U = 4;
  const int64_t per_block = 256 * U;  // 16 KiB
  for (int64_t base = blockIdx.x * per_block; base < n16; base += gridDim.x * per_block) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 256 + threadIdx.x;
      if (i < n16) v[u] = __ldcs(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 256 + threadIdx.x;
      if (i < n16) dst[i] = v[u];
    }
  }
}

constexpr int kStages = 6;
constexpr int kChunk = 32768;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void bulk_copy(const char* __restrict__ src, char* __restrict__ dst, int64_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t nchunks = (bytes + kChunk - 1) / kChunk;
  // this CTA's chunks: c = blockIdx.x + k * gridDim.x
  const int64_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto load = [&](int64_t k) {
    const int s = k % kStages;
    const int64_t c = blockIdx.x + k * gridDim.x;
    const uint32_t n = static_cast<uint32_t>((bytes - c * kChunk < kChunk ? bytes - c * kChunk : (int64_t)kChunk));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(n) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(smem + s * kChunk)),
                 "l"(src + c * kChunk), "r"(n), "r"(su32(&bar[s]))
                 : "memory");
  };
  for (int64_t k = 0; k < mine && k < kStages; ++k) load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int s = k % kStages;
    const uint32_t parity = (k / kStages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n@!p bra W;\n}\n" ::"r"(
            su32(&bar[s])),
        "r"(parity)
        : "memory");
    const int64_t c = blockIdx.x + k * gridDim.x;
    const uint32_t n = static_cast<uint32_t>((bytes - c * kChunk < kChunk ? bytes - c * kChunk : (int64_t)kChunk));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * kChunk),
                 "r"(su32(smem + s * kChunk)), "r"(n)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage of chunk k - 1 (its store was committed one iteration ago)
    if (k >= 1 && k - 1 + kStages < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(k - 1 + kStages);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("needs 2 GPUs\n");
    return 0;
  }
  const int64_t bytes = 512ll << 20;
  char *src = nullptr, *dst = nullptr;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&dst, bytes));
  int* stop = nullptr;
  CK(cudaHostAlloc(&stop, 4, cudaHostAllocMapped));
  cudaStream_t sb, sc;
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  int lo, hi;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&sc, cudaStreamNonBlocking, hi));
  CK(cudaFuncSetAttribute(blocker, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(bulk_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  {  // load the kernels now: a lazy load while the blocker spins would wait for it forever
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, ldst_copy));
    CK(cudaFuncGetAttributes(&fa, bulk_copy));
    CK(cudaFuncGetAttributes(&fa, blocker));
  }
  // same-device sanity first (local src), then peer
  {
    char* lsrc = nullptr;
    CK(cudaMalloc(&lsrc, bytes));
    CK(cudaMemset(lsrc, 1, bytes));
    bulk_copy<<<8, 32, kStages * kChunk, sc>>>(lsrc, dst, bytes);
    CK(cudaStreamSynchronize(sc));
    std::printf("local bulk ok\n");
    bulk_copy<<<8, 32, kStages * kChunk, sc>>>(src, dst, bytes);
    CK(cudaStreamSynchronize(sc));
    std::printf("peer bulk ok\n");
  }
  char* lsrc0 = nullptr;
  CK(cudaMalloc(&lsrc0, bytes));
  CK(cudaMemset(lsrc0, 1, bytes));
  char* pdst = nullptr;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&pdst, bytes));
  CK(cudaSetDevice(0));
  for (int push = 0; push < 2; ++push)
  for (int free_sms : {4, 8, 148}) {
    const char* s_ptr = push ? lsrc0 : src;
    char* d_ptr = push ? pdst : dst;
    for (int kind = 0; kind < 2; ++kind) {
      for (int grid : {4, 8, 16, 64, 148}) {
        if (kind == 1 && grid > free_sms * 1 && free_sms < 148 && grid != free_sms) continue;
        *stop = 0;
        if (free_sms < sms) blocker<<<sms - free_sms, 32, 200 * 1024, sb>>>(stop);
        CK(cudaGetLastError());
        float best = 1e9f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(a, sc));
          if (kind == 0)
            ldst_copy<<<grid * 8, 256, 0, sc>>>(reinterpret_cast<const uint4*>(s_ptr), reinterpret_cast<uint4*>(d_ptr), bytes / 16);
          else
            bulk_copy<<<grid, 32, kStages * kChunk, sc>>>(s_ptr, d_ptr, bytes);
          CK(cudaGetLastError());
          CK(cudaEventRecord(b, sc));
          CK(cudaEventSynchronize(b));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (ms < best) best = ms;
        }
        *stop = 1;
        CK(cudaDeviceSynchronize());
        std::printf("%s free_sms %3d %s grid %3d: %.1f GB/s\n", push ? "push" : "pull", free_sms, kind ? "bulk" : "ldst", kind ? grid : grid * 8,
                    bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  // correctness of the bulk path
  CK(cudaMemset(dst, 0, bytes));
  bulk_copy<<<8, 32, kStages * kChunk, sc>>>(src, dst, bytes);
  CK(cudaDeviceSynchronize());
  std::vector<char> h(1 << 20);
  CK(cudaMemcpy(h.data(), dst + bytes - h.size(), h.size(), cudaMemcpyDeviceToHost));
  int bad = 0;
  for (char c : h) bad += c != 1;
  std::printf("bulk copy check: %s\n", bad ? "MISMATCH" : "ok");
  return 0;
}
