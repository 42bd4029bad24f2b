// sm100.cuh — thin inline-PTX layer for Blackwell (sm_100a): mbarrier, TMA,
// tcgen05 (MMA / TMEM alloc / ld / st / commit) and the UMMA descriptors.
//
// Layout conventions used throughout the executor kernels:
//  * Tiles of 128 rows x 128 bf16 columns (D = 128) are staged in shared memory as
//    two "halves" of 128 rows x 64 columns, each row 128 B, written by TMA with
//    CU_TENSOR_MAP_SWIZZLE_128B. A half is 16 KiB; 8-row groups are 1024 B apart.
//  * K-major UMMA operand (rows = M or N, contiguous = K): SWIZZLE_128B descriptor,
//    SBO = 1024 B, LBO unused; the k-th 16-element K step inside a half advances the
//    start address by 32 B.
//  * MN-major UMMA operand (rows = K, contiguous = M/N): SWIZZLE_128B descriptor,
//    SBO = 1024 B (next 8 K-rows), LBO = byte distance between the two 64-column
//    halves; the k-th 16-row K step advances the start address by 2048 B.
//  * Accumulators (M = 128, cta_group::1): TMEM lane = row, column = n (fp32).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace dcpx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---- mbarrier ------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Default: try_wait without a suspend-time hint (the hardware's own short time limit, then
// the caller loops). Measured on cfg2 R1: the backward kernel is 1.6 % faster than with a
// 10 ms suspend hint (24.9 vs 25.3 ms, three alternating A/B runs); -DDCPX_SUSPEND_HINT
// restores the hinted form, -DDCPX_TEST_WAIT a non-blocking test_wait spin (2 % slower).
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
#if defined(DCPX_TEST_WAIT)
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#elif !defined(DCPX_SUSPEND_HINT)
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(0x989680u)
      : "memory");
#endif
  return ok != 0;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Hang diagnostics: when a wait times out, the waiting thread records (block, thread,
// barrier shared-address, parity) into host-mapped memory (if the host registered a
// buffer through the kernel parameters) before trapping, so a protocol bug can be located
// after the launch fails. Layout: word 0 = record count, then 4 words per record.
// Each translation unit gets its own copy (static); the host sets it per device through
// set_watchdog_buffer_* (attn_fwd.cu / attn_bwd.cu). Only read on the timeout path.
static __device__ uint32_t* g_watchdog_diag = nullptr;

__device__ __forceinline__ void watchdog_report(uint32_t* diag, uint32_t addr, uint32_t parity) {
  // producer / MMA warps (0-1) of every block, other roles of block 0 only
  if (diag && (threadIdx.x & 31) == 0 && (threadIdx.x < 64 || blockIdx.x == 0)) {
    const uint32_t i = atomicAdd(diag, 1u);
    if (i < 64) {
      diag[1 + 4 * i] = blockIdx.x;
      diag[2 + 4 * i] = threadIdx.x;
      diag[3 + 4 * i] = addr;
      diag[4 + 4 * i] = parity;
    }
    __threadfence_system();
  }
}

// Blocks until the phase with the given parity has completed. A watchdog traps after
// ~10 s of waiting so a protocol bug surfaces as a launch error instead of a hung GPU.
// Debug builds (-DDCPX_WATCHDOG_REPORT) also record the stuck barrier (watchdog_report)
// before trapping; that path costs registers, so it is off in production builds.
// Race-detection build (-DDCPX_JITTER, build/jitter/libdcpx.so; compute-sanitizer is closed
// on this pool): every wait returns after a pseudo-random delay of up to ~2 us for about a
// quarter of the calls, so each role's timing relative to the others is perturbed; a missing
// or misplaced barrier then changes results (tests/test_gpu_jitter.py compares the outputs
// with the product build's bit for bit where the computation is deterministic).
#ifdef DCPX_JITTER
__device__ __forceinline__ void jitter_point() {
  uint32_t x = static_cast<uint32_t>(clock64()) * 2654435761u ^ ((threadIdx.x >> 5) * 40503u) ^ (blockIdx.x * 9973u);
  x ^= x >> 13;
  x *= 0x5bd1e995u;
  x ^= x >> 15;
  if ((x & 3u) == 0) __nanosleep(x & 2047u);
}
#else
__device__ __forceinline__ void jitter_point() {}
#endif

__device__ __forceinline__ void mbar_wait_plain(uint64_t* bar, uint32_t parity);
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  mbar_wait_plain(bar, parity);
  jitter_point();
}

__device__ __forceinline__ void mbar_wait_plain(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const uint64_t t0 = global_ns();
  uint32_t spins = 0;
  while (!mbar_try_wait(addr, parity)) {
    if ((++spins & 1023u) == 0 && global_ns() - t0 > 10000000000ull) {
#ifdef DCPX_WATCHDOG_REPORT
      watchdog_report(g_watchdog_diag, addr, parity);
      const uint64_t t1 = global_ns();  // let the other stuck roles report before trapping
      while (global_ns() - t1 < 2000000000ull) {
      }
#endif
      __trap();
    }
  }
}

// CTA-scope release store / acquire load of a shared-memory word: cross-role sequence
// counters that, unlike an mbarrier phase parity, cannot alias when a waiter runs ahead.
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// ---- device-side dependency counters (persistent cross-division launches) ------------------
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Spins until *p reaches `target` (global, acquire); traps after ~20 s so a missing signal
// surfaces as a launch error. Then orders the generic-proxy acquire before later async-proxy
// (TMA) reads of the data the signal published.
__device__ __forceinline__ void wait_counter(const uint32_t* p, uint32_t target) {
  jitter_point();  // (race-detection build: late pollers)
  if (ld_acquire_gpu(p) < target) {
    const uint64_t t0 = global_ns();
    while (ld_acquire_gpu(p) < target) {
      __nanosleep(64);  // (exponential back-off to 2 us measured: no difference)
#ifdef DCPX_WATCHDOG_REPORT
      if (global_ns() - t0 > 5000000000ull) {  // report before the mbarrier watchdog fires
        printf("[wait_counter] block %d: counter %u < target %u\n", blockIdx.x, ld_acquire_gpu(p), target);
        __trap();
      }
#endif
      if (global_ns() - t0 > 20000000000ull) __trap();
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Spins until *p == v (an epoch stamp), acquire.
__device__ __forceinline__ void wait_stamp(const uint32_t* p, uint32_t v) {
  jitter_point();
  if (ld_acquire_gpu(p) == v) return;
  const uint64_t t0 = global_ns();
  while (ld_acquire_gpu(p) != v) {
    __nanosleep(64);
    if (global_ns() - t0 > 20000000000ull) __trap();
  }
}

// ---- dynamic unit scheduler -------------------------------------------------------------
// Persistent kernels take their work units from a global counter instead of a static
// blockIdx-strided walk: one lane of a scheduler warp fetches unit indices (atomicAdd) into
// a ring of shared-memory entries and every consumer warp reads the same sequence, so all
// roles of a CTA agree on its units. CTAs then advance through the (host-ordered) unit list
// together -- the units in flight at any time are ~gridDim.x consecutive ones, which keeps
// the rows they share resident in L2 and removes the static schedule's tail imbalance.
// The counter is never reset: every launch advances it by exactly num_units + gridDim.x
// (each CTA's scheduler stops after its first fetch past the end), so the host passes the
// launch's base value and keeps the running sum (modulo 2^32).
// Ring depth = how many units a CTA may claim ahead of its slowest role: 2 lets the TMA
// warp run two units ahead without one CTA hoarding a short launch's units
// (profiles/r2_n4_scheduler_queues_persistent.md); the forward kernel may use its own depth.
#ifndef DCPX_SCHED_RING
#define DCPX_SCHED_RING 2
#endif
constexpr int kSchedRing = DCPX_SCHED_RING;
template <int N>
struct SchedRingN {
  uint64_t full[N], empty[N];
  int32_t unit[N];
};
using SchedRing = SchedRingN<kSchedRing>;

template <int N>
__device__ __forceinline__ void sched_init(SchedRingN<N>& r, uint32_t consumer_warps) {
  for (int i = 0; i < N; ++i) {
    mbar_init(&r.full[i], 1);
    mbar_init(&r.empty[i], consumer_warps);
  }
}

// Scheduler side (one thread). Writes -1 once the units are exhausted and returns.
template <int N>
__device__ __forceinline__ void sched_produce(SchedRingN<N>& r, uint32_t* ctr, uint32_t base, int num_units) {
  for (uint32_t k = 0;; ++k) {
    const uint32_t s = k % N;
    mbar_wait(&r.empty[s], ((k / N) & 1) ^ 1);
    const uint32_t t = atomicAdd(ctr, 1u) - base;
    const int u = t < static_cast<uint32_t>(num_units) ? static_cast<int>(t) : -1;
    *reinterpret_cast<volatile int32_t*>(&r.unit[s]) = u;
    mbar_arrive(&r.full[s]);  // release: the entry is visible to the waiters' acquire
    if (u < 0) return;
  }
}

// Consumer side (a converged warp): the next unit of this CTA, or -1 at the end.
template <int N>
__device__ __forceinline__ int sched_next(SchedRingN<N>& r, uint32_t& k) {
  const uint32_t s = k % N;
  mbar_wait(&r.full[s], (k / N) & 1);
  const int u = *reinterpret_cast<volatile int32_t*>(&r.unit[s]);
  jitter_point();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&r.empty[s]);
  ++k;
  return u;
}

// ---- TMA -----------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
}

__device__ __forceinline__ void tma_load_2d(const void* desc, uint64_t* bar, void* smem, int32_t x,
                                            int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(desc), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// Non-tensor bulk copy global -> shared (16 B aligned, multiple of 16 B).
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bulk reduce-add of fp32 from shared to global (no return).
__device__ __forceinline__ void bulk_reduce_add_f32(float* gmem, const void* smem, uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gmem),
      "r"(smem_u32(smem)), "r"(bytes)
      : "memory");
}
// 2-D tensor reduce-add (fp32) from shared memory into global memory through TMA.
__device__ __forceinline__ void tma_reduce_add_2d(const void* desc, const void* smem, int32_t x, int32_t y) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(desc),
      "r"(smem_u32(smem)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- named barriers ----------------------------------------------------------------------
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- tcgen05: TMEM allocation ---------------------------------------------------------
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- tcgen05: MMA ----------------------------------------------------------------------
// Instruction descriptor, kind::f16 with bf16 inputs and fp32 accumulate
// (bit layout: cute/arch/mma_sm100_desc.hpp InstrDescriptor).
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                                  // D format: f32
         | (1u << 7)                                // A format: bf16
         | (1u << 10)                               // B format: bf16
         | (static_cast<uint32_t>(a_mn_major) << 15)  // A major (0 = K)
         | (static_cast<uint32_t>(b_mn_major) << 16)  // B major (0 = K)
         | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

// Shared-memory matrix descriptor (cute/arch/mma_sm100_desc.hpp SmemDescriptor),
// version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// The same descriptor split into a constant high word (SBO = 1024, version 1, SWIZZLE_128B)
// and a low word (start address >> 4 | LBO >> 4 << 16). A byte offset `off` into the
// operand advances the low word by off >> 4 (shared addresses stay below 2^18, so the
// 14-bit address field never carries), which keeps per-MMA issue down to one add.
constexpr uint32_t kSdescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
__host__ __device__ constexpr uint32_t sdesc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr >> 4) & 0x3FFFu) | ((lbo >> 4) << 16);
}

// D[tmem] (+)= A[smem] * B[smem], descriptors given by their low words
__device__ __forceinline__ void umma_ss_lo(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %5};\n\tmov.b64 db, {%2, %5};\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "n"(kSdescHi));
}

// D[tmem] (+)= A[tmem] * B[smem], B descriptor given by its low word
__device__ __forceinline__ void umma_ts_lo(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %5};\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "r"(b_lo), "r"(idesc), "r"(accumulate), "n"(kSdescHi));
}

// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrives on `bar` once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---- tcgen05: TMEM <-> registers (32 lanes x 32 bit, one lane per thread) ------------
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 16 consecutive 32-bit columns of this thread's lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

// TMEM address of (lane, column).
__device__ __forceinline__ uint32_t tmem_addr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Packed fp32x2 arithmetic (FFMA2 / FMUL2): two lanes of work per issue slot.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA / ALU pipes, for x <= 0 (softmax exponents), to take load off MUFU:
// x = j + f with j = rint(x) (magic-number rounding) and f in [-0.5, 0.5]; 2^f by a cubic
// fitted to relative error (max 7.5e-5, unbiased; bf16 P has a 3.9e-3 step); j is added
// straight into the exponent field. x <= -126 (including -inf) gives exactly 0, like
// ex2.approx.ftz, so fully masked rows keep l = 0.
__device__ __forceinline__ float soft_exp2(float x) {
  const float t = fmaxf(x, -127.f);
  const float jr = t + 12582912.f;  // 1.5 * 2^23: the low mantissa bits hold rint(t)
  const float f = t - (jr - 12582912.f);
  float p = fmaf(0.05515746f, f, 0.24261002f);
  p = fmaf(p, f, 0.6932636f);
  p = fmaf(p, f, 0.99992824f);
  const int bits = __float_as_int(p) + (__float_as_int(jr) << 23);
  return x > -126.f ? __int_as_float(bits) : 0.f;
}

}  // namespace dcpx
