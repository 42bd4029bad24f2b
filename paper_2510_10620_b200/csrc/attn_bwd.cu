// attn_bwd.cu — K1b: blockwise masked attention backward for DCP AttentionItems on
// sm_100a (tcgen05 + TMEM + TMA). No reference exists; the math is the
// gradient of exec_attention (simexec.hpp:33-76):
//   P = exp(s - LSE), dV = P^T dO, dP = dO V^T, Delta = rowsum(dO o O),
//   dS = P o (dP - Delta), dQ = scale * dS K, dK = scale * dS^T Q.
//
// Work unit = one 128-row kv sub-tile of one KV slot; it streams (item, 64-row q tile)
// steps of the division that touch it (all heads of the GQA group), accumulating dK and
// dV in TMEM. dQ of each step is reduce-added (fp32, TMA) into the q slot's accumulator.
//
// Software pipeline: the MMA issuer runs dP^T(g), S^T(g) one step ahead of the gradient
// MMAs dV(g-1), dK(g-1), dQ^T(g-1), and two compute warpgroups take alternate steps, so
// the softmax-gradient math of step g overlaps the tensor work of step g-1. K is also kept
// in TMEM for the whole unit, so S^T = K Q^T is a TS MMA (only Q read from shared memory:
// at N = 64 the SS form is shared-memory bound, 48 instead of 32 cycles per K=16 slice).
//
// CTA = 512 threads, persistent:
//   warp 0      TMA producer: Q, dO tiles + LSE/Delta rows per step (3 stages)
//   warp 1      TMEM owner + tcgen05.mma issuer
//   warp 2      TMA producer: K, V per unit
//   warp 3      unit scheduler (dynamic: global counter -> shared ring, see sched_produce)
//   warps 4-7   compute group 0 (even steps), warps 8-11 compute group 1 (odd steps):
//               TMEM lane = kv row; P^T (bf16) -> TMEM, dS^T -> smem (SW128). The group
//               taking a unit's first step first copies the unit's K tile into TMEM.
//   warps 12-15 dQ drain: dQ^T (TMEM lane = head dim) -> the step's Q/dO stage buffers
//               (fp32 [q][d], SW128) -> TMA bulk-tensor reduce-add into the accumulator.
// TMEM (512 cols): K (bf16 pairs, A operand of S^T) [0,64) | slot b in {0,1} = S^T
//       [64+64b, 128+64b) (then P^T and dS^T as bf16 in its two 32-col halves: A operands of
//       dV and dK; then dQ^T) | dP^T [192,256) (single: the compute group frees it as soon
//       as it has loaded it) | dV [256,384) | dK [384,512). dS^T also goes to smem: B operand
//       of dQ^T.
// Masks: for partial tiles each lane builds 32-bit words "q row -> kv rows of my warp"
// from the q rows' <= 2 attend ranges and transposes them across the warp (5 shuffles),
// giving every kv-row thread a bitmask over its q columns; the element loop is branch-free.
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdio>

#include "program.h"
#include "sm100.cuh"

namespace dcpx {

constexpr int kBwdThreads = 512;
// TMEM columns: K (bf16 pairs, A operand of S^T) | S^T slots 0, 1 (P^T / dS^T, then dQ^T) |
// dP^T (single) | dV | dK
constexpr uint32_t kTmK = 0, kTmS = 64, kTmDP = 192, kTmDV = 256, kTmDK = 384;
constexpr int kBwdStages = 3;
// K 32K | V 32K | dS^T[2] 32K | stages[3] x (Q 16K | dO 16K) | dQ / dK / dV staging 32K |
// LSE[3] 1K | Delta[3] 1K | barriers
constexpr int kBwdStageBytes = 32768;
constexpr int kBwdSmemMain = (96 + 32 * kBwdStages + 32) * 1024;
constexpr int kBwdSmem = kBwdSmemMain + 2048 + 512;
static_assert(kBwdSmem <= 232448, "backward shared memory exceeds the sm_100 opt-in limit");

struct BwdBarriers {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[kBwdStages], q_empty[kBwdStages];
  uint64_t s_full[2], p_ready[2], dq_full[2], dq_empty[2], ds_free[2];
  uint64_t acc_full, acc_empty;
  uint64_t ktm_full, dp_free;
  SchedRing sched;  // unit indices from the dynamic scheduler (warp 3)
  uint32_t tmem_base;
  uint32_t kv_seq;  // units whose K / V the MMA warp has seen land (monotonic)
};
static_assert(sizeof(BwdBarriers) <= 512, "barrier block exceeds its shared-memory reserve");

// Measured limits (B200, cfg3 / cfg2, tools/perf_probe.py; profiles/r2_bwd_experiments.md):
// two near-equal chains hold the kernel -- the dQ path (dQ^T MMA, drain, TMA reduce-add into
// the fp32 accumulator, whose L2 read-modify-write plus the Q / dO loads keep L2 near its
// throughput cap) and the MMA chain. Dropping the reduce alone: -7 %; dropping the dQ^T MMA
// alone: 0 %; both: -21 %; skipping the exponentials: 0 %. Not kept: dQ^T straight from
// registers by warp-wide red.global (no staging; equal or 3 % slower), rotating each unit's
// steps so concurrent units reduce into different dQ rows (equal).

// Bits [a, b) of a 32-bit word (a, b may lie outside [0, 32]).
__device__ __forceinline__ uint32_t bits_in(int64_t a, int64_t b) {
  a = a < 0 ? 0 : a;
  b = b > 32 ? 32 : b;
  if (b <= a) return 0u;
  const uint32_t hi = b == 32 ? 0xffffffffu : ((1u << b) - 1u);
  return hi & ~((1u << a) - 1u);
}

// 32x32 bit-matrix transpose across a warp: lane i holds row i (bit j = column j); on
// return lane j holds column j (bit i = row i).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
  }
  return x;
}

// Wait-cycle accounting for pipeline tuning (-DDCPX_BWD_PROFILE builds only): CTA 0's
// role leaders add the cycles spent in each wait and print them at exit.
#ifdef DCPX_BWD_PROFILE
#define BWD_PROF_DECL long long prof_[6] = {0, 0, 0, 0, 0, 0}; const long long prof_t0_ = clock64();
#define BWD_TIMED(i, stmt)                  \
  do {                                      \
    const long long t_ = clock64();         \
    stmt;                                   \
    prof_[i] += clock64() - t_;             \
  } while (0)
#define BWD_MARK(v) const long long v = clock64()
#define BWD_ADD(i, t0) prof_[i] += clock64() - (t0)
#define BWD_PROF_PRINT(name, a, b, c, d, e, f)                                                            \
  do {                                                                                                     \
    if (blockIdx.x == 0)                                                                                   \
      printf("[bwd prof] %-8s total %lld  %s %lld  %s %lld  %s %lld  %s %lld  %s %lld  %s %lld\n", name, \
             clock64() - prof_t0_, a, prof_[0], b, prof_[1], c, prof_[2], d, prof_[3], e, prof_[4], f, prof_[5]); \
  } while (0)
#else
#define BWD_PROF_DECL
#define BWD_TIMED(i, stmt) stmt
#define BWD_MARK(v)
#define BWD_ADD(i, t0)
#define BWD_PROF_PRINT(name, a, b, c, d, e, f) \
  do {                                         \
  } while (0)
#endif

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_dq,
                    const __grid_constant__ CUtensorMap tm_dkv, const BwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem;                 // [128 kv][128 d] as two SW128 halves of 64 d
  uint8_t* sV = smem + 32768;
  uint8_t* sDS = smem + 65536;        // [2][128 kv][64 q] bf16, SW128 rows of 128 B
  uint8_t* sStage = smem + 98304;     // [3] x (Q [64 q][128 d] | dO [64 q][128 d]), halves of 64 d
  uint8_t* sEpi = sStage + kBwdStages * kBwdStageBytes;  // staging: dQ [4][64 q][32] | dK/dV [2][128 kv][32] fp32
  float* sLSE = reinterpret_cast<float*>(smem + kBwdSmemMain);          // [4][64] (log2 units)
  float* sDelta = reinterpret_cast<float*>(smem + kBwdSmemMain + 1024);  // [4][64]
  BwdBarriers& bars = *reinterpret_cast<BwdBarriers*>(smem + kBwdSmemMain + 2048);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 operands need 1 KiB alignment

  if (threadIdx.x == 0) {
    mbar_init(&bars.kv_full, 1);
    mbar_init(&bars.kv_empty, 1);
    for (int i = 0; i < kBwdStages; ++i) {
      mbar_init(&bars.q_full[i], 1);
      mbar_init(&bars.q_empty[i], 1);  // MMA commit after dK, the stage's last reader
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.s_full[b], 1);
      mbar_init(&bars.p_ready[b], 128);
      mbar_init(&bars.dq_full[b], 1);
      mbar_init(&bars.dq_empty[b], 128);
      mbar_init(&bars.ds_free[b], 1);
    }
    mbar_init(&bars.acc_full, 1);
    mbar_init(&bars.acc_empty, 128);  // drain warpgroup: dK / dV read out of TMEM
    mbar_init(&bars.ktm_full, 128);   // compute group of the unit's first step: K in TMEM
    mbar_init(&bars.dp_free, 128);    // compute group of step g: dP^T(g) loaded
    bars.kv_seq = 0;
    sched_init(bars.sched, 15);  // consumers: warps 0-2, 8 compute warps, 4 drain warps
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_dq);
    tma_prefetch_desc(&tm_dkv);
  }
  if (warp == 1) tmem_alloc<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars.tmem_base;
  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");

  if (warp == 0) {
    // ------------------------------------------------------------ Q / dO producer
    // converged warp, one elected lane issues (keeps the TMA operands in uniform registers)
    {
      BWD_PROF_DECL
      uint32_t g = 0;
      for (uint32_t sk = 0;;) {
        const int u = sched_next(bars.sched, sk);
        if (u < 0) break;
        const BwdUnit U = p.units[u];
        for (int j = 0; j < U.step_count; ++j, ++g) {
          const BwdStep S = p.steps[U.step_begin + j];
          const int st = g % kBwdStages;
          uint8_t* stage = sStage + st * kBwdStageBytes;
          BWD_TIMED(1, mbar_wait(&bars.q_empty[st], ((g / kBwdStages) & 1) ^ 1));
          if (elect_one()) {
            mbar_arrive_expect_tx(&bars.q_full[st], kBwdStageBytes + 512);
            for (int h = 0; h < 2; ++h) {
              tma_load_2d(&tm_q, &bars.q_full[st], stage + h * 8192, 64 * h, S.q_row0);
              tma_load_2d(&tm_do, &bars.q_full[st], stage + 16384 + h * 8192, 64 * h, S.q_row0);
            }
            bulk_load(sLSE + st * 64, p.lse2 + S.q_row0, 256, &bars.q_full[st]);
            bulk_load(sDelta + st * 64, p.delta + S.q_row0, 256, &bars.q_full[st]);
          }
          __syncwarp();
        }
      }
      if (lane == 0) BWD_PROF_PRINT("q-prod", "-", "q_empty", "-", "-", "-", "-");
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ K / V producer
    // separate from the Q / dO stream so a unit boundary (waiting for the previous
    // unit's MMAs to release K and V) never stalls the Q / dO prefetch
    {
      BWD_PROF_DECL
      uint32_t it = 0;
      for (uint32_t sk = 0;; ++it) {
        const int u = sched_next(bars.sched, sk);
        if (u < 0) break;
        const int32_t kv_row0 = p.units[u].kv_row0;
        BWD_TIMED(0, mbar_wait(&bars.kv_empty, (it & 1) ^ 1));
        if (elect_one()) {
          mbar_arrive_expect_tx(&bars.kv_full, 65536);
          for (int h = 0; h < 2; ++h) {
            tma_load_2d(&tm_kv, &bars.kv_full, sK + h * 16384, 64 * h, kv_row0);
            tma_load_2d(&tm_kv, &bars.kv_full, sV + h * 16384, 64 * h, kv_row0 + p.slot_rows);
          }
        }
        __syncwarp();
      }
      if (lane == 0) BWD_PROF_PRINT("kv-prod", "kv_empty", "-", "-", "-", "-", "-");
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the issue loop (converged, so descriptors stay in uniform
    // registers) and one elected lane issues each batch of tcgen05 instructions; a
    // lane-0-only loop makes ptxas wrap every MMA in an R2UR waterfall loop.
    {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 64, 0, 0);   // S^T, dP^T: K-major A and B, N = 64 q
      constexpr uint32_t id_g = idesc_bf16_f32(128, 128, 0, 1);  // dV, dK: B = Q / dO MN-major, N = 128 d
      constexpr uint32_t id_q = idesc_bf16_f32(128, 64, 1, 1);   // dQ^T: A = K^T, B = dS^T, both MN-major
      // descriptor low words (sdesc_lo): K-major operands (LBO 16) for S^T / dP^T, MN-major
      // Q / dO (LBO 8192) for dV / dK, MN-major K (LBO 16384) and dS^T (LBO 8192) for dQ^T;
      // stage / slot / k-slice offsets are added as (byte offset >> 4)
      const uint32_t k_km = sdesc_lo(smem_u32(sK), 16), v_km = sdesc_lo(smem_u32(sV), 16);
      const uint32_t st_km = sdesc_lo(smem_u32(sStage), 16), st_mn = sdesc_lo(smem_u32(sStage), 8192);
      const uint32_t k_mn = sdesc_lo(smem_u32(sK), 16384), ds_mn = sdesc_lo(smem_u32(sDS), 8192);
      constexpr uint32_t kStageLo = kBwdStageBytes >> 4, kDoLo = 16384 >> 4;
      BWD_PROF_DECL
      // gradient MMAs of step g (stage st, slot b); first = first step of its unit
      auto grads = [&](uint32_t g, bool first, uint32_t it) {
        const uint32_t b = g & 1, st = g % kBwdStages;
        const uint32_t q_mn = st_mn + st * kStageLo, do_mn = q_mn + kDoLo, dsb = ds_mn + b * (16384 >> 4);
        BWD_TIMED(2, mbar_wait(&bars.p_ready[b], (g >> 1) & 1));
        tc_fence_after();
        if (first) {
          BWD_TIMED(3, mbar_wait(&bars.acc_empty, (it & 1) ^ 1));
          tc_fence_after();
        }
        if (elect_one()) {
          // dV += P^T dO   (A = P^T in TMEM, K = 64 q; B = dO MN-major)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_ts_lo(tbase + kTmDV, tbase + kTmS + 64 * b + kk * 8, do_mn + kk * 128, id_g, (!first || kk > 0) ? 1u : 0u);
          // dK += dS^T Q   (A = dS^T bf16 in TMEM slot cols [32,64); B = Q MN-major)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_ts_lo(tbase + kTmDK, tbase + kTmS + 64 * b + 32 + kk * 8, q_mn + kk * 128, id_g,
                       (!first || kk > 0) ? 1u : 0u);
          umma_commit(&bars.q_empty[st]);
          // dQ^T = K^T dS^T (A = K MN-major over d, B = dS^T MN-major over q; K = 128 kv) -> dP^T slot
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_ss_lo(tbase + kTmS + 64 * b, k_mn + kk * 128, dsb + kk * 128, id_q, kk > 0);
          umma_commit(&bars.dq_full[b]);
          umma_commit(&bars.ds_free[b]);
        }
        __syncwarp();
      };
      uint32_t g = 0, it = 0;
      for (uint32_t sk = 0;; ++it) {
        const int u = sched_next(bars.sched, sk);
        if (u < 0) break;
        const BwdUnit U = p.units[u];
        BWD_TIMED(4, mbar_wait(&bars.kv_full, it & 1));
        tc_fence_after();
        if (lane == 0) st_release_cta(&bars.kv_seq, it + 1);  // the K writer may copy K
        for (int j = 0; j < U.step_count; ++j, ++g) {
          const uint32_t b = g & 1, st = g % kBwdStages;
          const uint32_t q_km = st_km + st * kStageLo, do_km = q_km + kDoLo;
          BWD_TIMED(0, mbar_wait(&bars.q_full[st], (g / kBwdStages) & 1));
          tc_fence_after();
          // dP^T = V dO^T -> the dP^T columns, once the compute group of step g-1 has loaded
          // its dP^T (issued first: the drain of dQ^T(g-2) out of slot b overlaps it)
          if (g >= 1) {
            BWD_TIMED(5, mbar_wait(&bars.dp_free, (g - 1) & 1));
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_ss_lo(tbase + kTmDP, v_km + (kk >> 2) * 1024 + (kk & 3) * 2, do_km + (kk >> 2) * 512 + (kk & 3) * 2,
                         id_s, kk > 0);
          }
          __syncwarp();
          // S^T = K Q^T (A = K in TMEM) -> slot b, once dQ^T(g-2) has been drained from it
          if (g >= 2) {
            BWD_TIMED(1, mbar_wait(&bars.dq_empty[b], ((g >> 1) - 1) & 1));
            tc_fence_after();
          }
          if (j == 0) {
            BWD_TIMED(4, mbar_wait(&bars.ktm_full, it & 1));
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_ts_lo(tbase + kTmS + 64 * b, tbase + kTmK + kk * 8, q_km + (kk >> 2) * 512 + (kk & 3) * 2, id_s,
                         kk > 0);
            umma_commit(&bars.s_full[b]);
          }
          __syncwarp();
          if (j > 0) grads(g - 1, j == 1, it);
        }
        grads(g - 1, U.step_count == 1, it);
        if (elect_one()) {
          umma_commit(&bars.acc_full);
          umma_commit(&bars.kv_empty);
        }
        __syncwarp();
      }
      if (lane == 0) BWD_PROF_PRINT("mma", "q_full", "dq_empty", "p_ready", "acc_empty", "kv+ktm_full", "dp_free");
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ unit scheduler
    if (lane == 0) sched_produce(bars.sched, p.sched, p.sched_base, p.num_units);
    __syncwarp();
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ compute warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;");
    const uint32_t grp = (warp - 4) >> 2;           // steps with (g & 1) == grp
    const int wq = warp & 3;                        // TMEM lane quarter
    const int j = (wq << 5) + lane;                 // kv row
    const uint32_t lane_addr = tbase + ((uint32_t)(wq * 32) << 16);
    uint8_t* my_row0 = sDS + j * 128;
    BWD_PROF_DECL
    uint32_t g = 0, it = 0;
    for (uint32_t sk = 0;; ++it) {
      const int u = sched_next(bars.sched, sk);
      if (u < 0) break;
      const BwdUnit U = p.units[u];
      const bool kv_valid = j < U.n_kv;
      // descriptors of my next step are loaded a step ahead so their latency hides
      int s = (int)((grp - g) & 1);
      if (s == 0) {
        // the unit's first step is mine: copy its K tile (two SW128 halves of 64 d) into TMEM
        // cols [0,64), lane = kv row. The previous unit's S^T MMAs have completed (K / V of
        // this unit were loaded after the MMA's commit at the end of that unit). A group can
        // run units ahead (units without a step of its parity), so it waits for the MMA
        // warp's absolute unit count instead of a kv_full phase parity, which could alias.
        BWD_MARK(t_kv);
        while (ld_acquire_cta(&bars.kv_seq) < it + 1) __nanosleep(20);
        BWD_ADD(2, t_kv);
        const uint8_t* krow = sK + j * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t kr[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v4 = *reinterpret_cast<const uint4*>(krow + h * 16384 + ((c ^ (j & 7)) << 4));
            kr[4 * c] = v4.x;
            kr[4 * c + 1] = v4.y;
            kr[4 * c + 2] = v4.z;
            kr[4 * c + 3] = v4.w;
          }
          tmem_st32(lane_addr + kTmK + 32 * h, kr);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars.ktm_full);
      }
      BwdStep s_next{};
      ItemMask m_next{};
      if (s < U.step_count) {
        s_next = p.steps[U.step_begin + s];
        m_next = p.items[s_next.item];
      }
      for (; s < U.step_count; s += 2) {
        const uint32_t gs = g + s;
        const BwdStep S = s_next;
        const ItemMask im = m_next;
        if (s + 2 < U.step_count) {
          s_next = p.steps[U.step_begin + s + 2];
          m_next = p.items[s_next.item];
        }
        const uint32_t b = grp, st = gs % kBwdStages;
        BWD_MARK(t_mask);
        // ---- mask bits over the 64 q columns: mb[h] bit i <-> q column 32h + i
        uint32_t mb[2];
        if (S.cls == kTilePartial) {
          const int64_t base = im.kv_shift + S.col0 + 32 * wq;  // range coords of my warp's kv row 0
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int qi = 32 * h + lane;  // q row this lane describes
            uint32_t w = 0u;
            if (qi < S.n_q) {
              const int4 rg = __ldg(reinterpret_cast<const int4*>(p.ranges) + im.range_row0 + S.q_local0 + qi);
              w = bits_in((int64_t)rg.x - base, (int64_t)rg.y - base) | bits_in((int64_t)rg.z - base, (int64_t)rg.w - base);
            }
            mb[h] = warp_transpose32(w, lane);
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) mb[h] = bits_in(0, S.n_q - 32 * h);
        }
        if (!kv_valid) mb[0] = mb[1] = 0u;
        BWD_ADD(3, t_mask);
        BWD_TIMED(0, mbar_wait(&bars.s_full[b], (gs >> 1) & 1));
        tc_fence_after();
        if (gs >= 2) BWD_TIMED(1, mbar_wait(&bars.ds_free[b], ((gs >> 1) - 1) & 1));
        BWD_MARK(t_math);
        const float4* lse4 = reinterpret_cast<const float4*>(sLSE + st * 64);
        const float4* dlt4 = reinterpret_cast<const float4*>(sDelta + st * 64);
        const uint32_t slot = lane_addr + kTmS + 64 * b;
        // all of dP^T(gs) first, so the MMA may overwrite it with dP^T(gs+1) right away;
        // S^T in halves (half 1 is loaded before half 0's dS^T overwrites its columns)
        uint32_t sr[32], drr[2][32];
        tmem_ld32(lane_addr + kTmDP, drr[0]);
        tmem_ld32(lane_addr + kTmDP + 32, drr[1]);
        tmem_ld32(slot, sr);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars.dp_free);
        uint8_t* row = my_row0 + b * 16384;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* dr = drr[h];
          uint32_t pk[16], dk[16];
          const float2 c_s = make_float2(p.scale_log2, p.scale_log2), c_d = make_float2(p.scale, p.scale);
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            // -LSE * log2(e) and -Delta * scale per q column (delta_kernel stores them so)
            const float4 l4 = lse4[8 * h + e4];
            const float4 d4 = dlt4[8 * h + e4];
            const float2 nl[2] = {make_float2(l4.x, l4.y), make_float2(l4.z, l4.w)};
            const float2 nd[2] = {make_float2(d4.x, d4.y), make_float2(d4.z, d4.w)};
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
              const int i = 4 * e4 + 2 * e2;
              // P = 2^(s * scale * log2e - LSE * log2e); dS = P * (dP * scale - Delta * scale)
              const float2 x = ffma2(make_float2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])), c_s, nl[e2]);
              const float2 t = ffma2(make_float2(__uint_as_float(dr[i]), __uint_as_float(dr[i + 1])), c_d, nd[e2]);
              const float p0 = fast_exp2(x.x), p1 = fast_exp2(x.y);
              const float2 pv = make_float2(((mb[h] >> i) & 1u) ? p0 : 0.f, ((mb[h] >> (i + 1)) & 1u) ? p1 : 0.f);
              const float2 sv = fmul2(pv, t);
              pk[2 * e4 + e2] = pack_bf16(pv.x, pv.y);
              dk[2 * e4 + e2] = pack_bf16(sv.x, sv.y);
            }
          }
          if (h == 0) {
            tmem_ld32(slot + 32, sr);
            tmem_wait_ld();
          }
          // P^T / dS^T row j, q columns [32h, 32h+32) as bf16 pairs -> slot cols
          // [16h, 16h+16) / [32+16h, 48+16h) (A operands of dV / dK)
          tmem_st16(slot + 16 * h, pk);
          tmem_st16(slot + 32 + 16 * h, dk);
          // dS^T row j, q columns [32h, 32h+32): 16-byte chunks 4h..4h+3, 128B-swizzled
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int chunk = 4 * h + q4;
            *reinterpret_cast<uint4*>(row + ((chunk ^ (j & 7)) << 4)) =
                make_uint4(dk[4 * q4], dk[4 * q4 + 1], dk[4 * q4 + 2], dk[4 * q4 + 3]);
          }
        }
        tmem_wait_st();
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars.p_ready[b]);
        BWD_ADD(4, t_math);
      }
      g += U.step_count;
    }
    if (lane == 0 && wq == 0) BWD_PROF_PRINT(grp ? "compute1" : "compute0", "s_full", "ds_free", "kv_seq", "mask", "math", "-");
  } else if (warp >= 12) {
    // ------------------------------------------------------------ drain warpgroup
    // dQ^T of step g sits in S^T slot g&1 with TMEM lane = head dim d. Thread d
    // writes column d of four [64 q][32 d] fp32 chunks (128B-swizzled; chunk k = d / 32)
    // into the 32 KiB staging area, then one lane reduce-adds them into the dQ accumulator.
    // At the end of a unit the same warps move dV and dK out of TMEM (TMEM lane = kv row)
    // in [128 x 32] fp32 chunks through the staging area (two 16 KiB halves) into TMA
    // reduce-adds, so the compute warpgroups go straight on to the next unit.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;");
    const int wq = warp & 3;
    const int j = (wq << 5) + lane;  // kv row of the dK / dV epilogue
    const uint32_t lane_addr = tbase + ((uint32_t)(wq * 32) << 16);
    const uint32_t gran = (uint32_t)(lane >> 2), sub = (uint32_t)(lane & 3) * 4;
    BWD_PROF_DECL
    uint32_t g = 0, it = 0;
    for (uint32_t sk = 0;; ++it) {
      const int u = sched_next(bars.sched, sk);
      if (u < 0) break;
      const BwdUnit U = p.units[u];
      for (int s = 0; s < U.step_count; ++s, ++g) {
        const int q_row0 = p.steps[U.step_begin + s].q_row0;
        const uint32_t b = g & 1;
        BWD_TIMED(0, mbar_wait(&bars.dq_full[b], (g >> 1) & 1));
        tc_fence_after();
        uint32_t v[2][32];
        tmem_ld32(lane_addr + kTmS + 64 * b, v[0]);
        tmem_ld32(lane_addr + kTmS + 64 * b + 32, v[1]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars.dq_empty[b]);
        // the staging area is free once the previous reduce-adds have read it
        if (wq == 0) {
          if (elect_one()) BWD_TIMED(2, bulk_wait_read<0>());
          __syncwarp();
        }
        BWD_TIMED(1, named_bar_sync(2, 128));
        uint8_t* chunk = sEpi + wq * 8192 + sub;
#pragma unroll
        for (int q = 0; q < 64; ++q)
          *reinterpret_cast<uint32_t*>(chunk + q * 128 + ((gran ^ (q & 7)) << 4)) = v[q >> 5][q & 31];
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (wq == 0) {
          if (elect_one()) {
            for (int k = 0; k < 4; ++k) tma_reduce_add_2d(&tm_dq, sEpi + k * 8192, 32 * k, q_row0);
            bulk_commit();
          }
          __syncwarp();
        }
      }
      // ---- unit epilogue: dV (TMEM cols [256,384)) and dK ([384,512)), 8 chunks of 32
      BWD_TIMED(3, mbar_wait(&bars.acc_full, it & 1));
      BWD_MARK(t_epi);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t r[32];
        BWD_MARK(t_ld);
        tmem_ld32(lane_addr + kTmDV + 32 * c, r);
        tmem_wait_ld();
        BWD_ADD(1, t_ld);
        if (c == 7) {
          tc_fence_before();
          mbar_arrive(&bars.acc_empty);
        }
        // staging half c&1 was last read by the reduce-add two chunks back (chunk 0:
        // wait for everything, including the last step's dQ which used both halves)
        if (wq == 0) {
          if (elect_one()) {
            if (c == 0) BWD_TIMED(5, bulk_wait_read<0>());
            else BWD_TIMED(5, bulk_wait_read<1>());
          }
          __syncwarp();
        }
        BWD_TIMED(2, named_bar_sync(2, 128));
        uint8_t* row = sEpi + (c & 1) * 16384 + j * 128;
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          *reinterpret_cast<uint4*>(row + ((q4 ^ (j & 7)) << 4)) =
              make_uint4(r[4 * q4], r[4 * q4 + 1], r[4 * q4 + 2], r[4 * q4 + 3]);
        BWD_TIMED(3, fence_proxy_async_smem());
        BWD_TIMED(3, named_bar_sync(2, 128));
        if (wq == 0) {
          if (elect_one()) {
            tma_reduce_add_2d(&tm_dkv, sEpi + (c & 1) * 16384, 32 * (c & 3),
                              U.kv_row0 + (c < 4 ? p.slot_rows : 0));
            bulk_commit();
          }
          __syncwarp();
        }
      }
      BWD_ADD(4, t_epi);
    }
    if (wq == 0) {
      if (elect_one()) bulk_wait<0>();
      __syncwarp();
    }
    if (wq == 0 && lane == 0) BWD_PROF_PRINT("drain", "dq_full", "bar+ep_ld", "ep_bar1", "ep_fence+bar2", "epilogue", "epi_wait");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

void launch_attn_bwd(const CUtensorMap& tm_q, const CUtensorMap& tm_do, const CUtensorMap& tm_kv,
                     const CUtensorMap& tm_dq, const CUtensorMap& tm_dkv, const BwdParams& p, int grid,
                     cudaStream_t stream) {
  // the dynamic shared-memory opt-in is a per-device function attribute
  static uint64_t configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1ull << dev))) {
    cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    configured |= 1ull << dev;
  }
  attn_bwd_kernel<<<grid, kBwdThreads, kBwdSmem, stream>>>(tm_q, tm_do, tm_kv, tm_dq, tm_dkv, p);
}

void set_watchdog_buffer_bwd(uint32_t* diag) {
  cudaMemcpyToSymbol(g_watchdog_diag, &diag, sizeof(diag));
}

}  // namespace dcpx
