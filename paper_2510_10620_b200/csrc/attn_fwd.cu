// attn_fwd.cu — K1: blockwise masked attention forward for DCP AttentionItems on
// sm_100a (tcgen05 + TMEM + TMA), fused with the per-division rescale-and-sum merge.
//
// Reference semantics: exec_attention (simexec.hpp:33-76) per item, followed by
// exec_reduction (simexec.hpp:80-111) over all items of one output block. Because the
// (O, LSE) merge is associative, all kv sub-tiles of all items of a group are streamed
// through ONE online softmax; the result is written to the reduction's destination
// slot (optionally merged with that slot's current (O, LSE), i.e. the accumulator of
// earlier divisions). Rows with no attended key produce O = 0, LSE = -inf
// (simexec.hpp:61).
//
// CTA = 384 threads (3 warpgroups), persistent over FwdUnits:
//   warp 0      TMA producer: Q tiles (2 x 128 rows), K/V sub-tiles (2-stage ring)
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer
//   warp 2      unit scheduler (dynamic: global counter -> shared ring, see sched_produce)
//   warp 3      idle (warpgroup 0 donates registers: setmaxnreg 88)
//   warps 4-7   softmax / correction / epilogue for q tile 0 (warp w reads TMEM
//               lanes 32*(w%4)..+31, so the four warps cover rows 0-127); 208 regs
//   warps 8-11  same for q tile 1
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_t (bf16)
// overwrites the first 64 columns of S_t and feeds the PV MMA as the TMEM A operand.
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdio>

#include "program.h"
#include "sm100.cuh"

// The forward's scheduler ring holds one unit: its TMA warp needs no more look-ahead, and
// claiming later keeps short launches balanced (fwd kernel -0.6 % cfg3 N = 1, -5 % cfg2
// N = 4 vs depth 2; profiles/r2_n4_scheduler_queues_persistent.md section 7).
#ifndef DCPX_FWD_SCHED_RING
#define DCPX_FWD_SCHED_RING 1
#endif

namespace dcpx {

// Column pairs (of every 16) whose exp2 is evaluated by soft_exp2 instead of MUFU.
// Measured on cfg2 (B200): 0 -> 7.40 ms, 6 -> 7.60, 8 -> 8.91, 10 -> 10.1: the softmax
// warps are issue-bound rather than MUFU-bound here, so the default keeps MUFU for all.
#ifndef DCPX_SOFT_EXP_PAIRS
#define DCPX_SOFT_EXP_PAIRS 0
#endif
constexpr int kSoftExpPairs = DCPX_SOFT_EXP_PAIRS;
// Also measured (after the descriptor-issue change, 6.99 ms): exponent arguments as packed
// FFMA2 pairs 7.14 ms; plus 2 / 4 of 16 pairs through a packed-FMA soft_exp2: 7.13 / 7.17.
// Also measured and not kept: row max / row sum as 4 independent chains instead of one
// FMNMX3 / FADD chain (cfg2 7.51 vs 7.38 ms), and splitting the S load so the first half's
// max overlaps the second half's tcgen05.ld (much slower: the loaded registers spill).

// Per-phase cycle counters of the softmax warps (-DDCPX_FWD_PROFILE builds only): warp 4
// lane 0 of CTA 0 accumulates the cycles of each phase over its steps and prints them.
#ifdef DCPX_FWD_PROFILE
#define FWD_T(v) const long long v = clock64()
#define FWD_ACC(i, a, b) fprof[i] += (b) - (a)
#else
#define FWD_T(v)
#define FWD_ACC(i, a, b)
#endif

// P handed to the PV MMA in two halves (K-slices 0-3 after the first 64 columns are stored),
// so the first half of PV overlaps the second half of the exponentials. Measured (min of 10,
// alternating A/B on one B200): cfg2 7.05 -> 7.15 ms, cfg3 8.04 -> 8.00, shared-question
// 33.8 -> 34.5 ms (parity green), so it is off by default.
#ifndef DCPX_FWD_SPLIT_P
#define DCPX_FWD_SPLIT_P 0
#endif
constexpr bool kSplitP = DCPX_FWD_SPLIT_P != 0;
// Also measured and not kept (round 2): row max and row sum as 4 / 8 independent chains
// instead of one FMNMX3 / FADD chain: cfg3 8.00 -> 8.22 / 8.19 ms (the other tile's warp
// hides the chain latency; the extra live registers cost more).
// Also measured and not kept: the MMA warp issuing the two tiles' PV + next S in the order
// their P becomes ready (polling both barriers) instead of tile 0 first: 8.0 -> 9.0 ms (cfg3).

constexpr int kFwdThreads = 384;
constexpr int kFwdSmem = 6 * 32768 + 1024;  // Q0 Q1 K[2] V[2] + alignment slack
constexpr float kRescaleThreshold = 8.0f;   // log2 units: lazy O rescale (factor 256)

struct FwdBarriers {
  uint64_t q_full, q_empty;
  uint64_t k_full[2], v_full[2], kv_empty[2];
  uint64_t s_full[2], p_half[2], p_ready[2], o_full[2], o_empty[2];
  SchedRingN<DCPX_FWD_SCHED_RING> sched;  // unit indices from the dynamic scheduler (warp 2)
  uint32_t tmem_base;
};

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// Bits [a, b) of a 32-bit word (a, b may lie outside [0, 32]).
__device__ __forceinline__ uint32_t range_bits(int a, int b) {
  a = a < 0 ? 0 : a;
  b = b > 32 ? 32 : b;
  if (b <= a) return 0u;
  const uint32_t hi = b == 32 ? 0xffffffffu : ((1u << b) - 1u);
  return hi & ~((1u << a) - 1u);
}

__device__ __forceinline__ uint32_t cls_of(uint32_t cls, int t) { return (cls >> (2 * t)) & 3u; }

__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                    const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;              // [2 tiles][2 halves][16 KiB]
  uint8_t* sK = smem + 65536;      // [2 stages][2 halves][16 KiB]
  uint8_t* sV = smem + 131072;     // [2 stages][2 halves][16 KiB]
  __shared__ FwdBarriers bars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bars.q_full, 1);
    mbar_init(&bars.q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.k_full[i], 1);
      mbar_init(&bars.v_full[i], 1);
      mbar_init(&bars.kv_empty[i], 1);
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.p_half[i], 128);
      mbar_init(&bars.p_ready[i], 128);
      mbar_init(&bars.o_full[i], 1);
      mbar_init(&bars.o_empty[i], 128);
    }
    sched_init(bars.sched, 10);  // consumers: TMA warp, MMA warp, 8 softmax warps
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
  }
  if (warp == 1) tmem_alloc<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars.tmem_base;

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // converged warp, one elected lane issues (keeps the TMA operands in uniform registers)
    {
      uint32_t g = 0, it = 0;
      for (uint32_t sk = 0;; ++it) {
        const int u = sched_next(bars.sched, sk);
        if (u < 0) break;
        const FwdUnit U = p.units[u];
        const int ntiles = U.n_rows > kTileRows ? 2 : 1;
        const int division = (U.flags >> 8) & 0xff;
        if (p.rdy && division > 0) {  // persistent launch: the fetches of divisions <= this landed
          if (elect_one()) wait_counter(p.rdy, p.rdy_target[division]);
          __syncwarp();
        }
        mbar_wait(&bars.q_empty, (it & 1) ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&bars.q_full, ntiles * 32768);
          for (int t = 0; t < ntiles; ++t)
            for (int h = 0; h < 2; ++h)
              tma_load_2d(&tm_q, &bars.q_full, sQ + (t * 2 + h) * 16384, 64 * h, U.q_row0 + 128 * t);
        }
        __syncwarp();
        for (int j = 0; j < U.step_count; ++j, ++g) {
          const FwdStep S = p.steps[U.step_begin + j];
          const int st = g & 1;
          mbar_wait(&bars.kv_empty[st], ((g >> 1) & 1) ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&bars.k_full[st], 32768);
            tma_load_2d(&tm_kv, &bars.k_full[st], sK + (st * 2 + 0) * 16384, 0, S.kv_row0);
            tma_load_2d(&tm_kv, &bars.k_full[st], sK + (st * 2 + 1) * 16384, 64, S.kv_row0);
            mbar_arrive_expect_tx(&bars.v_full[st], 32768);
            tma_load_2d(&tm_kv, &bars.v_full[st], sV + (st * 2 + 0) * 16384, 0, S.kv_row0 + p.slot_rows);
            tma_load_2d(&tm_kv, &bars.v_full[st], sV + (st * 2 + 1) * 16384, 64, S.kv_row0 + p.slot_rows);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The converged warp runs the loop and one elected lane issues each batch of
    // tcgen05 instructions (a lane-0-only loop makes ptxas wrap every MMA in an R2UR
    // waterfall loop, which caps the issue rate well below the tensor pipe's).
    {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 128, 0, 0);  // Q K^T : both K-major
      constexpr uint32_t id_o = idesc_bf16_f32(128, 128, 0, 1);  // P V   : V is MN-major
      // descriptor low words (sdesc_lo); stage / k-slice offsets added as (bytes >> 4)
      const uint32_t q_lo = sdesc_lo(smem_u32(sQ), 16), k_lo = sdesc_lo(smem_u32(sK), 16);
      const uint32_t v_lo = sdesc_lo(smem_u32(sV), 16384);
      uint32_t g = 0, it = 0, cnt_p[2] = {0, 0}, cnt_o[2] = {0, 0};
      auto issue_s = [&](int t, int st) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 1024 + (kk & 3) * 2;
            umma_ss_lo(tbase + 128 * t, q_lo + t * 2048 + off, k_lo + st * 2048 + off, id_s, kk > 0);
          }
          umma_commit(&bars.s_full[t]);
        }
        __syncwarp();
      };
      for (uint32_t sk = 0;; ++it) {
        const int u = sched_next(bars.sched, sk);
        if (u < 0) break;
        const FwdUnit U = p.units[u];
        const FwdStep* steps = p.steps + U.step_begin;
        bool has[2] = {false, false};
        int last[2] = {-1, -1};  // each tile's last step: its O is final after that PV
        for (int j = 0; j < U.step_count; ++j) {
          const uint32_t c = steps[j].cls;
          if (cls_of(c, 0)) { has[0] = true; last[0] = j; }
          if (cls_of(c, 1)) { has[1] = true; last[1] = j; }
        }
        int issued[2] = {-1, -1};
        bool first[2] = {true, true};
        mbar_wait(&bars.q_full, it & 1);
        tc_fence_after();
        for (int j = 0; j < U.step_count; ++j, ++g) {
          const int st = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          const uint32_t c = steps[j].cls;
          mbar_wait(&bars.k_full[st], ph);
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (cls_of(c, t) && issued[t] < j) {
              issue_s(t, st);
              issued[t] = j;
            }
          if (j == U.step_count - 1) {  // every S of the unit is issued: Q may be refilled
            if (elect_one()) umma_commit(&bars.q_empty);
            __syncwarp();
          }
          mbar_wait(&bars.v_full[st], ph);
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (!cls_of(c, t)) continue;
            mbar_wait(kSplitP ? &bars.p_half[t] : &bars.p_ready[t], cnt_p[t] & 1);
            tc_fence_after();
            if (first[t]) {
              mbar_wait(&bars.o_empty[t], (cnt_o[t] & 1) ^ 1);
              tc_fence_after();
            }
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < (kSplitP ? 4 : 8); ++kk)
                umma_ts_lo(tbase + 256 + 128 * t, tbase + 128 * t + kk * 8, v_lo + st * 2048 + kk * 128, id_o,
                           (!first[t] || kk > 0) ? 1u : 0u);
            }
            __syncwarp();
            if (kSplitP) {
              mbar_wait(&bars.p_ready[t], cnt_p[t] & 1);
              tc_fence_after();
              if (elect_one()) {
#pragma unroll
                for (int kk = 4; kk < 8; ++kk)
                  umma_ts_lo(tbase + 256 + 128 * t, tbase + 128 * t + kk * 8, v_lo + st * 2048 + kk * 128, id_o, 1u);
              }
              __syncwarp();
            }
            // O_t is final once this tile's last PV retires: signal its epilogue now rather
            // than after the other tile's last PV (which waits for that tile's softmax)
            if (j == last[t]) {
              if (elect_one()) umma_commit(&bars.o_full[t]);
              __syncwarp();
            }
            ++cnt_p[t];
            first[t] = false;
            if (j + 1 < U.step_count && cls_of(steps[j + 1].cls, t)) {
              const uint32_t g2 = g + 1;
              mbar_wait(&bars.k_full[g2 & 1], (g2 >> 1) & 1);
              tc_fence_after();
              issue_s(t, g2 & 1);
              issued[t] = j + 1;
            }
          }
          if (elect_one()) umma_commit(&bars.kv_empty[st]);
          __syncwarp();
        }
        if (elect_one()) {
          // a unit without steps (rows that attend nothing) still took a Q buffer
          if (U.step_count == 0) umma_commit(&bars.q_empty);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (has[t]) ++cnt_o[t];
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ unit scheduler
    if (lane == 0) sched_produce(bars.sched, p.sched, p.sched_base, p.num_units);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    const int t = (warp - 4) >> 2;            // q tile handled by this warpgroup
    const int r = ((warp & 3) << 5) + lane;   // TMEM lane == row within the tile
    const uint32_t lane_addr = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t s_col = 128 * t, o_col = 256 + 128 * t;
    uint32_t cnt_s = 0, cnt_o = 0;
#ifdef DCPX_FWD_PROFILE
    long long fprof[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const long long fprof_t0 = clock64();
#endif
    for (uint32_t sk = 0;;) {
      const int u = sched_next(bars.sched, sk);
      if (u < 0) break;
      const FwdUnit U = p.units[u];
      if (t == 1 && U.n_rows <= kTileRows) continue;
      const FwdStep* steps = p.steps + U.step_begin;
      const bool row_valid = (128 * t + r) < U.n_rows;
      const int64_t q_local = U.q_local0 + 128 * t + r;
      const int64_t orow = (int64_t)U.out_row0 + 128 * t + r;
      __nv_bfloat16* out = p.o_arena + orow * kHeadDim;
      const bool merge = (U.flags & 1) != 0;
      float m_used = -CUDART_INF_F;  // running max, log2 domain (lazily updated)
      float l = 0.f;
      bool has = false;
#ifdef DCPX_FWD_PROFILE
      bool has_prev = false;
#endif
      for (int j = 0; j < U.step_count; ++j) {
        const FwdStep S = steps[j];
        const uint32_t cl = cls_of(S.cls, t);
        if (!cl) continue;
        FWD_T(t0);
        mbar_wait(&bars.s_full[t], cnt_s & 1);
        ++cnt_s;
        tc_fence_after();
        FWD_T(t1);
        uint32_t sraw[128];
#pragma unroll
        for (int c = 0; c < 128; c += 32) tmem_ld32(lane_addr + s_col + c, sraw + c);
        tmem_wait_ld();
        FWD_T(t2);
        float s[128];
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(sraw[c]);
        if (cl == kTilePartial) {
          int lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
          if (row_valid) {
            const ItemMask im = p.items[S.item];
            const int4 rg = __ldg(reinterpret_cast<const int4*>(p.ranges) + im.range_row0 + q_local);
            // intersect with the item's kv tile [0, n_k) (plan.hpp:231-242), then
            // express relative to this 128-column sub-tile
            const int64_t sh = im.kv_shift;
            const int64_t rb0 = imax64((int64_t)rg.x - sh, 0), re0 = imin64((int64_t)rg.y - sh, im.n_k);
            const int64_t rb1 = imax64((int64_t)rg.z - sh, 0), re1 = imin64((int64_t)rg.w - sh, im.n_k);
            lo0 = (int)imax64(rb0 - S.col0, 0);
            hi0 = (int)imin64(re0 - S.col0, 128);
            lo1 = (int)imax64(rb1 - S.col0, 0);
            hi1 = (int)imin64(re1 - S.col0, 128);
          }
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const uint32_t bits = range_bits(lo0 - 32 * w, hi0 - 32 * w) | range_bits(lo1 - 32 * w, hi1 - 32 * w);
#pragma unroll
            for (int c = 0; c < 32; ++c)
              s[32 * w + c] = ((bits >> c) & 1u) ? s[32 * w + c] : -CUDART_INF_F;
          }
        }
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int c = 0; c < 128; ++c) mx = fmaxf(mx, s[c]);
#ifdef DCPX_FWD_PROFILE
        mx = __shfl_sync(0xffffffffu, mx, lane);  // materialise before the timestamp
#endif
        FWD_T(t3);
        const float m_new = mx * p.scale_log2;
        float alpha = 1.f;
        const bool need = m_new > m_used + kRescaleThreshold || (m_used == -CUDART_INF_F && m_new > -CUDART_INF_F);
        if (need) {
          alpha = fast_exp2(m_used - m_new);  // m_used = -inf -> 0
          m_used = m_new;
        }
        if (__any_sync(0xffffffffu, need) && has) {
          // O(prev) is complete: s_full of this step implies the previous PV retired.
#pragma unroll 1
          for (int c = 0; c < 128; c += 32) {
            uint32_t o[32];
            tmem_ld32(lane_addr + o_col + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            tmem_st32(lane_addr + o_col + c, o);
          }
        }
        l *= alpha;
        const float msub = m_used == -CUDART_INF_F ? 0.f : m_used;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            // kSoftExpPairs of every 16 column pairs go to the FMA pipe (MUFU relief)
            const float x0 = fmaf(s[c + 2 * e], p.scale_log2, -msub);
            const float x1 = fmaf(s[c + 2 * e + 1], p.scale_log2, -msub);
            const float p0 = e < kSoftExpPairs ? soft_exp2(x0) : fast_exp2(x0);
            const float p1 = e < kSoftExpPairs ? soft_exp2(x1) : fast_exp2(x1);
            sum += p0 + p1;
            pk[e] = pack_bf16(p0, p1);
          }
          tmem_st16(lane_addr + s_col + (c >> 1), pk);
          if (kSplitP && c == 32) {  // P columns [0, 32) (K-slices 0-3) are in TMEM
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars.p_half[t]);
          }
        }
        l += sum;
        FWD_T(t4);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars.p_ready[t]);
        has = true;
        FWD_T(t5);
        FWD_ACC(0, t0, t1); FWD_ACC(1, t1, t2); FWD_ACC(2, t2, t3); FWD_ACC(3, t3, t4); FWD_ACC(4, t4, t5);
#ifdef DCPX_FWD_PROFILE
        ++fprof[5];
        if (!has_prev) fprof[7] += t1 - t0;
        has_prev = true;
#endif
      }
      FWD_T(te0);
      // ---- epilogue: O / l, LSE, optional merge with the destination's current value.
      // The merge operands (this row's previous O, 256 B, and LSE) are loaded before the wait
      // for the unit's last PV, all 16 vectors at once, so their global-memory latency
      // overlaps it instead of costing four round trips after it.
      float lse_prev = -CUDART_INF_F;
      uint4 prev[16];
      if (merge && U.dep >= 0) {  // persistent launch: the earlier division's unit has stored
        if (lane == 0) wait_stamp(p.unit_done + 2 * U.dep + t, p.epoch);
        __syncwarp();
      }
      if (merge && row_valid) {
        const uint4* src = reinterpret_cast<const uint4*>(out);
#pragma unroll
        for (int k = 0; k < 16; ++k) prev[k] = src[k];
        lse_prev = p.lse_arena[orow];
      }
      const float lse_new = l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994531f : -CUDART_INF_F;
      const float inv_l = l > 0.f ? 1.f / l : 0.f;
      float w_new = 1.f, w_prev = 0.f, lse_out = lse_new;
      if (merge && row_valid) {
        const float mm = fmaxf(lse_new, lse_prev);
        if (mm == -CUDART_INF_F) {
          w_new = 0.f; w_prev = 0.f; lse_out = -CUDART_INF_F;
        } else {
          const float a = __expf(lse_new - mm), b = __expf(lse_prev - mm);
          lse_out = mm + __logf(a + b);
          w_new = a / (a + b);
          w_prev = b / (a + b);
        }
      }
      if (has) {
        mbar_wait(&bars.o_full[t], cnt_o & 1);
        ++cnt_o;
        tc_fence_after();
      }
      const float scale_new = inv_l * w_new;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t oraw[32];
        if (has) {
          tmem_ld32(lane_addr + o_col + 32 * c, oraw);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) oraw[k] = 0u;
        }
        if (row_valid) {
          uint4* dst = reinterpret_cast<uint4*>(out + 32 * c);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float a = __uint_as_float(oraw[k * 8 + 2 * e]) * scale_new;
              float b = __uint_as_float(oraw[k * 8 + 2 * e + 1]) * scale_new;
              if (merge) {
                const uint32_t pv = (&prev[4 * c + k].x)[e];
                const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pv);
                a = fmaf(__bfloat162float(pb.x), w_prev, a);
                b = fmaf(__bfloat162float(pb.y), w_prev, b);
              }
              w[e] = pack_bf16(a, b);
            }
            dst[k] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      if (row_valid) p.lse_arena[orow] = lse_out;
      if (has) {
        tc_fence_before();
        mbar_arrive(&bars.o_empty[t]);
      }
      if (p.unit_done) {  // persistent launch: publish this tile's output (all 128 rows stored)
        named_bar_sync(1 + t, 128);
        if (r == 0) {
          __threadfence();
          st_release_gpu(p.unit_done + 2 * u + t, p.epoch);
          red_release_gpu_add(p.done + ((U.flags >> 8) & 0xff), 1u);
        }
      }
      FWD_T(te1);
      FWD_ACC(6, te0, te1);
#ifdef DCPX_FWD_PROFILE
      ++fprof[8];
#endif
    }
#ifdef DCPX_FWD_PROFILE
    if (blockIdx.x == 0 && (warp == 4 || warp == 8) && lane == 0)
      printf("[fwd prof] warp %d total %lld steps %lld  s_wait %lld (first of unit %lld)  ld %lld  max %lld  exp %lld  "
             "st+arrive %lld  units %lld epilogue %lld\n", warp, clock64() - fprof_t0, fprof[5], fprof[0], fprof[7],
             fprof[1], fprof[2], fprof[3], fprof[4], fprof[8], fprof[6]);
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

void launch_attn_fwd(const CUtensorMap& tm_q, const CUtensorMap& tm_kv, const FwdParams& p,
                     int grid, cudaStream_t stream) {
  // the dynamic shared-memory opt-in is a per-device function attribute
  static uint64_t configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1ull << dev))) {
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    configured |= 1ull << dev;
  }
  attn_fwd_kernel<<<grid, kFwdThreads, kFwdSmem, stream>>>(tm_q, tm_kv, p);
}

void set_watchdog_buffer_fwd(uint32_t* diag) {
  cudaMemcpyToSymbol(g_watchdog_diag, &diag, sizeof(diag));
}

}  // namespace dcpx
