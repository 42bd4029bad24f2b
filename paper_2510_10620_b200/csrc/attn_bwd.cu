// attn_bwd.cu — K1b: blockwise masked attention backward for DCP AttentionItems on
// sm_100a (tcgen05 + TMEM + TMA). No reference exists; the math is the
// gradient of exec_attention (simexec.hpp:33-76):
//   P = exp(s - LSE), dV = P^T dO, dP = dO V^T, Delta = rowsum(dO o O),
//   dS = P o (dP - Delta), dQ = scale * dS K, dK = scale * dS^T Q.
//
// Work unit = one 128-row kv sub-tile of one KV slot; it streams every (item, 128-row
// q tile) step of the division that touches it (all heads of the GQA group, all q tiles),
// accumulating dK and dV in TMEM. dQ of each step is reduce-added (fp32) into the
// q slot's dQ accumulator.
//
// CTA = 512 threads, persistent:
//   warp 0      TMA producer: K, V per unit; Q, dO tiles + LSE/Delta rows per step (2 stages)
//   warp 1      TMEM owner + tcgen05.mma issuer
//   warps 2-3   idle (register donors)
//   warps 4-11  compute: warp group c = 0/1 handles q columns [64c, 64c+64) of every kv row
//               (TMEM lane = kv row): P^T -> TMEM, dS^T -> smem (SW128); at the end of a
//               unit group 0 adds dV and group 1 adds dK to the fp32 accumulators.
//   warps 12-15 dQ drain: TMEM -> the step's Q/dO stage buffers (fp32, SW128) -> TMA
//               bulk-tensor reduce-add into the dQ accumulator.
// TMEM: S^T [0,128) (P^T bf16 overwrites [0,64)), dP^T [128,256) (reused for dQ),
//       dV [256,384), dK [384,512).
// Masks: for partial tiles each lane builds 32-bit words "q row -> kv rows of my warp"
// from the q rows' <= 2 attend ranges and transposes them across the warp (5 shuffles),
// giving every kv-row thread a bitmask over its q columns; the element loop is branch-free.
#include <cuda_bf16.h>
#include <math_constants.h>

#include "program.h"
#include "sm100.cuh"

namespace dcpx {

constexpr int kBwdThreads = 512;
// K 32K | V 32K | Q[2] 64K | dO[2] 64K | dS 32K | LSE[2] 1K | Delta[2] 1K | barriers
constexpr int kBwdSmemMain = 224 * 1024;
constexpr int kBwdSmem = kBwdSmemMain + 2048 + 256;

struct BwdBarriers {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[2], q_empty[2];
  uint64_t s_full, p_ready, dq_full, dq_empty, ds_free, acc_full, acc_empty;
  uint32_t tmem_base;
};

// fp32 vector reduce-add into global memory (accumulators are shared with other CTAs
// and with peer devices' gradient returns, so every update is atomic).
__device__ __forceinline__ void red_add_v4(float* dst, const uint32_t* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(__uint_as_float(v[0])),
               "f"(__uint_as_float(v[1])), "f"(__uint_as_float(v[2])), "f"(__uint_as_float(v[3]))
               : "memory");
}

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

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_dq,
                    const BwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem;
  uint8_t* sV = smem + 32768;
  uint8_t* sQ = smem + 65536;     // [2 stages][32 KiB]
  uint8_t* sDO = smem + 131072;   // [2 stages][32 KiB]
  uint8_t* sDS = smem + 196608;   // dS^T [kv rows][q], two q halves of 16 KiB, SW128
  float* sLSE = reinterpret_cast<float*>(smem + kBwdSmemMain);          // [2][128] (log2 units)
  float* sDelta = reinterpret_cast<float*>(smem + kBwdSmemMain + 1024);  // [2][128]
  BwdBarriers& bars = *reinterpret_cast<BwdBarriers*>(smem + kBwdSmemMain + 2048);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 operands need 1 KiB alignment

  if (threadIdx.x == 0) {
    mbar_init(&bars.kv_full, 1);
    mbar_init(&bars.kv_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.q_full[i], 1);
      mbar_init(&bars.q_empty[i], 2);  // MMA commit (dV, dK done) + drain (dQ staged and read)
    }
    mbar_init(&bars.s_full, 1);
    mbar_init(&bars.p_ready, 256);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.dq_empty, 128);
    mbar_init(&bars.ds_free, 1);
    mbar_init(&bars.acc_full, 1);
    mbar_init(&bars.acc_empty, 256);
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_dq);
  }
  if (warp == 1) tmem_alloc<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars.tmem_base;
  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t g = 0, it = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++it) {
        const BwdUnit U = p.units[u];
        mbar_wait(&bars.kv_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(&bars.kv_full, 65536);
        for (int h = 0; h < 2; ++h) {
          tma_load_2d(&tm_kv, &bars.kv_full, sK + h * 16384, 64 * h, U.kv_row0);
          tma_load_2d(&tm_kv, &bars.kv_full, sV + h * 16384, 64 * h, U.kv_row0 + p.slot_rows);
        }
        for (int j = 0; j < U.step_count; ++j, ++g) {
          const BwdStep S = p.steps[U.step_begin + j];
          const int st = g & 1;
          mbar_wait(&bars.q_empty[st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&bars.q_full[st], 65536 + 1024);
          for (int h = 0; h < 2; ++h) {
            tma_load_2d(&tm_q, &bars.q_full[st], sQ + st * 32768 + h * 16384, 64 * h, S.q_row0);
            tma_load_2d(&tm_do, &bars.q_full[st], sDO + st * 32768 + h * 16384, 64 * h, S.q_row0);
          }
          bulk_load(sLSE + st * 128, p.lse2 + S.q_row0, 512, &bars.q_full[st]);
          bulk_load(sDelta + st * 128, p.delta + S.q_row0, 512, &bars.q_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_kmaj = idesc_bf16_f32(128, 128, 0, 0);   // A K-major, B K-major
      const uint32_t id_bmn = idesc_bf16_f32(128, 128, 0, 1);    // A K-major, B MN-major
      const uint32_t id_abmn = idesc_bf16_f32(128, 128, 1, 1);   // A MN-major, B MN-major
      const uint32_t sk = smem_u32(sK), sv = smem_u32(sV), sq = smem_u32(sQ), sdo = smem_u32(sDO),
                     sds = smem_u32(sDS);
      uint32_t g = 0, it = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++it) {
        const BwdUnit U = p.units[u];
        mbar_wait(&bars.kv_full, it & 1);
        tc_fence_after();
        for (int j = 0; j < U.step_count; ++j, ++g) {
          const int st = g & 1;
          mbar_wait(&bars.q_full[st], (g >> 1) & 1);
          tc_fence_after();
          // S^T = K Q^T  -> cols [0,128)
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tbase, sdesc_sw128(sk + off, 16, 1024), sdesc_sw128(sq + st * 32768 + off, 16, 1024),
                    id_kmaj, kk > 0);
          }
          // dP^T = V dO^T -> cols [128,256) once the previous dQ has been drained
          if (g > 0) {
            mbar_wait(&bars.dq_empty, (g - 1) & 1);
            tc_fence_after();
          }
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tbase + 128, sdesc_sw128(sv + off, 16, 1024), sdesc_sw128(sdo + st * 32768 + off, 16, 1024),
                    id_kmaj, kk > 0);
          }
          umma_commit(&bars.s_full);
          mbar_wait(&bars.p_ready, g & 1);
          tc_fence_after();
          if (j == 0) {
            mbar_wait(&bars.acc_empty, (it & 1) ^ 1);
            tc_fence_after();
          }
          // dV += P^T dO   (A = P^T in TMEM, B = dO MN-major)
          for (int kk = 0; kk < 8; ++kk)
            umma_ts(tbase + 256, tbase + kk * 8, sdesc_sw128(sdo + st * 32768 + kk * 2048, 16384, 1024), id_bmn,
                    (j > 0 || kk > 0) ? 1u : 0u);
          // dK += dS^T Q   (A = dS^T K-major in smem, B = Q MN-major)
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tbase + 384, sdesc_sw128(sds + off, 16, 1024),
                    sdesc_sw128(sq + st * 32768 + kk * 2048, 16384, 1024), id_bmn, (j > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&bars.q_empty[st]);
          // dQ = dS K      (A = dS MN-major in smem, B = K MN-major) -> cols [128,256)
          for (int kk = 0; kk < 8; ++kk)
            umma_ss(tbase + 128, sdesc_sw128(sds + kk * 2048, 16384, 1024), sdesc_sw128(sk + kk * 2048, 16384, 1024),
                    id_abmn, kk > 0);
          umma_commit(&bars.dq_full);
          umma_commit(&bars.ds_free);
        }
        umma_commit(&bars.acc_full);
        umma_commit(&bars.kv_empty);
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ compute warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;");
    const int c = (warp - 4) >> 2;                  // q-column half handled by this group
    const int wq = warp & 3;                        // TMEM lane quarter
    const int j = (wq << 5) + lane;                 // kv row (P/dS) / q row (dQ drain)
    const uint32_t lane_addr = tbase + ((uint32_t)(wq * 32) << 16);
    uint32_t g = 0, it = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++it) {
      const BwdUnit U = p.units[u];
      const bool kv_valid = j < U.n_kv;
      // step descriptors are loaded one step ahead so their latency hides behind the work
      BwdStep s_next = p.steps[U.step_begin];
      ItemMask m_next = p.items[s_next.item];
      for (int s = 0; s < U.step_count; ++s, ++g) {
        const BwdStep S = s_next;
        const ItemMask im = m_next;
        if (s + 1 < U.step_count) {
          s_next = p.steps[U.step_begin + s + 1];
          m_next = p.items[s_next.item];
        }
        const int st = g & 1;
        // ---- mask bits over my 64 q columns: mb[h] bit i <-> q column 64c + 32h + i
        uint32_t mb[2];
        if (S.cls == kTilePartial) {
          const int64_t base = im.kv_shift + S.col0 + 32 * wq;  // range coords of my warp's kv row 0
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int qi = 64 * c + 32 * h + lane;           // q row this lane describes
            uint32_t w = 0u;
            if (qi < S.n_q) {
              const int4 rg = __ldg(reinterpret_cast<const int4*>(p.ranges) + im.range_row0 + S.q_local0 + qi);
              w = bits_in((int64_t)rg.x - base, (int64_t)rg.y - base) | bits_in((int64_t)rg.z - base, (int64_t)rg.w - base);
            }
            mb[h] = warp_transpose32(w, lane);
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) mb[h] = bits_in(0, S.n_q - 64 * c - 32 * h);
        }
        if (!kv_valid) mb[0] = mb[1] = 0u;
        mbar_wait(&bars.s_full, g & 1);
        tc_fence_after();
        if (g > 0) mbar_wait(&bars.ds_free, (g - 1) & 1);
        const float4* lse4 = reinterpret_cast<const float4*>(sLSE + st * 128 + 64 * c);
        const float4* dlt4 = reinterpret_cast<const float4*>(sDelta + st * 128 + 64 * c);
        // P^T (bf16) lands in S^T columns [0,64): every S^T column must be read by both
        // groups before either group stores P.
        uint32_t srr[2][32];
        tmem_ld32(lane_addr + 64 * c, srr[0]);
        tmem_ld32(lane_addr + 64 * c + 32, srr[1]);
        tmem_wait_ld();
        named_bar_sync(1, 256);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 64 * c + 32 * h;  // first q column of this chunk
          const uint32_t* sr = srr[h];
          uint32_t dr[32];
          tmem_ld32(lane_addr + 128 + col, dr);
          tmem_wait_ld();
          uint32_t pk[16], dk[16];
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 l4 = lse4[8 * h + e4];
            const float4 d4 = dlt4[8 * h + e4];
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
            const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
            float pv[4], sv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 4 * e4 + e;
              const float pe = fast_exp2(fmaf(__uint_as_float(sr[i]), p.scale_log2, -lv[e]));
              pv[e] = ((mb[h] >> i) & 1u) ? pe : 0.f;
              sv[e] = pv[e] * (__uint_as_float(dr[i]) - dv[e]) * p.scale;
            }
            pk[2 * e4] = pack_bf16(pv[0], pv[1]);
            pk[2 * e4 + 1] = pack_bf16(pv[2], pv[3]);
            dk[2 * e4] = pack_bf16(sv[0], sv[1]);
            dk[2 * e4 + 1] = pack_bf16(sv[2], sv[3]);
          }
          tmem_st16(lane_addr + (col >> 1), pk);
          // dS^T row j, q columns [col, col+32): 4 chunks of 16 B in half c, 128B-swizzled
          uint8_t* row = sDS + c * 16384 + j * 128;
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
        mbar_arrive(&bars.p_ready);
      }
      // ---- unit epilogue: group 0 adds dV [256,384), group 1 adds dK [384,512)
      mbar_wait(&bars.acc_full, it & 1);
      tc_fence_after();
      float* dst = p.dkv_acc + ((int64_t)U.kv_row0 + (c == 0 ? p.slot_rows : 0) + j) * 128;
      const uint32_t col = c == 0 ? 256 : 384;
#pragma unroll 1
      for (int cc = 0; cc < 128; cc += 32) {
        uint32_t r[32];
        tmem_ld32(lane_addr + col + cc, r);
        tmem_wait_ld();
        if (kv_valid) {
#pragma unroll
          for (int e = 0; e < 32; e += 4) red_add_v4(dst + cc + e, r + e);
        }
      }
      tc_fence_before();
      mbar_arrive(&bars.acc_empty);
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ dQ drain warpgroup
    // q row r of each step: dQ (TMEM cols [128,256)) -> four [128 x 32] fp32 chunks,
    // 128B-swizzled, staged in the step's own Q / dO stage buffers (free once dV and dK
    // retired: dq_full is committed after them) -> TMA bulk-tensor reduce-add into the
    // dQ accumulator; the stage is handed back to the producer after TMA has read it.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;");
    const int wq = warp & 3;
    const int r = (wq << 5) + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(wq * 32) << 16);
    uint32_t g = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
      const BwdUnit U = p.units[u];
      for (int s = 0; s < U.step_count; ++s, ++g) {
        const int q_row0 = p.steps[U.step_begin + s].q_row0;
        const int st = g & 1;
        mbar_wait(&bars.dq_full, g & 1);
        tc_fence_after();
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          uint32_t v[32];
          tmem_ld32(lane_addr + 128 + 32 * k, v);
          tmem_wait_ld();
          uint8_t* chunk = (k < 2 ? sQ : sDO) + st * 32768 + (k & 1) * 16384 + r * 128;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            *reinterpret_cast<uint4*>(chunk + ((q4 ^ (r & 7)) << 4)) =
                make_uint4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
        }
        tc_fence_before();
        mbar_arrive(&bars.dq_empty);
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (wq == 0 && lane == 0) {
          if (!(p.debug_flags & 1))
            for (int k = 0; k < 4; ++k)
              tma_reduce_add_2d(&tm_dq, (k < 2 ? sQ : sDO) + st * 32768 + (k & 1) * 16384, 32 * k, q_row0);
          bulk_commit();
          bulk_wait_read<0>();
          mbar_arrive(&bars.q_empty[st]);
        }
      }
    }
    if (wq == 0 && lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

void launch_attn_bwd(const CUtensorMap& tm_q, const CUtensorMap& tm_do, const CUtensorMap& tm_kv,
                     const CUtensorMap& tm_dq, const BwdParams& p, int grid, cudaStream_t stream) {
  // the dynamic shared-memory opt-in is a per-device function attribute
  static uint64_t configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1ull << dev))) {
    cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    configured |= 1ull << dev;
  }
  attn_bwd_kernel<<<grid, kBwdThreads, kBwdSmem, stream>>>(tm_q, tm_do, tm_kv, tm_dq, p);
}

void set_watchdog_buffer_bwd(uint32_t* diag) {
  cudaMemcpyToSymbol(g_watchdog_diag, &diag, sizeof(diag));
}

}  // namespace dcpx
