// program.h — device-side work descriptors shared by the host compiler (executor.cu)
// and the kernels. Everything here is POD so it can be memcpy'd to the device.
//
// Slot arenas (per plan device, HBM):
//   Q  arena : [cap_q ][slot_rows][128] bf16       one query head's tile per slot
//   KV arena : [cap_kv][2][slot_rows][128] bf16    K tile then V tile of one kv group
//   O  arena : [cap_o ][slot_rows][128] bf16       normalised partial / final output
//   LSE arena: [cap_o ][slot_rows] fp32            natural-log LSE of each O row
// Backward-only arenas mirror Q (dO bf16, LSE/Delta fp32, dQ fp32 accumulators) and
// KV (dK/dV fp32 accumulators). slot_rows = block size rounded up to 128.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace dcpx {

constexpr int kHeadDim = 128;
constexpr int kTileRows = 128;
constexpr int kBwdQRows = 64;  // q rows per backward step

// Mask classification of one (q tile, kv sub-tile) pair, 2 bits per q tile.
enum : uint32_t { kTileEmpty = 0, kTilePartial = 1, kTileFull = 2 };

// Attention item mask data: where the q rows' attend ranges live in the device
// `ranges` array and how to make them relative to the item's kv tile.
struct ItemMask {
  int64_t range_row0;  // ranges row of the item's q row 0
  int64_t kv_shift;    // subtracted from range values -> kv-tile-relative
  int32_t n_k;         // kv rows of the item's kv block
  int32_t _pad;
};

// One forward work unit: up to two 128-row q tiles of one output group (all items of
// a fused attention+reduction group share the same Q block), iterating over a list
// of kv sub-tile steps with a single online softmax.
struct FwdUnit {
  int32_t q_row0;      // Q arena row of q tile 0
  int32_t n_rows;      // valid q rows in this unit (1..256)
  int32_t step_begin;  // first FwdStep
  int32_t step_count;
  int32_t out_row0;    // O/LSE arena row of q tile 0 (destination slot)
  int32_t flags;       // bit0: merge with the destination's current (O, LSE);
                       // bits 8-15: division (persistent cross-division launch)
  int32_t q_local0;    // q row index (within the item) of q tile 0
  int32_t dep;         // persistent launch: the unit of an earlier division whose output this
                       // unit merges with (its epilogue waits for that unit's), else -1
};

struct FwdStep {
  int32_t kv_row0;  // KV arena row of the K sub-tile (V at kv_row0 + slot_rows)
  int32_t col0;     // kv-tile-relative index of column 0 (= 128 * kv_sub)
  int32_t item;     // ItemMask index
  uint32_t cls;     // bits [1:0] tile 0 class, [3:2] tile 1 class
};

// Unfused reduction (exec_reduction, simexec.hpp:80-111) of `n_src` O slots into dst.
struct MergeJob {
  int32_t dst_row0;   // O/LSE arena row of the destination slot
  int32_t n_rows;
  int32_t src_begin;  // into the src-row array (arena rows of each source slot)
  int32_t n_src;
};

// Row-block copy between arenas (scatter / gather / copy / transfers).
struct CopySeg {
  const void* src;
  void* dst;
  int64_t bytes;  // multiple of 16
};

// One backward work unit: a 128-row kv sub-tile of one KV slot, streaming 64-row q tiles
// of the items of the division that read it.
struct BwdUnit {
  int32_t kv_row0;  // KV arena row of the K sub-tile (V and the dV accumulator at + slot_rows)
  int32_t n_kv;     // valid kv rows (1..128)
  int32_t step_begin;
  int32_t step_count;
};

struct BwdStep {
  int32_t q_row0;    // Q / dO / LSE / Delta / dQ-accumulator row of this 64-row q tile
  int32_t n_q;       // valid q rows (1..64)
  int32_t item;      // ItemMask index
  int32_t q_local0;  // q row index within the item of tile row 0
  int32_t col0;      // kv-tile-relative index of the unit's kv row 0
  uint32_t cls;      // kTileEmpty / kTilePartial / kTileFull
};

struct BwdParams {
  const BwdUnit* units;
  const BwdStep* steps;
  const ItemMask* items;
  const int32_t* ranges;
  const float* lse2;   // -LSE * log2(e) per Q-arena row (negated for the packed FMA)
  const float* delta;  // -rowsum(dO o O) * scale per Q-arena row
  float* dq_acc;       // [Q-arena rows][128] fp32
  float* dkv_acc;      // [KV-arena rows][128] fp32
  int32_t num_units;
  int32_t slot_rows;
  float scale_log2;
  float scale;
  uint32_t* sched;      // dynamic-scheduler counter of the device (see sched_produce)
  uint32_t sched_base;  // its value at this launch
  int32_t _pad0;
};

struct FwdParams {
  const FwdUnit* units;
  const FwdStep* steps;
  const ItemMask* items;
  const int32_t* ranges;  // [rows][4] attend ranges (b0, e0, b1, e1)
  __nv_bfloat16* o_arena;
  float* lse_arena;
  int32_t num_units;
  int32_t slot_rows;
  float scale_log2;  // log2(e) / sqrt(D)
  uint32_t sched_base;  // dynamic-scheduler counter value at this launch
  uint32_t* sched;      // the device's scheduler counter (see sched_produce)
  // Persistent cross-division launch (all divisions' units in one launch; null otherwise):
  // a unit of division t > 0 starts loading once *rdy >= rdy_target[t] (every fetch of the
  // divisions <= t landed: each transfer adds 1 on the comm stream); each (unit, tile) epilogue
  // publishes unit_done[2 u + tile] = epoch and adds 1 to done[division] (the comm stream
  // waits on done before a receive overwrites slots freed by earlier divisions).
  uint32_t* rdy;
  const uint32_t* rdy_target;
  uint32_t* done;
  uint32_t* unit_done;
  uint32_t epoch;
  int32_t _pad;
};

}  // namespace dcpx
