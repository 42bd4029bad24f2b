/*
 * dcpx.h — C ABI of the B200-native DCP executor.
 *
 * This is the drop-in boundary for the executor half of DCP (arXiv 2510.10620).
 * The reference executes per-device ExecutionPlans with the single-threaded CPU
 * simulator `dcp::run(plans, g, payload, topo, opts) -> SimResult`
 * (reference: proj/include/dcp/simexec.hpp:207-209). This header replaces that
 * call with: create a context, prepare it with flat POD views of the same plans
 * (proj/include/dcp/plan.hpp:37-107) and block graph (proj/include/dcp/blocks.hpp:19-85),
 * load packed bf16 Q/K/V, run forward, run backward.
 *
 * Mapping to the reference interface (each entry point cites what it replaces):
 *   dcpx_create / dcpx_create_rank  -> construction of the per-device slot arenas in
 *                                      run() (simexec.hpp:216-222); one process owning
 *                                      all plan devices (like run) or one rank per GPU.
 *   dcpx_prepare                    -> plan ingestion + the resident-slot setup of run()
 *                                      (simexec.hpp:223-246); also what verify_plans
 *                                      checks statically (plan.hpp:388-475).
 *   dcpx_load_inputs                -> make_payload + resident copies (simexec.hpp:125-146,
 *                                      223-246): packed Q/K/V scattered to resident slots.
 *   dcpx_forward                    -> the lockstep interpreter of run() (simexec.hpp:258-395):
 *                                      Attention (:328-344, exec_attention :33-76),
 *                                      Reduction (:345-354, exec_reduction :80-111),
 *                                      Copy (:355-368), CommLaunch/CommWait (:263-327),
 *                                      deadlock / tag checks (:384-397), output assembly
 *                                      (:403-421), SimReport accounting (:153-162).
 *   dcpx_backward                   -> no reference. Gradients of the same
 *                                      masked blockwise attention under the same plan.
 *   dcpx_last_error                 -> dcp::Error::what() (types.hpp:17-45).
 *
 * Conventions
 *   - No C++ types cross this boundary; all views are caller-owned and borrowed only
 *     for the duration of the call.
 *   - Status codes map 1:1 onto the reference's exception hierarchy (types.hpp:17-45).
 *   - Tensors are device pointers (bf16 unless stated) in the caller's current CUDA
 *     context for the context's device; "host" variants take host pointers.
 *   - Packed token-major layouts: q/o/dq [T_total][H][D], k/v/dk/dv [T_total][G][D],
 *     lse [H][T_total] (fp32, natural log). Sequences are concatenated in batch order.
 *   - Only D = 128 is supported by the sm_100a kernels (north_star: d = 128).
 */
#ifndef DCPX_H_
#define DCPX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: types.hpp:17-45 --------------------------------------------- */
typedef enum {
  DCPX_OK = 0,
  DCPX_ERROR = 1,            /* dcp::Error */
  DCPX_DEADLOCK = 2,         /* dcp::DeadlockError      (simexec.hpp:384-394) */
  DCPX_TAG_MISMATCH = 3,     /* dcp::TagMismatchError   (simexec.hpp:267-273,317,396) */
  DCPX_BUFFER_OVERFLOW = 4,  /* dcp::BufferOverflowError (plan.hpp:368-380) */
  DCPX_INFEASIBLE = 5,       /* dcp::InfeasibleError (caller side: placement) */
  DCPX_CUDA_ERROR = 6,       /* CUDA / NCCL runtime failure */
  DCPX_UNSUPPORTED = 7       /* shape the sm_100a kernels do not handle (e.g. D != 128) */
} dcpx_status;

/* Block exchange between the plan devices of one context: LOCAL = copy kernels reading
 * the sender's slots over NVLink peer memory (default); NCCL = grouped ncclSend/ncclRecv
 * per message (one GPU per plan device). Gradient returns are peer-memory adds in both. */
typedef enum { DCPX_TRANSPORT_LOCAL = 0, DCPX_TRANSPORT_NCCL = 1 } dcpx_transport;

/* ---- block graph view: blocks.hpp:19-85 ---------------------------------------- */
enum { DCPX_KIND_Q = 0, DCPX_KIND_KV = 1, DCPX_KIND_O = 2 }; /* BlockKind, blocks.hpp:8 */

typedef struct {            /* DataBlock, blocks.hpp:19-27 */
  int32_t id, kind, seq, head, tile, _pad;
  int64_t tok_begin, tok_end; /* [start, end) within the sequence */
  uint64_t size_bytes;
} dcpx_data_block;

typedef struct {            /* ComputationBlock, blocks.hpp:29-40 */
  int32_t id, q_block, kv_block, o_block, seq, head, q_tile, kv_tile;
  uint64_t attended_pairs, flops_weight;
} dcpx_comp_block;

typedef struct {            /* BlockGraph + Batch (types.hpp:245-274) */
  int32_t heads, kv_groups, head_dim, bytes_per_element;
  int32_t num_seqs, num_data_blocks, num_comp_blocks, _pad;
  const int64_t* seq_lengths;        /* [num_seqs] */
  const int64_t* block_sizes;        /* [num_seqs]  BlockGraph::block_sizes */
  const dcpx_data_block* data_blocks;/* [num_data_blocks] */
  const dcpx_comp_block* comp_blocks;/* [num_comp_blocks] */
} dcpx_graph_view;

/* Per-sequence attend ranges (AttendRanges, types.hpp:232-243 / masks.hpp:10-67),
 * flattened: token i of sequence s is row seq_offsets[s] + i, four int32
 * (b0, e0, b1, e1) in sequence-local coordinates; an absent range is (0, 0). */
typedef struct {
  const int64_t* seq_offsets; /* [num_seqs + 1] */
  const int32_t* ranges;      /* [seq_offsets[num_seqs]][4] */
} dcpx_mask_view;

/* ---- execution plan view: plan.hpp:37-107 -------------------------------------- */
enum {
  DCPX_OP_ATTENTION = 0,   /* AttentionInstr  plan.hpp:50-52 */
  DCPX_OP_REDUCTION = 1,   /* ReductionInstr  plan.hpp:54-57 */
  DCPX_OP_COPY = 2,        /* CopyInstr       plan.hpp:59-66 */
  DCPX_OP_COMM_LAUNCH = 3, /* CommLaunchInstr plan.hpp:73-78 */
  DCPX_OP_COMM_WAIT = 4    /* CommWaitInstr   plan.hpp:80-82 */
};

typedef struct {           /* AttentionItem, plan.hpp:37-48 */
  int32_t comp_id, q_slot, kv_slot, out_slot, seq, head;
  int64_t q_begin, q_end;   /* q_tokens  */
  int64_t kv_begin, kv_end; /* kv_tokens */
  /* Row ranges (AttentionItem::rows, relative to kv_begin, plan.hpp:231-242).
   * -1: derive them from the mask view (bit-identical to compile_plans);
   * otherwise an offset into dcpx_plan_view.rows, (q_end-q_begin) rows of 4 int32. */
  int64_t rows_offset;
} dcpx_attention_item;

typedef struct { int32_t block, slot; } dcpx_block_slot; /* TransferBlock / ResidentBlock */
typedef struct { int32_t src_slot, dst_slot; } dcpx_copy_item; /* CopyItem */

typedef struct {           /* Instruction, plan.hpp:84-87 */
  int32_t op;              /* DCPX_OP_* */
  int32_t division;        /* Instruction::division */
  int32_t send;            /* CommLaunch: 1 = send, 0 = receive */
  int32_t peer;            /* CommLaunch: peer device */
  int32_t dst;             /* Reduction: destination slot */
  int32_t count;           /* items / srcs / copy items / blocks */
  int64_t offset;          /* first element in the op's pool below */
  const char* tag;         /* CommLaunch / CommWait tag (NUL-terminated) */
} dcpx_instruction;

typedef struct {           /* ExecutionPlan, plan.hpp:101-107 */
  int32_t version, device, divisions, _pad;
  int32_t capacity[3];     /* BufferLayout::capacity, indexed by kind */
  int32_t n_resident_q, n_resident_kv, n_resident_o;
  const dcpx_block_slot* resident_q;
  const dcpx_block_slot* resident_kv;
  const dcpx_block_slot* resident_o;
  int32_t n_instructions, _pad2;
  const dcpx_instruction* instructions;
  const dcpx_attention_item* items;  /* pool for DCPX_OP_ATTENTION */
  const int32_t* srcs;               /* pool for DCPX_OP_REDUCTION */
  const dcpx_copy_item* copies;      /* pool for DCPX_OP_COPY */
  const dcpx_block_slot* blocks;     /* pool for DCPX_OP_COMM_LAUNCH */
  const int32_t* rows;               /* optional explicit item rows, [n][4] */
} dcpx_plan_view;

/* ---- report: SimReport, simexec.hpp:153-162 ------------------------------------ */
typedef struct {
  int32_t devices, stages;           /* stages = divisions + 1 (stage T = output stage) */
  uint64_t total_bytes;              /* planned bytes moved (SimReport::total_bytes) */
  uint64_t total_flops;              /* 4 * pairs * D summed over executed items */
  uint64_t per_device_send[64];
  uint64_t per_device_recv[64];
  uint64_t wire_bytes;               /* bytes actually moved incl. fp32 LSE/Delta sidecars */
  double makespan;                   /* modeled, detail::cost_from_tables (schedule.hpp:217-236) */
  double device_ms;                  /* measured device time of the last call (max over devices) */
  int32_t kernel_launches;           /* executor kernels launched by the last call */
  int32_t attn_launches;             /* attention kernel (K1 / K1b) launches of the last call */
  double attn_ms;                    /* max over devices of the summed device time of those launches */
  double attn_ms_sum;                /* the same summed over devices (GPU-time spent in the kernel) */
  /* bytes the transfers of the call actually move per device (wire_bytes split by sender /
   * receiver): forward O transfers carry the fp32 LSE (4 B/row); backward Q fetches carry
   * Q + dO + fp32 LSE and Delta (8 B/row); gradient returns are fp32 (2x the planned bytes) */
  uint64_t wire_per_device_send[64];
  uint64_t wire_per_device_recv[64];
  int32_t units;                     /* attention work units of the call (K1 FwdUnit / K1b BwdUnit) */
  int32_t windowed;                  /* backward: attention instructions with q-windowed units */
} dcpx_report;

typedef struct dcpx_ctx dcpx_ctx;

/* One process executes all `ndev` plan devices; plan device d runs on CUDA device
 * cuda_ordinals[d] (several plan devices may share one GPU). Transfers run on per-device
 * comm streams: LOCAL = copy kernels reading the sender's slots over NVLink peer memory;
 * NCCL = ncclSend/ncclRecv groups (needs one distinct GPU per plan device).
 *
 * Stream contract: every load_inputs / forward / backward call is ordered after the work
 * already enqueued on the caller's stream of each plan device (by default the legacy
 * default stream; see dcpx_set_streams), and that stream waits for the call's device work,
 * so device inputs produced and outputs consumed on the caller's stream need no host
 * synchronisation. Host buffers (the _host calls) are valid after dcpx_synchronize. */
dcpx_status dcpx_create(int ndev, const int* cuda_ordinals, dcpx_transport transport,
                        dcpx_ctx** out);

/* One plan device per process (rank == plan device) on CUDA device cuda_ordinal: the
 * one-process-per-GPU deployment. Every rank prepares with ALL `world` plans (the
 * receiver of a transfer needs the sender's slot layout), then exchanges its arena
 * handles with the others:
 *     dcpx_create_rank(rank, world, ordinal, &ctx); dcpx_prepare(ctx, world, plans, ...);
 *     dcpx_rank_export(ctx, blob, cap, &size);      -> all-gather the blobs (any channel,
 *     dcpx_rank_connect(ctx, all_blobs, size);         e.g. torch.distributed), rank order
 * Transfers are then pulls over NVLink from the peers' CUDA-IPC-mapped arenas; ordering
 * across processes is by device-side epoch flags (no host round trip, no collective).
 * Every rank must issue the same sequence of load_inputs / forward / backward calls.
 * The I/O calls use this rank's buffers only (the _dev variants read entry [rank]). */
dcpx_status dcpx_create_rank(int rank, int world, int cuda_ordinal, dcpx_ctx** out);

/* Writes this rank's handle blob (after dcpx_prepare) into buf; *size = its length. With
 * cap too small nothing is written and *size tells the length needed. */
dcpx_status dcpx_rank_export(dcpx_ctx* ctx, void* buf, int64_t cap, int64_t* size);

/* Maps the peers' arenas; blobs = world blobs of blob_size bytes each, in rank order
 * (this rank's own entry is ignored). Required after every dcpx_prepare. */
dcpx_status dcpx_rank_connect(dcpx_ctx* ctx, const void* blobs, int64_t blob_size);

/* Ingests the plans: all ndev plans in device order (also per rank). Validates
 * shapes, slots and tag pairing, sizes the slot arenas from BufferLayout::capacity,
 * and compiles the instruction stream into the device program. */
dcpx_status dcpx_prepare(dcpx_ctx* ctx, int nplans, const dcpx_plan_view* plans,
                         const dcpx_graph_view* graph, const dcpx_mask_view* masks);

/* Packed bf16 inputs on the context's device(s): q [T][H][D], k, v [T][G][D].
 * In LOCAL mode with several GPUs, every device reads its resident rows from this one
 * buffer (peer-to-peer when it lives on another GPU; see dcpx_load_inputs_dev for the
 * distributed layout). Scatters rows into the resident slots. */
dcpx_status dcpx_load_inputs(dcpx_ctx* ctx, const void* q, const void* k, const void* v);
/* Same with host (pinned or pageable) pointers; host->device copies are inside.
 * Asynchronous: returns once the upload is enqueued (double-buffered device staging);
 * the host buffers must stay unchanged until the following dcpx_synchronize. */
dcpx_status dcpx_load_inputs_host(dcpx_ctx* ctx, const void* q, const void* k, const void* v);

/* Executes the plan forward. o_out [T][H][D] bf16 and lse_out [H][T] fp32 (may be
 * NULL) receive the rows owned by this context's device(s); other rows untouched. */
dcpx_status dcpx_forward(dcpx_ctx* ctx, void* o_out, float* lse_out, dcpx_report* rep);
dcpx_status dcpx_forward_host(dcpx_ctx* ctx, void* o_out, float* lse_out, dcpx_report* rep);

/* Executes the backward of the last forward. d_o [T][H][D] bf16 in (device memory, 16-byte
 * aligned: rows are read as 16-byte vectors; DCPX_ERROR otherwise); dq [T][H][D],
 * dk, dv [T][G][D] bf16 out (owned rows). */
dcpx_status dcpx_backward(dcpx_ctx* ctx, const void* d_o, void* dq, void* dk, void* dv,
                          dcpx_report* rep);
/* Host-buffer backward, asynchronous like dcpx_load_inputs_host: dq/dk/dv are valid after
 * the next dcpx_synchronize (uploads and downloads run on their own streams, so
 * consecutive steps overlap their PCIe traffic with compute). dcpx_forward_host is
 * asynchronous the same way: o_out / lse_out are valid after dcpx_synchronize. */
dcpx_status dcpx_backward_host(dcpx_ctx* ctx, const void* d_o, void* dq, void* dk, void* dv,
                               dcpx_report* rep);

/* Distributed layout (no reference counterpart: the reference's payload is one host
 * object). Entry d of every array is a packed buffer of the single-buffer calls' shape in
 * plan device d's own memory; device d reads only the input rows of the blocks resident
 * on it and writes only the output rows it owns, so no input or output crosses NVLink.
 * This is the layout a training step has, where each GPU produced its own tokens' Q/K/V.
 * Output arrays (or their entries) may be NULL to skip that output. */
dcpx_status dcpx_load_inputs_dev(dcpx_ctx* ctx, const void* const* q, const void* const* k,
                                 const void* const* v);
dcpx_status dcpx_forward_dev(dcpx_ctx* ctx, void* const* o_out, float* const* lse_out, dcpx_report* rep);
dcpx_status dcpx_backward_dev(dcpx_ctx* ctx, const void* const* d_o, void* const* dq, void* const* dk,
                              void* const* dv, dcpx_report* rep);

/* Synchronises all streams of the context. */
dcpx_status dcpx_synchronize(dcpx_ctx* ctx);

/* The caller's CUDA stream (cudaStream_t) on each of the n = ndev plan devices (per-rank
 * mode: n = world, only entry [rank] is used); NULL entries select the legacy default
 * stream. Applies to the following calls (stream contract above). */
dcpx_status dcpx_set_streams(dcpx_ctx* ctx, int n, void* const* streams);

/* Host-only plan check (no context, no GPU): ingests the views and runs the static checks
 * of verify_plans (plan.hpp:388-475) plus the lockstep replay of run() (deadlock and tag
 * errors, simexec.hpp:375-397). Returns the status the executor's prepare would raise for
 * these plans; err (may be NULL) receives the message, NUL-terminated, truncated to cap. */
dcpx_status dcpx_check_plans(int nplans, const dcpx_plan_view* plans, const dcpx_graph_view* graph,
                             const dcpx_mask_view* masks, char* err, int64_t cap);

/* GPU time of the attention kernel launches (K1 / K1b) recorded since the last read with
 * option "kernel_timing" = 2 (CUDA events around each launch on its stream, accumulated
 * without blocking the host): ms[0] / ms[1] = forward / backward summed over this context's
 * devices, ms[2] / ms[3] = the same, max over devices; launches[0..1] = launch counts.
 * Synchronises on those events, then resets the accumulation. */
dcpx_status dcpx_kernel_times(dcpx_ctx* ctx, double* ms, int32_t* launches);

/* Test / introspection hooks (not part of the reference surface). */
/* Device pointers of the slot arenas of plan device `dev`: kind 0 Q, 1 KV, 2 O, 3 LSE. */
dcpx_status dcpx_debug_arena(dcpx_ctx* ctx, int dev, int kind, void** ptr, int64_t* slot_rows);
/* Executor options: "fuse_reductions", "remap_copies", "timing" (report device_ms; blocks
 * the host at the end of each call; default off), "kernel_timing" (1: per-call attention
 * kernel times in the report, blocking; 2: deferred, see dcpx_kernel_times), "trace", "sm_transfers",
 * "sm_reserve" (SMs an attention launch leaves to the comm stream's copy kernels; default -1:
 * 4 on launches a fetch overlaps in multi-device plans, 0 otherwise; >= 0: that many on every
 * launch), "bwd_order", "bwd_window", "bwd_window_min_steps", "bwd_merge_heads",
 * "persistent" (1: one forward launch per device for all divisions, ordered on the device;
 * default 0), "aux_zero" (1, default: the gradient accumulators are re-zeroed on an aux
 * stream after each backward; 0: at the start of the next one).
 * The executor overlaps a compute and a comm stream per device; set
 * CUDA_DEVICE_MAX_CONNECTIONS=32 (or more) before the process creates its CUDA context so
 * they do not share a hardware work queue (the Python package does this on import). */
dcpx_status dcpx_set_option(dcpx_ctx* ctx, const char* key, int64_t value);

/* Op trace of the last forward/backward (option "trace"): rows of 7 doubles
 * (plan device, instruction, op kind, division, pass 0 fwd / 1 bwd, start ms, end ms),
 * times relative to the call's start on that device. Returns the number of rows. */
int dcpx_trace(dcpx_ctx* ctx, double* rows, int max_rows);
const char* dcpx_last_error(dcpx_ctx* ctx);
const char* dcpx_version(void);
void dcpx_destroy(dcpx_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* DCPX_H_ */
