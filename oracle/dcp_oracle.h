/*
 * dcp_oracle.h — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference DCP
 * executor (proj/include/dcp/simexec.hpp) in plain C, FP64.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 * It is the checker, never the thing measured or shipped: the product path
 * (paper_2510_10620_b200/, libdcpx.so) never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself compiled
 * from /root/reference (oracle/_ref/libdcpref.so, built by oracle/Makefile) and
 * against golden vectors committed under tests/golden/ (tests/golden/make_golden.py).
 * LSE and the backward are NOT in the reference: LSE = m + ln(l) of the final
 * accumulator (simexec.hpp:72-73,107-108) is kept through Copy (which zeroes it in
 * the reference, simexec.hpp:358-362) and pinned against a dense restatement; the
 * backward is pinned by finite differences of the forward ("parity unpinned" by
 * the reference).
 */
#ifndef DCP_ORACLE_H_
#define DCP_ORACLE_H_

#include <stdint.h>

#include "../include/dcpx.h"

#ifdef __cplusplus
extern "C" {
#endif

/* exec_attention (simexec.hpp:33-76). q [n_q][D], k, v [n_k][D] row-major; rows
 * [n_q][4] = (b0, e0, b1, e1) relative to the kv tile. Writes out [n_q][D], m, l.
 * Returns 0, or 1 when a range falls outside the kv tile (simexec.hpp:53). */
int orc_exec_attention(const double* q, const double* k, const double* v, int n_q, int n_k,
                       int D, const int32_t* rows, double* out, double* m, double* l);

/* exec_reduction (simexec.hpp:80-111): merges n partials (out_i [rows][D], m_i, l_i)
 * into (out, m, l). out may alias none of the inputs. */
void orc_exec_reduction(int n, const double* const* outs, const double* const* ms,
                        const double* const* ls, int rows, int D, double* out, double* m,
                        double* l);

typedef struct {
  uint64_t total_bytes, total_flops;
  uint64_t per_device_send[64], per_device_recv[64];
  uint64_t comm_bytes[64 * 64 * 8]; /* [stage][src][dst] flattened for R <= 64, stages <= 8 */
  uint64_t comp_flops[8 * 64];      /* [stage][device] */
  int32_t stages, devices;
} orc_report;

/* run (simexec.hpp:207-423) over the flat plan views of include/dcpx.h, numeric FP64.
 * Inputs packed token-major: q [T][H][D], k, v [T][G][D]. Outputs o [T][H][D] and
 * lse [H][T] (natural log; -inf for rows with no attended key). Returns a dcpx_status
 * (DCPX_DEADLOCK / DCPX_TAG_MISMATCH / DCPX_ERROR like the reference's exceptions);
 * err receives a message. numeric = 0 gives the cost-accounting-only mode. */
int orc_run(int nplans, const dcpx_plan_view* plans, const dcpx_graph_view* g,
            const dcpx_mask_view* masks, const double* q, const double* k, const double* v,
            double* o, double* lse, orc_report* rep, int numeric, char* err, int errlen);

/* Dense masked attention (tests/oracle.hpp:80-120) extended with LSE, over the
 * flattened masks: o [T][H][D], lse [H][T]. */
void orc_dense_forward(const dcpx_graph_view* g, const dcpx_mask_view* masks, const double* q,
                       const double* k, const double* v, double* o, double* lse);

/* Dense backward of the same masked attention (no reference):
 * P = softmax(masked s); dV = P^T dO; dP = dO V^T; Delta = rowsum(dO o O);
 * dS = P o (dP - Delta); dQ = dS K / sqrt(D); dK = dS^T Q / sqrt(D); GQA heads of a
 * group summed into dK, dV (types.hpp:259-261). */
void orc_dense_backward(const dcpx_graph_view* g, const dcpx_mask_view* masks, const double* q,
                        const double* k, const double* v, const double* d_o, double* dq,
                        double* dk, double* dv);

/* Item rows as compile_plans derives them (plan.hpp:231-242): mask row of each q
 * token intersected with [kv_begin, kv_end), made relative. rows_out [n_q][4]. */
void orc_item_rows(const dcpx_mask_view* masks, int seq, int64_t q_begin, int64_t q_end,
                   int64_t kv_begin, int64_t kv_end, int32_t* rows_out);

#ifdef __cplusplus
}
#endif

#endif
