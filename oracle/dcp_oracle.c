/*
 * dcp_oracle.c — TEST INFRASTRUCTURE ONLY (see dcp_oracle.h). Plain-C, FP64
 * restatement of the reference executor, proj/include/dcp/simexec.hpp, plus a dense
 * forward/backward. Each function cites the reference lines it restates.
 */
#include "dcp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NEG_INF (-INFINITY)

/* ---- exec_attention: simexec.hpp:33-76 ------------------------------------------- */
int orc_exec_attention(const double* q, const double* k, const double* v, int n_q, int n_k,
                       int D, const int32_t* rows, double* out, double* m_out, double* l_out) {
  const double scale = 1.0 / sqrt((double)D); /* :40 */
  double* scores = (double*)malloc(sizeof(double) * (size_t)(n_k > 0 ? n_k : 1));
  int bad = 0;
  memset(out, 0, sizeof(double) * (size_t)n_q * (size_t)D); /* :43 zero rows */
  for (int i = 0; i < n_q; ++i) {
    const int32_t* rr = rows + 4 * (size_t)i;
    double m = NEG_INF; /* :50 */
    for (int ri = 0; ri < 2; ++ri) {
      for (int32_t j = rr[2 * ri]; j < rr[2 * ri + 1]; ++j) { /* :51-60 */
        if (j < 0 || j >= n_k) { bad = 1; continue; }          /* :53 */
        double s = 0;
        for (int d = 0; d < D; ++d) s += q[(size_t)i * D + d] * k[(size_t)j * D + d];
        s *= scale;
        scores[j] = s;
        if (s > m) m = s;
      }
    }
    if (!isfinite(m)) { m_out[i] = NEG_INF; l_out[i] = 0.0; continue; } /* :61 */
    double l = 0;
    for (int ri = 0; ri < 2; ++ri) /* :62-65 */
      for (int32_t j = rr[2 * ri]; j < rr[2 * ri + 1]; ++j)
        if (j >= 0 && j < n_k) l += exp(scores[j] - m);
    for (int ri = 0; ri < 2; ++ri) { /* :66-71 */
      for (int32_t j = rr[2 * ri]; j < rr[2 * ri + 1]; ++j) {
        if (j < 0 || j >= n_k) continue;
        const double w = exp(scores[j] - m) / l;
        for (int d = 0; d < D; ++d) out[(size_t)i * D + d] += w * v[(size_t)j * D + d];
      }
    }
    m_out[i] = m; /* :72-73 */
    l_out[i] = l;
  }
  free(scores);
  return bad;
}

/* ---- exec_reduction: simexec.hpp:80-111 ------------------------------------------ */
void orc_exec_reduction(int n, const double* const* outs, const double* const* ms,
                        const double* const* ls, int rows, int D, double* out, double* m_out,
                        double* l_out) {
  memset(out, 0, sizeof(double) * (size_t)rows * (size_t)D);
  for (int i = 0; i < rows; ++i) {
    double mstar = NEG_INF; /* :94-96 */
    for (int p = 0; p < n; ++p)
      if (ls[p][i] > 0 && ms[p][i] > mstar) mstar = ms[p][i];
    if (!isfinite(mstar)) { m_out[i] = NEG_INF; l_out[i] = 0.0; continue; } /* :97 */
    double lstar = 0; /* :98-101 */
    for (int p = 0; p < n; ++p)
      if (ls[p][i] > 0) lstar += ls[p][i] * exp(ms[p][i] - mstar);
    for (int p = 0; p < n; ++p) { /* :102-106 */
      if (ls[p][i] <= 0) continue;
      const double w = ls[p][i] * exp(ms[p][i] - mstar) / lstar;
      for (int d = 0; d < D; ++d) out[(size_t)i * D + d] += w * outs[p][(size_t)i * D + d];
    }
    m_out[i] = mstar; /* :107-108 */
    l_out[i] = lstar;
  }
}

/* ---- item rows: plan.hpp:231-242 -------------------------------------------------- */
void orc_item_rows(const dcpx_mask_view* masks, int seq, int64_t q_begin, int64_t q_end,
                   int64_t kv_begin, int64_t kv_end, int32_t* rows_out) {
  const int64_t base = masks->seq_offsets[seq];
  for (int64_t i = q_begin; i < q_end; ++i) {
    const int32_t* r = masks->ranges + 4 * (size_t)(base + i);
    int32_t* o = rows_out + 4 * (size_t)(i - q_begin);
    int cnt = 0;
    o[0] = o[1] = o[2] = o[3] = 0;
    for (int ri = 0; ri < 2; ++ri) {
      int64_t b = r[2 * ri], e = r[2 * ri + 1];
      if (e <= b) continue;
      /* intersect (types.hpp:186-190) */
      int64_t ib = b > kv_begin ? b : kv_begin, ie = e < kv_end ? e : kv_end;
      if (ie <= ib) continue;
      /* TokenRanges::push (types.hpp:198-208): merge with the previous range when touching */
      int32_t rb = (int32_t)(ib - kv_begin), re = (int32_t)(ie - kv_begin);
      if (cnt > 0 && rb <= o[2 * (cnt - 1) + 1]) {
        if (re > o[2 * (cnt - 1) + 1]) o[2 * (cnt - 1) + 1] = re;
        continue;
      }
      o[2 * cnt] = rb;
      o[2 * cnt + 1] = re;
      ++cnt;
    }
  }
}

/* ---- run: simexec.hpp:207-423 ----------------------------------------------------- */
typedef struct {
  int rows;
  double* a;        /* [rows][D] */
} mat_t;

typedef struct {
  int rows;
  double *out, *m, *l;
} part_t;

typedef struct {
  const dcpx_plan_view* plan;
  size_t pc;
  mat_t* q;         /* [cap_q] */
  mat_t* k;         /* [cap_kv] */
  mat_t* v;
  part_t* o;        /* [cap_o] */
  /* posted receives: tag -> slots */
  int n_posted;
  const char* posted_tag[512];
  const dcpx_block_slot* posted_blocks[512];
  int posted_count[512];
} simdev_t;

typedef struct {
  const char* tag;
  int src, dst, division, nblocks;
  const dcpx_block_slot* blocks; /* sender's (block, slot) list */
  mat_t* q; mat_t* k; mat_t* v; part_t* o; /* snapshot payloads per block */
  int live;
} msg_t;

static void mat_set(mat_t* m, int rows, int D, const double* src) {
  free(m->a);
  m->rows = rows;
  m->a = (double*)malloc(sizeof(double) * (size_t)rows * (size_t)D + 8);
  if (src) memcpy(m->a, src, sizeof(double) * (size_t)rows * (size_t)D);
}

static void part_alloc(part_t* p, int rows, int D) {
  free(p->out); free(p->m); free(p->l);
  p->rows = rows;
  p->out = (double*)calloc((size_t)rows * (size_t)D + 1, sizeof(double));
  p->m = (double*)malloc(sizeof(double) * (size_t)rows + 8);
  p->l = (double*)calloc((size_t)rows + 1, sizeof(double));
  for (int i = 0; i < rows; ++i) p->m[i] = NEG_INF;
}

static void part_copy(part_t* dst, const part_t* src, int D) {
  part_alloc(dst, src->rows, D);
  memcpy(dst->out, src->out, sizeof(double) * (size_t)src->rows * (size_t)D);
  memcpy(dst->m, src->m, sizeof(double) * (size_t)src->rows);
  memcpy(dst->l, src->l, sizeof(double) * (size_t)src->rows);
}

#define ERR(code, ...)                                  \
  do {                                                  \
    if (err) snprintf(err, (size_t)errlen, __VA_ARGS__); \
    status = (code);                                    \
    goto done;                                          \
  } while (0)

int orc_run(int R, const dcpx_plan_view* plans, const dcpx_graph_view* g,
            const dcpx_mask_view* masks, const double* q, const double* k, const double* v,
            double* o, double* lse, orc_report* rep, int numeric, char* err, int errlen) {
  const int D = g->head_dim, H = g->heads, G = g->kv_groups;
  const int T = R > 0 ? plans[0].divisions : 0;
  const int64_t TT = masks->seq_offsets[g->num_seqs];
  int status = DCPX_OK;
  simdev_t* dev = (simdev_t*)calloc((size_t)R, sizeof(simdev_t));
  int nmsg_cap = 4096, nmsg = 0;
  msg_t* inbox = (msg_t*)calloc((size_t)nmsg_cap, sizeof(msg_t));
  if (R > 64 || T + 1 > 8) { if (err) snprintf(err, (size_t)errlen, "oracle limits"); free(dev); free(inbox); return DCPX_ERROR; }
  memset(rep, 0, sizeof(*rep));
  rep->stages = T + 1;
  rep->devices = R;

  /* slot arenas sized from capacity (:216-222); residents copied in (:223-246) */
  for (int d = 0; d < R; ++d) {
    simdev_t* sd = &dev[d];
    sd->plan = &plans[d];
    sd->q = (mat_t*)calloc((size_t)plans[d].capacity[0] + 1, sizeof(mat_t));
    sd->k = (mat_t*)calloc((size_t)plans[d].capacity[1] + 1, sizeof(mat_t));
    sd->v = (mat_t*)calloc((size_t)plans[d].capacity[1] + 1, sizeof(mat_t));
    sd->o = (part_t*)calloc((size_t)plans[d].capacity[2] + 1, sizeof(part_t));
    if (!numeric) continue;
    for (int i = 0; i < plans[d].n_resident_q; ++i) {
      const dcpx_data_block* db = &g->data_blocks[plans[d].resident_q[i].block];
      const int rows = (int)(db->tok_end - db->tok_begin);
      mat_t* m = &sd->q[plans[d].resident_q[i].slot];
      mat_set(m, rows, D, NULL);
      for (int r = 0; r < rows; ++r) {
        const int64_t t = masks->seq_offsets[db->seq] + db->tok_begin + r;
        memcpy(m->a + (size_t)r * D, q + ((size_t)t * H + db->head) * D, sizeof(double) * D);
      }
    }
    for (int i = 0; i < plans[d].n_resident_kv; ++i) {
      const dcpx_data_block* db = &g->data_blocks[plans[d].resident_kv[i].block];
      const int rows = (int)(db->tok_end - db->tok_begin);
      mat_t* mk = &sd->k[plans[d].resident_kv[i].slot];
      mat_t* mv = &sd->v[plans[d].resident_kv[i].slot];
      mat_set(mk, rows, D, NULL);
      mat_set(mv, rows, D, NULL);
      for (int r = 0; r < rows; ++r) {
        const int64_t t = masks->seq_offsets[db->seq] + db->tok_begin + r;
        memcpy(mk->a + (size_t)r * D, k + ((size_t)t * G + db->head) * D, sizeof(double) * D);
        memcpy(mv->a + (size_t)r * D, v + ((size_t)t * G + db->head) * D, sizeof(double) * D);
      }
    }
  }

  /* lockstep rounds (:375-395) */
  for (;;) {
    int all_done = 1, any_progress = 0;
    for (int d = 0; d < R; ++d) {
      simdev_t* sd = &dev[d];
      const dcpx_plan_view* pl = sd->plan;
      if (sd->pc >= (size_t)pl->n_instructions) continue;
      all_done = 0;
      while (sd->pc < (size_t)pl->n_instructions) { /* step (:258-372) */
        const dcpx_instruction* ins = &pl->instructions[sd->pc];
        if (ins->op == DCPX_OP_COMM_WAIT) { /* :263-293 */
          int mi = -1;
          for (int x = 0; x < nmsg; ++x)
            if (inbox[x].live && strcmp(inbox[x].tag, ins->tag) == 0) { mi = x; break; }
          if (mi < 0) break; /* blocked */
          msg_t* msg = &inbox[mi];
          if (msg->dst != d) ERR(DCPX_TAG_MISMATCH, "message %s delivered to wrong device", ins->tag);
          int pi = -1;
          for (int x = 0; x < sd->n_posted; ++x)
            if (sd->posted_tag[x] && strcmp(sd->posted_tag[x], ins->tag) == 0) { pi = x; break; }
          if (pi < 0) ERR(DCPX_TAG_MISMATCH, "device %d waits on %s without a posted receive", d, ins->tag);
          if (numeric) {
            for (int b = 0; b < msg->nblocks && b < sd->posted_count[pi]; ++b) {
              const int slot = sd->posted_blocks[pi][b].slot;
              const int kind = g->data_blocks[msg->blocks[b].block].kind;
              if (kind == DCPX_KIND_Q) { free(sd->q[slot].a); sd->q[slot] = msg->q[b]; msg->q[b].a = NULL; }
              else if (kind == DCPX_KIND_KV) {
                free(sd->k[slot].a); free(sd->v[slot].a);
                sd->k[slot] = msg->k[b]; sd->v[slot] = msg->v[b];
                msg->k[b].a = NULL; msg->v[b].a = NULL;
              } else { part_copy(&sd->o[slot], &msg->o[b], D); }
            }
          }
          for (int b = 0; b < msg->nblocks; ++b) {
            free(msg->q[b].a); free(msg->k[b].a); free(msg->v[b].a);
            free(msg->o[b].out); free(msg->o[b].m); free(msg->o[b].l);
          }
          free(msg->q); free(msg->k); free(msg->v); free(msg->o);
          msg->live = 0;
          sd->posted_tag[pi] = NULL;
          ++sd->pc; any_progress = 1;
          continue;
        }
        if (ins->op == DCPX_OP_COMM_LAUNCH) { /* :294-327 */
          if (ins->send) {
            for (int x = 0; x < nmsg; ++x)
              if (inbox[x].live && strcmp(inbox[x].tag, ins->tag) == 0)
                ERR(DCPX_TAG_MISMATCH, "duplicate message tag %s", ins->tag);
            if (nmsg == nmsg_cap) { nmsg_cap *= 2; inbox = (msg_t*)realloc(inbox, sizeof(msg_t) * (size_t)nmsg_cap); }
            msg_t* msg = &inbox[nmsg++];
            memset(msg, 0, sizeof(*msg));
            msg->tag = ins->tag; msg->src = d; msg->dst = ins->peer; msg->division = ins->division;
            msg->nblocks = ins->count; msg->blocks = pl->blocks + ins->offset; msg->live = 1;
            msg->q = (mat_t*)calloc((size_t)ins->count + 1, sizeof(mat_t));
            msg->k = (mat_t*)calloc((size_t)ins->count + 1, sizeof(mat_t));
            msg->v = (mat_t*)calloc((size_t)ins->count + 1, sizeof(mat_t));
            msg->o = (part_t*)calloc((size_t)ins->count + 1, sizeof(part_t));
            uint64_t bytes = 0;
            for (int b = 0; b < ins->count; ++b) {
              const dcpx_block_slot tb = pl->blocks[ins->offset + b];
              const dcpx_data_block* db = &g->data_blocks[tb.block];
              bytes += db->size_bytes; /* :303 */
              if (!numeric) continue;
              if (db->kind == DCPX_KIND_Q) mat_set(&msg->q[b], sd->q[tb.slot].rows, D, sd->q[tb.slot].a);
              else if (db->kind == DCPX_KIND_KV) {
                mat_set(&msg->k[b], sd->k[tb.slot].rows, D, sd->k[tb.slot].a);
                mat_set(&msg->v[b], sd->v[tb.slot].rows, D, sd->v[tb.slot].a);
              } else part_copy(&msg->o[b], &sd->o[tb.slot], D);
            }
            rep->total_bytes += bytes; /* :313-316 */
            rep->per_device_send[d] += bytes;
            rep->per_device_recv[ins->peer] += bytes;
            rep->comm_bytes[((size_t)ins->division * 64 + d) * 64 + ins->peer] += bytes;
          } else {
            if (sd->n_posted >= 512) ERR(DCPX_ERROR, "oracle: too many posted receives");
            sd->posted_tag[sd->n_posted] = ins->tag;
            sd->posted_blocks[sd->n_posted] = pl->blocks + ins->offset;
            sd->posted_count[sd->n_posted] = ins->count;
            sd->n_posted++;
          }
          ++sd->pc; any_progress = 1;
          continue;
        }
        if (ins->op == DCPX_OP_ATTENTION) { /* :328-344 */
          const dcpx_attention_item* items = pl->items + ins->offset;
          int bad = 0;
          for (int it = 0; it < ins->count; ++it) { /* flops from rows (:330-334) */
            const dcpx_attention_item* x = &items[it];
            const int nq = (int)(x->q_end - x->q_begin);
            int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(nq > 0 ? nq : 1));
            if (x->rows_offset >= 0) memcpy(rows, pl->rows + 4 * x->rows_offset, sizeof(int32_t) * 4 * (size_t)nq);
            else orc_item_rows(masks, x->seq, x->q_begin, x->q_end, x->kv_begin, x->kv_end, rows);
            uint64_t pairs = 0;
            for (int r = 0; r < nq; ++r) {
              if (rows[4 * r + 1] > rows[4 * r]) pairs += (uint64_t)(rows[4 * r + 1] - rows[4 * r]);
              if (rows[4 * r + 3] > rows[4 * r + 2]) pairs += (uint64_t)(rows[4 * r + 3] - rows[4 * r + 2]);
            }
            rep->comp_flops[(size_t)ins->division * 64 + d] += 4 * pairs * (uint64_t)D;
            rep->total_flops += 4 * pairs * (uint64_t)D;
            free(rows);
          }
          if (numeric) {
            #pragma omp parallel for schedule(dynamic, 1) reduction(|| : bad)
            for (int it = 0; it < ins->count; ++it) {
              const dcpx_attention_item* x = &items[it];
              const int nq = (int)(x->q_end - x->q_begin);
              int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(nq > 0 ? nq : 1));
              if (x->rows_offset >= 0) memcpy(rows, pl->rows + 4 * x->rows_offset, sizeof(int32_t) * 4 * (size_t)nq);
              else orc_item_rows(masks, x->seq, x->q_begin, x->q_end, x->kv_begin, x->kv_end, rows);
              part_t* p = &sd->o[x->out_slot];
              const mat_t* mq = &sd->q[x->q_slot];
              const mat_t* mk = &sd->k[x->kv_slot];
              part_alloc(p, mq->rows, D);
              if (orc_exec_attention(mq->a, mk->a, sd->v[x->kv_slot].a, mq->rows, mk->rows, D, rows,
                                     p->out, p->m, p->l)) bad = 1;
              free(rows);
            }
          }
          if (bad) ERR(DCPX_ERROR, "exec_attention: range outside kv tile");
          ++sd->pc; any_progress = 1;
          continue;
        }
        if (ins->op == DCPX_OP_REDUCTION) { /* :345-354 */
          if (numeric) {
            const int n = ins->count;
            const double** outs = (const double**)malloc(sizeof(double*) * (size_t)n);
            const double** ms = (const double**)malloc(sizeof(double*) * (size_t)n);
            const double** ls = (const double**)malloc(sizeof(double*) * (size_t)n);
            const int rows = sd->o[pl->srcs[ins->offset]].rows;
            for (int i = 0; i < n; ++i) {
              const part_t* p = &sd->o[pl->srcs[ins->offset + i]];
              if (p->rows != rows) ERR(DCPX_ERROR, "exec_reduction: partial shape mismatch");
              outs[i] = p->out; ms[i] = p->m; ls[i] = p->l;
            }
            part_t r = {0, NULL, NULL, NULL};
            part_alloc(&r, rows, D);
            orc_exec_reduction(n, outs, ms, ls, rows, D, r.out, r.m, r.l);
            part_t* dst = &sd->o[ins->dst];
            free(dst->out); free(dst->m); free(dst->l);
            *dst = r;
            free(outs); free(ms); free(ls);
          }
          ++sd->pc; any_progress = 1;
          continue;
        }
        if (ins->op == DCPX_OP_COPY) { /* :355-368; m and l are KEPT here (LSE) */
          if (numeric)
            for (int i = 0; i < ins->count; ++i) {
              const dcpx_copy_item ci = pl->copies[ins->offset + i];
              part_t tmp = {0, NULL, NULL, NULL};
              part_copy(&tmp, &sd->o[ci.src_slot], D);
              part_t* dst = &sd->o[ci.dst_slot];
              free(dst->out); free(dst->m); free(dst->l);
              *dst = tmp;
            }
          ++sd->pc; any_progress = 1;
          continue;
        }
        ERR(DCPX_ERROR, "run: unknown instruction");
      }
    }
    if (all_done) break;
    if (!any_progress) { /* :384-394 */
      char buf[1024];
      int off = snprintf(buf, sizeof buf, "deadlock: ");
      for (int d = 0; d < R && off < (int)sizeof buf - 64; ++d) {
        if (dev[d].pc >= (size_t)plans[d].n_instructions) continue;
        const dcpx_instruction* ins = &plans[d].instructions[dev[d].pc];
        if (ins->op == DCPX_OP_COMM_WAIT)
          off += snprintf(buf + off, sizeof buf - (size_t)off, "device %d waits on %s; ", d, ins->tag);
      }
      ERR(DCPX_DEADLOCK, "%s", buf);
    }
  }
  for (int x = 0; x < nmsg; ++x) /* :396-397 */
    if (inbox[x].live) ERR(DCPX_TAG_MISMATCH, "messages left undelivered at termination");

  /* output assembly (:403-421), plus LSE = m + ln l */
  if (numeric) {
    memset(o, 0, sizeof(double) * (size_t)TT * H * D);
    for (size_t i = 0; i < (size_t)H * (size_t)TT; ++i) lse[i] = NEG_INF;
    for (int d = 0; d < R; ++d)
      for (int i = 0; i < plans[d].n_resident_o; ++i) {
        const dcpx_data_block* db = &g->data_blocks[plans[d].resident_o[i].block];
        const part_t* p = &dev[d].o[plans[d].resident_o[i].slot];
        for (int r = 0; r < p->rows; ++r) {
          const int64_t t = masks->seq_offsets[db->seq] + db->tok_begin + r;
          memcpy(o + ((size_t)t * H + db->head) * D, p->out + (size_t)r * D, sizeof(double) * D);
          lse[(size_t)db->head * TT + t] = p->l[r] > 0 ? p->m[r] + log(p->l[r]) : NEG_INF;
        }
      }
  }
done:
  for (int d = 0; d < R; ++d) {
    if (!dev[d].plan) continue;
    for (int s = 0; s < plans[d].capacity[0]; ++s) free(dev[d].q[s].a);
    for (int s = 0; s < plans[d].capacity[1]; ++s) { free(dev[d].k[s].a); free(dev[d].v[s].a); }
    for (int s = 0; s < plans[d].capacity[2]; ++s) { free(dev[d].o[s].out); free(dev[d].o[s].m); free(dev[d].o[s].l); }
    free(dev[d].q); free(dev[d].k); free(dev[d].v); free(dev[d].o);
  }
  for (int x = 0; x < nmsg; ++x)
    if (inbox[x].live) {
      for (int b = 0; b < inbox[x].nblocks; ++b) {
        free(inbox[x].q[b].a); free(inbox[x].k[b].a); free(inbox[x].v[b].a);
        free(inbox[x].o[b].out); free(inbox[x].o[b].m); free(inbox[x].o[b].l);
      }
      free(inbox[x].q); free(inbox[x].k); free(inbox[x].v); free(inbox[x].o);
    }
  free(inbox);
  free(dev);
  return status;
}

/* ---- dense forward: tests/oracle.hpp:80-120 (mask as ranges, LSE added) ------------- */
void orc_dense_forward(const dcpx_graph_view* g, const dcpx_mask_view* masks, const double* q,
                       const double* k, const double* v, double* o, double* lse) {
  const int H = g->heads, G = g->kv_groups, D = g->head_dim;
  const int64_t TT = masks->seq_offsets[g->num_seqs];
  const double scale = 1.0 / sqrt((double)D);
  #pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int s = 0; s < g->num_seqs; ++s)
    for (int h = 0; h < H; ++h) {
      const int grp = (int)((long long)h * G / H); /* kv_group_of_head, types.hpp:259-261 */
      const int64_t off = masks->seq_offsets[s], L = g->seq_lengths[s];
      double* sc = (double*)malloc(sizeof(double) * (size_t)(L + 1));
      for (int64_t i = 0; i < L; ++i) {
        const int32_t* r = masks->ranges + 4 * (size_t)(off + i);
        const double* qi = q + ((size_t)(off + i) * H + h) * D;
        double* oi = o + ((size_t)(off + i) * H + h) * D;
        memset(oi, 0, sizeof(double) * D);
        double m = NEG_INF;
        for (int ri = 0; ri < 2; ++ri)
          for (int64_t j = r[2 * ri]; j < r[2 * ri + 1]; ++j) {
            const double* kj = k + ((size_t)(off + j) * G + grp) * D;
            double dot = 0;
            for (int d = 0; d < D; ++d) dot += qi[d] * kj[d];
            sc[j] = dot * scale;
            if (sc[j] > m) m = sc[j];
          }
        if (!isfinite(m)) { lse[(size_t)h * TT + off + i] = NEG_INF; continue; }
        double l = 0;
        for (int ri = 0; ri < 2; ++ri)
          for (int64_t j = r[2 * ri]; j < r[2 * ri + 1]; ++j) l += exp(sc[j] - m);
        for (int ri = 0; ri < 2; ++ri)
          for (int64_t j = r[2 * ri]; j < r[2 * ri + 1]; ++j) {
            const double w = exp(sc[j] - m) / l;
            const double* vj = v + ((size_t)(off + j) * G + grp) * D;
            for (int d = 0; d < D; ++d) oi[d] += w * vj[d];
          }
        lse[(size_t)h * TT + off + i] = m + log(l);
      }
      free(sc);
    }
}

/* ---- dense backward (no reference; formulas in dcp_oracle.h) ------------------------ */
void orc_dense_backward(const dcpx_graph_view* g, const dcpx_mask_view* masks, const double* q,
                        const double* k, const double* v, const double* d_o, double* dq,
                        double* dk, double* dv) {
  const int H = g->heads, G = g->kv_groups, D = g->head_dim;
  const int64_t TT = masks->seq_offsets[g->num_seqs];
  const double scale = 1.0 / sqrt((double)D);
  double* o = (double*)malloc(sizeof(double) * (size_t)TT * H * D);
  double* lse = (double*)malloc(sizeof(double) * (size_t)TT * H);
  orc_dense_forward(g, masks, q, k, v, o, lse);
  memset(dq, 0, sizeof(double) * (size_t)TT * H * D);
  memset(dk, 0, sizeof(double) * (size_t)TT * G * D);
  memset(dv, 0, sizeof(double) * (size_t)TT * G * D);
  /* parallel over (seq, group); heads of a group run serially so dK/dV need no atomics */
  #pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int s = 0; s < g->num_seqs; ++s)
    for (int grp = 0; grp < G; ++grp) {
      const int64_t off = masks->seq_offsets[s], L = g->seq_lengths[s];
      for (int h = 0; h < H; ++h) {
        if ((int)((long long)h * G / H) != grp) continue;
        for (int64_t i = 0; i < L; ++i) {
          const size_t qi_off = ((size_t)(off + i) * H + h) * D;
          const double li = lse[(size_t)h * TT + off + i];
          if (!isfinite(li)) continue;
          const int32_t* r = masks->ranges + 4 * (size_t)(off + i);
          double delta = 0;
          for (int d = 0; d < D; ++d) delta += d_o[qi_off + d] * o[qi_off + d];
          for (int ri = 0; ri < 2; ++ri)
            for (int64_t j = r[2 * ri]; j < r[2 * ri + 1]; ++j) {
              const size_t kj_off = ((size_t)(off + j) * G + grp) * D;
              double dot = 0, dp = 0;
              for (int d = 0; d < D; ++d) {
                dot += q[qi_off + d] * k[kj_off + d];
                dp += d_o[qi_off + d] * v[kj_off + d];
              }
              const double p = exp(dot * scale - li);
              const double ds = p * (dp - delta);
              for (int d = 0; d < D; ++d) {
                dv[kj_off + d] += p * d_o[qi_off + d];
                dq[qi_off + d] += ds * k[kj_off + d] * scale;
                dk[kj_off + d] += ds * q[qi_off + d] * scale;
              }
            }
        }
      }
    }
  free(o);
  free(lse);
}
