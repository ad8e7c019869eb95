/* s3_oracle.c -- TEST INFRASTRUCTURE ONLY (see s3_oracle.h).
 *
 * A plain state machine that executes the S^3 decode step exactly as the
 * paper states it, one sequence / layer / head / row at a time, in fp64 for
 * the attention.  No blocking, fusion or reordering.  Readings of points the
 * paper leaves open are DESIGN.md R1..R25 and are cited where used.
 *
 * Arena layout (part of the boundary):
 *   uint16 bf16 bits [R][L][2][H][D]; a sequence owns rows [off, off+cap).
 *   Host copy of an evicted sequence: its resident rows, same row layout.
 */
#include "s3_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= */
/* Closed forms                                                             */
/* ======================================================================= */

/* PAPER.md:111 [§2.1]: "The size of the KV cache is 4 l d_h bytes per token
 * when using half-precision numbers" -- with d_h = H*D (model dim).       */
int64_t s3o_kv_bytes_per_token(int64_t L, int64_t H, int64_t D) { return 4 * L * H * D; }

/* PAPER.md:15 [Analysis, Eviction Penalty]:
 *   2 ( S_P(x_i)/BW_H2D + sum_{j=i+1}^{n} S_P(x_j) / BW_HBM )             */
double s3o_eviction_penalty(double sp_i, double sum_sp_below, double bw_h2d, double bw_hbm) {
  return 2.0 * (sp_i / bw_h2d + sum_sp_below / bw_hbm);
}

/* PAPER.md:21 [Analysis]: 2 p N ( S_P(x)/BW_H2D + sum_0^n S_P(x_j) / (2 BW_HBM) )
 * with S_P(x) the mean reservation and the sum over the resident batch
 * (R14).                                                         */
double s3o_pool_penalty(double p, double N, double sp_mean, double sum_sp_resident,
                        double bw_h2d, double bw_hbm) {
  return 2.0 * p * N * (sp_mean / bw_h2d + sum_sp_resident / (2.0 * bw_hbm));
}

/* PAPER.md:36 [Analysis, Underutilization Penalty]: sum^N S_A(x) / sum^N S_P(x) */
double s3o_underutilization_ratio(int64_t n, const int64_t* s_actual, const int64_t* s_pred) {
  double a = 0.0, p = 0.0;
  for (int64_t i = 0; i < n; ++i) { a += (double)s_actual[i]; p += (double)s_pred[i]; }
  return a / p;
}

/* ======================================================================= */
/* Synthetic value generator          */
/* ======================================================================= */

uint64_t s3o_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint16_t float_to_bf16_bits_exact(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);   /* values here have <= 8 significant bits */
}

static int32_t kv_heads(const s3o_config* c) { return c->Hkv > 0 ? c->Hkv : c->H; }

/* tag 0 (K/V rows) runs over the Hkv KV heads, tag 1 (q) over the H query heads */
static void gen_values(const s3o_config* c, int tag, int64_t req, int32_t l, int32_t kv,
                       int32_t pos, float denom, uint16_t* out_hd) {
  const int32_t nh = tag == 0 ? kv_heads(c) : c->H;
  for (int32_t h = 0; h < nh; ++h) {
    for (int32_t d8 = 0; d8 < c->D / 8; ++d8) {
      uint64_t g = (((((uint64_t)req * (uint64_t)c->L + (uint64_t)l) * 2u + (uint64_t)kv)
                     * (uint64_t)c->max_len + (uint64_t)pos) * (uint64_t)nh + (uint64_t)h)
                   * (uint64_t)(c->D / 8) + (uint64_t)d8;
      uint64_t z = s3o_splitmix64(c->seed ^ ((uint64_t)tag << 60) ^ g);
      for (int j = 0; j < 8; ++j) {
        int k8 = (int)((z >> (8 * j)) & 0xFFu) - 128;
        out_hd[(int64_t)h * c->D + d8 * 8 + j] = float_to_bf16_bits_exact((float)k8 / denom);
      }
    }
  }
}

void s3o_gen_kv(const s3o_config* c, int64_t req, int32_t l, int32_t kv, int32_t pos, uint16_t* out_hd) {
  gen_values(c, 0, req, l, kv, pos, 128.0f, out_hd);
}

void s3o_gen_q(const s3o_config* c, int64_t req, int32_t l, int32_t pos, uint16_t* out_hd) {
  gen_values(c, 1, req, l, 0, pos, 32.0f, out_hd);
}

static double bf16_to_double(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* ======================================================================= */
/* First-fit decreasing                                                     */
/* ======================================================================= */

/* Sort order: cap descending, req ascending (R7). */
typedef struct { int64_t cap, req; int32_t idx; } ffd_key;

static int ffd_cmp(const void* a, const void* b) {
  const ffd_key* x = (const ffd_key*)a;
  const ffd_key* y = (const ffd_key*)b;
  if (x->cap != y->cap) return x->cap > y->cap ? -1 : 1;
  if (x->req != y->req) return x->req < y->req ? -1 : 1;
  return 0;
}

static ffd_key* sorted_keys(int32_t n, const int64_t* cap, const int64_t* req) {
  ffd_key* k = (ffd_key*)malloc(sizeof(ffd_key) * (size_t)(n > 0 ? n : 1));
  for (int32_t i = 0; i < n; ++i) { k[i].cap = cap[i]; k[i].req = req[i]; k[i].idx = i; }
  qsort(k, (size_t)n, sizeof(ffd_key), ffd_cmp);
  return k;
}

/* PAPER.md:164-166 [§3 Scheduler]: "sorts the sequences in the request pool
 * ... in a decreasing order.  It iterates through the pool and checks if the
 * KV cache of the current sequence does not exceed the available HBM.  If so,
 * it includes the sequence in the current batch and reduces the available
 * HBM by the size of the KV cache ... until either there is no available HBM
 * or it has iterated through the entire request pool."  Skip-and-continue
 * (R8).  max_items is the metadata capacity (R21).
 * admitted[i] = 1 + placement order for admitted items, 0 otherwise.       */
int32_t s3o_ffd(int32_t n, const int64_t* cap, const int64_t* req, int64_t free_rows,
                int32_t max_items, uint8_t* admitted) {
  ffd_key* k = sorted_keys(n, cap, req);
  int32_t count = 0;
  for (int32_t i = 0; i < n; ++i) admitted[i] = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (count >= max_items) break;
    if (k[i].cap <= free_rows) {
      free_rows -= k[i].cap;
      admitted[k[i].idx] = 1;
      ++count;
    }
  }
  free(k);
  return count;
}

/* Multi-bin FFD over ranks (R26): items in FFD order (PAPER.md:166,
 * "sorts ... in a decreasing order"); each item goes to the rank with the MOST
 * free rows among the ranks with a free metadata slot, ties to the lowest
 * rank (worst fit), if it fits there -- otherwise it fits nowhere and is
 * skipped.  The paper has one bin; the bin choice is R26's
 * reading for several GPUs in lockstep, where a step lasts as long as the
 * busiest rank, so the freed rows are filled evenly.  assigned_rank[i] =
 * rank or -1.  free_rows / slots_left are updated in place.                */
int32_t s3o_ffd_multibin(int32_t n, const int64_t* cap, const int64_t* req, int32_t world,
                         int64_t* free_rows, int64_t* slots_left, int32_t* assigned_rank) {
  ffd_key* k = sorted_keys(n, cap, req);
  int32_t count = 0;
  for (int32_t i = 0; i < n; ++i) assigned_rank[i] = -1;
  for (int32_t i = 0; i < n; ++i) {
    int32_t best = -1;
    for (int32_t r = 0; r < world; ++r)
      if (slots_left[r] > 0 && (best < 0 || free_rows[r] > free_rows[best])) best = r;
    if (best >= 0 && k[i].cap <= free_rows[best]) {
      free_rows[best] -= k[i].cap;
      slots_left[best] -= 1;
      assigned_rank[k[i].idx] = best;
      ++count;
    }
  }
  free(k);
  return count;
}

/* ======================================================================= */
/* State machine                                                            */
/* ======================================================================= */

typedef struct {
  int64_t req;
  int32_t prompt, alloc, gen, cap, evictions;
  int32_t evicted;        /* 1: carries host KV ("moves ... to the request pool") */
  uint16_t* host_kv;      /* [rows][L][2][H][D] */
  int64_t host_rows;
} item;

struct s3o_state {
  s3o_config c;
  int64_t row_elems;      /* elements per token row: 2*L*H*D */
  uint16_t* arena;
  s3o_slot* slots;
  uint8_t* status;
  int32_t B;
  int status_valid;
  int64_t tail;
  item* pool;
  int32_t npool, pool_cap;
  int64_t finished_total, evicted_total, tokens_total;
  int64_t moved_at_admit;  /* R27: bytes shifted by admission-time compactions */
};

s3o_state* s3o_create(const s3o_config* c) {
  if (c->L < 1 || c->H < 1 || c->D < 8 || c->D % 8 || c->max_len < 1 || c->R < c->max_len ||
      c->max_running < 1 || c->Hkv < 0 || (c->Hkv > 0 && c->H % c->Hkv))
    return NULL;
  s3o_state* s = (s3o_state*)calloc(1, sizeof(s3o_state));
  s->c = *c;
  if (s->c.Hkv == 0) s->c.Hkv = c->H;
  s->row_elems = 2LL * c->L * s->c.Hkv * c->D;
  s->arena = (uint16_t*)calloc((size_t)(c->R * s->row_elems), sizeof(uint16_t));
  s->slots = (s3o_slot*)calloc((size_t)c->max_running, sizeof(s3o_slot));
  s->status = (uint8_t*)calloc((size_t)c->max_running, 1);
  s->pool_cap = 64;
  s->pool = (item*)calloc((size_t)s->pool_cap, sizeof(item));
  if (!s->arena || !s->slots || !s->status || !s->pool) { s3o_destroy(s); return NULL; }
  return s;
}

void s3o_destroy(s3o_state* s) {
  if (!s) return;
  for (int32_t i = 0; i < s->npool; ++i) free(s->pool[i].host_kv);
  free(s->pool); free(s->slots); free(s->status); free(s->arena);
  free(s);
}

static void pool_push(s3o_state* s, item it) {
  if (s->npool == s->pool_cap) {
    s->pool_cap *= 2;
    s->pool = (item*)realloc(s->pool, sizeof(item) * (size_t)s->pool_cap);
  }
  s->pool[s->npool++] = it;
}

static void pool_remove_marked(s3o_state* s, const uint8_t* remove) {
  int32_t w = 0;
  for (int32_t i = 0; i < s->npool; ++i)
    if (!remove[i]) s->pool[w++] = s->pool[i];
  s->npool = w;
}

/* Reservation = P + predicted output (R4).  A reservation larger
 * than the whole arena is unschedulable -> error 6.          */
int s3o_submit(s3o_state* s, int32_t n, const int64_t* req, const int32_t* prompt,
               const int32_t* alloc) {
  for (int32_t i = 0; i < n; ++i) {
    if (prompt[i] < 0 || alloc[i] < 1 || prompt[i] + alloc[i] > s->c.max_len) return 1;
  }
  for (int32_t i = 0; i < n; ++i) {
    item it;
    memset(&it, 0, sizeof(it));
    it.req = req[i]; it.prompt = prompt[i]; it.alloc = alloc[i];
    it.cap = prompt[i] + alloc[i];
    pool_push(s, it);
  }
  return 0;
}

int32_t s3o_batch(const s3o_state* s, s3o_slot* slots) {
  if (slots) memcpy(slots, s->slots, sizeof(s3o_slot) * (size_t)s->B);
  return s->B;
}

const uint16_t* s3o_arena(const s3o_state* s) { return s->arena; }

int64_t s3o_host_kv(const s3o_state* s, int64_t req, const uint16_t** kv) {
  for (int32_t i = 0; i < s->npool; ++i)
    if (s->pool[i].req == req && s->pool[i].evicted) { *kv = s->pool[i].host_kv; return s->pool[i].host_rows; }
  return -1;
}

static uint16_t* row_ptr(s3o_state* s, int64_t row, int32_t l, int32_t kv) {
  return s->arena + row * s->row_elems + ((int64_t)l * 2 + kv) * s->c.Hkv * s->c.D;
}

/* Inputs of one decode step: for slot b at position pos = len_b,
 * k_new/v_new = KV(req, l, kv, pos) and q = Q(req, l, pos); the sampler's
 * EOS fires when this token is the request's last one (gen + 1 == O).
 * Layout: q [L][B][H][D], k and v [L][B][Hkv][D].                          */
void s3o_make_inputs(const s3o_state* s, const int32_t* out_len_by_req, uint16_t* q,
                     uint16_t* k, uint16_t* v, uint8_t* eos) {
  const int64_t HD = (int64_t)s->c.H * s->c.D, KD = (int64_t)s->c.Hkv * s->c.D;
  for (int32_t b = 0; b < s->B; ++b) {
    const s3o_slot* sl = &s->slots[b];
    for (int32_t l = 0; l < s->c.L; ++l) {
      s3o_gen_kv(&s->c, sl->req, l, 0, sl->len, k + ((int64_t)l * s->B + b) * KD);
      s3o_gen_kv(&s->c, sl->req, l, 1, sl->len, v + ((int64_t)l * s->B + b) * KD);
      s3o_gen_q(&s->c, sl->req, l, sl->len, q + ((int64_t)l * s->B + b) * HD);
    }
    eos[b] = (uint8_t)(sl->gen + 1 == out_len_by_req[sl->req]);
  }
}

/* softmax(q K^T / sqrt(D)) V for one layer, all H query heads, over n rows;
 * row j's K (all Hkv KV heads) starts at K0 + j*stride, V likewise; query
 * head h uses KV head h / (H/Hkv) (grouped-query attention; Hkv = H is MHA)
 * (PAPER.md:106).                                                          */
static void attend(const uint16_t* q_hd, const uint16_t* K0, const uint16_t* V0, int64_t stride,
                   int32_t n, int32_t H, int32_t Hkv, int32_t D, double* sc, double* out_hd) {
  const double inv_sqrt_d = 1.0 / sqrt((double)D);
  for (int32_t h = 0; h < H; ++h) {
    const uint16_t* qh = q_hd + (int64_t)h * D;
    const int64_t kvo = (int64_t)(h / (H / Hkv)) * D;
    /* scores s_j = q . K_j / sqrt(D), j = 0..n-1 */
    double m = -INFINITY;
    for (int32_t j = 0; j < n; ++j) {
      const uint16_t* kj = K0 + j * stride + kvo;
      double acc = 0.0;
      for (int32_t d = 0; d < D; ++d) acc += bf16_to_double(qh[d]) * bf16_to_double(kj[d]);
      sc[j] = acc * inv_sqrt_d;
      if (sc[j] > m) m = sc[j];
    }
    /* softmax weights and the weighted sum of V */
    double den = 0.0;
    for (int32_t j = 0; j < n; ++j) { sc[j] = exp(sc[j] - m); den += sc[j]; }
    double* o = out_hd + (int64_t)h * D;
    for (int32_t d = 0; d < D; ++d) {
      double acc = 0.0;
      for (int32_t j = 0; j < n; ++j) acc += sc[j] * bf16_to_double(V0[j * stride + kvo + d]);
      o[d] = acc / den;
    }
  }
}

/* One decode iteration for every running sequence.
 *
 * PAPER.md:103-109 [§2.1]: h_out = softmax(q_i K^T / sqrt(d_h)) V.  Reading
 * R1: the new token's K,V row is appended first and attended (self
 * included, rows 0..pos); R2: sqrt(d_h) is the per-head dim D.
 * [§2.2]: the reserved memory is filled "in an append-only fashion".
 * PAPER.md:174 [§3 Supervisor]: a sequence that is "not finished but used up
 * its reserved memory" is an overrun; R11: EOS at len == cap is FINISHED.
 * out: double [L][B][H][D].  status_out (optional): uint8 [B].            */
/* Threads for the attention loop of s3o_decode (1 = the plain sequential
 * oracle; used by bench.py's cpu_baseline to time it on all host cores).   */
static int s3o_threads = 1;
void s3o_set_threads(int n) { s3o_threads = n > 0 ? n : 1; }

int s3o_decode(s3o_state* s, const uint16_t* q, const uint16_t* k, const uint16_t* v,
               const uint8_t* eos, double* out, uint8_t* status_out) {
  if (s->status_valid) return 5;  /* previous statuses not yet consumed */
  const int32_t H = s->c.H, D = s->c.D, L = s->c.L, Hkv = s->c.Hkv;
  const int64_t HD = (int64_t)H * D, KD = (int64_t)Hkv * D;
  for (int32_t b = 0; b < s->B; ++b)
    if (s->slots[b].len >= s->slots[b].cap) return 5;
  /* append: row off+pos <- (k_new, v_new) for every (b, l) */
  for (int32_t b = 0; b < s->B; ++b) {
    const s3o_slot* sl = &s->slots[b];
    for (int32_t l = 0; l < L; ++l) {
      const int64_t ko = ((int64_t)l * s->B + b) * KD;
      memcpy(row_ptr(s, sl->off + sl->len, l, 0), k + ko, sizeof(uint16_t) * (size_t)KD);
      memcpy(row_ptr(s, sl->off + sl->len, l, 1), v + ko, sizeof(uint16_t) * (size_t)KD);
    }
  }
  /* attend over rows 0..pos (self included, R1).  The (b, l) pairs are
   * independent (each reads only its own slot's rows), so the optional
   * threads of s3o_set_threads split them; the arithmetic is unchanged.    */
  const int64_t pairs = (int64_t)s->B * L;
#pragma omp parallel num_threads(s3o_threads)
  {
    double* sc = (double*)malloc(sizeof(double) * (size_t)(s->c.max_len + 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t pr = 0; pr < pairs; ++pr) {
      const int32_t b = (int32_t)(pr / L), l = (int32_t)(pr % L);
      const s3o_slot* sl = &s->slots[b];
      const int64_t io = ((int64_t)l * s->B + b) * HD;
      attend(q + io, row_ptr(s, sl->off, l, 0), row_ptr(s, sl->off, l, 1), s->row_elems, sl->len + 1,
             H, Hkv, D, sc, out + io);
    }
    free(sc);
  }
  for (int32_t b = 0; b < s->B; ++b) {
    s3o_slot* sl = &s->slots[b];
    sl->len += 1;
    sl->gen += 1;
    s->tokens_total += 1;
    /* R28: a sequence at the maximum length stops like one that emitted EOS
     * ("prompt_tokens + output_tokens <= max_seq_len"; PAPER.md:127
     * "a maximum sequence length of 2048 tokens"): its reservation cannot grow. */
    if (eos[b] || sl->len == s->c.max_len) s->status[b] = S3O_FINISHED;
    else if (sl->len == sl->cap) s->status[b] = S3O_OVERRUN;
    else s->status[b] = S3O_RUNNING;
    if (status_out) status_out[b] = s->status[b];
  }
  s->status_valid = 1;
  return 0;
}

/* Eviction + row-shift compaction.
 *
 * PAPER.md:174 [§3 Supervisor]: overruns are evicted -- "moves the current
 * state of those sequences including the KV cache and the generated tokens
 * to the request pool and frees up the GPU memory" -- then "shifts the rows
 * below the blank one so that all rows are stored contiguously", and
 * "doubles the assigned memory for the evicted sequences" (R5: cap <-
 * min(2 cap, max_len)).  R6: finished sequences leave in the same single
 * compaction pass.  R10: evicted requests re-enter the pool at once.
 *
 * Byte counters:
 *   d2h_bytes        = sum over evicted of resident rows * kvpt (== S_P, len == cap)
 *   moved_bytes      = sum over kept sequences that change offset of len * kvpt
 *   paper_pcie_bytes = sum over evicted i of 2 S_P(x_i)
 *   paper_hbm_bytes  = sum over evicted i of 2 sum_{j>i} S_P(x_j)  (R12)
 */
int s3o_evict_compact(s3o_state* s, s3o_report* rep, int32_t* perm, s3o_evicted* ev,
                      int64_t* finished) {
  if (!s->status_valid) return 5;
  const int64_t kvpt = s3o_kv_bytes_per_token(s->c.L, s->c.Hkv, s->c.D);
  memset(rep, 0, sizeof(*rep));
  rep->n_before = s->B;
  rep->first_hole = s->B;
  for (int32_t b = 0; b < s->B; ++b) {
    s3o_slot* sl = &s->slots[b];
    if (s->status[b] != S3O_RUNNING && rep->first_hole == s->B) rep->first_hole = b;
    if (s->status[b] == S3O_FINISHED) {
      if (finished) finished[rep->n_finished] = sl->req;
      rep->n_finished++;
    } else if (s->status[b] == S3O_OVERRUN) {
      item it;
      memset(&it, 0, sizeof(it));
      it.req = sl->req; it.prompt = sl->prompt; it.gen = sl->gen;
      it.alloc = 0;
      it.evicted = 1;
      it.host_rows = sl->len;
      it.host_kv = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(sl->len * s->row_elems));
      memcpy(it.host_kv, s->arena + sl->off * s->row_elems,
             sizeof(uint16_t) * (size_t)(sl->len * s->row_elems));
      it.cap = sl->cap * 2 < s->c.max_len ? sl->cap * 2 : s->c.max_len;
      it.alloc = it.cap - it.prompt;
      rep->d2h_bytes += (int64_t)sl->len * kvpt;
      rep->paper_pcie_bytes += 2 * (int64_t)sl->cap * kvpt;
      int64_t below = 0;
      for (int32_t j = b + 1; j < s->B; ++j) below += s->slots[j].cap;
      rep->paper_hbm_bytes += 2 * below * kvpt;
      if (ev) {
        s3o_evicted* e = &ev[rep->n_evicted];
        e->req = sl->req; e->batch_index = b; e->prompt = sl->prompt; e->gen = sl->gen;
        e->len = sl->len; e->cap = sl->cap; e->new_cap = it.cap;
      }
      rep->n_evicted++;
      pool_push(s, it);
    }
  }
  /* Compaction in batch (= arena) order.  dst <= src, so a forward memmove
   * of each survivor in order is safe.  Policy "on demand" (R27):
   * shift only when the pool is non-empty after this step's evictions, i.e.
   * when an admission could use the freed rows; otherwise survivors keep
   * their rows and the tail is the end of the last survivor's slot. */
  const int do_compact = s->c.compact_policy == 0 || s->npool > 0;
  int64_t new_tail = 0;
  int32_t nb = 0;
  for (int32_t b = 0; b < s->B; ++b) {
    s3o_slot sl = s->slots[b];
    if (s->status[b] == S3O_RUNNING) {
      if (do_compact) {
        if (new_tail != sl.off) {
          memmove(s->arena + new_tail * s->row_elems, s->arena + sl.off * s->row_elems,
                  sizeof(uint16_t) * (size_t)(sl.len * s->row_elems));
          rep->moved_bytes += (int64_t)sl.len * kvpt;
        }
        sl.off = new_tail;
        new_tail += sl.cap;
      } else {
        new_tail = sl.off + sl.cap;
      }
      if (perm) perm[b] = nb;
      s->slots[nb++] = sl;
    } else if (perm) {
      perm[b] = -1;
    }
  }
  s->finished_total += rep->n_finished;
  s->evicted_total += rep->n_evicted;
  s->B = nb;
  s->tail = new_tail;
  rep->n_kept = nb;
  rep->tail = new_tail;
  s->status_valid = 0;
  return 0;
}

/* Place pool item i at the tail: fresh -> prompt rows are the generator's
 * rows 0..P-1 (stand-in for prefill); evicted -> host rows are copied back
 * ("reload", R10).                                                         */
static void place(s3o_state* s, const item* it) {
  s3o_slot* sl = &s->slots[s->B];
  sl->req = it->req; sl->prompt = it->prompt; sl->cap = it->cap; sl->off = s->tail;
  if (it->evicted) {
    sl->gen = it->gen;
    sl->len = (int32_t)it->host_rows;
    memcpy(s->arena + sl->off * s->row_elems, it->host_kv,
           sizeof(uint16_t) * (size_t)(it->host_rows * s->row_elems));
  } else {
    sl->gen = 0;
    sl->len = it->prompt;
    for (int32_t pos = 0; pos < it->prompt; ++pos)
      for (int32_t l = 0; l < s->c.L; ++l)
        for (int32_t kv = 0; kv < 2; ++kv)
          s3o_gen_kv(&s->c, it->req, l, kv, pos, row_ptr(s, sl->off + pos, l, kv));
  }
  s->tail += it->cap;
  s->B += 1;
}

/* R27 at admission: under the on-demand policy a step with an empty pool
 * leaves its holes in place; once requests wait again (a later submit), the
 * survivors are shifted up before the FFD so it sees the same free rows as
 * under the every-step policy ("shifts the rows below the blank
 * one so that all rows are stored contiguously").  Returns bytes moved.     */
static int64_t compact_holes(s3o_state* s) {
  const int64_t kvpt = s3o_kv_bytes_per_token(s->c.L, s->c.Hkv, s->c.D);
  int64_t new_tail = 0, moved = 0;
  for (int32_t b = 0; b < s->B; ++b) {
    s3o_slot* sl = &s->slots[b];
    if (sl->off != new_tail) {
      memmove(s->arena + new_tail * s->row_elems, s->arena + sl->off * s->row_elems,
              sizeof(uint16_t) * (size_t)(sl->len * s->row_elems));
      moved += (int64_t)sl->len * kvpt;
      sl->off = new_tail;
    }
    new_tail += sl->cap;
  }
  s->tail = new_tail;
  return moved;
}

static void compact_if_waiting(s3o_state* s) {
  if (s->c.compact_policy == 1 && s->npool > 0) s->moved_at_admit += compact_holes(s);
}

/* FFD over the pool items selected by `want` into this arena's free rows. */
static int32_t admit_selected(s3o_state* s, const uint8_t* want, int64_t* admitted) {
  int32_t n = 0;
  int32_t* map = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->npool + 1));
  int64_t* cap = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->npool + 1));
  int64_t* req = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->npool + 1));
  uint8_t* adm = (uint8_t*)malloc((size_t)(s->npool + 1));
  for (int32_t i = 0; i < s->npool; ++i)
    if (want[i]) { map[n] = i; cap[n] = s->pool[i].cap; req[n] = s->pool[i].req; ++n; }
  s3o_ffd(n, cap, req, s->c.R - s->tail, s->c.max_running - s->B, adm);
  /* placement in FFD scan order (R9) */
  ffd_key* k = sorted_keys(n, cap, req);
  uint8_t* remove = (uint8_t*)calloc((size_t)(s->npool + 1), 1);
  int32_t count = 0;
  for (int32_t t = 0; t < n; ++t) {
    int32_t i = k[t].idx;
    if (!adm[i]) continue;
    item* it = &s->pool[map[i]];
    place(s, it);
    if (admitted) admitted[count] = it->req;
    ++count;
    free(it->host_kv);
    it->host_kv = NULL;
    remove[map[i]] = 1;
  }
  pool_remove_marked(s, remove);
  free(remove); free(k); free(adm); free(req); free(cap); free(map);
  return count;
}

/* Single-bin admission, world == 1 ("a variant of the bin
 * packing problem with a single bin"): fresh and evicted requests compete in
 * one FFD.  Returns the number admitted; admitted[] gets their req ids in
 * placement order.                                                         */
int32_t s3o_admit(s3o_state* s, int64_t* admitted) {
  if (s->status_valid) return -5;
  compact_if_waiting(s);
  uint8_t* want = (uint8_t*)malloc((size_t)(s->npool + 1));
  for (int32_t i = 0; i < s->npool; ++i) want[i] = 1;
  int32_t n = admit_selected(s, want, admitted);
  free(want);
  return n;
}

/* world > 1, phase 1 (R26): re-admit this rank's own evicted
 * requests (their KV is in this rank's host store) by local FFD.          */
int32_t s3o_admit_home(s3o_state* s, int64_t* admitted) {
  if (s->status_valid) return -5;
  compact_if_waiting(s);      /* before the counters are exchanged (free rows = R - tail) */
  uint8_t* want = (uint8_t*)malloc((size_t)(s->npool + 1));
  for (int32_t i = 0; i < s->npool; ++i) want[i] = (uint8_t)s->pool[i].evicted;
  int32_t n = admit_selected(s, want, admitted);
  free(want);
  return n;
}

/* world > 1, phase 2 (R26): the fresh pool is identical on every
 * rank; multi-bin FFD over the all-reduced free rows / free slots; this
 * rank places its own assignments and drops every assigned request.       */
int32_t s3o_admit_shared(s3o_state* s, int32_t world, int32_t rank, const int64_t* free_by_rank,
                         const int64_t* slots_left_by_rank, int64_t* admitted) {
  if (s->status_valid) return -5;
  int32_t n = 0;
  int32_t* map = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->npool + 1));
  int64_t* cap = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->npool + 1));
  int64_t* req = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->npool + 1));
  int32_t* who = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->npool + 1));
  int64_t* fr = (int64_t*)malloc(sizeof(int64_t) * (size_t)world);
  int64_t* sl = (int64_t*)malloc(sizeof(int64_t) * (size_t)world);
  for (int32_t r = 0; r < world; ++r) { fr[r] = free_by_rank[r]; sl[r] = slots_left_by_rank[r]; }
  for (int32_t i = 0; i < s->npool; ++i)
    if (!s->pool[i].evicted) { map[n] = i; cap[n] = s->pool[i].cap; req[n] = s->pool[i].req; ++n; }
  s3o_ffd_multibin(n, cap, req, world, fr, sl, who);
  ffd_key* k = sorted_keys(n, cap, req);
  uint8_t* remove = (uint8_t*)calloc((size_t)(s->npool + 1), 1);
  int32_t count = 0;
  for (int32_t t = 0; t < n; ++t) {
    int32_t i = k[t].idx;
    if (who[i] < 0) continue;
    remove[map[i]] = 1;
    if (who[i] != rank) continue;
    place(s, &s->pool[map[i]]);
    if (admitted) admitted[count] = s->pool[map[i]].req;
    ++count;
  }
  pool_remove_marked(s, remove);
  free(remove); free(k); free(sl); free(fr); free(who); free(req); free(cap); free(map);
  return count;
}

/* Counter row exchanged between ranks each step (PAPER.md:172 [§3
 * Supervisor]: "check for the available space in the HBM and passes the
 * information to the scheduler"):
 *   0 free_rows, 1 running, 2 free_slots, 3 evicted_waiting, 4 fresh_waiting,
 *   5 finished_total, 6 evicted_total, 7 tokens_total                      */
int64_t s3o_moved_at_admit(const s3o_state* s) { return s->moved_at_admit; }

void s3o_counters(const s3o_state* s, int64_t row[8]) {
  int64_t ev = 0, fr = 0;
  for (int32_t i = 0; i < s->npool; ++i) { if (s->pool[i].evicted) ++ev; else ++fr; }
  row[0] = s->c.R - s->tail;
  row[1] = s->B;
  row[2] = s->c.max_running - s->B;
  row[3] = ev;
  row[4] = fr;
  row[5] = s->finished_total;
  row[6] = s->evicted_total;
  row[7] = s->tokens_total;
}

/* softmax(q K^T / sqrt(D)) V over n given rows, for inputs
 * that do not come from the generator (the GEMM-fed proxy model's q and
 * appended rows): row j's K at K0 + j*stride, V at V0 + j*stride.         */
void s3o_attend_rows(const uint16_t* q_hd, const uint16_t* K0, const uint16_t* V0, int64_t stride, int32_t n,
                     int32_t H, int32_t Hkv, int32_t D, double* out_hd) {
  double* sc = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  attend(q_hd, K0, V0, stride, n, H, Hkv, D, sc, out_hd);
  free(sc);
}

/* Attention of request `req` at position `pos` of layer l when its rows are
 * the generator's (invariant P2): K_j = G(req,l,0,j), V_j = G(req,l,1,j) for
 * j = 0..pos, q = Q(req,l,pos).  Lets tests check sampled outputs of a
 * full-size GPU run one at a time.  out: double [H][D].                    */
void s3o_attend_generated(const s3o_config* c, int64_t req, int32_t pos, int32_t l, double* out_hd) {
  const int32_t Hkv = kv_heads(c);
  const int64_t KD = (int64_t)Hkv * c->D;
  uint16_t* rows = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)((pos + 1) * 2 * KD));
  uint16_t* q = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)((int64_t)c->H * c->D));
  double* sc = (double*)malloc(sizeof(double) * (size_t)(pos + 1));
  for (int32_t j = 0; j <= pos; ++j) {
    s3o_gen_kv(c, req, l, 0, j, rows + (int64_t)j * 2 * KD);
    s3o_gen_kv(c, req, l, 1, j, rows + (int64_t)j * 2 * KD + KD);
  }
  s3o_gen_q(c, req, l, pos, q);
  attend(q, rows, rows + KD, 2 * KD, pos + 1, c->H, Hkv, c->D, sc, out_hd);
  free(sc); free(q); free(rows);
}
