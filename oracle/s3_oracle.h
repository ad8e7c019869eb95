/* s3_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle of the S^3 length-aware KV-cache
 * decode step (arXiv 2306.06000).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_2306_06000_b200/csrc); the two agree only through the written
 * definitions in DESIGN.md and the paper.
 *
 * Each function cites the passage it follows as PAPER.md:<line> [section].
 * Readings of silent/garbled passages are DESIGN.md "Readings" R1..R25.
 */
#ifndef S3_ORACLE_H
#define S3_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t L, H, D;        /* layers, heads, head dim                     */
  int32_t max_len;        /* max sequence length (cap on P + output)     */
  int64_t R;              /* arena rows                                  */
  int32_t max_running;    /* metadata capacity (admission stops at it)   */
  uint64_t seed;          /* synthetic value generator seed              */
  int32_t compact_policy; /* 0 = every step (R6), 1 = on demand (R27)    */
  int32_t Hkv;            /* KV heads (0 = H); query head h reads KV head h / (H/Hkv) */
} s3o_config;

enum { S3O_RUNNING = 0, S3O_FINISHED = 1, S3O_OVERRUN = 2 };

typedef struct { int64_t req; int32_t prompt, gen, len, cap; int64_t off; } s3o_slot;
typedef struct { int64_t req; int32_t batch_index, prompt, gen, len, cap, new_cap; } s3o_evicted;
typedef struct {
  int32_t n_before, n_finished, n_evicted, n_kept;
  int64_t tail;
  int64_t d2h_bytes, moved_bytes;
  int64_t paper_pcie_bytes, paper_hbm_bytes;
  int32_t first_hole;
} s3o_report;

typedef struct s3o_state s3o_state;

/* ---- closed forms of the paper ---------------------------------------- */
int64_t s3o_kv_bytes_per_token(int64_t L, int64_t H, int64_t D);
double  s3o_eviction_penalty(double sp_i, double sum_sp_below, double bw_h2d, double bw_hbm);
double  s3o_pool_penalty(double p, double N, double sp_mean, double sum_sp_resident,
                         double bw_h2d, double bw_hbm);
double  s3o_underutilization_ratio(int64_t n, const int64_t* s_actual, const int64_t* s_pred);

/* ---- synthetic value generator (own implementation of DESIGN.md contract) */
uint64_t s3o_splitmix64(uint64_t x);
void s3o_gen_kv(const s3o_config* c, int64_t req, int32_t l, int32_t kv, int32_t pos, uint16_t* out_hd);
void s3o_gen_q(const s3o_config* c, int64_t req, int32_t l, int32_t pos, uint16_t* out_hd);

/* ---- first-fit decreasing ---------------------------- */
int32_t s3o_ffd(int32_t n, const int64_t* cap, const int64_t* req, int64_t free_rows,
                int32_t max_items, uint8_t* admitted);
int32_t s3o_ffd_multibin(int32_t n, const int64_t* cap, const int64_t* req, int32_t world,
                         int64_t* free_rows, int64_t* slots_left, int32_t* assigned_rank);

/* ---- the state machine ------------------------------------------------ */
s3o_state* s3o_create(const s3o_config* c);
void s3o_destroy(s3o_state* s);
int  s3o_submit(s3o_state* s, int32_t n, const int64_t* req, const int32_t* prompt,
                const int32_t* alloc);
int32_t s3o_batch(const s3o_state* s, s3o_slot* slots);      /* returns B; slots may be NULL */
const uint16_t* s3o_arena(const s3o_state* s);
int64_t s3o_host_kv(const s3o_state* s, int64_t req, const uint16_t** kv);  /* rows or -1 */
void s3o_make_inputs(const s3o_state* s, const int32_t* out_len_by_req, uint16_t* q,
                     uint16_t* k, uint16_t* v, uint8_t* eos);
void s3o_set_threads(int n);   /* attention loop threads (1 = sequential, the default) */
int  s3o_decode(s3o_state* s, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                const uint8_t* eos, double* out, uint8_t* status_out);
int  s3o_evict_compact(s3o_state* s, s3o_report* rep, int32_t* perm, s3o_evicted* ev,
                       int64_t* finished);
int32_t s3o_admit(s3o_state* s, int64_t* admitted);
int32_t s3o_admit_home(s3o_state* s, int64_t* admitted);
int32_t s3o_admit_shared(s3o_state* s, int32_t world, int32_t rank, const int64_t* free_by_rank,
                         const int64_t* slots_left_by_rank, int64_t* admitted);
void s3o_counters(const s3o_state* s, int64_t row[8]);
int64_t s3o_moved_at_admit(const s3o_state* s);   /* R27 admission-time shifts, bytes */
void s3o_attend_rows(const uint16_t* q_hd, const uint16_t* K0, const uint16_t* V0, int64_t stride, int32_t n,
                     int32_t H, int32_t Hkv, int32_t D, double* out_hd);
void s3o_attend_generated(const s3o_config* c, int64_t req, int32_t pos, int32_t l, double* out_hd);

#ifdef __cplusplus
}
#endif
#endif
