/* s3.h -- C ABI of the B200-native S^3 length-aware KV-cache decode step.
 *
 * S^3 (arXiv 2306.06000): each sequence's KV slot is sized by its PREDICTED
 * output length (PAPER.md:153-178 [§3 Design]).  One iteration of the hot
 * path is four calls:
 *
 *   s3_decode_step    length-masked multi-head decode attention over each
 *                     slot's contiguous KV rows, fused with the KV append and
 *                     the overrun detection
 *   s3_evict_compact  eviction of overruns to pinned host memory and the
 *                     row-shift compaction of survivors
 *   s3_admit          first-fit-decreasing admission of queued requests into
 *                     the freed capacity, doubling the reservation of evicted
 *                     ones
 *   s3_kv_init        binds the arena and creates the context.
 *
 * Conventions
 * -----------
 * - Every function returns s3_status; nothing throws or longjmps across the ABI.
 * - Data layout: the KV arena is bf16
 *   [R][L][2][H_kv][D] -- one token ROW holds all layers' K and V of that
 *   token, kvpt = 4*L*H_kv*D bytes ("4 l d_h bytes per token").  A
 *   sequence owns rows [off, off+cap); rows [off, off+len) are resident.
 *   Slots are kept in arena order (batch index b increases with off).
 * - q is bf16 [nl][B][H][D], k_new / v_new bf16 [nl][B][H_kv][D] (H_kv = H
 *   unless num_kv_heads is set); out is fp32 [nl][B][H][D]; B is the running
 *   batch size (s3_batch_size), b the batch index.  Pointers 16-B aligned.
 * - All device pointers are on cfg.device; all device work is ordered on
 *   cfg.stream (a cudaStream_t, e.g. torch's current stream).
 * - Ownership: the caller allocates and frees every buffer in s3_buffers
 *   (sizes from s3_workspace_query).  The context owns host scheduling state,
 *   a side stream, CUDA events and small pinned host staging buffers.
 * - Errors: S3_E_INVAL / S3_E_UNSCHEDULABLE leave the state unchanged.
 *   S3_E_CUDA poisons the context: afterwards only s3_kv_destroy and
 *   s3_last_error are valid.  S3_E_STATE = call out of order (e.g. two decode
 *   steps without an s3_evict_compact in between).
 * - One context per GPU / process.  Calls are not reentrant.
 */
#ifndef S3_H
#define S3_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  S3_OK = 0,
  S3_E_INVAL = 1,          /* bad argument or config                                 */
  S3_E_NOMEM = 2,          /* caller buffer / host store too small                   */
  S3_E_CUDA = 3,           /* CUDA runtime error (context poisoned)                  */
  S3_E_NCCL = 4,           /* NCCL error or NCCL not loadable (s3_comm_*; poisons)    */
  S3_E_STATE = 5,          /* call out of order / logic error          */
  S3_E_UNSCHEDULABLE = 6   /* reservation larger than the whole arena  */
} s3_status;

/* Per-slot status after a decode step (R11). */
enum { S3_RUNNING = 0, S3_FINISHED = 1, S3_OVERRUN = 2 };

#define S3_NCOUNTERS 8
/* Counter row exchanged between ranks:
 * 0 free_rows, 1 running, 2 free_slots, 3 evicted_waiting, 4 fresh_waiting
 * (identical on every rank), 5 finished_total, 6 evicted_total, 7 tokens_total */

typedef struct s3_ctx s3_ctx;

typedef struct {
  int32_t num_layers, num_heads, head_dim;  /* L, H, D; head_dim in {64,128,256}; H*D <= 4096 */
  int32_t max_seq_len;                      /* cap on P + output (2048 for GPT-J runs)         */
  int64_t arena_rows;                       /* R >= max_seq_len                                */
  int32_t max_running;                      /* metadata capacity B_max (admission stops there) */
  int32_t chunk_rows;                       /* attention split-K chunk C in rows (0 = 512; <= 32768) */
  int32_t move_chunk_bytes;                 /* compaction chunk S (0 = 32768; 1024..36864, %16)*/
  int32_t device;                           /* CUDA device ordinal                             */
  void*   stream;                           /* cudaStream_t for all device work                */
  int32_t rank, world;                      /* multi-GPU partition by sequence (world >= 1)    */
  uint64_t synth_seed;                      /* generator seed for the prompt-fill stand-in     */
  int32_t attn_variant;                     /* 0 = TMA-staged ring (default), 1 = register stream */
  int32_t compact_mode;                     /* 0 = row shift fused into the decode step's
                                               attention pass when the step is whole (l0 = 0,
                                               nl = L) and the evictees fit in staging
                                               (default); 1 = separate ordered-move pass in
                                               s3_evict_compact                               */
  int32_t compact_policy;                   /* 0 = shift every step (the paper, R6);
                                               1 = on demand: only when the request pool is
                                               non-empty after the step's evictions (R27)     */
  int32_t num_kv_heads;                     /* KV heads H_kv (0 = num_heads; must divide it):
                                               grouped-query / multi-query KV, query head h
                                               reads KV head h / (H / H_kv); kvpt = 4*L*H_kv*D */
  int32_t reserve_sms;                      /* SMs the persistent attention grid leaves free so
                                               kernels on other streams (the counter all-reduce
                                               of a multi-GPU step) run DURING attention instead
                                               of after it: 0 = default (none at world 1, 4 at
                                               world > 1), -1 = none, else that many (< #SMs/2) */
} s3_config;

typedef struct {                            /* caller-owned memory                             */
  void* arena;      int64_t arena_bytes;    /* device, >= (R + 8) * kvpt (8 guard rows), 256-B aligned */
  void* workspace;  int64_t workspace_bytes;/* device, >= s3_workspace_query's figure          */
  void* staging;    int64_t staging_bytes;  /* device eviction staging (0 => synchronous D2H)  */
  void* host_store; int64_t host_store_bytes; /* pinned host memory for evicted KV             */
} s3_buffers;

/* Byte sizes of the caller buffers for cfg.  staging_min is the size that
 * always lets one max-length eviction stage (max_seq_len * kvpt).          */
s3_status s3_workspace_query(const s3_config* cfg, int64_t* arena_bytes, int64_t* workspace_bytes,
                             int64_t* staging_min, int64_t* host_store_min);

/* Validate cfg, bind the buffers, create the side stream and events. */
s3_status s3_kv_init(const s3_config* cfg, const s3_buffers* bufs, s3_ctx** out);
s3_status s3_kv_destroy(s3_ctx* ctx);
const char* s3_last_error(const s3_ctx* ctx);   /* static text; never NULL */

/* ---- request pool ("A text generation query arrives in a
 * request pool in the host DRAM") -------------------------------------- */
typedef struct { int64_t req_id; int32_t prompt_len, alloc_out; } s3_request;
/* Adds fresh requests; reservation cap = prompt_len + alloc_out rows
 * (R4).  S3_E_INVAL if prompt_len < 0, alloc_out < 1, the cap
 * exceeds max_seq_len, or a req_id is already live (queued, running or
 * evicted and not yet finished) or repeats within the call; nothing is added
 * then.  S3_E_UNSCHEDULABLE if cap > arena_rows.  With world > 1 every rank
 * must submit the same requests in the same order.                         */
s3_status s3_submit(s3_ctx* ctx, const s3_request* reqs, int32_t n);

/* ---- (a)+(b): decode attention + append + overrun detection -----------
 * For every running slot b and layer l in [l0, l0+nl): write k_new/v_new
 * into row off_b + len_b and compute
 *     out[l][b][h] = softmax( q K^T / sqrt(D) ) V   over rows 0..len_b
 * (PAPER.md:106 [§2.1]; R1 self-inclusive, R2 per-head D).
 * eos (device uint8 [B]) is read only when l0+nl == L: then len, gen += 1
 * and status_b = FINISHED if eos_b or len_b == max_seq_len (a length stop,
 * DESIGN.md R28), else OVERRUN if len_b == cap_b, else RUNNING (PAPER.md:174
 * "not finished but used up its reserved memory").  S3_E_STATE if a slot has
 * no free row (len >= cap; cannot happen through this API).
 * Stream-ordered on cfg.stream, no host synchronisation.                   */
s3_status s3_decode_step(s3_ctx* ctx, int32_t l0, int32_t nl, const void* q, const void* k_new,
                         const void* v_new, const uint8_t* eos, float* out);

/* The same whole step (l0 = 0, nl = L) fed from HOST memory: the call a
 * serving loop makes when the model's q / k_new / v_new / eos arrive from the
 * host and the attention output goes back to it.
 *   q, k_new, v_new, eos : pinned host (cudaHostAlloc / torch pin_memory),
 *                          layouts as s3_decode_step with nl = L, read-only;
 *   out                  : pinned host fp32 [L][B][H][D];
 *   q_dev, k_new_dev, v_new_dev, eos_dev : caller-owned device landing
 *                          buffers of the same sizes;
 *   out_dev              : device fp32 [L][B][H][D] or NULL.  Given (and
 *                          attn_variant 0), the kernels write out_dev and a
 *                          second copy stream moves each finished batch
 *                          range to `out` (the attention warps bump a
 *                          per-range counter with a release add; the stream
 *                          waits on it with cuStreamWaitValue32, so D2H
 *                          overlaps the kernel; split-K slots follow
 *                          k_combine).  NULL (or attn_variant 2): the
 *                          kernels store `out` directly over PCIe (mapped
 *                          pinned memory);
 *   chunks               : H2D pipeline depth (0 = 16, at most 64).
 * The H2D copies are split into `chunks` contiguous batch ranges on a copy
 * stream; after each range lands a stream write sets a ready word that the
 * attention kernel's producer waits on (acquire) before it touches that
 * range, so the copies overlap the HBM stream of earlier ranges (the
 * tensor-core kernel also appends each unit's new K/V row itself).  Where
 * the attention variant cannot wait on ready words (attn_variant 1, or no
 * stream-memory-operation support), the copies complete before the kernel.
 * All buffers are in use until cfg.stream reaches the end of this call's
 * work (synchronise cfg.stream before reading `out` or reusing inputs).
 * S3_E_INVAL if a host pointer is not pinned or a landing buffer is NULL.  */
typedef struct {
  const void* q; const void* k_new; const void* v_new; const uint8_t* eos;
  float* out;
  void* q_dev; void* k_new_dev; void* v_new_dev; uint8_t* eos_dev;
  int32_t chunks;
  float* out_dev;
} s3_host_io;
s3_status s3_decode_step_host(s3_ctx* ctx, const s3_host_io* io);

/* ---- (c)+(d): eviction + row-shift compaction ------------------------- */
typedef struct {
  int64_t req_id;
  int32_t batch_index, prompt_len, gen_len, len, cap_rows, new_cap_rows;
  int64_t host_off;          /* byte offset of its rows [len][L][2][H][D] in host_store */
} s3_evicted;
typedef struct {
  int32_t n_before, n_finished, n_evicted, n_kept;
  int64_t tail_rows;         /* sum of kept caps = first free row                        */
  int64_t d2h_bytes;         /* sum over evicted of len*kvpt (== S_P, len == cap)         */
  int64_t moved_bytes;       /* sum over moved survivors of len*kvpt (one way)            */
  int64_t paper_pcie_bytes;  /* sum over evicted i of 2 S_P(x_i)   */
  int64_t paper_hbm_bytes;   /* sum over evicted i of 2 sum_{j>i} S_P(x_j)  */
  int32_t first_hole;        /* batch index of the first non-running slot, or n_before   */
  int32_t sync_evict;        /* 1 if staging was too small and the D2H ran in-stream      */
} s3_evict_report;
/* Consumes the statuses of the last complete decode step: overruns' resident
 * KV goes to host_store (async D2H on the side stream, staged through
 * `staging`), survivors are shifted up in place preserving order
 * ("shifts the rows below the blank one so that all rows are stored
 * contiguously"), finished and evicted slots leave (R6), and
 * evicted requests re-enter the pool with cap <- min(2 cap, max_seq_len)
 * (R5).  perm[b] = new batch index or -1; evicted / finished_ids list the
 * leavers in batch order.  Each output array may be NULL, else it must hold
 * n_before entries.  Synchronises the host once on a small report readback.
 * S3_E_NOMEM if the host store cannot take this step's evictees (state
 * unchanged; retry after s3_evict_wait frees reloaded ranges).  A fused step
 * only stages evictions that fit the largest free host-store block, so this
 * cannot follow a fused step unless the store fragments; if it does, the
 * evictees' rows have already left the arena and the context is poisoned.   */
s3_status s3_evict_compact(s3_ctx* ctx, s3_evict_report* rep, int32_t* perm, s3_evicted* evicted,
                           int64_t* finished_ids);
/* Blocks until the host copy of every eviction so far is complete.        */
s3_status s3_evict_wait(s3_ctx* ctx);
/* Blocks until the host copy of request req_id's last eviction is complete
 * (each evictee's D2H records its own event on the side stream); S3_OK at
 * once when no copy of req_id is pending (never evicted, already waited for,
 * or re-admitted since).  SURVEY §8(b)'s s3_evict_wait(req).               */
s3_status s3_evict_wait_req(s3_ctx* ctx, int64_t req_id);

/* ---- (e): admission by first-fit decreasing --------------------------- */
typedef struct {
  int32_t n_admitted, n_fresh, n_reloaded, n_batch;
  int64_t tail_rows;
  int64_t fill_bytes;        /* prompt rows written for fresh admissions (prefill stand-in) */
  int64_t h2d_bytes;         /* evicted KV reloaded from host_store                        */
  int64_t moved_bytes;       /* compact_policy 1 (R27): rows shifted over holes a step with an
                                empty pool left in place, before this admission (one way)  */
  int64_t stage_reload_bytes;/* evicted KV re-admitted in the step that evicted it, reloaded
                                from the device staging copy (HBM) instead of host_store   */
} s3_admit_report;
/* compact_policy 1 (R27): when requests wait and an earlier step left holes
 * (its pool was empty), s3_admit / s3_admit_home first shift the survivors
 * up (keep-scan + ordered move), so the FFD sees the free rows of the
 * every-step policy; the bytes are reported in moved_bytes.
 * world == 1: one FFD over the whole pool, fresh and evicted alike, sorted
 * by (cap desc, req_id asc), skip-and-continue, into free = R - tail rows
 * (R7-R9).  Admitted slots are appended at the
 * tail in scan order; fresh ones get their P prompt rows, evicted ones get
 * their host rows back.  admitted_ids (may be NULL) receives the admitted
 * req ids in placement order (capacity: max_running).                     */
s3_status s3_admit(s3_ctx* ctx, s3_admit_report* rep, int64_t* admitted_ids);
/* world > 1 (R26), called in this order each step:
 *   s3_admit_home    re-admit this rank's evicted requests (local FFD);
 *   s3_counters_local + an all-reduce(sum) of the [world][S3_NCOUNTERS]
 *                    matrix by the caller (torch.distributed / NCCL);
 *   s3_admit_shared  multi-bin FFD of the shared fresh pool over ranks
 *                    (free rows = column 0, free slots = column 2): items in
 *                    FFD order, each to the rank with the most free rows
 *                    among ranks with a free slot (ties: lowest rank). */
s3_status s3_admit_home(s3_ctx* ctx, s3_admit_report* rep, int64_t* admitted_ids);
s3_status s3_admit_shared(s3_ctx* ctx, const int64_t* counters_all /* [world][S3_NCOUNTERS] */,
                          s3_admit_report* rep, int64_t* admitted_ids);
s3_status s3_counters_local(const s3_ctx* ctx, int64_t row[S3_NCOUNTERS]);

/* ---- (a8): the counter exchange over a library-owned NCCL communicator --
 * The supervisor "passes the information to the scheduler":
 * with ranks partitioned by sequence (R26) that is one all-reduce
 * (sum) of the [world][S3_NCOUNTERS] int64 matrix per step, between
 * s3_admit_home and s3_admit_shared.  NCCL is loaded at run time
 * (dlopen "libnccl.so.2" -- in a torch process, torch's copy); without it the
 * calls return S3_E_NCCL and the caller may all-reduce s3_counters_local
 * rows itself (torch.distributed) instead.
 *   s3_nccl_get_unique_id  rank 0 creates the id; the caller broadcasts its
 *                          S3_NCCL_ID_BYTES bytes to every rank (e.g.
 *                          torch.distributed.broadcast_object_list);
 *   s3_comm_init           every rank binds it (collective; rank / world from
 *                          s3_config).  The communicator, its stream (highest
 *                          priority, non-blocking) and a [world][S3_NCOUNTERS]
 *                          device + pinned host buffer belong to the context
 *                          (freed by s3_kv_destroy).  S3_E_STATE if already bound;
 *   s3_exchange_counters   fills this rank's row (s3_counters_local), all-reduces
 *                          the matrix on the communicator's stream -- which does
 *                          not wait for cfg.stream, so it runs while this step's
 *                          attention pass still streams (the persistent attention
 *                          grids leave s3_config.reserve_sms SMs free) -- and
 *                          returns it in counters_all (blocking until it is back);
 *   s3_counters_get        the last exchanged matrix as per-rank / total counters
 *                          (before any exchange: this rank's row alone).        */
#define S3_NCCL_ID_BYTES 128
#define S3_MAX_RANKS 64
s3_status s3_nccl_get_unique_id(uint8_t id[S3_NCCL_ID_BYTES]);
s3_status s3_comm_init(s3_ctx* ctx, const uint8_t id[S3_NCCL_ID_BYTES]);
s3_status s3_exchange_counters(s3_ctx* ctx, int64_t* counters_all /* [world][S3_NCOUNTERS] */);
typedef struct {
  int32_t world, exchanges;                       /* ranks; exchanges so far                  */
  int64_t rank_free_rows[S3_MAX_RANKS], rank_running[S3_MAX_RANKS];
  int64_t free_rows_total, running_total, evicted_waiting_total;
  int64_t fresh_waiting;                          /* the shared pool (identical on every rank) */
  int64_t finished_total, evicted_total, tokens_total;
} s3_counters;
s3_status s3_counters_get(const s3_ctx* ctx, s3_counters* counters);

/* ---- pure host planning helpers (no device work; callable without a GPU) */
/* Single-bin FFD: admitted[i] = 1 if item i is admitted.  Returns count.  */
int32_t s3_plan_ffd(int32_t n, const int64_t* cap, const int64_t* req_id, int64_t free_rows,
                    int32_t max_items, uint8_t* admitted);
/* Multi-bin FFD (worst fit over bins, R26): rank[i] = bin or -1;
 * free_rows / free_slots updated.                                          */
int32_t s3_plan_ffd_multibin(int32_t n, const int64_t* cap, const int64_t* req_id, int32_t world,
                             int64_t* free_rows, int64_t* free_slots, int32_t* rank);

/* ---- views ------------------------------------------------------------ */
typedef struct { int64_t req_id; int32_t prompt_len, gen_len, len, cap_rows; int64_t off; } s3_slot;
s3_status s3_batch_size(const s3_ctx* ctx, int32_t* B);
s3_status s3_batch_view(const s3_ctx* ctx, s3_slot* slots /* [B] */, int32_t* B);

/* ---- timing of the two dominant kernels (CUDA events on cfg.stream) ----- */
typedef struct {
  int64_t kernel_launches;          /* every kernel this context launched (always counted) */
  int64_t attn_launches, move_launches, fused_steps;
  double attn_ms, move_ms;          /* summed kernel durations                   */
  double attn_bytes, move_bytes;    /* algorithmic bytes of those launches        */
  double fused_move_bytes;          /* row-shift + staging bytes written by the attention
                                       launches of fused steps (part of their traffic)  */
  int64_t d2h_copies, h2d_copies;   /* eviction D2H batches / reload H2D copies timed   */
  double d2h_ms, d2h_bytes;         /* eviction copies (side stream, overlapped)        */
  double h2d_ms, h2d_bytes;         /* reload copies (main stream)                       */
  double d2h_overlap_ms;            /* part of d2h_ms during which an attention kernel ran
                                       (CUDA-event intervals on both streams)             */
  int64_t prep_launches;            /* k_prep launches timed (detection + keep-scan)     */
  double prep_ms;                   /* their summed durations                           */
} s3_profile;
s3_status s3_profile_enable(s3_ctx* ctx, int32_t on);   /* also resets the sums */
s3_status s3_profile_get(s3_ctx* ctx, s3_profile* prof); /* synchronises          */

/* ---- synthetic stand-ins (harness, not the method) ---------------------
 * s3_synth_inputs: the model's QKV projection + sampler stand-in; writes q,
 * k_new, v_new for layers [l0, l0+nl) at position len_b of every slot from
 * the counter-based generator and
 * eos_b = (gen_b + 1 == out_len_by_req[req_b]).  out_len_by_req: device
 * int32 [n_req] indexed by req_id.                                          */
s3_status s3_synth_inputs(s3_ctx* ctx, int32_t l0, int32_t nl, const int32_t* out_len_by_req,
                          int64_t n_req, void* q, void* k_new, void* v_new, uint8_t* eos);
/* Counts resident arena rows (all layers, K and V) that differ from the
 * generator (invariant P2).  Synchronises.                                  */
s3_status s3_verify_resident(s3_ctx* ctx, int64_t* bad_rows);

/* ---- batch-dependent decode cost ------------------------
 * The projections around attention share their weights across the batch, so
 * their cost per token falls as the batch grows -- the effect behind the
 * paper's ORCA vs S^3 vs Oracle throughput gap ("the
 * feed-forward layers ... batched", 247-249).  s3_gemm runs one such
 * projection on the tcgen05 tensor cores:
 *     D[M][N] = epi( A[M][K] . W[N][K]^T ),  bf16 operands, fp32 accumulate,
 *     epi 0: D = acc;  1: D = gelu_tanh(acc);  2: D = C + acc   (bf16 out).
 *   a      device bf16 [M][K] row-major (the batch's activations, M = B);
 *   w      device bf16 [N][K] row-major (the weight, nn.Linear layout);
 *   d[i]   device bf16 [M][seg_cols]: column segment i = columns
 *          [i seg_cols, (i+1) seg_cols) of D (N / seg_cols <= 3 segments, e.g.
 *          the QKV projection straight into q, k_new, v_new); unused = NULL;
 *   c      epi 2: device bf16 [M][N] (may be d[0], in place), else NULL.
 * K % 64 == 0, N % 128 == 0, seg_cols % 128 == 0; 16-B aligned pointers.
 * Stream-ordered on `stream` (a cudaStream_t); no context needed.  Launched
 * with programmatic dependent launch: a following s3_gemm's CTAs may start
 * (prologue only; every global access waits for this grid) on SMs this one
 * has left; the ordering a stream guarantees is unchanged.
 * S3_E_INVAL on a bad shape or pointer, S3_E_CUDA on a launch error.      */
typedef struct {
  const void* a; const void* w; void* d[3]; const void* c;
  int32_t M, N, K, seg_cols, epi;
  void* workspace; int64_t workspace_bytes;  /* device scratch for split-K partials
                                                (zero-filled once by the caller;
                                                every call leaves it reusable), or
                                                NULL: no split-K                  */
} s3_gemm_args;
s3_status s3_gemm(void* stream, const s3_gemm_args* g);
/* Workspace s3_gemm would use for this shape (0: it runs without).  Small
 * batches split K over idle SMs; a smaller workspace only limits the split. */
s3_status s3_gemm_workspace(const s3_gemm_args* g, int64_t* bytes);
/* dst (bf16, device) = round-to-nearest(src (fp32, device)), n elements
 * (n % 4 == 0, 16-B aligned): the attention output as the next GEMM's A.  */
s3_status s3_cast_bf16(void* stream, const float* src, void* dst, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* S3_H */
