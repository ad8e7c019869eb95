// s3_internal.h -- shared between the host control plane (s3_host.cpp) and
// the device kernels (s3_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace s3 {

// Device slot record (AoS, 32 B), kept in arena order.
struct DSlot {
  int64_t req;
  int32_t prompt, gen, len, cap, off, status;
};
static_assert(sizeof(DSlot) == 32, "DSlot must be 32 B");

// One attention work unit: rows [r0, r1) of slot b's resident rows, plus the
// new (appended) row when has_new.  part < 0: the unit covers the whole slot
// and writes `out` directly; else it writes partial (m, l, acc) record `part`.
//
// Fused attend-and-shift (compact_mode 0): mode says where the unit's rows go
// while they stream through shared memory: 0 = stay (only the new row is
// written, at off+len), 1 = move to arena rows dst+r, 2 = copy to the
// staging buffer at byte dst + r*kvpt (evicted), 3 = nowhere (finished).
enum { UNIT_STAY = 0, UNIT_MOVE = 1, UNIT_STAGE = 2, UNIT_DROP = 3 };
struct Unit {
  int32_t b, r0, r1, part;
  int32_t off, len, has_new, mode;
  int64_t dst;
  int32_t stage_base, pad;   // pad: eviction index of a STAGE unit (its staged-row counter)
};
static_assert(sizeof(Unit) == 48, "Unit must be 48 B");

// Per ring stage of a moving unit: the source units whose rows overlap the
// stage's destination rows, and how many of their rows must have been read
// (units strictly between ua and ub must be read completely).
struct DepDesc {
  int32_t ua, need_a, ub, need_b;
};
constexpr int AT_RPS = 4;      // rows per attention ring stage

struct Split {          // a slot whose attention is split over k units
  int32_t b, part0, k, pad;
};

enum { MOVE_ARENA = 0, MOVE_STAGE = 1 };
struct MoveEntry {      // one contiguous byte range to move, sources in arena order
  int64_t src, dst, bytes, chunk0;
  int32_t kind, pad0;
  int64_t pad1;
};
static_assert(sizeof(MoveEntry) == 48, "MoveEntry must be 48 B");

// ctrl words (int32 unless noted)
enum { CTRL_N_UNITS = 0, CTRL_N_SPLITS = 1, CTRL_ITEM = 2, CTRL_SPLIT_ITEM = 3, CTRL_FUSED = 4,
       CTRL_N_STAGES = 5, CTRL_WORDS = 16 };
// int64 ctrl words (separate array)
enum { CTRL64_TICKET = 0, CTRL64_N_CHUNKS = 1, CTRL64_WORDS = 8 };

// Packed report written by the keep-scan kernel; header then, for the
// pre-compaction batch size B: perm int32[B] | DEvicted[B] | int64 fin[B].
struct DReportHeader {
  int32_t n_before, n_finished, n_evicted, n_kept;
  int64_t tail, d2h_bytes, moved_bytes, pcie_bytes, hbm_bytes;
  int64_t n_chunks;
  int32_t n_entries, first_hole;
  int32_t fused, compacted;    // fused: the decode step already moved / staged the rows;
                               // compacted: survivors were shifted to prefix-sum offsets
  int64_t pad[6];
};
static_assert(sizeof(DReportHeader) == 128, "header 128 B");
struct DEvicted {
  int64_t req;
  int32_t b, prompt, gen, len, cap, pad;
  int64_t stage_off;
};
static_assert(sizeof(DEvicted) == 40, "DEvicted 40 B");

#ifdef __CUDACC__
#define S3_HD __host__ __device__
#else
#define S3_HD
#endif
S3_HD inline int64_t report_perm_off(int32_t) { return sizeof(DReportHeader); }
S3_HD inline int64_t report_ev_off(int32_t B) { return (sizeof(DReportHeader) + 4 * (int64_t)B + 15) / 16 * 16; }
S3_HD inline int64_t report_fin_off(int32_t B) { return report_ev_off(B) + (int64_t)sizeof(DEvicted) * B; }
S3_HD inline int64_t report_bytes(int32_t B) { return report_fin_off(B) + 8 * (int64_t)B; }

struct Shape {
  int32_t L, H, D, max_len;
  int32_t Hkv, pad;      // KV heads (grouped-query attention; Hkv == H is MHA)
  int64_t row_elems;     // 2*L*Hkv*D bf16 elements per token row
  int64_t kvpt;          // bytes per token row
};

// ---- kernel launchers (s3_kernels.cu) ----------------------------------
struct PrepArgs {
  Shape sh;
  DSlot* slots;        // current table (updated in place when not fused)
  DSlot* next;         // gathered table for the next step (fused only)
  int32_t B, C;
  const uint8_t* eos;
  int32_t finalize, fuse;
  int32_t compact_policy, pool_nonempty;   // on-demand compaction inputs (R27)
  int64_t staging_bytes;
  Unit* units;
  Split* splits;
  int32_t* ctrl;
  uint8_t* report;      // fused: the host-mapped pinned report (written over PCIe, no copy engine)
  int32_t* fused_out;   // host-mapped word: 1 if this step fused the row shift (or nullptr)
  // multi-CTA scan (B > PREP_CTA_SLOTS): per-CTA totals published with an epoch flag,
  // per-CTA header partials combined by the last CTA to finish
  long long* xagg;      // [PREP_MAX_CTAS][PREP_NX] block totals
  unsigned long long* xflag;   // [PREP_MAX_CTAS] epoch of the published totals
  long long* xpart;     // [PREP_MAX_CTAS][4] first_hole, hbm, moved, end
  int32_t* xdone;       // CTAs finished (reset by the last)
  uint32_t epoch;
};
constexpr int PREP_CTA_SLOTS = 1024;   // k_prep runs as one CTA up to 2 * PREP_CTA_SLOTS slots
constexpr int PREP_MAX_CTAS = 64;      // B <= 65535
constexpr int PREP_NX = 10;            // scanned quantities per slot
cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st);
cudaError_t launch_deps(const Unit* units, const int32_t* ctrl, DepDesc* desc, int32_t tc, int32_t grid,
                        cudaStream_t st);
// Host-fed step (s3_decode_step_host): slot b's q / k_new / v_new have landed
// once ready[b / cb] reaches epoch (written by the copy stream).  ready ==
// nullptr: inputs are resident before the launch.
struct Feed {
  const uint32_t* ready = nullptr;
  int32_t cb = 1;
  uint32_t epoch = 0;
  uint32_t* done = nullptr;    // per-chunk count of consumer warps whose final out rows are stored
};
cudaError_t launch_attn(const Shape& sh, const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                        uint16_t* arena, uint8_t* staging, float* out, float* partials, const Unit* units,
                        const Split* splits, const DepDesc* desc, unsigned long long* progress, uint32_t epoch,
                        int32_t* ctrl, int32_t B, int32_t l0, int32_t nl, int32_t grid_attn, int32_t grid_combine,
                        int32_t variant, const Feed& feed, uint32_t* evdone, cudaStream_t st);
cudaError_t launch_keep_scan(const Shape& sh, const DSlot* cur, DSlot* next, int32_t B, int64_t S,
                             void* report, MoveEntry* entries, int32_t* key_chunk0, int32_t* key_src,
                             int64_t* ctrl64, int32_t compact_policy, int32_t pool_nonempty, cudaStream_t st);
cudaError_t launch_move(uint8_t* arena, uint8_t* staging, const MoveEntry* entries, const int32_t* key_chunk0,
                        const int32_t* key_src, int32_t n_entries, int64_t n_chunks, int64_t S, int64_t kvpt,
                        int64_t* ctrl64, uint32_t* flags, uint32_t epoch, int32_t staging_enabled, int32_t grid,
                        cudaStream_t st);
int move_smem_bytes(int64_t S, int32_t n_entries, int32_t* keys_in_smem);
cudaError_t launch_fill(const Shape& sh, uint64_t seed, const DSlot* slots, const int32_t* list,
                        int32_t n, int32_t max_prompt, uint16_t* arena, cudaStream_t st);
cudaError_t launch_synth(const Shape& sh, uint64_t seed, const DSlot* slots, int32_t B, int32_t l0,
                         int32_t nl, const int32_t* out_len_by_req, int64_t n_req, uint16_t* q,
                         uint16_t* k, uint16_t* v, uint8_t* eos, cudaStream_t st);
cudaError_t launch_verify(const Shape& sh, uint64_t seed, const DSlot* slots, int32_t B,
                          const uint16_t* arena, unsigned long long* bad, cudaStream_t st);

// grouped-KV tensor-core path (s3_attn_tc.cu), attn_variant 2
cudaError_t launch_append(const Shape& sh, const DSlot* slots, int32_t B, int32_t l0, int32_t nl,
                          const uint16_t* k_new, const uint16_t* v_new, uint16_t* arena, cudaStream_t st);
bool attn_tc_supported(const Shape& sh);
int attn_tc_smem(int nc);
const void* attn_tc_kernel_ptr(int nc, bool pack, bool feed, bool r33);

cudaError_t launch_attn_tc(const Shape& sh, const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                           uint16_t* arena, int64_t arena_rows, uint8_t* staging, int64_t staging_bytes, float* out,
                           float* partials, const Unit* units, const Split* splits, const DepDesc* desc,
                           unsigned long long* progress, uint32_t epoch, int32_t* ctrl, int32_t B, int32_t l0,
                           int32_t nl, int32_t grid_attn, int32_t grid_combine, const Feed& feed, uint32_t* evdone,
                           int32_t mean_rows, int32_t nc_pick, cudaStream_t st);
cudaError_t launch_combine(const Shape& sh, const Split* splits, float* partials, float* out, int32_t* ctrl,
                           int32_t B, int32_t nl, int32_t grid, cudaStream_t st);

// bf16 tcgen05 GEMM (s3_gemm.cu): D = epi(A . W^T); see include/s3.h s3_gemm
struct GemmCall {
  const void* a;       // [M][K] bf16
  const void* w;       // [N][K] bf16
  void* d[3];          // output column segments [M][seg_cols] bf16
  const void* c;       // epi 2: [M][N] bf16 addend (may equal d[0])
  int32_t M, N, K, seg_cols, epi;
  void* workspace;     // split-K partials + counters (zeroed once), or NULL
  int64_t workspace_bytes;
};
int64_t gemm_workspace_bytes(const GemmCall& g);   // -1 on a bad shape
cudaError_t launch_gemm(const GemmCall& g, cudaStream_t st);
cudaError_t launch_cast_bf16(const float* src, void* dst, int64_t n, cudaStream_t st);

int attn_block_threads(const Shape& sh);
int attn_tma_stages(const Shape& sh);
int attn_tma_smem(const Shape& sh, int ns);
const void* attn_tma_kernel_ptr(const Shape& sh);
const void* attn_kernel_ptr(const Shape& sh);
const void* move_kernel_ptr();

}  // namespace s3
