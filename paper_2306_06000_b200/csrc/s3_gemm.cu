// s3_gemm.cu -- bf16 GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA)
// for the batch-dependent part of a decode step: the QKV,
// output and feed-forward projections of a GPT-J-shaped layer at M = B
// running sequences.  Their weights are shared by the whole batch, which is
// why a larger batch -- what S^3's length prediction buys (PAPER.md:168,
// 247-249) -- raises throughput; attention is the part that does not batch.
//
//   D[M][N] = epi( A[M][K] . W[N][K]^T )     A, W bf16 (K-major), fp32 accumulate
//   epi: STORE (bf16), GELU (tanh form, then bf16), ADD (D = C + acc, bf16; C may alias D)
//   D may be split into column segments of seg_cols columns (QKV -> q, k, v buffers).
//
// One persistent CTA per SM, 6 warps:
//   warp 0  TMA producer: per K block one 2-D box of A [128 x 64] and one of W
//           [BN x 64] (128B swizzle) into a ring of up to 6 stages (mbarrier full / empty);
//   warp 1  MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16,
//           M 128, N BN, K 16 (4 per K block), into one of two TMEM
//           accumulators (2 x BN fp32 columns), commits the stage back to the
//           producer and the finished accumulator to the epilogue;
//   warps 2-5 epilogue: tcgen05.ld 32 columns at a time (warp w reads TMEM
//           lanes 32 (w % 4) ..), applies the epilogue, stores bf16 rows; the
//           accumulator is released as soon as it has been read, so the next
//           tile's MMAs overlap this tile's stores.
// Tiles are walked n-major (the M tiles of one W column block run on
// neighbouring CTAs at the same time, so W streams from HBM once and the
// small A operand stays in L2).
// Small batches (M <= 64, SW = true): the operands swap roles -- the MMA's
// 128-row M side is a block of W rows and its N side (BN = 64) the
// batch, so a K block moves 16 KB of weights plus only BN x 128 B of
// activations (instead of a 128-row activation tile mostly zero-filled), and
// TMEM holds D^T: the epilogue transposes 32 x 32 blocks through shared memory
// into the row-major output.
// CTA pairs (cta_group::2, 256 x 256 tiles) for large M; stream-K over the
// ragged last wave, the groups sharing a tile adding their fp32 partials into
// one workspace tile by TMA reduce-add (the last to arrive reads it once).
// Programmatic dependent launch: the next GEMM's prologue overlaps this one's
// tail; every global access waits in griddepcontrol.wait.  DESIGN.md §10 NEXT-2.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "s3_internal.h"

namespace s3 {
namespace {

constexpr int GM = 128;          // tile rows (MMA M)
constexpr int GK = 64;           // K block: one 128-byte swizzle atom of bf16

constexpr int G_THREADS = 6 * 32;

__device__ __forceinline__ uint32_t gsu32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g_mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(gsu32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void g_mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gsu32(b)) : "memory");
}
__device__ __forceinline__ void g_mb_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gsu32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void g_mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
          gsu32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void g_tma2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(gsu32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(gsu32(bar))
      : "memory");
}
// K-major operand in 128B-swizzled smem: rows of 128 B, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t g_desc(const void* p) {
  return (uint64_t)((gsu32(p) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: bf16 x bf16 -> f32, both K-major, M m, N n
__host__ __device__ constexpr uint32_t g_idesc(int n, int m) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void g_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void g_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)gsu32(b)) : "memory");
}
__device__ __forceinline__ void g_tmem_ld32(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float gelu_tanh(float x) {
  // 0.5 x (1 + tanh( sqrt(2/pi) (x + 0.044715 x^3) ))  (GPT-J's "gelu_new")
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.f + t);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// as many ring stages as fit next to the epilogue staging (227 KB per CTA; 1 KB alignment
// slack + barriers), at most 6: deep rings keep enough weight bytes in flight when M is
// small and the GEMM streams W at HBM speed
__host__ __device__ constexpr int gemm_stages(int stage_bytes) {
  return (227 * 1024 - 4 * 16384 - 1024 - 512) / stage_bytes < 6 ? (227 * 1024 - 4 * 16384 - 1024 - 512) / stage_bytes
                                                                  : 6;
}

struct GemmMaps {
  CUtensorMap a, w;      // operands (loads)
  CUtensorMap d[3];      // output column segments (stores, box {64, 32})
  CUtensorMap c;         // epi 2 addend (loads, box {64, 32})
  CUtensorMap p;         // split-K fp32 partials (stores / loads, box {32, 32})
};
struct GemmArgs {
  int32_t M, N, K, epi, seg_cols, m_tiles, n_tiles;
  int32_t stage_tx;       // bytes one ring stage receives (SW: the activation box holds only the
                          //   batch's rows rounded to 8; the rest of its BN rows stay stale and
                          //   only feed D^T columns past M, which are never stored)
  int32_t dp_tiles;       // tiles [0, dp_tiles) data parallel, the rest stream-K (equal K-block ranges per group)
  int32_t cmax;           // stream-K: most CTA groups contributing to one tile (partial slots = cmax - 1)
  int32_t* cnt;           // stream-K: per (tile, CTA of the pair) [claim, done] counters (zero between calls)
  int32_t wpre;           // PDL: load the first stages' weight boxes before waiting for the previous grid
  int32_t red;            // stream-K: 1 = contributors TMA-reduce-add into one fp32 tile per tile (zero between
                          //   calls; the reducer reads it once and re-zeroes it), 0 = one partial slot each
};

// Work of one CTA group: whole tiles g, g + G, ... below dp_tiles (data
// parallel, n-major, so neighbouring groups share W blocks in L2), then --
// stream-K -- the K blocks [start(g), start(g+1)) of the remaining tiles'
// tile-major K-block sequence, cut at tile boundaries.  A tile touched by
// several groups (ncontrib > 1) is summed by the last group to finish its part.
struct Work {
  int tile, kb0, kb1, ncontrib;
};
struct WorkIter {
  int64_t dp_pos, pos, end, total;     // total: K blocks of the stream-K tiles
  int G, kblocks, dp_tiles;
  __host__ __device__ int64_t start(int grp) const { return (int64_t)grp * total / G; }
  __host__ __device__ int group_of(int64_t x) const {   // the group whose stream-K range holds K block x
    int grp = (int)(x * G / total);
    while (grp + 1 < G && start(grp + 1) <= x) ++grp;
    while (grp > 0 && start(grp) > x) --grp;
    return grp;
  }
  __host__ __device__ void init(int g, int groups, int tiles, int kb, int dp) {
    G = groups; kblocks = kb; dp_tiles = dp;
    dp_pos = g;
    total = (int64_t)(tiles - dp) * kb;
    pos = total ? start(g) : 0;
    end = total ? start(g + 1) : 0;
  }
  __host__ __device__ bool next(Work& w) {
    if (dp_pos < dp_tiles) {
      w.tile = (int)dp_pos; w.kb0 = 0; w.kb1 = kblocks; w.ncontrib = 1;
      dp_pos += G;
      return true;
    }
    if (pos >= end) return false;
    const int st = (int)(pos / kblocks);
    w.tile = dp_tiles + st;
    w.kb0 = (int)(pos - (int64_t)st * kblocks);
    const int64_t rest = (int64_t)w.kb0 + (end - pos);
    w.kb1 = rest < kblocks ? (int)rest : kblocks;
    w.ncontrib = group_of((int64_t)(st + 1) * kblocks - 1) - group_of((int64_t)st * kblocks) + 1;
    pos += w.kb1 - w.kb0;
    return true;
  }
};
__device__ __forceinline__ void g_tma_reduce_add2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(gsu32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void g_tma_store2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(gsu32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// 128B-swizzled staging tile of 32 rows x 128 B: 16-B chunk j of row r sits at chunk j ^ (r & 7)
__device__ __forceinline__ uint32_t swz(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }
__device__ __forceinline__ void sts128(uint8_t* base, uint32_t off, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(gsu32(base) + off), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(const uint8_t* base, uint32_t off) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(gsu32(base) + off)
               : "memory");
  return v;
}
constexpr int EPI_WARP_BYTES = 16384;   // per epilogue warp: 2 output + 2 input staging tiles of 4 KB

__device__ __forceinline__ bool g_elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// CTA pair: both CTAs' TMA loads complete on the leader's (rank 0) barrier
__device__ __forceinline__ void g_tma2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(gsu32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(gsu32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void g_mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// completion of the pair's MMAs arrives on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void g_commit_pair(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          gsu32(b)),
      "h"((uint16_t)3)
      : "memory");
}
// arrive on the leader CTA's barrier at the same offset
__device__ __forceinline__ void g_arrive_leader(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(gsu32(b) & 0xFEFFFFFFu) : "memory");
}

// CG = 1: one CTA per 128 x BN tile (tcgen05 cta_group::1, M 128).
// CG = 2: a CTA pair per 256 x BN tile (cta_group::2, M 256): each CTA loads
//   its 128 rows of A and half (BN/2 rows) of the W tile, the leader issues
//   the MMAs (the tensor cores read both CTAs' shared memory), each CTA's
//   TMEM holds its 128 accumulator rows.  W is read from L2 once per 256 rows
//   instead of once per 128, halving the operand traffic per flop.
// SW (CG = 1 only): maps.a is W (128-row boxes), maps.w the activations (BN-row
//   boxes); tile t covers W rows (t % m_tiles) x 128 and batch rows (t / m_tiles) x BN,
//   and the accumulator is D^T (TMEM lane = output column, column = batch row).
template <int BN, int CG, bool SW = false>
__global__ void __launch_bounds__(G_THREADS, 1) k_gemm(const __grid_constant__ GemmMaps maps, GemmArgs a) {
  static_assert(!SW || CG == 1, "swapped operands use single-CTA tiles");
  constexpr int A_BYTES = GM * GK * 2, W_BYTES = (BN / CG) * GK * 2, STAGE = A_BYTES + W_BYTES;
  constexpr int NSTG = gemm_stages(STAGE);
  constexpr int TMEM_COLS = 2 * BN;
  constexpr int TM_ROWS = GM * CG;                     // rows per tile
  extern __shared__ __align__(1024) uint8_t gsmem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsmem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_smem = smem + NSTG * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + 4 * EPI_WARP_BYTES);
  uint64_t* empty = full + NSTG;
  uint64_t* tfull = empty + NSTG;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;                        // [4 epilogue warps][2 input tiles]
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(inbar + 8);
  int32_t* s_role = reinterpret_cast<int32_t*>(tmem_base + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int unit0 = (int)blockIdx.x / CG, nunits = (int)gridDim.x / CG;   // tile scheduler per CTA group
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTG; ++i) { g_mb_init(&full[i], 1); g_mb_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { g_mb_init(&tfull[i], 1); g_mb_init(&tempty[i], 4 * CG); }
    for (int i = 0; i < 8; ++i) g_mb_init(&inbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.w) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gsu32(tmem_base)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gsu32(tmem_base)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base;
  const int tiles = a.m_tiles * a.n_tiles;
  const int kblocks = a.K / GK;
  auto work = [&]() {
    WorkIter w;
    w.init(unit0, nunits, tiles, kblocks, a.dp_tiles);
    return w;
  };

  // The producer and MMA roles run warp-wide with warp-uniform operands and one elected
  // lane issuing: a tcgen05.mma / TMA operand the compiler cannot prove uniform costs an
  // ELECT / R2UR.BROADCAST loop around every instruction (see s3_attn_tc.cu, uni()).
  // Programmatic dependent launch: let the next kernel on the stream start its CTAs on the
  // SMs this grid leaves (its prologue and weight prefetch overlap our tail); everything
  // that reads or writes data another kernel produces or consumes waits for the previous
  // grid (griddepcontrol.wait returns at once without a PDL launch).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    int s = 0;
    uint32_t ph = 0;
    WorkIter wi = work();
    // opt-in (S3_GEMM_PDL=2), CG = 1: the weight boxes of the first ring stages are loaded
    // BEFORE waiting for the previous grid -- only valid when the kernel just before this one
    // on the stream did not write W (off by default); their activation boxes follow the wait
    int pre = 0;
    bool waited = false;
    if constexpr (CG == 1) {
      WorkIter w0 = wi;
      Work wk;
      if (a.wpre && w0.next(wk)) {
        const int t = wk.tile;
        const int m0 = (t % a.m_tiles) * TM_ROWS, n0 = (t / a.m_tiles) * BN;
        pre = min(NSTG, wk.kb1 - wk.kb0);
        if (g_elect_one()) {
          for (int i = 0; i < pre; ++i) {
            uint8_t* sa = smem + i * STAGE;
            const int kb = wk.kb0 + i;
            g_mb_expect(&full[i], (uint32_t)a.stage_tx);
            if constexpr (SW) g_tma2d(sa, &maps.a, kb * GK, m0, &full[i]);            // W rows
            else g_tma2d(sa + A_BYTES, &maps.w, kb * GK, n0, &full[i]);
          }
        }
        __syncwarp();
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (Work wk; wi.next(wk);) {
      const int t = wk.tile;
      const int m0 = (t % a.m_tiles) * TM_ROWS + (int)rank * GM;
      const int n0 = (t / a.m_tiles) * BN + (int)rank * (BN / CG);
      for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
        uint8_t* sa = smem + s * STAGE;
        if (!waited && pre > 0) {   // a prefetched stage: its activation box only
          if (g_elect_one()) {
            if constexpr (SW) g_tma2d(sa + A_BYTES, &maps.w, kb * GK, n0, &full[s]);
            else g_tma2d(sa, &maps.a, kb * GK, m0, &full[s]);
          }
          __syncwarp();
          if (--pre == 0) waited = true;
          if (++s == NSTG) { s = 0; ph ^= 1u; }
          continue;
        }
        g_mb_wait(&empty[s], ph ^ 1u);
        if (g_elect_one()) {
          if constexpr (CG == 1) {
            g_mb_expect(&full[s], (uint32_t)a.stage_tx);
            g_tma2d(sa, &maps.a, kb * GK, m0, &full[s]);
            g_tma2d(sa + A_BYTES, &maps.w, kb * GK, n0, &full[s]);
          } else {
            if (leader) g_mb_expect(&full[s], (uint32_t)(2 * STAGE));   // both CTAs' bytes
            g_tma2d_pair(sa, &maps.a, kb * GK, m0, &full[s]);
            g_tma2d_pair(sa + A_BYTES, &maps.w, kb * GK, n0, &full[s]);
          }
        }
        __syncwarp();
        if (++s == NSTG) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (leader) {
      constexpr uint32_t id = g_idesc(BN, TM_ROWS);
      const uint32_t tm = (uint32_t)__shfl_sync(0xffffffffu, (int)tmem, 0);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      WorkIter wi = work();
      for (Work wk; wi.next(wk); ++it) {
        const int acc = it & 1;
        g_mb_wait(&tempty[acc], ((uint32_t)(it >> 1) & 1u) ^ 1u);   // the epilogue(s) drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tm + (uint32_t)(acc * BN);
        const int kb0 = wk.kb0, kb1 = wk.kb1;
        for (int kb = kb0; kb < kb1; ++kb) {
          g_mb_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sa = smem + s * STAGE;
          const uint64_t da = g_desc(sa), dw = g_desc(sa + A_BYTES);
          if (g_elect_one()) {   // MMAs and their commits from the same lane
#pragma unroll
            for (int k = 0; k < GK / 16; ++k) {      // +32 B per K = 16 inside the swizzle atom
              if constexpr (CG == 1) g_mma(d, da + (uint64_t)(k * 2), dw + (uint64_t)(k * 2), id, kb > kb0 || k);
              else g_mma_pair(d, da + (uint64_t)(k * 2), dw + (uint64_t)(k * 2), id, kb > kb0 || k);
            }
            // the stage is free once these MMAs have read it (in both CTAs of a pair)
            if constexpr (CG == 1) g_commit(&empty[s]); else g_commit_pair(&empty[s]);
            if (kb == kb1 - 1) {   // accumulator complete
              if constexpr (CG == 1) g_commit(&tfull[acc]); else g_commit_pair(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++s == NSTG) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else {
    // -------------------------------- epilogue --------------------------------
    // Warp w owns TMEM lanes 32 (w % 4) .. + 31 = 32 rows of the CTA's 128.  Values go
    // TMEM -> registers -> a 128B-swizzled staging tile -> one TMA store per 32 x 64
    // bf16 chunk (coalesced, asynchronous); addends and partials come in by TMA loads.
    asm volatile("griddepcontrol.wait;" ::: "memory");   // C, D, workspace: the previous grid is done
    const int quarter = warp & 3;
    uint8_t* eb = epi_smem + quarter * EPI_WARP_BYTES;
    uint64_t* ib = inbar + quarter * 2;
    uint32_t iph[2] = {0u, 0u};
    int ob = 0;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    auto load_in = [&](int buf, const CUtensorMap* map, int x, int y, uint32_t bytes = 4096u) {
      if (lane == 0) {
        g_mb_expect(&ib[buf], bytes);
        g_tma2d(eb + 8192 + buf * 4096, map, x, y, &ib[buf]);
      }
    };
    auto wait_in = [&](int buf) { g_mb_wait(&ib[buf], iph[buf]); iph[buf] ^= 1u; };
    auto out_tile = [&]() -> uint8_t* {        // the staging tile a TMA store finished reading
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      return eb + ob * 4096;
    };
    auto store_out = [&](const CUtensorMap* map, int x, int y, bool reduce_add = false) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (reduce_add) g_tma_reduce_add2d(map, x, y, eb + ob * 4096);
        else g_tma_store2d(map, x, y, eb + ob * 4096);
      }
      ob ^= 1;
    };
    // 64 accumulator columns -> epilogue (C already summed in for epi 2 by the caller) -> bf16 store
    auto finish64 = [&](float (&v)[64], const CUtensorMap* dmap, int x, int y) {
      if (a.epi == 1) {
#pragma unroll
        for (int i = 0; i < 64; ++i) v[i] = gelu_tanh(v[i]);
      }
      uint8_t* o = out_tile();
#pragma unroll
      for (int j = 0; j < 8; ++j)
        sts128(o, swz(lane, j), make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                           pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                                           pack_bf16(v[8 * j + 6], v[8 * j + 7])));
      store_out(dmap, x, y);
    };
    auto add_c = [&](float (&v)[64], int buf) {   // v += C tile in input buffer buf
      wait_in(buf);
      const uint8_t* cb = eb + 8192 + buf * 4096;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 x = lds128(cb, swz(lane, j));
        v[8 * j + 0] += bf16_lo(x.x); v[8 * j + 1] += bf16_hi(x.x);
        v[8 * j + 2] += bf16_lo(x.y); v[8 * j + 3] += bf16_hi(x.y);
        v[8 * j + 4] += bf16_lo(x.z); v[8 * j + 5] += bf16_hi(x.z);
        v[8 * j + 6] += bf16_lo(x.w); v[8 * j + 7] += bf16_hi(x.w);
      }
      __syncwarp();
    };
    auto add_p = [&](float* v, int buf) {         // 32 values += fp32 partial tile in input buffer buf
      wait_in(buf);
      const uint8_t* pb = eb + 8192 + buf * 4096;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 x = lds128(pb, swz(lane, j));
        v[4 * j + 0] += __uint_as_float(x.x); v[4 * j + 1] += __uint_as_float(x.y);
        v[4 * j + 2] += __uint_as_float(x.z); v[4 * j + 3] += __uint_as_float(x.w);
      }
      __syncwarp();
    };
    // SW: 32 accumulator columns (batch rows y .. y+31) of this lane's output column ->
    // a [32 rows][32 columns] bf16 staging block (64 B rows, unswizzled) -> one TMA store
    auto finishT = [&](float* v, const CUtensorMap* dmap, int x, int y) {
      if (a.epi == 1) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
      }
      uint8_t* o = out_tile();
      const uint32_t ob_s = gsu32(o) + (uint32_t)(lane * 2);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const __nv_bfloat16 h = __float2bfloat16_rn(v[i]);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(ob_s + (uint32_t)(i * 64)), "h"(*reinterpret_cast<const uint16_t*>(&h))
                     : "memory");
      }
      store_out(dmap, x, y);
    };
    auto add_cT = [&](float* v, int buf) {        // v += C^T block in input buffer buf
      wait_in(buf);
      const uint32_t cb = gsu32(eb + 8192 + buf * 4096) + (uint32_t)(lane * 2);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        uint16_t u;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(u) : "r"(cb + (uint32_t)(i * 64)) : "memory");
        v[i] += __uint_as_float((uint32_t)u << 16);
      }
      __syncwarp();
    };
    auto tmem_ld64 = [&](int col, float (&v)[64]) {
      uint32_t r[32];
      g_tmem_ld32(tl + (uint32_t)col, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
      g_tmem_ld32(tl + (uint32_t)(col + 32), r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[32 + i] = __uint_as_float(r[i]);
    };
    auto release = [&](int acc) {
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) g_mb_arrive(&tempty[acc]); else g_arrive_leader(&tempty[acc]);
      }
    };
    int it = 0;
    WorkIter wi = work();
    for (Work wk; wi.next(wk); ++it) {
      const int acc = it & 1;
      const int t = wk.tile;
      const int S = wk.ncontrib;
      const int y = (t % a.m_tiles) * TM_ROWS + (int)rank * GM + quarter * 32;   // first row of this warp
      const int n0 = (t / a.m_tiles) * BN;
      // SW: this warp's 32 output columns start at wn = y, the tile's batch rows at n0
      const int wn = SW ? y : n0;
      const int seg = wn / a.seg_cols, x0 = wn - seg * a.seg_cols;
      const CUtensorMap* dmap = &maps.d[seg];
      g_mb_wait(&tfull[acc], (uint32_t)(it >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (SW && S == 1) {
        const int rows = a.M - n0 < BN ? a.M - n0 : BN;   // batch rows present in this tile
        const int nch = (rows + 31) >> 5;
        if (a.epi == 2) load_in(0, &maps.c, wn, n0, 2048u);
#pragma unroll 1
        for (int i = 0; i < nch; ++i) {
          if (a.epi == 2 && i + 1 < nch) load_in((i + 1) & 1, &maps.c, wn, n0 + 32 * (i + 1), 2048u);
          uint32_t r[32];
          float v[32];
          g_tmem_ld32(tl + (uint32_t)(acc * BN + 32 * i), r);
          if (i + 1 == nch) release(acc);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (a.epi == 2) add_cT(v, i & 1);
          finishT(v, dmap, x0, n0 + 32 * i);
        }
        continue;
      }
      if (S == 1) {
        if (a.epi == 2) load_in(0, &maps.c, n0, y);
#pragma unroll 1
        for (int c = 0, i = 0; c < BN; c += 64, ++i) {
          if (a.epi == 2 && c + 64 < BN) load_in((i + 1) & 1, &maps.c, n0 + c + 64, y);   // prefetch the next
          float v[64];
          tmem_ld64(acc * BN + c, v);
          if (c + 64 >= BN) release(acc);
          if (a.epi == 2) add_c(v, i & 1);
          finish64(v, dmap, x0 + c, y);
        }
        continue;
      }
      // ---- several groups share this tile: the last of (tile, CTA) to arrive reduces;
      // the others store fp32 partials into slots 0..S-2 (claim order) ----
      int32_t* claim = a.cnt + 2 * (t * CG + (int)rank);
      if (threadIdx.x == 64) *s_role = atomicAdd(claim, 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int role = *s_role;
      if (role < S - 1) {
        const int prow = (a.red ? t : t * (a.cmax - 1) + role) * TM_ROWS + (int)rank * GM + quarter * 32;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          g_tmem_ld32(tl + (uint32_t)(acc * BN + c), r);
          if (c + 32 >= BN) release(acc);
          uint8_t* o = out_tile();
#pragma unroll
          for (int j = 0; j < 8; ++j) sts128(o, swz(lane, j), make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]));
          store_out(&maps.p, c, prow, a.red != 0);
        }
        if (lane == 0) {                               // partial in HBM/L2, then count this warp in
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(claim + 1) : "memory");
        }
      } else {
        // reduce-add mode, epi 2: the residual of the first 64 columns is requested before
        // waiting for the other splits, so its round trip overlaps the wait (BN = 64 when SW)
        const bool cpre = a.red && a.epi == 2;
        if (cpre) {
          if constexpr (SW) {
            load_in(0, &maps.c, wn, n0, 2048u);
            if (n0 + 32 < a.M) load_in(1, &maps.c, wn, n0 + 32, 2048u);
          } else {
            load_in(1, &maps.c, n0, y);
          }
        }
        if (lane == 0) {                               // every other split's 4 warps stored their partial
          const int want = 4 * (S - 1);
          for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(claim + 1) : "memory");
            if (v >= want) break;
            __nanosleep(64);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {
          float v[64];
          tmem_ld64(acc * BN + c, v);
          if (c + 64 >= BN) release(acc);
          if (a.red) {   // the other splits' sum, one TMA round trip; then zero it for the next call
            const int prow = t * TM_ROWS + (int)rank * GM + quarter * 32;
            if (cpre) {  // the residual first: it was requested before the wait above
              if constexpr (SW) {
                add_cT(v, 0);
                if (n0 + c + 32 < a.M) add_cT(v + 32, 1);
              } else {
                add_c(v, 1);
              }
            }
            load_in(0, &maps.p, c, prow);
            load_in(1, &maps.p, c + 32, prow);
            add_p(v, 0);
            add_p(v + 32, 1);
            if (!SW && cpre && c + 64 < BN) load_in(1, &maps.c, n0 + c + 64, y);   // next chunk's residual
#pragma unroll
            for (int h = 0; h < 2; ++h) {   // zeros back by TMA stores (generic stores here cost ~8 %)
              uint8_t* o = out_tile();
#pragma unroll
              for (int j = 0; j < 8; ++j) sts128(o, swz(lane, j), make_uint4(0u, 0u, 0u, 0u));
              store_out(&maps.p, c + 32 * h, prow);
            }
          } else {
            for (int j = 0; j < S - 1; ++j) {
              const int prow = (t * (a.cmax - 1) + j) * TM_ROWS + (int)rank * GM + quarter * 32;
              load_in(0, &maps.p, c, prow);
              load_in(1, &maps.p, c + 32, prow);
              add_p(v, 0);
              add_p(v + 32, 1);
            }
          }
          if constexpr (SW) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (n0 + c + 32 * h >= a.M) break;   // batch rows past M: nothing to store
              if (a.epi == 2 && !cpre) {
                load_in(0, &maps.c, wn, n0 + c + 32 * h, 2048u);
                add_cT(v + 32 * h, 0);
              }
              finishT(v + 32 * h, dmap, x0, n0 + c + 32 * h);
            }
            continue;
          }
          if (a.epi == 2 && !cpre) {
            load_in(0, &maps.c, n0 + c, y);
            add_c(v, 0);
          }
          finish64(v, dmap, x0 + c, y);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");   // all four warps saw the counts
        if (threadIdx.x == 64) { claim[0] = 0; claim[1] = 0; }   // reusable by the next call
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");     // s_role is read; the next tile may claim
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();   // the pair's MMAs are done with both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

typedef CUresult (*GEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
GEncodeFn g_encoder() {
  static GEncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (GEncodeFn)p;
  }
  return fn;
}
// row-major bf16 [rows][K]: box {64, box_rows}, 128B swizzle; rows past the end read as zero
bool encode_kmajor(CUtensorMap* m, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows) {
  GEncodeFn enc = g_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {K * 2};
  cuuint32_t box[2] = {(cuuint32_t)GK, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int CG>
int gemm_smem() {
  constexpr int STAGE = GM * GK * 2 + (BN / CG) * GK * 2;
  constexpr int NSTG = gemm_stages(STAGE);
  return NSTG * STAGE + 4 * EPI_WARP_BYTES + 1024 + 512;
}

// bf16 or fp32 row-major [rows][cols] map with a {box_cols, 32}-row box, 128B swizzle (TMA store / load)
bool encode_rows(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, int fp32, uint32_t box_cols,
                 bool swizzle = true) {
  GEncodeFn enc = g_encoder();
  if (!enc) return false;
  const uint64_t es = fp32 ? 4 : 2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * es};
  cuuint32_t box[2] = {box_cols, 32};
  cuuint32_t el[2] = {1, 1};
  return enc(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
             dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int CG, bool SW = false>
cudaError_t launch_one(const GemmMaps& maps, const GemmArgs& a, int grid, cudaStream_t st) {
  static const bool attr = cudaFuncSetAttribute(k_gemm<BN, CG, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                gemm_smem<BN, CG>()) == cudaSuccess;
  if (!attr) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(G_THREADS);
  cfg.dynamicSmemBytes = gemm_smem<BN, CG>();
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // programmatic dependent launch (S3_GEMM_PDL=0 turns it off: A/B; =2 adds the weight prefetch)
  static const int pdl = [] { const char* e = getenv("S3_GEMM_PDL"); return e ? atoi(e) : 1; }();
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_gemm<BN, CG, SW>, maps, a);
}

__global__ void __launch_bounds__(256) k_cast_bf16(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    dst[i] = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}

}  // namespace

cudaError_t launch_cast_bf16(const float* src, void* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n % 4 || ((uintptr_t)src | (uintptr_t)dst) % 16) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
  k_cast_bf16<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<uint2*>(dst), n4);
  return cudaGetLastError();
}

int gemm_num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Split-K factor: estimated time (in K blocks) = waves x (K blocks per split +
// pipeline fill) + the last split's reduction; S = 1 unless splitting fills
// idle SMs.  Needs S x tiles x rows x BN fp32 + counters of workspace.
// Most groups sharing one stream-K tile
int sk_cmax(int tiles, int kblocks, int G, int dp_tiles) {
  WorkIter w;
  w.init(0, G, tiles, kblocks, dp_tiles);
  int c = 1;
  for (int st = 0; st < tiles - dp_tiles; ++st)
    c = std::max(c, w.group_of((int64_t)(st + 1) * kblocks - 1) - w.group_of((int64_t)st * kblocks) + 1);
  return c;
}
// stream-K scratch: [claim, done] counters per (tile, CTA) at a FIXED place -- the first
// GEMM_CNT_BYTES, shared by every plan (each call leaves its counters zero, so GEMMs with
// different plans can share one workspace) -- then cmax - 1 fp32 partial tiles per tile
constexpr int64_t GEMM_CNT_BYTES = 32768;
// (or, reduce-add mode, one fp32 accumulation tile per tile)
static int gemm_red_mode() {
  static const int r = [] { const char* e = getenv("S3_GEMM_RED"); return e ? atoi(e) : 1; }();
  return r;
}
// Reduce-add for every stream-K plan (tools/gemm_sweep_red.sh: long-K projections
// 1.1-1.2x; with 2 contributors per tile about 3 % slower than a slot); one mode per
// process, so plans sharing a workspace agree on what it holds between calls.
bool gemm_red(int) { return gemm_red_mode() != 0; }
int64_t gemm_ws_bytes(int cmax, int tiles, int rows, int BN, int CG) {
  if ((int64_t)tiles * CG * 2 * 4 > GEMM_CNT_BYTES) return INT64_MAX;
  return GEMM_CNT_BYTES + (int64_t)(gemm_red(cmax) ? 1 : cmax - 1) * tiles * rows * BN * 4;
}

// Tile choice: a CTA pair per 256 x 256 tile (half the operand traffic per
// flop) when M > 128; one CTA per 128 x 256 tile for a single row tile; 128
// columns when 256-wide tiles would leave SMs idle.  Then the split-K factor.
struct GemmPlan {
  int CG, BN, rows, m_tiles, tiles, groups, sk, dp_tiles, cmax;
  bool SW;            // swapped operands (small batch): 128 W rows x BN batch rows per tile
  int64_t ws_bytes;   // workspace the plan needs (0 for data-parallel)
};
bool gemm_plan(const GemmCall& g, int64_t ws_avail, GemmPlan& p) {
  if (g.M < 1 || g.N < 128 || g.K < GK || g.K % GK || g.N % 128 || g.seg_cols < 128 || g.seg_cols % 128 ||
      g.N % g.seg_cols || g.N / g.seg_cols > 3 || g.epi < 0 || g.epi > 2)
    return false;
  const int sms = gemm_num_sms();
  const bool n256 = g.N % 256 == 0 && g.seg_cols % 256 == 0;
  static const int force_cg = [] { const char* e = getenv("S3_GEMM_CG"); return e ? atoi(e) : 0; }();
  static const int force_sk = [] { const char* e = getenv("S3_GEMM_SK"); return e ? atoi(e) : -1; }();
  // Configuration rules (tools/gemm_sweep.sh on B200, GPT-J projections at M = 256 .. 2048):
  //  * CTA-pair 256 x 256 tiles whenever M > 128 and the data-parallel waves are >= 85 % full;
  //  * fewer pair tiles than half the SMs' pairs: long K (>= 8192) -> stream-K over the pairs,
  //    else one CTA per 128 x 128 tile (more, smaller tiles);
  //  * 1 - 1.5 waves of pair tiles: stream-K over the last wave merged with the full one;
  //  * single-CTA tiles (M <= 128, or few pair tiles): stream-K when they fill less than
  //    half a wave (tools/gemm_sweep_small.sh: above that, data parallel streams the
  //    weights faster than stream-K's partial sums);
  //  * stream-K otherwise loses: groups at different K offsets of the same W block stop
  //    sharing it in L2.
  // Small batches (M <= 64): swapped operands, 64 batch columns per tile
  // (tools/gemm_sweep_swap.sh: 1.1-1.3x the unswapped tiles at M <= 64 on GPT-J's
  // projections, slower from M = 96 where the 128-row activation tile is mostly real rows);
  // stream-K when the N / 128 tiles fill at most half the SMs (GPT-J's output and
  // down projections: 32 tiles).  S3_GEMM_SWAP=0 turns it off (A/B).
  static const int swap_on = [] { const char* e = getenv("S3_GEMM_SWAP"); return e ? atoi(e) : 1; }();
  if (g.M <= 64 && swap_on && !force_cg) {
    p.SW = true;
    p.CG = 1;
    p.BN = 64;
    p.rows = GM;
    p.m_tiles = g.N / GM;
    p.tiles = p.m_tiles;                 // one batch tile
    const int kblocks = g.K / GK;
    const int rem = p.tiles % sms;
    const int sk_tiles = rem == 0 ? 0 : (p.tiles >= sms ? rem + sms : p.tiles);
    p.sk = (force_sk >= 0 ? force_sk : 2 * p.tiles <= sms) && sk_tiles > 0 && (int64_t)sk_tiles * kblocks >= 8LL * sms;
    p.dp_tiles = p.sk ? p.tiles - sk_tiles : p.tiles;
    p.cmax = 1;
    p.ws_bytes = 0;
    const int Gs = p.sk ? (int)std::min<int64_t>(sms, (int64_t)(p.tiles - p.dp_tiles) * kblocks) : sms;
    if (p.sk) {
      p.cmax = sk_cmax(p.tiles, kblocks, Gs, p.dp_tiles);
      p.ws_bytes = gemm_ws_bytes(p.cmax, p.tiles, p.rows, p.BN, 1);
      if (p.cmax == 1 || p.ws_bytes > ws_avail) { p.sk = 0; p.dp_tiles = p.tiles; p.cmax = 1; p.ws_bytes = 0; }
    }
    p.groups = p.sk ? Gs : std::min(p.tiles, sms);
    return true;
  }
  p.SW = false;
  const int sms2 = sms / 2;
  const int m2 = (g.M + 2 * GM - 1) / (2 * GM);
  const int tiles2 = m2 * (g.N / 256);
  const int waves2 = (tiles2 + sms2 - 1) / sms2;
  const double eff2 = (double)tiles2 / ((double)waves2 * sms2);
  int cg = 2, sk = 0;
  if (g.M <= GM || !n256) {
    cg = 1;
  } else if (eff2 >= 0.85) {
    cg = 2;
  } else if (2 * tiles2 < sms2) {
    if (g.K >= 8192) sk = 1; else cg = 1;
  } else if (tiles2 > sms2 && 2 * tiles2 < 3 * sms2) {
    sk = 1;
  }
  p.CG = force_cg ? force_cg : cg;
  if (p.CG == 2 && !n256) return false;
  p.rows = GM * p.CG;
  p.m_tiles = (g.M + p.rows - 1) / p.rows;
  const int G = sms / p.CG;
  static const int force_bn = [] { const char* e = getenv("S3_GEMM_BN"); return e ? atoi(e) : 0; }();
  p.BN = p.CG == 2 ? 256 : (n256 && (int64_t)p.m_tiles * (g.N / 256) >= sms ? 256 : 128);
  if (p.CG == 1 && (force_bn == 64 || force_bn == 128 || (force_bn == 256 && n256))) p.BN = force_bn;
  p.tiles = p.m_tiles * (g.N / p.BN);
  const int kblocks = g.K / GK;
  if (p.CG == 1 && force_sk < 0) sk = 2 * p.tiles < G;   // single-CTA tiles: stream-K below half a wave
  // stream-K covers the ragged last wave merged with one full wave (so every group gets
  // >= 1 tile of work); the waves before it stay data parallel
  const int rem = p.tiles % G;
  const int sk_tiles = rem == 0 ? 0 : (p.tiles >= G ? rem + G : p.tiles);
  p.sk = (force_sk >= 0 ? force_sk : sk) && sk_tiles > 0 && (int64_t)sk_tiles * kblocks >= 8LL * G;
  p.dp_tiles = p.sk ? p.tiles - sk_tiles : p.tiles;
  p.cmax = 1;
  p.ws_bytes = 0;
  // every stream-K group owns >= 1 K block (empty ranges would not count as contributors)
  const int Gs = p.sk ? (int)std::min<int64_t>(G, (int64_t)(p.tiles - p.dp_tiles) * kblocks) : G;
  if (p.sk) {
    p.cmax = sk_cmax(p.tiles, kblocks, Gs, p.dp_tiles);
    p.ws_bytes = gemm_ws_bytes(p.cmax, p.tiles, p.rows, p.BN, p.CG);
    if (p.cmax == 1 || p.ws_bytes > ws_avail) { p.sk = 0; p.dp_tiles = p.tiles; p.cmax = 1; p.ws_bytes = 0; }
  }
  p.groups = p.sk ? Gs : std::min(p.tiles, G);
  return true;
}

// SW: rows of the activation box -- the batch rounded up to 8 (TMA zero-fill of the
// remaining rows of a 64-row box made M = 8 ~30 % slower than M = 32)
int swap_box_rows(int M, int BN) { return std::min(BN, (M + 7) & ~7); }

int64_t gemm_workspace_bytes(const GemmCall& g) {
  GemmPlan p;
  return gemm_plan(g, INT64_MAX, p) ? p.ws_bytes : -1;
}

cudaError_t launch_gemm(const GemmCall& g, cudaStream_t st) {
  GemmPlan p;
  if (!gemm_plan(g, g.workspace ? g.workspace_bytes : 0, p) || !g.a || !g.w || !g.d[0] || (g.epi == 2 && !g.c))
    return cudaErrorInvalidValue;
  GemmMaps maps;
  if (p.SW) {   // the MMA's M side is W (128-row boxes), its N side the batch (BN-row boxes)
    if (!encode_kmajor(&maps.a, g.w, (uint64_t)g.N, (uint64_t)g.K, GM)) return cudaErrorInvalidValue;
    if (!encode_kmajor(&maps.w, g.a, (uint64_t)g.M, (uint64_t)g.K, (uint32_t)swap_box_rows(g.M, p.BN)))
      return cudaErrorInvalidValue;
  } else {
    if (!encode_kmajor(&maps.a, g.a, (uint64_t)g.M, (uint64_t)g.K, GM)) return cudaErrorInvalidValue;
    if (!encode_kmajor(&maps.w, g.w, (uint64_t)g.N, (uint64_t)g.K, (uint32_t)(p.BN / p.CG))) return cudaErrorInvalidValue;
  }
  // SW: 32 x 32 unswizzled output / addend blocks (the epilogue's transposed staging)
  const uint32_t obox = p.SW ? 32 : 64;
  const int nseg = g.N / g.seg_cols;
  for (int i = 0; i < 3; ++i) {
    const void* base = g.d[i < nseg ? i : 0];
    if (i < nseg && !g.d[i]) return cudaErrorInvalidValue;
    if (!encode_rows(&maps.d[i], base, (uint64_t)g.M, (uint64_t)g.seg_cols, 0, obox, !p.SW)) return cudaErrorInvalidValue;
  }
  maps.c = maps.d[0];
  if (g.epi == 2 && !encode_rows(&maps.c, g.c, (uint64_t)g.M, (uint64_t)g.N, 0, obox, !p.SW)) return cudaErrorInvalidValue;
  maps.p = maps.d[0];
  if (p.sk && !encode_rows(&maps.p, static_cast<uint8_t*>(g.workspace) + GEMM_CNT_BYTES,
                           (uint64_t)p.tiles * (gemm_red(p.cmax) ? 1 : p.cmax - 1) * p.rows, (uint64_t)p.BN, 1, 32))
    return cudaErrorInvalidValue;
  GemmArgs a;
  a.M = g.M; a.N = g.N; a.K = g.K; a.epi = g.epi; a.seg_cols = g.seg_cols;
  a.m_tiles = p.m_tiles; a.n_tiles = p.SW ? 1 : g.N / p.BN;
  a.stage_tx = GM * GK * 2 + (p.SW ? swap_box_rows(g.M, p.BN) : p.BN / p.CG) * GK * 2;
  a.dp_tiles = p.dp_tiles;
  a.cmax = p.cmax;
  a.cnt = p.sk ? static_cast<int32_t*>(g.workspace) : nullptr;
  a.red = p.sk && gemm_red(p.cmax);
  static const int pdl_mode = [] { const char* e = getenv("S3_GEMM_PDL"); return e ? atoi(e) : 1; }();
  a.wpre = pdl_mode == 2;   // opt-in: the caller guarantees the previous kernel did not write W
  const int groups = p.groups;
  cudaError_t e;
  if (p.SW) e = launch_one<64, 1, true>(maps, a, groups, st);
  else if (p.CG == 2) e = launch_one<256, 2>(maps, a, 2 * groups, st);
  else if (p.BN == 256) e = launch_one<256, 1>(maps, a, groups, st);
  else if (p.BN == 128) e = launch_one<128, 1>(maps, a, groups, st);
  else e = launch_one<64, 1>(maps, a, groups, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace s3
