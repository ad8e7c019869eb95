// s3_attn_tc.cu -- grouped-query / multi-query decode attention on the 5th-gen
// tensor cores (tcgen05 + TMEM + TMA).  attn_variant 2; D = 128, 2 <= G <= 16
// query heads per KV head.
//
// With grouped KV the G query heads that share KV head g turn the decode
// GEMV into a real contraction per 128-row tile of that head's rows:
//     S^T [128 x 16]  = K_tile [128 x D] . Q_g^T [D x 16]                 (A K-major, B K-major)
//     [O_hi|O_lo]^T  += V_tile^T [D x 128] . [P_hi|P_lo]^T [128 x 32]     (A MN-major, B K-major)
// (16 = G padded to the MMA N granularity; P is split into bf16 hi + lo so
// the product keeps ~16 bits, one N = 32 MMA per 16 rows).  Per CTA
// (persistent, one per SM, 11 warps) these roles:
//   producer warp : items (unit, layer, KV head) from the atomic queue (the
//                   next ticket and unit record fetched one ticket ahead); per
//                   tile ONE 4-D TMA box for K and one for V (all valid 8-row
//                   groups, both 64-column blocks; the smem tile layout is
//                   [8-row group][column block][8 rows][128 B]) and one 3-D box
//                   for the 16 q rows; K + q go to a 2-slot K ring that the S
//                   MMA releases, V to a 4-slot V ring that the O MMA releases.  Short units pack
//                   np = 2..NC/G KV heads into one tile, one segment of 128/np
//                   rows per head: the q box already holds those heads' np*G
//                   query rows, and the softmax masks S^T block-diagonally
//                   (segment s meets only columns [sG, (s+1)G)), so one MMA
//                   pair and one softmax pass serve np heads;
//   MMA warp      : one thread issues tcgen05.mma (kind::f16, M 128, K 16 per
//                   instruction) and routes tile t to softmax group iseq & 1;
//   softmax warps : two groups ("ping-pong"), each owning alternate items with
//                   its own S slots, P buffer and O buffer in TMEM; a group is
//                   4 warps per 8 query columns (NC = 16: two quads, one per
//                   column half, never synchronising); 4 warps = 128 TMEM lanes,
//                   lane j holds row j of S^T: mask rows >= nvalid, column
//                   max / sum across the 128 lanes, online softmax in the log2
//                   domain, P (bf16 hi / lo, swizzled) to shared memory, zero V
//                   rows >= nvalid (NaN safety), rescale O^T in TMEM; after the
//                   last tile of an item lane d holds O^T[d][:] and writes out
//                   / the split-K partial (same records as k_combine reads).
//   storer warp   : (fused steps only) the row shift of SURVEY §8 row (d),
//                   done on the tiles already in shared memory -- see below.
// The new token's K/V row is appended to the arena by k_append before this
// kernel, or -- in a host-fed step, where k_new / v_new stream in per chunk --
// by the producer warp just before the unit's tiles load; either way every
// tile reads rows straight from the arena.
//
// Fused row shift (same protocol as k_attn_tma, at tile granularity): when a
// tile lands the storer publishes its unit-layer's read progress
// (head * 2^16 + rows, monotone because a CTA walks a unit-layer's KV heads
// in order); for a MOVE tile it waits until every other unit whose source
// rows overlap the tile's destination rows (k_deps, tc mode) has read that
// far, then writes the tile's whole 8-row groups back with 4-D TMA tensor stores
// through the same layout and the ragged tail rows with a warp copy
// that undoes the 128B swizzle; STAGE (evicted) tiles go to the staging
// buffer the same way.  The K and V slots are released (kempty, vempty) only after the
// stores have read shared memory.  Deadlock freedom is the k_attn_tma
// argument: tickets are taken in unit order and destinations lie at or below
// their sources.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "s3_internal.h"

namespace s3 {
namespace {

// Diagnostic build only (-DTC_TRACE): SM-clock timestamps of CTA 0's tiles at
// fixed points of each role (0 producer got a stage, 1 producer issued the
// tile, 2 softmax finished the item's epilogue (last tiles only), 3 MMA saw the
// tile land, 4 MMA got P, 5 MMA committed O, 6 softmax got S, 7 softmax handed over P), read back with s3_debug_tc_trace.
#ifdef TC_TRACE
constexpr int TC_TRACE_TILES = 8192;
__device__ unsigned long long g_tc_trace[TC_TRACE_TILES * 8];
#define TC_TRACE_AT(t, slot)                                                        \
  do {                                                                             \
    if (blockIdx.x == 0 && (t) < TC_TRACE_TILES) g_tc_trace[(t) * 8 + (slot)] = clock64(); \
  } while (0)
#else
#define TC_TRACE_AT(t, slot) do { } while (0)
#endif

constexpr int TM = 128;                     // rows per tile (MMA M)
constexpr int NQ = 16;                      // query columns per KV head (MMA N)
constexpr int DH = 128;                     // head dim
// K and V ride separate rings: a K slot (with the tile's q) is free as soon as the S
// MMA has read it, a V slot only after the O MMA, so the V ring is the deeper one.
// With one 3-stage K|V ring a short tile held its stage for the whole chain (load,
// S, softmax, P hand-over, O: ~7.7k cycles) and 3 stages bounded the period.
// Ring shapes (per launch, template parameter R33): 2 K + 4 V slots when the step's items are short
// (mostly one tile), 3 + 3 otherwise -- with the fused row shift the storer holds a K slot
// while it waits for a MOVE tile's destination rows, which starves a 2-slot K ring on
// long, moving items (LLaMA-3-8B whole run: 0.66 vs 0.84 of the copy peak).
constexpr int NK_MAX = 3;                   // K (+ q) ring slots
constexpr int NV_MAX = 4;                   // V ring slots (tile t's header lives at hdr[t % nv])
constexpr int KV_BYTES = TM * DH * 2;       // 32 KB: two 64-column blocks of [128 rows x 128 B]
constexpr int Q_BYTES = NQ * DH * 2;        // 4 KB:  two blocks of [16 rows x 128 B]
constexpr int KSLOT_BYTES = KV_BYTES + Q_BYTES;   // 36 KB (multiple of 1024)
constexpr int VSLOT_BYTES = KV_BYTES;             // 32 KB
constexpr int RING_BYTES = 3 * KSLOT_BYTES + 3 * VSLOT_BYTES;   // >= 2 * KSLOT_BYTES + 4 * VSLOT_BYTES
static_assert(2 * KSLOT_BYTES + 4 * VSLOT_BYTES <= RING_BYTES, "ring shapes must fit the same bytes");
__device__ __forceinline__ uint8_t* kslot(uint8_t* smem, int t, int nk) { return smem + (t % nk) * KSLOT_BYTES; }
__device__ __forceinline__ uint8_t* vslot(uint8_t* smem, int t, int nk, int nv) {
  return smem + nk * KSLOT_BYTES + (t % nv) * VSLOT_BYTES;
}
// P as bf16 hi + lo parts (P = hi + lo to ~16 bits), one MMA operand [hi | lo] of N = 2 NC:
// two K blocks (tile rows j 0-63, 64-127) of [2 NC rows x 128 B] (rows 0..NC-1 hi, NC..2NC-1 lo)
__host__ __device__ constexpr int pblk_bytes(int nc) { return 2 * nc * 64 * 2; }   // per K block
__host__ __device__ constexpr int pbuf_bytes(int nc) { return 2 * pblk_bytes(nc); }  // 4 KB (NC 8) / 8 KB (NC 16)
constexpr float LAZY_THR = 8.0f;            // rescale only if a score beats the running max by 2^8
// NG softmax groups: group g takes the items with iseq % NG == g, so while one group runs a
// tile's softmax and epilogue the other runs its own.  NG = 2 ("ping-pong").  Measured on
// B200 (tools/attn_sweep.py, -DTC_NG8=3 / 4 builds with 4 KB P buffers and S^T issued NG - 1
// tiles ahead): 3 groups 0.64 / 0.79 / 0.66 and 4 groups 0.64 / 0.59 / 0.40 of the copy peak
// (400-row / 40-row / 20-row items) against 2 groups 1.00 / 0.94 / 0.70 -- the idle groups'
// mbarrier polling takes issue slots from the producer, MMA and working softmax warps.
// TMEM: S slot (g, b) at columns (2g + b)*16 in [0, 128); O buffer g at 128 + 32g:
// [0, NC) = V.P_hi, [NC, 2NC) = V.P_lo.
constexpr int NG_MAX = 4;
#ifndef TC_NG8
#define TC_NG8 2
#endif
__host__ __device__ constexpr int tc_groups(int nc) { return nc == 8 ? TC_NG8 : 2; }
constexpr int TMEM_COLS = 256;
__host__ __device__ constexpr uint32_t scol(int g, int b) { return (uint32_t)((2 * g + b) * 16); }
__host__ __device__ constexpr uint32_t ocol(int g) { return 32u * NG_MAX + 32u * (uint32_t)g; }
// warps: producer, MMA, 4 softmax (group 0), storer, then 4 softmax per further group
// A softmax group is 4 warps per 8 query columns: NC = 16 groups have two column halves
// (8 warps), each half running the 8-column chain on its own columns with its own named
// barrier -- softmax columns are independent (column max / sum), so the halves never
// synchronise -- which keeps the per-tile chain of the NC = 16 kernels (16 / G KV heads per
// short tile) at the 8-column latency.  Warps: producer, MMA, group 0 half 0, storer,
// group 1 half 0, then group 0 half 1, group 1 half 1.
__host__ __device__ constexpr int tc_halves(int nc) { return nc / 8; }
__host__ __device__ constexpr int tc_threads(int nc) { return 32 * (3 + 4 * tc_groups(nc) * tc_halves(nc)); }
constexpr int CW = 8;                       // query columns per softmax warp

struct TcHdr {
  int32_t item, r0, nvalid, flags;          // flags: 1 = first tile of the item, 2 = last;
                                            // bits 8..12: np (KV heads packed in the tile),
                                            // bits 16..20: seg / 8 (rows per packed head's segment)
                                            // bits 24..28: hoff + 1 (tail-packed items' full tiles)
  int32_t b, part, li, g;
  int32_t iseq, mode, drow;                 // iseq: per-CTA item sequence number (group / O buffer = iseq % NG)
  uint32_t prog;                            // read progress this tile completes (storer)
  DepDesc dep;                              // MOVE tiles: filled by the TMA engine with the tile
};
static_assert(sizeof(TcHdr) % 16 == 0, "TcHdr.dep must stay 16-B aligned");
constexpr uint32_t TC_PROG_FULL = 0x80000000u;
// KV heads g..g+np-1 share the tile, one segment of seg rows each (segment s at rows [s seg, (s+1) seg))
__device__ __forceinline__ int hdr_np(const TcHdr& h) { return (h.flags >> 8) & 31; }
__device__ __forceinline__ int hdr_seg(const TcHdr& h) { return ((h.flags >> 16) & 31) * 8; }
// tail-packed items (below): a full tile of head g + hoff inside the item of heads g.. (-1: none)
__device__ __forceinline__ int hdr_hoff(const TcHdr& h) { return ((h.flags >> 24) & 31) - 1; }
constexpr int TC_HEAD_STRIDE = 1 << 16;      // progress = head * 2^16 + rows (unit rows < 2^16)

struct alignas(16) TcSmem {                 // after the ring and the two P buffers (one per group)
  uint64_t kfull[NK_MAX], kempty[NK_MAX], vfull[NV_MAX], vempty[NV_MAX];
  uint64_t s_full[NG_MAX][2], s_empty[NG_MAX][2];   // [group][S slot]; s_full: MMA commit + the MMA thread's arrive
  uint64_t p_full[NG_MAX], o_done[NG_MAX], o_fin[NG_MAX], o_free[NG_MAX];   // [group] (= O buffer)
  alignas(16) TcHdr hdr[NV_MAX];            // tile t at hdr[t % nv]; hdr.dep is a 16-B bulk-copy destination
  float red[2 * NG_MAX][2][4][CW];          // [group + NG half][max / sum][warp][column]
  int32_t flag[2 * NG_MAX][4];
  int32_t gt[NG_MAX][2];                    // ring tile index in group g's S slot b (-1: no more tiles)
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// Warp-uniform issue of tcgen05 / TMA instructions.  Their operands live in uniform
// registers; a value the compiler cannot prove warp-uniform (anything loaded from memory,
// or computed in a lane-0-only branch) is moved there by an ELECT / R2UR.BROADCAST loop
// around EVERY instruction (~90 cycles per tcgen05.mma or cp.async.bulk.tensor, measured
// with the TC_TRACE build).  So the producer and MMA roles run warp-wide: memory values are
// broadcast with uni() (shfl from lane 0: provably uniform), and one elected lane issues.
__device__ __forceinline__ int uni(int x) { return __shfl_sync(0xffffffffu, x, 0); }
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s16(void* dst, const void* src, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void tma4d(void* dst, const CUtensorMap* map, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
          "r"(su32(dst)),
      "l"(map), "r"(0), "r"(c1), "r"(c2), "r"(0), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma4d_store(const CUtensorMap* map, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map), "r"(0),
               "r"(c1), "r"(c2), "r"(0), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
// UMMA shared-memory descriptor: 128B swizzle, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((su32(p) >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: bf16 x bf16 -> f32, M 128, N = n
__host__ __device__ constexpr uint32_t idesc(int a_mn_major, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(TM >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)su32(b)) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t addr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// named barrier of one softmax group's column half (4 warps); ids 1..4
__device__ __forceinline__ void softmax_bar(int bq) { asm volatile("bar.sync %0, 128;" ::"r"(1 + bq) : "memory"); }

// Column-wise reduction of 16 values per lane over the 128 softmax lanes.
// Within a warp a transposed butterfly halves the vector at each step (8 + 4
// + 2 + 1 + 1 shuffles); lane l ends with column 8*b4 + 4*b3 + 2*b2 + b1 of
// its bits.  Warp partials meet in shared memory; every lane gets all 16.
template <bool MAX>
__device__ __forceinline__ float rop(float x, float y) { return MAX ? fmaxf(x, y) : x + y; }

template <bool MAX, int NC>
__device__ __forceinline__ void col_reduce(float (&v)[NC], float (&red)[4][CW], int wq, int lane, int grp) {
  static_assert(NC <= CW, "one warp reduces at most CW columns");
  // NC = 16: 8 + 4 + 2 + 1 + 1 shuffles; NC = 8: 4 + 2 + 1 + 1 + 1
  float a8[8], a4[4], a2[2], a1;
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4, h2 = lane & 2;
  int col;
  if constexpr (NC == 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float send = h16 ? v[i] : v[8 + i];
      const float keep = h16 ? v[8 + i] : v[i];
      a8[i] = rop<MAX>(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) a8[i] = v[i];
  }
  const int o8 = NC == 16 ? 8 : 16;               // NC = 8: the first split uses lane bit 4
  const bool b8 = NC == 16 ? h8 : h16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b8 ? a8[i] : a8[4 + i];
    const float keep = b8 ? a8[4 + i] : a8[i];
    a4[i] = rop<MAX>(keep, __shfl_xor_sync(0xffffffffu, send, o8));
  }
  const int o4 = NC == 16 ? 4 : 8;
  const bool b4 = NC == 16 ? h4 : h8;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b4 ? a4[i] : a4[2 + i];
    const float keep = b4 ? a4[2 + i] : a4[i];
    a2[i] = rop<MAX>(keep, __shfl_xor_sync(0xffffffffu, send, o4));
  }
  const int o2 = NC == 16 ? 2 : 4;
  const bool b2 = NC == 16 ? h2 : h4;
  {
    const float send = b2 ? a2[0] : a2[1];
    const float keep = b2 ? a2[1] : a2[0];
    a1 = rop<MAX>(keep, __shfl_xor_sync(0xffffffffu, send, o2));
  }
  if constexpr (NC == 16) {
    a1 = rop<MAX>(a1, __shfl_xor_sync(0xffffffffu, a1, 1));
    col = (h16 ? 8 : 0) + (h8 ? 4 : 0) + (h4 ? 2 : 0) + (h2 ? 1 : 0);
  } else {
    a1 = rop<MAX>(a1, __shfl_xor_sync(0xffffffffu, a1, 2));
    a1 = rop<MAX>(a1, __shfl_xor_sync(0xffffffffu, a1, 1));
    col = (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
  }
  if (!(lane & (NC == 16 ? 1 : 3))) red[wq][col] = a1;
  softmax_bar(grp);
#pragma unroll
  for (int c = 0; c < NC; ++c) v[c] = rop<MAX>(rop<MAX>(red[0][c], red[1][c]), rop<MAX>(red[2][c], red[3][c]));
  softmax_bar(grp);
}

// Shared-memory tile layout: 16 groups of 8 rows; group j holds both 64-column
// blocks as adjacent 1 KB 128B-swizzle atoms, [j][block][8 rows][128 B], so a
// tile's K (or V) rows for one KV head arrive in ONE 4-D TMA box
// {64 columns, 8 rows, 2 blocks, n groups} whose row-group dimension (stride
// 8 rows) overlaps the row dimension -- a box may start at any row (see
// tools/tma_probe/tma4d.cu).  The UMMA descriptors read it with an 8-row-group
// stride of 2 KB and the second column block 1 KB after the first.
constexpr int NGRP = TM / 8;     // 8-row groups per tile
constexpr int NSTB = 5;          // store boxes of 16 / 8 / 4 / 2 / 1 groups (valid rows only)
struct TcMaps {
  CUtensorMap kvg[NGRP];         // loads: box of n + 1 groups
  CUtensorMap kvt[7];            // loads of a partial last group: box {64, r + 1 rows, 1 block, 1 group}
  CUtensorMap st_kv[NSTB];       // row-shift stores into the arena: box of 16 >> i groups
  CUtensorMap st_stage[NSTB];    // evictee stores into staging
  CUtensorMap q;                 // 16 q rows x both column blocks
};

struct TcArgs {
  int32_t H, Hkv, G, B, l0, nl;
  float qscale;
  float* out;
  float* partials;
  const Unit* units;
  int32_t* ctrl;
  // fused row shift
  uint8_t* arena;
  uint8_t* staging;
  int64_t kvpt;
  const DepDesc* desc;
  unsigned long long* progress;
  uint32_t epoch;
  int32_t pmax;          // most KV heads one tile may pack (NC / G; 1 = no packing)
  const uint16_t* k_new; // [nl][B][Hkv][D]: appended to the arena by the producer warp
  const uint16_t* v_new;
  uint32_t* evdone;      // per-evictee staged-row counters (cumulative; the D2H stream waits on them)
  Feed feed;             // host-fed step: per-chunk ready words (s3_decode_step_host)
  int32_t exact;         // 1: a segment's last, partial 8-row group loads only its valid rows
};

// Wait until a ready word written by the copy stream reaches `epoch` (host-fed
// step); trap after 20 s instead of hanging the device.
__device__ __noinline__ void tc_wait_ready(const uint32_t* p, uint32_t epoch) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    __nanosleep(200);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ uint4 ld_cg16(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}

// NC: query columns the softmax handles, G padded to 8 or 16 (the MMA always has N = 16);
// PACK: short units may pack several KV heads into one tile (NC / G >= 2)
// FEED: host-fed step (the producer warp waits on ready words and appends the new rows)
// R33: ring shape 3 K + 3 V slots (else 2 K + 4 V; compile-time so the slot arithmetic folds)
template <int NC, bool PACK, bool FEED, bool R33>
__global__ void __launch_bounds__(tc_threads(NC), 1) k_attn_tc(const __grid_constant__ TcMaps maps, TcArgs a) {
  constexpr int NG = tc_groups(NC);
  constexpr int PBLK = pblk_bytes(NC), PBUF = pbuf_bytes(NC);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128B-swizzle atoms, by pointer arithmetic so the
  // compiler keeps the shared-memory address space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* pbuf = smem + RING_BYTES;
  TcSmem& S = *reinterpret_cast<TcSmem*>(pbuf + NG * PBUF);
  const int tid = threadIdx.x, warp = uni(tid >> 5), lane = tid & 31;
  // the storer takes part in the ring only when this step shifts rows
  const bool fused = a.ctrl[CTRL_FUSED] != 0;
  constexpr int nk = R33 ? 3 : 2, nv = R33 ? 3 : 4;
  if (tid == 0) {
    for (int i = 0; i < nk; ++i) { mb_init(&S.kfull[i], 1); mb_init(&S.kempty[i], fused ? 2 : 1); }
    for (int i = 0; i < nv; ++i) { mb_init(&S.vfull[i], 1); mb_init(&S.vempty[i], fused ? 2 : 1); }
    for (int g = 0; g < NG; ++g) {
      for (int b = 0; b < 2; ++b) { mb_init(&S.s_full[g][b], 2); mb_init(&S.s_empty[g][b], 4 * tc_halves(NC)); }
      mb_init(&S.p_full[g], 4 * tc_halves(NC));
      mb_init(&S.o_done[g], 1);
      mb_init(&S.o_fin[g], 1);
      mb_init(&S.o_free[g], 4 * tc_halves(NC));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // V buffers start at zero: rows a tile does not load keep finite (zero or earlier valid) data
  for (int st = 0; st < nv; ++st)
    for (int i = tid; i < KV_BYTES / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(vslot(smem, st, nk, nv))[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&S.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;
  const int row_cols = 2 * a.Hkv * DH;      // elements of one layer inside a token row

  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    // One atomic per (unit, layer) covers its H_kv items (item = (u*nl + li)*H_kv + g),
    // so the queue and unit-record latencies are paid once per H_kv tiles.  In a host-fed
    // step the whole warp first appends the unit's new K/V row (all KV heads of the layer)
    // at arena row off + len -- the slot's first slack row, which no other unit reads or,
    // before this unit's progress covers it, writes -- then lane 0 issues the tiles.
    // Otherwise k_append has written every new row before the kernel (cheaper: the
    // loads would stall this warp's TMA issue).
    int t = 0, iseq = 0, ready_max = -1;
    const int groups_total = uni(a.ctrl[CTRL_N_UNITS]) * a.nl;
    const int kd8 = a.Hkv * DH / 8;               // 16-B vectors of one layer's new K (or V) row
    // The next ticket and its unit record are fetched one ticket ahead, so the
    // atomic and the dependent load (~2 us together) overlap this ticket's tile
    // issue instead of stalling the ring between tickets (short units have only a
    // few tiles per ticket).  Deadlock freedom is unchanged: the smallest
    // unfinished ticket is always some CTA's current one.
    // The whole warp runs the loop with warp-uniform values (uni()); elected lanes issue.
    auto load_unit = [&](int w) {
      const Unit* p = a.units + w / a.nl;
      Unit u;
      u.b = uni(p->b); u.r0 = uni(p->r0); u.r1 = uni(p->r1); u.part = uni(p->part);
      u.off = uni(p->off); u.len = uni(p->len); u.has_new = uni(p->has_new); u.mode = uni(p->mode);
      const long long d = p->dst;
      u.dst = (int64_t)(((unsigned long long)(uint32_t)uni((int)(d >> 32)) << 32) | (uint32_t)uni((int)d));
      u.stage_base = uni(p->stage_base); u.pad = uni(p->pad);
      return u;
    };
    int w_next = uni(lane == 0 ? atomicAdd(&a.ctrl[CTRL_ITEM], 1) : 0);
    Unit un_next{};
    if (w_next < groups_total) un_next = load_unit(w_next);
    for (;;) {
      const int w = w_next;
      const Unit un = un_next;
      if (w < groups_total) {
        w_next = uni(lane == 0 ? atomicAdd(&a.ctrl[CTRL_ITEM], 1) : 0);
        if (w_next < groups_total) un_next = load_unit(w_next);
      }
      if (w >= groups_total) {
        mb_wait(&S.kempty[t % nk], ((uint32_t)(t / nk) & 1u) ^ 1u);
        mb_wait(&S.vempty[t % nv], ((uint32_t)(t / nv) & 1u) ^ 1u);
        if (elect_one()) {
          S.hdr[t % nv].item = -1;
          mb_arrive(&S.kfull[t % nk]);
          mb_arrive(&S.vfull[t % nv]);
        }
        __syncwarp();
        break;
      }
      const int li = w % a.nl;
      if constexpr (FEED) {
        // host-fed step: this slot's q / k_new / v_new have landed once its chunk's word is set
        // (chunks land in order, so the highest chunk waited for covers every earlier one)
        const int c = un.b / a.feed.cb;
        if (c > ready_max) {
          if (lane == 0) tc_wait_ready(a.feed.ready + c, a.feed.epoch);
          ready_max = c;
          __syncwarp();
        }
      }
      if (FEED && un.has_new) {   // host-fed: k_new / v_new land during the kernel
        const int64_t src = ((int64_t)li * a.B + un.b) * a.Hkv * DH;
        uint16_t* dst = reinterpret_cast<uint16_t*>(a.arena) + (int64_t)(un.off + un.len) * (a.kvpt / 2) +
                        (int64_t)(a.l0 + li) * 2 * a.Hkv * DH;
        for (int i = lane; i < kd8; i += 32) {
          const uint4 kk = ld_cg16(a.k_new + src + i * 8);
          const uint4 vv = ld_cg16(a.v_new + src + i * 8);
          *reinterpret_cast<uint4*>(dst + i * 8) = kk;
          *reinterpret_cast<uint4*>(dst + a.Hkv * DH + i * 8) = vv;
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");   // the tile loads below read the new row
        __syncwarp();
      }
      {
        const int nrows = (un.r1 - un.r0) + (un.has_new ? 1 : 0);   // new row now in the arena
        const bool mv = un.mode == UNIT_MOVE;
        // destination row of the unit's first row: arena row (MOVE) or staging row (STAGE)
        const int drow0 = (int)(mv ? un.dst : un.dst / a.kvpt) + un.r0;
        // short units: up to pmax KV heads share one 128-row tile, one segment of seg =
        // nrows rounded up to 8 rows each, back to back (block-diagonal scores: segment s
        // only meets query columns [s G, (s+1) G)); the last tile of a unit-layer may hold
        // fewer heads (Hkv need not be a multiple of the packing)
        int npk = 1, seg = TM, tl = 0;
        bool tailpack = false;
        if constexpr (PACK) {
          const int rg = (nrows + 7) & ~7;
          if (2 * rg <= TM) {
            npk = min(min(a.pmax, TM / rg), a.Hkv);
            seg = rg;
          } else {
            // longer units: each head's rows past its last full 128-row tile (the tail) would
            // be a tile of its own; tails of up to 64 rows are packed instead, np heads per
            // tile, and those heads' full tiles come first in the same item (the item then
            // spans the np heads' query columns: a full tile of head g + hoff only meets
            // columns [hoff G, (hoff+1) G), the packed tail tile is block-diagonal)
            tl = nrows % TM;
            const int tg = (tl + 7) & ~7;
            if (tl > 0 && 2 * tg <= TM && a.pmax > 1) {
              npk = min(min(a.pmax, TM / tg), a.Hkv);
              seg = tg;
              tailpack = npk > 1;
            }
          }
        }
        // one tile: segments np_t of seg_t rows for heads hd.., rows [r, r + nrow) of the unit
        auto emit = [&](int g, int hd, int hoff, int np_t, int seg_t, int r, int nrow, bool first, bool last,
                        uint32_t prog) {
          const int ks = t % nk, vs = t % nv;
          mb_wait(&S.kempty[ks], ((uint32_t)(t / nk) & 1u) ^ 1u);
          mb_wait(&S.vempty[vs], ((uint32_t)(t / nv) & 1u) ^ 1u);
          if (elect_one()) {
            TC_TRACE_AT(t, 0);
            TcHdr& h = S.hdr[vs];
            h.item = w * a.Hkv + g; h.r0 = un.r0 + r; h.nvalid = nrow;
            h.flags = (first ? 1 : 0) | (last ? 2 : 0) | (np_t << 8) | ((seg_t >> 3) << 16) | ((hoff + 1) << 24);
            h.b = un.b; h.part = un.part; h.li = li; h.g = g; h.iseq = iseq;
            h.mode = un.mode; h.drow = drow0 + r;
            if (un.mode == UNIT_STAGE) h.dep.ua = un.pad;   // eviction index (dep is only loaded for MOVE)
            h.prog = prog;
            // 8-row groups (one 128B-swizzle atom per column block): fg whole groups in one
            // 4-D box, then (exact) the tr rows of a partial last group as one box per column
            // block -- the rows past nrow are never read (short items: ~5 % of the DRAM
            // traffic); the smem rows they leave stale are masked (K) / zeroed (V) like the
            // rows past a tile's last group
            const int fg = a.exact ? nrow >> 3 : (nrow + 7) >> 3;
            const int tr = a.exact ? nrow & 7 : 0;
            uint8_t* sk = kslot(smem, t, nk);
            uint8_t* sv = vslot(smem, t, nk, nv);
            uint8_t* sq = sk + KV_BYTES;
            const bool dep = fused && mv;
            const uint32_t sbytes = (uint32_t)(fg * 2048 + tr * 256);   // per segment, K (or V)
            mb_expect(&S.kfull[ks], (uint32_t)np_t * sbytes + (uint32_t)(Q_BYTES + (dep ? 16 : 0)));
            mb_expect(&S.vfull[vs], (uint32_t)np_t * sbytes);
            if (dep) bulk_g2s16(&h.dep, a.desc + un.stage_base + r / TM, &S.kfull[ks]);
            const int row0 = un.off + un.r0 + r;
            for (int sgi = 0; sgi < np_t; ++sgi) {   // one 4-D box per segment for K and one for V
              const int colk = (a.l0 + li) * row_cols + (hd + sgi) * DH;
              const int colv = colk + a.Hkv * DH;
              const int sgo = sgi * (seg_t / 8) * 2048;   // segment's first group
              if (fg > 0) {
                tma4d(sk + sgo, &maps.kvg[fg - 1], row0, colk / 64, &S.kfull[ks]);
                tma4d(sv + sgo, &maps.kvg[fg - 1], row0, colv / 64, &S.vfull[vs]);
              }
              if (tr > 0) {
                const int to = sgo + fg * 2048, tr0 = row0 + fg * 8;
                tma4d(sk + to, &maps.kvt[tr - 1], tr0, colk / 64, &S.kfull[ks]);
                tma4d(sk + to + 1024, &maps.kvt[tr - 1], tr0, colk / 64 + 1, &S.kfull[ks]);
                tma4d(sv + to, &maps.kvt[tr - 1], tr0, colv / 64, &S.vfull[vs]);
                tma4d(sv + to + 1024, &maps.kvt[tr - 1], tr0, colv / 64 + 1, &S.vfull[vs]);
              }
            }
            const int qrow = (li * a.B + un.b) * a.H + g * a.G;
            tma3d(sq, &maps.q, 0, qrow, 0, &S.kfull[ks]);   // both 64-column blocks of the 16 q rows
            TC_TRACE_AT(t, 1);
          }
          __syncwarp();
          ++t;
        };
        for (int g = 0; g < a.Hkv; g += npk, ++iseq) {
          const int np = min(npk, a.Hkv - g);
          const int glast = g + np - 1;
          const uint32_t full = glast == a.Hkv - 1 ? TC_PROG_FULL : 0u;
          if (!tailpack) {
            for (int r = 0; r < nrows; r += TM) {
              const int nrow = min(TM, nrows - r);
              // heads g..glast are read up to r + nrow rows once this tile lands
              emit(g, g, -1, np, seg, r, nrow, r == 0, r + TM >= nrows,
                   (uint32_t)(glast * TC_HEAD_STRIDE + r + nrow) | (r + TM >= nrows ? full : 0u));
            }
          } else {
            const int rfull = nrows - tl;
            // read progress: heads < g complete until the packed tail tile lands (conservative)
            for (int hh = 0; hh < np; ++hh)
              for (int r = 0; r < rfull; r += TM)
                emit(g, g + hh, hh, 1, TM, r, TM, hh == 0 && r == 0, false, (uint32_t)(g * TC_HEAD_STRIDE));
            emit(g, g, -1, np, seg, rfull, tl, false, true, (uint32_t)(glast * TC_HEAD_STRIDE + nrows) | full);
          }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // -------------------------------- MMA ---------------------------------
    // Tiles in ring order; tile t belongs to softmax group g = iseq % NG (its
    // item's group, which is also its O buffer) and is that group's k-th tile.
    // LA tiles of lookahead: S^T(t+LA) is issued before O^T(t), so the other
    // groups' softmax runs while this tile's P is being made.  LA < nv: the
    // tile t+LA must be able to land while O^T(t) is still pending.
    {
      // warp-wide with uniform values; one elected lane issues the MMAs and commits
      // S: N = 16 query columns; O: N = 2 NC ([P_hi | P_lo] in one MMA, halving the PV issue count)
      constexpr uint32_t id_s = idesc(0, NQ), id_o = idesc(1, 2 * NC);
      constexpr int LA = (NG - 1) < (nv - 1) ? (NG - 1) : (nv - 1);
      const uint32_t tm = (uint32_t)uni((int)tmem);
      int kc[NG];                               // tiles handed to each group so far
#pragma unroll
      for (int g = 0; g < NG; ++g) kc[g] = 0;
      int kq[4] = {0, 0, 0, 0};                 // tile t's index within its group, at kq[t & 3]
      auto issue_s = [&](int t) -> int {        // returns the tile's index within its group
        const int g = uni(S.hdr[t % nv].iseq) % NG;
        int k = 0;
#pragma unroll
        for (int i = 0; i < NG; ++i)
          if (i == g) k = kc[i]++;
        const int sb = k & 1;
        mb_wait(&S.s_empty[g][sb], ((uint32_t)(k >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* sk = kslot(smem, t, nk);
        const uint8_t* sq = sk + KV_BYTES;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {      // S^T = K . Q^T over d in steps of 16
            const int kb = kk >> 2, ko = (kk & 3) * 32;
            mma(tm + scol(g, sb), sdesc(sk + kb * 1024 + ko, 16, 2048), sdesc(sq + kb * 2048 + ko, 16, 1024), id_s,
                kk > 0);
          }
          commit(&S.s_full[g][sb]);
          commit(&S.kempty[t % nk]);            // the K slot is free once these MMAs have read it
          S.gt[g][sb] = t;
          mb_arrive(&S.s_full[g][sb]);          // releases gt together with the slot
        }
        __syncwarp();
        return k;
      };
      auto finish = [&]() {                     // tell every group there are no more tiles
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const int sb = kc[g] & 1;
          mb_wait(&S.s_empty[g][sb], ((uint32_t)(kc[g] >> 1) & 1u) ^ 1u);
          if (elect_one()) {
            S.gt[g][sb] = -1;
            mb_arrive(&S.s_full[g][sb]);
            mb_arrive(&S.s_full[g][sb]);
          }
          __syncwarp();
        }
      };
      // is tile j the end marker?  (waits for it to land)
      auto landed_end = [&](int j) -> bool {
        mb_wait(&S.kfull[j % nk], (uint32_t)(j / nk) & 1u);
        if (lane == 0) TC_TRACE_AT(j, 3);
        return uni(S.hdr[j % nv].item) < 0;
      };
      int end_t = 0x7fffffff;                   // the end marker's ring index, once seen
      for (int j = 0; j < LA && end_t > j; ++j) {
        if (landed_end(j)) end_t = j; else kq[j & 3] = issue_s(j);
      }
      if (end_t == 0) {
        finish();
      } else {
        for (int t = 0;; ++t) {
          const int vs = t % nv;
          const int j = t + LA;
          if (end_t > j) {
            if (landed_end(j)) end_t = j; else kq[j & 3] = issue_s(j);
          }
          const int kt = kq[t & 3];
          const int flags = uni(S.hdr[vs].flags);
          const bool first = flags & 1;
          const bool last = flags & 2;
          const int iseq = uni(S.hdr[vs].iseq), g = iseq % NG;
          if (first)   // O buffer g must have been read by the epilogue of item iseq - NG
            mb_wait(&S.o_free[g], ((uint32_t)(iseq / NG) & 1u) ^ 1u);
          mb_wait(&S.p_full[g], (uint32_t)kt & 1u);
          mb_wait(&S.vfull[vs], (uint32_t)(t / nv) & 1u);   // V landed (the softmax waited too if it zeroed rows)
          if (lane == 0) TC_TRACE_AT(t, 4);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sv = vslot(smem, t, nk, nv);
          const uint8_t* sp = pbuf + g * PBUF;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {        // [O_hi | O_lo]^T += V^T . [P_hi | P_lo]^T, rows in steps of 16
              const int kb = kk >> 2, ko = (kk & 3) * 32;
              mma(tm + ocol(g), sdesc(sv + kk * 4096, 1024, 2048), sdesc(sp + kb * PBLK + ko, 16, 1024), id_o,
                  (first && kk == 0) ? 0u : 1u);
            }
            commit(&S.o_done[g]);
            if (last) commit(&S.o_fin[g]);
            commit(&S.vempty[vs]);
            TC_TRACE_AT(t, 5);
          }
          __syncwarp();
          if (t + 1 == end_t) { finish(); break; }
        }
      }
    }
  } else if (warp == 6) {
    // ------------------------------- storer -------------------------------
    if (fused) {
      int pending = -1;                   // tile whose bulk stores may still read shared memory
      for (int t = 0;; ++t) {
        mb_wait(&S.kfull[t % nk], (uint32_t)(t / nk) & 1u);
        mb_wait(&S.vfull[t % nv], (uint32_t)(t / nv) & 1u);
        TcHdr h = S.hdr[t % nv];
        // fields that feed the TMA stores' operands: warp-uniform (see uni())
        h.item = uni(h.item); h.nvalid = uni(h.nvalid); h.flags = uni(h.flags); h.li = uni(h.li);
        h.g = uni(h.g); h.mode = uni(h.mode); h.drow = uni(h.drow);
        if (h.item < 0) break;
        const int w = h.item / a.Hkv;     // unit-layer ticket = progress slot
        if (lane == 0) {
          // the tile's rows are in shared memory: its source rows may be overwritten
          st_rlx_u64(a.progress + w, ((unsigned long long)a.epoch << 32) | h.prog);
          if (h.mode == UNIT_MOVE && h.dep.ua >= 0) {
            // the tile overwrites heads g..g+np-1 of its destination rows
            const uint32_t gbase =
                (uint32_t)((h.g + (PACK ? max(hdr_hoff(h), 0) + hdr_np(h) : 1) - 1) * TC_HEAD_STRIDE);
            for (int v = h.dep.ua; v <= h.dep.ub; ++v) {
              const int need = v == h.dep.ua ? h.dep.need_a : (v == h.dep.ub ? h.dep.need_b : -1);
              const int it = v * a.nl + h.li;
              if (it == w) continue;      // own rows: earlier tiles of this head, already read
              for (;;) {
                const unsigned long long x = ld_acq_u64(a.progress + it);
                const uint32_t lo = (uint32_t)x;
                if ((uint32_t)(x >> 32) == a.epoch && ((lo & TC_PROG_FULL) || (need >= 0 && lo >= gbase + need)))
                  break;
                __nanosleep(32);
              }
            }
          }
        }
        __syncwarp();
        const bool stores = (h.mode == UNIT_MOVE || h.mode == UNIT_STAGE) && h.nvalid > 0;
        if (stores) {
          const int full_groups = h.nvalid >> 3;     // whole 8-row groups go out as 4-D boxes
          if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
          const int np = PACK ? hdr_np(h) : 1;
          const int seg = PACK ? hdr_seg(h) : TM;
          for (int sgi = 0; sgi < np; ++sgi) {       // one segment per packed KV head
            const uint8_t* sk = kslot(smem, t, nk) + sgi * (seg / 8) * 2048;
            const uint8_t* sv = vslot(smem, t, nk, nv) + sgi * (seg / 8) * 2048;
            const int colk = (a.l0 + h.li) * 2 * a.Hkv * DH + (h.g + (PACK ? max(hdr_hoff(h), 0) : 0) + sgi) * DH;
            const int colv = colk + a.Hkv * DH;
            if (lane == 0) {
              const CUtensorMap* map = h.mode == UNIT_MOVE ? maps.st_kv : maps.st_stage;
#pragma unroll
              for (int i = 0; i < NSTB; ++i) {
                const int bg = NGRP >> i;
                if (full_groups & bg) {
                  const int done = full_groups & ~(2 * bg - 1);
                  tma4d_store(map + i, h.drow + done * 8, colk / 64, sk + done * 2048);
                  tma4d_store(map + i, h.drow + done * 8, colv / 64, sv + done * 2048);
                }
              }
            }
            // ragged tail rows: one 16-B chunk per lane (K/V, 64-column block, chunk)
            const int kv = lane >> 4, kb = (lane >> 3) & 1, c = lane & 7;
            uint8_t* gbase = (h.mode == UNIT_MOVE ? a.arena : a.staging) +
                             (int64_t)(kv ? colv : colk) * 2 + kb * 128 + c * 16;
            for (int row = full_groups * 8; row < h.nvalid; ++row) {
              const uint4 x = *reinterpret_cast<const uint4*>((kv ? sv : sk) + (row >> 3) * 2048 + kb * 1024 +
                                                              (row & 7) * 128 + ((c ^ (row & 7)) << 4));
              *reinterpret_cast<uint4*>(gbase + (int64_t)(h.drow + row) * a.kvpt) = x;
            }
          }
          __syncwarp();
        }
        if (lane == 0) {
          if (stores) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          // release the previous tile's K and V slots once its stores have read shared memory
          if (pending >= 0) {
            if (stores) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            mb_arrive(&S.kempty[pending % nk]);
            mb_arrive(&S.vempty[pending % nv]);
            pending = -1;
          }
          if (stores) {
            pending = t;
          } else {
            mb_arrive(&S.kempty[t % nk]);
            mb_arrive(&S.vempty[t % nv]);
          }
          if (h.mode == UNIT_STAGE && a.evdone) {
            // the tile's evictee rows are final in staging once its stores complete (the
            // ragged rows' generic stores are ordered by the __syncwarp above): count them
            // for the D2H stream, which copies each evictee as soon as its count is complete
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const uint32_t rows = (uint32_t)(h.nvalid * (PACK ? hdr_np(h) : 1));
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.evdone + h.dep.ua), "r"(rows) : "memory");
          }
        }
      }
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (pending >= 0) {
          mb_arrive(&S.kempty[pending % nk]);
          mb_arrive(&S.vempty[pending % nv]);
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
  } else {
    // ------------------------------ softmax -------------------------------
    // Two groups (warps 2-5 + 11-14: group 0, warps 7-10 + 15-18: group 1; the
    // second quad of each exists for NC = 16 and takes columns 8-15); group g
    // takes the tiles of items with iseq & 1 == g, in order, so the two
    // groups' per-tile chains (TMEM load, reductions, P, hand-over,
    // epilogue) overlap.  Lazy running max (log2 domain): the column max is
    // reduced across the 128 lanes only on an item's first tile or when some
    // score exceeds the running max by more than LAZY_THR; otherwise
    // p = 2^(s - m) <= 2^8 and nothing is rescaled.  Each lane keeps its own
    // row's partial sums; they are reduced once, in the epilogue.
    constexpr int HV = tc_halves(NC);
    const int sidx = warp < 6 ? warp - 2 : warp - 3;  // 0..3 g0 h0, 4..7 g1 h0, 8..11 g0 h1, 12..15 g1 h1
    const int grp = (sidx >> 2) & 1;
    const int hf = sidx >> 3;                         // column half: columns [CW hf, CW hf + CW)
    const int bq = grp + 2 * hf;                      // this quad's barrier / reduction slot
    const int co = CW * hf;
    const int wq = sidx & 3;                          // 0..3 within the quad
    const int lq = warp & 3;                          // TMEM lane quarter this warp may access
    const int row = lq * 32 + lane;                   // TMEM lane = tile row (S) = head-dim index (O)
    const uint32_t lane_base = tmem + ((uint32_t)(lq * 32) << 16);
    const uint32_t oc = ocol(grp);                    // this group's O buffer
    uint8_t* const pgrp = pbuf + grp * PBUF;          // this group's P buffer
    float m[CW], lrow[CW];
#pragma unroll
    for (int c = 0; c < CW; ++c) { m[c] = -INFINITY; lrow[c] = 0.f; }
    for (int k = 0;; ++k) {
      const int sb = k & 1;
      mb_wait(&S.s_full[grp][sb], (uint32_t)(k >> 1) & 1u);
      const int t = S.gt[grp][sb];
      if (t < 0) break;
      if (lane == 0 && sidx == 0) TC_TRACE_AT(t, 6);
      const TcHdr h = S.hdr[t % nv];
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float s[CW];
      tmem_ld8(lane_base + scol(grp, sb) + co, s);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive(&S.s_empty[grp][sb]);
      const bool first = h.flags & 1;
      bool valid, loaded;                             // loaded: row holds this item's (or slack) data
      const int np = PACK ? hdr_np(h) : 1;
      const int hoff = PACK ? hdr_hoff(h) : -1;
      if (!PACK || np == 1) {                          // warp-uniform: one KV head per tile
        valid = row < h.nvalid;
        loaded = row < ((h.nvalid + 15) & ~15);
        if (hoff < 0) {
#pragma unroll
          for (int c = 0; c < CW; ++c) s[c] = valid ? s[c] * a.qscale : -INFINITY;
        } else {                                       // tail-packed item: head g + hoff's full tile
          const int c0 = hoff * a.G - co, c1 = c0 + a.G;
#pragma unroll
          for (int c = 0; c < CW; ++c) s[c] = (valid && c >= c0 && c < c1) ? s[c] * a.qscale : -INFINITY;
        }
      } else {
        // block-diagonal mask of packed tiles: segment sgm only meets columns
        // [sgm G, (sgm+1) G); columns past np G stay unmasked (finite, never written out);
        // rows past the last segment are masked
        const int seg = hdr_seg(h);
        const int sgm = row / seg;
        const int rs = row - sgm * seg;
        loaded = sgm < np;
        valid = loaded && rs < h.nvalid;
        const int cg0 = sgm * a.G - co, cg1 = cg0 + a.G, cpad = a.G * np - co;   // in this half's columns
#pragma unroll
        for (int c = 0; c < CW; ++c)
          s[c] = (valid && ((c >= cg0 && c < cg1) || c >= cpad)) ? s[c] * a.qscale : -INFINITY;
      }
      // does any score need a larger running max?
      bool need = first;
      if (!first) {
        bool over = false;
#pragma unroll
        for (int c = 0; c < CW; ++c) over |= s[c] > m[c] + LAZY_THR;
        const bool wover = __any_sync(0xffffffffu, over);
        if (lane == 0) S.flag[bq][wq] = wover;
        softmax_bar(bq);
        need = S.flag[bq][0] | S.flag[bq][1] | S.flag[bq][2] | S.flag[bq][3];
        softmax_bar(bq);
      }
      float corr[CW];
      bool rescale = false;
      if (need) {
        float mt[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) mt[c] = s[c];
        col_reduce<true, CW>(mt, S.red[bq][0], wq, lane, bq);
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float mn = first ? mt[c] : fmaxf(m[c], mt[c]);
          // a column no tile of the item has met yet keeps m = -inf (tail-packed items)
          corr[c] = first ? 0.f : (mn == -INFINITY ? 1.f : ex2f(m[c] - mn));
          m[c] = mn;
          lrow[c] = first ? 0.f : lrow[c] * corr[c];
        }
        rescale = !first;
      }
      // this group's previous O MMA has read its P buffer (and O^T may be touched):
      // every o_done phase is waited, so no completion goes unobserved
      if (k > 0) {
        mb_wait(&S.o_done[grp], (uint32_t)(k - 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      // P = 2^(s - m) as bf16 hi + lo; row co + c (query column), column j = row; 128B swizzle
      uint8_t* sp = pgrp + (row >> 6) * PBLK;
      const uint32_t jj2 = (uint32_t)(row & 63) * 2u;
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const float pv = s[c] == -INFINITY ? 0.f : ex2f(s[c] - m[c]);
        lrow[c] += pv;
        const __nv_bfloat16 hi = __float2bfloat16_rn(pv);
        const __nv_bfloat16 lo = __float2bfloat16_rn(pv - __bfloat162float(hi));
        const uint32_t byte = (uint32_t)(co + c) * 128u + jj2;
        const uint32_t sw = byte ^ ((uint32_t)(c & 7) << 4);          // (co + c) & 7 == c
        *reinterpret_cast<__nv_bfloat16*>(sp + sw) = hi;
        *reinterpret_cast<__nv_bfloat16*>(sp + NC * 128 + sw) = lo;   // row NC + co + c: same swizzle phase
      }
      if (!valid && loaded) {                         // loaded rows past the slot's resident rows: V := 0
        mb_wait(&S.vfull[t % nv], (uint32_t)(t / nv) & 1u);   // after the V load has landed
        uint8_t* sv = vslot(smem, t, nk, nv);
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          if (HV == 2 && kb != hf) continue;          // the two halves zero one 64-column block each
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            *reinterpret_cast<uint4*>(sv + (row >> 3) * 2048 + kb * 1024 + (row & 7) * 128 + ch * 16) =
                make_uint4(0, 0, 0, 0);
        }
      }
      if (rescale) {                                // O^T *= corr (this item's previous tile is done)
        float o[CW], olo[CW];
        tmem_ld8(lane_base + oc + co, o);
        tmem_ld8(lane_base + oc + NC + co, olo);
#pragma unroll
        for (int c = 0; c < CW; ++c) { o[c] *= corr[c]; olo[c] *= corr[c]; }
        tmem_st8(lane_base + oc + co, o);
        tmem_st8(lane_base + oc + NC + co, olo);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive(&S.p_full[grp]);
      if (lane == 0 && sidx == 0) TC_TRACE_AT(t, 7);
      if (h.flags & 2) {
        // epilogue of the finished item: the other group keeps the tensor pipe busy meanwhile
        float pl[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) pl[c] = lrow[c];
        col_reduce<false, CW>(pl, S.red[bq][1], wq, lane, bq);
        mb_wait(&S.o_fin[grp], (uint32_t)(h.iseq / NG) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float o[CW], olo[CW];
        tmem_ld8(lane_base + oc + co, o);
        tmem_ld8(lane_base + oc + NC + co, olo);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(&S.o_free[grp]);
        const int d = row;
        const int ncol = PACK ? a.G * hdr_np(h) : a.G;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          if (co + c >= ncol) break;
          const int hq = h.g * a.G + co + c;        // packed heads: column c belongs to KV head g + c / G
          const float ov = o[c] + olo[c];
          if (h.part < 0) {
            a.out[((int64_t)(h.li * a.B + h.b) * a.H + hq) * DH + d] = ov / pl[c];
          } else {
            float* pr = a.partials + (((int64_t)h.part * a.nl + h.li) * a.H + hq) * (DH + 4);
            pr[d] = ov;
            if (d == 0) { pr[DH] = m[c]; pr[DH + 1] = pl[c]; }
          }
        }
        if (lane == 0 && sidx == 0) TC_TRACE_AT(t, 2);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}


// k_append: the new token's K/V row goes to row off+len before k_attn_tc reads it
__global__ void __launch_bounds__(256) k_append(Shape sh, const DSlot* __restrict__ slots, int32_t B, int32_t l0,
                                                int32_t nl, const uint16_t* __restrict__ k_new,
                                                const uint16_t* __restrict__ v_new, uint16_t* __restrict__ arena) {
  const int D8 = sh.D / 8;
  const int64_t total = (int64_t)nl * B * sh.Hkv * D8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    const int d8 = (int)(r % D8); r /= D8;
    const int g = (int)(r % sh.Hkv); r /= sh.Hkv;
    const int b = (int)(r % B);
    const int li = (int)(r / B);
    const DSlot s = slots[b];
    uint16_t* dst = arena + ((int64_t)s.off + s.len) * sh.row_elems + ((int64_t)(l0 + li) * 2 * sh.Hkv + g) * sh.D + d8 * 8;
    const uint4 kk = *reinterpret_cast<const uint4*>(k_new + i * 8);
    const uint4 vv = *reinterpret_cast<const uint4*>(v_new + i * 8);
    *reinterpret_cast<uint4*>(dst) = kk;
    *reinterpret_cast<uint4*>(dst + (int64_t)sh.Hkv * sh.D) = vv;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}


// K/V rows as a 4-D bf16 map {64 columns, rows (pitch), 64-column blocks of the row (128 B),
// 8-row groups (8 pitches)}; box {64, 8, 2, groups}.  The group dimension overlaps the row
// dimension, so a box starting at row r covers rows r .. r + 8 groups - 1; its extent is kept
// generous (the row dimension bounds the start row; reads past the arena's last row land in
// the 8 guard rows s3_workspace_query adds).
bool encode_4d(CUtensorMap* m, const void* base, uint64_t row_elems, uint64_t rows, uint64_t pitch, int groups,
               int box_rows = 8, int blocks = 2) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {64, rows, row_elems / 64, rows / 8 + 2};
  cuuint64_t strides[3] = {pitch, 128, 8 * pitch};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, (cuuint32_t)blocks, (cuuint32_t)groups};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// q as a 3-D bf16 map {64 columns, rows, 2 column blocks (stride 128 B)}: one box of 16 rows lands
// as [block][16 rows][64] -- the layout the S MMA reads -- in one instruction instead of two
bool encode_q3(CUtensorMap* m, const void* base, uint64_t rows, uint64_t pitch) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {64, rows, 2};
  cuuint64_t strides[2] = {pitch, 128};
  cuuint32_t box[3] = {64, 16, 2};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

#ifdef TC_TRACE
extern "C" int s3_debug_tc_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_tc_trace, sizeof(unsigned long long) * (size_t)std::min(n, TC_TRACE_TILES * 8));
}
#endif

int attn_tc_smem(int nc) { return RING_BYTES + tc_groups(nc) * pbuf_bytes(nc) + (int)sizeof(TcSmem) + 1024; }
template <bool R33>
const void* attn_tc_ptr(int nc, bool pack, bool feed) {
  if (feed) {
    if (nc == 8) return pack ? (const void*)k_attn_tc<8, true, true, R33> : (const void*)k_attn_tc<8, false, true, R33>;
    return pack ? (const void*)k_attn_tc<16, true, true, R33> : (const void*)k_attn_tc<16, false, true, R33>;
  }
  if (nc == 8) return pack ? (const void*)k_attn_tc<8, true, false, R33> : (const void*)k_attn_tc<8, false, false, R33>;
  return pack ? (const void*)k_attn_tc<16, true, false, R33> : (const void*)k_attn_tc<16, false, false, R33>;
}
const void* attn_tc_kernel_ptr(int nc, bool pack, bool feed, bool r33) {
  return r33 ? attn_tc_ptr<true>(nc, pack, feed) : attn_tc_ptr<false>(nc, pack, feed);
}

bool attn_tc_supported(const Shape& sh) {
  const int G = sh.Hkv > 0 ? sh.H / sh.Hkv : 0;
  return sh.D == DH && G >= 2 && G <= NQ && sh.H % sh.Hkv == 0 && encoder() != nullptr;
}


cudaError_t launch_append(const Shape& sh, const DSlot* slots, int32_t B, int32_t l0, int32_t nl,
                          const uint16_t* k_new, const uint16_t* v_new, uint16_t* arena, cudaStream_t st) {
  const int64_t tot = (int64_t)nl * B * sh.Hkv * (sh.D / 8);
  const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
  k_append<<<blocks, 256, 0, st>>>(sh, slots, B, l0, nl, k_new, v_new, arena);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const Shape& sh, const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                           uint16_t* arena, int64_t arena_rows, uint8_t* staging, int64_t staging_bytes, float* out,
                           float* partials, const Unit* units, const Split* splits, const DepDesc* desc,
                           unsigned long long* progress, uint32_t epoch, int32_t* ctrl, int32_t B, int32_t l0,
                           int32_t nl, int32_t grid_attn, int32_t grid_combine, const Feed& feed, uint32_t* evdone,
                           int32_t mean_rows, int32_t nc_pick, cudaStream_t st) {
  TcMaps maps;
  // staging rows (evicted slots' KV, token-major like the arena); without staging k_prep never fuses an eviction
  const int64_t stage_rows = staging ? staging_bytes / sh.kvpt : 0;
  for (int n = 1; n <= NGRP; ++n)
    if (!encode_4d(&maps.kvg[n - 1], arena, (uint64_t)sh.row_elems, (uint64_t)arena_rows, (uint64_t)sh.kvpt, n))
      return cudaErrorInvalidValue;
  for (int r = 1; r <= 7; ++r)
    if (!encode_4d(&maps.kvt[r - 1], arena, (uint64_t)sh.row_elems, (uint64_t)arena_rows, (uint64_t)sh.kvpt, 1, r, 1))
      return cudaErrorInvalidValue;
  for (int i = 0; i < NSTB; ++i) {
    if (!encode_4d(&maps.st_kv[i], arena, (uint64_t)sh.row_elems, (uint64_t)arena_rows, (uint64_t)sh.kvpt, NGRP >> i))
      return cudaErrorInvalidValue;
    if (stage_rows > 0) {
      if (!encode_4d(&maps.st_stage[i], staging, (uint64_t)sh.row_elems, (uint64_t)stage_rows, (uint64_t)sh.kvpt,
                     NGRP >> i))
        return cudaErrorInvalidValue;
    } else {
      maps.st_stage[i] = maps.st_kv[i];
    }
  }
  if (!encode_q3(&maps.q, q, (uint64_t)nl * B * sh.H, (uint64_t)sh.D * 2)) return cudaErrorInvalidValue;
  TcArgs a;
  a.H = sh.H; a.Hkv = sh.Hkv; a.G = sh.H / sh.Hkv; a.B = B; a.l0 = l0; a.nl = nl;
  a.qscale = 1.4426950408889634f / sqrtf((float)sh.D);
  a.out = out; a.partials = partials; a.units = units; a.ctrl = ctrl;
  a.arena = reinterpret_cast<uint8_t*>(arena); a.staging = staging; a.kvpt = sh.kvpt;
  a.desc = desc; a.progress = progress; a.epoch = epoch;
  a.k_new = k_new; a.v_new = v_new; a.feed = feed; a.evdone = evdone;
  static const int exact = [] { const char* e = getenv("S3_TC_EXACT"); return e ? atoi(e) : 1; }();   // A/B
  a.exact = exact;
  // Per launch, from the step's rows (s3_host.cpp):
  // * ring shape: 2 K + 4 V slots for short items (mostly one tile; mean <= 48 rows), else
  //   3 + 3 (the fused row shift holds K slots on long, moving items); LLaMA-3-8B threshold
  //   sweep 32 / 48 / 64 / 96: 48 keeps both the short-context window and the whole run best;
  // * softmax columns NC (nc_pick): 16 when G > 8, or when it needs fewer tiles than NC = 8
  //   (16 / G instead of 8 / G KV heads per short tile).  tools/attn_sweep.py, LLaMA-3-8B
  //   shape, NC 16 / NC 8: 25-row items 0.961 / 0.864, 33-row 0.943 / 0.837, 45-row 0.876 /
  //   0.915 (same tile count), 400-row 0.945 / 0.972.
  static const int ring = [] { const char* e = getenv("S3_TC_RING"); return e ? atoi(e) : 0; }();   // A/B: 24 or 33
  static const int short_rows = [] { const char* e = getenv("S3_TC_SHORT_ROWS"); return e ? atoi(e) : 48; }();
  const bool two_four = ring ? ring == 24 : mean_rows <= short_rows;
  static const int pack = [] { const char* e = getenv("S3_TC_PACK"); return e ? atoi(e) : 1; }();
  static const int nc_env = [] { const char* e = getenv("S3_TC_NC"); return e ? atoi(e) : 0; }();   // A/B: 8 or 16
  const int nc = a.G > 8 ? 16 : nc_env ? (nc_env == 16 ? 16 : 8) : (pack && nc_pick == 16 ? 16 : 8);
  a.pmax = pack ? nc / a.G : 1;   // S3_TC_PACK=0: one KV head per tile (A/B)
  const dim3 grid(grid_attn), block(tc_threads(nc));
  const int smem = attn_tc_smem(nc);
  const void* kfn = attn_tc_kernel_ptr(nc, a.pmax > 1, feed.ready != nullptr, !two_four);
  void* args[] = {(void*)&maps, (void*)&a};
  cudaError_t le = cudaLaunchKernel(kfn, grid, block, args, (size_t)smem, st);
  if (le != cudaSuccess) return le;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine(sh, splits, partials, out, ctrl, B, nl, grid_combine, st);
}

}  // namespace s3
