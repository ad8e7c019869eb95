// s3_kernels.cu -- sm_100a device kernels of the S^3 decode step.
//
//   k_prep       per-step work list (split-K units over each slot's rows) and
//                the overrun/finish detection epilogue
//   k_attn       length-masked decode attention + KV append
//   k_combine    merge of split-K partials
//   k_keep_scan  keep flags -> prefix sums -> new offsets, permutation,
//                eviction list, move list
//   k_move       ordered in-place row-shift compaction (+ eviction staging)
//   k_fill       prompt-row fill for fresh admissions (prefill stand-in)
//   k_synth      q / k_new / v_new / eos stand-in (harness)
//   k_verify     resident rows == generator (invariant P2, tests)
//
// Design notes are in DESIGN.md ("Kernels").  Everything here is HBM-bound
// integer / fp32-FMA work: decode attention has M = 1 per head (MHA), so the
// tensor cores have nothing to contract.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "s3_internal.h"

namespace s3 {

// ---------------------------------------------------------------------------
// small PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_plain(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// coherent (L2) load: for inputs that land while the kernel runs (host-fed step)
__device__ __forceinline__ uint4 ld_cg(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
// Wait until a ready word written by the copy stream reaches `epoch`
// (s3_decode_step_host).  A word that never arrives is a host bug: trap after
// 20 s instead of hanging the device.
__device__ __noinline__ void wait_ready(const uint32_t* p, uint32_t epoch) {
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
  asm volatile("fence.proxy.async.global;" ::: "memory");   // the bulk copies that follow read the landed bytes
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void unpack8(uint4 u, float (&f)[8]) {
  f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16); f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16); f[7] = __uint_as_float(u.w & 0xffff0000u);
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan of NV int64 (or int32) values per thread (1024 threads max).
// ---------------------------------------------------------------------------
template <int NV, typename T = long long>
__device__ void block_excl_scan(T (&x)[NV], T (&total)[NV]) {
  __shared__ T warp_sums[32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  T incl[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    T v = x[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    incl[i] = v;
  }
  if (lane == 31)
#pragma unroll
    for (int i = 0; i < NV; ++i) warp_sums[warp][i] = incl[i];
  __syncthreads();
  for (int i = warp; i < NV; i += nwarps) {   // warp i scans quantity i over the warps
    {
      T v = lane < nwarps ? warp_sums[lane][i] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
      }
      if (lane < nwarps) warp_sums[lane][i] = v;   // inclusive over warps
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    T before = warp == 0 ? 0 : warp_sums[warp - 1][i];
    total[i] = warp_sums[nwarps - 1][i];
    x[i] = before + incl[i] - x[i];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Counter-based generator
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// One byte of a 32-bit word as the float 2^23 + byte (PRMT with the 0x4B000000 exponent),
// then (byte - 128) * scale in one exact FFMA (scale a power of two); the bf16 of two such
// floats is their high halves, packed by one more PRMT.  Integer-pipe work per 16-B vector
// drops by ~2/3 against shift / mask / I2F / shift per element (k_synth is ALU-pipe bound).
__device__ __forceinline__ float byte_float(uint32_t word, uint32_t j, float scale) {
  const float f = __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7540u + j));
  return fmaf(f, scale, -8388736.0f * scale);
}
__device__ __forceinline__ uint32_t pack_hi(float lo, float hi) {
  return __byte_perm(__float_as_uint(lo), __float_as_uint(hi), 0x7632u);
}
__device__ __forceinline__ uint4 bytes_to_bf16x8(uint64_t z, float scale) {
  const uint32_t a = (uint32_t)z, b = (uint32_t)(z >> 32);
  return make_uint4(pack_hi(byte_float(a, 0, scale), byte_float(a, 1, scale)),
                    pack_hi(byte_float(a, 2, scale), byte_float(a, 3, scale)),
                    pack_hi(byte_float(b, 0, scale), byte_float(b, 1, scale)),
                    pack_hi(byte_float(b, 2, scale), byte_float(b, 3, scale)));
}
// 8 bf16 values (one 16-byte vector) for element group d8 of (req,l,kv,pos,h).
// tag 0 (K/V rows) indexes the Hkv KV heads, tag 1 (q) the H query heads.
// 8 generator values from counter g: bytes of splitmix64 minus 128, times scale
__device__ __forceinline__ uint4 gen8_at(uint64_t seed, uint64_t tag, uint64_t g, float scale) {
  return bytes_to_bf16x8(splitmix64(seed ^ (tag << 60) ^ g), scale);
}
// counter of the first 16-B vector of row (req, l, kv, pos): g = ((((req L + l) 2 + kv) M + pos) nh + h) D/8 + d8
__device__ __forceinline__ uint64_t gen_row_base(const Shape& sh, uint64_t nh, int64_t req, int l, int kv, int pos) {
  return ((((uint64_t)req * sh.L + l) * 2u + kv) * (uint64_t)sh.max_len + pos) * nh * (uint64_t)(sh.D / 8);
}
__device__ __forceinline__ uint4 gen8(const Shape& sh, uint64_t seed, uint64_t tag, int64_t req,
                                      int l, int kv, int pos, int h, int d8, float scale) {
  const uint64_t nh = tag == 0 ? (uint64_t)sh.Hkv : (uint64_t)sh.H;
  const uint64_t g =
      (((((uint64_t)req * sh.L + l) * 2u + kv) * (uint64_t)sh.max_len + pos) * nh + h) *
          (uint64_t)(sh.D / 8) + d8;
  return bytes_to_bf16x8(splitmix64(seed ^ (tag << 60) ^ g), scale);
}

// ---------------------------------------------------------------------------
// k_prep: one CTA of 1024 threads (B <= max_running; a few microseconds).
//  * detection (R11, R28): when finalize, status_b = FINISHED
//    if eos_b or len_b + 1 == max_len, else OVERRUN if len_b + 1 == cap_b,
//    else RUNNING;
//  * work list: slot b's len_b + 1 rows (with the new one) are cut into
//    ceil((len_b+1)/C) units (split-K); per unit, ceil(rows/AT_RPS) ring
//    stages;
//  * fused step (fuse && finalize && the evicted bytes fit in staging): the
//    keep-scan runs here, before the attention kernel, so that kernel can
//    write every survivor's rows straight to its compacted offset (the
//    paper's row shift) and every evictee's rows to the
//    staging buffer while it streams them.  Exclusive scans give new_off
//    (sum of kept caps before b), the permutation, evicted / finished lists
//    and the packed report; the gathered slot table goes to `next`.
// ---------------------------------------------------------------------------
// Detection after the step's append (len + 1 rows): FINISHED on EOS or at the
// maximum length (R28: the reservation cannot grow past max_len, so
// the sequence stops like one that emitted EOS), else OVERRUN when the
// reservation is used up, else RUNNING.
__device__ __forceinline__ int detect(const PrepArgs& a, const DSlot& sl, int b) {
  if (!a.finalize) return 0;
  if (a.eos[b] || sl.len + 1 >= a.sh.max_len) return 1;
  return sl.len + 1 == sl.cap ? 2 : 0;
}

#ifdef PREP_TRACE
#define PREP_T(i) do { if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ptt[i])); } while (0)
#else
#define PREP_T(i) do {} while (0)
#endif
__global__ void __launch_bounds__(1024) k_prep(PrepArgs a) {
#ifdef PREP_TRACE
  unsigned long long ptt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  PREP_T(0);
  __shared__ int s_first_hole;
  __shared__ unsigned long long s_hbm, s_moved;
  __shared__ long long s_end;
  __shared__ long long s_agg[PREP_MAX_CTAS][PREP_NX];
  __shared__ long long s_pre[PREP_NX], s_all[PREP_NX];
  __shared__ int s_last;
  if (threadIdx.x == 0) { s_first_hole = a.B; s_hbm = 0; s_moved = 0; s_end = 0; }
  const int B = a.B, C = a.C;
  const int64_t kvpt = a.sh.kvpt;
  const int nb = gridDim.x;                                  // > 1: one slot per thread, decoupled totals
  const int per = (B + nb * (int)blockDim.x - 1) / (nb * (int)blockDim.x);
  const int b0 = ((int)blockIdx.x * (int)blockDim.x + (int)threadIdx.x) * per, b1 = min(B, b0 + per);
  // x: 0 units, 1 splits, 2 parts, 3 stages, 4 keep, 5 keep*cap, 6 fin, 7 ev, 8 ev rows, 9 cap
  // (32-bit: counts and arena rows; evicted bytes = ev rows * kvpt)
  int x[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  DSlot sl0{};                                               // this thread's first slot, kept for pass 2
  int st0 = 0;
  for (int b = b0; b < b1; ++b) {
    const DSlot sl = a.slots[b];
    const int k = (sl.len + 1 + C - 1) / C;
    x[0] += k;
    x[1] += k > 1;
    x[2] += k > 1 ? k : 0;
    for (int i = 0; i < k; ++i) {
      const int rows = min((i + 1) * C, sl.len) - i * C;
      x[3] += rows > 0 ? (rows + AT_RPS - 1) / AT_RPS : 1;
    }
    const int st = detect(a, sl, b);
    if (b == b0) { sl0 = sl; st0 = st; }
    x[4] += st == 0;
    x[5] += st == 0 ? sl.cap : 0;
    x[6] += st == 1;
    x[7] += st == 2;
    x[8] += st == 2 ? sl.len + 1 : 0;
    x[9] += sl.cap;
  }
  int tot[10];
  PREP_T(1);
  block_excl_scan<10, int>(x, tot);
  PREP_T(2);
  if (nb > 1) {
    // publish this CTA's totals, then read every CTA's: the prefix of the CTAs before this one
    // and the grid totals (all CTAs are co-resident: nb <= 64 one-CTA-per-SM blocks)
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < PREP_NX; ++k) a.xagg[blockIdx.x * PREP_NX + k] = tot[k];
      // the release orders this thread's xagg stores before the flag (no separate fence)
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.xflag + blockIdx.x), "l"((unsigned long long)a.epoch)
                   : "memory");
    }
    if ((int)threadIdx.x < nb) {
      const int c = threadIdx.x;
      for (;;) {                          // all CTAs are co-resident and publish within microseconds: spin
        unsigned long long f;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(a.xflag + c) : "memory");
        if (f == (unsigned long long)a.epoch) break;
      }
#pragma unroll
      for (int k = 0; k < PREP_NX; ++k) s_agg[c][k] = __ldcg(a.xagg + c * PREP_NX + k);
    }
    __syncthreads();
    PREP_T(3);
    // warp k sums field k over the CTAs (lanes over c): the prefix of the CTAs before this one
    // and the grid total, once per CTA instead of once per thread
    {
      const int ln = threadIdx.x & 31;
      for (int w = threadIdx.x >> 5; w < PREP_NX; w += blockDim.x >> 5) {
        int pre = 0, all = 0;
        for (int c = ln; c < nb; c += 32) {
          const int v = (int)s_agg[c][w];
          all += v;
          if (c < (int)blockIdx.x) pre += v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          pre += __shfl_xor_sync(0xffffffffu, pre, o);
          all += __shfl_xor_sync(0xffffffffu, all, o);
        }
        if (ln == 0) { s_pre[w] = pre; s_all[w] = all; }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PREP_NX; ++k) {
      x[k] += s_pre[k];
      tot[k] = s_all[k];
    }
  }
  PREP_T(4);
  const bool fused = a.fuse && a.finalize && (int64_t)tot[8] * kvpt <= a.staging_bytes;
  // R27: shift unless the policy is on-demand and nobody could use the rows
  const bool compact = a.compact_policy == 0 || a.pool_nonempty || tot[7] > 0;
  int32_t* perm = reinterpret_cast<int32_t*>(a.report + report_perm_off(B));
  DEvicted* evl = reinterpret_cast<DEvicted*>(a.report + report_ev_off(B));
  int64_t* finl = reinterpret_cast<int64_t*>(a.report + report_fin_off(B));
  long long u = x[0], sp = x[1], p = x[2], stg = x[3];
  long long keep_i = x[4], keepcap = x[5], fin_i = x[6], ev_i = x[7], evb = (long long)x[8] * kvpt, capx = x[9];
  unsigned long long hbm = 0, moved = 0;
  long long end = 0;
  int first = B;
  for (int b = b0; b < b1; ++b) {
    DSlot sl = b == b0 ? sl0 : a.slots[b];
    const int k = (sl.len + 1 + C - 1) / C;
    const int st = b == b0 ? st0 : detect(a, sl, b);
    int mode = UNIT_STAY;
    int64_t dst = sl.off;
    if (fused) {
      if (st == 0) {
        const int64_t noff = compact ? keepcap : sl.off;
        mode = noff == sl.off ? UNIT_STAY : UNIT_MOVE;
        dst = noff;
      } else if (st == 2) {
        mode = UNIT_STAGE;
        dst = evb;
      } else {
        mode = UNIT_DROP;
        dst = 0;
      }
    }
    for (int i = 0; i < k; ++i) {
      Unit un;
      un.b = b;
      un.r0 = i * C;
      un.r1 = min((i + 1) * C, sl.len);
      un.part = k > 1 ? (int)(p + i) : -1;
      un.off = sl.off;
      un.len = sl.len;
      un.has_new = (i == k - 1);
      un.mode = mode;
      un.dst = dst;
      un.stage_base = (int)stg;
      un.pad = mode == UNIT_STAGE ? (int)ev_i : 0;   // eviction index: per-evictee completion counter
      a.units[u + i] = un;
      const int rows = un.r1 - un.r0;
      stg += rows > 0 ? (rows + AT_RPS - 1) / AT_RPS : 1;
    }
    if (k > 1) {
      Split spl;
      spl.b = b; spl.part0 = (int)p; spl.k = k; spl.pad = 0;
      a.splits[sp] = spl;
      ++sp;
      p += k;
    }
    u += k;
    if (a.finalize) {
      sl.len += 1;
      sl.gen += 1;
      sl.status = st;
    }
    if (!fused) {
      if (a.finalize) a.slots[b] = sl;
      continue;
    }
    // ---- fused keep-scan outputs ----
    if (st != 0 && b < first) first = b;
    if (st == 0) {
      perm[b] = (int)keep_i;
      if (mode == UNIT_MOVE) moved += (unsigned long long)sl.len * kvpt;
      sl.off = (int32_t)dst;
      sl.status = 0;
      end = max(end, (long long)sl.off + sl.cap);
      a.next[keep_i] = sl;
      ++keep_i;
      keepcap += sl.cap;
    } else {
      perm[b] = -1;
      if (st == 1) {
        finl[fin_i++] = sl.req;
      } else {
        DEvicted e;
        e.req = sl.req; e.b = b; e.prompt = sl.prompt; e.gen = sl.gen; e.len = sl.len;
        e.cap = sl.cap; e.pad = 0; e.stage_off = evb;
        evl[ev_i++] = e;
        evb += (int64_t)sl.len * kvpt;
        hbm += 2ull * (unsigned long long)(tot[9] - capx - sl.cap) * (unsigned long long)kvpt;
      }
    }
    capx += sl.cap;
  }
  if (fused) {
    // warp-reduce first: one shared atomic per warp instead of per thread
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
      hbm += __shfl_xor_sync(0xffffffffu, hbm, o);
      moved += __shfl_xor_sync(0xffffffffu, moved, o);
      end = max(end, __shfl_xor_sync(0xffffffffu, end, o));
    }
    if ((threadIdx.x & 31) == 0) {
      if (first < B) atomicMin(&s_first_hole, first);
      if (hbm) atomicAdd(&s_hbm, hbm);
      if (moved) atomicAdd(&s_moved, moved);
      if (end) atomicMax(&s_end, end);
    }
  }
  PREP_T(5);
  __syncthreads();
  PREP_T(6);
  if (nb > 1) {
    // the header's min / sums / max over CTAs: combined by the last CTA to finish
    if (threadIdx.x == 0) {
      long long* pt = a.xpart + blockIdx.x * 4;
      pt[0] = s_first_hole; pt[1] = (long long)s_hbm; pt[2] = (long long)s_moved; pt[3] = s_end;
      int old;                            // acq_rel: publishes pt, and the last CTA sees every CTA's
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(a.xdone) : "memory");
      s_last = old == nb - 1;
      if (s_last) {
        int fh = B;
        unsigned long long hb = 0, mv = 0;
        long long en = 0;
        for (int c = 0; c < nb; ++c) {
          const long long* q = a.xpart + c * 4;
          fh = min(fh, (int)__ldcg(q));
          hb += (unsigned long long)__ldcg(q + 1);
          mv += (unsigned long long)__ldcg(q + 2);
          en = max(en, __ldcg(q + 3));
        }
        s_first_hole = fh; s_hbm = hb; s_moved = mv; s_end = en;
        *a.xdone = 0;                                  // reusable by the next step
      }
    }
    __syncthreads();
#ifdef PREP_TRACE
    PREP_T(7);
    if (threadIdx.x == 0)
      printf("prep cta %d start %llu: pass1 %llu scan %llu wait %llu comb %llu pass2 %llu sync %llu last %llu\n",
             (int)blockIdx.x, ptt[0] % 1000000000ull, ptt[1] - ptt[0], ptt[2] - ptt[1], ptt[3] - ptt[2],
             ptt[4] - ptt[3], ptt[5] - ptt[4], ptt[6] - ptt[5], ptt[7] - ptt[6]);
#endif
    if (!s_last) return;
  }
#ifdef PREP_TRACE
  if (nb == 1 && threadIdx.x == 0)
    printf("prep 1 cta B %d: pass1 %llu scan %llu pass2 %llu sync %llu\n", B, ptt[1] - ptt[0], ptt[2] - ptt[1],
           ptt[5] - ptt[4], ptt[6] - ptt[5]);
#endif
  if (threadIdx.x == 0) {
    a.ctrl[CTRL_N_UNITS] = (int)tot[0];
    a.ctrl[CTRL_N_SPLITS] = (int)tot[1];
    a.ctrl[CTRL_ITEM] = 0;
    a.ctrl[CTRL_SPLIT_ITEM] = 0;
    a.ctrl[CTRL_FUSED] = fused ? 1 : 0;
    if (a.fused_out) *reinterpret_cast<volatile int32_t*>(a.fused_out) = fused ? 1 : 0;
    a.ctrl[CTRL_N_STAGES] = (int)tot[3];
    if (fused) {
      DReportHeader* h = reinterpret_cast<DReportHeader*>(a.report);
      h->n_before = B;
      h->n_finished = (int)tot[6];
      h->n_evicted = (int)tot[7];
      h->n_kept = (int)tot[4];
      h->tail = compact ? tot[5] : s_end;
      h->d2h_bytes = (int64_t)tot[8] * kvpt;
      h->moved_bytes = (int64_t)s_moved;
      h->pcie_bytes = 0;
      h->hbm_bytes = (int64_t)s_hbm;
      h->n_chunks = 0;
      h->n_entries = 0;
      h->first_hole = s_first_hole;
      h->fused = 1;
      h->compacted = compact ? 1 : 0;
    }
  }
}

// ---------------------------------------------------------------------------
// k_deps: for every ring stage of a MOVE unit, the source units whose rows
// overlap the stage's destination rows [d0, d1) (the new row included in a
// unit's last stage).  Sources are the units' arena rows [off+r0, off+r1),
// sorted and disjoint in unit order, so a binary search finds the first.
// One warp per unit, lanes over its stages.
// tc = 1 (k_attn_tc): stages are 128-row tiles and the new row is in the
// arena (row off+len; written by k_append, or in a host-fed step by the
// unit's producer warp just before its tiles load), so it is a source row of
// its unit and a tile row: no other unit stores into it before this unit's
// progress covers it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_deps(const Unit* __restrict__ units, const int32_t* __restrict__ ctrl,
                                              DepDesc* __restrict__ desc, int32_t tc) {
  const int n_units = ctrl[CTRL_N_UNITS];
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int tile = tc ? 128 : AT_RPS;
  for (int ui = gw; ui < n_units; ui += nw) {
    const Unit un = units[ui];
    const int rows = un.r1 - un.r0 + (tc ? un.has_new : 0);
    const int ns = rows > 0 ? (rows + tile - 1) / tile : 1;
    for (int s = lane; s < ns; s += 32) {
      DepDesc d;
      d.ua = -1; d.need_a = 0; d.ub = -1; d.need_b = 0;
      if (un.mode == UNIT_MOVE) {
        const int n = max(0, min(tile, rows - s * tile));
        const int64_t d0 = un.dst + un.r0 + (int64_t)s * tile;
        const int64_t d1 = d0 + n + ((!tc && s == ns - 1 && un.has_new) ? 1 : 0);
        int lo = 0, hi = n_units;              // first unit with source end > d0
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const Unit& m = units[mid];
          if ((int64_t)m.off + m.r1 + (tc ? m.has_new : 0) > d0) hi = mid; else lo = mid + 1;
        }
        for (int v = lo; v < n_units; ++v) {
          const Unit& m = units[v];
          const int64_t s0 = (int64_t)m.off + m.r0, s1 = (int64_t)m.off + m.r1 + (tc ? m.has_new : 0);
          if (s0 >= d1) break;
          if (s1 <= s0 || s1 <= d0) continue;  // empty source or no overlap
          const int need = (int)(min(d1, s1) - s0);
          if (d.ua < 0) { d.ua = v; d.need_a = need; }
          d.ub = v; d.need_b = need;
        }
      }
      desc[un.stage_base + s] = d;
    }
  }
}

// ---------------------------------------------------------------------------
// k_attn: persistent, dynamically scheduled over items (unit, layer).
// Each head is served by D/8 lanes; each lane owns 8 consecutive elements of
// the head (one 16-byte vector of K and of V per row).  Rows are streamed in
// groups of G with the next group's loads in flight while the current group
// is reduced: scores via lane-group xor shuffles, then an online softmax in
// the log2 domain (q is pre-scaled by log2(e)/sqrt(D)).
// ---------------------------------------------------------------------------
struct AttnArgs {
  Shape sh;
  const uint16_t* q;
  const uint16_t* k_new;
  const uint16_t* v_new;
  uint16_t* arena;
  uint8_t* staging;
  float* out;
  float* partials;
  const Unit* units;
  const DepDesc* desc;
  unsigned long long* progress;
  uint32_t epoch;
  int32_t* ctrl;
  int32_t B, l0, nl;
  float qscale;
  Feed feed;             // host-fed step: per-chunk ready words (s3_decode_step_host)
  uint32_t* evdone;      // per-evictee staged-row counters (cumulative; the D2H stream waits on them)
};

template <int D, int G>
__device__ __forceinline__ void attn_rows(const uint4 (&kc)[G], const uint4 (&vc)[G], int nvalid,
                                          const float (&qf)[8], float& m, float& s, float (&acc)[8]) {
  constexpr int LPH = D / 8;
  float sc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float kf[8];
    unpack8(kc[g], kf);
    float d = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) d = fmaf(qf[e], kf[e], d);
    sc[g] = d;
  }
#pragma unroll
  for (int o = LPH / 2; o > 0; o >>= 1)
#pragma unroll
    for (int g = 0; g < G; ++g) sc[g] += __shfl_xor_sync(0xffffffffu, sc[g], o);
  float mx = m;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (g >= nvalid) sc[g] = -INFINITY;
    mx = fmaxf(mx, sc[g]);
  }
  const float corr = ex2(m - mx);
  s *= corr;
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] *= corr;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float pr = ex2(sc[g] - mx);
    float vf[8];
    unpack8(vc[g], vf);
    s += pr;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = fmaf(pr, vf[e], acc[e]);
  }
  m = mx;
}

template <int D>
__global__ void __launch_bounds__(512, 1) k_attn(AttnArgs a) {
  constexpr int LPH = D / 8;    // lanes per head
  constexpr int HPW = 32 / LPH; // heads per warp
  constexpr int G = 4;          // rows per group
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int head = warp * HPW + lane / LPH;
  const int sub = lane % LPH;
  const int H = a.sh.H;
  const bool active = head < H;
  const int hh = active ? head : H - 1;
  const int hk = hh / (H / a.sh.Hkv);             // this query head's KV head
  const bool kv_writer = active && hh % (H / a.sh.Hkv) == 0;
  const int64_t HD = (int64_t)H * D, KD = (int64_t)a.sh.Hkv * D;
  const int64_t rowE = a.sh.row_elems;
  __shared__ int s_item;
  const int n_units = a.ctrl[CTRL_N_UNITS];
  const int total = n_units * a.nl;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&a.ctrl[CTRL_ITEM], 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= total) break;
    const int u = item / a.nl;
    const int li = item - u * a.nl;
    const int l = a.l0 + li;
    const Unit un = a.units[u];
    const uint16_t* kbase = a.arena + (int64_t)un.off * rowE + (int64_t)l * 2 * KD + hk * D + sub * 8;
    const uint16_t* vbase = kbase + KD;
    const int64_t io = ((int64_t)li * a.B + un.b) * HD + hh * D + sub * 8;
    const int64_t iok = ((int64_t)li * a.B + un.b) * KD + hk * D + sub * 8;
    float qf[8];
    unpack8(ld_plain(a.q + io), qf);
#pragma unroll
    for (int e = 0; e < 8; ++e) qf[e] *= a.qscale;
    float m = -INFINITY, s = 0.f, acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;

    uint4 kc[G], vc[G];
    int j = un.r0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const bool ok = j + g < un.r1;
      kc[g] = ok ? ld_stream(kbase + (int64_t)(j + g) * rowE) : make_uint4(0, 0, 0, 0);
      vc[g] = ok ? ld_stream(vbase + (int64_t)(j + g) * rowE) : make_uint4(0, 0, 0, 0);
    }
    while (j < un.r1) {
      const int jn = j + G;
      uint4 kn[G], vn[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool ok = jn + g < un.r1;
        kn[g] = ok ? ld_stream(kbase + (int64_t)(jn + g) * rowE) : make_uint4(0, 0, 0, 0);
        vn[g] = ok ? ld_stream(vbase + (int64_t)(jn + g) * rowE) : make_uint4(0, 0, 0, 0);
      }
      attn_rows<D, G>(kc, vc, min(G, un.r1 - j), qf, m, s, acc);
#pragma unroll
      for (int g = 0; g < G; ++g) { kc[g] = kn[g]; vc[g] = vn[g]; }
      j = jn;
    }
    if (un.has_new) {
      // append: row off+len <- (k_new, v_new), and attend to it from registers
      const uint4 kr = ld_plain(a.k_new + iok);
      const uint4 vr = ld_plain(a.v_new + iok);
      if (kv_writer) {
        st_v4((void*)(kbase + (int64_t)un.len * rowE), kr);
        st_v4((void*)(vbase + (int64_t)un.len * rowE), vr);
      }
      uint4 k1[1] = {kr}, v1[1] = {vr};
      attn_rows<D, 1>(k1, v1, 1, qf, m, s, acc);
    }
    if (active) {
      if (un.part < 0) {
        const float inv = 1.f / s;
        float4* o = reinterpret_cast<float4*>(a.out + io);
        o[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
        o[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
      } else {
        float* pr = a.partials + (((int64_t)un.part * a.nl + li) * H + hh) * (D + 4);
        float4* o = reinterpret_cast<float4*>(pr + sub * 8);
        o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        if (sub == 0) { pr[D] = m; pr[D + 1] = s; }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_combine: out = sum_i 2^(m_i - M) acc_i / sum_i 2^(m_i - M) l_i
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_combine(const Split* __restrict__ splits,
                                                 const float* __restrict__ partials,
                                                 float* __restrict__ out, int32_t* ctrl, int32_t H,
                                                 int32_t B, int32_t nl) {
  constexpr int EPL = D / 32;   // elements per lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int s_item;
  const int total = ctrl[CTRL_N_SPLITS] * nl;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&ctrl[CTRL_SPLIT_ITEM], 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= total) break;
    const Split sp = splits[item / nl];
    const int li = item % nl;
    for (int h = warp; h < H; h += nw) {
      float M = -INFINITY;
      for (int i = 0; i < sp.k; ++i)
        M = fmaxf(M, partials[(((int64_t)(sp.part0 + i) * nl + li) * H + h) * (D + 4) + D]);
      float acc[EPL], L = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
      for (int i = 0; i < sp.k; ++i) {
        const float* pr = partials + (((int64_t)(sp.part0 + i) * nl + li) * H + h) * (D + 4);
        const float w = ex2(pr[D] - M);
        L += w * pr[D + 1];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = fmaf(w, pr[lane * EPL + e], acc[e]);
      }
      const float inv = 1.f / L;
      float* o = out + (((int64_t)li * B + sp.b) * H + h) * D + lane * EPL;
#pragma unroll
      for (int e = 0; e < EPL; ++e) o[e] = acc[e] * inv;
    }
  }
}

// ---------------------------------------------------------------------------
// k_keep_scan: one CTA.  keep_b = (status == RUNNING); exclusive scans give
// new_idx, new_off (= sum of kept caps before b), evicted index and staging
// offset, finished index; a second scan numbers the move entries (moved
// survivors and evicted slots, in arena order) and their chunks.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_keep_scan(Shape sh, const DSlot* __restrict__ cur,
                                                    DSlot* __restrict__ next, int32_t B, int64_t S,
                                                    uint8_t* __restrict__ report,
                                                    MoveEntry* __restrict__ entries,
                                                    int32_t* __restrict__ key_chunk0,
                                                    int32_t* __restrict__ key_src,
                                                    int64_t* __restrict__ ctrl64,
                                                    int32_t compact_policy, int32_t pool_nonempty) {
  __shared__ int s_first_hole;
  __shared__ unsigned long long s_hbm;
  __shared__ long long s_end;
  if (threadIdx.x == 0) { s_first_hole = B; s_hbm = 0; s_end = 0; }
  const int per = (B + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(B, b0 + per);
  const int64_t kvpt = sh.kvpt;
  // pass A: keep, keep*cap, fin, ev, ev*len*kvpt, cap, ev*cap
  long long x[6] = {0, 0, 0, 0, 0, 0};
  for (int b = b0; b < b1; ++b) {
    const DSlot sl = cur[b];
    const int keep = sl.status == 0, fin = sl.status == 1, ev = sl.status == 2;
    x[0] += keep;
    x[1] += keep ? sl.cap : 0;
    x[2] += fin;
    x[3] += ev;
    x[4] += ev ? (long long)sl.len * kvpt : 0;
    x[5] += sl.cap;
  }
  long long tot[6];
  block_excl_scan<6>(x, tot);
  const bool compact = compact_policy == 0 || pool_nonempty || tot[3] > 0;   // R27
  int32_t* perm = reinterpret_cast<int32_t*>(report + report_perm_off(B));
  DEvicted* evl = reinterpret_cast<DEvicted*>(report + report_ev_off(B));
  int64_t* finl = reinterpret_cast<int64_t*>(report + report_fin_off(B));
  // pass B: move entries
  long long y[3] = {0, 0, 0};   // entries, chunks, moved bytes
  {
    long long keep_i = x[0], keepcap = x[1], fin_i = x[2], ev_i = x[3], evb = x[4], capx = x[5];
    unsigned long long hbm = 0;
    long long end = 0;
    int first = B;
    for (int b = b0; b < b1; ++b) {
      DSlot sl = cur[b];
      const int keep = sl.status == 0;
      if (!keep && b < first) first = b;
      if (keep) {
        perm[b] = (int)keep_i;
        const int64_t new_off = compact ? keepcap : sl.off;
        const int64_t bytes = (int64_t)sl.len * kvpt;
        if (new_off != sl.off && bytes > 0) { y[0] += 1; y[1] += (bytes + S - 1) / S; y[2] += bytes; }
        sl.off = (int32_t)new_off;
        sl.status = 0;
        end = max(end, (long long)new_off + sl.cap);
        next[keep_i] = sl;
        ++keep_i;
        keepcap += sl.cap;
      } else {
        perm[b] = -1;
        if (sl.status == 1) {
          finl[fin_i++] = sl.req;
        } else {
          const int64_t bytes = (int64_t)sl.len * kvpt;
          DEvicted e;
          e.req = sl.req; e.b = b; e.prompt = sl.prompt; e.gen = sl.gen; e.len = sl.len;
          e.cap = sl.cap; e.pad = 0; e.stage_off = evb;
          evl[ev_i++] = e;
          evb += bytes;
          hbm += 2ull * (unsigned long long)(tot[5] - capx - sl.cap) * (unsigned long long)kvpt;
          if (bytes > 0) { y[0] += 1; y[1] += (bytes + S - 1) / S; }
        }
      }
      capx += sl.cap;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {   // warp-reduce before the shared atomics (see k_prep)
      first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
      hbm += __shfl_xor_sync(0xffffffffu, hbm, o);
      end = max(end, __shfl_xor_sync(0xffffffffu, end, o));
    }
    if ((threadIdx.x & 31) == 0) {
      if (first < B) atomicMin(&s_first_hole, first);
      if (hbm) atomicAdd(&s_hbm, hbm);
      if (end) atomicMax(&s_end, end);
    }
  }
  long long ytot[3];
  block_excl_scan<3>(y, ytot);
  {
    long long e_i = y[0], chunk = y[1];
    long long keepcap = x[1], evb = x[4];
    for (int b = b0; b < b1; ++b) {
      const DSlot sl = cur[b];
      const int64_t bytes = (int64_t)sl.len * kvpt;
      if (sl.status == 0) {
        const int64_t new_off = compact ? keepcap : sl.off;
        if (new_off != sl.off && bytes > 0) {
          MoveEntry me;
          me.src = (int64_t)sl.off * kvpt; me.dst = new_off * kvpt; me.bytes = bytes;
          me.chunk0 = chunk; me.kind = MOVE_ARENA; me.pad0 = 0; me.pad1 = 0;
          key_chunk0[e_i] = (int32_t)chunk;
          key_src[e_i] = sl.off;
          entries[e_i++] = me;
          chunk += (bytes + S - 1) / S;
        }
        keepcap += sl.cap;
      } else if (sl.status == 2) {
        if (bytes > 0) {
          MoveEntry me;
          me.src = (int64_t)sl.off * kvpt; me.dst = evb; me.bytes = bytes;
          me.chunk0 = chunk; me.kind = MOVE_STAGE; me.pad0 = 0; me.pad1 = 0;
          key_chunk0[e_i] = (int32_t)chunk;
          key_src[e_i] = sl.off;
          entries[e_i++] = me;
          chunk += (bytes + S - 1) / S;
        }
        evb += bytes;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    DReportHeader* h = reinterpret_cast<DReportHeader*>(report);
    h->n_before = B;
    h->n_finished = (int)tot[2];
    h->n_evicted = (int)tot[3];
    h->n_kept = (int)tot[0];
    h->tail = compact ? tot[1] : s_end;
    h->d2h_bytes = tot[4];
    h->moved_bytes = ytot[2];
    h->pcie_bytes = 0;
    h->hbm_bytes = (int64_t)s_hbm;
    h->n_chunks = ytot[1];
    h->n_entries = (int)ytot[0];
    h->first_hole = s_first_hole;
    h->fused = 0;
    h->compacted = compact ? 1 : 0;
    ctrl64[CTRL64_TICKET] = 0;
    ctrl64[CTRL64_N_CHUNKS] = ytot[1];
    key_chunk0[ytot[0]] = (int32_t)ytot[1];
  }
}

// ---------------------------------------------------------------------------
// k_move: ordered in-place compaction (+ eviction staging) on the TMA bulk
// copy engine.
//
// The bytes to move form "entries" (moved survivors and evicted slots) in
// SOURCE order (= arena order), cut into chunks of S bytes numbered in that
// order.  Every CTA runs MV_NP independent (producer, consumer) thread pairs,
// each with MV_NB shared-memory buffers:
//   producer: take the next chunk ticket (atomic), cp.async.bulk G->S of its
//             source, completion on an mbarrier;
//   consumer: when the bytes have landed, publish "read done" for the chunk
//             (st.release), then -- only for arena destinations -- wait
//             (ld.acquire) until every chunk whose SOURCE overlaps this
//             chunk's DESTINATION has been read, and cp.async.bulk S->G.
// Every source lies at or above its destination, so the awaited chunks hold
// earlier tickets; the smallest unpublished ticket always sits at the head
// of its consumer and is published as soon as its load lands, so the wait
// chain strictly decreases and cannot deadlock.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

constexpr int MV_NP = 3;   // producer/consumer pairs per CTA
constexpr int MV_NB = 2;   // buffers per pair

struct MoveArgs {
  uint8_t* arena;
  uint8_t* staging;
  const MoveEntry* entries;
  const int32_t* key_chunk0;   // [n_entries + 1], last = n_chunks
  const int32_t* key_src;      // [n_entries] source row
  int32_t n_entries;
  int32_t keys_in_smem;
  int64_t n_chunks, S, kvpt;
  int64_t* ctrl64;
  uint32_t* flags;
  uint32_t epoch;
  int32_t staging_enabled;
};

__device__ __forceinline__ int chunk_entry(const int32_t* kc, int n, int64_t t) {
  int lo = 0, hi = n - 1;               // largest e with kc[e] <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (kc[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Wait until every chunk whose source overlaps [d0, d1) (arena bytes) has
// been read.  Entry i covers at most [src_i, src_i + nch_i*S); that bound is
// non-decreasing in i, so the first candidate is found by binary search.
__device__ void wait_sources(const int32_t* kc, const int32_t* ks, int n, int64_t kvpt, int64_t S,
                             int64_t d0, int64_t d1, int64_t self, const uint32_t* flags, uint32_t epoch) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)ks[mid] * kvpt + (int64_t)(kc[mid + 1] - kc[mid]) * S > d0) hi = mid; else lo = mid + 1;
  }
  for (int i = lo; i < n && (int64_t)ks[i] * kvpt < d1; ++i) {
    const int64_t src = (int64_t)ks[i] * kvpt, nch = kc[i + 1] - kc[i];
    const int64_t c_lo = d0 > src ? (d0 - src) / S : 0;
    const int64_t c_hi = min(nch - 1, (d1 - 1 - src) / S);
    for (int64_t c = c_lo; c <= c_hi; ++c) {
      const int64_t k = kc[i] + c;
      if (k == self) continue;
      while (ld_acquire_u32(flags + k) != epoch) __nanosleep(32);
    }
  }
}

__global__ void __launch_bounds__(64 * MV_NP) k_move(MoveArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t S = a.S;
  uint8_t* bufs = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)MV_NP * MV_NB * S);
  uint64_t* empty = full + MV_NP * MV_NB;
  long long* tix = reinterpret_cast<long long*>(empty + MV_NP * MV_NB);
  int32_t* ent = reinterpret_cast<int32_t*>(tix + MV_NP * MV_NB);
  int32_t* skeys = ent + MV_NP * MV_NB;
  const int n = a.n_entries;
  const int32_t* kc = a.key_chunk0;
  const int32_t* ks = a.key_src;
  if (a.keys_in_smem) {
    for (int i = threadIdx.x; i <= n; i += blockDim.x) skeys[i] = a.key_chunk0[i];
    for (int i = threadIdx.x; i < n; i += blockDim.x) skeys[n + 1 + i] = a.key_src[i];
    kc = skeys;
    ks = skeys + n + 1;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < MV_NP * MV_NB; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane != 0) return;
  const int pair = warp >> 1;
  uint8_t* pb = bufs + (size_t)pair * MV_NB * S;
  uint64_t* pf = full + pair * MV_NB;
  uint64_t* pe = empty + pair * MV_NB;
  long long* pt = tix + pair * MV_NB;
  int32_t* pen = ent + pair * MV_NB;
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(&a.ctrl64[CTRL64_TICKET]);
  if ((warp & 1) == 0) {
    // ---------------- producer ----------------
    for (int k = 0;; ++k) {
      const int i = k % MV_NB;
      const uint32_t ph = (uint32_t)(k / MV_NB) & 1u;
      mbar_wait(&pe[i], ph ^ 1u);                    // buffer free (passes at once on first use)
      const long long t = (long long)atomicAdd(ticket, 1ull);
      pt[i] = t;
      if (t >= a.n_chunks) { mbar_arrive(&pf[i]); break; }
      const int e = chunk_entry(kc, n, t);
      pen[i] = e;
      const MoveEntry me = a.entries[e];
      const int64_t pos = (t - kc[e]) * S;
      const uint32_t nb = (uint32_t)min(S, me.bytes - pos);
      if (me.kind == MOVE_ARENA || a.staging_enabled) {
        mbar_arrive_expect_tx(&pf[i], nb);
        bulk_g2s(pb + (size_t)i * S, a.arena + me.src + pos, nb, &pf[i]);
      } else {
        mbar_arrive(&pf[i]);                         // evicted, not staged: nothing to copy
      }
    }
  } else {
    // ---------------- consumer ----------------
    for (int k = 0;; ++k) {
      const int i = k % MV_NB;
      const uint32_t ph = (uint32_t)(k / MV_NB) & 1u;
      mbar_wait(&pf[i], ph);
      const long long t = pt[i];
      if (t >= a.n_chunks) break;
      const int e = pen[i];
      const MoveEntry me = a.entries[e];
      const int64_t pos = (t - kc[e]) * S;
      const uint32_t nb = (uint32_t)min(S, me.bytes - pos);
      st_release_u32(a.flags + t, a.epoch);          // source chunk t has been read
      if (me.kind == MOVE_ARENA) {
        wait_sources(kc, ks, n, a.kvpt, S, me.dst + pos, me.dst + pos + nb, t, a.flags, a.epoch);
        asm volatile("fence.proxy.async;" ::: "memory");
        bulk_s2g(a.arena + me.dst + pos, pb + (size_t)i * S, nb);
      } else if (a.staging_enabled) {
        bulk_s2g(a.staging + me.dst + pos, pb + (size_t)i * S, nb);
      }
      mbar_arrive(&pe[i]);
    }
  }
}

int move_smem_bytes(int64_t S, int32_t n_entries, int32_t* keys_in_smem) {
  const int64_t base = (int64_t)MV_NP * MV_NB * (S + 8 + 8 + 8 + 4);
  const int64_t keys = 4LL * (2LL * n_entries + 1);
  const int64_t limit = 227 * 1024;
  *keys_in_smem = base + keys <= limit;
  return (int)(base + (*keys_in_smem ? keys : 0));
}

// ---------------------------------------------------------------------------
// k_attn_tma: decode attention with the KV stream staged by the TMA bulk
// copy engine, fused with the row shift.
//
//  producer warp (1 thread): takes items (unit, layer) from the queue and
//    streams each item's rows -- one contiguous 4*H*D-byte layer-row (K of all
//    heads, then V) per cp.async.bulk -- plus the item's q into an
//    ns-stage shared-memory ring (mbarrier full/empty per stage);
//  consumer warps (H*D/256; D/8 lanes per head): 128-bit loads from the
//    stage, online softmax; at the item's end append the new row (k_new,
//    v_new) at its final position and write out / the split-K partial;
//  storer warp (1 thread): when a stage lands, publishes the item's read
//    progress (st.release), and for MOVE units waits (ld.acquire) until every
//    source unit overlapping the stage's destination rows has been read that
//    far (k_deps), then bulk-stores the stage's rows to their compacted rows;
//    STAGE units (evicted) are bulk-stored to the staging buffer.
// Deadlock freedom: items are handed out in unit order and every destination
// row lies at or below its source row, so a stage only waits on items with
// smaller tickets (or on rows of its own item that are already in shared
// memory); the smallest waiting item always progresses.
// ---------------------------------------------------------------------------
constexpr int AT_NS_MAX = 8;
constexpr unsigned long long PROG_FULL = 0x80000000ull;

struct StageHdr {
  DepDesc dep;                 // filled by the TMA engine (16 B, same transaction as the rows)
  int32_t item, r0, n, flags;  // flags: 1 = first stage of the item, 2 = last, 4 = unit has the new row
  int32_t b, part, off, len;   // the item's unit (so consumers never load it from global)
  int32_t mode, unit_r0, dep_ok, ev;    // dep_ok: storer's "destination free" stamp (stage seq + 1);
                                        // ev: eviction index of a STAGE unit
  int64_t dst, pad2;
};
static_assert(sizeof(StageHdr) % 16 == 0, "StageHdr must keep 16-B alignment");

__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_s32(int32_t* p, int32_t v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_cta_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void bulk_s2g_nocommit(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(576, 1) k_attn_tma(AttnArgs a, int32_t ns) {
  constexpr int LPH = D / 8;
  constexpr int HPW = 32 / LPH;
  extern __shared__ __align__(128) uint8_t smem[];
  const int H = a.sh.H;
  const int64_t HD = (int64_t)H * D, KD = (int64_t)a.sh.Hkv * D;
  const int64_t rowB = 4 * KD;                     // one layer-row: K and V of all KV heads
  const int64_t stageB = AT_RPS * rowB + 2 * HD;   // rows + q of the item (H query heads)
  const int64_t kvpt = a.sh.kvpt;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ns * stageB);
  uint64_t* empty = full + ns;
  StageHdr* hdr = reinterpret_cast<StageHdr*>(empty + ns);
  const int nwarps = blockDim.x >> 5;
  const int nwc = nwarps - 2;                      // consumer warps; then producer, storer
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the storer takes part in the ring only when this step moves rows
  const bool fused = a.ctrl[CTRL_FUSED] != 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], nwc + (fused ? 1 : 0));
      hdr[i].dep_ok = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_units = a.ctrl[CTRL_N_UNITS];
  const int total = n_units * a.nl;
  const uint8_t* arena = reinterpret_cast<const uint8_t*>(a.arena);
  if (warp == nwc) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      int k = 0;
      int ready_max = -1;               // host-fed step: highest chunk known to have landed
      for (;;) {
        const int item = atomicAdd(&a.ctrl[CTRL_ITEM], 1);
        if (item >= total) {
          const int st = k % ns;
          mbar_wait(&empty[st], ((uint32_t)(k / ns) & 1u) ^ 1u);
          hdr[st].item = -1;
          mbar_arrive(&full[st]);
          break;
        }
        const int u = item / a.nl, li = item - u * a.nl;
        const Unit un = a.units[u];
        if (a.feed.ready) {
          // chunks land in order: waiting for this unit's chunk covers every earlier one
          const int c = un.b / a.feed.cb;
          if (c > ready_max) { wait_ready(a.feed.ready + c, a.feed.epoch); ready_max = c; }
        }
        const uint8_t* base = arena + (int64_t)un.off * kvpt + (int64_t)(a.l0 + li) * rowB;
        const uint16_t* qsrc = a.q + ((int64_t)li * a.B + un.b) * HD;
        int r = un.r0, s = 0;
        do {
          const int st = k % ns;
          mbar_wait(&empty[st], ((uint32_t)(k / ns) & 1u) ^ 1u);
          const int n = min(AT_RPS, un.r1 - r);
          const bool first = r == un.r0;
          StageHdr& h = hdr[st];
          h.item = item; h.r0 = r; h.n = n;
          h.flags = (first ? 1 : 0) | (r + n >= un.r1 ? 2 : 0) | (un.has_new ? 4 : 0);
          h.b = un.b; h.part = un.part; h.off = un.off; h.len = un.len;
          h.mode = un.mode; h.unit_r0 = un.r0; h.dst = un.dst; h.ev = un.pad;
          const bool mv = un.mode == UNIT_MOVE;
          const uint32_t tx = (uint32_t)(n * rowB + (first ? 2 * HD : 0) + (mv ? sizeof(DepDesc) : 0));
          uint8_t* sb = smem + st * stageB;
          if (tx) {
            mbar_arrive_expect_tx(&full[st], tx);
            if (mv) bulk_g2s(&h.dep, a.desc + un.stage_base + s, (uint32_t)sizeof(DepDesc), &full[st]);
            if (first) bulk_g2s(sb + AT_RPS * rowB, qsrc, (uint32_t)(2 * HD), &full[st]);
            for (int i = 0; i < n; ++i)
              bulk_g2s(sb + i * rowB, base + (int64_t)(r + i) * kvpt, (uint32_t)rowB, &full[st]);
          } else {
            mbar_arrive(&full[st]);
          }
          r += n;
          ++s;
          ++k;
        } while (r < un.r1);
      }
    }
    return;
  }
  if (warp == nwc + 1) {
    // ------------------------------- storer -------------------------------
    if (lane == 0 && fused) {
      int pending = -1;                 // stage whose stores may still read shared memory
      uint32_t ev_rows = 0;             // rows of the current STAGE item written to staging so far
      int64_t seen_item = -1;           // progress cache: last observed source item / value
      unsigned long long seen_val = 0;
      for (int k = 0;; ++k) {
        const int st = k % ns;
        mbar_wait(&full[st], (uint32_t)(k / ns) & 1u);
        StageHdr& hs = hdr[st];
        const StageHdr h = hs;
        if (h.item < 0) break;
        const int li = h.item % a.nl;
        const unsigned long long done =
            (unsigned long long)(h.r0 + h.n - h.unit_r0) | ((h.flags & 2) ? PROG_FULL : 0ull);
        // the stage's bytes are in shared memory (mbarrier observed): the
        // source rows may be overwritten from now on
        st_relaxed_u64(a.progress + h.item, ((unsigned long long)a.epoch << 32) | done);
        bool stores = false;
        if (h.mode == UNIT_MOVE) {
          // destination rows free?  (own-item rows are already in shared memory)
          const DepDesc& d = h.dep;
          if (d.ua >= 0) {
            for (int v = d.ua; v <= d.ub; ++v) {
              const int need = v == d.ua ? d.need_a : (v == d.ub ? d.need_b : -1);
              const int64_t it = (int64_t)v * a.nl + li;
              if (it == h.item) continue;
              for (;;) {
                if (it != seen_item) { seen_item = it; seen_val = ld_acquire_u64(a.progress + it); }
                const unsigned long long x = seen_val;
                if ((uint32_t)(x >> 32) == a.epoch && ((x & PROG_FULL) || (need >= 0 && (int)(x & 0x7fffffffull) >= need)))
                  break;
                __nanosleep(32);
                seen_val = ld_acquire_u64(a.progress + it);
              }
            }
          }
          asm volatile("fence.proxy.async;" ::: "memory");
          st_release_cta_s32(&hs.dep_ok, k + 1);   // consumers may now write the new row
          stores = h.n > 0;
        } else if (h.mode == UNIT_STAGE) {
          stores = h.n > 0;
        }
        if (stores) {
          uint8_t* dbase = h.mode == UNIT_MOVE
                               ? reinterpret_cast<uint8_t*>(a.arena) + (h.dst + h.r0) * kvpt
                               : a.staging + h.dst + (int64_t)h.r0 * kvpt;
          const uint8_t* sb = smem + st * stageB;
          for (int i = 0; i < h.n; ++i)
            bulk_s2g_nocommit(dbase + (int64_t)i * kvpt + (int64_t)(a.l0 + li) * rowB, sb + i * rowB,
                              (uint32_t)rowB);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        // release the previous stage once its stores have read shared memory
        if (pending >= 0) {
          if (stores) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(&empty[pending]);
          pending = -1;
        }
        if (stores) pending = st;
        else mbar_arrive(&empty[st]);
        if (h.mode == UNIT_STAGE && a.evdone) {
          // an evictee's rows are final in staging once the item's stores have
          // completed (not just read shared memory): count them for the D2H
          // stream, which copies each evictee as soon as its count is complete
          ev_rows += (uint32_t)h.n;
          if (h.flags & 2) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.evdone + h.ev), "r"(ev_rows) : "memory");
            ev_rows = 0;
          }
        }
      }
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (pending >= 0) mbar_arrive(&empty[pending]);
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  // -------------------------------- consumers --------------------------------
  const int head = warp * HPW + lane / LPH;
  const int sub = lane % LPH;
  const bool active = head < H;
  const int hh = active ? head : H - 1;
  const int hk = hh / (H / a.sh.Hkv);             // this query head's KV head
  const bool kv_writer = active && hh % (H / a.sh.Hkv) == 0;
  const int64_t rowE = a.sh.row_elems;
  float qf[8], m = -INFINITY, ssum = 0.f, acc[8];
  int li = 0;
  for (int k = 0;; ++k) {
    const int st = k % ns;
    mbar_wait(&full[st], (uint32_t)(k / ns) & 1u);
    const StageHdr h = hdr[st];
    if (h.item < 0) break;
    const uint8_t* sb = smem + st * stageB;
    if (h.flags & 1) {
      li = h.item % a.nl;
      unpack8(lds128(sb + AT_RPS * rowB + (hh * D + sub * 8) * 2), qf);
#pragma unroll
      for (int e = 0; e < 8; ++e) { qf[e] *= a.qscale; acc[e] = 0.f; }
      m = -INFINITY;
      ssum = 0.f;
    }
    const int64_t io = ((int64_t)li * a.B + h.b) * HD + hh * D + sub * 8;
    const int64_t iok = ((int64_t)li * a.B + h.b) * KD + hk * D + sub * 8;
    uint4 kr = make_uint4(0, 0, 0, 0), vr = kr;
    const bool last_new = (h.flags & 2) && (h.flags & 4);
    if (last_new) {              // issue the new row's loads early; used after the stage
      if (a.feed.ready) {        // landed during this kernel (ordered by the producer's acquire)
        kr = ld_cg(a.k_new + iok);
        vr = ld_cg(a.v_new + iok);
      } else {
        kr = ld_plain(a.k_new + iok);
        vr = ld_plain(a.v_new + iok);
      }
    }
    if (h.n > 0) {
      uint4 kc[AT_RPS], vc[AT_RPS];
#pragma unroll
      for (int i = 0; i < AT_RPS; ++i) {
        if (i < h.n) {
          kc[i] = lds128(sb + i * rowB + (hk * D + sub * 8) * 2);
          vc[i] = lds128(sb + i * rowB + (KD + hk * D + sub * 8) * 2);
        } else {
          kc[i] = make_uint4(0, 0, 0, 0);
          vc[i] = kc[i];
        }
      }
      attn_rows<D, AT_RPS>(kc, vc, h.n, qf, m, ssum, acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (h.flags & 2) {
      if (last_new) {
        // append: the new row goes where the slot's rows end up
        uint16_t* kdst = nullptr;
        const int64_t lofs = (int64_t)(a.l0 + li) * 2 * KD + hk * D + sub * 8;
        if (h.mode == UNIT_STAY) {
          kdst = a.arena + (int64_t)(h.off + h.len) * rowE + lofs;
        } else if (h.mode == UNIT_MOVE) {
          // the storer stamps the stage once its destination rows (new row included) are free
          while (ld_acquire_cta_s32(&hdr[st].dep_ok) < k + 1) __nanosleep(20);
          kdst = a.arena + (h.dst + h.len) * rowE + lofs;
        } else if (h.mode == UNIT_STAGE) {
          kdst = reinterpret_cast<uint16_t*>(a.staging + h.dst + (int64_t)h.len * kvpt) + lofs;
        }
        if (kv_writer && kdst) {
          st_v4(kdst, kr);
          st_v4(kdst + KD, vr);
        }
        if (h.mode == UNIT_STAGE && a.evdone) {   // this warp's part of the evictee's new row is stored
          __syncwarp();
          if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.evdone + h.ev) : "memory");
        }
        uint4 k1[1] = {kr}, v1[1] = {vr};
        attn_rows<D, 1>(k1, v1, 1, qf, m, ssum, acc);
      }
      if (active) {
        if (h.part < 0) {
          const float inv = 1.f / ssum;
          float4* o = reinterpret_cast<float4*>(a.out + io);
          o[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
          o[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
        } else {
          float* pr = a.partials + (((int64_t)h.part * a.nl + li) * H + hh) * (D + 4);
          float4* o = reinterpret_cast<float4*>(pr + sub * 8);
          o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
          if (sub == 0) { pr[D] = m; pr[D + 1] = ssum; }
        }
      }
      if (a.feed.done && h.part < 0) {
        // host-fed step with a device out: count this warp's final rows for the
        // copy stream that waits on the chunk's counter (release orders the warp's stores)
        __syncwarp();
        if (lane == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.feed.done + h.b / a.feed.cb) : "memory");
      }
    }
  }
}

int attn_tma_stages(const Shape& sh) {
  const int64_t HD = (int64_t)sh.H * sh.D, KD = (int64_t)sh.Hkv * sh.D;
  const int64_t stageB = AT_RPS * 4 * KD + 2 * HD;
  const int64_t per = stageB + 16 + sizeof(StageHdr);
  const int64_t ns = (227 * 1024 - 64) / per;
  return (int)std::min<int64_t>(ns, AT_NS_MAX);
}
int attn_tma_smem(const Shape& sh, int ns) {
  const int64_t HD = (int64_t)sh.H * sh.D, KD = (int64_t)sh.Hkv * sh.D;
  return (int)(ns * (AT_RPS * 4 * KD + 2 * HD) + ns * (16 + (int64_t)sizeof(StageHdr)));
}
const void* attn_tma_kernel_ptr(const Shape& sh) {
  switch (sh.D) {
    case 64: return (const void*)k_attn_tma<64>;
    case 128: return (const void*)k_attn_tma<128>;
    case 256: return (const void*)k_attn_tma<256>;
    default: return nullptr;
  }
}

// ---------------------------------------------------------------------------
// k_fill: prompt rows 0..P-1 of freshly admitted slots (stand-in for the
// model's prefill).  grid = (row groups, admitted slots).
// ---------------------------------------------------------------------------
constexpr int FILL_ROWS = 4;
__global__ void __launch_bounds__(256) k_fill(Shape sh, uint64_t seed, const DSlot* __restrict__ slots,
                                              const int32_t* __restrict__ list, uint16_t* __restrict__ arena) {
  const DSlot sl = slots[list[blockIdx.y]];
  const int p0 = blockIdx.x * FILL_ROWS;
  if (p0 >= sl.prompt) return;
  const int p1 = min(sl.prompt, p0 + FILL_ROWS);
  const int D8 = sh.D / 8;
  const int per_row = sh.L * 2 * sh.Hkv * D8;   // 16-byte vectors per row
  const int total = (p1 - p0) * per_row;
  const int seg = sh.Hkv * D8;                  // vectors of one (layer, K/V) piece: counter base + u
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int pos = p0 + i / per_row;
    const int r = i % per_row;
    const int lkv = r / seg, u = r - lkv * seg;   // lkv = 2 l + kv; u = h D/8 + d8
    const uint4 v = gen8_at(seed, 0, gen_row_base(sh, (uint64_t)sh.Hkv, sl.req, lkv >> 1, lkv & 1, pos) + (uint64_t)u,
                            1.f / 128.f);
    st_v4(arena + ((int64_t)sl.off + pos) * sh.row_elems + (int64_t)r * 8, v);
  }
}

// ---------------------------------------------------------------------------
// k_synth: q / k_new / v_new [nl][B][H][D] at position len_b, and eos.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_synth(Shape sh, uint64_t seed, const DSlot* __restrict__ slots,
                                               int32_t B, int32_t l0, int32_t nl,
                                               const int32_t* __restrict__ out_len, int64_t n_req,
                                               uint16_t* q, uint16_t* k, uint16_t* v, uint8_t* eos) {
  // one (layer, slot) row per block iteration; 32-bit index math inside the row
  const int D8 = sh.D / 8;
  const int nq = sh.H * D8, nk = sh.Hkv * D8;          // 16-B vectors per row of q / of k_new, v_new
  for (int64_t row = blockIdx.x; row < (int64_t)nl * B; row += gridDim.x) {
    const int li = (int)(row / B), b = (int)(row - (int64_t)li * B);
    const DSlot sl = slots[b];
    const int l = l0 + li;
    // vector t of a row has counter row_base + t (h D/8 + d8 == t), so only the row bases are multiplied out
    const uint64_t gq = gen_row_base(sh, (uint64_t)sh.H, sl.req, l, 0, sl.len);
    const uint64_t gk = gen_row_base(sh, (uint64_t)sh.Hkv, sl.req, l, 0, sl.len);
    const uint64_t gv = gen_row_base(sh, (uint64_t)sh.Hkv, sl.req, l, 1, sl.len);
    for (int t = threadIdx.x; t < nq + nk; t += blockDim.x) {
      if (t < nq) {                                     // q: [nl][B][H][D]
        st_v4(q + (row * nq + t) * 8, gen8_at(seed, 1, gq + (uint64_t)t, 1.f / 32.f));
      } else {                                          // k_new, v_new: [nl][B][Hkv][D]
        const int u = t - nq;
        const int64_t o = (row * nk + u) * 8;
        st_v4(k + o, gen8_at(seed, 0, gk + (uint64_t)u, 1.f / 128.f));
        st_v4(v + o, gen8_at(seed, 0, gv + (uint64_t)u, 1.f / 128.f));
      }
    }
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    const DSlot s2 = slots[i];
    const int O = (s2.req >= 0 && s2.req < n_req) ? out_len[s2.req] : 0x7fffffff;
    eos[i] = (uint8_t)(s2.gen + 1 == O);
  }
}

// ---------------------------------------------------------------------------
// k_verify: count 16-byte vectors of resident rows that differ from G.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_verify(Shape sh, uint64_t seed, const DSlot* __restrict__ slots,
                                                const uint16_t* __restrict__ arena,
                                                unsigned long long* bad) {
  const DSlot sl = slots[blockIdx.y];
  const int D8 = sh.D / 8;
  const int64_t per_row = (int64_t)sh.L * 2 * sh.Hkv * D8;
  const int64_t total = (int64_t)sl.len * per_row;
  unsigned long long nbad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int pos = (int)(i / per_row);
    int64_t r = i % per_row;
    const int d8 = (int)(r % D8); r /= D8;
    const int h = (int)(r % sh.Hkv); r /= sh.Hkv;
    const int kv = (int)(r % 2);
    const int l = (int)(r / 2);
    const uint4 want = gen8(sh, seed, 0, sl.req, l, kv, pos, h, d8, 1.f / 128.f);
    const uint4 got = ld_plain(arena + ((int64_t)sl.off + pos) * sh.row_elems +
                               ((int64_t)(l * 2 + kv) * sh.Hkv + h) * sh.D + d8 * 8);
    nbad += (want.x != got.x) | (want.y != got.y) | (want.z != got.z) | (want.w != got.w);
  }
  if (nbad) atomicAdd(bad, nbad);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int attn_block_threads(const Shape& sh) {
  const int lanes = sh.H * sh.D / 8;
  return ((lanes + 31) / 32) * 32;
}

const void* attn_kernel_ptr(const Shape& sh) {
  switch (sh.D) {
    case 64: return (const void*)k_attn<64>;
    case 128: return (const void*)k_attn<128>;
    case 256: return (const void*)k_attn<256>;
    default: return nullptr;
  }
}
const void* move_kernel_ptr() { return (const void*)k_move; }

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st) {
  // up to 2 slots per thread one CTA is fastest; beyond, one CTA per 512 slots (B = 16384: 32
  // CTAs; 1024-slot CTAs measured 1.6x slower in-kernel: longer block scans and store queues)
  static const int single = [] { const char* e = getenv("S3_PREP_SINGLE_CTA"); return e ? atoi(e) : 0; }();  // A/B
  static const int thr = [] { const char* e = getenv("S3_PREP_THREADS"); return e ? atoi(e) : 512; }();
  static const int single_max = [] { const char* e = getenv("S3_PREP_SINGLE_MAX"); return e ? atoi(e) : 2 * PREP_CTA_SLOTS; }();
  const int nb = (single || a.B <= single_max) ? 1 : std::min((a.B + thr - 1) / thr, PREP_MAX_CTAS);
  k_prep<<<nb, nb == 1 ? 1024 : thr, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_deps(const Unit* units, const int32_t* ctrl, DepDesc* desc, int32_t tc, int32_t grid,
                        cudaStream_t st) {
  k_deps<<<grid, 256, 0, st>>>(units, ctrl, desc, tc);
  return cudaGetLastError();
}

cudaError_t launch_attn(const Shape& sh, const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                        uint16_t* arena, uint8_t* staging, float* out, float* partials, const Unit* units,
                        const Split* splits, const DepDesc* desc, unsigned long long* progress, uint32_t epoch,
                        int32_t* ctrl, int32_t B, int32_t l0, int32_t nl, int32_t grid_attn, int32_t grid_combine,
                        int32_t variant, const Feed& feed, uint32_t* evdone, cudaStream_t st) {
  AttnArgs a;
  a.feed = feed;
  a.evdone = evdone;
  a.sh = sh; a.q = q; a.k_new = k_new; a.v_new = v_new; a.arena = arena; a.staging = staging; a.out = out;
  a.partials = partials; a.units = units; a.desc = desc; a.progress = progress; a.epoch = epoch;
  a.ctrl = ctrl; a.B = B; a.l0 = l0; a.nl = nl;
  a.qscale = 1.4426950408889634f / sqrtf((float)sh.D);
  const int threads = attn_block_threads(sh);
  const int ns = attn_tma_stages(sh);
  const bool tma = variant == 0 && ns >= 2;
  const int smem = tma ? attn_tma_smem(sh, ns) : 0;
  switch (sh.D) {
    case 64:
      if (tma) k_attn_tma<64><<<grid_attn, threads + 64, smem, st>>>(a, ns);
      else k_attn<64><<<grid_attn, threads, 0, st>>>(a);
      k_combine<64><<<grid_combine, 256, 0, st>>>(splits, partials, out, ctrl, sh.H, B, nl);
      break;
    case 128:
      if (tma) k_attn_tma<128><<<grid_attn, threads + 64, smem, st>>>(a, ns);
      else k_attn<128><<<grid_attn, threads, 0, st>>>(a);
      k_combine<128><<<grid_combine, 256, 0, st>>>(splits, partials, out, ctrl, sh.H, B, nl);
      break;
    case 256:
      if (tma) k_attn_tma<256><<<grid_attn, threads + 64, smem, st>>>(a, ns);
      else k_attn<256><<<grid_attn, threads, 0, st>>>(a);
      k_combine<256><<<grid_combine, 256, 0, st>>>(splits, partials, out, ctrl, sh.H, B, nl);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_combine(const Shape& sh, const Split* splits, float* partials, float* out, int32_t* ctrl,
                           int32_t B, int32_t nl, int32_t grid, cudaStream_t st) {
  switch (sh.D) {
    case 64: k_combine<64><<<grid, 256, 0, st>>>(splits, partials, out, ctrl, sh.H, B, nl); break;
    case 128: k_combine<128><<<grid, 256, 0, st>>>(splits, partials, out, ctrl, sh.H, B, nl); break;
    case 256: k_combine<256><<<grid, 256, 0, st>>>(splits, partials, out, ctrl, sh.H, B, nl); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_keep_scan(const Shape& sh, const DSlot* cur, DSlot* next, int32_t B, int64_t S,
                             void* report, MoveEntry* entries, int32_t* key_chunk0, int32_t* key_src,
                             int64_t* ctrl64, int32_t compact_policy, int32_t pool_nonempty, cudaStream_t st) {
  k_keep_scan<<<1, 1024, 0, st>>>(sh, cur, next, B, S, (uint8_t*)report, entries, key_chunk0, key_src, ctrl64,
                                  compact_policy, pool_nonempty);
  return cudaGetLastError();
}

cudaError_t launch_move(uint8_t* arena, uint8_t* staging, const MoveEntry* entries, const int32_t* key_chunk0,
                        const int32_t* key_src, int32_t n_entries, int64_t n_chunks, int64_t S, int64_t kvpt,
                        int64_t* ctrl64, uint32_t* flags, uint32_t epoch, int32_t staging_enabled, int32_t grid,
                        cudaStream_t st) {
  MoveArgs a;
  a.arena = arena; a.staging = staging; a.entries = entries; a.key_chunk0 = key_chunk0; a.key_src = key_src;
  a.n_entries = n_entries; a.n_chunks = n_chunks; a.S = S; a.kvpt = kvpt; a.ctrl64 = ctrl64; a.flags = flags;
  a.epoch = epoch; a.staging_enabled = staging_enabled;
  const int smem = move_smem_bytes(S, n_entries, &a.keys_in_smem);
  k_move<<<grid, 64 * MV_NP, (size_t)smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fill(const Shape& sh, uint64_t seed, const DSlot* slots, const int32_t* list,
                        int32_t n, int32_t max_prompt, uint16_t* arena, cudaStream_t st) {
  if (n <= 0 || max_prompt <= 0) return cudaSuccess;
  dim3 grid((max_prompt + FILL_ROWS - 1) / FILL_ROWS, n);
  k_fill<<<grid, 256, 0, st>>>(sh, seed, slots, list, arena);
  return cudaGetLastError();
}

cudaError_t launch_synth(const Shape& sh, uint64_t seed, const DSlot* slots, int32_t B, int32_t l0,
                         int32_t nl, const int32_t* out_len_by_req, int64_t n_req, uint16_t* q,
                         uint16_t* k, uint16_t* v, uint8_t* eos, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((int64_t)nl * B, 148 * 16);
  k_synth<<<(int)blocks, 256, 0, st>>>(sh, seed, slots, B, l0, nl, out_len_by_req, n_req, q, k, v, eos);
  return cudaGetLastError();
}

cudaError_t launch_verify(const Shape& sh, uint64_t seed, const DSlot* slots, int32_t B,
                          const uint16_t* arena, unsigned long long* bad, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  dim3 grid(64, B);
  k_verify<<<grid, 256, 0, st>>>(sh, seed, slots, arena, bad);
  return cudaGetLastError();
}

}  // namespace s3
