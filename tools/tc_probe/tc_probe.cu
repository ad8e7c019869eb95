// tc_probe.cu -- standalone validation of the tcgen05 building blocks used by
// the grouped-KV attention kernel (not part of libs3.so).
//
//   test 1:  S^T[128 x 16] = K[128 x 128] . Q[16 x 128]^T
//            A = K tile, K-major, 128B swizzle (TMA tensor loads, 2 boxes)
//            B = Q tile, K-major, 128B swizzle
//   test 2:  O^T[128 x 16] = V^T . P^T,  V tile [128 j x 128 d] (MN-major A),
//            P [16 x 128 j] written by threads with a manual 128B swizzle (K-major B)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <cuda_bf16.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, 128B swizzle (layout type 2), version 1.
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;            // version (Blackwell)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
// instruction descriptor: bf16 x bf16 -> f32, M, N, A/B major
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                    // c_format f32
         | (1u << 7)                  // a_format bf16
         | (1u << 10)                 // b_format bf16
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)smem_u32(bar))
               : "memory");
}

}  // namespace

// one CTA of 128 threads
__global__ void __launch_bounds__(128) probe_kernel(const __grid_constant__ CUtensorMap map_k,
                                                    const __grid_constant__ CUtensorMap map_q,
                                                    const __grid_constant__ CUtensorMap map_v,
                                                    const float* __restrict__ p_in,  // [16][128] probabilities
                                                    float* __restrict__ s_out,       // [128][16]
                                                    float* __restrict__ o_out) {     // [128][16]
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sk = smem;                   // 2 x [128 rows x 128 B] = 32 KB
  uint8_t* sq = smem + 32768;           // 2 x [16 rows x 128 B]  = 4 KB
  uint8_t* sv = smem + 36864;           // 2 x [128 rows x 128 B] = 32 KB (j rows, d cols)
  uint8_t* sp = smem + 69632;           // 2 x [16 rows x 128 B]  = 4 KB (P, K-major over j)
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // P written by threads: row c (query), col j; block kb = j / 64; 128B swizzle
  for (int idx = tid; idx < 16 * 128; idx += 128) {
    const int c = idx / 128, j = idx % 128, kb = j / 64, jj = j % 64;
    const uint32_t byte = (uint32_t)c * 128u + (uint32_t)jj * 2u;
    const uint32_t sw = byte ^ (((byte >> 7) & 7u) << 4);
    __nv_bfloat16 v = __float2bfloat16(p_in[c * 128 + j]);
    *reinterpret_cast<__nv_bfloat16*>(sp + kb * 2048 + sw) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> async proxy (MMA)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_load, 32768 + 4096 + 32768);
    for (int kb = 0; kb < 2; ++kb) {
      tma_load_2d(sk + kb * 16384, &map_k, kb * 64, 0, &bar_load);   // K rows 0..127, cols kb*64..
      tma_load_2d(sq + kb * 2048, &map_q, kb * 64, 0, &bar_load);
      tma_load_2d(sv + kb * 16384, &map_v, kb * 64, 0, &bar_load);   // V rows j 0..127, d kb*64..
    }
    mbar_wait(&bar_load, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // test 1: S^T (TMEM cols 0..15) = K . Q^T, K-dim = d (128) in 8 steps of 16
    const uint32_t id1 = idesc_bf16(128, 16, 0, 0);
    for (int k = 0; k < 8; ++k) {
      const int kb = k / 4, ko = (k % 4) * 32;   // 16 bf16 = 32 B inside the 128-B swizzle row
      const uint64_t a = umma_desc(sk + kb * 16384 + ko, 16, 1024);
      const uint64_t b = umma_desc(sq + kb * 2048 + ko, 16, 1024);
      mma_bf16(tmem + 0, a, b, id1, k > 0);
    }
    // test 2: O^T (TMEM cols 32..47) = V^T . P^T; A = V^T MN-major (M = d, K = j),
    // B = P K-major (N = query, K = j); K-dim = j (128) in 8 steps of 16 rows
    const uint32_t id2 = idesc_bf16(128, 16, 1, 0);
    for (int k = 0; k < 8; ++k) {
      // A: MN-major; 16 j-rows = two 8-row atoms = 2048 B; the two 64-d blocks are 16 KB apart (LBO)
      const uint64_t a = umma_desc(sv + k * 2048, 16384, 1024);
      const int kb = k / 4, ko = (k % 4) * 32;
      const uint64_t b = umma_desc(sp + kb * 2048 + ko, 16, 1024);
      mma_bf16(tmem + 32, a, b, id2, k > 0);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // each warp reads its 32 TMEM lanes: lane = row
  uint32_t r[16], o[16];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7]),
        "=r"(o[8]), "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]), "=r"(o[13]), "=r"(o[14]), "=r"(o[15])
      : "r"(taddr + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 16; ++c) {
    s_out[tid * 16 + c] = __uint_as_float(r[c]);
    o_out[tid * 16 + c] = __uint_as_float(o[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (EncodeTiled)fn;
}

// 2-D map over a row-major [rows][cols] bf16 matrix with row pitch `pitch` bytes; box 64 x box_rows
static int make_map(CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint64_t pitch, uint32_t box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return (int)r;
}

extern "C" int tc_probe_run(void* k, void* q, void* v, const float* p, float* s_out, float* o_out, int pitch_k) {
  CUtensorMap mk, mq, mv;
  if (make_map(&mk, k, 128, 128, (uint64_t)pitch_k, 128)) return -1;
  if (make_map(&mq, q, 128, 16, 256, 16)) return -2;
  if (make_map(&mv, v, 128, 128, 256, 128)) return -3;
  const int smem = 73728 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(mk, mq, mv, p, s_out, o_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("cuda error %s\n", cudaGetErrorString(e));
    return -10;
  }
  return 0;
}
