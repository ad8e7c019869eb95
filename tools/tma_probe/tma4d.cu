// tma4d.cu -- does a 4-D TMA box with overlapping row strides load a tile's
// 8-row groups as [group][64-column block][8 rows][128 B] (both column blocks
// of a group adjacent) from an arbitrary starting row?  That layout would let
// one instruction load all groups of a K (or V) tile.  Prints PASS/FAIL.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void load4d(const __grid_constant__ CUtensorMap map, int row0, int ngroups, uint8_t* out, int bytes) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(su32(sm)), "l"(&map), "r"(0), "r"(row0), "r"(0), "r"(0), "r"(su32(&bar))
        : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(
                   su32(&bar))
               : "memory");
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 1000, kvpt = 4096;           // row pitch 4 KB; each row: 2048 bf16 elements
  std::vector<uint16_t> h((size_t)R * kvpt / 2);
  for (int r = 0; r < R; ++r)
    for (int e = 0; e < kvpt / 2; ++e) h[(size_t)r * (kvpt / 2) + e] = (uint16_t)((r * 131 + e * 7) & 0xFFFF);
  uint16_t* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)p;
  int fails = 0;
  const int col_base = 256;                  // start column (elements) of the head inside the row
  for (int ngroups : {1, 3, 6, 16}) {
    CUtensorMap m;
    // dims: 64 columns | rows (pitch kvpt) | column block (128 B) | row groups (8 * kvpt)
    cuuint64_t dims[4] = {64, (cuuint64_t)R, 2, (cuuint64_t)(R / 8)};
    cuuint64_t strides[3] = {(cuuint64_t)kvpt, 128, (cuuint64_t)8 * kvpt};
    cuuint32_t box[4] = {64, 8, 2, (cuuint32_t)ngroups};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)(d + col_base), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) { printf("ngroups %d: encode failed rc=%d\n", ngroups, (int)rc); ++fails; continue; }
    const int bytes = ngroups * 2 * 8 * 128;
    uint8_t* dout;
    cudaMalloc(&dout, bytes);
    cudaFuncSetAttribute(load4d, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    const int row0 = 37;
    load4d<<<1, 128, 40000>>>(m, row0, ngroups, dout, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("ngroups %d: kernel error %s\n", ngroups, cudaGetErrorString(e)); return 1; }
    std::vector<uint8_t> o(bytes);
    cudaMemcpy(o.data(), dout, bytes, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < ngroups; ++j)
      for (int kb = 0; kb < 2; ++kb)
        for (int i = 0; i < 8; ++i)
          for (int c = 0; c < 64; ++c) {
            const int r = row0 + 8 * j + i;
            const uint16_t want = h[(size_t)r * (kvpt / 2) + col_base + kb * 64 + c];
            const int chunk = c / 8, within = c % 8;
            const size_t off = (size_t)((j * 2 + kb) * 8 + i) * 128 + (size_t)(((chunk ^ (i & 7)) * 16) + within * 2);
            const uint16_t got = (uint16_t)(o[off] | (o[off + 1] << 8));
            if (got != want) ++bad;
          }
    printf("ngroups %d: %s (%d mismatches)\n", ngroups, bad ? "FAIL" : "PASS", bad);
    fails += bad != 0;
    cudaFree(dout);
  }
  printf(fails ? "RESULT FAIL\n" : "RESULT PASS\n");
  return 0;
}
