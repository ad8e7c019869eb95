// HBM ceiling probe: what a pure streaming kernel reaches on this B200, to put
// the attention kernel's achieved GB/s in context (the driver's peak is a
// torch copy, i.e. half reads, half writes).
//   read_ld   : 128-bit ld.global.nc, grid-stride, 148 x 4 CTAs x 512 threads
//   read_bulk : cp.async.bulk 16 KB pieces into a 4-stage shared ring per CTA
//   copy      : 128-bit load + store (the driver's "copy" pattern)
//   mix83     : read 5 parts, write 1 part (the fused attend-and-shift mix)
// Prints one JSON line (best of 10, CUDA events, 4 GiB buffers >> L2).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void read_ld(const uint4* __restrict__ p, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void copy_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = s[i];
}

// read 5/6 of the pieces, write the 6th back shifted (like attention + row shift)
__global__ void mix_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + i));
    if (((i >> 10) % 6) == 5) d[i] = v; else acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one thread per CTA streams 16 KB pieces with cp.async.bulk into NS stages
template <int NS>
__global__ void read_bulk(const uint8_t* __restrict__ p, size_t pieces, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NS];
  const uint32_t PB = 16384;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t acc = 0;
  size_t k = 0;
  auto issue = [&](size_t piece, int st) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(PB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm + st * PB)), "l"(p + piece * PB), "r"(PB), "r"(su32(&full[st]))
                 : "memory");
  };
  size_t first = blockIdx.x;
  int inflight = 0;
  for (size_t piece = first; piece < pieces && inflight < NS; piece += gridDim.x, ++inflight) issue(piece, inflight);
  for (size_t piece = first; piece < pieces; piece += gridDim.x, ++k) {
    const int st = k % NS;
    const uint32_t par = (uint32_t)(k / NS) & 1u;
    asm volatile("{\n .reg .pred q;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}\n" ::"r"(
                     su32(&full[st])), "r"(par) : "memory");
    acc ^= *reinterpret_cast<const uint32_t*>(sm + st * PB);
    const size_t nxt = piece + (size_t)NS * gridDim.x;
    if (nxt < pieces) issue(nxt, st);
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t N = 4ull << 30;
  uint8_t *a, *b;
  unsigned long long* sink;
  cudaMalloc(&a, N);
  cudaMalloc(&b, N);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 1, N);
  cudaMemset(b, 2, N);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(read_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto best = [&](auto fn) {
    float b = 1e9f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < b) b = ms;
    }
    return b;
  };
  const size_t n16 = N / 16;
  float t_ld = best([&] { read_ld<<<sms * 4, 512>>>((const uint4*)a, n16, sink); });
  float t_bulk = best([&] { read_bulk<8><<<sms, 32, 8 * 16384>>>(a, N / 16384, sink); });
  float t_bulk2 = best([&] { read_bulk<8><<<sms, 32, 8 * 16384>>>(a, N / 16384, sink); });
  float t_cp = best([&] { copy_k<<<sms * 4, 512>>>((const uint4*)a, (uint4*)b, n16 / 2); });
  float t_mix = best([&] { mix_k<<<sms * 4, 512>>>((const uint4*)a, (uint4*)b, n16, sink); });
  auto gbs = [&](double bytes, float ms) { return bytes / (ms / 1e3) / 1e9; };
  printf("{\"read_ld_gbs\": %.1f, \"read_bulk_gbs\": %.1f, \"copy_rw_gbs\": %.1f, \"mix_read5_write1_gbs\": %.1f, "
         "\"bytes\": %zu, \"err\": \"%s\"}\n",
         gbs(N, t_ld), gbs(N, t_bulk < t_bulk2 ? t_bulk : t_bulk2), gbs(N, t_cp), gbs(N + N / 6.0, t_mix), N,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
