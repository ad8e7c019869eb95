// Test-only stand-in for the multi-GPU counter all-reduce kernel: one CTA that
// needs a large dynamic shared-memory allocation (so it cannot share an SM
// with the persistent attention kernel) and spins for spin_ns nanoseconds.
#include <cuda_runtime.h>

__global__ void probe_kernel(unsigned long long* ts, long long spin_ns) {
  extern __shared__ unsigned char sm[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  sm[threadIdx.x] = (unsigned char)threadIdx.x;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while ((long long)(t - t0) < spin_ns);
  __syncthreads();
  if (threadIdx.x == 0) { ts[0] = t0; ts[1] = t + sm[5]; }
}

extern "C" int probe_launch(void* stream, int smem_bytes, long long spin_ns, unsigned long long* ts_dev) {
  cudaError_t e = cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return (int)e;
  probe_kernel<<<1, 128, smem_bytes, (cudaStream_t)stream>>>(ts_dev, spin_ns);
  return (int)cudaGetLastError();
}
