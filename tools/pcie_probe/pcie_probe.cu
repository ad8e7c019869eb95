// PCIe duplex probe for s3_decode_step_host's design: copy-engine H2D / D2H
// alone and concurrently, SM stores into mapped pinned memory alone and
// concurrently with a copy-engine H2D.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void sm_store(float4* __restrict__ dst, const float4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t N = 1ull << 30;
  void *hs, *hd, *da, *db;
  cudaHostAlloc(&hs, N, cudaHostAllocDefault);
  cudaHostAlloc(&hd, N, cudaHostAllocDefault);
  cudaMalloc(&da, N);
  cudaMalloc(&db, N);
  cudaMemset(db, 1, N);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, j1, j2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&j1); cudaEventCreate(&j2);
  void* hd_dev;
  cudaHostGetDevicePointer(&hd_dev, hd, 0);
  auto run = [&](int mode) {
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      if (mode == 0 || mode == 2 || mode == 4) cudaMemcpyAsync(da, hs, N, cudaMemcpyHostToDevice, s1);
      if (mode == 1 || mode == 2) cudaMemcpyAsync(hd, db, N, cudaMemcpyDeviceToHost, s2);
      if (mode == 3 || mode == 4) sm_store<<<148 * 4, 512, 0, s2>>>((float4*)hd_dev, (const float4*)db, N / 16);
      cudaEventRecord(j2, s2);
      cudaStreamWaitEvent(s1, j2, 0);
      cudaEventRecord(e1, s1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  const char* names[] = {"ce_h2d", "ce_d2h", "ce_both", "sm_store_d2h", "sm_store_plus_ce_h2d"};
  printf("{");
  for (int m = 0; m < 5; ++m) {
    float ms = run(m);
    double gb = (m == 2 || m == 4 ? 2.0 : 1.0) * N / 1e9;
    printf("%s\"%s\": {\"ms\": %.3f, \"total_gbs\": %.2f}", m ? ", " : "", names[m], ms, gb / (ms / 1e3));
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
