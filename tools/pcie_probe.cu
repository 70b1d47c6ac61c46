// dev probe: SM-issued stores to mapped pinned host memory vs copy-engine D2H
#include <cstdio>
#include <cuda_runtime.h>
__global__ void wr(unsigned long long* dst, size_t n_u2, int stride_rows) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  ulonglong2* d = reinterpret_cast<ulonglong2*>(dst);
  for (; i < n_u2; i += (size_t)gridDim.x * blockDim.x) d[i] = make_ulonglong2(i, i + 1);
}
int main() {
  const size_t bytes = 512ull << 20;
  unsigned long long* h = nullptr;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  unsigned long long* dh = nullptr;
  cudaHostGetDevicePointer(&dh, h, 0);
  void* d = nullptr;
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks : {148, 296, 592, 1184, 4096}) {
    wr<<<blocks, 256>>>(dh, bytes / 16, 0);
    cudaEventRecord(a);
    wr<<<blocks, 256>>>(dh, bytes / 16, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("SM stores to host, %d CTAs: %.1f GB/s\n", blocks, bytes / ms / 1e6);
  }
  cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
  cudaEventRecord(a);
  cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("cudaMemcpy D2H pinned: %.1f GB/s\n", bytes / ms / 1e6);
  return 0;
}
