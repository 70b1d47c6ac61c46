// dev probe: the e2e trace-streaming pattern — 4096 simulations, each
// appending 88 B rows into its own capacity-strided slice of mapped pinned
// host memory in 128-row flushes (16 B stores by one warp) — vs the same
// bytes written contiguously.
#include <cstdio>
#include <cstdlib>
#include <sys/mman.h>
#include <cuda_runtime.h>
__global__ void rows(char* dst, size_t slice, int rows_per_sim, int flush) {
  char* base = dst + blockIdx.x * slice;
  const int lane = threadIdx.x;
  for (int r0 = 0; r0 < rows_per_sim; r0 += flush) {
    const int r1 = r0 + flush < rows_per_sim ? r0 + flush : rows_per_sim;
    size_t b0 = (size_t)r0 * 88, b1 = (size_t)r1 * 88;
    b0 = (b0 + 15) & ~15ull;
    for (size_t b = b0 + lane * 16; b + 16 <= b1; b += 32 * 16)
      *reinterpret_cast<ulonglong2*>(base + b) = make_ulonglong2(b, r0);
    __syncwarp();
  }
}
static void run(const char* tag, char* dptr, size_t slice, int sims, int rows_per_sim) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  rows<<<sims, 32>>>(dptr, slice, rows_per_sim, 128);
  cudaEventRecord(a);
  rows<<<sims, 32>>>(dptr, slice, rows_per_sim, 128);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)sims * rows_per_sim * 88;
  printf("%-40s %.1f MB in %.2f ms: %.1f GB/s\n", tag, bytes / 1e6, ms, bytes / ms / 1e6);
}
int main() {
  const int sims = 4096, rps = 1600;
  for (size_t slice : {(size_t)4096 * 88, (size_t)1664 * 88}) {
    const size_t bytes = slice * sims;
    char* h = nullptr;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    char* d = nullptr;
    cudaHostGetDevicePointer(&d, h, 0);
    char tag[64];
    snprintf(tag, sizeof tag, "cudaHostAlloc, slice %zu KB", slice / 1024);
    run(tag, d, slice, sims, rps);
    cudaFreeHost(h);
    // huge-page backed, registered
    void* p = nullptr;
    const size_t hb = (bytes + (2u << 20) - 1) & ~((size_t)(2u << 20) - 1);
    if (posix_memalign(&p, 2u << 20, hb) == 0) {
      madvise(p, hb, MADV_HUGEPAGE);
      for (size_t i = 0; i < hb; i += 4096) static_cast<char*>(p)[i] = 0;
      if (cudaHostRegister(p, hb, cudaHostRegisterMapped) == cudaSuccess) {
        char* d2 = nullptr;
        cudaHostGetDevicePointer(&d2, p, 0);
        snprintf(tag, sizeof tag, "THP + cudaHostRegister, slice %zu KB", slice / 1024);
        run(tag, d2, slice, sims, rps);
        cudaHostUnregister(p);
      } else {
        printf("cudaHostRegister failed\n");
        cudaGetLastError();
      }
      free(p);
    }
  }
  return 0;
}
