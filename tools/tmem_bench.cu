// Microbenchmark: tcgen05.ld throughput (32x32b.x32, 128 B per lane per load)
// with 1..8 warps of one CTA; bytes per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tmem_bench.cu -o /tmp/tmem_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
#define LD32(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" \
  : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(taddr))

__global__ void bench(long long* out, int nwarps) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
    for (int i = 0; i < 256; ++i) {
      uint32_t r[64];
      LD32(base + (i & 1) * 64, r);
      LD32(base + (i & 1) * 64 + 32, (r + 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 64; ++c) acc += r[c];
    }
  }
  long long t1 = clock64();
  if (acc == 12345) out[2] = acc;
  if ((threadIdx.x & 31) == 0 && warp == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int nw : {1, 2, 4, 6, 8}) {
    long long h = 0;
    for (int r = 0; r < 3; ++r) { bench<<<148, 256>>>(d, nw); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = 256.0 * nw * 32 * 64 * 4;
    printf("%d warps: %lld cycles for 256 x 8 KB/warp -> %.1f B/cycle/SM, %.0f cycles per 8 KB warp-load  %s\n", nw, h,
           bytes / h, (double)h / 256, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
