// Microbenchmark: latency of tcgen05.commit -> mbarrier completion (no MMA
// outstanding / after one MMA), and of mbarrier arrive -> wait hand-offs between warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/sync_bench.cu -o /tmp/sync_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

__global__ void bench(long long* out, int mode) {
  __shared__ __align__(8) uint64_t b1, b2;
  __shared__ uint32_t slot;
  __shared__ __align__(1024) uint8_t sm[32768];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&b1)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&b2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const int N = 64;
  if (mode == 0 && threadIdx.x == 0) {  // commit (nothing outstanding) -> wait, same thread
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) { commit(&b1); wait(&b1, i & 1); }
    out[0] = (clock64() - t0) / N;
  }
  if (mode == 1 && threadIdx.x == 0) {  // one N=64 SS MMA then commit -> wait
    const uint64_t d = ((uint64_t)((smem_u32(sm) >> 4) & 0x3FFF)) | (1ull << 16) | ((uint64_t)64 << 32) | (1ull << 46) | (2ull << 61);
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
      asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(d), "l"(d), "r"(id));
      commit(&b1);
      wait(&b1, i & 1);
    }
    out[0] = (clock64() - t0) / N;
  }
  if (mode == 2) {  // ping-pong arrive/wait between warp 0 and warp 4 (lane 0 each)
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int i = 0; i < N; ++i) { arrive(&b1); wait(&b2, i & 1); }
      out[0] = (clock64() - t0) / N;
    } else if (threadIdx.x == 128) {
      for (int i = 0; i < N; ++i) { wait(&b1, i & 1); arrive(&b2); }
    }
  }
  if (mode == 3) {  // commit by warp 0 -> wait in warp 4 -> arrive back
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int i = 0; i < N; ++i) { commit(&b1); wait(&b2, i & 1); }
      out[0] = (clock64() - t0) / N;
    } else if (threadIdx.x == 128) {
      for (int i = 0; i < N; ++i) { wait(&b1, i & 1); arrive(&b2); }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  const char* names[] = {"commit->wait (same thread, idle pipe)", "mma N=64 + commit->wait", "arrive/wait ping-pong (2 warps)",
                         "commit -> other warp -> arrive back"};
  for (int m = 0; m < 4; ++m) {
    long long h = 0;
    for (int r = 0; r < 3; ++r) { bench<<<1, 256>>>(d, m); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-45s %lld cycles per round trip  %s\n", names[m], h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
