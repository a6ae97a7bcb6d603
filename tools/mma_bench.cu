// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) on one SM,
// A from shared memory (SS) or TMEM (TS), N in {32, 64, 128, 256},
// 1 or 4 independent accumulators. Build & run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (ignored for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// MODE 0: MMA thread alone; 1: + 8 warps spinning on an mbarrier; 2: + 8 warps streaming tcgen05.ld
template <bool TS, int N, int ACC, int NMMA, int MODE, bool RANDOM, int MMA_WARP>
__global__ void bench(long long* out, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2c;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    x ^= x >> 13;
    // random bf16 pairs in [-2, 2): sign/exponent near 1.0
    ((uint32_t*)sm)[i] = (RANDOM ? ((x & 0x807F807Fu) | 0x3F803F80u) : 0u);
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2c)));
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (RANDOM && threadIdx.x < 128 && MODE != 4) {  // random A operand in TMEM cols 384..447
    uint32_t r[4];
    for (int c = 0; c < 64; c += 4) {
      for (int e = 0; e < 4; ++e) r[e] = ((uint32_t*)sm)[(threadIdx.x * 64 + c + e) & 16383];
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + 384 + c),
                   "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp >= 4 && MODE == 1) {
    __shared__ __align__(8) uint64_t bar2;
    if (threadIdx.x == 128) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    while (!stop) {
      uint32_t d;
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(d) : "r"(smem_u32(&bar2)));
    }
  }
  if (warp >= 4 && MODE == 2) {
    uint32_t acc = 0;
    while (!stop) {
      uint32_t r0, r1, r2, r3;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 448));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += r0 + r3;
    }
    if (acc == 12345) out[3] = acc;
  }
  if (warp == 4 && MODE == 4 && (threadIdx.x & 31) == 0) {  // concurrent bulk copies global -> smem
    __shared__ __align__(8) uint64_t tbar;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    uint32_t phase = 0;
    int it = 0;
    while (!stop) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tbar)), "r"(16384));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(sm + 16384 * (it & 1))), "l"(gsrc + (size_t)(it % 512) * 16384),
                   "r"(16384), "r"(smem_u32(&tbar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(smem_u32(&tbar)), "r"(phase));
      phase ^= 1;
      ++it;
    }
  }
  if (warp >= 4 && MODE == 3) {  // dense ALU + MUFU like the softmax warps
    float x = threadIdx.x * 0.001f, y = 1.f;
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
        y = fmaf(y, 0.999f, e);
        x = fmaf(x, 1.0001f, -0.5f * e);
      }
    }
    if (y == 12345.f) out[3] = 1;
  }
  const int mma_warp = MMA_WARP;
  if (threadIdx.x == mma_warp * 32) {
    const uint32_t a_s = smem_u32(sm), b_s = smem_u32(sm + 32768);
    const uint32_t id = idesc(N);
    long long t0 = clock64();
    if (MODE == 7 || MODE == 8) {
      const uint32_t idqk = idesc(32);
      for (int u = 0; u < NMMA / 16; ++u) {
        const int b = u & 1, h = u & 1;
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t half = ks >> 2, in = (ks & 3) * 32;
          for (int mt = 0; mt < 2; ++mt) {
            const uint64_t bd = desc(b_s + half * 8192 + in + h * 4096);
            if (MODE == 7)
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                           ::"r"(tmem + 384 + 64 * mt + 32 * b), "r"(tmem + 256 + 64 * mt + 8 * ks), "l"(bd), "r"(idqk), "r"((uint32_t)(ks > 0)));
            else
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                           ::"r"(tmem + 384 + 64 * mt + 32 * b), "r"(tmem + 256 + 64 * mt + 8 * ks), "l"(desc(b_s + 32 * (ks & 3))), "r"(idqk), "r"((uint32_t)(ks > 0)));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2c)) : "memory");
      }
    } else
    for (int i = 0; i < NMMA; ++i) {
      if (MODE == 6 && (i & 7) == 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE == 5 && (i & 7) == 0 && i)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2c)) : "memory");
      const uint32_t d = tmem + (uint32_t)((i % ACC) * (N <= 64 ? 64 : 128)) % 384;
      const uint32_t acc = i >= ACC;
      if (TS) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                     ::"r"(d), "r"(tmem + 384 + 8 * (i & 7)), "l"(desc(b_s + 32 * (i & 3))), "r"(id), "r"(acc));
      } else {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                     ::"r"(d), "l"(desc(a_s + 32 * (i & 3))), "l"(desc(b_s + 32 * (i & 3))), "r"(id), "r"(acc));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static uint8_t* g_src = nullptr;
template <bool TS, int N, int ACC, int MODE = 0, bool RANDOM = false, int MW = 0>
void run(long long* d, int ctas = 1) {
  constexpr int NM = 256;
  auto k = bench<TS, N, ACC, NM, MODE, RANDOM, MW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  long long h[2];
  for (int rep = 0; rep < 3; ++rep) {
    k<<<ctas, MODE ? 384 : 128, 65536 + 1024>>>(d, g_src);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double floor = 128.0 * N / 256.0;
  printf("mma_warp %d %s mode %d ctas %3d %s N=%3d acc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %.0f)  %s\n", MW, RANDOM ? "rand" : "zero", MODE, ctas, TS ? "TS" : "SS", N, ACC,
         (double)h[0] / NM, (double)h[1] / NM, floor, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaMalloc(&g_src, 512 * 16384 + 16384);
  // dependent chains (acc=1) vs independent accumulators
  run<false, 64, 1, 0, true, 1>(d, 148);
  run<false, 64, 2, 0, true, 1>(d, 148);
  run<false, 64, 4, 0, true, 1>(d, 148);
  run<false, 128, 1, 0, true, 1>(d, 148);
  run<false, 128, 2, 0, true, 1>(d, 148);
  run<true, 128, 1, 0, true, 1>(d, 148);
  return 0;
}
