// Single-row weight streaming for the draft forward (reference: the projections
// of TinyTransformer.forward for the one pending row, model.py:283-285, 306-309,
// and the chained draft heads, model.py:104-120):  y[N] = x[K] . W[K][N], W bf16
// row-major [in, out] exactly as the reference stores it, x bf16, fp32 accumulate.
//
// With one row there is nothing for a tensor core to do; the layer is a pure
// HBM stream of its weights. Each CTA owns 256 columns (a lane holds 8 columns =
// one 16-byte load per weight row) and a slice of K; its 8 warps take
// interleaved rows, each warp keeping 8 rows of loads in flight, so an SM holds
// ~128 KB of weight loads in flight. The K slices of a column block are reduced
// by the last CTA to finish (arrival counter, reset after use), in slice order —
// deterministic — and the epilogue (fp32 store, or SiLU -> bf16 for the MLP
// up-projection) is applied after the full sum.
//
// Launched as a programmatic dependent (PDL): the weights do not depend on the
// previous kernel, so each CTA issues its first rows of weight loads before
// griddepcontrol.wait and only then reads x — the DRAM ramp of every layer's
// stream overlaps the tail of the kernel before it.
#include "common.cuh"

namespace sd {
namespace gv {

constexpr int COLS = 256;    // columns per CTA (32 lanes x 8)
constexpr int WARPS = 8;
#ifndef SD_GEMV_UNROLL
#define SD_GEMV_UNROLL 8
#endif
#ifndef SD_GEMV_CTAS_PER_SM
#define SD_GEMV_CTAS_PER_SM 4
#endif
constexpr int UNROLL = SD_GEMV_UNROLL;  // weight rows in flight per warp

__device__ __forceinline__ void fma8(float* acc, float xv, const uint4& w) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    acc[2 * e] = fmaf(xv, f.x, acc[2 * e]);
    acc[2 * e + 1] = fmaf(xv, f.y, acc[2 * e + 1]);
  }
}

__global__ void __launch_bounds__(WARPS * 32) gemv_kernel(const __nv_bfloat16* __restrict__ x,
                                                           const __nv_bfloat16* __restrict__ W, int K, int N,
                                                           int splits, int epi, void* __restrict__ y,
                                                           float* __restrict__ part, int* __restrict__ counters) {
  extern __shared__ float xs[];  // this CTA's K slice of x (fp32)
  __shared__ float red[WARPS][COLS];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cb = blockIdx.x, split = blockIdx.y;
  const int k0 = (int)((int64_t)split * K / splits), k1 = (int)((int64_t)(split + 1) * K / splits);
  const int col = cb * COLS + lane * 8;
  const bool live = col < N;  // N % 8 == 0: a lane's 8 columns are all in or all out
  const __nv_bfloat16* wp = W + col;
  // first batch of weight rows: independent of the previous kernel, issued before the wait
  uint4 w0[UNROLL];
  int k = k0 + warp;
  const bool first = live && k + (UNROLL - 1) * WARPS < k1;
  if (first) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) w0[u] = __ldcs(reinterpret_cast<const uint4*>(wp + (int64_t)(k + u * WARPS) * N));
  }
  pdl_trigger();
  pdl_wait();  // x is the previous kernel's output
  for (int kk = k0 + tid; kk < k1; kk += WARPS * 32) xs[kk - k0] = __bfloat162float(x[kk]);
  __syncthreads();
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (first) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) fma8(acc, xs[k + u * WARPS - k0], w0[u]);
    k += UNROLL * WARPS;
  }
  if (live) {
    for (; k + (UNROLL - 1) * WARPS < k1; k += UNROLL * WARPS) {
      uint4 w[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)  // streamed once: bypass L1
        w[u] = __ldcs(reinterpret_cast<const uint4*>(wp + (int64_t)(k + u * WARPS) * N));
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) fma8(acc, xs[k + u * WARPS - k0], w[u]);
    }
    for (; k < k1; k += WARPS) fma8(acc, xs[k - k0], __ldcs(reinterpret_cast<const uint4*>(wp + (int64_t)k * N)));
  }
  // warps -> CTA sum in warp order
#pragma unroll
  for (int e = 0; e < 8; ++e) red[warp][lane * 8 + e] = acc[e];
  __syncthreads();
  const int c = tid;  // one column per thread (256 threads == COLS)
  float v = 0.f;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) v += red[w][c];
  const int gcol = cb * COLS + c;
  auto store = [&](float s) {
    if (gcol >= N) return;
    if (epi == SD_GEMM_EPI_F32)
      ((float*)y)[gcol] = s;
    else
      ((__nv_bfloat16*)y)[gcol] = __float2bfloat16_rn(s / (1.f + __expf(-s)));
  };
  if (splits == 1) {
    store(v);
    return;
  }
  // K slices: partials, then the last CTA of the column block sums them in order
  if (gcol < N) part[(int64_t)split * N + gcol] = v;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&counters[cb], 1) == splits - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (gcol < N) {
    float s = 0.f;
#pragma unroll 8
    for (int sp = 0; sp < splits; ++sp) s += __ldcg(part + (int64_t)sp * N + gcol);
    store(s);
  }
  if (tid == 0) counters[cb] = 0;  // ready for the next launch / graph replay
}

// The workspace starts with a fixed 4 KB counter head (one int per column block)
// so that calls of different shapes sharing one workspace never see each other's
// partials in their counters.
constexpr size_t WS_HEAD = 4096;

static int splits_for(int K, int N) {
  const int blocks = (N + COLS - 1) / COLS;
  // ~4 CTAs per SM in flight, each with >= 256 weight rows; wide outputs (many
  // column blocks) keep longer K slices
  int s = (148 * (blocks >= 64 ? SD_GEMV_CTAS_PER_SM / 2 : SD_GEMV_CTAS_PER_SM) + blocks - 1) / blocks;
  const int max_s = K / 256 > 0 ? K / 256 : 1;
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

}  // namespace gv
}  // namespace sd

using namespace sd;

extern "C" {

size_t sd_gemv_workspace_bytes(int K, int N) {
  if (K <= 0 || N <= 0) return 0;
  const int s = gv::splits_for(K, N);
  return gv::WS_HEAD + (s > 1 ? (size_t)s * N * sizeof(float) : 0);
}

int sd_gemv(const void* x, int K, const void* w, int N, int epi, void* y, void* workspace, size_t workspace_bytes,
            sd_stream_t stream) {
  SD_REQUIRE(x && w && y && K > 0 && N > 0 && N % 8 == 0, "sd_gemv: K=%d N=%d (N %% 8 == 0)", K, N);
  SD_REQUIRE(((uintptr_t)w % 16) == 0, "sd_gemv: W must be 16-byte aligned");
  SD_REQUIRE(epi == SD_GEMM_EPI_F32 || epi == SD_GEMM_EPI_SILU_BF16, "sd_gemv: epilogue");
  const int s = gv::splits_for(K, N);
  SD_REQUIRE(s == 1 || (workspace && workspace_bytes >= sd_gemv_workspace_bytes(K, N)), "sd_gemv: workspace");
  const int blocks = (N + gv::COLS - 1) / gv::COLS;
  SD_REQUIRE((size_t)blocks * sizeof(int) <= gv::WS_HEAD, "sd_gemv: N=%d too wide for the counter head", N);
  const size_t head = gv::WS_HEAD;
  const int kslice = (K + s - 1) / s + 1;
  const size_t smem = (size_t)kslice * sizeof(float);
  SD_REQUIRE(smem <= 200 * 1024, "sd_gemv: K slice too long");
  if (smem > 48 * 1024) cudaFuncSetAttribute(gv::gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(gv::gemv_kernel, dim3(blocks, s), dim3(gv::WARPS * 32), smem, as_stream(stream),
             (const __nv_bfloat16*)x, (const __nv_bfloat16*)w, K, N, s, epi, y,
             s > 1 ? (float*)((char*)workspace + head) : nullptr, (int*)workspace);
  return check_launch("sd_gemv");
}

}  // extern "C"
