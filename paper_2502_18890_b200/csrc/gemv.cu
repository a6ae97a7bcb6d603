// Single-row weight streaming for the draft forward (reference: the projections
// of TinyTransformer.forward for the one pending row, model.py:283-285, 306-309,
// and the chained draft heads, model.py:104-120):  y[N] = x[K] . W[K][N], W bf16
// row-major [in, out] exactly as the reference stores it, x bf16, fp32 accumulate.
//
// With one row there is nothing for a tensor core to do; the layer is a pure
// HBM stream of its weights. Each CTA owns 256 columns and a slice of K. The K
// slices of a column block are reduced by the last CTA to finish (arrival
// counter, reset after use), in slice order — deterministic — and the epilogue
// (fp32 store, or SiLU -> bf16 for the MLP up-projection) is applied after the
// full sum.
//
// Two implementations of the stream (SD_GEMV_IMPL=tma|ld picks at run time):
//  * gemv_tma_kernel (default): one producer thread keeps a ring of 8 TMA boxes
//    (32 rows x 256 columns, 16 KB each) in flight per SM; 8 consumer warps read
//    them from shared memory. One CTA per SM, one wave. Measured on the cfg3
//    draft chain (tools/gemv_bench.py): 5.2 TB/s vs 4.7 for the register kernel.
//  * gemv_kernel: lanes hold 8 columns (one 16-byte load per weight row), 8 warps
//    take interleaved rows with 8 rows of loads in flight each, 4 CTAs per SM.
//
// Both are launched as programmatic dependents (PDL): the weights do not depend
// on the previous kernel, so the weight stream starts before griddepcontrol.wait
// and only x waits for the predecessor.
#include <unordered_map>

#include "tc_common.cuh"

namespace sd {
namespace gv {

constexpr int COLS = 256;    // columns per CTA (32 lanes x 8)
constexpr int WS_HEAD_INTS = 1024;
constexpr int ADDNORM_PER = 24, ADDNORM_MAX_N = ADDNORM_PER * 256;  // fused add+norm row length limit  // counter head: per column block, the last int is the row counter
constexpr int WARPS = 8;
#ifndef SD_GEMV_UNROLL
#define SD_GEMV_UNROLL 8
#endif
#ifndef SD_GEMV_CTAS_PER_SM
#define SD_GEMV_CTAS_PER_SM 4
#endif
#ifndef SD_GEMV_MINB
#define SD_GEMV_MINB 4
#endif
#ifndef SD_GEMV_TMA_DEFAULT
#define SD_GEMV_TMA_DEFAULT 1
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

__global__ void __launch_bounds__(WARPS * 32, SD_GEMV_MINB) gemv_kernel(const __nv_bfloat16* __restrict__ x,
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

// ---- TMA-streamed variant --------------------------------------------------
// The same column-block x K-slice decomposition, but the weight rows arrive by
// cp.async.bulk.tensor into a ring of TR-row x 256-column stages (16 KB at TR=32)
// issued by one producer thread, so an SM keeps NS stages (~96 KB per CTA) in
// flight without holding them in registers. The producer never reads x, so it
// does not wait on the previous kernel at all: under PDL a layer's whole first
// ring is in flight before its input exists. Consumer warp w takes rows
// 4w..4w+3 of each stage (a 512-byte row = one 16-byte lane load, conflict free).
#ifndef SD_GEMV_TR
#define SD_GEMV_TR 32
#endif
#ifndef SD_GEMV_NS
#define SD_GEMV_NS 8
#endif
#ifndef SD_GEMV_TMA_CPS
#define SD_GEMV_TMA_CPS 1
#endif
constexpr int TR = SD_GEMV_TR, NS = SD_GEMV_NS;
constexpr int STAGE_BYTES = TR * COLS * 2;
constexpr int RPW = TR / WARPS;  // stage rows per consumer warp

// Residual add + RMSNorm of the whole output row (model.py:278, 306-311), run by
// the last column block to finish: h += y; x = h * gain / rms(h). Replaces the
// separate sd_add_rmsnorm launch after a single-row projection.
struct AddNorm {
  float* h;           // [N] residual stream, updated in place
  const float* gain;  // [N]
  float eps;
  void* x;            // [N] normalised output
  int x_bf16;         // 1: bf16 x, 0: fp32 x
};

// The input row computed in the kernel from the residual stream instead of
// read as x (model.py:306-311 for one row: h <- h + delta; x = rmsnorm(h) *
// gain, rounded to bf16): every CTA sums the squares of the whole row in one
// fixed order (identical on all CTAs), then scales its K slice; the CTAs of
// column block 0 write the updated stream to h_out (not h_in: other CTAs are
// still reading it).
// RoPE + staging of the single draft row as the QKV projection's epilogue
// (model.py:216-232 for one row; the sd_rope_stage it replaces): pairs of
// adjacent columns (held by adjacent lanes) are rotated at the device position
// *pos; Q is scaled and written as bf16 [H][dh], K rotated into k [Hk][dh], V
// copied into v [Hk][dh].
struct RopeOut {
  const int32_t* pos;  // NULL: plain epilogue
  const float* cosT;   // [positions][dh / 2]
  const float* sinT;
  float q_scale;
  int H, Hk, dh;
  __nv_bfloat16* q;
  __nv_bfloat16* k;
  __nv_bfloat16* v;
};

struct XNorm {
  const float* h_in;   // [K] (NULL: plain bf16 x)
  const float* delta;  // [K]
  const float* gain;   // [K]
  float eps;
  float* h_out;        // [K]
};

template <bool ADDNORM>
__global__ void __launch_bounds__((WARPS + 1) * 32, 1)
    gemv_tma_kernel(const __grid_constant__ CUtensorMap wmap, const __nv_bfloat16* __restrict__ x, int K, int N,
                    int splits, int epi, void* __restrict__ y, float* __restrict__ part, int* __restrict__ counters,
                    AddNorm an, XNorm xn, RopeOut ro) {
  extern __shared__ __align__(1024) uint8_t gsm[];
  uint8_t* ring = gsm;                                    // NS stages
  float* xs = reinterpret_cast<float*>(gsm + NS * STAGE_BYTES);  // K slice of x
  __shared__ float red[WARPS][COLS];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cb = blockIdx.x, split = blockIdx.y;
  const int k0 = (int)((int64_t)split * K / splits), k1 = (int)((int64_t)(split + 1) * K / splits);
  const int nst = (k1 - k0 + TR - 1) / TR;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], WARPS);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  if (warp == WARPS) {  // producer: weights only, independent of the previous kernel
    if (lane == 0) {
      for (int i = 0; i < nst; ++i) {
        const int s = i % NS;
        if (i >= NS) tc::mbar_wait(&empty[s], ((i / NS) - 1) & 1);
        tc::mbar_expect_tx(&full[s], STAGE_BYTES);
        tc::tma_load_2d(ring + s * STAGE_BYTES, &wmap, &full[s], cb * COLS, k0 + i * TR);
      }
    }
    return;
  }
  pdl_wait();  // x (or h, delta) is the previous kernels' output
  if (xn.h_in) {
    // 16-byte loads, XN_U of each operand in flight per thread per round (K % 4 == 0)
    constexpr int XN_U = 4;
    float ss = 0.f;
    for (int k4 = tid; k4 < K / 4; k4 += WARPS * 32 * XN_U) {
      float4 hv[XN_U], dv[XN_U];
#pragma unroll
      for (int u = 0; u < XN_U; ++u) {
        const int i = k4 + u * WARPS * 32;
        hv[u] = i < K / 4 ? __ldcg(reinterpret_cast<const float4*>(xn.h_in) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        dv[u] = i < K / 4 ? __ldcg(reinterpret_cast<const float4*>(xn.delta) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < XN_U; ++u) {
        const float a = hv[u].x + dv[u].x, b = hv[u].y + dv[u].y, c = hv[u].z + dv[u].z, d = hv[u].w + dv[u].w;
        ss = fmaf(a, a, ss);
        ss = fmaf(b, b, ss);
        ss = fmaf(c, c, ss);
        ss = fmaf(d, d, ss);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[0][warp] = ss;
    asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) tot += red[0][w];  // fixed order: the same inv on every CTA
    const float inv = rsqrtf(tot / (float)K + xn.eps);
    for (int kk = k0 + tid; kk < k1; kk += WARPS * 32) {
      const float v = xn.h_in[kk] + xn.delta[kk];
      xs[kk - k0] = __bfloat162float(__float2bfloat16_rn(v * (xn.gain[kk] * inv)));
      if (cb == 0) xn.h_out[kk] = v;
    }
  } else {
    for (int kk = k0 + tid; kk < k1; kk += WARPS * 32) xs[kk - k0] = __bfloat162float(x[kk]);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int i = 0; i < nst; ++i) {
    const int s = i % NS;
    tc::mbar_wait(&full[s], (i / NS) & 1);
    const uint8_t* st = ring + s * STAGE_BYTES + lane * 16;
    uint4 w[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) w[r] = *reinterpret_cast<const uint4*>(st + (warp * RPW + r) * (COLS * 2));
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[s]);
    const int kb = k0 + i * TR + warp * RPW;
#pragma unroll
    for (int r = 0; r < RPW; ++r)
      if (kb + r < k1) fma8(acc, xs[kb + r - k0], w[r]);
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[warp][lane * 8 + e] = acc[e];
  asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
  const int c = tid;
  float v = 0.f;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) v += red[w][c];
  const int gcol = cb * COLS + c;
  auto store = [&](float sum) {
    if (gcol >= N) return;
    if (epi == SD_GEMM_EPI_SILU_BF16)
      ((__nv_bfloat16*)y)[gcol] = __float2bfloat16_rn(sum / (1.f + __expf(-sum)));
    else
      ((float*)y)[gcol] = sum;  // F32, or the row scratch of ADDNORM
  };
  if (splits > 1) {
    if (gcol < N) part[(int64_t)split * N + gcol] = v;
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
    if (tid == 0) s_last = atomicAdd(&counters[cb], 1) == splits - 1;
    asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
    if (!s_last) return;
    __threadfence();
    v = 0.f;
#pragma unroll 8
    for (int sp = 0; sp < splits; ++sp) v += gcol < N ? __ldcg(part + (int64_t)sp * N + gcol) : 0.f;
    if (tid == 0) counters[cb] = 0;
  }
  if (epi == SD_GEMM_EPI_ROPE) {
    // lanes c, c ^ 1 hold the pair (2i, 2i + 1) of one head (COLS and dh are even)
    const float other = __shfl_xor_sync(0xffffffffu, v, 1);
    if (gcol >= N) return;
    const int head = gcol / ro.dh, e = gcol - head * ro.dh;
    if (head < ro.H + ro.Hk) {
      const int64_t pos = *ro.pos;
      const int j = e >> 1, half = ro.dh >> 1;
      const float cs = ro.cosT[pos * half + j], sn = ro.sinT[pos * half + j];
      const float x0 = (c & 1) ? other : v, x1 = (c & 1) ? v : other;
      const float r = (c & 1) ? x0 * sn + x1 * cs : x0 * cs - x1 * sn;
      if (head < ro.H)
        ro.q[gcol] = __float2bfloat16_rn(r * ro.q_scale);
      else
        ro.k[(head - ro.H) * ro.dh + e] = __float2bfloat16_rn(r);
    } else {
      ro.v[(head - ro.H - ro.Hk) * ro.dh + e] = __float2bfloat16_rn(v);
    }
    return;
  }
  store(v);
  if constexpr (!ADDNORM) return;
  else {
  // ---- the last column block to finish normalises the whole row ----
  const int blocks = gridDim.x;
  int* row_counter = counters + (WS_HEAD_INTS - 1);
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
  if (tid == 0) s_last = atomicAdd(row_counter, 1) == blocks - 1;
  asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
  if (!s_last) return;
  __threadfence();
  // all loads of the row issued at once (N <= ADDNORM_MAX_N): one round trip, not N/256
  const float* yr = (const float*)y;
  float hv[ADDNORM_PER], gv_[ADDNORM_PER];
#pragma unroll
  for (int k = 0; k < ADDNORM_PER; ++k) {
    const int i = tid + k * WARPS * 32;
    hv[k] = i < N ? an.h[i] + __ldcg(yr + i) : 0.f;
    gv_[k] = i < N ? an.gain[i] : 0.f;
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < ADDNORM_PER; ++k) ss += hv[k] * hv[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[0][warp] = ss;
  asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) tot += red[0][w];
  const float inv = rsqrtf(tot / (float)N + an.eps);
#pragma unroll
  for (int k = 0; k < ADDNORM_PER; ++k) {
    const int i = tid + k * WARPS * 32;
    if (i < N) {
      an.h[i] = hv[k];
      const float xv = hv[k] * (gv_[k] * inv);
      if (an.x_bf16)
        ((__nv_bfloat16*)an.x)[i] = __float2bfloat16_rn(xv);
      else
        ((float*)an.x)[i] = xv;
    }
  }
  if (tid == 0) *row_counter = 0;
  }
}

static int tma_splits(int K, int N) {
  const int blocks = (N + COLS - 1) / COLS;
  int s = 148 * SD_GEMV_TMA_CPS / blocks;  // one wave
  const int max_s = K / (2 * TR) > 0 ? K / (2 * TR) : 1;
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

static bool use_tma() {  // SD_GEMV_IMPL=tma|ld overrides the build default (read per call: tests flip it)
  const char* e = getenv("SD_GEMV_IMPL");
  return e ? (e[0] == 't') : SD_GEMV_TMA_DEFAULT;
}

// tensor maps are built once per (weights, K, N): the draft's weights are static
static int weight_map(const void* w, int K, int N, CUtensorMap* out) {
  struct Key {
    const void* w;
    int K, N;
    bool operator==(const Key& o) const { return w == o.w && K == o.K && N == o.N; }
  };
  struct H {
    size_t operator()(const Key& k) const { return std::hash<const void*>()(k.w) ^ ((size_t)k.K << 20) ^ k.N; }
  };
  static std::unordered_map<Key, CUtensorMap, H> cache;
  const Key key{w, K, N};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return 0;
  }
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SD_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)N * 2};
  cuuint32_t box[2] = {(cuuint32_t)COLS, (cuuint32_t)TR};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SD_ECUDA;
  }
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return 0;
}

// one launch of the TMA kernel; false when its shared memory would not fit
static bool launch_tma(const void* x, int K, const void* w, int N, int epi, void* y, void* workspace,
                       const AddNorm& an, cudaStream_t st, int* rc, const XNorm& xn = XNorm{},
                       const RopeOut& ro = RopeOut{}) {
  const int blocks = (N + COLS - 1) / COLS;
  const int s = tma_splits(K, N);
  const size_t smem = (size_t)NS * STAGE_BYTES + ((K + s - 1) / s + 1) * sizeof(float);
  if (!use_tma() || smem > 212 * 1024) return false;
  CUtensorMap m;
  if (weight_map(w, K, N, &m)) {
    *rc = SD_ECUDA;
    return true;
  }
  // the attribute only grows: graph nodes captured with a larger size must still
  // launch after a smaller shape was captured (kernel replay re-checks it)
  auto kern = epi == SD_GEMM_EPI_ADDNORM ? gemv_tma_kernel<true> : gemv_tma_kernel<false>;
  static size_t attr[2] = {0, 0};
  size_t& at = attr[epi == SD_GEMM_EPI_ADDNORM];
  if (smem > at) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    at = smem;
  }
  launch_pdl(kern, dim3(blocks, s), dim3((WARPS + 1) * 32), smem, st, m, (const __nv_bfloat16*)x, K, N,
             s, epi, y, s > 1 ? (float*)((char*)workspace + WS_HEAD) : nullptr, (int*)workspace, an, xn, ro);
  *rc = check_launch("sd_gemv");
  return true;
}

static int launch_ld(const void* x, int K, const void* w, int N, int epi, void* y, void* workspace,
                     cudaStream_t st) {
  const int blocks = (N + COLS - 1) / COLS;
  const int s = splits_for(K, N);
  const int kslice = (K + s - 1) / s + 1;
  const size_t smem = (size_t)kslice * sizeof(float);
  SD_REQUIRE(smem <= 200 * 1024, "sd_gemv: K slice too long");
  static size_t attr = 48 * 1024;  // only grows (see above)
  if (smem > attr) {
    cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  launch_pdl(gemv_kernel, dim3(blocks, s), dim3(WARPS * 32), smem, st, (const __nv_bfloat16*)x,
             (const __nv_bfloat16*)w, K, N, s, epi, y, s > 1 ? (float*)((char*)workspace + WS_HEAD) : nullptr,
             (int*)workspace);
  return check_launch("sd_gemv");
}

static size_t partial_bytes(int K, int N) {
  int s = splits_for(K, N);
  const int st = tma_splits(K, N);
  if (st > s) s = st;  // either implementation fits
  return s > 1 ? (size_t)s * N * sizeof(float) : 0;
}

}  // namespace gv
}  // namespace sd

using namespace sd;

extern "C" {

size_t sd_gemv_workspace_bytes(int K, int N) {
  if (K <= 0 || N <= 0) return 0;
  // counter head | split partials | one fp32 row (the add+norm epilogue's scratch)
  return gv::WS_HEAD + gv::partial_bytes(K, N) + (size_t)N * sizeof(float);
}

int sd_gemv(const void* x, int K, const void* w, int N, int epi, void* y, void* workspace, size_t workspace_bytes,
            sd_stream_t stream) {
  SD_REQUIRE(x && w && y && K > 0 && N > 0 && N % 8 == 0, "sd_gemv: K=%d N=%d (N %% 8 == 0)", K, N);
  SD_REQUIRE(((uintptr_t)w % 16) == 0, "sd_gemv: W must be 16-byte aligned");
  SD_REQUIRE(epi == SD_GEMM_EPI_F32 || epi == SD_GEMM_EPI_SILU_BF16, "sd_gemv: epilogue");
  const int blocks = (N + gv::COLS - 1) / gv::COLS;
  SD_REQUIRE((size_t)blocks < (size_t)gv::WS_HEAD_INTS, "sd_gemv: N=%d too wide for the counter head", N);
  SD_REQUIRE(workspace && workspace_bytes >= sd_gemv_workspace_bytes(K, N), "sd_gemv: workspace");
  int rc = 0;
  if (gv::launch_tma(x, K, w, N, epi, y, workspace, gv::AddNorm{}, as_stream(stream), &rc)) return rc;
  return gv::launch_ld(x, K, w, N, epi, y, workspace, as_stream(stream));
}

int sd_gemv_norm(const float* h_in, const float* delta, const float* gain, float eps, float* h_out, int K,
                 const void* w, int N, int epi, void* y, void* workspace, size_t workspace_bytes, sd_stream_t stream) {
  SD_REQUIRE(h_in && delta && gain && h_out && h_out != h_in && w && y && K > 0 && K % 4 == 0 && N > 0 && N % 8 == 0,
             "sd_gemv_norm: K=%d N=%d", K, N);
  SD_REQUIRE(((uintptr_t)h_in % 16) == 0 && ((uintptr_t)delta % 16) == 0, "sd_gemv_norm: h / delta alignment");
  SD_REQUIRE(((uintptr_t)w % 16) == 0, "sd_gemv_norm: W must be 16-byte aligned");
  SD_REQUIRE(epi == SD_GEMM_EPI_F32 || epi == SD_GEMM_EPI_SILU_BF16, "sd_gemv_norm: epilogue");
  const int blocks = (N + gv::COLS - 1) / gv::COLS;
  SD_REQUIRE((size_t)blocks < (size_t)gv::WS_HEAD_INTS, "sd_gemv_norm: N=%d too wide for the counter head", N);
  SD_REQUIRE(workspace && workspace_bytes >= sd_gemv_workspace_bytes(K, N), "sd_gemv_norm: workspace");
  const gv::XNorm xn{h_in, delta, gain, eps, h_out};
  int rc = 0;
  if (gv::launch_tma(nullptr, K, w, N, epi, y, workspace, gv::AddNorm{}, as_stream(stream), &rc, xn)) return rc;
  set_error("sd_gemv_norm: the TMA weight stream does not fit this shape");
  return SD_EUNSUPPORTED;
}

int sd_gemv_rope(const void* x, const float* h_in, const float* delta, const float* gain, float eps, float* h_out,
                 int K, const void* w, int N, const int32_t* pos, const float* cos_table, const float* sin_table,
                 float q_scale, int H, int Hk, int dh, void* q_rot, void* k_rot, void* v, void* workspace,
                 size_t workspace_bytes, sd_stream_t stream) {
  SD_REQUIRE(w && pos && cos_table && sin_table && q_rot && k_rot && v && K > 0 && K % 4 == 0, "sd_gemv_rope: args");
  SD_REQUIRE(dh > 0 && dh % 2 == 0 && H > 0 && Hk > 0 && N == (H + 2 * Hk) * dh && N % 8 == 0,
             "sd_gemv_rope: N=%d must be (H + 2 Hk) * dh", N);
  SD_REQUIRE((x != nullptr) != (h_in != nullptr), "sd_gemv_rope: exactly one of x / h_in");
  SD_REQUIRE(!h_in || (delta && gain && h_out && h_out != h_in && ((uintptr_t)h_in % 16) == 0 &&
                       ((uintptr_t)delta % 16) == 0),
             "sd_gemv_rope: residual norm inputs");
  SD_REQUIRE(((uintptr_t)w % 16) == 0, "sd_gemv_rope: W must be 16-byte aligned");
  const int blocks = (N + gv::COLS - 1) / gv::COLS;
  SD_REQUIRE((size_t)blocks < (size_t)gv::WS_HEAD_INTS, "sd_gemv_rope: N=%d too wide for the counter head", N);
  SD_REQUIRE(workspace && workspace_bytes >= sd_gemv_workspace_bytes(K, N), "sd_gemv_rope: workspace");
  const gv::XNorm xn = h_in ? gv::XNorm{h_in, delta, gain, eps, h_out} : gv::XNorm{};
  const gv::RopeOut ro{pos, cos_table, sin_table, q_scale, H, Hk, dh, (__nv_bfloat16*)q_rot,
                       (__nv_bfloat16*)k_rot, (__nv_bfloat16*)v};
  int rc = 0;
  if (gv::launch_tma(x, K, w, N, SD_GEMM_EPI_ROPE, nullptr, workspace, gv::AddNorm{}, as_stream(stream), &rc, xn,
                     ro))
    return rc;
  set_error("sd_gemv_rope: the TMA weight stream does not fit this shape");
  return SD_EUNSUPPORTED;
}

int sd_gemv_addnorm(const void* x, int K, const void* w, int N, float* h, const float* gain, float eps, void* x_out,
                    int x_dtype, void* workspace, size_t workspace_bytes, sd_stream_t stream) {
  SD_REQUIRE(x && w && h && gain && x_out && K > 0 && N > 0 && N % 8 == 0, "sd_gemv_addnorm: K=%d N=%d", K, N);
  SD_REQUIRE(((uintptr_t)w % 16) == 0, "sd_gemv_addnorm: W must be 16-byte aligned");
  SD_REQUIRE(x_dtype == SD_BF16 || x_dtype == SD_F32, "sd_gemv_addnorm: x dtype");
  const int blocks = (N + gv::COLS - 1) / gv::COLS;
  SD_REQUIRE((size_t)blocks < (size_t)gv::WS_HEAD_INTS, "sd_gemv_addnorm: N=%d too wide", N);
  SD_REQUIRE(workspace && workspace_bytes >= sd_gemv_workspace_bytes(K, N), "sd_gemv_addnorm: workspace");
  float* yrow = (float*)((char*)workspace + gv::WS_HEAD + gv::partial_bytes(K, N));
  const gv::AddNorm an{h, gain, eps, x_out, x_dtype == SD_BF16};
  int rc = 0;
  if (N <= gv::ADDNORM_MAX_N &&
      gv::launch_tma(x, K, w, N, SD_GEMM_EPI_ADDNORM, yrow, workspace, an, as_stream(stream), &rc))
    return rc;
  // projection, then the separate add + norm (long rows, or the register-streaming kernel)
  if (gv::launch_tma(x, K, w, N, SD_GEMM_EPI_F32, yrow, workspace, gv::AddNorm{}, as_stream(stream), &rc)) {
    if (rc) return rc;
  } else {
    rc = gv::launch_ld(x, K, w, N, SD_GEMM_EPI_F32, yrow, workspace, as_stream(stream));
  }
  if (rc) return rc;
  return sd_add_rmsnorm(h, yrow, 1, N, gain, eps, x_out, x_dtype, 1, 0, stream);
}

}  // extern "C"
