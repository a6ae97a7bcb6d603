// Dense-layer plumbing around the cuBLAS GEMMs + RoPE/KV staging.
// Reference: model.py:216-236 (rope, rmsnorm), 276-289 (per-row q/k/v, stage),
// 306-311 (residual, SiLU MLP, final norm); kvcache.py:91-96 (stage).
#include <stdarg.h>

#include "common.cuh"

namespace sd {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SD_ECUDA;
  }
  return SD_OK;
}

template <typename T>
__global__ void embed_kernel(const int32_t* __restrict__ tok, const T* __restrict__ E, int d, float* __restrict__ h) {
  const int t = blockIdx.x;
  const T* row = E + (int64_t)tok[t] * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) h[(int64_t)t * d + i] = to_f(row[i]);
}

// bf16 rows, 8 elements (one 16-byte load) per thread
__global__ void embed8_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ E, int d,
                              float* __restrict__ h) {
  const int t = blockIdx.x;
  const uint4* row = reinterpret_cast<const uint4*>(E + (int64_t)tok[t] * d);
  float4* out = reinterpret_cast<float4*>(h + (int64_t)t * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    const uint4 v = row[i];
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
    const float2 a = __bfloat1622float2(p[0]), b = __bfloat1622float2(p[1]);
    const float2 c = __bfloat1622float2(p[2]), e = __bfloat1622float2(p[3]);
    out[2 * i] = make_float4(a.x, a.y, b.x, b.y);
    out[2 * i + 1] = make_float4(c.x, c.y, e.x, e.y);
  }
}

// one block per row: h += delta; x = h * gain / sqrt(mean(h^2) + eps).
// float4 vectors: every thread issues its loads before the reduction.
template <typename XT>
__device__ __forceinline__ void store4(XT* x, int64_t i, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4<float>(float* x, int64_t i, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(x + i) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* x, int64_t i, float a, float b, float c,
                                                      float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 v;
  v.x = *reinterpret_cast<uint32_t*>(&lo);
  v.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(x + i) = v;
}

// x[0] + x[s * stride] for s = 1 .. splits-1, summed in slice order (split-K
// slices of a projection); the loads of up to 8 slices are issued before any
// add, so a 9-slice sum costs two L2 round trips instead of nine
__device__ __forceinline__ float4 sum_slices4(const float* p, int splits, int64_t stride) {
  float4 acc = *reinterpret_cast<const float4*>(p);
  for (int s0 = 1; s0 < splits; s0 += 8) {
    float4 e[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      e[u] = s0 + u < splits ? *reinterpret_cast<const float4*>(p + (s0 + u) * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (s0 + u < splits) {
        acc.x += e[u].x;
        acc.y += e[u].y;
        acc.z += e[u].z;
        acc.w += e[u].w;
      }
  }
  return acc;
}

template <typename XT, int PER>
__global__ void add_rmsnorm_kernel(float* __restrict__ h, const float* __restrict__ delta, int d,
                                   const float* __restrict__ gain, float eps, XT* __restrict__ x, int splits,
                                   int64_t split_stride) {
  __shared__ float red[32];
  pdl_trigger();
  // the gains are weights (never written by a kernel): loaded before the wait
  float4 g[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = (threadIdx.x + k * blockDim.x) * 4;
    if (i < d) g[k] = *reinterpret_cast<const float4*>(gain + i);
  }
  pdl_wait();
  const int64_t base = (int64_t)blockIdx.x * d;
  float4 v[PER];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = (threadIdx.x + k * blockDim.x) * 4;
    if (i < d) {
      v[k] = *reinterpret_cast<const float4*>(h + base + i);
      if (delta) {
        const float4 dd = sum_slices4(delta + base + i, splits, split_stride);  // split-K slices, in order
        v[k].x += dd.x; v[k].y += dd.y; v[k].z += dd.z; v[k].w += dd.w;
        *reinterpret_cast<float4*>(h + base + i) = v[k];
      }
      ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
  }
  ss = block_reduce(ss, red, [](float a, float b) { return a + b; });
  const float inv = rsqrtf(ss / (float)d + eps);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = (threadIdx.x + k * blockDim.x) * 4;
    if (i < d)
      store4<XT>(x, base + i, v[k].x * (g[k].x * inv), v[k].y * (g[k].y * inv), v[k].z * (g[k].z * inv),
                 v[k].w * (g[k].w * inv));
  }
}

template <typename XT>
__global__ void add_rmsnorm_scalar_kernel(float* __restrict__ h, const float* __restrict__ delta, int d,
                                          const float* __restrict__ gain, float eps, XT* __restrict__ x, int splits,
                                          int64_t split_stride) {
  __shared__ float red[32];
  pdl_trigger();
  pdl_wait();
  const int64_t base = (int64_t)blockIdx.x * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = h[base + i];
    if (delta) {
      float dd = delta[base + i];
      for (int s = 1; s < splits; ++s) dd += delta[s * split_stride + base + i];
      v += dd;
      h[base + i] = v;
    }
    ss += v * v;
  }
  ss = block_reduce(ss, red, [](float a, float b) { return a + b; });
  const float inv = rsqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) x[base + i] = from_f<XT>(h[base + i] * (gain[i] * inv));
}

// 4 elements per thread: one 16-byte load, one 8-byte (bf16) / 16-byte (fp32) store
template <typename OT>
__global__ void silu4_kernel(const float4* __restrict__ a, OT* __restrict__ out, size_t n4,
                             const int32_t* __restrict__ rows_dev, int64_t row_quads) {
  pdl_trigger();
  pdl_wait();  // a is the projection before (PDL launch: may start under its tail)
  // rows_dev (the tree record's live row count): padded rows past it are skipped
  if (rows_dev) n4 = min(n4, (size_t)(*rows_dev) * (size_t)row_quads);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(a + i);
    const float r0 = v.x / (1.f + __expf(-v.x)), r1 = v.y / (1.f + __expf(-v.y));
    const float r2 = v.z / (1.f + __expf(-v.z)), r3 = v.w / (1.f + __expf(-v.w));
    if constexpr (sizeof(OT) == 2) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(r0, r1), hi = __floats2bfloat162_rn(r2, r3);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out)[i] = pk;
    } else {
      reinterpret_cast<float4*>(out)[i] = make_float4(r0, r1, r2, r3);
    }
  }
}

template <typename OT>
__global__ void silu_kernel(const float* __restrict__ a, OT* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = a[i];
    out[i] = from_f<OT>(v / (1.f + __expf(-v)));
  }
}

template <typename OT>
__global__ void add_cast_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                                OT* __restrict__ cast, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = a[i] + b[i];
    out[i] = v;
    if (cast) cast[i] = from_f<OT>(v);
  }
}

// grid: T rows; each thread rotates 2 adjacent pairs (4 elements) of one
// q/k head, or copies 4 elements of v.
template <typename T>
__device__ __forceinline__ void put2(T* p, float a, float b);
template <>
__device__ __forceinline__ void put2<float>(float* p, float a, float b) {
  *reinterpret_cast<float2*>(p) = make_float2(a, b);
}
template <>
__device__ __forceinline__ void put2<__nv_bfloat16>(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}

template <typename QT, typename KT>
__global__ void rope_stage_kernel(const float* __restrict__ qkv, int H, int Hk, int dh,
                                  const int32_t* __restrict__ positions, const float* __restrict__ cosT,
                                  const float* __restrict__ sinT, float q_scale, QT* __restrict__ q_rot,
                                  float* __restrict__ q_pre, KT* __restrict__ k_raw, KT* __restrict__ k_rot,
                                  KT* __restrict__ v, int64_t head_stride, int64_t row_offset,
                                  const int32_t* __restrict__ rows_dev, int splits, int64_t split_stride) {
  const int t = blockIdx.x;
  pdl_trigger();
  // positions / rows_dev come from the tree record or a host fill (never from a
  // programmatic-dependent kernel), and cos/sin are tables: all read before the
  // wait, so only the projection output waits for the kernel before
  if (rows_dev && t >= *rows_dev) {
    pdl_wait();
    return;
  }
  const int half = dh >> 1;
  const int width = (H + 2 * Hk) * dh;
  const float* row = qkv + (int64_t)t * width;
  const int64_t pos = positions[t];
  // row_offset < 0: rows go to positions[0] + t (verify rows staged after the
  // committed cache; device-resident step under graph replay)
  const int64_t dst_row = (row_offset >= 0 ? row_offset : (int64_t)positions[0]) + t;
  const int quads_rot = (H + Hk) * dh / 4, quads_all = width / 4;
  constexpr int PF = 4;  // rotation tables prefetched for a thread's first PF quads
  float2 pc[PF], ps[PF];
#pragma unroll
  // a row may be spread over gridDim.y CTAs (split-K input: the slice reads of
  // one row would otherwise bound a single CTA)
  const int u0 = threadIdx.x + blockIdx.y * blockDim.x, ustep = blockDim.x * gridDim.y;
  for (int k = 0; k < PF; ++k) {
    const int u = u0 + k * ustep;
    if (u < quads_rot) {
      const int j = ((4 * u) % dh) >> 1;
      pc[k] = *reinterpret_cast<const float2*>(cosT + pos * half + j);
      ps[k] = *reinterpret_cast<const float2*>(sinT + pos * half + j);
    }
  }
  pdl_wait();
  int k = 0;
  for (int u = u0; u < quads_all; u += ustep, ++k) {
    float4 x = sum_slices4(row + 4 * u, splits, split_stride);  // split-K slices of the QKV GEMM, in order
    const int col = 4 * u, head = col / dh, e = col - head * dh;
    if (u < quads_rot) {
      const int j = e >> 1;  // pair index of x.x/x.y; x.z/x.w is j + 1
      float2 c, s;
      if (k < PF) {
#pragma unroll
        for (int q = 0; q < PF; ++q)
          if (q == k) {
            c = pc[q];
            s = ps[q];
          }
      } else {
        c = *reinterpret_cast<const float2*>(cosT + pos * half + j);
        s = *reinterpret_cast<const float2*>(sinT + pos * half + j);
      }
      const float r0 = x.x * c.x - x.y * s.x, r1 = x.x * s.x + x.y * c.x;
      const float r2 = x.z * c.y - x.w * s.y, r3 = x.z * s.y + x.w * c.y;
      if (head < H) {
        const int64_t o = ((int64_t)t * H + head) * dh + e;
        put2<QT>(q_rot + o, r0 * q_scale, r1 * q_scale);
        put2<QT>(q_rot + o + 2, r2 * q_scale, r3 * q_scale);
        if (q_pre) *reinterpret_cast<float4*>(q_pre + o) = x;
      } else {
        const int64_t o = (head - H) * head_stride + dst_row * dh + e;
        put2<KT>(k_rot + o, r0, r1);
        put2<KT>(k_rot + o + 2, r2, r3);
        if (k_raw) {
          put2<KT>(k_raw + o, x.x, x.y);
          put2<KT>(k_raw + o + 2, x.z, x.w);
        }
      }
    } else {
      const int64_t o = (head - H - Hk) * head_stride + dst_row * dh + e;
      put2<KT>(v + o, x.x, x.y);
      put2<KT>(v + o + 2, x.z, x.w);
    }
  }
}

static int grid_for(size_t n) {
  size_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g ? g : 1);
}

}  // namespace sd

using namespace sd;

extern "C" {

int sd_version(void) { return 1; }
const char* sd_last_error(void) { return sd::g_err; }

int sd_embed(const int32_t* tokens, int T, const void* embed, int dtype, int d, float* h, sd_stream_t stream) {
  SD_REQUIRE(T > 0 && d > 0, "sd_embed: bad sizes");
  auto st = as_stream(stream);
  if (dtype == SD_BF16 && d % 8 == 0 && ((uintptr_t)embed % 16) == 0 && ((uintptr_t)h % 16) == 0)
    embed8_kernel<<<T, d / 8 < 512 ? ((d / 8 + 31) / 32) * 32 : 512, 0, st>>>(tokens, (const __nv_bfloat16*)embed,
                                                                          d, h);
  else if (dtype == SD_BF16)
    embed_kernel<<<T, 256, 0, st>>>(tokens, (const __nv_bfloat16*)embed, d, h);
  else if (dtype == SD_F32)
    embed_kernel<<<T, 256, 0, st>>>(tokens, (const float*)embed, d, h);
  else
    SD_REQUIRE(false, "sd_embed: dtype");
  return check_launch("sd_embed");
}

int sd_add_rmsnorm(float* h, const float* delta, int T, int d, const float* gain, float eps, void* x, int x_dtype,
                   int delta_splits, int64_t delta_split_stride, sd_stream_t stream) {
  if (delta_splits < 1) delta_splits = 1;
  SD_REQUIRE(T > 0 && d > 0, "sd_add_rmsnorm: bad sizes");
  SD_REQUIRE(x_dtype == SD_BF16 || x_dtype == SD_F32, "sd_add_rmsnorm: dtype");
  auto st = as_stream(stream);
  if (d % 4 == 0 && d <= 4 * 1024 * 2) {
    const int quads = d / 4;
    const int threads = quads >= 1024 ? 1024 : ((quads + 31) / 32) * 32;
    const bool two = quads > threads;
#define SD_NORM(XT, PER) \
  launch_pdl(add_rmsnorm_kernel<XT, PER>, dim3(T), dim3(threads), 0, st, h, delta, d, gain, eps, (XT*)x, delta_splits, \
             delta_split_stride)
    if (x_dtype == SD_BF16) {
      if (two) SD_NORM(__nv_bfloat16, 2); else SD_NORM(__nv_bfloat16, 1);
    } else {
      if (two) SD_NORM(float, 2); else SD_NORM(float, 1);
    }
#undef SD_NORM
  } else {
    const int threads = d >= 1024 ? 1024 : (d >= 256 ? 256 : 128);
    if (x_dtype == SD_BF16)
      launch_pdl(add_rmsnorm_scalar_kernel<__nv_bfloat16>, dim3(T), dim3(threads), 0, st, h, delta, d, gain, eps,
                 (__nv_bfloat16*)x, delta_splits, delta_split_stride);
    else
      launch_pdl(add_rmsnorm_scalar_kernel<float>, dim3(T), dim3(threads), 0, st, h, delta, d, gain, eps, (float*)x,
                 delta_splits, delta_split_stride);
  }
  return check_launch("sd_add_rmsnorm");
}

int sd_silu(const float* a, void* out, int out_dtype, size_t n, sd_stream_t stream) {
  auto st = as_stream(stream);
  const bool vec = n % 4 == 0 && ((uintptr_t)a % 16) == 0 && ((uintptr_t)out % 16) == 0;
  if (vec && out_dtype == SD_BF16)
    launch_pdl(silu4_kernel<__nv_bfloat16>, dim3(grid_for(n / 4)), dim3(256), 0, st, (const float4*)a,
               (__nv_bfloat16*)out, n / 4, (const int32_t*)nullptr, (int64_t)0);
  else if (vec && out_dtype == SD_F32)
    launch_pdl(silu4_kernel<float>, dim3(grid_for(n / 4)), dim3(256), 0, st, (const float4*)a, (float*)out, n / 4,
               (const int32_t*)nullptr, (int64_t)0);
  else if (out_dtype == SD_BF16)
    silu_kernel<<<grid_for(n), 256, 0, st>>>(a, (__nv_bfloat16*)out, n);
  else if (out_dtype == SD_F32)
    silu_kernel<<<grid_for(n), 256, 0, st>>>(a, (float*)out, n);
  else
    SD_REQUIRE(false, "sd_silu: dtype");
  return check_launch("sd_silu");
}

int sd_silu_rows(const float* a, void* out, int out_dtype, int T, int N, const int32_t* rows_dev,
                 sd_stream_t stream) {
  SD_REQUIRE(T > 0 && N > 0 && N % 4 == 0 && ((uintptr_t)a % 16) == 0 && ((uintptr_t)out % 16) == 0,
             "sd_silu_rows: N %% 4 and 16-byte alignment");
  auto st = as_stream(stream);
  const size_t n4 = (size_t)T * N / 4;
  if (out_dtype == SD_BF16)
    launch_pdl(silu4_kernel<__nv_bfloat16>, dim3(grid_for(n4)), dim3(256), 0, st, (const float4*)a,
               (__nv_bfloat16*)out, n4, rows_dev, (int64_t)(N / 4));
  else if (out_dtype == SD_F32)
    launch_pdl(silu4_kernel<float>, dim3(grid_for(n4)), dim3(256), 0, st, (const float4*)a, (float*)out, n4, rows_dev,
               (int64_t)(N / 4));
  else
    SD_REQUIRE(false, "sd_silu_rows: dtype");
  return check_launch("sd_silu_rows");
}

int sd_add_cast(const float* a, const float* b, float* out, void* cast_out, int cast_dtype, size_t n,
                sd_stream_t stream) {
  auto st = as_stream(stream);
  if (cast_dtype == SD_BF16)
    add_cast_kernel<<<grid_for(n), 256, 0, st>>>(a, b, out, (__nv_bfloat16*)cast_out, n);
  else
    add_cast_kernel<<<grid_for(n), 256, 0, st>>>(a, b, out, (float*)cast_out, n);
  return check_launch("sd_add_cast");
}

int sd_rope_stage(const float* qkv, int T, int H, int Hk, int dh, const int32_t* positions, const float* rope_cos,
                  const float* rope_sin, float q_scale, void* q_rot, int q_dtype, float* q_pre, void* k_raw,
                  void* k_rot, void* v, int kv_dtype, int64_t head_stride, int64_t row_offset,
                  const int32_t* rows_dev, int qkv_splits, int64_t qkv_split_stride, sd_stream_t stream) {
  if (qkv_splits < 1) qkv_splits = 1;
  SD_REQUIRE(T > 0 && H > 0 && Hk > 0 && dh > 0 && (dh % 4) == 0, "sd_rope_stage: head_dim must be a multiple of 4");
  auto st = as_stream(stream);
  // split-K input: one CTA per 512 quads of a row, so each row's slice reads spread over several SMs
  static const bool spread_all = getenv("SD_ROPE_SPREAD") && atoi(getenv("SD_ROPE_SPREAD")) != 0;  // A/B (tools)
  const int rc = (qkv_splits > 1 || (spread_all && T > 1)) ? ((H + 2 * Hk) * dh / 4 + 511) / 512 : 1;
#define SD_RS(QT, KT)                                                                                          \
  launch_pdl(rope_stage_kernel<QT, KT>, dim3(T, rc), dim3(512), 0, st, qkv, H, Hk, dh, positions, rope_cos, rope_sin,  \
             q_scale, (QT*)q_rot, q_pre, (KT*)k_raw, (KT*)k_rot, (KT*)v, head_stride, row_offset, rows_dev,       \
             qkv_splits, qkv_split_stride)
  if (q_dtype == SD_F32 && kv_dtype == SD_F32)
    SD_RS(float, float);
  else if (q_dtype == SD_BF16 && kv_dtype == SD_BF16)
    SD_RS(__nv_bfloat16, __nv_bfloat16);
  else if (q_dtype == SD_F32 && kv_dtype == SD_BF16)
    SD_RS(float, __nv_bfloat16);
  else
    SD_REQUIRE(false, "sd_rope_stage: dtype combo");
#undef SD_RS
  return check_launch("sd_rope_stage");
}

}  // extern "C"
