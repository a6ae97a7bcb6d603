// Split-KV attention for the decode step: tree verification over the full
// cache, draft attention over the rank-rotated partial cache, AR decode and
// causal prefill blocks — one kernel family, CUDA-core fp32 math.
//
// Reference semantics: model.py:238-247 (_attend: softmax(q.k/sqrt(dh)) V with
// query head j on kv head j // G), model.py:290-300 (masked: cache + ancestors
// + self), model.py:301-305 (causal), kvcache.py:158-165 (draft keys rotated at
// rank 0..m-1).
//
// Grid: x = cache chunk (chunk length is a function of ctx only, so the result
// is bitwise independent of how many GPUs share the heads) + 1 tree chunk,
// y = kv head, z = query-row tile. Each CTA writes an un-normalised partial
// (o / l, lse) per query row; sd_attention then merges chunks in fixed order.
#include <cuda_fp16.h>

#include "common.cuh"

namespace sd {

struct AttnParams {
  const void* q;
  int T, H, Hk, G;
  const void* k_cache;
  const void* v_cache;
  int64_t head_stride;
  int ctx;
  const int32_t* ranks;
  const float* cosT;
  const float* sinT;
  const void* k_tree;
  const void* v_tree;
  int64_t tree_head_stride;
  const uint32_t* mask;
  int mask_words;
  int chunk, n_chunks;
  float* ws_o;
  float* ws_lse;
  const int32_t* rows_dev;  // nullable: live row count (<= T) read on device
  const int32_t* ctx_dev;   // nullable: live cache length (<= ctx) read on device; the tree
                            // rows then sit right after it in k_cache / v_cache
  int x_base;               // chunk index of blockIdx.x == 0 (tree-only launches)
};

// live cache length and tree-row base pointers of kv head `kvh`
template <int DH, typename KT>
__device__ __forceinline__ int resolve_ctx(const AttnParams& p, int kvh, const KT*& Kt, const KT*& Vt) {
  if (p.ctx_dev) {
    const int c = *p.ctx_dev;
    Kt = (const KT*)p.k_cache + kvh * p.head_stride + (int64_t)c * DH;
    Vt = (const KT*)p.v_cache + kvh * p.head_stride + (int64_t)c * DH;
    return c;
  }
  Kt = (const KT*)p.k_tree + kvh * p.tree_head_stride;
  Vt = (const KT*)p.v_tree + kvh * p.tree_head_stride;
  return p.ctx;
}

__device__ __forceinline__ int live_rows(const AttnParams& p) {
  if (!p.rows_dev) return p.T;
  const int t = *p.rows_dev;
  return t < p.T ? t : p.T;
}

// partial-cache slots with rank < 0 are holes (evicted, not yet reused)
__device__ __forceinline__ uint32_t slot_valid_bits(const int32_t* __restrict__ ranks, int kb, int nk, int lane) {
  const bool ok = lane < nk && ranks[kb + lane] >= 0;
  return __ballot_sync(0xffffffffu, ok);
}

static inline int chunk_len_for(int ctx) {
  int c = (ctx + 31) / 32;
  c = (c + 255) / 256 * 256;
  return c < 256 ? 256 : c;
}
static inline int n_chunks_for(int ctx) {
  if (ctx <= 0) return 0;
  const int c = chunk_len_for(ctx);
  return (ctx + c - 1) / c;
}

// Stage 32 keys (rows key0.. of a source) into Ks [32][DH+1] / Vs [32][DH] as
// fp32; `lane_stride` threads cooperate (a warp or the whole CTA).
template <int DH, typename KT, bool ROT>
__device__ __forceinline__ void stage_tile(float* Ks, float* Vs, const KT* __restrict__ K, const KT* __restrict__ V,
                                           int key0, int nkeys, const int32_t* __restrict__ ranks,
                                           const float* __restrict__ cosT, const float* __restrict__ sinT, int tid,
                                           int nthreads) {
  constexpr int HALF = DH / 2;
  // K: pairs so RoPE can be applied on load
  for (int i = tid; i < 32 * HALF; i += nthreads) {
    const int j = i / HALF, e = i - j * HALF;
    float a = 0.f, b = 0.f;
    if (j < nkeys) {
      const int64_t row = key0 + j;
      a = to_f(K[row * DH + 2 * e]);
      b = to_f(K[row * DH + 2 * e + 1]);
      if (ROT) {
        int64_t r = ranks[row];
        if (r < 0) r = 0;  // hole slot: masked out by slot_valid_bits, keep the table read in bounds
        const float c = cosT[r * HALF + e], s = sinT[r * HALF + e];
        const float ra = a * c - b * s, rb = a * s + b * c;
        a = ra;
        b = rb;
      }
    }
    Ks[j * (DH + 1) + 2 * e] = a;
    Ks[j * (DH + 1) + 2 * e + 1] = b;
  }
  for (int i = tid; i < 32 * DH; i += nthreads) {
    const int j = i / DH, e = i - j * DH;
    Vs[j * DH + e] = j < nkeys ? to_f(V[(int64_t)(key0 + j) * DH + e]) : 0.f;
  }
}

// Online-softmax update of RPW query rows against one 32-key tile (lane = key).
// vis[r]: bitmask of visible keys of this tile for row r (0 = row inactive).
template <int DH, int RPW>
__device__ __forceinline__ void tile_update(const float* __restrict__ Ks, const float* __restrict__ Vs,
                                            const float* const* qrow, const uint32_t* vis, float* m, float* l,
                                            float (*acc)[(DH >= 32 ? DH / 32 : 1)], int lane) {
  constexpr int EPL = DH >= 32 ? DH / 32 : 1;
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    if (vis[r] == 0u) continue;  // warp-uniform
    const float* q = qrow[r];
    float s = 0.f;
#pragma unroll 16
    for (int d = 0; d < DH; ++d) s = fmaf(q[d], Ks[lane * (DH + 1) + d], s);
    const bool on = (vis[r] >> lane) & 1u;
    s = on ? s : -INFINITY;
    const float tmax = warp_max(s);
    const float mn = fmaxf(m[r], tmax);
    if (mn == -INFINITY) continue;         // nothing visible yet (warp-uniform)
    const float corr = __expf(m[r] - mn);  // m = -inf initially -> 0
    const float p = on ? __expf(s - mn) : 0.f;
    l[r] = l[r] * corr + warp_sum(p);
    m[r] = mn;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[r][e] *= corr;
    if (DH >= 32 || lane < DH) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[r][e] = fmaf(pj, Vs[j * DH + lane * EPL + e], acc[r][e]);
      }
    } else {
      for (int j = 0; j < 32; ++j) (void)__shfl_sync(0xffffffffu, p, j);
    }
  }
}

// visibility bits of tile keys [kt0, kt0+32) of the tree chunk for request row t
__device__ __forceinline__ uint32_t tree_vis(const uint32_t* __restrict__ mask, int mask_words, int t, int kt0,
                                             int nkeys) {
  uint32_t bits;
  if (mask) {
    const int w = kt0 >> 5;  // kt0 multiple of 32
    bits = w < mask_words ? mask[t * mask_words + w] : 0u;
  } else {
    bits = 0xffffffffu;
  }
  // only rows j <= t (ancestors and self); self always
  const int lim = t - kt0;  // keys kt0..kt0+lim visible by causality
  uint32_t causal = lim >= 31 ? 0xffffffffu : (lim < 0 ? 0u : ((1u << (lim + 1)) - 1u));
  bits &= causal;
  if (lim >= 0 && lim < 32) bits |= (1u << lim);
  const uint32_t valid = nkeys >= 32 ? 0xffffffffu : ((1u << nkeys) - 1u);
  return bits & valid;
}

// Mode A: 8 warps split 64 query rows (8 each); the CTA stages shared 32-key tiles.
template <int DH, typename QT, typename KT, bool ROT>
__global__ void __launch_bounds__(256) attn_rows_kernel(AttnParams p) {
  constexpr int EPL = DH >= 32 ? DH / 32 : 1;
  constexpr int RPW = 8;
  extern __shared__ float smem[];
  float* Qs = smem;                // [64][DH]
  float* Ks = Qs + 64 * DH;        // [32][DH+1]
  float* Vs = Ks + 32 * (DH + 1);  // [32][DH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kvh = blockIdx.y;
  const int Tl = live_rows(p);
  const int GT = p.G * Tl;
  const int rho0 = blockIdx.z * 64;
  if (rho0 >= GT) return;
  const int cx = (int)blockIdx.x + p.x_base;
  const bool tree = cx == p.n_chunks;
  // load Q rows of this tile
  for (int i = tid; i < 64 * DH; i += 256) {
    const int rr = i / DH, d = i - rr * DH;
    const int rho = rho0 + rr;
    float v = 0.f;
    if (rho < GT) {
      const int t = rho / p.G, g = rho - t * p.G;
      v = to_f(((const QT*)p.q)[((int64_t)t * p.H + kvh * p.G + g) * DH + d]);
    }
    Qs[i] = v;
  }
  const KT* K;
  const KT* V;
  int k_begin, k_end;
  const KT *Kt, *Vt;
  const int ctx = resolve_ctx<DH, KT>(p, kvh, Kt, Vt);
  if (tree) {
    K = Kt;
    V = Vt;
    k_begin = 0;
    k_end = Tl;
  } else {
    K = (const KT*)p.k_cache + kvh * p.head_stride;
    V = (const KT*)p.v_cache + kvh * p.head_stride;
    k_begin = cx * p.chunk;
    k_end = min(ctx, k_begin + p.chunk);
  }
  float m[RPW], l[RPW], acc[RPW][EPL];
  const float* qrow[RPW];
  int trow[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[r][e] = 0.f;
    const int rr = warp + 8 * r;
    qrow[r] = Qs + rr * DH;
    trow[r] = (rho0 + rr < GT) ? (rho0 + rr) / p.G : -1;
  }
  __syncthreads();
  for (int kb = k_begin; kb < k_end; kb += 32) {
    const int nk = min(32, k_end - kb);
    if (tree || !ROT)
      stage_tile<DH, KT, false>(Ks, Vs, K, V, kb, nk, nullptr, nullptr, nullptr, tid, 256);
    else
      stage_tile<DH, KT, true>(Ks, Vs, K, V, kb, nk, p.ranks, p.cosT, p.sinT, tid, 256);
    __syncthreads();
    uint32_t vis[RPW];
    uint32_t valid = nk >= 32 ? 0xffffffffu : ((1u << nk) - 1u);
    if (ROT && !tree) valid = slot_valid_bits(p.ranks, kb, nk, lane);
#pragma unroll
    for (int r = 0; r < RPW; ++r)
      vis[r] = trow[r] < 0 ? 0u : (tree ? tree_vis(p.mask, p.mask_words, trow[r], kb, nk) : valid);
    tile_update<DH, RPW>(Ks, Vs, qrow, vis, m, l, acc, lane);
    __syncthreads();
  }
  // write partials
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    if (trow[r] < 0) continue;
    const int rho = rho0 + warp + 8 * r;
    const int t = trow[r], g = rho - t * p.G, head = kvh * p.G + g;
    const int64_t oi = ((int64_t)cx * p.T + t) * p.H + head;
    const float inv = l[r] > 0.f ? 1.f / l[r] : 0.f;
    if (DH >= 32 || lane < DH) {
#pragma unroll
      for (int e = 0; e < EPL; ++e) p.ws_o[oi * DH + lane * EPL + e] = acc[r][e] * inv;
    }
    if (lane == 0) p.ws_lse[oi] = l[r] > 0.f ? m[r] + __logf(l[r]) : -INFINITY;
  }
}

// Mode B (G*T <= 8 rows: draft / AR): 4 warps split the chunk's keys, each warp
// handles every row, then the warps' states are merged in fixed order.
template <int DH, typename QT, typename KT, bool ROT>
__global__ void __launch_bounds__(128) attn_keys_kernel(AttnParams p) {
  constexpr int EPL = DH >= 32 ? DH / 32 : 1;
  constexpr int RPW = 8, NW = 4;
  extern __shared__ float smem[];
  float* Qs = smem;                         // [8][DH]
  float* Wk = Qs + 8 * DH;                  // per warp: K [32][DH+1], V [32][DH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* Ks = Wk + warp * (32 * (DH + 1) + 32 * DH);
  float* Vs = Ks + 32 * (DH + 1);
  const int kvh = blockIdx.y;
  const int Tl = live_rows(p);
  const int GT = p.G * Tl;
  const int cx = (int)blockIdx.x + p.x_base;
  const bool tree = cx == p.n_chunks;
  for (int i = tid; i < 8 * DH; i += 128) {
    const int rr = i / DH, d = i - rr * DH;
    float v = 0.f;
    if (rr < GT) {
      const int t = rr / p.G, g = rr - t * p.G;
      v = to_f(((const QT*)p.q)[((int64_t)t * p.H + kvh * p.G + g) * DH + d]);
    }
    Qs[i] = v;
  }
  const KT* K;
  const KT* V;
  int k_begin, k_end;
  const KT *Kt, *Vt;
  const int ctx = resolve_ctx<DH, KT>(p, kvh, Kt, Vt);
  if (tree) {
    K = Kt;
    V = Vt;
    k_begin = 0;
    k_end = Tl;
  } else {
    K = (const KT*)p.k_cache + kvh * p.head_stride;
    V = (const KT*)p.v_cache + kvh * p.head_stride;
    k_begin = cx * p.chunk;
    k_end = min(ctx, k_begin + p.chunk);
  }
  float m[RPW], l[RPW], acc[RPW][EPL];
  const float* qrow[RPW];
  int trow[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[r][e] = 0.f;
    qrow[r] = Qs + r * DH;
    trow[r] = r < GT ? r / p.G : -1;
  }
  __syncthreads();
  for (int kb = k_begin + 32 * warp; kb < k_end; kb += 32 * NW) {
    const int nk = min(32, k_end - kb);
    if (tree || !ROT)
      stage_tile<DH, KT, false>(Ks, Vs, K, V, kb, nk, nullptr, nullptr, nullptr, lane, 32);
    else
      stage_tile<DH, KT, true>(Ks, Vs, K, V, kb, nk, p.ranks, p.cosT, p.sinT, lane, 32);
    __syncwarp();
    uint32_t vis[RPW];
    uint32_t valid = nk >= 32 ? 0xffffffffu : ((1u << nk) - 1u);
    if (ROT && !tree) valid = slot_valid_bits(p.ranks, kb, nk, lane);
#pragma unroll
    for (int r = 0; r < RPW; ++r)
      vis[r] = trow[r] < 0 ? 0u : (tree ? tree_vis(p.mask, p.mask_words, trow[r], kb, nk) : valid);
    tile_update<DH, RPW>(Ks, Vs, qrow, vis, m, l, acc, lane);
    __syncwarp();
  }
  __syncthreads();
  // cross-warp merge through shared memory (reuse the staging area)
  float* Sm = Wk;                // [NW][RPW] m
  float* Sl = Sm + NW * RPW;     // [NW][RPW] l
  float* So = Sl + NW * RPW;     // [NW][RPW][DH]
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      Sm[warp * RPW + r] = m[r];
      Sl[warp * RPW + r] = l[r];
    }
  }
  if (DH >= 32 || lane < DH) {
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int e = 0; e < EPL; ++e) So[(warp * RPW + r) * DH + lane * EPL + e] = acc[r][e];
  }
  __syncthreads();
  for (int i = tid; i < RPW * DH; i += 128) {
    const int r = i / DH, d = i - r * DH;
    if (r >= GT) continue;
    float M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, Sm[w * RPW + r]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < NW; ++w) {
        const float sc = __expf(Sm[w * RPW + r] - M);
        L += Sl[w * RPW + r] * sc;
        O += So[(w * RPW + r) * DH + d] * sc;
      }
    }
    const int t = r / p.G, g = r - t * p.G, head = kvh * p.G + g;
    const int64_t oi = ((int64_t)cx * p.T + t) * p.H + head;
    p.ws_o[oi * DH + d] = L > 0.f ? O / L : 0.f;
    if (d == 0) p.ws_lse[oi] = L > 0.f ? M + __logf(L) : -INFINITY;
  }
}

// merge chunk partials in ascending chunk order -> out [T][H][DH]. One CTA per
// (t, head) row: the split weights exp(lse_c - max) are computed once into
// shared memory, then every thread accumulates its dims with independent loads.
constexpr int MERGE_MAX = 1024;
template <int DH, typename OT>
__global__ void attn_merge_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_lse, int nsplit,
                                  int TH, int H, const int32_t* __restrict__ rows_dev, OT* __restrict__ out) {
  __shared__ float wsh[MERGE_MAX];
  __shared__ float red[32];
  const int row = blockIdx.x;  // t * H + head
  if (rows_dev && row / H >= *rows_dev) {  // padded row: defined zeros
    for (int d = threadIdx.x; d < DH; d += blockDim.x) out[(int64_t)row * DH + d] = from_f<OT>(0.f);
    return;
  }
  float lm = -INFINITY;
  for (int c = threadIdx.x; c < nsplit; c += blockDim.x) {
    const float v = ws_lse[(int64_t)c * TH + row];
    wsh[c] = v;
    lm = fmaxf(lm, v);
  }
  const float M = block_reduce(lm, red, [](float a, float b) { return fmaxf(a, b); });
  float ls = 0.f;
  for (int c = threadIdx.x; c < nsplit; c += blockDim.x) {
    const float w = wsh[c] == -INFINITY ? 0.f : __expf(wsh[c] - M);
    wsh[c] = w;
    ls += w;
  }
  const float L = block_reduce(ls, red, [](float a, float b) { return a + b; });  // syncs: wsh visible
  const float inv = L > 0.f ? 1.f / L : 0.f;
  for (int d = threadIdx.x; d < DH; d += blockDim.x) {
    float O0 = 0.f, O1 = 0.f, O2 = 0.f, O3 = 0.f;
    int c = 0;
    // zero-weight splits (empty chunks past a device-resident context) are
    // skipped: their partial slots are not written
    for (; c + 4 <= nsplit; c += 4) {
      if (wsh[c] != 0.f) O0 = fmaf(wsh[c], ws_o[((int64_t)c * TH + row) * DH + d], O0);
      if (wsh[c + 1] != 0.f) O1 = fmaf(wsh[c + 1], ws_o[((int64_t)(c + 1) * TH + row) * DH + d], O1);
      if (wsh[c + 2] != 0.f) O2 = fmaf(wsh[c + 2], ws_o[((int64_t)(c + 2) * TH + row) * DH + d], O2);
      if (wsh[c + 3] != 0.f) O3 = fmaf(wsh[c + 3], ws_o[((int64_t)(c + 3) * TH + row) * DH + d], O3);
    }
    for (; c < nsplit; ++c)
      if (wsh[c] != 0.f) O0 = fmaf(wsh[c], ws_o[((int64_t)c * TH + row) * DH + d], O0);
    out[(int64_t)row * DH + d] = from_f<OT>(((O0 + O1) + (O2 + O3)) * inv);
  }
}

template <typename T> __device__ __forceinline__ void store4(T* p, float a, float b, float c, float d);
template <> __device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <> __device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c, float d) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 v;
  v.x = *reinterpret_cast<const uint32_t*>(&lo);
  v.y = *reinterpret_cast<const uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = v;
}

// head_dim 128: one warp per (t, head) row, lane = 4 dims. Split weights
// exp(lse_c - max) are recomputed per lane from a broadcast lse load, so every
// split's partial is an independent float4 load (all in flight) and the merge is
// a single L2 round trip; splits are accumulated in ascending order.
#ifndef SD_MERGE_U
#define SD_MERGE_U 8
#endif
constexpr int MU = SD_MERGE_U;  // split partials in flight per warp

// four consecutive partial values: fp32 (CUDA-core splits) or fp16 (tcgen05 splits)
__device__ __forceinline__ float4 load4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 load4(const __half* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

template <typename OT, typename PT = float, int MK = 3>
__global__ void __launch_bounds__(256) merge128_kernel(const PT* __restrict__ ws_o, const float* __restrict__ ws_lse,
                                                       int nsplit, int TH, int H, const int32_t* __restrict__ rows_dev,
                                                       OT* __restrict__ out, int fused_max_rows = 0) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);  // t * H + head
  pdl_trigger();
  pdl_wait();  // the split partials are the predecessor's output
  // fused_max_rows > 0: the tcgen05 kernel merged in place because the live rows
  // fit one row group (live rows <= fused_max_rows); nothing left to do here
  if (fused_max_rows > 0 && rows_dev && *rows_dev <= fused_max_rows) return;
  if (row >= TH) return;
  OT* dst = out + (int64_t)row * 128 + 4 * lane;
  if (rows_dev && row / H >= *rows_dev) {  // padded row: defined zeros
    store4<OT>(dst, 0.f, 0.f, 0.f, 0.f);
    return;
  }
  // lse of split c lives in lane c % 32, register c / 32 (nsplit <= 32 * MK)
  float lv[MK], wv[MK];
#pragma unroll
  for (int k = 0; k < MK; ++k) {
    const int c = lane + 32 * k;
    lv[k] = c < nsplit ? ws_lse[(int64_t)c * TH + row] : -INFINITY;
  }
  float m = lv[0];
#pragma unroll
  for (int k = 1; k < MK; ++k) m = fmaxf(m, lv[k]);
  m = warp_max(m);
  float lsum = 0.f;
#pragma unroll
  for (int k = 0; k < MK; ++k) {
    wv[k] = lv[k] == -INFINITY ? 0.f : __expf(lv[k] - m);
    lsum += wv[k];
  }
  lsum = warp_sum(lsum);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const PT* base = ws_o + (int64_t)row * 128 + 4 * lane;
  // only splits that hold data (empty ones — past a device-resident context —
  // were never written), in ascending order, MU partial loads in flight
#pragma unroll
  for (int k = 0; k < MK; ++k) {
    unsigned live = __ballot_sync(0xffffffffu, lv[k] != -INFINITY);
    while (live) {
      int cs[MU];
      float ws4[MU];
      int n = 0;
#pragma unroll
      for (int u = 0; u < MU; ++u) {
        cs[u] = live ? __ffs(live) - 1 : 0;
        ws4[u] = __shfl_sync(0xffffffffu, wv[k], cs[u]);
        if (live) {
          live &= live - 1;
          ++n;
        } else {
          ws4[u] = 0.f;
        }
      }
      float4 o[MU];
#pragma unroll
      for (int u = 0; u < MU; ++u) o[u] = load4(base + (int64_t)(32 * k + cs[u]) * TH * 128);
#pragma unroll
      for (int u = 0; u < MU; ++u) {
        if (u < n) {
          acc.x = fmaf(ws4[u], o[u].x, acc.x);
          acc.y = fmaf(ws4[u], o[u].y, acc.y);
          acc.z = fmaf(ws4[u], o[u].z, acc.z);
          acc.w = fmaf(ws4[u], o[u].w, acc.w);
        }
      }
    }
  }
  const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
  store4<OT>(dst, acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
}

template <typename OT>
static void launch_merge(const float* ws_o, const float* ws_lse, int nsplit, int TH, int H, const int32_t* rows_dev,
                         OT* out, int dh, cudaStream_t st) {
  if (dh == 128 && nsplit <= 96)
    launch_pdl(merge128_kernel<OT>, dim3((TH + 7) / 8), dim3(256), 0, st, ws_o, ws_lse, nsplit, TH, H, rows_dev, out, 0);
  else
    attn_merge_kernel<128, OT><<<TH, 128, 0, st>>>(ws_o, ws_lse, nsplit, TH, H, rows_dev, out);
}

template <int DH, typename QT, typename KT, typename OT>
static int launch_attention(const AttnParams& p0, int src_kind, void* out, cudaStream_t st, bool tree_only) {
  AttnParams p = p0;
  const int GT = p.G * p.T;
  dim3 grid(tree_only ? 1 : p.n_chunks + 1, p.Hk, 1);
  p.x_base = tree_only ? p.n_chunks : 0;
  if (GT <= 8) {
    const size_t smem = (8 * DH + 4 * (32 * (DH + 1) + 32 * DH)) * sizeof(float);
    auto kern = src_kind ? attn_keys_kernel<DH, QT, KT, true> : attn_keys_kernel<DH, QT, KT, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 128, smem, st>>>(p);
  } else {
    grid.z = (GT + 63) / 64;
    const size_t smem = (64 * DH + 32 * (DH + 1) + 32 * DH) * sizeof(float);
    auto kern = src_kind ? attn_rows_kernel<DH, QT, KT, true> : attn_rows_kernel<DH, QT, KT, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, st>>>(p);
  }
  int rc = check_launch("sd_attention(partial)");
  if (rc) return rc;
  if (DH == 128)
    launch_merge<OT>(p.ws_o, p.ws_lse, p.n_chunks + 1, p.T * p.H, p.H, p.rows_dev, (OT*)out, DH, st);
  else
    attn_merge_kernel<DH, OT><<<p.T * p.H, DH >= 128 ? 128 : (DH < 32 ? 32 : DH), 0, st>>>(
        p.ws_o, p.ws_lse, p.n_chunks + 1, p.T * p.H, p.H, p.rows_dev, (OT*)out);
  return check_launch("sd_attention(merge)");
}

template <int DH>
static int dispatch_types(const AttnParams& p, int q_dtype, int kv_dtype, int out_dtype, int src_kind, void* out,
                          cudaStream_t st, bool tree_only = false) {
  typedef __nv_bfloat16 bf;
  if (q_dtype == SD_BF16 && kv_dtype == SD_BF16 && out_dtype == SD_BF16)
    return launch_attention<DH, bf, bf, bf>(p, src_kind, out, st, tree_only);
  if (q_dtype == SD_F32 && kv_dtype == SD_BF16 && out_dtype == SD_BF16)
    return launch_attention<DH, float, bf, bf>(p, src_kind, out, st, tree_only);
  if (q_dtype == SD_F32 && kv_dtype == SD_F32 && out_dtype == SD_F32)
    return launch_attention<DH, float, float, float>(p, src_kind, out, st, tree_only);
  set_error("sd_attention: unsupported dtype combination q=%d kv=%d out=%d", q_dtype, kv_dtype, out_dtype);
  return SD_EUNSUPPORTED;
}


// ------------------------------------------------------------------------
// Single-row decode attention (draft over the partial cache, AR decode over
// the full cache): T == 1, G <= 8 query heads per kv head. A CTA takes one
// 64-key chunk of one kv head; each of its 4 warps streams 16 keys with lanes
// over head_dim: the warp's ranks arrive in one coalesced load and are
// broadcast by shuffles, then all 8 keys of a batch issue their K / V / cos /
// sin loads (8-byte vectors) before any math, so a warp has one memory
// round trip per batch. RoPE at the slot's rank is applied on load
// (kvcache.py:158-165); dots are reduced with warp shuffles; online softmax
// per query head; the 4 warps merge through shared memory.
constexpr int DEC_CHUNK = 64;

template <typename KT> struct Vec4;  // 4 consecutive elements
template <> struct Vec4<__nv_bfloat16> {
  using T = uint2;
  __device__ static void unpack(const T& v, float* f) {
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&v.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v.y);
    f[0] = __low2float(a); f[1] = __high2float(a); f[2] = __low2float(b); f[3] = __high2float(b);
  }
};
template <> struct Vec4<float> {
  using T = float4;
  __device__ static void unpack(const T& v, float* f) { f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w; }
};

template <int DH, typename QT, typename KT, bool ROT, int GM>
__global__ void __launch_bounds__(128, (GM == 4 && sizeof(KT) == 2) ? 4 : 2) decode_attn_kernel(AttnParams p, int chunk) {
  static_assert(DH == 128, "decode kernel: lanes hold 4 consecutive elements");
  constexpr int NB = 8;  // keys per load batch
  using V4 = typename Vec4<KT>::T;
  __shared__ float Sm[4][GM], Sl[4][GM], So[4][GM][DH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kvh = blockIdx.y, G = p.G;
  const int cx = blockIdx.x;
  const bool tree = cx == p.n_chunks;
  const KT* K;
  const KT* V;
  int k_begin, k_end;
  const KT *Kt, *Vt;
  const int ctx = resolve_ctx<DH, KT>(p, kvh, Kt, Vt);
  if (tree) {
    K = Kt;
    V = Vt;
    k_begin = 0;
    k_end = 1;
  } else {
    K = (const KT*)p.k_cache + kvh * p.head_stride;
    V = (const KT*)p.v_cache + kvh * p.head_stride;
    k_begin = cx * chunk;
    k_end = min(ctx, k_begin + chunk);
  }
  const int per_warp = chunk / 4;
  const int w0 = k_begin + warp * per_warp, w1 = min(k_end, w0 + per_warp);
  // ranks of this warp's keys (<= 32 per warp)
  int my_rank = 0;
  if (ROT && !tree && w0 + lane < w1) my_rank = p.ranks[w0 + lane];
  float q[GM][4];
#pragma unroll
  for (int g = 0; g < GM; ++g) {
    if (g < G) {
      const QT* qp = (const QT*)p.q + (int64_t)(kvh * G + g) * DH + lane * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) q[g][e] = to_f(qp[e]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) q[g][e] = 0.f;
    }
  }
  float m[GM], l[GM], acc[GM][4];
#pragma unroll
  for (int g = 0; g < GM; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[g][e] = 0.f;
  }
  for (int kb = w0; kb < w1; kb += NB) {
    V4 kv[NB], vv[NB];
    float2 cs[NB][2];
    bool ok[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = kb + b;
      const int rk = __shfl_sync(0xffffffffu, my_rank, (k - w0) & 31);
      ok[b] = k < w1 && (!ROT || tree || rk >= 0);
      const int kk = k < w1 ? k : w0;  // in-bounds address for masked keys
      kv[b] = *reinterpret_cast<const V4*>(K + (int64_t)kk * DH + lane * 4);
      vv[b] = *reinterpret_cast<const V4*>(V + (int64_t)kk * DH + lane * 4);
      if (ROT && !tree) {
        const int64_t r = rk > 0 ? rk : 0;
        cs[b][0] = *reinterpret_cast<const float2*>(p.cosT + r * (DH / 2) + lane * 2);
        cs[b][1] = *reinterpret_cast<const float2*>(p.sinT + r * (DH / 2) + lane * 2);
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float kf[4], vf[4];
      Vec4<KT>::unpack(kv[b], kf);
      Vec4<KT>::unpack(vv[b], vf);
      if (ROT && !tree) {  // pairs (0,1) and (2,3) of this lane
        const float a0 = kf[0], b0 = kf[1], a1 = kf[2], b1 = kf[3];
        kf[0] = a0 * cs[b][0].x - b0 * cs[b][1].x;
        kf[1] = a0 * cs[b][1].x + b0 * cs[b][0].x;
        kf[2] = a1 * cs[b][0].y - b1 * cs[b][1].y;
        kf[3] = a1 * cs[b][1].y + b1 * cs[b][0].y;
      }
      float sg[GM];
#pragma unroll
      for (int g = 0; g < GM; ++g) {
        float s = q[g][0] * kf[0];
        s = fmaf(q[g][1], kf[1], s);
        s = fmaf(q[g][2], kf[2], s);
        s = fmaf(q[g][3], kf[3], s);
        sg[g] = s;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int g = 0; g < GM; ++g) sg[g] += __shfl_xor_sync(0xffffffffu, sg[g], o);
      if (!ok[b]) continue;  // warp-uniform
#pragma unroll
      for (int g = 0; g < GM; ++g) {
        if (g < G) {
          const float mn = fmaxf(m[g], sg[g]);
          const float corr = __expf(m[g] - mn), pw = __expf(sg[g] - mn);
          l[g] = l[g] * corr + pw;
          m[g] = mn;
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[g][e] = fmaf(acc[g][e], corr, pw * vf[e]);
        }
      }
    }
  }
#pragma unroll
  for (int g = 0; g < GM; ++g) {
    if (g < G) {
      if (lane == 0) {
        Sm[warp][g] = m[g];
        Sl[warp][g] = l[g];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) So[warp][g][lane * 4 + e] = acc[g][e];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * DH; i += 128) {
    const int g = i / DH, d = i - g * DH;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, Sm[w][g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float sc = __expf(Sm[w][g] - M);
        L += Sl[w][g] * sc;
        O += So[w][g][d] * sc;
      }
    }
    const int64_t oi = (int64_t)cx * p.H + kvh * G + g;  // T == 1
    p.ws_o[oi * DH + d] = L > 0.f ? O / L : 0.f;
    if (d == 0) p.ws_lse[oi] = L > 0.f ? M + __logf(L) : -INFINITY;
  }
}

static inline int dec_chunk_for(int ctx) {
  int c = (ctx + 255) / 256;
  c = (c + DEC_CHUNK - 1) / DEC_CHUNK * DEC_CHUNK;
  return c < DEC_CHUNK ? DEC_CHUNK : c;
}

template <int DH, typename QT, typename KT, typename OT>
static int launch_decode(AttnParams p, int src_kind, void* out, cudaStream_t st) {
  const int chunk = dec_chunk_for(p.ctx);
  p.n_chunks = p.ctx > 0 ? (p.ctx + chunk - 1) / chunk : 0;
  p.ws_lse = p.ws_o + (size_t)(p.n_chunks + 1) * p.H * DH;
  dim3 grid(p.n_chunks + 1, p.Hk);
  if (p.G <= 4) {
    if (src_kind)
      decode_attn_kernel<DH, QT, KT, true, 4><<<grid, 128, 0, st>>>(p, chunk);
    else
      decode_attn_kernel<DH, QT, KT, false, 4><<<grid, 128, 0, st>>>(p, chunk);
  } else {
    if (src_kind)
      decode_attn_kernel<DH, QT, KT, true, 8><<<grid, 128, 0, st>>>(p, chunk);
    else
      decode_attn_kernel<DH, QT, KT, false, 8><<<grid, 128, 0, st>>>(p, chunk);
  }
  int rc = check_launch("sd_attention(decode)");
  if (rc) return rc;
  launch_merge<OT>(p.ws_o, p.ws_lse, p.n_chunks + 1, p.H, p.H, p.rows_dev, (OT*)out, DH, st);
  return check_launch("sd_attention(decode merge)");
}

template <int DH>
static int dispatch_decode(const AttnParams& p, int q_dtype, int kv_dtype, int out_dtype, int src_kind, void* out,
                           cudaStream_t st) {
  typedef __nv_bfloat16 bf;
  if (q_dtype == SD_BF16 && kv_dtype == SD_BF16 && out_dtype == SD_BF16)
    return launch_decode<DH, bf, bf, bf>(p, src_kind, out, st);
  if (q_dtype == SD_F32 && kv_dtype == SD_F32 && out_dtype == SD_F32)
    return launch_decode<DH, float, float, float>(p, src_kind, out, st);
  set_error("sd_attention(decode): unsupported dtype combination");
  return SD_EUNSUPPORTED;
}

// ------------------------------------------------------------------------
// Draft attention over the partial cache (model.py:301-305, kvcache.py:158-165):
// one query row, G <= 8 query heads per kv head, K_raw rotated on load at the
// slot's rank, holes (rank < 0) skipped, the pending token's own row (k_tree /
// v_tree) attended by the last chunk. Grid (chunks of DR_CHUNK slots, kv head),
// 8 warps x 16 keys per CTA so every SM holds ~2 CTAs with all key loads of a
// warp in flight. Chunk partials are merged by the LAST CTA of each kv head to
// finish (arrival counter in the zeroed workspace head, reset after use), in
// fixed chunk order — one launch, deterministic, no separate merge kernel.
#ifndef SD_DR_KPW
#define SD_DR_KPW 16
#endif
constexpr int DR_KPW = SD_DR_KPW;  // keys per warp: one batch of loads in flight per warp
constexpr int DR_WARPS = 8, DR_CHUNK = DR_WARPS * DR_KPW, DR_MAX_CHUNKS = 96;

template <typename KT, int GM>
__global__ void __launch_bounds__(256, GM == 4 ? 2 : 1) draft_attn_kernel(AttnParams p, int* __restrict__ counters,
                                                            __nv_bfloat16* __restrict__ out) {
  using V4 = typename Vec4<KT>::T;
  constexpr int DH = 128, NB = 8;
  __shared__ float Sm[DR_WARPS][GM], Sl[DR_WARPS][GM], So[DR_WARPS][GM][DH];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kvh = blockIdx.y, G = p.G, nc = gridDim.x, cx = blockIdx.x;
  const KT* K = (const KT*)p.k_cache + kvh * p.head_stride;
  const KT* V = (const KT*)p.v_cache + kvh * p.head_stride;
  const int w0 = cx * DR_CHUNK + warp * DR_KPW, w1 = min(p.ctx, w0 + DR_KPW);
  pdl_trigger();
  // the partial cache (slots, ranks) is written only by launches that do not
  // trigger dependents early (admit / evict / gather), so the first batch of key
  // loads is issued before waiting on the kernel before (which writes q and the
  // pending row)
  int my_rank = -1;
  if (lane < DR_KPW && w0 + lane < w1) my_rank = p.ranks[w0 + lane];
  V4 kv[NB], vv[NB];
  float2 cs[NB][2];
  bool ok[NB];
  auto load_batch = [&](int b0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = w0 + b0 + b;
      const int rk = __shfl_sync(0xffffffffu, my_rank, b0 + b);
      ok[b] = k < w1 && rk >= 0;
      const int kk = ok[b] ? k : 0;  // in-bounds address for masked keys
      kv[b] = *reinterpret_cast<const V4*>(K + (int64_t)kk * DH + lane * 4);
      vv[b] = *reinterpret_cast<const V4*>(V + (int64_t)kk * DH + lane * 4);
      const int64_t r = rk > 0 ? rk : 0;
      cs[b][0] = *reinterpret_cast<const float2*>(p.cosT + r * (DH / 2) + lane * 2);
      cs[b][1] = *reinterpret_cast<const float2*>(p.sinT + r * (DH / 2) + lane * 2);
    }
  };
  load_batch(0);
  pdl_wait();  // q and the pending row come from the kernel before
  float q[GM][4];
#pragma unroll
  for (int g = 0; g < GM; ++g) {
#pragma unroll
    for (int e = 0; e < 4; ++e) q[g][e] = 0.f;
    if (g < G) {
      const KT* qp = (const KT*)p.q + (int64_t)(kvh * G + g) * DH + lane * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) q[g][e] = to_f(qp[e]);
    }
  }
  float m[GM], l[GM], acc[GM][4];
#pragma unroll
  for (int g = 0; g < GM; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[g][e] = 0.f;
  }
  auto update = [&](const float* kf, const float* vf) {
    float sg[GM];
#pragma unroll
    for (int g = 0; g < GM; ++g) sg[g] = fmaf(q[g][0], kf[0], fmaf(q[g][1], kf[1], fmaf(q[g][2], kf[2], q[g][3] * kf[3])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int g = 0; g < GM; ++g) sg[g] += __shfl_xor_sync(0xffffffffu, sg[g], o);
#pragma unroll
    for (int g = 0; g < GM; ++g) {
      if (g < G) {
        const float mn = fmaxf(m[g], sg[g]);
        const float corr = __expf(m[g] - mn), pw = __expf(sg[g] - mn);
        l[g] = l[g] * corr + pw;
        m[g] = mn;
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[g][e] = fmaf(acc[g][e], corr, pw * vf[e]);
      }
    }
  };
  // batches of 8 keys: every load of a batch issued before any math. The
  // KG x GM partial dots of a key group (32 values per lane) are summed across
  // the warp by a butterfly reduce-scatter (31 shuffles; lane j ends with the
  // full dot of key j / GM, head j % GM), then one online-softmax update per
  // head covers the whole group: one exp per lane instead of one per key & head.
  constexpr int KG = 32 / GM;  // keys per reduction group
  const int my_g = lane % GM, my_b = lane / GM;
#pragma unroll
  for (int b0 = 0; b0 < DR_KPW; b0 += NB) {
    if (b0 > 0) load_batch(b0);
#pragma unroll
    for (int g0 = 0; g0 < NB; g0 += KG) {
      float d[32];
#pragma unroll
      for (int b = 0; b < KG; ++b) {
        float kf[4];
        Vec4<KT>::unpack(kv[g0 + b], kf);
        const float a0 = kf[0], c0 = kf[1], a1 = kf[2], c1 = kf[3];  // pairs (0,1), (2,3) of this lane
        const float2 cc = cs[g0 + b][0], sn = cs[g0 + b][1];
        const float r0 = a0 * cc.x - c0 * sn.x, r1 = a0 * sn.x + c0 * cc.x;
        const float r2 = a1 * cc.y - c1 * sn.y, r3 = a1 * sn.y + c1 * cc.y;
#pragma unroll
        for (int g = 0; g < GM; ++g) d[b * GM + g] = fmaf(q[g][0], r0, fmaf(q[g][1], r1, fmaf(q[g][2], r2, q[g][3] * r3)));
      }
#pragma unroll
      for (int c = 16; c >= 1; c >>= 1) {  // reduce-scatter: keep the half named by lane bit c
        const bool up = lane & c;
#pragma unroll
        for (int i = 0; i < c; ++i) {
          const float send = up ? d[i] : d[i + c];
          const float keep = up ? d[i + c] : d[i];
          d[i] = keep + __shfl_xor_sync(0xffffffffu, send, c);
        }
      }
      bool okb = false;
#pragma unroll
      for (int b = 0; b < KG; ++b) okb = my_b == b ? ok[g0 + b] : okb;
      const float sc = okb && my_g < G ? d[0] : -INFINITY;
      float bm = sc;  // group max per head: lanes of equal lane % GM
#pragma unroll
      for (int o = GM; o < 32; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
      float mo = m[0];
#pragma unroll
      for (int g = 1; g < GM; ++g) mo = my_g == g ? m[g] : mo;
      const float mn = fmaxf(mo, bm);
      const float pw = sc == -INFINITY ? 0.f : __expf(sc - mn);
      float ps = pw;
#pragma unroll
      for (int o = GM; o < 32; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      float corr[GM];
#pragma unroll
      for (int g = 0; g < GM; ++g) {
        const float mg = __shfl_sync(0xffffffffu, mn, g);
        const float sg = __shfl_sync(0xffffffffu, ps, g);
        corr[g] = m[g] == -INFINITY ? 0.f : __expf(m[g] - mg);
        l[g] = l[g] * corr[g] + sg;
        m[g] = mg;
      }
      float vf[KG][4];
#pragma unroll
      for (int b = 0; b < KG; ++b) Vec4<KT>::unpack(vv[g0 + b], vf[b]);
#pragma unroll
      for (int g = 0; g < GM; ++g) {
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[g][e] *= corr[g];
#pragma unroll
        for (int b = 0; b < KG; ++b) {
          const float pb = __shfl_sync(0xffffffffu, pw, b * GM + g);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[g][e] = fmaf(pb, vf[b][e], acc[g][e]);
        }
      }
    }
  }
  if (cx == nc - 1 && warp == DR_WARPS - 1) {  // the pending token's own row (always visible)
    const KT* Kt = (const KT*)p.k_tree + kvh * p.tree_head_stride;
    const KT* Vt = (const KT*)p.v_tree + kvh * p.tree_head_stride;
    float kf[4], vf[4];
    Vec4<KT>::unpack(*reinterpret_cast<const V4*>(Kt + lane * 4), kf);
    Vec4<KT>::unpack(*reinterpret_cast<const V4*>(Vt + lane * 4), vf);
    update(kf, vf);
  }
  // ---- CTA combine of the 8 warps' states -> chunk partial ----
#pragma unroll
  for (int g = 0; g < GM; ++g) {
    if (g < G) {
      if (lane == 0) {
        Sm[warp][g] = m[g];
        Sl[warp][g] = l[g];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) So[warp][g][lane * 4 + e] = acc[g][e];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * DH; i += 256) {
    const int g = i / DH, d = i - g * DH;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < DR_WARPS; ++w) M = fmaxf(M, Sm[w][g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < DR_WARPS; ++w) {
        const float sc = __expf(Sm[w][g] - M);
        L += Sl[w][g] * sc;
        O += So[w][g][d] * sc;
      }
    }
    const int64_t oi = (int64_t)cx * p.H + kvh * G + g;
    p.ws_o[oi * DH + d] = L > 0.f ? O / L : 0.f;
    if (d == 0) p.ws_lse[oi] = L > 0.f ? M + __logf(L) : -INFINITY;
  }
  // ---- the last CTA of this kv head merges the chunks in order ----
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&counters[kvh], 1) == nc - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // every warp takes (head row, part of the chunk range); parts summed in order
  const int parts = DR_WARPS / G, gi = warp % G, part = warp / G;
  const bool active = part < parts;
  const int row = kvh * G + gi;  // T == 1: row = head
  float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float L = 0.f;
  if (active) {
    float lv[3], wv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int c = lane + 32 * k;
      lv[k] = c < nc ? __ldcg(p.ws_lse + (int64_t)c * p.H + row) : -INFINITY;
    }
    const float M = warp_max(fmaxf(lv[0], fmaxf(lv[1], lv[2])));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      wv[k] = lv[k] == -INFINITY ? 0.f : __expf(lv[k] - M);
      L += wv[k];
    }
    L = warp_sum(L);
    const int ca = part * nc / parts, cb = (part + 1) * nc / parts;
#pragma unroll 8
    for (int c = ca; c < cb; ++c) {
      const float w = __shfl_sync(0xffffffffu, c < 32 ? wv[0] : (c < 64 ? wv[1] : wv[2]), c & 31);
      const float4 o = __ldcg(reinterpret_cast<const float4*>(p.ws_o + ((int64_t)c * p.H + row) * DH) + lane);
      if (w != 0.f) {
        o4.x = fmaf(w, o.x, o4.x);
        o4.y = fmaf(w, o.y, o4.y);
        o4.z = fmaf(w, o.z, o4.z);
        o4.w = fmaf(w, o.w, o4.w);
      }
    }
    *reinterpret_cast<float4*>(&So[part][gi][lane * 4]) = o4;
  }
  __syncthreads();
  if (warp < G) {
    float4 t = *reinterpret_cast<const float4*>(&So[0][gi][lane * 4]);
    for (int q = 1; q < parts; ++q) {
      const float4 u = *reinterpret_cast<const float4*>(&So[q][gi][lane * 4]);
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    store4<__nv_bfloat16>(out + (int64_t)row * DH + lane * 4, t.x * inv, t.y * inv, t.z * inv, t.w * inv);
  }
  if (tid == 0) counters[kvh] = 0;  // ready for the next launch / graph replay
}

int tc_make_kv_tmap(const void* base, int L, int Hk, int cap, int dh, void* out, int box_rows);
int launch_draft_mma(const void* tmap_k, const void* tmap_v, const void* q, int H, int Hk, int kv_heads_total,
                     int layer, int hi, const int32_t* ranks, const void* k_self, const void* v_self,
                     int64_t self_stride, float* ws_o, int* counters, void* out, cudaStream_t st);
int tc_set_trace(void* dev_ptr, int force_chunks);
int tc_split_target(int kv_heads_total);
int tc_grid_chunks(int ctx_bound, int n_target);
int launch_verify_tc(const void* tmap_k, const void* tmap_v, const void* q, int T, int H, int Hk, int layer, int ctx,
                     const int32_t* rows_dev, const int32_t* ctx_dev, const uint32_t* mask, int mask_words,
                     __half* ws_o, float* ws_lse, int n_chunks, int n_target, void* merge_out, int* merge_counters,
                     cudaStream_t st);
template <int DH, typename OT>
__global__ void attn_merge_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_lse, int nsplit,
                                  int TH, int H, const int32_t* __restrict__ rows_dev, OT* __restrict__ out);

// tensor-core path: all 16-bit, head_dim 128, full-cache source, >= one 64-key tile
static bool use_tc(const void* tk, const void* tv, int q_dtype, int kv_dtype, int out_dtype, int dh, int src_kind,
                   int ctx) {
  return tk && tv && q_dtype == SD_BF16 && kv_dtype == SD_BF16 && out_dtype == SD_BF16 && dh == 128 &&
         src_kind == 0 && ctx >= 64;
}

}  // namespace sd

using namespace sd;

extern "C" {

size_t sd_attention_workspace_bytes(int T, int H, int dh, int ctx) {
  int nc = n_chunks_for(ctx);
  if (nc < 148) nc = 148;  // tensor-core chunking may use up to 148 chunks
  if (T == 1 && ctx > 0) {
    const int dc = (ctx + dec_chunk_for(ctx) - 1) / dec_chunk_for(ctx);
    if (dc > nc) nc = dc;
  }
  return SD_ATTN_WS_HEAD + ((size_t)nc + 1) * (size_t)T * H * (dh + 1) * sizeof(float);
}

int sd_debug_tc_trace(void* trace_dev, int force_chunks) { return tc_set_trace(trace_dev, force_chunks); }

int sd_make_kv_tmap(const void* base, int L, int Hk, int cap, int dh, void* tmap_out_host) {
  SD_REQUIRE(base && tmap_out_host && dh == 128 && L > 0 && Hk > 0 && cap > 0, "sd_make_kv_tmap: args");
  return tc_make_kv_tmap(base, L, Hk, cap, dh, tmap_out_host, 128);
}

int sd_make_slot_tmap(const void* base, int L, int Hk, int cap, int dh, void* tmap_out_host) {
  SD_REQUIRE(base && tmap_out_host && dh == 128 && L > 0 && Hk > 0 && cap > 0, "sd_make_slot_tmap: args");
  return tc_make_kv_tmap(base, L, Hk, cap, dh, tmap_out_host, 64);
}

int sd_attention(const void* q, int q_dtype, int T, int H, int Hk, int dh, int src_kind, const void* k_cache,
                 const void* v_cache, int kv_dtype, int64_t head_stride, int ctx, const int32_t* ranks,
                 const float* rope_cos, const float* rope_sin, const void* k_tree, const void* v_tree,
                 int64_t tree_head_stride, const uint32_t* mask_bits, int mask_words, const int32_t* rows_dev,
                 const int32_t* ctx_dev, const void* tmap_k_host, const void* tmap_v_host, int layer,
                 int kv_heads_total, void* out, int out_dtype, void* workspace, size_t workspace_bytes,
                 sd_stream_t stream) {
  SD_REQUIRE(T > 0 && T <= SD_TREE_MAX_ROWS, "sd_attention: T=%d out of range", T);
  SD_REQUIRE(H > 0 && Hk > 0 && H % Hk == 0, "sd_attention: heads");
  SD_REQUIRE(ctx >= 0, "sd_attention: ctx");
  SD_REQUIRE(!mask_bits || mask_words * 32 >= T, "sd_attention: mask words");
  SD_REQUIRE(src_kind == 0 || (ranks && rope_cos && rope_sin), "sd_attention: partial source needs ranks/rope");
  SD_REQUIRE(!ctx_dev || (src_kind == 0 && tree_head_stride == head_stride),
             "sd_attention: ctx_dev needs the full-cache source with the tree rows in the cache arrays");
  SD_REQUIRE(workspace_bytes >= sd_attention_workspace_bytes(T, H, dh, ctx), "sd_attention: workspace too small");
  SD_REQUIRE(ctx <= 256 * 8192, "sd_attention: ctx too large for the merge split limit");
  AttnParams p;
  p.q = q;
  p.T = T;
  p.H = H;
  p.Hk = Hk;
  p.G = H / Hk;
  p.k_cache = k_cache;
  p.v_cache = v_cache;
  p.head_stride = head_stride;
  p.ctx = ctx;
  p.ranks = ranks;
  p.cosT = rope_cos;
  p.sinT = rope_sin;
  p.k_tree = k_tree;
  p.v_tree = v_tree;
  p.tree_head_stride = tree_head_stride;
  p.mask = mask_bits;
  p.mask_words = mask_words;
  p.chunk = chunk_len_for(ctx);
  p.n_chunks = n_chunks_for(ctx);
  int* counters = (int*)workspace;  // SD_ATTN_WS_HEAD bytes, zero between calls
  p.ws_o = (float*)((char*)workspace + SD_ATTN_WS_HEAD);
  p.ws_lse = p.ws_o + (size_t)(p.n_chunks + 1) * T * H * dh;
  p.rows_dev = rows_dev;
  p.ctx_dev = ctx_dev;
  p.x_base = 0;
  auto st = as_stream(stream);
  if (use_tc(tmap_k_host, tmap_v_host, q_dtype, kv_dtype, out_dtype, dh, src_kind, ctx)) {
    // cache chunks + the masked tree rows on tcgen05, then the chunk merge
    // ctx (host) or its upper bound (ctx_dev) sizes the grid; the splits
    // themselves are resolved in the kernel from the live context
    const int n_target = tc_split_target(kv_heads_total > 0 ? kv_heads_total : Hk);
    const int nc = tc_grid_chunks(ctx, n_target);
    // split partials in fp16 (normalised o / l: |values| <= max |v|; 2^-11
    // relative, below the bf16 output's own rounding), lse in fp32
    __half* ws_oh = reinterpret_cast<__half*>(p.ws_o);
    float* ws_lse = reinterpret_cast<float*>(ws_oh + (size_t)nc * T * H * dh);
    // the split merge fused into the kernel when the whole grid is co-resident
    // (one row group, one CTA per SM): CTAs of a kv head wait for each other
    static int n_sm = 0;
    if (!n_sm) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    // (the kernel checks the live rows on device: a padded launch whose live rows
    // need two row groups merges in merge128_kernel below instead)
    // off by default: measured no faster alone (52.8 vs 52.2 us at ctx 54K: the CTAs of a head wait for
    // its slowest chunk either way) and 0.19 ms slower per cfg3 step; SD_TC_FUSED_MERGE=1 turns it on
    static const bool fuse_env = getenv("SD_TC_FUSED_MERGE") && atoi(getenv("SD_TC_FUSED_MERGE")) != 0;
    const int max_rows_fused = 256 / (H / Hk);  // live rows whose G * rows fit one row group (tc ROWS)
    const bool fused = fuse_env && nc * Hk <= n_sm && 2 * Hk * (int)sizeof(int) <= 2048 && max_rows_fused > 0;
    int rc = launch_verify_tc(tmap_k_host, tmap_v_host, q, T, H, Hk, layer, ctx, rows_dev, ctx_dev, mask_bits,
                              mask_words, ws_oh, ws_lse, nc, n_target, fused ? out : nullptr,
                              fused ? counters + 512 : nullptr, st);
    if (rc) return rc;
    if (fused && T <= max_rows_fused) return SD_OK;  // every launch merges in the kernel
    if (nc > 160) {
      set_error("sd_attention(tc): %d splits > 160", nc);
      return SD_EINVAL;
    }
#ifndef SD_TC_NO_MERGE  // debug-only timing builds (tools/gpu_nomerge.sh): the split merge left out
    launch_pdl(nc <= 96 ? merge128_kernel<__nv_bfloat16, __half, 3> : merge128_kernel<__nv_bfloat16, __half, 5>, dim3((T * H + 7) / 8), dim3(256), 0, st, (const __half*)ws_oh,
               (const float*)ws_lse, nc, T * H, H, rows_dev, (__nv_bfloat16*)out, fused ? max_rows_fused : 0);
#endif
    return check_launch("sd_attention(tc merge)");
  }
  if (T == 1 && src_kind == 1 && dh == 128 && p.G <= 16 && !rows_dev && !ctx_dev && tmap_k_host && tmap_v_host &&
      q_dtype == SD_BF16 && kv_dtype == SD_BF16 && out_dtype == SD_BF16 && Hk * sizeof(int) <= SD_ATTN_WS_HEAD) {
    // draft attention on the warp-level tensor path: TMA-staged slots, rank-RoPE in
    // registers, split merge + pending row fused (last CTA per kv head)
    return launch_draft_mma(tmap_k_host, tmap_v_host, q, H, Hk, kv_heads_total, layer, ctx, ranks, k_tree, v_tree,
                            tree_head_stride, p.ws_o, counters, out, st);
  }
  if (T == 1 && src_kind == 1 && dh == 128 && p.G <= 8 && !rows_dev && q_dtype == kv_dtype &&
      out_dtype == SD_BF16 && kv_dtype == SD_BF16 && (ctx + DR_CHUNK - 1) / DR_CHUNK <= DR_MAX_CHUNKS &&
      Hk * sizeof(int) <= SD_ATTN_WS_HEAD) {
    // draft attention: rank-rotated partial cache, merge fused (last CTA per kv head)
    const int nc = ctx > 0 ? (ctx + DR_CHUNK - 1) / DR_CHUNK : 1;
    p.ws_lse = p.ws_o + (size_t)nc * H * dh;
    dim3 grid(nc, Hk);
    if (p.G <= 4)
      launch_pdl(draft_attn_kernel<__nv_bfloat16, 4>, grid, dim3(256), 0, st, p, counters, (__nv_bfloat16*)out);
    else
      launch_pdl(draft_attn_kernel<__nv_bfloat16, 8>, grid, dim3(256), 0, st, p, counters, (__nv_bfloat16*)out);
    return check_launch("sd_attention(draft)");
  }
  if (T == 1 && p.G <= 8 && dh == 128 && !rows_dev && !ctx_dev) {
    // single-row decode (draft / AR): latency-tolerant streaming kernel
    return dispatch_decode<128>(p, q_dtype, kv_dtype, out_dtype, src_kind, out, st);
  }
  switch (dh) {
    case 8: return dispatch_types<8>(p, q_dtype, kv_dtype, out_dtype, src_kind, out, st);
    case 16: return dispatch_types<16>(p, q_dtype, kv_dtype, out_dtype, src_kind, out, st);
    case 32: return dispatch_types<32>(p, q_dtype, kv_dtype, out_dtype, src_kind, out, st);
    case 64: return dispatch_types<64>(p, q_dtype, kv_dtype, out_dtype, src_kind, out, st);
    case 128: return dispatch_types<128>(p, q_dtype, kv_dtype, out_dtype, src_kind, out, st);
    default: set_error("sd_attention: head_dim %d unsupported", dh); return SD_EUNSUPPORTED;
  }
}

}  // extern "C"
