// Draft attention over the rank-rotated partial cache (reference model.py:301-305
// causal branch with one query row; keys rotated at their rank 0..m-1 in the
// draft view, kvcache.py:158-165, 227-240; the pending token's own row at rank m).
//
// One CTA = (slot split, kv head); one producer warp + 8 consumer warps.
//  * The producer streams the split's K_raw / V slots with TMA (64-slot stages,
//    128-byte swizzled boxes, 6-deep ring): every byte of the split is requested
//    at kernel start, before the dependency wait (the partial cache and its
//    ranks are written by ordinary launches, never by a programmatic-dependent
//    predecessor).
//  * Each consumer warp takes 16-slot tiles. S^T[heads, slots] = q . K_rot^T
//    runs on the warp-level tensor path (mma.m16n8k16, bf16 in, fp32 out) with
//    the query heads as the M rows; the K fragments come out of shared memory
//    by ldmatrix and are rotated in registers at the slot's rank before the
//    MMA (one RoPE pair per bf16x2 fragment register). cos / sin come from the
//    MUFU after an exact range reduction of rank * inv_freq (double-float
//    inv_freq / 2pi, fma remainder), so no table is read per slot.
//  * Online softmax in base 2 on the accumulator fragments (a quad of lanes
//    owns one head row), P repacked in registers as the A operand of
//    O[heads, dh] += P V (V fragments by ldmatrix.trans).
//  * The 8 warps' states merge in shared memory into the split's partial
//    (o / l, lse); the last CTA of each kv head to finish (arrival counter)
//    merges the splits in fixed order together with the pending row.
// Split count depends on the slot range and the model's total kv heads only,
// so a kv head's output is bitwise the same at any shard count.
#include <math.h>

#include "tc_common.cuh"

namespace sd {
namespace dr {

using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::pack_bf16;
using tc::smem_u32;

// debug-only pipeline experiments (tools/draft_bench.py): 1 = no rank-RoPE math, 2 = no split merge,
// 3 = no CTA combine / merge, 4 = no tile math (stream + barriers only)
#ifndef SD_DR_EXP
#define SD_DR_EXP 0
#endif
constexpr int DH = 128;
constexpr int STAGE_KEYS = 64;               // slots per TMA stage
constexpr int TILE = 16;                     // slots per MMA tile (two n-tiles of 8)
constexpr int TPS = STAGE_KEYS / TILE;       // tiles per stage
constexpr int NCW = 8;                       // consumer warps
constexpr int NST = 4;                       // ring depth
constexpr int THREADS = 32 * (NCW + 1);
constexpr int HALF_BYTES = STAGE_KEYS * 128; // one dh half of a stage (64 slots x 128 B)
constexpr int STAGE_BYTES = 4 * HALF_BYTES;  // K lo, K hi, V lo, V hi
constexpr int MAX_KPS = 2048;                // slots per split (ranks staged in shared memory)
#ifndef SD_DR_MIN_KPS
#define SD_DR_MIN_KPS 128
#endif
constexpr int MIN_KPS = SD_DR_MIN_KPS;                 // slots per split at least (merge cost vs parallelism)
constexpr int OFF_RANK = NST * STAGE_BYTES;
constexpr int OFF_FREQ = OFF_RANK + MAX_KPS * 4;
constexpr int OFF_BAR = OFF_FREQ + 64 * 8;
constexpr int SMEM_BYTES = OFF_BAR + 2 * NST * 8 + 16;
constexpr int SMEM_ALLOC = SMEM_BYTES + 1024;
constexpr float LOG2E = 1.4426950408889634f;
static_assert(NCW * 16 * DH * 4 + 2 * NCW * 16 * 4 <= NST * STAGE_BYTES, "combine scratch fits the ring");
static_assert(SMEM_ALLOC <= 227 * 1024, "shared memory");

struct Params {
  const __nv_bfloat16* q;       // [H][128], rotated at rank m and scaled by 1/sqrt(dh)
  const int32_t* ranks;         // [hi] ranks of this layer's slots (< 0: hole)
  const __nv_bfloat16* k_self;  // pending row, [Hk] x self_stride
  const __nv_bfloat16* v_self;
  int64_t self_stride;
  int H, G, layer, hi, kps, nsplit;
  float* ws_o;  // [nsplit][H][128]
  float* ws_lse;  // [nsplit][H] (base 2)
  int* counters;  // [Hk], zero between launches
  __nv_bfloat16* out;  // [H][128]
  float fh[64], fl[64];  // inv_freq_i / 2pi as a double-float
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// cos / sin of rank * inv_freq: the product is reduced modulo one turn exactly
// (fma remainder of the fp32 product + the low word of inv_freq / 2pi), so the
// MUFU sees |angle| <= pi and the error stays ~1e-6 absolute at any rank < 2^24
__device__ __forceinline__ void rope_cs(int r, float2 f, float& c, float& s) {
  const float rf = (float)r;
  const float ph = rf * f.x;
  const float pe = fmaf(rf, f.x, -ph);
  const float x = (ph - rintf(ph)) + fmaf(rf, f.y, pe);
  __sincosf(x * 6.283185307179586f, &s, &c);
}
// rotate one RoPE pair held as bf16x2 (low half = even element)
__device__ __forceinline__ uint32_t rot_pair(uint32_t w, float c, float s) {
  const float x1 = __uint_as_float(w << 16), x2 = __uint_as_float(w & 0xffff0000u);
  return pack_bf16(x1 * c - x2 * s, x1 * s + x2 * c);
}
__device__ __forceinline__ uint32_t sw_addr(uint32_t base, int row, int chunk) {
  // 16-byte chunk `chunk` (0..15 over the 128 dh) of slot row `row` in a stage
  return base + (chunk >> 3) * HALF_BYTES + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

template <bool BIG>  // BIG: G > 8, query rows 8..15 of the MMA tile are live
__global__ void __launch_bounds__(THREADS, 1)
    draft_mma_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + OFF_BAR);
  uint64_t* empty = full + NST;
  int* s_rank = (int*)(smem + OFF_RANK);
  float2* s_freq = (float2*)(smem + OFF_FREQ);
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kvh = blockIdx.y, split = blockIdx.x;
  const int k_begin = split * p.kps;
  const int n_keys = max(0, min(p.hi, k_begin + p.kps) - k_begin);
  const int n_tiles = (n_keys + TILE - 1) / TILE;
  const int n_stages = (n_keys + STAGE_KEYS - 1) / STAGE_KEYS;
  pdl_trigger();
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TPS);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ================= producer: every stage of the split, ring-recycled =================
    if (lane == 0) {
      tc::tma_prefetch(&tmk);
      tc::tma_prefetch(&tmv);
      for (int s = 0; s < n_stages; ++s) {
        const int slot = s % NST;
        if (s >= NST) mbar_wait(&empty[slot], ((s / NST) + 1) & 1);
        uint8_t* d = smem + slot * STAGE_BYTES;
        const int key0 = k_begin + s * STAGE_KEYS;
        mbar_expect_tx(&full[slot], STAGE_BYTES);
        tc::tma_load_4d(d, &tmk, &full[slot], 0, key0, kvh, p.layer);
        tc::tma_load_4d(d + HALF_BYTES, &tmk, &full[slot], 64, key0, kvh, p.layer);
        tc::tma_load_4d(d + 2 * HALF_BYTES, &tmv, &full[slot], 0, key0, kvh, p.layer);
        tc::tma_load_4d(d + 3 * HALF_BYTES, &tmv, &full[slot], 64, key0, kvh, p.layer);
      }
    }
    pdl_wait();
  } else {
    // ================= consumers =================
    for (int i = tid; i < n_keys; i += NCW * 32) s_rank[i] = p.ranks[k_begin + i];
    if (tid < 64) s_freq[tid] = make_float2(p.fh[tid], p.fl[tid]);
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
    const int g = lane >> 2, qd = lane & 3;
    pdl_wait();  // q comes from the RoPE staging launched just before
    uint32_t qa0[8], qa1[8], qa2[8], qa3[8];
    {
      const uint32_t* q32 = reinterpret_cast<const uint32_t*>(p.q);
      const int64_t rowA = (int64_t)(kvh * p.G + g) * (DH / 2), rowB = rowA + 8 * (DH / 2);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qa0[ks] = g < p.G ? q32[rowA + 8 * ks + qd] : 0u;
        qa2[ks] = g < p.G ? q32[rowA + 8 * ks + 4 + qd] : 0u;
        qa1[ks] = (BIG && g + 8 < p.G) ? q32[rowB + 8 * ks + qd] : 0u;
        qa3[ks] = (BIG && g + 8 < p.G) ? q32[rowB + 8 * ks + 4 + qd] : 0u;
      }
    }
    float o[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m0 = -INFINITY, l0 = 0.f, m1 = -INFINITY, l1 = 0.f;
    const int mi = lane >> 3, rr = lane & 7;
    for (int i = warp; i < n_tiles; i += NCW) {
      const int s = i / TPS, slot = s % NST;
      mbar_wait(&full[slot], (s / NST) & 1);
#if SD_DR_EXP == 4
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      continue;
#endif
      const uint32_t kbase = smem_u32(smem + slot * STAGE_BYTES);
      const uint32_t vbase = kbase + 2 * HALF_BYTES;
      const int r0 = (i % TPS) * TILE;  // tile's first row in the stage
      const int kl = i * TILE;          // tile's first slot in the split
      const int rA = kl + g < n_keys ? s_rank[kl + g] : -1;
      const int rB = kl + g + 8 < n_keys ? s_rank[kl + g + 8] : -1;
      // ---- S^T = q K_rot^T: rows = query heads, columns = the tile's 16 slots ----
      float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
      const int krow = r0 + rr + ((mi >> 1) << 3);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sw_addr(kbase, krow, 2 * ks + (mi & 1)), b0, b1, b2, b3);
        const float2 f0 = s_freq[8 * ks + qd], f1 = s_freq[8 * ks + 4 + qd];
#if SD_DR_EXP != 1
        {
          float c, sn;
          rope_cs(rA, f0, c, sn);
          b0 = rot_pair(b0, c, sn);
          rope_cs(rA, f1, c, sn);
          b1 = rot_pair(b1, c, sn);
          rope_cs(rB, f0, c, sn);
          b2 = rot_pair(b2, c, sn);
          rope_cs(rB, f1, c, sn);
          b3 = rot_pair(b3, c, sn);
        }
#else
        (void)f0;
        (void)f1;
#endif
        mma16816(sa, qa0[ks], qa1[ks], qa2[ks], qa3[ks], b0, b1);
        mma16816(sb, qa0[ks], qa1[ks], qa2[ks], qa3[ks], b2, b3);
      }
      // ---- online softmax (base 2) on the fragments: quad (lane >> 2) = head row ----
      bool ok[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = kl + 2 * qd + (e & 1) + 8 * (e >> 1);
        ok[e] = k < n_keys && s_rank[k] >= 0;
      }
      uint32_t pa0, pa1 = 0u, pa2, pa3 = 0u;
      {
        const float x0 = ok[0] ? sa[0] * LOG2E : -INFINITY, x1 = ok[1] ? sa[1] * LOG2E : -INFINITY;
        const float x2 = ok[2] ? sb[0] * LOG2E : -INFINITY, x3 = ok[3] ? sb[1] * LOG2E : -INFINITY;
        float mx = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(m0, mx);
        const float base = mn == -INFINITY ? 0.f : mn;
        const float corr = tc::ex2(m0 - base);  // m0 = -inf -> 0
        const float p0 = tc::ex2(x0 - base), p1 = tc::ex2(x1 - base), p2 = tc::ex2(x2 - base),
                    p3 = tc::ex2(x3 - base);
        l0 = l0 * corr + ((p0 + p1) + (p2 + p3));
        m0 = mn;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          o[nt][0] *= corr;
          o[nt][1] *= corr;
        }
        pa0 = pack_bf16(p0, p1);
        pa2 = pack_bf16(p2, p3);
      }
      if (BIG) {
        const float x0 = ok[0] ? sa[2] * LOG2E : -INFINITY, x1 = ok[1] ? sa[3] * LOG2E : -INFINITY;
        const float x2 = ok[2] ? sb[2] * LOG2E : -INFINITY, x3 = ok[3] ? sb[3] * LOG2E : -INFINITY;
        float mx = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(m1, mx);
        const float base = mn == -INFINITY ? 0.f : mn;
        const float corr = tc::ex2(m1 - base);
        const float p0 = tc::ex2(x0 - base), p1 = tc::ex2(x1 - base), p2 = tc::ex2(x2 - base),
                    p3 = tc::ex2(x3 - base);
        l1 = l1 * corr + ((p0 + p1) + (p2 + p3));
        m1 = mn;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          o[nt][2] *= corr;
          o[nt][3] *= corr;
        }
        pa1 = pack_bf16(p0, p1);
        pa3 = pack_bf16(p2, p3);
      }
      // ---- O[heads, dh] += P V ----
      const int vrow = r0 + rr + ((mi & 1) << 3);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(sw_addr(vbase, vrow, 2 * j + (mi >> 1)), v0, v1, v2, v3);
        mma16816(o[2 * j], pa0, pa1, pa2, pa3, v0, v1);
        mma16816(o[2 * j + 1], pa0, pa1, pa2, pa3, v2, v3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
#if SD_DR_EXP == 3
    if (tid == 0) p.out[kvh] = __float2bfloat16(l0 + o[0][0]);
    return;
#endif
    // ---- the 8 warps' states -> this split's partial (o / l, lse), ring reused as scratch ----
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");  // every tile consumed: the ring is free
    float* So = reinterpret_cast<float*>(smem);                    // [NCW][16][DH]
    float* Sm = So + NCW * 16 * DH;                                 // [NCW][16]
    float* Sl = Sm + NCW * 16;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      *reinterpret_cast<float2*>(&So[(warp * 16 + g) * DH + nt * 8 + 2 * qd]) = make_float2(o[nt][0], o[nt][1]);
      if (BIG)
        *reinterpret_cast<float2*>(&So[(warp * 16 + g + 8) * DH + nt * 8 + 2 * qd]) =
            make_float2(o[nt][2], o[nt][3]);
    }
    if (qd == 0) {
      Sm[warp * 16 + g] = m0;
      Sl[warp * 16 + g] = l0;
      Sm[warp * 16 + g + 8] = m1;
      Sl[warp * 16 + g + 8] = l1;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
    for (int e = tid; e < p.G * DH; e += NCW * 32) {
      const int row = e / DH, d = e - row * DH;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NCW; ++w) M = fmaxf(M, Sm[w * 16 + row]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < NCW; ++w) {
          const float sc = tc::ex2(Sm[w * 16 + row] - M);
          L += Sl[w * 16 + row] * sc;
          O += So[(w * 16 + row) * DH + d] * sc;
        }
      }
      const int64_t oi = (int64_t)split * p.H + kvh * p.G + row;
      p.ws_o[oi * DH + d] = L > 0.f ? O / L : 0.f;
      if (d == 0) p.ws_lse[oi] = L > 0.f ? M + __log2f(L) : -INFINITY;
    }
  }
  // ================= the last CTA of this kv head merges the splits + the pending row =================
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&p.counters[kvh], 1) == p.nsplit - 1;
  __syncthreads();
  if (!s_last) return;
#if SD_DR_EXP == 2
  if (tid == 0) p.counters[kvh] = 0;
  return;
#endif
  __threadfence();
  // One round of loads per thread: warp (part, row) reads the row's split lse
  // values, its part's partial outputs and the pending row, then combines;
  // the parts are summed in order afterwards (deterministic).
  const int ns = p.nsplit;
  const int parts = THREADS / (p.G * 32) < 1 ? 1 : THREADS / (p.G * 32);
  float* s_part = reinterpret_cast<float*>(smem);  // [parts][G][DH]
  float* s_inv = s_part + parts * p.G * DH;        // [G]
  for (int job = warp; job < parts * p.G; job += NCW + 1) {
    const int part = job / p.G, row = job - part * p.G, h = kvh * p.G + row;
    const int c0 = part * ns / parts, c1 = (part + 1) * ns / parts;
    const float4* src = reinterpret_cast<const float4*>(p.ws_o + (int64_t)h * DH) + lane;
    const int64_t cstride = (int64_t)p.H * DH / 4;
    constexpr int PRE = 8;
    float4 ob[PRE];
#pragma unroll
    for (int k = 0; k < PRE; ++k) ob[k] = c0 + k < c1 ? __ldcg(src + (c0 + k) * cstride) : make_float4(0.f, 0.f, 0.f, 0.f);
    float lv[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int c = lane + 32 * j;
      lv[j] = c < ns ? __ldcg(p.ws_lse + (int64_t)c * p.H + h) : -INFINITY;
    }
    const uint2 qu = *reinterpret_cast<const uint2*>(p.q + (int64_t)h * DH + lane * 4);
    const uint2 ku = *reinterpret_cast<const uint2*>(p.k_self + kvh * p.self_stride + lane * 4);
    const uint2 vu = *reinterpret_cast<const uint2*>(p.v_self + kvh * p.self_stride + lane * 4);
    // the pending token's own row (already rotated at rank m): always visible
    float sd = __uint_as_float(qu.x << 16) * __uint_as_float(ku.x << 16) +
               __uint_as_float(qu.x & 0xffff0000u) * __uint_as_float(ku.x & 0xffff0000u) +
               __uint_as_float(qu.y << 16) * __uint_as_float(ku.y << 16) +
               __uint_as_float(qu.y & 0xffff0000u) * __uint_as_float(ku.y & 0xffff0000u);
    sd = warp_sum(sd) * LOG2E;
    float M = fmaxf(fmaxf(fmaxf(lv[0], lv[1]), fmaxf(lv[2], lv[3])), lv[4]);
    M = fmaxf(warp_max(M), sd);
    float L = 0.f;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      lv[j] = tc::ex2(lv[j] - M);  // weights; -inf -> 0
      L += lv[j];
    }
    const float wsf = tc::ex2(sd - M);
    L = warp_sum(L) + wsf;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (part == 0)
      acc = make_float4(wsf * __uint_as_float(vu.x << 16), wsf * __uint_as_float(vu.x & 0xffff0000u),
                        wsf * __uint_as_float(vu.y << 16), wsf * __uint_as_float(vu.y & 0xffff0000u));
    auto weight = [&](int c) {
      const int j = c >> 5;
      const float wsel = j == 0 ? lv[0] : j == 1 ? lv[1] : j == 2 ? lv[2] : j == 3 ? lv[3] : lv[4];
      return __shfl_sync(0xffffffffu, wsel, c & 31);
    };
    auto fold = [&](float w, const float4& u) {
      acc.x = fmaf(w, u.x, acc.x);
      acc.y = fmaf(w, u.y, acc.y);
      acc.z = fmaf(w, u.z, acc.z);
      acc.w = fmaf(w, u.w, acc.w);
    };
#pragma unroll
    for (int k = 0; k < PRE; ++k)  // fixed split order
      if (c0 + k < c1) fold(weight(c0 + k), ob[k]);
    for (int cb = c0 + PRE; cb < c1; cb += PRE) {  // further splits: PRE loads in flight per round
#pragma unroll
      for (int k = 0; k < PRE; ++k)
        ob[k] = cb + k < c1 ? __ldcg(src + (cb + k) * cstride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < PRE; ++k)
        if (cb + k < c1) fold(weight(cb + k), ob[k]);
    }
    *reinterpret_cast<float4*>(s_part + (part * p.G + row) * DH + lane * 4) = acc;
    if (part == 0 && lane == 0) s_inv[row] = 1.f / L;
  }
  __syncthreads();
  for (int row = warp; row < p.G; row += NCW + 1) {
    const int h = kvh * p.G + row;
    float4 t = *reinterpret_cast<const float4*>(s_part + row * DH + lane * 4);
    for (int q = 1; q < parts; ++q) {
      const float4 u = *reinterpret_cast<const float4*>(s_part + (q * p.G + row) * DH + lane * 4);
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
    const float inv = s_inv[row];
    uint2 st;
    st.x = pack_bf16(t.x * inv, t.y * inv);
    st.y = pack_bf16(t.z * inv, t.w * inv);
    *reinterpret_cast<uint2*>(p.out + (int64_t)h * DH + lane * 4) = st;
  }
  if (tid == 0) p.counters[kvh] = 0;  // ready for the next launch / graph replay
}

}  // namespace dr

// splits per kv head: one CTA per SM when all of the model's kv heads sit on
// one GPU; a function of (slot range, total kv heads) only
static void draft_split(int hi, int kv_heads_total, int& nsplit, int& kps) {
  const int target = 148 / (kv_heads_total > 0 ? kv_heads_total : 1) > 0 ? 148 / kv_heads_total : 1;
  kps = (hi + target - 1) / target;
  kps = (kps + dr::TILE - 1) / dr::TILE * dr::TILE;
  if (kps < dr::MIN_KPS) kps = dr::MIN_KPS;
  if (kps > dr::MAX_KPS) kps = dr::MAX_KPS;
  nsplit = hi > 0 ? (hi + kps - 1) / kps : 1;
}

int draft_mma_splits(int hi, int kv_heads_total) {
  int n, k;
  draft_split(hi, kv_heads_total, n, k);
  return n;
}

int launch_draft_mma(const void* tmap_k, const void* tmap_v, const void* q, int H, int Hk, int kv_heads_total,
                     int layer, int hi, const int32_t* ranks, const void* k_self, const void* v_self,
                     int64_t self_stride, float* ws_o, int* counters, void* out, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(dr::draft_mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dr::SMEM_ALLOC);
    cudaFuncSetAttribute(dr::draft_mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dr::SMEM_ALLOC);
    attr_set = true;
  }
  dr::Params p;
  p.q = (const __nv_bfloat16*)q;
  p.ranks = ranks;
  p.k_self = (const __nv_bfloat16*)k_self;
  p.v_self = (const __nv_bfloat16*)v_self;
  p.self_stride = self_stride;
  p.H = H;
  p.G = H / Hk;
  p.layer = layer;
  p.hi = hi;
  draft_split(hi, kv_heads_total > 0 ? kv_heads_total : Hk, p.nsplit, p.kps);
  if (p.nsplit > 160) {  // the merge holds <= 160 split weights per row
    set_error("sd_attention(draft): %d slots need %d splits (max 160)", hi, p.nsplit);
    return SD_EINVAL;
  }
  p.ws_o = ws_o;
  p.ws_lse = ws_o + (size_t)p.nsplit * H * dr::DH;
  p.counters = counters;
  p.out = (__nv_bfloat16*)out;
  for (int i = 0; i < 64; ++i) {  // model.py:161: inv_freq_i = 10000^(-2i/dh), fp64
    const double f = pow(10000.0, -2.0 * i / dr::DH) / (2.0 * M_PI);
    p.fh[i] = (float)f;
    p.fl[i] = (float)(f - (double)p.fh[i]);
  }
  CUtensorMap mk, mv;
  memcpy(&mk, tmap_k, sizeof(CUtensorMap));
  memcpy(&mv, tmap_v, sizeof(CUtensorMap));
  dim3 grid(p.nsplit, Hk);
  if (p.G > 8)
    launch_pdl(dr::draft_mma_kernel<true>, grid, dim3(dr::THREADS), dr::SMEM_ALLOC, st, mk, mv, p);
  else
    launch_pdl(dr::draft_mma_kernel<false>, grid, dim3(dr::THREADS), dr::SMEM_ALLOC, st, mk, mv, p);
  return check_launch("sd_attention(draft mma)");
}

}  // namespace sd
