// Tree-verification attention on the 5th-generation tensor cores (sm_100a).
//
// Same contract as the split-KV path in attention.cu (reference model.py:238-247,
// 290-300): per kv head, the G*T query rows of the tree (query head j uses kv
// head j / G) attend to the full-cache rows of one key chunk; the CTA writes
// (o / l, lse) per row and sd_attention merges the chunks in fixed order.
//
// One CTA = (key chunk, kv head, 256-row group), 12 warps; the last chunk
// also covers the T staged tree rows (keys ctx..ctx+T-1) under the tree mask.
//   warps 0, 3  TMA producers for K and V: separate 5-deep rings of 64-key x
//               128-dh tiles (two 128-byte swizzled boxes each), started before
//               Q is staged;
//   warps 1, 2  one MMA-issuer thread per 128-row M-tile: S[mt][j%2] = Q K(j)^T
//               (M=128, N=64, SS) and O[mt] += P(j) V(j) (M=128, N=128, A = P
//               from TMEM, B = V MN-major straight from the TMA layout);
//   warps 4-15  softmax, 16 rows per warp and two threads per row (one per
//               32-key half of every 64-key tile; 16x32bx2 TMEM accesses, the
//               halves' maxima combined by one shuffle): warps 4-11 the first
//               128-row M-tile (two warps per TMEM sub-partition), warps 12-15
//               the second tile. A second tile of <= 64 rows runs as M=64 MMAs,
//               whose rows TMEM spreads over the four sub-partitions (lanes
//               0-15 of each); a larger one keeps thread = row. Online softmax
//               in base 2 with lazy rescale (O is rescaled in TMEM only when the
//               row max grows by > 2^8); full tiles take a third of their exps
//               on the FMA pipe (degree-3 polynomial); P (bf16x2) is written
//               back over the first 32 columns of the S buffer it came from.
// S(j+2) reuses buffer j%2, whose P(j) is still an operand of O += P(j) V(j).
// Both MMAs come from the same issuer thread with the PV first, and tcgen05.mma
// instructions of one thread execute in issue order (the pipelined-pair rule of
// the tcgen05 memory model), so the write-after-read on TMEM needs no barrier:
// the issuer never waits for an MMA to retire, and a tile costs it three
// barrier waits (K landed, V landed, P written) and four commits.
#include <cuda_fp16.h>

#include "tc_common.cuh"

namespace sd {
namespace tc {

constexpr int BN = 64;          // keys per tile
#ifndef SD_TC_MIN_CHUNK
#define SD_TC_MIN_CHUNK 256
#endif
constexpr int MIN_CHUNK = SD_TC_MIN_CHUNK;  // keys per split at least
constexpr int DH = 128;
// K and V stream in 128-key slots (one TMA pair = 2 x 16 KB per slot; one
// full/empty barrier pair per slot) while S / P / softmax work on 64-key
// sub-tiles: half the ring synchronisation per key of 64-key slots.
constexpr int SLOT_KEYS = 128;
constexpr int KST = 2;          // K ring depth (32 KB slots)
constexpr int VST = 3;          // V ring depth (V is held until the PV of its sub-tiles)
constexpr int THREADS = 512;    // 4 role warps + 12 softmax warps
#ifndef SD_TC_ROWS
#define SD_TC_ROWS 256
#endif
constexpr int ROWS = SD_TC_ROWS;  // query rows per CTA (2 M-tiles)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float TAU = 8.0f;     // lazy-rescale threshold (log2 units)
// 1 of every SD_POLY_DEN exp2 pairs of the softmax runs as a polynomial on the
// FMA pipe, the rest on the MUFU (0: all MUFU)
#ifndef SD_POLY_DEN
#define SD_POLY_DEN 3
#endif

constexpr int Q_BYTES = ROWS * DH * 2;          // 64 KB: [mt][dh half][128 rows][128 B]
constexpr int KV_SLOT = SLOT_KEYS * DH * 2;     // 32 KB: [dh half][128 rows][128 B]
constexpr int HALF = KV_SLOT / 2;               // 16 KB: one dh half of a slot
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + Q_BYTES;
constexpr int OFF_V = OFF_K + KST * KV_SLOT;
constexpr int OFF_BAR = OFF_V + VST * KV_SLOT;
constexpr int N_BAR = 2 * KST + 2 * VST + 3 * 4 + 2;
constexpr int SMEM_BYTES = OFF_BAR + N_BAR * 8 + 16;
constexpr int SMEM_ALLOC = SMEM_BYTES + 1024;   // slack for 1024-byte alignment

// TMEM columns (512): O[mt] fp32 128 each; S[mt][buf] fp32 64 each (double
// buffered); P[mt][buf] (bf16x2, the TMEM A operand of O += P V) overwrites the
// first 32 columns of the S buffer it was computed from.
constexpr uint32_t COL_O = 0;
constexpr uint32_t COL_S = 256;
constexpr uint32_t TMEM_COLS = 512;

// keys per split: ctx spread over n_target splits, at least MIN_CHUNK, whole tiles
__host__ __device__ __forceinline__ int chunk_len(int ctx, int n_target) {
  int c = (ctx + n_target - 1) / n_target;
  c = (c + BN - 1) / BN * BN;
  return c < MIN_CHUNK ? MIN_CHUNK : c;
}

struct Params {
  const __nv_bfloat16* q;  // [T][H][128]
  int T, H, G;
  int layer, ctx, n_target;  // n_target: chunks per kv head the split aims for (a function of the
                             // model's total kv heads, not of the shard: SURVEY H7)
  const int32_t* rows_dev;
  const int32_t* ctx_dev;  // nullable: live cache length (chunking resolved per launch on device)
  const uint32_t* mask;    // [T][mask_words] tree rows (NULL = causal)
  int mask_words;
  __half* ws_o;  // [split][T][H][128] fp16 partial o / l
  float* ws_lse;
  __nv_bfloat16* merge_out;  // non-null: the split merge runs in this kernel (fused_merge) into out [T][H][128]
  int* merge_counters;       // [Hk][2] arrival / departure counters, zero between launches
};


// Debug-only event timeline of CTA (0, 0, 0) (sd_debug_tc_trace); NULL in production.
// Compiled in only with -DSD_TC_TRACE (tools/tc_trace.py builds that variant):
// production kernels carry no instrumentation on the MMA critical path.
__device__ int64_t* g_tc_trace = nullptr;
// Debug-only pipeline experiments (-DSD_TC_EXPERIMENT=n, tools/gpu_tc_exp.sh):
// 1 = softmax skips its math, 2 = no PV MMAs, 3 = no QK MMAs, 4 = 1+2+3 (TMA stream only),
// 5 = 4 without the softmax's TMEM loads, 6 = 5 with plain mbarrier arrives instead of commits,
// 8 = bare TMA stream inside this kernel (producers recycle their own slots; no issuer / softmax),
// 9 = 6 without the softmax warps (the issuer does not wait for P).
#ifndef SD_TC_EXPERIMENT
#define SD_TC_EXPERIMENT 0
#endif
#define SD_TC_NOMMA (SD_TC_EXPERIMENT >= 4)
__device__ __forceinline__ void tc_signal(uint64_t* bar) {
#if SD_TC_EXPERIMENT == 6 || SD_TC_EXPERIMENT == 9
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
#else
  umma_commit(bar);
#endif
}
constexpr int TR_TILES = 64, TR_EV = 8;
__device__ __forceinline__ void trace(int role, int j, int ev) {
#ifdef SD_TC_TRACE
  int64_t* t = g_tc_trace;
  if (t && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < TR_TILES)
    t[(role * TR_TILES + j) * TR_EV + ev] = clock64();
#else
  (void)role;
  (void)j;
  (void)ev;
#endif
}

// MMA issue stream of one M-tile (warps 1 / 2; the whole warp runs the loop,
// one elected lane issues). TMEM base is 0: the CTA owns all 512 columns.
//   S[MT][j%2] = Q[MT] K(j)^T (8 K=16 steps), O[MT] += P(j) V(j) (4 steps)
__device__ __forceinline__ uint2 pack_half4(float4 f) {
  const __half2 a = __floats2half2_rn(f.x, f.y), b = __floats2half2_rn(f.z, f.w);
  return make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
}
// word w of a row's tree-visibility bits without dynamic register indexing
__device__ __forceinline__ uint32_t pick_word(const uint32_t (&m)[SD_MASK_WORDS], int w) {
  uint32_t r = 0u;
#pragma unroll
  for (int i = 0; i < SD_MASK_WORDS; ++i) r = w == i ? m[i] : r;
  return r;
}
// visibility of keys key0..key0+31 for one query row: committed-cache keys
// (< cache_end) are all visible; in the last chunk, key ctx + j (a staged tree
// row) is visible iff bit j of the row's ancestor-or-self mask is set (bits
// beyond the row's own index are zero). Bit arithmetic only, no per-key loop.
__device__ __forceinline__ uint32_t vis_bits32(int key0, int cache_end, int ctx, bool last,
                                               const uint32_t (&m)[SD_MASK_WORDS]) {
  const int nc = cache_end - key0;
  uint32_t v = nc >= 32 ? 0xffffffffu : (nc <= 0 ? 0u : ((1u << nc) - 1u));
  if (last) {
    const int j0 = key0 - ctx;
    uint32_t win;
    if (j0 >= 0) {
      const int w = j0 >> 5, o = j0 & 31;
      const uint32_t lo = pick_word(m, w), hi = pick_word(m, w + 1);
      win = o ? (lo >> o) | (hi << (32 - o)) : lo;
    } else {
      win = -j0 >= 32 ? 0u : pick_word(m, 0) << (-j0);
    }
    v |= win;
  }
  return v;
}

template <int MT, int M>
__device__ __forceinline__ void issue_loop(uint8_t* smem, int n_tiles, uint32_t p_bar_count, uint64_t* k_full,
                                           uint64_t* k_empty, uint64_t* v_full, uint64_t* v_empty, uint64_t* s_full,
                                           uint64_t* pv_done, uint64_t* o_final) {
  __syncwarp();
  const bool leader = elect_one();
  constexpr uint32_t id_qk = idesc_bf16(BN, false, M);
  constexpr uint32_t id_pv = idesc_bf16(DH, true, M);
  constexpr uint32_t O_COL = COL_O + 128 * MT;
  const uint32_t sb = smem_u32(smem);
  const uint32_t q_base = sb + OFF_Q + MT * 32768;
  auto issue_qk = [&](int j) {
    const int s = (j >> 1) % KST, b = j & 1;
    const uint32_t k_base = sb + OFF_K + s * KV_SLOT + (j & 1) * (BN * 128);
    if (leader) {
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        const uint32_t half = ks >> 2, in = (ks & 3) * 32;
        if (SD_TC_EXPERIMENT != 3 && !SD_TC_NOMMA)
          umma_bf16(COL_S + 128 * MT + 64 * b, umma_desc(q_base + half * 16384 + in, 16, 1024),
                    umma_desc(k_base + half * HALF + in, 16, 1024), id_qk, ks > 0);
      }
      tc_signal(&s_full[2 * MT + b]);
      if ((j & 1) || j == n_tiles - 1) tc_signal(&k_empty[s]);  // slot's last sub-tile
    }
    __syncwarp();
  };
  auto wait_k = [&](int j) {
    if (j & 1) return;  // the odd sub-tile shares its slot with the even one
    if (MT == 0) trace(1, j, 0);
    const int q = j >> 1;
    mbar_wait(&k_full[q % KST], (q / KST) & 1);
    if (MT == 0) trace(1, j, 1);
    tc_fence_after();
  };
  for (int j0 = 0; j0 < 2 && j0 < n_tiles; ++j0) {
    wait_k(j0);
    issue_qk(j0);
  }
  for (int j = 0; j < n_tiles; ++j) {
    const int q = j >> 1, s = q % VST, b = j & 1;
    if (MT == 0) trace(1, j, 3);
    if (!(j & 1)) mbar_wait(&v_full[s], (q / VST) & 1);
    const uint32_t v_base = sb + OFF_V + s * KV_SLOT + (j & 1) * (BN * 128);
#if SD_TC_EXPERIMENT != 9
    asm volatile("bar.sync %0, %1;" ::"r"(2 + 2 * MT + b), "r"(p_bar_count) : "memory");  // P(j) written
#endif
    if (MT == 0) trace(1, j, 4);
    tc_fence_after();
    if (leader) {
#pragma unroll
      for (int ks = 0; ks < BN / 16; ++ks)  // V tile [64 keys][dh] (MN-major B): dh halves LBO apart
        if (SD_TC_EXPERIMENT != 2 && !SD_TC_NOMMA)
          umma_bf16_ts(O_COL, COL_S + 128 * MT + 64 * b + 8 * ks, umma_desc(v_base + ks * 16 * 128, HALF, 1024),
                       id_pv, (j > 0 || ks > 0) ? 1u : 0u);
      tc_signal(&pv_done[2 * MT + b]);
      if (j == n_tiles - 1) tc_signal(&o_final[MT]);
      if ((j & 1) || j == n_tiles - 1) tc_signal(&v_empty[s]);
    }
    __syncwarp();
    if (MT == 0) trace(1, j, 6);
    // S(j+2) into buffer b: issued after PV(j) by this thread, so it is
    // ordered after PV(j)'s reads of P(j) (same-thread tcgen05.mma order)
    if (j + 2 < n_tiles) {
      wait_k(j + 2);
      issue_qk(j + 2);
    }
  }
}

// The split merge inside the kernel (replaces merge128_kernel when the whole
// grid is co-resident: one row group, <= one CTA per SM). Every live chunk CTA
// of a kv head publishes its fp16 partials, arrives on the head's counter and
// waits until all n_live have arrived; then CTA x merges rows [x R / n_live,
// (x+1) R / n_live) of the head's R = T*G output rows — the same arithmetic,
// in the same order, as merge128_kernel (bitwise equal output). The last CTA
// to leave resets the counters for the next launch (a graph replay, or the
// next layer: every launch passes griddepcontrol.wait first, i.e. after the
// previous launch's reset). Spinning cannot deadlock: the host fuses only when
// the grid fits on the SMs at one CTA each, and nothing the CTAs wait for
// depends on this kernel.
__device__ __noinline__ void fused_merge(const Params& p, int kvh, int n_live, int T_live) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int* arrive = p.merge_counters + 2 * kvh;
  int* depart = arrive + 1;
  __threadfence();  // this CTA's partials visible at gpu scope before it arrives
  __syncthreads();
  if (tid == 0) {
    atomicAdd(arrive, 1);
    int seen;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(arrive) : "memory");
      if (seen >= n_live) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
  const int G = p.G, R = p.T * G;
  const int r0 = (int)((int64_t)blockIdx.x * R / n_live), r1 = (int)((int64_t)(blockIdx.x + 1) * R / n_live);
  constexpr int MK = 5, MU = 8;  // <= 160 splits (lane c % 32, register c / 32); MU partials in flight
  for (int rho = r0 + warp; rho < r1; rho += THREADS / 32) {
    const int t = rho / G, h = kvh * G + (rho - t * G);
    __nv_bfloat16* dst = p.merge_out + ((int64_t)t * p.H + h) * DH + 4 * lane;
    if (t >= T_live) {  // padded row: defined zeros
      *reinterpret_cast<uint2*>(dst) = make_uint2(0u, 0u);
      continue;
    }
    float lv[MK], wv[MK];
#pragma unroll
    for (int k = 0; k < MK; ++k) {
      const int c = lane + 32 * k;
      lv[k] = c < n_live ? __ldcg(p.ws_lse + ((int64_t)c * p.T + t) * p.H + h) : -INFINITY;
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
    const __half* base = p.ws_o + ((int64_t)t * p.H + h) * DH + 4 * lane;
    const int64_t cstride = (int64_t)p.T * p.H * DH;
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
        for (int u = 0; u < MU; ++u) {
          const uint2 raw = __ldcg(reinterpret_cast<const uint2*>(base + (int64_t)(32 * k + cs[u]) * cstride));
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
          const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
          o[u] = make_float4(a.x, a.y, b.x, b.y);
        }
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
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv), hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(dst) = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(depart, 1) == n_live - 1) {  // everyone has passed the wait: reset for the next launch
      *arrive = 0;
      *depart = 0;
      __threadfence();
    }
  }
}

// FUSED: the fused_merge tail (SD_TC_FUSED_MERGE=1) is a separate instantiation so
// the production kernel's code is unchanged by it
template <bool FUSED>
__global__ void __launch_bounds__(THREADS, 1)
    verify_attn_tc_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                          Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + OFF_BAR);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;      // [mt][buf]: QK retired -> softmax
  uint64_t* p_full = s_full + 4;         // [mt][buf]: P(j) in TMEM -> PV(j), then QK(j+2)
  uint64_t* pv_done = p_full + 4;        // [mt][buf]: PV(j) retired -> O stable (lazy rescale)
  uint64_t* o_final = pv_done + 4;       // [mt]: single phase, after the last PV
  uint32_t* tmem_slot = (uint32_t*)(o_final + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kvh = blockIdx.y;
  // Programmatic dependent launch: this kernel may start while its predecessor
  // (the RoPE/KV staging of this layer) still runs. rows_dev / ctx_dev (the
  // tree record) and the committed cache rows come from earlier kernels and are
  // read at once; q and the staged tree rows only after pdl_wait.
  pdl_trigger();
#ifdef SD_TC_TRACE
  int64_t t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  const int T = p.rows_dev ? min(*p.rows_dev, p.T) : p.T;
  const int GT = p.G * T;
  const int rg = blockIdx.z * ROWS;
  if (rg >= GT) return;
  if (tid == 0) trace(0, 60, 0);
  // Split boundaries are a function of the live context and n_target only
  // (tc_chunk_len), identical for the host- and device-resident context and for
  // any number of GPUs sharing the kv heads: bitwise cross-P determinism (H7).
  const int ctx = p.ctx_dev ? *p.ctx_dev : p.ctx;
#ifndef SD_TC_LAST_RELIEF
#define SD_TC_LAST_RELIEF 0
#endif
  const int chunk = chunk_len(ctx + SD_TC_LAST_RELIEF, p.n_target);
  const int n_live = ctx > 0 ? (ctx + chunk - 1) / chunk : 1;
  if ((int)blockIdx.x >= n_live) {  // empty split: weight 0 in the merge
    for (int r = tid; r < ROWS; r += THREADS) {
      const int rho = rg + r;
      if (rho < GT) {
        const int t = rho / p.G, g = rho - t * p.G;
        p.ws_lse[((int64_t)blockIdx.x * p.T + t) * p.H + kvh * p.G + g] = -INFINITY;
      }
    }
    return;
  }
  const bool last = (int)blockIdx.x == n_live - 1;
  const int key_begin = blockIdx.x * chunk;
  const int cache_end = min(ctx, key_begin + chunk);
  const int key_end = last ? ctx + T : cache_end;  // the last chunk also takes the tree rows
  const int n_tiles = (key_end - key_begin + BN - 1) / BN;
  // The second M-tile runs as an M=64 MMA when it holds <= 64 rows: its rows
  // then sit in lanes 0-15 of each TMEM sub-partition (row 16k+i -> lane
  // 32k+i), so they spread over several SM sub-partitions instead of doubling
  // up on the first two with the first tile's rows, and each row is softmaxed
  // by two threads (one per 32-key half: 16x32bx2 TMEM accesses).
  const int rows1 = GT - rg - 128;
  const bool m1_64 = rows1 > 0 && rows1 <= 64;
  int act[2];  // softmax warps per tile (named-barrier arrivals)
  act[0] = 0;
  for (int g = 0; g < 8; ++g) act[0] += rg + 16 * g < GT;
  act[1] = 0;
  for (int w = 0; w < 4; ++w) act[1] += m1_64 ? (16 * w < rows1) : (32 * w < rows1);
  const int nm = act[1] > 0 ? 2 : 1;

  // ---- barriers first, so the TMA producers start streaming at once ----
  if (tid == 0) {
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], nm);  // one commit per M-tile issuer
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], nm);
    }
    for (int mt = 0; mt < 2; ++mt) {
      const uint32_t arrivals = act[mt] > 0 ? act[mt] : 1;  // one arrive per active softmax warp
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_full[2 * mt + b], 1);
        mbar_init(&p_full[2 * mt + b], arrivals);
        mbar_init(&pv_done[2 * mt + b], 1);
      }
      mbar_init(&o_final[mt], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t tmem = 0;
  if (warp != 0 && warp != 3) {
    // ---- stage Q (M-tiles, K-major SW128) while the first K/V tiles are in flight ----
    constexpr int NT = THREADS - 64;  // warps 1, 2, 4..15
    const int qt = tid < 96 ? tid - 32 : tid - 64;
    constexpr int PER = (ROWS * (DH / 8) + NT - 1) / NT;  // 16-byte chunks per thread
    uint4 v[PER];
    pdl_wait();  // q is the predecessor's output
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = qt + k * NT;
      const int row = i >> 4, c = i & 15;
      const int rho = rg + row;
      v[k] = make_uint4(0, 0, 0, 0);
      if (i < ROWS * 16 && rho < GT) {
        const int t = rho / p.G, g = rho - t * p.G;
        v[k] = __ldg(reinterpret_cast<const uint4*>(p.q + ((int64_t)t * p.H + kvh * p.G + g) * DH + c * 8));
      }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = qt + k * NT;
      if (i < ROWS * 16) {
        const int row = i >> 4, c = i & 15;
        const int mt = row >> 7, r = row & 127, half = c >> 3;
        *reinterpret_cast<uint4*>(smem + OFF_Q + mt * 32768 + half * 16384 + sw128(r, c & 7)) = v[k];
      }
    }
    if (warp == 2) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_async_smem();
    tc_fence_before();
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");  // Q staged + TMEM allocated (consumers only)
    tc_fence_after();
    tmem = *tmem_slot;
    if (tid == 32) trace(0, 60, 2);
  }

  if (warp == 0 || warp == 3) {
    // ================= TMA producers: K (warp 0) and V (warp 3), decoupled =================
    // K(j) is recycled when QK(j) retires, V(j) only after the softmax and PV
    // of tile j: one thread per ring keeps the K stream from queueing behind V.
    if (lane == 0) {
      const bool is_k = warp == 0;
      const CUtensorMap* map = is_k ? &tmap_k : &tmap_v;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      uint8_t* ring = smem + (is_k ? OFF_K : OFF_V);
      const int depth = is_k ? KST : VST;
      tma_prefetch(map);
      bool waited = false;
      const int n_slots = (n_tiles + 1) / 2;
      for (int q = 0; q < n_slots; ++q) {
        const int s = q % depth;
        const int key0 = key_begin + q * SLOT_KEYS;
        if (!waited && key0 + SLOT_KEYS > ctx) {  // slot reaches the tree rows staged by the predecessor
          pdl_wait();
          waited = true;
        }
#if SD_TC_EXPERIMENT == 8
        if (q >= depth) mbar_wait(&full[s], ((q / depth) + 1) & 1);
#else
        if (q >= depth) mbar_wait(&empty[s], ((q / depth) + 1) & 1);
#endif
        trace(0, q, is_k ? 1 : 2);
        uint8_t* d = ring + s * KV_SLOT;
        mbar_expect_tx(&full[s], KV_SLOT);
        tma_load_4d(d, map, &full[s], 0, key0, kvh, p.layer);
        tma_load_4d(d + HALF, map, &full[s], 64, key0, kvh, p.layer);
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ================= MMA issuers: one thread per M-tile =================
    // Each M-tile runs its own QK -> softmax -> PV chain on its own TMEM
    // columns; the two issuers share the K/V rings (a slot is free once both
    // have committed it) and their MMAs interleave in the tensor pipe, so one
    // tile's barrier waits never stall the other's MMAs.
    // The whole warp runs the issuer loop (lane 0 issues the MMAs and commits) so
    // that "P(j) written" can arrive as a hardware named barrier from the softmax
    // warpgroup instead of an mbarrier round trip.
    const int mt = warp - 1;
#if SD_TC_EXPERIMENT == 8
    if (lane == 0 && mt < nm) mbar_arrive(&o_final[mt]);
#else
    // M-tile as a template argument: every descriptor and TMEM address of the
    // issue stream is then warp-uniform (uniform datapath, no per-MMA R2UR /
    // ELECT waterfall); one elected lane issues.
    if (mt == 0)
      issue_loop<0, 128>(smem, n_tiles, 32u * (uint32_t)(act[0] + 1), k_full, k_empty, v_full, v_empty, s_full,
                         pv_done, o_final);
    else if (mt < nm && m1_64)
      issue_loop<1, 64>(smem, n_tiles, 32u * (uint32_t)(act[1] + 1), k_full, k_empty, v_full, v_empty, s_full,
                        pv_done, o_final);
    else if (mt < nm)
      issue_loop<1, 128>(smem, n_tiles, 32u * (uint32_t)(act[1] + 1), k_full, k_empty, v_full, v_empty, s_full,
                         pv_done, o_final);
#endif
  } else if (warp >= 4 && (warp < 12 || m1_64)) {
    // ================= softmax, 16 rows per warp, two threads per row =================
    // Tile 0 (M=128): warp 4+4s+q takes tile rows 32q+16s..+15 (TMEM lanes
    // 32q+16s..); an M=64 tile 1: warp 12+q takes rows 16q..16q+15 (lanes
    // 32q..32q+15). Thread lane&15 -> row, lane>>4 -> 32-key half of every
    // 64-key tile (16x32bx2 TMEM accesses). The two halves of a row combine
    // their maxima with one shuffle per tile and their sums at the end; each
    // rescales / writes its half of O and of P.
    const int mt = warp >= 12 ? 1 : 0;
    const int q = warp & 3, r16 = lane & 15, h = lane >> 4;
    const int sub = mt == 0 ? ((warp - 4) >> 2) : 0;
    const int lane0 = 32 * q + 16 * sub;                         // first TMEM lane of this warp
    const int row1 = mt == 0 ? lane0 + r16 : 16 * q + r16;       // row within the tile
    const int tile_rows = mt == 0 ? min(128, GT - rg) : rows1;
    const int rho = rg + 128 * mt + row1;
    if (row1 - r16 < tile_rows) {
      const bool valid = row1 < tile_rows;
      const int t = valid ? rho / p.G : 0;
      const uint32_t lane_base = (uint32_t)lane0 << 16;
      uint32_t tmask[SD_MASK_WORDS];
#pragma unroll
      for (int w = 0; w < SD_MASK_WORDS; ++w) {
        uint32_t bits = 0u;
        const int lo = 32 * w;
        if (lo <= t) {
          bits = p.mask ? (w < p.mask_words ? p.mask[(int64_t)t * p.mask_words + w] : 0u) : 0xffffffffu;
          const int lim = t - lo;
          if (lim < 31) bits &= (2u << lim) - 1u;
          if (lim < 32) bits |= 1u << lim;
        }
        tmask[w] = bits;
      }
      const uint32_t bar_count = 32u * (uint32_t)(act[mt] + 1);
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int b = j & 1;
        mbar_wait(&s_full[2 * mt + b], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t s_addr = tmem + lane_base + COL_S + 128 * mt + 64 * b;
        uint32_t sr[32];
        tmem_ld16x2_32<32>(s_addr, sr);
        tmem_wait_ld();
        const int key0 = key_begin + j * BN + 32 * h;
        const bool full = key_begin + j * BN + BN <= cache_end;  // tile-uniform
        if (!full) {
          const uint32_t vis = valid ? vis_bits32(key0, cache_end, ctx, last, tmask) : 0u;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (!((vis >> c) & 1u)) sr[c] = __float_as_uint(-INFINITY);
        }
        float m11[11];
#pragma unroll
        for (int c = 0; c < 10; ++c)
          m11[c] = fmax3(__uint_as_float(sr[c]), __uint_as_float(sr[c + 10]), __uint_as_float(sr[c + 20]));
        m11[10] = fmaxf(__uint_as_float(sr[30]), __uint_as_float(sr[31]));
        float mh = fmax3(fmax3(m11[0], m11[1], m11[2]), fmax3(m11[3], m11[4], m11[5]),
                         fmax3(fmax3(m11[6], m11[7], m11[8]), m11[9], m11[10]));
        mh = fmaxf(mh, __shfl_xor_sync(0xffffffffu, mh, 16));  // both halves of the row
        const float mx = mh * LOG2E;
        float scale = 1.f;
        bool rescale = false;
        if (mx > m_used + TAU) {
          scale = m_used == -INFINITY ? 0.f : ex2(m_used - mx);
          rescale = j > 0;
          m_used = mx;
          l *= scale;
        }
        uint32_t pk[16];
        const float nm_used = m_used == -INFINITY ? 0.f : -m_used;
        const uint64_t lg2 = f2(LOG2E, LOG2E), off = f2(nm_used, nm_used);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        if (full) {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 x = unf2(ffma2(f2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), lg2, off));
            float2 pp;
            if (SD_POLY_DEN > 0 && (c >> 1) % SD_POLY_DEN == SD_POLY_DEN - 1) {
              pp = exp2_poly3_pair(x.x, x.y);
            } else {
              pp.x = ex2(x.x);
              pp.y = ex2(x.y);
            }
            acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], f2(pp.x, pp.y));
            pk[c >> 1] = pack_bf16(pp.x, pp.y);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 x = unf2(ffma2(f2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), lg2, off));
            const float e0 = ex2(x.x), e1 = ex2(x.y);
            acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], f2(e0, e1));
            pk[c >> 1] = pack_bf16(e0, e1);
          }
        }
        {
          const float2 a2 = unf2(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
          l += a2.x + a2.y;
        }
        if (__any_sync(0xffffffffu, rescale)) {
          if (j > 0) mbar_wait(&pv_done[2 * mt + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {  // this half's 64 columns of O: [64h + 32 q2, +32)
            uint32_t o[32];
            const uint32_t ta = tmem + lane_base + COL_O + 128 * mt + 32 * q2;
            tmem_ld16x2_32<64>(ta, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * (rescale ? scale : 1.f));
            tmem_st16x2_32<64>(ta, o);
          }
          tmem_wait_st();
        }
        tmem_st16x2_16<16>(s_addr, pk);  // P(j): keys 32h.. -> columns 16h..16h+15
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.arrive %0, %1;" ::"r"(2 + 2 * mt + b), "r"(bar_count) : "memory");
      }
      // ---- epilogue ----
      for (int m2 = 0; m2 < nm; ++m2) mbar_wait(&o_final[m2], 0);
      tc_fence_after();
      const float lt = l + __shfl_xor_sync(0xffffffffu, l, 16);
      const int g = rho - t * p.G;
      const int64_t oi = ((int64_t)blockIdx.x * p.T + t) * p.H + kvh * p.G + g;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      uint8_t* stage = smem + OFF_K + (warp - 4) * (16 * DH * 4);  // 16 rows x 512 B
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2) {
        uint32_t o[32];
        tmem_ld16x2_32<64>(tmem + lane_base + COL_O + 128 * mt + 32 * q2, o);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int chunk = 16 * h + 8 * q2 + c;  // 16-byte chunk of the row (4 floats)
          *reinterpret_cast<float4*>(stage + r16 * 512 + ((chunk ^ r16) << 4)) =
              make_float4(__uint_as_float(o[4 * c]) * inv, __uint_as_float(o[4 * c + 1]) * inv,
                          __uint_as_float(o[4 * c + 2]) * inv, __uint_as_float(o[4 * c + 3]) * inv);
        }
      }
      __syncwarp();
      for (int rr = 0; rr < 16; ++rr) {
        const int64_t oi_r = __shfl_sync(0xffffffffu, oi, rr);
        const bool v_r = __shfl_sync(0xffffffffu, valid, rr);
        if (v_r) {
          const float4 f = *reinterpret_cast<const float4*>(stage + rr * 512 + ((lane ^ rr) << 4));
          reinterpret_cast<uint2*>(p.ws_o + oi_r * DH)[lane] = pack_half4(f);
        }
      }
      if (valid && h == 0) p.ws_lse[oi] = lt > 0.f ? (m_used + __log2f(lt)) / LOG2E : -INFINITY;
    }
  } else if (warp >= 12) {
    // ================= softmax of an M=128 second tile: thread = row =================
    const int mt = 1, wl = warp & 3;
    const int row = 32 * wl + lane;
    const int rho = rg + 128 * mt + row;
    const bool warp_active = (rg + 128 * mt + 32 * wl) < GT;
    if (mt < nm && warp_active) {
      const bool valid = rho < GT;
      const int t = valid ? rho / p.G : 0;
      const uint32_t lane_base = (uint32_t)(32 * wl) << 16;
      // tree-row visibility of this query row (ancestors + self; j <= t)
      uint32_t tmask[SD_MASK_WORDS];
#pragma unroll
      for (int w = 0; w < SD_MASK_WORDS; ++w) {
        uint32_t bits = 0u;
        const int lo = 32 * w;
        if (lo <= t) {
          bits = p.mask ? (w < p.mask_words ? p.mask[(int64_t)t * p.mask_words + w] : 0u) : 0xffffffffu;
          const int lim = t - lo;  // keep j <= t
          if (lim < 31) bits &= (2u << lim) - 1u;
          if (lim < 32) bits |= 1u << lim;  // self
        }
        tmask[w] = bits;
      }
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < (SD_TC_EXPERIMENT == 8 || SD_TC_EXPERIMENT == 9 ? 0 : n_tiles); ++j) {
        const int b = j & 1;
        const int role = (lane == 0 && wl == 0) ? 2 + mt : 99;
        if (role < 4) trace(role, j, 0);
        mbar_wait(&s_full[2 * mt + b], (j >> 1) & 1);
        if (role < 4) trace(role, j, 1);
        tc_fence_after();
        const uint32_t s_addr = tmem + lane_base + COL_S + 128 * mt + 64 * b;
        uint32_t sr[64];
#if SD_TC_EXPERIMENT < 5
        tmem_ld32(s_addr, sr);
        tmem_ld32(s_addr + 32, sr + 32);
        tmem_wait_ld();
#else
        for (int c = 0; c < 64; ++c) sr[c] = 0u;
#endif
        if (SD_TC_EXPERIMENT == 1 || SD_TC_NOMMA) {
          tc_fence_before();
          asm volatile("bar.arrive %0, %1;" ::"r"(2 + 2 * mt + b), "r"(32u * (uint32_t)(act[mt] + 1)) : "memory");
          l += __uint_as_float(sr[0]) + __uint_as_float(sr[63]);  // static indices: sr stays in registers
          continue;
        }
        const int key0 = key_begin + j * BN;
        // warp-uniform: a tile wholly inside the committed cache has no masked
        // keys (rows beyond GT hold zero queries: finite garbage, never written)
        const bool full = key0 + BN <= cache_end;
        if (!full) {
          const uint64_t vis = valid ? ((uint64_t)vis_bits32(key0 + 32, cache_end, ctx, last, tmask) << 32) |
                                           vis_bits32(key0, cache_end, ctx, last, tmask)
                                     : 0ull;
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (!((vis >> c) & 1ull)) sr[c] = __float_as_uint(-INFINITY);
        }
        // tile max: 3-input max tree (short dependency chain)
        float m21[22];
#pragma unroll
        for (int c = 0; c < 21; ++c)
          m21[c] = fmax3(__uint_as_float(sr[c]), __uint_as_float(sr[c + 21]), __uint_as_float(sr[c + 42]));
        m21[21] = __uint_as_float(sr[63]);
        float m8[8];
#pragma unroll
        for (int c = 0; c < 7; ++c) m8[c] = fmax3(m21[c], m21[c + 7], m21[c + 14]);
        m8[7] = m21[21];
        const float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7])) * LOG2E;
        float scale = 1.f;
        bool rescale = false;
        if (mx > m_used + TAU) {
          scale = m_used == -INFINITY ? 0.f : ex2(m_used - mx);
          rescale = j > 0;
          m_used = mx;
          l *= scale;
        }
        uint32_t pk[32];
        const float nm_used = m_used == -INFINITY ? 0.f : -m_used;
        const uint64_t lg2 = f2(LOG2E, LOG2E), off = f2(nm_used, nm_used);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        // p = 2^(s log2e - m): packed scale, packed row sums; the exps split
        // between the MUFU and (1 of every SD_POLY_DEN pairs) the FMA pipe: a
        // degree-3 polynomial on full tiles, the -inf-exact one on masked tiles
        if (full) {
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 x = unf2(ffma2(f2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), lg2, off));
            float2 pp;
            if (SD_POLY_DEN > 0 && (c >> 1) % SD_POLY_DEN == SD_POLY_DEN - 1) {
              pp = exp2_poly3_pair(x.x, x.y);
            } else {
              pp.x = ex2(x.x);
              pp.y = ex2(x.y);
            }
            acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], f2(pp.x, pp.y));
            pk[c >> 1] = pack_bf16(pp.x, pp.y);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 x = unf2(ffma2(f2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), lg2, off));
            float2 pp;
            if (SD_POLY_DEN > 0 && (c >> 1) % SD_POLY_DEN == SD_POLY_DEN - 1) {
              pp = exp2_poly2(x.x, x.y);
            } else {
              pp.x = ex2(x.x);
              pp.y = ex2(x.y);
            }
            acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], f2(pp.x, pp.y));
            pk[c >> 1] = pack_bf16(pp.x, pp.y);
          }
        }
        {
          const float2 a = unf2(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
          l += a.x + a.y;
        }
        if (role < 4) trace(role, j, 2);
        if (__any_sync(0xffffffffu, rescale)) {
          // O must be stable: wait for every earlier O += P V of this M-tile (PV(j-1) retires last)
          if (j > 0) mbar_wait(&pv_done[2 * mt + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t o[32];
            const uint32_t ta = tmem + lane_base + COL_O + 128 * mt + 32 * q4;
            tmem_ld32(ta, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * (rescale ? scale : 1.f));
            tmem_st32(ta, o);
          }
          tmem_wait_st();
        }
        if (role < 4) trace(role, j, 3);
        tmem_st32(s_addr, pk);  // P(j) (bf16x2) over the consumed S columns
        tmem_wait_st();
        tc_fence_before();  // P(j) in TMEM -> the issuer warp's bar.sync releases it to the MMA
        asm volatile("bar.arrive %0, %1;" ::"r"(2 + 2 * mt + b), "r"(32u * (uint32_t)(act[mt] + 1)) : "memory");
        if (role < 4) trace(role, j, 4);
      }
      // ---- epilogue: O / l, lse (natural log) ----
      // Every MMA of the CTA has retired once both M-tiles' o_final fired, so the
      // K/V rings are free: each warp stages its 32 rows x 512 B there (16-byte
      // chunks XOR-swizzled by row: conflict-free both ways) and writes them out
      // one contiguous row per instruction instead of 32 rows x 16 B.
      if (row == 0 && mt == 0) trace(0, 60, 3);
      for (int m2 = 0; m2 < nm; ++m2) mbar_wait(&o_final[m2], 0);
      if (row == 0 && mt == 0) trace(0, 60, 4);
      tc_fence_after();
      const int g = rho - t * p.G;
      const int64_t oi = ((int64_t)blockIdx.x * p.T + t) * p.H + kvh * p.G + g;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      uint8_t* stage = smem + OFF_K + 8 * (16 * DH * 4) + (warp - 12) * (32 * DH * 4);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t o[32];
        tmem_ld32(tmem + lane_base + COL_O + 128 * mt + 32 * q4, o);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int chunk = 8 * q4 + c;  // 16-byte chunk of this row
          *reinterpret_cast<float4*>(stage + lane * 512 + ((chunk ^ lane) << 4)) =
              make_float4(__uint_as_float(o[4 * c]) * inv, __uint_as_float(o[4 * c + 1]) * inv,
                          __uint_as_float(o[4 * c + 2]) * inv, __uint_as_float(o[4 * c + 3]) * inv);
        }
      }
      __syncwarp();
      for (int rr = 0; rr < 32; ++rr) {
        const int64_t oi_r = __shfl_sync(0xffffffffu, oi, rr);
        const bool v_r = __shfl_sync(0xffffffffu, valid, rr);
        if (v_r) {
          const float4 f = *reinterpret_cast<const float4*>(stage + rr * 512 + ((lane ^ rr) << 4));
          reinterpret_cast<uint2*>(p.ws_o + oi_r * DH)[lane] = pack_half4(f);
        }
      }
      if (valid) p.ws_lse[oi] = l > 0.f ? (m_used + __log2f(l)) / LOG2E : -INFINITY;
      if (row == 0 && mt == 0) trace(0, 60, 5);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) trace(0, 60, 6);
#ifdef SD_TC_TRACE
  if (tid == 0 && g_tc_trace) {  // per-CTA start / end (globaltimer, ns) after the event block
    const int c = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    g_tc_trace[4 * 64 * 8 + 64 + 2 * c] = t_start;
    g_tc_trace[4 * 64 * 8 + 64 + 2 * c + 1] = (int64_t)now;
  }
#endif
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
  if constexpr (FUSED) {
    if (p.merge_out && GT <= ROWS) fused_merge(p, kvh, n_live, T);  // live rows in one row group: merge here
  }
}

}  // namespace tc

// ---------------------------------------------------------------- host -----
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  return fn;
}

int tc_make_kv_tmap(const void* base, int L, int Hk, int cap, int dh, void* out, int box_rows) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SD_ECUDA;
  }
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out);
  cuuint64_t dims[4] = {(cuuint64_t)dh, (cuuint64_t)cap, (cuuint64_t)Hk, (cuuint64_t)L};
  cuuint64_t strides[3] = {(cuuint64_t)dh * 2, (cuuint64_t)cap * dh * 2, (cuuint64_t)Hk * cap * dh * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SD_ECUDA;
  }
  return SD_OK;
}

static int g_force_chunks = 0;  // debug only (sd_debug_tc_trace)

int tc_set_trace(void* dev_ptr, int force_chunks) {
  g_force_chunks = force_chunks;
  if (dev_ptr) {  // watchdog report area just past the trace block
    void* stuck = (char*)dev_ptr + 4 * 64 * 8 * sizeof(int64_t);
    cudaMemcpyToSymbol(tc::g_tc_stuck, &stuck, sizeof(void*));
  }
  cudaError_t e = cudaMemcpyToSymbol(tc::g_tc_trace, &dev_ptr, sizeof(void*));
  return e == cudaSuccess ? SD_OK : SD_ECUDA;
}

// chunks per kv head the split aims for: one wave of one CTA per SM when the
// model's kv heads all sit on one GPU (148 SMs); a function of the model, never
// of the shard, so every GPU count computes the same splits
int tc_split_target(int kv_heads_total) {
  if (g_force_chunks > 0) return g_force_chunks;
  const int t = 148 / (kv_heads_total > 0 ? kv_heads_total : 1);
  return t < 1 ? 1 : t;
}

// grid width covering every live split of any context <= ctx_bound
int tc_grid_chunks(int ctx_bound, int n_target) {
  const int by_ctx = (ctx_bound + tc::MIN_CHUNK - 1) / tc::MIN_CHUNK;
  const int n = by_ctx < n_target ? by_ctx : n_target;
  return n < 1 ? 1 : n;
}

int launch_verify_tc(const void* tmap_k, const void* tmap_v, const void* q, int T, int H, int Hk, int layer, int ctx,
                     const int32_t* rows_dev, const int32_t* ctx_dev, const uint32_t* mask, int mask_words,
                     __half* ws_o, float* ws_lse, int n_chunks, int n_target, void* merge_out, int* merge_counters,
                     cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc::verify_attn_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_ALLOC);
    cudaFuncSetAttribute(tc::verify_attn_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_ALLOC);
    attr_set = true;
  }
  tc::Params p;
  p.q = (const __nv_bfloat16*)q;
  p.T = T;
  p.H = H;
  p.G = H / Hk;
  p.layer = layer;
  p.ctx = ctx;
  p.n_target = n_target;
  p.rows_dev = rows_dev;
  p.ctx_dev = ctx_dev;
  p.mask = mask;
  p.mask_words = mask_words;
  p.ws_o = ws_o;
  p.ws_lse = ws_lse;
  p.merge_out = (__nv_bfloat16*)merge_out;
  p.merge_counters = merge_counters;
  const int groups = (p.G * T + tc::ROWS - 1) / tc::ROWS;
  dim3 grid(n_chunks, Hk, groups);
  CUtensorMap mk, mv;
  memcpy(&mk, tmap_k, sizeof(CUtensorMap));
  memcpy(&mv, tmap_v, sizeof(CUtensorMap));
  if (merge_out)
    launch_pdl(tc::verify_attn_tc_kernel<true>, grid, dim3(tc::THREADS), tc::SMEM_ALLOC, st, mk, mv, p);
  else
    launch_pdl(tc::verify_attn_tc_kernel<false>, grid, dim3(tc::THREADS), tc::SMEM_ALLOC, st, mk, mv, p);
  return check_launch("sd_attention(tcgen05)");
}

}  // namespace sd
