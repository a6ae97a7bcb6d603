// Weight-streaming GEMM for the decode step's dense layers on the 5th-generation
// tensor cores (sm_100a):  Y[M, N] = X[M, K] . W[K, N], bf16 in, fp32 accumulate.
//
// Reference: the projections of TinyTransformer.forward (model.py:283-285 q/k/v,
// 306 o, 307-309 non-gated SiLU MLP) — x @ w with w stored [in, out]. Decode
// forwards have few rows (1 draft row; 101 padded verify rows), so every layer is
// a stream of its weights: the kernel is HBM-bound and is built to keep HBM
// busy — persistent CTAs (one per SM) walk (128-column N-tile, K split) work
// items with the TMA stream running on across items, a 10-deep TMA ring of weight tiles (160 KB in flight per SM; the
// bare stream needs >= 128 KB to reach 6 TB/s, tools/tma_bench.cu) beside a
// 4-deep ring of activation tiles sized to the live rows, one MMA thread
// (M=128, N=128, K=16 per instruction, A = X K-major, B = W MN-major straight
// from the weight), two TMEM accumulators so an item's epilogue overlaps the
// next item's MMAs. Weights are stored N-tiled,
// [N/128][K][128], so each CTA's weight stream is one contiguous run (the
// row-major [K][N] stripe of a tile touches only 256 B per 8-32 KB row). Split-K
// partials go out as [S][M][N] slices that the consumer (sd_add_rmsnorm /
// sd_rope_stage) sums in fixed split order — deterministic, no extra pass. The
// SiLU of the MLP is fused into the epilogue (that GEMM is never split).
#include "tc_common.cuh"

namespace sd {
namespace gm {

using namespace ::sd::tc;

constexpr int BM = 128, BN = 128, BK = 64;
// Ring depths are chosen per call from the row count: the X slot is sized to
// the live rows (1 KB at 1-8 rows, 13 KB at 101), the W ring takes the rest of
// shared memory (13 x 16 KB = 208 KB in flight per SM for the draft rows,
// 9 x 16 KB for the verify rows).
constexpr int WST_MAX = 14;
constexpr int XST_MAX = 16;  // the X loads queue behind the W loads in the SM's TMA unit: they need
                             // as much lookahead as W (16 x 1 KB at <= 8 rows; 6 x 13 KB at 101 rows)
constexpr int SILU_SPLIT_MAX_M = 16; // split-K SiLU (last CTA of a tile reduces) only for draft-sized M
constexpr int X_TILE = BM * BK * 2;  // 16 KB: [128 rows][64 K * 2 B] K-major SW128 (rows >= M unused)
constexpr int W_TILE = BK * BN * 2;  // 16 KB: [N half][64 K rows][128 B] MN-major SW128
constexpr int N_BAR = 2 * WST_MAX + 2 * XST_MAX + 4;
constexpr int RING_BYTES = 224 * 1024;                // W ring + X ring
constexpr int OFF_BAR = RING_BYTES;
constexpr int SMEM_ALLOC = OFF_BAR + N_BAR * 8 + 16 + 1024;
constexpr int THREADS = 224;  // warp 0 W TMA, warp 1 MMA, warps 2-5 epilogue (TMEM lane quarters 2,3,0,1), warp 6 X TMA
constexpr int EPI_THREADS = 128;

struct Params {
  int M, N, K, splits, epi;
  int x_rows;  // X box rows = M rounded up to 8 (rows >= M of the A tile are never stored)
  int wst;     // W ring depth
  int xst;     // X ring depth
  int x_slot;  // X slot bytes (x_rows * 128 rounded up to 1 KB). X ring first, W ring after it:
               // the MMA reads 128 A rows, so a short X slot's unused rows fall inside the W ring
  void* y;     // [splits][M][ldy] (fp32) or [M][ldy] (bf16 SiLU)
  int64_t ldy;
  float* ws;      // SiLU with splits > 1: fp32 partials [splits][M][N]
  int* counters;  // SiLU with splits > 1: per N-tile arrival counters (zero between launches)
};

__global__ void __launch_bounds__(THREADS, 1)
    gemm_stream_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                       Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* w_full = (uint64_t*)(smem + OFF_BAR);
  uint64_t* w_empty = w_full + WST_MAX;
  uint64_t* x_full = w_empty + WST_MAX;
  uint64_t* x_empty = x_full + XST_MAX;
  uint64_t* acc_full = x_empty + XST_MAX;  // [2]: accumulator b holds a finished work item
  uint64_t* acc_empty = acc_full + 2;  // [2]: epilogue has drained accumulator b
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = p.K / BK;
  const int n_items = (p.N / BN) * p.splits;  // item = (N-tile, split); CTA g takes g, g + G, ...
  const int G = gridDim.x, g = blockIdx.x;
  const int my_items = g < n_items ? (n_items - 1 - g) / G + 1 : 0;
  auto item_range = [&](int j, int& tile, int& split, int& k0, int& k1) {
    const int item = g + j * G;
    tile = item / p.splits;
    split = item - tile * p.splits;
    k0 = (int)((int64_t)split * nk / p.splits);
    k1 = (int)((int64_t)(split + 1) * nk / p.splits);
  };

  if (tid == 0) {
    for (int s = 0; s < p.wst; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < p.xst; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], EPI_THREADS);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the weights never depend on the kernel before,
  // so the W stream starts at once; X loads and every global store wait for it
  pdl_trigger();

  if (warp == 0 || warp == 6) {
    if (lane == 0) {  // ---- TMA producers: W (warp 0, deep ring) and X (warp 6), continuous across items ----
      const bool is_w = warp == 0;
      tma_prefetch(is_w ? &tmap_w : &tmap_x);
      if (!is_w) pdl_wait();
      const int depth = is_w ? p.wst : p.xst;
      uint8_t* x_ring = smem;
      uint8_t* w_ring = smem + p.xst * p.x_slot;
      uint64_t* full = is_w ? w_full : x_full;
      uint64_t* empty = is_w ? w_empty : x_empty;
      const uint32_t bytes = is_w ? W_TILE : (uint32_t)p.x_rows * BK * 2;
      int i = 0;
      for (int j = 0; j < my_items; ++j) {
        int tile, split, k0, k1;
        item_range(j, tile, split, k0, k1);
        for (int kk = k0; kk < k1; ++kk, ++i) {
          const int s = i % depth;
          if (i >= depth) mbar_wait(&empty[s], ((i / depth) + 1) & 1);
          mbar_expect_tx(&full[s], bytes);
          if (is_w) {
            uint8_t* st = w_ring + s * W_TILE;
            tma_load_3d(st, &tmap_w, &full[s], 0, kk * BK, 2 * tile);                // tile cols 0..63
            tma_load_3d(st + W_TILE / 2, &tmap_w, &full[s], 0, kk * BK, 2 * tile + 1);  // tile cols 64..127
          } else {
            tma_load_2d(x_ring + s * p.x_slot, &tmap_x, &full[s], kk * BK, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: accumulators alternate so the epilogue overlaps the next item ----
      const uint32_t idesc = idesc_bf16(BN, true);
      int i = 0;
      for (int j = 0; j < my_items; ++j) {
        int tile, split, k0, k1;
        item_range(j, tile, split, k0, k1);
        const int b = j & 1;
        if (j >= 2) mbar_wait(&acc_empty[b], ((j - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + BN * b;
        for (int kk = k0; kk < k1; ++kk, ++i) {
          const int s = i % p.wst, sx = i % p.xst;
          mbar_wait(&x_full[sx], (i / p.xst) & 1);
          mbar_wait(&w_full[s], (i / p.wst) & 1);
          tc_fence_after();
          const uint32_t xs = smem_u32(smem + sx * p.x_slot), ws = smem_u32(smem + p.xst * p.x_slot + s * W_TILE);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            const uint64_t a = umma_desc(xs + ks * 32, 16, 1024);
            const uint64_t bd = umma_desc(ws + ks * 16 * 128, W_TILE / 2, 1024);
            umma_bf16(acc, a, bd, idesc, (kk > k0 || ks > 0) ? 1u : 0u);
          }
          umma_commit(&w_empty[s]);
          umma_commit(&x_empty[sx]);
        }
        umma_commit(&acc_full[b]);
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    pdl_wait();  // y / partials / counters may still be in use by the kernel before
    // ---- epilogue: TMEM -> registers -> split slice (fp32) | silu (bf16) ----
    const int quarter = warp & 3;
    const int row = 32 * quarter + lane;
    for (int j = 0; j < my_items; ++j) {
      int tile, split, k0, k1;
      item_range(j, tile, split, k0, k1);
      const int b = j & 1, n0 = tile * BN;
      mbar_wait(&acc_full[b], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + BN * b + ((uint32_t)(32 * quarter) << 16);
#pragma unroll
      for (int q4 = 0; q4 < BN / 32; ++q4) {
        uint32_t r[32];
        tmem_ld32(taddr + 32 * q4, r);
        tmem_wait_ld();
        if (row < p.M) {
          const bool slice = p.epi == SD_GEMM_EPI_F32 || p.splits > 1;
          if (slice) {  // split slice `split` of the fp32 output (SiLU: of the workspace)
            float* base = p.epi == SD_GEMM_EPI_F32 ? (float*)p.y + ((int64_t)split * p.M + row) * p.ldy
                                                   : p.ws + ((int64_t)split * p.M + row) * p.N;
            float4* d4 = reinterpret_cast<float4*>(base + n0 + 32 * q4);
#pragma unroll
            for (int c = 0; c < 8; ++c)
              d4[c] = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                  __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
          } else {  // SiLU -> bf16 (model.py:308)
            uint4* d4 = reinterpret_cast<uint4*>((__nv_bfloat16*)p.y + row * p.ldy + n0 + 32 * q4);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float a0 = __uint_as_float(r[8 * c + 2 * e]), a1 = __uint_as_float(r[8 * c + 2 * e + 1]);
                const __nv_bfloat162 h = __floats2bfloat162_rn(a0 / (1.f + __expf(-a0)), a1 / (1.f + __expf(-a1)));
                w[e] = *reinterpret_cast<const uint32_t*>(&h);
              }
              d4[c] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[b]);
      if (p.epi != SD_GEMM_EPI_F32 && p.splits > 1) {
        // split SiLU (M <= 16): the last CTA to finish a slice of this tile sums
        // the slices in split order and applies the SiLU (deterministic)
        __shared__ int s_last;
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
        if (tid == 64) s_last = atomicAdd(&p.counters[tile], 1) == p.splits - 1;
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
        if (s_last) {
          __threadfence();
          const int c = tid - 64;
          for (int m = 0; m < p.M; ++m) {
            float a = 0.f;
            for (int t = 0; t < p.splits; ++t) a += __ldcg(p.ws + ((int64_t)t * p.M + m) * p.N + n0 + c);
            ((__nv_bfloat16*)p.y)[m * p.ldy + n0 + c] = __float2bfloat16_rn(a / (1.f + __expf(-a)));
          }
          if (c == 0) p.counters[tile] = 0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
  }
}

// split-K factor: the (N-tile x split) items spread over the persistent CTAs
// with the best balance (max items per CTA vs the mean), preferring fewer
// splits (each slice is read back by the consumer) at equal balance
static int splits_for(int M, int N, int K, int epi) {
  if (epi != SD_GEMM_EPI_F32 && M > SILU_SPLIT_MAX_M) return 1;  // the in-kernel SiLU reduce is for small M
  const int tiles = N / BN, nk = K / BK;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 12 && s <= nk / 4; ++s) {
    const int items = tiles * s;
    const int per = (items + 147) / 148;
    const double eff = (double)items / (per * 148.0) * (items < 148 ? 1.0 : 1.0);
    if (eff > best_eff + 0.03) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

// [K][N] row-major -> [N/128][2][K][64]: each 64-column half of an N-tile is one
// contiguous stream, so every TMA box is a contiguous 8 KB run
__global__ void tile_weight_kernel(const uint4* __restrict__ w, int K, int N, uint4* __restrict__ wt) {
  const int64_t total = (int64_t)K * N / 8;  // 16-byte chunks
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / (N / 8), n8 = i - k * (N / 8);
    const int64_t half = n8 / 8, c8 = n8 - half * 8;  // half = 2 * tile + (64-column half)
    wt[(half * K + k) * 8 + c8] = w[i];
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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

// 2-D bf16 map over a row-major [rows][cols] matrix, 64-column x box_rows boxes, 128-byte swizzle
static int make_map(const void* base, int rows, int cols, int box_rows, CUtensorMap* m) {
  auto enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SD_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SD_ECUDA;
  }
  return SD_OK;
}

static int make_tiled_weight_map(const void* wt, int K, int N, CUtensorMap* m) {
  auto enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SD_ECUDA;
  }
  cuuint64_t dims[3] = {64, (cuuint64_t)K, (cuuint64_t)(2 * N / BN)};
  cuuint64_t strides[2] = {128, (cuuint64_t)K * 128};
  cuuint32_t box[3] = {64, (cuuint32_t)BK, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(wt), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SD_ECUDA;
  }
  return SD_OK;
}

}  // namespace gm
}  // namespace sd

using namespace sd;

extern "C" {

int sd_tile_weight(const void* w, int K, int N, void* w_tiled, sd_stream_t stream) {
  SD_REQUIRE(w && w_tiled && K > 0 && N > 0 && K % gm::BK == 0 && N % gm::BN == 0,
             "sd_tile_weight: W [K=%d][N=%d] needs K %% 64 == 0 and N %% 128 == 0", K, N);
  gm::tile_weight_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>((const uint4*)w, K, N, (uint4*)w_tiled);
  return check_launch("sd_tile_weight");
}

int sd_make_weight_tmap(const void* w_tiled, int K, int N, void* tmap_out_host) {
  SD_REQUIRE(w_tiled && tmap_out_host && K > 0 && N > 0 && K % gm::BK == 0 && N % gm::BN == 0,
             "sd_make_weight_tmap: W [K=%d][N=%d] must be bf16 with K %% 64 == 0 and N %% 128 == 0", K, N);
  return gm::make_tiled_weight_map(w_tiled, K, N, reinterpret_cast<CUtensorMap*>(tmap_out_host));
}

int sd_gemm_splits(int M, int N, int K, int epi) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  return epi == SD_GEMM_EPI_F32 ? gm::splits_for(M, N, K, epi) : 1;  // slices the caller sees
}

size_t sd_gemm_workspace_bytes(int M, int N, int K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  const int s = gm::splits_for(M, N, K, SD_GEMM_EPI_SILU_BF16);
  if (s <= 1) return 0;
  return (size_t)4096 + (size_t)s * M * N * sizeof(float);  // fixed counter head: shapes may share a workspace
}

int sd_gemm(const void* x, int M, int K, const void* w_tmap_host, int N, int epi, void* y, int64_t ldy,
            void* workspace, size_t workspace_bytes, sd_stream_t stream) {
  SD_REQUIRE(x && w_tmap_host && y && M > 0 && M <= gm::BM, "sd_gemm: M=%d must be in [1, 128]", M);
  SD_REQUIRE(K % gm::BK == 0 && N % gm::BN == 0, "sd_gemm: K %% 64 and N %% 128");
  SD_REQUIRE(epi == SD_GEMM_EPI_F32 || epi == SD_GEMM_EPI_SILU_BF16, "sd_gemm: epilogue");
  SD_REQUIRE(ldy >= N && ((uintptr_t)y % 16) == 0 && (ldy % 8) == 0, "sd_gemm: output row stride / alignment");
  SD_REQUIRE(((uintptr_t)x % 16) == 0, "sd_gemm: X must be 16-byte aligned");
  const size_t need = epi == SD_GEMM_EPI_F32 ? 0 : sd_gemm_workspace_bytes(M, N, K);
  SD_REQUIRE(need == 0 || (workspace && workspace_bytes >= need), "sd_gemm: workspace too small");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gm::gemm_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gm::SMEM_ALLOC);
    attr = true;
  }
  CUtensorMap mx, mw;
  const int x_rows = (M + 7) / 8 * 8;
  int rc = gm::make_map(x, M, K, x_rows, &mx);
  if (rc) return rc;
  memcpy(&mw, w_tmap_host, sizeof(CUtensorMap));
  gm::Params p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.splits = gm::splits_for(M, N, K, epi);
  p.epi = epi;
  p.x_rows = x_rows;
  p.x_slot = (x_rows * 128 + 1023) / 1024 * 1024;
  p.xst = p.x_slot <= 2048 ? gm::XST_MAX : 6;
  p.wst = (gm::RING_BYTES - p.xst * p.x_slot) / gm::W_TILE;
  if (p.wst > gm::WST_MAX) p.wst = gm::WST_MAX;
  p.y = y;
  p.ldy = ldy;
  p.counters = (int*)workspace;
  SD_REQUIRE((N / gm::BN) * sizeof(int) <= 4096, "sd_gemm: N too wide for the counter head");
  p.ws = need ? (float*)((char*)workspace + 4096) : nullptr;
  const int items = (N / gm::BN) * p.splits;
  dim3 grid(items < 148 ? items : 148);
  launch_pdl(gm::gemm_stream_kernel, grid, dim3(gm::THREADS), gm::SMEM_ALLOC, as_stream(stream), mx, mw, p);
  return check_launch("sd_gemm");
}

}  // extern "C"
