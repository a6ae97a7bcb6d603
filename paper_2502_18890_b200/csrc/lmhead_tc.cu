// Verification LM head fused with the first pass of the penalised sampler
// on the 5th-generation tensor cores:
//
//   s[r][v] = penalise(h0[r] . embed[v]) / temperature        (engine.py:237-245,
//             sampling.py:98-153: Eq. 3 on the row's window + tree branch)
//   stats[r][t] = (max_v s, sum_v exp(s - max)) over 128-token tile t
//
// The tied head is embed [V][d] (model.py:312 `h0 @ embed.T`). The kernel
// streams the 1.05 GB cfg3 embedding once per verification (HBM-bound), from a
// box-contiguous copy (sd_tile_lmhead: [V/128][d/64][128][64], every 16 KB TMA box
// one contiguous run). Persistent CTAs (one per SM) take 128-token tiles round
// robin, two tiles per pass sharing each h0 box (the last pass or two single, to
// keep the exposed epilogue short). Swap-AB MMA: M = 128 tokens (A = embedding box,
// K-major), N = the h0 rows rounded up to 16 (B = h0 box), fp32 accumulators in
// TMEM (lane = token, column = row), double-buffered so the epilogue of pass j
// overlaps the MMAs of pass j+1. Epilogue (4 warps, thread = token): the row's
// penalty membership (window count of the token, overridden by a shared-memory
// table of the tokens the tree rows' window splices patch, with row bitmasks),
// the scaled fp32 logits (coalesced: a warp writes 32 consecutive tokens of a
// row), and per-row tile statistics through a padded shared-memory transpose; the
// four warps' partials are combined in a fixed order. sd_sample_rows with
// SD_IN_SCALED_F32 then skips its first pass: every CTA of a row's cluster
// combines the row's tile statistics in the same order (same Z everywhere) and
// only re-reads the scaled logits it owns. Measured (tools/lmhead_bench.py, cfg3
// T=101 with 41 live rows): 203-212 us for the LM head + statistics against
// cuBLAS's 199 us plain GEMM, 256-260 us with the sampler against 274-277 us.
#include "sample_common.cuh"
#include "tc_common.cuh"

namespace sd {
namespace lh {

using namespace ::sd::tc;

// Swap-AB: the MMA's M side is 128 vocabulary entries (A = an embedding box,
// K-major straight from embed [V][d]) and its N side the h0 rows (B = an h0 box,
// N = rows rounded up to 16): one h0 box feeds the MMAs of TWO vocabulary tiles,
// so per k-block a CTA pulls 2 x 16 KB of embedding (HBM) and one <= 16 KB h0 box
// (L2) instead of an h0 box per 16 KB. Accumulators: TMEM lane = vocabulary
// entry, column = row.
constexpr int BV = 128, BK = 64;
constexpr int WST_MAX = 10, XST = 3;
constexpr int TBUF_BYTES = 4 * 32 * 33 * 4;
constexpr int W_TILE = BV * BK * 2;  // 16 KB: [128 tokens][64 K] K-major SW128
constexpr int N_BAR = 2 * WST_MAX + 2 * XST + 4;
constexpr int THREADS = 224;  // warp 0 embedding TMA, warp 1 MMA, warps 2-5 epilogue, warp 6 h0 TMA
constexpr int EPI_THREADS = 128;
constexpr int BLOOM_WORDS = 512;  // 16384-bit filter of every live row's patched tokens
constexpr int PATCH_INTS = 1 + 2 * MAX_PATCH;  // per row: n, tok[MAX_PATCH], val[MAX_PATCH] (setup only)
// patched tokens, each with the rows that patch it and the patched membership
// (bit r of word r/32); at most one new token per row beyond the window drops
struct PatchTok {
  int tok;
  uint32_t rows[4], val[4];
};
constexpr int SMEM_BUDGET = 227 * 1024;

struct Params {
  int M, K, V, tiles, n_rows;  // n_rows: MMA N (rows rounded up to 16)
  int wst, x_slot;
  int off_w, off_scr, off_bloom, off_utab, off_tbuf, off_bar;
  int utab_cap;
  float* logits;   // [M][V] scaled, penalised
  double* stats;   // [M][tiles][2]
};

__device__ __forceinline__ int live_rows(const SampleDev& a, int M) {
  if (a.member_kind == SD_MEMBER_TREE) {
    const int t = a.tree[tree_off::T];
    return t < M ? t : M;
  }
  return M;
}

// a CTA's tiles (round robin, n of them) go in passes of two sharing each h0 box,
// except that the last one or two passes take one tile each: the epilogue of the
// final pass is the kernel's exposed tail
struct PassPlan {
  int pairs, passes;
  __device__ PassPlan(int n) {
    const int singles = n == 0 ? 0 : (n % 2 == 1 ? 1 : (n >= 2 ? 2 : 1));
    pairs = (n - singles) / 2;
    passes = pairs + singles;
  }
  __device__ int first(int j) const { return j < pairs ? 2 * j : 2 * pairs + (j - pairs); }
  __device__ int count(int j) const { return j < pairs ? 2 : 1; }
};

// ctrl-style penalty of a member (sampling.py Eq. 3 variant): out of line, the
// IEEE division keeps the unfused sampler's arithmetic
static __device__ __noinline__ float scale_ctrl(float l, float inv_t, float th) {
  return (l < 0.f ? l * th : l / th) * inv_t;
}

__global__ void __launch_bounds__(THREADS, 1)
    lmhead_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w, Params p,
                  SampleDev a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* x_ring = smem;
  uint8_t* w_ring = smem + p.off_w;
  float2* scr = (float2*)(smem + p.off_scr);           // [2 parity][4 quarters][128 rows] (max, sum)
  uint32_t* bloom = (uint32_t*)(smem + p.off_bloom);  // [BLOOM_WORDS]
  PatchTok* utab = (PatchTok*)(smem + p.off_utab);   // [utab_cap] + count in utab_n
  float* tbuf = (float*)(smem + p.off_tbuf);          // [4 warps][32 rows][33]; setup: per-row patches
  int* patch = (int*)tbuf;                            // [M][PATCH_INTS], setup only

  uint64_t* bars = (uint64_t*)(smem + p.off_bar);
  uint64_t* w_full = bars;
  uint64_t* w_empty = w_full + WST_MAX;
  uint64_t* x_full = w_empty + WST_MAX;
  uint64_t* x_empty = x_full + XST;
  uint64_t* acc_full = x_empty + XST;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
  int* utab_n = (int*)(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = p.K / BK;
  const int G = gridDim.x, g = blockIdx.x;
  const int my_tiles = g < p.tiles ? (p.tiles - 1 - g) / G + 1 : 0;
  const PassPlan plan(my_tiles);
  const int my_passes = plan.passes;
  const int wst = p.wst;

  if (tid == 0) {
    for (int s = 0; s < wst; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < XST; ++s) {
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
                 "r"(4 * BV)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // the embedding stream never depends on the kernel before

  if (warp == 0 || warp == 6) {
    if (lane == 0) {  // ---- TMA producers: embedding boxes (warp 0), h0 boxes (warp 6) ----
      const bool is_w = warp == 0;
      tma_prefetch(is_w ? &tmap_w : &tmap_x);
      if (!is_w) pdl_wait();
      int iw = 0, ix = 0;
      for (int j = 0; j < my_passes; ++j) {
        const int t0 = g + plan.first(j) * G;
        const int nt = plan.count(j);
        for (int kk = 0; kk < nk; ++kk) {
          if (is_w) {
            for (int u = 0; u < nt; ++u, ++iw) {
              const int s = iw % wst;
              if (iw >= wst) mbar_wait(&w_empty[s], ((iw / wst) + 1) & 1);
              mbar_expect_tx(&w_full[s], W_TILE);
              tma_load_3d(w_ring + s * W_TILE, &tmap_w, &w_full[s], 0, 0, (t0 + u * G) * nk + kk);  // contiguous 16 KB
            }
          } else {
            const int s = ix % XST;
            if (ix >= XST) mbar_wait(&x_empty[s], ((ix / XST) + 1) & 1);
            mbar_expect_tx(&x_full[s], (uint32_t)p.n_rows * BK * 2);
            tma_load_2d(x_ring + s * p.x_slot, &tmap_x, &x_full[s], kk * BK, 0);
            ++ix;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: D[vocab][row] += E_box . h0_box^T ----
      const uint32_t idesc = idesc_bf16(p.n_rows, false);
      int iw = 0, ix = 0;
      for (int j = 0; j < my_passes; ++j) {
        const int nt = plan.count(j);
        const int b = j & 1;
        if (j >= 2) mbar_wait(&acc_empty[b], ((j - 2) >> 1) & 1);
        tc_fence_after();
        for (int kk = 0; kk < nk; ++kk, ++ix) {
          const int sx = ix % XST;
          mbar_wait(&x_full[sx], (ix / XST) & 1);
          const uint32_t xs = smem_u32(x_ring + sx * p.x_slot);
          for (int u = 0; u < nt; ++u, ++iw) {
            const int s = iw % wst;
            mbar_wait(&w_full[s], (iw / wst) & 1);
            tc_fence_after();
            const uint32_t ws = smem_u32(w_ring + s * W_TILE);
            const uint32_t acc = tmem + 2 * BV * b + BV * u;
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks)
              umma_bf16(acc, umma_desc(ws + ks * 32, 16, 1024), umma_desc(xs + ks * 32, 16, 1024), idesc,
                        (kk > 0 || ks > 0) ? 1u : 0u);
            umma_commit(&w_empty[s]);
          }
          umma_commit(&x_empty[sx]);
        }
        umma_commit(&acc_full[b]);
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ---- epilogue: thread = one vocabulary entry of the tile (TMEM lane), rows along columns ----
    const int quarter = warp & 3;
    const int et = tid - 64;  // 0..127
    pdl_wait();  // tree record / window / state come from the kernels before
    const int rows = live_rows(a, p.M);
    // per-row window splice (row_setup) -> per-row patch lists -> one table of the
    // patched tokens with row bitmasks, plus a filter so a tile's threads skip the lookup
    for (int i = et; i < BLOOM_WORDS; i += EPI_THREADS) bloom[i] = 0u;
    if (et < rows) {
      RowCtx rc;
      row_setup(a, et, rc);
      int* pr = patch + et * PATCH_INTS;
      pr[0] = rc.n_patch;
      for (int i = 0; i < rc.n_patch; ++i) {
        pr[1 + i] = rc.patch_tok[i];
        pr[1 + MAX_PATCH + i] = rc.patch_val[i];
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
    if (et == 0) {  // serial: a few dozen entries
      int n = 0;
      for (int r = 0; r < rows; ++r) {
        const int* pr = patch + r * PATCH_INTS;
        for (int i = 0; i < pr[0]; ++i) {
          const int t = pr[1 + i];
          int k = 0;
          while (k < n && utab[k].tok != t) ++k;
          if (k == n) {
            if (n == p.utab_cap) continue;  // cannot happen: <= rows + 2 * depth distinct tokens
            utab[n].tok = t;
            for (int w = 0; w < 4; ++w) utab[n].rows[w] = utab[n].val[w] = 0u;
            bloom[(t >> 5) & (BLOOM_WORDS - 1)] |= 1u << (t & 31);
            ++n;
          }
          utab[k].rows[r >> 5] |= 1u << (r & 31);
          if (pr[1 + MAX_PATCH + i]) utab[k].val[r >> 5] |= 1u << (r & 31);
        }
      }
      *utab_n = n;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
    const int n_utab = *utab_n;
    const bool tree = a.member_kind == SD_MEMBER_TREE, win = a.member_kind >= SD_MEMBER_WINDOW && a.window > 0;
    const float inv_t = (float)(1.0 / a.temperature), inv_tt = (float)(1.0 / (a.temperature * a.theta));
    const float th = (float)a.theta;
    const int ctrl = a.ctrl_style;
    int it = 0;  // tiles done (scratch parity)
#ifdef LH_EXP_TIME
    long long tr[12];
    int ntr = 0;
    auto gt = []() { long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; };
    const long long tk0 = gt();
#define LH_T0()
#define LH_T(k) do { if ((k) == 0 || (k) == 4) { if (ntr < 12) tr[ntr++] = gt() - tk0; } } while (0)
#else
#define LH_T0()
#define LH_T(k)
#endif
    for (int j = 0; j < my_passes; ++j) {
      const int nt = plan.count(j);
      const int b = j & 1;
      LH_T0();
      mbar_wait(&acc_full[b], (j >> 1) & 1);
      tc_fence_after();
      LH_T(0);
      for (int u = 0; u < nt; ++u, ++it) {
        const int tile = g + (plan.first(j) + u) * G;
        const int v = tile * BV + 32 * quarter + lane;  // this thread's TMEM lane
        const bool vok = v < p.V;
        const int base = (win && vok) ? (a.win_count[v] > 0) : 0;
        // rows whose branch / window splice patches token v (rare: filter first)
        uint32_t pr0 = 0, pr1 = 0, pr2 = 0, pr3 = 0, pv0 = 0, pv1 = 0, pv2 = 0, pv3 = 0;
        if (tree && vok && ((bloom[(v >> 5) & (BLOOM_WORDS - 1)] >> (v & 31)) & 1u)) {
          for (int k = 0; k < n_utab; ++k)
            if (utab[k].tok == v) {
              pr0 = utab[k].rows[0], pr1 = utab[k].rows[1], pr2 = utab[k].rows[2], pr3 = utab[k].rows[3];
              pv0 = utab[k].val[0], pv1 = utab[k].val[1], pv2 = utab[k].val[2], pv3 = utab[k].val[3];
            }
        }
        float2* sc = scr + (it & 1) * 4 * 128;
        const uint32_t taddr = tmem + 2 * BV * b + BV * u + ((uint32_t)(32 * quarter) << 16);
        float* tb = tbuf + quarter * 32 * 33;  // this warp's [32 rows][33] transpose buffer
        for (int r0 = 0; r0 < rows; r0 += 32) {
          const int nr = rows - r0 < 32 ? rows - r0 : 32;
          const uint32_t prw = r0 == 0 ? pr0 : r0 == 32 ? pr1 : r0 == 64 ? pr2 : pr3;
          const uint32_t pvw = r0 == 0 ? pv0 : r0 == 32 ? pv1 : r0 == 64 ? pv2 : pv3;
          // scaled logits of rows r0.. for this thread's token, 8 TMEM columns at a time
          for (int g8 = 0; g8 < nr; g8 += 8) {
            uint32_t r[8];
            tmem_ld8(taddr + r0 + g8, r);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int row = r0 + g8 + k;
              const float l = __uint_as_float(r[k]);
              // scaled_w of sample_rows_cluster_kernel (same float arithmetic)
              const int bit = (g8 + k) & 31;
              const int m = ((prw >> bit) & 1u) ? (int)((pvw >> bit) & 1u) : base;
              float sv = l * (m ? inv_tt : inv_t);
              if (ctrl && m) sv = scale_ctrl(l, inv_t, th);
              if (vok && row < rows) p.logits[(int64_t)row * p.V + v] = sv;  // 32 consecutive v per warp
              tb[(g8 + k) * 33 + lane] = vok ? sv : -INFINITY;
            }
          }
          __syncwarp();
          // row statistics over the warp's 32 tokens: lane i reads row r0 + i back from
          // the transpose buffer (padded rows: conflict-free both ways)
          if (lane < nr) {
            const float* rp = tb + lane * 33;
            float m = -INFINITY;
#pragma unroll 8
            for (int k = 0; k < 32; ++k) m = fmaxf(m, rp[k]);
            float z = 0.f;
            if (m != -INFINITY) {
#pragma unroll 8
              for (int k = 0; k < 32; ++k) z += __expf(rp[k] - m);
            }
            sc[quarter * 128 + r0 + lane] = make_float2(m, z);
          }
          __syncwarp();
        }
        if (u == nt - 1) {  // both accumulators of the pass drained
          tc_fence_before();
          mbar_arrive(&acc_empty[b]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
        if (et < rows) {  // combine the four quarters in a fixed order
          double m = -INFINITY;
          for (int q = 0; q < 4; ++q) m = fmax(m, (double)sc[q * 128 + et].x);
          double z = 0.0;
          for (int q = 0; q < 4; ++q) {
            const float2 w = sc[q * 128 + et];
            if (w.x != -INFINITY) z += (double)(w.y * __expf(w.x - (float)m));
          }
          reinterpret_cast<double2*>(p.stats)[(int64_t)et * p.tiles + tile] = make_double2(m, z);
        }
        LH_T(4);
      }
    }
#ifdef LH_EXP_TIME
    if (et == 0) {
      double* o = p.stats + (int64_t)g * 16;
      int pc = 0;
      for (int i = 0; i < BLOOM_WORDS; ++i) pc += __popc(bloom[i]);
      o[14] = pc;
      o[0] = my_tiles;
      o[1] = ntr;
      for (int k = 0; k < ntr; ++k) o[2 + k] = (double)tr[k];
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(4 * BV) : "memory");
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

// 2-D bf16 map over a row-major [rows][cols] matrix: 64-column x box_rows boxes, SW128
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

// embed [V][K] -> [tiles][K/64][128][64]: every (vocabulary tile, k-block) box is
// one contiguous 16 KB run (a box of the row-major embedding touches 128 B of each
// of 128 rows 2*K bytes apart); rows past V are zero
__global__ void tile_embed_kernel(const uint4* __restrict__ e, int V, int K, uint4* __restrict__ out, int tiles) {
  const int nk = K / BK;
  const int64_t total = (int64_t)tiles * BV * K / 8;  // 16-byte chunks of the output
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i & 7);               // 16-byte chunk within the 128-byte row piece
    const int64_t rowpiece = i >> 3;           // (t * nk + kk) * 128 + r
    const int r = (int)(rowpiece % BV);
    const int64_t blk = rowpiece / BV;
    const int kk = (int)(blk % nk);
    const int64_t t = blk / nk;
    const int64_t v = t * BV + r;
    out[i] = v < V ? e[(v * K + (int64_t)kk * BK) / 8 + c8] : make_uint4(0u, 0u, 0u, 0u);
  }
}

static int make_tiled_map(const void* tiled, int V, int K, CUtensorMap* m) {
  auto enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SD_ECUDA;
  }
  const int tiles = (V + BV - 1) / BV;
  cuuint64_t dims[3] = {64, (cuuint64_t)BV, (cuuint64_t)tiles * (K / BK)};
  cuuint64_t strides[2] = {128, (cuuint64_t)BV * 128};
  cuuint32_t box[3] = {64, (cuuint32_t)BV, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(tiled), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SD_ECUDA;
  }
  return SD_OK;
}

}  // namespace lh
}  // namespace sd

using namespace sd;

extern "C" {

size_t sd_lmhead_tiled_bytes(int V, int K) {
  if (V <= 0 || K <= 0) return 0;
  return (size_t)((V + lh::BV - 1) / lh::BV) * lh::BV * K * 2;
}

int sd_tile_lmhead(const void* embed, int V, int K, void* tiled, sd_stream_t stream) {
  SD_REQUIRE(embed && tiled && V > 0 && K > 0 && K % lh::BK == 0 && ((uintptr_t)embed % 16) == 0 &&
                 ((uintptr_t)tiled % 16) == 0,
             "sd_tile_lmhead: embed [V=%d][K=%d] bf16, K %% 64 == 0, 16-byte aligned", V, K);
  const int tiles = (V + lh::BV - 1) / lh::BV;
  lh::tile_embed_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>((const uint4*)embed, V, K, (uint4*)tiled, tiles);
  return check_launch("sd_tile_lmhead");
}

int sd_make_lmhead_tmap(const void* tiled, int V, int K, void* tmap_out_host) {
  SD_REQUIRE(tiled && tmap_out_host && V > 0 && K > 0 && K % lh::BK == 0 && ((uintptr_t)tiled % 16) == 0,
             "sd_make_lmhead_tmap: tiled embedding of [V=%d][K=%d], K %% 64 == 0", V, K);
  return lh::make_tiled_map(tiled, V, K, reinterpret_cast<CUtensorMap*>(tmap_out_host));
}

int sd_lmhead_tiles(int V) { return V > 0 ? (V + lh::BV - 1) / lh::BV : 0; }

int sd_lmhead_sample_stats(const void* x, int M, int K, const void* embed_tmap_host, int V,
                           const sd_sample_args* args_host, float* logits, double* stats, sd_stream_t stream) {
  SD_REQUIRE(x && embed_tmap_host && args_host && logits && stats, "sd_lmhead_sample_stats: null argument");
  SD_REQUIRE(M > 0 && M <= 128 && K > 0 && K % lh::BK == 0 && V > 0,
             "sd_lmhead_sample_stats: M=%d in [1,128], K=%d %% 64", M, K);
  SD_REQUIRE(((uintptr_t)x % 16) == 0 && ((uintptr_t)logits % 16) == 0 && ((uintptr_t)stats % 16) == 0,
             "sd_lmhead_sample_stats: 16-byte alignment");
  const sd_sample_args& h = *args_host;
  SD_REQUIRE(h.V == V && h.temperature > 0.0 && h.theta >= 1.0, "sd_lmhead_sample_stats: sampler arguments");
  SD_REQUIRE(h.member_kind == SD_MEMBER_NONE || h.member_kind == SD_MEMBER_WINDOW || h.member_kind == SD_MEMBER_TREE,
             "sd_lmhead_sample_stats: membership kind");
  SD_REQUIRE(h.member_kind < SD_MEMBER_WINDOW || h.window == 0 || (h.win_count && h.state),
             "sd_lmhead_sample_stats: window");
  SD_REQUIRE(h.member_kind != SD_MEMBER_TREE || h.tree, "sd_lmhead_sample_stats: tree");
  SD_REQUIRE(h.positions || h.tree, "sd_lmhead_sample_stats: need positions or tree");
  lh::Params p;
  p.M = M;
  p.K = K;
  p.V = V;
  p.tiles = (V + lh::BV - 1) / lh::BV;
  p.n_rows = (M + 15) / 16 * 16;
  p.x_slot = p.n_rows * 128;  // multiple of 2 KB: SW128 atoms stay 1 KB aligned
  p.logits = logits;
  p.stats = stats;
  p.utab_cap = M + 2 * SD_TREE_MAX_DEPTH;
  const int utab_bytes = p.utab_cap * (int)sizeof(lh::PatchTok);
  SD_REQUIRE(M * lh::PATCH_INTS * 4 <= lh::TBUF_BYTES, "sd_lmhead_sample_stats: patch lists");
  const int rest = 2 * 4 * 128 * 8 + lh::BLOOM_WORDS * 4 + utab_bytes + lh::TBUF_BYTES + lh::N_BAR * 8 + 16 + 1024;
  const int x_bytes = lh::XST * p.x_slot;
  p.wst = (lh::SMEM_BUDGET - rest - x_bytes) / lh::W_TILE;
  if (p.wst > lh::WST_MAX) p.wst = lh::WST_MAX;
  SD_REQUIRE(p.wst >= 4, "sd_lmhead_sample_stats: shared memory");
  p.off_w = x_bytes;
  p.off_scr = p.off_w + p.wst * lh::W_TILE;
  p.off_bloom = p.off_scr + 2 * 4 * 128 * 8;
  p.off_utab = p.off_bloom + lh::BLOOM_WORDS * 4;
  p.off_tbuf = p.off_utab + utab_bytes;
  p.off_bar = (p.off_tbuf + lh::TBUF_BYTES + 7) / 8 * 8;
  const int smem = p.off_bar + lh::N_BAR * 8 + 16 + 1024;
  static int attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(lh::lmhead_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lh::SMEM_BUDGET);
    attr = lh::SMEM_BUDGET;
  }
  SD_REQUIRE(smem <= lh::SMEM_BUDGET, "sd_lmhead_sample_stats: shared memory %d", smem);
  CUtensorMap mx, mw;
  int rc = lh::make_map(x, M, K, p.n_rows, &mx);
  if (rc) return rc;
  memcpy(&mw, embed_tmap_host, sizeof(CUtensorMap));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dim3 grid(p.tiles < sms ? p.tiles : sms);
  launch_pdl(lh::lmhead_kernel, grid, dim3(lh::THREADS), (size_t)smem, as_stream(stream), mx, mw, p, to_dev(h));
  return check_launch("sd_lmhead_sample_stats");
}

}  // extern "C"
