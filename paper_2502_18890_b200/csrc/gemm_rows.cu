// Few-row weight streaming for the verification forward's projections
// (reference: TinyTransformer.forward's QKV / O projections over the tree rows,
// model.py:283-285, 306-309): y[S][T][N] = split-K slices of x[T][K] . W[K][N],
// W bf16 row-major [in, out] as the reference stores it, x bf16, fp32 accumulate.
// The consumers (sd_rope_stage, sd_add_rmsnorm) sum the S slices in slice order.
//
// The tree has at most 101 rows (41 at the default tree), so the projection is a
// weight stream like the single-row draft projections (gemv.cu): each CTA owns
// 256 output columns and a slice of K; one producer thread keeps a ring of
// stages in flight, each stage = 64 weight rows x 256 columns (four 128-byte-
// swizzled TMA boxes straight from the row-major weight, 32 KB) + the live x
// rows for those 64 k (K-major boxes of 16 rows, <= 14 KB, read from L2).
// Swap-AB on the 5th-generation tensor cores: M = 128 output columns (A = the
// weight boxes, MN-major), N = the live rows rounded up to 16 (B = the x boxes,
// K-major), fp32 accumulators in TMEM (lane = column, TMEM column = row), two
// M-tiles per stage issued by one thread, stage released by tcgen05.commit. The
// legacy warp-level path (mma.sync) was measured first: at 48 rows its issue
// rate caps the stream at ~3.3 TB/s; the tcgen05 MMAs of a stage take ~200
// cycles against the ~2000 the stage's bytes take to arrive.
//
// Launched as a programmatic dependent: the weight stages are requested before
// griddepcontrol.wait (weights do not depend on the previous kernel), x and the
// live row count (tree record) after it. Only live rows are computed and
// written; rows >= live in y keep stale values, as padded rows of a library GEMM
// would hold garbage-in-garbage-out values (nothing reads them).
#include <unordered_map>

#include "tc_common.cuh"

namespace sd {
namespace gr2 {

using namespace ::sd::tc;

constexpr int COLS = 256;                 // output columns per CTA (two M=128 tiles)
constexpr int TR = 64;                    // k rows per stage
constexpr int WARPS = 8;                  // warp 0: MMA issuer; all 8: epilogue
constexpr int NS = 4;                     // ring depth
constexpr int MAXM = 112;                 // live rows at most (MMA N <= 112)
constexpr int W_BOX = TR * 128;           // 8 KB: [64 k][64 n] bf16, 128B swizzle (MN-major A atom rows)
constexpr int W_BYTES = 4 * W_BOX;        // 32 KB
constexpr int X_BOX = 16 * 128;           // 2 KB: [16 rows][64 k] bf16, 128B swizzle (K-major B)
constexpr int X_BYTES = (MAXM / 16) * X_BOX;  // 14 KB
constexpr int STAGE = W_BYTES + X_BYTES;  // 46 KB (multiple of 1 KB)
constexpr int SMEM_ALLOC = NS * STAGE + 1024;
constexpr uint32_t TMEM_COLS = 256;       // accumulator of M-tile j at column 128 j
static_assert(STAGE % 1024 == 0, "stage alignment");

// A (weights) MN-major: two 64-column boxes per M-tile, LBO = box stride; B K-major
constexpr uint32_t idesc_rows(int n) { return idesc_bf16(n, false, 128) | (1u << 15); }

__global__ void __launch_bounds__((WARPS + 1) * 32, 1)
    gemm_rows_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap, int T,
                     int K, int N, int splits, const int32_t* __restrict__ rows_dev, float* __restrict__ y) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[NS], empty[NS], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cb = blockIdx.x, split = blockIdx.y;
  const int nbox = K / TR;
  const int b0 = (int)((int64_t)split * nbox / splits), b1 = (int)((int64_t)(split + 1) * nbox / splits);
  const int nst = b1 - b0;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 2);  // weights + x, each an arrive with its transaction bytes
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_trigger();
  if (warp == WARPS) {  // ================= producer =================
    if (lane == 0) {
      tma_prefetch(&wmap);
      tma_prefetch(&xmap);
      const int pre = nst < NS ? nst : NS;
      for (int i = 0; i < pre; ++i) {  // weights first: independent of the previous kernel
        uint8_t* st = smem + i * STAGE;
        mbar_expect_tx(&full[i], W_BYTES);
        const int k = (b0 + i) * TR;
        for (int b = 0; b < 4; ++b) tma_load_2d(st + b * W_BOX, &wmap, &full[i], cb * COLS + b * 64, k);
      }
      pdl_wait();  // x (and the tree record's row count) come from earlier kernels
      const int rows = rows_dev ? min(*rows_dev, T) : T;
      const int mtn = (rows + 15) >> 4;
      for (int i = 0; i < nst; ++i) {
        const int s = i % NS;
        uint8_t* st = smem + s * STAGE;
        const int k = (b0 + i) * TR;
        if (i >= NS) {
          mbar_wait(&empty[s], ((i / NS) - 1) & 1);
          mbar_expect_tx(&full[s], W_BYTES);
          for (int b = 0; b < 4; ++b) tma_load_2d(st + b * W_BOX, &wmap, &full[s], cb * COLS + b * 64, k);
        }
        mbar_expect_tx(&full[s], (uint32_t)mtn * X_BOX);
        for (int m = 0; m < mtn; ++m) tma_load_2d(st + W_BYTES + m * X_BOX, &xmap, &full[s], k, m * 16);
      }
    }
    return;
  }
  pdl_wait();
  const int rows = rows_dev ? min(*rows_dev, T) : T;
  const int mtn = (rows + 15) >> 4;
  if (warp == 0) {  // ================= MMA issuer =================
    __syncwarp();
    const bool leader = elect_one();
    const uint32_t idesc = idesc_rows(mtn * 16);
    for (int i = 0; i < nst; ++i) {
      const int s = i % NS;
      mbar_wait(&full[s], (i / NS) & 1);
      tc_fence_after();
      if (leader) {
        const uint32_t ws = smem_u32(smem + s * STAGE), xs = ws + W_BYTES;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int ks = 0; ks < TR / 16; ++ks)
            umma_bf16(tmem + 128 * mt, umma_desc(ws + mt * 2 * W_BOX + ks * 16 * 128, W_BOX, 1024),
                      umma_desc(xs + ks * 32, 16, 1024), idesc, (i > 0 || ks > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
        if (i == nst - 1) umma_commit(&done);
      }
      __syncwarp();
    }
  }
  // ================= epilogue: warp w reads M-tile w/4, TMEM lanes 32 (w % 4) .. + 31 =================
  mbar_wait(&done, 0);
  tc_fence_after();
  const int mt = warp >> 2, sp = warp & 3;
  const int col = cb * COLS + mt * 128 + sp * 32 + lane;
  float* ys = y + (int64_t)split * T * N + col;
  const uint32_t taddr = tmem + ((uint32_t)(sp * 32) << 16) + 128 * mt;
  uint32_t r[MAXM];  // every live accumulator column requested before one wait
#pragma unroll
  for (int c = 0; c < MAXM / 8; ++c)
    if (c < 2 * mtn) tmem_ld8(taddr + 8 * c, r + 8 * c);
  tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < MAXM; ++j)
    if (j < rows) ys[(int64_t)j * N] = __uint_as_float(r[j]);
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"n"(WARPS * 32) : "memory");  // consumers only (the producer warp returned)
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  return enc;
}

// 2-D map over a row-major bf16 [rows][cols] array, box {bc, br}, cached per (ptr, shape)
static int map2d(const void* p, int rows, int cols, int bc, int br, CUtensorMapSwizzle sw, CUtensorMap* out) {
  struct Key {
    const void* p;
    int r, c, bc;
    bool operator==(const Key& o) const { return p == o.p && r == o.r && c == o.c && bc == o.bc; }
  };
  struct H {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.p) ^ ((size_t)k.r << 20) ^ ((size_t)k.c << 40) ^ (size_t)k.bc;
    }
  };
  static std::unordered_map<Key, CUtensorMap, H> cache;
  const Key key{p, rows, cols, bc};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return SD_OK;
  }
  auto enc = encoder();
  SD_REQUIRE(enc, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("sd_gemm_rows: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SD_ECUDA;
  }
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return SD_OK;
}

static int splits_for(int K, int N) {
  const int blocks = N / COLS;
  int s = 148 / (blocks > 0 ? blocks : 1);
  static const int cap = getenv("SD_ROWS_MAX_SPLITS") ? atoi(getenv("SD_ROWS_MAX_SPLITS")) : 0;  // tuning only
  if (cap > 0 && s > cap) s = cap;
  if (s < 1) s = 1;
  if (s > K / TR) s = K / TR;
  return s;
}

}  // namespace gr2
}  // namespace sd

using namespace sd;

extern "C" {

int sd_gemm_rows_splits(int K, int N) { return gr2::splits_for(K, N); }

int sd_gemm_rows(const void* x, int T, int K, const void* w, int N, const int32_t* rows_dev, float* y,
                 sd_stream_t stream) {
  SD_REQUIRE(x && w && y, "sd_gemm_rows: null pointer");
  SD_REQUIRE(T >= 1 && T <= gr2::MAXM, "sd_gemm_rows: %d rows (1..%d)", T, gr2::MAXM);
  SD_REQUIRE(K % gr2::TR == 0 && K >= gr2::TR, "sd_gemm_rows: K=%d must be a multiple of %d", K, gr2::TR);
  SD_REQUIRE(N % gr2::COLS == 0, "sd_gemm_rows: N=%d must be a multiple of %d", N, gr2::COLS);
  SD_REQUIRE(((uintptr_t)x & 15) == 0 && ((uintptr_t)w & 15) == 0, "sd_gemm_rows: 16-byte aligned operands");
  CUtensorMap wm, xm;
  int rc = gr2::map2d(w, K, N, 64, gr2::TR, CU_TENSOR_MAP_SWIZZLE_128B, &wm);  // box [64 k][64 n]
  if (rc) return rc;
  rc = gr2::map2d(x, T, K, 64, 16, CU_TENSOR_MAP_SWIZZLE_128B, &xm);  // box [16 rows][64 k]
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gr2::gemm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gr2::SMEM_ALLOC);
    attr = true;
  }
  const int s = gr2::splits_for(K, N);
  launch_pdl(gr2::gemm_rows_kernel, dim3(N / gr2::COLS, s), dim3((gr2::WARPS + 1) * 32), gr2::SMEM_ALLOC,
             (cudaStream_t)stream, wm, xm, T, K, N, s, rows_dev, y);
  return check_launch("sd_gemm_rows");
}

}  // extern "C"
