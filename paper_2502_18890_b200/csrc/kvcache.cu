// Dynamic partial-KV maintenance: Eq. 2 scoring, the fused refresh (scores ->
// exact top-K with the reference's (-score, pos) order -> gather -> per-layer
// importance ring), mirror build, the per-step admit/evict (device-resident
// bookkeeping, launched inside the step's CUDA graph), and reconcile of
// accepted tree rows.
// Reference: kvcache.py:116-127 (reconcile), 215-225 (admit), 243-265
// (importance), 268-319 (prefill/mirror build), 332-354 (evict);
// engine.py:128-148 (per-layer body scores over pre-rotation keys), 280.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sd {

// ---------------------------------------------------------------- scores ----
// Eq. 2 dot products of one full-cache row, kv head by kv head. A warp covers
// RPW head rows per 16-byte load (LPH lanes per row, VEC elements per lane);
// a lane's VEC products are chained in ascending dim order, then summed by an
// xor butterfly inside its LPH-lane group. The fused refresh and
// sd_importance_scores share this exact tree, so per-head partials summed in
// ascending head order (the sharded refresh) equal the unsharded total bit for
// bit (reference sums every head, kvcache.py:264).
template <int DH, typename KT>
struct ScoreShape {
  static constexpr int ES = sizeof(KT);
  static constexpr int VEC = 16 / ES;            // elements per lane per load
  static constexpr int LPH = DH / VEC;           // lanes per head row
  static constexpr int RPW = 32 / LPH;           // head rows per warp-load
  static_assert(DH * ES >= 16 && LPH <= 32 && 32 % LPH == 0, "row must be >= 16 B and split evenly");
};

// U consecutive rows at once (loads of all U rows first); rows >= n_valid skipped
template <int DH, typename KT, int HKMAX, int U>
__device__ __forceinline__ void score_rows(const float* __restrict__ qg, const KT* __restrict__ Kl, int64_t head_stride,
                                           int64_t pos0, int n_valid, int Hk, int lane, float (&parts)[U][HKMAX]) {
  using S = ScoreShape<DH, KT>;
  constexpr int NL = (HKMAX + S::RPW - 1) / S::RPW;
  const int sub = lane / S::LPH, d0 = (lane % S::LPH) * S::VEC;
  uint4 raw[U][NL];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int it = 0; it < NL; ++it) {
      const int h = it * S::RPW + sub;
      raw[u][it] = make_uint4(0, 0, 0, 0);
      if (h < Hk && u < n_valid)
        raw[u][it] = __ldg(reinterpret_cast<const uint4*>(Kl + h * head_stride + (pos0 + u) * DH + d0));
    }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float p[NL];
#pragma unroll
    for (int it = 0; it < NL; ++it) {
      const int h = it * S::RPW + sub;
      const KT* e = reinterpret_cast<const KT*>(&raw[u][it]);
      float acc = 0.f;
      if (h < Hk) {
#pragma unroll
        for (int v = 0; v < S::VEC; ++v) acc = fmaf(qg[h * DH + d0 + v], to_f(e[v]), acc);
      }
#pragma unroll
      for (int o = S::LPH / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      p[it] = acc;
    }
#pragma unroll
    for (int h = 0; h < HKMAX; ++h) parts[u][h] = __shfl_sync(0xffffffffu, p[h / S::RPW], (h % S::RPW) * S::LPH);
  }
}

// grouped query per kv head, g summed in ascending order (kvcache.py:262-264)
__device__ __forceinline__ void load_grouped_query(const float* __restrict__ q, int H, int Hk, int dh, float* qg) {
  const int G = H / Hk;
  for (int i = threadIdx.x; i < Hk * dh; i += blockDim.x) {
    const int k = i / dh, d = i - k * dh;
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += q[(k * G + g) * dh + d];
    qg[i] = s;
  }
}

template <int HKMAX>
__device__ __forceinline__ float sum_heads(const float (&parts)[HKMAX], int Hk) {
  float t = parts[0];
#pragma unroll
  for (int h = 1; h < HKMAX; ++h)
    if (h < Hk) t += parts[h];  // ascending head order
  return t;
}

// grid (ceil(n / 64), L), 256 threads: a warp scores 8 positions
template <int DH, typename KT, int HKMAX>
__global__ void __launch_bounds__(256) score_kernel(const float* __restrict__ q_sum, const KT* __restrict__ K,
                                                    int64_t layer_stride, int64_t head_stride, int H, int Hk,
                                                    int start, int end, float* __restrict__ scores,
                                                    float* __restrict__ per_head) {
  extern __shared__ float qg[];  // [Hk][DH]
  const int layer = blockIdx.y;
  load_grouped_query(q_sum + (int64_t)layer * H * DH, H, Hk, DH, qg);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = end - start;
  const KT* Kl = K + layer * layer_stride;
  for (int r = 0; r < 8; r += 4) {
    const int i0 = blockIdx.x * 64 + warp * 8 + r;
    if (i0 >= n) break;
    float parts[4][HKMAX];
    score_rows<DH, KT, HKMAX, 4>(qg, Kl, head_stride, start + i0, n - i0, Hk, lane, parts);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u;
      if (i >= n) break;
      if (per_head && lane < Hk) {
#pragma unroll
        for (int h = 0; h < HKMAX; ++h)
          if (h == lane) per_head[((int64_t)layer * Hk + h) * n + i] = parts[u][h];
      }
      if (lane == 0 && scores) scores[(int64_t)layer * n + i] = sum_heads(parts[u], Hk);
    }
  }
}

__global__ void sum_head_scores_kernel(const float* __restrict__ per_head, int L, int Hk, int n,
                                       float* __restrict__ scores) {
  const int64_t total = (int64_t)L * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = idx / n, i = idx - l * n;
    float s = per_head[(l * Hk) * n + i];
    for (int k = 1; k < Hk; ++k) s += per_head[(l * Hk + k) * n + i];
    scores[idx] = s;
  }
}

// -------------------------------------------------------------- top-K ------
__device__ __forceinline__ uint32_t ord_f32(float f) {
  if (f == 0.0f) f = 0.0f;  // -0.0 ties with +0.0, as in the reference's comparison
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// larger key = better: higher score first, then lower position (kvcache.py:286)
__device__ __forceinline__ uint64_t sel_key(float score, int pos) {
  return ((uint64_t)ord_f32(score) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)pos);
}

constexpr int RF_CLUSTER = 4;     // CTAs per layer in the fused refresh
constexpr int RF_THREADS = 512;
constexpr int RF_MAX_TAKE = 8192;
constexpr int RF_UNROLL = 4;     // positions per warp iteration in the scoring phase
constexpr float QNAN = __builtin_nanf("");

struct RefreshArgs {
  const float* q_sum;        // [L][H][dh] (NULL with scores_in)
  const float* scores_in;    // [L][n] precomputed (sharded refresh) or NULL
  float* scores_ws;          // [L][n] scratch (scores_in == NULL)
  uint64_t* keys_ws;         // [L][take] scratch
  const void* fk;            // full K_raw
  const void* fv;            // full V
  int64_t f_ls, f_hs;        // full layer / head strides (elements)
  void* pk;
  void* pv;
  int64_t p_ls, p_hs;
  int32_t *ppos, *prank, *ring, *freel, *meta;
  float* pscore;
  int slot_cap;
  int H, Hk, n, sink, take;
};

// copy the K_raw / V rows of `pos` into partial slot `slot` (all kv heads);
// a warp moves 512 B per instruction
template <int DH, typename KT>
__device__ __forceinline__ void copy_rows(const RefreshArgs& a, int layer, int64_t pos, int slot, int Hk, int lane) {
  constexpr int RW = DH * (int)sizeof(KT) / 16;  // uint4 per head row
  const uint4* fk = reinterpret_cast<const uint4*>(static_cast<const KT*>(a.fk) + layer * a.f_ls);
  const uint4* fv = reinterpret_cast<const uint4*>(static_cast<const KT*>(a.fv) + layer * a.f_ls);
  uint4* pk = reinterpret_cast<uint4*>(static_cast<KT*>(a.pk) + layer * a.p_ls);
  uint4* pv = reinterpret_cast<uint4*>(static_cast<KT*>(a.pv) + layer * a.p_ls);
  const int64_t fhs = a.f_hs * (int64_t)sizeof(KT) / 16, phs = a.p_hs * (int64_t)sizeof(KT) / 16;
  for (int w = lane; w < Hk * RW; w += 32) {
    const int h = w / RW, c = w - h * RW;
    const uint4 k = __ldg(fk + h * fhs + pos * RW + c);
    const uint4 v = __ldg(fv + h * fhs + pos * RW + c);
    pk[h * phs + (int64_t)slot * RW + c] = k;
    pv[h * phs + (int64_t)slot * RW + c] = v;
  }
}

// Fused refresh (kvcache.py:243-297 via engine.py:128-148): one cluster of
// RF_CLUSTER CTAs per layer, each owning a contiguous 1/RF_CLUSTER of the
// candidate positions [sink, sink+n).
//   1. Eq. 2 score of every owned position (score_row), kept in scores_ws
//      (L2-resident), unless precomputed scores are given;
//   2. exact radix select of the take-th largest 64-bit key (score, ~pos):
//      8-bit digits from the top, per-CTA shared histograms summed through
//      distributed shared memory, stopping early once a digit bucket is taken
//      whole; keys are unique, so exactly `take` keys are >= the threshold;
//   3. compaction in ascending position order (cluster prefix over the CTAs'
//      counts): body entry j lands in slot sink + j (rank = slot, position
//      order), score kept, K_raw / V rows gathered by the CTA that owns it;
//   4. cluster rank 0 sorts the selected keys (bitonic, descending; key low
//      word = ~j, order-equivalent to ~pos among the selected) into the
//      layer's importance ring: ring[i] = slot of the i-th most important body
//      entry; the layer's meta is reset (count = hi = sink + take).
template <int DH, typename KT, int HKMAX>
__global__ void __cluster_dims__(RF_CLUSTER, 1, 1) __launch_bounds__(RF_THREADS)
    refresh_kernel(RefreshArgs a) {
  extern __shared__ __align__(16) uint8_t rf_smem[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(rf_smem);                         // [RF_MAX_TAKE] (rank 0 sort)
  float* qg = reinterpret_cast<float*>(rf_smem + RF_MAX_TAKE * 8);             // [Hk][DH]
  __shared__ uint32_t hist[2][256];
  __shared__ uint32_t tot[256];
  __shared__ uint32_t wsum[RF_THREADS / 32];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_k, s_done, s_total;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int layer = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = a.n, sink = a.sink, take = a.take, Hk = a.Hk;
  const int i0 = (int)((int64_t)n * rank / RF_CLUSTER), i1 = (int)((int64_t)n * (rank + 1) / RF_CLUSTER);
  const float* sc = a.scores_in ? a.scores_in + (int64_t)layer * n : a.scores_ws + (int64_t)layer * n;

  // ---- 1. scores ----
  if (!a.scores_in) {
    load_grouped_query(a.q_sum + (int64_t)layer * a.H * DH, a.H, Hk, DH, qg);
    __syncthreads();
    const KT* Kl = static_cast<const KT*>(a.fk) + layer * a.f_ls;
    float* out = a.scores_ws + (int64_t)layer * n;
    // RF_UNROLL positions per warp iteration: all their loads are issued before
    // the first dot product (RF_UNROLL x NL x 16 B in flight per lane)
    for (int i = i0 + warp * RF_UNROLL; i < i1; i += (RF_THREADS / 32) * RF_UNROLL) {
      float p[RF_UNROLL][HKMAX];
      score_rows<DH, KT, HKMAX, RF_UNROLL>(qg, Kl, a.f_hs, sink + i, i1 - i, Hk, lane, p);
#pragma unroll
      for (int u = 0; u < RF_UNROLL; ++u)
        if (lane == u && i + u < i1) out[i + u] = sum_heads(p[u], Hk);
    }
    __syncthreads();
  }

  // ---- 2. radix select of the take-th largest key ----
  uint64_t prefix = 0, pmask = 0, thresh = 0;
  if (take < n) {
    uint32_t k = (uint32_t)take;
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass, buf = pass & 1;
      if (tid < 256) hist[buf][tid] = 0;
      __syncthreads();
      for (int i = i0 + tid; i < i1; i += RF_THREADS) {
        const uint64_t key = sel_key(sc[i], sink + i);
        if ((key & pmask) == prefix) atomicAdd(&hist[buf][(key >> shift) & 255u], 1u);
      }
      cluster.sync();  // every CTA's histogram of this digit complete
      if (tid < 256) {
        uint32_t t = 0;
        for (int r = 0; r < RF_CLUSTER; ++r) t += cluster.map_shared_rank(&hist[buf][0], r)[tid];
        tot[tid] = t;
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t cum = 0;
        int b = 255;
        for (; b > 0; --b) {
          if (cum + tot[b] >= k) break;
          cum += tot[b];
        }
        s_prefix = prefix | ((uint64_t)b << shift);
        s_k = k - cum;
        s_done = (tot[b] == k - cum) ? 1u : 0u;  // the whole bucket is taken
      }
      __syncthreads();
      prefix = s_prefix;
      k = s_k;
      pmask |= (uint64_t)255 << shift;
      if (s_done) break;
    }
    thresh = prefix;  // lower digits zero: keys >= thresh are exactly the top `take`
  }

  // ---- 3. compaction in position order + gather ----
  const int len = i1 - i0;
  const int seg = (len + RF_THREADS - 1) / RF_THREADS;
  const int b0 = i0 + tid * seg, b1 = min(i1, b0 + seg);
  uint32_t cnt = 0;
  for (int i = b0; i < b1; ++i) cnt += sel_key(sc[i], sink + i) >= thresh;
  uint32_t v = cnt;  // block inclusive scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < RF_THREADS / 32 ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < RF_THREADS / 32) wsum[lane] = w;
    if (lane == RF_THREADS / 32 - 1) s_total = w;
  }
  cluster.sync();  // CTA totals published
  uint32_t base = 0;
  for (int r = 0; r < rank; ++r) base += *cluster.map_shared_rank(&s_total, r);
  uint32_t off = base + v - cnt + (warp ? wsum[warp - 1] : 0u);
  int32_t* lpos = a.ppos + (int64_t)layer * a.slot_cap;
  int32_t* lrank = a.prank + (int64_t)layer * a.slot_cap;
  float* lsc = a.pscore + (int64_t)layer * a.slot_cap;
  uint64_t* keys = a.keys_ws + (int64_t)layer * take;
  for (int i = b0; i < b1; ++i) {
    const float s = sc[i];
    if (sel_key(s, sink + i) >= thresh) {
      const int slot = sink + (int)off;
      lpos[slot] = sink + i;
      lrank[slot] = slot;
      lsc[slot] = s;
      keys[off] = ((uint64_t)ord_f32(s) << 32) | (uint64_t)(0xFFFFFFFFu - off);
      ++off;
    }
  }
  if (rank == 0) {
    for (int s = tid; s < sink; s += RF_THREADS) {
      lpos[s] = s;
      lrank[s] = s;
      lsc[s] = QNAN;
    }
    for (int s = sink + take + tid; s < a.slot_cap; s += RF_THREADS) {  // beyond the budget: holes
      lpos[s] = -1;
      lrank[s] = -1;
      lsc[s] = QNAN;
    }
  }
  __syncthreads();
  {
    const int j0 = (int)base, j1 = (int)(base + s_total);
    for (int j = j0 + warp; j < j1; j += RF_THREADS / 32) copy_rows<DH, KT>(a, layer, lpos[sink + j], sink + j, Hk, lane);
    if (rank == 0)
      for (int s = warp; s < sink; s += RF_THREADS / 32) copy_rows<DH, KT>(a, layer, s, s, Hk, lane);
  }
  __threadfence();
  cluster.sync();  // every key written (no DSMEM access after this point)
  if (rank != 0) return;

  // ---- 4. importance ring (rank 0) ----
  int N = 1;
  while (N < take) N <<= 1;
  for (int i = tid; i < N; i += RF_THREADS) sk[i] = i < take ? keys[i] : 0ull;
  __syncthreads();
  for (int kk = 2; kk <= N; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < N; i += RF_THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = sk[i], y = sk[ixj];
          if ((x < y) == ((i & kk) == 0)) {  // descending
            sk[i] = y;
            sk[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  int32_t* ring = a.ring + (int64_t)layer * a.slot_cap;
  for (int i = tid; i < take; i += RF_THREADS) ring[i] = sink + (int)(0xFFFFFFFFu - (uint32_t)(sk[i] & 0xFFFFFFFFull));
  if (tid == 0) {
    int32_t* m = a.meta + layer * SD_PM_WORDS;
    m[SD_PM_COUNT] = sink + take;
    m[SD_PM_HI] = sink + take;
    m[SD_PM_HEAD] = 0;
    m[SD_PM_LEN] = take;
    m[SD_PM_NFREE] = 0;
    m[SD_PM_ERR] = 0;
  }
}

// mirror (kvcache.py:300-319): slot s <- position s for s < upto (rank = s);
// the layer's ring lists the body newest first. grid (x, L)
template <int DH, typename KT>
__global__ void __launch_bounds__(256) mirror_kernel(RefreshArgs a, int upto) {
  const int layer = blockIdx.y, lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  int32_t* lpos = a.ppos + (int64_t)layer * a.slot_cap;
  int32_t* lrank = a.prank + (int64_t)layer * a.slot_cap;
  float* lsc = a.pscore + (int64_t)layer * a.slot_cap;
  int32_t* ring = a.ring + (int64_t)layer * a.slot_cap;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int s = gt; s < a.slot_cap; s += nt) {
    const bool live = s < upto;
    lpos[s] = live ? s : -1;
    lrank[s] = live ? s : -1;
    lsc[s] = QNAN;
    if (s < upto - a.sink) ring[s] = upto - 1 - s;
  }
  for (int s = gw; s < upto; s += nw) copy_rows<DH, KT>(a, layer, s, s, a.Hk, lane);
  if (gt == 0) {
    int32_t* m = a.meta + layer * SD_PM_WORDS;
    m[SD_PM_COUNT] = upto;
    m[SD_PM_HI] = upto;
    m[SD_PM_HEAD] = 0;
    m[SD_PM_LEN] = upto > a.sink ? upto - a.sink : 0;
    m[SD_PM_NFREE] = 0;
    m[SD_PM_ERR] = 0;
  }
}

// ------------------------------------------------------ admit / evict ------
constexpr int PS_MAX = 1024;  // entries moved each way per launch

struct StepArgs {
  const int32_t* result;  // device step result (engine) or NULL (a_host / first_pos_host)
  int a_host, first_pos_host, evict, protected_host, sink, budget;
  RefreshArgs r;
};

// One CTA per layer (kvcache.py:215-225 admit, 332-354 evict_to_budget, as
// called at engine.py:281-283): evict the over-budget tail of the layer's
// importance ring (slots become holes and go to the free stack), admit the `a`
// newly committed positions into free slots (or fresh slots at hi) at the ring
// head in position order, keep ranks a dense position order (survivors drop
// one rank per evicted entry with a smaller position), copy the new K_raw / V
// rows from the full cache. Reads the accepted count and base from the device
// step result inside the CUDA graph: no host round trip.
template <int DH, typename KT>
__global__ void __launch_bounds__(256) partial_step_kernel(StepArgs sa) {
  __shared__ int ev_slot[PS_MAX], ev_pos[PS_MAX], new_slot[PS_MAX];
  __shared__ int s_a, s_over, s_first, s_count_after, s_hi, s_bad;
  const RefreshArgs& a = sa.r;
  const int layer = blockIdx.x, tid = threadIdx.x, cap = a.slot_cap;
  int32_t* lpos = a.ppos + (int64_t)layer * cap;
  int32_t* lrank = a.prank + (int64_t)layer * cap;
  float* lsc = a.pscore + (int64_t)layer * cap;
  int32_t* ring = a.ring + (int64_t)layer * cap;
  int32_t* fl = a.freel + (int64_t)layer * cap;
  int32_t* m = a.meta + layer * SD_PM_WORDS;
  if (tid < 32) {  // warp 0: the ring / free-stack bookkeeping, lanes in parallel
    const int lane = tid;
    const int na = sa.result ? sa.result[SD_RES_ACCEPTED] : sa.a_host;
    const int first = sa.result ? sa.result[SD_RES_BASE] : sa.first_pos_host;
    const int prot = sa.result ? na : sa.protected_host;
    const int count = m[SD_PM_COUNT], hi0 = m[SD_PM_HI], head = m[SD_PM_HEAD], len = m[SD_PM_LEN];
    const int nfree = m[SD_PM_NFREE];
    int over = sa.evict ? count + na - sa.budget : 0;
    if (over < 0) over = 0;
    const int nf = nfree + over;  // free slots after the eviction
    const int fresh = na > nf ? na - nf : 0;
    const bool bad = na > PS_MAX || over > PS_MAX || over > len || (over > 0 && count + na - sa.sink - over < prot) ||
                     hi0 + fresh > cap;
    if (!bad) {
      for (int e = lane; e < over; e += 32) {  // pop the least important tail; push onto the free stack
        const int slot = ring[(head + len - 1 - e) % cap];
        ev_slot[e] = slot;
        ev_pos[e] = lpos[slot];
        fl[nfree + e] = slot;
      }
      __syncwarp();
      for (int i = lane; i < na; i += 32) {  // pop the free stack (top first), then fresh slots at hi
        const int slot = i < nf ? fl[nf - 1 - i] : hi0 + (i - nf);
        new_slot[i] = slot;
        ring[((head - na + i) % cap + cap) % cap] = slot;  // ring head, in position order
      }
    }
    if (lane == 0) {
      if (!bad) {
        m[SD_PM_COUNT] = count + na - over;
        m[SD_PM_HI] = hi0 + fresh;
        m[SD_PM_HEAD] = ((head - na) % cap + cap) % cap;
        m[SD_PM_LEN] = len - over + na;
        m[SD_PM_NFREE] = nf - (na < nf ? na : nf);
      } else {
        m[SD_PM_ERR] = 1;  // SinkViolation / capacity: nothing changed
      }
      s_bad = bad;
      s_a = na;
      s_over = over;
      s_first = first;
      s_count_after = count + na - over;
      s_hi = hi0 + fresh;
    }
  }
  __syncthreads();
  if (s_bad) return;
  const int na = s_a, over = s_over, hi = s_hi;
  if (over > 0) {
    // survivors drop one rank per evicted entry with a smaller position; slots
    // are read PS_U at a time so their loads are in flight together
    constexpr int PS_U = 8;
    for (int s0 = tid; s0 < hi; s0 += PS_U * blockDim.x) {
      int p[PS_U], r[PS_U];
#pragma unroll
      for (int u = 0; u < PS_U; ++u) {
        const int s = s0 + u * blockDim.x;
        p[u] = s < hi ? lpos[s] : -1;
        r[u] = s < hi ? lrank[s] : -1;
      }
#pragma unroll
      for (int u = 0; u < PS_U; ++u) {
        if (p[u] < 0) continue;
        int dec = 0;
        for (int e = 0; e < over; ++e) dec += ev_pos[e] < p[u];
        if (dec) lrank[s0 + u * blockDim.x] = r[u] - dec;
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < over; e += blockDim.x) {
    lpos[ev_slot[e]] = -1;
    lrank[ev_slot[e]] = -1;
    lsc[ev_slot[e]] = QNAN;
  }
  __syncthreads();
  for (int i = tid; i < na; i += blockDim.x) {
    lpos[new_slot[i]] = s_first + i;
    lrank[new_slot[i]] = s_count_after - na + i;
    lsc[new_slot[i]] = QNAN;
  }
  const int lane = tid & 31;
  for (int i = tid >> 5; i < na; i += blockDim.x >> 5) copy_rows<DH, KT>(a, layer, s_first + i, new_slot[i], a.Hk, lane);
}

// grid (L, Hk): rows base+keep[i] -> base+i for three arrays (read all, then write)
__global__ void reconcile_kernel(const int32_t* __restrict__ result, int base, uint32_t* k_raw, uint32_t* k_rot,
                                 uint32_t* v, int64_t layer_w, int64_t head_w, int row_w) {
  extern __shared__ uint32_t buf[];  // [3][depth][row_w]
  const int layer = blockIdx.x, h = blockIdx.y;
  const int a = result[SD_RES_ACCEPTED];
  if (base < 0) base = result[SD_RES_BASE];  // device-resident step (graph replay)
  const int64_t off = layer * layer_w + h * head_w;
  uint32_t* arrs[3] = {k_raw, k_rot, v};
  const int per = a * row_w;
  for (int idx = threadIdx.x; idx < 3 * per; idx += blockDim.x) {
    const int which = idx / per, r = idx - which * per, i = r / row_w, w = r - i * row_w;
    buf[idx] = arrs[which][off + (int64_t)(base + result[SD_RES_KEEP + i]) * row_w + w];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 3 * per; idx += blockDim.x) {
    const int which = idx / per, r = idx - which * per, i = r / row_w, w = r - i * row_w;
    arrs[which][off + (int64_t)(base + i) * row_w + w] = buf[idx];
  }
}

// grid (L, H): q_sum[l][h][:] = sum_i q_pre[l][keep[i]][h][:] in keep order
__global__ void qsum_kernel(const int32_t* __restrict__ result, const float* __restrict__ q_pre, int q_rows, int H,
                            int dh, float* __restrict__ q_sum) {
  const int layer = blockIdx.x, h = blockIdx.y;
  const int a = result[SD_RES_ACCEPTED];
  for (int d = threadIdx.x; d < dh; d += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < a; ++i) s += q_pre[(((int64_t)layer * q_rows + result[SD_RES_KEEP + i]) * H + h) * dh + d];
    q_sum[((int64_t)layer * H + h) * dh + d] = s;
  }
}

template <int DH, typename KT>
static int launch_scores_t(const float* q_sum, const void* k_raw, int64_t ls, int64_t hs, int L, int H, int Hk,
                           int start, int end, float* scores, float* per_head, cudaStream_t st) {
  dim3 grid((end - start + 63) / 64, L);
  const size_t smem = (size_t)Hk * DH * 4;
  if (Hk <= 8)
    score_kernel<DH, KT, 8><<<grid, 256, smem, st>>>(q_sum, (const KT*)k_raw, ls, hs, H, Hk, start, end, scores,
                                                     per_head);
  else if (Hk <= 32)
    score_kernel<DH, KT, 32><<<grid, 256, smem, st>>>(q_sum, (const KT*)k_raw, ls, hs, H, Hk, start, end, scores,
                                                      per_head);
  else {
    set_error("sd_importance_scores: more than 32 kv heads");
    return SD_EUNSUPPORTED;
  }
  return check_launch("sd_importance_scores");
}

template <int DH>
static int launch_scores(const float* q_sum, const void* k_raw, int kv_dtype, int64_t ls, int64_t hs, int L, int H,
                         int Hk, int start, int end, float* scores, float* per_head, cudaStream_t st) {
  if (kv_dtype == SD_BF16)
    return launch_scores_t<DH, __nv_bfloat16>(q_sum, k_raw, ls, hs, L, H, Hk, start, end, scores, per_head, st);
  return launch_scores_t<DH, float>(q_sum, k_raw, ls, hs, L, H, Hk, start, end, scores, per_head, st);
}

static int esize(int dtype) { return dtype == SD_BF16 ? 2 : 4; }

// dispatch over (head_dim, dtype): f(DH, KT) via a templated functor
template <template <int, typename> class F, typename... Args>
static int dispatch_dh(int dh, int dtype, Args... args) {
  switch (dh) {
#define SD_CASE(D)                                                         \
  case D:                                                                  \
    return dtype == SD_BF16 ? F<D, __nv_bfloat16>::run(args...) : F<D, float>::run(args...);
    SD_CASE(8) SD_CASE(16) SD_CASE(32) SD_CASE(64) SD_CASE(128)
#undef SD_CASE
    default:
      set_error("partial cache: head_dim %d", dh);
      return SD_EUNSUPPORTED;
  }
}

template <int DH, typename KT>
struct RefreshLaunch {
  static int run(const RefreshArgs& a, int L, cudaStream_t st) {
    const size_t smem = (size_t)RF_MAX_TAKE * 8 + (size_t)a.Hk * DH * 4;
    auto kern = a.Hk <= 8 ? refresh_kernel<DH, KT, 8> : refresh_kernel<DH, KT, 32>;
    static size_t attr8 = 0, attr32 = 0;
    size_t& attr = a.Hk <= 8 ? attr8 : attr32;
    if (smem > attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
    kern<<<dim3(RF_CLUSTER, L), RF_THREADS, smem, st>>>(a);
    return check_launch("sd_partial_refresh");
  }
};

template <int DH, typename KT>
struct MirrorLaunch {
  static int run(const RefreshArgs& a, int L, int upto, cudaStream_t st) {
    int gx = (a.slot_cap + 255) / 256;
    if (gx > 16) gx = 16;
    mirror_kernel<DH, KT><<<dim3(gx, L), 256, 0, st>>>(a, upto);
    return check_launch("sd_partial_mirror");
  }
};

template <int DH, typename KT>
struct StepLaunch {
  static int run(const StepArgs& a, int L, cudaStream_t st) {
    partial_step_kernel<DH, KT><<<L, 256, 0, st>>>(a);
    return check_launch("sd_partial_step");
  }
};

static RefreshArgs make_refresh_args(const void* full_k_raw, const void* full_v, int64_t fls, int64_t fhs, int Hk,
                                     void* pk, void* pv, int64_t pls, int64_t phs, int slot_cap, int32_t* ppos,
                                     int32_t* prank, float* pscore, int32_t* ring, int32_t* freel, int32_t* meta) {
  RefreshArgs a = {};
  a.fk = full_k_raw;
  a.fv = full_v;
  a.f_ls = fls;
  a.f_hs = fhs;
  a.Hk = Hk;
  a.pk = pk;
  a.pv = pv;
  a.p_ls = pls;
  a.p_hs = phs;
  a.slot_cap = slot_cap;
  a.ppos = ppos;
  a.prank = prank;
  a.pscore = pscore;
  a.ring = ring;
  a.freel = freel;
  a.meta = meta;
  return a;
}

}  // namespace sd

using namespace sd;

extern "C" {

int sd_importance_scores(const float* q_sum, const void* k_raw, int kv_dtype, int64_t layer_stride,
                         int64_t head_stride, int L, int H, int Hk, int dh, int start, int end, float* scores,
                         float* per_head, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && H > 0 && Hk > 0 && H % Hk == 0 && Hk <= 32, "sd_importance_scores: heads");
  SD_REQUIRE(end > start && start >= 0, "sd_importance_scores: range");
  auto st = as_stream(stream);
  switch (dh) {
    case 8: return launch_scores<8>(q_sum, k_raw, kv_dtype, layer_stride, head_stride, L, H, Hk, start, end, scores, per_head, st);
    case 16: return launch_scores<16>(q_sum, k_raw, kv_dtype, layer_stride, head_stride, L, H, Hk, start, end, scores, per_head, st);
    case 32: return launch_scores<32>(q_sum, k_raw, kv_dtype, layer_stride, head_stride, L, H, Hk, start, end, scores, per_head, st);
    case 64: return launch_scores<64>(q_sum, k_raw, kv_dtype, layer_stride, head_stride, L, H, Hk, start, end, scores, per_head, st);
    case 128: return launch_scores<128>(q_sum, k_raw, kv_dtype, layer_stride, head_stride, L, H, Hk, start, end, scores, per_head, st);
    default: set_error("sd_importance_scores: head_dim %d", dh); return SD_EUNSUPPORTED;
  }
}

int sd_sum_head_scores(const float* per_head, int L, int Hk, int n, float* scores, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && Hk > 0 && n > 0, "sd_sum_head_scores: sizes");
  sum_head_scores_kernel<<<148 * 4, 256, 0, as_stream(stream)>>>(per_head, L, Hk, n, scores);
  return check_launch("sd_sum_head_scores");
}

size_t sd_refresh_workspace_bytes(int L, int n_cand, int take) {
  return (size_t)L * ((size_t)(n_cand > 0 ? n_cand : 1) * 4 + (size_t)(take > 0 ? take : 1) * 8) + 16;
}

int sd_partial_refresh(const float* q_sum, const float* scores_in, int L, int H, int Hk, int dh, int upto, int sink,
                       int budget, const void* full_k_raw, const void* full_v, int kv_dtype, int64_t full_layer_stride,
                       int64_t full_head_stride, void* pk, void* pv, int64_t part_layer_stride,
                       int64_t part_head_stride, int slot_cap, int32_t* ppos, int32_t* prank, float* pscore,
                       int32_t* ring, int32_t* freel, int32_t* meta, void* workspace, size_t workspace_bytes,
                       sd_stream_t stream) {
  SD_REQUIRE(L > 0 && Hk > 0 && Hk <= 32 && H % Hk == 0, "sd_partial_refresh: heads");
  SD_REQUIRE(budget > sink && sink >= 0, "sd_partial_refresh: budget %d <= sink %d", budget, sink);
  SD_REQUIRE(upto >= budget, "sd_partial_refresh: %d entries < budget %d", upto, budget);
  const int n = upto - sink, take = budget - sink;
  SD_REQUIRE(take <= RF_MAX_TAKE, "sd_partial_refresh: body %d > %d", take, RF_MAX_TAKE);
  SD_REQUIRE(budget <= slot_cap, "sd_partial_refresh: slot capacity");
  SD_REQUIRE(q_sum || scores_in, "sd_partial_refresh: need q_sum or scores");
  SD_REQUIRE(workspace_bytes >= sd_refresh_workspace_bytes(L, n, take), "sd_partial_refresh: workspace");
  SD_REQUIRE((dh * esize(kv_dtype)) % 16 == 0, "sd_partial_refresh: row bytes");
  RefreshArgs a = make_refresh_args(full_k_raw, full_v, full_layer_stride, full_head_stride, Hk, pk, pv,
                                    part_layer_stride, part_head_stride, slot_cap, ppos, prank, pscore, ring, freel,
                                    meta);
  a.q_sum = q_sum;
  a.scores_in = scores_in;
  a.scores_ws = reinterpret_cast<float*>(workspace);
  a.keys_ws = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(workspace) +
                                          (((size_t)L * n * 4 + 15) & ~(size_t)15));
  a.H = H;
  a.n = n;
  a.sink = sink;
  a.take = take;
  return dispatch_dh<RefreshLaunch>(dh, kv_dtype, a, L, as_stream(stream));
}

int sd_partial_mirror(int L, int Hk, int dh, int upto, int sink, const void* full_k_raw, const void* full_v,
                      int kv_dtype, int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                      int64_t part_layer_stride, int64_t part_head_stride, int slot_cap, int32_t* ppos, int32_t* prank,
                      float* pscore, int32_t* ring, int32_t* freel, int32_t* meta, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && Hk > 0 && upto >= sink && upto <= slot_cap, "sd_partial_mirror: sizes");
  SD_REQUIRE((dh * esize(kv_dtype)) % 16 == 0, "sd_partial_mirror: row bytes");
  RefreshArgs a = make_refresh_args(full_k_raw, full_v, full_layer_stride, full_head_stride, Hk, pk, pv,
                                    part_layer_stride, part_head_stride, slot_cap, ppos, prank, pscore, ring, freel,
                                    meta);
  a.sink = sink;
  return dispatch_dh<MirrorLaunch>(dh, kv_dtype, a, L, upto, as_stream(stream));
}

int sd_partial_step(int L, const int32_t* result, int a_host, int first_pos_host, int evict, int protected_host,
                    int sink, int budget, int Hk, int dh, const void* full_k_raw, const void* full_v, int kv_dtype,
                    int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                    int64_t part_layer_stride, int64_t part_head_stride, int slot_cap, int32_t* ppos, int32_t* prank,
                    float* pscore, int32_t* ring, int32_t* freel, int32_t* meta, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && Hk > 0 && budget > sink, "sd_partial_step: sizes");
  SD_REQUIRE(result || (a_host >= 0 && a_host <= PS_MAX), "sd_partial_step: a=%d (max %d per launch)", a_host, PS_MAX);
  SD_REQUIRE((dh * esize(kv_dtype)) % 16 == 0, "sd_partial_step: row bytes");
  StepArgs s = {};
  s.result = result;
  s.a_host = a_host;
  s.first_pos_host = first_pos_host;
  s.evict = evict;
  s.protected_host = protected_host;
  s.sink = sink;
  s.budget = budget;
  s.r = make_refresh_args(full_k_raw, full_v, full_layer_stride, full_head_stride, Hk, pk, pv, part_layer_stride,
                          part_head_stride, slot_cap, ppos, prank, pscore, ring, freel, meta);
  return dispatch_dh<StepLaunch>(dh, kv_dtype, s, L, as_stream(stream));
}

int sd_reconcile(int L, const int32_t* result, int base_len, void* k_raw, void* k_rot, void* v, int kv_dtype,
                 int64_t layer_stride, int64_t head_stride, int Hk, int dh, const float* q_pre, int q_rows, int H,
                 float* q_sum, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && Hk > 0 && dh > 0, "sd_reconcile: sizes");
  const int es = esize(kv_dtype), fw = 4 / es, row_w = dh / fw;
  auto st = as_stream(stream);
  const size_t smem = 3 * SD_TREE_MAX_DEPTH * row_w * 4;
  reconcile_kernel<<<dim3(L, Hk), 128, smem, st>>>(result, base_len, (uint32_t*)k_raw, (uint32_t*)k_rot,
                                                    (uint32_t*)v, layer_stride / fw, head_stride / fw, row_w);
  int rc = check_launch("sd_reconcile");
  if (rc || !q_pre) return rc;
  qsum_kernel<<<dim3(L, H), dh < 32 ? 32 : (dh > 256 ? 256 : dh), 0, st>>>(result, q_pre, q_rows, H, dh, q_sum);
  return check_launch("sd_reconcile(qsum)");
}

}  // extern "C"
