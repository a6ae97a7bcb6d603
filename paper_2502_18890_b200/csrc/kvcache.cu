// Dynamic partial-KV maintenance: Eq. 2 scoring, exact top-K selection with
// the reference's (-score, pos) order, slot gather, admit/evict with
// incremental rank upkeep, and reconcile of accepted tree rows.
// Reference: kvcache.py:116-127 (reconcile), 215-225 (admit), 243-265
// (importance), 268-319 (prefill/mirror build), 332-354 (evict);
// engine.py:128-148 (per-layer body scores over pre-rotation keys), 280.
#include "common.cuh"

namespace sd {

// ---------------------------------------------------------------- scores ----
// grid (ceil(n/64), L), 256 threads: warp handles 8 positions, lanes over dh.
template <int DH, typename KT>
__global__ void __launch_bounds__(256) score_kernel(const float* __restrict__ q_sum, const KT* __restrict__ K,
                                                    int64_t layer_stride, int64_t head_stride, int H, int Hk,
                                                    int start, int end, float* __restrict__ scores,
                                                    float* __restrict__ per_head) {
  constexpr int EPL = DH >= 32 ? DH / 32 : 1;
  __shared__ float qg[64 * DH];  // Hk <= 64
  const int layer = blockIdx.y, G = H / Hk;
  const float* q = q_sum + (int64_t)layer * H * DH;
  // grouped query per kv head, g summed in ascending order
  for (int i = threadIdx.x; i < Hk * DH; i += blockDim.x) {
    const int k = i / DH, d = i - k * DH;
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += q[(k * G + g) * DH + d];
    qg[i] = s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = end - start;
  const KT* Kl = K + layer * layer_stride;
  for (int r = 0; r < 8; ++r) {
    const int i = blockIdx.x * 64 + warp * 8 + r;
    if (i >= n) break;
    const int64_t pos = start + i;
    float total = 0.f;
    for (int k = 0; k < Hk; ++k) {
      float part = 0.f;
      if (DH >= 32 || lane < DH) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int d = lane * EPL + e;
          part = fmaf(qg[k * DH + d], to_f(Kl[k * head_stride + pos * DH + d]), part);
        }
      }
      part = warp_sum(part);
      if (per_head && lane == 0) per_head[((int64_t)layer * Hk + k) * n + i] = part;
      total = k == 0 ? part : total + part;  // ascending head order
    }
    if (lane == 0 && scores) scores[(int64_t)layer * n + i] = total;
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
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// larger key = better: higher score first, then lower position
__device__ __forceinline__ uint64_t sel_key(float score, int pos) {
  if (score == 0.0f) score = 0.0f;  // -0.0 ties with +0.0, as in the reference's comparison
  return ((uint64_t)ord_f32(score) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)pos);
}

constexpr int SEL_THREADS = 1024;
constexpr int SEL_MAX_TAKE = 8192;

// one CTA per layer
__global__ void __launch_bounds__(SEL_THREADS) select_kernel(const float* __restrict__ scores, int n, int sink,
                                                             int take, int32_t* __restrict__ ppos,
                                                             int32_t* __restrict__ prank, float* __restrict__ pscore,
                                                             int slot_cap, int32_t* __restrict__ asc_ws) {
  extern __shared__ uint64_t sk[];  // [pow2 >= take]
  __shared__ uint32_t hist[256];
  __shared__ uint32_t red[32];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_k;
  const int layer = blockIdx.x, tid = threadIdx.x;
  const float* sc = scores + (int64_t)layer * n;
  int32_t* asc = asc_ws + (int64_t)layer * n;
  int32_t* lpos = ppos + (int64_t)layer * slot_cap;
  int32_t* lrank = prank + (int64_t)layer * slot_cap;
  float* lsc = pscore + (int64_t)layer * slot_cap;
  // --- radix select: the take-th largest key ---
  uint64_t prefix = 0, pmask = 0;
  uint32_t k = (uint32_t)take;
  if (take < n) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += SEL_THREADS) hist[b] = 0;
      __syncthreads();
      for (int i = tid; i < n; i += SEL_THREADS) {
        const uint64_t key = sel_key(sc[i], sink + i);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t cum = 0;
        int b = 255;
        for (; b > 0; --b) {
          if (cum + hist[b] >= k) break;
          cum += hist[b];
        }
        s_prefix = prefix | ((uint64_t)b << shift);
        s_k = k - cum;
      }
      __syncthreads();
      prefix = s_prefix;
      k = s_k;
      pmask |= (uint64_t)255 << shift;
    }
  }
  const uint64_t thresh = take < n ? prefix : 0;  // keys >= thresh selected
  // --- compaction in ascending position order ---
  const int seg = (n + SEL_THREADS - 1) / SEL_THREADS;
  const int b0 = tid * seg, b1 = min(n, b0 + seg);
  uint32_t cnt = 0;
  for (int i = b0; i < b1; ++i) cnt += sel_key(sc[i], sink + i) >= thresh;
  // block exclusive scan of cnt
  uint32_t v = cnt;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = red[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    red[lane] = w;
  }
  __syncthreads();
  uint32_t off = v - cnt + (wid ? red[wid - 1] : 0);
  for (int i = b0; i < b1; ++i)
    if (sel_key(sc[i], sink + i) >= thresh) asc[off++] = sink + i;
  __syncthreads();
  // --- bitonic sort of selected keys, descending ---
  int N = 1;
  while (N < take) N <<= 1;
  for (int i = tid; i < N; i += SEL_THREADS) sk[i] = i < take ? sel_key(sc[asc[i] - sink], asc[i]) : 0ull;
  __syncthreads();
  for (int kk = 2; kk <= N; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < N; i += SEL_THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = sk[i], b = sk[ixj];
          const bool up = (i & kk) == 0;
          if ((a < b) == up) {
            sk[i] = b;
            sk[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // --- write slots: sink first, then body in importance order ---
  for (int j = tid; j < sink; j += SEL_THREADS) {
    lpos[j] = j;
    lrank[j] = j;
    lsc[j] = __int_as_float(0x7fc00000);
  }
  for (int i = tid; i < take; i += SEL_THREADS) {
    const int pos = (int)(0xFFFFFFFFu - (uint32_t)(sk[i] & 0xFFFFFFFFull));
    int lo = 0, hi = take;  // lower_bound in asc
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (asc[mid] < pos) lo = mid + 1; else hi = mid;
    }
    lpos[sink + i] = pos;
    lrank[sink + i] = sink + lo;
    lsc[sink + i] = sc[pos - sink];
  }
}

__global__ void mirror_kernel(int upto, int sink, int32_t* __restrict__ ppos, int32_t* __restrict__ prank,
                              float* __restrict__ pscore, int slot_cap) {
  const int layer = blockIdx.y;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < upto; s += gridDim.x * blockDim.x) {
    const int pos = s < sink ? s : upto - 1 - (s - sink);
    ppos[(int64_t)layer * slot_cap + s] = pos;
    prank[(int64_t)layer * slot_cap + s] = pos;
    pscore[(int64_t)layer * slot_cap + s] = __int_as_float(0x7fc00000);
  }
}

// copy rows (K_raw, V) of the full cache at ppos into partial slots, uint32 words
__global__ void gather_kernel(int count, const int32_t* __restrict__ ppos, int slot_cap,
                              const uint32_t* __restrict__ fk, const uint32_t* __restrict__ fv,
                              int64_t f_layer_w, int64_t f_head_w, uint32_t* __restrict__ pk,
                              uint32_t* __restrict__ pv, int64_t p_layer_w, int64_t p_head_w, int Hk, int row_w) {
  const int layer = blockIdx.y;
  const int64_t per_layer = (int64_t)count * Hk * row_w;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < per_layer;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % row_w);
    const int64_t sh = idx / row_w;
    const int h = (int)(sh % Hk);
    const int s = (int)(sh / Hk);
    const int64_t pos = ppos[(int64_t)layer * slot_cap + s];
    const int64_t src = layer * f_layer_w + h * f_head_w + pos * row_w + w;
    const int64_t dst = layer * p_layer_w + h * p_head_w + (int64_t)s * row_w + w;
    pk[dst] = fk[src];
    pv[dst] = fv[src];
  }
}

struct UpdateArgs {
  int new_slots[SD_TREE_MAX_DEPTH];
  int evict_slots[SD_TREE_MAX_DEPTH];
};

// one CTA per layer over slots [0, hi): evicted slots become holes (pos = rank
// = -1), surviving entries drop one rank per evicted entry with a smaller
// position, admitted entries (the newest positions) take the top ranks.
__global__ void partial_update_kernel(int hi, int count_after, int first_pos, int a, int n_evict, UpdateArgs ua,
                                      int32_t* __restrict__ ppos, int32_t* __restrict__ prank,
                                      float* __restrict__ pscore, int slot_cap, const uint32_t* __restrict__ fk,
                                      const uint32_t* __restrict__ fv, int64_t f_layer_w, int64_t f_head_w,
                                      uint32_t* __restrict__ pk, uint32_t* __restrict__ pv, int64_t p_layer_w,
                                      int64_t p_head_w, int Hk, int row_w) {
  __shared__ int ep[SD_TREE_MAX_DEPTH];
  const int layer = blockIdx.x;
  int32_t* lp = ppos + (int64_t)layer * slot_cap;
  int32_t* lr = prank + (int64_t)layer * slot_cap;
  float* ls = pscore + (int64_t)layer * slot_cap;
  if ((int)threadIdx.x < n_evict) ep[threadIdx.x] = lp[ua.evict_slots[threadIdx.x]];
  __syncthreads();
  for (int s = threadIdx.x; s < hi; s += blockDim.x) {
    int ni = -1;
    bool ev = false;
    for (int i = 0; i < a; ++i) ni = ua.new_slots[i] == s ? i : ni;
    for (int e = 0; e < n_evict; ++e) ev |= ua.evict_slots[e] == s;
    if (ni >= 0) {
      lp[s] = first_pos + ni;
      lr[s] = count_after - a + ni;
      ls[s] = __int_as_float(0x7fc00000);
    } else if (ev) {
      lp[s] = -1;
      lr[s] = -1;
      ls[s] = __int_as_float(0x7fc00000);
    } else {
      const int p = lp[s];
      if (p < 0) continue;  // hole
      int dec = 0;
      for (int e = 0; e < n_evict; ++e) dec += ep[e] < p;
      lr[s] -= dec;
    }
  }
  const int per = a * Hk * row_w;
  for (int idx = threadIdx.x; idx < per; idx += blockDim.x) {
    const int w = idx % row_w, sh = idx / row_w, h = sh % Hk, i = sh / Hk;
    const int64_t src = layer * f_layer_w + h * f_head_w + (int64_t)(first_pos + i) * row_w + w;
    const int64_t dst = layer * p_layer_w + h * p_head_w + (int64_t)ua.new_slots[i] * row_w + w;
    pk[dst] = fk[src];
    pv[dst] = fv[src];
  }
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

template <int DH>
static int launch_scores(const float* q_sum, const void* k_raw, int kv_dtype, int64_t ls, int64_t hs, int L, int H,
                         int Hk, int start, int end, float* scores, float* per_head, cudaStream_t st) {
  dim3 grid((end - start + 63) / 64, L);
  if (kv_dtype == SD_BF16)
    score_kernel<DH, __nv_bfloat16><<<grid, 256, 0, st>>>(q_sum, (const __nv_bfloat16*)k_raw, ls, hs, H, Hk, start,
                                                          end, scores, per_head);
  else
    score_kernel<DH, float><<<grid, 256, 0, st>>>(q_sum, (const float*)k_raw, ls, hs, H, Hk, start, end, scores,
                                                  per_head);
  return check_launch("sd_importance_scores");
}

static int esize(int dtype) { return dtype == SD_BF16 ? 2 : 4; }

}  // namespace sd

using namespace sd;

extern "C" {

int sd_importance_scores(const float* q_sum, const void* k_raw, int kv_dtype, int64_t layer_stride,
                         int64_t head_stride, int L, int H, int Hk, int dh, int start, int end, float* scores,
                         float* per_head, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && H > 0 && Hk > 0 && H % Hk == 0 && Hk <= 64, "sd_importance_scores: heads");
  SD_REQUIRE(end > start && start >= 0, "sd_importance_scores: range");
  SD_REQUIRE(dh * Hk <= 64 * 128, "sd_importance_scores: Hk*dh too large");
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

size_t sd_select_workspace_bytes(int L, int n_cand) { return (size_t)L * (size_t)(n_cand > 0 ? n_cand : 1) * 4; }

int sd_select_topk(const float* scores, int L, int n_cand, int sink, int take, int32_t* ppos, int32_t* prank,
                   float* pscore, int slot_cap, void* workspace, size_t workspace_bytes, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && take > 0 && take <= n_cand, "sd_select_topk: take=%d n_cand=%d", take, n_cand);
  SD_REQUIRE(take <= SEL_MAX_TAKE, "sd_select_topk: take %d > %d", take, SEL_MAX_TAKE);
  SD_REQUIRE(sink + take <= slot_cap, "sd_select_topk: slot capacity");
  SD_REQUIRE(workspace_bytes >= sd_select_workspace_bytes(L, n_cand), "sd_select_topk: workspace");
  int N = 1;
  while (N < take) N <<= 1;
  const size_t smem = (size_t)N * 8;
  static size_t attr = 0;  // only grows: earlier captured launches keep fitting
  if (smem > attr) {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  select_kernel<<<L, SEL_THREADS, smem, as_stream(stream)>>>(scores, n_cand, sink, take, ppos, prank, pscore,
                                                             slot_cap, (int32_t*)workspace);
  return check_launch("sd_select_topk");
}

int sd_mirror_positions(int L, int upto, int sink, int32_t* ppos, int32_t* prank, float* pscore, int slot_cap,
                        sd_stream_t stream) {
  SD_REQUIRE(L > 0 && upto >= sink && upto <= slot_cap, "sd_mirror_positions: sizes");
  if (upto == 0) return SD_OK;
  dim3 grid((upto + 255) / 256, L);
  mirror_kernel<<<grid, 256, 0, as_stream(stream)>>>(upto, sink, ppos, prank, pscore, slot_cap);
  return check_launch("sd_mirror_positions");
}

int sd_gather_slots(int L, int count, const int32_t* ppos, int slot_cap, const void* full_k_raw, const void* full_v,
                    int kv_dtype, int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                    int64_t part_layer_stride, int64_t part_head_stride, int Hk, int dh, sd_stream_t stream) {
  SD_REQUIRE(L > 0 && count >= 0, "sd_gather_slots: sizes");
  if (count == 0) return SD_OK;
  const int es = esize(kv_dtype);
  SD_REQUIRE((dh * es) % 4 == 0, "sd_gather_slots: row bytes");
  const int fw = 4 / es;  // elements per word
  const int row_w = dh / fw;
  const int64_t per = (int64_t)count * Hk * row_w;
  int gx = (int)((per + 255) / 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, L);
  gather_kernel<<<grid, 256, 0, as_stream(stream)>>>(count, ppos, slot_cap, (const uint32_t*)full_k_raw,
                                                     (const uint32_t*)full_v, full_layer_stride / fw,
                                                     full_head_stride / fw, (uint32_t*)pk, (uint32_t*)pv,
                                                     part_layer_stride / fw, part_head_stride / fw, Hk, row_w);
  return check_launch("sd_gather_slots");
}

int sd_partial_update(int L, int hi, int count_after, int first_pos, int a, const int32_t* new_slots_host,
                      int n_evict, const int32_t* evict_slots_host, int32_t* ppos, int32_t* prank, float* pscore,
                      int slot_cap, const void* full_k_raw, const void* full_v, int kv_dtype,
                      int64_t full_layer_stride, int64_t full_head_stride, void* pk, void* pv,
                      int64_t part_layer_stride, int64_t part_head_stride, int Hk, int dh, sd_stream_t stream) {
  SD_REQUIRE(a >= 0 && a <= SD_TREE_MAX_DEPTH && n_evict >= 0 && n_evict <= SD_TREE_MAX_DEPTH,
             "sd_partial_update: counts");
  SD_REQUIRE(hi <= slot_cap && count_after >= a && count_after <= hi, "sd_partial_update: capacity");
  UpdateArgs ua;
  for (int i = 0; i < SD_TREE_MAX_DEPTH; ++i) {
    ua.new_slots[i] = i < a ? new_slots_host[i] : -1;
    ua.evict_slots[i] = i < n_evict ? evict_slots_host[i] : -1;
    SD_REQUIRE(i >= a || (ua.new_slots[i] >= 0 && ua.new_slots[i] < hi), "sd_partial_update: new slot");
    SD_REQUIRE(i >= n_evict || (ua.evict_slots[i] >= 0 && ua.evict_slots[i] < hi), "sd_partial_update: evict slot");
  }
  const int es = esize(kv_dtype), fw = 4 / es, row_w = dh / fw;
  partial_update_kernel<<<L, 256, 0, as_stream(stream)>>>(
      hi, count_after, first_pos, a, n_evict, ua, ppos, prank, pscore, slot_cap, (const uint32_t*)full_k_raw,
      (const uint32_t*)full_v, full_layer_stride / fw, full_head_stride / fw, (uint32_t*)pk, (uint32_t*)pv,
      part_layer_stride / fw, part_head_stride / fw, Hk, row_w);
  return check_launch("sd_partial_update");
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
