// Contextual-penalty sampling on device, fp64 arithmetic like the reference.
// Reference: sampling.py:142-162 (Eq. 3 penalty + softmax), 193-216
// (top-p / min-p / eta truncation), 219-224 (inverse-CDF at the (seed, pos)
// deviate), 120-139 (shrunk window masks); engine.py:155-181 (per verify row
// window splice), 207-215 (draft per-head top-w, ties to the lower id),
// 237-245 (row draw positions).
//
// One CTA per row. Membership of token v in row r is computed on the fly from
// the window's count array plus at most 2*depth patched tokens (tokens slid
// out of the window by the branch, tokens of the branch itself), so the
// [T, V] boolean mask of the reference is never materialised.
#include <cooperative_groups.h>

#include "common.cuh"
#include "sample_common.cuh"

namespace cg = cooperative_groups;

namespace sd {

constexpr int SMP_THREADS = 1024;
struct DI {
  double v;
  int i;
};
__device__ __forceinline__ DI better(DI x, DI y) {  // larger value, ties -> lower index
  if (x.v > y.v) return x;
  if (y.v > x.v) return y;
  return x.i <= y.i ? x : y;
}

__device__ DI block_argmax(DI x, DI* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DI y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = better(x, y);
  }
  __syncthreads();
  if (lane == 0) scratch[wid] = x;
  __syncthreads();
  DI r = scratch[0];
  for (int w = 1; w < nw; ++w) r = better(r, scratch[w]);
  __syncthreads();
  return r;
}

// inclusive block scan (fp64) -> returns exclusive prefix of this thread
__device__ double block_exclusive_scan(double v, double* scratch, double* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    double w = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) scratch[lane] = w;
  }
  __syncthreads();
  const double before = (wid ? scratch[wid - 1] : 0.0) + (x - v);
  *total = scratch[nw - 1];
  __syncthreads();
  return before;
}

template <int IN>
__global__ void __launch_bounds__(SMP_THREADS) sample_rows_kernel(const void* __restrict__ in, SampleDev a) {
  __shared__ RowCtx rc;
  __shared__ double dred[32];
  __shared__ DI ared[32];
  __shared__ unsigned long long s_u64[4];
  __shared__ double hmass[256];
  __shared__ unsigned int hcnt[256];
  __shared__ int s_int[4];
  const int row = blockIdx.x, tid = threadIdx.x;
  if (row >= a.rows) return;
  if (a.member_kind == SD_MEMBER_TREE && row >= a.tree[tree_off::T]) return;
  if (tid == 0) row_setup(a, row, rc);
  __syncthreads();
  const int V = a.V;
  const int64_t base = (int64_t)row * V;
  auto sum_op = [](double x, double y) { return x + y; };
  auto max_op = [](double x, double y) { return fmax(x, y); };

  // ---- penalised softmax (or given probabilities) ----
  // fp64 logits (API path): fp64 throughout, like the reference.
  // fp32 logits (engine path): fp32 scaled logits and expf, fp64 sums.
  constexpr bool FAST = IN == SD_IN_LOGITS_F32;
  double m = 0.0, Z = 1.0, invZ = 1.0;
  float mf = 0.f;
  const float inv_t = (float)(1.0 / a.temperature), inv_tt = (float)(1.0 / (a.temperature * a.theta));
  const float th = (float)a.theta;
  auto scaled_f = [&](int v) -> float {
    const float l = ((const float*)in)[base + v];
    if (!is_member(a, rc, row, v)) return l * inv_t;
    if (a.ctrl_style) return (l < 0.f ? l * th : l / th) * inv_t;
    return l * inv_tt;
  };
  const bool is_probs = IN == SD_IN_PROBS_F64;
  if (FAST) {
    // one pass: running max and sum of exp per thread, combined in fp64
    float lm = -INFINITY;
    double lz = 0.0;
    for (int v = tid; v < V; v += SMP_THREADS) {
      const float s = scaled_f(v);
      if (s > lm) {
        lz = lz * (double)expf(lm - s);  // exp(-inf) = 0 on the first element
        lm = s;
      }
      lz += (double)expf(s - lm);
    }
    mf = block_reduce(lm, (float*)dred, [](float x, float y) { return fmaxf(x, y); });
    lz = lm == -INFINITY ? 0.0 : lz * exp((double)lm - (double)mf);
    Z = block_reduce(lz, dred, sum_op);
    invZ = 1.0 / Z;
  } else if (!is_probs) {
    double lm = -INFINITY;
    for (int v = tid; v < V; v += SMP_THREADS) lm = fmax(lm, scaled(load_in<IN>(in, base + v), is_member(a, rc, row, v), a));
    m = block_reduce(lm, dred, max_op);
    double lz = 0.0;
    for (int v = tid; v < V; v += SMP_THREADS) lz += exp(scaled(load_in<IN>(in, base + v), is_member(a, rc, row, v), a) - m);
    Z = block_reduce(lz, dred, sum_op);
  }
  auto prob = [&](int v) -> double {
    if (is_probs) return load_in<IN>(in, base + v);
    if (FAST) return (double)expf(scaled_f(v) - mf) * invZ;
    const double s = scaled(load_in<IN>(in, base + v), is_member(a, rc, row, v), a);
    const double e = exp(s - m);
    return e / Z;
  };
  if (a.probs_out)
    for (int v = tid; v < V; v += SMP_THREADS) a.probs_out[base + v] = prob(v);
  if (!a.trunc_out && !a.token_out) return;

  // ---- truncation support: keep(v) ----
  // kinds: none; min_p: p >= thr; eta: p >= thr (or argmax only); top_p: p > pstar or (p == pstar and v <= vcut)
  double thr = -1.0;  // keep p >= thr
  double pstar = -1.0;
  int vcut = -1, only = -1;
  const int tk = a.trunc_kind;
  if (tk == SD_TRUNC_MIN_P && !is_probs) {
    // p_max = exp(0) / Z: no pass needed (sampling.py:207)
    thr = a.trunc_value * (FAST ? invZ : 1.0 / Z);
  } else if (tk == SD_TRUNC_MIN_P || tk == SD_TRUNC_ETA || tk == SD_TRUNC_TOP_P) {
    // pmax and argmax (lowest index)
    DI best{-1.0, 0x7fffffff};
    for (int v = tid; v < V; v += SMP_THREADS) best = better(best, DI{prob(v), v});
    best = block_argmax(best, ared);
    if (tk == SD_TRUNC_MIN_P) {
      thr = a.trunc_value * best.v;
    } else if (tk == SD_TRUNC_ETA) {
      double le = 0.0;
      for (int v = tid; v < V; v += SMP_THREADS) {
        const double p = prob(v);
        if (p > 0.0) le += p * log(p);
      }
      const double ent = -block_reduce(le, dred, sum_op);
      const double alpha = a.eta_alpha < 0.0 ? sqrt(a.trunc_value) : a.eta_alpha;
      const double eta = fmin(a.trunc_value, alpha * exp(-ent));
      if (best.v < eta) only = best.i;  // nothing survives: keep the argmax
      thr = eta;
    } else {
      // ---- top-p: radix descent over fp64 bit patterns with mass histograms ----
      double total_l = 0.0;
      for (int v = tid; v < V; v += SMP_THREADS) total_l += prob(v);
      const double total = block_reduce(total_l, dred, sum_op);
      if (a.trunc_value >= total) {
        thr = -1.0;  // keep everything
      } else {
        unsigned long long prefix = 0, mask = 0;
        double above = 0.0;
        for (int shift = 56; shift >= 0; shift -= 8) {
          for (int b = tid; b < 256; b += SMP_THREADS) {
            hmass[b] = 0.0;
            hcnt[b] = 0;
          }
          __syncthreads();
          for (int v = tid; v < V; v += SMP_THREADS) {
            const double p = prob(v);
            const unsigned long long bits = (unsigned long long)__double_as_longlong(p);
            if ((bits & mask) == prefix) {
              const int bkt = (int)((bits >> shift) & 255ull);
              atomicAdd(&hmass[bkt], p);
              atomicAdd(&hcnt[bkt], 1u);
            }
          }
          __syncthreads();
          if (tid == 0) {
            int b = 255;
            double acc = above;
            int chosen = -1, lowest = -1;
            for (; b >= 0; --b) {
              if (hcnt[b] == 0) continue;
              lowest = b;
              if (acc + hmass[b] >= a.trunc_value) {
                chosen = b;
                break;
              }
              acc += hmass[b];
            }
            if (chosen < 0) {  // rounding: mass never reached; take the lowest bucket
              chosen = lowest < 0 ? 0 : lowest;
              acc -= lowest < 0 ? 0.0 : hmass[lowest];
            }
            s_u64[0] = prefix | ((unsigned long long)chosen << shift);
            dred[0] = acc;
          }
          __syncthreads();
          prefix = s_u64[0];
          above = dred[0];
          mask |= 255ull << shift;
          __syncthreads();
        }
        pstar = __longlong_as_double((long long)prefix);
        // number of elements equal to pstar needed, lowest indices first
        unsigned int ceq_l = 0;
        for (int v = tid; v < V; v += SMP_THREADS) ceq_l += prob(v) == pstar;
        double ceq_d = block_reduce((double)ceq_l, dred, sum_op);
        const int ceq = (int)ceq_d;
        int need = (int)ceil((a.trunc_value - above) / pstar);
        if (need < 1) need = 1;
        if (need > ceq) need = ceq;
        if (need >= ceq) {
          vcut = V;  // all equal elements kept
        } else {
          // index of the need-th equal element: segment scan in index order
          const int seg = (V + SMP_THREADS - 1) / SMP_THREADS;
          const int b0 = tid * seg, b1 = min(V, b0 + seg);
          double c = 0.0;
          for (int v = b0; v < b1; ++v) c += prob(v) == pstar;
          double tot;
          const double before = block_exclusive_scan(c, dred, &tot);
          if (tid == 0) s_int[0] = V;
          __syncthreads();
          if (before < need && before + c >= need) {
            int k = (int)before;
            for (int v = b0; v < b1; ++v) {
              if (prob(v) == pstar && ++k == need) {
                s_int[0] = v;
                break;
              }
            }
          }
          __syncthreads();
          vcut = s_int[0];
        }
      }
    }
  }
  auto kept = [&](int v, double p) -> double {
    if (tk == SD_TRUNC_NONE) return p;
    if (only >= 0) return v == only ? p : 0.0;
    if (tk == SD_TRUNC_TOP_P) {
      if (pstar < 0.0) return p;
      return (p > pstar || (p == pstar && v <= vcut)) ? p : 0.0;
    }
    return p >= thr ? p : 0.0;
  };
  // ---- kept mass in warp-contiguous chunks (coalesced; chunk w = [w*S, (w+1)*S)) ----
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int NWARP = SMP_THREADS / 32;
  const int S = (V + NWARP * 32 - 1) / (NWARP * 32) * 32;
  const int c0 = wid * S, c1 = min(V, c0 + S);
  double lk = 0.0;
  for (int v = c0 + lane; v < c1; v += 32) lk += kept(v, prob(v));
  lk = warp_sum_d(lk);
  __shared__ double wtot[NWARP];
  if (lane == 0) wtot[wid] = lk;
  __syncthreads();
  double K = 0.0;
  for (int w = 0; w < NWARP; ++w) K += wtot[w];
  if (a.trunc_out)
    for (int v = tid; v < V; v += SMP_THREADS) a.trunc_out[base + v] = kept(v, prob(v)) / K;
  if (!a.token_out) return;
  // ---- inverse CDF: first v with cumsum(kept / K) > u ----
  // the warp whose chunk holds the crossing walks it 32 keys at a time
  const double u = uniform_at(a.seed, (uint64_t)rc.pos);
  double before = 0.0;
  for (int w = 0; w < wid; ++w) before += wtot[w] / K;
  const double mine = wtot[wid] / K;
  const bool last_warp = c1 >= V || wid == NWARP - 1;
  if (tid == 0) s_int[1] = V;
  __syncthreads();
  // (chunk prefix sums and the walk round differently: neighbouring warps within
  // 1e-12 of the crossing also walk; the lowest hit wins)
  if (c0 < c1 && before <= u + 1e-12 && (before + mine > u - 1e-12 || last_warp)) {
    double c = before;
    for (int v0 = c0; v0 < c1; v0 += 32) {
      const int v = v0 + lane;
      double x = v < c1 ? kept(v, prob(v)) / K : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, v < c1 && c + x > u);
      if (hit) {
        if (lane == 0) atomicMin(&s_int[1], v0 + __ffs(hit) - 1);
        break;
      }
      c += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int idx = s_int[1];
    if (idx > V - 1) idx = V - 1;
    a.token_out[row] = idx;
  }
}

// Engine path (fp32 logits; no truncation, min-p or top-p; token draw only): a
// cluster of SC_CTAS CTAs per row, each owning a contiguous 1/SC_CTAS of the
// vocabulary, so a row is spread over 8 SMs instead of one. Cross-CTA
// reductions go through distributed shared memory and are combined in CTA
// order on every CTA (identical results everywhere, deterministic):
//   1. online max / sum-exp of the penalised scaled logits (sampling.py:142-162);
//   2. truncation: min-p keeps p >= p_base * p_max (sampling.py:207-210); top-p
//      bisects the nucleus threshold over the bit patterns of e = exp(s - max)
//      (fp32, positive: bit order == value order == order of p = e / Z, and equal
//      bits <=> equal p) with cluster-summed masses, ties at the threshold kept
//      lowest index first (sampling.py:198-205); then kept mass per CTA;
//   3. the CTA whose prefix holds u = uniform_at(seed, pos) walks its slice in
//      32-key warp chunks for the first cumsum > u (sampling.py:219-224).
constexpr int SC_CTAS = 8, SC_THREADS = 512;

__global__ void __cluster_dims__(SC_CTAS, 1, 1) __launch_bounds__(SC_THREADS, 3)
    sample_rows_cluster_kernel(const float* __restrict__ logits, SampleDev a) {
  extern __shared__ float ecache[];  // e = exp(s - max) of this CTA's slice
  __shared__ RowCtx rc;
  __shared__ float s_m;
  __shared__ double s_z, s_k;
  __shared__ double dred[32];
  __shared__ float fred[32];
  __shared__ double wtot[SC_THREADS / 32];
  __shared__ int s_hit;
  __shared__ double s_tot;
  __shared__ int s_cnt, s_vcut;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int row = blockIdx.x / SC_CTAS, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool live = row < a.rows && !(a.member_kind == SD_MEMBER_TREE && row >= a.tree[tree_off::T]);
  // a padded row's whole cluster leaves before any cluster barrier or DSMEM access
  // (every CTA of the cluster sees the same row and the same tree size)
  if (!live) return;
  const int V = a.V;
  const int v0 = (int)((int64_t)V * rank / SC_CTAS), v1 = (int)((int64_t)V * (rank + 1) / SC_CTAS);
  const float* lg = logits + (int64_t)row * V;
  if (live && tid == 0) {
    if (a.in_kind == SD_IN_SCALED_F32)
      rc.pos = row_pos(a, row);  // the LM head already applied the row's penalty splice
    else
      row_setup(a, row, rc);
  }
  __syncthreads();
  const float inv_t = (float)(1.0 / a.temperature), inv_tt = (float)(1.0 / (a.temperature * a.theta));
  const float th = (float)a.theta;
  // ---- 1. online max / sum-exp over this CTA's slice; the scaled logits are kept
  // in ecache (shared memory) so pass 2 never touches global memory ----
  auto scaled_w = [&](float l, int v, int word) -> float {
    if (!member_from(a, rc, v, word)) return l * inv_t;
    if (a.ctrl_style) return (l < 0.f ? l * th : l / th) * inv_t;
    return l * inv_tt;
  };
  float mf = -INFINITY;
  double Z = 0.0;
  if (a.in_kind == SD_IN_SCALED_F32) {
    // the LM-head epilogue (sd_lmhead_sample_stats) already penalised and scaled
    // the logits and left (max, sum-exp) per 128-token tile: this CTA only loads
    // its slice, and every CTA of the cluster combines the row's tile statistics
    // in the same fixed order (identical mf and Z on all eight)
    for (int v = v0 + tid; v < v1; v += SC_THREADS) ecache[v - v0] = lg[v];
    const double2* st = reinterpret_cast<const double2*>(a.stats) + (int64_t)row * a.stats_tiles;
    double tm = -INFINITY;
    for (int t = tid; t < a.stats_tiles; t += SC_THREADS) tm = fmax(tm, st[t].x);
    mf = (float)block_reduce(tm, dred, [](double x, double y) { return fmax(x, y); });
    double tz = 0.0;
    for (int t = tid; t < a.stats_tiles; t += SC_THREADS) {
      const double2 e = st[t];
      if (e.x != -INFINITY) tz += e.y * exp(e.x - (double)mf);
    }
    Z = block_reduce(tz, dred, [](double x, double y) { return x + y; });
  } else {
    float lm = -INFINITY;
    double lz = 0.0;
    constexpr int UB = 4;  // elements per thread per batch: all their loads issued first
    for (int vb = v0 + tid; vb < v1; vb += SC_THREADS * UB) {
      float lv[UB];
      int wv[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int v = vb + u * SC_THREADS;
        lv[u] = v < v1 ? lg[v] : 0.f;
        wv[u] = v < v1 ? member_word(a, row, v) : 0;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int v = vb + u * SC_THREADS;
        if (v < v1) {
          const float sv = scaled_w(lv[u], v, wv[u]);
          ecache[v - v0] = sv;
          if (sv > lm) {
            lz = lz * (double)expf(lm - sv);
            lm = sv;
          }
          lz += (double)expf(sv - lm);
        }
      }
    }
    const float cm = block_reduce(lm, fred, [](float x, float y) { return fmaxf(x, y); });
    lz = lm == -INFINITY ? 0.0 : lz * exp((double)lm - (double)cm);
    const double cz = block_reduce(lz, dred, [](double x, double y) { return x + y; });
    if (tid == 0) {
      s_m = cm;
      s_z = cz;
    }
    cluster.sync();
    for (int r = 0; r < SC_CTAS; ++r) mf = fmaxf(mf, *cluster.map_shared_rank(&s_m, r));
    for (int r = 0; r < SC_CTAS; ++r) {
      const float mr = *cluster.map_shared_rank(&s_m, r);
      const double zr = *cluster.map_shared_rank(&s_z, r);
      Z += mr == -INFINITY ? 0.0 : zr * exp((double)mr - (double)mf);
    }
  }
  const double invZ = 1.0 / Z;
  // warp-contiguous chunks of this CTA's slice (coalesced; chunk w = [c0, c1))
  constexpr int NW = SC_THREADS / 32;
  const int S = ((v1 - v0) + NW * 32 - 1) / (NW * 32) * 32;
  const int c0 = v0 + wid * S, c1 = min(v1, c0 + S);
  for (int i = tid; i < v1 - v0; i += SC_THREADS) ecache[i] = expf(ecache[i] - mf);  // same thread wrote i
  __syncthreads();
  auto ebits = [&](int v) -> int { return __float_as_int(ecache[v - v0]); };
  auto prob = [&](int v) -> double { return (double)ecache[v - v0] * invZ; };
  // min-p: p_max = exp(0) / Z, so keep p >= p_base / Z
  const double thr = a.trunc_kind == SD_TRUNC_MIN_P ? a.trunc_value * invZ : -1.0;
  int pbits = -1;  // top-p threshold: keep bits > pbits, and bits == pbits up to index vcut
  int vcut = V;
  if (a.trunc_kind == SD_TRUNC_TOP_P) {
    // cluster-wide masses of {e >= t_i} for NQ thresholds at once (fp64, CTA order):
    // an NQ+1-ary search over the bit range needs ~ceil(31 / log2(NQ+1)) passes
    constexpr int NQ = 1;  // binary search measured fastest (fp64 partial sums per threshold cost more than passes)
    __shared__ double s_q[SC_THREADS / 32][NQ];
    __shared__ double s_qc[NQ];
    auto mass_ge_n = [&](const int* t, double* out) {
      double ml[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) ml[i] = 0.0;
      double all = 0.0;  // elements at or above the top threshold count for every t_i
      if (live)
        for (int v = v0 + tid; v < v1; v += SC_THREADS) {
          const int b = ebits(v);
          if (b < t[0]) continue;  // the common case once the range has narrowed
          const double e = (double)ecache[v - v0];
          if (b >= t[NQ - 1]) {
            all += e;
          } else {
#pragma unroll
            for (int i = 0; i < NQ - 1; ++i) ml[i] += b >= t[i] ? e : 0.0;
          }
        }
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const double w = warp_sum_d(ml[i] + all);
        if (lane == 0) s_q[wid][i] = w;
      }
      __syncthreads();
      if (tid < NQ) {
        double c = 0.0;
        for (int w = 0; w < SC_THREADS / 32; ++w) c += s_q[w][tid];
        s_qc[tid] = c;
      }
      cluster.sync();
      if (tid < NQ) {
        double t2 = 0.0;
        for (int r = 0; r < SC_CTAS; ++r) t2 += cluster.map_shared_rank(s_qc, r)[tid];
        s_q[0][tid] = t2 * invZ;  // own smem scratch: peers only read s_qc
      }
      cluster.sync();  // s_qc is rewritten by the next query
#pragma unroll
      for (int i = 0; i < NQ; ++i) out[i] = s_q[0][i];
      __syncthreads();
    };
    int t0[NQ];
    double m0[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) t0[i] = i == 0 ? 0 : 0x7f800001;
    mass_ge_n(t0, m0);
    const double total = m0[0];
    if (a.trunc_value < total) {
      // largest b with mass(e >= b) >= top_p: an element's value; above = mass(e > b)
      int lo = 0, hi = 0x7f800001;
      double above = 0.0;
      while (hi - lo > 1) {
        int t[NQ];
        double mm[NQ];
        const int64_t span = (int64_t)hi - lo;
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
          int64_t ti = lo + span * (i + 1) / (NQ + 1);
          if (ti <= lo) ti = lo + 1;
          if (ti >= hi) ti = hi - 1;
          t[i] = (int)ti;
        }
        mass_ge_n(t, mm);
        // thresholds ascend, masses descend: lo = the largest t_i with mass >= top_p
        int nlo = lo, nhi = hi;
        double nabove = above;
#pragma unroll
        for (int i = NQ - 1; i >= 0; --i) {
          if (mm[i] >= a.trunc_value) {
            if (t[i] > nlo) nlo = t[i];
          } else if (t[i] < nhi) {
            nhi = t[i];
            nabove = mm[i];
          }
        }
        lo = nlo;
        hi = nhi;
        above = nabove;
      }
      pbits = lo;
      const double pstar = (double)__int_as_float(lo) * invZ;
      // elements equal to pstar: keep the lowest-index `need` of them
      int ce = 0;
      if (live)
        for (int v = v0 + tid; v < v1; v += SC_THREADS) ce += ebits(v) == lo;
      ce = (int)block_reduce((double)ce, dred, [](double x, double y) { return x + y; });
      if (tid == 0) {
        s_cnt = ce;
        s_vcut = V;
      }
      cluster.sync();
      int ceq = 0, before_eq = 0;
      for (int r = 0; r < SC_CTAS; ++r) {
        const int cr = *cluster.map_shared_rank(&s_cnt, r);
        if (r < rank) before_eq += cr;
        ceq += cr;
      }
      int need = (int)ceil((a.trunc_value - above) / pstar);
      if (need < 1) need = 1;
      if (need > ceq) need = ceq;
      if (need < ceq && before_eq < need && need <= before_eq + ce && live) {
        // the need-th equal element (index order) is in this CTA's slice: warp-chunk scan
        const int want = need - before_eq;
        int cw = 0;
        for (int v = c0 + lane; v < c1; v += 32) cw += ebits(v) == lo;
        cw = (int)warp_sum_d((double)cw);
        if (lane == 0) wtot[wid] = (double)cw;
        __syncthreads();
        int bw = 0;
        for (int w = 0; w < wid; ++w) bw += (int)wtot[w];
        if (bw < want && want <= bw + cw) {
          int cnt = bw;
          for (int vb = c0; vb < c1; vb += 32) {
            const int v = vb + lane;
            const unsigned eq = __ballot_sync(0xffffffffu, v < c1 && ebits(v) == lo);
            const int n_eq = __popc(eq);
            if (cnt + n_eq >= want) {
              unsigned m2 = eq;
              for (int k = cnt; k < want - 1; ++k) m2 &= m2 - 1;  // drop the lowest (want-1-cnt) bits
              if (lane == 0) *cluster.map_shared_rank(&s_vcut, 0) = vb + __ffs(m2) - 1;
              break;
            }
            cnt += n_eq;
          }
        }
        __syncthreads();
      }
      cluster.sync();
      vcut = need >= ceq ? V : *cluster.map_shared_rank(&s_vcut, 0);
    }
  }
  auto kept = [&](int v) -> double {
    const double p = prob(v);
    if (pbits >= 0) {
      const int b = ebits(v);
      return (b > pbits || (b == pbits && v <= vcut)) ? p : 0.0;
    }
    return p >= thr ? p : 0.0;
  };
  // ---- 2. kept mass in warp-contiguous chunks of this CTA's slice ----
  double lk = 0.0;
  if (live)
    for (int v = c0 + lane; v < c1; v += 32) lk += kept(v);
  lk = warp_sum_d(lk);
  if (lane == 0) wtot[wid] = lk;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += wtot[w];
    s_k = t;
    s_hit = 0x7fffffff;
  }
  cluster.sync();
  double K = 0.0, prefix = 0.0;
  for (int r = 0; r < SC_CTAS; ++r) {
    const double kr = *cluster.map_shared_rank(&s_k, r);
    if (r < rank) prefix += kr;
    K += kr;
  }
  // ---- 3. inverse CDF: first v with cumsum(kept / K) > u ----
  const double u = live ? uniform_at(a.seed, (uint64_t)rc.pos) : 2.0;
  double before = prefix / K;
  for (int w = 0; w < wid; ++w) before += wtot[w] / K;
  const double mine = wtot[wid] / K;
  const bool last_chunk = c1 >= V;
  if (live && c0 < c1 && before <= u + 1e-12 && (before + mine > u - 1e-12 || last_chunk)) {
    double c = before;
    for (int vb = c0; vb < c1; vb += 32) {
      const int v = vb + lane;
      double x = v < c1 ? kept(v) / K : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, v < c1 && c + x > u);
      if (hit) {
        if (lane == 0) atomicMin(cluster.map_shared_rank(&s_hit, 0), vb + __ffs(hit) - 1);
        break;
      }
      c += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  cluster.sync();
  if (live && rank == 0 && tid == 0) {
    int idx = s_hit;
    if (idx > V - 1) idx = V - 1;
    a.token_out[row] = idx;
  }
}

// draft per-head top-w (engine.py:207-215): a cluster of TW_CTAS CTAs per head,
// each CTA owning a contiguous 1/TW_CTAS of the vocabulary. Candidates are ranked
// by the penalised scaled logit s (exp(s - m) / Z is monotone in s), ties to the
// lower id. Each thread keeps a sorted top-W list; W rounds of block argmax give
// the CTA's top-W; cluster rank 0 reads every CTA's list through distributed
// shared memory and picks the head's top-w with the same order (slices ascend,
// so "lower id" stays exact across CTAs).
constexpr int TW_CTAS = 8, TW_THREADS = 512;

template <int W>
__global__ void __cluster_dims__(TW_CTAS, 1, 1) __launch_bounds__(TW_THREADS)
    draft_topw_kernel(const float* __restrict__ logits, int V, const int32_t* __restrict__ cnt, double t,
                      double theta, int ctrl, int w0, int w1, int w2, int w3, int w4, int w5, int w6, int w7,
                      int32_t* __restrict__ out) {
  __shared__ DI ared[32];
  __shared__ DI cand[W];  // this CTA's top-W, best first
  __shared__ DI all[TW_CTAS * W];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int head = blockIdx.x / TW_CTAS, tid = threadIdx.x;
  const int ws[8] = {w0, w1, w2, w3, w4, w5, w6, w7};
  int off = 0;
  for (int k = 0; k < head; ++k) off += ws[k];
  const int w = ws[head];
  const float* row = logits + (int64_t)head * V;
  const int v0 = (int)((int64_t)V * rank / TW_CTAS), v1 = (int)((int64_t)V * (rank + 1) / TW_CTAS);
  const double inv_t = 1.0 / t, inv_tt = 1.0 / (t * theta);
  double bv[W];
  int bi[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    bv[k] = -INFINITY;
    bi[k] = 0x7fffffff;
  }
  for (int v = v0 + tid; v < v1; v += TW_THREADS) {
    const double l = (double)row[v];
    const bool mem = cnt != nullptr && cnt[v] > 0;
    double sv;
    if (!mem) sv = l * inv_t;
    else if (ctrl) sv = (l < 0.0 ? l * theta : l / theta) * inv_t;
    else sv = l * inv_tt;
    // v increases within a thread: ties keep the earlier (lower) id
    if (sv > bv[W - 1]) {
      double cv = sv;
      int ci = v;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (cv > bv[k]) {
          const double tv = bv[k];
          const int ti = bi[k];
          bv[k] = cv;
          bi[k] = ci;
          cv = tv;
          ci = ti;
        }
      }
    }
  }
  int head_pos = 0;
  for (int j = 0; j < w; ++j) {
    DI mine{-INFINITY, 0x7fffffff};
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k == head_pos) mine = DI{bv[k], bi[k]};
    const DI best = block_argmax(mine, ared);
    if (best.i == mine.i && best.v == mine.v) ++head_pos;
    if (tid == 0) cand[j] = best;
  }
  cluster.sync();
  if (rank == 0 && tid < 32) {
    // gather the cluster's lists, then w rounds of warp argmax over them
    for (int e = tid; e < TW_CTAS * W; e += 32) {
      const int r = e / W, j = e - r * W;
      all[e] = j < w ? cluster.map_shared_rank(cand, r)[j] : DI{-INFINITY, 0x7fffffff};
    }
    __syncwarp();
    for (int j = 0; j < w; ++j) {
      DI b{-INFINITY, 0x7fffffff};
      int be = -1;
      for (int e = tid; e < TW_CTAS * W; e += 32) {
        const DI c = all[e];
        if (c.i != 0x7fffffff || c.v != -INFINITY) {
          const DI nb = better(b, c);
          if (nb.i != b.i || nb.v != b.v) be = e;
          b = nb;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        DI y;
        y.v = __shfl_xor_sync(0xffffffffu, b.v, o);
        y.i = __shfl_xor_sync(0xffffffffu, b.i, o);
        const int ye = __shfl_xor_sync(0xffffffffu, be, o);
        const DI nb = better(b, y);
        if (nb.i != b.i || nb.v != b.v) be = ye;
        b = nb;
      }
      if (tid == 0) {
        out[off + j] = b.i;
        if (be >= 0) all[be] = DI{-INFINITY, 0x7fffffff};  // taken
      }
      __syncwarp();
    }
  }
  cluster.sync();  // peers' lists stay alive until rank 0 has read them
}

}  // namespace sd

using namespace sd;

extern "C" {

int sd_sample_rows(const void* in, const sd_sample_args* args_host, sd_stream_t stream) {
  SD_REQUIRE(args_host && args_host->rows > 0 && args_host->V > 0, "sd_sample_rows: sizes");
  const sd_sample_args& h = *args_host;
  SD_REQUIRE(h.temperature > 0.0 && h.theta >= 1.0, "sd_sample_rows: temperature/theta");
  SD_REQUIRE(h.member_kind != SD_MEMBER_MASK || h.member_mask, "sd_sample_rows: mask");
  SD_REQUIRE(h.member_kind < SD_MEMBER_WINDOW || h.window == 0 || (h.win_count && h.state),
             "sd_sample_rows: window");
  SD_REQUIRE(h.member_kind != SD_MEMBER_TREE || h.tree, "sd_sample_rows: tree");
  SD_REQUIRE(h.positions || h.tree, "sd_sample_rows: need positions or tree");
  SampleDev d = to_dev(h);
  auto st = as_stream(stream);
  const bool cluster_ok = !h.probs_out && !h.trunc_out && h.token_out &&
      (h.trunc_kind == SD_TRUNC_NONE || h.trunc_kind == SD_TRUNC_MIN_P || h.trunc_kind == SD_TRUNC_TOP_P);
  if (h.in_kind == SD_IN_SCALED_F32)
    SD_REQUIRE(cluster_ok && h.stats && h.stats_tiles == (h.V + 127) / 128,
               "sd_sample_rows: scaled input needs the token draw only (no probs/trunc outputs, none/min-p/top-p) "
               "and the LM head's tile statistics");
  if ((h.in_kind == SD_IN_LOGITS_F32 || h.in_kind == SD_IN_SCALED_F32) && cluster_ok) {
    // engine path: one CTA cluster per row
    const size_t smem = (size_t)((h.V + SC_CTAS - 1) / SC_CTAS) * sizeof(float);
    SD_REQUIRE(smem <= 200 * 1024, "sd_sample_rows: vocabulary too large for the cluster path");
    static size_t attr_smem = 0;
    if (smem > 48 * 1024 && smem > attr_smem) {
      cudaFuncSetAttribute(sample_rows_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_smem = smem;
    }
    sample_rows_cluster_kernel<<<h.rows * SC_CTAS, SC_THREADS, smem, st>>>((const float*)in, d);
    return check_launch("sd_sample_rows(cluster)");
  }
  switch (h.in_kind) {
    case SD_IN_LOGITS_F32: sample_rows_kernel<SD_IN_LOGITS_F32><<<h.rows, SMP_THREADS, 0, st>>>(in, d); break;
    case SD_IN_LOGITS_F64: sample_rows_kernel<SD_IN_LOGITS_F64><<<h.rows, SMP_THREADS, 0, st>>>(in, d); break;
    case SD_IN_PROBS_F64: sample_rows_kernel<SD_IN_PROBS_F64><<<h.rows, SMP_THREADS, 0, st>>>(in, d); break;
    default: SD_REQUIRE(false, "sd_sample_rows: in_kind");
  }
  return check_launch("sd_sample_rows");
}

int sd_draft_topw(const float* logits, int heads, int V, const int32_t* win_count, double temperature, double theta,
                  int ctrl_style, const int32_t* widths_host, int32_t* out, sd_stream_t stream) {
  SD_REQUIRE(heads > 0 && heads <= SD_TREE_MAX_DEPTH && V > 0, "sd_draft_topw: sizes");
  int w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int wmax = 0;
  for (int k = 0; k < heads; ++k) {
    SD_REQUIRE(widths_host[k] >= 1 && widths_host[k] <= 16 && widths_host[k] <= V, "sd_draft_topw: width");
    w[k] = widths_host[k];
    wmax = w[k] > wmax ? w[k] : wmax;
  }
  auto st = as_stream(stream);
#define SD_TOPW(W) draft_topw_kernel<W><<<heads * TW_CTAS, TW_THREADS, 0, st>>>(logits, V, win_count, temperature, theta, \
                                                                       ctrl_style, w[0], w[1], w[2], w[3], w[4], \
                                                                       w[5], w[6], w[7], out)
  if (wmax <= 4) SD_TOPW(4); else if (wmax <= 8) SD_TOPW(8); else SD_TOPW(16);
#undef SD_TOPW
  return check_launch("sd_draft_topw");
}

}  // extern "C"
