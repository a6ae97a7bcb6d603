// Sampler arguments, per-row window splice and membership tests shared by the
// sampling kernels (sampling.cu) and the LM-head epilogue that computes the
// penalised logits' statistics (gemm_tc.cu). Reference: sampling.py:98-153,
// engine.py:155-181, 237-245.
#pragma once
#include "common.cuh"

namespace sd {

struct SampleDev {
  int rows, V, in_kind;
  double temperature, theta;
  int ctrl_style, member_kind;
  const uint8_t* member_mask;
  const int32_t* win_count;
  const int32_t* win_ring;
  const int64_t* state;
  int window;
  const int32_t* tree;
  int depth;
  int trunc_kind;
  double trunc_value, eta_alpha;
  uint64_t seed;
  const int32_t* positions;
  int64_t n;
  double* probs_out;
  double* trunc_out;
  int32_t* token_out;
  const double* stats;  // SD_IN_SCALED_F32: [rows][stats_tiles][2] (max, sum exp(s - max)) of the scaled logits
  int stats_tiles;
};

constexpr int MAX_PATCH = 2 * SD_TREE_MAX_DEPTH;


struct RowCtx {
  int n_patch;
  int patch_tok[MAX_PATCH];
  int patch_val[MAX_PATCH];
  uint32_t bloom[32];  // bit (v & 1023) set for every patched token v
  int64_t pos;
};

static __device__ __forceinline__ bool is_member(const SampleDev& a, const RowCtx& rc, int row, int v) {
  switch (a.member_kind) {
    case SD_MEMBER_MASK: return a.member_mask[(int64_t)row * a.V + v] != 0;
    case SD_MEMBER_WINDOW: return a.window > 0 && a.win_count[v] > 0;
    case SD_MEMBER_TREE: {
      if (a.window <= 0) return false;
      bool m = a.win_count[v] > 0;
      if ((rc.bloom[(v >> 5) & 31] >> (v & 31)) & 1u)  // rare: v may be a patched token
        for (int i = 0; i < rc.n_patch; ++i)
          if (rc.patch_tok[i] == v) m = rc.patch_val[i] != 0;
      return m;
    }
    default: return false;
  }
}

// is_member split in two: the per-element word (loaded in batches, so a thread
// keeps several global loads in flight) and the decision from it
static __device__ __forceinline__ int member_word(const SampleDev& a, int row, int v) {
  switch (a.member_kind) {
    case SD_MEMBER_MASK: return a.member_mask[(int64_t)row * a.V + v];
    case SD_MEMBER_WINDOW:
    case SD_MEMBER_TREE: return a.window > 0 ? a.win_count[v] : 0;
    default: return 0;
  }
}
static __device__ __forceinline__ bool member_from(const SampleDev& a, const RowCtx& rc, int v, int word) {
  switch (a.member_kind) {
    case SD_MEMBER_MASK: return word != 0;
    case SD_MEMBER_WINDOW: return a.window > 0 && word > 0;
    case SD_MEMBER_TREE: {
      if (a.window <= 0) return false;
      bool m = word > 0;
      if ((rc.bloom[(v >> 5) & 31] >> (v & 31)) & 1u)
        for (int i = 0; i < rc.n_patch; ++i)
          if (rc.patch_tok[i] == v) m = rc.patch_val[i] != 0;
      return m;
    }
    default: return false;
  }
}

template <int IN>
static __device__ __forceinline__ double load_in(const void* in, int64_t idx) {
  if (IN == SD_IN_LOGITS_F32) return (double)((const float*)in)[idx];
  return ((const double*)in)[idx];
}

// scaled logit l / (t * I) (sampling.py:142-153)
static __device__ __forceinline__ double scaled(double l, bool member, const SampleDev& a) {
  if (!member) return l / a.temperature;
  if (a.ctrl_style) return (l < 0.0 ? l * a.theta : l / a.theta) / a.temperature;
  return l / (a.temperature * a.theta);
}

// thread 0: per-row patches (engine.py:155-181) and draw position
// the draw key of a row: explicit positions, or n / n + depth + 1 from the tree
static __device__ __forceinline__ int64_t row_pos(const SampleDev& a, int row) {
  if (a.positions) return a.positions[row];
  const int64_t n = a.n >= 0 ? a.n : a.state[SD_ST_BASE] + 1;  // n < 0: device-resident step
  return row == 0 ? n : n + a.tree[tree_off::NDEPTH + row - 1] + 1;
}

static __device__ __noinline__ void row_setup(const SampleDev& a, int row, RowCtx& rc) {
  rc.n_patch = 0;
  for (int i = 0; i < 32; ++i) rc.bloom[i] = 0u;
  rc.pos = row_pos(a, row);
  if (a.member_kind != SD_MEMBER_TREE || a.window <= 0 || row == 0) return;
  const int W = a.window;
  const int node = row - 1;
  int branch[SD_TREE_MAX_DEPTH];
  int b = 0;
  for (int x = node; x >= 0 && b < SD_TREE_MAX_DEPTH; x = a.tree[tree_off::PARENT + x])
    branch[b++] = a.tree[tree_off::TOK + 1 + x];  // deepest first
  const int64_t ring = a.state[SD_ST_RING_LEN], head = a.state[SD_ST_RING_HEAD];
  int64_t cap = a.depth < ring ? a.depth : ring;
  int64_t drop = ring + b - W;
  if (drop < 0) drop = 0;
  if (drop > cap) drop = cap;
  // tokens slid out of the window (oldest first), with their removal counts
  for (int64_t j = 0; j < drop; ++j) {
    const int tok = a.win_ring[(head + j) % W];
    int found = -1;
    for (int i = 0; i < rc.n_patch; ++i)
      if (rc.patch_tok[i] == tok) found = i;
    if (found < 0) {
      found = rc.n_patch++;
      rc.patch_tok[found] = tok;
      rc.patch_val[found] = 0;  // used as removal counter for now
    }
    rc.patch_val[found] += 1;
  }
  for (int i = 0; i < rc.n_patch; ++i) rc.patch_val[i] = (a.win_count[rc.patch_tok[i]] - rc.patch_val[i]) > 0;
  const int tail = b < W ? b : W;  // last min(b, W) branch tokens = the deepest `tail`
  for (int j = 0; j < tail; ++j) {
    const int tok = branch[j];
    int found = -1;
    for (int i = 0; i < rc.n_patch; ++i)
      if (rc.patch_tok[i] == tok) found = i;
    if (found < 0) {
      found = rc.n_patch++;
      rc.patch_tok[found] = tok;
    }
    rc.patch_val[found] = 1;
  }
  for (int i = 0; i < rc.n_patch; ++i) {
    const int v = rc.patch_tok[i];
    rc.bloom[(v >> 5) & 31] |= 1u << (v & 31);
  }
}


static inline SampleDev to_dev(const sd_sample_args& h) {
  SampleDev d;
  d.rows = h.rows;
  d.V = h.V;
  d.in_kind = h.in_kind;
  d.temperature = h.temperature;
  d.theta = h.theta;
  d.ctrl_style = h.ctrl_style;
  d.member_kind = h.member_kind;
  d.member_mask = h.member_mask;
  d.win_count = h.win_count;
  d.win_ring = h.win_ring;
  d.state = h.state;
  d.window = h.window;
  d.tree = h.tree;
  d.depth = h.depth;
  d.trunc_kind = h.trunc_kind;
  d.trunc_value = h.trunc_value;
  d.eta_alpha = h.eta_alpha;
  d.seed = h.seed;
  d.positions = h.positions;
  d.n = h.n;
  d.probs_out = h.probs_out;
  d.trunc_out = h.trunc_out;
  d.token_out = h.token_out;
  d.stats = h.stats;
  d.stats_tiles = h.stats_tiles;
  return d;
}


}  // namespace sd
