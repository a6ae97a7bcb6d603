// Integer-exact control path of the decode step, device resident:
//  * n-gram table (ngram.py:18-66): open-addressing hash of n-token keys with
//    per-first-token chains, exact counts and a global recency clock;
//  * candidate tree (tree.py:87-175): Cartesian-product head trie in DFS order
//    plus greedily merged n-gram chains, ancestor-closure row masks;
//  * acceptance (engine.py:247-274): exact-match path validity, uniform pick
//    among the longest at uniform_at(select_seed, n), bonus token;
//  * commit (engine.py:276-290): history, penalty window ring, n-gram update,
//    pending token for the next step.
// These are latency-bound (a few hundred integer ops per step), run by one
// thread of one CTA so the whole step needs no host round trip.
#include "common.cuh"

namespace sd {

// ------------------------------------------------------------- n-gram ------
struct NgView {
  int64_t* hdr;  // [0] n [1] cap [2] V [3] size [4] clock [5] error
  int64_t* last;
  int32_t* keys;
  int32_t* freq;
  int32_t* next;
  int32_t* head;
};

__host__ __device__ inline size_t ng_align(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline NgView ng_view(void* base, int n, int cap, int V) {
  char* p = (char*)base;
  NgView v;
  v.hdr = (int64_t*)p;
  p += 256;
  v.last = (int64_t*)p;
  p += ng_align((size_t)cap * 8);
  v.keys = (int32_t*)p;
  p += ng_align((size_t)cap * n * 4);
  v.freq = (int32_t*)p;
  p += ng_align((size_t)cap * 4);
  v.next = (int32_t*)p;
  p += ng_align((size_t)cap * 4);
  v.head = (int32_t*)p;
  (void)V;
  return v;
}

__device__ inline NgView ng_dev(void* base) {
  const int64_t* h = (const int64_t*)base;
  return ng_view(base, (int)h[0], (int)h[1], (int)h[2]);
}

__device__ inline uint64_t ng_hash(const int32_t* g, int n) {
  uint64_t x = 0x51ED27A3ull;
  for (int i = 0; i < n; ++i) x = splitmix64(x ^ (uint64_t)(uint32_t)g[i]);
  return x;
}

// find slot of gram (or the empty slot where it would go); -1 if table full
__device__ inline int ng_find(const NgView& t, const int32_t* g, int n, int cap, bool* found) {
  int idx = (int)(ng_hash(g, n) & (uint64_t)(cap - 1));
  for (int probe = 0; probe < cap; ++probe) {
    const int32_t* k = t.keys + (int64_t)idx * n;
    if (k[0] == -1) {
      *found = false;
      return idx;
    }
    bool eq = true;
    for (int i = 0; i < n; ++i) eq &= k[i] == g[i];
    if (eq) {
      *found = true;
      return idx;
    }
    idx = (idx + 1) & (cap - 1);
  }
  *found = false;
  return -1;
}

// count every window of length n ending in seq[n_tail, n_tail + n_new)
__device__ void ng_update_dev(void* base, const int32_t* seq, int n_tail, int n_new) {
  NgView t = ng_dev(base);
  const int n = (int)t.hdr[0], cap = (int)t.hdr[1];
  for (int end = n_tail; end < n_tail + n_new; ++end) {
    const int start = end + 1 - n;
    if (start < 0) continue;
    const int32_t* g = seq + start;
    const int64_t clock = ++t.hdr[4];
    bool found;
    const int idx = ng_find(t, g, n, cap, &found);
    if (idx < 0) {
      t.hdr[5] = 1;  // overflow
      continue;
    }
    if (found) {
      t.freq[idx] += 1;
    } else {
      for (int i = 0; i < n; ++i) t.keys[(int64_t)idx * n + i] = g[i];
      t.freq[idx] = 1;
      t.next[idx] = t.head[g[0]];
      t.head[g[0]] = idx;
      t.hdr[3] += 1;
    }
    t.last[idx] = clock;
  }
}

// top-k by (freq desc, last desc) among grams starting with `first`
__device__ int ng_retrieve_dev(const void* base, int first, int k, int32_t* out) {
  NgView t = ng_dev((void*)base);
  const int n = (int)t.hdr[0], V = (int)t.hdr[2];
  if (k <= 0 || first < 0 || first >= V) return 0;
  int sel[64];
  int cnt = 0;
  for (int e = t.head[first]; e >= 0; e = t.next[e]) {
    // insertion into sorted `sel`
    const int f = t.freq[e];
    const int64_t l = t.last[e];
    int pos = cnt;
    while (pos > 0) {
      const int o = sel[pos - 1];
      const bool worse = t.freq[o] > f || (t.freq[o] == f && t.last[o] > l);
      if (worse) break;
      --pos;
    }
    if (pos >= k) continue;
    const int upto = cnt < k ? cnt : k - 1;
    for (int j = upto; j > pos; --j) sel[j] = sel[j - 1];
    sel[pos] = e;
    if (cnt < k) ++cnt;
  }
  for (int i = 0; i < cnt; ++i)
    for (int j = 0; j < n; ++j) out[i * n + j] = t.keys[(int64_t)sel[i] * n + j];
  return cnt;
}

__global__ void ng_init_kernel(void* base, int n, int cap, int V) {
  NgView t = ng_view(base, n, cap, V);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < (int64_t)cap * n; i += stride) t.keys[i] = -1;
  for (int64_t i = tid; i < cap; i += stride) {
    t.freq[i] = 0;
    t.next[i] = -1;
    t.last[i] = 0;
  }
  for (int64_t i = tid; i < V; i += stride) t.head[i] = -1;
  if (tid == 0) {
    t.hdr[0] = n;
    t.hdr[1] = cap;
    t.hdr[2] = V;
    t.hdr[3] = 0;
    t.hdr[4] = 0;
    t.hdr[5] = 0;
  }
}

__global__ void ng_update_kernel(void* base, const int32_t* seq, int n_tail, int n_new) {
  if (threadIdx.x == 0 && blockIdx.x == 0) ng_update_dev(base, seq, n_tail, n_new);
}

__global__ void ng_retrieve_kernel(const void* base, const int32_t* first, int k, int32_t* out, int32_t* count) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *count = ng_retrieve_dev(base, *first, k, out);
}

__global__ void ng_frequency_kernel(const void* base, const int32_t* grams, int count, int32_t* out) {
  NgView t = ng_dev((void*)base);
  const int n = (int)t.hdr[0], cap = (int)t.hdr[1];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    bool found;
    const int idx = ng_find(t, grams + (int64_t)i * n, n, cap, &found);
    out[i] = (idx >= 0 && found) ? t.freq[idx] : 0;
  }
}

__global__ void ng_size_kernel(const void* base, int32_t* out) {
  if (threadIdx.x == 0) *out = (int32_t)((const int64_t*)base)[3];
}

// --------------------------------------------------------------- tree ------
struct Widths {
  int w[SD_TREE_MAX_DEPTH];
};

// Single-thread build into `tr` (a zeroed shared-memory copy of the record; the
// trie links live in shared memory too). The ancestor masks are left to
// tree_masks_dev, which the whole block runs afterwards.
__device__ void tree_build_dev(const int32_t* per_head, const Widths& W, int K, const int32_t* grams, int n_grams,
                               int pending, int64_t base_pos, int32_t* tr, int64_t* state, int16_t* first_child,
                               int16_t* next_sib) {
  using namespace tree_off;
  int n_nodes = 0, n_paths = 0;
  int root_first = -1;
  bool overflow = false;
  int hoff[SD_TREE_MAX_DEPTH];
  int acc = 0;
  for (int d = 0; d < K; ++d) {
    hoff[d] = acc;
    acc += W.w[d];
  }
  auto add_node = [&](int parent, int tok, int dep) -> int {
    if (n_nodes + 1 >= SD_TREE_MAX_ROWS) {
      overflow = true;
      return -1;
    }
    const int id = n_nodes++;
    tr[TOK + 1 + id] = tok;
    tr[POS + 1 + id] = (int32_t)(base_pos + 1 + dep);
    tr[PARENT + id] = parent;
    tr[NDEPTH + id] = dep;
    first_child[id] = -1;
    next_sib[id] = -1;
    // append to the parent's child list (lookup is by token, order is irrelevant)
    if (parent < 0) {
      next_sib[id] = root_first;
      root_first = id;
    } else {
      next_sib[id] = first_child[parent];
      first_child[parent] = id;
    }
    return id;
  };
  auto find_child = [&](int parent, int tok) -> int {
    for (int c = parent < 0 ? root_first : first_child[parent]; c >= 0; c = next_sib[c])
      if (tr[TOK + 1 + c] == tok) return c;
    return -1;
  };
  // head trie: Cartesian product in lexicographic (DFS) order
  int digit[SD_TREE_MAX_DEPTH];
  int cur[SD_TREE_MAX_DEPTH];
  for (int d = 0; d < K; ++d) digit[d] = 0;
  int changed = 0;  // lowest depth whose digit changed
  bool done = K == 0;
  int rank = 0;
  while (!done && !overflow) {
    for (int d = changed; d < K; ++d) cur[d] = add_node(d ? cur[d - 1] : -1, per_head[hoff[d] + digit[d]], d);
    if (overflow || n_paths >= SD_TREE_MAX_PATHS) {
      overflow = true;
      break;
    }
    for (int d = 0; d < K; ++d) tr[PNODES + n_paths * SD_TREE_MAX_DEPTH + d] = cur[d];
    tr[PORIGIN + n_paths] = 0;
    tr[POIDX + n_paths] = rank++;
    ++n_paths;
    // increment mixed-radix counter (last digit fastest)
    int d = K - 1;
    while (d >= 0 && ++digit[d] == W.w[d]) digit[d--] = 0;
    if (d < 0) done = true;
    changed = d;
  }
  const int head_nodes = n_nodes;
  for (int r = 0; r < n_grams && !overflow; ++r) {
    const int32_t* g = grams + r * K;
    bool dup = false;
    for (int p = 0; p < n_paths && !dup; ++p) {
      bool eq = true;
      for (int d = 0; d < K && eq; ++d) eq = tr[TOK + 1 + tr[PNODES + p * SD_TREE_MAX_DEPTH + d]] == g[d];
      dup = eq;
    }
    if (dup) continue;
    int c = -1;
    for (int d = 0; d < K; ++d) {
      int nx = find_child(c, g[d]);
      if (nx < 0) nx = add_node(c, g[d], d);
      if (nx < 0) break;
      cur[d] = nx;
      c = nx;
    }
    if (overflow || n_paths >= SD_TREE_MAX_PATHS) {
      overflow = true;
      break;
    }
    for (int d = 0; d < K; ++d) tr[PNODES + n_paths * SD_TREE_MAX_DEPTH + d] = cur[d];
    tr[PORIGIN + n_paths] = 1;
    tr[POIDX + n_paths] = r;
    ++n_paths;
  }
  const int T = 1 + n_nodes;
  tr[tree_off::T] = T;
  tr[NPATHS] = n_paths;
  tr[HEADNODES] = head_nodes;
  tr[DEPTH] = K;
  tr[NGRAMS] = n_grams;
  tr[TOK] = pending;
  tr[POS] = (int32_t)base_pos;
  // padded rows (a fixed-shape verify forward reads them): root token / position
  for (int r = T; r < SD_TREE_MAX_ROWS; ++r) {
    tr[TOK + r] = pending < 0 ? 0 : pending;
    tr[POS + r] = (int32_t)base_pos;
  }
  if (overflow && state) state[SD_ST_ERROR] |= 2;
}

// ancestor-closure row masks over request rows (row 0 = root), one row per thread
__device__ void tree_masks_dev(int32_t* tr) {
  using namespace tree_off;
  const int T = tr[tree_off::T];
  for (int r = threadIdx.x; r < T; r += blockDim.x) {
    uint32_t bits[SD_MASK_WORDS];
    for (int w = 0; w < SD_MASK_WORDS; ++w) bits[w] = 0;
    bits[0] = 1u;
    for (int x = r - 1; x >= 0; x = tr[PARENT + x]) bits[(x + 1) >> 5] |= 1u << ((x + 1) & 31);
    for (int w = 0; w < SD_MASK_WORDS; ++w) tr[MASK + r * SD_MASK_WORDS + w] = (int32_t)bits[w];
  }
}

// The record is assembled in shared memory (zeroed first, so every field the
// build does not set reads as 0) and written out with 16-byte stores.
constexpr int TREE_THREADS = 128;
static_assert(tree_off::TOTAL % 4 == 0, "tree record copied as int4");

__device__ void tree_stage_zero(int32_t* str) {
  for (int i = threadIdx.x; i < tree_off::TOTAL / 4; i += blockDim.x)
    reinterpret_cast<int4*>(str)[i] = make_int4(0, 0, 0, 0);
  __syncthreads();
}
__device__ void tree_stage_out(const int32_t* str, int32_t* tree) {
  __syncthreads();
  tree_masks_dev(const_cast<int32_t*>(str));
  __syncthreads();
  for (int i = threadIdx.x; i < tree_off::TOTAL / 4; i += blockDim.x)
    reinterpret_cast<int4*>(tree)[i] = reinterpret_cast<const int4*>(str)[i];
}

__global__ void tree_build_kernel(const int32_t* per_head, Widths W, int K, const int32_t* grams,
                                  const int32_t* n_grams_dev, int n_grams_host, const int64_t* state,
                                  int64_t base_pos, int32_t* tree) {
  __shared__ __align__(16) int32_t str[tree_off::TOTAL];
  __shared__ int16_t fc[SD_TREE_MAX_ROWS], nsib[SD_TREE_MAX_ROWS];
  if (base_pos < 0) base_pos = state[SD_ST_BASE];
  tree_stage_zero(str);
  if (threadIdx.x == 0) {
    const int ng = n_grams_dev ? *n_grams_dev : n_grams_host;
    const int pending = state ? (int)state[SD_ST_PENDING] : -1;
    tree_build_dev(per_head, W, K, grams, ng, pending, base_pos, str, (int64_t*)state, fc, nsib);
  }
  tree_stage_out(str, tree);
}

__global__ void draft_tree_kernel(const void* ngram, int k, const int32_t* per_head, Widths W, int K,
                                  const int64_t* state, int64_t base_pos, int32_t* grams, int32_t* tree) {
  __shared__ __align__(16) int32_t str[tree_off::TOTAL];
  __shared__ int16_t fc[SD_TREE_MAX_ROWS], nsib[SD_TREE_MAX_ROWS];
  if (base_pos < 0) base_pos = state[SD_ST_BASE];
  tree_stage_zero(str);
  if (threadIdx.x == 0) {
    int ng = 0;
    if (ngram && k > 0) ng = ng_retrieve_dev(ngram, per_head[0], k, grams);
    tree_build_dev(per_head, W, K, grams, ng, (int)state[SD_ST_PENDING], base_pos, str, (int64_t*)state, fc, nsib);
  }
  tree_stage_out(str, tree);
}

// ----------------------------------------------------- accept + commit -----
__device__ void window_push_dev(int tok, int64_t* state, int32_t* ring, int32_t* cnt, int W) {
  if (W <= 0) return;
  int64_t head = state[SD_ST_RING_HEAD], len = state[SD_ST_RING_LEN];
  if (len == W) {
    cnt[ring[head]] -= 1;
    ring[head] = tok;
    head = (head + 1) % W;
  } else {
    ring[(head + len) % W] = tok;
    ++len;
  }
  cnt[tok] += 1;
  state[SD_ST_RING_HEAD] = head;
  state[SD_ST_RING_LEN] = len;
}

__global__ void accept_commit_kernel(const int32_t* __restrict__ tr, const int32_t* __restrict__ y,
                                     uint64_t select_seed, int64_t n, int K, int bonus, int64_t* state,
                                     int32_t* ring, int32_t* cnt, int W, int32_t* history, void* ngram,
                                     int32_t* result) {
  using namespace tree_off;
  __shared__ int best[SD_TREE_MAX_PATHS];
  if (blockIdx.x) return;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  if (n < 0) n = state[SD_ST_BASE] + 1;  // device-resident step (graph replay)
  const int P = tr[NPATHS];
  // path validity, one path per lane; the longest valid prefix and the paths that
  // reach it, in ascending path order (ballot compaction)
  constexpr int PK = SD_TREE_MAX_PATHS / 32;
  int vloc[PK];
  int best_v = -1;
#pragma unroll
  for (int k = 0; k < PK; ++k) {
    const int p = k * 32 + lane;
    int v = -1;
    if (k * 32 < P && p < P) {
      int expect = y[0];
      v = 0;
      for (int j = 0; j < K; ++j) {
        const int node = tr[PNODES + p * SD_TREE_MAX_DEPTH + j];
        if (tr[TOK + 1 + node] != expect) break;
        ++v;
        expect = y[1 + node];
      }
    }
    vloc[k] = v;
    best_v = max(best_v, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best_v = max(best_v, __shfl_xor_sync(0xffffffffu, best_v, o));
  int nb = 0;
#pragma unroll
  for (int k = 0; k < PK; ++k) {
    const bool hit = k * 32 + lane < P && vloc[k] == best_v;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) best[nb + __popc(m & ((1u << lane) - 1u))] = k * 32 + lane;
    nb += __popc(m);
  }
  __syncwarp();
  if (lane) return;  // the commit below is sequential
  const int pick = best[(int)(uniform_at(select_seed, (uint64_t)n) * (double)nb)];
  int a = bonus ? (best_v + 1 < K ? best_v + 1 : K) : (best_v > 1 ? best_v : 1);
  int ys[SD_TREE_MAX_DEPTH], keep[SD_TREE_MAX_DEPTH];
  ys[0] = y[0];
  keep[0] = 0;
  for (int j = 0; j + 1 < a; ++j) {
    const int node = tr[PNODES + pick * SD_TREE_MAX_DEPTH + j];
    ys[j + 1] = y[1 + node];
    keep[j + 1] = 1 + node;
  }
  result[SD_RES_ACCEPTED] = a;
  result[SD_RES_BEST] = best_v;
  result[SD_RES_PICK] = pick;
  result[SD_RES_ORIGIN] = tr[PORIGIN + pick];
  result[SD_RES_ROWS] = tr[tree_off::T];
  result[SD_RES_PATHS] = P;
  result[SD_RES_BASE] = (int32_t)(n - 1);
  for (int j = 0; j < SD_TREE_MAX_DEPTH; ++j) {
    result[SD_RES_YS + j] = j < a ? ys[j] : -1;
    result[SD_RES_KEEP + j] = j < a ? keep[j] : -1;
  }
  // commit: tail of the emitted history (before this step), then append
  const int64_t hl = state[SD_ST_HIST_LEN];
  const int tail = (int)((K - 1) < hl ? (K - 1) : hl);
  int32_t seq[2 * SD_TREE_MAX_DEPTH];
  for (int j = 0; j < tail; ++j) seq[j] = history[hl - tail + j];
  for (int j = 0; j < a; ++j) {
    seq[tail + j] = ys[j];
    history[hl + j] = ys[j];
    window_push_dev(ys[j], state, ring, cnt, W);
  }
  state[SD_ST_HIST_LEN] = hl + a;
  state[SD_ST_BASE] = n - 1 + a;
  state[SD_ST_PENDING] = ys[a - 1];
  result[SD_RES_PENDING] = ys[a - 1];
  if (ngram) ng_update_dev(ngram, seq, tail, a);
}

__global__ void window_push_kernel(const int32_t* tokens, int count, int64_t* state, int32_t* ring, int32_t* cnt,
                                   int W) {
  if (threadIdx.x || blockIdx.x) return;
  for (int i = 0; i < count; ++i) window_push_dev(tokens[i], state, ring, cnt, W);
}

static Widths widths_from(const int32_t* w, int K) {
  Widths W;
  for (int d = 0; d < SD_TREE_MAX_DEPTH; ++d) W.w[d] = d < K ? w[d] : 0;
  return W;
}

}  // namespace sd

using namespace sd;

extern "C" {

size_t sd_ngram_bytes(int n, int cap, int V) {
  return 256 + ng_align((size_t)cap * 8) + ng_align((size_t)cap * n * 4) + 2 * ng_align((size_t)cap * 4) +
         ng_align((size_t)V * 4);
}

int sd_ngram_init(void* table, int n, int cap, int V, sd_stream_t stream) {
  SD_REQUIRE(n >= 1 && n <= 16 && cap >= 2 && (cap & (cap - 1)) == 0 && V > 0, "sd_ngram_init: n/cap/V");
  ng_init_kernel<<<256, 256, 0, as_stream(stream)>>>(table, n, cap, V);
  return check_launch("sd_ngram_init");
}

int sd_ngram_update(void* table, const int32_t* seq, int n_tail, int n_new, sd_stream_t stream) {
  SD_REQUIRE(n_tail >= 0 && n_new >= 0, "sd_ngram_update: sizes");
  ng_update_kernel<<<1, 32, 0, as_stream(stream)>>>(table, seq, n_tail, n_new);
  return check_launch("sd_ngram_update");
}

int sd_ngram_retrieve(const void* table, const int32_t* first, int k, int32_t* out_grams, int32_t* out_count,
                      sd_stream_t stream) {
  SD_REQUIRE(k >= 0 && k <= 64, "sd_ngram_retrieve: k %d", k);
  ng_retrieve_kernel<<<1, 32, 0, as_stream(stream)>>>(table, first, k, out_grams, out_count);
  return check_launch("sd_ngram_retrieve");
}

int sd_ngram_frequency(const void* table, const int32_t* grams, int count, int32_t* out, sd_stream_t stream) {
  if (count <= 0) return SD_OK;
  ng_frequency_kernel<<<(count + 127) / 128, 128, 0, as_stream(stream)>>>(table, grams, count, out);
  return check_launch("sd_ngram_frequency");
}

int sd_ngram_size(const void* table, int32_t* out, sd_stream_t stream) {
  ng_size_kernel<<<1, 32, 0, as_stream(stream)>>>(table, out);
  return check_launch("sd_ngram_size");
}

int sd_tree_layout(int32_t* o, int n) {
  using namespace tree_off;
  const int32_t v[] = {tree_off::T, NPATHS, HEADNODES, DEPTH, NGRAMS, TOK, POS, PARENT, NDEPTH,
                       PNODES, PORIGIN, POIDX, MASK, TOTAL, SD_TREE_MAX_ROWS, SD_TREE_MAX_PATHS,
                       SD_TREE_MAX_DEPTH, SD_MASK_WORDS};
  const int cnt = (int)(sizeof(v) / sizeof(v[0]));
  for (int i = 0; i < n && i < cnt; ++i) o[i] = v[i];
  return cnt;
}

int sd_tree_build(const int32_t* per_head, const int32_t* widths_host, int depth, const int32_t* grams,
                  const int32_t* n_grams_dev, int n_grams_host, const int64_t* state, int64_t base_pos,
                  int32_t* tree, sd_stream_t stream) {
  SD_REQUIRE(depth >= 1 && depth <= SD_TREE_MAX_DEPTH, "sd_tree_build: depth");
  tree_build_kernel<<<1, TREE_THREADS, 0, as_stream(stream)>>>(per_head, widths_from(widths_host, depth), depth, grams,
                                                     n_grams_dev, n_grams_host, state, base_pos, tree);
  return check_launch("sd_tree_build");
}

int sd_draft_tree(const void* ngram_table, int k, const int32_t* per_head, const int32_t* widths_host, int depth,
                  const int64_t* state, int64_t base_pos, int32_t* grams_scratch, int32_t* tree, sd_stream_t stream) {
  SD_REQUIRE(depth >= 1 && depth <= SD_TREE_MAX_DEPTH && k >= 0 && k <= 64, "sd_draft_tree: depth/k");
  draft_tree_kernel<<<1, TREE_THREADS, 0, as_stream(stream)>>>(ngram_table, k, per_head, widths_from(widths_host, depth),
                                                     depth, state, base_pos, grams_scratch, tree);
  return check_launch("sd_draft_tree");
}

int sd_accept_commit(const int32_t* tree, const int32_t* y, uint64_t select_seed, int64_t n, int depth, int bonus,
                     int64_t* state, int32_t* win_ring, int32_t* win_count, int window, int32_t* history,
                     void* ngram_table, int32_t* result, sd_stream_t stream) {
  SD_REQUIRE(depth >= 1 && depth <= SD_TREE_MAX_DEPTH, "sd_accept_commit: depth");
  accept_commit_kernel<<<1, 32, 0, as_stream(stream)>>>(tree, y, select_seed, n, depth, bonus, state, win_ring,
                                                        win_count, window, history, ngram_table, result);
  return check_launch("sd_accept_commit");
}

int sd_window_push(const int32_t* tokens, int count, int64_t* state, int32_t* win_ring, int32_t* win_count,
                   int window, sd_stream_t stream) {
  if (count <= 0) return SD_OK;
  window_push_kernel<<<1, 32, 0, as_stream(stream)>>>(tokens, count, state, win_ring, win_count, window);
  return check_launch("sd_window_push");
}

}  // extern "C"
