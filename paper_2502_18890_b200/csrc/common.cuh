// Shared device helpers for libswiftdec_b200 (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "swiftdec_b200.h"

namespace sd {

// ---- error plumbing (thread-local message, no global mutable device state) ----
void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define SD_REQUIRE(cond, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      ::sd::set_error(__VA_ARGS__);    \
      return SD_EINVAL;                \
    }                                  \
  } while (0)

inline cudaStream_t as_stream(sd_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- element conversions ----
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// ---- warp / block reductions ----
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide reductions; `scratch` needs blockDim/32 entries; all threads get the result
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* scratch, Op op) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T r = scratch[0];
  for (int i = 1; i < nw; ++i) r = op(r, scratch[i]);  // fixed order: deterministic
  __syncthreads();
  return r;
}

// ---- programmatic dependent launch (PDL) ----
// Kernels on the decode chain are launched with programmatic stream
// serialization: each lets its successor launch early (pdl_trigger) and waits for
// its predecessor's results before touching them (pdl_wait). Every such kernel
// calls pdl_wait before it finishes, so completion stays transitive.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// SD_NO_PDL=1 (profiling only): plain stream-ordered launches, so per-kernel
// durations are not inflated by early-launched kernels waiting on their inputs.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SD_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- splitmix64 counter RNG (rng.py:16-30) ----
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t counter) {
  return splitmix64(splitmix64(seed) ^ counter);
}
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t counter) {
  return (double)(mix64(seed, counter) >> 11) * (1.0 / 9007199254740992.0);
}

// ---- device tree record layout (int32 words) ----
// [0] T (rows = 1 + nodes)   [1] n_paths   [2] head_nodes   [3] depth
// row arrays (SD_TREE_MAX_ROWS each): tok, pos, parent(node index, -1 root-level), ndepth
// paths: nodes [SD_TREE_MAX_PATHS][SD_TREE_MAX_DEPTH], origin [P], origin_index [P]
// mask bits [SD_TREE_MAX_ROWS][SD_MASK_WORDS] (row r sees request row j)
namespace tree_off {
constexpr int T = 0, NPATHS = 1, HEADNODES = 2, DEPTH = 3, NGRAMS = 4;
constexpr int TOK = 16;
constexpr int POS = TOK + SD_TREE_MAX_ROWS;
constexpr int PARENT = POS + SD_TREE_MAX_ROWS;  // per node (row - 1)
constexpr int NDEPTH = PARENT + SD_TREE_MAX_ROWS;  // per node
constexpr int PNODES = NDEPTH + SD_TREE_MAX_ROWS;
constexpr int PORIGIN = PNODES + SD_TREE_MAX_PATHS * SD_TREE_MAX_DEPTH;
constexpr int POIDX = PORIGIN + SD_TREE_MAX_PATHS;
constexpr int MASK = POIDX + SD_TREE_MAX_PATHS;
constexpr int TOTAL = MASK + SD_TREE_MAX_ROWS * SD_MASK_WORDS;
}  // namespace tree_off

}  // namespace sd
