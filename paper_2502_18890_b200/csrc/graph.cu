// Step-graph post-processing: early launch across library kernels.
//
// Inside the captured decode step, every kernel of this library is launched
// with programmatic stream serialization and waits (griddepcontrol.wait) before
// it reads its predecessor's output. Between two of our kernels the captured
// edge is programmatic and fires when the predecessor calls
// griddepcontrol.launch_dependents (at its start). A cuBLAS projection never
// calls it, so the edge from a cuBLAS kernel to the RMSNorm / RoPE / SiLU
// launch after it only fires when the projection has finished: the dependent's
// launch latency and ramp sit in the step's critical path four times per
// verify layer. sd_graph_relax_library_edges moves those edges to the
// predecessor's launch-completion port: the dependent may be scheduled once
// every block of the projection has started (it co-resides in the shared
// memory the projection leaves free), runs its pre-wait prologue, and waits in
// griddepcontrol.wait for the projection's completion and memory flush — the
// same guarantee as before, minus the launch gap.
#include <cuda.h>

#include <cstring>
#include <vector>

#include "common.cuh"

namespace sd {
namespace gr {

typedef CUresult (*PFN_nodeParams)(CUgraphNode, CUDA_KERNEL_NODE_PARAMS*);
typedef CUresult (*PFN_funcName)(const char**, CUfunction);

template <typename F>
static F entry(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (F)f;
}

// mangled names of this library's kernels live in namespace sd
static bool ours(const char* name) { return name && strstr(name, "_ZN2sd") != nullptr; }

}  // namespace gr
}  // namespace sd

using namespace sd;

extern "C" {

int sd_graph_relax_library_edges(void* graph, int* relaxed_out) {
  SD_REQUIRE(graph, "sd_graph_relax_library_edges: graph");
  auto node_params = gr::entry<gr::PFN_nodeParams>("cuGraphKernelNodeGetParams");
  auto func_name = gr::entry<gr::PFN_funcName>("cuFuncGetName");
  SD_REQUIRE(node_params && func_name, "sd_graph_relax_library_edges: driver entry points unavailable");
  cudaGraph_t g = (cudaGraph_t)graph;
  size_t n = 0;
  if (cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &n) != cudaSuccess) return check_launch("graph edges");
  std::vector<cudaGraphNode_t> from(n), to(n);
  std::vector<cudaGraphEdgeData> data(n);
  if (n && cudaGraphGetEdges_v2(g, from.data(), to.data(), data.data(), &n) != cudaSuccess)
    return check_launch("graph edges");
  int relaxed = 0;
  static const bool verbose = getenv("SD_GRAPH_VERBOSE") != nullptr;  // tuning only
  int prog = 0, named = 0;
  for (size_t i = 0; i < n; ++i) {
    const cudaGraphEdgeData& e = data[i];
    if (verbose) {
      cudaGraphNodeType a, b;
      cudaGraphNodeGetType(from[i], &a);
      cudaGraphNodeGetType(to[i], &b);
      CUDA_KERNEL_NODE_PARAMS qa, qb;
      memset(&qa, 0, sizeof(qa));
      memset(&qb, 0, sizeof(qb));
      const char* na = "-";
      const char* nb = "-";
      if (a == cudaGraphNodeTypeKernel && node_params((CUgraphNode)from[i], &qa) == CUDA_SUCCESS && qa.func)
        func_name(&na, qa.func);
      if (b == cudaGraphNodeTypeKernel && node_params((CUgraphNode)to[i], &qb) == CUDA_SUCCESS && qb.func)
        func_name(&nb, qb.func);
      fprintf(stderr, "edge type %d port %d: %.60s -> %.60s\n", (int)e.type, (int)e.from_port, na, nb);
    }
    if (e.type != cudaGraphDependencyTypeProgrammatic || e.from_port != cudaGraphKernelNodePortProgrammatic) continue;
    ++prog;
    cudaGraphNodeType tf, tt;
    if (cudaGraphNodeGetType(from[i], &tf) != cudaSuccess || cudaGraphNodeGetType(to[i], &tt) != cudaSuccess) continue;
    if (tf != cudaGraphNodeTypeKernel || tt != cudaGraphNodeTypeKernel) continue;
    CUDA_KERNEL_NODE_PARAMS pf, pt;
    memset(&pf, 0, sizeof(pf));
    memset(&pt, 0, sizeof(pt));
    if (node_params((CUgraphNode)from[i], &pf) != CUDA_SUCCESS || node_params((CUgraphNode)to[i], &pt) != CUDA_SUCCESS)
      continue;
    const char* nf = nullptr;
    const char* nt = nullptr;
    if (!pf.func || !pt.func || func_name(&nf, pf.func) != CUDA_SUCCESS || func_name(&nt, pt.func) != CUDA_SUCCESS)
      continue;
    ++named;
    if (gr::ours(nf) || !gr::ours(nt)) continue;  // only library kernel -> our (waiting) kernel
    cudaGraphEdgeData ne = e;
    ne.from_port = cudaGraphKernelNodePortLaunchCompletion;
    if (cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &data[i], 1) != cudaSuccess ||
        cudaGraphAddDependencies_v2(g, &from[i], &to[i], &ne, 1) != cudaSuccess)
      return check_launch("graph edge rewrite");
    ++relaxed;
  }
  if (verbose) fprintf(stderr, "graph: %zu edges, %d programmatic, %d named, %d relaxed\n", n, prog, named, relaxed);
  if (relaxed_out) *relaxed_out = relaxed;
  return SD_OK;
}

}  // extern "C"
