// Probe: does a cuBLAS (nvjet) kernel honour a programmatic graph edge, i.e.
// execute griddepcontrol.wait before reading its operands? (tools/pdl_probe.py)
//   probe_late_write: triggers its dependents at once, spins, then writes x.
//   probe_prog_edges: turns every edge probe kernel -> other kernel into a
//   programmatic edge (fires at the probe's trigger).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

__global__ void probe_late_write_kernel(__nv_bfloat16* x, int n, float v, long long spin) {
  asm volatile("griddepcontrol.launch_dependents;");
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = __float2bfloat16(v);
}

typedef CUresult (*PFN_nodeParams)(CUgraphNode, CUDA_KERNEL_NODE_PARAMS*);
typedef CUresult (*PFN_funcName)(const char**, CUfunction);

extern "C" int probe_late_write(void* x, int n, float v, long long spin, void* stream) {
  probe_late_write_kernel<<<148, 256, 0, (cudaStream_t)stream>>>((__nv_bfloat16*)x, n, v, spin);
  return (int)cudaGetLastError();
}

extern "C" int probe_prog_edges(void* graph) {
  void* f1 = nullptr;
  void* f2 = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuGraphKernelNodeGetParams", &f1, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuFuncGetName", &f2, cudaEnableDefault, &q);
  auto node_params = (PFN_nodeParams)f1;
  auto func_name = (PFN_funcName)f2;
  cudaGraph_t g = (cudaGraph_t)graph;
  size_t n = 0;
  cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &n);
  std::vector<cudaGraphNode_t> from(n), to(n);
  std::vector<cudaGraphEdgeData> data(n);
  cudaGraphGetEdges_v2(g, from.data(), to.data(), data.data(), &n);
  int changed = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType a, b;
    cudaGraphNodeGetType(from[i], &a);
    cudaGraphNodeGetType(to[i], &b);
    if (a != cudaGraphNodeTypeKernel || b != cudaGraphNodeTypeKernel) continue;
    CUDA_KERNEL_NODE_PARAMS pa;
    memset(&pa, 0, sizeof(pa));
    const char* na = nullptr;
    if (node_params((CUgraphNode)from[i], &pa) != CUDA_SUCCESS || func_name(&na, pa.func) != CUDA_SUCCESS) continue;
    if (!na || !strstr(na, "probe_late_write")) continue;
    cudaGraphEdgeData ne;
    memset(&ne, 0, sizeof(ne));
    ne.type = cudaGraphDependencyTypeProgrammatic;
    ne.from_port = cudaGraphKernelNodePortProgrammatic;
    if (cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &data[i], 1) != cudaSuccess) return -1;
    if (cudaGraphAddDependencies_v2(g, &from[i], &to[i], &ne, 1) != cudaSuccess) return -2;
    ++changed;
  }
  return changed;
}
