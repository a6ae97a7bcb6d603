"""Does cuBLAS's GEMM kernel wait on a programmatic graph edge?

A probe kernel triggers its dependents at once, spins ~spin cycles, then writes
A = 1. torch.mm(A, W) is captured after it; the probe -> GEMM edge is made
programmatic. If the GEMM executes griddepcontrol.wait before reading A, the
product equals W's column sums every replay; if not, it reads A before the
probe's write (A is zeroed before each replay) and the product is ~0.
Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC
       -o tools/pdl_probe.so tools/pdl_probe.cu -lcuda
"""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "pdl_probe.so"))
lib.probe_late_write.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_longlong, ctypes.c_void_p]
lib.probe_prog_edges.argtypes = [ctypes.c_void_p]


def run(M, K, N, spin, prog):
    dev = torch.device("cuda:0")
    A = torch.zeros((M, K), dtype=torch.bfloat16, device=dev)
    W = torch.randn((K, N), dtype=torch.bfloat16, device=dev)
    ref = W.float().sum(0)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.mm(A, W, out_dtype=torch.float32)  # warm-up / kernel selection
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g, stream=s):
        lib.probe_late_write(A.data_ptr(), A.numel(), 1.0, spin, s.cuda_stream)
        out = torch.mm(A, W, out_dtype=torch.float32)
    changed = lib.probe_prog_edges(g.raw_cuda_graph()) if prog else 0
    g.instantiate()
    bad = 0
    for _ in range(20):
        A.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        err = (out - ref[None, :]).abs().max().item()
        bad += err > 1e-2 * (ref.abs().max().item() + 1)
    print(f"M={M} K={K} N={N} spin={spin} prog={prog} edges_changed={changed}: {bad}/20 replays wrong")
    return bad


if __name__ == "__main__":
    spin = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    for (K, N) in ((4096, 6144), (4096, 4096), (4096, 16384), (16384, 4096)):
        run(101, K, N, spin, False)
        run(101, K, N, spin, True)
