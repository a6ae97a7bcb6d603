"""ctypes binding of libswiftdec_b200.so (the C ABI in include/swiftdec_b200.h).

There is no fallback: if the library is missing or no CUDA device is present
the product path raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SD_LIB_OVERRIDE") or os.path.join(HERE, "libswiftdec_b200.so")  # override: tools/ experiments only

SD_F32, SD_BF16, SD_F64 = 0, 1, 2
TREE_MAX_ROWS, TREE_MAX_PATHS, TREE_MAX_DEPTH, MASK_WORDS = 256, 512, 8, 8
MEMBER_NONE, MEMBER_MASK, MEMBER_WINDOW, MEMBER_TREE = 0, 1, 2, 3
TRUNC_NONE, TRUNC_TOP_P, TRUNC_MIN_P, TRUNC_ETA = 0, 1, 2, 3
IN_LOGITS_F32, IN_LOGITS_F64, IN_PROBS_F64, IN_SCALED_F32 = 0, 1, 2, 3
GEMM_EPI_F32, GEMM_EPI_SILU_BF16 = 0, 1
ST_RING_HEAD, ST_RING_LEN, ST_HIST_LEN, ST_PENDING, ST_ERROR, ST_BASE = 0, 1, 2, 3, 4, 5
RES_ACCEPTED, RES_BEST, RES_PICK, RES_ORIGIN, RES_ROWS, RES_PATHS, RES_PENDING, RES_BASE = 0, 1, 2, 3, 4, 5, 6, 7
RES_YS, RES_KEEP = 8, 16
PM_COUNT, PM_HI, PM_HEAD, PM_LEN, PM_NFREE, PM_ERR, PM_WORDS = 0, 1, 2, 3, 4, 5, 8

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
INT = C.c_int
F32 = C.c_float
F64 = C.c_double
SZ = C.c_size_t
U64 = C.c_uint64


class SampleArgs(C.Structure):
    _fields_ = [
        ("rows", INT), ("V", INT), ("in_kind", INT),
        ("temperature", F64), ("theta", F64),
        ("ctrl_style", INT), ("member_kind", INT),
        ("member_mask", P), ("win_count", P), ("win_ring", P), ("state", P),
        ("window", INT), ("tree", P), ("depth", INT), ("trunc_kind", INT),
        ("trunc_value", F64), ("eta_alpha", F64), ("seed", U64),
        ("positions", P), ("n", I64),
        ("probs_out", P), ("trunc_out", P), ("token_out", P),
        ("stats", P), ("stats_tiles", INT),
    ]


_SIGS = {
    "sd_version": (INT, []),
    "sd_graph_relax_library_edges": (INT, [P, C.POINTER(INT)]),
    "sd_last_error": (C.c_char_p, []),
    "sd_embed": (INT, [P, INT, P, INT, INT, P, P]),
    "sd_add_rmsnorm": (INT, [P, P, INT, INT, P, F32, P, INT, INT, I64, P]),
    "sd_silu": (INT, [P, P, INT, SZ, P]),
    "sd_silu_rows": (INT, [P, P, INT, INT, INT, P, P]),
    "sd_add_cast": (INT, [P, P, P, P, INT, SZ, P]),
    "sd_rope_stage": (INT, [P, INT, INT, INT, INT, P, P, P, F32, P, INT, P, P, P, P, INT, I64, I64, P, INT, I64, P]),
    "sd_attention_workspace_bytes": (SZ, [INT, INT, INT, INT]),
    "sd_attention": (INT, [P, INT, INT, INT, INT, INT, INT, P, P, INT, I64, INT, P, P, P, P, P, I64, P, INT, P, P,
                           P, P, INT, INT, P, INT, P, SZ, P]),
    "sd_make_kv_tmap": (INT, [P, INT, INT, INT, INT, P]),
    "sd_make_slot_tmap": (INT, [P, INT, INT, INT, INT, P]),
    "sd_gemv_workspace_bytes": (SZ, [INT, INT]),
    "sd_gemv": (INT, [P, INT, P, INT, INT, P, P, SZ, P]),
    "sd_gemm_rows_splits": (INT, [INT, INT]),
    "sd_gemm_rows": (INT, [P, INT, INT, P, INT, P, P, P]),
    "sd_gemv_addnorm": (INT, [P, INT, P, INT, P, P, F32, P, INT, P, SZ, P]),
    "sd_gemv_norm": (INT, [P, P, P, F32, P, INT, P, INT, INT, P, P, SZ, P]),
    "sd_gemv_rope": (INT, [P, P, P, P, F32, P, INT, P, INT, P, P, P, F32, INT, INT, INT, P, P, P, P, SZ, P]),
    "sd_tile_weight": (INT, [P, INT, INT, P, P]),
    "sd_make_weight_tmap": (INT, [P, INT, INT, P]),
    "sd_gemm_splits": (INT, [INT, INT, INT, INT]),
    "sd_gemm_workspace_bytes": (SZ, [INT, INT, INT]),
    "sd_gemm": (INT, [P, INT, INT, P, INT, INT, P, I64, P, SZ, P]),
    "sd_debug_tc_trace": (INT, [P, INT]),
    "sd_importance_scores": (INT, [P, P, INT, I64, I64, INT, INT, INT, INT, INT, INT, P, P, P]),
    "sd_sum_head_scores": (INT, [P, INT, INT, INT, P, P]),
    "sd_refresh_workspace_bytes": (SZ, [INT, INT, INT]),
    "sd_partial_refresh": (INT, [P, P, INT, INT, INT, INT, INT, INT, INT, P, P, INT, I64, I64, P, P, I64, I64, INT,
                                 P, P, P, P, P, P, P, SZ, P]),
    "sd_partial_mirror": (INT, [INT, INT, INT, INT, INT, P, P, INT, I64, I64, P, P, I64, I64, INT, P, P, P, P, P, P,
                                P]),
    "sd_partial_step": (INT, [INT, P, INT, INT, INT, INT, INT, INT, INT, INT, P, P, INT, I64, I64, P, P, I64, I64,
                              INT, P, P, P, P, P, P, P]),
    "sd_reconcile": (INT, [INT, P, INT, P, P, P, INT, I64, I64, INT, INT, P, INT, INT, P, P]),
    "sd_sample_rows": (INT, [P, C.POINTER(SampleArgs), P]),
    "sd_lmhead_tiled_bytes": (SZ, [INT, INT]),
    "sd_tile_lmhead": (INT, [P, INT, INT, P, P]),
    "sd_make_lmhead_tmap": (INT, [P, INT, INT, P]),
    "sd_lmhead_tiles": (INT, [INT]),
    "sd_lmhead_sample_stats": (INT, [P, INT, INT, P, INT, C.POINTER(SampleArgs), P, P, P]),
    "sd_draft_topw": (INT, [P, INT, INT, P, F64, F64, INT, P, P, P]),
    "sd_ngram_bytes": (SZ, [INT, INT, INT]),
    "sd_ngram_init": (INT, [P, INT, INT, INT, P]),
    "sd_ngram_update": (INT, [P, P, INT, INT, P]),
    "sd_ngram_retrieve": (INT, [P, P, INT, P, P, P]),
    "sd_ngram_frequency": (INT, [P, P, INT, P, P]),
    "sd_ngram_size": (INT, [P, P, P]),
    "sd_tree_layout": (INT, [P, INT]),
    "sd_tree_build": (INT, [P, P, INT, P, P, INT, P, I64, P, P]),
    "sd_draft_tree": (INT, [P, INT, P, P, INT, P, I64, P, P, P]),
    "sd_accept_commit": (INT, [P, P, U64, I64, INT, INT, P, P, P, INT, P, P, P, P]),
    "sd_window_push": (INT, [P, INT, P, P, P, INT, P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class LibraryError(RuntimeError):
    pass


def load(require_cuda: bool = True):
    """Load the library (once). Raises when it is missing — there is no CPU path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryError(
            f"{LIB_PATH} not built; run `python -m paper_2502_18890_b200.build_lib` (nvcc, sm_100a)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require_cuda():
    if not torch.cuda.is_available():
        raise LibraryError("paper_2502_18890_b200 needs a CUDA device (sm_100a); no CPU fallback exists")


# kernels launched per successful entry-point call (for the bench's gpu_launches)
_LAUNCHES = {"sd_attention": 2, "sd_reconcile": 2}  # attention: split kernel + merge (see _launches)


def _launches(name: str, args) -> int:
    """Kernels one successful call launches (the bench's gpu_launches claim):
    the tensor-core draft attention (src_kind 1 with slot descriptors) merges
    its splits in the same kernel."""
    if name == "sd_attention" and args[6] == 1 and args[22] is not None:
        return 1
    return _LAUNCHES.get(name, 1)
_NO_LAUNCH = {"sd_version", "sd_graph_relax_library_edges", "sd_last_error", "sd_attention_workspace_bytes", "sd_refresh_workspace_bytes",
              "sd_ngram_bytes", "sd_tree_layout", "sd_make_kv_tmap", "sd_make_slot_tmap", "sd_debug_tc_trace", "sd_make_weight_tmap",
              "sd_gemm_splits", "sd_gemm_workspace_bytes", "sd_gemv_workspace_bytes", "sd_make_lmhead_tmap",
              "sd_lmhead_tiles", "sd_lmhead_tiled_bytes", "sd_gemm_rows_splits"}
launch_count = 0


# PROFILING ONLY: SD_DEBUG_SKIP="sd_attention:0,sd_add_rmsnorm,mm,..." drops those
# launches (results become garbage) to measure each kernel's marginal cost in the
# real overlapped step; ":k" matches an sd_attention src_kind (0 verify, 1 draft),
# the row count of sd_rope_stage / sd_add_rmsnorm (1: draft, 101: verify).
DEBUG_SKIP = frozenset(x for x in os.environ.get("SD_DEBUG_SKIP", "").split(",") if x)


def call(name: str, *args):
    global launch_count
    if DEBUG_SKIP and (name in DEBUG_SKIP or (name == "sd_attention" and f"{name}:{args[6]}" in DEBUG_SKIP)
                       or (name == "sd_gemv" and f"{name}:{args[3]}" in DEBUG_SKIP)
                       or (name == "sd_rope_stage" and f"{name}:{args[1]}" in DEBUG_SKIP)
                       or (name == "sd_add_rmsnorm" and f"{name}:{args[2]}" in DEBUG_SKIP)):
        return 0
    if name not in _NO_LAUNCH:
        launch_count += _launches(name, args)
    rc = getattr(load(), name)(*args)
    if rc != 0:
        msg = load().sd_last_error().decode(errors="replace")
        raise LibraryError(f"{name} failed (code {rc}): {msg}")
    return rc


def ptr(t) -> int | None:
    """Device pointer of a tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def dcode(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return SD_BF16
    if dtype == torch.float32:
        return SD_F32
    if dtype == torch.float64:
        return SD_F64
    raise ValueError(f"unsupported dtype {dtype}")


def host_i32(values):
    arr = (I32 * max(1, len(values)))(*[int(v) for v in values])
    return arr


_TREE_LAYOUT = None


def tree_layout() -> dict:
    global _TREE_LAYOUT
    if _TREE_LAYOUT is None:
        buf = (I32 * 32)()
        n = load().sd_tree_layout(buf, 32)
        names = ["T", "NPATHS", "HEADNODES", "DEPTH", "NGRAMS", "TOK", "POS", "PARENT", "NDEPTH", "PNODES",
                 "PORIGIN", "POIDX", "MASK", "TOTAL", "MAX_ROWS", "MAX_PATHS", "MAX_DEPTH", "MASK_WORDS"]
        _TREE_LAYOUT = {k: int(buf[i]) for i, k in enumerate(names[:n])}
    return _TREE_LAYOUT
