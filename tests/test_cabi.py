"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
exactly the symbols include/swiftdec_b200.h declares (no compute calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "swiftdec_b200.h")
LIB = os.path.join(ROOT, "paper_2502_18890_b200", "libswiftdec_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sd_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2502_18890_b200.build_lib import build
        build()
    return ctypes.CDLL(LIB)


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "sd_attention" in syms and "sd_partial_refresh" in syms and "sd_sample_rows" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_table_matches_header():
    from paper_2502_18890_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_pure_host_queries(lib):
    # size queries touch no device
    lib.sd_attention_workspace_bytes.restype = ctypes.c_size_t
    assert lib.sd_attention_workspace_bytes(41, 32, 128, 54000) > 0
    lib.sd_ngram_bytes.restype = ctypes.c_size_t
    assert lib.sd_ngram_bytes(4, 1 << 16, 128256) > (1 << 16) * 16
    buf = (ctypes.c_int32 * 32)()
    assert lib.sd_tree_layout(buf, 32) == 18
    assert buf[14] == 256  # SD_TREE_MAX_ROWS


def test_product_has_no_cpu_fallback():
    """The product package must not import the oracle."""
    pkg = os.path.join(ROOT, "paper_2502_18890_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_missing_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2502_18890_b200 import ModelConfig, TinyTransformer, _lib
    with pytest.raises(_lib.LibraryError):
        TinyTransformer(ModelConfig(vocab_size=16, hidden_dim=8, num_heads=2, num_kv_heads=1))
