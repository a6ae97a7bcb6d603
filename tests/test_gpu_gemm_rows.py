"""sd_gemm_rows (few-row weight streaming on the warp-level tensor path, the
verification forward's QKV / O projections, model.py:283-285, 306-309) against
a plain PyTorch fp32 product of the same bf16 operands; the split-K slices sum
to the product. Tolerance: fp32 accumulation of bf16 products in a different
order, |err| <= 1e-3 * (1 + |ref|) at K <= 16384."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2502_18890_b200 import _lib
    _lib.load()
    return _lib


@pytest.mark.parametrize("T,live,K,N", [(101, 41, 4096, 6144), (101, 101, 4096, 4096), (41, 41, 4096, 6144),
                                        (2, 1, 256, 256), (112, 97, 1536, 2048), (101, 17, 16384, 4096),
                                        (60, 60, 5120, 7168)])
def test_gemm_rows_matches_fp32(lib, T, live, K, N):
    g = torch.Generator(device="cuda")
    g.manual_seed(T * 7 + K + N)
    x = (torch.randn((T, K), device="cuda", generator=g)).to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda", generator=g) * K ** -0.5).to(torch.bfloat16)
    rows = torch.tensor([live], dtype=torch.int32, device="cuda")
    S = lib.load().sd_gemm_rows_splits(K, N)
    y = torch.full((S, T, N), 7.0, dtype=torch.float32, device="cuda")
    lib.call("sd_gemm_rows", lib.ptr(x), T, K, lib.ptr(w), N, lib.ptr(rows), lib.ptr(y), lib.stream())
    torch.cuda.synchronize()
    ref = x.float() @ w.float()
    got = y.sum(0)
    err = (got[:live] - ref[:live]).abs()
    assert float((err / (1 + ref[:live].abs())).max()) <= 1e-3
    # rows past the live count are not written
    assert bool((y[:, live:] == 7.0).all())


def test_gemm_rows_without_row_hint_computes_every_row(lib):
    T, K, N = 37, 2048, 1024
    x = torch.randn((T, K), device="cuda").to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda") * K ** -0.5).to(torch.bfloat16)
    S = lib.load().sd_gemm_rows_splits(K, N)
    y = torch.empty((S, T, N), dtype=torch.float32, device="cuda")
    lib.call("sd_gemm_rows", lib.ptr(x), T, K, lib.ptr(w), N, None, lib.ptr(y), lib.stream())
    torch.cuda.synchronize()
    ref = x.float() @ w.float()
    assert float(((y.sum(0) - ref).abs() / (1 + ref.abs())).max()) <= 1e-3


def test_gemm_rows_rejects_bad_shapes(lib):
    x = torch.zeros((4, 100), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((100, 256), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros((8, 4, 256), dtype=torch.float32, device="cuda")
    with pytest.raises(lib.LibraryError):
        lib.call("sd_gemm_rows", lib.ptr(x), 4, 100, lib.ptr(w), 256, None, lib.ptr(y), lib.stream())


@pytest.mark.parametrize("live", [41, 101, 1])
def test_silu_rows_skips_padding(lib, live):
    """sd_silu_rows: silu of the live verify rows (engine path: the tree record's
    row count), padded rows untouched."""
    T, N = 101, 16384
    a = torch.randn((T, N), device="cuda")
    out = torch.full((T, N), 3.0, dtype=torch.bfloat16, device="cuda")
    rows = torch.tensor([live], dtype=torch.int32, device="cuda")
    lib.call("sd_silu_rows", lib.ptr(a), lib.ptr(out), lib.SD_BF16, T, N, lib.ptr(rows), lib.stream())
    torch.cuda.synchronize()
    want = torch.nn.functional.silu(a[:live]).to(torch.bfloat16).float()
    torch.testing.assert_close(out[:live].float(), want, rtol=1e-2, atol=1e-2)
    assert bool((out[live:] == 3.0).all())
