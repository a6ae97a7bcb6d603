"""torch.ops.swiftdec_b200.* shim (the C ABI wrapped as PyTorch
operators): every §8(b) operator is registered with its schema, in-place
outputs are declared mutable, and only a CUDA kernel is registered (no CPU
fallback: calling with CPU tensors fails loudly)."""

import pytest
import torch

import paper_2502_18890_b200  # noqa: F401  (registers the operators)
from paper_2502_18890_b200 import ops

NAMES = ["verify_attention", "draft_attention", "stage_kv_rope", "score_select_gather", "partial_admit_evict",
         "reconcile_rows", "ngram_update", "ngram_retrieve", "draft_topw", "tree_build", "verify_sample", "accept"]


def test_every_boundary_operator_is_registered():
    assert sorted(ops.schemas()) == sorted(NAMES)
    for n in NAMES:
        op = getattr(torch.ops.swiftdec_b200, n).default
        assert op._schema.name == f"swiftdec_b200::{n}"
        assert any(a.alias_info is not None and a.alias_info.is_write for a in op._schema.arguments), n


def test_operators_have_no_cpu_kernel():
    t = torch.zeros(4, dtype=torch.int32)
    with pytest.raises(NotImplementedError):
        torch.ops.swiftdec_b200.ngram_update(t, t, 1, 1)
