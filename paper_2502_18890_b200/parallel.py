"""KV-head sharding across GPUs of one node (one process per GPU, NCCL).

The reference has no parallelism. The decode step shards
naturally by KV head: rank r owns kv heads [r*Hk/P, (r+1)*Hk/P), their G query
heads, their slice of every cache (full and partial) and their slice of the
Eq. 2 scores. Two exchanges per step:

* after attention, every layer: all-gather of O [T, H/P*dh] -> [T, H*dh]
  (rank-major == global head order), then the replicated O projection / MLP /
  LM head;
* at a partial-cache refresh: all-gather of per-kv-head score partials,
  summed in ascending global head order (sd_sum_head_scores) so every rank
  selects the identical top-K, bitwise equal to the single-GPU sum.

Sampling, tree, n-gram and acceptance run replicated; they are deterministic
functions of identical inputs, so ranks stay in lock step without further
communication.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import _lib as L


def init_from_env(backend: str = "nccl"):
    """(rank, world, local_rank) from torchrun's environment; initialises the
    default process group when world > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return rank, world, local


def gather_rank_major(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather x from every rank -> [world, *x.shape] in rank order (NCCL
    over NVLink on the product path; gloo in the CPU tests)."""
    if x.is_cuda and dist.get_backend(group) == "gloo":  # CPU-side collectives (single-GPU multi-rank checks)
        return gather_rank_major(x.cpu(), world, group).to(x.device)
    flat = torch.empty((world * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(flat, x.contiguous(), group=group)
    return flat.view((world,) + tuple(x.shape))


def shard_heads(num_heads: int, num_kv_heads: int, head_dim: int, rank: int, world: int):
    """Column ranges of this rank's query and kv heads in Wq / Wk / Wv
    (rank r owns kv heads [r*Hk/P, (r+1)*Hk/P) and their G query heads)."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} kv heads cannot be sharded over {world} ranks")
    hk = num_kv_heads // world
    h = hk * (num_heads // num_kv_heads)
    return (rank * h * head_dim, (rank + 1) * h * head_dim), (rank * hk * head_dim, (rank + 1) * hk * head_dim)


def all_gather_heads(o: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[T, H_local*dh] per rank -> [T, H*dh] with heads in global order."""
    g = gather_rank_major(o, world, group)        # [P, T, Hl*dh]
    return g.permute(1, 0, 2).reshape(o.shape[0], world * o.shape[1])


def gather_head_partials(per_head: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[L, Hk_local, n] per rank -> [L, Hk, n] with kv heads in global order."""
    g = gather_rank_major(per_head, world, group)  # [P, L, Hkl, n]
    P, Ln, Hkl, n = g.shape
    return g.permute(1, 0, 2, 3).reshape(Ln, P * Hkl, n)


class ShardDivergence(RuntimeError):
    """Ranks of a sharded session disagree on a step result."""


def check_lockstep(result: torch.Tensor, world: int, group=None, step: int = -1) -> None:
    """Guard for the replicated sampling / tree / acceptance: all-gather this
    rank's step result (accepted count, tokens, path; a few dozen ints) and
    raise ShardDivergence unless every rank holds rank 0's copy. The replicated
    stages are deterministic functions of identical inputs, so a mismatch means
    a rank's inputs differed (a collective or kernel fault), and stepping on
    would silently desynchronise the caches."""
    if world <= 1:
        return
    g = gather_rank_major(result.reshape(-1), world, group).cpu()
    bad = [r for r in range(1, world) if not torch.equal(g[r], g[0])]
    if bad:
        raise ShardDivergence(f"step {step}: ranks {bad} disagree with rank 0 on the step result "
                              f"({g[bad[0]].tolist()[:8]} vs {g[0].tolist()[:8]})")


def sharded_scores(full, q_sum: torch.Tensor, model, start: int, end: int) -> torch.Tensor:
    """Eq. 2 scores over rows [start, end) for all layers, identical on every rank."""
    n = end - start
    per_head = torch.empty((full.num_layers, full.num_kv_heads, n), dtype=torch.float32, device=full.device)
    L.call("sd_importance_scores", L.ptr(q_sum), L.ptr(full.k_raw), L.dcode(full.dtype), full.layer_stride,
           full.head_stride, full.num_layers, model.H, full.num_kv_heads, full.head_dim, start, end, None,
           L.ptr(per_head), L.stream())
    allh = gather_head_partials(per_head, model.world, model.group).contiguous()
    scores = torch.empty((full.num_layers, n), dtype=torch.float32, device=full.device)
    L.call("sd_sum_head_scores", L.ptr(allh), full.num_layers, allh.shape[1], n, L.ptr(scores), L.stream())
    return scores
