"""KV-head sharding host logic on CPU: world_size 2 over gloo (127.0.0.1).

The GPU path runs the same functions over NCCL (paper_2502_18890_b200/parallel.py).
Checked here with the numpy oracle doing each rank's per-head math:

* head sharding: rank r's column ranges of Wq / Wk / Wv select exactly its kv
  heads and their query heads (model.py:241 — query head j uses kv head j//G);
* attention-output all-gather: per-rank attention over its kv heads, gathered
  rank-major, equals the unsharded attention (global head order);
* refresh score exchange: per-kv-head Eq. 2 partials gathered from both ranks and
  summed in ascending global head order give the same top-K selection as the
  unsharded scores (kvcache.py:243-297).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kvcache as OK

WORLD = 2
H, HK, DH, T, CTX = 8, 4, 16, 5, 96


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _attend(q, K, V):
    """q [T, H, dh]; K, V [n, Hk, dh] -> [T, H, dh] (oracle softmax attention, GQA)."""
    t, h, dh = q.shape
    hk = K.shape[1]
    g = h // hk
    s = np.einsum("tkgd,nkd->tkgn", q.reshape(t, hk, g, dh), K) / np.sqrt(dh)
    w = np.exp(s - s.max(-1, keepdims=True))
    w /= w.sum(-1, keepdims=True)
    return np.einsum("tkgn,nkd->tkgd", w, V).reshape(t, h, dh)


def _data():
    g = np.random.default_rng(11)
    return (g.normal(size=(T, H, DH)), g.normal(size=(CTX, HK, DH)), g.normal(size=(CTX, HK, DH)),
            g.normal(size=(H, DH)))


def _worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2502_18890_b200.parallel import all_gather_heads, gather_head_partials, shard_heads
        q, K, V, qsum = _data()
        (q0, q1), (k0, k1) = shard_heads(H, HK, DH, rank, WORLD)
        hl, hkl = (q1 - q0) // DH, (k1 - k0) // DH
        # this rank's heads: query columns [q0, q1) and kv columns [k0, k1)
        ql = q.reshape(T, H * DH)[:, q0:q1].reshape(T, hl, DH)
        Kl = K.reshape(CTX, HK * DH)[:, k0:k1].reshape(CTX, hkl, DH)
        Vl = V.reshape(CTX, HK * DH)[:, k0:k1].reshape(CTX, hkl, DH)
        o_local = torch.as_tensor(_attend(ql, Kl, Vl).reshape(T, hl * DH))
        o_all = all_gather_heads(o_local, WORLD).numpy()
        # per-kv-head Eq. 2 partials over this rank's heads, [L=1, Hk_local, n]
        G = H // HK
        kh = [k0 // DH + i for i in range(hkl)]
        per_head = np.stack([OK.importance_scores(qsum[h * G:(h + 1) * G], K[:, h:h + 1], G) for h in kh])
        allh = gather_head_partials(torch.as_tensor(per_head[None]), WORLD).numpy()
        out_q.put((rank, o_all, allh))
    except Exception as e:  # surface worker failures to the test process
        out_q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gathered():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        r, o, s = q.get(timeout=120)
        assert s is not None, f"rank {r} failed: {o}"
        res[r] = (o, s)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_shard_heads_partition():
    from paper_2502_18890_b200.parallel import shard_heads
    for world in (1, 2, 4):
        qs, ks = [], []
        for r in range(world):
            (q0, q1), (k0, k1) = shard_heads(32, 8, 128, r, world)
            qs.append((q0, q1))
            ks.append((k0, k1))
            # the rank's query heads are exactly the G heads of each of its kv heads
            assert (q1 - q0) == 4 * (k1 - k0) and q0 == 4 * k0
        assert qs[0][0] == 0 and qs[-1][1] == 32 * 128 and all(a[1] == b[0] for a, b in zip(qs, qs[1:]))
        assert ks[0][0] == 0 and ks[-1][1] == 8 * 128 and all(a[1] == b[0] for a, b in zip(ks, ks[1:]))
    with pytest.raises(ValueError):
        shard_heads(32, 8, 128, 0, 3)


def test_attention_all_gather_equals_unsharded(gathered):
    q, K, V, _ = _data()
    want = _attend(q, K, V).reshape(T, H * DH)
    for r in range(WORLD):
        np.testing.assert_array_equal(gathered[r][0], gathered[0][0])  # every rank holds the same O
        np.testing.assert_allclose(gathered[r][0], want, rtol=1e-12, atol=1e-12)


def test_score_exchange_selects_the_unsharded_top_k(gathered):
    q, K, V, qsum = _data()
    want = OK.importance_scores(qsum, K, H // HK)
    for r in range(WORLD):
        allh = gathered[r][1][0]  # [Hk, n] in global kv-head order
        assert allh.shape == (HK, CTX)
        summed = np.zeros(CTX)
        for k in range(HK):  # ascending global head order (sd_sum_head_scores)
            summed = summed + allh[k]
        np.testing.assert_allclose(summed, want, rtol=1e-12, atol=1e-12)
        sink, take = 4, 40
        assert OK.select_body(summed[sink:], sink, CTX, take) == OK.select_body(want[sink:], sink, CTX, take)


def _lockstep_worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2502_18890_b200.parallel import ShardDivergence, check_lockstep
        same = torch.arange(32, dtype=torch.int32)
        check_lockstep(same, WORLD, step=0)  # identical results: no error
        diverged = same.clone()
        diverged[3] += rank  # rank 1's accepted tokens differ
        try:
            check_lockstep(diverged, WORLD, step=1)
            out_q.put((rank, "no error"))
        except ShardDivergence as e:
            out_q.put((rank, str(e)))
    except Exception as e:  # surface worker failures to the test process
        out_q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_lockstep_guard_detects_divergent_ranks():
    """the replicated sampler / tree / acceptance are checked
    every sharded step; a rank whose step result differs from rank 0's raises
    ShardDivergence on every rank (each sees the gathered results)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lockstep_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(WORLD):
        assert res[r].startswith("step 1: ranks [1] disagree"), res[r]
