"""Forward + end-to-end parity of the device model/engine against the oracle.

Tolerances (north star): logits within 1e-4 relative in the fp32 build and
1e-2 relative in bf16; token sequences identical wherever the top-1 margin
exceeds that tolerance (we check exact equality on seeds where margins are
comfortable, and report the first divergence otherwise).
"""

import json
import os
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import engine as OE
from oracle import model as OM
from oracle import sampling as OS

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
J = json.load(open(os.path.join(HERE, "golden.json")))
A = np.load(os.path.join(HERE, "golden.npz"))


def rel_err(got, want):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want)) / max(1e-9, np.max(np.abs(want))))


def dev_model(cfgd, dtype):
    from paper_2502_18890_b200 import ModelConfig, TinyTransformer
    return TinyTransformer(ModelConfig(**cfgd), dtype=dtype)


@pytest.mark.parametrize("name", ["gqa", "mha", "g4"])
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 1e-2)])
def test_forward_prefill_and_tree_vs_oracle(name, dtype, tol):
    from paper_2502_18890_b200 import ForwardRequest
    meta = J["model"][name]
    m = dev_model(meta["cfg"], dtype)
    om = OM.TinyTransformer(OM.ModelConfig(**meta["cfg"]), params=m.parameters_host())
    pre = meta["prefix"]
    cache = m.new_cache(64)
    r = m.forward(ForwardRequest(tokens=pre, positions=list(range(len(pre))), cache=cache))
    ocache = om.new_cache()
    ob, oq = om.forward(pre, list(range(len(pre))), ocache)
    assert rel_err(r.bundles.cpu().numpy(), ob) < tol
    assert rel_err(r.queries.cpu().numpy(), oq) < tol
    par = meta["tree_parent"]
    rows, ctx = len(par), len(pre)
    from oracle.tree import closure
    mask = np.zeros((rows, ctx + rows), dtype=bool)
    mask[:, :ctx] = True
    mask[:, ctx:] = closure(par)
    r2 = m.forward(ForwardRequest(tokens=meta["tree_tokens"], positions=[ctx + d for d in meta["tree_depth"]],
                                  cache=cache, attention_mask=mask, heads_needed=1))
    ob2, oq2 = om.forward(meta["tree_tokens"], [ctx + d for d in meta["tree_depth"]], ocache, mask, heads_needed=1)
    assert rel_err(r2.bundles[:, 0].cpu().numpy(), ob2[:, 0]) < tol
    assert torch.all(torch.isinf(r2.bundles[:, 1:]))
    if dtype == torch.float32:
        # fp32 device weights are the fp64 reference weights rounded once: still within 1e-4 of the reference
        assert rel_err(r2.bundles[:, 0].cpu().numpy(), A[f"m_{name}_tree_b"]) < 1e-4


def test_forward_matches_reference_contract():
    """test_model.py:116-175 restated: batched == incremental, chain mask ==
    causal, append-only cache, heads_needed, queries shape, errors."""
    from paper_2502_18890_b200 import (ForwardRequest, MaskShapeMismatch, ModelConfig, PositionOverflow,
                                       TinyTransformer)
    cfg = ModelConfig(vocab_size=64, num_layers=2, hidden_dim=32, num_heads=4, num_kv_heads=4, gamma=2,
                      max_positions=4096, init_seed=9)
    m = TinyTransformer(cfg, dtype=torch.float32)
    toks = [5, 9, 2, 44, 17]
    c1 = m.new_cache(64)
    batch = m.forward(ForwardRequest(toks, list(range(5)), c1)).bundles
    c2 = m.new_cache(64)
    rows = [m.forward(ForwardRequest([t], [i], c2)).bundles[0] for i, t in enumerate(toks)]
    np.testing.assert_allclose(batch.cpu().numpy(), torch.stack(rows).cpu().numpy(), rtol=1e-5, atol=1e-5)
    # masked chain == causal
    c3, c4 = m.new_cache(64), m.new_cache(64)
    m.forward(ForwardRequest([3, 1, 4], [0, 1, 2], c3))
    m.forward(ForwardRequest([3, 1, 4], [0, 1, 2], c4))
    causal = m.forward(ForwardRequest([1, 5, 9], [3, 4, 5], c3)).bundles
    mask = np.zeros((3, 6), dtype=bool)
    mask[:, :3] = True
    for i in range(3):
        mask[i, 3:4 + i] = True
    masked = m.forward(ForwardRequest([1, 5, 9], [3, 4, 5], c4, attention_mask=mask)).bundles
    np.testing.assert_allclose(causal.cpu().numpy(), masked.cpu().numpy(), rtol=1e-6, atol=1e-6)
    # append-only
    before = c1.rotated_keys(0, 5).clone()
    m.forward(ForwardRequest([5, 6], [5, 6], c1))
    assert len(c1) == 7 and torch.equal(c1.rotated_keys(0, 5), before)
    lim = m.forward(ForwardRequest([1, 2], [0, 1], m.new_cache(8), heads_needed=1)).bundles
    full = m.forward(ForwardRequest([1, 2], [0, 1], m.new_cache(8))).bundles
    np.testing.assert_allclose(lim[:, 0].cpu().numpy(), full[:, 0].cpu().numpy(), rtol=1e-6)
    assert torch.all(torch.isinf(lim[:, 1:]))
    assert m.forward(ForwardRequest([1, 2, 3], [0, 1, 2], m.new_cache(8))).queries.shape == (3, 2, 4, 8)
    with pytest.raises(PositionOverflow):
        m.forward(ForwardRequest([1], [4096], m.new_cache(8)))
    with pytest.raises(MaskShapeMismatch):
        m.forward(ForwardRequest([1, 2], [0, 1], m.new_cache(8), attention_mask=np.ones((2, 5), dtype=bool)))


def oracle_session_cfg(run):
    mk, ek = run["model"], run["engine"]
    sp = ek["sampler"]
    smp = OS.SamplerConfig(temperature=sp.get("temperature", 1.0), theta=sp["theta"], window=sp["window"],
                           truncation=OS.Truncation(sp["kind"], sp["value"]), seed=sp["seed"])
    ecfg = OE.EngineConfig(target_length=ek["target_length"], sink_size=ek["sink_size"], budget=ek["budget"],
                           widths=tuple(ek["widths"]), k=ek["k"], sampler=smp, seed=ek["seed"],
                           bonus=ek.get("bonus", True))
    mcfg = dict(vocab_size=mk["vocab"], num_layers=2, hidden_dim=mk.get("hidden", 32), num_heads=mk.get("heads", 4),
                num_kv_heads=mk["kv"], gamma=3, init_seed=mk["seed"])
    return mcfg, ecfg


def device_cfg(ecfg):
    from paper_2502_18890_b200 import EngineConfig, SamplerConfig, TreeConfig, Truncation
    s = ecfg.sampler
    smp = SamplerConfig(temperature=s.temperature, theta=s.theta, window=s.window,
                        truncation=Truncation(s.truncation.kind, s.truncation.value), seed=s.seed)
    return EngineConfig(target_length=ecfg.target_length, sink_size=ecfg.sink_size, budget=ecfg.budget,
                        tree=TreeConfig(tuple(ecfg.widths)), k=ecfg.k, sampler=smp, seed=ecfg.seed, bonus=ecfg.bonus)


def rec_tuple(r):
    return [r.accepted, r.ngram_accepted, r.origin, r.matched, list(r.tokens), r.refreshed, r.draft_ctx,
            r.verify_ctx, r.verify_rows, r.path_index]


@pytest.mark.parametrize("idx", range(5))
def test_engine_fp32_equals_reference_golden(idx):
    """fp32 device session vs the reference's own run (golden): identical
    tokens and iteration records."""
    from paper_2502_18890_b200 import generate
    run = J["engine"][idx]
    mcfg, ecfg = oracle_session_cfg(run)
    m = dev_model(mcfg, torch.float32)
    out, _ = generate(m, run["prompt"], device_cfg(ecfg))
    assert out == run["emitted"]


@pytest.mark.parametrize("idx", [0, 3, 4])
def test_engine_records_and_partial_vs_oracle(idx):
    from paper_2502_18890_b200 import prefill
    run = J["engine"][idx]
    mcfg, ecfg = oracle_session_cfg(run)
    m = dev_model(mcfg, torch.float32)
    om = OM.TinyTransformer(OM.ModelConfig(**mcfg), params=m.parameters_host())
    s = prefill(m, run["prompt"], device_cfg(ecfg))
    o = OE.Session(om, run["prompt"], ecfg)
    while not s.done:
        r = s.step()
        ro = o.step()
        assert rec_tuple(r) == rec_tuple(ro), f"step {ro.step}"
        assert s.partial.positions == o.partial.positions
        assert s.partial.mark == o.partial.mark
        assert len(s.full) == len(o.full)
    assert s.emitted == o.emitted
    assert s.device_error() == 0
    # n-gram table and window end in the same state
    for f in set(s.emitted[:20]):
        assert s.ngrams.retrieve(f, 20) == o.ngrams.retrieve(f, 20)
    assert s.window.member_mask().tolist() == o.window.member_mask().tolist()


def _oracle_margin(om, prompt, emitted, i, smp):
    """Relative top-1 margin of the oracle's penalised logits before token i."""
    cache = om.new_cache()
    seq = list(prompt) + list(emitted[:i])
    b, _ = om.forward(seq, list(range(len(seq))), cache, heads_needed=1)
    win = OS.PenaltyWindow(smp.window, om.config.vocab_size)
    for t in emitted[:i]:
        win.push(t)
    s = OS.scale_logits(b[-1, 0], win.member_mask(), smp.temperature, smp.theta)
    top = np.sort(s)[-2:]
    return float((top[1] - top[0]) / max(1e-9, abs(top[1])))


@pytest.mark.parametrize("idx,seed", [(4, 0), (4, 1), (0, 2)])
def test_engine_bf16_greedy_vs_oracle_same_weights(idx, seed):
    """bf16 device session vs the oracle running the same bf16-rounded
    weights in fp64, greedy (min-p 1.0): the token sequences agree up to the
    first position whose oracle top-1 margin is below the bf16 tolerance."""
    from paper_2502_18890_b200 import generate
    run = J["engine"][idx]
    mcfg, ecfg = oracle_session_cfg(run)
    mcfg = dict(mcfg, init_seed=mcfg["init_seed"] + seed)
    ecfg = replace(ecfg, sampler=replace(ecfg.sampler, truncation=OS.Truncation.min_p(1.0)), target_length=120)
    m = dev_model(mcfg, torch.bfloat16)
    om = OM.TinyTransformer(OM.ModelConfig(**mcfg), params=m.parameters_host())
    out, _ = generate(m, run["prompt"], device_cfg(ecfg))
    want, _ = OE.generate(om, run["prompt"], ecfg)
    n = min(len(out), len(want))
    i = next((j for j in range(n) if out[j] != want[j]), n)
    if i < n:
        margin = _oracle_margin(om, run["prompt"], want, i, ecfg.sampler)
        assert margin < 2e-2, f"diverged at token {i} with oracle margin {margin:.3e}"


def test_generate_ar_lossless():
    from paper_2502_18890_b200 import generate, generate_ar
    run = J["engine"][0]
    mcfg, ecfg = oracle_session_cfg(run)
    m = dev_model(mcfg, torch.float32)
    out, _ = generate(m, run["prompt"], device_cfg(ecfg))
    ar = generate_ar(m, run["prompt"], replace(device_cfg(ecfg), target_length=len(out)))
    assert ar == run["ar"]
    assert out[:len(ar)] == ar


def test_session_mechanics():
    """test_engine.py:167-262 restated on device."""
    from paper_2502_18890_b200 import (ConfigError, EngineConfig, ModelConfig, PromptTooShort, SamplerConfig,
                                       SessionExhausted, TinyTransformer, TreeConfig, Truncation, prefill)
    m = TinyTransformer(ModelConfig(vocab_size=64, num_layers=2, hidden_dim=32, num_heads=4, num_kv_heads=2,
                                    gamma=3, init_seed=8), dtype=torch.float32)
    base = dict(target_length=40, sink_size=2, budget=12, tree=TreeConfig((1, 2, 2, 2)), k=4,
                sampler=SamplerConfig(seed=3, theta=1.0, window=0, truncation=Truncation.top_p(1.0)), seed=3)
    with pytest.raises(PromptTooShort):
        prefill(m, [1, 2], EngineConfig(**base))
    with pytest.raises(ConfigError):
        EngineConfig(**{**base, "budget": 5}).validate(3)
    s = prefill(m, list(range(10)), EngineConfig(**{**base, "budget": 8}))
    assert len(s.full) == 10 and len(s.partial) == 8 and s.partial.mark == 9
    cfg = EngineConfig(**{**base, "target_length": 80, "budget": 10, "sink_size": 3,
                          "sampler": SamplerConfig(seed=1, truncation=Truncation.top_p(0.9))})
    s = prefill(m, list(range(12)), cfg)
    sink0 = s.partial.pk[:, :, :3].clone()
    while not s.done:
        s.step()
        assert torch.equal(s.partial.pk[:, :, :3], sink0)
        assert all(p[:3] == [0, 1, 2] for p in s.partial.positions)
        assert len(s.partial) <= cfg.budget
    assert 80 <= len(s.emitted) <= 83
    assert sum(r.accepted for r in s.records) == len(s.emitted)
    with pytest.raises(SessionExhausted):
        s.step()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_graph_replay_equals_eager(dtype):
    """The CUDA-graph step (device-resident base / context, whole slot range in
    the draft) is the same computation as the eager step: identical tokens,
    records and partial caches, across refreshes and evictions."""
    from paper_2502_18890_b200 import Session
    run = J["engine"][4]
    mcfg, ecfg = oracle_session_cfg(run)
    cfg = replace(device_cfg(ecfg), target_length=160)
    m = dev_model(mcfg, dtype)
    a = Session(m, run["prompt"], cfg, graph=False)
    b = Session(m, run["prompt"], cfg, graph=True)
    while not a.done:
        ra, rb = a.step(), b.step()
        assert rec_tuple(ra) == rec_tuple(rb), f"step {ra.step}"
        assert a.partial.positions == b.partial.positions
    assert a.emitted == b.emitted
    assert b._graph is not None and b.device_error() == 0
    assert torch.equal(a.q_sum, b.q_sum)
    n = len(a.full)
    assert torch.equal(a.full.k_rot[:, :, :n], b.full.k_rot[:, :, :n])


def test_cli_generate_trace_report_roundtrip(tmp_path, capsys):
    """`generate` on the device engine writes the reference's trace / metrics
    formats; `report` reads them back (reference cli.py:192-345)."""
    import json as _json

    from paper_2502_18890_b200 import cli
    from paper_2502_18890_b200 import metrics as M
    cfgf = tmp_path / "m.cfg"
    cfgf.write_text("vocab_size = 512\nnum_layers = 2\nhidden_dim = 64\nnum_heads = 4\nnum_kv_heads = 2\n"
                    "max_positions = 4096\n")
    out, trace, met = tmp_path / "o.txt", tmp_path / "t.jsonl", tmp_path / "m.json"
    rc = cli.main(["generate", "--model", str(cfgf), "--random-prompt", "48", "--target", "40", "--budget", "32",
                   "--sink", "4", "--min-p", "0.5", "--dtype", "fp32", "--out", str(out), "--trace", str(trace),
                   "--metrics", str(met)])
    assert rc == 0
    toks = [int(t) for t in out.read_text().split()]
    recs = M.read_trace(trace)
    assert len(toks) >= 40 and [t for r in recs for t in r.tokens] == toks
    m = _json.loads(met.read_text())
    assert m["emitted"] == len(toks) and m["iterations"] == len(recs)
    capsys.readouterr()
    assert cli.main(["report", "--trace", str(trace), "--prefix-len", "48"]) == 0
    rep = _json.loads(capsys.readouterr().out)
    assert rep["alpha"] == m["alpha"] and rep["emitted"] == len(toks)


_CFG1 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg1_run.json")


@pytest.mark.skipif(not os.path.exists(_CFG1), reason="tests/golden/cfg1_run.json not generated")
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
def test_cfg1_full_run_vs_reference(dtype):
    """BASELINE cfg1 end to end against the reference's own 2000-token run
    (tests/golden/make_golden_cfg1.py; SURVEY §8(c) layering (3)): fp32 —
    identical tokens and every IterationRecord; bf16 — the greedy tokens equal
    the oracle's wherever its top-1 margin exceeds 2e-2 (teacher forced on the
    device's own prefix, oracle/checks.py)."""
    import json as _json

    from oracle import checks as OC
    from oracle import model as OM
    from oracle import sampling as OS
    from paper_2502_18890_b200 import (EngineConfig, ModelConfig, SamplerConfig, TinyTransformer, TreeConfig,
                                       Truncation, prefill)
    from paper_2502_18890_b200.rng import random_prompt
    g = _json.load(open(_CFG1))
    mcfg = g["model"]
    prompt = random_prompt(g["prompt_len"], mcfg["vocab_size"])
    m = TinyTransformer(ModelConfig(**mcfg), dtype=dtype)
    cfg = EngineConfig(target_length=g["engine"]["target_length"], sink_size=g["engine"]["sink_size"],
                       budget=g["engine"]["budget"], tree=TreeConfig((1, 3, 3, 3)), k=g["engine"]["k"],
                       sampler=SamplerConfig(theta=1.2, window=1024, truncation=Truncation.min_p(1.0)))
    s = prefill(m, prompt, cfg)
    while not s.done:
        s.step()
    assert s.device_error() == 0
    if dtype == torch.float32:
        assert s.emitted == g["emitted"]
        got = [_json.loads(r.to_json()) for r in s.records]
        assert got == g["records"]
        assert g["lossless"] and g["ar"] == g["emitted"][:len(g["ar"])]
    else:
        om = OM.TinyTransformer(OM.ModelConfig(**mcfg), params=m.parameters_host())
        osmp = OS.SamplerConfig(theta=1.2, window=1024, truncation=OS.Truncation.min_p(1.0))
        bad, undecided = OC.greedy_mismatches(om, prompt, s.emitted, osmp, 2e-2)
        assert not bad, bad[:4]
