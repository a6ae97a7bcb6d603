"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference.

The fixtures come from tests/golden/make_golden.py, which ran the reference
implementation (swiftdec) in the build container. CPU-only.
"""

import json
import os

import numpy as np
import pytest

from oracle import engine as OE
from oracle import kvcache as OK
from oracle import model as OM
from oracle import ngram as ON
from oracle import rng as OR
from oracle import sampling as OS
from oracle import tree as OT

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
J = json.load(open(os.path.join(HERE, "golden.json")))
A = np.load(os.path.join(HERE, "golden.npz"))


def test_rng_golden():
    for s, c, want in J["mix"]:
        assert OR.mix(s, c) == want
    for s, c, want in J["uniform_at"]:
        assert OR.uniform_at(s, c) == want
    for s, t, want in J["derive_seed"]:
        assert OR.derive_seed(s, t) == want
    assert OR.random_prompt(32, 128256) == J["prompt_128256"]
    # survey-quoted constants
    assert OR.mix(0, 0) == 0xA706DD2F4D197E6F
    assert OR.derive_seed(0, "branch-select") == 0xC1A92C4D55330423


@pytest.mark.parametrize("trial", range(24))
def test_sampling_golden(trial):
    case = J["sampling"][trial]
    logits = A[f"samp{trial}_logits"]
    members = A[f"samp{trial}_members"]
    cfg = OS.SamplerConfig(temperature=case["t"], theta=case["theta"], window=64, ctrl_style=case["ctrl"])
    probs = OS.penalized_probs_masked(logits, members, cfg)
    np.testing.assert_allclose(probs, A[f"samp{trial}_probs"], rtol=1e-12, atol=1e-300)
    rules = [OS.Truncation.min_p(0.1), OS.Truncation.top_p(0.9), OS.Truncation.eta(0.02),
             OS.Truncation.top_p(0.5), OS.Truncation.min_p(0.5)]
    for ri, rule in enumerate(rules):
        d = OS.truncate(A[f"samp{trial}_probs"], rule)
        np.testing.assert_allclose(d, A[f"samp{trial}_trunc{ri}"], rtol=1e-12, atol=1e-300)
        got = [OS.sample_at(A[f"samp{trial}_trunc{ri}"], pos, seed)
               for pos, seed in [(0, 0), (5, 1), (777, 3), (4096, 0)]]
        assert got == case["draws"][str(ri)]


def test_shrunk_masks_golden():
    s = J["shrunk"]
    w = OS.PenaltyWindow(s["cap"], s["V"])
    for t in s["tokens"]:
        w.push(t)
    got = [np.nonzero(m)[0].tolist() for m in w.shrunk_masks(5)]
    assert got == s["masks"]


@pytest.mark.parametrize("trial", range(40))
def test_tree_golden(trial):
    c = J["trees"][trial]
    t = OT.build_tree(c["heads"], [tuple(g) for g in c["grams"]], c["widths"])
    assert t.tokens == c["tokens"]
    assert t.parent == c["parent"]
    assert t.depth == c["depth"]
    assert t.head_node_count == c["head_node_count"]
    assert [[list(p.tokens), list(p.nodes), p.origin, p.origin_index] for p in t.paths] == c["paths"]
    assert [np.nonzero(r)[0].tolist() for r in t.mask] == c["mask"]


@pytest.mark.parametrize("trial", range(6))
def test_ngram_golden(trial):
    c = J["ngram"][trial]
    tab = ON.NGramTable(n=c["n"], k_max=64)
    seq = []
    for chunk in c["ops"]:
        tab.update(chunk, seq[-(c["n"] - 1):] if c["n"] > 1 else [])
        seq.extend(chunk)
    assert len(tab) == c["size"]
    for f, want in c["retrieve"].items():
        assert [list(g) for g in tab.retrieve(int(f), 20)] == want
    for g, fr in c["freqs"]:
        assert tab.frequency(tuple(g)) == fr


def test_importance_and_select_golden():
    for gs in J["imp_groups"]:
        got = OK.importance_scores(A[f"imp_q{gs}"], A[f"imp_k{gs}"], gs)
        np.testing.assert_allclose(got, A[f"imp_s{gs}"], rtol=1e-12)
    for trial, c in enumerate(J["select"]):
        sc = A[f"sel{trial}_scores"]
        for layer in range(2):
            body = OK.select_body(sc[layer], c["sink"], c["n"], c["budget"] - c["sink"])
            assert list(range(c["sink"])) + body == c["positions"][layer]


@pytest.mark.parametrize("name", ["gqa", "mha", "g4"])
def test_model_forward_golden(name):
    meta = J["model"][name]
    cfg = OM.ModelConfig(**meta["cfg"])
    model = OM.TinyTransformer(cfg)
    cache = model.new_cache()
    pre = meta["prefix"]
    b, q = model.forward(pre, list(range(len(pre))), cache)
    np.testing.assert_allclose(b, A[f"m_{name}_prefill_b"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(q, A[f"m_{name}_prefill_q"], rtol=1e-10, atol=1e-12)
    par = meta["tree_parent"]
    rows = len(par)
    ctx = len(pre)
    mask = np.zeros((rows, ctx + rows), dtype=bool)
    mask[:, :ctx] = True
    mask[:, ctx:] = OT.closure(par)
    b2, q2 = model.forward(meta["tree_tokens"], [ctx + d for d in meta["tree_depth"]], cache, mask, heads_needed=1)
    np.testing.assert_allclose(b2[:, 0], A[f"m_{name}_tree_b"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(q2, A[f"m_{name}_tree_q"], rtol=1e-10, atol=1e-12)


def oracle_run(run):
    mk, ek = run["model"], run["engine"]
    cfg = OM.ModelConfig(vocab_size=mk["vocab"], num_layers=2, hidden_dim=mk.get("hidden", 32),
                         num_heads=mk.get("heads", 4), num_kv_heads=mk["kv"], gamma=3, init_seed=mk["seed"])
    sp = ek["sampler"]
    smp = OS.SamplerConfig(temperature=sp.get("temperature", 1.0), theta=sp["theta"], window=sp["window"],
                           truncation=OS.Truncation(sp["kind"], sp["value"]), seed=sp["seed"])
    ecfg = OE.EngineConfig(target_length=ek["target_length"], sink_size=ek["sink_size"], budget=ek["budget"],
                           widths=tuple(ek["widths"]), k=ek["k"], sampler=smp, seed=ek["seed"],
                           bonus=ek.get("bonus", True))
    return OM.TinyTransformer(cfg), ecfg


@pytest.mark.parametrize("idx", range(5))
def test_engine_golden(idx):
    run = J["engine"][idx]
    model, ecfg = oracle_run(run)
    out, sess = OE.generate(model, run["prompt"], ecfg)
    assert out == run["emitted"]
    got = [[r.accepted, r.ngram_accepted, r.origin, r.matched, r.tokens, r.refreshed,
            r.draft_ctx, r.verify_ctx, r.verify_rows, r.path_index] for r in sess.records]
    assert got == run["records"]
    assert sess.partial.positions == run["final_partial_positions"]
    assert sess.partial.mark == run["final_mark"]


def test_ar_golden():
    run = J["engine"][0]
    model, ecfg = oracle_run(run)
    from dataclasses import replace
    ar = OE.generate_ar(model, run["prompt"], replace(ecfg, target_length=len(run["ar"])))
    assert ar == run["ar"]


def test_teacher_forced_check_on_oracle_ar():
    """oracle/checks.py: the oracle's own AR output passes its teacher-forced
    check at every position (and a corrupted token is caught)."""
    from oracle import checks as OC
    from oracle import engine as OE
    from oracle import model as OM
    from oracle import sampling as OS
    mc = OM.ModelConfig(vocab_size=97, num_layers=2, hidden_dim=32, num_heads=4, num_kv_heads=2, gamma=3, init_seed=4)
    om = OM.TinyTransformer(mc)
    smp = OS.SamplerConfig(theta=1.2, window=16, truncation=OS.Truncation.min_p(1.0))
    cfg = OE.EngineConfig(target_length=40, sink_size=4, budget=16, sampler=smp)
    prompt = [int(x) for x in np.random.default_rng(0).integers(0, 97, size=12)]
    out = OE.generate_ar(om, prompt, cfg)
    res = OC.teacher_forced(om, prompt, out, smp)
    assert [w for _, w, _ in res] == out
    bad, _ = OC.greedy_mismatches(om, prompt, out, smp, 0.0)
    assert bad == []
    wrong = list(out)
    wrong[5] = (wrong[5] + 1) % 97
    bad, _ = OC.greedy_mismatches(om, prompt, wrong, smp, 0.0)
    assert bad and bad[0][0] == 5
