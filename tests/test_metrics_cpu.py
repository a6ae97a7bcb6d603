"""Run statistics, traces and the cost model (metrics.py) on known answers:
the definitions of swiftdec/metrics.py:29-213 (Eq. 5 alpha, Eq. 7 beta,
distinct-n, the roofline replay of a trace). Host-only: no GPU needed."""

import math

import pytest

from paper_2502_18890_b200 import metrics as M


def _recs():
    return [M.IterationRecord(step=0, accepted=4, ngram_accepted=4, origin="ngram", matched=3, tokens=[5, 6, 7, 8],
                              draft_ctx=100, verify_ctx=200, verify_rows=41),
            M.IterationRecord(step=1, accepted=1, ngram_accepted=0, origin="head", matched=0, tokens=[9],
                              draft_ctx=104, verify_ctx=204, verify_rows=41, refreshed=True),
            M.IterationRecord(step=2, accepted=2, ngram_accepted=0, origin="head", matched=1, tokens=[5, 6],
                              draft_ctx=105, verify_ctx=205, verify_rows=1)]


def test_rates_and_distinct():
    r = _recs()
    assert M.acceptance_rate(r, 3) == 7 / 12
    assert M.ngram_acceptance_rate(r, 3) == 4 / 12
    toks = [t for x in r for t in x.tokens]  # 5 6 7 8 9 5 6
    assert M.distinct_n(toks, 1) == 5 / 7
    assert M.distinct_n(toks, 2) == 5 / 6  # (5,6) twice
    assert M.distinct_n(toks, 4) == 1.0
    with pytest.raises(M.SequenceTooShort):
        M.distinct_n([1, 2], 3)
    with pytest.raises(ValueError):
        M.acceptance_rate([], 3)
    m = M.collect_metrics(r, 3, toks, {"draft": 3}, {"draft": 0.5})
    assert m.iterations == 3 and m.emitted == 7 and m.accepted == [4, 1, 2] and m.ngram_accepted == [4, 0, 0]
    d = m.to_dict()
    assert d["distinct"]["2"] == 5 / 6 and d["forward_counts"] == {"draft": 3}


def test_trace_roundtrip(tmp_path):
    r = _recs()
    p = tmp_path / "t.jsonl"
    M.write_trace(r, p)
    assert M.read_trace(p) == r
    assert '"verify_rows": 41' in r[0].to_json()


def test_cost_model():
    p = M.CostParams(bandwidth=1e12, flops=1e14, weight_bytes=1e9, kv_bytes_per_token=1e3)
    assert M.forward_time(p, 1000, 1) == (1e9 + 1e6) / 1e12
    # compute-bound at many rows: rows * row_ops / flops
    assert M.forward_time(p, 0, 1000) == 1000 * 1e9 / 1e14
    ar = M.ar_generation_cost(p, 10, 3)
    assert math.isclose(ar, sum((1e9 + 1e3 * (10 + i)) / 1e12 for i in range(3)))
    r = _recs()
    sw = M.swift_generation_cost(p, r)
    want = sum(M.forward_time(p, x.draft_ctx, 1) + M.forward_time(p, x.verify_ctx, max(x.verify_rows, 1)) for x in r)
    assert math.isclose(sw, want)
    s = M.simulated_speedup(p, r, 64)
    assert math.isclose(s, (M.ar_generation_cost(p, 64, 7) / 7) / (sw / 7))
    with pytest.raises(ValueError):
        M.CostParams(bandwidth=0)
    # B200 preset: the SURVEY §8d step bound at cfg3 ctx 54K (~4.96 ms)
    assert 4.8e-3 < M.step_bound_seconds(M.B200, 54096, 4096) < 5.1e-3


def test_cli_report_matches_metrics(tmp_path, capsys):
    """`report` (cli.py:324-345 of the reference): the reference's payload from a
    trace, the (Gen. Len., alpha, x) CSV row, exit code 2 on a missing trace."""
    import json as _json

    from paper_2502_18890_b200 import cli
    r = _recs()
    p = tmp_path / "t.jsonl"
    M.write_trace(r, p)
    csvp = tmp_path / "r.csv"
    assert cli.main(["report", "--trace", str(p), "--prefix-len", "64", "--csv", str(csvp)]) == 0
    out = _json.loads(capsys.readouterr().out)
    want = M.collect_metrics(r, 3, [t for x in r for t in x.tokens]).to_dict()
    for k, v in want.items():
        assert out[k] == v
    assert math.isclose(out["simulated_speedup"], M.simulated_speedup(M.CostParams(), r, 64))
    lines = csvp.read_text().splitlines()
    assert lines[0] == "Gen. Len.,alpha,x" and lines[1].startswith("7,0.5833,")
    assert cli.main(["report", "--trace", str(p), "--b200"]) == 0
    assert math.isclose(_json.loads(capsys.readouterr().out)["simulated_speedup"],
                        M.simulated_speedup(M.B200, r, 64))
    assert cli.main(["report", "--trace", str(tmp_path / "missing.jsonl")]) == 2


def test_cli_model_config_parsing(tmp_path):
    from paper_2502_18890_b200 import cli
    from paper_2502_18890_b200.engine import ConfigError
    f = tmp_path / "m.cfg"
    f.write_text("# tiny\nvocab_size = 512\nnum_layers = 2\nhidden_dim = 256\nnum_heads = 8\nnum_kv_heads = 2\n")
    assert cli.read_model_config(str(f))["num_kv_heads"] == "2"
    f.write_text("vocab_size = 512\nbogus = 1\n")
    with pytest.raises(ConfigError):
        cli.read_model_config(str(f))
    f.write_text("backend = table\n")
    with pytest.raises(ConfigError):
        cli.read_model_config(str(f))
