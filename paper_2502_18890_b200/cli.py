"""Command-line entry points on the device engine (the reference's `swiftdec`
CLI surface for the decode path, cli.py:192-345):

    python -m paper_2502_18890_b200.cli generate --model m.cfg --random-prompt 512 --target 2000 \\
        [--trace t.jsonl] [--metrics m.json] [--out tokens.txt]
    python -m paper_2502_18890_b200.cli report --trace t.jsonl [--gamma 3] [--prefix-len 512] [--b200] [--csv r.csv]
    python -m paper_2502_18890_b200.cli bench --model m.cfg --gen-lens 256,1024 --ks 0,20 [--out grid.csv]

Model configs are the reference's flat `key = value` files (model.py:487-507:
vocab_size, num_layers, hidden_dim, num_heads, num_kv_heads, gamma,
max_positions, init_seed; backend `tiny` only). Traces are the reference's
JSONL, so `swiftdec report` reads ours and this `report` reads the
reference's. `report` prints the reference's payload (RunMetrics.to_dict() +
simulated_speedup) and can append its (Gen. Len., alpha, x) CSV row; `--b200`
swaps the reference's A100 cost defaults for the B200 preset. `bench` writes
the reference's grid CSV header. Exit codes: 0 ok, 2 configuration error,
3 runtime error (cli.py:396-401).
"""

from __future__ import annotations

import argparse
import csv
import itertools
import json
import statistics
import sys
from pathlib import Path

from . import metrics
from .engine import ConfigError, EngineConfig, Session
from .sampling import SamplerConfig, Truncation
from .tree import TreeConfig

_MODEL_KEYS = ("backend", "vocab_size", "num_layers", "hidden_dim", "num_heads", "num_kv_heads", "gamma",
               "max_positions", "init_seed")


def read_model_config(path: str) -> dict[str, str]:
    p = Path(path)
    if not p.exists():
        raise ConfigError(f"model config not found: {path}")
    out: dict[str, str] = {}
    for line in p.read_text(encoding="utf-8").splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, sep, val = line.partition("=")
        if not sep or key.strip() not in _MODEL_KEYS:
            raise ConfigError(f"{path}: bad line {line!r}")
        out[key.strip()] = val.strip()
    if out.get("backend", "tiny") != "tiny":
        raise ConfigError("only the tiny transformer backend runs on the device engine")
    return out


def build_model(values: dict[str, str], dtype: str = "bf16"):
    import torch

    from .model import ModelConfig, TinyTransformer
    g = lambda k, d: int(values.get(k, d))  # noqa: E731
    cfg = ModelConfig(vocab_size=g("vocab_size", 256), num_layers=g("num_layers", 2), hidden_dim=g("hidden_dim", 64),
                      num_heads=g("num_heads", 4), num_kv_heads=g("num_kv_heads", g("num_heads", 4)),
                      gamma=g("gamma", 3), max_positions=g("max_positions", 65536), init_seed=g("init_seed", 0))
    return TinyTransformer(cfg, dtype=torch.float32 if dtype == "fp32" else torch.bfloat16)


def _truncation(args) -> Truncation:
    if args.top_p is not None:
        return Truncation.top_p(args.top_p)
    if args.eta is not None:
        return Truncation.eta(args.eta)
    return Truncation.min_p(args.min_p if args.min_p is not None else 0.1)


def _engine_config(args, target: int, k: int, tree: str, theta: float, window: int, seed: int) -> EngineConfig:
    smp = SamplerConfig(temperature=args.temperature, theta=theta, window=window, truncation=_truncation(args),
                        seed=seed)
    return EngineConfig(target_length=target, sink_size=args.sink, budget=args.budget,
                        tree=TreeConfig(tuple(int(w) for w in tree.split(","))), k=k, sampler=smp, seed=seed,
                        bonus=not args.no_bonus)


def _prompt(args, vocab: int, seed: int) -> list[int]:
    from .rng import random_prompt
    if args.prompt is not None:
        return [int(t) for t in args.prompt.split()]
    if args.prompt_file is not None:
        p = Path(args.prompt_file)
        if not p.exists():
            raise ConfigError(f"prompt file not found: {p}")
        return [int(t) for t in p.read_text().split()]
    return random_prompt(args.random_prompt if args.random_prompt is not None else 64, vocab, seed)


def _run(model, prompt, ecfg) -> Session:
    s = Session(model, prompt, ecfg)
    while not s.done:
        s.step()
    return s


def _cost_params(args) -> metrics.CostParams:
    if getattr(args, "b200", False):
        return metrics.B200
    return metrics.CostParams(bandwidth=args.bandwidth, flops=args.flops, weight_bytes=args.weight_bytes,
                              kv_bytes_per_token=args.kv_bytes)


def cmd_generate(args) -> int:
    model = build_model(read_model_config(args.model), args.dtype)
    prompt = _prompt(args, model.config.vocab_size, args.seed)
    s = _run(model, prompt, _engine_config(args, args.target, args.k, args.tree, args.theta, args.window, args.seed))
    text = " ".join(str(t) for t in s.emitted)
    if args.out:
        Path(args.out).write_text(text + "\n", encoding="utf-8")
    else:
        print(text)
    if args.trace:
        metrics.write_trace(s.records, args.trace)
    if args.metrics:
        Path(args.metrics).write_text(json.dumps(s.metrics().to_dict(), indent=2) + "\n", encoding="utf-8")
    return 0


def cmd_report(args) -> int:
    path = Path(args.trace)
    if not path.exists():
        raise ConfigError(f"trace not found: {path}")
    records = metrics.read_trace(path)
    if not records:
        raise ConfigError(f"trace {path} is empty")
    emitted = [t for r in records for t in r.tokens]
    run = metrics.collect_metrics(records, args.gamma, emitted)
    sim = metrics.simulated_speedup(_cost_params(args), records, args.prefix_len)
    payload = run.to_dict()
    payload["simulated_speedup"] = sim
    print(json.dumps(payload, indent=2))
    if args.csv:
        new = not Path(args.csv).exists()
        with open(args.csv, "a", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            if new:
                w.writerow(["Gen. Len.", "alpha", "x"])
            w.writerow([run.emitted, f"{run.alpha:.4f}", f"{sim:.4f}"])
    return 0


def _fmt(values: list[float]) -> str:
    if len(values) == 1:
        return f"{values[0]:.4f}"
    return f"{statistics.fmean(values):.4f}±{statistics.pstdev(values):.4f}"


def cmd_bench(args) -> int:
    values = read_model_config(args.model)
    grid = list(itertools.product([int(x) for x in args.gen_lens.split(",")], [int(x) for x in args.ks.split(",")],
                                  args.trees.split(";"), [float(x) for x in args.thetas.split(",")],
                                  [int(x) for x in args.windows.split(",")]))
    seeds = [int(x) for x in args.seeds.split(",")]
    if not grid or not seeds:
        raise ConfigError("bench grid must not be empty")
    params = _cost_params(args)
    model = build_model(values, args.dtype)  # weights are immutable and shared by the sessions
    rows = []
    for gen_len, k, tree, theta, window in grid:
        st = {"alpha": [], "beta": [], "speedup": [], "distinct": []}
        for seed in seeds:
            prompt = _prompt(args, model.config.vocab_size, seed)
            s = _run(model, prompt, _engine_config(args, gen_len, k, tree, theta, window, seed))
            m = s.metrics()
            st["alpha"].append(m.alpha)
            st["beta"].append(m.beta)
            st["speedup"].append(metrics.simulated_speedup(params, s.records, len(prompt)))
            st["distinct"].append(statistics.fmean(m.distinct.values()))
        rows.append({"gen_len": gen_len, "k": k, "tree": tree, "theta": theta, "W": window,
                     "alpha": _fmt(st["alpha"]), "beta": _fmt(st["beta"]),
                     "simulated_speedup": _fmt(st["speedup"]), "distinct_avg": _fmt(st["distinct"])})
    header = ["gen_len", "k", "tree", "theta", "W", "alpha", "beta", "simulated_speedup", "distinct_avg"]
    fh = open(args.out, "w", newline="", encoding="utf-8") if args.out else sys.stdout
    try:
        w = csv.DictWriter(fh, fieldnames=header)
        w.writeheader()
        w.writerows(rows)
    finally:
        if args.out:
            fh.close()
    return 0


def _run_flags(p) -> None:
    p.add_argument("--model", required=True, help="model config file (key = value lines)")
    src = p.add_mutually_exclusive_group()
    src.add_argument("--prompt")
    src.add_argument("--prompt-file")
    src.add_argument("--random-prompt", type=int, metavar="N")
    p.add_argument("--sink", type=int, default=4)
    p.add_argument("--budget", type=int, default=64)
    p.add_argument("--temperature", type=float, default=1.0)
    trunc = p.add_mutually_exclusive_group()
    trunc.add_argument("--top-p", type=float)
    trunc.add_argument("--min-p", type=float)
    trunc.add_argument("--eta", type=float)
    p.add_argument("--no-bonus", action="store_true")
    p.add_argument("--dtype", choices=["bf16", "fp32"], default="bf16")


def _cost_flags(p) -> None:
    p.add_argument("--bandwidth", type=float, default=2.04e12, help="bytes/s")
    p.add_argument("--flops", type=float, default=312e12)
    p.add_argument("--weight-bytes", type=float, default=15.0e9)
    p.add_argument("--kv-bytes", type=float, default=131072.0, help="per token")
    p.add_argument("--b200", action="store_true", help="use the B200 preset (metrics.B200)")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2502_18890_b200", description="TokenSwift decode on B200")
    sub = ap.add_subparsers(dest="command", required=True)
    g = sub.add_parser("generate", help="run one decode on the GPU")
    _run_flags(g)
    g.add_argument("--target", type=int, default=256)
    g.add_argument("--k", type=int, default=20)
    g.add_argument("--tree", default="1,3,3,3")
    g.add_argument("--theta", type=float, default=1.2)
    g.add_argument("--window", type=int, default=1024)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--out")
    g.add_argument("--trace")
    g.add_argument("--metrics")
    g.set_defaults(func=cmd_generate)
    b = sub.add_parser("bench", help="sweep a config grid into CSV")
    _run_flags(b)
    _cost_flags(b)
    b.add_argument("--gen-lens", default="256")
    b.add_argument("--ks", default="20")
    b.add_argument("--thetas", default="1.2")
    b.add_argument("--windows", default="1024")
    b.add_argument("--trees", default="1,3,3,3", help="semicolon-separated width lists")
    b.add_argument("--seeds", default="0")
    b.add_argument("--out")
    b.set_defaults(func=cmd_bench)
    r = sub.add_parser("report", help="trace JSONL to metrics JSON")
    _cost_flags(r)
    r.add_argument("--trace", required=True)
    r.add_argument("--gamma", type=int, default=3)
    r.add_argument("--prefix-len", type=int, default=64)
    r.add_argument("--csv")
    r.set_defaults(func=cmd_report)
    return ap


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ConfigError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (RuntimeError, OSError) as exc:
        print(f"runtime error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
