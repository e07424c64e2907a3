"""``moeplace.cli`` — configuration-driven experiments.

Orchestration only: every hot operation it calls (trace synthesis, frequency estimation, hop
matrix, cost matrix, coefficients, evaluation, communication map) runs on the GPU engine.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

from .errors import ConfigError, InfeasibleError, MoeplaceError, exit_code
from .eval import communication_map, evaluate_many, gain, objective_value, report_from_sums, score_sums
from .model_trace import (ModelSpec, default_attention_placement, estimate_frequencies, generate_trace,
                          parse_trace, split_trace, trace_stats, write_trace)
from .placement import (Constraints, cost_matrix, place_greedy, place_round_robin, read_placement, validate,
                        write_placement)
from .solver import UniformFrequencies, build_instance, solve_exact, write_solve_report
from .topology import TopologySpec, all_pairs_hops, build_topology, locality_order

METHODS = ("rr", "greedy", "ilp", "ilpload")

# flat configuration keys (mirroring Table 5) and their defaults
DEFAULTS = {
    "model": "custom", "L": None, "E": None, "K": None,
    "c_exp": None, "c_layer": 1,
    "topology": "FatTree", "topologies": None,
    "num_leaf_switches": 16, "num_nodes_per_leaf": 4, "num_gpus_per_server": 4,
    "spines": 4, "groups": 4, "group_size": 4, "spines_per_group": 2,
    "trace_file": None, "zipf_s": 1.2, "n_tokens": 20000, "n_chunks": 150, "seed": 0,
    "train_chunks": 100, "test_chunks": 50,
    "methods": list(METHODS), "output_dir": "moeplace_out",
}


@dataclass
class ExperimentConfig:
    """SPEC.md:404-407.  A single flat JSON document; unknown keys are rejected."""

    values: dict = field(default_factory=dict)

    def __getattr__(self, k):
        v = self.__dict__.get("values", {})
        if k in v:
            return v[k]
        raise AttributeError(k)

    @classmethod
    def from_dict(cls, d: dict) -> "ExperimentConfig":
        unknown = sorted(set(d) - set(DEFAULTS))
        if unknown:
            raise ConfigError(f"unknown config key(s): {', '.join(unknown)}")
        v = dict(DEFAULTS)
        v.update(d)
        for k in ("L", "E", "K", "c_exp"):
            if v[k] is None:
                raise ConfigError(f"config key {k!r} is required")
        bad = [m for m in v["methods"] if m not in METHODS]
        if bad or not v["methods"]:
            raise ConfigError(f"methods must be a non-empty subset of {METHODS}, got {v['methods']}")
        cfg = cls(v)
        cfg.model_spec()
        cfg.constraints()
        for kind in cfg.kinds():
            cfg.topology_spec(kind)
        return cfg

    @staticmethod
    def read_json(path) -> dict:
        """The raw config document: a JSON object, else ConfigError (CLI exit 2)."""
        try:
            with open(path) as f:
                d = json.load(f)
        except (json.JSONDecodeError, UnicodeDecodeError) as e:
            raise ConfigError(f"{path}: invalid JSON ({e})") from None
        if not isinstance(d, dict):
            raise ConfigError(f"{path}: the config must be a JSON object")
        return d

    @classmethod
    def load(cls, path) -> "ExperimentConfig":
        return cls.from_dict(cls.read_json(path))

    def model_spec(self) -> ModelSpec:
        return ModelSpec(int(self.values["L"]), int(self.values["E"]), int(self.values["K"]))

    def constraints(self) -> Constraints:
        return Constraints(int(self.values["c_exp"]), int(self.values["c_layer"]))

    def kinds(self) -> list:
        t = self.values["topologies"]
        return list(t) if t else [self.values["topology"]]

    def topology_spec(self, kind: str) -> TopologySpec:
        v = self.values
        extra = {"FatTree": {"spines": v["spines"]}, "FatTreeHier": {"groups": v["groups"]},
                 "Dragonfly": {"group_size": v["group_size"]},
                 "DragonflyPlus": {"group_size": v["group_size"], "spines_per_group": v["spines_per_group"]}}.get(kind, {})
        return TopologySpec(kind, int(v["num_leaf_switches"]), int(v["num_nodes_per_leaf"]),
                            int(v["num_gpus_per_server"]), extra)

    def with_(self, **kw) -> "ExperimentConfig":
        d = dict(self.values)
        d.update(kw)
        return ExperimentConfig.from_dict(d)


def _atomic_write(path: Path, writer) -> None:
    """Write an artifact atomically."""
    path.parent.mkdir(parents=True, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=str(path.parent), prefix=".tmp_")
    os.close(fd)
    try:
        writer(tmp)
        os.replace(tmp, path)
    finally:
        if os.path.exists(tmp):
            os.unlink(tmp)


def _load_trace(cfg: ExperimentConfig):
    model = cfg.model_spec()
    v = cfg.values
    if v["trace_file"]:
        tr = parse_trace(v["trace_file"])
        if tr.model != model:
            raise ConfigError(f"trace file shape {tr.model} does not match config {model}")
        return tr
    return generate_trace(model, float(v["zipf_s"]), int(v["n_tokens"]), int(v["n_chunks"]), int(v["seed"]))


def _place_all(cfg, kind, model, c, train, need_freq=True):
    """Topology -> hop matrix -> cost matrix -> requested placements (plus f_train)."""
    g = build_topology(cfg.topology_spec(kind))
    c.check_feasible(model, g.n_devices)
    dist = all_pairs_hops(g)
    order = locality_order(g, dist)
    attn = default_attention_placement(model, order)
    cost = cost_matrix(dist, attn)
    placements = {}
    for m in cfg.values["methods"]:
        if m == "rr":
            placements[m] = place_round_robin(model, attn, order, c)
        elif m == "greedy":
            placements[m] = place_greedy(model, attn, cost, c)
        elif m == "ilp":
            placements[m], _ = solve_exact(build_instance(cost, UniformFrequencies(model.E), c))
            placements[m].label = "ilp"
    freq = None
    if "ilpload" in cfg.values["methods"] or need_freq:
        freq = estimate_frequencies(train, model)
    if "ilpload" in cfg.values["methods"]:
        placements["ilpload"], _ = solve_exact(build_instance(cost, freq, c))
        placements["ilpload"].label = "ilpload"
    for m, p in placements.items():
        p.label = m
        bad = validate(p, c, model, g.n_devices)
        if bad:
            raise InfeasibleError(f"{m} placement violates {len(bad)} constraint(s): {bad[0]}")
    return g, dist, attn, cost, placements, freq


def run_experiment(cfg: ExperimentConfig) -> dict:
    """SPEC.md:409-417.  Writes, per topology: topology JSON, distance CSV, placement CSVs,
    EvalReport JSONs, CommMap CSVs of the two best methods; plus one comparison CSV
    (network,placement,hops_mean,hops_std,gain_pct) with RR as the gain baseline."""
    if isinstance(cfg, dict):
        cfg = ExperimentConfig.from_dict(cfg)
    model, c = cfg.model_spec(), cfg.constraints()
    out = Path(cfg.values["output_dir"])
    trace = _load_trace(cfg)
    train, test = split_trace(trace, int(cfg.values["train_chunks"]), int(cfg.values["test_chunks"]))
    rows, results = [], {}
    multi = len(cfg.kinds()) > 1
    for kind in cfg.kinds():
        g, dist, attn, cost, placements, freq = _place_all(cfg, kind, model, c, train)
        d = out / kind if multi else out
        _atomic_write(d / "topology.json", lambda p: Path(p).write_text(json.dumps(g.to_json())))
        _atomic_write(d / "distance.csv", dist.to_csv)
        methods = list(placements)
        # one pass over train + test chunks (they are contiguous): per-chunk sums, split after
        n_tr, n_te = int(cfg.values["train_chunks"]), int(cfg.values["test_chunks"])
        both = trace.view(0, n_tr + n_te)
        sums = score_sums(both, [placements[m] for m in methods], cost)
        tok = both.chunk_token_counts()
        reports = [report_from_sums(sums[i, n_tr:], tok[n_tr:], m) for i, m in enumerate(methods)]
        train_reports = [report_from_sums(sums[i, :n_tr], tok[:n_tr], m) for i, m in enumerate(methods)]
        res = {}
        for m, rep, trep in zip(methods, reports, train_reports):
            rep.label = m
            rep.objective_train = objective_value(placements[m], freq, cost)
            res[m] = {"test": rep, "train": trep}
            _atomic_write(d / f"placement_{m}.csv", lambda p, m=m: write_placement(placements[m], p))
            _atomic_write(d / f"eval_{m}.json", rep.write)
            if getattr(placements[m], "solve_report", None):
                _atomic_write(d / f"solve_{m}.json", lambda p, m=m: write_solve_report(placements[m], p))
        base = res["rr"]["test"].mean_hops_per_token if "rr" in res else None
        for m in methods:
            r = res[m]["test"]
            gp = gain(base, r.mean_hops_per_token) if base is not None else 0.0
            rows.append((kind, m, r.mean_hops_per_token, r.std_hops, gp))
        best = sorted(methods, key=lambda m: (res[m]["test"].mean_hops_per_token, methods.index(m)))[:2]
        for m in best:
            cm = communication_map(test, placements[m], cost)
            _atomic_write(d / f"commmap_{m}.csv", cm.to_csv)
        results[kind] = res
    _atomic_write(out / "comparison.csv", lambda p: Path(p).write_text(
        "network,placement,hops_mean,hops_std,gain_pct\n" +
        "".join(f"{k},{m},{mean!r},{std!r},{gp!r}\n" for k, m, mean, std, gp in rows)))
    return {"rows": rows, "results": results, "output_dir": str(out)}


def ablate_clayer(cfg: ExperimentConfig, values) -> list:
    """one row per (topology, method, c_layer), with the exact-solver
    objective on the train frequencies.  Writes ablation.csv."""
    if isinstance(cfg, dict):
        cfg = ExperimentConfig.from_dict(cfg)
    rows = []
    base_out = Path(cfg.values["output_dir"])
    for cl in values:
        sub = cfg.with_(c_layer=int(cl), output_dir=str(base_out / f"c_layer_{cl}"))
        res = run_experiment(sub)
        for kind, per in res["results"].items():
            for m, r in per.items():
                t = r["test"]
                rows.append((kind, m, int(cl), t.mean_hops_per_token, t.std_hops, t.objective_train))
    _atomic_write(base_out / "ablation.csv", lambda p: Path(p).write_text(
        "network,placement,c_layer,hops_mean,hops_std,objective_train\n" +
        "".join(f"{k},{m},{cl},{a!r},{b!r},{o!r}\n" for k, m, cl, a, b, o in rows)))
    return rows


def _cfg_from_args(a) -> ExperimentConfig:
    d = {}
    if getattr(a, "config", None):
        d = ExperimentConfig.read_json(a.config)  # invalid JSON / non-object -> ConfigError (exit 2)
    for k in DEFAULTS:
        v = getattr(a, k, None)
        if v is not None and k not in d:  # --config overrides flags
            d[k] = v
    return ExperimentConfig.from_dict(d)


def _add_cfg_flags(p):
    p.add_argument("--config")
    for k, dv in DEFAULTS.items():
        typ = {"zipf_s": float, "topology": str, "trace_file": str, "output_dir": str, "model": str}.get(k, int)
        if k in ("methods", "topologies"):
            p.add_argument("--" + k.replace("_", "-"), dest=k, type=lambda s: s.split(","))
        else:
            p.add_argument("--" + k.replace("_", "-"), dest=k, type=typ)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="moeplace", description="topology-aware MoE expert placement (B200 engine)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("topo")
    p.add_argument("action", choices=["build"])
    _add_cfg_flags(p)
    p.add_argument("--out", required=True)
    p.add_argument("--dist-csv")
    p = sub.add_parser("trace")
    p.add_argument("action", choices=["gen", "stats"])
    _add_cfg_flags(p)
    p.add_argument("--out")
    p.add_argument("--trace")
    p = sub.add_parser("place")
    p.add_argument("method", choices=METHODS)
    _add_cfg_flags(p)
    p.add_argument("--out", required=True)
    p = sub.add_parser("eval")
    _add_cfg_flags(p)
    p.add_argument("--placement", required=True)
    p = sub.add_parser("compare")
    _add_cfg_flags(p)
    p = sub.add_parser("ablate")
    _add_cfg_flags(p)
    p.add_argument("--values", required=True, type=lambda s: [int(x) for x in s.split(",")])
    a = ap.parse_args(argv)
    try:
        if a.cmd == "topo":
            cfg = _cfg_from_args(a)
            g = build_topology(cfg.topology_spec(cfg.kinds()[0]))
            _atomic_write(Path(a.out), lambda p: Path(p).write_text(json.dumps(g.to_json())))
            if a.dist_csv:
                all_pairs_hops(g).to_csv(a.dist_csv)
        elif a.cmd == "trace" and a.action == "gen":
            cfg = _cfg_from_args(a)
            if not a.out:
                raise ConfigError("trace gen needs --out")
            tr = _load_trace(cfg.with_(trace_file=None))
            _atomic_write(Path(a.out), lambda p: write_trace(tr, p))
        elif a.cmd == "trace":
            if not a.trace:
                raise ConfigError("trace stats needs --trace")
            print(json.dumps(trace_stats(parse_trace(a.trace)), sort_keys=True))
        elif a.cmd == "place":
            cfg = _cfg_from_args(a).with_(methods=[a.method])
            train, _ = split_trace(_load_trace(cfg), int(cfg.train_chunks), int(cfg.test_chunks))
            _, _, _, _, pl, _ = _place_all(cfg, cfg.kinds()[0], cfg.model_spec(), cfg.constraints(), train,
                                           need_freq=False)
            _atomic_write(Path(a.out), lambda p: write_placement(pl[a.method], p))
        elif a.cmd == "eval":
            cfg = _cfg_from_args(a)
            model, c = cfg.model_spec(), cfg.constraints()
            g = build_topology(cfg.topology_spec(cfg.kinds()[0]))
            dist = all_pairs_hops(g)
            attn = default_attention_placement(model, locality_order(g, dist))
            cost = cost_matrix(dist, attn)
            pl = read_placement(a.placement, model, c, g.n_devices)
            _, test = split_trace(_load_trace(cfg), int(cfg.train_chunks), int(cfg.test_chunks))
            print(json.dumps(evaluate_many(test, [pl], cost)[0].to_json(), sort_keys=True))
        elif a.cmd == "compare":
            res = run_experiment(_cfg_from_args(a))
            print(Path(res["output_dir"]) / "comparison.csv")
        elif a.cmd == "ablate":
            ablate_clayer(_cfg_from_args(a), a.values)
        return 0
    except (MoeplaceError, OSError) as e:
        print(f"moeplace: error: {e}", file=sys.stderr)
        return exit_code(e)


if __name__ == "__main__":
    sys.exit(main())
