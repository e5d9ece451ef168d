"""Run manifests and replay for GPU solves.

The reference CLI records every run as a JSON manifest -- the command, its
full configuration, the FNV-1a digest of every input file -- and `replay`
re-executes a manifest after checking that no input changed; with
`--clock none` the data outputs are byte-identical across replays
(otaccel_cli.cpp:1-5, 40-95, 256-400, 543-580).  This module restates that for
the two solver commands on the device path:

* `solve`   one solver on one instance -> solve_trace.csv, solve_result.json,
            solve_manifest.json (otaccel_cli.cpp:333-349)
* `compare` Sinkhorn against acc-homotopy -> compare_trace.csv,
            compare_summary.json, compare_manifest.json (:351-395)
* `replay`  re-run a manifest (:543-580); the image / word-vector pipeline
            commands are out of scope here and refused.

Manifests written here carry `"device": "gpu"` at the top level (the
reference's replay reads only `command`, `config` and `inputs`, so the file
stays replayable there).  JSON is written with sorted keys and a two-space
indent, the layout of nlohmann::json's `dump(2)` over its ordered map.

CLI:  python -m paper_2605_30267_b200.replay solve --synthetic n=200,m=150,seed=7 --eps 0.05 \
          --clock none --out-dir out
      python -m paper_2605_30267_b200.replay replay --manifest out/solve_manifest.json
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import sys
from dataclasses import asdict, dataclass, field
from typing import Dict

from . import ot

VERSION = "0.1.0"  # the reference CLI's manifest version (otaccel_cli.cpp:32)


def file_digest(path: str) -> str:
    """FNV-1a 64 over the raw file bytes, 16 hex digits (otaccel_cli.cpp:49-65)."""
    h = 0xcbf29ce484222325
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise ot.IoError(f"cannot read input for digest: {path}") from e
    for byte in data:
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def write_file_atomic(path: str, content: str):
    """Write through a .partial name renamed on success (otaccel_cli.cpp:67-79)."""
    tmp = path + ".partial"
    try:
        with open(tmp, "w", newline="") as f:
            f.write(content)
    except OSError as e:
        raise ot.IoError(f"cannot write {tmp}") from e
    os.replace(tmp, path)


def _dump(obj) -> str:
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def _utc_now() -> str:
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def resolve_out_dir(flag: str) -> str:  # otaccel_cli.cpp:87-91
    if flag:
        return flag
    return os.environ.get("OTACCEL_OUT_DIR", ".")


# ------------------------------------------------------------ configs ----
@dataclass
class InstanceConfig:  # otaccel_cli.cpp:97-120
    kind: str = "synthetic"  # "synthetic" | "csv"
    n: int = 100
    m: int = 100
    seed: int = 1
    path: str = ""
    eps: float = 1e-2


@dataclass
class SolverConfig:  # otaccel_cli.cpp:122-150
    solver: str = "acc-homotopy"
    mu: float = 0.5
    mu0: float = 0.5
    m0: int = 4
    max_iters: int = 2000000
    trace_stride: int = 1
    clock: str = "wall"  # "wall" | "none"

    def spec(self) -> ot.SolverSpec:  # to_spec, otaccel_cli.cpp:152-163
        return ot.SolverSpec(kind=ot.solver_kind_from_name(self.solver), mu=self.mu,
                             mu0=self.mu0, m0=self.m0, max_iters=self.max_iters,
                             record_trace=True, trace_stride=self.trace_stride,
                             wall_clock=self.clock == "wall")


@dataclass
class SolveCmdConfig:  # otaccel_cli.cpp:165-184 (solve and compare share the layout)
    instance: InstanceConfig = field(default_factory=InstanceConfig)
    solver: SolverConfig = field(default_factory=SolverConfig)
    tol_l1: str = "auto"
    out_dir: str = ""

    def to_json(self) -> dict:
        return {"instance": asdict(self.instance), "solver": asdict(self.solver),
                "tol_l1": self.tol_l1, "out_dir": self.out_dir}

    @staticmethod
    def from_json(j: dict) -> "SolveCmdConfig":
        try:
            inst = InstanceConfig(**{k: j["instance"][k] for k in InstanceConfig.__dataclass_fields__})
            sol = SolverConfig(**{k: j["solver"][k] for k in SolverConfig.__dataclass_fields__})
            return SolveCmdConfig(inst, sol, j["tol_l1"], j["out_dir"])
        except (KeyError, TypeError) as e:
            raise ot.OtError(f"malformed manifest config: missing {e}") from e


# ------------------------------------------------------------ helpers ----
def load_instance(c: InstanceConfig, inputs: Dict[str, str]) -> ot.TransportProblem:
    """otaccel_cli.cpp:258-275: synthetic (data.cpp:17-41) or an instance CSV."""
    if c.kind == "synthetic":
        a, b, C = ot.synthetic_instance(c.n, c.m, c.seed)
        return ot.with_epsilon(ot.make_problem(a, b, C, 1.0), c.eps)
    if c.kind != "csv":
        raise ot.OtError("instance kind must be synthetic or csv")
    inputs[c.path] = file_digest(c.path)
    p = ot.read_instance_csv(c.path)
    if c.eps > 0.0:
        p = ot.with_epsilon(p, c.eps)
    else:
        c.eps = p.epsilon  # record the file's strength so a replay matches
    c.n, c.m = p.n(), p.m()
    return p


def resolve_tol(tol: str, n: int, alignment_style: bool = False) -> float:
    """otaccel_cli.cpp:277-292: "auto" = 2 / n (1% of that for alignment)."""
    if tol == "auto":
        base = 2.0 / n
        return 0.01 * base if alignment_style else base
    try:
        v = float(tol)
    except ValueError:
        raise ot.OtError(f"bad --tol-l1 value: {tol}") from None
    if not v > 0.0:
        raise ot.OtError(f"bad --tol-l1 value: {tol}")
    return v


def write_manifest(path: str, command: str, config: dict, seed: int, inputs: Dict[str, str],
                   started: str):
    """otaccel_cli.cpp:294-301, plus the device the run used."""
    m = {"command": command, "version": VERSION, "seed": seed, "config": config,
         "inputs": dict(inputs), "started": started, "finished": _utc_now(), "device": "gpu"}
    write_file_atomic(path, _dump(m))


def result_json(r: ot.SolveResult, solver: str, eps: float, tol: float) -> dict:
    """otaccel_cli.cpp:320-331."""
    return {"solver": solver, "eps": eps, "tol_l1": tol, "converged": bool(r.converged),
            "iterations": int(r.iterations), "evaluations": int(r.evaluations),
            "outer_stages": int(r.outer_stages), "final_violation": float(r.final_violation),
            "final_reduced_f": float(r.final_reduced_f), "max_v_inf": float(r.max_v_inf)}


# ----------------------------------------------------------- commands ----
def run_solve(cfg: SolveCmdConfig) -> int:
    """otaccel_cli.cpp:333-349: exit 0 when converged, 2 otherwise."""
    out = resolve_out_dir(cfg.out_dir)
    os.makedirs(out, exist_ok=True)
    inputs: Dict[str, str] = {}
    started = _utc_now()
    prob = load_instance(cfg.instance, inputs)
    scaled = ot.rescale_problem(prob)
    tol = resolve_tol(cfg.tol_l1, scaled.n())
    r = ot.run_solver(scaled, cfg.solver.spec(), tol)
    write_file_atomic(os.path.join(out, "solve_trace.csv"), r.trace.to_csv())
    write_file_atomic(os.path.join(out, "solve_result.json"),
                      _dump(result_json(r, cfg.solver.solver, cfg.instance.eps, tol)))
    write_manifest(os.path.join(out, "solve_manifest.json"), "solve", cfg.to_json(),
                   cfg.instance.seed, inputs, started)
    return 0 if r.converged else 2


def run_compare(cfg: SolveCmdConfig) -> int:
    """otaccel_cli.cpp:351-395: both solvers, one joined trace, a summary."""
    out = resolve_out_dir(cfg.out_dir)
    os.makedirs(out, exist_ok=True)
    inputs: Dict[str, str] = {}
    started = _utc_now()
    prob = load_instance(cfg.instance, inputs)
    scaled = ot.rescale_problem(prob)
    tol = resolve_tol(cfg.tol_l1, scaled.n())
    sink = SolverConfig(**{**asdict(cfg.solver), "solver": "sinkhorn"})
    acc = SolverConfig(**{**asdict(cfg.solver), "solver": "acc-homotopy"})
    rs = ot.run_solver(scaled, sink.spec(), tol)
    ra = ot.run_solver(scaled, acc.spec(), tol)
    joined = ["solver," + ot.SolverTrace.csv_header()]
    for name, r in (("sinkhorn", rs), ("acc-homotopy", ra)):
        joined += [f"{name},{line}" for line in r.trace.to_csv().splitlines()[1:]]
    write_file_atomic(os.path.join(out, "compare_trace.csv"), "\n".join(joined) + "\n")
    summary = {"eps": cfg.instance.eps, "tol_l1": tol, "n": cfg.instance.n,
               "m": cfg.instance.m,
               "sinkhorn": result_json(rs, "sinkhorn", cfg.instance.eps, tol),
               "acc_homotopy": result_json(ra, "acc-homotopy", cfg.instance.eps, tol)}
    if rs.converged and ra.converged:
        speedup = 1.0
        if rs.iterations or ra.iterations:
            speedup = rs.iterations / max(ra.iterations, 1)
        summary["speedup_inner_iterations"] = speedup
    else:
        summary["speedup_inner_iterations"] = None
    write_file_atomic(os.path.join(out, "compare_summary.json"), _dump(summary))
    write_manifest(os.path.join(out, "compare_manifest.json"), "compare", cfg.to_json(),
                   cfg.instance.seed, inputs, started)
    return 0 if (rs.converged and ra.converged) else 2


def run_replay(manifest_path: str, out_dir_override: str = "") -> int:
    """otaccel_cli.cpp:543-580: refuse a changed input, then re-run."""
    try:
        with open(manifest_path) as f:
            m = json.load(f)
    except OSError as e:
        raise ot.IoError(f"cannot read manifest: {manifest_path}") from e
    for path, digest in m.get("inputs", {}).items():
        now = file_digest(path)
        if now != digest:
            raise ot.IoError(f"input changed since the recorded run: {path} (digest {now}, "
                             f"manifest {digest})")
    command = m.get("command")
    cfg = SolveCmdConfig.from_json(m.get("config", {})) if command in ("solve", "compare") else None
    if cfg is not None and out_dir_override:
        cfg.out_dir = out_dir_override
    if command == "solve":
        return run_solve(cfg)
    if command == "compare":
        return run_compare(cfg)
    if command in ("color-transfer", "word-align"):
        raise ot.OtError(f"manifest command {command} is a reference pipeline, not the GPU path")
    raise ot.OtError(f"unknown command in manifest: {command}")


# ----------------------------------------------------------------- CLI ----
def _parse_synthetic(spec: str, inst: InstanceConfig):  # otaccel_cli.cpp:583-606
    inst.kind = "synthetic"
    for part in spec.split(","):
        if "=" not in part:
            raise ot.OtError(f"--synthetic expected key=value: {part}")
        key, val = part.split("=", 1)
        if key == "n":
            inst.n = int(val)
        elif key == "m":
            inst.m = int(val)
        elif key == "seed":
            inst.seed = int(val)
        else:
            raise ot.OtError(f"--synthetic unknown key: {key}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="otg-replay", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("solve", "compare"):
        s = sub.add_parser(name)
        s.add_argument("--synthetic", default="n=100,m=100,seed=1")
        s.add_argument("--instance", default="", help="instance CSV (name,index,value)")
        s.add_argument("--eps", type=float, default=1e-2)
        s.add_argument("--solver", default="acc-homotopy")
        s.add_argument("--mu", type=float, default=0.5)
        s.add_argument("--mu0", type=float, default=0.5)
        s.add_argument("--m0", type=int, default=4)
        s.add_argument("--max-iters", type=int, default=2000000)
        s.add_argument("--trace-stride", type=int, default=1)
        s.add_argument("--clock", default="wall", choices=["wall", "none"])
        s.add_argument("--tol-l1", default="auto")
        s.add_argument("--out-dir", default="")
    r = sub.add_parser("replay")
    r.add_argument("--manifest", required=True)
    r.add_argument("--out-dir", default="")
    a = ap.parse_args(argv)
    if a.cmd == "replay":
        return run_replay(a.manifest, a.out_dir)
    inst = InstanceConfig(eps=a.eps)
    if a.instance:
        inst.kind, inst.path = "csv", a.instance
    else:
        _parse_synthetic(a.synthetic, inst)
    cfg = SolveCmdConfig(inst, SolverConfig(a.solver, a.mu, a.mu0, a.m0, a.max_iters,
                                            a.trace_stride, a.clock), a.tol_l1, a.out_dir)
    return run_solve(cfg) if a.cmd == "solve" else run_compare(cfg)


if __name__ == "__main__":
    sys.exit(main())
