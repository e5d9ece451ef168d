"""Run manifests and replay (otaccel_cli.cpp:40-95, 294-301, 543-580): the
host-side logic on CPU, the byte-identical replay of a GPU solve on the GPU."""
import json
import os

import numpy as np
import pytest

from paper_2605_30267_b200 import ot
from paper_2605_30267_b200 import replay as R


def test_fnv1a_known_answers(tmp_path):
    # published FNV-1a 64 test vectors
    for data, want in ((b"", "cbf29ce484222325"), (b"a", "af63dc4c8601ec8c"),
                       (b"foobar", "85944171f73967e8")):
        f = tmp_path / "x.bin"
        f.write_bytes(data)
        assert R.file_digest(str(f)) == want
    with pytest.raises(ot.IoError):
        R.file_digest(str(tmp_path / "missing"))


def test_resolve_tol():
    assert R.resolve_tol("auto", 100) == 0.02
    assert R.resolve_tol("auto", 100, alignment_style=True) == pytest.approx(2e-4)
    assert R.resolve_tol("1e-6", 100) == 1e-6
    for bad in ("0", "-1", "x", "nan"):
        with pytest.raises(ot.OtError):
            R.resolve_tol(bad, 100)


def test_config_round_trip():
    cfg = R.SolveCmdConfig(R.InstanceConfig("synthetic", 7, 5, 3, "", 0.25),
                           R.SolverConfig("sinkhorn", 0.4, 0.3, 6, 1000, 2, "none"), "1e-8", "o")
    j = json.loads(json.dumps(cfg.to_json()))
    assert R.SolveCmdConfig.from_json(j) == cfg
    with pytest.raises(ot.OtError):
        R.SolveCmdConfig.from_json({"instance": {}, "solver": {}})


def test_replay_refusals(tmp_path):
    f = tmp_path / "inst.csv"
    f.write_text("name,index,value\n")
    m = {"command": "solve", "config": {}, "inputs": {str(f): "0000000000000000"}}
    (tmp_path / "m.json").write_text(json.dumps(m))
    with pytest.raises(ot.IoError):  # the input changed since the recorded run
        R.run_replay(str(tmp_path / "m.json"))
    for cmd in ("word-align", "frobnicate"):
        (tmp_path / "m.json").write_text(json.dumps({"command": cmd, "config": {}, "inputs": {}}))
        with pytest.raises(ot.OtError):
            R.run_replay(str(tmp_path / "m.json"))
    with pytest.raises(ot.IoError):
        R.run_replay(str(tmp_path / "nope.json"))


@pytest.mark.gpu
def test_solve_replay_is_byte_identical(tmp_path):
    out = str(tmp_path / "run")
    rc = R.main(["solve", "--synthetic", "n=60,m=45,seed=8", "--eps", "0.05", "--clock", "none",
                 "--tol-l1", "1e-9", "--out-dir", out])
    assert rc == 0
    trace = open(os.path.join(out, "solve_trace.csv")).read()
    result = open(os.path.join(out, "solve_result.json")).read()
    man = json.load(open(os.path.join(out, "solve_manifest.json")))
    assert man["command"] == "solve" and man["device"] == "gpu" and man["version"] == R.VERSION
    res = json.loads(result)
    assert res["converged"] and res["iterations"] == len(trace.splitlines()) - 2
    out2 = str(tmp_path / "again")
    assert R.run_replay(os.path.join(out, "solve_manifest.json"), out2) == 0
    assert open(os.path.join(out2, "solve_trace.csv")).read() == trace
    assert open(os.path.join(out2, "solve_result.json")).read() == result


@pytest.mark.gpu
def test_compare_from_instance_csv(tmp_path):
    a, b, C = ot.synthetic_instance(30, 20, 4)
    csv_path = str(tmp_path / "inst.csv")
    ot.write_instance_csv(csv_path, ot.with_epsilon(ot.make_problem(a, b, C, 1.0), 0.1))
    out = str(tmp_path / "cmp")
    assert R.main(["compare", "--instance", csv_path, "--eps", "0", "--clock", "none",
                   "--out-dir", out]) == 0
    s = json.load(open(os.path.join(out, "compare_summary.json")))
    assert s["eps"] == 0.1 and s["n"] == 30 and s["m"] == 20
    assert s["sinkhorn"]["converged"] and s["acc_homotopy"]["converged"]
    man = json.load(open(os.path.join(out, "compare_manifest.json")))
    assert man["inputs"] == {csv_path: R.file_digest(csv_path)}
    joined = open(os.path.join(out, "compare_trace.csv")).read()
    out2 = str(tmp_path / "cmp2")
    assert R.run_replay(os.path.join(out, "compare_manifest.json"), out2) == 0
    assert open(os.path.join(out2, "compare_trace.csv")).read() == joined
