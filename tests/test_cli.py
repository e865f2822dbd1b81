"""CLI flows (reference test_cli.py's coverage): generate -> check -> enumerate
on CPU; simulate / optimize / --check-delta through the GPU path."""

import json
import re

import pytest

import paper_1807_05358_b200 as ps
from paper_1807_05358_b200.cli import main


@pytest.fixture
def inputs(tmp_path):
    g, t = tmp_path / "graph.json", tmp_path / "topo.json"
    assert main(["generate", "rnnlm-like", "--steps", "1", "--layers", "1", "--batch", "4", "--hidden", "4",
                 "--vocab", "8", "--out", str(g)]) == 0
    assert main(["generate", "p100-node", "--gpus", "2", "--out", str(t)]) == 0
    return g, t


def test_generate_and_check(inputs, capsys):
    g, t = inputs
    assert ps.validate_graph(ps.load_graph(g)).ok
    assert main(["check", "--graph", str(g), "--topology", str(t)]) == 0
    out = capsys.readouterr().out
    assert "graph ok" in out and "topology ok" in out


def test_generate_stdout_and_errors(capsys):
    assert main(["generate", "rnn3"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert doc["format_version"] == 1 and doc["ops"]
    assert main(["generate", "resnet-9000"]) == 2
    assert "unknown generator" in capsys.readouterr().err
    assert main(["generate", "rnn3", "--gpus", "4"]) == 2
    assert "does not take --gpus" in capsys.readouterr().err
    assert main(["check"]) == 2
    assert main(["generate", "inception-v3"]) == 0
    assert len(json.loads(capsys.readouterr().out)["ops"]) == 125


def test_check_rejects_bad_files(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert main(["check", "--graph", str(bad)]) == 2
    assert main(["check", "--graph", str(tmp_path / "missing.json")]) == 2
    assert "not found" in capsys.readouterr().err


def test_enumerate(inputs, capsys):
    g, t = inputs
    assert main(["enumerate", "--graph", str(g), "--topology", str(t), "--max-degree", "2"]) == 0
    out = capsys.readouterr().out
    assert "configs up to degree 2" in out and "tasks=" in out
    assert main(["enumerate", "--graph", str(g), "--topology", str(t), "--op", "nope"]) == 2


def _makespan(out):
    m = re.search(r"makespan: ([0-9eE+.inf-]+) s", out)
    assert m, out
    return float(m.group(1))


@pytest.mark.gpu
def test_simulate_and_check_delta(inputs, tmp_path, capsys):
    g, t = inputs
    trace, csv = tmp_path / "trace.json", tmp_path / "tl.csv"
    assert main(["simulate", "--graph", str(g), "--topology", str(t), "--trace", str(trace), "--csv", str(csv),
                 "--check-delta", "8"]) == 0
    out = capsys.readouterr().out
    assert _makespan(out) > 0 and "all matched full rebuilds" in out
    assert json.loads(trace.read_text())["traceEvents"]
    assert csv.read_text().startswith("task,device,start,end")


@pytest.mark.gpu
def test_optimize_is_reproducible(inputs, tmp_path, capsys):
    g, t = inputs
    r1, r2, s1 = tmp_path / "r1.json", tmp_path / "r2.json", tmp_path / "s.json"
    for rep in (r1, r2):
        assert main(["optimize", "--graph", str(g), "--topology", str(t), "--max-proposals", "60", "--seed", "3",
                     "--max-degree", "2", "--report", str(rep), "--out-strategy", str(s1)]) == 0
    assert r1.read_text() == r2.read_text()
    assert "best cost" in capsys.readouterr().out
    assert main(["simulate", "--graph", str(g), "--topology", str(t), "--strategy", str(s1)]) == 0
    best = json.loads(r1.read_text())["best_cost"]
    assert _makespan(capsys.readouterr().out) == best
    assert main(["optimize", "--graph", str(g), "--topology", str(t)]) == 2
