"""The reference's CLI driver (proj/tools/fmm_bench.cpp) over the B200 path: flags, exit codes,
run / sweep CSV (engine.cpp:127-166), stage trace CSV (scheduler.cpp:305-317), DOT
(scheduler.cpp:287-303), and the reference generator (dataset.cpp:76-111) it feeds."""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1203_0889_b200", "bin", "fmm_bench")
GOLD = os.path.join(ROOT, "tests", "golden", "ref_cases.npz")


def run(*args, **kw):
    if not os.path.exists(BIN):
        pytest.skip("fmm_bench not built (python -c 'import __graft_entry__ as g; g.build()')")
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=kw.get("timeout", 600))


def test_help_and_argument_errors():
    r = run("--help")
    assert r.returncode == 0 and "--sweep" in r.stdout and "--mutual" in r.stdout
    # CLI11 exit codes of the reference driver: conversion 104, validation 105, extras 109
    assert run("--n", "abc").returncode == 104
    assert run("--theta", "1.5").returncode == 105
    assert run("--n", "0").returncode == 105
    assert run("--ncrit", "-3").returncode == 105
    assert run("--sweep", "x=1").returncode == 105
    assert run("--bogus").returncode == 109


def test_runtime_errors_exit_1():
    r = run("--dist", "nowhere", "--n", "10")
    assert r.returncode == 1 and "unknown distribution name: nowhere" in r.stderr


def test_reference_generator_matches_golden_bodies():
    """fmm_generate_bodies 10/11/12 = the reference's generate_bodies(cube / sphere-surface /
    cluster) bit-for-bit (bodies of the committed fixtures came from the reference build)."""
    import paper_1203_0889_b200 as fb
    fx = np.load(GOLD)
    for name, cfg, n, seed in (("cube2048_p6", 10, 2048, 15), ("cluster512_p3", 12, 512, 12),
                               ("sphere2000_p5", 11, 2000, 18), ("cube4096_p3_q", 10, 4096, 3)):
        assert np.array_equal(fb.generate_bodies(cfg, n, seed), fx[f"{name}/bodies"]), name


@pytest.mark.gpu
def test_cli_run_check_csv_trace_dag(tmp_path):
    csv_path, trace, dag = tmp_path / "run.csv", tmp_path / "trace.csv", tmp_path / "dag.dot"
    for mutual in ("--non-mutual", "--mutual"):
        r = run("--n", "20000", "--p", "6", "--dist", "cluster", "--check", mutual, "--csv", str(csv_path),
                "--trace", str(trace), "--dag", str(dag))
        assert r.returncode == 0, r.stderr
        assert "check     rel_l2=" in r.stdout and ("mutual" in r.stdout)
    rows = list(csv.DictReader(io.StringIO(csv_path.read_text())))
    assert len(rows) == 2 and [row["mutual"] for row in rows] == ["0", "1"]
    assert list(rows[0].keys()) == ("n,p,q,threads,theta,ncrit,mutual,dist,seed,t_build,t_upward,"
                                    "t_traversal,t_downward,t_total,tasks,rel_l2,rel_linf").split(",")
    for row in rows:
        assert row["dist"] == "cluster" and row["q"] == "200" and int(row["tasks"]) > 0
        assert float(row["rel_l2"]) < 1e-4  # p = 6 (test_output.txt: 5.89e-5 at N=1e4, cube)
        assert abs(float(row["t_total"]) - sum(float(row[k]) for k in
                   ("t_build", "t_upward", "t_traversal", "t_downward"))) < 1e-6
    tr = list(csv.DictReader(io.StringIO(trace.read_text())))
    assert [t["kind"] for t in tr] == ["build", "traversal", "upward", "m2l", "p2p", "downward"]
    assert all(int(t["end_ns"]) >= int(t["start_ns"]) >= 0 for t in tr)
    text = dag.read_text()
    assert text.startswith("digraph tasks {") and text.count("->") == 7 and 't5 [label="downward #5"]' in text
    # a failed accuracy check exits 2 (fmm_bench.cpp:141-145)
    r = run("--n", "5000", "--p", "2", "--check", "--check-tol", "1e-12")
    assert r.returncode == 2 and "check failed" in r.stderr


@pytest.mark.gpu
def test_cli_sweep(tmp_path):
    out = tmp_path / "sweep.csv"
    r = run("--sweep", "n=4000,8000;p=3,5;t=1", "--csv", str(out), "--dist", "sphere-surface")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert len(rows) == 4 and {(row["n"], row["p"]) for row in rows} == {("4000", "3"), ("8000", "3"),
                                                                         ("4000", "5"), ("8000", "5")}
    assert all(float(row["speedup_vs_T1"]) == 1.0 for row in rows)
    assert "wrote 4 rows" in r.stdout


@pytest.mark.gpu
def test_stage_trace_python(fmmlib):
    ctx = fmmlib.Context(order=4, n_crit=64, theta=0.5)
    ctx.set_bodies(fmmlib.generate_bodies(1, 30000, 2))
    ctx.evaluate()
    tr = ctx.stage_trace()
    assert [r[2] for r in tr] == ["build", "traversal", "upward", "m2l", "p2p", "downward"]
    assert tr[2][1] == 1  # default overlap: the upward pass runs on the second stream
    t = ctx.stage_times()
    assert abs((tr[-1][4] - tr[0][3]) * 1e-6 - t.total_ms) < 1e-2
    ctx.close()
