"""CPU: host logic of the experiment driver (paper_2412_20980_b200/experiment.py, the mirror of gapa::bench and
of the file loaders) against golden values produced by the unmodified reference (tests/golden/experiments.json,
tests/golden/make_golden.py).  No compute call is made here."""
import hashlib
import json
import os
import struct
import subprocess

import numpy as np
import pytest

import golden_cases as gc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ex(gp):
    from paper_2412_20980_b200 import experiment
    return experiment


@pytest.fixture(scope="module")
def golden():
    return gc.load("experiments.json")


def test_format_double_is_std_to_chars(ex, tmp_path):
    """bench.cpp:378-382 formats every metric with std::to_chars(double): compare on edge cases and random bit
    patterns against a two-line C++ program."""
    src = tmp_path / "fmt.cpp"
    src.write_text('#include <charconv>\n#include <cstdio>\n#include <cstring>\nint main(){unsigned long long b;char buf[64];'
                   'while(std::scanf("%llx",&b)==1){double v;std::memcpy(&v,&b,8);auto r=std::to_chars(buf,buf+64,v);*r.ptr=0;'
                   'std::puts(buf);}}\n')
    exe = tmp_path / "fmt"
    subprocess.run(["g++", "-std=c++17", "-O1", str(src), "-o", str(exe)], check=True)
    rng = np.random.default_rng(8)
    values = [0.0, -0.0, 0.5, 34.0, 1e5, 1e-4, 1e-5, 1e22, 1e21, 123456789012345678.0, 0.1, 1 / 3, 5e-324, 1.7976931348623157e308,
              447931.0, 499999500000.0, -0.5, 0.26156030286641424, 100000.5, 1e15, 1e16, 1e17, 0.001, 0.00101]
    values += [float(x) for x in rng.random(300)] + [float(x) for x in rng.integers(0, 10**12, 200)]
    values += [float(10.0 ** e * m) for e, m in zip(rng.integers(-30, 30, 300), rng.random(300))]
    bits = rng.integers(0, 2**63 - 1, 500, dtype=np.int64)
    values += [v for v in (struct.unpack("<d", struct.pack("<q", int(b)))[0] for b in bits) if v == v and abs(v) != float("inf")]
    text = "\n".join("%x" % struct.unpack("<Q", struct.pack("<d", v))[0] for v in values)
    want = subprocess.run([str(exe)], input=text, capture_output=True, text=True, check=True).stdout.split("\n")
    for v, w in zip(values, want):
        assert ex.format_double(v) == w, (v, w)


def test_loaders(ex, golden):
    for name, c in golden["datasets"].items():
        res = ex.load_edge_list_file(os.path.join(ROOT, "tests", "golden", "datasets", name))
        e = np.asarray(res.graph.edges(), dtype=np.int32)
        assert (res.graph.n, len(e)) == (c["n"], c["m"]) and gc.sha(e) == c["sha"] and e[:5].tolist() == c["first"], name
    noisy = ex.load_edge_list_file(os.path.join(ROOT, "tests", "golden", "datasets", "sbm60.txt"))
    assert (noisy.self_loops_dropped, noisy.duplicates_dropped) == (1, 1)
    g = ex.load_edge_list("a b\n# c\n\n b   c \n% x\nc a\r\n").graph  # graph.cpp:65-118
    assert g.n == 3 and g.labels == ["a", "b", "c"] and g.edges().tolist() == [[0, 1], [1, 2], [0, 2]]
    with pytest.raises(ex.ParseError, match="edge list line 2: expected exactly 2 tokens"):
        ex.load_edge_list("a b\na b c\n")
    with pytest.raises(ex.DatasetError, match="cannot open edge list file"):
        ex.load_edge_list_file("/nonexistent/file.txt")
    truth = ex.load_community_file(os.path.join(ROOT, "tests", "golden", "datasets", "sbm60_truth.txt"), noisy.graph)
    assert len(truth) == 60 and len(set(truth.tolist())) == 4
    labels = noisy.graph.labels
    assert all(truth[i] == truth[j] for i in range(60) for j in range(60) if labels[i][1:3] != "" and int(labels[i][1:]) // 15 == int(labels[j][1:]) // 15)


def test_nmi_and_precision_match_the_reference(ex, golden, oracle):
    for c in golden["metrics"]["nmi"]:
        assert ex.nmi(c["a"], c["b"]) == c["nmi"]
    for c in golden["metrics"]["lp"]:
        og = oracle.graph_from_edges(c["n"], np.asarray(c["edges"], dtype=np.int32).reshape(-1, 2))
        sp = oracle.split_build(og, c["fraction"], c["split_seed"])
        scores = np.asarray(c["scores"])
        assert ex.precision_at_test_count(scores[:sp.T], scores[sp.T:], sp.test, sp.probe) == c["precision"]
        genes = np.asarray(c["genes"], dtype=np.int32).reshape(1, -1)
        assert oracle.eval_batch(sp, 3, genes)[0] == c["auc"]  # the oracle's AUC on the same individual


def test_config_rules(ex):
    cfg = ex.parse_config('{"algorithm": "qattack", "dataset": "d.txt"}')
    assert (cfg.task, cfg.pool_kind, cfg.params.pc, cfg.params.pm, cfg.params.iterations, cfg.params.pop_size) == \
           (ex.Task.CdaModularity, ex.PoolKind.EdgeAddition, 0.8, 0.1, 1500, 100)  # bench.cpp:72-79
    cfg = ex.parse_config('{"algorithm": "lpa-eda", "dataset": "d.txt", "pop_size": 20}')
    assert cfg.params.eda_interval == 1 and cfg.params.pc == 0.0 and cfg.params.pop_size == 20
    assert ex.parse_config('{"task": "cnd-pc", "dataset": "d"}').pool_kind == ex.PoolKind.NodeRemoval  # default_pool_kind
    assert ex.parse_config('{"task": "cda-modularity", "dataset": "d"}').pool_kind == ex.PoolKind.EdgeAddition
    for bad, msg in [('{"dataset": "d"}', "either 'algorithm' or 'task' is required"), ('[1]', "expected a JSON object"),
                     ('{"task": "cnd-pc", "dataset": "d", "colour": 1}', "unknown key 'colour'"), ('{', "invalid JSON"),
                     ('{"task": "cnd-pc"}', "dataset path is required"), ('{"task": "nope", "dataset": "d"}', "unknown task"),
                     ('{"task": "cnd-pc", "dataset": "d", "pool": "edge-removal"}', "cnd-\\* tasks require a node-removal pool"),
                     ('{"task": "lpa-similarity", "dataset": "d", "pool": "edge-addition"}', "requires an edge-removal pool"),
                     ('{"task": "cda-modularity", "dataset": "d", "pool": "node-removal"}', "edge-removal or edge-addition"),
                     ('{"task": "cnd-pc", "dataset": "d", "mode": "s", "pn": 2}', "serial and s modes fix pn = qn = 1"),
                     ('{"task": "cnd-pc", "dataset": "d", "mode": "x"}', "unknown mode"),
                     ('{"task": "cnd-pc", "dataset": "d", "pop_size": 1}', "pop_size must be >= 2"),
                     ('{"task": "cnd-pc", "dataset": "d", "iterations": 0}', "iterations must be >= 1"),
                     ('{"task": "cnd-pc", "dataset": "d", "test_fraction": 0.6}', "test_fraction"),
                     ('{"task": "cnd-pc", "dataset": "d", "perturbation_rate": 0}', "perturbation_rate"),
                     ('{"task": "cnd-pc", "dataset": "d", "repetitions": 0}', "repetitions"),
                     ('{"algorithm": "fancy", "dataset": "d"}', "unknown algorithm preset")]:
        with pytest.raises(ex.ConfigError, match=msg):
            ex.parse_config(bad)
    with pytest.raises(ex.ConfigError, match="strictly ascending"):
        ex.sweep(ex.parse_config('{"task": "cnd-pc", "dataset": "d"}'), "pop_size", [8, 8])
    with pytest.raises(ex.ConfigError, match="unknown sweep axis"):
        ex.sweep(ex.parse_config('{"task": "cnd-pc", "dataset": "d"}'), "qn", [2])


def test_report_round_trip_is_byte_identical(ex, golden):
    """parse_rows_csv -> report reproduces the reference's CSV bytes; csv_without_wall_time matches its output."""
    for c in golden["experiments"]:
        rows = ex.parse_rows_csv(c["csv"])
        assert ex.report(rows, "csv") == c["csv"]
        assert ex.csv_without_wall_time(c["csv"]) == c["csv_without_wall_time"]
        table = ex.report(rows, "table").split("\n")
        assert len({len(line) for line in table[:-1]}) == 1 and table[0].startswith("task")
    with pytest.raises(ex.ParseError, match="wrong column count in header"):
        ex.parse_rows_csv("task,algorithm\n")
    with pytest.raises(ex.ParseError, match="rows CSV line 2: bad number 'x'"):
        ex.parse_rows_csv(golden["experiments"][0]["csv"].split("\n")[0] + "\n" + "t,a,d,s,x,1,2,3,4,0.1" + "," * 12 + "\n")


def test_cli_report_and_exit_codes(ex, golden, tmp_path, capsys):
    rows = tmp_path / "rows.csv"
    rows.write_text(golden["experiments"][3]["csv"])
    assert ex.main(["report", str(rows), "--format", "csv"]) == 0
    assert capsys.readouterr().out == golden["experiments"][3]["csv"]
    bad = tmp_path / "bad.json"
    bad.write_text('{"task": "cnd-pc", "dataset": "d", "colour": 1}')
    assert ex.main(["run", str(bad)]) == 2  # gapa_main.cpp:13-15
    missing = tmp_path / "missing.json"
    missing.write_text(json.dumps({"task": "cnd-pc", "dataset": str(tmp_path / "nope.txt")}))
    assert ex.main(["run", str(missing)]) == 3
