"""GPU: the experiment driver on the CUDA path against the reference's own bench::run_experiment / sweep
(SURVEY §8 f-4).  The reference's determinism contract is byte identity of the rows CSV with the wall_time_s
column blanked (bench.hpp:83-85); tests/golden/experiments.json holds that CSV from the unmodified reference
(CPU) for every config below, and the GPU run must produce the same bytes — fitness trajectories, metric
columns (Q, NMI, MCN, PC, AUC, precision) and number formatting included."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import golden_cases as gc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = gc.load("experiments.json")


@pytest.fixture(scope="module")
def ex(gp, cuda_device):
    from paper_2412_20980_b200 import experiment
    return experiment


@pytest.fixture(autouse=True)
def _repo_root(monkeypatch):
    monkeypatch.chdir(ROOT)  # dataset paths in the golden configs are repo-relative


@pytest.mark.parametrize("index", range(len(GOLDEN["experiments"])),
                         ids=[c["config"].get("algorithm", c["config"].get("task")) + "-" + os.path.basename(c["config"]["dataset"])
                              + ("-sweep" if c["axis"] else "") for c in GOLDEN["experiments"]])
def test_experiment_csv_is_byte_identical_to_the_reference(ex, index, tmp_path):
    c = GOLDEN["experiments"][index]
    cfg = ex.parse_config(json.dumps(c["config"]))
    cfg.output = str(tmp_path / "rows.csv")
    rows = ex.sweep(cfg, c["axis"], c["values"]) if c["axis"] else ex.run_experiment(cfg)
    text = ex.report(rows, "csv")
    assert ex.csv_without_wall_time(text) == c["csv_without_wall_time"]
    assert open(cfg.output).read() == text and all(r.wall_time_s > 0 for r in rows)


def test_detected_partitions_match_the_reference(gp, cuda_device):
    for c in GOLDEN["metrics"]["detect"]:
        g = gp.Graph(c["n"], gc.i32(c["edges"], 2))
        obj = gp.ModularityAttackObjective(g, gp.build_gene_pool(g, gp.PoolKind(c["kind"])))
        genes = gc.i32(c["genes"]).reshape(-1)
        out = np.zeros(c["n"], dtype=np.int32)
        q = C.c_double(0)
        gp.capi.check(obj.dgraph.lib.gapa_cuda_detect_communities(
            obj.dgraph.handle, genes.ctypes.data_as(C.c_void_p) if genes.size else None, genes.size,
            out.ctypes.data_as(C.c_void_p), C.byref(q)))
        assert out.tolist() == c["assignment"]
        assert q.value == obj.evaluate_one(genes)
    g = gp.Graph(5, np.zeros((0, 2), np.int32))  # edgeless: everyone stays a singleton
    obj = gp.ModularityAttackObjective(g, gp.build_gene_pool(g, gp.PoolKind.EdgeAddition))
    out = np.zeros(5, dtype=np.int32)
    gp.capi.check(obj.dgraph.lib.gapa_cuda_detect_communities(obj.dgraph.handle, None, 0, out.ctypes.data_as(C.c_void_p), None))
    assert out.tolist() == [0, 1, 2, 3, 4]


def test_ra_scores_auc_and_precision_match_the_reference(gp, ex, cuda_device):
    for c in GOLDEN["metrics"]["lp"]:
        g = gp.Graph(c["n"], gc.i32(c["edges"], 2))
        split = gp.build_lp_split(g, c["fraction"], c["split_seed"])
        obj = gp.LinkPredictionAttackObjective(split, gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval))
        genes = gc.i32(c["genes"]).reshape(-1)
        T, P = len(split.test_edges), len(split.probe_nonedges)
        t, p, auc = np.zeros(T), np.zeros(P), C.c_double(0)
        gp.capi.check(obj.dgraph.lib.gapa_cuda_lpa_scores(
            obj.dgraph.handle, genes.ctypes.data_as(C.c_void_p) if genes.size else None, genes.size,
            t.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p), C.byref(auc)))
        assert np.concatenate([t, p]).tolist() == c["scores"] and auc.value == c["auc"]
        assert ex.precision_at_test_count(t, p, split.test_edges, split.probe_nonedges) == c["precision"]


def test_cli_run_writes_the_reference_bytes(ex, tmp_path, capsys):
    c = GOLDEN["experiments"][3]
    cfg = dict(c["config"], output=str(tmp_path / "out.csv"))
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    assert ex.main(["run", str(path)]) == 0
    out = capsys.readouterr().out
    assert out.startswith("task") and out.rstrip().endswith("rows written to " + cfg["output"])
    assert ex.csv_without_wall_time(open(cfg["output"]).read()) == c["csv_without_wall_time"]
