"""Generates tests/golden/*.json from the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference/proj by oracle/Makefile).  Run in the authoring container only:

    python tests/golden/make_golden.py

The JSON files are committed; nothing in tests/ or bench.py reads /root/reference at run
time.  Doubles are stored with repr() and round-trip exactly.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.bindings import (MODE_M, MODE_S, MODE_SERIAL, TASK_CDA, TASK_CDA_ADD, TASK_LPA, TASK_MCN, TASK_PC, TASK_SIXDST,
                             Ref)  # noqa: E402

r = Ref()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=None, separators=(",", ":"))
    print(name, os.path.getsize(os.path.join(HERE, name)), "bytes")


def ints(a):
    return np.asarray(a).astype(np.int64).tolist()


def floats(a):
    return [float(x) for x in np.asarray(a, dtype=np.float64)]


# ------------------------------------------------------------------ rng + operators
rng_cases = []
for seed, gen, role, row in [(1, 0, 1, 0), (1, 3, 4, 7), (2**63 + 5, 100, 2, 4095), (0, 0, 5, 0), (20240601, 50, 3, 19)]:
    rng_cases.append({
        "seed": seed, "generation": gen, "role": role, "row": row,
        "u64": [int(x) for x in r.stream_u64(seed, gen, role, row, 8)],
        "unit": floats(r.stream_unit(seed, gen, role, row, 8)),
        "index_1000": ints(r.stream_index(seed, gen, role, row, 1000, 8)),
        "index_big": ints(r.stream_index(seed, gen, role, row, 4_000_000_000, 8)),
    })
ops = {"mix64": {str(x): r.mix64(x) for x in (0, 1, 2**64 - 1, 0x9E3779B97F4A7C15)}, "streams": rng_cases}

gen = np.random.default_rng(12345)
ops["init"] = []
for pool, s, k, seed, g_ in [(1000, 4, 6, 1, 0), (1000, 100, 50, 1, 0), (7, 33, 1, 9, 0), (2_000_000_000, 5, 300, 3, 4)]:
    m = r.init_population(pool, s, k, seed, g_)
    ops["init"].append({"pool": pool, "s": s, "k": k, "seed": seed, "generation": g_, "sha": sha(m),
                        "row0": ints(m[0][:16]), "block_1_3_sha": sha(r.init_population_block(pool, 1, 3, k, seed, g_))})

ops["selection"] = []
for s, ties, minimize in [(4, True, True), (4, True, False), (100, False, True), (257, True, True), (257, True, False), (1000, False, False)]:
    f = gen.integers(0, 20, s).astype(float) if ties else gen.random(s)
    if s == 4:
        f = np.array([5.0, 3.0, 3.0, 9.0])
    pop = gen.integers(0, 50, (s, 3)).astype(np.int32)
    idx, partners = r.roulette_select(pop, f, minimize, 5, s)
    assert np.array_equal(pop[idx], partners)
    ops["selection"].append({"fitness": floats(f), "minimize": minimize, "seed": 5, "generation": s,
                             "weights": floats(r.selection_weights(f, minimize)), "partner_index": ints(idx)})

ops["variation"] = []
for s, k, pool, pc, pm in [(12, 7, 1000, 0.6, 0.2), (5, 40, 9, 0.0, 1.0), (5, 40, 9, 1.0, 0.0), (30, 11, 2**31 - 1, 0.8, 0.1)]:
    pop = gen.integers(0, pool, (s, k)).astype(np.int32)
    f = gen.random(s)
    idx, partners = r.roulette_select(pop, f, True, 3, 17)
    crossed = r.crossover(pop, partners, pc, 3, 17)
    mutated = r.mutate(crossed, pm, pool, 3, 17)
    assert np.array_equal(mutated[2:5], r.mutate_block(crossed[2:5], 2, pm, pool, 3, 17))
    ops["variation"].append({"pop": ints(pop), "partner_index": ints(idx), "pool": pool, "pc": pc, "pm": pm, "seed": 3,
                             "generation": 17, "crossed": ints(crossed), "mutated": ints(mutated)})

ops["elitism"] = []
for s, k, minimize in [(4, 2, True), (4, 2, False), (37, 3, True), (64, 1, False)]:
    pop, mp = gen.integers(0, 50, (s, k)).astype(np.int32), gen.integers(0, 50, (s, k)).astype(np.int32)
    f, fm = gen.integers(0, 6, s).astype(float), gen.integers(0, 6, s).astype(float)
    nxt, nf = r.elitism(pop, mp, f, fm, minimize)
    ops["elitism"].append({"pop": ints(pop), "m_pop": ints(mp), "fit": floats(f), "fit_m": floats(fm), "minimize": minimize,
                           "next": ints(nxt), "next_fit": floats(nf)})

ops["eda"] = []
for ec, smooth in [(30, True), (5, True), (30, False)]:
    elite = gen.integers(0, 40, (30, 12)).astype(np.int32)
    ops["eda"].append({"elite": ints(elite), "elite_count": ec, "pool": 40, "seed": 4, "generation": 6, "smoothing": smooth,
                       "out": ints(r.eda_sample(elite, ec, 40, 4, 6, smooth))})
ops["partition_rows"] = [{"s": s, "pn": pn, "blocks": r.partition_rows(s, pn)} for s, pn in [(10, 3), (4096, 8), (7, 8), (100, 1), (5, 2)]]
dump("ops.json", ops)

# ------------------------------------------------------------------ graphs + fitness
fit = {"graphs": {}, "pc_mcn": [], "cda": [], "lpa": []}
for name, g in [("ba_1000_2_1", r.graph_ba(1000, 2, 1)), ("er_500_0.03_1", r.graph_er(500, 0.03, 1)),
                ("sbm_10_50_0.2_0.01_1", r.graph_sbm(10, 50, 0.2, 0.01, 1)), ("ba_3000_5_7", r.graph_ba(3000, 5, 7)),
                ("er_100_0.04_665", r.graph_er(100, 0.04, 665)), ("sbm_4_16_0.28_0.02_671", r.graph_sbm(4, 16, 0.28, 0.02, 671))]:
    e = r.graph_edges(g)
    fit["graphs"][name] = {"n": r.graph_n(g), "m": r.graph_m(g), "sha": sha(e), "first": ints(e[:6])}

# acceptance #3 style: random graphs x individuals, PC and MCN (exact)
for trial in range(40):
    n = int(gen.integers(4, 70))
    dens = float(gen.uniform(0.02, 0.4))
    iu = np.triu_indices(n, 1)
    keep = gen.random(len(iu[0])) < dens
    edges = np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.int32)
    g = r.graph_from_edges(n, edges)
    k = int(gen.integers(0, n + 1))
    batch = gen.integers(0, n, (3, k)).astype(np.int32)
    fit["pc_mcn"].append({"n": n, "edges": ints(edges), "genes": ints(batch),
                          "pc": floats(r.eval_batch(g, TASK_PC, batch)), "mcn": floats(r.eval_batch(g, TASK_MCN, batch))})
g = r.graph_ba(1000, 2, 1)
pop = r.init_population(1000, 4, 50, 1)
fit["config1"] = {"pc": floats(r.eval_batch(g, TASK_PC, pop)), "mcn": floats(r.eval_batch(g, TASK_MCN, pop))}
g = r.graph_ba(3000, 5, 7)
pop = r.init_population(3000, 70, 150, 2)
fit["ba_3000"] = {"pc": floats(r.eval_batch(g, TASK_PC, pop, threads=8)), "mcn": floats(r.eval_batch(g, TASK_MCN, pop[:6], threads=6))}

# CDA: small graphs (edges inline) + the SURVEY KAT instance
for trial in range(14):
    kind = trial % 3
    n = int(gen.integers(6, 60))
    if kind == 0:
        g = r.graph_er(n, float(gen.uniform(0.05, 0.35)), 100 + trial)
    elif kind == 1:
        g = r.graph_ba(n, int(gen.integers(1, 4)), 100 + trial)
    else:
        g = r.graph_sbm(int(gen.integers(2, 5)), int(gen.integers(4, 14)), 0.5, 0.04, 100 + trial)
    m = r.graph_m(g)
    if m == 0:
        continue
    k = int(gen.integers(0, m + 1))
    batch = gen.integers(0, m, (3, k)).astype(np.int32)
    fit["cda"].append({"n": r.graph_n(g), "edges": ints(r.graph_edges(g)), "genes": ints(batch),
                       "q": floats(r.eval_batch(g, TASK_CDA, batch)), "q0": r.modularity_unattacked(g),
                       "communities": ints(r.detect_communities(g))})
g = r.graph_sbm(10, 50, 0.2, 0.01, 1)
k = r.budget(g, 0, 0.05)
pop = r.init_population(r.graph_m(g), 3, k, 1)
fit["cda_kat"] = {"k": k, "q": floats(r.eval_batch(g, TASK_CDA, pop)), "q0": r.modularity_unattacked(g)}
kar = r.graph_load("/root/reference/proj/data/karate.txt")
fit["karate"] = {"n": r.graph_n(kar), "edges": ints(r.graph_edges(kar)), "q0": r.modularity_unattacked(kar),
                 "communities": ints(r.detect_communities(kar))}
pop = r.init_population(r.graph_m(kar), 5, 8, 11)
fit["karate"]["genes"] = ints(pop)
fit["karate"]["q"] = floats(r.eval_batch(kar, TASK_CDA, pop))

# LPA
for trial, (gname, g) in enumerate([("er", r.graph_er(120, 0.08, 2)), ("ba", r.graph_ba(150, 3, 4)),
                                    ("sbm", r.graph_sbm(4, 16, 0.28, 0.02, 671))]):
    frac, sseed = [0.2, 0.1, 0.1][trial], [5, 6, 672][trial]
    sp = r.split_build(g, frac, sseed)
    test, probe = r.split_pairs(sp)
    train = r.split_train(sp)
    mt = r.graph_m(train)
    k = r.budget(train, 0, 0.1)
    batch = r.init_population(mt, 4, k, 3)
    fit["lpa"].append({"n": r.graph_n(g), "edges": ints(r.graph_edges(g)), "fraction": frac, "split_seed": sseed,
                       "test": ints(test), "probe": ints(probe), "train_sha": sha(r.graph_edges(train)), "genes": ints(batch),
                       "auc": floats(r.eval_batch(sp, TASK_LPA, batch)), "auc0": r.auc_unattacked(sp),
                       "ra_first_test": [r.ra_score(train, int(u), int(v)) for u, v in test[:5]]})
g = r.graph_er(500, 0.03, 1)
sp = r.split_build(g, 0.1, 1)
train = r.split_train(sp)
k = r.budget(train, 0, 0.1)
pop = r.init_population(r.graph_m(train), 3, k, 1)
fit["lpa_kat"] = {"T": len(r.split_pairs(sp)[0]), "train_m": r.graph_m(train), "k": k,
                  "auc": floats(r.eval_batch(sp, TASK_LPA, pop)), "auc0": r.auc_unattacked(sp)}
dump("fitness.json", fit)

# ------------------------------------------------------------------ trajectories
runs = {}


def run_case(name, ctx, task, pc, pm, s, k, iters, seed, eda=0, modes=((MODE_S, 1, 1),)):
    base = r.run_ga(ctx, task, pc, pm, s, k, iters, seed, eda, MODE_SERIAL)
    for mode, pn, qn in modes:  # every topology reproduces the serial run bit for bit
        other = r.run_ga(ctx, task, pc, pm, s, k, iters, seed, eda, mode, pn, qn)
        assert np.array_equal(base["best"], other["best"]) and np.array_equal(base["mean"], other["mean"])
        assert np.array_equal(base["population"], other["population"])
    runs[name] = {"task": task, "pc": pc, "pm": pm, "pop_size": s, "budget": k, "iterations": iters, "seed": seed,
                  "eda_interval": eda, "best": floats(base["best"]), "mean": floats(base["mean"]),
                  "final_fitness": floats(base["fitness"]), "final_population_sha": sha(base["population"]),
                  "best_individual": ints(base["population"][0])}


run_case("config1_pc_ba1000", r.graph_ba(1000, 2, 1), TASK_PC, 0.6, 0.2, 100, 50, 100, 1, modes=((MODE_S, 1, 1), (MODE_M, 8, 1)))
run_case("acceptance6_sixdst_er100", r.graph_er(100, 0.04, 665), TASK_MCN, 0.5, 0.3, 20, 10, 50, 20240601, modes=((MODE_S, 1, 1), (MODE_M, 2, 1)))
run_case("pc_er100_eda3", r.graph_er(100, 0.04, 665), TASK_PC, 0.8, 0.1, 30, 8, 25, 4, eda=3)
g = r.graph_sbm(4, 16, 0.28, 0.02, 671)
sp = r.split_build(g, 0.1, 672)
k = r.budget(r.split_train(sp), 0, 0.1)
run_case("acceptance10_lpa_sbm64", sp, TASK_LPA, 0.7, 0.1, 50, k, 200, 673)
runs["acceptance10_lpa_sbm64"]["auc0"] = r.auc_unattacked(sp)
run_case("cda_sbm80", r.graph_sbm(4, 20, 0.3, 0.03, 1), TASK_CDA, 0.8, 0.1, 16, 10, 12, 2)
run_case("cda_karate", kar, TASK_CDA, 0.8, 0.1, 20, 4, 30, 7)
dump("runs.json", runs)
print("acceptance #6 final MCN", runs["acceptance6_sixdst_er100"]["best"][-1], "(reference test_output.txt:50 says 81)")
print("acceptance #10 AUC", runs["acceptance10_lpa_sbm64"]["auc0"], "->", runs["acceptance10_lpa_sbm64"]["best"][-1])
print("config 1 best", runs["config1_pc_ba1000"]["best"][0], "->", runs["config1_pc_ba1000"]["best"][-1])


# ------------------------------------------------------------------ truncated closure, edge addition
# (own generator so that the files above stay byte-identical when this section grows)
gen2 = np.random.default_rng(777)
wide = {"sixdst": [], "cda_add": []}
path40 = np.stack([np.arange(39), np.arange(1, 40)], 1).astype(np.int32)  # test_fitness.cpp:94-103
for trial in range(16):
    if trial == 0:
        n, edges = 40, path40
    else:
        n = int(gen2.integers(10, 150))
        iu = np.triu_indices(n, 1)
        keep = gen2.random(len(iu[0])) < float(gen2.uniform(0.6, 2.2)) / n
        edges = np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.int32)
        if trial % 4 == 1:  # a long path through everything plus the random chords: large diameter
            chain = np.stack([np.arange(n - 1), np.arange(1, n)], 1).astype(np.int32)
            edges = np.unique(np.concatenate([edges, chain]), axis=0)
    g = r.graph_from_edges(n, edges)
    k = 0 if trial == 0 else int(gen2.integers(0, n // 5 + 1))
    batch = gen2.integers(0, n, (3, k)).astype(np.int32)
    wide["sixdst"].append({"n": n, "edges": ints(edges), "genes": ints(batch),
                           "six": floats(r.eval_batch(g, TASK_SIXDST, batch)), "mcn": floats(r.eval_batch(g, TASK_MCN, batch))})
g = r.graph_ba(1000, 2, 1)
pop = r.init_population(1000, 4, 50, 1)
wide["sixdst_config1"] = floats(r.eval_batch(g, TASK_SIXDST, pop))

for trial in range(12):
    n = int(gen2.integers(5, 60))
    iu = np.triu_indices(n, 1)
    keep = gen2.random(len(iu[0])) < (0.0 if trial == 0 else float(gen2.uniform(0.03, 0.3)))
    edges = np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.int32)
    g = r.graph_from_edges(n, edges)
    pu, pv = r.pool_genes(g, 1)
    k = int(gen2.integers(0, 30))
    batch = gen2.integers(0, len(pu), (3, k)).astype(np.int32)
    if k > 2:
        batch[1, 2] = batch[1, 0]
    wide["cda_add"].append({"n": n, "edges": ints(edges), "pool_size": len(pu), "pool_sha": sha(np.stack([pu, pv], 1)),
                            "genes": ints(batch), "q": floats(r.eval_batch(g, TASK_CDA_ADD, batch))})
pu, pv = r.pool_genes(kar, 1)
pop = r.init_population(len(pu), 5, 8, 11)
wide["karate_add"] = {"pool_size": len(pu), "pool_first": ints(np.stack([pu, pv], 1)[:6]), "genes": ints(pop),
                      "q": floats(r.eval_batch(kar, TASK_CDA_ADD, pop))}
dump("widen.json", wide)

runs = {}
# acceptance #8 (acceptance.cpp:207-246): karate, QAttack defaults over the EdgeAddition pool, 300 iterations
run_case("acceptance8_cda_add_karate", kar, TASK_CDA_ADD, 0.8, 0.1, 100, r.budget(kar, 1, 0.1), 300, 667)
runs["acceptance8_cda_add_karate"]["q0"] = r.modularity_unattacked(kar)
run_case("sixdegrees_ba300", r.graph_ba(300, 1, 668), TASK_SIXDST, 0.5, 0.3, 24, r.budget(r.graph_ba(300, 1, 668), 2, 0.1), 30, 670,
         modes=((MODE_S, 1, 1), (MODE_M, 3, 1)))
dump("runs_widen.json", runs)
print("acceptance #8 Q", runs["acceptance8_cda_add_karate"]["q0"], "->", runs["acceptance8_cda_add_karate"]["best"][-1],
      "(reference test_output.txt:52 says 0.380671 -> 0.26156 @300)")


# ------------------------------------------------------------------ loaders, reporting metrics, experiment CSV
# Datasets are written here (committed under tests/golden/datasets/) and read back by the reference's own
# load_edge_list_file / run_experiment, so the golden CSV rows and the files always belong together.
DS = os.path.join(HERE, "datasets")
os.makedirs(DS, exist_ok=True)
gen3 = np.random.default_rng(4242)


def write_edge_list(name, n, edges, label=lambda i: str(i), noise=False):
    lines = ["# synthetic dataset for tests/golden/experiments.json (tests/golden/make_golden.py)", ""]
    order = gen3.permutation(len(edges))
    for idx, e in enumerate(order):
        u, v = (int(x) for x in edges[e])
        if gen3.random() < 0.5:
            u, v = v, u
        lines.append(f"{label(u)}\t{label(v)}" if idx % 3 else f"  {label(u)} {label(v)}  ")
        if noise and idx == 5:
            lines += ["% comment in the other style", f"{label(u)} {label(u)}", f"{label(v)} {label(u)}", "   "]
    with open(os.path.join(DS, name), "w") as f:
        f.write("\n".join(lines) + "\n")


kar_edges = np.asarray(fit["karate"]["edges"], dtype=np.int32)
write_edge_list("karate.txt", 34, kar_edges, label=lambda i: str(i + 1))
sbm_g = r.graph_sbm(4, 15, 0.35, 0.03, 9)
sbm_edges = r.graph_edges(sbm_g)
write_edge_list("sbm60.txt", 60, sbm_edges, label=lambda i: f"n{i:02d}", noise=True)
with open(os.path.join(DS, "sbm60_truth.txt"), "w") as f:
    f.write("# label community\n" + "".join(f"n{i:02d} block{i // 15}\n" for i in gen3.permutation(60)))
tree_edges = r.graph_edges(r.graph_ba(120, 1, 31))
write_edge_list("tree120.txt", 120, tree_edges)
er_edges = r.graph_edges(r.graph_er(90, 0.09, 17))
write_edge_list("er90.txt", 90, er_edges, label=lambda i: f"v{i}")

rel = lambda name: "tests/golden/datasets/" + name  # configs use repo-relative paths: run from the repo root
os.chdir(os.path.dirname(os.path.dirname(HERE)))
experiments = []
for cfg, axis, values in [
    ({"algorithm": "qattack", "dataset": rel("karate.txt"), "iterations": 40, "pop_size": 20, "seed": 667, "repetitions": 2}, "", ()),
    ({"algorithm": "cda-eda", "dataset": rel("karate.txt"), "iterations": 12, "pop_size": 16, "seed": 5, "eda_interval": 3}, "", ()),
    ({"task": "cda-modularity", "pool": "edge-removal", "dataset": rel("sbm60.txt"), "ground_truth": rel("sbm60_truth.txt"),
      "pc": 0.8, "pm": 0.1, "iterations": 10, "pop_size": 12, "seed": 3, "perturbation_rate": 0.15}, "", ()),
    ({"algorithm": "cutoff-pc", "dataset": rel("tree120.txt"), "iterations": 30, "pop_size": 16, "seed": 11, "mode": "m", "pn": 2}, "", ()),
    ({"algorithm": "sixdst", "dataset": rel("tree120.txt"), "iterations": 25, "pop_size": 14, "seed": 12, "fast_closure": True,
      "perturbation_rate": 0.05}, "", ()),
    ({"algorithm": "sixdst", "dataset": rel("er90.txt"), "iterations": 20, "pop_size": 10, "seed": 13}, "", ()),
    ({"algorithm": "lpa-ga", "dataset": rel("sbm60.txt"), "iterations": 20, "pop_size": 12, "seed": 21, "repetitions": 2,
      "test_fraction": 0.2}, "", ()),
    ({"algorithm": "lpa-eda", "dataset": rel("er90.txt"), "iterations": 8, "pop_size": 10, "seed": 22}, "", ()),
    ({"task": "cnd-pc", "dataset": rel("er90.txt"), "pc": 0.6, "pm": 0.2, "iterations": 10, "seed": 30}, "pop_size", (8, 12)),
]:
    csv = r.run_experiment(json.dumps(cfg), axis, list(values))
    experiments.append({"config": cfg, "axis": axis, "values": list(values), "csv": csv,
                        "csv_without_wall_time": r.csv_without_wall_time(csv)})
    print(csv.splitlines()[1][:150])

metrics = {"nmi": [], "lp": [], "detect": []}
for trial in range(12):
    n = int(gen3.integers(1, 60))
    a, b = gen3.integers(0, int(gen3.integers(1, 8)), n), gen3.integers(0, int(gen3.integers(1, 8)), n)
    if trial == 0:
        b = a.copy()
    if trial == 1:
        a, b = np.zeros(n, int), np.zeros(n, int)
    metrics["nmi"].append({"a": ints(a), "b": ints(b), "nmi": r.nmi(a, b)})
for kind, g, edges in [(0, sbm_g, sbm_edges), (1, sbm_g, sbm_edges), (1, kar, kar_edges)]:
    psize = len(r.pool_genes(g, kind)[0])
    for k in (0, 7, 25):
        genes = gen3.integers(0, psize, k).astype(np.int32)
        metrics["detect"].append({"n": r.graph_n(g), "edges": ints(edges), "kind": kind, "genes": ints(genes),
                                  "assignment": ints(r.detect_perturbed(g, kind, genes))})
for gname, g, frac, sseed in [("sbm", sbm_g, 0.2, 21), ("er", r.graph_er(90, 0.09, 17), 0.1, 22)]:
    sp = r.split_build(g, frac, sseed)
    mt = r.graph_m(r.split_train(sp))
    for k in (0, 9):
        genes = gen3.integers(0, mt, k).astype(np.int32)
        auc, prec, scores = r.lp_metrics(sp, genes)
        metrics["lp"].append({"n": r.graph_n(g), "edges": ints(r.graph_edges(g)), "fraction": frac, "split_seed": sseed,
                              "genes": ints(genes), "auc": auc, "precision": prec, "scores": floats(scores)})
datasets = {}
for name in ("karate.txt", "sbm60.txt", "tree120.txt", "er90.txt"):
    g = r.graph_load(rel(name))
    e = r.graph_edges(g)
    datasets[name] = {"n": r.graph_n(g), "m": r.graph_m(g), "sha": sha(e), "first": ints(e[:5])}
dump("experiments.json", {"experiments": experiments, "metrics": metrics, "datasets": datasets})

# ------------------------------------------------------------------ mask matrices (ga_ops.cpp:84-103)
mask_cases = []
for rows, cols, rate, role, seed, g_ in [(6, 10, 0.6, 3, 1, 1), (100, 50, 0.2, 4, 1, 7), (33, 1, 0.0, 3, 9, 2), (5, 300, 1.0, 4, 3, 4),
                                         (17, 129, 0.37, 3, 2**63 + 5, 100), (40, 64, 1e-3, 4, 5, 12)]:
    a = r.make_mask(rows, cols, rate, role, seed, g_)
    mask_cases.append({"rows": rows, "cols": cols, "rate": rate, "role": role, "seed": seed, "generation": g_, "sha": sha(a),
                       "row0": [int(x) for x in a[0][:24]], "ones": int(a.sum())})
index_cases = []
for rows, cols, pool, seed, g_ in [(6, 10, 1000, 1, 1), (100, 50, 1000, 1, 7), (33, 1, 7, 9, 2), (5, 300, 2_000_000_000, 3, 4)]:
    a = r.make_mutation_indices(rows, cols, pool, seed, g_)
    index_cases.append({"rows": rows, "cols": cols, "pool": pool, "seed": seed, "generation": g_, "sha": sha(a),
                        "row0": [int(x) for x in a[0][:16]]})
dump("masks.json", {"_source": "compiled unmodified reference (oracle/_ref): make_crossover_mask / make_mutation_mask / "
                               "make_mutation_indices, ga_ops.cpp:84-103; generated by tests/golden/make_golden.py (masks section)",
                    "masks": mask_cases, "indices": index_cases})
