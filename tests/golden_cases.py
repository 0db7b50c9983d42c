"""Golden-vector checks shared by the CPU suite (oracle) and the GPU suite (CUDA path).

An *impl* is a small adaptor exposing the same operations over either the C oracle
(oracle/bindings.py) or the CUDA path (paper_2412_20980_b200); every check compares it
with tests/golden/*.json, which were produced by the unmodified reference
(tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TASK_PC, TASK_MCN, TASK_CDA, TASK_LPA = 0, 1, 2, 3
TASK_SIXDST, TASK_CDA_ADD = 4, 5  # sixdst_fitness(SixDegrees); cda_fitness over the EdgeAddition pool


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def i32(x, cols=None):
    a = np.asarray(x, dtype=np.int32)
    if cols is not None and a.size == 0:
        a = a.reshape(-1, cols)
    return a


class OracleImpl:
    """Adaptor over oracle.bindings.Oracle."""

    def __init__(self, oracle):
        self.o = oracle

    def stream_u64(self, *a): return self.o.stream_u64(*a)
    def init_population(self, *a): return self.o.init_population(*a)
    def init_population_block(self, *a): return self.o.init_population_block(*a)
    def selection_weights(self, f, minimize): return self.o.selection_weights(f, minimize)
    def roulette_pick(self, f, minimize, seed, gen): return self.o.roulette_pick(f, minimize, seed, gen)
    def crossover(self, pop, idx, pc, seed, gen): return self.o.crossover(pop, idx, pc, seed, gen)
    def mutate_block(self, b, off, pm, pool, seed, gen): return self.o.mutate_block(b, off, pm, pool, seed, gen)
    def elitism(self, pop, mp, f, fm, minimize): return self.o.elitism(pop, mp, f, fm, minimize)
    def eda_sample(self, e, ec, pool, seed, gen, sm): return self.o.eda_sample(e, ec, pool, seed, gen, sm)
    def partition_rows(self, s, pn): return self.o.partition_rows(s, pn)
    def graph(self, n, edges): return self.o.graph_from_edges(n, edges)
    def graph_named(self, kind, *a): return getattr(self.o, "graph_" + kind)(*a)
    def edges_of(self, g): return g.edges
    def split(self, g, frac, seed):
        s = self.o.split_build(g, frac, seed)
        return s, s.test, s.probe, s.train.edges
    def addition_pool(self, g): return np.stack(self.o.addition_pool(g), 1)
    def eval(self, ctx, task, genes):
        if task == TASK_CDA_ADD:
            self.o.addition_pool(ctx)
        return self.o.eval_batch(ctx, task, genes)
    def run(self, ctx, task, c):
        if task == TASK_CDA_ADD:
            self.o.addition_pool(ctx)
        r = self.o.run_ga(ctx, task, c["pc"], c["pm"], c["pop_size"], c["budget"], c["iterations"], c["seed"],
                          eda_interval=c["eda_interval"], threads=8)
        return r["best"], r["mean"], r["population"], r["fitness"]


class CudaImpl:
    """Adaptor over the product package (through the C ABI)."""

    def __init__(self, gp):
        self.gp = gp
        self.D = lambda minimize: gp.Direction.Minimize if minimize else gp.Direction.Maximize

    def stream_u64(self, seed, gen, role, row, count): return self.gp.rng_draws(seed, gen, role, row, count)
    def init_population(self, *a): return self.gp.init_population(*a)
    def init_population_block(self, *a): return self.gp.init_population_block(*a)
    def selection_weights(self, f, minimize): return self.gp.selection_weights(f, self.D(minimize))
    def roulette_pick(self, f, minimize, seed, gen): return self.gp.roulette_pick(f, self.D(minimize), seed, gen)
    def crossover(self, pop, idx, pc, seed, gen): return self.gp.crossover(pop, i32(pop)[i32(idx)], pc, seed, gen)
    def mutate_block(self, b, off, pm, pool, seed, gen): return self.gp.mutate_block(b, off, pm, pool, seed, gen)
    def elitism(self, pop, mp, f, fm, minimize): return self.gp.elitism(pop, mp, f, fm, self.D(minimize))
    def eda_sample(self, e, ec, pool, seed, gen, sm): return self.gp.eda_sample(e, ec, pool, seed, gen, sm)
    def partition_rows(self, s, pn): return self.gp.partition_rows(s, pn)
    def graph(self, n, edges): return self.gp.Graph(n, edges)
    def graph_named(self, kind, *a):
        return {"ba": self.gp.barabasi_albert, "er": self.gp.erdos_renyi, "sbm": self.gp.planted_partition}[kind](*a)
    def edges_of(self, g): return g.edges()
    def split(self, g, frac, seed):
        s = self.gp.build_lp_split(g, frac, seed)
        return s, s.test_edges, s.probe_nonedges, s.train.edges()
    def objective(self, ctx, task):
        gp = self.gp
        if task == TASK_LPA:
            return gp.LinkPredictionAttackObjective(ctx, gp.build_gene_pool(ctx.train, gp.PoolKind.EdgeRemoval))
        if task == TASK_CDA:
            return gp.ModularityAttackObjective(ctx, gp.build_gene_pool(ctx, gp.PoolKind.EdgeRemoval))
        if task == TASK_CDA_ADD:
            return gp.ModularityAttackObjective(ctx, gp.build_gene_pool(ctx, gp.PoolKind.EdgeAddition))
        if task == TASK_SIXDST:
            return gp.SixDstObjective(ctx, gp.build_gene_pool(ctx, gp.PoolKind.NodeRemoval), policy=gp.ClosurePolicy.SixDegrees)
        cls = gp.PairwiseConnectivityObjective if task == TASK_PC else gp.SixDstObjective
        return cls(ctx, gp.build_gene_pool(ctx, gp.PoolKind.NodeRemoval))
    def addition_pool(self, g):
        p = self.gp.build_gene_pool(g, self.gp.PoolKind.EdgeAddition)
        return np.stack([p.u, p.v], 1)
    def eval(self, ctx, task, genes): return self.objective(ctx, task).evaluate_batch(genes)
    def run(self, ctx, task, c):
        obj = self.objective(ctx, task)
        p = self.gp.GAParams(pc=c["pc"], pm=c["pm"], pop_size=c["pop_size"], budget=c["budget"],
                             iterations=c["iterations"], seed=c["seed"], eda_interval=c["eda_interval"] or None)
        r = self.gp.run_ga(p, obj.pool, obj)
        return r.history_best, r.history_mean, r.final_population, r.final_fitness


# ------------------------------------------------------------------------------ checks
def check_rng_and_init(impl):
    g = load("ops.json")
    for c in g["streams"]:
        got = impl.stream_u64(c["seed"], c["generation"], c["role"], c["row"], 8)
        assert [int(x) for x in got] == c["u64"]
    for c in g["init"]:
        m = impl.init_population(c["pool"], c["s"], c["k"], c["seed"], c["generation"])
        assert sha(m) == c["sha"] and m[0][:16].tolist() == c["row0"]
        assert sha(impl.init_population_block(c["pool"], 1, 3, c["k"], c["seed"], c["generation"])) == c["block_1_3_sha"]


def check_selection(impl):
    for c in load("ops.json")["selection"]:
        f = np.array(c["fitness"])
        assert impl.selection_weights(f, c["minimize"]).tolist() == c["weights"]
        assert impl.roulette_pick(f, c["minimize"], c["seed"], c["generation"]).tolist() == c["partner_index"]


def check_variation(impl):
    for c in load("ops.json")["variation"]:
        pop = i32(c["pop"])
        crossed = impl.crossover(pop, c["partner_index"], c["pc"], c["seed"], c["generation"])
        assert crossed.tolist() == c["crossed"]
        mutated = impl.mutate_block(crossed, 0, c["pm"], c["pool"], c["seed"], c["generation"])
        assert mutated.tolist() == c["mutated"]
        assert impl.mutate_block(crossed[2:5], 2, c["pm"], c["pool"], c["seed"], c["generation"]).tolist() == c["mutated"][2:5]


def check_elitism_eda_partition(impl):
    g = load("ops.json")
    for c in g["elitism"]:
        nxt, nf = impl.elitism(i32(c["pop"]), i32(c["m_pop"]), c["fit"], c["fit_m"], c["minimize"])
        assert nxt.tolist() == c["next"] and nf.tolist() == c["next_fit"]
    for c in g["eda"]:
        out = impl.eda_sample(i32(c["elite"]), c["elite_count"], c["pool"], c["seed"], c["generation"], c["smoothing"])
        assert out.tolist() == c["out"]
    for c in g["partition_rows"]:
        assert [list(b) for b in impl.partition_rows(c["s"], c["pn"])] == c["blocks"]


def check_generators(impl):
    for name, c in load("fitness.json")["graphs"].items():
        kind, *args = name.split("_")
        args = [float(a) if "." in a else int(a) for a in args]
        g = impl.graph_named(kind, *args)
        e = np.asarray(impl.edges_of(g), dtype=np.int32)
        assert len(e) == c["m"] and sha(e) == c["sha"] and e[:6].tolist() == c["first"], name


def check_pc_mcn(impl):
    g = load("fitness.json")
    for c in g["pc_mcn"]:
        ctx = impl.graph(c["n"], i32(c["edges"], 2))
        genes = i32(c["genes"]).reshape(3, -1)
        assert impl.eval(ctx, TASK_PC, genes).tolist() == c["pc"]
        assert impl.eval(ctx, TASK_MCN, genes).tolist() == c["mcn"]
    ctx = impl.graph_named("ba", 1000, 2, 1)
    pop = impl.init_population(1000, 4, 50, 1)
    assert impl.eval(ctx, TASK_PC, pop).tolist() == g["config1"]["pc"]
    assert impl.eval(ctx, TASK_MCN, pop).tolist() == g["config1"]["mcn"]
    ctx = impl.graph_named("ba", 3000, 5, 7)
    pop = impl.init_population(3000, 70, 150, 2)
    assert impl.eval(ctx, TASK_PC, pop).tolist() == g["ba_3000"]["pc"]
    assert impl.eval(ctx, TASK_MCN, pop[:6]).tolist() == g["ba_3000"]["mcn"]


def check_cda(impl):
    g = load("fitness.json")
    for c in g["cda"] + [g["karate"]]:
        ctx = impl.graph(c["n"], i32(c["edges"], 2))
        genes = i32(c["genes"])
        genes = genes.reshape(len(c["q"]), -1)
        assert impl.eval(ctx, TASK_CDA, genes).tolist() == c["q"]
        assert impl.eval(ctx, TASK_CDA, np.zeros((1, 0), np.int32)).tolist() == [c["q0"]]  # empty == unattacked, exactly
    ctx = impl.graph_named("sbm", 10, 50, 0.2, 0.01, 1)
    pop = impl.init_population(len(impl.edges_of(ctx)), 3, g["cda_kat"]["k"], 1)
    assert impl.eval(ctx, TASK_CDA, pop).tolist() == g["cda_kat"]["q"]


def check_lpa(impl):
    g = load("fitness.json")
    for c in g["lpa"]:
        full = impl.graph(c["n"], i32(c["edges"], 2))
        split, test, probe, train_edges = impl.split(full, c["fraction"], c["split_seed"])
        assert np.asarray(test).tolist() == c["test"] and np.asarray(probe).tolist() == c["probe"]
        assert sha(np.asarray(train_edges, dtype=np.int32)) == c["train_sha"]
        assert impl.eval(split, TASK_LPA, i32(c["genes"])).tolist() == c["auc"]
        assert impl.eval(split, TASK_LPA, np.zeros((1, 0), np.int32)).tolist() == [c["auc0"]]
    full = impl.graph_named("er", 500, 0.03, 1)
    split, test, _, train_edges = impl.split(full, 0.1, 1)
    k = g["lpa_kat"]
    assert (len(test), len(train_edges)) == (k["T"], k["train_m"])
    assert impl.eval(split, TASK_LPA, impl.init_population(k["train_m"], 3, k["k"], 1)).tolist() == k["auc"]


def check_sixdegrees(impl):
    """sixdst_fitness(SixDegrees): largest radius-8 ball (fitness.cpp:18-26, accessibility.cpp:20-37)."""
    g = load("widen.json")
    for c in g["sixdst"]:
        ctx = impl.graph(c["n"], i32(c["edges"], 2))
        genes = i32(c["genes"]).reshape(3, -1)
        assert impl.eval(ctx, TASK_SIXDST, genes).tolist() == c["six"]
        assert impl.eval(ctx, TASK_MCN, genes).tolist() == c["mcn"]
    assert g["sixdst"][0]["six"] == [17.0] * 3 and g["sixdst"][0]["mcn"] == [40.0] * 3  # P40: 8 each side + self
    ctx = impl.graph_named("ba", 1000, 2, 1)
    assert impl.eval(ctx, TASK_SIXDST, impl.init_population(1000, 4, 50, 1)).tolist() == g["sixdst_config1"]


def check_cda_add(impl):
    """cda_fitness over EdgeAddition pools (gene_pool.cpp:57-60, :81-87)."""
    g = load("widen.json")
    for c in g["cda_add"]:
        ctx = impl.graph(c["n"], i32(c["edges"], 2))
        pool = impl.addition_pool(ctx)
        assert len(pool) == c["pool_size"] and sha(np.asarray(pool, dtype=np.int32)) == c["pool_sha"]
        genes = i32(c["genes"]).reshape(3, -1)
        assert impl.eval(ctx, TASK_CDA_ADD, genes).tolist() == c["q"]
    k = load("fitness.json")["karate"]
    ctx = impl.graph(k["n"], i32(k["edges"], 2))
    ka = g["karate_add"]
    pool = impl.addition_pool(ctx)
    assert len(pool) == ka["pool_size"] and np.asarray(pool)[:6].tolist() == ka["pool_first"]
    assert impl.eval(ctx, TASK_CDA_ADD, i32(ka["genes"])).tolist() == ka["q"]
    assert impl.eval(ctx, TASK_CDA_ADD, np.zeros((1, 0), np.int32)).tolist() == [k["q0"]]


def _run_ctx(impl, name):
    if name == "config1_pc_ba1000":
        return impl.graph_named("ba", 1000, 2, 1)
    if name in ("acceptance6_sixdst_er100", "pc_er100_eda3"):
        return impl.graph_named("er", 100, 0.04, 665)
    if name == "acceptance10_lpa_sbm64":
        return impl.split(impl.graph_named("sbm", 4, 16, 0.28, 0.02, 671), 0.1, 672)[0]
    if name == "cda_sbm80":
        return impl.graph_named("sbm", 4, 20, 0.3, 0.03, 1)
    if name == "sixdegrees_ba300":
        return impl.graph_named("ba", 300, 1, 668)
    if name in ("cda_karate", "acceptance8_cda_add_karate"):
        k = load("fitness.json")["karate"]
        return impl.graph(k["n"], i32(k["edges"], 2))
    raise KeyError(name)


def check_run(impl, name):
    c = load("runs_widen.json" if name in WIDE_RUN_NAMES else "runs.json")[name]
    best, mean, pop, fit = impl.run(_run_ctx(impl, name), c["task"], c)
    assert np.asarray(best).tolist() == c["best"]
    assert np.asarray(mean).tolist() == c["mean"]          # sequential-sum mean, bit for bit
    assert np.asarray(fit).tolist() == c["final_fitness"]
    assert sha(np.asarray(pop, dtype=np.int32)) == c["final_population_sha"]
    assert np.asarray(pop)[0].tolist() == c["best_individual"]


WIDE_RUN_NAMES = ["acceptance8_cda_add_karate", "sixdegrees_ba300"]
RUN_NAMES = ["config1_pc_ba1000", "acceptance6_sixdst_er100", "pc_er100_eda3", "acceptance10_lpa_sbm64", "cda_sbm80",
             "cda_karate"] + WIDE_RUN_NAMES
