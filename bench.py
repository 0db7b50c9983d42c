#!/usr/bin/env python
"""bench.py — the driver's measurement contract for the GAPA hot path on B200.

    python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload c4|c1|...]

A *step* is one generation of the hot path over the whole population:
select -> crossover+mutate -> batched fitness evaluation of M_POP -> elitism
(modes.cpp:159-175), population resident in HBM.  `value` = fitness evaluations per second
of the whole job (all ranks), device-timed with CUDA events on the stream the kernels run
on, max over ranks.  `e2e` = the same metric through the reference-facing plugin call
FitnessFunction::evaluate_batch with HOST buffers (pinned H2D of the gene matrix + kernels
+ D2H of the fitness vector inside the timed region).

Default workload = BASELINE.json configs[3] ("C4"): critical-node detection, pairwise-
connectivity fitness, Barabasi-Albert n = 1,000,000 attach 5 (m = 4,999,985), budget
k = 50,000, population 4096 — the configuration north_star's roofline target is quoted on
and the largest that the metric names; it fits one GPU.  With N > 1 the population is
sharded over ranks (strong scaling: total population fixed) and the only exchange is one
NCCL all-gather of fitness doubles per generation.

`--impl reference` times the reference's CPU path for the same config on the host cores:
the unmodified reference (oracle/_ref) where its dense n x n storage can hold the graph
(n <= 20,000), else the CSR port of the same algorithm (oracle/), on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (task, graph kind, graph args, pool kind, rate, pop, pc, pm, description)
    "c4": dict(task="pc", graph=("ba", 1_000_000, 5, 1), rate=0.05, pop=4096, pc=0.6, pm=0.2,
               name="C4: CND pairwise-connectivity GA, Barabasi-Albert n=1e6 attach=5 (m=4,999,985), k=50,000, pop 4096"),
    "c1": dict(task="pc", graph=("ba", 1000, 2, 1), rate=0.05, pop=100, pc=0.6, pm=0.2,
               name="C1: CND pairwise-connectivity GA, Barabasi-Albert n=1000 attach=2 (m=1997), k=50, pop 100"),
    "c2": dict(task="cda", graph=("sbm", 10, 500, 0.02, 0.0005, 1), rate=0.05, pop=100, pc=0.8, pm=0.1,
               name="C2: CDA modularity GA, SBM 10x500 (m=30,321), 5% edge deletion k=1517, pop 100"),
    "c3": dict(task="lpa", graph=("er", 10_000, 10 / 9999, 1), rate=0.1, pop=50, pc=0.7, pm=0.1,
               name="C3: LPA RA-AUC GA, Erdos-Renyi n=1e4 <d>=10 (m=50,277), 10% hidden, k=4525, pop 50"),
    "n1e5": dict(task="pc", graph=("ba", 100_000, 5, 1), rate=0.05, pop=4096, pc=0.6, pm=0.2,
                 name="C5 point: CND-PC, BA n=1e5 attach=5, k=5000, pop 4096"),
    "n1e4": dict(task="pc", graph=("ba", 10_000, 5, 1), rate=0.05, pop=4096, pc=0.6, pm=0.2,
                 name="C5 point: CND-PC, BA n=1e4 attach=5, k=500, pop 4096"),
    "n5e5": dict(task="pc", graph=("ba", 500_000, 5, 1), rate=0.05, pop=4096, pc=0.6, pm=0.2,
                 name="between the C5 points: CND-PC, BA n=5e5 attach=5, k=25,000, pop 4096"),
}
TASK_ID = {"pc": 0, "mcn": 1, "cda": 2, "lpa": 3}


def algorithmic_bytes(task: str, n: int, m: int, k: int, T: int = 0, P: int = 0, dbar: float = 0.0) -> float:
    """algorithmic bytes per evaluation (int32 indices, FP64 outputs)."""
    if task in ("pc", "mcn"):
        return 4 * (n + 1) + 8 * m + 4 * k + 2 * ((n + 7) // 8) + 8 * n + 8
    if task == "lpa":
        return 4 * k + 2 * ((m + 7) // 8) + 8 * n + (T + P) * (16 + 2 * 8 * dbar) + 8 * (T + P) + 8
    return 4 * (n + 1) + 8 * m + 4 * m + 4 * k + 2 * ((m + 7) // 8) + 16 * m + 8 * n + 8  # cda


def peaks() -> tuple[float, str]:
    """HBM peak in GB/s: the driver-written MEASURED_PEAKS.json (burst figure: the evaluation is timed alone,
    kernel by kernel), else the fallback B200_PROFILING.md states."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            doc = json.load(f)
        flat = {}

        def walk(prefix, node):
            if isinstance(node, dict):
                for k, v in node.items():
                    walk(f"{prefix}.{k}" if prefix else str(k), v)
            elif isinstance(node, (int, float)) and not isinstance(node, bool):
                flat[prefix.lower()] = float(node)

        walk("", doc)
        for want in ("hbm_gbs", "hbm_gbs_burst", "hbm.burst_gbs", "hbm_burst_gbs"):
            if want in flat:
                return flat[want], f"measured (MEASURED_PEAKS.json {want})"
        cands = [(k, v) for k, v in flat.items() if "hbm" in k and 1000.0 < v < 20000.0]
        if cands:
            burst = [kv for kv in cands if "burst" in kv[0]] or [kv for kv in cands if "sustain" not in kv[0]] or cands
            k, v = max(burst, key=lambda kv: kv[1])
            return v, f"measured (MEASURED_PEAKS.json {k})"
    except Exception:
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (B200_PROFILING.md recipe)."""

    def __init__(self, index: int):
        self.rows, self.proc, self.index = [], None, index

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------------- CPU arms
def cpu_reference_throughput(w: dict, target_seconds: float, threads: int) -> dict:
    """evals/s of the reference CPU path on a bounded sample of workload `w` (the checker is the
    thing timed here, and only here)."""
    from oracle.bindings import Oracle, Ref
    o = Oracle()
    kind, *args = w["graph"]
    task = TASK_ID[w["task"]]
    use_ref = Ref.available() and args[0] * (args[1] if kind == "sbm" else 1) <= 20_000
    if use_ref:
        r = Ref()
        g = getattr(r, "graph_" + kind)(*args)
        if task == 3:
            ctx = r.split_build(g, 0.1, 1)
            basis = r.graph_m(r.split_train(ctx))
        else:
            ctx, basis = g, (r.graph_n(g) if task in (0, 1) else r.graph_m(g))
        impl, label = r, "reference"
    else:
        g = getattr(o, "graph_" + kind)(*args)
        if task == 3:
            ctx = o.split_build(g, 0.1, 1)
            basis = ctx.train.m
        else:
            ctx, basis = g, (g.n if task in (0, 1) else g.m)
        impl, label = o, "port"
    k = o.budget(basis, w["rate"])
    rows = max(threads, 1)
    cap_rows = int(max(w["pop"] * 4, min(1_000_000, 2e8 / max(k, 1))))  # bounded sample: <= 0.8 GB of genes
    total_rows, total_t = 0, 0.0
    while True:
        batch = o.init_population(basis, rows, k, 1)
        t0 = time.perf_counter()
        impl.eval_batch(ctx, task, batch, threads=threads)
        dt = time.perf_counter() - t0
        total_rows, total_t = rows, dt
        if dt >= target_seconds / 3 or rows >= cap_rows:
            break
        rows = int(min(cap_rows, max(rows * 2, rows * (target_seconds / 2) / max(dt, 1e-3))))
    return {"value": total_rows / total_t, "unit": "evals/s", "cores": threads, "kind": label, "rows": total_rows, "seconds": total_t,
            "sample": f"{total_rows} individuals of the workload evaluated once on {threads} host threads "
                      f"({'unmodified reference, dense BitMatrix' if use_ref else 'CSR port of the reference algorithm; the reference itself needs n^2/8 bytes per individual'}) in {total_t:.2f} s"}


def workload_shape(w: dict) -> dict:
    """n, m, k of a workload without touching a GPU (host generators of the product library: problem setup, CPU)."""
    import paper_2412_20980_b200 as gp
    kind, *gargs = w["graph"]
    graph = {"ba": gp.barabasi_albert, "er": gp.erdos_renyi, "sbm": gp.planted_partition}[kind](*gargs)
    if w["task"] == "lpa":
        graph = gp.build_lp_split(graph, 0.1, 1).train
    kindp = gp.PoolKind.NodeRemoval if w["task"] in ("pc", "mcn") else gp.PoolKind.EdgeRemoval
    return {"n": graph.node_count(), "m": graph.edge_count(), "budget": gp.perturbation_budget(graph, kindp, w["rate"])}


def config_of(w: dict, s: int, k: int, n: int, m: int, world: int, rows_per_rank: int) -> dict:
    """the `config` object — identical keys and values in both arms"""
    return {"workload": w["name"], "population": s, "budget": k, "n": n, "m": m,
            "step": "one generation of the in-library loop: select -> crossover+mutate -> evaluate(M_POP) -> elitism, population in HBM",
            "parallelism": f"population rows sharded over {world} GPU(s), graph replicated, 1 fitness all-gather/generation",
            "l2": "inputs larger than L2 (gene matrix %.0f MB + alive/reached words %.0f MB per step vs 126 MB L2)"
                  % (4.0 * s * k / 1e6, 16.0 * n * ((rows_per_rank + 63) // 64) / 1e6)}


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = host_threads()
    steps = max(args.steps, 1)
    per_step = min(60.0, 150.0 / (steps + args.warmup))
    vals, secs, rows = [], [], []
    base = None
    for i in range(args.warmup + steps):
        base = cpu_reference_throughput(w, per_step, threads)
        if i >= args.warmup:
            vals.append(base["value"])
            secs.append(base["seconds"])
            rows.append(base["rows"])
    value = float(np.sum(rows) / np.sum(secs))
    base["value"] = value
    s = (args.pop or w["pop"]) * (max(args.gpus, 1) if args.scaling == "weak" else 1)  # weak: the workload's population PER GPU
    world = max(args.gpus, 1)
    shape = workload_shape(w)
    # A step of this arm is a BOUNDED SAMPLE of the workload's step (rows_per_step individuals of the population,
    # evaluated once on the host cores): ms_per_step is the measured time of that sample, not of a whole generation.
    line = {"impl": "reference", "metric": "fitness_evals_per_sec", "value": value, "unit": "evals/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)), "rows_per_step": int(np.mean(rows)),
            "step_is_sample": True, "ms_per_full_step_extrapolated": 1e3 * s / value,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "int64" if w["task"] in ("pc", "mcn") else "f64", "data": "synthetic",
            "config": config_of(w, s, shape["budget"], shape["n"], shape["m"], world, (s + world - 1) // world),
            "cpu_baseline": base,
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------- GPU arm
def run_gpu_arm(args, w):
    import torch
    import torch.distributed as dist
    import paper_2412_20980_b200 as gp
    from paper_2412_20980_b200.driver import Comm, Shard, torch_bytes_allgather

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the hot path has no CPU fallback")
    if world != max(args.gpus, 1):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # development aid: all ranks on GPU 0 (separate processes, time-sliced; rendezvous over gloo because NCCL refuses two
    # ranks on one device) — exercises the N > 1 code path of this script on a one-GPU box; never a benchmark
    shared_gpu = world > 1 and os.environ.get("GAPA_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    elif torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: --gpus {world} but only {torch.cuda.device_count()} CUDA device(s) are visible")
    torch.cuda.set_device(local)
    if world > 1 and shared_gpu:
        dist.init_process_group("gloo")
    elif world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if rank == 0:
            print(f"[bench] NCCL communicator: nranks={dist.get_world_size()} backend={dist.get_backend()}", file=sys.stderr, flush=True)

    kind, *gargs = w["graph"]
    graph = {"ba": gp.barabasi_albert, "er": gp.erdos_renyi, "sbm": gp.planted_partition}[kind](*gargs)
    task = w["task"]
    T = P = 0
    if task == "lpa":
        split = gp.build_lp_split(graph, 0.1, 1)
        pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
        obj = gp.LinkPredictionAttackObjective(split, pool, device=local)
        base_graph, T, P = split.train, len(split.test_edges), len(split.probe_nonedges)
    elif task == "cda":
        pool = gp.build_gene_pool(graph, gp.PoolKind.EdgeRemoval)
        obj = gp.ModularityAttackObjective(graph, pool, device=local)
        base_graph = graph
    else:
        pool = gp.build_gene_pool(graph, gp.PoolKind.NodeRemoval)
        obj = (gp.PairwiseConnectivityObjective if task == "pc" else gp.SixDstObjective)(graph, pool, device=local)
        base_graph = graph
    n, m = base_graph.node_count(), base_graph.edge_count()
    k = gp.perturbation_budget(base_graph, pool.kind(), w["rate"])
    s = (args.pop or w["pop"]) * (max(args.gpus, 1) if args.scaling == "weak" else 1)  # weak: the workload's population PER GPU
    params = gp.GAParams(pc=w["pc"], pm=w["pm"], pop_size=s, budget=k, iterations=args.warmup + args.steps + 1, seed=1)
    shard = Shard(rank, world, s)
    lib = gp.capi.load()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    # The generation loop runs inside the library (gapa_cuda_ga_*: what a C++ host's run_ga_cuda executes), one rank per
    # GPU.  The once-per-generation exchange is the library's own: peer mailboxes over NVLink where every GPU can reach
    # every other (surviving children of other ranks are then read from their builder's HBM on demand), else NCCL.
    comm, transport = None, None
    if world > 1:
        transport = args.exchange
        if transport == "auto" and shared_gpu:
            transport = "peer"
        if transport == "auto":
            reach = all(torch.cuda.can_device_access_peer(local, d) for d in range(world) if d != local)
            flags = [None] * world
            dist.all_gather_object(flags, bool(reach))
            transport = "peer" if all(flags) else "nccl"
        if transport == "peer":
            comm = Comm.peer(obj, rank, world, s, torch_bytes_allgather())
        else:
            def broadcast_bytes(data):
                box = [data]
                dist.broadcast_object_list(box, src=0)
                return box[0]
            comm = Comm.nccl(obj, rank, world, broadcast_bytes)
        if rank == 0:
            print(f"[bench] exchange transport: {transport} (world {world})", file=sys.stderr, flush=True)
    loop = gp.GaLoop(params, obj, rank=rank, world=world, comm=comm)
    loop.advance(args.warmup)  # generation 1 carries the initialisation and the first evaluation of the parents
    barrier()
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    calls0, eval_s0, _ = loop.counters()
    launches0 = lib.gapa_cuda_launch_count()
    step_ms_total = loop.advance(args.steps)  # device time of exactly K generations: CUDA events on the run's stream
    barrier()
    launches = lib.gapa_cuda_launch_count() - launches0
    clocks = sampler.stop() if rank == 0 else None
    calls1, eval_s1, _ = loop.counters()
    eval_ms = [1e3 * (eval_s1 - eval_s0) / max(calls1 - calls0, 1)]  # variation + evaluation of the timed generations
    mine = loop.result()

    # pure fitness evaluation (no variation fused in), device-resident: this rank's block of the current parents
    # — what the roofline figures are computed from
    lo, hi = shard.rows
    block_dev = torch.from_numpy(mine.final_population[lo:hi]).cuda()
    fit_dev = torch.empty(max(hi - lo, 1), dtype=torch.float64, device="cuda")
    pure_ms = []
    for i in range(3 + args.steps):
        obj.dgraph.eval_batch_device(obj.task, block_dev.data_ptr(), hi - lo, k, fit_dev.data_ptr(), 0)
        if i >= 3:
            pure_ms.append(obj.dgraph.last_eval_ms())
    torch.cuda.synchronize()
    assert np.array_equal(fit_dev[:hi - lo].cpu().numpy(), mine.final_fitness[lo:hi]), "re-evaluating the parents changed their fitness"

    # e2e: the plugin boundary with HOST buffers — evaluate_batch(host genes) -> host fitness,
    # this rank's block of the current M_POP, pinned memory, copies inside the timed region.
    host_genes = torch.empty((hi - lo, k), dtype=torch.int32, pin_memory=True)
    host_genes.copy_(torch.from_numpy(mine.final_population[lo:hi]))  # this rank's block of the current parents
    host_out = torch.empty(max(hi - lo, 1), dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()

    def e2e_once():
        gp.capi.check(lib.gapa_cuda_eval_batch(obj.dgraph.handle, obj.task, host_genes.data_ptr(), hi - lo, k,
                                               host_out.data_ptr()))

    for _ in range(min(args.warmup, 3)):
        e2e_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_once()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    assert np.array_equal(host_out[:hi - lo].numpy(), mine.final_fitness[lo:hi]), "e2e result differs from the device path"

    # the same call with a PAGEABLE gene matrix — what the C++ adapter's evaluate_batch(const PopulationMatrix&) passes
    # (a std::vector): the library stages it through its own pinned ring
    pageable_genes = host_genes.numpy().copy()
    pageable_out = np.empty(max(hi - lo, 1), dtype=np.float64)

    def e2e_pageable_once():
        gp.capi.check(lib.gapa_cuda_eval_batch(obj.dgraph.handle, obj.task, pageable_genes.ctypes.data, hi - lo, k,
                                               pageable_out.ctypes.data))

    for _ in range(2):
        e2e_pageable_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_pageable_once()
    e2e_pageable_s = time.perf_counter() - t0
    assert np.array_equal(pageable_out[:hi - lo], mine.final_fitness[lo:hi]), "pageable e2e result differs from the device path"

    # N > 1: the sharded run must BE the 1-GPU run (test_parallel.cpp:86-104): rank 0 repeats the same generations
    # unsharded with the same seed and compares history and final population bit for bit.
    verify = None
    if world > 1:
        if rank == 0:
            solo = gp.GaLoop(params, obj)
            solo.advance(loop.generation)
            ref = solo.result()
            solo.close()
            g = loop.generation
            verify = {"generations": g, "transport": transport,
                      "history_best_equal": bool(np.array_equal(mine.history_best[:g], ref.history_best[:g])),
                      "history_mean_equal": bool(np.array_equal(mine.history_mean[:g], ref.history_mean[:g])),
                      "final_population_equal": bool(np.array_equal(mine.final_population, ref.final_population)),
                      "final_fitness_equal": bool(np.array_equal(mine.final_fitness, ref.final_fitness))}
        barrier()

    times = torch.tensor([step_ms_total, e2e_s * 1e3, float(np.mean(pure_ms)), float(np.mean(eval_ms)), e2e_pageable_s * 1e3],
                         dtype=torch.float64, device="cpu" if shared_gpu else "cuda")
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    step_ms_total, e2e_ms_total, eval_ms_mean, fused_ms_mean, e2e_pageable_ms_total = (float(x) for x in times.cpu())

    if rank == 0:
        ms_per_step = step_ms_total / args.steps
        value = s * args.steps / (step_ms_total * 1e-3)
        e2e_value = s * args.steps / (e2e_ms_total * 1e-3)
        dbar = 2.0 * m / max(n, 1)
        b_eval = algorithmic_bytes(task, n, m, k, T, P, dbar)
        peak, peak_src = peaks()
        rows_per_rank = shard.block
        survey = b_eval * rows_per_rank / (eval_ms_mean * 1e-3) / 1e9
        traffic = traffic_src = None
        try:
            with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as f:
                entry = json.load(f).get(args.workload if not args.pop else f"{args.workload}@{args.pop}")
            if isinstance(entry, dict):
                traffic, traffic_src = entry.get("bytes"), entry.get("source")
            elif entry:
                traffic = entry
        except Exception:
            pass
        if task in ("pc", "mcn"):
            # What the bit-sliced algorithm has to move for this rank's batch: the CSR once per super-group
            # of 256 individuals (one pass serves all of them), and per individual its genome (4k), its removal bitmap
            # (written, read by the transpose: 2 n/8), its alive bits (written + read: 2 n/8) and its reached bits
            # (cleared, read, written: 3 n/8).
            sg = (rows_per_rank + 255) // 256
            b_algo = sg * (4 * (n + 1) + 8 * m) + rows_per_rank * (4 * k + 7 * (n / 8.0))
            algo_note = ("batched algorithm: CSR once per 256 individuals + per individual 4k genome + 7 n/8 bitmap / alive / reached "
                         "bytes (the clear of the reached records included)")
        else:
            b_algo = b_eval * rows_per_rank
            algo_note = "SURVEY 8(d) bytes per evaluation x evaluations per launch sequence (working set is L2-resident: no roofline claim)"
        achieved = b_algo / (eval_ms_mean * 1e-3) / 1e9
        # ncu-measured DRAM bytes of one full-population evaluation (tools/ncu_traffic.py), scaled to this rank's rows
        actual = traffic * (rows_per_rank / s) / (eval_ms_mean * 1e-3) / 1e9 if traffic else None
        line = {
            "metric": "fitness_evals_per_sec", "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "int64" if task in ("pc", "mcn") else "f64", "data": "synthetic",
            "config": config_of(w, s, k, n, m, world, rows_per_rank),
            "generations_per_sec": 1e3 / ms_per_step,
            "fitness_eval_ms_per_step": eval_ms_mean,
            "variation_plus_eval_ms_per_step": fused_ms_mean,
            "fitness_evals_per_sec_kernels_only": rows_per_rank * world / (eval_ms_mean * 1e-3),
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": int(4 * (hi - lo) * k) * world,
                    "d2h_bytes_per_step": int(8 * (hi - lo)) * world,
                    "path": "gapa_cuda_eval_batch(pinned host genes) -> host fitness (FitnessFunction::evaluate_batch boundary)"},
            "e2e_pageable": {"value": s * args.steps / (e2e_pageable_ms_total * 1e-3), "unit": "evals/s",
                             "path": "the same call with a pageable gene matrix (what CudaObjective::evaluate_batch(const "
                                     "PopulationMatrix&) passes): staged through the library's pinned ring by host threads"},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "comm": {"transport": transport, "bootstrap": ("torch.distributed gloo (ranks share one GPU: development aid, not a benchmark)" if shared_gpu else "torch.distributed nccl") if world > 1 else None, "nranks": world},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                         "kernel": "fitness evaluation pipeline (k_pc_sweep dominant)" if task in ("pc", "mcn") else f"{task} fitness pipeline",
                         "algorithmic_bytes_per_launch": b_algo, "algorithmic_bytes_model": algo_note,
                         "actual_dram_gbs": actual, "actual_dram_frac": (actual / peak) if actual else None,
                         "vs_survey_model": {"bytes_per_eval": b_eval, "achieved": survey, "frac": survey / peak,
                                             "note": "SURVEY 8(d) charges every individual a private pass over the CSR; the bit-sliced "
                                                     "kernels share one pass among 256 individuals, so this ratio exceeds 1 and is NOT "
                                                     "a fraction of the HBM peak"},
                         "note": "achieved = algorithmic bytes of the launch sequence / device time of the whole evaluation (CUDA events "
                                 "on the launch stream); traffic = ncu dram__bytes_read+write of the same launch sequence "
                                 "(profiles/dram_traffic.json, produced by tools/ncu_traffic.py); actual_dram_* = traffic / the same time"},
        }
        if verify is not None:
            line["verify"] = verify
        if task == "cda":
            # the merge phase is on-chip / L2 traffic and serial merge depth, not HBM — report merges/s.
            # Merges of one detection = n - communities of its partition; estimated from 8 individuals' partitions.
            from paper_2412_20980_b200.experiment import _detect
            sample = mine.final_population[np.linspace(0, s - 1, 8).astype(int)]
            merges = float(np.mean([n - len(np.unique(_detect(obj.dgraph, row))) for row in sample]))
            line["merges_per_individual"] = merges
            line["merges_per_sec"] = merges * rows_per_rank * world / (eval_ms_mean * 1e-3)
            line["roofline"]["note"] += ("; CDA is bound by the serial depth of the greedy merge sequence (one block-wide step per "
                                         "merge), not by HBM: see merges_per_sec")
        if world == 1:
            # the same generations through the in-library loop (gapa_cuda_run: no host round trip per
            # operator) — what a C++ host gets from run_ga_cuda(); reported beside the stepwise driver
            iters = max(args.steps, 5) if ms_per_step > 1.0 else 200  # short generations: amortise init + the final read-back
            run = gp.run_ga(gp.GAParams(pc=w["pc"], pm=w["pm"], pop_size=s, budget=k, iterations=iters, seed=1), pool, obj)
            line["library_loop"] = {"generations_per_sec": iters / run.total_wall_seconds, "iterations": iters,
                                    "evals_per_sec": s * (iters + 1) / run.total_wall_seconds,
                                    "eval_ms_per_generation": 1e3 * run.eval_seconds / (iters + 1)}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_reference_throughput(w, 30.0, host_threads())
        print(json.dumps(line), flush=True)
    loop.close()
    if comm is not None:
        barrier()
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--pop", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = the workload's population sharded over the GPUs (north_star's C4); weak = that population per GPU")
    ap.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                    help="N > 1: the library's exchange transport (auto = peer mailboxes where every GPU reaches every other)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, w)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` on its own: re-launch under torch.distributed.run, one rank per GPU
        import socket
        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")  # the communicator's "nranks N" line goes to stderr
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd, env=env))
    run_gpu_arm(args, w)


if __name__ == "__main__":
    main()
