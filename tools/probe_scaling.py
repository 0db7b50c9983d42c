"""Per-rank critical path of the sharded generation at world = N, measured on ONE GPU.

Runs driver.ShardedGa as rank 0 of N with a stand-in for the all-gather that fills the other ranks'
fitness blocks with a cyclic copy of this rank's block (so the elitism mix of surviving rows is
realistic).  What it measures is everything a rank does per generation except the NCCL all-gather
itself (s doubles; latency-bound, ~20-50 us on NVSwitch).  It is a projection aid, not a scaling result."""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2412_20980_b200 as gp
from paper_2412_20980_b200.driver import CudaOps, Shard, ShardedGa

n, attach, s, rate = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000, 5, 4096, 0.05
g = gp.barabasi_albert(n, attach, 1)
pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, rate)
obj = gp.PairwiseConnectivityObjective(g, pool)
out = {}
for world in (1, 2, 4, 8):
    shard = Shard(0, world, s)
    lo, hi = shard.rows

    def gather(fit, shard_):
        if shard_.world == 1:
            return
        block = fit[lo:hi]
        for r in range(1, shard_.world):
            fit[r * (hi - lo):(r + 1) * (hi - lo)] = block

    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=s, budget=k, iterations=40, seed=1)
    ga = ShardedGa(params, CudaOps(obj, 0), shard, gather)
    ga.initialize()
    for _ in range(3):
        ga.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    steps = 15
    for _ in range(steps):
        ga.step()
    e1.record()
    torch.cuda.synchronize()
    out[world] = e0.elapsed_time(e1) / steps
    del ga
base = out[1]
print(json.dumps({"n": n, "pop": s, "k": k, "ms_per_generation_per_rank": out,
                  "projected_speedup_excluding_allgather": {w: base / t for w, t in out.items()}}))
