"""ONE generation of the in-library loop bracketed by cudaProfilerStart/Stop (for `ncu --profile-from-start off --set full`).
usage: python tools/probe_gen.py [workload] [pop]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_20980_b200 as gp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = bench.WORKLOADS[name]
s = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) else w["pop"]
kind, *gargs = w["graph"]
graph = {"ba": gp.barabasi_albert, "er": gp.erdos_renyi, "sbm": gp.planted_partition}[kind](*gargs)
task = w["task"]
if task == "lpa":
    split = gp.build_lp_split(graph, 0.1, 1)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    obj, base = gp.LinkPredictionAttackObjective(split, pool), split.train
elif task == "cda":
    pool = gp.build_gene_pool(graph, gp.PoolKind.EdgeRemoval)
    obj, base = gp.ModularityAttackObjective(graph, pool), graph
else:
    pool = gp.build_gene_pool(graph, gp.PoolKind.NodeRemoval)
    obj, base = gp.PairwiseConnectivityObjective(graph, pool), graph
k = gp.perturbation_budget(base, pool.kind(), w["rate"])
loop = gp.GaLoop(gp.GAParams(pc=w["pc"], pm=w["pm"], pop_size=s, budget=k, iterations=8, seed=1), obj)
loop.advance(4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ms = loop.advance(1)
torch.cuda.cudart().cudaProfilerStop()
print(f"{name}: one generation {ms:.4f} ms")
loop.close()
