"""Per-kernel device time of ONE generation of the in-library loop, from torch's CUPTI profiler (no ncu needed):
usage: python tools/probe_gen_kernels.py [workload] [pop]   -> one line per kernel, ms summed over the generation"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2412_20980_b200 as gp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = bench.WORKLOADS[name]
s = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) else w["pop"]
kind, *gargs = w["graph"]
graph = {"ba": gp.barabasi_albert, "er": gp.erdos_renyi, "sbm": gp.planted_partition}[kind](*gargs)
pool = gp.build_gene_pool(graph, gp.PoolKind.NodeRemoval)
obj = gp.PairwiseConnectivityObjective(graph, pool)
k = gp.perturbation_budget(graph, pool.kind(), w["rate"])
loop = gp.GaLoop(gp.GAParams(pc=w["pc"], pm=w["pm"], pop_size=s, budget=k, iterations=40, seed=1), obj)
loop.advance(4)
torch.cuda.synchronize()
ms = loop.advance(10) / 10
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    loop.advance(5)
    torch.cuda.synchronize()
rows = sorted(((e.key, e.device_time_total / 5 / 1000.0, e.count / 5) for e in prof.key_averages()), key=lambda r: -r[1])
print(f"{name}: generation {ms:.4f} ms; " + "; ".join(f"{k_.split('(')[0].replace('void gapa_b200::', '')[:28]} {t:.4f}" for k_, t, c in rows[:6]))
loop.close()
