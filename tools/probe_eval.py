"""One device-resident fitness evaluation of a bench.py workload's initial population (for ncu / timing probes;
not the bench contract).  usage: python tools/probe_eval.py [workload] [pop] [repeats]

The evaluations after the warm-up are bracketed by cudaProfilerStart/Stop, so
`ncu --profile-from-start off` lists exactly `repeats` evaluations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_20980_b200 as gp  # noqa: E402
from paper_2412_20980_b200 import capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = bench.WORKLOADS[name]
s = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) else w["pop"]
repeats = int(sys.argv[3]) if len(sys.argv) > 3 else 1
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
lib = capi.load()
genes = torch.empty((s, k), dtype=torch.int32, device="cuda")
out = torch.empty(s, dtype=torch.float64, device="cuda")
capi.check(lib.gapa_cuda_ga_init_device(pool.size(), 0, s, k, 1, 0, genes.data_ptr(), 0))
for _ in range(3):
    obj.dgraph.eval_batch_device(obj.task, genes.data_ptr(), s, k, out.data_ptr(), 0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ms = []
for _ in range(repeats):
    obj.dgraph.eval_batch_device(obj.task, genes.data_ptr(), s, k, out.data_ptr(), 0)
    ms.append(obj.dgraph.last_eval_ms())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"{name}: n={base.node_count()} m={base.edge_count()} k={k} pop={s}: evaluation {sum(ms) / len(ms):.4f} ms "
      f"({s / (sum(ms) / len(ms)) * 1e3:.0f} evals/s), fitness[:3] = {out[:3].tolist()}", flush=True)
