"""PC evaluation timing on Erdos-Renyi / shuffled-label graphs (the hub-first relabelling path)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2412_20980_b200 as gp
from paper_2412_20980_b200 import capi
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000
deg = float(sys.argv[2]) if len(sys.argv) > 2 else 8.0
s = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
rng = np.random.default_rng(1)
m = int(n * deg / 2)
e = rng.integers(0, n, (m, 2)).astype(np.int32)
e = e[e[:, 0] != e[:, 1]]
e.sort(axis=1)
e = np.unique(e, axis=0)
g = gp.Graph(n, e)
pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.05)
obj = gp.PairwiseConnectivityObjective(g, pool)
lib = capi.load()
genes = torch.empty((s, k), dtype=torch.int32, device="cuda")
out = torch.empty(s, dtype=torch.float64, device="cuda")
capi.check(lib.gapa_cuda_ga_init_device(pool.size(), 0, s, k, 1, 0, genes.data_ptr(), 0))
torch.cuda.synchronize()
for it in range(4):
    l0 = lib.gapa_cuda_launch_count()
    obj.dgraph.eval_batch_device(0, genes.data_ptr(), s, k, out.data_ptr(), 0)
    torch.cuda.synchronize()
    print(f"ER n={n} m={len(e)} iter {it}: device {obj.dgraph.last_eval_ms():.2f} ms launches {lib.gapa_cuda_launch_count()-l0}", flush=True)
if n <= 300_000:
    from oracle.bindings import Oracle
    o = Oracle(); og = o.graph_from_edges(g.n, g.edges())
    print("oracle match:", np.array_equal(o.eval_batch(og, 0, genes[:32].cpu().numpy(), threads=8), out[:32].cpu().numpy()))
