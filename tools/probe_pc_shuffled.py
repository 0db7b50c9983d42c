"""PC eval time on a BA graph with shuffled labels (tests the hub-first internal order)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2412_20980_b200 as gp
from paper_2412_20980_b200 import capi
n, s = int(float(sys.argv[1])), int(sys.argv[2])
base = gp.barabasi_albert(n, 5, 1)
perm = np.random.default_rng(1).permutation(n).astype(np.int32)
g = gp.Graph(n, perm[base.edges()])
pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.05)
obj = gp.PairwiseConnectivityObjective(g, pool)
lib = capi.load()
genes = torch.empty((s, k), dtype=torch.int32, device="cuda"); out = torch.empty(s, dtype=torch.float64, device="cuda")
capi.check(lib.gapa_cuda_ga_init_device(pool.size(), 0, s, k, 1, 0, genes.data_ptr(), 0))
for it in range(4):
    l0 = lib.gapa_cuda_launch_count(); t0 = time.time()
    obj.dgraph.eval_batch_device(0, genes.data_ptr(), s, k, out.data_ptr(), 0); torch.cuda.synchronize()
    print(f"iter {it}: wall {(time.time()-t0)*1e3:.2f} ms device {obj.dgraph.last_eval_ms():.2f} ms launches {lib.gapa_cuda_launch_count()-l0}", flush=True)
