"""PC evaluation timing on graph families other than Barabasi-Albert (sanity of the sweep heuristics)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2412_20980_b200 as gp
from paper_2412_20980_b200 import capi
from oracle.bindings import Oracle
o = Oracle()
lib = capi.load()


def run(name, g, s):
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.05)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    genes = torch.empty((s, k), dtype=torch.int32, device="cuda")
    out = torch.empty(s, dtype=torch.float64, device="cuda")
    capi.check(lib.gapa_cuda_ga_init_device(pool.size(), 0, s, k, 1, 0, genes.data_ptr(), 0))
    for it in range(3):
        l0 = lib.gapa_cuda_launch_count()
        obj.dgraph.eval_batch_device(0, genes.data_ptr(), s, k, out.data_ptr(), 0)
        torch.cuda.synchronize()
    og = o.graph_from_edges(g.n, g.edges())
    ok = np.array_equal(o.eval_batch(og, 0, genes[:16].cpu().numpy(), threads=8), out[:16].cpu().numpy())
    print(f"{name}: n={g.n} m={g.edge_count()} rows={s}: device {obj.dgraph.last_eval_ms():.2f} ms launches {lib.gapa_cuda_launch_count()-l0} oracle {ok}", flush=True)


n = 100_000
run("sbm 100x1000", gp.planted_partition(100, 1000, 0.008, 0.00002, 1), 1024)
run("ring", gp.Graph(n, np.stack([np.arange(n), (np.arange(n) + 1) % n], 1).astype(np.int32)), 512)
side = 300
idx = np.arange(side * side).reshape(side, side)
grid = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1), np.stack([idx[:-1].ravel(), idx[1:].ravel()], 1)]).astype(np.int32)
run("grid 300x300", gp.Graph(side * side, grid), 512)
rng = np.random.default_rng(2)
perm = rng.permutation(n).astype(np.int32)
ba = gp.barabasi_albert(n, 3, 4)
run("BA shuffled labels", gp.Graph(n, perm[ba.edges()]), 1024)
star = np.stack([np.zeros(n - 1, np.int32), np.arange(1, n, dtype=np.int32)], 1)
run("star", gp.Graph(n, star), 512)
