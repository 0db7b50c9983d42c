"""Device-side timing probe for the truncated-closure SixDST kernel."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2412_20980_b200 as gp
for n, attach, rows in ((500, 1, 80), (1000, 2, 100), (5000, 2, 100), (12000, 3, 100), (20000, 3, 100)):
    g = gp.barabasi_albert(n, attach, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.1)
    obj = gp.SixDstObjective(g, pool, policy=gp.ClosurePolicy.SixDegrees)
    pop = gp.init_population(pool.size(), rows, k, 1)
    for it in range(3):
        f = obj.evaluate_batch(pop)
    print(f"n={n} m={g.edge_count()} k={k} rows={rows}: device {obj.dgraph.last_eval_ms():.3f} ms  fit[0]={f[0]}", flush=True)
