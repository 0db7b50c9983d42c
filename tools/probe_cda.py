"""Device-side timing probe for the CDA fitness kernel (C2 shape by default)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2412_20980_b200 as gp
blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 500
rows = int(sys.argv[3]) if len(sys.argv) > 3 else 100
g = gp.planted_partition(blocks, bs, 0.02 * 500 / bs, 0.0005 * 500 / bs, 1)
pool = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)
k = gp.perturbation_budget(g, gp.PoolKind.EdgeRemoval, 0.05)
obj = gp.ModularityAttackObjective(g, pool)
pop = gp.init_population(pool.size(), rows, k, 1)
for it in range(3):
    t0 = time.time(); f = obj.evaluate_batch(pop); dt = time.time() - t0
    print(f"n={g.n} m={g.edge_count()} k={k} rows={rows}: wall {dt*1e3:.1f} ms device {obj.dgraph.last_eval_ms():.1f} ms  Q[0]={f[0]:.6f}", flush=True)

import ctypes as C
lib = gp.capi.load()
if hasattr(lib, "gapa_cuda_cda_phase_cycles") or True:
    try:
        fn = lib.gapa_cuda_cda_phase_cycles
        buf = (C.c_ulonglong * 8)()
        fn(buf, 1)
        obj.evaluate_batch(pop[:1])
        fn(buf, 0)
        names = ["argmax", "room+mark", "fold", "drop", "scan list(a)", "list work (short)", "list work (long)", "best(a)+map reset"]
        tot = sum(buf)
        print("phase cycles of one individual (CTA 0):", {n: f"{100 * v / tot:.1f}%" for n, v in zip(names, buf)}, f"total {tot / 1.965e6:.1f} ms")
    except AttributeError:
        pass
