"""Quick device-side timing probe for the PC fitness path (not the bench contract)."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2412_20980_b200 as gp
from paper_2412_20980_b200 import capi

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
rate = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
attach = int(sys.argv[4]) if len(sys.argv) > 4 else 5
t0 = time.time(); g = gp.barabasi_albert(n, attach, 1); print(f"graph n={g.n} m={g.edge_count()} gen {time.time()-t0:.2f}s", flush=True)
pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, rate)
t0 = time.time(); obj = gp.PairwiseConnectivityObjective(g, pool); print(f"ctx {time.time()-t0:.2f}s k={k}", flush=True)
lib = capi.load()
genes = torch.empty((s, k), dtype=torch.int32, device="cuda")
out = torch.empty(s, dtype=torch.float64, device="cuda")
capi.check(lib.gapa_cuda_ga_init_device(pool.size(), 0, s, k, 1, 0, genes.data_ptr(), 0))
torch.cuda.synchronize()
for it in range(5):
    l0 = lib.gapa_cuda_launch_count()
    t0 = time.time()
    obj.dgraph.eval_batch_device(0, genes.data_ptr(), s, k, out.data_ptr(), 0)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ms = obj.dgraph.last_eval_ms()
    print(f"iter {it}: wall {dt*1e3:.2f} ms, device {ms:.2f} ms, {s/ms*1e3:.0f} evals/s, launches {lib.gapa_cuda_launch_count()-l0}", flush=True)
print("fitness[:4]", out[:4].tolist())
if n <= 200_000:
    from oracle.bindings import Oracle
    o = Oracle(); og = o.graph_from_edges(g.n, g.edges())
    want = o.eval_batch(og, 0, genes[:64].cpu().numpy(), threads=8)
    print("oracle match:", np.array_equal(want, out[:64].cpu().numpy()))
