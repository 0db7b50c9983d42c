"""Per-rank critical path of the sharded generation at world = N, measured on ONE GPU (a projection aid, not a scaling
result: the box has one GPU).

Runs the in-library loop (gapa_cuda_ga_*) as rank 0 of N with a stand-in exchange that fills the other ranks' fitness
blocks with a copy of this rank's block, so the elitism mix of surviving rows is realistic.  Two ways of getting the
surviving children of other ranks:
  rebuild   every rank recomputes them from the replicated parents (NCCL transport; round 1's only way)
  peer      they are read from their builder's pool on demand and kept (peer-mailbox transport) — timed here with
            GAPA_PEER_ROWS_LOOPBACK: the "remote" pool is this GPU's own, so the bookkeeping and the write-through copies
            are in the number, the NVLink latency of the remote reads is not.
The exchange itself (one 4 KB-per-rank all-gather per generation: a few microseconds of NVLink stores and a flag per
peer) is not in either number."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2412_20980_b200 as gp  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
weak = len(sys.argv) > 3 and sys.argv[3] == "weak"
g = gp.barabasi_albert(n, 5, 1)
pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.05)
obj = gp.PairwiseConnectivityObjective(g, pool)
cudart = C.CDLL("libcudart.so.12")
out = {}
for mode in os.environ.get("PROBE_MODES", "rebuild,peer").split(","):
    os.environ.pop("GAPA_PEER_ROWS_LOOPBACK", None)
    if mode == "peer":
        os.environ["GAPA_PEER_ROWS_LOOPBACK"] = "1"
    out[mode] = {}
    for world in [int(w) for w in os.environ.get("PROBE_WORLDS", "1,2,4,8").split(",")]:
        pop = s * world if weak else s
        block = (pop + world - 1) // world

        def exchange(user, fit_dev, s_, padded_block, stream, world=world):  # stand-in all-gather: copies of block 0
            for r in range(1, world):
                cudart.cudaMemcpyAsync(C.c_void_p(fit_dev + 8 * r * padded_block), C.c_void_p(fit_dev), C.c_size_t(8 * padded_block),
                                       C.c_int(3), C.c_void_p(stream))
            return 0

        params = gp.GAParams(pc=0.6, pm=0.2, pop_size=pop, budget=k, iterations=40, seed=1)
        loop = gp.GaLoop(params, obj, rank=0, world=world, exchange=exchange if world > 1 else None)
        loop.advance(5)
        out[mode][world] = loop.advance(20) / 20
        if os.environ.get("PROBE_PROFILE"):  # per-kernel device time of a generation at this world size (stderr)
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                loop.advance(5)
                torch.cuda.synchronize()
            rows = sorted(((e.key, e.device_time_total / 5 / 1000.0) for e in prof.key_averages()), key=lambda r: -r[1])
            print(f"[{mode} world {world}] " + "; ".join(f"{k_.split('(')[0].replace('void gapa_b200::', '')[:26]} {t:.4f}" for k_, t in rows[:14]),
                  file=sys.stderr)
        loop.close()
        del block
res = {"n": n, "pop": s, "k": k, "scaling": "weak (pop x world)" if weak else "strong", "ms_per_generation_per_rank": out,
       "projected_speedup_excluding_exchange": {m: {w: (out[m][1] / t) * (w if weak else 1) for w, t in out[m].items()} for m in out if 1 in out[m]}}
print(json.dumps(res))
