"""The library's own exchange and the sharded run built on it on the ONE GPU the test box has:
ranks are host threads of one process (gapa_cuda_run_multi: peer mailboxes between two contexts on the same device)
or separate processes (CUDA IPC mailboxes), plus the NCCL transport with a one-rank communicator.  The determinism
contract of test_parallel.cpp:86-104: every rank of every world size reproduces the single-GPU run and the oracle."""
import multiprocessing as mp
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert np.array_equal(a.history_best, b.history_best) and np.array_equal(a.history_mean, b.history_mean)
    assert np.array_equal(a.final_population, b.final_population) and np.array_equal(a.final_fitness, b.final_fitness)


@pytest.mark.parametrize("peer_rows", ["1", "0"], ids=["peer-rows", "rebuild"])
@pytest.mark.parametrize("world,eda", [(2, 0), (3, 4), (4, 0)])
def test_run_multi_threads_equal_the_single_run(gp, oracle, cuda_device, world, eda, peer_rows, monkeypatch):
    """gapa_cuda_run_multi: `world` contexts on device 0, one host thread each, peer-mailbox exchange (raw pointers inside
    one process).  Ragged blocks (37 rows over 2 / 3 / 4 ranks), EDA generations included.  Surviving children of other
    ranks are read from their builder's pool on demand (default), or rebuilt locally (GAPA_PEER_ROWS=0)."""
    monkeypatch.setenv("GAPA_PEER_ROWS", peer_rows)
    g = gp.barabasi_albert(600, 2, 4)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    s, k, iters = 37, 15, 12
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=s, budget=k, iterations=iters, seed=11, eda_interval=eda or None)
    want = oracle.run_ga(oracle.graph_from_edges(g.n, g.edges()), 0, 0.6, 0.2, s, k, iters, 11, eda_interval=eda)
    objs = [gp.PairwiseConnectivityObjective(g, pool) for _ in range(world)]
    results = gp.run_ga_multi(params, objs, transport="peer")
    assert len(results) == world
    for res in results:
        assert np.array_equal(res.history_best, want["best"]) and np.array_equal(res.history_mean, want["mean"])
        assert np.array_equal(res.final_population, want["population"]) and np.array_equal(res.final_fitness, want["fitness"])
        assert all(h.messages == 2 if i == 0 else h.messages == 1 for i, h in enumerate(res.history))  # one exchange per evaluation


def test_run_multi_bit_sliced_path_and_large_population(gp, cuda_device, monkeypatch):
    """The same through the bit-sliced PC pipeline (forced) with a population beyond the one-launch operators."""
    monkeypatch.setenv("GAPA_PC_SMALL", "0")
    g = gp.barabasi_albert(5000, 3, 2)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=700, budget=250, iterations=6, seed=3)
    single = gp.run_ga(params, pool, gp.PairwiseConnectivityObjective(g, pool))
    for res in gp.run_ga_multi(params, [gp.PairwiseConnectivityObjective(g, pool) for _ in range(2)]):
        _same(res, single)


def test_run_multi_other_tasks(gp, cuda_device):
    g = gp.erdos_renyi(300, 0.03, 5)
    split = gp.build_lp_split(g, 0.2, 2)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    params = gp.GAParams(pc=0.7, pm=0.1, pop_size=21, budget=30, iterations=7, seed=4, eda_interval=3)
    single = gp.run_ga(params, pool, gp.LinkPredictionAttackObjective(split, pool))
    for res in gp.run_ga_multi(params, [gp.LinkPredictionAttackObjective(split, pool) for _ in range(2)]):
        _same(res, single)
    g2 = gp.planted_partition(3, 20, 0.3, 0.03, 6)
    pool2 = gp.build_gene_pool(g2, gp.PoolKind.EdgeRemoval)
    params2 = gp.GAParams(pc=0.8, pm=0.1, pop_size=12, budget=9, iterations=5, seed=8)
    single2 = gp.run_ga(params2, pool2, gp.ModularityAttackObjective(g2, pool2))
    for res in gp.run_ga_multi(params2, [gp.ModularityAttackObjective(g2, pool2) for _ in range(3)]):
        _same(res, single2)


def test_nccl_transport_loads_and_gathers(gp, cuda_device):
    """libnccl.so.2 resolved at run time: unique id, communicator of one rank, an in-place all-gather on a device
    buffer; and run_multi(world = 1, transport = nccl).  (NCCL refuses two ranks on one GPU, so a one-rank
    communicator is what this box can exercise.)"""
    import ctypes as C

    import torch
    from paper_2412_20980_b200.driver import Comm
    g = gp.barabasi_albert(300, 2, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    comm = Comm.nccl(obj, 0, 1, lambda data: data)
    lib = gp.capi.load()
    kind, rank, world = C.c_int(-1), C.c_int(-1), C.c_int(-1)
    gp.capi.check(lib.gapa_cuda_comm_info(comm.handle, C.byref(kind), C.byref(rank), C.byref(world)))
    assert (kind.value, rank.value, world.value) == (1, 0, 1)
    fit = torch.arange(8, dtype=torch.float64, device="cuda")
    gp.capi.check(lib.gapa_cuda_comm_allgather(comm.handle, fit.data_ptr(), 8, 8, 0))
    torch.cuda.synchronize()
    assert fit.cpu().tolist() == list(range(8))
    out = C.create_string_buffer(5)
    gp.capi.check(lib.gapa_cuda_comm_allgather_bytes(comm.handle, b"hello", 5, out))
    assert out.raw == b"hello"
    comm.close()
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=20, budget=10, iterations=5, seed=2)
    _same(gp.run_ga_multi(params, [obj], transport="nccl")[0], gp.run_ga(params, pool, obj))


def _file_allgather(tmpdir, rank, world):
    """out-of-band all-gather through files (any channel will do: the handles are 128 opaque bytes)"""
    import time
    state = {"round": 0}

    def gather(mine: bytes):
        tag = state["round"]
        state["round"] += 1
        final = os.path.join(tmpdir, f"r{tag}_{rank}.bin")
        with open(final + ".tmp", "wb") as f:
            f.write(mine)
        os.replace(final + ".tmp", final)
        out = []
        for r in range(world):
            path = os.path.join(tmpdir, f"r{tag}_{r}.bin")
            deadline = time.time() + 240
            while not os.path.exists(path):
                if time.time() > deadline:
                    raise TimeoutError(path)
                time.sleep(0.01)
            with open(path, "rb") as f:
                out.append(f.read())
        return out

    return gather


def _ipc_rank(rank, world, tmpdir, out_q):
    """one rank of a two-PROCESS run on the same GPU: handles travel through files, mailboxes through CUDA IPC"""
    try:
        import paper_2412_20980_b200 as gp
        from paper_2412_20980_b200.driver import Comm
        g = gp.barabasi_albert(600, 2, 4)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        obj = gp.PairwiseConnectivityObjective(g, pool)
        params = gp.GAParams(pc=0.6, pm=0.2, pop_size=37, budget=15, iterations=8, seed=11, eda_interval=3)
        allgather_bytes = _file_allgather(tmpdir, rank, world)
        comm = Comm.peer(obj, rank, world, params.pop_size, allgather_bytes)
        res = gp.run_ga(params, pool, obj, rank=rank, world=world, comm=comm)
        comm.status()
        out_q.put((rank, res.history_best, res.history_mean, res.final_population, res.final_fitness))
        # every rank has finished its last exchange before anybody frees a mailbox the others may still read
        allgather_bytes(b"done")
        comm.close()
    except Exception as exc:  # noqa: BLE001
        out_q.put((rank, repr(exc)))


def test_two_processes_exchange_through_cuda_ipc(gp, oracle, cuda_device, tmp_path, monkeypatch):
    monkeypatch.setenv("GAPA_COMM_TIMEOUT_MS", "60000")
    ctx = mp.get_context("spawn")
    world = 2
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, world, str(tmp_path), q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    g = gp.barabasi_albert(600, 2, 4)
    want = oracle.run_ga(oracle.graph_from_edges(g.n, g.edges()), 0, 0.6, 0.2, 37, 15, 8, 11, eda_interval=3)
    for item in got:
        assert len(item) == 5, item
        _, best, mean, population, fitness = item
        assert np.array_equal(best, want["best"]) and np.array_equal(mean, want["mean"])
        assert np.array_equal(population, want["population"]) and np.array_equal(fitness, want["fitness"])


def test_resumable_loop_equals_one_run(gp, cuda_device):
    """gapa_cuda_ga_*: blocks of generations with the population resident in between == gapa_cuda_run."""
    g = gp.barabasi_albert(3000, 3, 2)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=64, budget=150, iterations=40, seed=3, eda_interval=7)
    whole = gp.run_ga(params, pool, obj)
    loop = gp.GaLoop(params, obj, want_stats=True)
    ms = []
    for block in (1, 5, 16, 3, 100):
        ms.append(loop.advance(block))
    assert loop.generation == 40 and all(t > 0 for t in ms[:4])
    part = loop.result()
    _same(part, whole)
    assert part.fitness_batch_calls == 41
    assert all(h.wall_seconds > 0 for h in part.history)
    early = gp.GaLoop(params, obj)
    early.advance(10)
    mid = early.result()
    assert np.array_equal(mid.history_best[:10], whole.history_best[:10]) and np.all(mid.history_best[10:] == 0)
    assert np.all(np.diff(mid.final_fitness) >= 0)
    early.close()
    loop.close()
