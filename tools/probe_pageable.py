"""Host -> device staging of a PAGEABLE gene matrix through gapa_cuda_eval_batch (C4 shape): the library's pinned ring
with N copy threads against the plain cudaMemcpyAsync from pageable memory.  usage: python tools/probe_pageable.py"""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import time
    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2412_20980_b200 as gp
    g = gp.barabasi_albert(1_000_000, 5, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    rows, k = 4096, 50_000
    genes = gp.init_population(pool.size(), rows, k, 1)
    out = np.empty(rows)
    lib = gp.capi.load()
    for _ in range(2):
        gp.capi.check(lib.gapa_cuda_eval_batch(obj.dgraph.handle, obj.task, genes.ctypes.data, rows, k, out.ctypes.data))
    t0 = time.perf_counter()
    for _ in range(5):
        gp.capi.check(lib.gapa_cuda_eval_batch(obj.dgraph.handle, obj.task, genes.ctypes.data, rows, k, out.ctypes.data))
    dt = (time.perf_counter() - t0) / 5
    print(f"{os.environ.get('GAPA_PINNED_RING', '1')} ring, slice {os.environ.get('GAPA_PINNED_SLICE_MB', '16')} MB, copy {os.environ.get('GAPA_PINNED_RING_COPY', 'memcpy')}, threads {os.environ.get('GAPA_PINNED_RING_THREADS', 'default')}: "
          f"{dt * 1e3:.1f} ms per call, {rows / dt:.0f} evals/s, {4 * rows * k / dt / 1e9:.1f} GB/s")
elif len(sys.argv) > 1 and sys.argv[1] == "host":
    # the host's own copy ceiling, no GPU involved: N threads memcpy an 819 MB pageable array into another buffer
    import threading
    import time
    import numpy as np
    src = np.random.default_rng(1).integers(0, 1 << 20, size=4096 * 50_000, dtype=np.int32)
    dst = np.empty_like(src)
    for nthreads in (1, 2, 4, 8, 16):
        parts = np.array_split(np.arange(src.size), nthreads)
        bounds = [(int(p[0]), int(p[-1]) + 1) for p in parts]
        def run(lo, hi):
            np.copyto(dst[lo:hi], src[lo:hi])
        best = 1e9
        for _ in range(3):
            ts = [threading.Thread(target=run, args=b) for b in bounds]
            t0 = time.perf_counter()
            [t.start() for t in ts]
            [t.join() for t in ts]
            best = min(best, time.perf_counter() - t0)
        print(f"host copy (numpy.copyto releases the GIL), {nthreads} threads: {src.nbytes / best / 1e9:.1f} GB/s")
else:
    subprocess.call([sys.executable, __file__, "host"])
    for env in ({"GAPA_PINNED_RING_COPY": "memcpy", "GAPA_PINNED_RING_THREADS": "4"}, {"GAPA_PINNED_RING_COPY": "memcpy", "GAPA_PINNED_RING_THREADS": "8"},
                {"GAPA_PINNED_SLICE_MB": "4", "GAPA_PINNED_RING_THREADS": "8"}, {"GAPA_PINNED_SLICE_MB": "8", "GAPA_PINNED_RING_THREADS": "8"},
                {"GAPA_PINNED_SLICE_MB": "32", "GAPA_PINNED_RING_THREADS": "8"}, {"GAPA_PINNED_SLICE_MB": "64", "GAPA_PINNED_RING_THREADS": "8"},{"GAPA_PINNED_RING": "0"}, {"GAPA_PINNED_RING_THREADS": "1"}, {"GAPA_PINNED_RING_THREADS": "2"}, {"GAPA_PINNED_RING_THREADS": "4"},
                {"GAPA_PINNED_RING_THREADS": "8"}, {"GAPA_PINNED_RING_THREADS": "12"}, {"GAPA_PINNED_RING_THREADS": "16"}):
        subprocess.call([sys.executable, __file__, "child"], env={**os.environ, **env})
