"""Could a pageable batch be pinned IN PLACE instead of being copied into a pinned ring?  Times cudaHostRegister +
cudaHostUnregister over an 819 MB pageable array in slices, from 1..8 host threads.  usage: python tools/probe_hostregister.py"""
import ctypes as C
import threading
import time

import numpy as np
import torch  # noqa: F401  (loads libcudart and creates the context)

torch.cuda.init()
torch.zeros(1, device="cuda")
rt = C.CDLL("libcudart.so.12")
src = np.random.default_rng(1).integers(0, 1 << 20, size=4096 * 50_000, dtype=np.int32)
base = src.ctypes.data
for slice_mb in (16, 64):
    step = slice_mb << 20
    offs = list(range(0, src.nbytes - step + 1, step))
    for nthreads in (1, 2, 4, 8):
        def run(mine):
            for off in mine:
                a = (base + off + 4095) & ~4095
                rc = rt.cudaHostRegister(C.c_void_p(a), C.c_size_t(step - 4096), C.c_uint(0))
                assert rc == 0, rc
                rc = rt.cudaHostUnregister(C.c_void_p(a))
                assert rc == 0, rc
        parts = [offs[i::nthreads] for i in range(nthreads)]
        ts = [threading.Thread(target=run, args=(p,)) for p in parts]
        t0 = time.perf_counter()
        [t.start() for t in ts]
        [t.join() for t in ts]
        dt = time.perf_counter() - t0
        print(f"register+unregister {slice_mb} MB slices, {nthreads} threads: {len(offs) * step / dt / 1e9:.1f} GB/s ({dt * 1e3:.0f} ms for the batch)")
