"""ctypes binding of include/gapa_cuda.h — one Python function per exported symbol.

Loading fails loudly when the CUDA library has not been built; there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB, build

c_i32p = C.POINTER(C.c_int32)
c_f64p = C.POINTER(C.c_double)
c_u64p = C.POINTER(C.c_uint64)
VP = C.c_void_p


class GapaCudaError(RuntimeError):
    """Mirror of gapa::Error (include/gapa/error.hpp:9-30) for a non-zero C-ABI status."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


E_INVALID, E_RANGE, E_NAN, E_CUDA, E_NOMEM = 1, 2, 3, 4, 5


class RunParams(C.Structure):
    _fields_ = [("pc", C.c_double), ("pm", C.c_double), ("pop_size", C.c_int32), ("budget", C.c_int32),
                ("iterations", C.c_int32), ("minimize", C.c_int32), ("eda_interval", C.c_int32), ("task", C.c_int32),
                ("seed", C.c_uint64), ("rank", C.c_int32), ("world", C.c_int32)]


class RunResult(C.Structure):
    _fields_ = [("history_best", c_f64p), ("history_mean", c_f64p), ("final_population", c_i32p),
                ("final_fitness", c_f64p), ("fitness_batch_calls", C.c_uint64), ("total_wall_seconds", C.c_double),
                ("eval_seconds", C.c_double), ("gen_wall_seconds", c_f64p), ("gen_compute_seconds", c_f64p),
                ("gen_exchange_seconds", c_f64p), ("gen_lifecycle_seconds", c_f64p), ("gen_messages", C.POINTER(C.c_uint64))]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, VP, VP, C.c_int, C.c_int, VP)

# name -> (restype, argtypes); exactly the symbols include/gapa_cuda.h declares
SIGNATURES = {
    "gapa_cuda_last_error": (C.c_char_p, []),
    "gapa_cuda_abi_version": (C.c_int, []),
    "gapa_cuda_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "gapa_cuda_graph_create": (C.c_int, [C.c_int32, C.c_int64, VP, C.c_int, C.POINTER(VP)]),
    "gapa_cuda_graph_create_csr": (C.c_int, [C.c_int32, C.c_int64, VP, VP, C.c_int, C.POINTER(VP)]),
    "gapa_cuda_destroy": (C.c_int, [VP]),
    "gapa_cuda_graph_info": (C.c_int, [VP, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "gapa_cuda_pool_set": (C.c_int, [VP, C.c_int, C.c_int32, VP, VP]),
    "gapa_cuda_pool_info": (C.c_int, [VP, C.POINTER(C.c_int), C.POINTER(C.c_int32)]),
    "gapa_cuda_lp_split_set": (C.c_int, [VP, C.c_int32, VP, C.c_int32, VP]),
    "gapa_cuda_lp_score_set": (C.c_int, [VP, C.c_int]),
    "gapa_cuda_eval_batch": (C.c_int, [VP, C.c_int, VP, C.c_int, C.c_int, VP]),
    "gapa_cuda_eval_batch_device": (C.c_int, [VP, C.c_int, VP, C.c_int, C.c_int, VP, VP]),
    "gapa_cuda_ga_init_device": (C.c_int, [C.c_int32, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP, VP]),
    "gapa_cuda_ga_mask_device": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP, VP]),
    "gapa_cuda_ga_mutation_indices_device": (C.c_int, [C.c_int32, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP, VP]),
    "gapa_cuda_ga_mask": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP]),
    "gapa_cuda_ga_mutation_indices": (C.c_int, [C.c_int, C.c_int32, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP]),
    "gapa_cuda_ga_select_device": (C.c_int, [VP, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP, VP, VP]),
    "gapa_cuda_ga_crossover_mutate_device": (C.c_int, [VP, VP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                                       C.c_double, C.c_int32, C.c_uint64, C.c_uint64, VP, VP]),
    "gapa_cuda_ga_mutate_device": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int32, C.c_uint64,
                                             C.c_uint64, VP, VP]),
    "gapa_cuda_ga_eda_device": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.c_int32, C.c_uint64, C.c_uint64, C.c_int,
                                          VP, VP]),
    "gapa_cuda_ga_elitism_device": (C.c_int, [VP, VP, C.c_int, C.c_int, VP, VP, C.c_int, VP, VP, VP]),
    "gapa_cuda_ga_elitism_sharded_device": (C.c_int, [VP, VP, C.c_int, C.c_int, VP, C.c_int, C.c_int, VP, VP, C.c_int,
                                                      C.c_double, C.c_double, C.c_int32, C.c_uint64, C.c_uint64, VP, VP, VP]),
    "gapa_cuda_ga_slots_identity_device": (C.c_int, [C.c_int, VP, VP, VP]),
    "gapa_cuda_ga_slots_variation_device": (C.c_int, [VP, VP, VP, VP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                                      C.c_double, C.c_int32, C.c_uint64, C.c_uint64, VP]),
    "gapa_cuda_ga_slots_variation_eval_device": (C.c_int, [VP, C.c_int, VP, VP, VP, VP, C.c_int, C.c_int, C.c_int, C.c_int,
                                                           C.c_double, C.c_double, C.c_uint64, C.c_uint64, VP, VP]),
    "gapa_cuda_ga_slots_elitism_device": (C.c_int, [VP, VP, VP, VP, C.c_int, C.c_int, C.c_int, C.c_int, VP, VP, C.c_int,
                                                    C.c_double, C.c_double, C.c_int32, C.c_uint64, C.c_uint64, VP, VP, VP, VP]),
    "gapa_cuda_ga_slots_gather_device": (C.c_int, [VP, VP, C.c_int, C.c_int, VP, VP]),
    "gapa_cuda_eval_rows_device": (C.c_int, [VP, C.c_int, VP, VP, C.c_int, C.c_int, VP, VP]),
    "gapa_cuda_ga_stats_device": (C.c_int, [VP, C.c_int, VP, VP, VP]),
    "gapa_cuda_ga_init": (C.c_int, [C.c_int, C.c_int32, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP]),
    "gapa_cuda_ga_selection_weights": (C.c_int, [C.c_int, VP, C.c_int, C.c_int, VP]),
    "gapa_cuda_ga_select": (C.c_int, [C.c_int, VP, C.c_int, C.c_int, C.c_uint64, C.c_uint64, VP]),
    "gapa_cuda_ga_crossover_mutate": (C.c_int, [C.c_int, VP, VP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                                C.c_double, C.c_int32, C.c_uint64, C.c_uint64, VP]),
    "gapa_cuda_ga_mutate": (C.c_int, [C.c_int, VP, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int32, C.c_uint64,
                                      C.c_uint64, VP]),
    "gapa_cuda_ga_eda": (C.c_int, [C.c_int, VP, C.c_int, C.c_int, C.c_int, C.c_int32, C.c_uint64, C.c_uint64, C.c_int,
                                   VP]),
    "gapa_cuda_ga_elitism": (C.c_int, [C.c_int, VP, VP, C.c_int, C.c_int, VP, VP, C.c_int, VP, VP]),
    "gapa_cuda_rng_draws": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, VP]),
    "gapa_cuda_run": (C.c_int, [VP, C.POINTER(RunParams), ALLGATHER_FN, VP, C.POINTER(RunResult)]),
    "gapa_cuda_ga_create": (C.c_int, [VP, C.POINTER(RunParams), ALLGATHER_FN, VP, C.c_int, C.POINTER(VP)]),
    "gapa_cuda_ga_advance": (C.c_int, [VP, C.c_int, C.POINTER(C.c_float)]),
    "gapa_cuda_ga_generation": (C.c_int, [VP, C.POINTER(C.c_int)]),
    "gapa_cuda_ga_result": (C.c_int, [VP, C.POINTER(RunResult)]),
    "gapa_cuda_ga_destroy": (C.c_int, [VP]),
    "gapa_cuda_comm_create": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.POINTER(VP), VP]),
    "gapa_cuda_comm_connect": (C.c_int, [VP, VP]),
    "gapa_cuda_nccl_unique_id": (C.c_int, [VP]),
    "gapa_cuda_comm_create_nccl": (C.c_int, [VP, VP, C.c_int, C.c_int, C.POINTER(VP)]),
    "gapa_cuda_comm_allgather": (C.c_int, [VP, VP, C.c_int, C.c_int, VP]),
    "gapa_cuda_comm_allgather_bytes": (C.c_int, [VP, VP, C.c_int, VP]),
    "gapa_cuda_comm_status": (C.c_int, [VP]),
    "gapa_cuda_comm_info": (C.c_int, [VP, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "gapa_cuda_comm_destroy": (C.c_int, [VP]),
    "gapa_cuda_run_multi": (C.c_int, [C.POINTER(VP), C.c_int, C.POINTER(RunParams), C.c_int, C.POINTER(RunResult)]),
    "gapa_host_barabasi_albert": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, VP, C.c_int64, C.POINTER(C.c_int64)]),
    "gapa_host_erdos_renyi": (C.c_int, [C.c_int32, C.c_double, C.c_uint64, VP, C.c_int64, C.POINTER(C.c_int64)]),
    "gapa_host_planted_partition": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, VP, C.c_int64,
                                              C.POINTER(C.c_int64)]),
    "gapa_host_lp_split": (C.c_int, [C.c_int32, C.c_int64, VP, C.c_double, C.c_uint64, VP, VP, VP,
                                     C.POINTER(C.c_int32)]),
    "gapa_cuda_detect_communities": (C.c_int, [VP, VP, C.c_int, VP, C.POINTER(C.c_double)]),
    "gapa_cuda_lpa_scores": (C.c_int, [VP, VP, C.c_int, VP, VP, C.POINTER(C.c_double)]),
    "gapa_host_budget": (C.c_int, [C.c_int64, C.c_double, C.POINTER(C.c_int32)]),
    "gapa_host_nonedges": (C.c_int, [C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "gapa_cuda_malloc": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(VP)]),
    "gapa_cuda_free": (C.c_int, [C.c_int, VP]),
    "gapa_cuda_memcpy_h2d": (C.c_int, [C.c_int, VP, VP, C.c_uint64]),
    "gapa_cuda_memcpy_d2h": (C.c_int, [C.c_int, VP, VP, C.c_uint64]),
    "gapa_cuda_stream_sync": (C.c_int, [C.c_int, VP]),
    "gapa_cuda_launch_count": (C.c_uint64, []),
    "gapa_cuda_last_eval_ms": (C.c_int, [VP, C.POINTER(C.c_float)]),
}

_lib = None


def load(rebuild_if_stale: bool = True) -> C.CDLL:
    """dlopen the in-tree library (building it first when sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    path = LIB
    if rebuild_if_stale and os.environ.get("GAPA_B200_NO_REBUILD") != "1":
        try:
            path = build()
        except Exception:
            if not os.path.exists(LIB):
                raise
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_2412_20980_b200.build`; "
                           "there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError here == a symbol the header declares is not exported
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        raise GapaCudaError(status, load().gapa_cuda_last_error().decode())
