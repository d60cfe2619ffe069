"""ctypes mirror of include/tpgen.h (argument marshalling only)."""
from __future__ import annotations

import ctypes
import os

from ctypes import (CFUNCTYPE, POINTER, Structure, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t,
                    c_uint64, c_void_p)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtpgen.so")

TPGEN_OK = 0
STATUS_NAMES = {
    0: "TPGEN_OK", 1: "TPGEN_ERR_INVALID_ARGUMENT", 2: "TPGEN_ERR_INVALID_GRAPH",
    3: "TPGEN_ERR_LIMIT_EXCEEDED", 4: "TPGEN_ERR_OUT_OF_MEMORY", 5: "TPGEN_ERR_UNREACHABLE",
    6: "TPGEN_ERR_CUDA", 7: "TPGEN_ERR_INTERNAL", 8: "TPGEN_ERR_UNSUPPORTED",
}
OUT_MATERIALIZE = 0
OUT_COUNT_HASH = 1
ENGINE_DFS = 0
ENGINE_FRONTIER = 1
ENGINE_ALG3 = 2
TP_PER_PP = 0
TP_UNIQUE = 1
TP_GREEDY = 2

ALLOC_FN = CFUNCTYPE(c_void_p, c_size_t, c_void_p, c_void_p)
FREE_FN = CFUNCTYPE(None, c_void_p, c_void_p, c_void_p)


class Paths(Structure):
    _fields_ = [("n_paths", c_int64), ("offsets", POINTER(c_int64)), ("vertices", POINTER(c_int32)),
                ("on_device", c_int32), ("device", c_int32), ("_owner", c_void_p)]


class Options(Structure):
    _fields_ = [("device", c_int32), ("stream", c_void_p), ("output_on_device", c_int32),
                ("output_mode", c_int32), ("shard_rank", c_int32), ("shard_count", c_int32),
                ("start_lo", c_int32), ("start_hi", c_int32),
                ("max_paths", c_int64), ("max_extensions", c_int64), ("tp_mode", c_int32),
                ("compute_digest", c_int32), ("device_alloc", ALLOC_FN), ("device_free", FREE_FN),
                ("alloc_ctx", c_void_p), ("host_out", c_void_p), ("host_out_bytes", c_size_t),
                ("engine", c_int32), ("no_plan_cache", c_int32), ("shard_prefix", c_int32),
                ("prune", c_int32)]


class Metrics(Structure):
    _fields_ = [("nodes", c_int64), ("edges", c_int64), ("sccs", c_int64), ("scc_nodes", c_int64),
                ("scc_edges", c_int64), ("weak_components", c_int64), ("cc", c_int64), ("npath", c_uint64),
                ("npath_status", c_int32), ("pad", c_int32)]


class Stats(Structure):
    _fields_ = [("n_paths", c_int64), ("total_vertices", c_int64), ("n_extensions", c_int64),
                ("n_cross", c_int64), ("n_units", c_int64), ("n_heads", c_int64), ("n_segments", c_int64),
                ("hash_lo", c_uint64), ("hash_hi", c_uint64), ("n_scc", c_int32),
                ("n_scc_nontrivial", c_int32), ("max_scc", c_int32), ("n_count_rounds", c_int32),
                ("gpu_launches", c_int64), ("shard_lo", c_int32), ("shard_hi", c_int32),
                ("ms_plan", c_double), ("ms_count", c_double), ("ms_write", c_double), ("ms_stitch", c_double),
                ("ms_device", c_double), ("ms_total", c_double), ("ms_dfs_write", c_double),
                ("ms_dfs_count", c_double), ("ms_linearize", c_double), ("ms_dominant", c_double),
                ("ext_dominant", c_int64), ("unit_lo", c_int64), ("unit_hi", c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


# Every symbol declared in include/tpgen.h (tests check the library exports them all).
SYMBOLS = {
    "tpgen_options_init": (None, [POINTER(Options)]),
    "tpgen_status_string": (c_char_p, [c_int]),
    "tpgen_last_error_message": (c_char_p, []),
    "tpgen_version": (c_char_p, []),
    "tpgen_prime_paths": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, POINTER(Options),
                                  POINTER(Paths), POINTER(Stats)]),
    "tpgen_test_paths": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, POINTER(Paths), c_int32, c_int32,
                                 POINTER(Options), POINTER(Paths), POINTER(Stats)]),
    "tpgen_paths_free": (None, [POINTER(Paths)]),
    "tpgen_components": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, POINTER(c_int32), POINTER(c_int32),
                                 POINTER(c_int32)]),
    "tpgen_shard_range": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, c_int32, c_int32, POINTER(c_int32),
                                  POINTER(c_int32)]),
    "tpgen_shard_units": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, c_int32, c_int32, POINTER(c_int32),
                                  POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int32),
                                  POINTER(c_int32)]),
    "tpgen_shard_unit_paths": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, c_int32, c_int32,
                                       POINTER(c_int64), POINTER(c_int32), POINTER(c_int32), c_int64, c_int64,
                                       POINTER(c_int64), POINTER(c_int64)]),
    "tpgen_metrics_compute": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, c_int32, c_int32,
                                      POINTER(Metrics)]),
    "tpgen_normalize_outdeg2": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, POINTER(c_int32),
                                        POINTER(c_int64), POINTER(c_int64), POINTER(c_int32), POINTER(c_int32)]),
    "tpgen_plan_create": (c_int, [POINTER(c_int64), POINTER(c_int32), c_int32, POINTER(Options),
                                  POINTER(c_void_p)]),
    "tpgen_plan_prime_paths": (c_int, [c_void_p, POINTER(Options), POINTER(Paths), POINTER(Stats)]),
    "tpgen_plan_test_paths": (c_int, [c_void_p, POINTER(Paths), c_int32, c_int32, POINTER(Options), POINTER(Paths),
                                      POINTER(Stats)]),
    "tpgen_plan_classify": (c_int, [c_void_p, POINTER(Paths), c_int32, c_int32, POINTER(Options),
                                    POINTER(c_int64)]),
    "tpgen_plan_destroy": (None, [c_void_p]),
    "tpgen_release_cache": (None, []),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libtpgen.so; raises if the CUDA library has not been built (no fallback).
    TPGEN_LIB_VARIANT=<name> loads the experiment build libtpgen_<name>.so instead."""
    global _lib
    if _lib is None:
        if os.environ.get("TPGEN_LIB_VARIANT"):
            path = os.path.join(HERE, f"libtpgen_{os.environ['TPGEN_LIB_VARIANT']}.so")
        if not os.path.exists(path):
            # build the CUDA library in-tree (nvcc, sm_100a) -- never a fallback: if nvcc
            # fails the import fails
            import sys

            from . import build as _build

            sys.stderr.write(f"[tpgen] {path} missing: building it with nvcc (sm_100a)\n")
            try:
                _build.build()
            except Exception as e:  # noqa: BLE001
                raise ImportError(f"libtpgen.so not found at {path} and the nvcc build failed: {e}") from e
        lib = ctypes.CDLL(path)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
