"""ctypes binding of liblamg_b200.so (include/lamg_b200.h).

The shared library is the product: hand-written sm_100a CUDA behind a C-ABI.
There is no CPU path -- if the library is missing or no CUDA device is
present, the calls below raise instead of falling back.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblamg_b200.so")

# exported symbols declared in include/lamg_b200.h (checked by tests/test_capi_symbols.py)
HEADER = os.path.join(os.path.dirname(HERE), "include", "lamg_b200.h")

_lib = None


class lamg_csr(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int64), ("row_ptr", C.c_void_p), ("col", C.c_void_p),
                ("val", C.c_void_p), ("diag", C.c_void_p)]


class lamg_setup_opts(C.Structure):
    _fields_ = [("gamma", C.c_double), ("rng_seed", C.c_uint64), ("coarsest_n", C.c_int32),
                ("tv_sweeps", C.c_int32), ("tv_count_finest", C.c_int32), ("tv_count_max", C.c_int32)]


class lamg_cycle_cfg(C.Structure):
    _fields_ = [("gamma", C.c_double), ("correction", C.c_int32), ("mu", C.c_double),
                ("max_cycles", C.c_int32), ("target_reduction", C.c_double),
                ("divergence_factor", C.c_double), ("rng_seed", C.c_uint64)]


class lamg_solve_stats(C.Structure):
    _fields_ = [("acf", C.c_double), ("solve_work", C.c_double), ("cycles", C.c_int32),
                ("converged", C.c_int32), ("recombinations", C.c_int64), ("recomb_max_growth", C.c_double),
                ("nresiduals", C.c_int32), ("relax_sweeps", C.c_int32)]


class lamg_level_info(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("m", C.c_int64), ("gamma", C.c_double),
                ("nu_pre", C.c_int32), ("nu_post", C.c_int32), ("tv_count", C.c_int32),
                ("coarsest", C.c_int32), ("nstages", C.c_int32), ("coarse_n", C.c_int32),
                ("alpha", C.c_double), ("stage_used", C.c_int32), ("dummy_aggregate", C.c_int32),
                ("gs_fronts", C.c_int32), ("colors", C.c_int32)]


def lib():
    """Loads liblamg_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C paper_1108_1310_b200/csrc` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.lamg_last_error.restype = C.c_char_p
        L.lamg_version.restype = C.c_char_p
        L.lamg_flat_mu.restype = C.c_double
        L.lamg_flat_mu.argtypes = [C.c_double]
        L.lamg_rng_derive.restype = C.c_uint64
        L.lamg_rng_derive.argtypes = [C.c_uint64, C.c_uint64]
        L.lamg_ctx_destroy.restype = None
        L.lamg_hier_destroy.restype = None
        L.lamg_graph_destroy.restype = None
        L.lamg_comm_destroy.restype = None
        L.lamg_part_level_destroy.restype = None
        L.lamg_mm_destroy.restype = None
        _lib = L
    return _lib


def declared_symbols() -> list[str]:
    """Function names declared in include/lamg_b200.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lamg_[a-z0-9_]+)\s*\(", txt)))
