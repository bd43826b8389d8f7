"""ctypes binding of the C-ABI in include/cfcent_b200.h.

The shared library ``libcfcent_b200.so`` is built in-tree by
``paper_1607_02955_b200._build.build()`` (nvcc, sm_100a).  There is no
fallback: if the library is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import ConvergenceError, DomainError

HERE = os.path.dirname(os.path.abspath(__file__))
# CF_LIB_VARIANT=<name> loads an experiment build libcfcent_b200_<name>.so
# (_build.py ``variant``); the default is the product library.
LIB_PATH = os.path.join(HERE, "libcfcent_b200.so" if not os.environ.get("CF_LIB_VARIANT")
                        else f"libcfcent_b200_{os.environ['CF_LIB_VARIANT']}.so")

CF_OK, CF_DOMAIN, CF_CONVERGENCE, CF_RUNTIME = 0, 1, 2, 3

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class CfLevelDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("n", C.c_int32), ("n_coarse", C.c_int32),
        ("nnz_off", C.c_int64), ("rowptr", i64p), ("col", i32p), ("val", f64p), ("diag", f64p),
        ("n_colors", C.c_int32), ("color_ptr", i32p), ("color_rows", i32p),
        ("agg", i32p), ("agg_ptr", i32p), ("agg_members", i32p),
        ("n_f", C.c_int32), ("f_nodes", i32p), ("c_nodes", i32p), ("f_degree", f64p),
        ("wcf_ptr", i64p), ("wcf_col", i32p), ("wcf_val", f64p),
        ("wfc_ptr", i64p), ("wfc_col", i32p), ("wfc_val", f64p),
        ("coarse_op", f64p),
    ]


class CfSolveParams(C.Structure):
    _fields_ = [
        ("tau", C.c_double), ("max_cycles", C.c_int32), ("nu1", C.c_int32), ("nu2", C.c_int32),
        ("fcg_max_iters", C.c_int32), ("jpcg_max_iters", C.c_int32),
        ("stop_margin", C.c_double), ("stagnation_factor", C.c_double),
        ("stagnation_cycles", C.c_int32),
    ]


class CfSolveStats(C.Structure):
    _fields_ = [
        ("solves", C.c_int64), ("fallback_solves", C.c_int64), ("vcycles", C.c_int64),
        ("outer_iterations", C.c_int64), ("max_residual", C.c_double),
        ("best_residual", C.c_double), ("krylov_solves", C.c_int64),
    ]


_lib = None
_lock = threading.Lock()

_SIGS = {
    "cf_last_error": (C.c_char_p, []),
    "cf_version": (C.c_int, []),
    "cf_device_count": (C.c_int, []),
    "cf_hier_create": (C.c_int, [C.c_int32, C.POINTER(CfLevelDesc), C.c_int32,
                                 C.POINTER(C.c_void_p)]),
    "cf_hier_destroy": (C.c_int, [C.c_void_p]),
    "cf_hier_device_bytes": (C.c_int64, [C.c_void_p]),
    "cf_hier_set_order": (C.c_int, [C.c_void_p, i32p, C.c_int64]),
    "cf_solve_rows": (C.c_int, [C.c_void_p, f64p, C.c_int64, C.POINTER(CfSolveParams), f64p,
                                f64p, C.POINTER(CfSolveStats)]),
    "cf_solve_block_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                     C.POINTER(CfSolveParams), f64p, C.POINTER(CfSolveStats),
                                     C.c_void_p]),
    "cf_residual_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  f64p, C.c_void_p]),
    "cf_graph_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, i64p, i32p, i32p, f64p,
                                  C.POINTER(C.c_void_p)]),
    "cf_graph_destroy": (C.c_int, [C.c_void_p]),
    "cf_jl_rhs_rows": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                 C.c_int64, C.c_int64, C.c_int32, f64p]),
    "cf_jl_sketch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                               C.c_int64, C.c_int64, C.c_int64, C.c_double, i64p, C.c_int64,
                               C.POINTER(CfSolveParams), f64p, f64p, f64p, f64p,
                               C.POINTER(CfSolveStats)]),
    "cf_jl_combine": (C.c_int, [f64p, C.c_int64, C.c_int64, C.c_int64, f64p]),
    "cf_node_solutions": (C.c_int, [C.c_void_p, i64p, C.c_int64, C.POINTER(CfSolveParams), f64p,
                                    f64p, f64p, C.POINTER(CfSolveStats)]),
    "cf_exact_sums": (C.c_int, [C.c_void_p, i64p, C.c_int64, C.POINTER(CfSolveParams), f64p,
                                f64p, C.POINTER(CfSolveStats)]),
    "cf_hier_stream": (C.c_void_p, [C.c_void_p]),
    "cf_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "cf_profile_report": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, i64p]),
    "cf_setup_elim_select": (C.c_int, [C.c_int64, i64p, i64p, C.c_int32, i64p, i64p]),
    "cf_setup_aggregate": (C.c_int, [C.c_int64, i64p, i64p, f64p, C.c_int32, C.c_int32,
                                     C.c_double, i64p, i64p]),
    "cf_setup_matching": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, i64p, i64p, i64p]),
    "cf_setup_colour": (C.c_int, [C.c_int64, i64p, i64p, i32p, i32p]),
    "cf_setup_permute": (C.c_int, [C.c_int64, i64p, i64p, f64p, i64p, i64p, i64p, i64p, f64p]),
    "cf_rebuild_laplacian": (C.c_int, [C.c_int64, i64p, i64p, f64p, i64p, i64p, f64p, i64p]),
    "cf_build_csr": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, f64p, i64p, i64p, f64p, i64p]),
    "cf_csr_from_edges_dev": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, i64p, i64p, f64p, i64p,
                                        i64p, f64p, i32p]),
    "cf_components_dev": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, i64p, i64p, i64p, i32p]),
    "cf_coarse_operator_dev": (C.c_int, [C.c_int32, C.c_int64, i64p, i64p, f64p, i64p, C.c_int64,
                                         C.c_int64, i64p, i64p]),
    "cf_coarse_fetch_dev": (C.c_int, [i64p, i64p, f64p]),
    "cf_setup_relax": (C.c_int, [C.c_int64, i64p, i64p, f64p, C.c_int32, C.c_int32, f64p]),
    "cf_validate_laplacian_dev": (C.c_int, [C.c_int32, C.c_int64, i64p, i64p, f64p, f64p, i64p]),
}


def lib():
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` "
                        "(there is no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, stats: CfSolveStats | None = None):
    if status == CF_OK:
        return
    msg = lib().cf_last_error().decode(errors="replace")
    if status == CF_DOMAIN:
        raise DomainError(msg)
    if status == CF_CONVERGENCE:
        # the library formats the message; ConvergenceError appends the residual
        best = stats.best_residual if stats is not None else float("nan")
        raise ConvergenceError(msg, best)
    raise RuntimeError(f"cfcent_b200 native failure: {msg}")


def ptr(a: np.ndarray | None, t):
    if a is None:
        return C.cast(None, t)
    return a.ctypes.data_as(t)


def device_available() -> bool:
    try:
        return lib().cf_device_count() > 0
    except Exception:
        return False
