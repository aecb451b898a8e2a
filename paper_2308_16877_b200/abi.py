"""ctypes view of the C-ABI in include/hpac_offload.h.

Struct layouts mirror the header field for field. This module only loads
the in-tree product library (paper_2308_16877_b200/libhpac_b200.so); it
fails loudly when it is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("HPAC_LIB", PKG / "libhpac_b200.so"))  # HPAC_LIB: tuning builds only

# ---- status / enums (hpac_offload.h) -------------------------------------
OK, ERR_CONFIG, ERR_ARENA_OVERFLOW, ERR_BARRIER_DIVERGENCE, ERR_CUDA, ERR_DIRECTIVE, ERR_UNSUPPORTED = range(7)
MAP_PER_THREAD, MAP_PER_TEAM = 0, 1
TECH_TAF, TECH_IACT, TECH_PERFO = 0, 1, 2
LEVEL_THREAD, LEVEL_WARP, LEVEL_TEAM = 0, 1, 2
PERFO_SMALL, PERFO_LARGE, PERFO_INI, PERFO_FINI, PERFO_HERDED_SMALL, PERFO_HERDED_LARGE, PERFO_RANDOM = range(7)
APP_TABLE, APP_SYNTHETIC, APP_BLACKSCHOLES, APP_BINOMIAL, APP_KMEANS, APP_LAVAMD = range(6)
SYNTH_CONSTANT, SYNTH_SLOW_DRIFT, SYNTH_NOISE = range(3)
REGION_STORE_ACCUMULATE = 1
REGION_BARRIER_IN_EVALUATE = 2
REGION_KMEANS_FAST_MATH = 4

PERFO_KINDS = {"small": PERFO_SMALL, "large": PERFO_LARGE, "ini": PERFO_INI, "fini": PERFO_FINI,
               "herded_small": PERFO_HERDED_SMALL, "herded_large": PERFO_HERDED_LARGE,
               "random": PERFO_RANDOM}
LEVELS = {"thread": LEVEL_THREAD, "warp": LEVEL_WARP, "team": LEVEL_TEAM, "block": LEVEL_TEAM}


class Grid(C.Structure):
    _fields_ = [("num_teams", C.c_int32), ("threads_per_team", C.c_int32),
                ("warp_size", C.c_int32), ("items_per_thread", C.c_int32),
                ("shared_mem_budget_bytes", C.c_uint64)]


class Spec(C.Structure):
    _fields_ = [("technique", C.c_int32), ("level", C.c_int32),
                ("taf_h_size", C.c_int32), ("taf_p_size", C.c_int32), ("taf_threshold", C.c_double),
                ("iact_table_size", C.c_int32), ("iact_tables_per_warp", C.c_int32),
                ("iact_threshold", C.c_double),
                ("perfo_kind", C.c_int32), ("perfo_modulus", C.c_int32),
                ("perfo_skip_percent", C.c_int32), ("reserved0", C.c_int32),
                ("perfo_seed", C.c_uint64),
                ("n_input_sections", C.c_int32), ("n_output_sections", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("total_invocations", C.c_uint64), ("approx_invocations", C.c_uint64),
                ("divergent_warp_steps", C.c_uint64), ("total_warp_steps", C.c_uint64),
                ("resident_warps", C.c_int32), ("barrier_divergence_detected", C.c_int32),
                ("arena_required", C.c_uint64), ("arena_available", C.c_uint64),
                ("fail_step", C.c_int64), ("fail_team", C.c_int32), ("fail_missing", C.c_int32),
                ("kernel_ms", C.c_double), ("lattice_fallbacks", C.c_uint64),
                ("lattice_nodes", C.c_uint64), ("zero_copy", C.c_int32), ("reserved0", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Region(C.Structure):
    _fields_ = [("app", C.c_int32), ("input_dims", C.c_int32), ("output_dims", C.c_int32),
                ("flags", C.c_int32), ("synthetic_profile", C.c_int32),
                ("binomial_steps", C.c_int32), ("binomial_american", C.c_int32),
                ("binomial_put", C.c_int32), ("kmeans_dims", C.c_int32), ("kmeans_k", C.c_int32),
                ("lavamd_boxes1d", C.c_int32), ("lavamd_particles", C.c_int32),
                ("seed", C.c_uint64), ("lavamd_alpha", C.c_double),
                ("in_", C.c_void_p), ("table_out", C.c_void_p), ("encounters", C.c_void_p),
                ("out", C.c_void_p), ("centroids", C.c_void_p), ("labels", C.c_void_p)]


class Launch(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("team_begin", C.c_int32), ("team_end", C.c_int32),
                ("paths", C.c_void_p), ("synchronous", C.c_int32), ("reserved", C.c_int32)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
KMEANS_CENTROIDS_GIVEN = 8
KMEANS_HOST_LOOP = 16


class KmeansProblem(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("dims", C.c_int32), ("k", C.c_int32),
                ("points", C.c_void_p), ("centroids", C.c_void_p), ("assignments", C.c_void_p),
                ("max_iters", C.c_int32), ("flags", C.c_int32), ("perfo_seed_base", C.c_uint64),
                ("allreduce", ALLREDUCE_FN), ("allreduce_user", C.c_void_p),
                ("reduce_buf", C.c_void_p)]


class KmeansResult(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("stats", Stats),
                ("region_ms", C.c_double), ("update_ms", C.c_double), ("graph", C.c_int32)]


def _declare(lib):
    P = C.POINTER
    sig = {
        "hpac_abi_version": (C.c_int, []),
        "hpac_status_name": (C.c_char_p, [C.c_int]),
        "hpac_resolve_grid": (C.c_int, [C.c_char_p, C.c_int64, P(Grid), P(Grid), P(C.c_int32), C.c_char_p, C.c_size_t]),
        "hpac_parse_directive": (C.c_int, [C.c_char_p, P(Spec), P(C.c_int32), P(C.c_int64), C.c_char_p, C.c_size_t]),
        "hpac_unparse": (C.c_int, [P(Spec), C.c_char_p, C.c_size_t]),
        "hpac_region_bind": (C.c_int, [P(Region), C.c_char_p, C.c_size_t]),
        "hpac_arena_required": (C.c_int, [P(Grid), P(Region), P(Spec), P(C.c_uint64), P(C.c_uint64), C.c_char_p, C.c_size_t]),
        "hpac_run_region": (C.c_int, [P(Grid), C.c_int64, C.c_int32, P(Region), P(Spec), P(Launch), P(Stats), C.c_char_p, C.c_size_t]),
        "hpac_run_region_host": (C.c_int, [P(Grid), C.c_int64, C.c_int32, P(Region), P(Spec), P(Stats), C.c_char_p, C.c_size_t]),
        "hpac_run_region_host_teams": (C.c_int, [P(Grid), C.c_int64, C.c_int32, P(Region), P(Spec), C.c_int32, C.c_int32,
                                                 P(Stats), C.c_char_p, C.c_size_t]),
        "hpac_stats_fetch": (C.c_int, [P(Stats)]),
        "hpac_kmeans_run": (C.c_int, [P(Grid), P(KmeansProblem), P(Spec), C.c_void_p, P(KmeansResult), C.c_char_p, C.c_size_t]),
        "hpac_make_bs_portfolio": (C.c_int, [C.c_int64, C.c_uint64, C.c_int32, C.c_double, C.c_void_p]),
        "hpac_make_binomial_portfolio": (C.c_int, [C.c_int64, C.c_uint64, C.c_double, C.c_void_p]),
        "hpac_make_blobs": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_void_p]),
        "hpac_mape": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, P(C.c_double)]),
        "hpac_mcr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, P(C.c_double)]),
        "hpac_probe_fp64_peak": (C.c_int, [P(C.c_double)]),
        "hpac_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "hpac_nccl_allreduce": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
        "hpac_nccl_check": (C.c_int, [C.c_void_p]),
        "hpac_nccl_comm_init_rank": (C.c_int, [C.c_int, C.c_char_p, C.c_int, P(C.c_void_p)]),
        "hpac_probe_dmma_peak": (C.c_int, [P(C.c_double)]),
        "hpac_make_lavamd": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]),
        "hpac_fm_eval": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_LIB = None


def lib():
    """The product library; raises if it has not been built."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(the CUDA path has no CPU fallback)")
        _LIB = _declare(C.CDLL(str(LIB_PATH)))
    return _LIB


def exported_symbols():
    """Names declared in include/*.h (checked against the .so exports)."""
    import re
    names = []
    for h in (PKG.parent / "include").glob("*.h"):
        names += re.findall(r"^\s*(?:int|const char\*)\s+(hpac_\w+)\s*\(", h.read_text(), re.M)
    return sorted(set(names))
