"""ctypes binding of libssqa_b200.so (include/ssqa_cuda.h + include/ssqa_host.h).

The library is built in-tree by ``paper_2302_12454_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("SSQA_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libssqa_b200.so")

SSQA_OK, SSQA_EINVAL, SSQA_ERANGE, SSQA_ECUDA, SSQA_EUNSUP = 0, 1, 2, 3, 4
ENGINE_AUTO, ENGINE_SIMT, ENGINE_TCGEN05 = 0, 1, 2
ENGINE_NAMES = {ENGINE_SIMT: "simt", ENGINE_TCGEN05: "tcgen05"}


class ParamsC(C.Structure):
    """ssqa_params_c == ssqa::SsqaParams (annealer.hpp:14-30)."""
    _fields_ = [
        ("r", C.c_int), ("jperp_min", C.c_double), ("jperp_max", C.c_double),
        ("beta", C.c_int), ("tau", C.c_int), ("delay", C.c_int), ("i0", C.c_double),
        ("n_rnd", C.c_double), ("alpha", C.c_double), ("sc", C.c_long),
        ("bidirectional", C.c_int),
    ]


class SsaParamsC(C.Structure):
    """ssqa_ssa_params_c == ssqa::SsaParams (annealer.hpp:38-50)."""
    _fields_ = [
        ("i0_min", C.c_double), ("i0_max", C.c_double), ("beta", C.c_double),
        ("tau", C.c_int), ("n_rnd", C.c_double), ("alpha", C.c_double), ("sc", C.c_long),
    ]


class ResultC(C.Structure):
    """ssqa_result_c == scalar fields of ssqa::AnnealResult (annealer.hpp:102-111)."""
    _fields_ = [
        ("best_energy", C.c_double), ("best_replica", C.c_int), ("reached_target", C.c_int),
        ("first_hit_cycle", C.c_long), ("cycles_used", C.c_long), ("wall_seconds", C.c_double),
    ]


# (name, restype, argtypes) for every exported C entry point.
VP, DP, I8P, U64P = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int8), C.POINTER(C.c_uint64)
IP, LP = C.POINTER(C.c_int), C.POINTER(C.c_long)
SIGNATURES = [
    ("ssqa_last_error", C.c_char_p, []),
    ("ssqa_version", C.c_char_p, []),
    ("ssqa_pool_trim", C.c_longlong, [C.c_int]),
    ("ssqa_tune_set", C.c_int, [C.c_char_p, C.c_long]),
    ("ssqa_tune_trace", C.c_int, [C.c_char_p]),
    ("ssqa_tune_reset", None, []),
    ("ssqa_pool_stats", C.c_int, [C.c_int, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    ("ssqa_problem_create", C.c_int, [C.c_int, DP, DP, C.c_double, C.c_int, C.POINTER(VP)]),
    ("ssqa_problem_destroy", C.c_int, [VP]),
    ("ssqa_problem_create_many", C.c_int, [C.c_int, C.c_int, DP, DP, DP, C.c_int,
                                           C.POINTER(VP)]),
    ("ssqa_problem_count", C.c_int, [VP]),
    ("ssqa_problem_create_dense", C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_void_p]),
    ("ssqa_problem_create_gi", C.c_int, [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                         C.c_double, C.c_double, C.c_int, C.c_void_p]),
    ("ssqa_problem_create_zero", C.c_int, [C.c_int, C.c_int, C.c_void_p]),
    ("ssqa_problem_export", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("ssqa_gi_compact", C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_double,
                                  C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("ssqa_problem_info", C.c_int, [VP, IP, IP, IP, IP, IP]),
    ("ssqa_quantize_info", C.c_int, [C.c_int, DP, DP, IP, IP, IP, IP]),
    ("ssqa_plan_geometry", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, IP, IP, IP, IP]),
    ("ssqa_problem_fp4", C.c_int, [VP]),
    ("ssqa_problem_int16", C.c_int, [C.c_void_p]),
    ("ssqa_params_validate", C.c_int, [C.POINTER(ParamsC), C.c_int]),
    ("ssqa_jperp_schedule", C.c_int, [C.c_long, C.POINTER(ParamsC), DP]),
    ("ssqa_run_batch", C.c_int, [VP, C.POINTER(ParamsC), U64P, C.c_int, C.c_int, C.c_double,
                                 C.c_int, C.c_int, C.c_int, C.POINTER(ResultC), I8P, DP]),
    ("ssqa_ssa_params_validate", C.c_int, [C.POINTER(SsaParamsC), C.c_int]),
    ("ssqa_i0_schedule", C.c_int, [C.c_long, C.POINTER(SsaParamsC), DP]),
    ("ssqa_i0_levels", C.c_int, [C.POINTER(SsaParamsC), DP, IP]),
    ("ssqa_ssa_run_batch", C.c_int, [VP, C.POINTER(SsaParamsC), U64P, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(ResultC), I8P, DP]),
    ("ssqa_batch_create_ssa", C.c_int, [VP, C.POINTER(SsaParamsC), C.c_int, C.c_int, C.c_int,
                                        C.POINTER(VP)]),
    ("ssqa_batch_create", C.c_int, [VP, C.POINTER(ParamsC), C.c_int, C.c_int, C.c_int,
                                    C.POINTER(VP)]),
    ("ssqa_batch_destroy", C.c_int, [VP]),
    ("ssqa_batch_stream", VP, [VP]),
    ("ssqa_batch_engine", C.c_int, [VP]),
    ("ssqa_batch_operand_bits", C.c_int, [VP]),
    ("ssqa_batch_set_seeds", C.c_int, [VP, U64P]),
    ("ssqa_batch_launch", C.c_int, [VP, C.c_int, C.c_double, C.c_int]),
    ("ssqa_batch_fetch", C.c_int, [VP, C.POINTER(ResultC), I8P, DP]),
    ("ssqa_batch_launch_count", C.c_long, [VP]),
    ("ssqa_batch_elapsed_ms", C.c_int, [VP, DP]),
    ("ssqa_batch_synchronize", C.c_int, [C.c_void_p]),
    ("ssqa_batch_profile_field", C.c_int, [VP, C.c_int, DP]),
    ("ssqa_batch_set_shard", C.c_int, [VP, C.c_int, C.c_int]),
    ("ssqa_batch_shard_bytes", C.c_long, [VP]),
    ("ssqa_batch_shard_begin", C.c_int, [VP, C.c_int, C.c_double, C.c_int]),
    ("ssqa_batch_shard_pass", C.c_int, [VP, VP]),
    ("ssqa_batch_shard_merge", C.c_int, [VP, VP]),
    ("ssqa_batch_shard_pass_to", C.c_int, [VP, C.POINTER(VP), C.POINTER(VP), C.c_int, C.c_uint]),
    ("ssqa_batch_shard_merge_from", C.c_int, [VP, VP, VP, C.c_int, C.c_uint]),
    ("ssqa_batch_shard_direct_ok", C.c_int, [VP]),
    ("ssqa_batch_sig4", C.c_int, [VP, C.POINTER(VP)]),
    ("ssqa_batch_shard_pass_direct", C.c_int, [VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP),
                                               C.c_int, C.c_uint]),
    ("ssqa_batch_shard_merge_direct", C.c_int, [VP, VP, C.c_longlong, VP, C.c_int, C.c_uint]),
    ("ssqa_exchange_alloc", C.c_int, [C.c_int, C.c_longlong, C.POINTER(VP)]),
    ("ssqa_exchange_free", C.c_int, [VP]),
    ("ssqa_ipc_handle", C.c_int, [VP, C.c_char_p]),
    ("ssqa_ipc_open", C.c_int, [C.c_char_p, C.c_int, C.POINTER(VP)]),
    ("ssqa_ipc_close", C.c_int, [VP]),
    ("ssqa_batch_shard_end", C.c_int, [VP]),
    ("ssqa_batch_init", C.c_int, [VP]),
    ("ssqa_batch_sweep", C.c_int, [VP, C.c_long]),
    ("ssqa_batch_sweep_with", C.c_int, [VP, C.c_double, C.c_double]),
    ("ssqa_batch_energies", C.c_int, [VP, DP]),
    ("ssqa_batch_read_lattice", C.c_int, [VP, C.c_int, DP, DP, DP, LP]),
    ("ssqa_batch_write_lattice", C.c_int, [VP, C.c_int, DP, DP, DP, C.c_long]),
    # ssqa_host.h
    ("ssqa_gi_ising", C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_double,
                                C.c_double, DP, DP, DP]),
    ("ssqa_dense_ising", C.c_int, [C.c_int, C.c_int, C.c_uint64, DP, DP, DP]),
    ("ssqa_ising_energy", C.c_int, [C.c_int, DP, DP, C.c_double, I8P, DP]),
    ("ssqa_host_last_error", C.c_char_p, []),
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2302_12454_b200.build` "
                "(the engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SsqaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int, host: bool = False) -> None:
    if rc != SSQA_OK:
        L = lib()
        msg = (L.ssqa_host_last_error() if host else L.ssqa_last_error()).decode()
        if rc in (SSQA_EINVAL, SSQA_EUNSUP) and not host:
            raise SsqaInvalidArgument(rc, msg)
        if host and rc == 1:
            raise SsqaInvalidArgument(rc, msg)
        raise SsqaError(rc, msg)


class SsqaInvalidArgument(SsqaError, ValueError):
    """The reference's std::invalid_argument."""
