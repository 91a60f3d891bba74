"""ctypes binding of libgcmc_b200.so (include/gcmc_b200.h).

The library is built in-tree by ``paper_1408_3764_b200.build`` (nvcc,
sm_100a). There is no fallback: if the shared object is missing or cannot
be loaded, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("GCMC_LIB") or os.path.join(PKG, "libgcmc_b200.so")

_d, _u64, _i32, _p = C.c_double, C.c_uint64, C.c_int32, C.c_void_p
_dp = C.POINTER(C.c_double)

GCMC_OK = 0
STATUS = {0: "OK", 1: "INVALID_PID", 2: "CELL_OVERFLOW", 3: "NOT_FOUND", 4: "OVERLAP",
          5: "CUDA", 6: "ARG", 7: "STATE"}
ALL_PAIRS, CELL_LIST, MICROCELL = 0, 1, 2


class GcmcParams(C.Structure):
    _fields_ = [("box_length", _d), ("epsilon", _d), ("sigma", _d), ("r_cut", _d),
                ("temperature", _d), ("chemical_potential", _d), ("lambda_", _d),
                ("displace_percent", _d), ("max_displacement", _d),
                ("equilibration_steps", _u64), ("sampling_interval", _u64),
                ("strategy", _i32), ("cell_capacity", _i32), ("microcell_capacity", _i32),
                ("tail_corrections", _i32), ("max_particles", _u64), ("engine_ctas", _i32),
                ("engine_group", _i32), ("engine_variants", _i32), ("engine_bias", _i32),
                ("engine_mode", _i32), ("engine_share", _i32)]


class GcmcState(C.Structure):
    _fields_ = [("step", _u64), ("n", _u64), ("energy", _d), ("virial", _d),
                ("attempted", _u64 * 3), ("accepted", _u64 * 3), ("samples", _u64),
                ("sum_u", _d), ("sum_p", _d), ("sum_n", _d), ("sum_n2", _d),
                ("peak_occupancy", _i32), ("pad", _i32)]


class GcmcRunResult(C.Structure):
    _fields_ = [("state", GcmcState), ("moves", _u64), ("rounds", _u64), ("device_ms", _d),
                ("gen_ms", _d), ("pair_evals", _u64), ("engine", _i32), ("pad", _i32)]


TRACE_DTYPE = np.dtype([("kind", "<i4"), ("accepted", "<i4"), ("delta_u", "<f8"),
                        ("delta_w", "<f8"), ("acceptance_prob", "<f8"), ("n_after", "<u8")])

EXPORTS = [
    "gcmc_last_error", "gcmc_version", "gcmc_create", "gcmc_destroy", "gcmc_upload_positions",
    "gcmc_download_positions", "gcmc_build", "gcmc_store_set", "gcmc_grid_info", "gcmc_download_grid",
    "gcmc_rebuild_check", "gcmc_peak_occupancy", "gcmc_delta_displace", "gcmc_delta_insert",
    "gcmc_delta_delete", "gcmc_delta_batch", "gcmc_commit_displace", "gcmc_commit_insert",
    "gcmc_commit_delete", "gcmc_total_energy", "gcmc_energy_drift", "gcmc_seed_rng", "gcmc_set_rng_state",
    "gcmc_get_rng_state", "gcmc_set_state", "gcmc_get_state", "gcmc_run_moves",
    "gcmc_random_initial_configuration", "gcmc_run_chains", "gcmc_energy_timing",
    "gcmc_total_energy_bruteforce", "gcmc_device_initial_configuration",
]

_lib = None


class GcmcError(RuntimeError):
    """A non-OK gcmc_status; ``code`` is the status, the message is the
    reference's exception text."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.status = STATUS.get(code, str(code))


def load(path: str = SO):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_1408_3764_b200.build`"
                          " (there is no CPU fallback)")
    lib = C.CDLL(path)
    lib.gcmc_last_error.restype = C.c_char_p
    lib.gcmc_version.restype = C.c_char_p
    P = C.POINTER
    sig = {
        "gcmc_create": [P(GcmcParams), C.c_int, P(_p)],
        "gcmc_destroy": [_p],
        "gcmc_upload_positions": [_p, _dp, _u64],
        "gcmc_download_positions": [_p, _dp, _u64, P(_u64)],
        "gcmc_build": [_p],
        "gcmc_store_set": [_p, _u64, _dp],
        "gcmc_grid_info": [_p, P(_i32), P(_i32), P(_u64)],
        "gcmc_download_grid": [_p, P(_i32), P(_i32)],
        "gcmc_rebuild_check": [_p, C.c_char_p, C.c_size_t, P(_i32)],
        "gcmc_peak_occupancy": [_p, P(_i32)],
        "gcmc_delta_displace": [_p, _u64, _dp, _dp, _dp],
        "gcmc_delta_insert": [_p, _dp, _dp, _dp],
        "gcmc_delta_delete": [_p, _u64, _dp, _dp],
        "gcmc_delta_batch": [_p, _u64, P(_i32), P(_u64), _dp, _dp, _dp],
        "gcmc_commit_displace": [_p, _u64, _dp],
        "gcmc_commit_insert": [_p, _dp, P(_u64)],
        "gcmc_commit_delete": [_p, _u64],
        "gcmc_total_energy": [_p, _dp, _dp],
        "gcmc_energy_drift": [_p, _dp, _dp],
        "gcmc_seed_rng": [_p, _u64],
        "gcmc_set_rng_state": [_p, P(_u64), _u64, _u64],
        "gcmc_get_rng_state": [_p, P(_u64), P(_u64), P(_u64)],
        "gcmc_set_state": [_p, P(GcmcState)],
        "gcmc_get_state": [_p, P(GcmcState)],
        "gcmc_run_moves": [_p, _u64, _p, P(GcmcRunResult)],
        "gcmc_random_initial_configuration": [_u64, _d, _d, _u64, _dp, P(_u64), P(_u64), P(_u64)],
        "gcmc_run_chains": [P(_p), _i32, P(_u64), P(GcmcRunResult)],
        "gcmc_energy_timing": [_p, _dp, _dp],
        "gcmc_total_energy_bruteforce": [_p, _dp, _dp],
        "gcmc_device_initial_configuration": [C.c_int, _u64, _d, _d, _u64, _dp, P(_u64), P(_u64),
                                              P(_u64)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != GCMC_OK:
        raise GcmcError(rc, load().gcmc_last_error().decode())


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)
