"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU oracles.

* ``ref``  : the real reference (its unmodified headers compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libgcmc_ref.so``).
* ``port`` : the C restatement ``oracle/gcmc_oracle.c`` (``liboracle.so``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this package; the
product (``paper_1408_3764_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgcmc_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_INC = "/root/reference/proj/include"

_d = C.c_double
_u64 = C.c_uint64
_i32 = C.c_int32
_p = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


SHIM = os.path.join(HERE, "_ref", "shim_check")


def build(ref: bool = True) -> None:
    """Compile the restatement, and the reference (plus the drop-in shim
    check, which links the product library) when its headers exist."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref and os.path.isdir(REF_INC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        subprocess.run(["make", "-s", "-C", HERE, "shim"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_INC)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip)


# --------------------------------------------------------------------------
# Reference (oracle/_ref)
# --------------------------------------------------------------------------
class RefConfig(C.Structure):
    _fields_ = [
        ("temperature", _d), ("chemical_potential", _d), ("lambda_", _d), ("epsilon", _d),
        ("sigma", _d), ("r_cut", _d), ("box_length", _d), ("initial_particles", _u64),
        ("density", _d), ("displace_percent", _d), ("steps", _u64), ("seed", _u64),
        ("checkpoint_interval", _u64), ("strategy", _i32), ("tail_corrections", _i32),
        ("cell_capacity", _i32), ("microcell_capacity", _i32),
        ("equilibration_steps", _u64), ("sampling_interval", _u64), ("max_displacement", _d),
    ]


class RefOutcome(C.Structure):
    _fields_ = [("kind", _i32), ("accepted", _i32), ("delta_u", _d), ("delta_w", _d),
                ("acceptance_prob", _d), ("n_after", _u64)]


OUTCOME_DTYPE = np.dtype([("kind", "<i4"), ("accepted", "<i4"), ("delta_u", "<f8"),
                          ("delta_w", "<f8"), ("acceptance_prob", "<f8"), ("n_after", "<u8")])


class RefState(C.Structure):
    _fields_ = [("step", _u64), ("n", _u64), ("energy", _d), ("virial", _d),
                ("attempted", _u64 * 3), ("accepted", _u64 * 3), ("samples", _u64),
                ("sum_u", _d), ("sum_p", _d), ("sum_n", _d), ("sum_n2", _d), ("draws", _u64),
                ("peak_occupancy", _i32), ("pad", _i32), ("pressure", _d),
                ("reported_energy", _d)]


STRATEGIES = {"all_pairs": 0, "cell_list": 1, "microcell": 2}

_ref_lib = None


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_index_from.restype = _u64
        lib.ref_min_image_dist2.restype = _d
        for f in ("ref_displacement_acceptance", "ref_insertion_acceptance",
                  "ref_deletion_acceptance"):
            getattr(lib, f).restype = _d
        lib.ref_displacement_acceptance.argtypes = [_d, _d]
        lib.ref_insertion_acceptance.argtypes = [_d, _u64, _d, _d, _d, _d]
        lib.ref_deletion_acceptance.argtypes = [_d, _u64, _d, _d, _d, _d]
        lib.ref_microcell_extent.restype = _i32
        lib.ref_microcell_extent.argtypes = [_d, _d]
        lib.ref_default_cell_capacity.restype = _i32
        lib.ref_default_cell_capacity.argtypes = [_d, _d]
        lib.ref_strat_size.restype = _u64
        lib.ref_strat_peak.restype = _i32
        lib.ref_strat_cell_of.restype = _i32
        lib.ref_strat_neighborhood_of_cell.restype = _u64
        lib.ref_strat_neighborhood_of_pos.restype = _u64
        lib.ref_cube_cells.restype = _u64
        lib.ref_index_from.argtypes = [_d, _u64]
        lib.ref_min_image_dist2.argtypes = [_dp, _dp, _d]
        lib.ref_microcell_axis_arc.argtypes = [_d, _d, _d, _d, _i32, _ip, _ip]
        lib.ref_microcell_axis_window.argtypes = [_i32, _d, _d, _i32, _d, _ip, _ip]
        lib.ref_microcell_dims.argtypes = [_d, _d, _ip, _dp]
        lib.ref_compute_cell_dims.argtypes = [_d, _d, _ip, _dp]
        lib.ref_lj_pair.argtypes = [_d, _d, _d, _d, C.c_int, _dp, _dp]
        lib.ref_tail_corrections.argtypes = [_d, _d, _d, _d, _dp, _dp]
        lib.ref_mt_uniforms.argtypes = [_u64, _u64, _u64, _dp]
        lib.ref_rng_hex.argtypes = [_u64, _u64, C.c_char_p, _u64]
        lib.ref_total_energy.argtypes = [_dp, _u64, _d, _d, _d, _d, _dp, _dp]
        lib.ref_random_initial_configuration.argtypes = [_u64, _d, _d, _u64, _dp, C.c_char_p, _u64]
        lib.ref_strat_create.argtypes = [_i32, _dp, _u64, _d, _d, _d, _d, _i32, C.POINTER(_p)]
        lib.ref_strat_destroy.argtypes = [_p]
        for f in ("ref_strat_size", "ref_strat_peak", "ref_strat_build"):
            getattr(lib, f).argtypes = [_p]
        lib.ref_strat_positions.argtypes = [_p, _dp]
        lib.ref_strat_delta_displace.argtypes = [_p, _u64, _dp, _dp, _dp]
        lib.ref_strat_delta_insert.argtypes = [_p, _dp, _dp, _dp]
        lib.ref_strat_delta_delete.argtypes = [_p, _u64, _dp, _dp]
        lib.ref_strat_commit_displace.argtypes = [_p, _u64, _dp]
        lib.ref_strat_commit_insert.argtypes = [_p, _dp, C.POINTER(_u64)]
        lib.ref_strat_commit_delete.argtypes = [_p, _u64]
        lib.ref_strat_grid_info.argtypes = [_p, _ip, _ip, C.POINTER(_u64)]
        lib.ref_strat_grid.argtypes = [_p, _ip, _ip]
        lib.ref_strat_cell_of.argtypes = [_p, _dp]
        lib.ref_strat_neighborhood_of_cell.argtypes = [_p, _i32, _ip, _u64]
        lib.ref_strat_neighborhood_of_pos.argtypes = [_p, _dp, _ip, _u64]
        lib.ref_strat_rebuild_check.argtypes = [_p, C.c_char_p, _u64, _ip]
        lib.ref_sim_create.argtypes = [C.POINTER(RefConfig), _i32, _dp, _u64, C.c_char_p, _u64,
                                       _d, _d, C.POINTER(_p)]
        lib.ref_sim_destroy.argtypes = [_p]
        lib.ref_sim_run.argtypes = [_p, _u64, _p, _dp]
        lib.ref_sim_state.argtypes = [_p, C.POINTER(RefState)]
        lib.ref_sim_positions.argtypes = [_p, _dp]
        lib.ref_sim_rng_hex.argtypes = [_p, C.c_char_p, _u64]
        lib.ref_sim_audit.argtypes = [_p, _dp, _dp, _ip, C.c_char_p, _u64]
        lib.ref_sim_checkpoint_text.argtypes = [_p, C.c_char_p, _u64, C.POINTER(_u64)]
        lib.ref_sim_stats_row.argtypes = [_p, C.c_char_p, _u64]
        lib.ref_sim_from_checkpoint.argtypes = [C.c_char_p, C.POINTER(_p)]
        lib.ref_sim_grid_info.argtypes = [_p, _ip, _ip, C.POINTER(_u64)]
        lib.ref_sim_grid.argtypes = [_p, _ip, _ip]
        lib.ref_sim_store_set.argtypes = [_p, _u64, _dp]
        lib.ref_run_with_files.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(_u64)]
        lib.ref_format_g17.argtypes = [_d, C.c_char_p, _u64]
        lib.ref_parse_config.argtypes = [C.c_char_p, C.POINTER(RefConfig)]
        lib.ref_serialize_config.argtypes = [C.POINTER(RefConfig), C.c_char_p, _u64]
        lib.ref_run_concurrent.argtypes = [C.POINTER(RefConfig), _dp, _u64, C.c_char_p, _d, _d,
                                           _i32, _u64, _dp]
        lib.ref_cross_strategy_equivalence.argtypes = [_u64, _d, _d, _i32, _d, _u64, _dp, _dp, _ip]
        _ref_lib = lib
    return _ref_lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _chk(rc: int):
    if rc != 0:
        raise RefError(rc, ref_lib().ref_last_error().decode())


def ref_config(**kw) -> RefConfig:
    """RunConfig with the reference defaults (config.hpp:42-64)."""
    c = RefConfig(temperature=0.0, chemical_potential=0.0, lambda_=1.0, epsilon=1.0, sigma=1.0,
                  r_cut=2.5, box_length=0.0, initial_particles=0, density=0.6,
                  displace_percent=0.30, steps=0, seed=1, checkpoint_interval=10000,
                  strategy=0, tail_corrections=0, cell_capacity=0, microcell_capacity=5,
                  equilibration_steps=0, sampling_interval=1, max_displacement=0.0)
    for k, v in kw.items():
        if k == "strategy" and isinstance(v, str):
            v = STRATEGIES[v]
        if k == "lambda":
            k = "lambda_"
        setattr(c, k, v)
    return c


def ref_uniforms(seed: int, n: int, skip: int = 0) -> np.ndarray:
    out = np.empty(n, np.float64)
    _chk(ref_lib().ref_mt_uniforms(seed, skip, n, dptr(out)))
    return out


def ref_initial_configuration(n: int, box: float, seed: int, min_sep: float = 0.85):
    """(positions (n,3), rng_hex) from init_config.hpp:19-64 with RngStream(seed)."""
    xyz = np.empty((max(n, 1), 3), np.float64)
    buf = C.create_string_buffer(16384)
    _chk(ref_lib().ref_random_initial_configuration(n, box, min_sep, seed, dptr(xyz), buf, 16384))
    return xyz[:n].copy(), buf.value.decode()


class RefStrategy:
    """A reference NeighborStrategy over its own store (validate.hpp:51-53)."""

    def __init__(self, kind, xyz, box, eps=1.0, sigma=1.0, rc=2.5, capacity=0):
        lib = ref_lib()
        self.kind = STRATEGIES[kind] if isinstance(kind, str) else kind
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        h = _p()
        _chk(lib.ref_strat_create(self.kind, dptr(xyz), len(xyz), box, eps, sigma, rc, capacity,
                                  C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_strat_destroy(self.h)
            self.h = None

    def size(self):
        return ref_lib().ref_strat_size(self.h)

    def positions(self):
        out = np.empty((max(self.size(), 1), 3), np.float64)
        ref_lib().ref_strat_positions(self.h, dptr(out))
        return out[: self.size()].copy()

    def _d(self, fn, *args):
        du, dw = _d(), _d()
        _chk(fn(self.h, *args, C.byref(du), C.byref(dw)))
        return du.value, dw.value

    def delta_displace(self, pid, pos):
        p = np.asarray(pos, np.float64)
        return self._d(ref_lib().ref_strat_delta_displace, pid, dptr(p))

    def delta_insert(self, pos):
        p = np.asarray(pos, np.float64)
        return self._d(ref_lib().ref_strat_delta_insert, dptr(p))

    def delta_delete(self, pid):
        return self._d(ref_lib().ref_strat_delta_delete, pid)

    def commit_displace(self, pid, pos):
        p = np.asarray(pos, np.float64)
        _chk(ref_lib().ref_strat_commit_displace(self.h, pid, dptr(p)))

    def commit_insert(self, pos):
        p = np.asarray(pos, np.float64)
        pid = _u64()
        _chk(ref_lib().ref_strat_commit_insert(self.h, dptr(p), C.byref(pid)))
        return pid.value

    def commit_delete(self, pid):
        _chk(ref_lib().ref_strat_commit_delete(self.h, pid))

    def grid(self):
        d, cap, nc = _i32(), _i32(), _u64()
        ref_lib().ref_strat_grid_info(self.h, C.byref(d), C.byref(cap), C.byref(nc))
        occ = np.empty(nc.value, np.int32)
        slots = np.empty(nc.value * cap.value, np.int32)
        ref_lib().ref_strat_grid(self.h, iptr(occ), iptr(slots))
        return occ, slots

    def grid_info(self):
        d, cap, nc = _i32(), _i32(), _u64()
        ref_lib().ref_strat_grid_info(self.h, C.byref(d), C.byref(cap), C.byref(nc))
        return d.value, cap.value, nc.value

    def peak(self):
        return ref_lib().ref_strat_peak(self.h)

    def cell_of(self, pos):
        return ref_lib().ref_strat_cell_of(self.h, dptr(np.asarray(pos, np.float64)))

    def neighborhood_of_pos(self, pos):
        out = np.empty(4096, np.int32)
        n = ref_lib().ref_strat_neighborhood_of_pos(self.h, dptr(np.asarray(pos, np.float64)),
                                                    iptr(out), 4096)
        return out[:n].copy()

    def neighborhood_of_cell(self, cell):
        out = np.empty(4096, np.int32)
        n = ref_lib().ref_strat_neighborhood_of_cell(self.h, cell, iptr(out), 4096)
        return out[:n].copy()

    def rebuild_check(self):
        buf = C.create_string_buffer(512)
        clean = _i32()
        _chk(ref_lib().ref_strat_rebuild_check(self.h, buf, 512, C.byref(clean)))
        return None if clean.value else buf.value.decode()


class RefSim:
    """The reference gcmc::Simulation (engine.hpp:214-437)."""

    def __init__(self, cfg: RefConfig, mode=0, xyz=None, rng_hex="", step=0, energy=0.0,
                 virial=0.0, _handle=None):
        lib = ref_lib()
        if _handle is not None:
            self.h = _handle
            return
        if xyz is None:
            xyz = np.zeros((1, 3))
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        n = len(xyz) if mode else 0
        h = _p()
        _chk(lib.ref_sim_create(C.byref(cfg), mode, dptr(xyz), n, rng_hex.encode(), step, energy,
                                virial, C.byref(h)))
        self.h = h

    @classmethod
    def from_checkpoint(cls, text: str):
        h = _p()
        _chk(ref_lib().ref_sim_from_checkpoint(text.encode(), C.byref(h)))
        return cls(None, _handle=h)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_sim_destroy(self.h)
            self.h = None

    def run(self, n: int, trace: bool = False):
        """Runs n steps; returns (seconds, trace-or-None)."""
        secs = _d()
        tr = np.zeros(n, OUTCOME_DTYPE) if trace else None
        _chk(ref_lib().ref_sim_run(self.h, n, tr.ctypes.data if trace else None, C.byref(secs)))
        return secs.value, tr

    def state(self) -> RefState:
        s = RefState()
        ref_lib().ref_sim_state(self.h, C.byref(s))
        return s

    def positions(self):
        n = self.state().n
        out = np.empty((max(n, 1), 3), np.float64)
        ref_lib().ref_sim_positions(self.h, dptr(out))
        return out[:n].copy()

    def rng_hex(self):
        buf = C.create_string_buffer(16384)
        ref_lib().ref_sim_rng_hex(self.h, buf, 16384)
        return buf.value.decode()

    def audit(self):
        u, w, ok = _d(), _d(), _i32()
        buf = C.create_string_buffer(1024)
        _chk(ref_lib().ref_sim_audit(self.h, C.byref(u), C.byref(w), C.byref(ok), buf, 1024))
        return u.value, w.value, bool(ok.value), buf.value.decode()

    def checkpoint_text(self):
        need = _u64()
        _chk(ref_lib().ref_sim_checkpoint_text(self.h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _chk(ref_lib().ref_sim_checkpoint_text(self.h, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def stats_row(self):
        buf = C.create_string_buffer(512)
        _chk(ref_lib().ref_sim_stats_row(self.h, buf, 512))
        return buf.value.decode()

    def grid(self):
        """(occupancy_view, slots_view) of the live strategy (empty for all_pairs)."""
        d, cap, nc = _i32(), _i32(), _u64()
        ref_lib().ref_sim_grid_info(self.h, C.byref(d), C.byref(cap), C.byref(nc))
        occ = np.zeros(nc.value, np.int32)
        slots = np.zeros(nc.value * cap.value, np.int32)
        ref_lib().ref_sim_grid(self.h, iptr(occ), iptr(slots))
        return occ, slots

    def store_set(self, i, pos):
        """ParticleStore::set behind the strategy's back (T/test_engine.cpp:186-192)."""
        _chk(ref_lib().ref_sim_store_set(self.h, i, dptr(np.ascontiguousarray(pos, np.float64))))


def ref_run_with_files(cfg_text: str, out_dir: str, resume: str | None = None) -> int:
    """gcmc::run_with_files (driver.hpp:47-116); returns the final step."""
    fs = _u64()
    _chk(ref_lib().ref_run_with_files(cfg_text.encode(), out_dir.encode(),
                                      resume.encode() if resume else None, C.byref(fs)))
    return fs.value


def ref_format_g17(v: float) -> str:
    buf = C.create_string_buffer(64)
    ref_lib().ref_format_g17(v, buf, 64)
    return buf.value.decode()


# --------------------------------------------------------------------------
# Restatement (oracle/liboracle.so)
# --------------------------------------------------------------------------
class OrcRng(C.Structure):
    _fields_ = [("mt", _u64 * 312), ("idx", _u64), ("draws", _u64)]


class OrcParams(C.Structure):
    _fields_ = [("temperature", _d), ("chemical_potential", _d), ("lambda_", _d),
                ("epsilon", _d), ("sigma", _d), ("r_cut", _d), ("box_length", _d),
                ("displace_percent", _d), ("max_displacement", _d),
                ("equilibration_steps", _u64), ("sampling_interval", _u64), ("strategy", _i32),
                ("tail_corrections", _i32), ("cell_capacity", _i32), ("microcell_capacity", _i32)]


class OrcState(C.Structure):
    _fields_ = [("step", _u64), ("energy", _d), ("virial", _d), ("attempted", _u64 * 3),
                ("accepted", _u64 * 3), ("samples", _u64), ("sum_u", _d), ("sum_p", _d),
                ("sum_n", _d), ("sum_n2", _d)]


_port_lib = None


def port_lib():
    global _port_lib
    if _port_lib is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        lib = C.CDLL(PORT_SO)
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_rng_next.restype = _u64
        lib.orc_uniform.restype = _d
        lib.orc_index_from.restype = _u64
        lib.orc_index_from.argtypes = [_d, _u64]
        lib.orc_wrap_axis.restype = _d
        lib.orc_wrap_axis.argtypes = [_d, _d]
        lib.orc_wrap_position.argtypes = [_dp, _d, _dp]
        lib.orc_min_image_dist2.restype = _d
        lib.orc_min_image_dist2.argtypes = [_dp, _dp, _d]
        for f in ("orc_displacement_acceptance", "orc_insertion_acceptance",
                  "orc_deletion_acceptance"):
            getattr(lib, f).restype = _d
        lib.orc_displacement_acceptance.argtypes = [_d, _d]
        lib.orc_insertion_acceptance.argtypes = [_d, _u64, _d, _d, _d, _d]
        lib.orc_deletion_acceptance.argtypes = [_d, _u64, _d, _d, _d, _d]
        lib.orc_rng_seed.argtypes = [C.POINTER(OrcRng), _u64]
        lib.orc_rng_next.argtypes = [C.POINTER(OrcRng)]
        lib.orc_uniform.argtypes = [C.POINTER(OrcRng)]
        lib.orc_microcell_axis_arc.argtypes = [_d, _d, _d, _d, _i32, _ip, _ip]
        lib.orc_microcell_axis_window.argtypes = [_i32, _d, _d, _i32, _d, _ip, _ip]
        lib.orc_microcell_dims.argtypes = [_d, _d, _ip, _dp]
        lib.orc_compute_cell_dims.argtypes = [_d, _d, _ip, _dp]
        lib.orc_microcell_extent.restype = _i32
        lib.orc_microcell_extent.argtypes = [_d, _d]
        lib.orc_total_energy.argtypes = [_dp, _u64, _d, _d, _d, _d, _dp, _dp]
        lib.orc_random_initial_configuration.argtypes = [_u64, _d, _d, C.POINTER(OrcRng), _dp]
        lib.orc_grid_create.restype = _p
        lib.orc_grid_create.argtypes = [_i32, _dp, _u64, _u64, _d, _d, _d, _d, _i32, _ip]
        lib.orc_grid_destroy.argtypes = [_p]
        lib.orc_grid_size.restype = _u64
        lib.orc_grid_size.argtypes = [_p]
        lib.orc_grid_positions.restype = _dp
        lib.orc_grid_positions.argtypes = [_p]
        lib.orc_grid_info.argtypes = [_p, _ip, _ip, C.POINTER(_u64)]
        lib.orc_grid_occ.restype = _ip
        lib.orc_grid_occ.argtypes = [_p]
        lib.orc_grid_slots.restype = _ip
        lib.orc_grid_slots.argtypes = [_p]
        lib.orc_grid_peak.restype = _i32
        lib.orc_grid_peak.argtypes = [_p]
        lib.orc_grid_cell_of.restype = _i32
        lib.orc_grid_cell_of.argtypes = [_p, _dp]
        lib.orc_delta_displace.argtypes = [_p, _u64, _dp, _dp, _dp]
        lib.orc_delta_insert.argtypes = [_p, _dp, _dp, _dp]
        lib.orc_delta_delete.argtypes = [_p, _u64, _dp, _dp]
        lib.orc_commit_displace.argtypes = [_p, _u64, _dp]
        lib.orc_commit_insert.argtypes = [_p, _dp, C.POINTER(_u64)]
        lib.orc_commit_delete.argtypes = [_p, _u64]
        lib.orc_rebuild_check.argtypes = [_p]
        lib.orc_sim_create.restype = _p
        lib.orc_sim_create.argtypes = [C.POINTER(OrcParams), _dp, _u64, C.POINTER(OrcRng), _u64,
                                       _d, _d, _ip]
        lib.orc_sim_destroy.argtypes = [_p]
        lib.orc_sim_run.argtypes = [_p, _u64, _p]
        lib.orc_sim_state.argtypes = [_p, C.POINTER(OrcState)]
        lib.orc_sim_grid.restype = _p
        lib.orc_sim_grid.argtypes = [_p]
        lib.orc_sim_rng.restype = C.POINTER(OrcRng)
        lib.orc_sim_rng.argtypes = [_p]
        _port_lib = lib
    return _port_lib


def rng_from_hex(text: str) -> OrcRng:
    """RngStream::serialize_hex text (rng.hpp:47-58) -> OrcRng."""
    parts = text.split()
    count, draws = int(parts[0], 16), int(parts[1], 16)
    words = [int(w, 16) for w in parts[2: 2 + count]]
    assert count == 313, count
    r = OrcRng()
    for i in range(312):
        r.mt[i] = words[i]
    r.idx = words[312]
    r.draws = draws
    return r


def rng_to_hex(r: OrcRng) -> str:
    words = list(r.mt) + [r.idx]
    return " ".join([format(313, "x"), format(r.draws, "x")] + [format(w, "x") for w in words])


def port_rng(seed: int) -> OrcRng:
    r = OrcRng()
    port_lib().orc_rng_seed(C.byref(r), seed)
    return r


class PortGrid:
    def __init__(self, kind, xyz, box, eps=1.0, sigma=1.0, rc=2.5, capacity=0, capn=0):
        lib = port_lib()
        self.kind = STRATEGIES[kind] if isinstance(kind, str) else kind
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        st = _i32()
        self.h = lib.orc_grid_create(self.kind, dptr(xyz), len(xyz), capn, box, eps, sigma, rc,
                                     capacity, C.byref(st))
        if st.value:
            msg = lib.orc_last_error().decode()
            lib.orc_grid_destroy(self.h)
            self.h = None
            raise RefError(st.value, msg)

    def __del__(self):
        if getattr(self, "h", None):
            port_lib().orc_grid_destroy(self.h)
            self.h = None

    def _chk(self, rc):
        if rc:
            raise RefError(rc, port_lib().orc_last_error().decode())

    def size(self):
        return port_lib().orc_grid_size(self.h)

    def positions(self):
        n = self.size()
        p = port_lib().orc_grid_positions(self.h)
        return np.ctypeslib.as_array(p, shape=(n * 3,)).reshape(n, 3).copy() if n else np.zeros((0, 3))

    def grid(self):
        d, cap, nc = _i32(), _i32(), _u64()
        port_lib().orc_grid_info(self.h, C.byref(d), C.byref(cap), C.byref(nc))
        occ = np.ctypeslib.as_array(port_lib().orc_grid_occ(self.h), shape=(nc.value,)).copy()
        slots = np.ctypeslib.as_array(port_lib().orc_grid_slots(self.h),
                                      shape=(nc.value * cap.value,)).copy()
        return occ, slots

    def peak(self):
        return port_lib().orc_grid_peak(self.h)

    def _dd(self, fn, *args):
        du, dw = _d(), _d()
        self._chk(fn(self.h, *args, C.byref(du), C.byref(dw)))
        return du.value, dw.value

    def delta_displace(self, pid, pos):
        return self._dd(port_lib().orc_delta_displace, pid, dptr(np.asarray(pos, np.float64)))

    def delta_insert(self, pos):
        return self._dd(port_lib().orc_delta_insert, dptr(np.asarray(pos, np.float64)))

    def delta_delete(self, pid):
        return self._dd(port_lib().orc_delta_delete, pid)

    def commit_displace(self, pid, pos):
        self._chk(port_lib().orc_commit_displace(self.h, pid, dptr(np.asarray(pos, np.float64))))

    def commit_insert(self, pos):
        pid = _u64()
        self._chk(port_lib().orc_commit_insert(self.h, dptr(np.asarray(pos, np.float64)),
                                               C.byref(pid)))
        return pid.value

    def commit_delete(self, pid):
        self._chk(port_lib().orc_commit_delete(self.h, pid))

    def rebuild_check(self):
        ok = port_lib().orc_rebuild_check(self.h)
        return None if ok else port_lib().orc_last_error().decode()


def port_params(**kw) -> OrcParams:
    p = OrcParams(temperature=2.0, chemical_potential=-2.0, lambda_=1.0, epsilon=1.0, sigma=1.0,
                  r_cut=2.5, box_length=10.0, displace_percent=0.30, max_displacement=0.0,
                  equilibration_steps=0, sampling_interval=1, strategy=2, tail_corrections=0,
                  cell_capacity=0, microcell_capacity=5)
    for k, v in kw.items():
        if k == "strategy" and isinstance(v, str):
            v = STRATEGIES[v]
        if k == "lambda":
            k = "lambda_"
        setattr(p, k, v)
    return p


class PortSim:
    def __init__(self, params: OrcParams, xyz, rng: OrcRng, step=0, energy=0.0, virial=0.0):
        lib = port_lib()
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        st = _i32()
        self.h = lib.orc_sim_create(C.byref(params), dptr(xyz), len(xyz), C.byref(rng), step,
                                    energy, virial, C.byref(st))
        if st.value:
            raise RefError(st.value, lib.orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            port_lib().orc_sim_destroy(self.h)
            self.h = None

    def run(self, n, trace=False):
        tr = np.zeros(n, OUTCOME_DTYPE) if trace else None
        rc = port_lib().orc_sim_run(self.h, n, tr.ctypes.data if trace else None)
        if rc:
            raise RefError(rc, port_lib().orc_last_error().decode())
        return tr

    def state(self) -> OrcState:
        s = OrcState()
        port_lib().orc_sim_state(self.h, C.byref(s))
        return s

    def grid(self):
        g = PortGrid.__new__(PortGrid)
        g.h = None
        g.kind = None
        h = port_lib().orc_sim_grid(self.h)
        n = port_lib().orc_grid_size(h)
        p = port_lib().orc_grid_positions(h)
        pos = np.ctypeslib.as_array(p, shape=(n * 3,)).reshape(n, 3).copy() if n else np.zeros((0, 3))
        d, cap, nc = _i32(), _i32(), _u64()
        port_lib().orc_grid_info(h, C.byref(d), C.byref(cap), C.byref(nc))
        occ = slots = None
        if nc.value:
            occ = np.ctypeslib.as_array(port_lib().orc_grid_occ(h), shape=(nc.value,)).copy()
            slots = np.ctypeslib.as_array(port_lib().orc_grid_slots(h),
                                          shape=(nc.value * cap.value,)).copy()
        return pos, occ, slots

    def rng(self) -> OrcRng:
        r = OrcRng()
        C.memmove(C.byref(r), port_lib().orc_sim_rng(self.h), C.sizeof(OrcRng))
        return r
