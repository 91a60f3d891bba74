"""Host mirror of the reference's engine API over the C ABI.

* :class:`GpuNeighborStrategy` — ``gcmc::NeighborStrategy``
  (proj/include/gcmc/strategy.hpp:27-50): build / delta_* / commit_* /
  rebuild_check / peak_cell_occupancy, executed on the B200.
* :class:`Simulation` — ``gcmc::Simulation`` (engine.hpp:214-437): the three
  constructors (fresh, prepared, resume), step / run_to / audit / state /
  statistics / pressure / reported_energy, with the move loop batched on the
  device (one ``gcmc_run_moves`` per checkpoint interval instead of one call
  per move — PAPER.md:481).
* :class:`RngState` — RngStream state with the reference's hex text form
  (rng.hpp:47-77), so checkpoints interoperate with the reference.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib as L
from .config import RunConfig, STRATEGIES

MOVE_KINDS = ("displace", "insert", "remove")  # engine.hpp:100


@dataclass
class PairInteraction:
    u: float = 0.0
    w: float = 0.0


@dataclass
class MoveOutcome:
    """engine.hpp:104-110."""
    kind: str = "displace"
    accepted: bool = False
    delta_u: float = 0.0
    delta_w: float = 0.0
    acceptance_prob: float = 0.0


@dataclass
class RngState:
    """std::mt19937_64 state (312 words + _M_p) + RngStream draw counter."""
    words: np.ndarray
    index: int
    draws: int = 0

    @classmethod
    def from_seed(cls, seed: int) -> "RngState":
        # Same as RngStream(seed): use the library's host initializer with n=0.
        words = (C.c_uint64 * 312)()
        idx, draws = C.c_uint64(), C.c_uint64()
        dummy = np.zeros(3)
        L.check(L.load().gcmc_random_initial_configuration(0, 1.0, 0.5, seed, L.dptr(dummy), words,
                                                           C.byref(idx), C.byref(draws)))
        return cls(np.frombuffer(words, dtype=np.uint64).copy(), idx.value, 0)

    def serialize_hex(self) -> str:
        """rng.hpp:47-58: "count draws w0 ... w312" in hex."""
        ws = [int(w) for w in self.words] + [int(self.index)]
        return " ".join([format(len(ws), "x"), format(self.draws, "x")] + [format(w, "x") for w in ws])

    @classmethod
    def deserialize_hex(cls, text: str) -> "RngState":
        parts = text.split()
        if len(parts) < 2:
            raise ValueError("rng state: bad header")
        count, draws = int(parts[0], 16), int(parts[1], 16)
        if len(parts) < 2 + count:
            raise ValueError("rng state: truncated")
        ws = [int(w, 16) for w in parts[2: 2 + count]]
        if count != 313:
            raise ValueError("rng state: malformed")
        return cls(np.array(ws[:312], dtype=np.uint64), ws[312], draws)


@dataclass
class SystemState:
    """engine.hpp:112-123."""
    energy: float = 0.0
    virial: float = 0.0
    attempted: list = field(default_factory=lambda: [0, 0, 0])
    accepted: list = field(default_factory=lambda: [0, 0, 0])

    def acceptance_ratio(self, kind: int) -> float:
        return self.accepted[kind] / self.attempted[kind] if self.attempted[kind] else 0.0


@dataclass
class RunStatistics:
    """engine.hpp:125-140."""
    samples: int = 0
    sum_u: float = 0.0
    sum_p: float = 0.0
    sum_n: float = 0.0
    sum_n2: float = 0.0

    def mean_u(self):
        return self.sum_u / self.samples if self.samples else 0.0

    def mean_p(self):
        return self.sum_p / self.samples if self.samples else 0.0

    def mean_n(self):
        return self.sum_n / self.samples if self.samples else 0.0

    def variance_n(self):
        if not self.samples:
            return 0.0
        m = self.mean_n()
        return self.sum_n2 / self.samples - m * m


K_AUDIT_REL = 1e-8  # engine.hpp:146-147
K_AUDIT_ABS = 1e-12


@dataclass
class AuditReport:
    """engine.hpp:149-177."""
    u_tracked: float = 0.0
    u_recomputed: float = 0.0
    w_tracked: float = 0.0
    w_recomputed: float = 0.0
    grid_issue: Optional[str] = None

    @staticmethod
    def within_tolerance(tracked, reference):
        tol = max(K_AUDIT_ABS, K_AUDIT_REL * max(1.0, abs(reference)))
        return abs(tracked - reference) <= tol

    def energy_ok(self):
        return self.within_tolerance(self.u_tracked, self.u_recomputed)

    def virial_ok(self):
        return self.within_tolerance(self.w_tracked, self.w_recomputed)

    def passed(self):
        return self.energy_ok() and self.virial_ok() and not self.grid_issue

    def describe(self):
        s = ""
        if not self.energy_ok():
            s += f"energy drift: tracked {self.u_tracked:f} vs recomputed {self.u_recomputed:f}; "
        if not self.virial_ok():
            s += f"virial drift: tracked {self.w_tracked:f} vs recomputed {self.w_recomputed:f}; "
        if self.grid_issue:
            s += "grid: " + self.grid_issue
        return s or "ok"


class AuditFailure(RuntimeError):
    """engine.hpp:180-183."""


def tail_corrections(rho, epsilon, sigma, r_cut):
    """potential.hpp:63-72 (same operation order)."""
    sr3 = (sigma / r_cut) * (sigma / r_cut) * (sigma / r_cut)
    sr9 = sr3 * sr3 * sr3
    s3 = sigma * sigma * sigma
    pi = math.pi
    u = (8.0 / 3.0) * pi * rho * epsilon * s3 * (sr9 / 3.0 - sr3)
    pr = (16.0 / 3.0) * pi * rho * rho * epsilon * s3 * (2.0 / 3.0 * sr9 - sr3)
    return u, pr


def random_initial_configuration(n: int, box_length: float, min_sep: float, seed: int,
                                 device: Optional[int] = 0):
    """init_config.hpp:19-64 (same MT draws, bit-identical result) on the
    given device (gcmc_device_initial_configuration), or on the host with
    device=None. Returns (positions (n,3), RngState left for the MC stream)."""
    out = np.zeros((max(n, 1), 3))
    words = (C.c_uint64 * 312)()
    idx, draws = C.c_uint64(), C.c_uint64()
    if device is None:
        L.check(L.load().gcmc_random_initial_configuration(n, box_length, min_sep, seed, L.dptr(out),
                                                           words, C.byref(idx), C.byref(draws)))
    else:
        L.check(L.load().gcmc_device_initial_configuration(device, n, box_length, min_sep, seed,
                                                           L.dptr(out), words, C.byref(idx),
                                                           C.byref(draws)))
    return out[:n].copy(), RngState(np.frombuffer(words, dtype=np.uint64).copy(), idx.value,
                                    draws.value)


def _params(cfg: RunConfig, engine_ctas=0, engine_group=0, engine_variants=0, engine_bias=0,
            max_particles=0, engine_mode=0, engine_share=0) -> L.GcmcParams:
    return L.GcmcParams(
        box_length=cfg.box_length, epsilon=cfg.epsilon, sigma=cfg.sigma, r_cut=cfg.r_cut,
        temperature=cfg.temperature, chemical_potential=cfg.chemical_potential,
        lambda_=cfg.lambda_, displace_percent=cfg.displace_percent,
        max_displacement=cfg.max_displacement, equilibration_steps=cfg.equilibration_steps,
        sampling_interval=cfg.sampling_interval, strategy=STRATEGIES.index(cfg.strategy),
        cell_capacity=cfg.cell_capacity, microcell_capacity=cfg.microcell_capacity,
        tail_corrections=int(cfg.tail_corrections), max_particles=max_particles,
        engine_ctas=engine_ctas, engine_group=engine_group, engine_variants=engine_variants,
        engine_bias=engine_bias, engine_mode=engine_mode, engine_share=engine_share)


class _Device:
    """Owns one gcmc_dev handle."""

    def __init__(self, cfg: RunConfig, device: int = 0, **engine_kw):
        lib = L.load()
        self.lib = lib
        self.cfg = cfg
        h = C.c_void_p()
        p = _params(cfg, **engine_kw)
        L.check(lib.gcmc_create(C.byref(p), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.gcmc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass

    # ---- store
    def upload(self, xyz):
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        L.check(self.lib.gcmc_upload_positions(self.h, L.dptr(xyz), len(xyz)))

    def size(self) -> int:
        n = C.c_uint64()
        L.check(self.lib.gcmc_download_positions(self.h, None, 0, C.byref(n)))
        return n.value

    def positions(self) -> np.ndarray:
        n = self.size()
        out = np.zeros((max(n, 1), 3))
        cnt = C.c_uint64()
        L.check(self.lib.gcmc_download_positions(self.h, L.dptr(out), max(n, 1), C.byref(cnt)))
        return out[: cnt.value].copy()

    # ---- rng
    def set_rng(self, r: RngState):
        w = np.ascontiguousarray(r.words, np.uint64)
        L.check(self.lib.gcmc_set_rng_state(self.h, w.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            int(r.index), int(r.draws)))

    def get_rng(self) -> RngState:
        w = np.zeros(312, np.uint64)
        idx, dr = C.c_uint64(), C.c_uint64()
        L.check(self.lib.gcmc_get_rng_state(self.h, w.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            C.byref(idx), C.byref(dr)))
        return RngState(w, idx.value, dr.value)

    # ---- state
    def get_state(self) -> L.GcmcState:
        s = L.GcmcState()
        L.check(self.lib.gcmc_get_state(self.h, C.byref(s)))
        return s

    def set_state(self, s: L.GcmcState):
        L.check(self.lib.gcmc_set_state(self.h, C.byref(s)))

    def total_energy(self):
        u, w = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_total_energy(self.h, C.byref(u), C.byref(w)))
        return u.value, w.value

    def total_energy_bruteforce(self):
        """O(N^2) device cross-check of total_energy() (no cell structure)."""
        u, w = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_total_energy_bruteforce(self.h, C.byref(u), C.byref(w)))
        return u.value, w.value

    def energy_timing(self):
        """Device ms of the last total_energy(): (whole pass, pair kernel)."""
        a, b = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_energy_timing(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def energy_drift(self):
        """Largest |maintained - fresh| per-particle pair energy / virial
        (gcmc_energy_drift; 0, 0 when the per-window engine ran last)."""
        u, w = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_energy_drift(self.h, C.byref(u), C.byref(w)))
        return u.value, w.value

    def rebuild(self):
        """NeighborStrategy::build() (strategy.hpp:34): bins the store afresh,
        ascending ids per cell, as the reference's constructors do."""
        L.check(self.lib.gcmc_build(self.h))

    def store_set(self, pid: int, pos):
        """ParticleStore::set (particles.hpp:26): the store only, grid untouched."""
        L.check(self.lib.gcmc_store_set(self.h, pid, L.dptr(np.ascontiguousarray(pos, np.float64))))

    def rebuild_check(self) -> Optional[str]:
        buf = C.create_string_buffer(512)
        clean = C.c_int32()
        L.check(self.lib.gcmc_rebuild_check(self.h, buf, 512, C.byref(clean)))
        return None if clean.value else buf.value.decode()

    def grid_info(self):
        d, cap, nc = C.c_int32(), C.c_int32(), C.c_uint64()
        L.check(self.lib.gcmc_grid_info(self.h, C.byref(d), C.byref(cap), C.byref(nc)))
        return d.value, cap.value, nc.value

    def grid(self):
        d, cap, nc = self.grid_info()
        occ = np.zeros(nc, np.int32)
        slots = np.zeros(nc * cap, np.int32)
        if nc:
            L.check(self.lib.gcmc_download_grid(self.h, occ.ctypes.data_as(C.POINTER(C.c_int32)),
                                                slots.ctypes.data_as(C.POINTER(C.c_int32))))
        return occ, slots

    def peak(self) -> int:
        p = C.c_int32()
        L.check(self.lib.gcmc_peak_occupancy(self.h, C.byref(p)))
        return p.value


class GpuNeighborStrategy(_Device):
    """NeighborStrategy (strategy.hpp:27-50) on the device. The strategy owns
    its store (device positions); ``positions()`` downloads it."""

    def __init__(self, strategy: str, positions, box_length: float, epsilon=1.0, sigma=1.0,
                 r_cut=2.5, capacity=0, device=0):
        cfg = RunConfig(temperature=1.0, box_length=box_length, epsilon=epsilon, sigma=sigma,
                        r_cut=r_cut, strategy=strategy,
                        cell_capacity=capacity if strategy == "cell_list" else 0,
                        microcell_capacity=capacity if strategy == "microcell" and capacity else 5)
        super().__init__(cfg, device)
        self.upload(positions)  # the reference ctor builds immediately

    def name(self) -> str:
        return self.cfg.strategy

    def build(self):
        self.rebuild()

    def delta_displace(self, pid: int, pos) -> PairInteraction:
        p = np.asarray(pos, np.float64)
        u, w = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_delta_displace(self.h, pid, L.dptr(p), C.byref(u), C.byref(w)))
        return PairInteraction(u.value, w.value)

    def delta_insert(self, pos) -> PairInteraction:
        p = np.asarray(pos, np.float64)
        u, w = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_delta_insert(self.h, L.dptr(p), C.byref(u), C.byref(w)))
        return PairInteraction(u.value, w.value)

    def delta_delete(self, pid: int) -> PairInteraction:
        u, w = C.c_double(), C.c_double()
        L.check(self.lib.gcmc_delta_delete(self.h, pid, C.byref(u), C.byref(w)))
        return PairInteraction(u.value, w.value)

    def delta_batch(self, kinds, pids, xyz):
        """Many proposals against the same state (one warp each)."""
        kinds = np.ascontiguousarray(kinds, np.int32)
        pids = np.ascontiguousarray(pids, np.uint64)
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        n = len(kinds)
        du, dw = np.zeros(n), np.zeros(n)
        L.check(self.lib.gcmc_delta_batch(self.h, n, kinds.ctypes.data_as(C.POINTER(C.c_int32)),
                                          pids.ctypes.data_as(C.POINTER(C.c_uint64)), L.dptr(xyz),
                                          L.dptr(du), L.dptr(dw)))
        return du, dw

    def commit_displace(self, pid: int, pos):
        L.check(self.lib.gcmc_commit_displace(self.h, pid, L.dptr(np.asarray(pos, np.float64))))

    def commit_insert(self, pos) -> int:
        pid = C.c_uint64()
        L.check(self.lib.gcmc_commit_insert(self.h, L.dptr(np.asarray(pos, np.float64)),
                                            C.byref(pid)))
        return pid.value

    def commit_delete(self, pid: int):
        L.check(self.lib.gcmc_commit_delete(self.h, pid))

    def peak_cell_occupancy(self) -> int:
        return self.peak()

    def occupancy_view(self):
        return self.grid()[0]

    def slots_view(self):
        return self.grid()[1]


def total_energy(positions, box_length, epsilon=1.0, sigma=1.0, r_cut=2.5, device=0):
    """engine.hpp:74-94 on the device (raises GcmcError OVERLAP like the
    reference's runtime_error)."""
    d = _Device(RunConfig(temperature=1.0, box_length=box_length, epsilon=epsilon, sigma=sigma,
                          r_cut=r_cut, strategy="all_pairs"), device)
    d.upload(positions)
    try:
        return d.total_energy()
    finally:
        d.close()


class Simulation:
    """gcmc::Simulation (engine.hpp:214-437) with the move loop on the B200.

    Simulation(cfg)                                   fresh   (engine.hpp:216-227)
    Simulation(cfg, positions, rng)                   prepared (engine.hpp:231-239)
    Simulation(cfg, positions, rng, step, U, W)       resume  (engine.hpp:244-252)
    """

    def __init__(self, cfg: RunConfig, positions=None, rng: Optional[RngState] = None,
                 step: Optional[int] = None, energy: float = 0.0, virial: float = 0.0,
                 device: int = 0, **engine_kw):
        cfg.validate()
        self.cfg = cfg
        self.dev = _Device(cfg, device, **engine_kw)
        if positions is None:
            if cfg.initial_particles > 0:
                positions, rng = random_initial_configuration(cfg.initial_particles,
                                                              cfg.box_length, 0.85 * cfg.sigma,
                                                              cfg.seed, device=device)
            else:
                positions, rng = np.zeros((0, 3)), RngState.from_seed(cfg.seed)
        if rng is None:
            raise ValueError("an RNG state is required with explicit positions")
        self.dev.upload(positions)
        self.dev.set_rng(rng)
        st = self.dev.get_state()
        if step is None:  # fresh / prepared: total energy
            st.step = 0
            st.energy, st.virial = self.dev.total_energy()
        else:  # resume: adopt verbatim
            st.step = step
            st.energy, st.virial = energy, virial
        self.dev.set_state(st)
        self.last_run = None

    # ---- accessors (engine.hpp:261-291)
    def config(self):
        return self.cfg

    def current_step(self) -> int:
        return self.dev.get_state().step

    def particle_count(self) -> int:
        return self.dev.get_state().n

    def particles(self) -> np.ndarray:
        return self.dev.positions()

    def rng(self) -> RngState:
        return self.dev.get_rng()

    def state(self) -> SystemState:
        s = self.dev.get_state()
        return SystemState(s.energy, s.virial, list(s.attempted), list(s.accepted))

    def statistics(self) -> RunStatistics:
        s = self.dev.get_state()
        return RunStatistics(s.samples, s.sum_u, s.sum_p, s.sum_n, s.sum_n2)

    def density(self) -> float:
        return self.particle_count() / self.cfg.volume()

    def pressure(self) -> float:
        s = self.dev.get_state()
        rho = s.n / self.cfg.volume()
        p = rho * self.cfg.temperature + s.virial / (3.0 * self.cfg.volume())
        if self.cfg.tail_corrections:
            p += tail_corrections(rho, self.cfg.epsilon, self.cfg.sigma, self.cfg.r_cut)[1]
        return p

    def reported_energy(self) -> float:
        s = self.dev.get_state()
        u = s.energy
        if self.cfg.tail_corrections:
            rho = s.n / self.cfg.volume()
            u += s.n * tail_corrections(rho, self.cfg.epsilon, self.cfg.sigma, self.cfg.r_cut)[0]
        return u

    def peak_cell_occupancy(self) -> int:
        return self.dev.peak()

    # ---- moves
    def run(self, n: int, trace: bool = False):
        """n x step() on the device; returns the per-move trace if asked."""
        tr = np.zeros(max(n, 1), L.TRACE_DTYPE) if trace else None
        res = L.GcmcRunResult()
        L.check(self.dev.lib.gcmc_run_moves(self.dev.h, n, tr.ctypes.data if trace else None,
                                            C.byref(res)))
        self.last_run = res
        return tr[:n] if trace else None

    def step(self) -> MoveOutcome:
        t = self.run(1, trace=True)[0]
        return MoveOutcome(MOVE_KINDS[t["kind"]], bool(t["accepted"]), float(t["delta_u"]),
                           float(t["delta_w"]), float(t["acceptance_prob"]))

    def audit(self) -> AuditReport:
        """engine.hpp:333-342 on the device."""
        s = self.dev.get_state()
        u, w = self.dev.total_energy()
        return AuditReport(s.energy, u, s.virial, w, self.dev.rebuild_check())

    def run_to(self, target_step: int, on_checkpoint: Optional[Callable] = None):
        """engine.hpp:314-325: audits at every checkpoint boundary and at the
        target; one device batch per interval."""
        step = self.current_step()
        ci = self.cfg.checkpoint_interval
        while step < target_step:
            nxt = min(target_step, (step // ci + 1) * ci)
            self.run(nxt - step)
            step = nxt
            report = self.audit()
            if not report.passed():
                raise AuditFailure(f"audit failed at step {step}: {report.describe()}")
            if on_checkpoint:
                on_checkpoint(self, report)

    def close(self):
        self.dev.close()


def run_chains(sims, n):
    """Advance independent Simulations concurrently (gcmc_run_chains): the
    points of a mu/T sweep as K chains on one device (create each with
    ``engine_share=K``). ``n`` is one move count for all or one per chain.
    Every chain ends exactly where ``sim.run(n)`` alone would leave it."""
    sims = list(sims)
    k = len(sims)
    counts = [int(n)] * k if np.isscalar(n) else [int(x) for x in n]
    if len(counts) != k:
        raise ValueError("one move count per chain")
    hs = (C.c_void_p * k)(*[s.dev.h for s in sims])
    ns = (C.c_uint64 * k)(*counts)
    res = (L.GcmcRunResult * k)()
    L.check(L.load().gcmc_run_chains(hs, k, ns, res))
    for s, r in zip(sims, res):
        s.last_run = r
    return list(res)
