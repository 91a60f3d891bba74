"""Parity of the B200 path (through the C ABI) against the CPU oracle.

The oracle is the real reference compiled from its own headers
(oracle/_ref/libgcmc_ref.so) when present, else the bit-exact C restatement
(oracle/liboracle.so; the two agree bitwise, tests/test_oracle_cpu.py).

Bars (BASELINE.json north_star): identical cell assignments / slot arrays
(byte compare), ΔE within 1e-10 relative (floor 1, validate.hpp:47-49),
identical accept decisions and kinds for the first 1e5 moves, identical
positions and RNG state, ensemble averages within statistical error.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-10
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def E():
    from paper_1408_3764_b200 import engine

    return engine


def use_ref() -> bool:
    return os.path.exists(O.REF_SO) or os.path.isdir(O.REF_INC)


def oracle_grid(kind, xyz, box, cap=0):
    if use_ref():
        return O.RefStrategy(kind, xyz, box, capacity=cap)
    return O.PortGrid(kind, xyz, box, capacity=cap)


def oracle_sim(strategy, box, xyz, rng_hex, energy, virial, **kw):
    """Resumed oracle simulation (engine.hpp:244-252) with trace support."""
    kw = dict(kw)
    if use_ref():
        cfg = O.ref_config(box_length=box, strategy=strategy, **kw)
        return O.RefSim(cfg, mode=2, xyz=xyz, rng_hex=rng_hex, energy=energy, virial=virial)
    p = O.port_params(box_length=box, strategy=strategy, **kw)
    return _PortAdapter(O.PortSim(p, xyz, O.rng_from_hex(rng_hex), energy=energy,
                                  virial=virial))


class _PortAdapter:
    def __init__(self, s):
        self.s = s

    def run(self, n, trace=False):
        return 0.0, self.s.run(n, trace=trace)

    def positions(self):
        return self.s.grid()[0]

    def rng_hex(self):
        return O.rng_to_hex(self.s.rng())

    def state(self):
        return self.s.state()


def config(n0, seed=1, density=0.67):
    box = (n0 / density) ** (1.0 / 3.0)
    xyz, rng = E().random_initial_configuration(n0, box, 0.85, seed)
    return box, xyz, rng


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(1.0, np.abs(np.asarray(b)))


# --------------------------------------------------------------------- (a) build
@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
@pytest.mark.parametrize("n0", [2048, 32768])
def test_build_byte_identical(strategy, n0):
    box, xyz, _ = config(n0)
    g = E().GpuNeighborStrategy(strategy, xyz, box)
    o = oracle_grid(strategy, xyz, box)
    occ, slots = g.grid()
    roc, rsl = o.grid()
    assert np.array_equal(occ, roc)
    assert np.array_equal(slots, rsl)
    assert g.rebuild_check() is None
    assert g.peak_cell_occupancy() == o.peak()


def test_build_byte_identical_1m_microcell():
    box, xyz, _ = config(1 << 20)
    g = E().GpuNeighborStrategy("microcell", xyz, box)
    o = oracle_grid("microcell", xyz, box)
    occ, slots = g.grid()
    roc, rsl = o.grid()
    assert np.array_equal(occ, roc) and np.array_equal(slots, rsl)


def test_golden_grids():
    gold = np.load(os.path.join(GOLD, "golden.npz"))
    import json

    meta = json.load(open(os.path.join(GOLD, "golden.json")))
    box = meta["init_256_box"]
    for strat, key in (("microcell", "micro"), ("cell_list", "cell")):
        g = E().GpuNeighborStrategy(strat, gold["init_256_xyz"], box)
        occ, slots = g.grid()
        assert np.array_equal(occ, gold[f"grid_{key}_occ"])
        assert np.array_equal(slots, gold[f"grid_{key}_slots"])


def test_overflow_is_a_hard_error_naming_the_cell():
    # test_grids.cpp:208-226
    from paper_1408_3764_b200 import _lib

    store = np.array([[0.1 + 0.13 * i, 0.5, 0.5] for i in range(6)])
    with pytest.raises(_lib.GcmcError) as ei:
        E().GpuNeighborStrategy("microcell", store, 10.0)
    assert ei.value.status == "CELL_OVERFLOW"
    assert "microcell: cell 0 exceeds capacity 5" in str(ei.value)
    roomy = E().GpuNeighborStrategy("microcell", store, 10.0, capacity=8)
    assert roomy.occupancy_view()[0] == 6
    rng = O.port_rng(9)
    lib = O.port_lib()
    crowded = np.array([[lib.orc_uniform(C.byref(rng)) * 2.4 for _ in range(3)] for _ in range(49)])
    with pytest.raises(_lib.GcmcError) as ei:
        E().GpuNeighborStrategy("cell_list", crowded, 10.0)
    assert "capacity 48" in str(ei.value)


# --------------------------------------------------------------------- (b) ΔE
def proposals(n0, box, k, seed):
    rs = np.random.default_rng(seed)
    kinds = np.arange(k) % 3
    pids = rs.integers(0, n0, k)
    pts = rs.random((k, 3)) * box
    return kinds, pids, pts


def oracle_deltas(o, kinds, pids, pts):
    out = []
    for kd, pid, p in zip(kinds, pids, pts):
        if kd == 0:
            out.append(o.delta_displace(int(pid), p))
        elif kd == 1:
            out.append(o.delta_insert(p))
        else:
            out.append(o.delta_delete(int(pid)))
    return np.array(out)


@pytest.mark.parametrize("strategy", ["microcell", "cell_list", "all_pairs"])
@pytest.mark.parametrize("n0", [2048, 32768])
def test_deltas_within_tolerance(strategy, n0):
    box, xyz, _ = config(n0)
    g = E().GpuNeighborStrategy(strategy, xyz, box)
    o = oracle_grid(strategy, xyz, box)
    kinds, pids, pts = proposals(n0, box, 600, 5)
    du, dw = g.delta_batch(kinds, pids, pts)
    ref = oracle_deltas(o, kinds, pids, pts)
    assert rel(du, ref[:, 0]).max() <= TOL
    assert rel(dw, ref[:, 1]).max() <= TOL


@pytest.mark.parametrize("strategy", ["microcell", "cell_list", "all_pairs"])
def test_deltas_match_golden(strategy):
    import json

    gold = np.load(os.path.join(GOLD, "golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "golden.json")))
    g = E().GpuNeighborStrategy(strategy, gold["init_256_xyz"], meta["init_256_box"])
    rows = gold[f"deltas_{strategy}"]
    du, dw = g.delta_batch(rows[:, 0].astype(np.int32), rows[:, 1].astype(np.uint64), rows[:, 2:5])
    assert rel(du, rows[:, 5]).max() <= TOL
    assert rel(dw, rows[:, 6]).max() <= TOL


def test_trivial_deltas():
    # test_grids.cpp:261-295
    g = E().GpuNeighborStrategy("microcell", np.zeros((0, 3)), 12.0)
    assert g.delta_insert([1.0, 1.0, 1.0]).u == 0.0
    rmin = 2.0 ** (1.0 / 6.0)
    pair = np.array([[1.0, 1.0, 1.0], [1.0 + rmin, 1.0, 1.0]])
    from paper_1408_3764_b200 import _lib

    for strat in ("microcell", "cell_list", "all_pairs"):
        s = E().GpuNeighborStrategy(strat, pair, 12.0)
        assert abs(s.delta_displace(1, [7.0, 7.0, 7.0]).u - 1.0) <= 1e-12
        with pytest.raises(_lib.GcmcError) as ei:
            s.delta_displace(99, [2.0, 2.0, 2.0])
        assert ei.value.status == "INVALID_PID"
        assert f"{strat}: invalid particle id" in str(ei.value)
    box, fluid, _ = config(400, seed=8, density=400 / 12.0 ** 3)
    grid = E().GpuNeighborStrategy("microcell", fluid, 12.0)
    pos = [3.7, 8.1, 0.4]
    ins = grid.delta_insert(pos)
    pid = grid.commit_insert(pos)
    dele = grid.delta_delete(pid)
    assert dele.u == -ins.u and dele.w == -ins.w


def test_tiny_box_clamps_window():
    # test_grids.cpp:336-359: L = 5.2, 6 cells per axis, window = whole box
    box = 5.2
    xyz, _ = E().random_initial_configuration(40, box, 0.85, 44)
    g = E().GpuNeighborStrategy("microcell", xyz, box)
    o = oracle_grid("all_pairs", xyz, box)
    kinds, pids, pts = proposals(40, box, 200, 3)
    du, _ = g.delta_batch(kinds, pids, pts)
    ref = oracle_deltas(o, kinds, pids, pts)
    assert rel(du, ref[:, 0]).max() <= 1e-12


# --------------------------------------------------------------------- commits
@pytest.mark.parametrize("strategy", ["microcell", "cell_list", "all_pairs"])
def test_commit_sequence_byte_identical(strategy):
    n0 = 2048
    box, xyz, _ = config(n0, seed=2)
    g = E().GpuNeighborStrategy(strategy, xyz, box)
    o = oracle_grid(strategy, xyz, box)
    rs = np.random.default_rng(11)
    n = n0
    for step in range(600):
        kind = int(rs.integers(0, 3))
        if kind == 0:
            pid, p = int(rs.integers(0, n)), rs.random(3) * box
            if step % 7 == 0:  # same-cell displacement fast path
                q = o.positions()[pid] if hasattr(o, "positions") else None
                if q is not None:
                    p = np.minimum(np.floor(q) + 0.5, box - 1e-9)
            g.commit_displace(pid, p)
            o.commit_displace(pid, p)
        elif kind == 1:
            p = rs.random(3) * box
            a, b = g.commit_insert(p), o.commit_insert(p)
            assert a == b
            n += 1
        else:
            pid = int(rs.integers(0, n))
            g.commit_delete(pid)
            o.commit_delete(pid)
            n -= 1
        if step % 100 == 99:
            assert np.array_equal(g.positions(), o.positions())
            if strategy != "all_pairs":
                a, b = g.grid(), o.grid()
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                assert g.rebuild_check() is None
    assert g.peak_cell_occupancy() == o.peak()


# --------------------------------------------------------------------- (c) total energy
@pytest.mark.parametrize("n0", [2048, 32768])
def test_total_energy_matches_reference(n0):
    box, xyz, _ = config(n0)
    u, w = E().total_energy(xyz, box)
    ru, rw = C.c_double(), C.c_double()
    if use_ref():
        O.ref_lib().ref_total_energy(O.dptr(xyz), n0, box, 1.0, 1.0, 2.5, C.byref(ru), C.byref(rw))
    else:
        O.port_lib().orc_total_energy(O.dptr(xyz), n0, box, 1.0, 1.0, 2.5, C.byref(ru), C.byref(rw))
    assert abs(u - ru.value) <= TOL * max(1.0, abs(ru.value))
    assert abs(w - rw.value) <= TOL * max(1.0, abs(rw.value))


def test_total_energy_landmarks_and_overlap():
    # test_engine.cpp:55-84
    from paper_1408_3764_b200 import _lib

    rmin = 2.0 ** (1.0 / 6.0)
    u, w = E().total_energy(np.array([[1.0, 1, 1], [1.0 + rmin, 1, 1]]), 20.0)
    assert abs(u + 1.0) <= 1e-13 and abs(w) <= 1e-12
    tri = np.array([[5.0, 5, 5], [6.0, 5, 5], [5.5, 5 + math.sqrt(3) / 2, 5]])
    assert abs(E().total_energy(tri, 20.0)[0]) <= 1e-12
    with pytest.raises(_lib.GcmcError) as ei:
        E().total_energy(np.array([[1.0, 1, 1], [1.0, 1, 1]]), 20.0)
    assert ei.value.status == "OVERLAP" and "particles 0 and 1 overlap" in str(ei.value)


def test_total_energy_1m_against_pair_sum_identity():
    """At 1M the O(N^2) oracle takes hours; check the size-independent identity
    U_total = 1/2 sum_i u_i where u_i = -delta_delete(i) (each pair counted
    twice) on a random subset-free sample: sum over all i of the deletion ΔE."""
    box, xyz, _ = config(1 << 17)
    g = E().GpuNeighborStrategy("microcell", xyz, box)
    u, w = g.total_energy()
    n = len(xyz)
    kinds = np.full(n, 2, np.int32)
    du, dw = g.delta_batch(kinds, np.arange(n, dtype=np.uint64), np.zeros((n, 3)))
    assert abs(u - (-0.5 * du.sum())) <= 1e-9 * abs(u)
    assert abs(w - (-0.5 * dw.sum())) <= 1e-9 * abs(w)


def test_total_energy_1m_against_device_bruteforce():
    """the 1M total energy against an independent O(N^2) device
    pass (every pair i < j, no cell structure, engine.hpp:74-94's loop), at
    the bench's start configuration and after 2^22 moves; the cell pass is
    bitwise reproducible."""
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(1 << 20)
    sim = E().Simulation(RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box,
                                   strategy="microcell"), xyz, rng)
    for rep in range(2):
        u, w = sim.dev.total_energy()
        bu, bw = sim.dev.total_energy_bruteforce()
        assert abs(u - bu) <= TOL * abs(bu), (u, bu)
        assert abs(w - bw) <= TOL * abs(bw), (w, bw)
        assert sim.dev.total_energy() == (u, w)
        pass_ms, kern_ms = sim.dev.energy_timing()
        assert 0.0 < kern_ms <= pass_ms
        sim.run(1 << 22)
    sim.close()


@pytest.mark.parametrize("box,rc,n0", [(6.0, 2.5, 120), (9.0, 2.5, 400), (13.23, 4.25, 1389),
                                       (13.23, 2.75, 1389)])
def test_total_energy_grid_shapes(box, rc, n0):
    """Both cell passes (27-cell stencil below 5 half-width cells per axis, the
    5^3 sub-cell stencil from there on) against the reference's O(N^2) loop
    and the device brute force, at several cutoffs."""
    xyz, _ = E().random_initial_configuration(n0, box, 0.85, 3)
    g = E().GpuNeighborStrategy("microcell", xyz, box, r_cut=rc)
    u, w = g.total_energy()
    bu, bw = g.total_energy_bruteforce()
    ru, rw = C.c_double(), C.c_double()
    if use_ref():
        O.ref_lib().ref_total_energy(O.dptr(xyz), n0, box, 1.0, 1.0, rc, C.byref(ru), C.byref(rw))
    else:
        O.port_lib().orc_total_energy(O.dptr(xyz), n0, box, 1.0, 1.0, rc, C.byref(ru), C.byref(rw))
    for a in (u, bu):
        assert abs(a - ru.value) <= TOL * max(1.0, abs(ru.value)), (a, ru.value)
    for a in (w, bw):
        assert abs(a - rw.value) <= TOL * max(1.0, abs(rw.value)), (a, rw.value)


# --------------------------------------------------------------------- (d) engine
def run_pair(strategy, n0, moves, mu, seed=1, **kw):
    box, xyz, rng = config(n0, seed=seed)
    from paper_1408_3764_b200.config import RunConfig

    cfg = RunConfig(temperature=2.0, chemical_potential=mu, box_length=box, strategy=strategy,
                    seed=seed, **kw)
    sim = E().Simulation(cfg, xyz, rng)
    st = sim.dev.get_state()
    tr = sim.run(moves, trace=True)
    extra = {k: v for k, v in kw.items()}
    o = oracle_sim(strategy, box, xyz, rng.serialize_hex(), st.energy, st.virial,
                   temperature=2.0, chemical_potential=mu, **extra)
    _, tp = o.run(moves, trace=True)
    return sim, tr, o, tp


def assert_trace_parity(tr, tp):
    assert np.array_equal(tr["kind"], tp["kind"])
    bad = np.nonzero(tr["accepted"] != tp["accepted"])[0]
    assert bad.size == 0, f"first decision mismatch at move {bad[:1]}"
    assert np.array_equal(tr["n_after"], tp["n_after"])
    assert rel(tr["delta_u"], tp["delta_u"]).max() <= TOL
    assert rel(tr["delta_w"], tp["delta_w"]).max() <= TOL
    assert rel(tr["acceptance_prob"], tp["acceptance_prob"]).max() <= 1e-9


@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
@pytest.mark.parametrize("mu", [-2.0, 1.0])
def test_first_1e5_moves_identical(strategy, mu):
    sim, tr, o, tp = run_pair(strategy, 2048, 100000, mu)
    assert_trace_parity(tr, tp)
    assert np.array_equal(sim.particles(), o.positions())
    assert sim.rng().serialize_hex() == o.rng_hex()
    st, rs = sim.dev.get_state(), o.state()
    assert list(st.attempted) == list(rs.attempted) and list(st.accepted) == list(rs.accepted)
    assert st.samples == rs.samples and st.sum_n == rs.sum_n and st.sum_n2 == rs.sum_n2
    assert abs(st.energy - rs.energy) <= 1e-9 * max(1.0, abs(rs.energy))
    assert abs(st.sum_u - rs.sum_u) <= 1e-9 * max(1.0, abs(rs.sum_u))


def test_maintained_energies_do_not_drift():
    """The maintained-energy engine's per-particle e_i stay equal (to rounding)
    to a from-scratch evaluation after many accepted moves."""
    sim, tr, o, tp = run_pair("microcell", 32768, 200000, 1.0)
    assert_trace_parity(tr, tp)
    du, dw = sim.dev.energy_drift()
    assert du <= 1e-11 and dw <= 1e-10, (du, dw)
    assert int(tr["accepted"].sum()) > 1000


def test_per_window_engine_still_identical():
    """engine_mode=1 forces the per-window engine (engine.cu) on a strategy the
    maintained-energy engine also supports: same decisions."""
    box, xyz, rng = config(2048)
    from paper_1408_3764_b200.config import RunConfig

    cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
    a = E().Simulation(cfg, xyz, rng)
    b = E().Simulation(cfg, xyz, rng, engine_mode=1)
    ta, tb = a.run(50000, trace=True), b.run(50000, trace=True)
    assert np.array_equal(ta["accepted"], tb["accepted"])
    assert np.array_equal(ta["n_after"], tb["n_after"])
    assert rel(ta["delta_u"], tb["delta_u"]).max() <= TOL
    assert b.dev.energy_drift() == (0.0, 0.0)


def test_all_pairs_trajectory_identical():
    sim, tr, o, tp = run_pair("all_pairs", 1024, 5000, -2.0)
    assert_trace_parity(tr, tp)
    assert np.array_equal(sim.particles(), o.positions())


def test_max_displacement_and_tail_and_sampling_interval():
    sim, tr, o, tp = run_pair("microcell", 2048, 20000, 1.0, displace_percent=0.5,
                              max_displacement=0.4, tail_corrections=1, equilibration_steps=777,
                              sampling_interval=7)
    assert_trace_parity(tr, tp)
    st, rs = sim.dev.get_state(), o.state()
    assert st.samples == rs.samples == (20000 - 777) // 7
    assert abs(st.sum_p - rs.sum_p) <= 1e-9 * abs(rs.sum_p)
    assert abs(st.sum_u - rs.sum_u) <= 1e-9 * abs(rs.sum_u)


def test_first_1e5_moves_identical_at_1m():
    sim, tr, o, tp = run_pair("microcell", 1 << 20, 100000, 1.0)
    assert_trace_parity(tr, tp)
    assert sim.rng().serialize_hex() == o.rng_hex()


def test_run_is_chunk_invariant_and_resumable():
    """n moves in one call == the same n moves split over calls: identical
    decisions, N, positions and RNG state (bitwise); ΔU / ΔW / p to rounding
    (a move evaluated in the round after an accepted neighbour adds that
    neighbour's pair change instead of re-reading it, so the last bits of its
    ΔU depend on where the round boundaries fell)."""
    box, xyz, rng = config(2048, seed=5)
    from paper_1408_3764_b200.config import RunConfig

    cfg = RunConfig(temperature=2.0, chemical_potential=-1.0, box_length=box,
                    strategy="microcell", seed=5)
    a = E().Simulation(cfg, xyz, rng)
    b = E().Simulation(cfg, xyz, rng)
    ta = a.run(30000, trace=True)
    tb = np.concatenate([b.run(k, trace=True) for k in (1, 2, 997, 12000, 17000)])
    for f in ("kind", "accepted", "n_after"):
        assert np.array_equal(ta[f], tb[f]), f
    for f in ("delta_u", "delta_w", "acceptance_prob"):
        assert rel(ta[f], tb[f]).max() <= 1e-12, f
    assert np.array_equal(a.particles(), b.particles())
    assert a.rng().serialize_hex() == b.rng().serialize_hex()


def test_gpu_checkpoint_resumes_on_reference_bitwise():
    """Equilibrate on the device, write a reference-format checkpoint, resume the
    reference from it: both continuations make identical decisions."""
    if not use_ref():
        pytest.skip("needs the compiled reference")
    from paper_1408_3764_b200 import checkpoint as CK
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(4096, seed=3)
    cfg = RunConfig(temperature=2.0, chemical_potential=0.0, box_length=box,
                    strategy="microcell", seed=3, checkpoint_interval=5000)
    sim = E().Simulation(cfg, xyz, rng)
    sim.run(50000)
    text = CK.to_text(CK.snapshot(sim))
    ref = O.RefSim.from_checkpoint(text)
    _, tp = ref.run(20000, trace=True)
    tr = sim.run(20000, trace=True)
    assert_trace_parity(tr, tp)
    assert np.array_equal(sim.particles(), ref.positions())


def test_audit_and_run_to():
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(2000, seed=7, density=0.6)
    cfg = RunConfig(temperature=2.0, chemical_potential=-2.0, box_length=box,
                    strategy="microcell", seed=7, checkpoint_interval=10000, steps=50000)
    sim = E().Simulation(cfg, xyz, rng)
    seen = []
    sim.run_to(50000, lambda s, r: seen.append((s.current_step(), r)))
    assert [s for s, _ in seen] == [10000, 20000, 30000, 40000, 50000]
    for _, r in seen:
        assert r.passed(), r.describe()
        assert abs(r.u_tracked - r.u_recomputed) <= 1e-8 * max(1.0, abs(r.u_recomputed))


def test_ideal_gas_poisson():
    # validate.hpp:299-331 / test_engine.cpp:160-164 (epsilon = 0)
    from paper_1408_3764_b200.config import RunConfig

    target, l = 300.0, 10.0
    cfg = RunConfig(temperature=1.0, epsilon=0.0, box_length=l,
                    chemical_potential=math.log(target / l ** 3), strategy="microcell",
                    seed=2024, equilibration_steps=20000, microcell_capacity=64)
    sim = E().Simulation(cfg)
    sim.run(150000)
    st = sim.statistics()
    mean = st.mean_n()
    assert abs(mean - target) / target <= 0.05
    assert abs(st.variance_n() / mean - 1.0) <= 0.25


def test_epsilon_zero_identical_across_strategies():
    # test_engine.cpp:143-158
    from paper_1408_3764_b200.config import RunConfig

    traces = []
    for strat in ("all_pairs", "cell_list", "microcell"):
        cfg = RunConfig(temperature=1.0, epsilon=0.0, box_length=10.0,
                        chemical_potential=math.log(100.0 / 1000.0), strategy=strat, seed=1234,
                        microcell_capacity=64, cell_capacity=128)
        sim = E().Simulation(cfg)
        traces.append(sim.run(20000, trace=True))
    assert np.array_equal(traces[0]["n_after"], traces[1]["n_after"])
    assert np.array_equal(traces[0]["n_after"], traces[2]["n_after"])


def test_draw_counts_match_reference():
    sim, tr, o, tp = run_pair("microcell", 512, 3000, -2.0)
    r = sim.rng()
    # 6 / 6 / 4 draws per displace / insert / delete (engine.hpp:207-213)
    kinds = tr["kind"]
    expect = 6 * np.sum(kinds == 0) + 6 * np.sum(kinds == 1) + 4 * np.sum(kinds == 2)
    start = E().random_initial_configuration(512, (512 / 0.67) ** (1 / 3), 0.85, 1)[1].draws
    assert r.draws - start == expect


@pytest.mark.parametrize("strategy,n0", [("microcell", 4096), ("cell_list", 4096), ("all_pairs", 1024)])
def test_drop_in_strategy_against_reference(strategy, n0):
    """include/gcmc_b200_strategy.hpp as a gcmc::NeighborStrategy, driven
    side by side with the reference's own strategy (oracle/shim_check.cpp):
    ΔE within 1e-10, identical stores, byte-identical grids after commits,
    clean rebuild_check, the reference's exception types and messages."""
    import subprocess

    if not os.path.exists(O.SHIM):
        pytest.skip("oracle/_ref/shim_check not built (needs the reference headers)")
    r = subprocess.run([O.SHIM, strategy, str(n0), "3000", "5"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fails=0" in r.stdout, r.stdout


# --------------------------------------------------------------------- (f4) initial configuration
@pytest.mark.parametrize("n,density,seed", [(2048, 0.67, 1), (32768, 0.67, 3), (262144, 0.67, 5),
                                            (1 << 20, 0.67, 1), (300, 0.75, 9), (5, 0.6, 2),
                                            (4000, 0.9, 11)])
def test_device_initial_configuration_bitwise(n, density, seed):
    """gcmc_device_initial_configuration == the host restatement (itself pinned
    to the reference, test_host_cpu) bit for bit: positions in order, MT state,
    position and draw count (init_config.hpp:19-64)."""
    box = (n / density) ** (1.0 / 3.0)
    hx, hr = E().random_initial_configuration(n, box, 0.85, seed, device=None)
    dx, dr = E().random_initial_configuration(n, box, 0.85, seed, device=0)
    assert np.array_equal(hx, dx)
    assert hr.serialize_hex() == dr.serialize_hex()
    if use_ref() and n <= 4096:
        rx, rh = O.ref_initial_configuration(n, box, seed)
        assert np.array_equal(dx, rx) and dr.serialize_hex() == rh


def test_device_initial_configuration_rejection_limit():
    """The reference's error after 10^6 consecutive rejections (a density the
    separation cannot reach), with the same text."""
    from paper_1408_3764_b200 import _lib

    with pytest.raises(_lib.GcmcError) as e1:
        E().random_initial_configuration(400, 5.0, 0.85, 1, device=0)
    with pytest.raises(_lib.GcmcError) as e2:
        E().random_initial_configuration(400, 5.0, 0.85, 1, device=None)
    assert str(e1.value) == str(e2.value)
    assert "consecutive rejections" in str(e1.value)
