"""Parity of the device ENGINE path (gcmc_run_moves) against the reference.

test_gpu_parity.py covers the plugin calls (build / ΔE / host-API commits)
and traces from the random start. This file covers what every benchmarked
move goes through:

* the reference grid the engine's committer maintains, byte-compared with the
  reference Simulation's own strategy (occupancy_view / slots_view after
  remove_id / relabel_id, microcell_grid.hpp:485-513, cell_grid.hpp:250-275)
  every 10^4 moves at 2k, 32k and 1M for both grid strategies;
* the bench regime: 1M particles after >= 2^24 warm-up moves (acceptance
  ~2.6 %, ~366 moves per round), then 2x10^5 traced moves against the
  reference resumed there (engine.hpp:244-252), full state compared;
* 256k (BASELINE configs[2]) in the same way;
* other cutoffs (T/acceptance.cpp:114-128: r_c in {2.75, 3.0, 3.75, 4.25} at
  L = 13.23 with a 0.23 sigma boundary microcell): ΔE and 10^4-move traces;
* the overlap clamp (potential.hpp:51-54, T/test_potential.cpp:82-92) on the
  device ΔE path;
* audit / rebuild_check fault injection (T/test_engine.cpp:186-192).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import (TOL, E, assert_trace_parity, config, oracle_deltas, oracle_grid,
                             oracle_sim, proposals, rel, use_ref)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not use_ref(), reason="needs the compiled reference (oracle/_ref)")]


def RC():
    from paper_1408_3764_b200.config import RunConfig

    return RunConfig


def grid_of(o):
    g = getattr(o, "grid", None)
    if g is not None:
        return g()
    pos, occ, slots = o.s.grid()  # restatement adapter
    return occ, slots


def sim_pair(strategy, n0, mu, seed=1, density=0.67, **kw):
    box, xyz, rng = config(n0, seed=seed, density=density)
    cfg = RC()(temperature=2.0, chemical_potential=mu, box_length=box, strategy=strategy,
               seed=seed, **kw)
    sim = E().Simulation(cfg, xyz, rng)
    st = sim.dev.get_state()
    o = oracle_sim(strategy, box, xyz, rng.serialize_hex(), st.energy, st.virial,
                   temperature=2.0, chemical_potential=mu, **kw)
    return sim, o


def assert_same_grid(sim, o, where=""):
    occ, slots = sim.dev.grid()
    roc, rsl = grid_of(o)
    assert np.array_equal(occ, roc), f"occupancy differs {where}"
    bad = np.nonzero(slots != rsl)[0]
    assert bad.size == 0, f"slots differ {where}: first at {bad[:4]} ({slots[bad[:4]]} vs {rsl[bad[:4]]})"


# ------------------------------------------------------------ engine-path grids
@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
@pytest.mark.parametrize("n0,chunks", [(2048, 10), (32768, 10), (1 << 20, 6)])
def test_engine_grid_byte_identical(strategy, n0, chunks):
    """The engine committer's reference grid equals the reference's after
    every 10^4 moves (and positions are bitwise equal)."""
    sim, o = sim_pair(strategy, n0, 1.0)
    acc = 0
    for k in range(chunks):
        tr = sim.run(10000, trace=True)
        _, tp = o.run(10000, trace=True)
        assert_trace_parity(tr, tp)
        acc += int(tr["accepted"].sum())
        assert np.array_equal(sim.particles(), o.positions()), f"positions after chunk {k}"
        assert_same_grid(sim, o, f"after chunk {k}")
    assert acc > 100  # the committer really ran
    assert sim.dev.rebuild_check() is None
    assert sim.peak_cell_occupancy() == o.state().peak_occupancy


def test_engine_grid_byte_identical_mu_minus2_2k():
    """mu = -2 at 2k: one accept per ~9 moves, mostly deletions and insertions
    (relabel chains in the committer)."""
    for strategy in ("microcell", "cell_list"):
        sim, o = sim_pair(strategy, 2048, -2.0)
        for k in range(5):
            tr = sim.run(20000, trace=True)
            _, tp = o.run(20000, trace=True)
            assert_trace_parity(tr, tp)
            assert_same_grid(sim, o, f"{strategy} chunk {k}")


# ------------------------------------------------------------ the bench regime
def warmed_pair(n0, warm, strategy="microcell", mu=1.0):
    """A device chain warmed for `warm` moves and the reference resumed from
    its exact state (positions, RNG, step, U, W)."""
    box, xyz, rng = config(n0)
    cfg = RC()(temperature=2.0, chemical_potential=mu, box_length=box, strategy=strategy)
    sim = E().Simulation(cfg, xyz, rng)
    sim.run(warm)
    return sim, resume_ref(sim, box, strategy, mu)


def resume_ref(sim, box, strategy, mu):
    st = sim.dev.get_state()
    xyz = sim.particles()
    if use_ref():
        cfg = O.ref_config(box_length=box, strategy=strategy, temperature=2.0,
                           chemical_potential=mu)
        return O.RefSim(cfg, mode=2, xyz=xyz, rng_hex=sim.rng().serialize_hex(), step=st.step,
                        energy=st.energy, virial=st.virial)
    p = O.port_params(box_length=box, strategy=strategy, temperature=2.0, chemical_potential=mu)
    from test_gpu_parity import _PortAdapter

    return _PortAdapter(O.PortSim(p, xyz, O.rng_from_hex(sim.rng().serialize_hex()), step=st.step,
                                  energy=st.energy, virial=st.virial))


def assert_full_state(sim, o, st0, rs0=None):
    """Positions and RNG bitwise; counters exact; energies within 1e-10."""
    assert np.array_equal(sim.particles(), o.positions())
    assert sim.rng().serialize_hex() == o.rng_hex()
    st, rs = sim.dev.get_state(), o.state()
    assert st.step == rs.step and st.n == rs.n
    for k in range(3):
        assert st.attempted[k] - st0.attempted[k] == rs.attempted[k] - (rs0.attempted[k] if rs0 else 0)
        assert st.accepted[k] - st0.accepted[k] == rs.accepted[k] - (rs0.accepted[k] if rs0 else 0)
    assert st.samples - st0.samples == rs.samples - (rs0.samples if rs0 else 0)
    assert st.sum_n - st0.sum_n == rs.sum_n - (rs0.sum_n if rs0 else 0)
    assert abs(st.energy - rs.energy) <= TOL * max(1.0, abs(rs.energy))
    assert abs(st.virial - rs.virial) <= TOL * max(1.0, abs(rs.virial))


def bench_regime(n0, warm, traced, after_rebuild):
    sim, o = warmed_pair(n0, warm)
    st0 = sim.dev.get_state()
    tr = sim.run(traced, trace=True)
    _, tp = o.run(traced, trace=True)
    assert_trace_parity(tr, tp)
    acc = tr["accepted"].mean()
    assert_full_state(sim, o, st0)
    # Grids: the reference's resume ctor bins the store into a fresh grid
    # (ascending ids, unused slots -1); re-uploading the store is the same
    # "new strategy over this store" on the device (checkpoint / resume).
    sim.dev.upload(sim.particles())
    box = sim.cfg.box_length
    o2 = resume_ref(sim, box, "microcell", 1.0)
    assert_same_grid(sim, o2, "after rebuild")
    st1 = sim.dev.get_state()
    tr = sim.run(after_rebuild, trace=True)
    _, tp = o2.run(after_rebuild, trace=True)
    assert_trace_parity(tr, tp)
    assert_full_state(sim, o2, st1)
    assert_same_grid(sim, o2, f"after {after_rebuild} moves")
    return acc


def test_bench_regime_1m():
    """BASELINE configs[3] in the window bench.py times: 2^24 warm-up moves,
    then 2x10^5 traced moves (and 10^5 more after a rebuild, grid compared)."""
    acc = bench_regime(1 << 20, 1 << 24, 200000, 100000)
    assert acc < 0.06  # the equilibrated regime, not the random start (~18 %)


def test_256k_liquid_trace():
    """BASELINE configs[2]: 256k at liquid density, mixed moves."""
    bench_regime(1 << 18, 1 << 22, 100000, 50000)


# ------------------------------------------------------------ other cutoffs
CUT_BOX = 13.23  # T/acceptance.cpp:114-128: 0.23 sigma boundary microcell


@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
@pytest.mark.parametrize("rc", [2.75, 3.0, 3.75, 4.25])
def test_other_cutoffs(strategy, rc):
    """validate.hpp:164-172 (the C5 coverage check): n = max(64, 0.4 V) at
    L = 13.23, seed 17. At r_c >= 3.75 the cell list has 3^3 cells of 4.41
    sigma side (~34 particles each at rho = 0.4, default capacity 48), so the
    chains run it with cell_capacity = 96 on both sides (config.hpp:60)."""
    n0 = max(64, int(0.4 * CUT_BOX ** 3))
    cap = 96 if strategy == "cell_list" else 0
    xyz, rng = E().random_initial_configuration(n0, CUT_BOX, 0.85, 17)
    g = E().GpuNeighborStrategy(strategy, xyz, CUT_BOX, r_cut=rc, capacity=cap)
    o = O.RefStrategy(strategy, xyz, CUT_BOX, rc=rc, capacity=cap) if use_ref() else \
        O.PortGrid(strategy, xyz, CUT_BOX, rc=rc, capacity=cap)
    occ, slots = g.grid()
    roc, rsl = o.grid()
    assert np.array_equal(occ, roc) and np.array_equal(slots, rsl)
    kinds, pids, pts = proposals(n0, CUT_BOX, 600, 23)
    du, dw = g.delta_batch(kinds, pids, pts)
    ref = oracle_deltas(o, kinds, pids, pts)
    assert rel(du, ref[:, 0]).max() <= TOL
    assert rel(dw, ref[:, 1]).max() <= TOL
    # 10^4-move trace through the engine
    kw = {"cell_capacity": cap} if cap else {}
    cfg = RC()(temperature=2.0, chemical_potential=-1.0, box_length=CUT_BOX, strategy=strategy,
               r_cut=rc, seed=17, **kw)
    sim = E().Simulation(cfg, xyz, rng)
    st = sim.dev.get_state()
    os_ = oracle_sim(strategy, CUT_BOX, xyz, rng.serialize_hex(), st.energy, st.virial,
                     temperature=2.0, chemical_potential=-1.0, r_cut=rc, **kw)
    tr = sim.run(10000, trace=True)
    _, tp = os_.run(10000, trace=True)
    assert_trace_parity(tr, tp)
    assert tr["accepted"].sum() > 200
    assert np.array_equal(sim.particles(), os_.positions())
    assert_same_grid(sim, os_, f"rc={rc}")


# ------------------------------------------------------------ overlap clamp
@pytest.mark.parametrize("strategy", ["microcell", "cell_list", "all_pairs"])
def test_overlap_clamp_on_device(strategy):
    """lj_pair_clamped: r^2 < 1e-12 sigma^2 -> (1e30, 1e30) (potential.hpp:51-54),
    through the device ΔE path, against the reference's strategy."""
    box = 12.0
    xyz, _ = E().random_initial_configuration(500, box, 0.85, 31)
    g = E().GpuNeighborStrategy(strategy, xyz, box)
    o = oracle_grid(strategy, xyz, box)
    p = xyz[7]
    pts = np.array([p, p + [1e-7, 0, 0], p + [0, 0, 5e-7], p + [1.1e-6, 0, 0]])
    for q in pts:
        a = g.delta_insert(q)
        b = o.delta_insert(q)
        assert abs(a.u - b[0]) <= TOL * max(1.0, abs(b[0])), (a.u, b[0])
        assert abs(a.w - b[1]) <= TOL * max(1.0, abs(b[1]))
    assert g.delta_insert(pts[1]).u >= 1e30
    # just above the floor: the unclamped LJ term (~1e72 here), not the clamp value
    big = g.delta_insert(pts[3]).u
    assert math.isfinite(big) and big != 1e30 and big > 1e60
    # a displacement onto another particle
    a = g.delta_displace(3, pts[2])
    b = o.delta_displace(3, pts[2])
    assert a.u >= 1e30 and abs(a.u - b[0]) <= TOL * abs(b[0])


# ------------------------------------------------------------ fault injection
@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
def test_audit_detects_store_edit(strategy):
    """T/test_engine.cpp:186-192: a particle moved behind the engine's back
    fails the audit (energy drift and a stale grid slot), with the same
    rebuild_check message as the reference; run_to raises AuditFailure."""
    box, xyz, rng = config(2000, seed=7, density=0.6)
    cfg = RC()(temperature=2.0, chemical_potential=-2.5, box_length=box, strategy=strategy,
               seed=7, checkpoint_interval=1 << 62)
    sim = E().Simulation(cfg, xyz, rng)
    assert sim.audit().passed()
    sim.run(5000)
    mid = sim.audit()
    assert mid.passed(), mid.describe()
    st = sim.dev.get_state()
    ref = None
    if use_ref():
        rc = O.ref_config(box_length=box, strategy=strategy, temperature=2.0,
                          chemical_potential=-2.5)
        ref = O.RefSim(rc, mode=2, xyz=sim.particles(), rng_hex=sim.rng().serialize_hex(),
                       step=st.step, energy=st.energy, virial=st.virial)
    p = sim.particles()[0]
    q = np.array([math.fmod(p[0] + 3.1, box), math.fmod(p[1] + 2.2, box), p[2]])
    sim.dev.store_set(0, q)
    bad = sim.audit()
    assert not bad.passed()
    assert not bad.energy_ok()
    assert bad.grid_issue is not None
    if ref is not None:
        ref.store_set(0, q)
        _, _, ok, text = ref.audit()
        assert not ok
        assert "grid: " + bad.grid_issue in text, (bad.grid_issue, text)
    with pytest.raises(E().AuditFailure):
        sim.run_to(sim.current_step() + 1)


def test_rebuild_check_detects_mirror_and_slot_corruption():
    """rebuild_check is not only ever clean: a store edit inside the same
    reference cell leaves the reference grid consistent but the coordinate
    mirror stale, and that is reported too."""
    box = 12.0
    xyz, _ = E().random_initial_configuration(400, box, 0.85, 5)
    g = E().GpuNeighborStrategy("microcell", xyz, box)
    assert g.rebuild_check() is None
    p = xyz[11]
    q = np.floor(p) + 0.5  # same microcell
    g.store_set(11, q)
    msg = g.rebuild_check()
    assert msg is not None and "mirror" in msg
    g.build()  # a fresh binning of the edited store is consistent again
    assert g.rebuild_check() is None


@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
def test_build_on_a_live_strategy_keeps_stale_slots_like_the_reference(strategy):
    """build() resets only the occupancy (microcell_grid.hpp:194-198,
    cell_grid.hpp:88-92): slots past a cell's new occupancy keep their old
    ids, byte for byte as in the reference."""
    box, xyz, _ = config(2048, seed=4)
    g = E().GpuNeighborStrategy(strategy, xyz, box)
    o = O.RefStrategy(strategy, xyz, box)
    rs = np.random.default_rng(3)
    n = len(xyz)
    for _ in range(300):
        if rs.random() < 0.5 and n > 10:
            pid = int(rs.integers(0, n))
            g.commit_delete(pid)
            o.commit_delete(pid)
            n -= 1
        else:
            p = rs.random(3) * box
            assert g.commit_insert(p) == o.commit_insert(p)
            n += 1
    g.build()
    O.ref_lib().ref_strat_build(o.h)
    a, b = g.grid(), o.grid()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_pair_evaluations_are_counted():
    """gcmc_run_result.pair_evals: the device's own count of FP64 pair
    evaluations: one pruned brick window per evaluated non-deletion slot plus
    the neighbour updates of accepted moves; all-pairs scans N per window."""
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(32768)
    sim = E().Simulation(RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box,
                                   strategy="microcell"), xyz, rng)
    sim.run(20000)
    r = sim.last_run
    # every evaluated slot counts, consumed or discarded by its round (from
    # the random start most rounds end early: ~1.1e3 per consumed move; in the
    # bench regime ~140)
    per_move = r.pair_evals / r.moves
    assert 50 < per_move < 5000, per_move
    sim.close()
    sim = E().Simulation(RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box,
                                   strategy="all_pairs"), xyz, rng)
    sim.run(2000)
    assert sim.last_run.pair_evals >= 2000 * 0.6 * len(xyz) * 0.9
    sim.close()


def test_all_pairs_on_the_maintained_energy_engine_32k():
    """BASELINE configs[1]'s all-pairs arm: the all-pairs strategy on the
    maintained-energy engine (S(n) by a scan of the whole store, in-flight
    moves corrected) is trace-identical to the reference's AllPairsStrategy
    (strategy.hpp:64-116) and to the per-window engine (engine_mode = 1)."""
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(32768)
    cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="all_pairs")
    sim = E().Simulation(cfg, xyz, rng)
    st0 = sim.dev.get_state()
    o = oracle_sim("all_pairs", box, xyz, rng.serialize_hex(), st0.energy, st0.virial,
                   temperature=2.0, chemical_potential=1.0)
    tr = sim.run(20000, trace=True)
    _, tp = o.run(20000, trace=True)
    assert_trace_parity(tr, tp)
    assert_full_state(sim, o, st0)
    assert sim.last_run.pair_evals > 20000 * 0.5 * len(xyz)  # whole-store scans
    old = E().Simulation(cfg, xyz, rng, engine_mode=1)
    to = old.run(20000, trace=True)
    assert np.array_equal(to["accepted"], tr["accepted"])
    assert np.array_equal(old.particles(), sim.particles())
    sim.close()
    old.close()
