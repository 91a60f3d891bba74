"""The chain-per-SM engine (engine_sm.cu, engine_mode = 2): one CTA runs a
whole chain, so K chains of a mu/T sweep each own an SM (SURVEY §8f rank 3,
PAPER.md:632). The chain must be the reference's, move for move: traces,
full state, the engine committer's reference grid (byte-identical), the
maintained per-particle energies, and the same trajectory as the multi-SM
engine (engine2.cu) from the same start."""
from __future__ import annotations

import numpy as np
import pytest

from test_gpu_parity import TOL, E, assert_trace_parity, config, oracle_sim, rel, use_ref
from test_gpu_engine_parity import assert_full_state, assert_same_grid, resume_ref

pytestmark = [pytest.mark.gpu]


def RC():
    from paper_1408_3764_b200.config import RunConfig

    return RunConfig


def sm_pair(strategy, n0, mu, seed=1, **kw):
    box, xyz, rng = config(n0, seed=seed)
    cfg = RC()(temperature=2.0, chemical_potential=mu, box_length=box, strategy=strategy,
               seed=seed, **kw)
    sim = E().Simulation(cfg, xyz, rng, engine_mode=2)
    st = sim.dev.get_state()
    o = oracle_sim(strategy, box, xyz, rng.serialize_hex(), st.energy, st.virial,
                   temperature=2.0, chemical_potential=mu, **kw)
    return sim, o, st


@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
@pytest.mark.parametrize("n0,mu,chunks", [(2048, 1.0, 5), (2048, -2.0, 5), (32768, 1.0, 4),
                                          (65536, -3.0, 4), (1 << 20, 1.0, 2)])
def test_sm_engine_trace_state_and_grid(strategy, n0, mu, chunks):
    """Trace parity, full state and the byte-identical reference grid after
    every chunk (2k dense / dilute, 32k, the 64k sweep's mu = -3, and 1M,
    where the mirror occupancies are read from global memory: no shared
    replica fits)."""
    sim, o, st0 = sm_pair(strategy, n0, mu)
    acc = 0
    for k in range(chunks):
        tr = sim.run(20000, trace=True)
        assert sim.last_run.engine == 3
        _, tp = o.run(20000, trace=True)
        assert_trace_parity(tr, tp)
        acc += int(tr["accepted"].sum())
        assert_full_state(sim, o, st0)
        if use_ref():
            assert_same_grid(sim, o, f"after chunk {k}")
    assert acc > 200
    assert sim.dev.rebuild_check() is None
    assert sim.peak_cell_occupancy() == o.state().peak_occupancy
    du, dw = sim.dev.energy_drift()
    assert du <= 1e-10 and dw <= 1e-9, (du, dw)
    # a speculative round really consumed several moves
    assert sim.last_run.moves / max(1, sim.last_run.rounds) > 4


@pytest.mark.parametrize("n0,mu", [(16384, -1.0), (65536, -3.0)])
def test_sm_engine_equals_multi_sm_engine(n0, mu):
    """Same start, same stream: the one-CTA engine and the whole-GPU engine
    follow the same trajectory (positions and RNG bitwise), and each keeps
    the other's maintained energies usable (switching mid-run)."""
    box, xyz, rng = config(n0, seed=3)
    cfg = RC()(temperature=2.0, chemical_potential=mu, box_length=box, seed=3, strategy="microcell")
    a = E().Simulation(cfg, xyz, rng)
    b = E().Simulation(cfg, xyz, rng, engine_mode=2)
    ta, tb = a.run(60000, trace=True), b.run(60000, trace=True)
    assert a.last_run.engine == 2 and b.last_run.engine == 3
    assert np.array_equal(ta["accepted"], tb["accepted"])
    assert np.array_equal(ta["n_after"], tb["n_after"])
    assert rel(ta["delta_u"], tb["delta_u"]).max() <= TOL
    assert np.array_equal(a.particles(), b.particles())
    assert a.rng().serialize_hex() == b.rng().serialize_hex()
    sa, sb = a.dev.get_state(), b.dev.get_state()
    assert (sa.n, sa.step, list(sa.accepted), sa.samples) == (sb.n, sb.step, list(sb.accepted), sb.samples)
    assert abs(sa.energy - sb.energy) <= TOL * max(1.0, abs(sa.energy))
    a.close()
    b.close()


def test_sm_engine_resumed_bench_regime_64k():
    """The sweep regime after a long warm-up on the whole-GPU engine: resume
    the reference there, continue on the one-CTA engine."""
    box, xyz, rng = config(65536)
    cfg = RC()(temperature=2.0, chemical_potential=-3.0, box_length=box, strategy="microcell")
    sim = E().Simulation(cfg, xyz, rng, engine_mode=2)
    sim.run(1 << 21)
    o = resume_ref(sim, box, "microcell", -3.0)
    st0 = sim.dev.get_state()
    tr = sim.run(200000, trace=True)
    _, tp = o.run(200000, trace=True)
    assert_trace_parity(tr, tp)
    assert_full_state(sim, o, st0)
    sim.close()


def test_sm_engine_chains_match_their_reference_chains():
    """Eight concurrent one-CTA chains (gcmc_run_chains), each the reference's."""
    k, n0 = 8, 8192
    sims, refs, st0 = [], [], []
    for c in range(k):
        box, xyz, rng = config(n0, seed=1 + c)
        mu = -3.0 + c
        cfg = RC()(temperature=2.0, chemical_potential=mu, box_length=box, seed=1 + c,
                   strategy="microcell")
        sim = E().Simulation(cfg, xyz, rng, engine_mode=2, engine_share=k)
        st = sim.dev.get_state()
        sims.append(sim)
        st0.append(st)
        refs.append(oracle_sim("microcell", box, xyz, rng.serialize_hex(), st.energy, st.virial,
                               temperature=2.0, chemical_potential=mu))
    moves = [20000 + 1000 * c for c in range(k)]
    for rep in range(2):
        res = E().run_chains(sims, moves)
        assert all(r.engine == 3 for r in res)
        for c in range(k):
            refs[c].run(moves[c])
            assert_full_state(sims[c], refs[c], st0[c])
    for s in sims:
        s.close()


def test_sm_engine_sampling_tail_and_equilibration():
    """Statistics in the decided rounds: sampling interval, equilibration
    cut-off and tail corrections, as the reference accumulates them."""
    sim, o, st0 = sm_pair("microcell", 2048, 1.0, tail_corrections=1, equilibration_steps=777,
                          sampling_interval=7)
    tr = sim.run(30000, trace=True)
    _, tp = o.run(30000, trace=True)
    assert_trace_parity(tr, tp)
    st, rs = sim.dev.get_state(), o.state()
    assert st.samples == rs.samples and st.sum_n == rs.sum_n and st.sum_n2 == rs.sum_n2
    assert abs(st.sum_u - rs.sum_u) <= 1e-9 * max(1.0, abs(rs.sum_u))
    assert abs(st.sum_p - rs.sum_p) <= 1e-9 * max(1.0, abs(rs.sum_p))


@pytest.mark.parametrize("engine_mode", [0, 2])
def test_engine_cell_overflow_like_the_reference(engine_mode):
    """An accepted insertion into a full reference cell (microcell capacity 2,
    mu = +4 at 400 particles) ends the run with the reference's error at the
    same move (cell_grid / microcell_grid insert_id: runtime_error), on both
    engines; everything before it is committed and identical."""
    from paper_1408_3764_b200 import _lib

    import oracle as O

    n0 = 400
    box = (n0 / 0.5) ** (1.0 / 3.0)
    xyz, rng = E().random_initial_configuration(n0, box, 0.85, 1)
    cfg = RC()(temperature=2.0, chemical_potential=4.0, box_length=box, strategy="microcell",
               microcell_capacity=2)
    sim = E().Simulation(cfg, xyz, rng, engine_mode=engine_mode)
    with pytest.raises(_lib.GcmcError) as ei:
        sim.run(20000)
    assert ei.value.status == "CELL_OVERFLOW"
    msg = str(ei.value)
    assert "microcell: cell" in msg and "exceeds capacity 2" in msg
    st = sim.dev.get_state()
    if use_ref():
        ref = O.RefSim(O.ref_config(box_length=box, strategy="microcell", temperature=2.0,
                                    chemical_potential=4.0, microcell_capacity=2),
                       mode=2, xyz=xyz, rng_hex=rng.serialize_hex(), step=0, energy=0.0, virial=0.0)
        with pytest.raises(O.RefError) as er:
            ref.run(20000)
        assert str(er.value).split("microcell: ")[-1] in msg
        assert st.step == ref.state().step
    sim.close()


@pytest.mark.parametrize("strategy", ["microcell", "cell_list"])
@pytest.mark.parametrize("engine_mode", [0, 2])
def test_sm_engine_filling_a_dilute_box(strategy, engine_mode):
    """mu = +6 from density 0.1: nearly every insertion is accepted, so rounds
    end at the N-offset range (d = +8) or at max_acc and almost every commit
    is an insertion (index chains, forwarded relabels when a deletion follows);
    the store starts at 4096 + 64 particles and grows with N (store
    reallocation between launches). Trace, state and grid bytes stay the
    reference's, on both maintained-energy engines."""
    box, xyz, rng = config(4096, seed=7, density=0.1)
    cfg = RC()(temperature=2.0, chemical_potential=6.0, box_length=box, strategy=strategy, seed=7)
    sim = E().Simulation(cfg, xyz, rng, engine_mode=engine_mode, max_particles=4096 + 64)
    st0 = sim.dev.get_state()
    o = oracle_sim(strategy, box, xyz, rng.serialize_hex(), st0.energy, st0.virial,
                   temperature=2.0, chemical_potential=6.0)
    for k in range(3):
        tr = sim.run(10000, trace=True)
        assert sim.last_run.engine == (3 if engine_mode == 2 else 2)
        _, tp = o.run(10000, trace=True)
        assert_trace_parity(tr, tp)
        assert_full_state(sim, o, st0)
        if use_ref():
            assert_same_grid(sim, o, f"chunk {k}")
    assert sim.particle_count() > 4096 * 2  # the box really filled
    du, dw = sim.dev.energy_drift()
    assert du <= 1e-9 and dw <= 1e-8, (du, dw)
    sim.close()


def _ideal_gas_pair(engine_mode, **kw):
    box, xyz, rng = config(2048)
    cfg = RC()(temperature=2.0, chemical_potential=3.0, box_length=box, strategy="cell_list",
               epsilon=0.0)
    sim = E().Simulation(cfg, xyz, rng, engine_mode=engine_mode, **kw)
    st = sim.dev.get_state()
    o = oracle_sim("cell_list", box, xyz, rng.serialize_hex(), st.energy, st.virial,
                   temperature=2.0, chemical_potential=3.0, epsilon=0.0)
    return sim, o, st


@pytest.mark.parametrize("engine_mode", [0, 2])
def test_mirror_growth_then_reference_overflow(engine_mode):
    """epsilon = 0 at mu = +3: an ideal gas that fills the box. The brick
    mirror (32 records per brick) overflows first — the engine doubles it and
    continues at that move, invisibly — then the reference's cell list (48)
    overflows: the same error at the same move (T/test_engine.cpp:143-158's
    epsilon = 0 case; cell_grid.hpp insert_id)."""
    from paper_1408_3764_b200 import _lib

    sim, o, st0 = _ideal_gas_pair(engine_mode)
    failed = False
    for k in range(20):
        try:
            tr = sim.run(1000, trace=True)
        except _lib.GcmcError as e:
            assert e.status == "CELL_OVERFLOW" and "exceeds capacity 48" in str(e)
            with pytest.raises(Exception) as er:
                o.run(1000, trace=True)
            assert "exceeds capacity 48" in str(er.value)
            assert sim.dev.get_state().step == o.state().step
            failed = True
            break
        _, tp = o.run(1000, trace=True)
        assert_trace_parity(tr, tp)
        assert_full_state(sim, o, st0)
        peak = sim.peak_cell_occupancy()
    assert failed
    # cells and bricks partition this box alike (5^3 of side L/5 >= r_c): a
    # cell past 32 means the mirror grew
    assert peak > 32, peak
    sim.close()


def test_mirror_growth_in_a_batched_launch():
    """The same ideal gas as two chain-per-SM chains in one launch: a chain
    whose mirror overflows mid-chunk finishes the chunk on its own launches
    (grown mirror); both stay the reference's chain up to the overflow."""
    from paper_1408_3764_b200 import _lib

    pairs = [_ideal_gas_pair(2, engine_share=2) for _ in range(2)]
    sims = [p[0] for p in pairs]
    for k in range(6):
        E().run_chains(sims, 1000)
        for sim, o, st0 in pairs:
            o.run(1000)
            assert_full_state(sim, o, st0)
    assert all(s.peak_cell_occupancy() > 32 for s in sims)  # past the mirror's 32 per brick
    with pytest.raises(_lib.GcmcError):
        E().run_chains(sims, 4000)
    for s in sims:
        s.close()


def test_batched_chains_of_different_shapes():
    """One launch over chains with different strategies, box sizes and state
    points (the shared-memory plan takes the largest replica): each chain is
    its own reference chain."""
    specs = [("microcell", 2048, -2.0, 11), ("cell_list", 32768, 1.0, 12), ("microcell", 65536, -3.0, 13)]
    sims, refs, st0 = [], [], []
    for strategy, n0, mu, seed in specs:
        box, xyz, rng = config(n0, seed=seed)
        cfg = RC()(temperature=2.0, chemical_potential=mu, box_length=box, strategy=strategy, seed=seed)
        sim = E().Simulation(cfg, xyz, rng, engine_mode=2)
        st = sim.dev.get_state()
        sims.append(sim)
        st0.append(st)
        refs.append(oracle_sim(strategy, box, xyz, rng.serialize_hex(), st.energy, st.virial,
                               temperature=2.0, chemical_potential=mu))
    for rep in range(2):
        res = E().run_chains(sims, [15000, 20000, 25000])
        assert all(r.engine == 3 for r in res)
        for c, (sim, o) in enumerate(zip(sims, refs)):
            o.run([15000, 20000, 25000][c])
            assert_full_state(sim, o, st0[c])
            if use_ref():
                assert_same_grid(sim, o, f"chain {c} rep {rep}")
    for s in sims:
        s.close()
