"""Many chains per GPU: K independent chains
advanced concurrently by gcmc_run_chains, each sharing the device
(engine_share = K), every one trace-identical to its own reference chain."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import E, assert_trace_parity, config, oracle_sim, use_ref
from test_gpu_engine_parity import assert_full_state, assert_same_grid

pytestmark = [pytest.mark.gpu]


def _chains(k, n0, mus, strategy="microcell"):
    from paper_1408_3764_b200.config import RunConfig

    sims, refs = [], []
    for c in range(k):
        box, xyz, rng = config(n0, seed=1 + c)
        cfg = RunConfig(temperature=2.0, chemical_potential=mus[c], box_length=box,
                        strategy=strategy, seed=1 + c)
        sim = E().Simulation(cfg, xyz, rng, engine_share=k)
        st = sim.dev.get_state()
        sims.append(sim)
        refs.append(oracle_sim(strategy, box, xyz, rng.serialize_hex(), st.energy, st.virial,
                               temperature=2.0, chemical_potential=mus[c]))
    return sims, refs


@pytest.mark.parametrize("k,n0", [(2, 32768), (4, 8192)])
def test_concurrent_chains_match_their_reference_chains(k, n0):
    mus = [-3.0 + c for c in range(k)]
    sims, refs = _chains(k, n0, mus)
    st0 = [s.dev.get_state() for s in sims]
    moves = [30000 + 1000 * c for c in range(k)]  # different lengths: chains finish apart
    for rep in range(3):
        E().run_chains(sims, moves)
        for c in range(k):
            refs[c].run(moves[c])
            assert_full_state(sims[c], refs[c], st0[c])
            if use_ref():
                assert_same_grid(sims[c], refs[c], f"chain {c} rep {rep}")
    for s in sims:
        assert s.last_run.moves == moves[sims.index(s)]
        s.close()


def test_chain_share_equals_solo_trace():
    """A chain in a shared device gives the same trace as the same chain alone
    on the whole device (round boundaries differ; the trajectory does not)."""
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(16384, seed=5)
    cfg = RunConfig(temperature=2.0, chemical_potential=-1.0, box_length=box, seed=5)
    solo = E().Simulation(cfg, xyz, rng)
    shared = E().Simulation(cfg, xyz, rng, engine_share=3)
    other = E().Simulation(cfg, xyz, rng, engine_share=3)
    t_solo = solo.run(40000, trace=True)
    E().run_chains([shared, other], [40000, 40000])
    assert np.array_equal(solo.particles(), shared.particles())
    assert np.array_equal(shared.particles(), other.particles())
    assert solo.rng().serialize_hex() == shared.rng().serialize_hex()
    a, b = solo.dev.get_state(), shared.dev.get_state()
    assert (a.n, a.step, list(a.accepted)) == (b.n, b.step, list(b.accepted))
    assert t_solo["accepted"].sum() == sum(b.accepted) - 0
    for s in (solo, shared, other):
        s.close()


def test_run_chains_rejects_duplicates():
    from paper_1408_3764_b200 import _lib as L
    from paper_1408_3764_b200.config import RunConfig

    box, xyz, rng = config(2048)
    sim = E().Simulation(RunConfig(temperature=2.0, box_length=box), xyz, rng)
    with pytest.raises(L.GcmcError, match="twice"):
        E().run_chains([sim, sim], 10)
    sim.close()
