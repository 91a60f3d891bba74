"""Pins the CPU restatement (oracle/gcmc_oracle.c) before it is trusted as
the parity checker: against the golden fixtures produced by the real
reference (tests/golden/make_golden.py), the reference tests' own
known-answer values (file:line cited per test), and the C++ standard's
mt19937_64 known-answer value. CPU only."""
from __future__ import annotations

import ctypes as C
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "golden.npz"))


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def test_mt19937_64_known_answer():
    # [rand.predef]: 10000th output of default-seeded mt19937_64.
    lib = O.port_lib()
    r = O.port_rng(5489)
    for _ in range(9999):
        lib.orc_rng_next(C.byref(r))
    assert lib.orc_rng_next(C.byref(r)) == 9981545732273789042


def test_uniforms_match_golden(gold):
    lib = O.port_lib()
    r = O.port_rng(1)
    got = np.array([lib.orc_uniform(C.byref(r)) for _ in range(16)])
    assert np.array_equal(got, gold["mt_seed1_first16"])
    # SURVEY §8c seed-1 values, printed by the reference.
    assert got[0] == 0.13387664401253263 and got[5] == 0.91135804791117681
    r = O.port_rng(42)
    for _ in range(1000):
        lib.orc_uniform(C.byref(r))
    got = np.array([lib.orc_uniform(C.byref(r)) for _ in range(16)])
    assert np.array_equal(got, gold["mt_seed42_skip1000_16"])


def test_index_from_kats():
    lib = O.port_lib()  # test_core.cpp:108-109
    assert lib.orc_index_from(0.9999999999999999, 3) == 2
    assert lib.orc_index_from(0.0, 3) == 0


def test_wrap_and_min_image_kats():
    lib = O.port_lib()  # test_core.cpp:19-35, 56-62
    out = np.empty(3)
    lib.orc_wrap_position(O.dptr(np.array([10.5, 0.2, -0.1])), 10.0, O.dptr(out))
    assert np.allclose(out, [0.5, 0.2, 9.9], rtol=1e-14)
    lib.orc_wrap_position(O.dptr(np.array([25.0, 25.0, 25.0])), 10.0, O.dptr(out))
    assert list(out) == [5.0, 5.0, 5.0]
    assert lib.orc_wrap_position(O.dptr(np.array([math.inf, 0, 0])), 10.0, O.dptr(out)) == -1
    d = lib.orc_min_image_dist2(O.dptr(np.array([0.1, 0, 0])), O.dptr(np.array([9.9, 0, 0])), 10.0)
    assert abs(d - 0.04) <= 1e-12 * 0.04
    assert lib.orc_min_image_dist2(O.dptr(np.array([1.0, 2, 3])), O.dptr(np.array([4.0, 6, 3])),
                                   100.0) == 25.0


def test_grid_geometry_kats():
    lib = O.port_lib()
    d, s = C.c_int32(), C.c_double()
    for l, want in ((23.9, 9), (7.0, 3), (10.0, 4)):  # test_grids.cpp:15-27
        lib.orc_compute_cell_dims(l, 2.5, C.byref(d), C.byref(s))
        assert d.value == want
    lib.orc_microcell_dims(50.23, 1.0, C.byref(d), C.byref(s))  # test_grids.cpp:35-43
    assert d.value == 51 and abs(s.value - 0.23) < 1e-9
    lib.orc_microcell_dims(10.0, 1.0, C.byref(d), C.byref(s))
    assert d.value == 10 and s.value == 1.0
    assert [lib.orc_microcell_extent(rc, 1.0) for rc in (2.5, 2.75, 4.25)] == [3, 3, 5]
    lo, cnt = C.c_int32(), C.c_int32()
    # test_grids.cpp:45-74
    for c, lw, want in ((7, 0.23, (-3, 7)), (12, 0.23, (-3, 8)), (0, 0.23, (-4, 8)),
                        (12, 0.6, (-3, 7)), (5, 1.0, (-3, 7))):
        lib.orc_microcell_axis_window(c, 2.5, 1.0, 14, lw, C.byref(lo), C.byref(cnt))
        assert (lo.value, cnt.value) == want
    # test_grids.cpp:76-103
    for x, rc, want in ((7.51, 2.5, (5, 6)), (7.2, 2.5, (4, 6)), (13.1, 2.5, (10, 7)),
                        (1.0, 2.5, (12, 7))):
        lib.orc_microcell_axis_arc(x, rc, 1.0, 14.23, 15, C.byref(lo), C.byref(cnt))
        assert (lo.value, cnt.value) == want
    lib.orc_microcell_axis_arc(3.0, 14.23 / 2, 1.0, 14.23, 15, C.byref(lo), C.byref(cnt))
    assert cnt.value == 15


def test_acceptance_kats():
    lib = O.port_lib()  # test_engine.cpp:11-34
    assert lib.orc_displacement_acceptance(-5.0, 1.0) == 1.0
    assert abs(lib.orc_displacement_acceptance(math.log(2.0), 1.0) - 0.5) <= 1e-15
    assert lib.orc_displacement_acceptance(1e30, 1.0) == 0.0
    assert lib.orc_insertion_acceptance(0.0, 99, 100.0, 1.0, 0.0, 1.0) == 1.0
    assert abs(lib.orc_insertion_acceptance(0.0, 199, 100.0, 1.0, 0.0, 1.0) - 0.5) <= 1e-15
    assert abs(lib.orc_deletion_acceptance(0.0, 50, 100.0, 1.0, 0.0, 1.0) - 0.5) <= 1e-15


def test_total_energy_kats():
    lib = O.port_lib()  # test_engine.cpp:55-84
    u, w = C.c_double(), C.c_double()
    rmin = 2.0 ** (1.0 / 6.0)
    pair = np.array([[1.0, 1.0, 1.0], [1.0 + rmin, 1.0, 1.0]])
    assert lib.orc_total_energy(O.dptr(pair), 2, 20.0, 1.0, 1.0, 2.5, C.byref(u), C.byref(w)) == 0
    assert abs(u.value + 1.0) < 1e-13 and abs(w.value) <= 1e-12
    ov = np.array([[1.0, 1, 1], [1.0, 1, 1]])
    assert lib.orc_total_energy(O.dptr(ov), 2, 20.0, 1.0, 1.0, 2.5, C.byref(u), C.byref(w)) == 4


def test_initial_configuration_matches_golden(gold, meta):
    box = meta["init_256_box"]
    r = O.port_rng(7)
    pos = np.empty((256, 3))
    assert O.port_lib().orc_random_initial_configuration(256, box, 0.85, C.byref(r),
                                                         O.dptr(pos)) == 0
    assert np.array_equal(pos, gold["init_256_xyz"])
    assert O.rng_to_hex(r) == meta["init_256_rng"]


def test_build_matches_golden_grids(gold, meta):
    box = meta["init_256_box"]
    occ, slots = O.PortGrid("microcell", gold["init_256_xyz"], box).grid()
    assert np.array_equal(occ, gold["grid_micro_occ"])
    assert np.array_equal(slots, gold["grid_micro_slots"])
    occ, slots = O.PortGrid("cell_list", gold["init_256_xyz"], box).grid()
    assert np.array_equal(occ, gold["grid_cell_occ"])
    assert np.array_equal(slots, gold["grid_cell_slots"])


@pytest.mark.parametrize("strat", ["all_pairs", "cell_list", "microcell"])
def test_deltas_match_golden_bitwise(gold, meta, strat):
    box = meta["init_256_box"]
    g = O.PortGrid(strat, gold["init_256_xyz"], box)
    for kind, pid, x, y, z, du, dw in gold[f"deltas_{strat}"]:
        pid = int(pid)
        if kind == 0:
            got = g.delta_displace(pid, [x, y, z])
        elif kind == 1:
            got = g.delta_insert([x, y, z])
        else:
            got = g.delta_delete(pid)
        assert got == (du, dw)


@pytest.mark.parametrize("strat", ["all_pairs", "cell_list", "microcell"])
@pytest.mark.parametrize("mu", ["m2", "p1"])
def test_trajectory_matches_golden_bitwise(gold, meta, strat, mu):
    box = meta["init_256_box"]
    xyz = gold["init_256_xyz"]
    key = f"{strat}_{mu}"
    e0, w0 = meta[f"initial_energy_{key}"]
    u, w = C.c_double(), C.c_double()
    O.port_lib().orc_total_energy(O.dptr(xyz), len(xyz), box, 1.0, 1.0, 2.5, C.byref(u),
                                  C.byref(w))
    assert (u.value, w.value) == (e0, w0)
    params = O.port_params(box_length=box, strategy=strat,
                           chemical_potential=-2.0 if mu == "m2" else 1.0, tail_corrections=1)
    sim = O.PortSim(params, xyz, O.rng_from_hex(meta["init_256_rng"]), energy=e0, virial=w0)
    tr = sim.run(2000, trace=True)
    assert np.array_equal(tr, gold[f"trace_{key}"])
    st = sim.state()
    final = gold[f"final_{key}"]
    assert [st.energy, st.virial, st.sum_u, st.sum_p, st.sum_n, st.sum_n2] == list(final[:6])
    pos, _, _ = sim.grid()
    assert np.array_equal(pos, gold[f"final_{key}_xyz"])
    assert O.rng_to_hex(sim.rng()) == meta[f"final_{key}_rng"]


@pytest.mark.skipif(not O.ref_available(), reason="reference not available")
def test_port_equals_reference_at_4096_mixed_state_points():
    """Larger cross-check against the live reference (not a fixture)."""
    n0 = 4096
    box = (n0 / 0.67) ** (1 / 3)
    xyz, hexs = O.ref_initial_configuration(n0, box, 3)
    for strat in ("microcell", "cell_list"):
        cfg = O.ref_config(temperature=2.0, chemical_potential=1.0, box_length=box,
                           strategy=strat, displace_percent=0.4, max_displacement=0.7)
        ref = O.RefSim(cfg, mode=2, xyz=xyz, rng_hex=hexs)
        _, tr = ref.run(5000, trace=True)
        port = O.PortSim(O.port_params(box_length=box, strategy=strat, chemical_potential=1.0,
                                       displace_percent=0.4, max_displacement=0.7),
                         xyz, O.rng_from_hex(hexs))
        tp = port.run(5000, trace=True)
        assert np.array_equal(tr, tp)
        assert O.rng_to_hex(port.rng()) == ref.rng_hex()
