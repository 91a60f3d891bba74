"""run_with_files / stats.csv / checkpoints on the device against the
reference's own driver (driver.hpp:15-116, checkpoint.hpp:45-132).

Integer columns (step, N), acceptance ratios, RNG state, the config block and
the positions block of every checkpoint are compared byte for byte; U and P
(running sums of ΔU whose last bits depend on summation order) within 1e-10
relative. On an identical state the stats row is byte-identical."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import TOL, use_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not use_ref(), reason="needs the compiled reference (oracle/_ref)")]

CFG_TEXT = """# 1500 particles at rho 0.5 (the reference's particles/density form)
temperature=2.0
chemical_potential=-1.0
particles=1500
density=0.5
steps=30000
checkpoint_interval=10000
strategy=microcell
seed=3
"""


def D():
    from paper_1408_3764_b200 import checkpoint, config, driver, engine

    return checkpoint, config, driver, engine


def close(a: str, b: str) -> bool:
    x, y = float(a), float(b)
    return abs(x - y) <= TOL * max(1.0, abs(y))


def compare_rows(ours: str, ref: str):
    a, b = ours.split(","), ref.split(",")
    assert len(a) == len(b) == 7
    assert a[0] == b[0] and a[1] == b[1], (ours, ref)  # step, N
    assert close(a[2], b[2]) and close(a[3], b[3]), (ours, ref)  # U, P
    assert a[4:] == b[4:], (ours, ref)  # acceptance ratios of identical counts


def compare_checkpoints(pa: str, pb: str):
    ta, tb = open(pa).read(), open(pb).read()
    ha, pos_a = ta.split("positions\n")
    hb, pos_b = tb.split("positions\n")
    assert pos_a == pos_b, "positions block differs"
    la, lb = ha.splitlines(), hb.splitlines()
    assert len(la) == len(lb)
    for x, y in zip(la, lb):
        if x.startswith(("energy=", "virial=")):
            assert x.split("=")[0] == y.split("=")[0] and close(x.split("=")[1], y.split("=")[1])
        else:
            assert x == y, (x, y)


def test_stats_row_byte_identical_on_the_same_state():
    ck, cf, _, E = D()
    cfg = cf.parse_config_text(CFG_TEXT)
    sim = E.Simulation(cfg)
    sim.run(12345)
    text = ck.to_text(ck.snapshot(sim))
    ref = O.RefSim.from_checkpoint(text)
    ours = ck.checkpoint_from_text(text).restore()  # the same resume on the device
    assert ck.stats_csv_row(ours) == ref.stats_row()
    assert ck.to_text(ck.snapshot(ours)) == ref.checkpoint_text()
    ours.run(20000)
    ref.run(20000)
    compare_rows(ck.stats_csv_row(ours), ref.stats_row())
    # ... and once more from an identical state after the run
    text2 = ref.checkpoint_text()
    again = ck.checkpoint_from_text(text2).restore()
    ref2 = O.RefSim.from_checkpoint(text2)
    assert ck.stats_csv_row(again) == ref2.stats_row()


def test_run_with_files_matches_reference(tmp_path):
    _, cf, dr, _ = D()
    ref_dir, our_dir = str(tmp_path / "ref"), str(tmp_path / "ours")
    assert O.ref_run_with_files(CFG_TEXT, ref_dir) == 30000
    res = dr.run_with_files(cf.parse_config_text(CFG_TEXT), our_dir)
    assert res.final_step == 30000
    assert sorted(os.listdir(ref_dir)) == sorted(os.listdir(our_dir))
    assert os.path.basename(res.final_checkpoint_path) == "checkpoint_30000.txt"
    ra = open(os.path.join(ref_dir, "stats.csv")).read().splitlines()
    oa = open(os.path.join(our_dir, "stats.csv")).read().splitlines()
    assert ra[0] == oa[0] == "step,N,U,P,acc_disp,acc_ins,acc_del"
    assert len(ra) == len(oa) == 5  # start row + 3 checkpoints
    for x, y in zip(oa[1:], ra[1:]):
        compare_rows(x, y)
    for step in (10000, 20000, 30000):
        compare_checkpoints(os.path.join(our_dir, f"checkpoint_{step}.txt"),
                            os.path.join(ref_dir, f"checkpoint_{step}.txt"))


def test_run_with_files_resume_is_seamless(tmp_path):
    """driver.hpp:42-46: a resumed run continues the uninterrupted trajectory;
    a device checkpoint resumes on the reference and vice versa."""
    _, cf, dr, _ = D()
    cfg20 = cf.parse_config_text(CFG_TEXT.replace("steps=30000", "steps=20000"))
    cfg30 = cf.parse_config_text(CFG_TEXT)
    a, b, c = (str(tmp_path / k) for k in "abc")
    dr.run_with_files(cfg20, a)
    res = dr.run_with_files(cfg30, b, resume=os.path.join(a, "checkpoint_20000.txt"))
    assert res.final_step == 30000
    # the reference resumes from the device's checkpoint to the same end state
    O.ref_run_with_files(CFG_TEXT, c, os.path.join(a, "checkpoint_20000.txt"))
    compare_checkpoints(os.path.join(b, "checkpoint_30000.txt"),
                        os.path.join(c, "checkpoint_30000.txt"))
    # uninterrupted device run
    d = str(tmp_path / "d")
    dr.run_with_files(cfg30, d)
    pa = open(os.path.join(b, "checkpoint_30000.txt")).read().split("positions\n")[1]
    pd = open(os.path.join(d, "checkpoint_30000.txt")).read().split("positions\n")[1]
    assert pa == pd
    # zero-length resume: audit + the final checkpoint rewritten
    e = str(tmp_path / "e")
    res = dr.run_with_files(cfg30, e, resume=os.path.join(b, "checkpoint_30000.txt"))
    assert res.final_step == 30000 and os.path.exists(os.path.join(e, "checkpoint_30000.txt"))
    assert len(open(os.path.join(e, "stats.csv")).read().splitlines()) == 2


def test_resume_rejects_other_physics(tmp_path):
    _, cf, dr, _ = D()
    a = str(tmp_path / "a")
    dr.run_with_files(cf.parse_config_text(CFG_TEXT.replace("steps=30000", "steps=10000")), a)
    other = cf.parse_config_text(CFG_TEXT.replace("temperature=2.0", "temperature=1.5"))
    with pytest.raises(RuntimeError, match="resume: config does not match"):
        dr.run_with_files(other, str(tmp_path / "b"), resume=os.path.join(a, "checkpoint_10000.txt"))
    # steps / seed / interval / strategy may change on resume (driver.hpp:59-66)
    ok = cf.parse_config_text(CFG_TEXT.replace("strategy=microcell", "strategy=cell_list")
                              .replace("seed=3", "seed=9"))
    assert dr.run_with_files(ok, str(tmp_path / "c"),
                             resume=os.path.join(a, "checkpoint_10000.txt")).final_step == 30000
