"""Run driver with checkpoints and stats.csv — gcmc::run_with_files
(proj/include/gcmc/driver.hpp:15-116) over the device Simulation.

Same files, names and formats as the reference: ``stats.csv`` with the header
``step,N,U,P,acc_disp,acc_ins,acc_del`` and one row per checkpoint boundary
(plus the starting row), ``checkpoint_<step>.txt`` in the reference's text
format (checkpoint.hpp:45-58, written atomically via tmp + rename). The move
loop between boundaries is one device batch; every boundary runs the device
audit (full-system energy + rebuild_check, engine.hpp:333-342) and an
``AuditFailure`` propagates to the caller, as in the reference. A checkpoint
written here resumes the reference bit for bit, and vice versa.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, TextIO

from .checkpoint import STATS_HEADER, read_checkpoint, snapshot, stats_csv_row, write_checkpoint
from .config import RunConfig, format_g17
from .engine import AuditFailure, RngState, Simulation


@dataclass
class RunFilesResult:
    """driver.hpp:36-40."""
    final_step: int = 0
    stats_path: str = ""
    final_checkpoint_path: str = ""


def _physics_only(cfg: RunConfig) -> str:
    # driver.hpp:59-66: steps, seed, interval and strategy may differ on resume
    return cfg.copy(steps=0, seed=0, checkpoint_interval=0, strategy="all_pairs").serialize()


def run_with_files(cfg: RunConfig, out_dir: str, resume: Optional[str] = None,
                   log: Optional[TextIO] = None, device: int = 0, **engine_kw) -> RunFilesResult:
    """driver.hpp:47-116: runs to cfg.steps writing a checkpoint and a stats
    row at every checkpoint boundary; with ``resume``, continues from that
    checkpoint (the trajectory is identical to an uninterrupted run)."""
    os.makedirs(out_dir, exist_ok=True)
    if resume:
        c = read_checkpoint(resume)
        if _physics_only(c.config) != _physics_only(cfg):
            raise RuntimeError("resume: config does not match the checkpoint's parameters")
        sim = Simulation(cfg, c.positions, RngState.deserialize_hex(c.rng_state_hex), c.step,
                         c.energy, c.virial, device=device, **engine_kw)
    else:
        sim = Simulation(cfg, device=device, **engine_kw)
    try:
        result = RunFilesResult(stats_path=os.path.join(out_dir, "stats.csv"))

        def checkpoint_path(step: int) -> str:
            return os.path.join(out_dir, f"checkpoint_{step}.txt")

        with open(result.stats_path, "wb") as stats:
            stats.write((STATS_HEADER + "\n" + stats_csv_row(sim) + "\n").encode())
            initial_step = sim.current_step()

            def on_checkpoint(s, _report):
                write_checkpoint(checkpoint_path(s.current_step()), snapshot(s))
                stats.write((stats_csv_row(s) + "\n").encode())
                if log:
                    st = s.state()
                    log.write(f"step {s.current_step()}: N={s.particle_count()} "
                              f"U={format_g17(st.energy)}\n")

            sim.run_to(cfg.steps, on_checkpoint)
            # a zero-length run still leaves a restorable final state behind
            if sim.current_step() == initial_step:
                report = sim.audit()
                if not report.passed():
                    raise AuditFailure("final audit failed: " + report.describe())
                write_checkpoint(checkpoint_path(sim.current_step()), snapshot(sim))
        result.final_step = sim.current_step()
        result.final_checkpoint_path = checkpoint_path(result.final_step)
        if log:
            st, rs = sim.state(), sim.statistics()
            log.write(f"done: steps={sim.current_step()} N={sim.particle_count()} "
                      f"U={format_g17(st.energy)} P={format_g17(sim.pressure())}\n"
                      f"samples={rs.samples} <N>={format_g17(rs.mean_n())} "
                      f"<U>={format_g17(rs.mean_u())} <P>={format_g17(rs.mean_p())}\n"
                      f"acceptance: displace={format_g17(st.acceptance_ratio(0))} "
                      f"insert={format_g17(st.acceptance_ratio(1))} "
                      f"delete={format_g17(st.acceptance_ratio(2))}\n")
        return result
    finally:
        sim.close()
