"""Reference-format checkpoints and stats rows (checkpoint.hpp:16-132,
driver.hpp:15-34): a GPU run writes text the reference's read_checkpoint()
restores bit-for-bit, and vice versa."""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .config import RunConfig, format_g17, parse_config_text

MAGIC = "gcmc-checkpoint 1"
STATS_HEADER = "step,N,U,P,acc_disp,acc_ins,acc_del"


@dataclass
class Checkpoint:
    config: RunConfig
    step: int
    energy: float
    virial: float
    rng_state_hex: str
    positions: np.ndarray

    def restore(self, **kw):
        from .engine import RngState, Simulation

        return Simulation(self.config, self.positions, RngState.deserialize_hex(self.rng_state_hex),
                          self.step, self.energy, self.virial, **kw)


def snapshot(sim) -> Checkpoint:
    s = sim.dev.get_state()
    return Checkpoint(sim.cfg, s.step, s.energy, s.virial, sim.rng().serialize_hex(),
                      sim.particles())


def to_text(c: Checkpoint) -> str:
    lines = [MAGIC, c.config.serialize().rstrip("\n"), f"step={c.step}",
             f"count={len(c.positions)}", f"energy={format_g17(c.energy)}",
             f"virial={format_g17(c.virial)}", f"rng={c.rng_state_hex}", "positions"]
    body = "\n".join(f"{format_g17(x)} {format_g17(y)} {format_g17(z)}" for x, y, z in c.positions)
    return "\n".join(lines) + "\n" + (body + "\n" if len(c.positions) else "")


def checkpoint_from_text(text: str) -> Checkpoint:
    it = iter(text.split("\n"))
    if next(it, "").strip(" \t\r") != MAGIC:
        raise ValueError("checkpoint: bad or missing format line")
    cfg_lines, hdr = [], {}
    for line in it:
        l = line.strip(" \t\r")
        if l == "positions":
            break
        if "=" not in l:
            raise ValueError(f"checkpoint: expected key=value, got '{l}'")
        k, v = l.split("=", 1)
        if k in ("step", "count", "energy", "virial", "rng"):
            hdr[k] = v
        else:
            cfg_lines.append(l)
    if set(hdr) != {"step", "count", "energy", "virial", "rng"}:
        raise ValueError("checkpoint: incomplete header")
    cfg = parse_config_text("\n".join(cfg_lines) + "\n")
    count = int(hdr["count"])
    pos = np.zeros((count, 3))
    for i in range(count):
        line = next(it, None)
        if line is None:
            raise ValueError("checkpoint: truncated positions block")
        parts = line.split()
        if len(parts) < 3:
            raise ValueError(f"checkpoint: malformed position line {i}")
        pos[i] = [float(parts[0]), float(parts[1]), float(parts[2])]
    return Checkpoint(cfg, int(hdr["step"]), float(hdr["energy"]), float(hdr["virial"]),
                      hdr["rng"], pos)


def write_checkpoint(path: str, c: Checkpoint) -> None:
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(to_text(c).encode())
    os.replace(tmp, path)


def read_checkpoint(path: str) -> Checkpoint:
    with open(path, "rb") as f:
        return checkpoint_from_text(f.read().decode())


def stats_csv_row(sim) -> str:
    s = sim.state()
    return ",".join([str(sim.current_step()), str(sim.particle_count()),
                     format_g17(sim.reported_energy()), format_g17(sim.pressure()),
                     format_g17(s.acceptance_ratio(0)), format_g17(s.acceptance_ratio(1)),
                     format_g17(s.acceptance_ratio(2))])
