"""RunConfig and its key=value text format — the reference's config API
(proj/include/gcmc/config.hpp:16-219), kept so a reference config file or
checkpoint header drives this engine unchanged."""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

STRATEGIES = ("all_pairs", "cell_list", "microcell")  # config.hpp:16


def format_g17(v: float) -> str:
    """std::to_chars(general, 17) (text.hpp:14-18)."""
    return "%.17g" % v


def _parse_double(text: str) -> float:
    try:
        if text.strip() != text or text.startswith("+"):
            raise ValueError
        return float(text)
    except ValueError:
        raise ValueError(f"bad floating-point value: '{text}'") from None


def _parse_u64(text: str) -> int:
    """text.hpp:28-34: std::from_chars over the whole text — ASCII digits only,
    no sign, no overflow past 2^64 - 1."""
    if not text or any(c not in "0123456789" for c in text) or int(text) >= 1 << 64:
        raise ValueError(f"bad integer value: '{text}'")
    return int(text)


@dataclass
class RunConfig:
    """gcmc::RunConfig (config.hpp:42-64), same fields and defaults."""

    temperature: float = 0.0
    chemical_potential: float = 0.0
    lambda_: float = 1.0
    epsilon: float = 1.0
    sigma: float = 1.0
    r_cut: float = 2.5
    box_length: float = 0.0
    initial_particles: int = 0
    density: float = 0.6
    displace_percent: float = 0.30
    steps: int = 0
    seed: int = 1
    checkpoint_interval: int = 10000
    strategy: str = "all_pairs"
    tail_corrections: bool = False
    cell_capacity: int = 0
    microcell_capacity: int = 5
    equilibration_steps: int = 0
    sampling_interval: int = 1
    max_displacement: float = 0.0

    def beta(self) -> float:
        return 1.0 / self.temperature

    def volume(self) -> float:
        return self.box_length * self.box_length * self.box_length

    def copy(self, **kw) -> "RunConfig":
        return dataclasses.replace(self, **kw)

    def validate(self) -> None:
        """config.hpp:69-87 (same messages)."""
        def fail(why: str):
            raise ValueError("config: " + why)
        if not self.temperature > 0.0:
            fail("temperature must be > 0")
        if not self.lambda_ > 0.0:
            fail("lambda must be > 0")
        if not self.sigma > 0.0:
            fail("sigma must be > 0")
        if self.epsilon < 0.0:
            fail("epsilon must be >= 0")
        if not self.r_cut > 0.0:
            fail("r_cut must be > 0")
        if not self.box_length > 0.0:
            fail("box length must be > 0")
        if self.r_cut > self.box_length / 2.0:
            fail("r_cut must be <= box_length/2 for the minimum image convention (r_cut="
                 f"{format_g17(self.r_cut)}, L={format_g17(self.box_length)})")
        if self.displace_percent < 0.0 or self.displace_percent > 1.0:
            fail("displace_percent must lie in [0, 1]")
        if self.checkpoint_interval == 0:
            fail("checkpoint_interval must be >= 1")
        if self.sampling_interval == 0:
            fail("sampling_interval must be >= 1")
        if self.cell_capacity < 0:
            fail("cell_capacity must be >= 1 (or 0 for automatic)")
        if self.microcell_capacity < 1:
            fail("microcell_capacity must be >= 1")
        if self.max_displacement < 0.0:
            fail("max_displacement must be >= 0")
        if self.strategy not in STRATEGIES:
            fail(f"unknown strategy '{self.strategy}'")

    def serialize(self) -> str:
        """config.hpp:90-111, byte-identical."""
        return (
            f"temperature={format_g17(self.temperature)}\n"
            f"chemical_potential={format_g17(self.chemical_potential)}\n"
            f"lambda={format_g17(self.lambda_)}\n"
            f"epsilon={format_g17(self.epsilon)}\n"
            f"sigma={format_g17(self.sigma)}\n"
            f"r_cut={format_g17(self.r_cut)}\n"
            f"box_length={format_g17(self.box_length)}\n"
            f"displace_percent={format_g17(self.displace_percent)}\n"
            f"steps={self.steps}\n"
            f"seed={self.seed}\n"
            f"checkpoint_interval={self.checkpoint_interval}\n"
            f"strategy={self.strategy}\n"
            f"tail_corrections={'on' if self.tail_corrections else 'off'}\n"
            f"cell_capacity={self.cell_capacity}\n"
            f"microcell_capacity={self.microcell_capacity}\n"
            f"equilibration_steps={self.equilibration_steps}\n"
            f"sampling_interval={self.sampling_interval}\n"
            f"max_displacement={format_g17(self.max_displacement)}\n"
        )


_KNOWN = ("temperature", "chemical_potential", "lambda", "epsilon", "sigma", "r_cut",
          "box_length", "particles", "density", "displace_percent", "steps", "seed",
          "checkpoint_interval", "strategy", "tail_corrections", "cell_capacity",
          "microcell_capacity", "equilibration_steps", "sampling_interval", "max_displacement")


def _on_off(v: str) -> bool:
    if v in ("on", "true", "1"):
        return True
    if v in ("off", "false", "0"):
        return False
    raise ValueError(f"expected on/off, got '{v}'")


def _trim(s: str) -> str:
    return s.strip(" \t\r")


def parse_config_text(text: str) -> RunConfig:
    """config.hpp:128-211: key=value lines, '#' comments; unknown and
    duplicate keys are errors; exactly one of box_length / particles."""
    entries: dict[str, str] = {}
    for lineno, raw in enumerate(text.split("\n"), 1):
        line = raw.split("#", 1)[0]
        line = _trim(line)
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"config line {lineno}: expected key=value, got '{line}'")
        key, value = line.split("=", 1)
        key, value = _trim(key), _trim(value)
        if not key or not value:
            raise ValueError(f"config line {lineno}: empty key or value")
        if key in entries:
            raise ValueError(f"config line {lineno}: duplicate key '{key}'")
        entries[key] = value
    for key in sorted(entries):
        if key not in _KNOWN:
            raise ValueError(f"config: unknown key '{key}'")
    cfg = RunConfig()
    if "temperature" not in entries:
        raise ValueError("config: temperature is required")
    cfg.temperature = _parse_double(entries["temperature"])
    if "chemical_potential" not in entries:
        raise ValueError("config: chemical_potential is required")
    cfg.chemical_potential = _parse_double(entries["chemical_potential"])
    for key, attr in (("lambda", "lambda_"), ("epsilon", "epsilon"), ("sigma", "sigma"),
                      ("r_cut", "r_cut"), ("displace_percent", "displace_percent"),
                      ("max_displacement", "max_displacement")):
        if key in entries:
            setattr(cfg, attr, _parse_double(entries[key]))
    for key in ("steps", "seed", "checkpoint_interval", "cell_capacity", "microcell_capacity",
                "equilibration_steps", "sampling_interval"):
        if key in entries:
            setattr(cfg, key, _parse_u64(entries[key]))
    if "strategy" in entries:
        s = entries["strategy"]
        if s not in STRATEGIES:
            raise ValueError(f"unknown strategy '{s}' (expected all_pairs, cell_list or microcell)")
        cfg.strategy = s
    if "tail_corrections" in entries:
        cfg.tail_corrections = _on_off(entries["tail_corrections"])
    box, particles, density = (entries.get("box_length"), entries.get("particles"),
                               entries.get("density"))
    if box and particles:
        raise ValueError("config: give either box_length or particles, not both")
    if not box and not particles:
        raise ValueError("config: one of box_length / particles is required")
    if box:
        if density:
            raise ValueError("config: density only applies with particles")
        cfg.box_length = _parse_double(box)
        cfg.initial_particles = 0
    else:
        cfg.initial_particles = _parse_u64(particles)
        if density:
            cfg.density = _parse_double(density)
        if not cfg.density > 0.0:
            raise ValueError("config: density must be > 0")
        cfg.box_length = math.cbrt(cfg.initial_particles / cfg.density)
    cfg.validate()
    return cfg


def parse_config_file(path: str) -> RunConfig:
    try:
        with open(path, "rb") as f:
            return parse_config_text(f.read().decode())
    except OSError:
        raise ValueError(f"cannot open config file '{path}'") from None
