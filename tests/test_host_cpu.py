"""Host-side mirror and C-ABI surface, CPU only (no device calls)."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_1408_3764_b200 import config as CFG

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "gcmc_b200.h")


def header_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(gcmc_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1408_3764_b200 import _lib

    lib = _lib.load()  # loads without a GPU (libcudart is linked, not initialised)
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.gcmc_version().decode().startswith("gcmc_b200")


def test_abi_struct_layouts_match_the_header(tmp_path):
    """ctypes mirrors of the C ABI structs (_lib.py) have the header's sizes
    and field offsets (compiled here with gcc against include/gcmc_b200.h)."""
    import shutil
    import subprocess

    from paper_1408_3764_b200 import _lib as L

    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    structs = {"gcmc_params": L.GcmcParams, "gcmc_state": L.GcmcState,
               "gcmc_run_result": L.GcmcRunResult}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "gcmc_b200.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f in cls._fields_:
            lines.append(f'  printf("{name} {f[0]} %zu\\n", offsetof({name}, {f[0].rstrip("_")}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for name, cls in structs.items():
        assert got[(name, "size")] == C.sizeof(cls), name
        for f in cls._fields_:
            assert got[(name, f[0])] == getattr(cls, f[0]).offset, (name, f[0])


def test_library_is_sm100a_cubin():
    so = os.path.join(ROOT, "paper_1408_3764_b200", "libgcmc_b200.so")
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_random_initial_configuration_matches_reference():
    from paper_1408_3764_b200 import engine as E

    for n, seed in ((300, 3), (2048, 1)):
        box = (n / 0.67) ** (1 / 3)
        xyz, rng = E.random_initial_configuration(n, box, 0.85, seed, device=None)  # host form
        if O.ref_available():
            rx, rh = O.ref_initial_configuration(n, box, seed)
            assert np.array_equal(xyz, rx)
            assert rng.serialize_hex() == rh
        # restatement (always available)
        r = O.port_rng(seed)
        pos = np.empty((n, 3))
        O.port_lib().orc_random_initial_configuration(n, box, 0.85, C.byref(r), O.dptr(pos))
        assert np.array_equal(xyz, pos)
        assert rng.serialize_hex() == O.rng_to_hex(r)


def test_rng_state_hex_roundtrip():
    from paper_1408_3764_b200 import engine as E

    r = E.RngState.from_seed(42)
    assert E.RngState.deserialize_hex(r.serialize_hex()).serialize_hex() == r.serialize_hex()
    if O.ref_available():
        buf = C.create_string_buffer(16384)
        O.ref_lib().ref_rng_hex(42, 0, buf, 16384)
        assert r.serialize_hex() == buf.value.decode()


SMALL = """# small LJ system
temperature = 2.0
chemical_potential = -2.0
particles = 250
density = 0.5
steps = 600
seed = 99
checkpoint_interval = 200
strategy = microcell
"""


def test_config_parse_matches_reference():
    cfg = CFG.parse_config_text(SMALL)  # test_harness.cpp:46-59
    assert cfg.temperature == 2.0 and cfg.initial_particles == 250
    assert cfg.strategy == "microcell" and cfg.displace_percent == 0.30
    assert cfg.microcell_capacity == 5 and not cfg.tail_corrections
    if O.ref_available():
        rc = O.RefConfig()
        assert O.ref_lib().ref_parse_config(SMALL.encode(), C.byref(rc)) == 0
        assert rc.box_length == cfg.box_length
        buf = C.create_string_buffer(4096)
        O.ref_lib().ref_serialize_config(C.byref(rc), buf, 4096)
        assert buf.value.decode() == cfg.serialize()


@pytest.mark.parametrize("bad", [
    "temperature=2\nchemical_potential=1\nbox_length=10\nfoo=1\n",        # unknown key
    "temperature=2\nchemical_potential=1\nbox_length=10\nbox_length=11\n",  # duplicate
    "chemical_potential=1\nbox_length=10\n",                                # missing T
    "temperature=2\nchemical_potential=1\n",                                # no geometry
    "temperature=2\nchemical_potential=1\nbox_length=4\n",                  # rc > L/2
    "temperature=2\nchemical_potential=1\nbox_length=10\nstrategy=verlet\n",
])
def test_config_rejects_like_reference(bad):
    with pytest.raises(ValueError):
        CFG.parse_config_text(bad)
    if O.ref_available():
        rc = O.RefConfig()
        assert O.ref_lib().ref_parse_config(bad.encode(), C.byref(rc)) != 0


def test_reference_configs_parse():
    for name in ("ideal_gas.cfg", "lj_small.cfg"):
        path = os.path.join("/root/reference/proj/configs", name)
        if not os.path.exists(path):
            pytest.skip("reference configs not present")
        cfg = CFG.parse_config_file(path)
        cfg.validate()


def test_checkpoint_text_roundtrip_and_reference_format():
    from paper_1408_3764_b200 import checkpoint as CK
    from paper_1408_3764_b200 import engine as E

    n = 64
    box = (n / 0.5) ** (1 / 3)
    xyz, rng = E.random_initial_configuration(n, box, 0.85, 4, device=None)
    cfg = CFG.RunConfig(temperature=2.0, chemical_potential=-2.0, box_length=box,
                        strategy="microcell", seed=4)
    c = CK.Checkpoint(cfg, 17, -12.5, 3.25, rng.serialize_hex(), xyz)
    txt = CK.to_text(c)
    back = CK.checkpoint_from_text(txt)
    assert back.step == 17 and back.energy == -12.5 and np.array_equal(back.positions, xyz)
    if O.ref_available():
        # the reference restores our text bit-for-bit and writes the same text back
        sim = O.RefSim.from_checkpoint(txt)
        assert sim.checkpoint_text() == txt
