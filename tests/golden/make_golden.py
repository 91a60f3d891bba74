"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs only in the build container (needs /root/reference, compiled through
oracle/_ref/libgcmc_ref.so). The fixtures travel with the repo, so the GPU
box and the CPU tests check against them without the reference.

    python tests/golden/make_golden.py

Contents of golden.npz (all produced by the unmodified reference):
  mt_seed1_first16, mt_seed42_skip1000_16   RngStream::uniform() outputs
  init_256_xyz, init_256_rng                random_initial_configuration(256, L, 0.85, RngStream(7))
  trace_<strategy>_<mu>                     2000-move step() traces (kind, accepted, dU, dW, p, N)
  final_<strategy>_<mu>                     (energy, virial, sum_u, sum_p, sum_n, sum_n2, N)
  final_<strategy>_<mu>_rng                 RNG state after the trace (serialize_hex)
  grid_micro_occ/slots, grid_cell_occ/slots after build of init_256
  deltas_<strategy>                         (kind, pid, x, y, z, dU, dW) for 300 proposals
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def main() -> None:
    out: dict[str, np.ndarray] = {}
    meta: dict = {}
    out["mt_seed1_first16"] = O.ref_uniforms(1, 16)
    out["mt_seed42_skip1000_16"] = O.ref_uniforms(42, 16, skip=1000)

    n0 = 256
    box = (n0 / 0.67) ** (1.0 / 3.0)
    meta["init_256_box"] = box
    xyz, rng_hex = O.ref_initial_configuration(n0, box, 7)
    out["init_256_xyz"] = xyz
    meta["init_256_rng"] = rng_hex

    for strat in ("all_pairs", "cell_list", "microcell"):
        for mu in (-2.0, 1.0):
            cfg = O.ref_config(temperature=2.0, chemical_potential=mu, box_length=box,
                               strategy=strat, tail_corrections=1)
            sim = O.RefSim(cfg, mode=1, xyz=xyz, rng_hex=rng_hex)
            st0 = sim.state()
            _, tr = sim.run(2000, trace=True)
            st = sim.state()
            key = f"{strat}_{'m2' if mu < 0 else 'p1'}"
            out[f"trace_{key}"] = tr
            out[f"final_{key}"] = np.array([st.energy, st.virial, st.sum_u, st.sum_p, st.sum_n,
                                            st.sum_n2, float(st.n)])
            meta[f"initial_energy_{key}"] = [st0.energy, st0.virial]
            meta[f"final_{key}_rng"] = sim.rng_hex()
            out[f"final_{key}_xyz"] = sim.positions()

    micro = O.RefStrategy("microcell", xyz, box)
    out["grid_micro_occ"], out["grid_micro_slots"] = micro.grid()
    cell = O.RefStrategy("cell_list", xyz, box)
    out["grid_cell_occ"], out["grid_cell_slots"] = cell.grid()

    rng = np.random.default_rng(123)
    for strat in ("all_pairs", "cell_list", "microcell"):
        s = O.RefStrategy(strat, xyz, box)
        rows = []
        for k in range(300):
            kind = k % 3
            pid = int(rng.integers(0, n0))
            p = rng.random(3) * box
            if kind == 0:
                du, dw = s.delta_displace(pid, p)
            elif kind == 1:
                du, dw = s.delta_insert(p)
            else:
                du, dw = s.delta_delete(pid)
            rows.append([kind, pid, p[0], p[1], p[2], du, dw])
        out[f"deltas_{strat}"] = np.array(rows)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
