"""K chains of the 64k mu-sweep on one GPU with a chosen engine: aggregate
moves/s after a warm-up (wall clock around gcmc_run_chains, which returns
when every chain is done).

    python tools/sm_sweep.py --mode 2 --k 1 8 32 64 --moves 200000
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--k", type=int, nargs="+", default=[1, 8])
    ap.add_argument("--n0", type=int, default=65536)
    ap.add_argument("--moves", type=int, default=200000)
    ap.add_argument("--warm", type=int, default=400000)
    ap.add_argument("--mu0", type=float, default=-3.0)
    ap.add_argument("--spread", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    from paper_1408_3764_b200 import engine as E
    from paper_1408_3764_b200.config import RunConfig

    box = (a.n0 / 0.67) ** (1.0 / 3.0)
    for K in a.k:
        sims = []
        for c in range(K):
            mu = a.mu0 + a.spread * c / K
            xyz, rng = E.random_initial_configuration(a.n0, box, 0.85, 1 + c, device=0)
            cfg = RunConfig(temperature=2.0, chemical_potential=mu, box_length=box, seed=1 + c,
                            strategy="microcell")
            kw = {"engine_mode": a.mode}
            if K > 1:
                kw["engine_share"] = K
            sims.append(E.Simulation(cfg, xyz, rng, **kw))
        E.run_chains(sims, a.warm) if K > 1 else sims[0].run(a.warm)
        best = None
        for _ in range(a.reps):
            t0 = time.perf_counter()
            res = E.run_chains(sims, a.moves) if K > 1 else [sims[0].run(a.moves) or sims[0].last_run]
            dt = time.perf_counter() - t0
            rounds = sum(r.rounds for r in res)
            dev = max(r.device_ms for r in res)
            v = K * a.moves / dt
            if best is None or v > best["moves_per_s"]:
                best = {"k": K, "mode": a.mode, "moves_per_s": v, "per_chain": v / K,
                        "moves_per_round": K * a.moves / max(1, rounds), "wall_s": dt,
                        "max_device_ms": dev, "engine": [r.engine for r in res][:4], "n": [s.dev.get_state().n for s in sims[:4]]}
        print(json.dumps(best), flush=True)
        for s in sims:
            s.close()


if __name__ == "__main__":
    main()
