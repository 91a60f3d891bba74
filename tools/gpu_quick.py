"""First-contact GPU check: prints parity numbers for each subsystem."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig

def step(name, f):
    t = time.time()
    try:
        r = f()
        print(f"[ok] {name} ({time.time()-t:.2f}s): {r}", flush=True)
    except Exception as e:
        print(f"[FAIL] {name}: {e}", flush=True)
        traceback.print_exc()

for n0 in (2048, 32768):
    box = (n0 / 0.67) ** (1 / 3)
    xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
    for strat in ("microcell", "cell_list", "all_pairs"):
        if strat == "all_pairs" and n0 > 4096: continue
        def grid():
            g = E.GpuNeighborStrategy(strat, xyz, box)
            r = O.RefStrategy(strat, xyz, box)
            if strat == "all_pairs": return "n/a"
            a, b = g.grid(); c, d = r.grid()
            return f"occ eq {np.array_equal(a,c)} slots eq {np.array_equal(b,d)} check={g.rebuild_check()}"
        step(f"{strat} {n0} build", grid)
        def deltas():
            g = E.GpuNeighborStrategy(strat, xyz, box)
            r = O.RefStrategy(strat, xyz, box)
            rs = np.random.default_rng(5)
            k = 300
            kinds = np.arange(k) % 3
            pids = rs.integers(0, n0, k)
            pts = rs.random((k, 3)) * box
            du, dw = g.delta_batch(kinds, pids, pts)
            ref = []
            for i in range(k):
                if kinds[i] == 0: ref.append(r.delta_displace(int(pids[i]), pts[i]))
                elif kinds[i] == 1: ref.append(r.delta_insert(pts[i]))
                else: ref.append(r.delta_delete(int(pids[i])))
            ref = np.array(ref)
            ru = np.abs(du - ref[:, 0]) / np.maximum(1, np.abs(ref[:, 0]))
            rw = np.abs(dw - ref[:, 1]) / np.maximum(1, np.abs(ref[:, 1]))
            return f"max rel dU {ru.max():.3e} dW {rw.max():.3e} bitwise {np.mean(du==ref[:,0]):.2f}"
        step(f"{strat} {n0} deltas", deltas)
    def energy():
        g = E.GpuNeighborStrategy("microcell", xyz, box)
        u, w = g.total_energy()
        t = time.time(); ru, rw = O.RefSim(O.ref_config(temperature=2.0, box_length=box, strategy=2), mode=1, xyz=xyz, rng_hex=rng.serialize_hex()).state().energy, 0
        return f"gpu U={u!r} ref U={ru!r} rel={abs(u-ru)/abs(ru):.2e} (ref {time.time()-t:.1f}s)"
    step(f"total energy {n0}", energy)
    for mu in (-2.0, 1.0):
        def traj():
            cfg = RunConfig(temperature=2.0, chemical_potential=mu, box_length=box, strategy="microcell")
            sim = E.Simulation(cfg, xyz, rng)
            nm = 20000
            t = time.time()
            tr = sim.run(nm, trace=True)
            dt = time.time() - t
            st = sim.dev.get_state()
            u0 = O.RefSim(O.ref_config(temperature=2.0, chemical_potential=mu, box_length=box, strategy=2), mode=1, xyz=xyz, rng_hex=rng.serialize_hex())
            _, tp = u0.run(nm, trace=True)
            same_k = np.array_equal(tr["kind"], tp["kind"]); same_a = np.array_equal(tr["accepted"], tp["accepted"])
            first_bad = np.argmax((tr["accepted"] != tp["accepted"]) | (tr["kind"] != tp["kind"])) if not (same_k and same_a) else -1
            rel = np.abs(tr["delta_u"] - tp["delta_u"]) / np.maximum(1, np.abs(tp["delta_u"]))
            res = sim.last_run
            peq = np.array_equal(sim.particles(), u0.positions()); req = sim.rng().serialize_hex()==u0.rng_hex()
            t2 = time.time(); sim.run(200000); dt2 = time.time() - t2
            r2 = sim.last_run
            return (f"kinds {same_k} acc {same_a} first_bad {first_bad} relmax {rel.max():.2e} acc={tr['accepted'].sum()} "
                    f"pos eq {peq} rng eq {req} "
                    f"rounds {res.rounds} dev_ms {res.device_ms:.2f} gen_ms {res.gen_ms:.2f} wall {dt:.2f}s | "
                    f"200k: dev_ms {r2.device_ms:.1f} gen_ms {r2.gen_ms:.1f} rounds {r2.rounds} -> {200000/(r2.device_ms/1e3):.3e} moves/s")
        step(f"traj {n0} mu={mu}", traj)
