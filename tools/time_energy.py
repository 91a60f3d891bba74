"""Time gcmc_total_energy (cell pass) and the O(N^2) brute force at several N.
python tools/time_energy.py [--bf-max N]"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1408_3764_b200 import engine as E

ap = argparse.ArgumentParser()
ap.add_argument("--bf-max", type=int, default=1 << 18)
ap.add_argument("--sizes", default="32768,131072,262144,1048576")
a = ap.parse_args()
for n in [int(x) for x in a.sizes.split(",")]:
    box = (n / 0.67) ** (1 / 3)
    xyz, _ = E.random_initial_configuration(n, box, 0.85, 1)
    g = E.GpuNeighborStrategy("microcell", xyz, box)
    for _ in range(3):
        u, w = g.total_energy()
    p, k = g.energy_timing()
    line = f"n={n} cell pass {1e3*p:.1f} us kernel {1e3*k:.1f} us U={u:.10e}"
    if n <= a.bf_max:
        t = time.time()
        bu, bw = g.total_energy_bruteforce()
        line += f" | brute force {time.time()-t:.3f} s U={bu:.10e} rel {abs(u-bu)/abs(bu):.2e}"
    print(line, flush=True)
    g.close()
