"""Initial configuration (init_config.hpp:19-64) on the device vs the host
restatement: wall time and bitwise equality.  python tools/time_init.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E

for n in (32768, 262144, 1 << 20, 1 << 22):
    box = (n / 0.67) ** (1 / 3)
    E.random_initial_configuration(2048, (2048 / 0.67) ** (1 / 3), 0.85, 1, device=0)  # warm
    t = time.time(); dx, dr = E.random_initial_configuration(n, box, 0.85, 1, device=0); td = time.time() - t
    t = time.time(); hx, hr = E.random_initial_configuration(n, box, 0.85, 1, device=None); th = time.time() - t
    same = np.array_equal(dx, hx) and dr.serialize_hex() == hr.serialize_hex()
    print(f"n={n} device {td:.3f} s host {th:.3f} s ({th / td:.1f}x) draws {dr.draws} identical={same}", flush=True)
