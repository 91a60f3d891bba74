"""Attribute ncu per-SASS stall samples to source lines (via nvdisasm -g).
usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTR [topN]"""
import csv, re, subprocess, sys, tempfile, os, collections
rep, obj, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}; data = rows[2:]
f = lambda r, k: float(r[ix[k]]) if r[ix[k]] else 0.0
base = min(int(r[ix["Address"]], 16) for r in data)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [x for x in os.listdir(d) if x.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
# find function block
lines = sass.splitlines()
start = next(i for i, l in enumerate(lines) if ".text." in l and kname in l and l.strip().startswith(".section"))
cur = None; off2line = {}
for l in lines[start + 1:]:
    if l.strip().startswith(".section") and ".text." in l: break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"; continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur: off2line[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in data:
    off = int(r[ix["Address"]], 16) - base
    key = off2line.get(off, "?")
    a = agg[key]; a[0] += f(r, "Warp Stall Sampling (All Samples)"); a[1] += f(r, "Instructions Executed")
    for s in stalls: a[2][s[6:]] += f(r, s)
tot = sum(a[0] for a in agg.values())
print(f"total samples {tot:.0f}")
# samples of warps that are not parked at a barrier or asleep (the serial chains)
act = lambda a: a[0] - a[2]["barrier"] - a[2]["sleep"]
tact = sum(act(a) for a in agg.values())
print(f"active samples {tact:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -act(kv[1]))[:top]:
    c = a[2].copy(); c.pop("barrier", None); c.pop("sleep", None)
    print(f"{act(a):7.0f} {100*act(a)/tact:5.1f}% inst {a[1]:10.0f}  {k:28s} {c.most_common(3)}")
