"""Markdown table of moves/s (and reference-equivalent pair evals/s) vs N from
bench.py JSON lines: python tools/vs_n_table.py gpurun_out/vsn/vs_n.jsonl

pair evals per move follow SURVEY §8d (reference work, not the engine's):
1.3 windows per move (0.3 displace x 2 + 0.7 x 1) x candidates per window,
216 rho (microcell arc), 434 rho (27-cell list), N (all pairs); rho = final N / V.
"""
import json, sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
print("| N0 | strategy | mu | moves/step | GPU moves/s (device) | GPU moves/s (e2e) | CPU ref moves/s (1 core, same moves) | e2e / CPU | ns/move | final N | ref-equiv. pair evals/s |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    c = r["config"]
    n0 = c["n0"]
    vol = n0 / c["density"]
    nf = r.get("n_final", n0)
    rho = nf / vol
    per_win = {"microcell": 216 * rho, "cell_list": 434 * rho, "all_pairs": nf}[c["strategy"]]
    pe = r["value"] * 1.3 * per_win
    cpu = r.get("cpu_baseline") or {}
    cv = cpu.get("value")
    e2e = r["e2e"]["value"]
    print(f"| {n0} | {c['strategy']} | {c['mu']:+g} | {c['moves_per_step']} | {r['value']/1e6:.2f} M | {e2e/1e6:.2f} M | "
          f"{(cv or 0)/1e3:.1f} k | {e2e/cv if cv else float('nan'):.0f}x | {1e9/r['value']:.0f} | {nf} | {pe:.2e} |")
