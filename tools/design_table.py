"""Print the DESIGN.md / README.md measurement table from profiles/r02/bench_*_<tag>.json.

    python tools/design_table.py r02h
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02h"
NAMES = [("default", "C2b (headline): N = 2^24, M = 2^10"), ("c2a", "C2a: M = 2^6"), ("c2c", "C2c: M = 2^14"),
         ("c3", "C3: 4096 × 2^16, M = 256, per batch"), ("c4", "C4: N = 6,220,800, M = 1000"),
         ("c1", "C1: N = 2^20, M = 64"), ("c5", "C5: N = 2^30, M = 2^12 (1 GPU)")]


def load(c):
    return json.loads((ROOT / "profiles" / "r02" / f"bench_{c}_{TAG}.json").read_text())


def t(ms):
    return f"{ms * 1e3:.1f} µs" if ms < 0.5 else f"{ms:.3f} ms"


print("| config | per execute, chained | isolated (device) | p / r / P1 × P2, tail | frac (chained) | parity vs oracle |")
print("|---|---|---|---|---|---|")
for c, name in NAMES:
    r = load(c)
    cfg, clk = r["config"], r["clocks"]
    note = f" (SM {clk['sm_mhz']} MHz, sw_power_cap)" if clk["reasons"] else ""
    tail = cfg["tail"].split(" (")[0]
    print(f"| {name} | {t(r['ms_per_step'])}{note} | {t(r['latency_us_isolated'] / 1e3)} | "
          f"{cfg['p']} / {cfg['r']} / {cfg['P1']} × {cfg['P2']}, {tail} | {r['roofline']['frac']:.2f} | "
          f"{r['parity_rel_l2']:.1e} |")
r = load("c5_sharded")
print(f"| C5 via `pft_execute_sharded` (1-rank NCCL) | {t(r['ms_per_step'])} | -- | {r['config'].get('p', '')} / "
      f"{r['config'].get('r', '')}, sharded planner | {r['roofline']['frac']:.2f} | = plain execute (rel "
      f"{r.get('sharded_vs_plain_rel_l2', 0):.0e}) |")
r = load("2d")
print(f"| 2-D 4096², (64, 64) (`tools/bench_2d.py`) | {t(r['ms_per_step'])} | -- | rows p = {r['config'].get('p2')}, "
      f"columns p = {r['config'].get('p1')} | {r.get('roofline', {}).get('frac', 0):.2f} | tests |")
d, ref, an = load("default"), load("reference"), load("anomaly")
print()
print(f"e2e {d['e2e']['value']:.0f}/s; reference arm {ref['value']:.1f}/s; our p on the CPU "
      f"{d['cpu_baseline']['value']:.1f}/s (1 thread {d['cpu_baseline']['one_thread']['value']:.1f}/s); anomaly "
      f"{an['value']:.0f} series/s")
