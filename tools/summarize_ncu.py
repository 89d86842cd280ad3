"""Summarise ncu captures into profiles/ (committed evidence for the bench's roofline line).

    python tools/summarize_ncu.py --tag r01 --config c2b

Reads gpurun_out/launches_<tag>.csv (gpu__time_duration.sum per launch) and the --set full
reports gpurun_out/prof_k1_<tag>.ncu-rep / prof_k2_<tag>.ncu-rep; writes
profiles/<tag>_ncu_summary.md and updates profiles/k1_dram_traffic.json (per-launch DRAM
bytes of K1, which bench.py reports as roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep: Path) -> dict:
    # a capture too large to copy back is exported on the box (`ncu -i X --page raw --csv`)
    alt = rep.with_name(rep.name.replace(".ncu-rep", ".raw.csv"))
    if not rep.exists() and alt.exists():
        out = alt.read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    units = dict(zip(rows[0], rows[1]))
    return {h: (v, units.get(h, "")) for h, v in zip(rows[0], rows[2])}


def stalls(d: dict) -> list[tuple[str, float]]:
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[0])) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v[0]
          and float(v[0]) > 0]
    tot = sum(x for _, x in st) or 1.0
    return [(n, x / tot) for n, x in sorted(st, key=lambda x: -x[1])[:8]]


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def launch_shares(path: Path) -> list[tuple[str, int, float, float]]:
    rows = list(csv.reader(path.read_text().splitlines()))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    acc = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            acc[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for k, v in acc.items() if "generate" not in k and "elementwise" not in k) or 1.0
    return [(k, len(v), sum(v) / len(v), sum(v) / total) for k, v in acc.items()]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="c2b")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    lines = [f"# ncu summary {a.tag} ({a.config})", "", a.note, "",
             "Captured with `tools/profile_run.sh` on one B200 (`ncu --set full --clock-control none`, "
             "cold caches, one launch each); the launch list is `--metrics gpu__time_duration.sum`.", ""]
    lp = OUT / f"launches_{a.tag}.csv"
    if lp.exists():
        lines += ["## Launch list (share of PFT kernel time)", "", "| kernel | launches | mean us | share |",
                  "|---|---|---|---|"]
        for k, n, mean, share in launch_shares(lp):
            if "generate" in k or "elementwise" in k:
                continue  # input generation / torch fills, outside the timed region
            lines.append(f"| `{k}` | {n} | {mean / 1e3:.2f} | {share:.1%} |")
        lines.append("")
    traffic = {}
    for kern in ("k1", "k2"):
        rep = OUT / f"prof_{kern}_{a.tag}.ncu-rep"
        if not rep.exists() and not (OUT / f"prof_{kern}_{a.tag}.raw.csv").exists():
            continue
        d = raw(rep)
        lines += [f"## {kern.upper()} (`--set full`)", "", "| metric | value |", "|---|---|"]
        for key, label in METRICS:
            if key in d:
                v, u = d[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        lines += ["", "Top stall reasons (share of sampled stalls): " +
                  ", ".join(f"{n} {x:.0%}" for n, x in stalls(d)), ""]
        if kern == "k1":
            rd = to_bytes(*d["dram__bytes_read.sum"])
            wr = to_bytes(*d["dram__bytes_write.sum"])
            traffic = {"dram_bytes_read": rd, "dram_bytes_write": wr, "traffic": rd + wr,
                       "source": f"profiles/{a.tag}_ncu_summary.md"}
    (PROF / f"{a.tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    if traffic:
        tf = PROF / "k1_dram_traffic.json"
        cur = json.loads(tf.read_text()) if tf.exists() else {}
        cur[a.config] = traffic["traffic"]
        cur[f"{a.config}_detail"] = traffic
        tf.write_text(json.dumps(cur, indent=1) + "\n")
    print((PROF / f"{a.tag}_ncu_summary.md").read_text())


if __name__ == "__main__":
    main()
