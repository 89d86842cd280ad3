"""Regenerate the shipped ScopeTable artifact (cmd_gen_table).

    python -m paper_2008_12559_b200.gen_table [--out PATH] [--r-max 25] [--eps 1e-1,...]

Defaults: eps in {1e-1, ..., 1e-13} x r in 1..25 (SPEC.md:103's grid extended to cover
BASELINE.json's eps = 1e-12).  Generation is deterministic: the same
flags give a byte-identical file.
"""
from __future__ import annotations

import argparse
import time
from pathlib import Path

from . import ScopeTable

DEFAULT_OUT = Path(__file__).resolve().parent / "data" / "scope_table_v1.pftt"
DEFAULT_EPS = [10.0 ** -k for k in range(1, 14)]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(DEFAULT_OUT))
    ap.add_argument("--r-max", type=int, default=25)
    ap.add_argument("--eps", default="")
    ap.add_argument("--csv", default="")
    a = ap.parse_args()
    eps = [float(x) for x in a.eps.split(",")] if a.eps else [float(f"1e-{k}") for k in range(1, 14)]
    t0 = time.time()
    tab = ScopeTable.generate(eps, a.r_max)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    tab.save(a.out)
    if a.csv:
        tab.save_csv(a.csv)
    print(f"wrote {a.out}: {len(tab)} entries in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
