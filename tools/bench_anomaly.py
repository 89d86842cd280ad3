"""cmd_anomaly throughput (SPEC.md cli `anomaly`, §4.4).

    python tools/bench_anomaly.py [--n 19735] [--m 125] [--k 20] [--series 200]

One call = one spike-injected series through `pft.anomaly` (host series -> H2D -> one GPU PFT
execute for the 2M+1 coefficients on R_{0,M} -> D2H -> reconstruction + top-k scoring on the
host, inside libpft_b200.so).  Beside it, the same scoring fed by the CPU oracle's PFT
(oracle/, test infrastructure) on the same plan.  Wall clock over `--series` calls after 3
warm-ups; prints one JSON line with both rates and the top-k agreement count.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2008_12559_b200 as pft  # noqa: E402


def series(N, M, k, seed):
    rng = np.random.default_rng(seed)
    n = np.arange(N)
    x = np.zeros(N)
    for _ in range(6):
        f = rng.integers(1, M)
        x += rng.uniform(0.2, 1.0) * np.cos(2 * np.pi * f * n / N + rng.uniform(0, 2 * np.pi))
    x += 0.01 * rng.standard_normal(N)
    x[rng.choice(N, size=k, replace=False)] += rng.choice([-1, 1], size=k) * rng.uniform(0.8, 2.0, size=k)
    return x


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=19735)
    ap.add_argument("--m", type=int, default=125)
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--series", type=int, default=200)
    a = ap.parse_args()
    xs = [series(a.n, a.m, a.k, 1000 + i) for i in range(a.series)]
    for x in xs[:3]:
        pft.anomaly(x, a.m, a.k)
    t0 = time.perf_counter()
    gpu_idx = [pft.anomaly(x, a.m, a.k)[0] for x in xs]
    gpu_s = time.perf_counter() - t0

    import oracle  # the checker / CPU baseline only
    plan = pft.build_plan(a.n, a.m, 0, None, 1e-12)
    t0 = time.perf_counter()
    cpu_idx = []
    for x in xs:
        c = oracle.execute(plan, x.astype(np.complex128))
        cpu_idx.append(pft.anomaly_from_coeffs(x, c, a.m, a.k)[0])
    cpu_s = time.perf_counter() - t0
    agree = sum(set(g.tolist()) == set(c.tolist()) for g, c in zip(gpu_idx, cpu_idx))
    print(json.dumps({
        "metric": "anomaly series/sec", "value": a.series / gpu_s, "unit": "series/s",
        "config": {"workload": f"cmd_anomaly: N = {a.n}, M = {a.m}, k = {a.k}, spike-injected tones + noise",
                   "p": plan.p, "r": plan.r, "series": a.series,
                   "timing": "host wall clock around pft.anomaly (H2D, GPU execute, D2H, host scoring)"},
        "cpu_baseline": {"value": a.series / cpu_s, "unit": "series/s", "kind": "port",
                         "sample": f"{a.series} series: oracle execute + the same scoring"},
        "topk_sets_identical": f"{agree}/{a.series}",
    }))


if __name__ == "__main__":
    main()
