"""2-D PFT throughput on one B200 (measurement beside bench.py's 1-D lines).

    python tools/bench_2d.py [--n1 4096] [--n2 4096] [--m1 64] [--m2 64] [--steps 200] [--warmup 5]

A step = one pft_execute_2d (axis-2 pass batched over the N1 rows, tiled transpose, axis-1
pass over the 2M2+1 columns, final transpose) on a device-resident N1 x N2 complex128 grid.
Inputs: 2 rotating seeded U[-1,1] grids of 16*N1*N2 bytes each (> L2 at the default 268 MB).
Timing: K steps captured in one CUDA graph, CUDA events on the launch stream, W warm-up steps.
Roofline: algorithmic bytes = the 16*N1*N2 input bytes per transform (the first pass streams
them once; everything after is O(N1*M2)), against MEASURED_PEAKS.json hbm_gbs.
CPU baseline: the oracle's execute_2d (oracle/, test infrastructure) on a bounded sample,
all host threads.  Prints one JSON line; parity is tests/test_pft2d.py's job, but the line
records the GPU-vs-oracle relative l2 on the sample input.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2008_12559_b200 as pft  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n1", type=int, default=4096)
    ap.add_argument("--n2", type=int, default=4096)
    ap.add_argument("--m1", type=int, default=64)
    ap.add_argument("--m2", type=int, default=64)
    ap.add_argument("--mu1", type=int, default=0)
    ap.add_argument("--mu2", type=int, default=0)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--spec-p", action="store_true", help="keep SPEC's CPU p per axis (no device autotune)")
    a = ap.parse_args()
    N1, N2, M1, M2 = a.n1, a.n2, a.m1, a.m2
    W1, W2 = 2 * M1 + 1, 2 * M2 + 1
    plan = pft.build_plan_2d(N1, N2, M1, M2, a.mu1, a.mu2, epsilon=1e-12)
    dev = torch.device("cuda:0")
    bufs = []
    for i in range(2):
        x = torch.empty(N1 * N2, dtype=torch.complex128, device=dev)
        pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 50 + i, N1 * N2)
        bufs.append(x)
    spec_p = (plan.plan1.p, plan.plan2.p)
    if not a.spec_p:  # device-measured p per axis (autotune_2d), the oracle gets the same plans
        plan = pft.autotune_2d(plan, bufs[0].data_ptr())
    ws = torch.zeros(-(-plan.workspace_bytes() // 16), dtype=torch.complex128, device=dev)  # zeroed once
    out = torch.empty(W1 * W2, dtype=torch.complex128, device=dev)
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    with torch.cuda.stream(stream):
        for i in range(a.warmup):
            plan.execute_ptr(bufs[i % 2].data_ptr(), out.data_ptr(), ws.data_ptr(), stream=sp)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(a.steps):
            plan.execute_ptr(bufs[i % 2].data_ptr(), out.data_ptr(), ws.data_ptr(), stream=sp)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        g.replay()  # warm replay
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    value = 1e3 / ms
    gbs = 16.0 * N1 * N2 * value / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 7672.0))

    # parity of the timed path on the last input, and the CPU oracle on a bounded sample
    import oracle  # test infrastructure: the checker and the CPU baseline only
    host = bufs[(a.steps - 1) % 2].cpu().numpy().reshape(N1, N2)
    plan.execute_ptr(bufs[(a.steps - 1) % 2].data_ptr(), out.data_ptr(), ws.data_ptr())
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(W1, W2)
    nthreads = os.cpu_count() or 1
    t0, n_cpu, ref = time.perf_counter(), 0, None
    while True:
        r = oracle.execute_2d(plan.plan1, plan.plan2, host, plan.parenthesization)
        ref = r if ref is None else ref
        n_cpu += 1
        if time.perf_counter() - t0 >= a.cpu_seconds:
            break
    cpu_s = time.perf_counter() - t0
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    line = {
        "metric": "2-D PFT transforms/sec", "value": value, "unit": "transforms/s", "n_gpus": 1,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "dtype": "f64 (complex128)", "data": "synthetic",
        "config": {"workload": f"2-D PFT N1 x N2 = {N1} x {N2}, (M1, M2) = ({M1}, {M2}), "
                               f"mu = ({a.mu1}, {a.mu2}), eps = 1e-12, U[-1,1] re/im",
                   "p1": plan.plan1.p, "r1": plan.plan1.r, "p2": plan.plan2.p, "r2": plan.plan2.r,
                   "p_choice": "SPEC select_divisor per axis" if a.spec_p else
                               f"autotune_2d (pft_autotune_divisor per axis at its batch; SPEC picks {spec_p})",
                   "l2": f"2 rotating inputs of {16 * N1 * N2 / 2**20:.0f} MiB",
                   "timing": "CUDA graph of K steps, CUDA events on the launch stream"},
        "input_gbs": gbs,
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                     "algorithmic_bytes_per_transform": 16 * N1 * N2,
                     "note": "whole 2-D execute (4 launches) against the input bytes"},
        "rel_l2_gpu_vs_oracle": rel,
        "cpu_baseline": {"value": n_cpu / cpu_s, "unit": "transforms/s", "cores": nthreads, "kind": "port",
                         "sample": f"{n_cpu} full 2-D transforms in {cpu_s:.1f} s (oracle execute_2d)"},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
