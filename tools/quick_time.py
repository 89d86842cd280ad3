"""Quick device timing of the execute path for a few plans (development aid)."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402


def time_plan(N, M, mu, p, p2=0, reps=50, label=""):
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    d = pft.DevicePlan(plan, p2=p2)
    bufs = [torch.empty(N, dtype=torch.complex128, device="cuda") for _ in range(2)]
    for i, b in enumerate(bufs):
        pft.generate_signal_device(b.data_ptr(), pft.KIND_UNIFORM, 1 + i, N)
    out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for i in range(5):
        d.execute_ptr(bufs[i % 2].data_ptr(), out.data_ptr(), stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        d.execute_ptr(bufs[i % 2].data_ptr(), out.data_ptr(), stream=st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = 16 * N / (ms * 1e-3) / 1e9
    print(json.dumps({"label": label, "N": N, "M": M, "p": plan.p, "q": plan.q, "r": plan.r, "P1": d.P1,
                      "P2": d.P2, "us": round(ms * 1e3, 2), "GB/s": round(gbs, 1)}), flush=True)


if __name__ == "__main__":
    time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b p=2^15")
    time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, p2=256, label="C2b p=2^15 P2=256")
    time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, p2=1024, label="C2b p=2^15 P2=1024")
    time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 16, label="C2b p=2^16")
    time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label="C2b p=2^14")
    time_plan(2 ** 24, 2 ** 6, 2 ** 22, None, label="C2a")
    time_plan(2 ** 24, 2 ** 14, 2 ** 22, None, label="C2c")
    time_plan(2 ** 20, 64, 0, None, label="C1")
    time_plan(6220800, 1000, -12345, 62208, label="C4")
