"""Where a 2-D PFT execute spends its time, and which per-axis p the device prefers (dev aid).

    python tools/probe_2d.py N1 N2 M1 M2
Times (CUDA events, 20 executes after 3 warm-ups): the full pft_execute_2d at the SPEC plans;
the axis-2 row pass alone (batch N1, stride N2) at each candidate p; the axis-1 column pass
alone (batch 2M2+1, stride N1) at each candidate p.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


N1, N2, M1, M2 = (int(x) for x in sys.argv[1:5])
plan = pft.build_plan_2d(N1, N2, M1, M2, 0, 0, epsilon=1e-12)
x = torch.empty(N1 * N2, dtype=torch.complex128, device="cuda")
pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 5, N1 * N2)
ws = torch.zeros(-(-plan.workspace_bytes() // 16), dtype=torch.complex128, device="cuda")
out = torch.empty((2 * M1 + 1) * (2 * M2 + 1), dtype=torch.complex128, device="cuda")
print(f"full 2-D (SPEC p1={plan.plan1.p} r1={plan.plan1.r}, p2={plan.plan2.p} r2={plan.plan2.r}): "
      f"{timeit(lambda: plan.execute_ptr(x.data_ptr(), out.data_ptr(), ws.data_ptr())):.1f} us")


def axis(N, M, batch, label):
    W = 2 * M + 1
    o = torch.empty(W * batch, dtype=torch.complex128, device="cuda")
    for p in [d for d in range(2, N + 1) if N % d == 0 and d >= 16 and N // d >= 2]:
        try:
            pl = pft.build_plan(N, M, 0, p, 1e-12)
            d = pft.DevicePlan(pl, batch_hint=batch)
        except Exception as e:  # noqa: BLE001
            print(f"  {label} p={p}: {e}")
            continue
        w = torch.zeros(-(-d.workspace_bytes(batch) // 16), dtype=torch.complex128, device="cuda")
        t = timeit(lambda: d.execute_ptr(x.data_ptr(), o.data_ptr(), batch=batch, in_stride=N, d_ws=w.data_ptr()))
        print(f"  {label} p={p:6d} r={pl.r:2d} P1={d.P1} P2={d.P2} {d.tail_kind():9s}: {t:9.1f} us "
              f"({16 * N * batch / t / 1e3:7.0f} GB/s)")


axis(N2, M2, N1, "rows")
axis(N1, M1, 2 * M2 + 1, "cols")
