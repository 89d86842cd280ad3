"""2-D column-pass form check: sum tail (forced) vs the planner's choice at batch 2M2+1 (dev aid)."""
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

for (N, M, B) in [(4096, 64, 129), (1024, 32, 513), (2 ** 16, 256, 64)]:
    x = torch.empty(N * B, dtype=torch.complex128, device="cuda")
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 5, N * B)
    o = torch.empty((2 * M + 1) * B, dtype=torch.complex128, device="cuda")
    for p in [d for d in range(32, N // 2 + 1) if N % d == 0]:
        for mode in (0, 5):
            try:
                pl = pft.build_plan(N, M, 0, p, 1e-12)
                d = pft.DevicePlan(pl, batch_hint=B, k2_mode=mode)
            except Exception:  # noqa: BLE001
                continue
            w = torch.zeros(-(-d.workspace_bytes(B) // 16), dtype=torch.complex128, device="cuda")
            t = timeit(lambda: d.execute_ptr(x.data_ptr(), o.data_ptr(), batch=B, in_stride=N, d_ws=w.data_ptr()))
            print(f"N={N} M={M} B={B} p={p:5d} r={pl.r:2d} P2={d.P2:3d} mode={mode} {d.tail_kind():8s} {t:8.1f} us")
