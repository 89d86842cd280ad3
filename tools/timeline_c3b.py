"""Per-CTA phases of the batched sum-tail K1 including the reduction (PFT_TIMELINE build).

    PFT_LIB=variants/lib_tl.so python tools/timeline_c3b.py [N] [M] [p] [batch]
K1 stamps: 0 start, 1 first stage, 2 loop end, 3 barrier, 4 FFT end, 5 row written;
sum-tail stamps (timeline2): 0 ticket taken, 1 rows ready (reducers), 2 reduction done, 3 exit.
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 16
M = int(sys.argv[2]) if len(sys.argv) > 2 else 256
p = int(sys.argv[3]) if len(sys.argv) > 3 else 256
B = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
plan = pft.build_plan(N, M, 0, p, 1e-12)
d = pft.DevicePlan(plan, batch_hint=B)
x = torch.empty(N * B, dtype=torch.complex128, device="cuda")
pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 3, N * B)
ws = torch.zeros(-(-d.workspace_bytes(B) // 16), dtype=torch.complex128, device="cuda")
out = torch.empty((2 * M + 1) * B, dtype=torch.complex128, device="cuda")
for _ in range(6):
    d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=B, in_stride=N, d_ws=ws.data_ptr())
torch.cuda.synchronize()
L = pft.lib()
b1 = (C.c_ulonglong * (4 * 4096 * 6))()
b2 = (C.c_ulonglong * (4 * 4096 * 6))()
L.pft_debug_timeline(b1)
L.pft_debug_timeline2(b2)
t1 = np.array(b1, dtype=np.float64).reshape(4, 4096, 6)
t2 = np.array(b2, dtype=np.float64).reshape(4, 4096, 6)
k = max(range(4), key=lambda i: t1[i, 0, 0])  # the last execute
n = min(4096, d.P2 * B)
a, z = t1[k, :n] / 1e3, t2[k, :n] / 1e3
print(f"N={N} M={M} p={p} r={plan.r} P1={d.P1} P2={d.P2} batch={B} reducers(plan)")
red = z[:, 1] > 0
rows = [("wait first stage", a[:, 1] - a[:, 0]), ("stream", a[:, 2] - a[:, 1]), ("barrier", a[:, 3] - a[:, 2]),
        ("FFT", a[:, 4] - a[:, 3]), ("tail row", a[:, 5] - a[:, 4]), ("fence+ticket", z[:, 0] - a[:, 5]),
        ("reducer: wait rows", (z[:, 1] - z[:, 0])[red]), ("reducer: reduce", (z[:, 2] - z[:, 1])[red]),
        ("reducer: re-arm+exit", (z[:, 3] - z[:, 2])[red]), ("non-reducer exit", (z[:, 3] - z[:, 0])[~red]),
        ("CTA total", z[:, 3] - a[:, 0])]
for nm, v in rows:
    if len(v):
        print(f"{nm:>22}: mean {v.mean():7.2f} us  med {np.median(v):7.2f}  max {v.max():7.2f}  (n={len(v)})")
print(f"{'span of these CTAs':>22}: {z[:, 3].max() - a[:, 0].min():.1f} us")
