"""Per-CTA phase durations of the batched C3 K1 (PFT_TIMELINE build; development aid).

    PFT_LIB=variants/lib_tl.so python tools/timeline_c3.py [p] [batch]

Stamps (kernel PFT_STAMP slots): 0 start, 1 first TMA stage landed, 2 contraction loop end,
3 after the block barrier, 4 first FFT pass end, 5 sum-tail row written.
"""
import sys
from pathlib import Path
import ctypes as C
import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
N, M = 2 ** 16, 256
plan = pft.build_plan(N, M, 0, p, 1e-12)
d = pft.DevicePlan(plan, batch_hint=B)
x = torch.empty(B * N, dtype=torch.complex128, device="cuda")
pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 3, B * N)
out = torch.empty(B * (2 * M + 1), dtype=torch.complex128, device="cuda")
ws = torch.zeros(d.workspace_bytes(B), dtype=torch.uint8, device="cuda")
for i in range(6):
    d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=B, d_ws=ws.data_ptr())
torch.cuda.synchronize()
L = pft.lib()
b1 = (C.c_ulonglong * (4 * 4096 * 6))()
L.pft_debug_timeline(b1)
t = np.array(b1, dtype=np.float64).reshape(4, 4096, 6)
k = int(np.argmax(t[:, 0, 0]))
a = t[k]
ok = a[:, 0] > 0
a = a[ok]
t0 = a[:, 0].min()
print(f"p={p} P1={d.P1} P2={d.P2} r={plan.r} CTAs recorded {ok.sum()}  span {(a[:, 5].max() - t0) / 1e3:.1f} us")
names = ["first data", "stream", "barrier", "fft", "tail row"]
for i in range(1, 6):
    dd = (a[:, i] - a[:, i - 1]) / 1e3
    print(f"{names[i - 1]:>11}: med {np.median(dd):7.2f} us  p10 {np.percentile(dd, 10):7.2f} p90 {np.percentile(dd, 90):7.2f}")
tot = (a[:, 5] - a[:, 0]) / 1e3
print(f"{'CTA total':>11}: med {np.median(tot):7.2f} us")
# concurrency: CTAs resident at the median time
mid = np.median(a[:, 0])
print("resident CTAs at median start:", int(((a[:, 0] <= mid) & (a[:, 5] >= mid)).sum()))
