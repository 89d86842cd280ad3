"""K1 per-CTA phase timeline from the PFT_TIMELINE build (development aid).

    PFT_LIB=variants/lib_timeline.so python tools/timeline.py
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402

N, M, mu, p = 2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15
plan = pft.build_plan(N, M, mu, p, 1e-12)
d = pft.DevicePlan(plan)
x = torch.empty(N, dtype=torch.complex128, device="cuda")
pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 1, N)
Y = torch.empty(plan.p * plan.r, dtype=torch.complex128, device="cuda")
for _ in range(5):
    d.execute_partial_ptr(x.data_ptr(), Y.data_ptr())
torch.cuda.synchronize()
n = d.P2
buf = (C.c_ulonglong * (6 * n))()
pft.lib().pft_debug_timeline.restype = C.c_int
assert pft.lib().pft_debug_timeline(buf, n) == 0
t = np.array(buf, dtype=np.float64).reshape(n, 6)
t -= t[:, 0].min()
t /= 1e3  # us
names = ["start", "first data", "main loop end", "after sync", "fft end", "end"]
print("CTAs:", n)
for i, nm in enumerate(names):
    print(f"{nm:>15}: min {t[:, i].min():7.2f}  median {np.median(t[:, i]):7.2f}  max {t[:, i].max():7.2f} us")
for a, b, nm in [(0, 1, "first-data latency"), (1, 2, "main loop"), (2, 3, "barrier"), (3, 4, "fft"), (4, 5, "Y write")]:
    dd = t[:, b] - t[:, a]
    print(f"{nm:>20}: min {dd.min():6.2f} median {np.median(dd):6.2f} max {dd.max():6.2f}")
# which CTAs are slow: by SM co-residency proxy (blockIdx >= 148 ~ second slot)
late = t[:, 5]
print("end time blockIdx<148 median", np.median(late[:148]), " >=148 median", np.median(late[148:]))
