"""K1 + K2 timeline of one transform (single stream, after warm-up) from the PFT_TIMELINE build."""
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
out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
for _ in range(5):
    d.execute_ptr(x.data_ptr(), out.data_ptr())
torch.cuda.synchronize()
L = pft.lib()
b1 = (C.c_ulonglong * (6 * d.P2))()
b2 = (C.c_ulonglong * (6 * d.P1))()
L.pft_debug_timeline(b1, d.P2)
L.pft_debug_timeline2(b2, d.P1)
t1 = np.array(b1, dtype=np.float64).reshape(d.P2, 6)
t2 = np.array(b2, dtype=np.float64).reshape(d.P1, 6)
t0 = t1[:, 0].min()
t1 = (t1 - t0) / 1e3
t2 = (t2 - t0) / 1e3
for nm, i in [("K1 start", 0), ("K1 first data", 1), ("K1 loop end", 2), ("K1 fft end", 4), ("K1 end", 5)]:
    print(f"{nm:>16}: min {t1[:, i].min():7.2f} med {np.median(t1[:, i]):7.2f} max {t1[:, i].max():7.2f}")
for nm, i in [("K2 start", 0), ("K2 prologue", 1), ("K2 after wait", 2), ("K2 slab loaded", 3), ("K2 fft end", 4),
              ("K2 end", 5)]:
    print(f"{nm:>16}: min {t2[:, i].min():7.2f} med {np.median(t2[:, i]):7.2f} max {t2[:, i].max():7.2f}")
