"""C2c K1 + K2 timeline, K2 grid vs K2 tail (PFT_TIMELINE build; development aid).

    PFT_LIB=variants/lib_tl.so python tools/timeline_k2tail.py [on|off] [reducers]
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402

tail = sys.argv[1] if len(sys.argv) > 1 else "on"
red = int(sys.argv[2]) if len(sys.argv) > 2 else 0
N, M, mu, p = 2 ** 24, 2 ** 14, 2 ** 22, 2 ** 15
plan = pft.build_plan(N, M, mu, p, 1e-12)
d = pft.DevicePlan(plan, k2_tail=1 if tail == "on" else -1, reducers=red)
print(d.tail_kind(), d.P1, d.P2)
xs = [torch.empty(N, dtype=torch.complex128, device="cuda") for _ in range(2)]
for i, x in enumerate(xs):
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 1 + i, N)
out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
torch.cuda.synchronize()
for i in range(40):
    d.execute_ptr(xs[i % 2].data_ptr(), out.data_ptr())
torch.cuda.synchronize()
L = pft.lib()
b1 = (C.c_ulonglong * (4 * 4096 * 6))()
b2 = (C.c_ulonglong * (4 * 4096 * 6))()
L.pft_debug_timeline(b1)
L.pft_debug_timeline2(b2)
t1 = np.array(b1, dtype=np.float64).reshape(4, 4096, 6)
t2 = np.array(b2, dtype=np.float64).reshape(4, 4096, 6)
order = sorted(range(4), key=lambda k: t1[k, 0, 0])
n1 = d.P2
n2 = red if (tail == "on" and red) else (min(64, d.P1) if tail == "on" else d.P1)
t0 = t1[order[1], :n1, 0].min()
names2 = ([("W start", 0), ("W wait done", 1), ("W slab0", 2), ("W fft0", 3), ("W m1 done", 4), ("W end", 5)]
          if tail == "on" else
          [("K2 start", 0), ("K2 prologue", 1), ("K2 after wait", 2), ("K2 slab", 3), ("K2 fft", 4), ("K2 end", 5)])
for k in order[1:]:
    a = (t1[k, :n1] - t0) / 1e3
    print(f"--- execute slot {k}")
    for nm, i in [("K1 start", 0), ("K1 first data", 1), ("K1 loop end", 2), ("K1 w fold", 3), ("K1 fft end", 4),
                  ("K1 slab written", 5)]:
        print(f"{nm:>16}: min {a[:, i].min():8.2f} med {np.median(a[:, i]):8.2f} max {a[:, i].max():8.2f}")
    b = (t2[k, :n2] - t0) / 1e3
    for nm, i in names2:
        print(f"{nm:>16}: min {b[:, i].min():8.2f} med {np.median(b[:, i]):8.2f} max {b[:, i].max():8.2f}")
