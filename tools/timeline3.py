"""Steady-state K1/K2 timeline of a PDL chain of executes (PFT_TIMELINE build; development aid).

    PFT_LIB=variants/lib_tl.so python tools/timeline3.py [c2b|c4] [k2_mode] [k2_ctas]

Runs 40 executes back to back on one stream (no graph, so each launch gets its own sequence
number), then prints, for the last 3 executes, per-phase min/median/max stamps relative to
the first K1 CTA start of the earliest of them.
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2b"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
kc = int(sys.argv[3]) if len(sys.argv) > 3 else 0
red = int(sys.argv[4]) if len(sys.argv) > 4 else 0
N, M, mu, p = {"c2b": (2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15), "c4": (6220800, 1000, -12345, 62208)}[cfg]
plan = pft.build_plan(N, M, mu, p, 1e-12)
d = pft.DevicePlan(plan, k2_mode=mode, k2_ctas=kc, reducers=red)
xs = [torch.empty(N, dtype=torch.complex128, device="cuda") for _ in range(2)]
for i, x in enumerate(xs):
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 1 + i, N)
out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
torch.cuda.synchronize()
n = 40
for i in range(n):
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
n2 = kc if kc else (2 * M + 1 + 7) // 8
t0 = t1[order[1], :n1, 0].min()
for k in order[1:]:
    a = (t1[k, :n1] - t0) / 1e3
    print(f"--- execute slot {k}")
    for nm, i in [("K1 start", 0), ("K1 first data", 1), ("K1 loop end", 2), ("K1 fft end", 3), ("K1 tail end", 4),
                  ("K1 end", 5)]:
        if a[:, i].min() < -1e6:
            continue
        print(f"{nm:>16}: min {a[:, i].min():7.2f} med {np.median(a[:, i]):7.2f} max {a[:, i].max():7.2f}")
    nz = t2[k, :n2]
    if len(nz):
        b = (nz - t0) / 1e3
        for nm, i in [("K2 start", 0), ("K2 after wait", 2), ("K2 end", 5)]:
            if b[:, i].min() < -1e6:
                continue
            print(f"{nm:>16}: min {b[:, i].min():7.2f} med {np.median(b[:, i]):7.2f} max {b[:, i].max():7.2f}")
