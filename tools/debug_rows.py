"""Which rows of C are wrong in a bad residue class, and does the error look like a
stale/misplaced TMA stage?  (development aid)"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402

N, M, mu, p = 2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15
plan = pft.build_plan(N, M, mu, p, 1e-12)
d = pft.DevicePlan(plan)
P1, P2, r, q = d.P1, d.P2, plan.r, plan.q
a = pft.generate_signal(pft.KIND_UNIFORM, 1, N)
x = torch.from_numpy(a).cuda()
Y = torch.zeros(P1 * P2 * r, dtype=torch.complex128, device="cuda")
d.execute_partial_ptr(x.data_ptr(), 0, q, q, Y.data_ptr())
torch.cuda.synchronize()
Yg = Y.cpu().numpy().reshape(P1, P2, r)
Cg = np.fft.ifft(Yg, axis=0)  # [k1][c][j]
A = a.reshape(P1, P2, q)       # row k = c + P2 k1 -> A[k1][c][:]
Bm = plan.B                    # q x r
CH = 32
nch = q // CH
# per-chunk contributions contrib[k1][c][ch][j]
contrib = np.einsum("kcxl,lxj->kcxj", A.reshape(P1, P2, nch, CH), Bm.reshape(nch, CH, r).transpose(1, 0, 2))
Cr = contrib.sum(axis=2)
diff = Cg - Cr
badc = sorted(set(np.argwhere(np.abs(diff) > 1e-9)[:, 1].tolist()))
print("bad residues", badc)
for c in badc[:3]:
    rows = np.argwhere(np.abs(diff[:, c, 0]) > 1e-9)[:, 0]
    print(f"c={c}: bad rows k1={rows.tolist()}")
    for k1 in rows[:4]:
        dv = diff[k1, c]
        m = np.abs(dv[None, :] + contrib[k1, c]).sum(-1)   # missing chunk
        dbl = np.abs(dv[None, :] - contrib[k1, c]).sum(-1) # double-counted chunk
        # stale: chunk ch read the data of chunk ch-4 (previous use of the same stage)
        st = [np.abs(dv - (contrib[k1, c, ch - 4] - contrib[k1, c, ch])).sum() if ch >= 4 else 1e9 for ch in range(nch)]
        # partial: one row in the box read another row's chunk (same stage)
        print(f"   k1={k1}: |diff|={np.abs(dv).max():.3e} missing(ch={m.argmin()}): {m.min():.2e}  "
              f"double(ch={dbl.argmin()}): {dbl.min():.2e}  stale(ch={int(np.argmin(st))}): {min(st):.2e}")
