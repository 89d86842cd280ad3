"""Stage-isolating parity check: K1's partial slab Y vs a numpy model, then K2."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402


def check(N, M, mu, p, p2=0, seed=1):
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    d = pft.DevicePlan(plan, p2=p2)
    P1, P2, r, q = d.P1, d.P2, plan.r, plan.q
    a = pft.generate_signal(pft.KIND_UNIFORM, seed, N)
    x = torch.from_numpy(a).cuda()
    Y = torch.zeros(P1 * P2 * r, dtype=torch.complex128, device="cuda")
    d.execute_partial_ptr(x.data_ptr(), Y.data_ptr())
    out = torch.zeros(2 * M + 1, dtype=torch.complex128, device="cuda")
    d.finalize_ptr(Y.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    Yg = Y.cpu().numpy().reshape(P1, P2, r)
    Cm = oracle.matmul(a.reshape(plan.p, q), plan.B)        # p x r
    Cr = Cm.reshape(P1, P2, r)                              # [k1][c][j]
    Ym = np.fft.fft(Cr, axis=0)                             # over k1 -> [m1][c][j]
    err = np.abs(Yg - Ym)
    relY = np.linalg.norm(Yg - Ym) / np.linalg.norm(Ym)
    bad = np.argwhere(err > 1e-9 * np.abs(Ym).max())
    ref = oracle.execute(plan, a)
    relO = np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref)
    global LAST
    LAST = sorted(set(int(x) for x in bad[:, 1])) if len(bad) else []
    print(f"N={N} M={M} mu={mu} p={plan.p} q={q} r={r} P1={P1} P2={P2}: relY={relY:.3e} relOut={relO:.3e} "
          f"bad={len(bad)} first={bad[:5].tolist()}", flush=True)


LAST = []

if __name__ == "__main__":
    for rep in range(3):
        check(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15)
        print("  bad residues:", LAST)
    check(2 ** 22, 2 ** 10, 2 ** 20, 2 ** 15, p2=256)   # q = 128
    check(2 ** 23, 2 ** 10, 2 ** 21, 2 ** 15, p2=256)   # q = 256
    check(2 ** 24, 2 ** 10, 0, 2 ** 15, p2=256)         # mu = 0
    check(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 16, p2=128)   # P1 = 512? (r=6 -> 48KB)
    check(2 ** 25, 2 ** 10, 0, 2 ** 15, p2=256)         # q = 1024
    check(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, p2=128)   # q = 1024, 128 CTAs
