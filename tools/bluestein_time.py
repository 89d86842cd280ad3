"""Timing of the second pass over a P2 with a large prime factor: Bluestein (chirp-z) vs the
dot and direct forms on the same plan.  One JSON line per case."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402

CASES = [  # (N, M, mu, p, P2)
    (2 ** 16 * 2039, 2 ** 14, 0, 2039 * 2 ** 7, 2039),
    (2 ** 16 * 1021, 2 ** 14, 0, 1021 * 2 ** 7, 1021),
    (2 ** 10 * 1021, 2 ** 12, 77, 1021 * 2 ** 7, 1021),
]
for N, M, mu, p, P2 in CASES:
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    x = torch.empty(N, dtype=torch.complex128, device="cuda")
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 3, N)
    out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
    ref = oracle.execute(plan, x.cpu().numpy()) if N <= 2 ** 24 else None
    for form in ("k2-bluestein", "k2-dot", "k2-direct"):
        try:
            d = pft.DevicePlan(plan, p2=P2, second_pass=form)
        except Exception as e:
            print(json.dumps({"N": N, "P2": P2, "form": form, "error": str(e)}), flush=True)
            continue
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                d.execute_ptr(x.data_ptr(), out.data_ptr(), stream=st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(20):
                d.execute_ptr(x.data_ptr(), out.data_ptr(), stream=st.cuda_stream)
            e1.record(st)
        torch.cuda.synchronize()
        rel = None
        if ref is not None:
            g = out.cpu().numpy()
            rel = float(np.linalg.norm(g - ref) / np.linalg.norm(ref))
        print(json.dumps({"N": N, "M": M, "p": p, "r": plan.r, "P1": d.P1, "P2": d.P2, "form": d.second_pass,
                          "us_per_execute": e0.elapsed_time(e1) / 20 * 1e3, "rel_l2_vs_oracle": rel}), flush=True)
        d.close()
