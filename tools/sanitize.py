"""Small executes of every device form, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  Each form runs 3 times on one workspace (re-armed counters, PDL overlap where the
form chains) and is checked against the CPU oracle; exits non-zero on a parity failure.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402

FORMS = [
    # (label, N, M, mu, p, batch, DevicePlan options)
    ("sum tail, many classes", 2 ** 18, 200, 33, 2 ** 11, 1, dict(second_pass="sum")),
    ("sum tail, fast reduction (tensor cores)", 2 ** 14, 64, 0, 2 ** 8, 3, dict(batch_hint=64)),
    ("sum tail, one class per signal", 4096, 64, 5, 64, 3, dict(batch_hint=64)),
    ("K2 grid (FFT form)", 2 ** 18, 2 ** 11, -7, 2 ** 12, 1, dict(second_pass="k2-fft", k2_at="grid")),
    ("K2 dot form", 2 ** 18, 2 ** 9, 7, 2 ** 12, 1, dict(second_pass="k2-dot")),
    ("K2 direct form", 2 ** 18, 2 ** 9, 7, 2 ** 12, 1, dict(second_pass="k2-direct")),
    ("K2 L2 form", 2 ** 18, 2 ** 6, 7, 2 ** 12, 1, dict(second_pass="k2-l2")),
    ("K2 tail (last arrivals)", 2 ** 18, 2 ** 9, -5, 2 ** 12, 1, dict(second_pass="k2-fft", k2_at="tail")),
    ("fused K2 (grid barrier)", 2 ** 16, 128, 77, 2 ** 12, 2, dict(second_pass="k2-fft", k2_at="fused")),
    ("K2 workers inside K1's grid (chained)", 2 ** 20, 2 ** 11, -7, 2 ** 13, 1, dict(second_pass="k2-fft", k2_at="tail")),
    ("K2 workers, 3 workers, odd r", 2 ** 20, 1500, 0, 2 ** 13, 1, dict(second_pass="k2-fft", k2_at="tail", tail_ctas=3)),
    ("ring K2 kernel, 6 CTAs looping over m1", 2 ** 20, 2 ** 11, -7, 2 ** 13, 1, dict(second_pass="k2-fft", k2_grid_ctas=6)),
    ("ring K2 kernel, one CTA per m1", 2 ** 20, 2 ** 11, -7, 2 ** 13, 1, dict(second_pass="k2-fft", k2_at="grid")),
]


def run_form(label, N, M, mu, p, batch, kw) -> float:
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    d = pft.DevicePlan(plan, **kw)
    a = pft.generate_signal(pft.KIND_UNIFORM, 7, N * batch)
    x = torch.from_numpy(a).cuda()
    ws = torch.zeros(-(-d.workspace_bytes(batch) // 16), dtype=torch.complex128, device="cuda")
    outs = [torch.empty(batch * (2 * M + 1), dtype=torch.complex128, device="cuda") for _ in range(3)]
    s = torch.cuda.current_stream().cuda_stream
    for i in range(3):  # chained with PDL overlap (distinct outputs, the input is never an output)
        d.execute_ptr(x.data_ptr(), outs[i].data_ptr(), batch=batch, in_stride=N, d_ws=ws.data_ptr(), stream=s,
                      overlap=True)
    torch.cuda.synchronize()
    if d.status(d_ws=ws.data_ptr()) != 0:
        return float("inf")
    worst = 0.0
    for i in range(3):
        got = outs[i].cpu().numpy().reshape(batch, 2 * M + 1)
        for b in range(batch):
            ref = oracle.execute(plan, a[b * N:(b + 1) * N])
            worst = max(worst, float(np.linalg.norm(got[b] - ref) / np.linalg.norm(ref)))
    return worst


def run_2d() -> float:
    plan = pft.build_plan_2d(256, 256, 8, 8, 3, -5)
    a = np.random.default_rng(3).random((256, 256)).astype(np.complex128)
    got = pft.execute_2d(plan, a).values
    ref = oracle.execute_2d(plan.plan1, plan.plan2, a)
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


def run_sharded() -> float:
    plan = pft.build_plan(2 ** 18, 2 ** 9, 11, 2 ** 12, 1e-12)
    d = pft.DevicePlan(plan)
    a = pft.generate_signal(pft.KIND_UNIFORM, 5, plan.N)
    slab = torch.zeros(plan.p * plan.r, dtype=torch.complex128, device="cuda")
    part = torch.empty_like(slab)
    for rank in range(2):
        local = torch.from_numpy(np.ascontiguousarray(pft.shard_gather(a, plan.p, plan.q, 2, rank))).cuda()
        d.execute_partial_ptr(local.data_ptr(), part.data_ptr(), world=2, rank=rank)
        torch.cuda.synchronize()
        slab += part
    out = torch.empty(2 * plan.M + 1, dtype=torch.complex128, device="cuda")
    d.finalize_ptr(slab.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    ref = oracle.execute(plan, a)
    return float(np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref))


def main() -> int:
    bad = 0
    for f in FORMS:
        e = run_form(*f)
        print(f"{f[0]:50s} rel_l2 {e:.2e}", flush=True)
        bad += e > 1e-11
    for label, fn in (("2-D (two batched passes + transposes)", run_2d), ("sharded partial + finalize", run_sharded)):
        e = fn()
        print(f"{label:50s} rel_l2 {e:.2e}", flush=True)
        bad += e > 1e-11
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
