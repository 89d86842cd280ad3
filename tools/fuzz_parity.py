"""Randomised parity sweep on the GPU (development aid): random shapes (N = 2^a 3^b 5^c 7^d, M, mu, a
device-model or random divisor p, batch) through the default device plan, isolated and as a PDL
chain, each output against the CPU oracle on the same plan.  Prints one line per case; exit 1 on
any relative l2 > 1e-11 or non-zero status."""
import random
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402


def rand_n(rng, lo, hi):
    while True:
        n = 2 ** rng.randint(4, 20) * 3 ** rng.randint(0, 3) * 5 ** rng.randint(0, 2) * 7 ** rng.randint(0, 1)
        if lo <= n <= hi:
            return n


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cases = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    pow2 = len(sys.argv) > 3 and sys.argv[3] == "pow2"  # power-of-two N, many bins: the K2 worker / ring forms
    rng = random.Random(seed)
    bad = 0
    for i in range(cases):
        big_batch = rng.random() < 0.3 and not pow2
        N = rand_n(rng, 2 ** 8, 2 ** 13) if big_batch else rand_n(rng, 2 ** 10, 2 ** 22)
        M = rng.randint(0, max(0, min(N // 4, 3000)))
        if pow2:
            N = 2 ** rng.randint(16, 23)
            M = rng.randint(N // 4096, N // 512)
        mu = rng.choice([0, rng.randint(-N, 2 * N)])
        divs = [p for p in pft.divisors(N) if p >= max(2 * M, 1) and N // p >= 2] if hasattr(pft, "divisors") else []
        try:
            if divs and rng.random() < 0.5:
                p = rng.choice(divs)
            else:
                p = pft.select_divisor_device(N, M)[0]
            plan = pft.build_plan(N, M, mu, p, 1e-12)
            batch = rng.choice([700, 1301, 2402]) if big_batch else rng.choice([1, 1, 2, 3])
            d = pft.DevicePlan(plan, batch_hint=batch)
        except Exception as e:  # infeasible shape for the planner / device plan
            print(f"[{i}] N={N} M={M} mu={mu}: skipped ({str(e)[:60]})", flush=True)
            continue
        W = 2 * M + 1
        a = pft.generate_signal(pft.KIND_NORMAL, 100 + i, N * batch)
        x = torch.from_numpy(a).cuda()
        ws = torch.zeros(-(-d.workspace_bytes(batch) // 16), dtype=torch.complex128, device="cuda")
        outs = [torch.full((batch * W,), np.nan, dtype=torch.complex128, device="cuda") for _ in range(3)]
        s = torch.cuda.current_stream().cuda_stream
        d.execute_ptr(x.data_ptr(), outs[0].data_ptr(), batch=batch, in_stride=N, d_ws=ws.data_ptr(), stream=s)
        for o in outs[1:]:
            d.execute_ptr(x.data_ptr(), o.data_ptr(), batch=batch, in_stride=N, d_ws=ws.data_ptr(), stream=s, overlap=True)
        torch.cuda.synchronize()
        st = d.status(d_ws=ws.data_ptr())
        worst = 0.0
        sig = sorted(set([0, batch - 1, batch // 2]))
        for b in sig:
            ref = oracle.execute(plan, a[b * N:(b + 1) * N])
            nr = np.linalg.norm(ref) or 1.0
            for o in outs:
                got = o.cpu().numpy().reshape(batch, W)[b]
                worst = max(worst, float(np.linalg.norm(got - ref) / nr))
        ok = worst <= 1e-11 and st == 0
        bad += not ok
        print(f"[{i}] N={N} M={M} mu={mu} p={plan.p} r={plan.r} batch={batch} P1xP2={d.P1}x{d.P2} "
              f"tail={d.tail_kind()[:10].replace(' ', '_')} g={d.signals_per_cta(batch)} rel_l2={worst:.2e} status={st} "
              f"{'ok' if ok else 'FAIL'}", flush=True)
    print(f"{bad} failures")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
