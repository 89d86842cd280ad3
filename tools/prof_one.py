"""Run a few executes of one config with given DevicePlan options (for ncu captures).

    python tools/prof_one.py c2b [k=v,...] [reps]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402
from tools.quick_time import PICKS, parse_opts  # noqa: E402

cfg = sys.argv[1]
opts = parse_opts(sys.argv[2] if len(sys.argv) > 2 else "")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
N, M, mu, _, kind, _ = bench.CONFIGS[cfg]
B = bench.BATCH.get(cfg, 1)
x = torch.empty(N * B, dtype=torch.complex128, device="cuda")
bench.make_input_device(pft, x, N * B, mu, M, bench.SEEDS[cfg], kind, N=N)
plan = pft.build_plan(N, M, mu, PICKS[cfg], bench.EPS)
d = pft.DevicePlan(plan, batch_hint=B, **opts)
ws = torch.zeros(-(-d.workspace_bytes(B) // 16), dtype=torch.complex128, device="cuda")
out = torch.empty((2 * M + 1) * B, dtype=torch.complex128, device="cuda")
for _ in range(reps):
    d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=B, in_stride=N, d_ws=ws.data_ptr())
torch.cuda.synchronize()
print(cfg, opts, d.P1, d.P2, d.tail_kind(), "status", d.status(d_ws=ws.data_ptr()))
