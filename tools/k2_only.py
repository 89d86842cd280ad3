"""Run K2 (finalize) alone repeatedly for profiling (development aid)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
plan = pft.build_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, 1e-12)
d = pft.DevicePlan(plan, k2_mode=mode)
x = torch.empty(plan.N, dtype=torch.complex128, device="cuda")
pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 1, plan.N)
Y = torch.empty(plan.p * plan.r, dtype=torch.complex128, device="cuda")
out = torch.empty(2 * plan.M + 1, dtype=torch.complex128, device="cuda")
d.execute_partial_ptr(x.data_ptr(), Y.data_ptr())
for _ in range(10):
    d.finalize_ptr(Y.data_ptr(), out.data_ptr())
torch.cuda.synchronize()
print("ok")
