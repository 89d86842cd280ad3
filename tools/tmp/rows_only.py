import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2008_12559_b200 as pft
N1, N2, M, p = 4096, 4096, 64, 64
plan = pft.build_plan(N2, M, 0, p, 1e-12)
d = pft.DevicePlan(plan, batch_hint=N1)
x = torch.randn(N1 * N2, dtype=torch.complex128, device="cuda")
out = torch.empty(N1 * (2 * M + 1), dtype=torch.complex128, device="cuda")
ws = torch.zeros(-(-d.workspace_bytes(N1) // 16), dtype=torch.complex128, device="cuda")
for i in range(8):
    d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=N1, in_stride=N2, d_ws=ws.data_ptr())
torch.cuda.synchronize()
print("signals per CTA", d.signals_per_cta(N1), "r", plan.r)
