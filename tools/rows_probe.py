import sys, os, json
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2008_12559_b200 as pft
N1, N2, M, p = 4096, 4096, 64, 64
plan = pft.build_plan(N2, M, 0, p, 1e-12)
d = pft.DevicePlan(plan, batch_hint=N1)
x = torch.randn(N1 * N2, dtype=torch.complex128, device="cuda")
x2 = torch.randn(N1 * N2, dtype=torch.complex128, device="cuda")
out = torch.empty(N1 * (2 * M + 1), dtype=torch.complex128, device="cuda")
ws = torch.zeros(-(-d.workspace_bytes(N1) // 16), dtype=torch.complex128, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for i in range(3):
        d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=N1, in_stride=N2, d_ws=ws.data_ptr(), stream=st.cuda_stream, overlap=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(20):
            d.execute_ptr((x if i % 2 else x2).data_ptr(), out.data_ptr(), batch=N1, in_stride=N2, d_ws=ws.data_ptr(), stream=st.cuda_stream, overlap=True)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); g.replay(); e1.record(st)
torch.cuda.synchronize()
print(os.environ.get("PFT_DBG_PHASE", "full"), "rows pass us per execute:", e0.elapsed_time(e1) / 20 * 1e3, "r", plan.r, "g", d.signals_per_cta(N1))
