"""Same-box A/B of the execute path between library builds (PFT_LIB; development aid).

    PFT_LIB=variants/lib_old.so python tools/ab_exec.py
Times 1000 executes captured in one CUDA graph per config (C2b p = 2^14, C4 p = 11520, C1
p = 2048), inputs rotated over buffers totalling > 2x L2.
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402

CFG = {k: v for k, v in {"c2b": (2 ** 24, 2 ** 10, 2 ** 22, 16384), "c4": (6220800, 1000, -12345, 11520), "c1": (2 ** 20, 64, 0, 2048)}.items() if k in os.environ.get("AB_CFGS", "c2b c4 c1").split()}
lib = os.environ.get("PFT_LIB", "main")
for name, (N, M, mu, p) in CFG.items():
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    d = pft.DevicePlan(plan)
    nb = max(2, -(-2 * 126 * 2 ** 20 // (16 * N)))
    bufs = [torch.empty(N, dtype=torch.complex128, device="cuda") for _ in range(nb)]
    for i, b in enumerate(bufs):
        pft.generate_signal_device(b.data_ptr(), pft.KIND_UNIFORM, 1 + i, N)
    out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
    s = torch.cuda.Stream()
    reps = 1000
    with torch.cuda.stream(s):
        for i in range(5):
            d.execute_ptr(bufs[i % nb].data_ptr(), out.data_ptr(), stream=s.cuda_stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                d.execute_ptr(bufs[i % nb].data_ptr(), out.data_ptr(), stream=s.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{lib} {name} {e0.elapsed_time(e1) / reps * 1e3:.2f} us")
