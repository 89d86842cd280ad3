"""2-D PFT: time each axis pass alone (batched 1-D executes) for several residue-class counts P2
(development aid for the device plans pft_execute_2d uses)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402


def time_pass(N, M, p, batch, p2, reps=50, spc=0):
    plan = pft.build_plan(N, M, 0, p, 1e-12)
    try:
        d = pft.DevicePlan(plan, p2=p2, batch_hint=batch, signals_per_cta=spc)
    except Exception as e:
        return {"N": N, "p": p, "batch": batch, "p2": p2, "error": str(e)[:80]}
    x = torch.empty(N * batch, dtype=torch.complex128, device="cuda")
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 5, N * batch)
    out = torch.empty((2 * M + 1) * batch, dtype=torch.complex128, device="cuda")
    ws = torch.zeros(-(-d.workspace_bytes(batch) // 16), dtype=torch.complex128, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=batch, in_stride=N, d_ws=ws.data_ptr(), stream=st.cuda_stream, overlap=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=batch, in_stride=N, d_ws=ws.data_ptr(), stream=st.cuda_stream, overlap=True)
        e1.record(st)
    torch.cuda.synchronize()
    return {"N": N, "M": M, "p": p, "r": plan.r, "batch": batch, "P1": d.P1, "P2": d.P2, "tail": d.tail_kind(), "spc": spc,
            "us": e0.elapsed_time(e1) / reps * 1e3}


for spc in (1, 2, 4, 8, 16):  # rows pass of 4096 x 4096, (64, 64): 4096 signals of 4096
    for p in (64, 128):
        print(json.dumps(time_pass(4096, 64, p, 4096, 1, reps=20, spc=spc)), flush=True)
for spc in (1, 2, 4):  # 1024 x 16384 rows pass (M2 = 256)
    print(json.dumps(time_pass(16384, 256, 512, 1024, 1, reps=20, spc=spc)), flush=True)
