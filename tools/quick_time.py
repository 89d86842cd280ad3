"""Quick device timing of the execute path (and K1 alone) for a few plans (development aid).

Times K consecutive executes captured in a CUDA graph, inputs rotated over 2 buffers.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_12559_b200 as pft  # noqa: E402


def graph_time(fn, reps, stream):
    with torch.cuda.stream(stream):
        for i in range(3):
            fn(i)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(reps):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def time_plan(N, M, mu, p, p2=0, stages=0, reps=200, label="", k2_mode=0, k2_ctas=0, fuse=False, red=0):
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    d = pft.DevicePlan(plan, p2=p2, k1_stages=stages, k2_mode=k2_mode, k2_ctas=k2_ctas, fuse=fuse, reducers=red)
    bufs = [torch.empty(N, dtype=torch.complex128, device="cuda") for _ in range(2)]
    for i, b in enumerate(bufs):
        pft.generate_signal_device(b.data_ptr(), pft.KIND_UNIFORM, 1 + i, N)
    out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
    Y = torch.empty(plan.p * plan.r, dtype=torch.complex128, device="cuda")
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    ms = graph_time(lambda i: d.execute_ptr(bufs[i % 2].data_ptr(), out.data_ptr(), stream=sp), reps, s)
    k1 = graph_time(lambda i: d.execute_partial_ptr(bufs[i % 2].data_ptr(), Y.data_ptr(), stream=sp), reps, s)
    # K2 alone (finalize of the same slab), and a 2-stream pipeline of independent transforms
    k2 = graph_time(lambda i: d.finalize_ptr(Y.data_ptr(), out.data_ptr(), stream=sp), reps, s)
    s2 = torch.cuda.Stream()
    ws = [torch.zeros(-(-d.workspace_bytes(1) // 16), dtype=torch.complex128, device="cuda") for _ in range(2)]
    outs = [torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda") for _ in range(2)]
    ev = [torch.cuda.Event() for _ in range(2)]

    def two_stream(i):
        # fork s2 from s at the start of a pair, join back at the end (graph-capturable)
        if i % 2 == 0:
            ev[0].record(s)
            s2.wait_event(ev[0])
        st = s if i % 2 == 0 else s2
        d.execute_ptr(bufs[i % 2].data_ptr(), outs[i % 2].data_ptr(), d_ws=ws[i % 2].data_ptr(),
                      stream=st.cuda_stream)
        if i % 2 == 1:
            ev[1].record(s2)
            s.wait_event(ev[1])
    ms2 = graph_time(two_stream, reps, s)

    # split: the K1 chain stays on stream s (PDL back-to-back), each transform's K2 runs on s2
    evk = [torch.cuda.Event() for _ in range(reps + 8)]
    evf = [torch.cuda.Event() for _ in range(reps + 8)]

    def split(i):
        if i >= 2:
            s.wait_event(evf[i - 2])  # K2(i-2) done reading workspace i % 2
        d.execute_partial_ptr(bufs[i % 2].data_ptr(), ws[i % 2].data_ptr(), stream=s.cuda_stream)
        evk[i].record(s)
        s2.wait_event(evk[i])
        d.finalize_ptr(ws[i % 2].data_ptr(), outs[i % 2].data_ptr(), stream=s2.cuda_stream)
        evf[i].record(s2)
        if i == reps - 1 or i == 2:
            s.wait_event(evf[i])
    ms3 = graph_time(split, reps, s)
    print(json.dumps({"label": label, "k2_us": round(k2 * 1e3, 2), "pipelined_us": round(ms2 * 1e3, 2), "split_us": round(ms3 * 1e3, 2), "N": N, "M": M, "p": plan.p, "q": plan.q, "r": plan.r, "P1": d.P1,
                      "P2": d.P2, "stages": stages, "us": round(ms * 1e3, 2), "k1_us": round(k1 * 1e3, 2),
                      "GB/s": round(16 * N / (ms * 1e-3) / 1e9, 1),
                      "k1_GB/s": round(16 * N / (k1 * 1e-3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    import os
    which = os.environ.get("QT", "main")
    if which == "split":
        for rep in range(2):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b", reps=500)
            time_plan(6220800, 1000, -12345, 62208, label="C4", reps=500)
            time_plan(2 ** 20, 64, 0, None, label="C1", reps=500)
    if which == "sum":
        for rep in range(2):
            for mode in (5, 1):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b k2_mode={mode}", k2_mode=mode, reps=500)
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label=f"C2b p=2^14 k2_mode={mode}", k2_mode=mode, reps=500)
                time_plan(6220800, 1000, -12345, 62208, label=f"C4 k2_mode={mode}", k2_mode=mode, reps=500)
                time_plan(2 ** 20, 64, 0, None, label=f"C1 k2_mode={mode}", k2_mode=mode, reps=500)
    if which == "sumc":
        for rep in range(2):
            for kc in (64, 148, 296, 592):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b sum k2_ctas={kc}", k2_mode=5, k2_ctas=kc, reps=500)
                time_plan(6220800, 1000, -12345, 62208, label=f"C4 sum k2_ctas={kc}", k2_mode=5, k2_ctas=kc, reps=500)
            for st in ():
                for kc in (0, 16):
                    time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b sum st={st} k2_ctas={kc}", k2_mode=5,
                              k2_ctas=kc, stages=st, reps=500)
    if which == "sumq":
        for rep in range(2):
            for red in (0, 32, 128):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b sum red={red}", k2_mode=5, red=red, reps=500)
                time_plan(6220800, 1000, -12345, 62208, label=f"C4 sum red={red}", k2_mode=5, red=red, reps=500)
                time_plan(2 ** 20, 64, 0, None, label=f"C1 sum red={red}", k2_mode=5, red=red, reps=500)
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b fft", k2_mode=1, reps=500)
            time_plan(6220800, 1000, -12345, 62208, label="C4 fft", k2_mode=1, reps=500)
            time_plan(2 ** 20, 64, 0, None, label="C1 l2", k2_mode=4, reps=500)
    if which == "sumv":
        for rep in range(2):
            for red in (0, 16, 64):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b sum red={red}", k2_mode=5, red=red, reps=500)
                time_plan(6220800, 1000, -12345, 62208, label=f"C4 sum red={red}", k2_mode=5, red=red, reps=500)
                time_plan(2 ** 20, 64, 0, None, label=f"C1 sum red={red}", k2_mode=5, red=red, reps=500)
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b fft", k2_mode=1, reps=500)
    if which == "sum1":
        for rep in range(2):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b sum", reps=500)
            time_plan(6220800, 1000, -12345, 62208, label="C4 sum", reps=500)
    if which == "redsweep":
        for rep in range(2):
            for red in (0, 20, 24, 40, 48):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b sum red={red}", red=red, reps=500)
                time_plan(6220800, 1000, -12345, 62208, label=f"C4 sum red={red}", red=red, reps=500)
    if which == "psweep":
        for rep in range(2):
            for pp, p2 in ((2 ** 15, 256), (2 ** 15, 512), (2 ** 16, 256), (2 ** 16, 512), (2 ** 14, 256), (2 ** 14, 128)):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, pp, p2=p2, label=f"C2b p={pp} P2={p2}", reps=500)
            for pp, p2 in ((62208, 256), (62208, 243), (27648, 256), (62208, 324)):
                time_plan(6220800, 1000, -12345, pp, p2=p2, label=f"C4 p={pp} P2={p2}", reps=500)
    if which == "psweep2":
        for rep in range(2):
            for pp, p2 in ((2 ** 14, 128), (2 ** 15, 128), (2 ** 16, 128), (2 ** 13, 128), (2 ** 14, 64), (2 ** 15, 64)):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, pp, p2=p2, label=f"C2b p={pp} P2={p2}", reps=500)
            for pp, p2 in ((27648, 128), (27648, 144), (27648, 216), (62208, 128), (62208, 144), (62208, 162)):
                time_plan(6220800, 1000, -12345, pp, p2=p2, label=f"C4 p={pp} P2={p2}", reps=500)
            for pp, p2 in ((16384, 128), (16384, 64), (8192, 128), (4096, 64)):
                time_plan(2 ** 20, 64, 0, pp, p2=p2, label=f"C1 p={pp} P2={p2}", reps=500)
    if which == "dev":
        for rep in range(2):
            for pp in (2 ** 14, 2 ** 15):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, pp, label=f"C2b p={pp}", reps=500)
            for pp in (2048, 4096, 16384, 65536):
                time_plan(2 ** 24, 2 ** 6, 2 ** 22, pp, label=f"C2a p={pp}", reps=500)
            for pp in (32768, 65536, 262144):
                time_plan(2 ** 24, 2 ** 14, 2 ** 22, pp, label=f"C2c p={pp}", reps=300)
            for pp in (16200, 27648, 62208, 10368):
                time_plan(6220800, 1000, -12345, pp, label=f"C4 p={pp}", reps=500)
            for pp in (1024, 2048, 4096):
                time_plan(2 ** 20, 64, 0, pp, label=f"C1 p={pp}", reps=500)
    if which == "k1ab":
        for rep in range(2):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label="C2b p=2^14", reps=500)
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 13, label="C2b p=2^13 r=10", reps=500)
            time_plan(6220800, 1000, -12345, 15360, label="C4 p=15360", reps=500)
            time_plan(2 ** 24, 2 ** 14, 2 ** 22, 2 ** 15, label="C2c p=2^15 r=14", reps=200)
            time_plan(2 ** 20, 64, 0, 2048, label="C1 p=2048", reps=500)
    if which == "fuse":
        for rep in range(2):
            for fz in (True, False):
                time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b fuse={fz}", fuse=fz, reps=500)
                time_plan(6220800, 1000, -12345, 62208, label=f"C4 fuse={fz}", fuse=fz, reps=500)
    if which == "rep":
        for _ in range(3):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b", reps=1000)
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label="C2b p=2^14", reps=1000)
    if which == "l2":
        for mode in (4, 1):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b k2_mode={mode}", k2_mode=mode)
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label=f"C2b p=2^14 k2_mode={mode}", k2_mode=mode)
            time_plan(6220800, 1000, -12345, 62208, label=f"C4 k2_mode={mode}", k2_mode=mode)
            time_plan(2 ** 20, 64, 0, None, label=f"C1 k2_mode={mode}", k2_mode=mode)
    if which == "k2c":
        for kc in (16, 32, 64, 128):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b k2_ctas={kc}", k2_ctas=kc)
        time_plan(6220800, 1000, -12345, 62208, label="C4")
        time_plan(2 ** 24, 2 ** 14, 2 ** 22, 2 ** 16, label="C2c p=2^16")
    if which == "k2":
        for mode in (1, 2, 3):
            time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label=f"C2b k2_mode={mode}", k2_mode=mode)
            time_plan(2 ** 24, 2 ** 14, 2 ** 22, 2 ** 16, label=f"C2c k2_mode={mode}", k2_mode=mode)
            time_plan(6220800, 1000, -12345, 62208, label=f"C4 k2_mode={mode}", k2_mode=mode)
    if which == "k1":
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b p=2^15")
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label="C2b p=2^14")
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 16, label="C2b p=2^16")
        time_plan(2 ** 24, 0, 2 ** 22, 2 ** 15, label="C2b-shape r=1")
    if which == "main":
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 15, label="C2b p=2^15")
        time_plan(2 ** 24, 0, 2 ** 22, 2 ** 15, label="C2b-shape r=1 (memory-pattern ceiling)")
        time_plan(2 ** 24, 0, 2 ** 22, 2 ** 14, label="p=2^14 r=1")
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 14, label="C2b p=2^14")
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 13, label="C2b p=2^13")
        time_plan(2 ** 24, 2 ** 10, 2 ** 22, 2 ** 16, label="C2b p=2^16")
        time_plan(2 ** 24, 2 ** 6, 2 ** 22, None, label="C2a")
        time_plan(2 ** 24, 2 ** 14, 2 ** 22, 2 ** 16, label="C2c p=2^16")
        time_plan(2 ** 20, 64, 0, None, label="C1")
        time_plan(6220800, 1000, -12345, 62208, label="C4")
