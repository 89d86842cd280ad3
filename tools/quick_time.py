"""Device timing of the execute path for A/B comparisons on one box (development aid).

    python tools/quick_time.py c2b c2c c4 [--opt k=v ...] [--json]

For each BASELINE config (bench.py's CONFIGS, p from --p or the bench's autotuned picks) it
times K executes captured in one CUDA graph with PFT_EXEC_OVERLAP_PREVIOUS (chained throughput)
and the median of single isolated executes, inputs rotated over buffers > 2x L2, and checks the
last output against the CPU oracle.  --opt passes DevicePlan keyword options (second_pass=sum,
k2_at=grid, tail_ctas=8, p2=256, ...); several --variant 'k=v,k=v' run side by side.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402

PICKS = {"c1": 2048, "c2a": 2048, "c2b": 16384, "c2c": 32768, "c3": 256, "c4": 10368, "c5": 524288}


def parse_opts(text: str) -> dict:
    out = {}
    for kv in filter(None, (text or "").split(",")):
        k, v = kv.split("=")
        out[k] = int(v) if v.lstrip("-").isdigit() else v
        if k == "split":
            out[k] = bool(out[k])
    return out


def run(cfg: str, p: int, opts: dict, reps: int, check: bool, streams: int = 1) -> dict:
    N, M, mu, _, kind, _ = bench.CONFIGS[cfg]
    B = bench.BATCH.get(cfg, 1)
    W = 2 * M + 1
    nbuf = 1 if (B > 1 or 16 * N >= 16 * bench.L2_BYTES) else max(4, -(-8 * bench.L2_BYTES // (16 * N)))
    bufs = [torch.empty(N * B, dtype=torch.complex128, device="cuda") for _ in range(nbuf)]
    for i, b in enumerate(bufs):
        bench.make_input_device(pft, b, N * B, mu, M, bench.SEEDS[cfg], kind, offset=(0 if B > 1 else i * N), N=N)
    plan = pft.build_plan(N, M, mu, p, bench.EPS)
    d = pft.DevicePlan(plan, batch_hint=B, **opts)
    ws = torch.zeros(-(-d.workspace_bytes(B) // 16), dtype=torch.complex128, device="cuda")
    out = torch.empty(W * B, dtype=torch.complex128, device="cuda")
    st = torch.cuda.Stream()
    # streams > 1: free-running PDL chains, one per stream, each with its own workspace and output
    # (forked once at the start of the graph, joined once at its end); execute i runs on chain i % streams
    sts = [st] + [torch.cuda.Stream() for _ in range(streams - 1)]
    wss = [ws] + [torch.zeros_like(ws) for _ in range(streams - 1)]
    outs = [out] + [torch.empty_like(out) for _ in range(streams - 1)]

    def ex(i, overlap=True, k=0):
        d.execute_ptr(bufs[i % nbuf].data_ptr(), outs[k].data_ptr(), batch=B, in_stride=N, d_ws=wss[k].data_ptr(),
                      stream=sts[k].cuda_stream, overlap=overlap)

    with torch.cuda.stream(st):
        for i in range(3):
            ex(i)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            if streams > 1:
                fork = torch.cuda.Event()
                fork.record(st)
                for s2 in sts[1:]:
                    s2.wait_event(fork)
            for i in range(reps):
                ex(i, k=i % streams)
            for s2 in sts[1:]:
                j = torch.cuda.Event()
                j.record(s2)
                st.wait_event(j)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    chained = e0.elapsed_time(e1) / reps * 1e3
    out_chained = outs[(reps - 1) % streams][:W * min(B, 4)].clone()  # the last execute (input bufs[(reps - 1) % nbuf])
    with torch.cuda.stream(st):  # serialized executes (no overlap flag): device time per execute
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=st):
            for i in range(min(reps, 50)):
                ex(i + 1, overlap=False)
        g2.replay()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        g2.replay()
        a1.record(st)
    torch.cuda.synchronize()
    iso = [a0.elapsed_time(a1) * 1e3 / min(reps, 50)]
    res = {"cfg": cfg, "p": p, "opts": opts, "streams": streams, "P1": d.P1, "P2": d.P2, "tail": d.tail_kind(),
           "chained_us": chained, "isolated_us": float(np.median(iso)),
           "frac": 16 * N * B / (chained * 1e-6) / 1e9 / bench.measured_hbm_peak()[0]}
    if check:
        import oracle
        src = bufs[(reps - 1) % nbuf]
        ex(reps - 1, overlap=False)
        torch.cuda.synchronize()
        nb = min(B, 4)
        got = out[:W * nb].cpu().numpy().reshape(nb, W)
        src_c = bufs[(reps - 1) % nbuf]
        got_c = out_chained.cpu().numpy().reshape(min(B, 4), W)
        res["rel_l2_chained"] = max(float(np.linalg.norm(got_c[b] - (r := oracle.execute(plan, src_c[b * N:(b + 1) * N].cpu().numpy())))
                                          / np.linalg.norm(r)) for b in range(min(B, 4)))
        res["rel_l2"] = max(float(np.linalg.norm(got[b] - (r := oracle.execute(plan, src[b * N:(b + 1) * N].cpu().numpy())))
                                  / np.linalg.norm(r)) for b in range(nb))
    res["status"] = d.status(d_ws=ws.data_ptr())
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--variant", action="append", default=None, help="DevicePlan options k=v,k=v")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--streams", type=int, default=1, help="free-running PDL chains (streams, workspaces, outputs)")
    a = ap.parse_args()
    variants = a.variant or [""]
    for cfg in a.configs:
        for v in variants:
            reps = a.reps if cfg not in ("c3", "c5") else 10
            r = run(cfg, a.p or PICKS[cfg], parse_opts(v), reps, not a.no_check, a.streams)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
