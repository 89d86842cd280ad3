#!/usr/bin/env python3
"""Benchmark of the PFT execute hot path (BASELINE.json metric: PFT transforms/sec and input
GB/s, fraction of the HBM roofline) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2b] [--impl ours|reference]

A "step" is one transform (one pass of transform.execute) over one
synthetic input already resident in HBM.  Default workload = BASELINE.json configs[1] at
M = 2^10 (the north-star "C2b": N = 2^24, mu = N/4, eps = 1e-12, 32 seeded tones + CN
noise).  Multi-GPU: one process per GPU (torchrun), each rank runs an independent replica
stream of transforms ("replicas only" for single transforms, weak scaling); the step time
is the max over ranks of the device time.  Prints ONE JSON line on rank 0.

--impl reference times the reference algorithm's CPU restatement (oracle/, the
reference ships no runnable implementation -- SURVEY.md §8(c)) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (N, M, mu, p, kind, description); p None: our arm autotunes p on the device
    # (pft_autotune_divisor), the reference arm uses SPEC's CPU cost model (select_divisor)
    "c1": (2 ** 20, 64, 0, None, "uniform", "BASELINE configs[0]: N=2^20, M=64, mu=0, U[-1,1] re/im"),
    "c2a": (2 ** 24, 2 ** 6, 2 ** 22, None, "sparse", "BASELINE configs[1]: N=2^24, M=2^6, mu=N/4, 32 tones + CN noise"),
    "c2b": (2 ** 24, 2 ** 10, 2 ** 22, None, "sparse", "BASELINE configs[1]: N=2^24, M=2^10, mu=N/4, 32 tones + CN noise"),
    "c2c": (2 ** 24, 2 ** 14, 2 ** 22, None, "sparse", "BASELINE configs[1]: N=2^24, M=2^14, mu=N/4, 32 tones + CN noise"),
    "c3": (2 ** 16, 256, 0, None, "uniform", "BASELINE configs[2]: 4096 signals x N=2^16, M=256, mu=0, U[-1,1] re/im"),
    "c4": (6220800, 1000, -12345, None, "normal", "BASELINE configs[3]: N=2^10 3^5 5^2, M=1000, mu=-12345, CN(0,1)"),
    "c5": (2 ** 30, 2 ** 12, 0, None, "uniform", "BASELINE configs[4]: N=2^30, M=2^12, mu=0, U[-1,1] re/im; "
                                                 "contraction-axis sharded over the GPUs"),
}
SHARDED = {"c5"}  # one transform split along the contraction axis when run on > 1 GPU
BATCH = {"c3": 4096}
SEEDS = {"c1": 1, "c2a": 2, "c2b": 2, "c2c": 2, "c3": 3, "c4": 4, "c5": 5}
EPS = 1e-12
L2_BYTES = 126 * 1024 * 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_hbm_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def committed_traffic(config):
    f = ROOT / "profiles" / "k1_dram_traffic.json"
    try:
        return json.loads(f.read_text()).get(config)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi style clocks/throttle sampling (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("NVML unavailable:", e)
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        s = sorted(self.samples)
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(s)}


def make_input_host(pft, cfg, N, mu, M, seed, kind):
    if kind == "sparse":
        freqs, amps = pft.sparse_tones(seed, 32, mu - M, mu + M)
        return pft.generate_signal(pft.KIND_SPARSE, seed, N, N=N, freqs=freqs, amps=amps, sigma=1e-3)
    return pft.generate_signal(pft.KIND_NORMAL if kind == "normal" else pft.KIND_UNIFORM, seed, N)


def make_input_device(pft, buf, count, mu, M, seed, kind, offset=0, N=None):
    """`count` elements at global element index `offset` (signal length N for the tones)."""
    N = N or count
    if kind == "sparse":
        freqs, amps = pft.sparse_tones(seed, 32, mu - M, mu + M)
        pft.generate_signal_device(buf.data_ptr(), pft.KIND_SPARSE, seed, count, N=N, offset=offset, freqs=freqs,
                                   amps=amps, sigma=1e-3)
    else:
        pft.generate_signal_device(buf.data_ptr(), pft.KIND_NORMAL if kind == "normal" else pft.KIND_UNIFORM, seed,
                                   count, offset=offset)


def omp_threads(n: int) -> None:
    """Set the OpenMP team size of the oracle library (libgomp is shared by the process)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


def host_cpu() -> dict:
    """CPU model, logical CPUs and the OpenMP team size of the CPU legs."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "omp_num_threads": int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()}


def cpu_oracle_rate(pft_mod, plan, a, budget_s: float):
    """Transforms/s of the CPU oracle (all host threads) on the same plan and input."""
    import oracle
    oracle.execute(plan, a)  # warm (twiddle tables, page faults)
    n, t0 = 0, time.perf_counter()
    while True:
        oracle.execute(plan, a)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            return n / el, n, el


def run_reference(args):
    """--impl reference: the reference algorithm (CPU restatement) on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    import oracle
    import paper_2008_12559_b200 as pft
    N, M, mu, p, kind, desc = CONFIGS[args.config]
    if 16 * N > 4 * 2 ** 30:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.config}: one CPU transform of a "
                          f"{16 * N / 2**30:.0f} GiB signal exceeds the bounded per-step sample"}), flush=True)
        return
    plan = pft.build_plan(N, M, mu, p, EPS)
    a = make_input_host(pft, args.config, N, mu, M, SEEDS[args.config], kind)
    cores = os.cpu_count()
    for _ in range(max(args.warmup, 0)):
        oracle.execute(plan, a)
    # each step is one full transform; cap the run at ~150 s of CPU time
    t0 = time.perf_counter()
    oracle.execute(plan, a)
    per = time.perf_counter() - t0
    steps = max(1, min(args.steps, int(150.0 / max(per, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.execute(plan, a)
    el = time.perf_counter() - t0
    value = steps / el
    line = {
        "impl": "reference", "metric": "PFT transforms/sec", "value": value, "unit": "transforms/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": el / steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if BATCH.get(args.config, 1) > 1 else "weak",
        "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
        "config": {"workload": desc, "p": plan.p, "q": plan.q, "r": plan.r, "epsilon": EPS,
                   "p_choice": "SPEC select_divisor (the reference's CPU cost model)",
                   "sample": "each step = one signal" + (f" of the {BATCH[args.config]}-signal batch"
                                                         if args.config in BATCH else "")},
        "input_gbs": value * 16 * N / 1e9,
        "cpu_baseline": {"value": value, "unit": "transforms/s", "cores": cores, "kind": "port",
                         "sample": f"{steps} full transforms (oracle/oracle.cpp, OpenMP {cores} threads)",
                         **host_cpu()},
        "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2008_12559_b200 as pft

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.config in SHARDED and (world > 1 or args.force_sharded):
        return run_sharded(args, world, rank, local, dev)

    N, M, mu, p, kind, desc = CONFIGS[args.config]
    W = 2 * M + 1
    # batched config (C3): the fixed global batch is sharded by signal over the ranks, no
    # communication (strong scaling); single-signal configs run one replica per GPU (weak)
    B_total = BATCH.get(args.config, 1)
    if B_total > 1 and B_total % world:
        raise SystemExit(f"{args.config}: global batch {B_total} not divisible by {world} GPUs")
    B = B_total // world if B_total > 1 else 1
    scaling = "strong" if B_total > 1 else "weak"

    # inputs: >= 4 buffers, together >= 8x L2 (126 MiB), rotated so no step re-reads an input still
    # in L2 (a batched input is one buffer far larger than L2; C5 one 16 GiB signal)
    nbuf = 1 if (B > 1 or 16 * N >= 16 * L2_BYTES) else max(4, -(-8 * L2_BYTES // (16 * N)))
    bufs = [torch.empty(N * B, dtype=torch.complex128, device=dev) for _ in range(nbuf)]
    for i, b in enumerate(bufs):
        make_input_device(pft, b, N * B, mu, M, SEEDS[args.config] + (0 if B > 1 else 100 * rank), kind,
                          offset=(rank * B * N if B > 1 else i * N), N=N)
    p_src = "--p"
    if args.p:
        p = args.p
    elif p is None:  # device-aware planner: model-ranked candidates, timed on this GPU
        p, tuned_us = pft.autotune_divisor(N, M, mu, bufs[0].data_ptr(), epsilon=EPS, device=local, batch=B)
        p_src = f"pft_autotune_divisor ({tuned_us:.1f} us per execute in the tuning run)"
    else:
        p_src = "config"
    plan = pft.build_plan(N, M, mu, p, EPS)
    d = pft.DevicePlan(plan, device=local, p2=args.p2, batch_hint=B, second_pass=args.second_pass,
                       k2_at=args.k2_at, tail_ctas=args.tail_ctas, k2_grid_ctas=args.k2_grid_ctas)
    overlap = not args.no_pdl  # independent inputs: PFT_EXEC_OVERLAP_PREVIOUS is the caller's promise
    launches = d.launches_per_execute()
    if overlap and B == 1 and d.tail_kind().startswith("K2 workers"):
        launches = 1  # chained single executes: the K2 work rides in K1's grid (one kernel per execute)

    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    # Independent transforms alternate between two streams, each with its own workspace and
    # output (pft_execute is re-entrant on distinct (stream, workspace) pairs), so one
    # transform's K2 and K1 FFT tail overlap the next transform's streaming K1.
    side = torch.cuda.Stream(device=dev)
    ws_elems = -(-d.workspace_bytes(B) // 16)
    ws = [torch.zeros(ws_elems, dtype=torch.complex128, device=dev) for _ in range(args.streams)]  # zeroed once
    outs = [torch.empty(W * B, dtype=torch.complex128, device=dev) for _ in range(2)]
    out = outs[0]
    fork, join = torch.cuda.Event(), torch.cuda.Event()

    def step(i):
        if args.streams == 1:
            d.execute_ptr(bufs[i % nbuf].data_ptr(), out.data_ptr(), batch=B, in_stride=N,
                          d_ws=ws[0].data_ptr(), stream=sp, overlap=overlap)
            return
        if i % 2 == 0:
            fork.record(stream)
            side.wait_event(fork)
        st = stream if i % 2 == 0 else side
        d.execute_ptr(bufs[i % nbuf].data_ptr(), outs[i % 2].data_ptr(), batch=B, in_stride=N,
                      d_ws=ws[i % 2].data_ptr(), stream=st.cuda_stream, overlap=overlap)
        if i % 2 == 1 or i == args.steps - 1:
            join.record(st)
            stream.wait_event(join)

    def capture(fn, n):
        with torch.cuda.stream(stream):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(n):
                    fn(i)
            g.replay()  # warm replay
        torch.cuda.synchronize(dev)
        return g

    def timed(g):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()  # replays on the current stream == `stream`
            e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize(dev)
    # capture exactly K steps into one graph (launch overhead off the timed path)
    graph = capture(step, args.steps)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        torch.cuda.synchronize(dev)
        e0.record(stream)
        graph.replay()  # replays on the current stream == `stream`
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    # chained latency: one stream, executes back to back (the overlap flag as in the timed chain)
    n_lat = min(args.steps, 200)
    lat_graph = capture(lambda i: d.execute_ptr(bufs[i % nbuf].data_ptr(), out.data_ptr(), batch=B, in_stride=N,
                                                d_ws=ws[0].data_ptr(), stream=sp, overlap=overlap), n_lat)
    latency_us = timed(lat_graph) / n_lat * 1e3
    # isolated latency: executes WITHOUT the overlap flag, so each starts only after the previous
    # one completed (no two transforms share the device) -- K executes captured in a graph, device
    # time per execute (launch gaps of the graph included, host API overhead not)
    iso_graph = capture(lambda i: d.execute_ptr(bufs[(i + 1) % nbuf].data_ptr(), out.data_ptr(), batch=B, in_stride=N,
                                                d_ws=ws[0].data_ptr(), stream=sp), n_lat)
    latency_iso_us = timed(iso_graph) / n_lat * 1e3
    # and one call on an idle device from the host: synchronise, CUDA events around one
    # pft_execute (host API overhead included); median
    iso = []
    for i in range(max(5, min(args.steps, 30))):
        torch.cuda.synchronize(dev)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a0.record(stream)
            d.execute_ptr(bufs[(i + 1) % nbuf].data_ptr(), out.data_ptr(), batch=B, in_stride=N,
                          d_ws=ws[0].data_ptr(), stream=sp)
            a1.record(stream)
        torch.cuda.synchronize(dev)
        iso.append(a0.elapsed_time(a1) * 1e3)
    iso.sort()
    latency_call_us = iso[len(iso) // 2]
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * B * args.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (K1).  Its launches are the transform's streaming pass;
    # the follow-up kernel of a 2-launch execute (row sum / K2) overlaps the next K1 under PDL, so
    # the K1 launch duration is bounded by the step time: achieved = 16 N B / ms_per_step is a
    # LOWER bound on K1's rate (exact when K1 is the only kernel).  The ncu launch list of the
    # same command (profiles/) gives each kernel's share.
    peak, peak_src = measured_hbm_peak()
    k1_ms = ms_step
    k1_gbs = 16 * N * B / (k1_ms * 1e-3) / 1e9
    k1_note = ("K1 is the only kernel of an execute: achieved = 16 N B / ms_per_step" if launches == 1 else
               f"{launches} kernels per execute, overlapped under PDL: achieved = 16 N B / ms_per_step "
               "(a lower bound for K1)")
    status = d.status(stream=sp, d_ws=ws[0].data_ptr())
    # parity of this run: the last timed input through the same plan (untimed, no overlap) vs the
    # CPU oracle on the same plan (batched: the first <= 64 signals)
    parity = None
    if rank == 0 and not args.no_parity:
        import numpy as np
        import oracle
        src = bufs[(args.steps - 1) % nbuf]
        # in the timed chain's form: two chained executes (the overlap flag as timed), the last on src
        for x in (bufs[(args.steps - 2) % nbuf], src):
            d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=B, in_stride=N, d_ws=ws[0].data_ptr(), stream=sp,
                          overlap=overlap)
        torch.cuda.synchronize(dev)
        nb = min(B, 64)
        got = out[:W * nb].cpu().numpy().reshape(nb, W)
        t0 = time.perf_counter()
        worst = 0.0
        for b in range(nb):
            ref = oracle.execute(plan, src[b * N:(b + 1) * N].cpu().numpy())
            worst = max(worst, float(np.linalg.norm(got[b] - ref) / np.linalg.norm(ref)))
        parity = {"rel_l2_vs_oracle": worst, "gate": 1e-11, "pass": worst <= 1e-11,
                  "signals_checked": nb, "oracle_seconds": time.perf_counter() - t0,
                  "what": "last timed input, same plan (p, r, P1, P2, tail) and execute form as the timed "
                          "chain, CPU oracle oracle/oracle.cpp"}
        if worst > 1e-11:
            log(f"PARITY FAILURE: rel_l2 {worst:.3e} > 1e-11")

    line = None
    if rank == 0:
        # ---- e2e through the public host API (H2D of the input + D2H of the spectrum)
        e2e = None
        huge = 16 * N > 4 * 2 ** 30  # C5: a host copy / pinned buffer of the whole signal is not sampled
        if huge:
            e2e = {"value": None, "skipped": "input > 4 GiB: no pinned host copy in the bench"}
        if not args.no_e2e and not huge:
            Be = min(B, 64)  # batched: a 64-signal slice per call keeps the pinned buffer small
            h_in = torch.empty(N * Be, dtype=torch.complex128, pin_memory=True)
            h_in.copy_(bufs[0][:N * Be].cpu())
            h_out = torch.empty(W * Be, dtype=torch.complex128, pin_memory=True)
            d_in2 = torch.empty(N * Be, dtype=torch.complex128, device=dev)
            import ctypes as C
            L = pft.lib()
            def e2e_call():
                st = L.pft_execute_host(d.handle, C.c_void_p(h_in.data_ptr()), Be, C.c_void_p(h_out.data_ptr()),
                                        C.c_void_p(d_in2.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(sp))
                if st != 0:
                    raise RuntimeError(f"pft_execute_host failed: {st}")
            for _ in range(2):
                e2e_call()
            n_e2e = max(3, min(args.steps, 20))
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                e2e_call()
            el = time.perf_counter() - t0
            e2e = {"value": n_e2e * Be / el, "unit": "transforms/s", "h2d_bytes_per_step": 16 * N * Be,
                   "d2h_bytes_per_step": 16 * W * Be, "steps": n_e2e, "signals_per_call": Be,
                   "timer": "host wall clock around synchronous pft_execute_host (pinned host buffers)"}
        # ---- CPU baseline: the oracle on this host, bounded sample
        cpu = None
        if huge:
            cpu = {"value": None, "skipped": "input > 4 GiB: one oracle transform exceeds the bounded sample"}
        if not args.no_cpu and world == 1 and not huge:
            try:
                a_host = bufs[0][:N].cpu().numpy()
                rate, n, el = cpu_oracle_rate(pft, plan, a_host, args.cpu_seconds)
                cpu = {"value": rate, "unit": "transforms/s", "cores": os.cpu_count(), "kind": "port",
                       "sample": f"{n} full {args.config} transforms (one signal each) in {el:.1f} s "
                                 f"(oracle/oracle.cpp, OpenMP {os.cpu_count()} threads)", **host_cpu()}
                omp_threads(1)  # report the 1-thread rate as well
                r1, n1, el1 = cpu_oracle_rate(pft, plan, a_host, min(args.cpu_seconds, 5.0))
                omp_threads(os.cpu_count())
                cpu["one_thread"] = {"value": r1, "sample": f"{n1} transforms in {el1:.1f} s, 1 thread"}
            except Exception as e:  # the baseline is reported, never required
                cpu = {"value": None, "error": str(e)}
        line = {
            "metric": "PFT transforms/sec", "value": value, "unit": "transforms/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
            "config": {"workload": f"{args.config}: {desc}", "N": N, "M": M, "mu": mu, "epsilon": EPS,
                       "global_batch": B_total, "batch_per_gpu": B,
                       "p": plan.p, "q": plan.q, "r": plan.r, "P1": d.P1, "P2": d.P2, "p_choice": p_src,
                       "parallelism": (f"signals sharded over {world} GPUs" if B_total > 1 else
                                       f"replicas x{world}") if world > 1 else "single GPU",
                       "l2": (f"one input of {16 * N * B / 2**30:.2f} GiB (> L2 126 MiB)" if nbuf == 1 else
                              f"{nbuf} rotating inputs of {16 * N / 2**20:.1f} MiB ({nbuf * 16 * N / L2_BYTES:.1f}x L2)"),
                       "timing": "CUDA graph of K steps, CUDA events on the launch stream",
                       "streams": args.streams, "overlap_previous": overlap,
                       "tail": {"sum tail": "sum tail in K1 (one kernel per execute)",
                                "K2 tail": "K2 work by K1's last-arriving CTAs (one kernel per execute)",
                                "fused K2": "K2 in K1 behind a grid barrier (one kernel per execute)",
                                "K2 workers in K1 (chained) / K2 grid":
                                    ("K2 worker CTAs inside K1's grid (one kernel per execute)" if overlap else
                                     "K1 + K2 grid (2 kernels per execute)")}.get(
                                    d.tail_kind(), f"K2 ({launches} kernels per execute)"),
                       "pipelining": "independent transforms alternate over 2 streams with separate "
                                     "workspaces" if args.streams == 2 else
                                     "single stream; execute i+1's K1 starts streaming while execute "
                                     "i finishes, via programmatic dependent launch"},
            "latency_us_isolated": latency_iso_us,
            "latency_us_single_call": latency_call_us,
            "latency_us_chained": latency_us,
            "parity_rel_l2": parity["rel_l2_vs_oracle"] if parity else None,
            "parity": parity,
            "input_gbs": value * 16 * N / 1e9,
            "input_gbs_frac_of_peak": value * 16 * N / 1e9 / world / peak,
            "roofline": {"bound": "hbm", "kernel": "k1_contract_fft", "achieved": k1_gbs, "peak": peak,
                         "unit": "GB/s", "frac": k1_gbs / peak, "peak_source": peak_src,
                         "traffic": committed_traffic(args.config),
                         "algorithmic_bytes_per_launch": 16 * N * B, "k1_ms": k1_ms,
                         "note": k1_note},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "status_flags": status,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_sharded(args, world, rank, local, dev):
    """One huge transform split along the contraction axis: every rank
    runs pft_execute_sharded -- K1 on its column slice into a partial slab, ncclReduce of the
    slabs onto rank 0 over NVLink, K2 on rank 0 -- as ONE library call per step, K steps captured
    in one CUDA graph.  Strong scaling: value = whole-job transforms/s, time = max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2008_12559_b200 as pft
    from paper_2008_12559_b200.sharded import ShardedTransform, gather_local_device, init_comm, select_divisor_sharded

    N, M, mu, p, kind, desc = CONFIGS[args.config]
    W = 2 * M + 1
    if args.p:
        p, p_src = args.p, "--p"
    else:
        p, _, est = select_divisor_sharded(N, M, world, epsilon=EPS)
        p_src = f"pft_select_divisor_sharded (model incl. the collective: {est:.0f} us at {world} GPUs)"
    plan = pft.build_plan(N, M, mu, p, EPS)
    st = ShardedTransform(plan, world, rank, root=0, device=local, p2=args.p2)
    comm = init_comm(world, rank, local)
    # this rank's slice of the (device-generated) global signal; setup, not timed
    full = torch.empty(N, dtype=torch.complex128, device=dev)
    make_input_device(pft, full, N, mu, M, SEEDS[args.config], kind, N=N)
    x = gather_local_device(full, plan.p, plan.q, world, rank)
    ref = None
    if world == 1:  # --force-sharded on one GPU: checked against the plain execute below
        ref = torch.empty(W, dtype=torch.complex128, device=dev)
        st.dplan.execute_ptr(full.data_ptr(), ref.data_ptr())
        torch.cuda.synchronize(dev)
    del full
    torch.cuda.empty_cache()
    slab = torch.empty(plan.p * plan.r, dtype=torch.complex128, device=dev)
    out = torch.empty(W, dtype=torch.complex128, device=dev)
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    launches = 2 if rank == 0 else 1  # K1 (+ K2 on the root); the NCCL kernel is NCCL's

    def step():
        st.execute_nccl(comm, x.data_ptr(), slab.data_ptr(), out.data_ptr(), stream=sp)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(args.steps):
                step()
        g.replay()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        torch.cuda.synchronize(dev)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    t = torch.tensor([e0.elapsed_time(e1)], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = args.steps / (ms / 1e3)
    peak, peak_src = measured_hbm_peak()
    local_bytes = 16 * plan.p * st.layout.row_len
    check = None
    if ref is not None:
        check = float(torch.linalg.vector_norm(out - ref) / torch.linalg.vector_norm(ref))
    status = st.dplan.status() if rank == 0 else 0
    if rank == 0:
        line = {
            "metric": "PFT transforms/sec", "value": value, "unit": "transforms/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
            "config": {"workload": f"{args.config}: {desc}", "N": N, "M": M, "mu": mu, "epsilon": EPS,
                       "p": plan.p, "q": plan.q, "r": plan.r, "P1": st.dplan.P1, "P2": st.dplan.P2,
                       "p_choice": p_src,
                       "parallelism": f"contraction axis split over {world} GPUs + ncclReduce of the "
                                      f"{16 * plan.p * plan.r / 2**20:.1f} MiB partial slab inside pft_execute_sharded",
                       "l2": f"per-rank slice of {local_bytes / 2**30:.2f} GiB (> L2 126 MiB)",
                       "timing": "CUDA graph of K pft_execute_sharded steps (K1 | ncclReduce | K2 on rank 0), "
                                 "CUDA events, max over ranks"},
            "input_gbs": value * 16 * N / 1e9,
            "input_gbs_frac_of_peak": value * 16 * N / 1e9 / world / peak,
            "roofline": {"bound": "hbm", "kernel": "k1_contract_fft", "achieved": local_bytes / (ms_step * 1e-3) / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": local_bytes / (ms_step * 1e-3) / 1e9 / peak,
                         "peak_source": peak_src, "traffic": None,
                         "algorithmic_bytes_per_launch": local_bytes,
                         "note": "per-rank K1 bytes over the whole step (K1 + reduce + K2): a lower bound"},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "status_flags": status,
            "sharded_vs_plain_rel_l2": check,
        }
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=0, help="override p (0 = autotune on the device)")
    ap.add_argument("--p2", type=int, default=0, help="override K1 residue classes (0 = planner)")
    ap.add_argument("--streams", type=int, default=1, choices=[1, 2],
                    help="1 (default): one stream; consecutive transforms overlap through programmatic "
                         "dependent launch (K2 releases the next K1).  2: alternate two streams")
    ap.add_argument("--second-pass", default="auto", choices=["auto", "sum", "k2-fft", "k2-dot", "k2-direct", "k2-l2"],
                    help="second-pass form (PFT_PASS2_*)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="c5: run the contraction-axis sharded path even on one GPU (checks it)")
    ap.add_argument("--no-pdl", action="store_true",
                    help="no PFT_EXEC_OVERLAP_PREVIOUS: each execute waits for the previous one")
    ap.add_argument("--k2-at", default="auto", choices=["auto", "grid", "tail", "fused"],
                    help="where the K2 FFT form runs (PFT_K2_AT_*)")
    ap.add_argument("--k2-grid-ctas", type=int, default=0, help="K2 grid width (L2 form)")
    ap.add_argument("--tail-ctas", type=int, default=0, help="sum tail / K2 tail working CTAs per signal (0 = plan)")
    ap.add_argument("--no-parity", action="store_true", help="skip the untimed oracle check of the output")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
