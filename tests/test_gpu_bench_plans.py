"""Parity at exactly the plans bench.py times, and execute chains (VERDICT r1 "pin every number
that gets credited").

Each BASELINE config is run here through the device decomposition (p, r, P1, P2, tail form)
that its bench line reports, against the CPU oracle on the same plan (gate: relative l2 <= 1e-11,
BASELINE.json north_star).  The chains check what the throughput mode relies on: executes with
PFT_EXEC_OVERLAP_PREVIOUS (programmatic dependent launch: execute i+1 streams while execute i
finishes in the shared workspace) captured in one CUDA graph, each on its own input and output,
each at the oracle; the default mode with an execute consuming the previous one's output; and a
workspace sized for batch 3 reused by a batch-2 call (control words at batch-independent
offsets).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GATE = 1e-11


def rel_l2(x, y) -> float:
    x, y = np.asarray(x), np.asarray(y)
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


def sparse_c2(pft, M, seed=2):
    N, mu = 2 ** 24, 2 ** 22
    f, a = pft.sparse_tones(seed, 32, mu - M, mu + M)
    return N, mu, pft.generate_signal(pft.KIND_SPARSE, seed, N, N=N, freqs=f, amps=a, sigma=1e-3)


# (config, p, expected (P1, P2, tail kind)) -- the autotuned picks in the bench lines
# (profiles/r01i_bench_*.json, r02*_bench_*.json)
def test_c2b_headline_plan(pft, oracle):
    """C2b (north star): N = 2^24, M = 2^10, mu = N/4, p = 2^14, r = 8, P1 = P2 = 128, sum tail."""
    import torch
    N, mu, a = sparse_c2(pft, 2 ** 10)
    plan = pft.build_plan(N, 2 ** 10, mu, 2 ** 14, 1e-12)
    d = pft.DevicePlan(plan)
    assert (plan.r, d.P1, d.P2, d.tail_kind()) == (8, 128, 128, "sum tail")
    x = torch.from_numpy(a).cuda()
    out = torch.empty(plan.M * 2 + 1, dtype=torch.complex128, device="cuda")
    d.execute_ptr(x.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    assert rel_l2(out.cpu().numpy(), oracle.execute(plan, a)) <= GATE


def test_c2c_full_size_plan(pft, oracle):
    """C2c: M = 2^14 (W = 32769), p = 2^15, r = 14 (FP64 tensor-core K1), K2 grid."""
    import torch
    N, mu, a = sparse_c2(pft, 2 ** 14)
    plan = pft.build_plan(N, 2 ** 14, mu, 2 ** 15, 1e-12)
    d = pft.DevicePlan(plan)
    assert plan.r == 14 and (d.P1, d.P2) == (128, 256) and d.tail_kind().startswith("K2 workers")
    x = torch.from_numpy(a).cuda()
    out = torch.empty(plan.M * 2 + 1, dtype=torch.complex128, device="cuda")
    d.execute_ptr(x.data_ptr(), out.data_ptr())  # isolated: K1 + K2 grid
    torch.cuda.synchronize()
    ref = oracle.execute(plan, a)
    assert rel_l2(out.cpu().numpy(), ref) <= GATE
    # the benchmarked form: a chain with PFT_EXEC_OVERLAP_PREVIOUS (K2 workers inside K1's grid),
    # distinct inputs and outputs in one CUDA graph, then an isolated execute on the same workspace
    K = 4
    xs = [a] + [pft.generate_signal(pft.KIND_UNIFORM, 900 + i, N) for i in range(1, K)]
    dx = [x] + [torch.from_numpy(v).cuda() for v in xs[1:]]
    outs = [torch.full((plan.M * 2 + 1,), np.nan, dtype=torch.complex128, device="cuda") for _ in range(K)]
    ws = torch.zeros(-(-d.workspace_bytes(1) // 16), dtype=torch.complex128, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(K):
                d.execute_ptr(dx[i].data_ptr(), outs[i].data_ptr(), d_ws=ws.data_ptr(), stream=st.cuda_stream,
                              overlap=True)
        for _ in range(3):
            g.replay()
        out.fill_(np.nan)
        d.execute_ptr(dx[1].data_ptr(), out.data_ptr(), d_ws=ws.data_ptr(), stream=st.cuda_stream)
        g.replay()
    torch.cuda.synchronize()
    refs = [ref] + [oracle.execute(plan, v) for v in xs[1:]]
    for i in range(K):
        assert rel_l2(outs[i].cpu().numpy(), refs[i]) <= GATE, i
    assert rel_l2(out.cpu().numpy(), refs[1]) <= GATE
    assert d.status(d_ws=ws.data_ptr()) == 0


def test_c4_autotuned_plan(pft, oracle):
    """C4: N = 6220800, M = 1000, mu = -12345 at the bench's p = 10368 (r = 9, P2 = 81)."""
    N, M, mu = 6220800, 1000, -12345
    a = pft.generate_signal(pft.KIND_NORMAL, 4, N)
    plan = pft.build_plan(N, M, mu, 10368, 1e-12)
    d = plan.device_plan()
    assert d.P2 == 81 and d.tail_kind() == "sum tail"
    assert rel_l2(pft.execute(plan, a).values, oracle.execute(plan, a)) <= GATE


def test_c3_batched_plan_slice(pft, oracle):
    """C3: 4096 x 2^16 signals, M = 256, at the bench's p = 256 (r = 18, tensor cores, P2 = 2,
    last-arrival reduction), batch_hint 4096; a 64-signal slice of the global batch (signals
    4032..4095: global element offsets as the bench generates them) -- every signal checked."""
    import torch
    N, M, B = 2 ** 16, 256, 64
    plan = pft.build_plan(N, M, 0, 256, 1e-12)
    d = pft.DevicePlan(plan, batch_hint=4096)
    assert (plan.r, d.P2, d.tail_kind()) == (18, 2, "sum tail")
    x = torch.empty(N * B, dtype=torch.complex128, device="cuda")
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 3, N * B, offset=(4096 - B) * N)
    ws = torch.zeros(-(-d.workspace_bytes(B) // 16), dtype=torch.complex128, device="cuda")
    out = torch.empty(B * (2 * M + 1), dtype=torch.complex128, device="cuda")
    d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=B, in_stride=N, d_ws=ws.data_ptr())
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(B, 2 * M + 1)
    a = x.cpu().numpy()
    for b in range(B):
        assert rel_l2(got[b], oracle.execute(plan, a[b * N:(b + 1) * N])) <= GATE, b


@pytest.mark.timeout(900)
def test_c5_full_size_plan(pft, oracle):
    """C5: N = 2^30 (16 GiB), M = 2^12 at the bench's plans -- the device planner's p and the
    autotuned p bench.py times (K2 tail, 16 GiB byte offsets) -- against the CPU oracle on the
    same plan (~17 GB of host memory)."""
    import torch
    N, M = 2 ** 30, 2 ** 12
    x = torch.empty(N, dtype=torch.complex128, device="cuda")
    pft.generate_signal_device(x.data_ptr(), pft.KIND_UNIFORM, 5, N)
    p_model, _, _ = pft.select_divisor_device(N, M)
    p_tuned, _ = pft.autotune_divisor(N, M, 0, x.data_ptr())
    got = {}
    for p in sorted({p_model, p_tuned}):
        plan = pft.build_plan(N, M, 0, p, 1e-12)
        d = pft.DevicePlan(plan)
        out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
        d.execute_ptr(x.data_ptr(), out.data_ptr())
        torch.cuda.synchronize()
        got[p] = (plan, out.cpu().numpy(), d.tail_kind())
        d.close()
    a = x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    for p, (plan, g, kind) in got.items():
        assert rel_l2(g, oracle.execute(plan, a)) <= GATE, (p, kind)


@pytest.mark.parametrize("N,M,mu,p,kw", [
    (2 ** 22, 2 ** 8, 2 ** 20, 2 ** 12, {}),                                        # sum tail (C2b-like)
    (2 ** 22, 2 ** 12, 2 ** 20, 2 ** 14, dict(second_pass="k2-fft", k2_at="grid")),  # K1 + K2 grid (C2c-like)
    (2 ** 22, 2 ** 9, -5, 2 ** 15, dict(second_pass="k2-fft", k2_at="tail")),       # K2 tail (C5-like)
    # K2 worker CTAs inside K1's grid (the chained C2c form): default count, few workers (many m1
    # rounds each), more than the free slots (capped), an odd r (column groups 6 + 5), mu = 0
    (2 ** 22, 2 ** 12, 2 ** 20, 2 ** 14, dict(second_pass="k2-fft", k2_at="tail")),
    (2 ** 22, 2 ** 12, 2 ** 20, 2 ** 14, dict(second_pass="k2-fft", k2_at="tail", tail_ctas=3)),
    (2 ** 22, 2 ** 12, 2 ** 20, 2 ** 14, dict(second_pass="k2-fft", k2_at="tail", tail_ctas=200)),
    (2 ** 22, 3000, 0, 2 ** 14, dict(second_pass="k2-fft", k2_at="tail", p2=128)),
    # the ring K2 kernel on a narrow grid (opt-in, k2_grid_ctas)
    (2 ** 22, 2 ** 12, 2 ** 20, 2 ** 14, dict(second_pass="k2-fft", k2_grid_ctas=12)),
])
def test_overlap_chain_distinct_inputs_in_one_graph(pft, oracle, N, M, mu, p, kw):
    """K executes of distinct inputs into distinct outputs with PFT_EXEC_OVERLAP_PREVIOUS,
    captured in ONE CUDA graph on one stream and one shared workspace: execute i+1's K1 streams
    while execute i still reduces; every output matches the oracle on its own input."""
    import torch
    K = 6
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    d = pft.DevicePlan(plan, **kw)
    if kw.get("k2_at") == "tail" and 8 <= plan.r <= 18:
        assert d.tail_kind().startswith("K2 workers"), (plan.r, d.P1, d.P2, d.tail_kind())
    xs = [pft.generate_signal(pft.KIND_UNIFORM, 500 + i, N) for i in range(K)]
    dx = [torch.from_numpy(x).cuda() for x in xs]
    outs = [torch.full((2 * M + 1,), np.nan, dtype=torch.complex128, device="cuda") for _ in range(K)]
    ws = torch.zeros(-(-d.workspace_bytes(1) // 16), dtype=torch.complex128, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(K):
                d.execute_ptr(dx[i].data_ptr(), outs[i].data_ptr(), d_ws=ws.data_ptr(), stream=st.cuda_stream,
                              overlap=True)
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    for i in range(K):
        assert rel_l2(outs[i].cpu().numpy(), oracle.execute(plan, xs[i])) <= GATE, i
    assert d.status(d_ws=ws.data_ptr()) == 0


def test_default_mode_consumes_previous_output(pft, oracle):
    """Without the overlap flag an execute may read the previous execute's output: plan A's
    2M+1 = 4097 outputs are plan B's input (N_B = 4097 = 17 * 241), same stream, no sync."""
    import torch
    A = pft.build_plan(2 ** 20, 2048, 77, None, 1e-12)
    B = pft.build_plan(4097, 100, 3, None, 1e-12)
    da, db = pft.DevicePlan(A), pft.DevicePlan(B)
    a = pft.generate_signal(pft.KIND_UNIFORM, 71, A.N)
    x = torch.from_numpy(a).cuda()
    y = torch.empty(4097, dtype=torch.complex128, device="cuda")
    z = torch.empty(201, dtype=torch.complex128, device="cuda")
    wa = torch.zeros(-(-da.workspace_bytes(1) // 16), dtype=torch.complex128, device="cuda")
    wb = torch.zeros(-(-db.workspace_bytes(1) // 16), dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        y.fill_(np.nan)
        da.execute_ptr(x.data_ptr(), y.data_ptr(), d_ws=wa.data_ptr(), stream=s)
        db.execute_ptr(y.data_ptr(), z.data_ptr(), d_ws=wb.data_ptr(), stream=s)
    torch.cuda.synchronize()
    ya = oracle.execute(A, a)
    assert rel_l2(y.cpu().numpy(), ya) <= GATE
    assert rel_l2(z.cpu().numpy(), oracle.execute(B, y.cpu().numpy())) <= GATE


@pytest.mark.parametrize("kw", [{}, dict(second_pass="k2-fft", k2_at="tail"), dict(second_pass="k2-fft", k2_at="grid")])
def test_workspace_for_batch3_serves_batch2(pft, oracle, kw):
    """a workspace sized and zeroed for batch 3, then used by batch-3 and batch-2
    calls alternately (a remainder batch): control words sit at batch-independent offsets."""
    import torch
    N, M, mu = 2 ** 16, 128, 77
    plan = pft.build_plan(N, M, mu, 4096, 1e-12)
    d = pft.DevicePlan(plan, batch_hint=3, **kw)
    a = pft.generate_signal(pft.KIND_UNIFORM, 9, N * 3)
    x = torch.from_numpy(a).cuda()
    ws = torch.zeros(-(-d.workspace_bytes(3) // 16), dtype=torch.complex128, device="cuda")
    assert d.workspace_bytes(2) <= d.workspace_bytes(3)
    refs = [oracle.execute(plan, a[b * N:(b + 1) * N]) for b in range(3)]
    for batch in (3, 2, 3, 2, 1, 3):
        out = torch.full((batch * (2 * M + 1),), np.nan, dtype=torch.complex128, device="cuda")
        d.execute_ptr(x.data_ptr(), out.data_ptr(), batch=batch, in_stride=N, d_ws=ws.data_ptr())
        torch.cuda.synchronize()
        got = out.cpu().numpy().reshape(batch, 2 * M + 1)
        for b in range(batch):
            assert rel_l2(got[b], refs[b]) <= GATE, (batch, b)
