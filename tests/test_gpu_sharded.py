"""The sharded transform with its collective inside the library (pft_execute_sharded: K1 on the
local slice -> ncclReduce onto the root -> K2 on the root), on the one GPU a gpurun box has.

A 1-rank NCCL communicator makes the reduce an in-place no-op, so the library call must equal
the split steps (pft_execute_partial + pft_finalize on the same plan) bitwise and the oracle
within the gate; it must also be capturable in a CUDA graph.  Multi-rank orchestration (shard
layout, per-rank slices, the reduce over ranks) is covered by tests/test_sharding_gloo.py and by
test_gpu_parity.py::test_sharded_partials_sum_to_unsharded (ranks emulated one after another).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GATE = 1e-11


@pytest.mark.parametrize("N,M,mu,p", [(2 ** 20, 64, 0, 2 ** 14), (2 ** 22, 2 ** 9, 2 ** 20, 2 ** 13),
                                     (3 * 5 * 7 * 64, 20, 11, 3 * 5 * 64),
                                     # a plan whose chained executes take the K2 workers (r = 12): the sharded
                                     # steps keep the plain slab layout and the K2 finalize
                                     (2 ** 20, 2 ** 11, -7, 2 ** 13)])
def test_execute_sharded_one_rank(pft, oracle, N, M, mu, p):
    import torch
    from paper_2008_12559_b200.sharded import NcclComm, ShardedTransform, nccl_available, nccl_unique_id
    assert nccl_available()
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    st = ShardedTransform(plan, 1, 0)
    comm = NcclComm(1, 0, nccl_unique_id(), 0)
    a = pft.generate_signal(pft.KIND_UNIFORM, 5, N)
    x = torch.from_numpy(np.ascontiguousarray(st.gather_local(a)).reshape(-1)).cuda()
    slab = torch.empty(plan.p * plan.r, dtype=torch.complex128, device="cuda")
    out = torch.empty(2 * M + 1, dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    st.execute_nccl(comm, x.data_ptr(), slab.data_ptr(), out.data_ptr(), stream=s)
    # the split steps on the same plan
    slab2 = torch.empty_like(slab)
    out2 = torch.empty_like(out)
    st.partial(x.data_ptr(), slab2.data_ptr(), s)
    st.finalize(slab2.data_ptr(), out2.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    ref = oracle.execute(plan, a)
    got = out.cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= GATE
    # graph capture of K steps
    outs = [torch.empty_like(out) for _ in range(3)]
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for o in outs:
                st.execute_nccl(comm, x.data_ptr(), slab.data_ptr(), o.data_ptr(), stream=cs.cuda_stream)
        g.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, out)
    comm.close()


def test_execute_sharded_rejects_foreign_device_and_missing_output(pft):
    import torch  # noqa: F401
    from paper_2008_12559_b200.sharded import NcclComm, ShardedTransform, nccl_unique_id
    plan = pft.build_plan(2 ** 16, 32, 0, 2 ** 10, 1e-12)
    st = ShardedTransform(plan, 1, 0)
    comm = NcclComm(1, 0, nccl_unique_id(), 0)
    with pytest.raises(ValueError):
        st.execute_nccl(comm, 16, 16, 0)  # root without d_out
    comm.close()
