"""Multi-process (world_size 2 and 3, gloo on CPU) coverage of the sharded paths' host logic:
shard layout -> per-rank partial contraction -> torch.distributed reduce -> finalize, checked
against the unsharded transform.  The per-rank device kernel (K1 partial) is stood in for by
the oracle's contraction of the same columns (tests may use the oracle); the partial-slab
sum over ranks is linear in the same way on the GPU (tests/test_gpu_parity.py covers the
kernel side on one GPU)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, N, M, mu, p, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2008_12559_b200 as pft
        from paper_2008_12559_b200.sharded import ShardedTransform, batch_shard

        plan = pft.build_plan(N, M, mu, p, 1e-12)
        a = pft.generate_signal(pft.KIND_UNIFORM, 11, N)  # every rank can regenerate its data
        st = ShardedTransform(plan, world, rank)
        local = st.gather_local(a)                      # p x row_len
        v = st.layout
        gcols = np.array([int(x.real) for x in pft.shard_gather(np.arange(plan.q, dtype=complex), 1, plan.q,
                                                                  world, rank)[0]], dtype=np.int64)
        # partial contraction over this rank's columns (oracle stand-in for K1's contraction)
        partial = oracle.matmul(local, plan.B[gcols, :]) if v.row_len else np.zeros((plan.p, plan.r), complex)
        slab = torch.from_numpy(np.ascontiguousarray(partial).reshape(-1).copy())
        st.reduce(slab)                                  # dist.reduce over gloo
        if rank == 0:
            C = slab.numpy().reshape(plan.p, plan.r)
            out = oracle.post(plan, oracle.batch_fft_columns(C))
            ref = oracle.execute(plan, a)
            results[rank] = float(np.linalg.norm(out - ref) / np.linalg.norm(ref))
        else:
            results[rank] = 0.0
        # batch sharding covers every signal exactly once
        counts = [batch_shard(4096, world, r) for r in range(world)]
        assert counts[0][0] == 0 and sum(c for _, c in counts) == 4096
        assert all(counts[i][0] + counts[i][1] == counts[i + 1][0] for i in range(world - 1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,M,mu,p", [(2, 2 ** 16, 64, 1000, 2 ** 10), (3, 105 * 64, 20, 11, 15 * 64),
                                            (2, 2 ** 18, 256, -77, 2 ** 12)])
def test_contraction_sharding_over_gloo(world, N, M, mu, p):
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, port, N, M, mu, p, results), nprocs=world, join=True)
        assert results[0] <= 1e-13, dict(results)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_gather_local_device_matches_shard_gather(pft, world):
    """bench.py's C5 setup slices a device-resident signal with torch (sharded.gather_local_device);
    it must equal the library's shard_gather layout for every rank (run here on CPU tensors)."""
    import torch
    from paper_2008_12559_b200.sharded import gather_local_device, local_columns
    p, q = 16, 50
    a = pft.generate_signal(pft.KIND_UNIFORM, 5, p * q)
    seen = []
    for rank in range(world):
        ref = pft.shard_gather(a, p, q, world, rank)
        got = gather_local_device(torch.from_numpy(a), p, q, world, rank).numpy().reshape(p, -1)
        assert np.array_equal(ref, got)
        cols = local_columns(q, world, rank)
        seen += [int(c) for c in cols if c >= 0]
    assert sorted(seen) == list(range(q))  # every column on exactly one rank
