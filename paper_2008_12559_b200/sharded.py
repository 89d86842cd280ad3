"""Multi-GPU execution of one huge transform (BASELINE.json configs[4]: N = 2^30 split along
the contraction axis over 2/4/8 B200s) and batch sharding (configs[2]).

One process per GPU (torchrun).  For a single transform each rank owns, for every row k of A,
the column pairs of pft_shard_layout(q, world, rank); the only exchange is one reduction of the
p x r partial slab (8.4 MB at p = 2^16, r = 8 -- SURVEY.md §8(e)):

    K1 (local slice) -> ncclReduce(slab, sum, root) -> K2 on root

On GPUs the whole step is ONE library call per rank, pft_execute_sharded (C++: K1, the NCCL
reduce over NVLink and K2 on the caller's stream, graph-capturable), over a communicator from
pft_nccl_comm_init (`NcclComm`; the 128-byte unique id travels over torch.distributed).  The
`partial` / `reduce` / `finalize` steps below are the same split with torch.distributed as the
collective: the gloo CPU tests drive the orchestration through it.

The slab is the K1 output Y (the contraction fused with the first FFT pass); both steps are
linear, so the sum over ranks of the partial slabs equals the unsharded slab.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import PftPlan, ShardLayout, _check, lib, shard_gather, shard_layout


def nccl_available() -> bool:
    a = C.c_int()
    _check(lib().pft_nccl_available(C.byref(a)))
    return bool(a.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().pft_nccl_get_unique_id(buf))
    return buf.raw


class NcclComm:
    """A NCCL communicator made by the library (pft_nccl_comm_init) for pft_execute_sharded.
    `uid`: nccl_unique_id() from one rank, shared with the others (e.g. dist.broadcast_object_list)."""

    def __init__(self, world: int, rank: int, uid: bytes, device: int = 0):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.world, self.rank, self.device = world, rank, device
        h = C.c_void_p()
        _check(lib().pft_nccl_comm_init(int(world), int(rank), C.create_string_buffer(uid, 128), int(device),
                                        C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _check(lib().pft_nccl_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


def init_comm(world: int, rank: int, device: int, group=None) -> NcclComm:
    """Collective over torch.distributed: rank 0 makes the NCCL unique id, every rank joins."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return NcclComm(world, rank, obj[0], device)


def select_divisor_sharded(N: int, M: int, world: int, epsilon: float = 1e-12, n_sms: int = 148,
                           table=None) -> tuple[int, int, float]:
    """Device-aware p for the transform sharded over `world` GPUs (collective term included):
    (p, r, modelled microseconds per transform)."""
    from . import _table
    p, r, us = C.c_uint64(), C.c_int(), C.c_double()
    _check(lib().pft_select_divisor_sharded(_table(table).handle, int(N), int(M), float(epsilon), int(n_sms),
                                            int(world), C.byref(p), C.byref(r), C.byref(us)))
    return p.value, r.value, us.value


class ShardedTransform:
    """Contraction-axis sharded execute of `plan` on this rank."""

    def __init__(self, plan: PftPlan, world: int, rank: int, root: int = 0, group=None, device: int = 0,
                 p2: int = 0):
        self.plan, self.world, self.rank, self.root, self.group = plan, world, rank, root, group
        self.layout: ShardLayout = shard_layout(plan.q, world, rank)
        self.device = device
        self._p2 = p2
        self._dplan = None

    # --------------------------------------------------------------- host helpers
    def gather_local(self, a) -> np.ndarray:
        """This rank's slice (p x row_len) of the global signal, in the shard layout."""
        return shard_gather(a, self.plan.p, self.plan.q, self.world, self.rank)

    def slab_elems(self) -> int:
        return self.plan.p * self.plan.r

    # --------------------------------------------------------------- device steps
    @property
    def dplan(self):
        if self._dplan is None:
            from . import DevicePlan
            self._dplan = DevicePlan(self.plan, device=self.device, p2=self._p2)
        return self._dplan

    def partial(self, d_local: int, d_slab: int, stream: int = 0) -> None:
        """K1 on the local slice: writes this rank's partial slab (p*r complex128)."""
        self.dplan.execute_partial_ptr(d_local, d_slab, world=self.world, rank=self.rank,
                                       row_stride=self.layout.row_len, stream=stream)

    def reduce(self, slab) -> None:
        """Sum the partial slabs onto the root (torch tensor, complex128, any backend)."""
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.reduce(torch.view_as_real(slab), dst=self.root, op=dist.ReduceOp.SUM, group=self.group)

    def finalize(self, d_slab: int, d_out: int, stream: int = 0) -> None:
        """K2 on the root: the remaining FFT pass + Eq. (7) post-process."""
        if self.rank == self.root:
            self.dplan.finalize_ptr(d_slab, d_out, stream=stream)

    def execute_nccl(self, comm: NcclComm, d_local: int, d_slab: int, d_out: int, stream: int = 0) -> None:
        """The whole sharded step in the library (pft_execute_sharded): K1 on the slice, ncclReduce
        onto the root, K2 on the root.  Device pointers; asynchronous on `stream`."""
        _check(lib().pft_execute_sharded(self.dplan.handle, C.c_void_p(d_local), self.layout.row_len, comm.handle,
                                         int(self.root), C.c_void_p(d_slab), C.c_void_p(d_out or None),
                                         C.c_void_p(stream or None)))

    def execute(self, local, slab, out) -> None:
        """Sharded transform on CUDA tensors through torch.distributed's reduce (the split steps):
        local (p*row_len), slab (p*r), out (2M+1)."""
        import torch
        stream = torch.cuda.current_stream().cuda_stream
        self.partial(local.data_ptr(), slab.data_ptr(), stream)
        self.reduce(slab)
        self.finalize(slab.data_ptr(), out.data_ptr(), stream)


def local_columns(q: int, world: int, rank: int) -> np.ndarray:
    """Global column of each local column of `rank`'s row layout (-1 = padding)."""
    idx = np.arange(1, q + 1, dtype=np.float64).astype(np.complex128)
    return shard_gather(idx, 1, q, world, rank).reshape(-1).real.astype(np.int64) - 1


def gather_local_device(full, p: int, q: int, world: int, rank: int):
    """Device-side shard_gather: `rank`'s local slice (p * row_len complex128) of a CUDA
    tensor holding the whole signal (setup only: it reads all of `full`)."""
    import torch
    cols = local_columns(q, world, rank)
    sel = torch.from_numpy(np.where(cols < 0, 0, cols)).to(full.device)
    local = full.view(p, q).index_select(1, sel)
    if (cols < 0).any():
        local[:, torch.from_numpy(np.nonzero(cols < 0)[0]).to(full.device)] = 0
    return local.contiguous().view(-1)


def batch_shard(n_signals: int, world: int, rank: int) -> tuple[int, int]:
    """Signals [start, start + count) of rank `rank` when a batch is sharded by signal
    (BASELINE configs[2]); contiguous near-equal split, no communication."""
    base, extra = divmod(n_signals, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)
