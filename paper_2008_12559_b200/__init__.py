"""B200-native Partial Fourier Transform (arXiv 2008.12559) -- Python mirror of the API.

The product is libpft_b200.so: a C++20 host library (minimax table, planner) and sm_100a
CUDA kernels behind the C ABI in include/pft_capi.h.  This module mirrors the reference's
plan-then-execute interface (SPEC.md modules minimax / planner / transform; type names of
proj/include/pft/types.hpp) with the same argument meaning and error behaviour, so tests
read like the reference's own acceptance tests.  Every call goes through the C ABI; the
transform itself runs only on the GPU (no CPU fallback -- see oracle/ for the checker).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import c128

__all__ = [
    "PftError", "ApproxPoly", "ScopeTable", "CostEstimate", "TargetRange", "PartialSpectrum", "PftPlan",
    "DevicePlan", "best_approx", "scope_xi", "translate_poly", "divisors", "min_terms", "select_divisor", "select_divisor_device", "autotune_divisor",
    "Pft2dPlan", "PartialSpectrum2d", "build_plan_2d", "execute_2d", "parenthesization", "autotune_2d",
    "build_plan", "execute", "mod_index", "l1_norm", "generate_signal", "sparse_tones", "shard_layout",
    "shard_gather",
    "device_count", "lib",
]

DEFAULT_EPSILON = 1e-12  # BASELINE.json configs


def lib() -> C.CDLL:
    return _capi.load()


# ----------------------------------------------------------------------------- errors

class PftError(Exception):
    """A non-OK pft_status from the C ABI."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.name = _capi.STATUS_NAMES.get(status, f"status {status}")
        super().__init__(f"{self.name}: {message}")


class PftValueError(PftError, ValueError):
    pass


class PftIOError(PftError, OSError):
    pass


class PftDeviceError(PftError, RuntimeError):
    pass


_VALUE = {1, 2, 3, 4, 5, 6, 7, 12, 14}
_IO = {8, 9}


def _check(status: int) -> None:
    if status == 0:
        return
    msg = (lib().pft_last_error() or b"").decode() or lib().pft_status_string(status).decode()
    cls = PftValueError if status in _VALUE else PftIOError if status in _IO else PftDeviceError
    raise cls(status, msg)


def _cbuf(n: int) -> np.ndarray:
    return np.zeros(max(n, 1), dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------------------- types.hpp mirror

def mod_index(m: int, n: int) -> int:
    """Non-negative m mod n (types.hpp:15-20)."""
    return m % n


def l1_norm(v) -> float:
    """sum |v_i| (types.hpp:92-96)."""
    return float(np.sum(np.abs(np.asarray(v, dtype=np.complex128))))


@dataclasses.dataclass(frozen=True)
class TargetRange:
    """R_{mu,M} = [mu - M, mu + M] (types.hpp:24-43)."""
    mu: int = 0
    half_width: int = 0

    def count(self) -> int:
        return 2 * self.half_width + 1

    def first(self) -> int:
        return self.mu - self.half_width

    def last(self) -> int:
        return self.mu + self.half_width

    def contains(self, m: int) -> bool:
        return self.first() <= m <= self.last()

    def slot(self, m: int) -> int:
        if not self.contains(m):
            raise IndexError(f"TargetRange::slot: index {m} outside [{self.first()}, {self.last()}]")
        return m - self.first()


@dataclasses.dataclass
class PartialSpectrum:
    """values[slot(m)] estimates coefficient m (types.hpp:47-53)."""
    range: TargetRange
    values: np.ndarray
    plan_id: int = 0

    def at(self, m: int) -> complex:
        return complex(self.values[self.range.slot(m)])


# ----------------------------------------------------------------------------- minimax

@dataclasses.dataclass
class ApproxPoly:
    """SPEC.md:35-41."""
    coeffs: np.ndarray
    base_frequency: float
    scope: float
    achieved_error: float

    @property
    def degree(self) -> int:
        return len(self.coeffs) - 1

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        acc = np.zeros(x.shape, dtype=np.complex128)
        pw = np.ones(x.shape)
        for c in self.coeffs:
            acc = acc + c * pw
            pw = pw * x
        return acc


def best_approx(r: int, xi: float, u: float) -> ApproxPoly:
    """Near-minimax degree r-1 polynomial for e^{iux} on |x| <= xi."""
    out = _cbuf(r)
    ach = C.c_double()
    _check(lib().pft_best_approx(int(r), float(xi), float(u), _ptr(out), C.byref(ach)))
    return ApproxPoly(out[:r].copy(), float(u), abs(float(xi)), ach.value)


def scope_xi(epsilon: float, r: int) -> tuple[float, ApproxPoly]:
    """Largest certified xi with error <= epsilon, and its polynomial."""
    out = _cbuf(r)
    xi = C.c_double()
    ach = C.c_double()
    _check(lib().pft_scope_xi(float(epsilon), int(r), C.byref(xi), _ptr(out), C.byref(ach)))
    return xi.value, ApproxPoly(out[:r].copy(), float(np.pi), xi.value, ach.value)


def translate_poly(poly: ApproxPoly, u: float, mu: float) -> ApproxPoly:
    """Q(x) = e^{iu mu} P(x - mu) (Lemma 1)."""
    c = np.ascontiguousarray(poly.coeffs, dtype=np.complex128)
    out = _cbuf(len(c))
    _check(lib().pft_translate_poly(_ptr(c), len(c), float(u), float(mu), _ptr(out)))
    return ApproxPoly(out[:len(c)].copy(), float(u), poly.scope, poly.achieved_error)


@dataclasses.dataclass
class TableEntry:
    epsilon: float
    r: int
    xi: float
    coeffs: np.ndarray
    achieved_error: float


class ScopeTable:
    """Persisted map (eps, r) -> (xi, coeffs) (PFTT v1 SPEC.md:108)."""

    version = 1

    def __init__(self, handle, owned: bool):
        self._h = handle
        self._owned = owned

    def __del__(self):
        if getattr(self, "_owned", False) and self._h:
            try:
                lib().pft_table_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def default(cls) -> "ScopeTable":
        h = C.c_void_p()
        _check(lib().pft_table_default(C.byref(h)))
        return cls(h, owned=False)

    @classmethod
    def generate(cls, epsilons: Optional[Sequence[float]] = None, r_max: int = 25) -> "ScopeTable":
        h = C.c_void_p()
        if epsilons:
            arr = np.ascontiguousarray(epsilons, dtype=np.float64)
            _check(lib().pft_table_generate(_ptr(arr), len(arr), int(r_max), C.byref(h)))
        else:
            _check(lib().pft_table_generate(None, 0, int(r_max), C.byref(h)))
        return cls(h, owned=True)

    @classmethod
    def load(cls, path) -> "ScopeTable":
        h = C.c_void_p()
        _check(lib().pft_table_load(str(path).encode(), C.byref(h)))
        return cls(h, owned=True)

    def save(self, path) -> None:
        _check(lib().pft_table_save(self._h, str(path).encode()))

    def save_csv(self, path) -> None:
        _check(lib().pft_table_save_csv(self._h, str(path).encode()))

    def __len__(self) -> int:
        n = C.c_size_t()
        _check(lib().pft_table_size(self._h, C.byref(n)))
        return n.value

    def entry(self, i: int) -> TableEntry:
        eps, xi, ach = C.c_double(), C.c_double(), C.c_double()
        r = C.c_int()
        buf = _cbuf(25)
        _check(lib().pft_table_entry(self._h, i, C.byref(eps), C.byref(r), C.byref(xi), _ptr(buf), C.byref(ach)))
        return TableEntry(eps.value, r.value, xi.value, buf[:r.value].copy(), ach.value)

    @property
    def entries(self) -> list[TableEntry]:
        return [self.entry(i) for i in range(len(self))]

    def lookup(self, epsilon: float, r: int) -> TableEntry:
        xi, ach = C.c_double(), C.c_double()
        buf = _cbuf(25)
        _check(lib().pft_table_lookup(self._h, float(epsilon), int(r), C.byref(xi), _ptr(buf), C.byref(ach)))
        return TableEntry(float(epsilon), int(r), xi.value, buf[:r].copy(), ach.value)

    @property
    def epsilon_grid(self) -> list[float]:
        seen: list[float] = []
        for e in self.entries:
            if not any(abs(e.epsilon - s) <= 1e-9 * s for s in seen):
                seen.append(e.epsilon)
        return seen

    @property
    def r_max(self) -> int:
        return max(e.r for e in self.entries)


# ----------------------------------------------------------------------------- planner

@dataclasses.dataclass(frozen=True)
class CostEstimate:
    """SPEC.md:130-133."""
    p: int
    r: int
    cost: float


def _table(table: Optional[ScopeTable]) -> ScopeTable:
    return table if table is not None else ScopeTable.default()


def divisors(N: int) -> list[int]:
    """All divisors of N, ascending."""
    cnt = C.c_size_t()
    st = lib().pft_divisors(int(N), None, 0, C.byref(cnt))
    if st not in (0, 14):
        _check(st)
    arr = np.zeros(max(cnt.value, 1), dtype=np.uint64)
    _check(lib().pft_divisors(int(N), _ptr(arr), cnt.value, C.byref(cnt)))
    return [int(x) for x in arr[:cnt.value]]


def min_terms(epsilon: float, M: int, p: int, table: Optional[ScopeTable] = None) -> int:
    """min{r : xi(eps, r) >= M/p}."""
    r = C.c_int()
    _check(lib().pft_min_terms(_table(table).handle, float(epsilon), int(M), int(p), C.byref(r)))
    return r.value


def select_divisor(N: int, M: int, table: Optional[ScopeTable] = None,
                   epsilon: float = DEFAULT_EPSILON) -> tuple[int, CostEstimate]:
    """Cost-model choice of p."""
    p = C.c_uint64()
    r = C.c_int()
    cost = C.c_double()
    _check(lib().pft_select_divisor(_table(table).handle, int(N), int(M), float(epsilon), C.byref(p),
                                    C.byref(r), C.byref(cost)))
    return p.value, CostEstimate(p.value, r.value, cost.value)


def select_divisor_device(N: int, M: int, table: Optional[ScopeTable] = None,
                          epsilon: float = DEFAULT_EPSILON, n_sms: int = 148) -> tuple[int, int, float]:
    """Device-aware choice of p for the B200 path (not in the reference):
    returns (p, r, modelled microseconds per transform).  Pass p to build_plan."""
    p = C.c_uint64()
    r = C.c_int()
    est = C.c_double()
    _check(lib().pft_select_divisor_device(_table(table).handle, int(N), int(M), float(epsilon), int(n_sms),
                                           C.byref(p), C.byref(r), C.byref(est)))
    return p.value, r.value, est.value


class PartialSpectrum2d:
    """(2M1+1) x (2M2+1) values on the rectangle R_{(mu1,mu2),(M1,M2)}."""

    def __init__(self, values: np.ndarray, mu1: int, mu2: int, M1: int, M2: int):
        self.values, self.mu1, self.mu2, self.M1, self.M2 = values, mu1, mu2, M1, M2

    def at(self, m1: int, m2: int) -> complex:
        i, j = m1 - (self.mu1 - self.M1), m2 - (self.mu2 - self.M2)
        if not (0 <= i < self.values.shape[0] and 0 <= j < self.values.shape[1]):
            raise IndexError("(m1, m2) outside the target rectangle")
        return complex(self.values[i, j])


def parenthesization(q1: int, r1: int, q2: int, r2: int) -> str:
    """SPEC.md:285 / Appendix B: LeftFirst ((B1^T A) B2) iff q2 r1 (q1 + r2) <= q1 r2 (q2 + r1)."""
    return "LeftFirst" if q2 * r1 * (q1 + r2) <= q1 * r2 * (q2 + r1) else "RightFirst"


class Pft2dPlan:
    """2-D PFT configuration (Algorithm 3): one 1-D plan per dimension --
    plan1 for axis 1 (N1, M1, mu1, p1), plan2 for axis 2 -- and the CPU parenthesization
    (LeftFirst iff q2 r1 (q1 + r2) <= q1 r2 (q2 + r1)), which only matters for the CPU cost."""

    def __init__(self, plan1: "PftPlan", plan2: "PftPlan"):
        self.plan1, self.plan2 = plan1, plan2
        self.parenthesization = parenthesization(plan1.q, plan1.r, plan2.q, plan2.r)
        self.achieved_epsilon = max(plan1.achieved_epsilon, plan2.achieved_epsilon)
        self._dplans = None

    @property
    def shape(self) -> tuple[int, int]:
        return self.plan1.N, self.plan2.N

    def device_plans(self, device: int = 0):
        """(rows, cols): the axis-2 plan batched over the N1 rows, the axis-1 plan over the
        2M2+1 columns of the first pass."""
        if self._dplans is None:
            rows = DevicePlan(self.plan2, device=device, batch_hint=self.plan1.N)
            cols = DevicePlan(self.plan1, device=device, batch_hint=2 * self.plan2.M + 1)
            self._dplans = (rows, cols)
        return self._dplans

    def workspace_bytes(self, device: int = 0) -> int:
        rows, cols = self.device_plans(device)
        n = C.c_size_t()
        _check(lib().pft_workspace_bytes_2d(rows.handle, cols.handle, C.byref(n)))
        return n.value

    def execute_ptr(self, d_in: int, d_out: int, d_ws: int, stream: int = 0, device: int = 0) -> None:
        rows, cols = self.device_plans(device)
        _check(lib().pft_execute_2d(rows.handle, cols.handle, C.c_void_p(d_in), C.c_void_p(d_out),
                                    C.c_void_p(d_ws), C.c_void_p(stream or None)))


def build_plan_2d(N1: int, N2: int, M1: int, M2: int, mu1: int, mu2: int, p1: Optional[int] = None,
                  p2: Optional[int] = None, epsilon: float = DEFAULT_EPSILON,
                  table: Optional[ScopeTable] = None) -> Pft2dPlan:
    """Algorithm 3: per-dimension plans (p_d auto via select_divisor)."""
    for N, M in ((N1, M1), (N2, M2)):
        if 2 * M > N:
            raise PftValueError(1, "build_plan_2d: M_d > N_d / 2")
    return Pft2dPlan(build_plan(N1, M1, mu1, p1, epsilon, table), build_plan(N2, M2, mu2, p2, epsilon, table))


def autotune_2d(plan: Pft2dPlan, d_in: int, device: int = 0, candidates: int = 8) -> Pft2dPlan:
    """Device-measured p per axis (SURVEY.md §8(f) row 1 applied to Algorithm 3).  SPEC's CPU
    cost model picks each p_d for one length-N_d signal; on the GPU the axis-2 pass runs N1
    short signals as one batch and the axis-1 pass 2M2+1 of them, where the per-signal FFT and
    tail costs decide (tools/probe_2d.py: 4096 x 4096, M = 64: rows p = 64 208 us vs SPEC's 128
    232 us, columns p = 256 33 us vs 80 us).  Each axis is timed with pft_autotune_divisor at
    its batch: the rows over the caller's device grid `d_in` (N1 x N2 complex128), the columns
    over the first (2M2+1) x N1 elements of the same buffer (timing only).  Returns a new plan
    with those p; the oracle must be given that plan."""
    p1, p2 = plan.plan1, plan.plan2
    pr, _ = autotune_divisor(p2.N, p2.M, p2.mu, d_in, epsilon=p2.epsilon, device=device, candidates=candidates,
                             batch=p1.N)
    pc, _ = autotune_divisor(p1.N, p1.M, p1.mu, d_in, epsilon=p1.epsilon, device=device, candidates=candidates,
                             batch=2 * p2.M + 1)
    return Pft2dPlan(build_plan(p1.N, p1.M, p1.mu, pc, p1.epsilon), build_plan(p2.N, p2.M, p2.mu, pr, p2.epsilon))


def execute_2d(plan: Pft2dPlan, a, device: int = 0) -> PartialSpectrum2d:
    """Algorithm 4 on the GPU: a is N1 x N2 (row-major) complex128."""
    N1, N2 = plan.shape
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if a.size != N1 * N2:
        raise PftValueError(6, "execute_2d: grid shape does not match the plan")
    W1, W2 = 2 * plan.plan1.M + 1, 2 * plan.plan2.M + 1
    out = np.zeros((W1, W2), dtype=np.complex128)
    rows, cols = plan.device_plans(device)
    _check(lib().pft_execute_2d_host(rows.handle, cols.handle, _ptr(a), _ptr(out)))
    return PartialSpectrum2d(out, plan.plan1.mu, plan.plan2.mu, plan.plan1.M, plan.plan2.M)


def autotune_divisor(N: int, M: int, mu: int, d_in: int, table: Optional[ScopeTable] = None,
                     epsilon: float = DEFAULT_EPSILON, device: int = 0, candidates: int = 4,
                     batch: int = 1) -> tuple[int, float]:
    """Measured choice of p: times the `candidates` best modelled divisors on the device with the
    caller's input (device pointer to batch x N complex128); returns (p, microseconds per execute
    of the batch)."""
    p = C.c_uint64()
    us = C.c_double()
    _check(lib().pft_autotune_divisor(_table(table).handle, int(N), int(M), int(mu), float(epsilon), int(device),
                                      C.c_void_p(int(d_in)), int(batch), int(candidates), C.byref(p), C.byref(us)))
    return p.value, us.value


class PftPlan:
    """Frozen configuration of Algorithm 1.  Arrays are host copies of the
    plan tables the GPU consumes; the oracle consumes the same arrays."""

    def __init__(self, handle):
        self._h = handle
        info = _capi.PlanInfo()
        _check(lib().pft_plan_info_get(handle, C.byref(info)))
        self.N, self.M, self.mu = int(info.N), int(info.M), int(info.mu)
        self.p, self.q, self.r = int(info.p), int(info.q), int(info.r)
        self.epsilon = float(info.epsilon)
        self.achieved_epsilon = float(info.achieved_epsilon)
        self.xi = float(info.xi)
        self.estimated_cost = float(info.estimated_cost)
        self.plan_id = int(info.plan_id)
        self._cache: dict = {}
        self._dplans: dict = {}

    def __del__(self):
        for d in getattr(self, "_dplans", {}).values():
            d.close()
        if getattr(self, "_h", None):
            try:
                lib().pft_plan_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def range(self) -> TargetRange:
        return TargetRange(self.mu, self.M)

    def _get(self, name: str, n: int, dtype, fn):
        if name not in self._cache:
            arr = np.zeros(max(n, 1), dtype=dtype)
            _check(fn(self._h, _ptr(arr)))
            self._cache[name] = arr[:n]
        return self._cache[name]

    @property
    def B(self) -> np.ndarray:
        return self._get("B", self.q * self.r, np.complex128, lib().pft_plan_copy_B).reshape(self.q, self.r)

    @property
    def w(self) -> np.ndarray:
        return self._get("w", self.r, np.complex128, lib().pft_plan_copy_w)

    @property
    def phase(self) -> np.ndarray:
        return self._get("phase", self.q, np.complex128, lib().pft_plan_copy_phase)

    @property
    def tvals(self) -> np.ndarray:
        return self._get("tvals", self.q, np.float64, lib().pft_plan_copy_tvals)

    @property
    def post_powers(self) -> np.ndarray:
        W = 2 * self.M + 1
        return self._get("pp", W * self.r, np.float64, lib().pft_plan_copy_post_powers).reshape(W, self.r)

    @property
    def post_twiddles(self) -> np.ndarray:
        return self._get("pt", 2 * self.M + 1, np.complex128, lib().pft_plan_copy_post_twiddles)

    def json(self) -> str:
        need = C.c_size_t()
        lib().pft_plan_json(self._h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        _check(lib().pft_plan_json(self._h, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def device_plan(self, device: int = 0, p2: int = 0) -> "DevicePlan":
        key = (device, p2)
        if key not in self._dplans:
            self._dplans[key] = DevicePlan(self, device=device, p2=p2)
        return self._dplans[key]


def build_plan(N: int, M: int, mu: int = 0, p: Optional[int] = None, epsilon: float = DEFAULT_EPSILON,
               table: Optional[ScopeTable] = None) -> PftPlan:
    """Algorithm 1.  p=None selects p with the SPEC cost model."""
    h = C.c_void_p()
    _check(lib().pft_plan_build(_table(table).handle, int(N), int(M), int(mu), int(p or 0), float(epsilon),
                                C.byref(h)))
    return PftPlan(h)


# ----------------------------------------------------------------------------- transform (GPU)

def device_count() -> int:
    n = C.c_int()
    _check(lib().pft_device_count(C.byref(n)))
    return n.value


PASS2 = {"auto": 0, "sum": 1, "k2-fft": 2, "k2-dot": 3, "k2-direct": 4, "k2-l2": 5,
         "k2-bluestein": 6}                                                          # PFT_PASS2_*
K2_AT = {"auto": 0, "grid": 1, "tail": 2, "fused": 3}                                 # PFT_K2_AT_*
EXEC_OVERLAP_PREVIOUS = 1                                                             # PFT_EXEC_*


class DevicePlan:
    """A plan uploaded to one B200 (pft_dplan_t).  Device buffers are passed as raw
    pointers (e.g. torch.Tensor.data_ptr() of complex128 CUDA tensors).

    second_pass: "auto" | "sum" (sum tail in K1) | "k2-fft" | "k2-dot" | "k2-direct" | "k2-l2"
    k2_at: where the k2-fft form runs: "auto" | "grid" (own launch) | "tail" (inside K1: its last
    arrivals for r = 4..7, K2 worker CTAs riding in K1's grid for r = 8..18 on overlapped
    executes) | "fused" (K1 behind a grid barrier).  tail_ctas: sum-tail reducers / K2-tail or
    K2 workers per signal (0 = plan).  k2_grid_ctas: width of the ring K2 kernel's grid (0 = one
    CTA per m1).  batch_hint: typical batch per execute.  split: isolated
    executes may run two K1 CTAs (a cluster) per residue class (PFT_EXEC_OVERLAP_PREVIOUS
    executes never do)."""

    def __init__(self, plan: PftPlan, device: int = 0, p2: int = 0, k1_stages: int = 0, second_pass: str = "auto",
                 k2_at: str = "auto", tail_ctas: int = 0, k2_grid_ctas: int = 0, batch_hint: int = 1,
                 split: bool = True):
        self.plan = plan
        opts = _capi.DPlanOpts()
        opts.device = device
        opts.p2 = p2
        opts.k1_stages = k1_stages
        opts.second_pass = PASS2[second_pass]
        opts.k2_at = K2_AT[k2_at]
        opts.tail_ctas = tail_ctas
        opts.k2_grid_ctas = k2_grid_ctas
        opts.k1_split = 0 if split else 1
        opts.batch_hint = batch_hint
        h = C.c_void_p()
        _check(lib().pft_dplan_create(plan.handle, C.byref(opts), C.byref(h)))
        self._h = h
        p1, pp2 = C.c_uint64(), C.c_uint64()
        _check(lib().pft_dplan_layout(h, C.byref(p1), C.byref(pp2)))
        self.P1, self.P2 = p1.value, pp2.value
        self.device = device

    def close(self) -> None:
        if getattr(self, "_h", None):
            try:
                lib().pft_dplan_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    def workspace_bytes(self, batch: int = 1) -> int:
        n = C.c_size_t()
        _check(lib().pft_workspace_bytes(self._h, batch, C.byref(n)))
        return n.value

    def signals_per_cta(self, batch: int) -> int:
        """Signals a K1 CTA holds for a contiguous batch of this size (pft_dplan_signals_per_cta)."""
        n = C.c_int()
        _check(lib().pft_dplan_signals_per_cta(self._h, C.c_size_t(batch), C.byref(n)))
        return n.value

    def launches_per_execute(self) -> int:
        n = C.c_int()
        _check(lib().pft_launches_per_execute(self._h, C.byref(n)))
        return n.value

    TAIL_KINDS = ("K2 grid", "sum tail", "K2 tail", "fused K2", "K2 workers in K1 (chained) / K2 grid")

    def tail_kind(self) -> str:
        """How execute finishes after K1: "K2 grid", "sum tail", "K2 tail" (K2's work by K1's
        last arrivals), "fused K2" (grid barrier, opt-in) or "K2 workers in K1 (chained) / K2 grid"
        (overlapped executes: K2 worker CTAs inside K1's grid; isolated ones: K1 + K2 grid)."""
        n = C.c_int()
        _check(lib().pft_dplan_tail_kind(self._h, C.byref(n)))
        return self.TAIL_KINDS[n.value]

    @property
    def second_pass(self) -> str:
        """The second-pass form this plan runs ("sum", "k2-fft", "k2-dot", "k2-direct", "k2-l2",
        "k2-bluestein")."""
        n = C.c_int()
        _check(lib().pft_dplan_second_pass(self._h, C.byref(n)))
        return {v: k for k, v in PASS2.items()}[n.value]

    def execute_ptr(self, d_in: int, d_out: int, batch: int = 1, in_stride: int = 0, d_ws: int = 0,
                    stream: int = 0, overlap: bool = False) -> None:
        """pft_execute_ex.  overlap=True (PFT_EXEC_OVERLAP_PREVIOUS): K1 may stream while the
        preceding kernel on the stream finishes; d_in must not be that kernel's output."""
        _check(lib().pft_execute_ex(self._h, C.c_void_p(d_in), batch, in_stride, C.c_void_p(d_out),
                                    C.c_void_p(d_ws or None), C.c_void_p(stream or None),
                                    EXEC_OVERLAP_PREVIOUS if overlap else 0))

    def execute_partial_ptr(self, d_in_local: int, d_partial: int, world: int = 1, rank: int = 0,
                            row_stride: int = 0, stream: int = 0) -> None:
        """K1 only, on rank `rank`'s slice (shard_layout) of A: writes the reducible slab."""
        _check(lib().pft_execute_partial(self._h, C.c_void_p(d_in_local), int(world), int(rank), row_stride,
                                         C.c_void_p(d_partial), C.c_void_p(stream or None)))

    def finalize_ptr(self, d_partial: int, d_out: int, batch: int = 1, stream: int = 0) -> None:
        _check(lib().pft_finalize(self._h, C.c_void_p(d_partial), batch, C.c_void_p(d_out),
                                  C.c_void_p(stream or None)))

    def status(self, stream: int = 0, reset: bool = True, d_ws: int = 0) -> int:
        """Non-finite flag word of workspace d_ws (0 = the plan's own workspace)."""
        f = C.c_int()
        _check(lib().pft_workspace_status(self._h, C.c_void_p(d_ws or None), C.c_void_p(stream or None), C.byref(f),
                                          int(reset)))
        return f.value

    def execute_host(self, a: np.ndarray, batch: int = 1) -> np.ndarray:
        """End-to-end: host input -> H2D -> kernels -> D2H (raises on non-finite input)."""
        a = np.ascontiguousarray(a, dtype=np.complex128)
        if a.size != self.plan.N * batch:
            raise PftValueError(6, f"length mismatch: got {a.size}, plan N*batch = {self.plan.N * batch}")
        out = np.zeros(batch * (2 * self.plan.M + 1), dtype=np.complex128)
        _check(lib().pft_execute_host(self._h, _ptr(a), batch, _ptr(out), None, None, None))
        return out


def naive_dft(a, first_m: int, count: int) -> np.ndarray:
    """Exact-angle direct DFT on the GPU at bins first_m .. first_m + count - 1:
    the verification path of the CLI (not the transform)."""
    a = np.ascontiguousarray(np.asarray(a), dtype=np.complex128).reshape(-1)
    out = np.zeros(max(count, 1), dtype=np.complex128)
    _check(lib().pft_naive_dft_host(_ptr(a), a.size, int(first_m), int(count), _ptr(out)))
    return out[:count]


def execute(plan: PftPlan, a, device: int = 0) -> PartialSpectrum:
    """Algorithm 2 on the GPU: host vector in, PartialSpectrum out."""
    a = np.ascontiguousarray(np.asarray(a), dtype=np.complex128).reshape(-1)
    if a.size != plan.N:
        raise PftValueError(6, f"execute: length mismatch (a.len={a.size}, plan.N={plan.N})")
    vals = plan.device_plan(device).execute_host(a)
    return PartialSpectrum(plan.range, vals, plan.plan_id)


# ----------------------------------------------------------------------------- sharding + inputs

@dataclasses.dataclass(frozen=True)
class ShardLayout:
    """Contraction-axis slice of one rank (pft_shard_info): mirror column pairs
    (l, q-l) for l in [pair_begin, pair_end), plus the unpaired columns on rank 0."""
    pair_begin: int
    pair_end: int
    row_len: int
    front_col: int
    mirror_col: int
    single0_col: int
    singleh_col: int


def shard_layout(q: int, world: int, rank: int) -> ShardLayout:
    info = _capi.ShardInfo()
    _check(lib().pft_shard_layout(int(q), int(world), int(rank), C.byref(info)))
    return ShardLayout(info.pair_begin, info.pair_end, info.row_len, info.front_col, info.mirror_col,
                       info.single0_col, info.singleh_col)


def shard_gather(a, p: int, q: int, world: int, rank: int) -> np.ndarray:
    """Host scatter of the global signal into `rank`'s local layout (p x row_len)."""
    a = np.ascontiguousarray(a, dtype=np.complex128).reshape(-1)
    v = shard_layout(q, world, rank)
    out = np.zeros(max(p * v.row_len, 1), dtype=np.complex128)
    _check(lib().pft_shard_gather_host(int(p), int(q), int(world), int(rank), _ptr(a), _ptr(out), v.row_len))
    return out[:p * v.row_len].reshape(p, v.row_len)


def sparse_tones(seed: int, n: int, lo: int, hi: int) -> tuple[np.ndarray, np.ndarray]:
    f = np.zeros(max(n, 1), dtype=np.int64)
    a = _cbuf(n)
    _check(lib().pft_sparse_tones(int(seed), int(n), int(lo), int(hi), _ptr(f), _ptr(a)))
    return f[:n].copy(), a[:n].copy()


KIND_UNIFORM, KIND_NORMAL, KIND_SPARSE = 0, 1, 2


def _desc(kind: int, seed: int, N: int, offset: int, freqs=None, amps=None, sigma: float = 0.0):
    d = _capi.SignalDesc()
    d.kind, d.seed, d.N, d.index_offset = kind, seed, N, offset
    keep = []
    if kind == KIND_SPARSE:
        f = np.ascontiguousarray(freqs, dtype=np.int64)
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        keep = [f, a]
        d.n_tones = len(f)
        d.freqs = f.ctypes.data_as(C.POINTER(C.c_int64))
        d.amps = a.ctypes.data_as(C.POINTER(c128))
        d.sigma = sigma
    return d, keep


def generate_signal(kind: int, seed: int, count: int, N: int = 0, offset: int = 0, freqs=None, amps=None,
                    sigma: float = 0.0) -> np.ndarray:
    """Seeded synthetic input on the host (bit-identical to the device generator for kind 0)."""
    d, keep = _desc(kind, seed, N, offset, freqs, amps, sigma)
    out = np.zeros(max(count, 1), dtype=np.complex128)
    _check(lib().pft_generate_host(C.byref(d), _ptr(out), count))
    del keep
    return out[:count]


def generate_signal_device(d_out: int, kind: int, seed: int, count: int, N: int = 0, offset: int = 0,
                           freqs=None, amps=None, sigma: float = 0.0, stream: int = 0) -> None:
    d, keep = _desc(kind, seed, N, offset, freqs, amps, sigma)
    _check(lib().pft_generate_device(C.byref(d), C.c_void_p(d_out), count, C.c_void_p(stream or None)))
    del keep


# ----------------------------------------------------------------------------- data formats

SIGNAL_CSV, SIGNAL_F64LE = 0, 1


def _signal_format(path: str, fmt: Optional[int]) -> int:
    if fmt is not None:
        return int(fmt)
    return SIGNAL_CSV if str(path).lower().endswith(".csv") else SIGNAL_F64LE


def read_signal(path, fmt: Optional[int] = None) -> tuple[np.ndarray, bool]:
    """SignalFile read (SPEC.md cli "SignalFile"): csv rows "re" / "re,im", or f64le with the
    16-byte {"PFTS", u32 complex flag, u32 length} header.  Returns (complex128 values,
    is_complex).  Format from the extension (.csv) unless given."""
    f = _signal_format(path, fmt)
    n, cx = C.c_uint64(), C.c_int()
    _check(lib().pft_signal_read(str(path).encode(), f, None, 0, C.byref(n), C.byref(cx)))
    out = np.zeros(n.value, dtype=np.complex128)
    _check(lib().pft_signal_read(str(path).encode(), f, _ptr(out), out.size, C.byref(n), C.byref(cx)))
    return out, bool(cx.value)


def write_signal(path, values, fmt: Optional[int] = None, is_complex: Optional[bool] = None) -> None:
    v = np.ascontiguousarray(np.asarray(values, dtype=np.complex128))
    if is_complex is None:
        is_complex = bool(np.iscomplexobj(values))
    _check(lib().pft_signal_write(str(path).encode(), _signal_format(path, fmt), _ptr(v), v.size, int(is_complex)))


def write_spectrum_csv(path, spectrum: "PartialSpectrum") -> None:
    """cmd_transform output: CSV "m,re,im" over [mu - M, mu + M], bit-exact on re-read."""
    v = np.ascontiguousarray(spectrum.values, dtype=np.complex128)
    _check(lib().pft_spectrum_write_csv(str(path).encode(), int(spectrum.range.mu), int(spectrum.range.half_width),
                                        _ptr(v)))


def read_spectrum_csv(path) -> tuple[int, np.ndarray]:
    """(first m, values) of a "m,re,im" file."""
    n, m0 = C.c_uint64(), C.c_int64()
    _check(lib().pft_spectrum_read_csv(str(path).encode(), C.byref(m0), None, 0, C.byref(n)))
    out = np.zeros(n.value, dtype=np.complex128)
    _check(lib().pft_spectrum_read_csv(str(path).encode(), C.byref(m0), _ptr(out), out.size, C.byref(n)))
    return m0.value, out


# ----------------------------------------------------------------------------- anomaly pipeline

def anomaly_from_coeffs(x, coeffs, M: int, k: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """cmd_anomaly scoring (SPEC.md cli; §4.4) from coefficients on R_{0,M}
    (coeffs[s] = a_{s-M}): (top-k indices, their scores, fitted curve)."""
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    cv = np.ascontiguousarray(np.asarray(coeffs, dtype=np.complex128))
    if cv.size != 2 * M + 1:
        raise PftValueError(6, f"coeffs length {cv.size} != 2M+1 = {2 * M + 1}")
    idx = np.zeros(k, dtype=np.uint64)
    sc = np.zeros(k, dtype=np.float64)
    fit = np.zeros(xv.size, dtype=np.float64)
    _check(lib().pft_anomaly_from_coeffs(_ptr(xv), xv.size, _ptr(cv), M, k, _ptr(idx), _ptr(sc), _ptr(fit)))
    return idx.astype(np.int64), sc, fit


_ANOMALY_PLANS: dict = {}


def anomaly(x, M: int, k: int, p: Optional[int] = None, epsilon: float = DEFAULT_EPSILON,
            device: int = 0) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """cmd_anomaly with source = pft: coefficients on R_{0,M} from one GPU execute, then the
    scoring of anomaly_from_coeffs (inside the library: pft_anomaly)."""
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    key = (xv.size, M, p, epsilon, device)
    d = _ANOMALY_PLANS.get(key)
    if d is None:  # plans are immutable and reusable: one per shape, not per call
        d = DevicePlan(build_plan(xv.size, M, 0, p, epsilon), device=device)
        _ANOMALY_PLANS[key] = d
    idx = np.zeros(k, dtype=np.uint64)
    sc = np.zeros(k, dtype=np.float64)
    fit = np.zeros(xv.size, dtype=np.float64)
    _check(lib().pft_anomaly(d._h, _ptr(xv), k, _ptr(idx), _ptr(sc), _ptr(fit)))
    return idx.astype(np.int64), sc, fit
