"""CPU oracle for the PFT execute path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference leg
may import this package.  It loads oracle/_build/liboracle.so (oracle.cpp, a plain
restatement of SPEC.md's transform and oracle modules; see its header for the file:line
each function follows).  Parity pinning: SPEC.md's known-answer examples and an
independent exact DFT (tests/golden, generated with mpmath) -- the reference ships no
implementation to run.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        vp, sz, u64, i64, d, i = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int64, C.c_double, C.c_int
        sig = {
            "oracle_fft": (i, [sz, vp, vp]),
            "oracle_ifft": (i, [sz, vp, vp]),
            "oracle_batch_fft_columns": (i, [sz, sz, vp, vp]),
            "oracle_matmul": (i, [sz, sz, sz, vp, sz, vp, vp]),
            "oracle_build_B": (i, [u64, u64, i, i64, vp, vp, vp]),
            "oracle_post": (i, [u64, u64, i64, i, vp, vp, vp, vp]),
            "oracle_execute": (i, [u64, u64, i64, u64, i, vp, vp, vp, vp, vp]),
            "oracle_contract_slice": (i, [u64, u64, i, u64, u64, vp, vp, vp]),
            "oracle_naive_dft": (i, [u64, vp, i64, u64, vp]),
            "oracle_l1": (d, [vp, u64]),
            "oracle_compare": (i, [vp, vp, u64, d, d, i, vp]),
            "oracle_certify": (d, [vp, i, d, d]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _ok(rc: int) -> None:
    if rc != 0:
        raise ValueError(f"oracle call failed (rc={rc})")


def fft(x) -> np.ndarray:
    x = _c(x)
    out = np.empty_like(x)
    _ok(lib().oracle_fft(len(x), _p(x), _p(out)))
    return out


def ifft(x) -> np.ndarray:
    x = _c(x)
    out = np.empty_like(x)
    _ok(lib().oracle_ifft(len(x), _p(x), _p(out)))
    return out


def batch_fft_columns(Cm) -> np.ndarray:
    Cm = _c(Cm)
    p, r = Cm.shape
    out = np.empty_like(Cm)
    _ok(lib().oracle_batch_fft_columns(p, r, _p(Cm), _p(out)))
    return out


def matmul(A, B) -> np.ndarray:
    A, B = _c(A), _c(B)
    p, q = A.shape
    q2, r = B.shape
    if q != q2:
        raise ValueError("dimension mismatch")
    out = np.zeros((p, r), dtype=np.complex128)
    _ok(lib().oracle_matmul(p, q, r, _p(A), q, _p(B), _p(out)))
    return out


def build_B(N: int, q: int, r: int, mu: int, w):
    w = _c(w)
    B = np.zeros((q, r), dtype=np.complex128)
    tv = np.zeros(q)
    _ok(lib().oracle_build_B(N, q, r, mu, _p(w), _p(B), tv.ctypes.data_as(C.c_void_p)))
    return B, tv


def execute(plan, a) -> np.ndarray:
    """Algorithm 2 on the CPU with the plan's own tables (same plan as the GPU)."""
    a = _c(a).reshape(-1)
    if a.size != plan.N:
        raise ValueError("length mismatch")
    B = _c(plan.B)
    pp = np.ascontiguousarray(plan.post_powers, dtype=np.float64)
    pt = _c(plan.post_twiddles)
    out = np.zeros(2 * plan.M + 1, dtype=np.complex128)
    _ok(lib().oracle_execute(plan.N, plan.M, plan.mu, plan.p, plan.r, _p(B), pp.ctypes.data_as(C.c_void_p),
                             _p(pt), _p(a), _p(out)))
    return out


def contract_slice(plan, a, l0: int, lq: int) -> np.ndarray:
    """Partial C (p x r) over columns [l0, l0+lq) of A -- host model of one shard."""
    a = _c(a).reshape(-1)
    B = _c(plan.B)
    out = np.zeros((plan.p, plan.r), dtype=np.complex128)
    _ok(lib().oracle_contract_slice(plan.p, plan.q, plan.r, l0, lq, _p(B), _p(a), _p(out)))
    return out


def post(plan, Chat) -> np.ndarray:
    Chat = _c(Chat)
    pp = np.ascontiguousarray(plan.post_powers, dtype=np.float64)
    pt = _c(plan.post_twiddles)
    out = np.zeros(2 * plan.M + 1, dtype=np.complex128)
    _ok(lib().oracle_post(plan.p, plan.M, plan.mu, plan.r, _p(Chat), pp.ctypes.data_as(C.c_void_p), _p(pt),
                          _p(out)))
    return out


def naive_dft(a, mu: int, M: int) -> np.ndarray:
    """Exact-angle direct DFT on R_{mu,M}."""
    a = _c(a).reshape(-1)
    out = np.zeros(2 * M + 1, dtype=np.complex128)
    _ok(lib().oracle_naive_dft(len(a), _p(a), mu, M, _p(out)))
    return out


def l1(a) -> float:
    a = _c(a).reshape(-1)
    return float(lib().oracle_l1(_p(a), a.size))


class _Report(C.Structure):
    _fields_ = [("relative_l2", C.c_double), ("max_abs", C.c_double), ("l1_input", C.c_double),
                ("bound", C.c_double), ("bound_satisfied", C.c_int)]


@dataclasses.dataclass
class ErrorReport:
    """SPEC.md:337-340."""
    relative_l2: float
    max_abs: float
    l1_input: float
    bound: float
    bound_satisfied: bool


def compare(actual, estimate, l1_input: float, epsilon: float, two_d: bool = False) -> ErrorReport:
    actual, estimate = _c(actual).reshape(-1), _c(estimate).reshape(-1)
    if actual.size != estimate.size:
        raise ValueError("range mismatch")
    rep = _Report()
    _ok(lib().oracle_compare(_p(actual), _p(estimate), actual.size, l1_input, epsilon, int(two_d), C.byref(rep)))
    return ErrorReport(rep.relative_l2, rep.max_abs, rep.l1_input, rep.bound, bool(rep.bound_satisfied))


def certify(coeffs, xi: float, u: float = np.pi) -> float:
    c = _c(coeffs)
    return float(lib().oracle_certify(_p(c), len(c), float(xi), float(u)))


def execute_2d(plan1, plan2, a, parenthesization: str = "LeftFirst") -> np.ndarray:
    """execute_2d (Algorithm 4) on the CPU: per (k1, k2) block
    C = B1^T A B2 in the given parenthesization (oracle matmul, ascending l), the r1 r2 2-D
    FFTs of size p1 x p2 as row-column passes of the 1-D provider, then the
    Eq. (14) weighted sum with the per-dimension post factors of the two 1-D plans."""
    p1, q1, r1, p2, q2, r2 = plan1.p, plan1.q, plan1.r, plan2.p, plan2.q, plan2.r
    A4 = _c(a).reshape(p1, q1, p2, q2)  # A^{(k1,k2)}[l1][l2] = a[q1 k1 + l1][q2 k2 + l2]
    B1, B2 = _c(plan1.B), _c(plan2.B)
    if parenthesization == "LeftFirst":  # (B1^T A) B2
        T = matmul(A4.transpose(0, 2, 3, 1).reshape(-1, q1), B1).reshape(p1, p2, q2, r1)
        Cb = matmul(T.transpose(0, 1, 3, 2).reshape(-1, q2), B2).reshape(p1, p2, r1, r2)
    else:  # B1^T (A B2)
        T = matmul(A4.reshape(-1, q2), B2).reshape(p1, q1, p2, r2)
        Cb = matmul(T.transpose(0, 2, 3, 1).reshape(-1, q1), B1).reshape(p1, p2, r2, r1).transpose(0, 1, 3, 2)
    # 2-D FFT over (k1, k2) for every (j1, j2): columns along k1, then along k2
    F = batch_fft_columns(Cb.reshape(p1, -1)).reshape(p1, p2, r1, r2)
    F = batch_fft_columns(F.transpose(1, 0, 2, 3).reshape(p2, -1)).reshape(p2, p1, r1, r2).transpose(1, 0, 2, 3)
    M1, M2 = plan1.M, plan2.M
    m1 = np.arange(plan1.mu - M1, plan1.mu + M1 + 1)
    m2 = np.arange(plan2.mu - M2, plan2.mu + M2 + 1)
    G = F[np.mod(m1, p1)][:, np.mod(m2, p2)]  # (W1, W2, r1, r2)
    pw1 = np.asarray(plan1.post_powers, dtype=np.float64).reshape(2 * M1 + 1, r1)
    pw2 = np.asarray(plan2.post_powers, dtype=np.float64).reshape(2 * M2 + 1, r2)
    S = np.einsum("abjk,aj,bk->ab", G, pw1, pw2)
    tw1 = _c(plan1.post_twiddles).reshape(-1)
    tw2 = _c(plan2.post_twiddles).reshape(-1)
    return S * tw1[:, None] * tw2[None, :]


def naive_dft_2d(a, mu1: int, M1: int, mu2: int, M2: int) -> np.ndarray:
    """Exact-angle 2-D DFT on the rectangle (separable: naive_dft along axis 2, then axis 1)."""
    a = _c(a)
    rows = np.stack([naive_dft(row, mu2, M2) for row in a])          # (N1, W2)
    return np.stack([naive_dft(col, mu1, M1) for col in rows.T]).T   # (W1, W2)
