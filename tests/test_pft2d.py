"""2-D PFT (Algorithms 3-4).

CPU: the oracle's execute_2d (block contraction B1^T A B2 in either parenthesization, row-column
2-D FFT, Eq. (14)) against an exact-angle 2-D DFT and SPEC's examples/invariants.
GPU (marked): the device path (two batched 1-D passes, pft_execute_2d) against that oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

GATE = 1e-11


def rel_l2(x, y) -> float:
    return float(np.linalg.norm(np.asarray(x) - np.asarray(y)) / np.linalg.norm(y))


def grid(seed, N1, N2):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((N1, N2)) + 1j * rng.standard_normal((N1, N2))


def test_parenthesization_rule(pft):
    """q1=8, r2=2, q2=4, r1=4 -> LeftFirst 160 vs RightFirst 128 -> RightFirst;
    the symmetric case ties -> LeftFirst."""
    assert pft.parenthesization(8, 4, 4, 2) == "RightFirst"
    assert pft.parenthesization(16, 5, 16, 5) == "LeftFirst"


def test_build_plan_2d(pft):
    """per-dimension plans; (64,64),(4,4),eps 1e-6 is valid; M_d > N_d/2 fails."""
    P = pft.build_plan_2d(64, 64, 4, 4, 0, 0, epsilon=1e-6)
    for pl, N in ((P.plan1, 64), (P.plan2, 64)):
        assert pl.p * pl.q == N and pl.r >= 1
    assert P.parenthesization == "LeftFirst"
    with pytest.raises(ValueError):
        pft.build_plan_2d(8, 8, 5, 1, 0, 0)


@pytest.mark.parametrize("order", ["LeftFirst", "RightFirst"])
def test_oracle_2d_impulse_and_separable(pft, oracle, order):
    """the impulse spectrum is all ones; a separable grid gives the outer
    product of the 1-D spectra."""
    N1, N2, M1, M2, mu1, mu2 = 64, 96, 5, 7, 3, -11
    P = pft.build_plan_2d(N1, N2, M1, M2, mu1, mu2)
    bound = P.achieved_epsilon ** 2 + 2 * P.achieved_epsilon
    d = np.zeros((N1, N2), dtype=np.complex128)
    d[0, 0] = 1
    assert np.max(np.abs(oracle.execute_2d(P.plan1, P.plan2, d, order) - 1)) <= bound + 1e-14
    f, g = grid(1, 1, N1)[0], grid(2, 1, N2)[0]
    out = oracle.execute_2d(P.plan1, P.plan2, np.outer(f, g), order)
    outer = np.outer(oracle.naive_dft(f, mu1, M1), oracle.naive_dft(g, mu2, M2))
    assert np.max(np.abs(out - outer)) <= (np.abs(f).sum() * np.abs(g).sum()) * bound + 1e-12


def test_oracle_2d_random_and_parenthesizations(pft, oracle):
    """N=(128,128), M=(8,8), mu=(5,-3): rel l2 vs the naive 2-D DFT < 1e-6 (1e-11 at
    eps = 1e-12); both parenthesizations agree within 1e-10."""
    P = pft.build_plan_2d(128, 128, 8, 8, 5, -3)
    a = grid(3, 128, 128)
    L = oracle.execute_2d(P.plan1, P.plan2, a, "LeftFirst")
    R = oracle.execute_2d(P.plan1, P.plan2, a, "RightFirst")
    assert rel_l2(L, R) <= 1e-10
    assert rel_l2(L, oracle.naive_dft_2d(a, 5, 8, -3, 8)) < 1e-11


def test_oracle_2d_theorem4(pft, oracle):
    """Theorem 4: max abs error <= ||a||_1 (eps^2 + 2 eps) over random small cases
    (with binary64 roundoff slack, as for Theorem 2)."""
    rng = np.random.default_rng(7)
    for t in range(20):
        N1, N2 = int(rng.choice([16, 24, 32, 48])), int(rng.choice([16, 20, 32, 40]))
        M1, M2 = int(rng.integers(0, N1 // 4 + 1)), int(rng.integers(0, N2 // 4 + 1))
        mu1, mu2 = int(rng.integers(-50, 50)), int(rng.integers(-50, 50))
        eps = float(rng.choice([1e-6, 1e-9, 1e-12]))
        P = pft.build_plan_2d(N1, N2, M1, M2, mu1, mu2, epsilon=eps)
        a = grid(100 + t, N1, N2)
        err = np.max(np.abs(oracle.execute_2d(P.plan1, P.plan2, a, P.parenthesization)
                            - oracle.naive_dft_2d(a, mu1, M1, mu2, M2)))
        l1 = np.abs(a).sum()
        assert err <= l1 * (P.achieved_epsilon ** 2 + 2 * P.achieved_epsilon) + 64 * 2.2e-16 * l1, t


CASES_2D = [
    # (N1, N2, M1, M2, mu1, mu2, eps)
    (64, 64, 4, 4, 0, 0, 1e-6),
    (128, 128, 8, 8, 5, -3, 1e-12),
    (96, 200, 6, 10, -7, 33, 1e-12),
    (1024, 2048, 20, 40, 300, -77, 1e-12),
    (4096, 4096, 64, 32, 1000, 2000, 1e-12),
]


@pytest.mark.gpu
@pytest.mark.parametrize("N1,N2,M1,M2,mu1,mu2,eps", CASES_2D)
def test_execute_2d_matches_oracle(pft, oracle, N1, N2, M1, M2, mu1, mu2, eps):
    P = pft.build_plan_2d(N1, N2, M1, M2, mu1, mu2, epsilon=eps)
    a = grid(N1 + N2, N1, N2)
    gpu = pft.execute_2d(P, a).values
    ref = oracle.execute_2d(P.plan1, P.plan2, a, P.parenthesization)
    assert gpu.shape == (2 * M1 + 1, 2 * M2 + 1)
    assert rel_l2(gpu, ref) <= GATE
    if N1 * N2 <= 2 ** 16:
        exact = oracle.naive_dft_2d(a, mu1, M1, mu2, M2)
        assert abs(rel_l2(gpu, exact) - rel_l2(ref, exact)) <= 0.05 * rel_l2(ref, exact) + 2e-14
        l1 = np.abs(a).sum()
        assert np.max(np.abs(gpu - exact)) <= l1 * (P.achieved_epsilon ** 2 + 2 * P.achieved_epsilon) + 1e-9
    assert P.plan1.mu == mu1 and abs(pft.execute_2d(P, a).at(mu1, mu2) - gpu[M1, M2]) == 0


@pytest.mark.gpu
def test_execute_2d_device_pointers_and_nonfinite(pft, oracle):
    """pft_execute_2d on device buffers with a caller workspace (zeroed once, reused); a NaN
    input is reported as PFT_ERR_NON_FINITE by the host entry point."""
    import torch
    N1, N2, M1, M2 = 256, 512, 9, 17
    P = pft.build_plan_2d(N1, N2, M1, M2, -4, 100)
    a = grid(5, N1, N2)
    x = torch.from_numpy(a).cuda()
    out = torch.empty((2 * M1 + 1) * (2 * M2 + 1), dtype=torch.complex128, device="cuda")
    ws = torch.zeros(-(-P.workspace_bytes() // 16), dtype=torch.complex128, device="cuda")
    for _ in range(2):
        P.execute_ptr(x.data_ptr(), out.data_ptr(), ws.data_ptr())
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(2 * M1 + 1, 2 * M2 + 1)
    assert rel_l2(got, oracle.execute_2d(P.plan1, P.plan2, a)) <= GATE
    a[7, 9] = np.nan
    with pytest.raises(ValueError) as e:
        pft.execute_2d(P, a)
    assert e.value.status == 7


@pytest.mark.gpu
@pytest.mark.parametrize("N1,N2,M1,M2,mu1,mu2", [(1024, 2048, 16, 64, 3, -50), (512, 4096, 40, 100, -9, 7)])
def test_autotune_2d_plan_parity(pft, oracle, N1, N2, M1, M2, mu1, mu2):
    """autotune_2d picks p per axis on the device (rows at batch N1, columns at batch 2M2+1);
    the tuned plan passes the same gate against the oracle run on that plan."""
    import torch
    P = pft.build_plan_2d(N1, N2, M1, M2, mu1, mu2)
    a = grid(77, N1, N2)
    x = torch.from_numpy(a).cuda()
    T = pft.autotune_2d(P, x.data_ptr())
    assert N1 % T.plan1.p == 0 and N2 % T.plan2.p == 0
    assert (T.plan1.M, T.plan2.M, T.plan1.mu, T.plan2.mu) == (M1, M2, mu1, mu2)
    gpu = pft.execute_2d(T, a).values
    assert rel_l2(gpu, oracle.execute_2d(T.plan1, T.plan2, a, T.parenthesization)) <= GATE
