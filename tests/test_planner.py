"""planner module (Algorithm 1) and the shard layout."""
from __future__ import annotations

import math

import numpy as np
import pytest


def test_divisors(pft):
    assert pft.divisors(12) == [1, 2, 3, 4, 6, 12]
    assert pft.divisors(19735) == [1, 5, 3947, 19735]           # SPEC.md:143 (PAPER §4.2)
    assert pft.divisors(1000003) == [1, 1000003]                # prime
    assert pft.divisors(1) == [1]
    for n in (360, 6220800, 2 ** 30):
        d = pft.divisors(n)
        assert d == sorted(d) and all(n % x == 0 for x in d)
        assert len(d) == sum(1 for x in range(1, int(math.isqrt(n)) + 1) if n % x == 0) * 2 - (
            1 if math.isqrt(n) ** 2 == n else 0)


def test_select_divisor_air_condition(pft):
    """N = 19735, M = 125 -> p = 3947."""
    for eps in (1e-6, 1e-12):
        p, est = pft.select_divisor(19735, 125, epsilon=eps)
        assert p == 3947 and est.p == 3947


def test_select_divisor_m0_and_errors(pft):
    p, est = pft.select_divisor(19735, 0)
    assert (p, est.r) == (5, 1)
    assert pft.select_divisor(3947, 0)[0] == 3947                # prime N -> p = N
    with pytest.raises(ValueError):
        pft.select_divisor(1, 0)                                 # N = 1 rejected
    with pytest.raises(ValueError):
        pft.select_divisor(16, 17)                               # M > N rejected


def lemma2_window_has_divisor(divs, M, b):
    lo, hi = M / math.sqrt(b), M * math.sqrt(b)
    return any(lo <= d < hi for d in divs)


def test_lemma2_examples(pft):
    assert lemma2_window_has_divisor([512], 2 ** 9, 2) and 512 in pft.divisors(2 ** 22)
    assert lemma2_window_has_divisor(pft.divisors(12), 12, 3)


def test_lemma2_property(pft):
    """Acceptance #4: 500 random b-smooth N <= 1e6 per b in {2,3,5,7}."""
    rng = np.random.default_rng(4)
    for b in (2, 3, 5, 7):
        primes = [q for q in (2, 3, 5, 7) if q <= b]
        count = 0
        while count < 500:
            N = 1
            for _ in range(rng.integers(1, 25)):
                f = int(rng.choice(primes))
                if N * f > 10 ** 6:
                    break
                N *= f
            M = int(rng.integers(1, N + 1))
            assert lemma2_window_has_divisor(pft.divisors(N), M, b), (N, M, b)
            count += 1


def test_min_terms(pft):
    assert pft.min_terms(1e-12, 0, 32) == 1
    assert pft.min_terms(1e-6, 1, 32) == 4                        # SPEC.md:163, App. A.1
    t = pft.ScopeTable.default()
    for M, p in [(1, 32), (1, 8), (1, 2), (1, 1), (2, 1)]:
        rs = [pft.min_terms(eps, M, p, t) for eps in (1e-2, 1e-4, 1e-6, 1e-8, 1e-12)]
        assert rs == sorted(rs), (M, p, rs)
    with pytest.raises(ValueError) as e:
        pft.min_terms(1e-12, 1000, 1)                             # ratio out of range
    assert e.value.status == 5
    with pytest.raises(ValueError) as e:
        pft.min_terms(3e-7, 1, 32)                                # eps not in table
    assert e.value.status == 4


def test_spec_cost_model_picks_match_survey(pft):
    """SURVEY.md App. A.2 (SPEC cost model over this build's table at eps = 1e-12)."""
    cases = {(2 ** 20, 64): (16384, 5), (2 ** 24, 64): (65536, 4), (2 ** 24, 1024): (65536, 6),
             (2 ** 24, 16384): (262144, 8), (2 ** 16, 256): (2048, 10), (6220800, 1000): (62208, 6),
             (2 ** 30, 4096): (4194304, 4)}
    for (N, M), (p, r) in cases.items():
        got, est = pft.select_divisor(N, M)
        assert (got, est.r) == (p, r), (N, M)


def test_device_divisor_model(pft):
    """pft_select_divisor_device (B200 time model, DESIGN.md §2 'Plan choice'): a valid divisor
    whose r is min_terms(p); at the calibration point (C2b) it picks the measured-best p = 2^14
    (SPEC's CPU model picks 2^16)."""
    for N, M in [(2 ** 20, 64), (2 ** 24, 64), (2 ** 24, 1024), (2 ** 24, 16384), (2 ** 16, 256),
                 (6220800, 1000), (2 ** 30, 4096), (32000, 100)]:
        p, r, est = pft.select_divisor_device(N, M)
        assert N % p == 0 and 1 < p < N
        assert r == pft.min_terms(1e-12, M, p)
        assert est > 0
    assert pft.select_divisor_device(2 ** 24, 1024)[0] == 2 ** 14
    with pytest.raises(ValueError):
        pft.select_divisor_device(2 ** 20, 64, n_sms=0)


def test_cost_model_sanity(pft):
    """the selected p minimises r (N + p log2 p + M) over all valid divisors."""
    for N, M in [(2 ** 20, 512), (32000, 100), (6220800, 1000)]:
        p, est = pft.select_divisor(N, M)
        for d in pft.divisors(N)[1:]:
            try:
                r = pft.min_terms(1e-12, M, d)
            except ValueError:
                continue
            assert est.cost <= r * (N + d * math.log2(max(d, 2)) + M) + 1e-6


def test_build_plan_examples(pft, oracle):
    plan = pft.build_plan(16, 2, 0, 4, 1e-6)
    assert plan.q == 4
    assert np.all(plan.B[2, 1:] == 0) and plan.B[2, 0] == plan.w[0]   # invariant SPEC.md:127
    assert np.all(plan.phase == 1)                                # mu = 0
    plan = pft.build_plan(32000, 100, 0, None, 1e-6)
    assert 32000 % plan.p == 0 and plan.p * plan.q == 32000
    assert pft.scope_xi(1e-6, plan.r)[0] >= 100 / plan.p


def test_build_plan_errors(pft):
    with pytest.raises(ValueError) as e:
        pft.build_plan(16, 2, 0, 5, 1e-6)
    assert e.value.status == 2                                    # p does not divide N
    with pytest.raises(ValueError) as e:
        pft.build_plan(16, 9, 0, 4, 1e-6)
    assert e.value.status == 3                                    # M > N/2
    with pytest.raises(ValueError) as e:
        pft.build_plan(16, 2, 0, 4, 5e-7)
    assert e.value.status == 4                                    # eps missing from table


@pytest.mark.parametrize("N,M,mu,p", [(4096, 32, 37, 128), (4096, 32, -200, 64), (105 * 64, 20, 11, 15 * 64),
                                      (2 ** 20, 64, 2 ** 18, 2 ** 14), (6220800, 1000, -12345, 62208),
                                      (2 ** 30, 4096, 2 ** 29 + 7, 2 ** 16)])
def test_plan_tables_match_formulas(pft, oracle, N, M, mu, p):
    """B[l][j] = e^{-2 pi i mu (l-q/2)/N} w_j (1-2l/q)^j, independently re-derived
    by the oracle; post_powers ((m-mu)/p)^j and post_twiddles e^{-pi i m/p}."""
    plan = pft.build_plan(N, M, mu, p, 1e-12)
    if plan.q <= 1 << 16:
        B, tv = oracle.build_B(N, plan.q, plan.r, mu, plan.w)
        np.testing.assert_allclose(plan.B, B, rtol=0, atol=4e-16 * np.abs(plan.w).max())
        np.testing.assert_array_equal(plan.tvals, tv)
    s = np.arange(2 * M + 1)
    x = (s - M) / plan.p
    np.testing.assert_allclose(plan.post_powers, x[:, None] ** np.arange(plan.r)[None, :], rtol=1e-15, atol=0)
    m = mu - M + s
    ang = np.pi * ((-m) % (2 * plan.p)) / plan.p
    np.testing.assert_allclose(plan.post_twiddles, np.exp(1j * ang), rtol=0, atol=2e-15)


def test_plan_determinism(pft):
    """Identical inputs -> bit-identical plans."""
    a = pft.build_plan(2 ** 20, 64, 12345, None, 1e-12)
    b = pft.build_plan(2 ** 20, 64, 12345, None, 1e-12)
    assert a.plan_id == b.plan_id
    for name in ("B", "w", "phase", "tvals", "post_powers", "post_twiddles"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    c = pft.build_plan(2 ** 20, 64, 12346, None, 1e-12)
    assert c.plan_id != a.plan_id


def test_odd_q_and_large_mu_phase(pft):
    """SURVEY.md Hard part 4: for odd q the B phase flips by (-1)^q under mu -> mu + N."""
    N, p = 105 * 64, 15 * 64  # q = 7
    a = pft.build_plan(N, 20, 11, p, 1e-12)
    b = pft.build_plan(N, 20, 11 + N, p, 1e-12)
    c = pft.build_plan(N, 20, 11 + 2 * N, p, 1e-12)
    np.testing.assert_allclose(b.phase, -a.phase, atol=1e-15)
    np.testing.assert_allclose(c.phase, a.phase, atol=1e-15)


def test_plan_json(pft):
    import json
    d = json.loads(pft.build_plan(2 ** 24, 1024, 2 ** 22, 2 ** 15, 1e-12).json())
    assert (d["N"], d["M"], d["mu"], d["p"], d["q"], d["r"]) == (2 ** 24, 1024, 2 ** 22, 2 ** 15, 512, 7)
    assert d["achieved_epsilon"] <= d["epsilon"] and d["estimated_cost"] > 0


@pytest.mark.parametrize("q", [1, 2, 3, 7, 8, 64, 255, 512, 1000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_layout_partitions_columns(pft, q, world):
    """Contraction-axis sharding: the ranks' local columns cover [0, q) exactly once, in
    mirror pairs, with the unpaired columns on rank 0."""
    seen = []
    for rank in range(world):
        v = pft.shard_layout(q, world, rank)
        a = np.arange(q, dtype=np.complex128)  # one row whose value is its column index
        local = pft.shard_gather(a, 1, q, world, rank)[0]
        cols = [int(z.real) for z in local]
        assert len(cols) == v.row_len
        n = v.pair_end - v.pair_begin
        for t in range(n):
            assert cols[v.front_col + t] == v.pair_begin + t
            assert cols[v.mirror_col - t] == q - (v.pair_begin + t)
        if v.single0_col >= 0:
            assert rank == 0 and cols[v.single0_col] == 0
        if v.singleh_col >= 0:
            assert rank == 0 and cols[v.singleh_col] == q // 2
        seen += cols
    assert sorted(seen) == list(range(q))


def test_shard_layout_errors(pft):
    with pytest.raises(ValueError):
        pft.shard_layout(512, 2, 2)
    with pytest.raises(ValueError):
        pft.shard_layout(0, 1, 0)


def test_select_divisor_sharded_collective_term(pft):
    """pft_select_divisor_sharded (the comm-aware planner): C5 (N = 2^30,
    M = 2^12) over 1..8 GPUs.  The pick divides N and is feasible; the modelled time falls with
    G; the reduced slab (16 p r bytes) stays far below SPEC's p = 2^22 choice (268 MB, SURVEY.md
    §8(e)); and with G > 1 the collective term never favours a larger slab than G = 1 does."""
    from paper_2008_12559_b200.sharded import select_divisor_sharded
    N, M = 2 ** 30, 2 ** 12
    prev_us, slab1 = None, None
    for G in (1, 2, 4, 8):
        p, r, us = select_divisor_sharded(N, M, G)
        assert N % p == 0 and r == pft.min_terms(1e-12, M, p)
        slab = 16 * p * r
        assert slab <= 64 * 2 ** 20
        if prev_us is not None:
            assert us < prev_us
            assert slab <= slab1
        else:
            slab1 = slab
        prev_us = us
