"""minimax module: best_approx, scope_xi, translate_poly, ScopeTable."""
from __future__ import annotations

import math

import numpy as np
import pytest

PI = math.pi


def test_best_approx_degenerate(pft):
    """(r=1, xi=0, u=pi) -> constant 1, achieved 0 (Definition 1)."""
    P = pft.best_approx(1, 0.0, PI)
    assert list(P.coeffs) == [1.0]
    assert P.achieved_error == 0.0
    P = pft.best_approx(4, 0.5, 0.0)  # u = 0 degenerate clause
    assert P.coeffs[0] == 1.0 and np.all(P.coeffs[1:] == 0) and P.achieved_error == 0.0


def test_best_approx_r3_xi01(pft):
    """SPEC.md:59.  The stated '< 1e-4' is infeasible (the minimax floor of the odd part is
    ~(pi xi)^3/24 = 1.3e-3); assert the stated Taylor ceiling instead, plus a
    floor that shows the number is a real near-minimax error."""
    P = pft.best_approx(3, 0.1, PI)
    assert abs(P.coeffs[0] - 1) < 1e-2
    assert 1.0e-3 < P.achieved_error < (PI * 0.1) ** 3 / 6  # 5.2e-3
    # w = (1, 3.103i, -4.904)
    np.testing.assert_allclose(P.coeffs, [1.0, 3.103j, -4.904], atol=2e-3)


def test_rescaling_law(pft):
    """P(vx/u) approximates e^{vix} on |x| <= u xi / v with the same error."""
    for r, xi in [(2, 0.3), (5, 0.2), (9, 0.7)]:
        P1 = pft.best_approx(r, xi, PI)
        P2 = pft.best_approx(r, xi / 2, 2 * PI)
        assert abs(P1.achieved_error - P2.achieved_error) <= 1e-12 + 1e-9 * P1.achieved_error
        np.testing.assert_allclose(P2.coeffs, P1.coeffs * (2.0 ** np.arange(r)), rtol=1e-9, atol=1e-12)


def test_error_decreases_with_xi(pft):
    """at fixed r, error strictly decreases as xi decreases."""
    for r in (3, 7, 12):
        errs = [pft.best_approx(r, xi, PI).achieved_error for xi in (0.8, 0.4, 0.2, 0.1)]
        assert all(a > b for a, b in zip(errs, errs[1:])), errs


def test_value_at_zero(pft):
    """P(0) is within achieved_error of 1."""
    for r, xi in [(3, 0.1), (8, 0.5), (15, 1.0)]:
        P = pft.best_approx(r, xi, PI)
        assert abs(P(0.0) - 1.0) <= P.achieved_error


def test_scope_xi_examples(pft):
    """SPEC.md:68-70."""
    xi1, _ = pft.scope_xi(1e-3, 1)
    assert xi1 > 0
    x8, _ = pft.scope_xi(1e-2, 8)
    x9, _ = pft.scope_xi(1e-2, 9)
    assert x9 >= x8
    # minimal r with xi(1e-6, r) >= 1/32 is 4 (xi(1e-6,4)=0.03745)
    xs = {r: pft.scope_xi(1e-6, r)[0] for r in (3, 4)}
    assert xs[3] < 1 / 32 <= xs[4]


def test_scope_xi_certified_and_tight(pft, oracle):
    xi, P = pft.scope_xi(1e-12, 7)
    assert P.achieved_error <= 1e-12
    assert oracle.certify(P.coeffs, xi) <= 1e-12          # independent re-certification
    assert pft.best_approx(7, xi * 1.01, PI).achieved_error > 1e-12  # bisection tolerance 1e-3


def test_translate_poly(pft):
    """Lemma 1 / SPEC.md:76-80."""
    _, P = pft.scope_xi(1e-8, 10)
    Q = pft.translate_poly(P, PI, 0.0)
    np.testing.assert_array_equal(Q.coeffs, P.coeffs)  # mu = 0 -> identity
    P = pft.best_approx(8, 0.25, PI)
    Q = pft.translate_poly(P, PI, 3.0)
    x = np.linspace(2.75, 3.25, 4001)
    err = np.max(np.abs(Q(x) - np.exp(1j * PI * x)))
    # exact in real arithmetic; in binary64 the re-expanded coefficients carry round-off of
    # order eps_mach * sum_j |q_j| |x|^j ("within expansion round-off")
    roundoff = 64 * np.finfo(float).eps * np.sum(np.abs(Q.coeffs) * 3.25 ** np.arange(len(Q.coeffs)))
    assert err <= P.achieved_error + roundoff, (err, P.achieved_error, roundoff)
    assert err >= P.achieved_error * (1 - 1e-3)  # and it is the same error, not a better one


def test_default_table_shape(pft):
    t = pft.ScopeTable.default()
    assert len(t) == 13 * 25 and t.r_max == 25
    grid = t.epsilon_grid
    assert grid[0] == pytest.approx(1e-1) and grid[-1] == pytest.approx(1e-13)
    assert any(abs(e - 1e-12) < 1e-24 for e in grid)  # BASELINE.json's eps


def test_default_table_invariants(pft, oracle):
    """certified <= eps (re-checked independently); monotone in r and eps."""
    t = pft.ScopeTable.default()
    entries = t.entries
    by = {(round(math.log10(e.epsilon)), e.r): e for e in entries}
    for e in entries:
        assert e.achieved_error <= e.epsilon
    rng = np.random.default_rng(0)
    for e in rng.choice(entries, 20, replace=False):
        assert oracle.certify(e.coeffs, e.xi) <= e.epsilon
    for k in range(1, 14):
        xs = [by[(-k, r)].xi for r in range(1, 26)]
        assert all(a <= b for a, b in zip(xs, xs[1:])), k
    for r in range(1, 26):
        xs = [by[(-k, r)].xi for k in range(13, 0, -1)]  # increasing eps
        assert all(a <= b for a, b in zip(xs, xs[1:])), r


def test_default_table_matches_survey_values(pft):
    """SURVEY.md App. A.1 (xi(1e-12, r), same method, derived independently)."""
    t = pft.ScopeTable.default()
    expect = {1: 3.2e-13, 2: 6.37e-7, 3: 9.17e-5, 4: 1.18e-3, 5: 5.75e-3, 6: 0.01697, 7: 0.03762, 8: 0.06946,
              10: 0.1697, 12: 0.3181, 14: 0.5101, 18: 1.0031, 20: 1.2939}
    for r, xi in expect.items():
        assert t.lookup(1e-12, r).xi == pytest.approx(xi, rel=6e-3), r


def test_table_round_trip(pft, tmp_path):
    """save then load -> equal table, bit-exact."""
    t = pft.ScopeTable.generate([1e-2, 1e-6], 6)
    f = tmp_path / "t.pftt"
    t.save(f)
    u = pft.ScopeTable.load(f)
    assert len(u) == len(t) == 12
    for a, b in zip(t.entries, u.entries):
        assert (a.epsilon, a.r, a.xi) == (b.epsilon, b.r, b.xi)
        assert np.array_equal(a.coeffs, b.coeffs)
    # query after load returns the values at save time
    assert u.lookup(1e-6, 5).xi == t.lookup(1e-6, 5).xi
    t.save_csv(tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text().count("\n") == 13


def test_table_errors(pft, tmp_path):
    f = tmp_path / "t.pftt"
    pft.ScopeTable.generate([1e-3], 2).save(f)
    raw = bytearray(f.read_bytes())
    raw[4] = 2  # version 2
    (tmp_path / "v2.pftt").write_bytes(bytes(raw))
    with pytest.raises(OSError) as e:
        pft.ScopeTable.load(tmp_path / "v2.pftt")
    assert e.value.status == 9  # version mismatch
    (tmp_path / "bad.pftt").write_bytes(bytes(raw[:20]))
    with pytest.raises(OSError):
        pft.ScopeTable.load(tmp_path / "bad.pftt")
    with pytest.raises(OSError):
        pft.ScopeTable.load(tmp_path / "missing.pftt")
    with pytest.raises(ValueError):  # missing entry requested later
        pft.ScopeTable.load(f).lookup(1e-7, 1)


def test_table_regeneration_is_byte_identical(pft, tmp_path):
    """cmd_gen_table is deterministic: regenerating the shipped artifact's
    cells gives the same bytes.  (Subset of cells to keep the CPU suite fast.)"""
    t = pft.ScopeTable.generate([1e-2, 1e-12], 10)
    shipped = pft.ScopeTable.default()
    for e in t.entries:
        s = shipped.lookup(e.epsilon, e.r)
        assert s.xi == e.xi and np.array_equal(s.coeffs, e.coeffs)
    a, b = tmp_path / "a.pftt", tmp_path / "b.pftt"
    t.save(a)
    pft.ScopeTable.generate([1e-2, 1e-12], 10).save(b)
    assert a.read_bytes() == b.read_bytes()
