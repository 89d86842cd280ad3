"""Data formats either side of execute and the anomaly pipeline that calls it (SURVEY.md §8(f)
row 4; SPEC.md cli module: SignalFile, cmd_transform's "m,re,im" output, cmd_anomaly).

The PFTS layout is pinned by bytes built here with struct/numpy (independent of the library).
SPEC's header is "16-byte ... {magic "PFTS", u32 complex flag, u32 length}": those fields fill
12 bytes, so this build keeps the stated 16-byte size with 4 reserved zero bytes (ignored on
read) -- a decision recorded in DESIGN.md.
CSV files round-trip bit-exactly (SPEC.md cli "File round-trip"); the anomaly scoring is
checked against a numpy restatement of the same formula with exact FFT coefficients.
"""
from __future__ import annotations

import struct

import numpy as np
import pytest


def rand_c(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    v[:4] = [1e-300 + 0j, -2.5e307 + 1e-17j, np.pi + 0j, 0.1 - 0.3j][: min(4, n)]
    return v


def test_pfts_layout_is_pinned(pft, tmp_path):
    v = rand_c(37, 1)
    p = tmp_path / "a.f64"
    pft.write_signal(p, v, pft.SIGNAL_F64LE)
    raw = np.empty(2 * v.size)
    raw[0::2], raw[1::2] = v.real, v.imag
    assert p.read_bytes() == b"PFTS" + struct.pack("<III", 1, v.size, 0) + raw.astype("<f8").tobytes()
    back, cx = pft.read_signal(p)
    assert cx and np.array_equal(back.view(np.float64), v.view(np.float64))


def test_pfts_real_channel(pft, tmp_path):
    x = np.random.default_rng(2).uniform(-1, 1, 101)
    p = tmp_path / "r.bin"
    (p).write_bytes(b"PFTS" + struct.pack("<III", 0, x.size, 0) + x.astype("<f8").tobytes())
    back, cx = pft.read_signal(p)
    assert not cx and np.array_equal(back.real, x) and not back.imag.any()
    q = tmp_path / "r2.bin"
    pft.write_signal(q, x.astype(np.complex128), is_complex=False)
    assert q.read_bytes() == p.read_bytes()


@pytest.mark.parametrize("complex_", [True, False])
def test_csv_signal_round_trip_bit_exact(pft, tmp_path, complex_):
    v = rand_c(200, 3)
    if not complex_:
        v = v.real.astype(np.complex128)
    p = tmp_path / "s.csv"
    pft.write_signal(p, v, is_complex=complex_)
    rows = p.read_text().splitlines()
    assert len(rows) == v.size and all(r.count(",") == (1 if complex_ else 0) for r in rows)
    back, cx = pft.read_signal(p)
    assert cx == complex_ and np.array_equal(back.view(np.float64), v.view(np.float64))


def test_csv_reader_accepts_spec_rows(pft, tmp_path):
    p = tmp_path / "h.csv"
    p.write_text("1\n0\n\n  0 \n0\n")  # impulse, blank line skipped, whitespace trimmed
    back, cx = pft.read_signal(p)
    assert not cx and np.array_equal(back, np.array([1, 0, 0, 0], dtype=np.complex128))
    p.write_text("1.5,-2\n3,4e-3\n")
    back, cx = pft.read_signal(p)
    assert cx and np.array_equal(back, np.array([1.5 - 2j, 3 + 4e-3j]))


@pytest.mark.parametrize("content,suffix", [
    (b"PFTX" + struct.pack("<III", 1, 1, 0) + b"\0" * 16, ".f64"),        # bad magic
    (b"PFTS" + struct.pack("<III", 1, 3, 0) + b"\0" * 16, ".f64"),        # truncated payload
    (b"PFTS" + struct.pack("<III", 0, 1, 0) + b"\0" * 9, ".f64"),         # trailing bytes
    (b"PFTS" + struct.pack("<III", 2, 0, 0), ".f64"),                     # channel flag 2
    (b"PFTS\1\0", ".f64"),                                                # truncated header
    (b"1,2,3\n", ".csv"),                                                 # three fields
    (b"1\nabc\n", ".csv"),                                                # not a number
    (b"1\n2,3\n", ".csv"),                                                # mixed rows
])
def test_malformed_signal_files_are_io_errors(pft, tmp_path, content, suffix):
    p = tmp_path / ("bad" + suffix)
    p.write_bytes(content)
    with pytest.raises(pft.PftIOError) as e:
        pft.read_signal(p)
    assert e.value.status == 8  # PFT_ERR_IO: the CLI's exit code 1 (SPEC.md cli)


def test_missing_file_is_io_error(pft, tmp_path):
    with pytest.raises(pft.PftIOError):
        pft.read_signal(tmp_path / "nope.csv")


def test_spectrum_csv_round_trip_bit_exact(pft, tmp_path):
    M, mu = 40, -12345
    vals = rand_c(2 * M + 1, 4)
    spec = pft.PartialSpectrum(pft.TargetRange(mu, M), vals)
    p = tmp_path / "out.csv"
    pft.write_spectrum_csv(p, spec)
    rows = p.read_text().splitlines()
    assert rows[0] == "m,re,im" and len(rows) == 2 * M + 2
    assert [int(r.split(",")[0]) for r in rows[1:]] == list(range(mu - M, mu + M + 1))
    m0, back = pft.read_spectrum_csv(p)
    assert m0 == mu - M and np.array_equal(back.view(np.float64), vals.view(np.float64))


def _numpy_anomaly(x, coeffs, M, k):
    """Restatement of cmd_anomaly's scoring (SPEC.md cli) for the check."""
    N = x.size
    n = np.arange(N)
    fit = np.full(N, coeffs[M].real)
    for m in range(1, M + 1):
        ang = 2 * np.pi * ((m * n) % N) / N
        fit += 2 * (coeffs[M + m].real * np.cos(ang) - coeffs[M + m].imag * np.sin(ang))
    fit /= N
    score = np.abs(x - fit)
    order = np.lexsort((np.arange(N), -score))[:k]
    return order, score[order], fit


def _exact_coeffs(x, M):
    full = np.fft.fft(x)
    return full[np.arange(-M, M + 1) % x.size]


def test_anomaly_scoring_matches_restatement(pft):
    rng = np.random.default_rng(5)
    N, M, k = 1000, 12, 15
    n = np.arange(N)
    x = np.sin(2 * np.pi * 3 * n / N) + 0.3 * np.cos(2 * np.pi * 7 * n / N) + 0.05 * rng.standard_normal(N)
    x[[17, 400, 401, 777]] += [4.0, -3.0, 2.5, 5.0]
    c = _exact_coeffs(x, M)
    idx, sc, fit = pft.anomaly_from_coeffs(x, c, M, k)
    ridx, rsc, rfit = _numpy_anomaly(x, c, M, k)
    assert np.allclose(fit, rfit, rtol=0, atol=1e-12)
    assert np.allclose(sc, rsc, rtol=0, atol=1e-12)
    assert set(idx[:4].tolist()) == {17, 400, 401, 777}
    assert np.all(np.diff(sc) <= 0)


def test_anomaly_low_frequency_input_has_no_residual(pft):
    N, M = 777, 9
    n = np.arange(N)
    x = sum(np.cos(2 * np.pi * f * n / N + f) for f in range(0, M + 1))
    _, sc, _ = pft.anomaly_from_coeffs(x, _exact_coeffs(x, M), M, 5)
    assert sc.max() < 1e-6 * np.abs(x).max()


def test_anomaly_k_equals_n_ties_by_index(pft):
    x = np.zeros(64)
    x[[5, 9]] = 1.0
    c = np.zeros(3, dtype=np.complex128)  # M = 1, zero coefficients: fit = 0, scores = |x|
    idx, sc, _ = pft.anomaly_from_coeffs(x, c, 1, 64)
    assert idx[:2].tolist() == [5, 9] and idx[2:].tolist() == [i for i in range(64) if i not in (5, 9)]
    assert sc[0] == sc[1] == 1.0


def test_anomaly_argument_errors(pft):
    with pytest.raises(pft.PftValueError):
        pft.anomaly_from_coeffs(np.zeros(8), np.zeros(3, dtype=complex), 1, 0)   # k = 0
    with pytest.raises(pft.PftValueError):
        pft.anomaly_from_coeffs(np.zeros(8), np.zeros(11, dtype=complex), 5, 1)  # M > N/2


@pytest.mark.gpu
def test_anomaly_pft_matches_fft_source(pft):
    """Acceptance criterion 7 (SPEC.md; Fig. 4 "does not change the result of the
    detection"): 50 spike-injected series, N = 19735, M = 125, k = 20 -- the top-k index sets
    from the GPU PFT source and from exact FFT coefficients are identical."""
    N, M, k = 19735, 125, 20
    n = np.arange(N)
    for case in range(50):
        rng = np.random.default_rng(1000 + case)
        x = np.zeros(N)
        for _ in range(6):
            f = rng.integers(1, M)
            x += rng.uniform(0.2, 1.0) * np.cos(2 * np.pi * f * n / N + rng.uniform(0, 2 * np.pi))
        x += 0.01 * rng.standard_normal(N)
        spikes = rng.choice(N, size=k, replace=False)
        x[spikes] += rng.choice([-1, 1], size=k) * rng.uniform(0.8, 2.0, size=k)
        idx_pft, _, _ = pft.anomaly(x, M, k)
        idx_fft, _, _ = pft.anomaly_from_coeffs(x, _exact_coeffs(x, M), M, k)
        assert set(idx_pft.tolist()) == set(idx_fft.tolist()), case
