"""The command-line surface (cli module): the `pft` binary built next to the
library.  Host-only verbs (gen-table, plan) and the exit codes run anywhere; the GPU verbs are
marked gpu.  Exit codes: 0 ok, 1 I/O or parse, 2 invalid parameters, 3 verification failure
(SPEC.md:458), 4 no usable GPU (this build has no CPU fallback)."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
PFT = ROOT / "paper_2008_12559_b200" / "pft"


def run(*args, timeout=600):
    return subprocess.run([str(PFT), *map(str, args)], capture_output=True, text=True, timeout=timeout)


def test_cli_built_and_version():
    assert PFT.exists(), "build the library (python -m paper_2008_12559_b200.build) to get the CLI"
    r = run("version")
    assert r.returncode == 0 and "sm_100a" in r.stdout


def test_gen_table_is_deterministic_and_loadable(tmp_path, pft):
    """cmd_gen_table: same flags -> byte-identical file; r_max = 1 -> constants."""
    a, b = tmp_path / "a.pftt", tmp_path / "b.pftt"
    for p in (a, b):
        r = run("gen-table", "--epsilons", "1e-2,1e-6", "--r-max", "8", "--out", p)
        assert r.returncode == 0, r.stderr
    assert a.read_bytes() == b.read_bytes()
    t = pft.ScopeTable.load(a)
    assert len(t) == 16 and t.r_max == 8
    r = run("gen-table", "--epsilons", "1e-1", "--r-max", "1", "--out", tmp_path / "c.pftt")
    assert r.returncode == 0 and json.loads(r.stdout)["entries"] == 1


def test_plan_json_and_device_choices():
    r = run("plan", "--N", 2 ** 24, "--M", 2 ** 10, "--mu", 2 ** 22, "--device", "--world", 8)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines()]
    assert lines[0]["p"] == 65536 and lines[0]["r"] == 6       # SPEC cost model
    assert lines[1]["device_p"] == 16384 and lines[1]["device_r"] == 8
    assert lines[2]["world"] == 8 and (2 ** 24) % lines[2]["sharded_p"] == 0


@pytest.mark.parametrize("args,code", [
    (["plan", "--N", 16, "--M", 9], 2),                      # M > N/2 -> invalid parameters
    (["plan", "--N", 16, "--M", 2, "--p", 5], 2),            # p does not divide N
    (["plan", "--N", "abc", "--M", 2], 2),                   # not an integer
    (["plan", "--M", 2], 2),                                 # missing --N
    (["transform", "--input", "/nonexistent.csv", "--M", 4, "--output", "/tmp/x.csv"], 1),
    (["gen-table", "--epsilons", "1e-6", "--out", "/nonexistent/dir/t.pftt"], 1),
    (["bench", "--mode", "vary-x", "--out", "/tmp/b.csv"], 2),
    (["frobnicate"], 2),
])
def test_exit_codes(args, code):
    r = run(*args)
    assert r.returncode == code, (args, r.returncode, r.stderr)


def test_transform_parse_error_is_exit_1(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("1.0\nnot-a-number\n")
    r = run("transform", "--input", bad, "--M", 0, "--output", tmp_path / "o.csv")
    assert r.returncode == 1, r.stderr


@pytest.mark.gpu
def test_transform_impulse_and_verify(tmp_path, pft):
    """cmd_transform: impulse CSV, M = 4, mu = 0 -> nine rows ~ (1, 0); --verify prints
    the ErrorReport and exits 0; the CSV re-reads bit-exactly."""
    sig = tmp_path / "imp.csv"
    sig.write_text("1\n" + "0\n" * 255)
    out = tmp_path / "o.csv"
    r = run("transform", "--input", sig, "--M", 4, "--output", out, "--verify")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["relative_l2"] < 1e-6 and rep["bound_satisfied"]
    m0, vals = pft.read_spectrum_csv(out)
    assert m0 == -4 and len(vals) == 9 and np.max(np.abs(vals - 1)) < 1e-9


@pytest.mark.gpu
def test_transform_air_condition_size_verify(tmp_path, pft):
    """random N = 19735 file, M = 125, auto p, --verify -> exit 0, relative l2 < 1e-6."""
    x = np.random.default_rng(19735).random(19735)
    sig = tmp_path / "x.f64"
    pft.write_signal(sig, x, is_complex=False)
    r = run("transform", "--input", sig, "--M", 125, "--output", tmp_path / "o.csv", "--verify")
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout.strip().splitlines()[-1])["relative_l2"] < 1e-6


@pytest.mark.gpu
def test_transform_verify_failure_is_exit_3(tmp_path, pft):
    """A loose table (eps = 1e-2) cannot meet the 1e-6 verification threshold: exit 3."""
    table = tmp_path / "loose.pftt"
    assert run("gen-table", "--epsilons", "1e-2", "--r-max", "25", "--out", table).returncode == 0
    x = np.random.default_rng(1).random(4096) + 1j * np.random.default_rng(2).random(4096)
    sig = tmp_path / "x.csv"
    pft.write_signal(sig, x)
    r = run("transform", "--input", sig, "--M", 200, "--epsilon", 1e-2, "--table", table,
            "--output", tmp_path / "o.csv", "--verify")
    assert r.returncode == 3, (r.stdout, r.stderr)


@pytest.mark.gpu
def test_transform2d_verify(tmp_path, pft):
    x = np.random.default_rng(5).random(64 * 128)
    sig = tmp_path / "g.f64"
    pft.write_signal(sig, x, is_complex=False)
    out = tmp_path / "o.csv"
    r = run("transform2d", "--input", sig, "--N1", 64, "--N2", 128, "--M1", 5, "--M2", 9, "--mu1", 3,
            "--mu2", -4, "--output", out, "--verify")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["relative_l2"] < 1e-6 and rep["bound_satisfied"]
    rows = out.read_text().splitlines()
    assert rows[0] == "m1,m2,re,im" and len(rows) == 1 + 11 * 19


@pytest.mark.gpu
def test_anomaly_pft_and_fft_sources_agree(tmp_path, pft):
    """injected spikes -> identical top-k between --source pft and --source fft."""
    rng = np.random.default_rng(44)
    N = 19735
    n = np.arange(N)
    x = np.sin(2 * np.pi * 3 * n / N) + 0.5 * np.cos(2 * np.pi * 11 * n / N) + 0.01 * rng.standard_normal(N)
    spikes = rng.choice(N, 20, replace=False)
    x[spikes] += 5.0
    sig = tmp_path / "s.f64"
    pft.write_signal(sig, x, is_complex=False)
    res = {}
    for src in ("pft", "fft"):
        r = run("anomaly", "--input", sig, "--M", 125, "--k", 20, "--source", src)
        assert r.returncode == 0, r.stderr
        res[src] = json.loads(r.stdout)
        assert res[src]["fitted_curve_source"] == src and len(res[src]["indices"]) == 20
    assert res["pft"]["indices"] == res["fft"]["indices"]
    assert set(res["pft"]["indices"]) == set(int(s) for s in spikes)


@pytest.mark.gpu
def test_bench_vary_n_csv(tmp_path):
    """cmd_bench: BenchRecord CSV with the SPEC header; PFT rows carry rel_l2 < 1e-6 against the
    naive DFT where the oracle runs (N <= 2^16)."""
    out = tmp_path / "b.csv"
    r = run("bench", "--mode", "vary-n", "--reps", 3, "--warmup", 1, "--max-n", 2 ** 16, "--out", out)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "algo,N,M,mu,p,r,reps,mean_ms,stddev_ms,rel_l2"
    recs = [l.split(",") for l in lines[1:]]
    pft_rows = [x for x in recs if x[0] == "pft"]
    assert [int(x[1]) for x in pft_rows] == [2 ** e for e in range(12, 17)]
    for x in pft_rows:
        assert float(x[7]) > 0 and float(x[9]) < 1e-6
