"""Generate the golden fixtures in tests/golden/ (committed; rerun to regenerate).

    python tests/golden/make_golden.py

The reference ships no implementation and no golden files, so the pins
are (1) SPEC.md's worked known-answer examples (encoded directly in the tests) and (2)
these fixtures: seeded inputs with their exact DFT on a target range, computed here in
40-digit arithmetic with mpmath -- independent of every line of product and oracle code.
A third fixture pins the seeded input generators (host == device for the uniform kind).
"""
from __future__ import annotations

import json
from pathlib import Path

import mpmath as mp
import numpy as np

HERE = Path(__file__).resolve().parent
mp.mp.dps = 40

# (name, N, mu, M, kind, seed)
CASES = [
    ("impulse_n16", 16, 0, 8, "impulse", 0),
    ("real01_n256_mu37", 256, 37, 16, "real01", 1),        # SPEC.md:241 setting
    ("cplx_n97_prime", 97, -5, 12, "cplx", 2),
    ("cplx_n1000_mu_neg", 1000, -200, 40, "cplx", 3),
    ("real01_n4096_m32", 4096, 0, 32, "real01", 4),         # acceptance #1 setting
    ("cplx_n3947_prime", 3947, 125, 20, "cplx", 5),
    ("tone_n2048", 2048, 300, 10, "tone", 6),
]


def make_input(N, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "impulse":
        a = np.zeros(N, dtype=np.complex128)
        a[0] = 1.0
    elif kind == "real01":
        a = rng.random(N).astype(np.complex128)
    elif kind == "tone":
        n = np.arange(N)
        a = np.exp(2j * np.pi * ((303 * n) % N) / N) + 0.5 * np.exp(2j * np.pi * ((295 * n) % N) / N)
    else:
        a = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
    return a


def exact_dft(a, mu, M):
    N = len(a)
    ar = [mp.mpc(float(z.real), float(z.imag)) for z in a]
    out = []
    for m in range(mu - M, mu + M + 1):
        acc = mp.mpc(0)
        for n in range(N):
            k = (m * n) % N
            acc += ar[n] * mp.expjpi(mp.mpf(-2 * k) / N)
        out.append(complex(acc))
    return np.array(out, dtype=np.complex128)


def main():
    index = {}
    for name, N, mu, M, kind, seed in CASES:
        a = make_input(N, kind, seed)
        ex = exact_dft(a, mu, M)
        np.savez_compressed(HERE / f"{name}.npz", a=a, exact=ex, N=N, mu=mu, M=M)
        index[name] = {"N": N, "mu": mu, "M": M, "kind": kind, "seed": seed}
        print(name, "done")
    (HERE / "index.json").write_text(json.dumps(index, indent=1) + "\n")


if __name__ == "__main__":
    main()
