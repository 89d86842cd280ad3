"""Same-box A/B of the K2-worker form against the K2 grid over sizes (development aid):
for each (N, M) the device-model p and the next candidates; prints one JSON line per (shape, p, variant)."""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2008_12559_b200 as pft  # noqa: E402
from tools import quick_time  # noqa: E402

SHAPES = [(2 ** 22, 2 ** 12), (2 ** 23, 2 ** 13), (2 ** 24, 2 ** 13), (2 ** 24, 2 ** 14), (2 ** 25, 2 ** 14),
          (2 ** 26, 2 ** 15), (2 ** 26, 2 ** 13)]
for N, M in SHAPES:
    name = f"x{N.bit_length() - 1}_{M.bit_length() - 1}"
    bench.CONFIGS[name] = (N, M, N // 4, None, "sparse", name)
    bench.SEEDS[name] = 2
    p0, r0, _ = pft.select_divisor_device(N, M)
    for p in sorted({p0, 2 * p0, max(p0 // 2, 2 * M)}):
        if N % p or p < 2 * M:
            continue
        for v in ("", "k2_at=grid"):
            try:
                r = quick_time.run(name, p, quick_time.parse_opts(v), 100, True)
            except Exception as e:  # plan not feasible at this p
                r = {"cfg": name, "p": p, "opts": v, "error": str(e)[:80]}
            print(json.dumps(r), flush=True)
