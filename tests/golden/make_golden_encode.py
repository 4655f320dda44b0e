"""Golden outputs of the reference ICM encoder (assign_codes, train.py:196-243).

Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_encode.py

Cases: reference-initialised books (train.py:_init_books) on clustered data,
the committed BASELINE c4 books (bench_data/: d=128, K=16), d=960 data (c3),
starting codes with a sweep cap, and a few-codeword odd shape.
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from icq.train import _init_books, assign_codes  # noqa: E402  (reference)

from tools.workloads import CONFIGS, load_books, sample_numpy  # noqa: E402


def main():
    rng = np.random.default_rng(123)
    out = {}
    means = rng.standard_normal((12, 32)) * 1.5
    x = (means[rng.integers(0, 12, 4000)] + 0.3 * rng.standard_normal((4000, 32))).astype(np.float32)
    books = _init_books(x[:2000].astype(np.float64), 8, 256, rng).astype(np.float32)
    out["a"] = (x, books, None, 10)
    w = CONFIGS["c4"]
    b4, _ = load_books(w)
    out["c4"] = (sample_numpy(w, 2500, rng), b4, None, 10)
    w = CONFIGS["c3"]  # d = 960 (many d slabs); small reference-initialised books
    x3 = sample_numpy(w, 600, rng)
    b3 = _init_books(x3[:300].astype(np.float64), 4, 64, rng).astype(np.float32)
    out["c3"] = (x3, b3, None, 10)
    start = rng.integers(0, 256, size=(4000, 8))
    out["start"] = (x, books, start, 3)
    xs = rng.standard_normal((700, 5)).astype(np.float32)
    bs = rng.standard_normal((3, 7, 5)).astype(np.float32)
    out["odd"] = (xs, bs, None, 10)
    save = {}
    for name, (xx, bb, cc, sw) in out.items():
        codes = assign_codes(xx, bb, codes=cc, max_sweeps=sw).codes
        save[f"{name}_x"] = xx
        save[f"{name}_books"] = bb
        save[f"{name}_codes"] = codes.astype(np.uint8)
        save[f"{name}_sweeps"] = np.int64(sw)
        if cc is not None:
            save[f"{name}_start"] = cc.astype(np.uint8)
        print(name, xx.shape, bb.shape, flush=True)
    np.savez_compressed(HERE / "encode_cases.npz", **save)


if __name__ == "__main__":
    sys.exit(main())
