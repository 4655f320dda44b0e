"""Train the bench codebooks with the REAL reference trainer (build container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tools/train_books.py c1 c2 c4 c5 [c3]

For each BASELINE config: draw a seeded sample of its distribution
(tools/workloads.py), run ``icq.train.train`` (train.py:287) with a recorded
budget, and store the trained books plus the learned model (xi, fast set,
sigma, lambdas) in bench_data/books_<cfg>.npz.  The index-construction rule
 is applied at bench time: fast = [0..F-1] when the learned
fast set does not have the configured size; sigma = the learned margin.
"""

import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools.workloads import BOOKS_DIR, CONFIGS, SEED_TRAIN, sample_numpy  # noqa: E402

from icq import Config, EmbeddedDataset  # noqa: E402  (reference)
from icq.train import train  # noqa: E402

BUDGET = {  # (training sample rows, epochs) — recorded in the npz.  Rows are
    # BASELINE's stated training samples (c1: the full 100k database); the
    # epoch count is BASELINE-unspecified (Config default 50 would take hours
    # at 1M rows on the build host), recorded with the books.
    "c1": (100_000, 2),
    "c2": (100_000, 2),
    "c3": (100_000, 1),
    "c4": (200_000, 2),
    "c5": (1_000_000, 2),
}
OUT_DIR = Path(os.environ.get("ICQ_BOOKS_OUT", str(BOOKS_DIR)))


def main(names):
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    for name in names:
        w = CONFIGS[name]
        rows, epochs = BUDGET[name]
        x = sample_numpy(w, rows, np.random.default_rng(SEED_TRAIN))
        cfg = Config(K=w.K, m=256, epochs=epochs, seed=0)
        t0 = time.time()
        index, _ = train(EmbeddedDataset(x), cfg)
        dt = time.time() - t0
        np.savez_compressed(
            OUT_DIR / f"books_{name}.npz",
            books=index.books.codewords.astype(np.float32),
            learned_fast=index.fast.astype(np.uint32),
            learned_sigma=np.float64(index.sigma),
            xi=index.xi,
            lambdas=index.lambdas,
            train_rows=np.int64(rows),
            epochs=np.int64(epochs),
            seed=np.int64(0),
            train_seconds=np.float64(dt),
        )
        print(f"{name}: trained in {dt:.0f}s psi={int(index.xi.sum())}/{w.d} "
              f"fast={index.fast.tolist()} sigma={index.sigma!r}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4", "c5", "c3"])
