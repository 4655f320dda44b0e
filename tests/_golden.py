"""Loader for the golden vectors produced by tests/golden/make_golden.py."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem not in ("eval_cli", "encode_cases"))


class Row:
    def __init__(self, z, i, r):
        self.query = int(r[0])
        self.k = int(r[1])
        self.sigma = None if r[2] == -1.0 else float(r[2])
        self.is_exact = bool(r[3])
        self.sigma_f32 = len(r) > 4 and bool(r[4])
        if self.sigma_f32:  # the reference was called with a numpy float32 sigma
            self.sigma = np.float32(self.sigma)
        self.ids = z[f"r{i}_ids"]
        self.scores = z[f"r{i}_scores"]
        ops = z[f"r{i}_ops"]
        self.fast_adds, self.exact_adds, self.lut_ops, self.evaluations, self.refinements = (
            int(x) for x in ops[:5])
        self.fallback = bool(ops[5])


class Case:
    def __init__(self, name):
        z = np.load(GOLDEN / f"{name}.npz")
        self.name = name
        self.books = z["books"]
        self.codes = z["codes"].astype(np.uint32)
        self.fast = z["fast"]
        self.sigma = float(z["sigma"])
        self.queries = z["queries"]
        self.luts = z["luts"]
        self.rows = [Row(z, i, r) for i, r in enumerate(z["rows"])]

    @property
    def K(self):
        return self.books.shape[0]

    @property
    def m(self):
        return self.books.shape[1]

    @property
    def d(self):
        return self.books.shape[2]

    @property
    def n(self):
        return self.codes.shape[0]


def load(name):
    return Case(name)
