"""Seeded synthetic workloads for the BASELINE configs (bench / test infrastructure).

BASELINE.json names no public dataset; each config is a seeded synthetic
distribution with the stated shapes.  Seeds are fixed here
and recorded in every bench line:

    mixture means / training sample : numpy default_rng(SEED_MEANS / SEED_TRAIN)
    database rows                   : torch CUDA generator SEED_DB + chunk index
    queries                         : torch CUDA generator SEED_QUERIES

Codebooks are trained by the reference (tools/train_books.py, run in the build
container) and committed under bench_data/.  The database is encoded on the
GPU by the package's float64 ICM encoder (paper_1912_08756_b200.encode_device,
icq_encode.cu: the reference's assign_codes, train.py:196-243, pinned to it
by tests/test_gpu_encode.py), chunk by chunk as it is generated.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
BOOKS_DIR = ROOT / "bench_data"

SEED_MEANS = 0
SEED_TRAIN = 1
SEED_DB = 1000
SEED_QUERIES = 7


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    K: int
    F: int
    Q: int
    k: int
    batch: int
    dist: str
    comps: int = 0
    std: float = 0.0
    train_n: int = 0  # BASELINE's stated training sample (we train on a recorded subsample)


CONFIGS = {
    "c1": Workload("c1", 100_000, 128, 8, 2, 1000, 10, 1000, "gmm", 32, 0.3, 100_000),
    "c2": Workload("c2", 1_000_000, 128, 8, 2, 10_000, 100, 10_000, "lognormal", train_n=100_000),
    "c3": Workload("c3", 1_000_000, 960, 16, 4, 1000, 10, 1000, "gamma", train_n=100_000),
    "c4": Workload("c4", 10_000_000, 128, 16, 4, 10_000, 100, 256, "gmm", 256, 0.25, 200_000),
    "c5": Workload("c5", 100_000_000, 96, 8, 2, 10_000, 100, 512, "gmm", 1024, 0.2, 1_000_000),
}


def mixture_means(w: Workload) -> np.ndarray | None:
    if w.dist != "gmm":
        return None
    return np.random.default_rng(SEED_MEANS).standard_normal((w.comps, w.d))


def sample_numpy(w: Workload, n: int, rng: np.random.Generator) -> np.ndarray:
    """Host sample of the config's distribution (used to train the books)."""
    if w.dist == "gmm":
        means = mixture_means(w)
        lab = rng.integers(0, w.comps, size=n)
        return (means[lab] + w.std * rng.standard_normal((n, w.d))).astype(np.float32)
    if w.dist == "lognormal":
        return np.round(np.clip(np.exp(rng.normal(2.0, 1.0, size=(n, w.d))), 0, 255)).astype(
            np.float32)
    if w.dist == "gamma":
        return np.clip(rng.gamma(2.0, 0.05, size=(n, w.d)), 0.0, 1.0).astype(np.float32)
    raise ValueError(w.dist)


def sample_torch(w: Workload, n: int, seed: int, device="cuda"):
    """Device sample of the config's distribution (database rows / queries)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if w.dist == "gmm":
        means = torch.from_numpy(mixture_means(w)).to(device=device, dtype=torch.float32)
        lab = torch.randint(0, w.comps, (n,), generator=g, device=device)
        return means[lab] + w.std * torch.randn((n, w.d), generator=g, device=device)
    if w.dist == "lognormal":
        x = torch.randn((n, w.d), generator=g, device=device) + 2.0
        return torch.round(torch.clamp(torch.exp(x), 0, 255))
    if w.dist == "gamma":
        # Gamma(shape=2, scale=0.05) = 0.05 * (E1 + E2), E ~ Exp(1)
        u = torch.rand((2, n, w.d), generator=g, device=device).clamp_min_(1e-12)
        x = -0.05 * torch.log(u).sum(0)
        return torch.clamp(x, 0.0, 1.0)
    raise ValueError(w.dist)


def load_books(w: Workload):
    z = np.load(BOOKS_DIR / f"books_{w.name}.npz", allow_pickle=False)
    meta = {k: z[k].item() if z[k].ndim == 0 else z[k] for k in z.files if k != "books"}
    return z["books"].astype(np.float32), meta


def build_database(w: Workload, books, sweeps: int = 10, chunk_rows: int = 1 << 22,
                   device="cuda", stats: dict | None = None):
    """Generate the config's database chunk by chunk on the GPU, encode it with
    the float64 ICM encoder, and keep only the uint8 codes (n, K) on the device."""
    import time

    import torch

    from paper_1912_08756_b200.encode import encode_device

    codes = torch.empty((w.n, w.K), dtype=torch.uint8, device=device)
    used, t_enc = 0, 0.0
    for ci, s in enumerate(range(0, w.n, chunk_rows)):
        e = min(w.n, s + chunk_rows)
        x = sample_torch(w, e - s, SEED_DB + ci, device).float()
        torch.cuda.synchronize()
        t0 = time.time()
        c, u = encode_device(x, books, max_sweeps=sweeps)
        torch.cuda.synchronize()
        t_enc += time.time() - t0
        codes[s:e] = c
        used = max(used, u)
        del x, c
    if stats is not None:
        stats.update(encode_seconds=t_enc, sweeps_used=used, max_sweeps=sweeps)
    return codes


def queries(w: Workload, device="cuda"):
    import torch

    return sample_torch(w, w.Q, SEED_QUERIES, device).to(torch.float64)


def index_rule(w: Workload, meta: dict, sigma_override: float | None = None):
    """Index-construction rule, recorded with every result.

    fast set: the learned one when it has the configured size, else the first
    |F| books of the residual chain (they carry most of the energy).
    sigma: the learned margin when the learned model has a fast set; when the
    reference learned an empty fast set (psi = {} — c3, c4 here) its margin
    belongs to no fast set and sigma = 0 is imposed (the learned value of
    c1, c2, c5).  A sigma sweep is reported separately.
    """
    learned_fast = np.asarray(meta["learned_fast"], dtype=np.uint32)
    learned_sigma = float(meta["learned_sigma"])
    if learned_fast.size == w.F:
        fast, frule = learned_fast, "learned"
    else:
        fast = np.arange(w.F, dtype=np.uint32)
        frule = f"first {w.F} books (learned fast set {learned_fast.tolist()})"
    if sigma_override is not None:
        sigma, srule = float(sigma_override), "override"
    elif learned_fast.size:
        sigma, srule = learned_sigma, "learned"
    else:
        sigma, srule = 0.0, f"0 (learned fast set empty; learned sigma {learned_sigma:.4g} unused)"
    return fast, sigma, frule, srule
