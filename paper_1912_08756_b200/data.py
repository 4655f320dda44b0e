"""Argument containers of the query path (mirror of icq.data, data.py:32-263).

The B200 engines accept either these containers or the reference's own
``icq.SearchIndex`` objects (duck-typed: ``books.codewords``, ``codes.codes``,
``fast``, ``sigma``, ``cfg.K``/``cfg.m``).  Validation restates
``SearchIndex.__post_init__`` (data.py:136-176) so the same inputs are
rejected with the same exception class.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _reference_classes():
    """The reference's exception classes when its package is importable.

    A drop-in must raise the *same* classes the reference's callers catch
    (``except icq.ValidationError``, ``pytest.raises(ValidationError)`` in
    pkg/tests/test_search.py:126-141, :218-221).  When ``icq`` is importable
    the mirror's classes derive from the reference's, so both the local and
    the reference class match; without it they are plain ValueError /
    Exception subclasses with the reference's names and meanings.
    ``ICQ_B200_STANDALONE=1`` skips the probe.
    """
    import importlib.util
    import os

    if os.environ.get("ICQ_B200_STANDALONE"):
        return ValueError, Exception, Exception
    try:
        if importlib.util.find_spec("icq") is None:
            return ValueError, Exception, Exception
        import icq.data as ref
    except Exception:  # pragma: no cover - a broken reference install
        return ValueError, Exception, Exception
    return ref.ValidationError, ref.FormatError, ref.UnsupportedVersionError


_VE_BASE, _FE_BASE, _UVE_BASE = _reference_classes()


class ValidationError(_VE_BASE):  # type: ignore[misc,valid-type]
    """Invalid values: non-finite data, bad shapes, out-of-range parameters (data.py:32)."""


class FormatError(_FE_BASE):  # type: ignore[misc,valid-type]
    """Malformed file: bad magic, truncated payload, inconsistent lengths (data.py:36)."""


class UnsupportedVersionError(FormatError, _UVE_BASE):  # type: ignore[misc,valid-type]
    """Index file written with an unknown format version (data.py:40)."""


class UnsupportedError(RuntimeError):
    """Inputs valid for the reference but outside this build's kernels (m > 256, K > 16)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the native library."""


@dataclass
class Config:
    """Quantizer hyperparameters carried by an index (data.py:80-121; only K, m used here)."""

    K: int = 8
    m: int = 256
    gamma1: float = 0.1
    gamma2: float = 1.0
    pi1: float = 0.9
    pi2: float = 0.1
    alpha2: float = -10.0
    sigma_scale: float = 1.0
    epochs: int = 50
    batch_size: int = 256
    learning_rate: float = 1e-2
    seed: int = 0

    def __post_init__(self):  # data.py:102-122
        if self.K < 1:
            raise ValidationError(f"K must be >= 1, got {self.K}")
        if self.m < 2:
            raise ValidationError(f"m must be >= 2, got {self.m}")
        if self.gamma1 < 0 or self.gamma2 < 0:
            raise ValidationError("gamma1 and gamma2 must be non-negative")
        if not (self.pi1 > self.pi2 > 0):
            raise ValidationError(f"need pi1 > pi2 > 0, got {self.pi1}, {self.pi2}")
        if abs(self.pi1 + self.pi2 - 1.0) > 1e-12:
            raise ValidationError(f"pi1 + pi2 must equal 1, got {self.pi1 + self.pi2}")
        if self.alpha2 >= 0:
            raise ValidationError(f"alpha2 must be negative, got {self.alpha2}")
        if self.sigma_scale < 0:
            raise ValidationError(f"sigma_scale must be >= 0, got {self.sigma_scale}")
        if self.epochs < 1 or self.batch_size < 1:
            raise ValidationError("epochs and batch_size must be >= 1")
        if self.learning_rate <= 0:
            raise ValidationError(f"learning_rate must be > 0, got {self.learning_rate}")
        if self.seed < 0:
            raise ValidationError(f"seed must be >= 0, got {self.seed}")


@dataclass
class EmbeddedDataset:
    """Vectors plus optional labels (data.py:44-77): (n, d) float32, (n,) uint32."""

    vectors: np.ndarray
    labels: np.ndarray | None = None

    def __post_init__(self):
        vectors = np.ascontiguousarray(self.vectors, dtype=np.float32)
        if vectors.ndim != 2:
            raise ValidationError(f"vectors must be 2-d, got shape {vectors.shape}")
        self.vectors = vectors
        if self.labels is not None:
            labels = np.asarray(self.labels)
            if labels.shape != (vectors.shape[0],):
                raise ValidationError(
                    f"labels shape {labels.shape} does not match n={vectors.shape[0]}")
            if labels.size and (np.any(labels < 0)
                                or not np.issubdtype(labels.dtype, np.integer)):
                raise ValidationError("labels must be non-negative integers")
            self.labels = np.ascontiguousarray(labels, dtype=np.uint32)

    @property
    def n(self) -> int:
        return self.vectors.shape[0]

    @property
    def d(self) -> int:
        return self.vectors.shape[1]


@dataclass
class CodebookSet:
    """K codebooks of m codewords, (K, m, d) (data.py:136-164)."""

    codewords: np.ndarray

    def __post_init__(self):
        cw = np.ascontiguousarray(self.codewords)
        if cw.ndim != 3:
            raise ValidationError(f"codewords must be (K, m, d), got shape {cw.shape}")
        self.codewords = cw

    @property
    def K(self) -> int:
        return self.codewords.shape[0]

    @property
    def m(self) -> int:
        return self.codewords.shape[1]

    @property
    def d(self) -> int:
        return self.codewords.shape[2]


@dataclass
class CodeMatrix:
    """(n, K) codeword choices (data.py:167-190); stored uint32 like the reference."""

    codes: np.ndarray

    def __post_init__(self):
        c = np.ascontiguousarray(self.codes)
        if c.ndim != 2:
            raise ValidationError(f"codes must be (n, K), got shape {c.shape}")
        if c.size and np.any(c < 0):
            raise ValidationError("codes must be non-negative")
        self.codes = c.astype(np.uint32, copy=False)

    @property
    def n(self) -> int:
        return self.codes.shape[0]

    @property
    def K(self) -> int:
        return self.codes.shape[1]


@dataclass
class SearchIndex:
    """Query-time state of a trained quantizer (data.py:193-263)."""

    books: CodebookSet
    codes: CodeMatrix
    xi: np.ndarray
    fast: np.ndarray
    sigma: float
    lambdas: np.ndarray
    cfg: Config = field(default_factory=Config)

    def __post_init__(self):
        # (duck-typed: the reference's own CodebookSet / CodeMatrix are accepted too)
        books = self.books if isinstance(self.books, CodebookSet) else CodebookSet(
            getattr(self.books, "codewords", self.books))
        codes = self.codes if isinstance(self.codes, CodeMatrix) else CodeMatrix(
            getattr(self.codes, "codes", self.codes))
        self.books = CodebookSet(books.codewords.astype(np.float32, copy=False))
        self.codes = codes
        if codes.K != books.K:
            raise ValidationError(f"codes have {codes.K} books, codebooks have {books.K}")
        if codes.codes.size and codes.codes.max() >= books.m:
            raise ValidationError("codes reference codewords beyond m")
        if self.cfg.K != books.K or self.cfg.m != books.m:
            raise ValidationError("config K/m disagree with the codebooks")
        xi = np.ascontiguousarray(np.asarray(self.xi), dtype=np.uint8)
        if xi.shape != (books.d,):
            raise ValidationError(f"xi length {xi.shape} does not match d={books.d}")
        if xi.size and xi.max() > 1:
            raise ValidationError("xi entries must be 0 or 1")
        self.xi = xi
        fast = np.ascontiguousarray(np.asarray(self.fast), dtype=np.uint32)
        if fast.ndim != 1 or (fast.size and fast.max() >= books.K):
            raise ValidationError("fast set must hold codebook indices in [0, K)")
        if fast.size and np.any(np.diff(fast.astype(np.int64)) <= 0):
            raise ValidationError("fast set must be sorted and unique")
        self.fast = fast
        lam = np.ascontiguousarray(np.asarray(self.lambdas), dtype=np.float32)
        if lam.shape != (books.d,):
            raise ValidationError(f"lambdas length {lam.shape} does not match d={books.d}")
        if lam.size and (not np.all(np.isfinite(lam)) or lam.min() < 0):
            raise ValidationError("lambdas must be finite and non-negative")
        self.lambdas = lam
        sigma = float(np.float32(self.sigma))
        if not np.isfinite(sigma) or sigma < 0:
            raise ValidationError(f"sigma must be finite and >= 0, got {self.sigma}")
        self.sigma = sigma

    @property
    def n(self) -> int:
        return self.codes.n

    @property
    def d(self) -> int:
        return self.books.d
