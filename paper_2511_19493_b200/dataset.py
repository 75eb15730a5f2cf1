"""Training-matrix type of the proximity path.

Mirrors the reference ``Dataset`` / ``ColumnKind`` / ``from_arrays``
(dataset.py:23-111, :252-283) so callers can pass either the reference's
objects or these: the proximity path only reads ``values`` (column-major
(n, p) float64, categorical cells holding level codes), ``labels`` and the
column kinds.  CSV ingestion (dataset.py:135-249) is host I/O and out of
scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError

MAX_CATEGORICAL_LEVELS = 32  # dataset.py:19-20


@dataclass(frozen=True)
class ColumnKind:
    kind: str  # "numeric" | "categorical"
    levels: tuple = ()

    def __post_init__(self):
        if self.kind not in ("numeric", "categorical"):
            raise DataError(f"unknown column kind {self.kind!r}")
        if self.kind == "categorical":
            if not 2 <= len(self.levels) <= MAX_CATEGORICAL_LEVELS:
                raise DataError("categorical columns need 2..32 levels")
            if len(set(self.levels)) != len(self.levels):
                raise DataError("duplicate level names in categorical column")

    @property
    def is_categorical(self) -> bool:
        return self.kind == "categorical"

    @property
    def level_count(self) -> int:
        return len(self.levels)


@dataclass(frozen=True)
class Dataset:
    """Immutable (n, p) matrix, column-major float64, plus int32 labels."""

    feature_names: tuple
    columns: tuple
    values: np.ndarray
    labels: np.ndarray
    class_names: tuple

    def __post_init__(self):
        n, p = self.values.shape
        if n < 2:
            raise DataError(f"need at least 2 samples, got {n}")
        if len(self.class_names) < 2:
            raise DataError("need at least 2 classes")
        if len(self.columns) != p or len(self.feature_names) != p:
            raise DataError("column metadata does not match value matrix width")
        if self.labels.shape != (n,):
            raise DataError("labels length does not match sample count")
        if self.labels.min() < 0 or self.labels.max() >= len(self.class_names):
            raise DataError("label code out of range")
        for j, col in enumerate(self.columns):
            if col.is_categorical:
                c = self.values[:, j]
                if c.min() < 0 or c.max() >= col.level_count:
                    raise DataError(f"categorical code out of range in column {j}")
        self.values.setflags(write=False)
        self.labels.setflags(write=False)

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def p(self) -> int:
        return self.values.shape[1]

    @property
    def class_count(self) -> int:
        return len(self.class_names)


def column_arrays(columns):
    """(col_cat uint8, col_levels int32) per feature (forest.py:204-209)."""
    cat = np.array([1 if c.is_categorical else 0 for c in columns], dtype=np.uint8)
    lev = np.array([c.level_count if c.is_categorical else 0 for c in columns],
                   dtype=np.int32)
    return cat, lev


def from_arrays(values, labels, columns=None, feature_names=None,
                class_names=None) -> Dataset:
    """dataset.py:252-283: numeric columns by default; labels re-coded in
    first-appearance order unless ``class_names`` is given."""
    vals = np.asfortranarray(np.asarray(values, dtype=np.float64))
    raw = np.asarray(labels)
    n, p = vals.shape
    columns = tuple(columns) if columns is not None else tuple(
        ColumnKind("numeric") for _ in range(p))
    feature_names = tuple(feature_names) if feature_names is not None else tuple(
        f"x{j}" for j in range(p))
    if class_names is None:
        order: dict = {}
        codes = np.empty(n, dtype=np.int32)
        for i, lab in enumerate(raw):
            codes[i] = order.setdefault(str(lab), len(order))
        class_names = tuple(sorted(order, key=order.get))
    else:
        codes = raw.astype(np.int32)
    return Dataset(feature_names=feature_names, columns=columns, values=vals,
                   labels=codes, class_names=tuple(class_names))


def make_synthetic(n: int, p: int, n_classes: int = 4, seed: int = 0, p_inf=None,
                   sep: float = 1.0):
    """The synthetic workload of SURVEY §8(d): Gaussian class centres on the
    first ``p_inf`` features, float32-exact values.  Returns (X, y)."""
    p_inf = min(p, 10) if p_inf is None else p_inf
    rng = np.random.default_rng(seed)
    y = rng.integers(0, n_classes, n)
    centers = rng.normal(0, sep, (n_classes, p_inf))
    X = rng.standard_normal((n, p)).astype(np.float32)
    X[:, :p_inf] += centers[y].astype(np.float32)
    return X.astype(np.float64), y
