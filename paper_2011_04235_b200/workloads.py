"""Seeded synthetic workloads standing in for the paper's corpora.

The paper's Amazon / RCV / Eurlex / Bibtex corpora (reference
``PAPER.md:688-697``) are not available offline, so the five configurations
of ``BASELINE.json`` are generated here from a seed with the shapes, nnz
targets and degree / value distributions that file states.  Everything is
host-side numpy; this is input generation, not part of the solve.

Conventions (documented in DESIGN.md):

* Row degrees follow the named distribution, are rescaled by one common
  factor so that the total hits the nnz target, and are capped at ``n``
  (the excess is lost to the cap; the scale factor compensates).
* Columns inside a row are distinct and drawn with probability proportional
  to the column popularity weights (with-replacement draws, deduplicated and
  topped up for a few rounds; rows that cannot be completed keep fewer).
* Values are uniform on (0, 1] (or TF-IDF-like for config 2); rows are
  L2-normalised where the config says so.  The result is canonical CSR
  (sorted indices, no duplicates, no explicit zeros) -- exactly what
  ``check_csr`` (reference ``validation.py:38-55``) would produce.
* Labels: per-row counts ~ Poisson(lambda), labels drawn distinct with Zipf
  popularity over the label set, values exactly 1.0.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration."""

    name: str
    m: int
    n: int
    nnz: int
    n_labels: int
    rank: int
    k: float
    seed: int
    row_dist: tuple
    col_dist: tuple
    values: str = "uniform"
    normalize_rows: bool = False
    labels_per_row: float = 4.0
    label_zipf: float = 1.2
    notes: str = ""

    @property
    def alpha(self) -> float:
        return self.rank / self.n


WORKLOADS = {
    "c1": Workload("c1", 2_000, 500, 10_000, 100, 100, 0.01, 0,
                   ("zipf", 1.2), ("zipf", 1.5), "uniform", True, 4.0, 1.3,
                   "tiny CPU-runnable case, BASELINE configs[0]"),
    "c2": Workload("c2", 7_400, 1_840, 500_000, 159, 368, 0.01, 1,
                   ("lognormal", 68.0, 0.6), ("zipf", 1.3), "tfidf", True, 2.4, 1.2,
                   "Bibtex-shaped, BASELINE configs[1]"),
    "c3r50": Workload("c3r50", 16_000, 500, 320_000, 983, 50, 0.01, 2,
                      ("poisson", 20.0), ("hubtail", 0.05, 0.40), "uniform", False, 19.0, 1.1,
                      "BASELINE configs[2], r=50"),
    "c3r100": Workload("c3r100", 16_000, 500, 320_000, 983, 100, 0.01, 2,
                       ("poisson", 20.0), ("hubtail", 0.05, 0.40), "uniform", False, 19.0, 1.1,
                       "BASELINE configs[2], r=100"),
    "c3r200": Workload("c3r200", 16_000, 500, 320_000, 983, 200, 0.01, 2,
                       ("poisson", 20.0), ("hubtail", 0.05, 0.40), "uniform", False, 19.0, 1.1,
                       "BASELINE configs[2], r=200"),
    "c4": Workload("c4", 200_000, 50_000, 5_000_000, 4_000, 500, 0.005, 3,
                   ("zipf", 1.4), ("zipf", 1.6), "uniform", False, 5.0, 1.2,
                   "BASELINE configs[3]; A11 blocks sharded across 1/2/4/8 GPUs"),
    "c5": Workload("c5", 2_000_000, 200_000, 30_000_000, 3_000, 1_000, 0.005, 4,
                   ("lognormal", 15.0, 1.0), ("zipf", 1.5), "uniform", True, 4.0, 1.2,
                   "BASELINE configs[4]; U rows partitioned across GPUs"),
}


def _raw_row_weights(rng, m, dist, cap):
    kind = dist[0]
    if kind == "zipf":
        raw = rng.zipf(dist[1], size=m).astype(np.float64)
    elif kind == "lognormal":
        mean, sigma = dist[1], dist[2]
        raw = rng.lognormal(math.log(mean) - 0.5 * sigma * sigma, sigma, size=m)
    elif kind == "poisson":
        raw = 1.0 + rng.poisson(dist[1], size=m).astype(np.float64)
    else:
        raise ValueError(f"unknown row distribution {dist!r}")
    return np.minimum(raw, float(cap))


def _row_degrees(rng, m, n, target, dist):
    """Degrees with the named shape, rescaled so the capped total hits ``target``."""
    raw = _raw_row_weights(rng, m, dist, n)

    def total(c):
        return int(np.clip(np.rint(raw * c), 1, n).sum())

    lo, hi = 1e-6, 1.0
    while total(hi) < target and hi < 1e12:
        hi *= 2.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if total(mid) < target:
            lo = mid
        else:
            hi = mid
    return np.clip(np.rint(raw * hi), 1, n).astype(np.int64)


def _col_probs(rng, n, dist):
    kind = dist[0]
    if kind == "zipf":
        ranks = rng.permutation(n).astype(np.float64)
        w = (ranks + 1.0) ** (-dist[1])
    elif kind == "hubtail":
        frac_cols, frac_mass = dist[1], dist[2]
        n_hub = max(1, int(round(frac_cols * n)))
        order = rng.permutation(n)
        w = np.empty(n)
        w[order[:n_hub]] = frac_mass / n_hub
        w[order[n_hub:]] = (1.0 - frac_mass) / (n - n_hub)
        w *= rng.uniform(0.8, 1.2, size=n)
    else:
        raise ValueError(f"unknown column distribution {dist!r}")
    return w / w.sum()


def _uniq(keys):
    keys = np.sort(keys)
    if len(keys) < 2:
        return keys
    return keys[np.concatenate(([True], keys[1:] != keys[:-1]))]


def _sample_distinct(rng, deg, p, n, rounds=12):
    """Per-row distinct column draws with probabilities ``p``; returns sorted keys row*n+col."""
    m = len(deg)
    cdf = np.cumsum(p)
    cdf[-1] = 1.0

    def draw(rows_rep):
        u = rng.random(len(rows_rep))
        cols = np.searchsorted(cdf, u, side="right")
        np.minimum(cols, n - 1, out=cols)
        return rows_rep * n + cols

    keys = _uniq(draw(np.repeat(np.arange(m, dtype=np.int64), deg)))
    budget = 2 * int(deg.sum()) + 1024
    for rnd in range(rounds):
        have = np.bincount(keys // n, minlength=m)
        deficit = deg - have
        need = deficit > 0
        if not need.any():
            break
        # Oversample geometrically: the still-missing columns live in the thin tail of p.
        extra = np.where(need, (deficit + 1) << min(rnd + 1, 6), 0)
        if extra.sum() > budget:
            extra = np.where(need, np.minimum(extra, 4 * (deficit + 1)), 0)
        keys = _uniq(np.concatenate([keys, draw(np.repeat(np.arange(m, dtype=np.int64), extra))]))
    have = np.bincount(keys // n, minlength=m)
    short = np.flatnonzero(deg > have)
    if len(short):
        # Exact weighted draw without replacement for the few rows still short.
        bounds = np.searchsorted(keys, np.arange(m + 1, dtype=np.int64) * n)
        add = []
        for i in short:
            got = keys[bounds[i]:bounds[i + 1]] % n
            q = p.copy()
            q[got] = 0.0
            q_sum = q.sum()
            want = min(int(deg[i] - len(got)), int(np.count_nonzero(q)))
            if want > 0 and q_sum > 0:
                add.append(i * n + rng.choice(n, size=want, replace=False, p=q / q_sum))
        if add:
            keys = _uniq(np.concatenate([keys] + add))
    # Trim rows that overshot, dropping a uniformly random subset of their columns.
    rows = keys // n
    have = np.bincount(rows, minlength=m)
    if (have > deg).any():
        prio = rng.random(len(keys))
        order = np.lexsort((prio, rows))
        start = np.concatenate([[0], np.cumsum(have)[:-1]])
        pos = np.arange(len(keys)) - start[rows[order]]
        kept = order[pos < deg[rows[order]]]
        keys = np.sort(keys[kept])
    return keys


def _feature_matrix(w: Workload, rng) -> sp.csr_matrix:
    deg = _row_degrees(rng, w.m, w.n, w.nnz, w.row_dist)
    p = _col_probs(rng, w.n, w.col_dist)
    keys = _sample_distinct(rng, deg, p, w.n)
    rows = keys // w.n
    cols = keys % w.n
    if w.values == "uniform":
        vals = 1.0 - rng.random(len(keys))  # (0, 1]
    elif w.values == "tfidf":
        tf = np.log1p(np.maximum(rng.poisson(2.0, size=len(keys)), 1).astype(np.float64))
        df = np.bincount(cols, minlength=w.n).astype(np.float64)
        idf = np.log((1.0 + w.m) / (1.0 + df)) + 1.0
        vals = tf * idf[cols]
    else:
        raise ValueError(w.values)
    indptr = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=w.m))]).astype(np.int64)
    if w.normalize_rows:
        sq = np.add.reduceat(vals * vals, indptr[:-1]) if len(vals) else np.zeros(w.m)
        norms = np.sqrt(np.where(np.diff(indptr) > 0, sq, 1.0))
        vals = vals / np.repeat(norms, np.diff(indptr))
    A = sp.csr_matrix((vals, cols.astype(np.int32), indptr), shape=(w.m, w.n))
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    return A


def _label_matrix(w: Workload, rng) -> sp.csr_matrix:
    counts = np.minimum(rng.poisson(w.labels_per_row, size=w.m), w.n_labels).astype(np.int64)
    ranks = rng.permutation(w.n_labels).astype(np.float64)
    p = (ranks + 1.0) ** (-w.label_zipf)
    p /= p.sum()
    keys = _sample_distinct(rng, counts, p, w.n_labels)
    rows = keys // w.n_labels
    cols = (keys % w.n_labels).astype(np.int32)
    indptr = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=w.m))]).astype(np.int64)
    Y = sp.csr_matrix((np.ones(len(keys)), cols, indptr), shape=(w.m, w.n_labels))
    Y.sort_indices()
    return Y


@dataclass
class Problem:
    workload: Workload
    A: sp.csr_matrix
    Y: sp.csr_matrix
    meta: dict = field(default_factory=dict)


def make_problem(name: str) -> Problem:
    """Deterministic (A, Y) for one named workload."""
    w = WORKLOADS[name]
    rng = np.random.default_rng([w.seed, 20110423])
    A = _feature_matrix(w, rng)
    Y = _label_matrix(w, rng)
    return Problem(w, A, Y, {"nnz": int(A.nnz), "nnz_Y": int(Y.nnz)})


def fastpi_config_kwargs(w: Workload) -> dict:
    """FastpiConfig(alpha, k, seed) for a workload (reference ``pinv.py:32-46``)."""
    return {"alpha": w.alpha, "k": w.k, "seed": w.seed}
