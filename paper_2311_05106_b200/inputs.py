"""Seeded synthetic inputs shared by the product path, the tests and the bench.

This module holds NONE of the method's arithmetic (no scatter, no
connectivity rule, no neuron update): only seeded random numbers in the
shapes of the paper's workloads and bit packing.
Both the CUDA path and the CPU oracle consume what it produces.
"""
from __future__ import annotations

import numpy as np

# Listing S3: 4000 * scale neurons, 80 % excitatory, p = 80/N.
V0_MEAN, V0_STD = -55.0, 2.0          # V_initializer=Normal(-55., 2.)
V0_SEED = 42


def n_words(n: int) -> int:
    return (n + 31) // 32


def pack_bits(events: np.ndarray) -> np.ndarray:
    """uint8/bool [n] -> uint32 [ceil(n/32)], bit r&31 of word r>>5 (little-endian)."""
    ev = np.asarray(events).astype(bool)
    n = ev.shape[0]
    padded = np.zeros(n_words(n) * 32, bool)
    padded[:n] = ev
    bits = padded.reshape(-1, 32).astype(np.uint64)
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))
    return (bits * weights).sum(axis=1).astype(np.uint32)


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    """uint32 words -> uint8 [n]."""
    w = np.asarray(words, dtype=np.uint32)
    bits = ((w[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(np.uint8)
    return bits.reshape(-1)[:n].copy()


def spike_pattern(n: int, density: float, seed: int) -> np.ndarray:
    """Bernoulli(density) events, i.e. rate*dt per neuron (reading R27)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.random(n) < density).astype(np.uint8)


def lif_v0(n: int, seed: int = V0_SEED) -> np.ndarray:
    """V0 ~ Normal(-55, 2) in fp64 from PCG64, cast to fp32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.normal(V0_MEAN, V0_STD, n).astype(np.float32)


def hh_init(n: int, seed: int = V0_SEED):
    """COBA-HH initial state: V0 = E_L + 5 N(0,1) - 5 = -65 + 5 N(0,1) mV
    (the Brette 2007 / Brian2 COBAHH benchmark's initialiser, EXTERNAL).
    Gating variables start at fixed values near rest (m, h, n) = (0.05, 0.6,
    0.32); they are initial conditions, not derived from the model."""
    rng = np.random.Generator(np.random.PCG64(seed))
    v = (-65.0 + 5.0 * rng.standard_normal(n)).astype(np.float32)
    m = np.full(n, 0.05, np.float32)
    h = np.full(n, 0.6, np.float32)
    nk = np.full(n, 0.32, np.float32)
    return v, m, h, nk


def random_csr(n_rows: int, n_cols: int, p: float, seed: int,
               weights: str = "homo", w0: float = 1.0, w1: float = 0.0,
               integer_weights: bool = False):
    """Random CSR with Bernoulli(p)-like rows: per-row count ~ Binomial(n_cols, p),
    columns drawn uniformly without replacement, sorted (canonical CSR).
    weights: 'homo' -> data None; 'uniform' -> U[w0, w1); 'normal' -> N(w0, w1);
    integer_weights -> small integers in [-4, 4] (exact in any summation order).
    Returns (indptr int64, indices int32, data float32 | None)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    counts = rng.binomial(n_cols, p, n_rows).astype(np.int64)
    indptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    indices = np.empty(nnz, np.int32)
    for r in range(n_rows):
        c = int(counts[r])
        if c:
            cols = rng.choice(n_cols, size=c, replace=False)
            cols.sort()
            indices[indptr[r]:indptr[r + 1]] = cols
    data = None
    if integer_weights:
        data = rng.integers(-4, 5, nnz).astype(np.float32)
    elif weights == "uniform":
        data = rng.uniform(w0, w1, nnz).astype(np.float32)
    elif weights == "normal":
        data = rng.normal(w0, w1, nnz).astype(np.float32)
    return indptr, indices, data


def fixed_fanin_csr_fast(n_rows: int, n_cols: int, p: float, seed: int):
    """Large random CSR, vectorised: per-row Binomial(n_cols, p) counts and
    uniform columns with replacement, sorted per row; duplicates within a
    row are dropped (their share is ~ count^2 / (2 n_cols), < 0.1 % at the
    configs' fan-outs).  Used for the 400k-neuron HH network and the CSR
    microbenchmark, where the per-row loop of random_csr is too slow."""
    rng = np.random.Generator(np.random.PCG64(seed))
    counts = rng.binomial(n_cols, p, n_rows).astype(np.int64)
    rows = np.repeat(np.arange(n_rows, dtype=np.int64), counts)
    cols = rng.integers(0, n_cols, rows.shape[0], dtype=np.int64)
    key = rows * np.int64(n_cols) + cols
    key = np.unique(key)                       # sorts and drops duplicates
    rows = key // n_cols
    cols = (key - rows * n_cols).astype(np.int32)
    indptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=indptr[1:])
    return indptr, cols, None


def bernoulli_csr(n_rows: int, n_cols: int, p: float, seed: int, weights: str = "homo",
                  w0: float = 1.0, w1: float = 0.0, chunk: int = 2048):
    """Large random CSR with every entry present independently with
    probability p (per-row Binomial(n_cols, p) fan-out, no duplicates),
    vectorised by rows of Geo(p) column gaps: row r's columns are the
    partial sums of its gaps (minus one) below n_cols.  Sorted per row.
    weights: 'homo' -> data None; 'uniform' -> U[w0, w1).
    Returns (indptr int64, indices int32, data float32 | None)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    mean = n_cols * p
    width = int(mean + 10.0 * np.sqrt(mean + 1.0) + 16)
    idx_parts, counts = [], np.zeros(n_rows, np.int64)
    for r0 in range(0, n_rows, chunk):
        r1 = min(n_rows, r0 + chunk)
        pos = np.cumsum(rng.geometric(p, size=(r1 - r0, width)), axis=1, dtype=np.int64) - 1
        short = np.nonzero(pos[:, -1] < n_cols)[0]
        while short.size:                       # extend the rare rows that need more gaps
            ext = pos[short, -1:] + np.cumsum(rng.geometric(p, size=(short.size, width)),
                                              axis=1, dtype=np.int64)
            grown = np.full((pos.shape[0], pos.shape[1] + width), np.iinfo(np.int64).max,
                            np.int64)
            grown[:, :pos.shape[1]] = pos
            grown[short, pos.shape[1]:] = ext
            pos = grown
            short = np.nonzero(pos[:, -1] < n_cols)[0]
        keep = pos < n_cols
        counts[r0:r1] = keep.sum(axis=1)
        idx_parts.append(pos[keep].astype(np.int32))
    indptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = np.concatenate(idx_parts) if idx_parts else np.zeros(0, np.int32)
    data = None
    if weights == "uniform":
        data = rng.uniform(w0, w1, indices.shape[0]).astype(np.float32)
    return indptr, indices, data
