"""Config-size parity: digests of full-size outputs (test infrastructure).

The generator (tests/golden/make_config_digests.py, run in the container that
has /root/reference) and the GPU tests (tests/test_gpu_config.py) share these
helpers, so a digest computed from the device's output on the GPU box is
computed by exactly the same numpy code as the committed one.

Per output array:
* ``sha256`` of the C-order bytes (bitwise claims: stencils, elementwise);
* ``rowsum`` = ``X.reshape(X.shape[0], -1).sum(axis=1)`` (numpy pairwise);
* ``min`` / ``max`` / ``nan``;
* ``samples`` at ``sample_index(size)``, a fixed multiplicative-hash index
  set (no stored indices), or the full array (``values``) when small;
* for re-associated float outputs: ``exact`` (an 80-bit long-double
  evaluation of the same chain) and ``terms`` (the chain's first-order
  rounding-error magnitude, Σ|terms| per element) at the same points, for the
  criterion ``|gpu - exact| <= |oracle - exact| + 4 eps terms``.
"""

from __future__ import annotations

import hashlib

import numpy as np

N_SAMPLES = 100_000
FULL_MAX = 100_000
EPS = np.finfo(np.float64).eps


def sample_index(size: int) -> np.ndarray:
    """Deterministic spread of N_SAMPLES flat indices (Knuth multiplicative
    hash of 0..K-1 modulo size), sorted and de-duplicated."""
    k = np.arange(min(N_SAMPLES, size), dtype=np.uint64)
    idx = (k * np.uint64(2654435761) + np.uint64(12345)) % np.uint64(size)
    return np.unique(idx.astype(np.int64))


def picks(size: int) -> np.ndarray:
    """The flat indices a digest records values at (all when small)."""
    return np.arange(size, dtype=np.int64) if size <= FULL_MAX else sample_index(size)


def digest(x) -> dict:
    x = np.ascontiguousarray(x)
    d = {
        "shape": np.asarray(x.shape, dtype=np.int64),
        "sha256": np.frombuffer(hashlib.sha256(x.tobytes()).digest(), dtype=np.uint8),
        "min": np.asarray(np.nanmin(x) if x.size else 0.0),
        "max": np.asarray(np.nanmax(x) if x.size else 0.0),
        "nan": np.asarray(int(np.isnan(x).sum()) if x.dtype.kind == "f" else 0),
    }
    if x.ndim >= 1 and x.size:
        d["rowsum"] = x.reshape(x.shape[0], -1).sum(axis=1)
    d["values"] = x.reshape(-1)[picks(x.size)] if x.size else x.reshape(-1)
    return d


def pack(prefix: str, d: dict) -> dict:
    return {f"{prefix}/{k}": v for k, v in d.items()}


def unpack(blob, prefix: str) -> dict:
    p = prefix + "/"
    return {k[len(p):]: blob[k] for k in blob.files if k.startswith(p)}


def sha(x) -> bytes:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).digest()


def rel_err(a, b) -> float:
    """pkg/tests/conftest.py:85-93: max |a-b| / max(|b|, 1)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    with np.errstate(invalid="ignore"):
        d = np.abs(a - b) / np.maximum(np.abs(b), 1.0)
    d = np.where(np.isnan(a) & np.isnan(b), 0.0, d)
    return float(np.max(np.nan_to_num(d, nan=np.inf)))


def exact_criterion(gpu, oracle, exact, terms, k: float = 4.0):
    """Per element: |gpu - exact| <= |oracle - exact| + k eps terms.
    Returns (ok, worst slack ratio, gpu max abs error vs exact, oracle max
    abs error vs exact)."""
    gpu = np.asarray(gpu, dtype=np.longdouble)
    oracle = np.asarray(oracle, dtype=np.longdouble)
    exact = np.asarray(exact, dtype=np.longdouble)
    eg = np.abs(gpu - exact)
    eo = np.abs(oracle - exact)
    bound = eo + k * EPS * np.asarray(terms, dtype=np.longdouble)
    ratio = np.where(bound > 0, eg / np.where(bound > 0, bound, 1), np.where(eg > 0, np.inf, 0))
    return bool(np.all(eg <= bound)), float(np.max(ratio)), float(np.max(eg)), float(np.max(eo))


def make_inputs(param_order, shapes: dict, seed: int, round_f32=()):
    """pkg/tests/conftest.py:38-49 semantics in signature order: arrays
    uniform(-1, 1), f64 scalars uniform(0.5, 1.5); integer params are
    bindings and draw nothing.  ``shapes[name]`` is a tuple (array) or ()
    (f64 scalar); names missing from ``shapes`` are integer params.
    ``round_f32``: arrays rounded to float32 after drawing (the f32 configs)."""
    rng = np.random.default_rng(seed)
    out = {}
    for p in param_order:
        if p not in shapes:
            continue
        shp = shapes[p]
        if shp:
            out[p] = rng.uniform(-1.0, 1.0, size=shp)
            if p in round_f32:
                out[p] = out[p].astype(np.float32).astype(np.float64)
        else:
            out[p] = float(rng.uniform(0.5, 1.5))
    return out
