"""Synthetic inputs of the correction loop (BASELINE.json configs).

f = the reference's deterministic synthetic field (field.cpp:229-250), ξ = rel ×
(max − min) (field.cpp:42-50), f̂ = the reference base codec's reconstruction
(base_codec.cpp:76-120) — all restated bit-exactly in ``csrc/inputs.cpp`` and
parallelised (tests/test_inputs.py pins them against the reference).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from .build import INPUTS_SO

KINDS = {"gaussian-mixture": 0, "trig": 1, "random-smooth": 2, "multi-scale": 3}

_lib = None


def _library():
    global _lib
    if _lib is None:
        if not os.path.exists(INPUTS_SO):
            raise RuntimeError(f"{INPUTS_SO} missing (run paper_2406_09423_b200.build())")
        _lib = C.CDLL(INPUTS_SO)
    return _lib


def _suf(dtype):
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


def generate(kind: str, dims, seed: int = 0, dtype=np.float32, a: float = 0.2) -> np.ndarray:
    """generate_synthetic<T> (field.cpp:229-250); 'multi-scale' = gm(seed) + a*rs(seed+1)."""
    out = np.empty(int(np.prod(dims)), dtype)
    d = (C.c_uint64 * len(dims))(*dims)
    rc = getattr(_library(), f"mssz_in_generate_{_suf(dtype)}")(
        KINDS[kind], len(dims), d, C.c_uint64(seed), C.c_double(a), out.ctypes.data_as(C.c_void_p))
    if rc:
        raise ValueError(f"generate failed ({rc}) for {kind} {dims}")
    return out


def value_range(values: np.ndarray):
    lo = C.c_double()
    hi = C.c_double()
    getattr(_library(), f"mssz_in_value_range_{_suf(values.dtype)}")(
        C.c_uint64(values.size), values.ctypes.data_as(C.c_void_p), C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def resolve_rel(values: np.ndarray, magnitude: float) -> float:
    """resolve_bound with a relative bound (field.cpp:42-50)."""
    if not magnitude > 0:
        raise ValueError("error bound must be > 0")
    lo, hi = value_range(values)
    if hi == lo:
        raise ValueError("relative bound over a constant field (zero range)")
    return magnitude * (hi - lo)


def compress_base(dims, values: np.ndarray, xi: float) -> np.ndarray:
    """compress_base(...).reconstruction (base_codec.cpp:76-120)."""
    recon = np.empty_like(values)
    esc = C.c_uint64()
    d = (C.c_uint64 * len(dims))(*dims)
    rc = getattr(_library(), f"mssz_in_compress_base_recon_{_suf(values.dtype)}")(
        len(dims), d, values.ctypes.data_as(C.c_void_p), C.c_double(xi),
        recon.ctypes.data_as(C.c_void_p), C.byref(esc))
    if rc:
        raise ValueError(f"compress_base failed ({rc})")
    return recon


@dataclass(frozen=True)
class Config:
    name: str
    kind: str
    dims: tuple
    rel: float
    seed: int = 0
    subloop_cap: int = 640
    a: float = 0.2
    note: str = ""


# BASELINE.json "configs"
CONFIGS = {
    "C1": Config("C1", "gaussian-mixture", (512, 512), 1e-3,
                 note="2D 512x512 Gaussian-mixture, rel eb 1e-3"),
    "C2": Config("C2", "random-smooth", (177, 95, 48), 1e-3,
                 note="3D 177x95x48 AT-shaped (random-smooth), rel eb 1e-3"),
    "C2-trig": Config("C2-trig", "trig", (177, 95, 48), 1e-3,
                      note="3D 177x95x48 AT-shaped (trig), rel eb 1e-3"),
    "C3": Config("C3", "random-smooth", (512, 512, 512), 1e-3, subloop_cap=100000,
                 note="3D 512^3 Nyx-shaped (random-smooth), rel eb 1e-3"),
    "C4": Config("C4", "multi-scale", (1024, 1024, 1024), 1e-3, subloop_cap=100000,
                 note="3D 1024^3 multi-scale gm + 0.2*rs, rel eb 1e-3"),
    "C5": Config("C5", "gaussian-mixture", (3600, 2400), 1e-4, subloop_cap=100000,
                 note="2D 3600x2400 CESM-shaped Gaussian-mixture, rel eb 1e-4"),
}


def make_inputs(cfg: Config, dims=None, dtype=np.float32):
    """(f, f̂, ξ) for a config (optionally at other dims, e.g. a bounded CPU sample)."""
    dims = tuple(dims or cfg.dims)
    f = generate(cfg.kind, dims, cfg.seed, dtype, cfg.a)
    xi = resolve_rel(f, cfg.rel)
    fh = compress_base(dims, f, xi)
    return f, fh, xi
