"""mssz-b200: B200-native MSz segmentation-correction loop (arXiv 2406.09423).

Python host mirror of the reference's ``proj/core`` hot-path API
(``edit_engine.hpp``, ``mss.hpp``, ``grid.hpp``, ``errors.hpp``) over the
C-ABI in ``include/mssz_cuda.h``.  Names, argument meaning and error kinds
follow the reference so callers (and the parity tests) read like the
reference's own:

    topo  = build_topology([512, 512])                       # grid.hpp:51
    edits = derive_edits(topo, f, fhat, xi, DeriveOptions(), stats)  # edit_engine.hpp:183
    g     = apply_edits(topo, fhat, edits)                    # edit_engine.hpp:188

Every compute entry point runs on the GPU through ``_lib/libmssz_b200.so``;
there is no CPU fallback — without the built library or a CUDA device the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Optional, Union

import numpy as np

from .build import CUDA_SO, INPUTS_SO, build  # noqa: F401

__all__ = [
    "ErrKind", "Error", "GridTopology", "build_topology", "DeriveOptions", "EditStats",
    "EditSet", "DirectionField", "SegmentationLabels", "CriticalSet", "FalseCriticalReport",
    "derive_edits", "derive_edits_into", "derive_edits_device", "compute_directions",
    "compute_direction_codes", "compute_labels", "classify_critical", "detect_false_critical",
    "detect_kind", "lower_step", "representable_floor", "apply_edits", "segmentation_equal",
    "library", "build", "slab_range", "derive_edits_slabs", "SlabComm",
    "VerificationReport", "build_report", "build_report_device", "segmentation", "export_labels",
    "compress_base", "decompress_base", "encode_edits", "PROF_CLASSES", "profile_mask",
]

FPMAX, FPMIN, FNMAX, FNMIN = 0, 1, 2, 3


class ErrKind(IntEnum):
    """errors.hpp:9-16 (1:1 with CLI exit codes)."""

    usage = 2
    io = 3
    bound_violation = 4
    non_convergence = 5
    corrupt_archive = 6
    internal = 7
    callback = 98  # on_batch raised: the correction was abandoned (the exception is re-raised)
    cuda = 99


ERR_CALLBACK = 98


class Error(RuntimeError):
    """errors.hpp:18-28 — ``kind()`` and ``exit_code()`` as in the reference."""

    def __init__(self, kind: int, msg: str):
        super().__init__(msg)
        try:
            self._kind = ErrKind(kind)
        except ValueError:
            self._kind = ErrKind.internal
        self.msg = msg

    def kind(self) -> ErrKind:
        return self._kind

    def exit_code(self) -> int:
        return int(self._kind)


# ---------------------------------------------------------------- topology
_MAX_VERTICES = 1 << 40  # grid.cpp:19


@dataclass(frozen=True)
class GridTopology:
    """grid.hpp:25-47 (row-major, axis 0 fastest; dims[2] == 1 in 2D)."""

    ndims: int
    dims: tuple
    vertex_count: int

    def coords_of(self, v: int):
        x = v % self.dims[0]
        y = (v // self.dims[0]) % self.dims[1]
        z = v // (self.dims[0] * self.dims[1])
        return x, y, z

    def index_of(self, x: int, y: int, z: int = 0) -> int:
        return x + self.dims[0] * (y + self.dims[1] * z)

    @property
    def extents(self):
        return list(self.dims[: self.ndims])


def build_topology(dims) -> GridTopology:
    """build_topology (grid.cpp:39-55): usage error on bad extents."""
    dims = [int(d) for d in dims]
    if len(dims) not in (2, 3):
        raise Error(ErrKind.usage, "dims must have 2 or 3 extents")
    count = 1
    for d in dims:
        if d < 2:
            raise Error(ErrKind.usage, "every grid extent must be >= 2")
        if d > _MAX_VERTICES // count:
            raise Error(ErrKind.usage, "grid exceeds the address-space cap")
        count *= d
    full = tuple(dims + [1] * (3 - len(dims)))
    return GridTopology(len(dims), full, count)


# ---------------------------------------------------------------- results
@dataclass
class DeriveOptions:
    """DeriveOptions<T> (edit_engine.hpp:70-82); ``device`` replaces ExecPolicy."""

    outer_cap: int = 1000
    subloop_cap: int = 640
    r_cap: int = 100000
    force: bool = False
    device: int = -1
    on_batch: Optional[Callable[[np.ndarray], None]] = None
    # "every": after every fix batch (the reference's call sites); "phases": only
    # after each complete C pass and each R iteration, the device loop running
    # at full speed in between (snapshots of large fields)
    on_batch_mode: str = "every"
    # per-kernel CUDA-event timing into EditStats.kernel_ms: True = every class,
    # or an int mask from profile_mask(...) for selected classes only
    profile: Union[bool, int] = False


@dataclass
class EditStats:
    """EditStats (edit_engine.hpp:54-68) plus the device counters."""

    outer_iterations: int = 0
    c_passes: int = 0
    sub_iterations: list = field(default_factory=lambda: [0, 0, 0, 0])
    r_iterations: int = 0
    effective_edits: int = 0
    touched: int = 0
    input_bound_violations: int = 0
    direction_seconds: float = 0.0
    label_seconds: float = 0.0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    device_seconds: float = 0.0
    label_passes: int = 0
    label_rounds: int = 0
    detect_sweeps: int = 0
    frontier_vertices: int = 0
    kernel_launches: int = 0
    big_batches: int = 0
    huge_batches: int = 0
    label_tiles: int = 0
    rfix_tiles: int = 0
    sparse_iterations: int = 0
    sparse_up: int = 0
    rfix_divergent: int = 0
    subloop_items: int = 0
    subloop_edits: int = 0
    skipped_subloops: int = 0
    kernel_count: list = field(default_factory=lambda: [0] * 16)
    kernel_ms: list = field(default_factory=lambda: [0.0] * 16)

    def kernel_profile(self) -> dict:
        return {name: {"launches": self.kernel_count[i], "ms": self.kernel_ms[i]}
                for i, name in enumerate(PROF_CLASSES)}

    def sub_iterations_total(self) -> int:
        return sum(self.sub_iterations)


@dataclass
class EditSet:
    """EditSet<T> (edit_engine.hpp:45-52): strictly increasing indices, absolute values."""

    indices: np.ndarray
    values: np.ndarray

    def size(self) -> int:
        return int(self.indices.size)

    def empty(self) -> bool:
        return self.indices.size == 0


@dataclass
class DirectionField:
    """mss.hpp:24-31."""

    asc: np.ndarray
    desc: np.ndarray

    def is_max(self, v: int) -> bool:
        return int(self.asc[v]) == v

    def is_min(self, v: int) -> bool:
        return int(self.desc[v]) == v


@dataclass
class SegmentationLabels:
    """mss.hpp:37-42."""

    max_label: np.ndarray
    min_label: np.ndarray

    def __eq__(self, other) -> bool:
        return bool(np.array_equal(self.max_label, other.max_label)
                    and np.array_equal(self.min_label, other.min_label))


@dataclass
class CriticalSet:
    """mss.hpp:32-35."""

    maxima: np.ndarray
    minima: np.ndarray


@dataclass
class FalseCriticalReport:
    """edit_engine.hpp:29-41 (first matching class wins)."""

    fp_max: np.ndarray
    fp_min: np.ndarray
    fn_max: np.ndarray
    fn_min: np.ndarray

    def empty(self) -> bool:
        return self.total() == 0

    def total(self) -> int:
        return int(self.fp_max.size + self.fp_min.size + self.fn_max.size + self.fn_min.size)


# ---------------------------------------------------------------- C-ABI
class _Options(C.Structure):
    _fields_ = [
        ("outer_cap", C.c_uint64), ("subloop_cap", C.c_uint64), ("r_cap", C.c_uint64),
        ("force", C.c_int32), ("device", C.c_int32),
        ("on_batch", C.c_void_p), ("on_batch_user", C.c_void_p),
        ("profile", C.c_int32), ("on_batch_mode", C.c_int32),
    ]


class _Stats(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_uint64), ("c_passes", C.c_uint64),
        ("sub_iterations", C.c_uint64 * 4), ("r_iterations", C.c_uint64),
        ("effective_edits", C.c_uint64), ("touched", C.c_uint64),
        ("input_bound_violations", C.c_uint64), ("direction_seconds", C.c_double),
        ("label_seconds", C.c_double), ("h2d_seconds", C.c_double),
        ("d2h_seconds", C.c_double), ("device_seconds", C.c_double),
        ("label_passes", C.c_uint64), ("label_rounds", C.c_uint64),
        ("detect_sweeps", C.c_uint64), ("frontier_vertices", C.c_uint64),
        ("kernel_launches", C.c_uint64), ("big_batches", C.c_uint64),
        ("huge_batches", C.c_uint64), ("label_tiles", C.c_uint64), ("rfix_tiles", C.c_uint64),
        ("sparse_iterations", C.c_uint64), ("sparse_up", C.c_uint64), ("rfix_divergent", C.c_uint64),
        ("subloop_items", C.c_uint64), ("subloop_edits", C.c_uint64),
        ("skipped_subloops", C.c_uint64),
        ("kernel_count", C.c_uint64 * 16), ("kernel_ms", C.c_double * 16),
    ]

    def fill(self, st: EditStats) -> EditStats:
        for name, _ in self._fields_:
            v = getattr(self, name)
            setattr(st, name, list(v) if name in _ARRAY_FIELDS else v)
        return st


_ARRAY_FIELDS = ("sub_iterations", "kernel_count", "kernel_ms")
PROF_CLASSES = ["validate", "directions", "detect_kind", "detect_all", "subloop", "label_init",
                "label_jump", "rfix", "frontier", "compact", "label_finish", "fix", "sparse",
                "detect_dirty"]


def profile_mask(*classes: str) -> int:
    """DeriveOptions.profile value that times only the named kernel classes."""
    return sum(1 << (PROF_CLASSES.index(c) + 1) for c in classes)


_BATCH_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_void_p)

# every symbol include/mssz_cuda.h declares (tests check the exports)
EXPORTS = [
    "mssz_cu_default_options", "mssz_cu_last_error", "mssz_cu_free", "mssz_cu_device_count",
    "mssz_cu_version", "mssz_cu_release_workspace", "mssz_cu_compute_labels",
    "mssz_cu_classify_critical", "mssz_cu_slab_range", "mssz_cu_comm_unique_id",
    "mssz_cu_comm_init", "mssz_cu_comm_destroy", "mssz_cu_batch_phase",
] + [
    f"mssz_cu_{name}_{suf}" for suf in ("f32", "f64") for name in (
        "derive_edits", "derive_edits_into", "derive_edits_device", "compute_directions",
        "compute_direction_codes", "detect_false_critical", "detect_kind", "lower_step",
        "representable_floor", "apply_edits", "derive_edits_slab", "derive_edits_slab_device",
        "derive_edits_slabs_local", "verify", "verify_device", "segmentation", "compress_base",
        "decompress_base", "encode_edits", "r_targets")
]

_lib = None


def _nccl_path() -> Optional[str]:
    """torch's bundled libnccl.so.2 (nvidia-nccl wheel), if installed."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(base, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return cand
    return None


def library() -> C.CDLL:
    """Loads ``_lib/libmssz_b200.so`` (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if "MSSZ_NCCL_LIBRARY" not in os.environ:
            path = _nccl_path()
            if path:
                os.environ["MSSZ_NCCL_LIBRARY"] = path
        if not os.path.exists(CUDA_SO):
            raise Error(ErrKind.cuda, f"CUDA extension missing: {CUDA_SO} (run build())")
        lib = C.CDLL(CUDA_SO)
        lib.mssz_cu_last_error.restype = C.c_char_p
        lib.mssz_cu_version.restype = C.c_char_p
        lib.mssz_cu_free.argtypes = [C.c_void_p]
        _lib = lib
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise Error(rc, library().mssz_cu_last_error().decode())


def _suf(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise Error(ErrKind.usage, f"unsupported dtype {dt} (f32 or f64)")


def _ctype(dtype):
    return C.c_float if np.dtype(dtype) == np.float32 else C.c_double


def _dims(topo: GridTopology):
    return (C.c_uint64 * 3)(*topo.dims)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _field(topo: GridTopology, a, name: str, dtype=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.size != topo.vertex_count:
        raise Error(ErrKind.io, f"{name}: {a.size} values for a grid of {topo.vertex_count}")
    return a.reshape(-1)


def _options(opts: Optional[DeriveOptions], dtype, keep: list) -> _Options:
    o = opts or DeriveOptions()
    if o.on_batch_mode not in ("every", "phases"):
        raise Error(ErrKind.usage, f"on_batch_mode must be 'every' or 'phases', not {o.on_batch_mode!r}")
    co = _Options(o.outer_cap, o.subloop_cap, o.r_cap, int(o.force), o.device, None, None,
                  int(o.profile), 0 if o.on_batch_mode == "every" else 1)
    if o.on_batch is not None:
        ctype = _ctype(dtype)

        def _cb(ptr, n, user):
            # an exception must not be swallowed by ctypes: store it, tell the
            # engine to abort (nonzero), re-raise it after the call (_check_cb)
            try:
                arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,))
                o.on_batch(arr.copy())
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised by _check_cb
                keep.append(_CallbackFailure(e))
                return 1

        cb = _BATCH_CB(_cb)
        keep.append(cb)
        co.on_batch = C.cast(cb, C.c_void_p)
    return co


class _CallbackFailure:
    def __init__(self, exc: BaseException):
        self.exc = exc


PHASE_KINDS = ("batch", "c_pass", "r_iteration")


def batch_phase() -> tuple:
    """Inside an on_batch callback: (kind, outer iteration, index) of the snapshot,
    kind in PHASE_KINDS (mssz_cu_batch_phase)."""
    out = np.zeros(3, np.uint64)
    _check(library().mssz_cu_batch_phase(_p(out)))
    return PHASE_KINDS[int(out[0])], int(out[1]), int(out[2])


def _check_cb(rc: int, keep: list) -> None:
    """_check, re-raising an on_batch exception as the reference's would propagate."""
    if rc == ERR_CALLBACK:
        for k in keep:
            if isinstance(k, _CallbackFailure):
                raise k.exc
    _check(rc)


def derive_edits(topo: GridTopology, original, decompressed, xi: float,
                 opts: Optional[DeriveOptions] = None,
                 stats: Optional[EditStats] = None) -> EditSet:
    """derive_edits<T> (edit_engine.hpp:183-186) on the GPU; host arrays in, EditSet out."""
    f = _field(topo, original, "original")
    fh = _field(topo, decompressed, "decompressed", f.dtype)
    suf = _suf(f.dtype)
    keep: list = []
    co = _options(opts, f.dtype, keep)
    idx = C.POINTER(C.c_uint64)()
    val = C.POINTER(_ctype(f.dtype))()
    count = C.c_uint64()
    st = _Stats()
    lib = library()
    rc = getattr(lib, f"mssz_cu_derive_edits_{suf}")(
        topo.ndims, _dims(topo), _p(f), _p(fh), C.c_double(xi), C.byref(co), C.byref(idx),
        C.byref(val), C.byref(count), C.byref(st))
    _check_cb(rc, keep)
    k = count.value
    indices = np.ctypeslib.as_array(idx, shape=(max(k, 1),))[:k].copy()
    values = np.ctypeslib.as_array(val, shape=(max(k, 1),))[:k].copy()
    lib.mssz_cu_free(C.cast(idx, C.c_void_p))
    lib.mssz_cu_free(C.cast(val, C.c_void_p))
    if stats is not None:
        st.fill(stats)
    return EditSet(indices, values)


def derive_edits_into(topo: GridTopology, f_ptr: int, fh_ptr: int, xi: float, idx_ptr: int,
                      val_ptr: int, capacity: int, dtype=np.float32,
                      opts: Optional[DeriveOptions] = None) -> tuple:
    """Host-pointer variant with caller-owned (e.g. pinned) output buffers -> (count, EditStats)."""
    suf = _suf(dtype)
    keep: list = []
    co = _options(opts, dtype, keep)
    count = C.c_uint64()
    st = _Stats()
    rc = getattr(library(), f"mssz_cu_derive_edits_into_{suf}")(
        topo.ndims, _dims(topo), C.c_void_p(f_ptr), C.c_void_p(fh_ptr), C.c_double(xi),
        C.byref(co), C.c_void_p(idx_ptr), C.c_void_p(val_ptr), C.c_uint64(capacity),
        C.byref(count), C.byref(st))
    _check_cb(rc, keep)
    return count.value, st.fill(EditStats())


def derive_edits_device(topo: GridTopology, d_f: int, d_fh: int, xi: float, d_idx: int,
                        d_val: int, capacity: int, dtype=np.float32,
                        opts: Optional[DeriveOptions] = None, stream: int = 0) -> tuple:
    """Device-resident variant (CUDA pointers, optional stream) -> (count, EditStats)."""
    suf = _suf(dtype)
    keep: list = []
    co = _options(opts, dtype, keep)
    count = C.c_uint64()
    st = _Stats()
    rc = getattr(library(), f"mssz_cu_derive_edits_device_{suf}")(
        topo.ndims, _dims(topo), C.c_void_p(d_f), C.c_void_p(d_fh), C.c_double(xi),
        C.byref(co), C.c_void_p(d_idx), C.c_void_p(d_val), C.c_uint64(capacity),
        C.byref(count), C.byref(st), C.c_void_p(stream or None))
    _check_cb(rc, keep)
    return count.value, st.fill(EditStats())


def compute_directions(topo: GridTopology, values) -> DirectionField:
    """compute_directions<T> (mss.hpp:44-50): u64 steepest neighbour ids, SELF = own id."""
    v = _field(topo, values, "values")
    asc = np.empty(topo.vertex_count, np.uint64)
    desc = np.empty(topo.vertex_count, np.uint64)
    _check(getattr(library(), f"mssz_cu_compute_directions_{_suf(v.dtype)}")(
        topo.ndims, _dims(topo), _p(v), _p(asc), _p(desc)))
    return DirectionField(asc, desc)


def compute_direction_codes(topo: GridTopology, values) -> np.ndarray:
    """Packed device representation: low nibble asc slot, high nibble desc slot, 15 = SELF."""
    v = _field(topo, values, "values")
    out = np.empty(topo.vertex_count, np.uint8)
    _check(getattr(library(), f"mssz_cu_compute_direction_codes_{_suf(v.dtype)}")(
        topo.ndims, _dims(topo), _p(v), _p(out)))
    return out


def compute_labels(topo: GridTopology, directions: DirectionField) -> SegmentationLabels:
    """compute_labels (mss.hpp:58-60); raises internal on a corrupt (cyclic) field."""
    asc = _field(topo, directions.asc, "asc", np.uint64)
    desc = _field(topo, directions.desc, "desc", np.uint64)
    M = np.empty(topo.vertex_count, np.uint64)
    m = np.empty(topo.vertex_count, np.uint64)
    _check(library().mssz_cu_compute_labels(topo.ndims, _dims(topo), _p(asc), _p(desc), _p(M),
                                            _p(m)))
    return SegmentationLabels(M, m)


def classify_critical(directions: DirectionField) -> CriticalSet:
    """classify_critical (mss.cpp:40-47): sorted maxima / minima."""
    asc = np.ascontiguousarray(directions.asc, np.uint64)
    desc = np.ascontiguousarray(directions.desc, np.uint64)
    n = asc.size
    mx = np.empty(n, np.uint64)
    mn = np.empty(n, np.uint64)
    nmx = C.c_uint64()
    nmn = C.c_uint64()
    _check(library().mssz_cu_classify_critical(C.c_uint64(n), _p(asc), _p(desc), _p(mx),
                                               C.byref(nmx), _p(mn), C.byref(nmn)))
    return CriticalSet(mx[: nmx.value].copy(), mn[: nmn.value].copy())


def detect_false_critical(topo: GridTopology, original, edited) -> FalseCriticalReport:
    """EditState::detect_false_critical (edit_engine.cpp:134-158) for (f, g)."""
    f = _field(topo, original, "original")
    g = _field(topo, edited, "edited", f.dtype)
    n = topo.vertex_count
    counts = np.zeros(4, np.uint64)
    lists = np.zeros(4 * n, np.uint64)
    _check(getattr(library(), f"mssz_cu_detect_false_critical_{_suf(f.dtype)}")(
        topo.ndims, _dims(topo), _p(f), _p(g), _p(counts), _p(lists)))
    parts = [lists[k * n: k * n + int(counts[k])].copy() for k in range(4)]
    return FalseCriticalReport(*parts)


def detect_kind(topo: GridTopology, original, edited, kind: int) -> np.ndarray:
    """EditState::detect_kind (edit_engine.cpp:104-132): sorted, per kind, non-exclusive."""
    f = _field(topo, original, "original")
    g = _field(topo, edited, "edited", f.dtype)
    out = np.empty(topo.vertex_count, np.uint64)
    cnt = C.c_uint64()
    _check(getattr(library(), f"mssz_cu_detect_kind_{_suf(f.dtype)}")(
        topo.ndims, _dims(topo), _p(f), _p(g), int(kind), _p(out), C.byref(cnt)))
    return out[: cnt.value].copy()


@dataclass
class RBatchTargets:
    """One R batch's target set (run_r_loop, edit_engine.cpp:336-352)."""

    targets: np.ndarray      # sorted distinct troublemaker targets v_t
    false_critical: int      # false critical points of (f, g): the R gate (:338)
    sources: int             # divergent mismatched (vertex, family) pairs = distinct v_i
    path: str                # "tiled" or "sparse"


def r_targets(topo: GridTopology, original, edited, mode: str = "tiled") -> RBatchTargets:
    """The R-batch targets the engine computes for (f, g): tiled pass or sparse Up(X) pass."""
    f = _field(topo, original, "original")
    g = _field(topo, edited, "edited", f.dtype)
    out = np.empty(topo.vertex_count, np.uint64)
    cnt = C.c_uint64()
    info = np.zeros(3, np.uint64)
    _check(getattr(library(), f"mssz_cu_r_targets_{_suf(f.dtype)}")(
        topo.ndims, _dims(topo), _p(f), _p(g), {"tiled": 0, "sparse": 1}[mode], _p(out),
        C.byref(cnt), _p(info)))
    return RBatchTargets(out[: cnt.value].copy(), int(info[0]), int(info[1]),
                         "sparse" if info[2] else "tiled")


def lower_step(g, f, xi: float):
    """Element-wise EditState::lower_step (edit_engine.cpp:75-86) -> (new g, moved mask)."""
    f = np.ascontiguousarray(f).reshape(-1)
    g = np.ascontiguousarray(g, f.dtype).reshape(-1)
    out = np.empty_like(g)
    moved = np.empty(g.size, np.uint8)
    _check(getattr(library(), f"mssz_cu_lower_step_{_suf(f.dtype)}")(
        C.c_uint64(g.size), _p(g), _p(f), C.c_double(xi), _p(out), _p(moved)))
    return out, moved.astype(bool)


def representable_floor(f, xi: float) -> np.ndarray:
    """Element-wise representable_floor (edit_engine.cpp:22-29)."""
    f = np.ascontiguousarray(f).reshape(-1)
    out = np.empty_like(f)
    _check(getattr(library(), f"mssz_cu_representable_floor_{_suf(f.dtype)}")(
        C.c_uint64(f.size), _p(f), C.c_double(xi), _p(out)))
    return out


def apply_edits(topo: GridTopology, decompressed, edits: EditSet) -> np.ndarray:
    """apply_edits<T> (edit_engine.hpp:188-190); corrupt_archive on bad input."""
    fh = _field(topo, decompressed, "decompressed")
    if edits.indices.size != edits.values.size:
        raise Error(ErrKind.corrupt_archive, "edit set index/value length mismatch")
    idx = np.ascontiguousarray(edits.indices, np.uint64)
    vals = np.ascontiguousarray(edits.values, fh.dtype)
    out = np.empty_like(fh)
    _check(getattr(library(), f"mssz_cu_apply_edits_{_suf(fh.dtype)}")(
        C.c_uint64(fh.size), _p(fh), _p(idx), _p(vals), C.c_uint64(idx.size), _p(out)))
    return out


def segmentation_equal(a: SegmentationLabels, b: SegmentationLabels):
    """segmentation_equal (mss.cpp:122-133) -> (match mask, mismatches)."""
    if a.max_label.size != b.max_label.size:
        raise Error(ErrKind.usage, "segmentation_equal: topology mismatch")
    match = (a.max_label == b.max_label) & (a.min_label == b.min_label)
    return match.astype(np.uint8), int(match.size - int(match.sum()))


# ---------------------------------------------------------------- z-slab sharding
def slab_range(z_extent: int, nranks: int, rank: int) -> tuple:
    """(z0, z1, wz0, wz1): owned planes [z0, z1) and window planes [wz0, wz1) of a rank."""
    out = (C.c_uint64 * 4)()
    _check(library().mssz_cu_slab_range(C.c_uint64(z_extent), nranks, rank, out))
    return tuple(int(v) for v in out)


def derive_edits_slabs(topo: GridTopology, original, decompressed, xi: float, nslabs: int,
                       opts: Optional[DeriveOptions] = None, stats: Optional[EditStats] = None,
                       devices=None) -> EditSet:
    """derive_edits on ``nslabs`` z-slabs run as virtual ranks in this process
    (host threads; all on ``opts.device`` unless ``devices`` is given).  The
    result equals derive_edits on the whole field (the sharding acceptance
    test)."""
    f = _field(topo, original, "original")
    fh = _field(topo, decompressed, "decompressed", f.dtype)
    suf = _suf(f.dtype)
    keep: list = []
    co = _options(opts, f.dtype, keep)
    cap = topo.vertex_count
    idx = np.empty(cap, np.uint64)
    val = np.empty(cap, f.dtype)
    count = C.c_uint64()
    st = _Stats()
    devs = None if not devices else (C.c_int * len(devices))(*devices)
    rc = getattr(library(), f"mssz_cu_derive_edits_slabs_local_{suf}")(
        nslabs, devs, len(devices) if devices else 0, topo.ndims, _dims(topo), _p(f), _p(fh),
        C.c_double(xi), C.byref(co), _p(idx), _p(val), C.c_uint64(cap), C.byref(count),
        C.byref(st))
    _check(rc)
    if stats is not None:
        st.fill(stats)
    k = count.value
    return EditSet(idx[:k].copy(), val[:k].copy())


class SlabComm:
    """One rank of a z-slab sharded run (one process per GPU, NCCL underneath).

    ``SlabComm.unique_id()`` on rank 0, broadcast (e.g. torch.distributed), then
    ``SlabComm(uid, nranks, rank, device)`` everywhere.  ``derive_edits`` takes
    this rank's window (planes ``slab_range(...)[2:4]``) and returns the edits in
    its owned planes (global ids) plus their offset in the global EditSet."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        if len(uid) != 128:
            raise Error(ErrKind.usage, "NCCL unique id must be 128 bytes")
        self.nranks, self.rank, self.device = nranks, rank, device
        self._c = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(library().mssz_cu_comm_init(buf, nranks, rank, device, C.byref(self._c)))

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(library().mssz_cu_comm_unique_id(buf))
        return bytes(buf)

    def close(self) -> None:
        if self._c:
            _check(library().mssz_cu_comm_destroy(self._c))
            self._c = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def derive_edits(self, dims, original_window, decompressed_window, xi: float,
                     opts: Optional[DeriveOptions] = None, stats: Optional[EditStats] = None):
        """-> (EditSet of this slab, offset in the global EditSet)."""
        f = np.ascontiguousarray(original_window).reshape(-1)
        fh = np.ascontiguousarray(decompressed_window, dtype=f.dtype).reshape(-1)
        z0, z1, wz0, wz1 = slab_range(int(dims[2]), self.nranks, self.rank)
        want = int(dims[0]) * int(dims[1]) * (wz1 - wz0)
        if f.size != want or fh.size != want:
            raise Error(ErrKind.io, f"window holds {f.size} values, expected {want}")
        keep: list = []
        co = _options(opts, f.dtype, keep)
        cap = int(dims[0]) * int(dims[1]) * (z1 - z0)
        idx = np.empty(cap, np.uint64)
        val = np.empty(cap, f.dtype)
        count, offset, st = C.c_uint64(), C.c_uint64(), _Stats()
        rc = getattr(library(), f"mssz_cu_derive_edits_slab_{_suf(f.dtype)}")(
            self._c, 3, (C.c_uint64 * 3)(*[int(d) for d in dims]), _p(f), _p(fh), C.c_double(xi),
            C.byref(co), _p(idx), _p(val), C.c_uint64(cap), C.byref(count), C.byref(offset),
            C.byref(st))
        _check(rc)
        if stats is not None:
            st.fill(stats)
        k = count.value
        return EditSet(idx[:k].copy(), val[:k].copy()), offset.value

    def derive_edits_into(self, dims, f_ptr: int, fh_ptr: int, xi: float, idx_ptr: int,
                          val_ptr: int, capacity: int, dtype=np.float32,
                          opts: Optional[DeriveOptions] = None) -> tuple:
        """Host-pointer window (e.g. pinned) -> (count, offset, EditStats)."""
        keep: list = []
        co = _options(opts, dtype, keep)
        count, offset, st = C.c_uint64(), C.c_uint64(), _Stats()
        rc = getattr(library(), f"mssz_cu_derive_edits_slab_{_suf(dtype)}")(
            self._c, 3, (C.c_uint64 * 3)(*[int(d) for d in dims]), C.c_void_p(f_ptr),
            C.c_void_p(fh_ptr), C.c_double(xi), C.byref(co), C.c_void_p(idx_ptr),
            C.c_void_p(val_ptr), C.c_uint64(capacity), C.byref(count), C.byref(offset), C.byref(st))
        _check(rc)
        return count.value, offset.value, st.fill(EditStats())

    def derive_edits_device(self, dims, d_f: int, d_fh: int, xi: float, d_idx: int, d_val: int,
                            capacity: int, dtype=np.float32, opts: Optional[DeriveOptions] = None,
                            stream: int = 0) -> tuple:
        """Device-resident window -> (count, offset, EditStats)."""
        keep: list = []
        co = _options(opts, dtype, keep)
        count, offset, st = C.c_uint64(), C.c_uint64(), _Stats()
        rc = getattr(library(), f"mssz_cu_derive_edits_slab_device_{_suf(dtype)}")(
            self._c, 3, (C.c_uint64 * 3)(*[int(d) for d in dims]), C.c_void_p(d_f), C.c_void_p(d_fh),
            C.c_double(xi), C.byref(co), C.c_void_p(d_idx), C.c_void_p(d_val), C.c_uint64(capacity),
            C.byref(count), C.byref(offset), C.byref(st), C.c_void_p(stream or None))
        _check(rc)
        return count.value, offset.value, st.fill(EditStats())


# ---------------------------------------------------------------- verification report
@dataclass
class VerificationReport:
    """VerificationReport (metrics.hpp:14-23) plus the device extras."""

    mss_distortion: float = 0.0
    right_labeled_ratio: float = 1.0
    psnr: float = 0.0
    edit_ratio: float = 0.0
    ocr: float = 0.0
    obr: float = 0.0
    bound_violations: int = 0
    fp_max: int = 0
    fp_min: int = 0
    fn_max: int = 0
    fn_min: int = 0
    mismatches: int = 0
    sum_sq: float = 0.0
    value_lo: float = 0.0
    value_hi: float = 0.0
    device_seconds: float = 0.0
    kernel_launches: int = 0

    def passed(self) -> bool:
        """The reference CLI's verify exit criterion (tools/mssz.cpp:250)."""
        return self.mss_distortion == 0.0 and self.bound_violations == 0


class _Report(C.Structure):
    _fields_ = [
        ("mss_distortion", C.c_double), ("right_labeled_ratio", C.c_double), ("psnr", C.c_double),
        ("edit_ratio", C.c_double), ("ocr", C.c_double), ("obr", C.c_double),
        ("bound_violations", C.c_uint64), ("fp_max", C.c_uint64), ("fp_min", C.c_uint64),
        ("fn_max", C.c_uint64), ("fn_min", C.c_uint64), ("mismatches", C.c_uint64),
        ("sum_sq", C.c_double), ("value_lo", C.c_double), ("value_hi", C.c_double),
        ("device_seconds", C.c_double), ("kernel_launches", C.c_uint64),
    ]

    def to_report(self) -> VerificationReport:
        return VerificationReport(**{name: getattr(self, name) for name, _ in self._fields_})


def build_report(topo: GridTopology, original, candidate, xi: float, edit_count: int = 0,
                 archive_bytes: int = 0, opts: Optional[DeriveOptions] = None) -> VerificationReport:
    """build_report<T> (tools/mssz.cpp:84-104) on the GPU; host arrays in."""
    f = _field(topo, original, "original")
    g = _field(topo, candidate, "candidate", f.dtype)
    keep: list = []
    co = _options(opts, f.dtype, keep)
    r = _Report()
    _check(getattr(library(), f"mssz_cu_verify_{_suf(f.dtype)}")(
        topo.ndims, _dims(topo), _p(f), _p(g), C.c_double(xi), C.c_uint64(edit_count),
        C.c_uint64(archive_bytes), C.byref(co), C.byref(r)))
    return r.to_report()


def build_report_device(topo: GridTopology, d_f: int, d_g: int, xi: float, dtype=np.float32,
                        edit_count: int = 0, archive_bytes: int = 0,
                        opts: Optional[DeriveOptions] = None, stream: int = 0) -> VerificationReport:
    """Device-resident variant (CUDA pointers, optional stream)."""
    keep: list = []
    co = _options(opts, dtype, keep)
    r = _Report()
    _check(getattr(library(), f"mssz_cu_verify_device_{_suf(dtype)}")(
        topo.ndims, _dims(topo), C.c_void_p(d_f), C.c_void_p(d_g), C.c_double(xi),
        C.c_uint64(edit_count), C.c_uint64(archive_bytes), C.byref(co), C.byref(r),
        C.c_void_p(stream or None)))
    return r.to_report()


def segmentation(topo: GridTopology, values) -> SegmentationLabels:
    """compute_labels(compute_directions(values)) in one device pass (the `mss` subcommand)."""
    v = _field(topo, values, "values")
    M = np.empty(topo.vertex_count, np.uint64)
    m = np.empty(topo.vertex_count, np.uint64)
    _check(getattr(library(), f"mssz_cu_segmentation_{_suf(v.dtype)}")(
        topo.ndims, _dims(topo), _p(v), _p(M), _p(m)))
    return SegmentationLabels(M, m)


def export_labels(labels: SegmentationLabels, path: str) -> None:
    """export_labels (mss.cpp:135-145): the M array then the m array, u64 little-endian."""
    with open(path, "wb") as fp:
        fp.write(np.ascontiguousarray(labels.max_label, "<u8").tobytes())
        fp.write(np.ascontiguousarray(labels.min_label, "<u8").tobytes())


# ---------------------------------------------------------------- base codec (GPU)
def compress_base(topo: GridTopology, values, xi: float, timing: Optional[dict] = None):
    """compress_base<T> (base_codec.cpp:76-120) on the GPU -> (reconstruction, symbols,
    literals): symbols are what huffman::encode_stream codes (0 = escape, else
    1 + zigzag(q)), literals the escaped values in index order."""
    v = _field(topo, values, "values")
    recon = np.empty_like(v)
    sym = np.empty(topo.vertex_count, np.uint32)
    esc = C.c_uint64()
    ms = C.c_double()
    _check(getattr(library(), f"mssz_cu_compress_base_{_suf(v.dtype)}")(
        topo.ndims, _dims(topo), _p(v), C.c_double(xi), _p(recon), _p(sym), C.byref(esc),
        C.byref(ms)))
    if timing is not None:
        timing["device_ms"] = ms.value
    lits = v[sym == 0]
    assert lits.size == esc.value
    return recon, sym, lits


def decompress_base(topo: GridTopology, symbols, literals, xi: float, dtype=np.float32,
                    timing: Optional[dict] = None) -> np.ndarray:
    """decompress_base<T> (base_codec.cpp:122-152) after the Huffman decode, on the GPU."""
    sym = np.ascontiguousarray(symbols, np.uint32).reshape(-1)
    if sym.size != topo.vertex_count:
        raise Error(ErrKind.corrupt_archive, "code count does not match the grid")
    lit = np.ascontiguousarray(literals, dtype).reshape(-1)
    out = np.empty(topo.vertex_count, dtype)
    ms = C.c_double()
    _check(getattr(library(), f"mssz_cu_decompress_base_{_suf(dtype)}")(
        topo.ndims, _dims(topo), _p(sym), _p(lit) if lit.size else None, C.c_uint64(lit.size),
        C.c_double(xi), _p(out), C.byref(ms)))
    if timing is not None:
        timing["device_ms"] = ms.value
    return out


# ---------------------------------------------------------------- edit-set encoding
def encode_edits(edits: EditSet, codec: int = 1, timing: Optional[dict] = None) -> bytes:
    """encode_edits<T> (edit_codec.cpp:188-222): the archive's edit payload, byte-identical
    to the reference; codec 0 = store, 1 = raw DEFLATE."""
    idx = np.ascontiguousarray(edits.indices, np.uint64)
    val = np.ascontiguousarray(edits.values)
    out = C.POINTER(C.c_uint8)()
    n = C.c_uint64()
    ms = C.c_double()
    lib = library()
    _check(getattr(lib, f"mssz_cu_encode_edits_{_suf(val.dtype)}")(
        _p(idx) if idx.size else None, _p(val) if val.size else None, C.c_uint64(idx.size), codec,
        C.byref(out), C.byref(n), C.byref(ms)))
    data = C.string_at(out, n.value)
    lib.mssz_cu_free(C.cast(out, C.c_void_p))
    if timing is not None:
        timing["device_ms"] = ms.value
    return data
