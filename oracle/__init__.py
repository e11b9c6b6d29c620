"""TEST INFRASTRUCTURE ONLY — ctypes front-ends of the two CPU checkers.

* ``Ref``    — the UNMODIFIED reference core (``oracle/_ref/libmssz_ref.so``,
  built from /root/reference/proj/core/src by ``oracle/Makefile``).
* ``Oracle`` — our plain-C restatement (``oracle/_ref/libmssz_oracle.so``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the
product library never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REF_SO = os.path.join(REF_DIR, "libmssz_ref.so")
ORACLE_SO = os.path.join(REF_DIR, "libmssz_oracle.so")
REFERENCE_SRC = "/root/reference/proj/core"

GAUSS_SEIDEL = 0
JACOBI = 1

KINDS = {"gaussian-mixture": 0, "trig": 1, "random-smooth": 2}


def build(quiet: bool = True) -> None:
    """Build the checkers: the C restatement always, the reference only when its sources exist."""
    targets = ["oracle"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    out = subprocess.run(["make", "-C", HERE, *targets], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{out.stdout}\n{out.stderr}")


class StatsC(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_uint64),
        ("c_passes", C.c_uint64),
        ("sub_iterations", C.c_uint64 * 4),
        ("r_iterations", C.c_uint64),
        ("effective_edits", C.c_uint64),
        ("touched", C.c_uint64),
        ("input_bound_violations", C.c_uint64),
        ("direction_seconds", C.c_double),
        ("label_seconds", C.c_double),
    ]

    def to_dict(self) -> dict:
        return {
            "outer_iterations": self.outer_iterations,
            "c_passes": self.c_passes,
            "sub_iterations": list(self.sub_iterations),
            "r_iterations": self.r_iterations,
            "effective_edits": self.effective_edits,
            "touched": self.touched,
            "input_bound_violations": self.input_bound_violations,
            "direction_seconds": self.direction_seconds,
            "label_seconds": self.label_seconds,
        }


class RefOptionsC(C.Structure):
    _fields_ = [
        ("outer_cap", C.c_uint64),
        ("subloop_cap", C.c_uint64),
        ("r_cap", C.c_uint64),
        ("force", C.c_int),
        ("threads", C.c_int),
    ]


class OracleOptionsC(C.Structure):
    _fields_ = [
        ("outer_cap", C.c_uint64),
        ("subloop_cap", C.c_uint64),
        ("r_cap", C.c_uint64),
        ("force", C.c_int),
        ("schedule", C.c_int),
    ]


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


@dataclass
class EditResult:
    indices: np.ndarray
    values: np.ndarray
    stats: dict = field(default_factory=dict)
    batches: list = field(default_factory=list)


def _dims_arr(dims):
    return (C.c_uint64 * len(dims))(*dims)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _suffix(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"unsupported dtype {dt}")


CB_F32 = C.CFUNCTYPE(None, C.POINTER(C.c_float), C.c_uint64, C.c_void_p)
CB_F64 = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_uint64, C.c_void_p)


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(f"{self.path} missing (run `make -C oracle`)")
        self.lib = C.CDLL(self.path)
        self.lib.__getattr__(self.prefix + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc: int):
        if rc != 0:
            msg = self._fn("last_error")().decode()
            raise CheckerError(rc, msg)

    def compute_directions(self, dims, values: np.ndarray, threads: int = 1):
        values = np.ascontiguousarray(values)
        n = int(np.prod(dims))
        asc = np.empty(n, np.uint64)
        desc = np.empty(n, np.uint64)
        args = [len(dims), _dims_arr(dims), _ptr(values), _ptr(asc), _ptr(desc)]
        if self.prefix == "mssz_ref_":
            args.append(threads)
        self._check(self._fn("compute_directions_" + _suffix(values.dtype))(*args))
        return asc, desc

    def compute_labels(self, dims, asc: np.ndarray, desc: np.ndarray, threads: int = 1):
        n = int(np.prod(dims))
        M = np.empty(n, np.uint64)
        m = np.empty(n, np.uint64)
        asc = np.ascontiguousarray(asc, np.uint64)
        desc = np.ascontiguousarray(desc, np.uint64)
        args = [len(dims), _dims_arr(dims), _ptr(asc), _ptr(desc), _ptr(M), _ptr(m)]
        if self.prefix == "mssz_ref_":
            args.append(threads)
        self._check(self._fn("compute_labels")(*args))
        return M, m

    def detect_false_critical(self, dims, f: np.ndarray, g: np.ndarray, xi: float = 1.0,
                              threads: int = 1):
        n = int(np.prod(dims))
        counts = np.zeros(4, np.uint64)
        lists = np.zeros(4 * n, np.uint64)
        suf = _suffix(f.dtype)
        args = [len(dims), _dims_arr(dims), _ptr(f), _ptr(g)]
        name = "detect_false_critical_"
        if self.prefix == "mssz_ref_":
            args.append(C.c_double(xi))
        args += [_ptr(counts), _ptr(lists)]
        if self.prefix == "mssz_ref_" and threads != 1:
            name = "detect_false_critical_mt_"
            args.append(threads)
        self._check(self._fn(name + suf)(*args))
        return [lists[k * n : k * n + int(counts[k])].copy() for k in range(4)]

    def _derive(self, fn, dims, f, fhat, xi, opts, record_batches):
        f = np.ascontiguousarray(f)
        fhat = np.ascontiguousarray(fhat, dtype=f.dtype)
        suf = _suffix(f.dtype)
        T = C.c_float if suf == "f32" else C.c_double
        idx = C.POINTER(C.c_uint64)()
        val = C.POINTER(T)()
        count = C.c_uint64()
        st = StatsC()
        batches = []
        cb = None
        if record_batches:
            CB = CB_F32 if suf == "f32" else CB_F64
            n = int(np.prod(dims))

            def _on_batch(ptr, size, user):
                batches.append(np.ctypeslib.as_array(ptr, shape=(size,)).copy())

            cb = CB(_on_batch)
        rc = fn(len(dims), _dims_arr(dims), _ptr(f), _ptr(fhat), C.c_double(xi), C.byref(opts),
                cb, None, C.byref(idx), C.byref(val), C.byref(count), C.byref(st))
        self._check(rc)
        k = count.value
        indices = np.ctypeslib.as_array(idx, shape=(max(k, 1),))[:k].copy()
        values = np.ctypeslib.as_array(val, shape=(max(k, 1),))[:k].copy()
        self._fn("free")(idx)
        self._fn("free")(val)
        return EditResult(indices, values, st.to_dict(), batches)


class Ref(_Lib):
    """The unmodified reference (edit_engine.cpp, mss.cpp, field.cpp, base_codec.cpp)."""

    prefix = "mssz_ref_"
    path = REF_SO

    def __init__(self):
        super().__init__()
        self.lib.mssz_ref_free.argtypes = [C.c_void_p]

    def derive_edits(self, dims, f, fhat, xi, outer_cap=1000, subloop_cap=640, r_cap=100000,
                     force=False, threads=1, record_batches=False) -> EditResult:
        opts = RefOptionsC(outer_cap, subloop_cap, r_cap, int(force), threads)
        fn = self._fn("derive_edits_" + _suffix(np.asarray(f).dtype))
        return self._derive(fn, dims, f, fhat, xi, opts, record_batches)

    def oracle_labels(self, dims, values):
        n = int(np.prod(dims))
        M = np.empty(n, np.uint64)
        m = np.empty(n, np.uint64)
        self._check(self._fn("oracle_labels_" + _suffix(values.dtype))(
            len(dims), _dims_arr(dims), _ptr(values), _ptr(M), _ptr(m)))
        return M, m

    def generate(self, kind: str, dims, seed: int, dtype=np.float32) -> np.ndarray:
        out = np.empty(int(np.prod(dims)), dtype)
        self._check(self._fn("generate_" + _suffix(dtype))(
            KINDS[kind], len(dims), _dims_arr(dims), C.c_uint64(seed), _ptr(out)))
        return out

    def compress_base(self, dims, values: np.ndarray, xi: float) -> np.ndarray:
        recon = np.empty_like(values)
        nbytes = C.c_uint64()
        self._check(self._fn("compress_base_" + _suffix(values.dtype))(
            len(dims), _dims_arr(dims), _ptr(values), C.c_double(xi), _ptr(recon),
            C.byref(nbytes)))
        return recon

    def resolve_rel(self, dims, values: np.ndarray, magnitude: float) -> float:
        xi = C.c_double()
        self._check(self._fn("resolve_rel_" + _suffix(values.dtype))(
            len(dims), _dims_arr(dims), _ptr(values), C.c_double(magnitude), C.byref(xi)))
        return xi.value

    def lower_step_trace(self, dims, f, g, xi, v, max_steps=200):
        T = f.dtype
        trace = np.zeros(max_steps + 1, T)
        steps = C.c_int()
        floor = np.zeros(1, T)
        self._check(self._fn("lower_step_" + _suffix(T))(
            len(dims), _dims_arr(dims), _ptr(f), _ptr(g), C.c_double(xi), C.c_uint64(v),
            max_steps, _ptr(trace), C.byref(steps), _ptr(floor)))
        return trace[: steps.value + 1], floor[0]

    def r_targets(self, dims, f, g, threads=0):
        """run_r_loop's target collection (edit_engine.cpp:336-352) on (f, g):
        (sorted distinct targets, false critical points, distinct (v_i, family)
        sources, mismatched vertices)."""
        f = np.ascontiguousarray(f)
        g = np.ascontiguousarray(g, f.dtype)
        n = int(np.prod(dims))
        out = np.empty(2 * n, np.uint64)
        cnt = C.c_uint64()
        info = np.zeros(3, np.uint64)
        self._check(self._fn("r_targets_" + _suffix(f.dtype))(
            len(dims), _dims_arr(dims), _ptr(f), _ptr(g), threads, _ptr(out), C.byref(cnt),
            _ptr(info)))
        return out[: cnt.value].copy(), int(info[0]), int(info[1]), int(info[2])

    def encode_edits(self, indices: np.ndarray, values: np.ndarray, codec: int = 1) -> bytes:
        """encode_edits<T> (edit_codec.cpp:188-222): the reference edit payload."""
        idx = np.ascontiguousarray(indices, np.uint64)
        val = np.ascontiguousarray(values)
        out = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        self._check(self._fn(f"encode_edits_{_suffix(val.dtype)}")(
            _ptr(idx), _ptr(val), C.c_uint64(idx.size), codec, C.byref(out), C.byref(n)))
        data = bytes(C.cast(out, C.POINTER(C.c_uint8 * max(n.value, 1))).contents)[:n.value]
        self.lib.mssz_ref_free(C.cast(out, C.c_void_p))
        return data

    def find_troublemaker(self, dims, f, g, xi, v, descending=False):
        vi = C.c_uint64()
        vt = C.c_uint64()
        self._check(self._fn("find_troublemaker_" + _suffix(f.dtype))(
            len(dims), _dims_arr(dims), _ptr(f), _ptr(g), C.c_double(xi), C.c_uint64(v),
            int(descending), C.byref(vi), C.byref(vt)))
        return vi.value, vt.value


class Oracle(_Lib):
    """Our plain-C restatement (mssz_oracle.c)."""

    prefix = "mssz_oracle_"
    path = ORACLE_SO

    def __init__(self):
        super().__init__()
        self.lib.mssz_oracle_free.argtypes = [C.c_void_p]
        self.lib.mssz_oracle_representable_floor_f32.restype = C.c_float
        self.lib.mssz_oracle_representable_floor_f32.argtypes = [C.c_float, C.c_double]
        self.lib.mssz_oracle_representable_floor_f64.restype = C.c_double
        self.lib.mssz_oracle_representable_floor_f64.argtypes = [C.c_double, C.c_double]

    def derive_edits(self, dims, f, fhat, xi, outer_cap=1000, subloop_cap=640, r_cap=100000,
                     force=False, schedule=JACOBI, record_batches=False) -> EditResult:
        opts = OracleOptionsC(outer_cap, subloop_cap, r_cap, int(force), schedule)
        fn = self._fn("derive_edits_" + _suffix(np.asarray(f).dtype))
        return self._derive(fn, dims, f, fhat, xi, opts, record_batches)

    def detect_kind(self, dims, f, g, kind: int) -> np.ndarray:
        n = int(np.prod(dims))
        out = np.zeros(n, np.uint64)
        cnt = C.c_uint64()
        self._check(self._fn("detect_kind_" + _suffix(f.dtype))(
            len(dims), _dims_arr(dims), _ptr(f), _ptr(g), kind, _ptr(out), C.byref(cnt)))
        return out[: cnt.value].copy()

    def representable_floor(self, f: float, xi: float, dtype=np.float64):
        return self._fn("representable_floor_" + _suffix(dtype))(f, xi)

    def lower_step(self, g: float, f: float, xi: float, dtype=np.float64):
        T = C.c_float if _suffix(dtype) == "f32" else C.c_double
        gv = T(g)
        moved = self._fn("lower_step_" + _suffix(dtype))(C.byref(gv), T(f), C.c_double(xi))
        return bool(moved), gv.value

    def neighbors(self, dims, v: int):
        out = (C.c_uint64 * 14)()
        n = C.c_int()
        self._check(self._fn("neighbors")(len(dims), _dims_arr(dims), C.c_uint64(v), out,
                                          C.byref(n)))
        return [out[i] for i in range(n.value)]

    def build_topology(self, dims) -> int:
        n = C.c_uint64()
        self._check(self._fn("build_topology")(len(dims), _dims_arr(dims), C.byref(n)))
        return n.value


_ref = None
_oracle = None


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle()
    return _oracle


def have_ref() -> bool:
    return os.path.exists(REF_SO)
