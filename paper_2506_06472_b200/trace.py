"""Trace model: one training iteration as kernels + tensor access lists.

Mirrors the reference data model and file format (`offloader/trace.py`):
`TensorKind` (trace.py:47-49), `KernelRecord` (:52-60), `TensorRecord`
(:63-84), `Trace` (:87-110), `validate_trace` (:125-157), the JSONL parser
(:160-275), `write_trace` (:278-301), `load_trace`/`save_trace` (:304-311),
`make_trace` (:314-321).

What is different is the representation.  A `Trace` here is backed by a
structure-of-arrays (`TraceArrays`, numpy) that is what the device path
consumes: kernel durations (int64[N]), tensor ids/sizes/kinds (int64/int64/
int8 [T]) and the tensor-major access CSR (`access_ptr` int64[T+1],
`accesses` int64[E]).  The record lists (`trace.kernels`, `trace.tensors`)
are materialised lazily for traces built from arrays, so a 10M-event trace
never becomes ten million Python objects unless somebody asks for them.
All integers must fit in int64 (the reference uses unbounded Python ints);
values outside that range are rejected when the arrays are built.
"""

from __future__ import annotations

import io
import json
import operator
from dataclasses import dataclass, field
from enum import Enum
from typing import IO, Iterable

import numpy as np

TRACE_FORMAT_VERSION = 1
NONE_I64 = np.iinfo(np.int64).min  # sentinel for "None" in optional int columns
KIND_INTERMEDIATE = 0
KIND_GLOBAL = 1
KIND_UNKNOWN = -1


class TraceParseError(ValueError):
    """Malformed trace stream; carries the 1-based line number."""

    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line


class TraceValidationError(ValueError):
    """A well-formed trace that breaks a model invariant."""

    def __init__(self, violations: list[str]):
        super().__init__("; ".join(violations))
        self.violations = violations


class TensorKind(str, Enum):
    INTERMEDIATE = "intermediate"
    GLOBAL = "global"


@dataclass(frozen=True)
class KernelRecord:
    index: int
    name: str
    duration_us: int
    stage: int | None = None
    layer: int | None = None


@dataclass(frozen=True)
class TensorRecord:
    id: int
    size_bytes: int
    kind: TensorKind
    accesses: tuple[int, ...]
    layer: int | None = None

    @property
    def first_access(self) -> int:
        return self.accesses[0]

    @property
    def last_access(self) -> int:
        return self.accesses[-1]


# --------------------------------------------------------------------------
# structure-of-arrays form

def _i64(values, what: str) -> np.ndarray:
    try:
        return np.asarray(values, dtype=np.int64)
    except OverflowError:
        raise ValueError(f"{what}: value outside int64") from None


def _opt_i64(values, what: str) -> np.ndarray:
    return _i64([NONE_I64 if v is None else v for v in values], what)


@dataclass
class TraceArrays:
    """Column form of a trace (host numpy arrays).

    `accesses[access_ptr[i]:access_ptr[i+1]]` are tensor i's kernel indices.
    Optional int columns (stage/layer) use NONE_I64 for None.  Kernel names
    are interned: `kernel_name_code[k]` indexes `name_table`.
    """

    duration_us: np.ndarray        # int64[N]
    kernel_index: np.ndarray       # int64[N]
    kernel_name_code: np.ndarray   # int32[N]
    name_table: list[str]
    kernel_stage: np.ndarray       # int64[N]
    kernel_layer: np.ndarray       # int64[N]
    tensor_id: np.ndarray          # int64[T]
    size_bytes: np.ndarray         # int64[T]
    kind: np.ndarray               # int8[T]  (0 intermediate, 1 global, -1 unknown)
    tensor_layer: np.ndarray       # int64[T]
    access_ptr: np.ndarray         # int64[T+1]
    accesses: np.ndarray           # int64[E]
    bad_kinds: dict = field(default_factory=dict)  # position -> original kind object

    @property
    def num_kernels(self) -> int:
        return int(self.duration_us.shape[0])

    @property
    def num_tensors(self) -> int:
        return int(self.tensor_id.shape[0])

    @property
    def num_events(self) -> int:
        return int(self.accesses.shape[0])

    @staticmethod
    def empty() -> "TraceArrays":
        z = np.zeros(0, dtype=np.int64)
        return TraceArrays(z, z.copy(), np.zeros(0, np.int32), [], z.copy(), z.copy(),
                           z.copy(), z.copy(), np.zeros(0, np.int8), z.copy(),
                           np.zeros(1, np.int64), z.copy())

    def equals(self, other: "TraceArrays") -> bool:
        a, b = self, other
        if a.num_kernels != b.num_kernels or a.num_tensors != b.num_tensors:
            return False
        names_a = [a.name_table[c] for c in a.kernel_name_code.tolist()]
        names_b = [b.name_table[c] for c in b.kernel_name_code.tolist()]
        return (names_a == names_b and a.bad_kinds == b.bad_kinds
                and all(np.array_equal(getattr(a, f), getattr(b, f)) for f in (
                    "duration_us", "kernel_index", "kernel_stage", "kernel_layer",
                    "tensor_id", "size_bytes", "kind", "tensor_layer",
                    "access_ptr", "accesses")))


def _kind_code(kind) -> int:
    # our TensorKind, or an equal-valued enum member of the reference package
    # (records coming straight from `offloader` objects)
    if isinstance(kind, Enum):
        if kind.value == "global":
            return KIND_GLOBAL
        if kind.value == "intermediate":
            return KIND_INTERMEDIATE
    return KIND_UNKNOWN


def arrays_from_records(kernels: list[KernelRecord], tensors: list[TensorRecord]) -> TraceArrays:
    name_index: dict[str, int] = {}
    codes = []
    for k in kernels:
        codes.append(name_index.setdefault(k.name, len(name_index)))
    kinds = np.array([_kind_code(t.kind) for t in tensors], dtype=np.int8)
    bad = {i: t.kind for i, t in enumerate(tensors) if kinds[i] == KIND_UNKNOWN}
    lengths = np.array([len(t.accesses) for t in tensors], dtype=np.int64)
    ptr = np.zeros(len(tensors) + 1, dtype=np.int64)
    np.cumsum(lengths, out=ptr[1:])
    flat = [a for t in tensors for a in t.accesses]
    return TraceArrays(
        duration_us=_i64([k.duration_us for k in kernels], "kernel duration_us"),
        kernel_index=_i64([k.index for k in kernels], "kernel index"),
        kernel_name_code=np.array(codes, dtype=np.int32),
        name_table=list(name_index),
        kernel_stage=_opt_i64([k.stage for k in kernels], "kernel stage"),
        kernel_layer=_opt_i64([k.layer for k in kernels], "kernel layer"),
        tensor_id=_i64([t.id for t in tensors], "tensor id"),
        size_bytes=_i64([t.size_bytes for t in tensors], "tensor size_bytes"),
        kind=kinds,
        tensor_layer=_opt_i64([t.layer for t in tensors], "tensor layer"),
        access_ptr=ptr,
        accesses=_i64(flat, "tensor access"),
        bad_kinds=bad,
    )


def _opt(v: int):
    return None if v == NONE_I64 else int(v)


def records_from_arrays(a: TraceArrays) -> tuple[list[KernelRecord], list[TensorRecord]]:
    names = a.name_table
    kernels = [KernelRecord(int(i), names[c], int(d), _opt(s), _opt(l))
               for i, c, d, s, l in zip(a.kernel_index.tolist(), a.kernel_name_code.tolist(),
                                        a.duration_us.tolist(), a.kernel_stage.tolist(),
                                        a.kernel_layer.tolist())]
    acc = a.accesses.tolist()
    ptr = a.access_ptr.tolist()
    kinds = a.kind.tolist()
    tensors = []
    for i, (tid, size, layer) in enumerate(zip(a.tensor_id.tolist(), a.size_bytes.tolist(),
                                               a.tensor_layer.tolist())):
        kc = kinds[i]
        kind = (TensorKind.GLOBAL if kc == KIND_GLOBAL else
                TensorKind.INTERMEDIATE if kc == KIND_INTERMEDIATE else a.bad_kinds[i])
        tensors.append(TensorRecord(tid, size, kind, tuple(acc[ptr[i]:ptr[i + 1]]), _opt(layer)))
    return kernels, tensors


class Trace:
    """One training iteration (reference `Trace`, trace.py:87-110).

    Construct from record lists like the reference (`Trace(kernels, tensors,
    meta)`), or from columns with `Trace.from_arrays`.  `arrays()` returns the
    column form the device path consumes; for record-built traces it is
    rebuilt whenever the record lists change: the records are frozen, so the
    lists are compared element by element (by identity) with the snapshot
    the columns were built from; the snapshot holds the records, so their
    ids cannot be reused while it exists.  Every device-side cache entry
    (`device_cache`) is dropped with the columns.
    """

    def __init__(self, kernels: list[KernelRecord] | None = None,
                 tensors: list[TensorRecord] | None = None,
                 meta: dict | None = None):
        self._kernels = kernels if kernels is not None else []
        self._tensors = tensors if tensors is not None else []
        self.meta = meta if meta is not None else {}
        self._arrays: TraceArrays | None = None
        self._snap: tuple | None = None
        self._from_arrays = False
        self.device_cache: dict = {}

    @classmethod
    def from_arrays(cls, arrays: TraceArrays, meta: dict | None = None) -> "Trace":
        t = cls(None, None, meta)
        t._kernels = None
        t._tensors = None
        t._arrays = arrays
        t._from_arrays = True
        return t

    # -- record views (reference API) -------------------------------------
    def _materialise(self) -> None:
        if self._kernels is None:
            self._kernels, self._tensors = records_from_arrays(self._arrays)
            # from now on the lists are the source of truth
            self._from_arrays = False
            self._snap = self._snapshot()

    @property
    def kernels(self) -> list[KernelRecord]:
        self._materialise()
        return self._kernels

    @kernels.setter
    def kernels(self, value):
        self._materialise()
        self._kernels = value

    @property
    def tensors(self) -> list[TensorRecord]:
        self._materialise()
        return self._tensors

    @tensors.setter
    def tensors(self, value):
        self._materialise()
        self._tensors = value

    def _snapshot(self) -> tuple:
        return tuple(self._kernels), tuple(self._tensors)

    def _stale(self) -> bool:
        if self._arrays is None or self._snap is None:
            return True
        for cur, old in ((self._kernels, self._snap[0]), (self._tensors, self._snap[1])):
            if len(cur) != len(old) or not all(map(operator.is_, cur, old)):
                return True
        return False

    def arrays(self) -> TraceArrays:
        if self._from_arrays:
            return self._arrays
        if self._stale():
            self._arrays = arrays_from_records(self._kernels, self._tensors)
            self._snap = self._snapshot()
            self.device_cache.clear()
        return self._arrays

    # -- derived quantities (trace.py:94-110) --------------------------------
    @property
    def num_kernels(self) -> int:
        if self._from_arrays:
            return self._arrays.num_kernels
        return len(self._kernels)

    @property
    def num_tensors(self) -> int:
        if self._from_arrays:
            return self._arrays.num_tensors
        return len(self._tensors)

    def kernel_start_times(self) -> list[int]:
        d = self.arrays().duration_us
        starts = np.zeros(d.shape[0], dtype=np.int64)
        if d.shape[0] > 1:
            np.cumsum(d[:-1], out=starts[1:])
        return starts.tolist()

    def iteration_length(self) -> int:
        return int(self.arrays().duration_us.sum())

    def tensor_by_id(self) -> dict[int, TensorRecord]:
        return {t.id: t for t in self.tensors}

    def __eq__(self, other) -> bool:
        if not isinstance(other, Trace):
            return NotImplemented
        return self.meta == other.meta and self.arrays().equals(other.arrays())

    def __repr__(self) -> str:
        return (f"Trace(num_kernels={self.num_kernels}, num_tensors={self.num_tensors}, "
                f"meta={self.meta!r})")


@dataclass
class ValidationReport:
    violations: list[str] = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.violations

    def add(self, message: str) -> None:
        self.violations.append(message)


def validate_arrays(a: TraceArrays) -> ValidationReport:
    """Vectorised restatement of `validate_trace` (trace.py:125-157).

    Finds offending rows with numpy and formats messages only for them, in the
    reference's order (kernels by position, then tensors by position, each
    tensor's checks in the reference's order).
    """
    report = ValidationReport()
    n = a.num_kernels
    pos = np.arange(n, dtype=np.int64)
    bad_index = a.kernel_index != pos
    bad_dur = a.duration_us <= 0
    for p in np.flatnonzero(bad_index | bad_dur).tolist():
        idx = int(a.kernel_index[p])
        if bad_index[p]:
            report.add(f"kernel at position {p}: index {idx} not contiguous")
        if bad_dur[p]:
            report.add(f"kernel {idx}: duration {int(a.duration_us[p])} must be > 0")

    t = a.num_tensors
    if t == 0:
        return report
    ids = a.tensor_id
    # duplicate = id already seen at an earlier position
    order = np.argsort(ids, kind="stable")
    sorted_ids = ids[order]
    dup_sorted = np.zeros(t, dtype=bool)
    dup_sorted[1:] = sorted_ids[1:] == sorted_ids[:-1]
    dup = np.zeros(t, dtype=bool)
    dup[order] = dup_sorted
    bad_size = a.size_bytes <= 0
    bad_kind = a.kind == KIND_UNKNOWN
    lengths = np.diff(a.access_ptr)
    empty = lengths == 0
    acc = a.accesses
    e = acc.shape[0]
    owner = np.repeat(np.arange(t, dtype=np.int64), lengths)
    if e > 1:
        same = owner[1:] == owner[:-1]
        nonmono_ev = same & (acc[1:] <= acc[:-1])
        nonmono = np.zeros(t, dtype=bool)
        nonmono[owner[1:][nonmono_ev]] = True
    else:
        nonmono = np.zeros(t, dtype=bool)
    oor_ev = (acc < 0) | (acc >= n)
    oor = np.zeros(t, dtype=bool)
    oor[owner[oor_ev]] = True
    bad = dup | bad_size | bad_kind | empty | nonmono | oor
    ptr = a.access_ptr
    for i in np.flatnonzero(bad).tolist():
        label = f"tensor {int(ids[i])}"
        if dup[i]:
            report.add(f"{label}: duplicate tensor id")
        if bad_size[i]:
            report.add(f"{label}: size {int(a.size_bytes[i])} must be > 0")
        if bad_kind[i]:
            report.add(f"{label}: unknown kind {a.bad_kinds[i]!r}")
        mine = acc[ptr[i]:ptr[i + 1]].tolist()
        if empty[i]:
            report.add(f"{label}: accesses must be non-empty")
            continue
        if nonmono[i]:
            report.add(f"{label}: accesses {mine} not strictly increasing")
        if oor[i]:
            first_bad = next(x for x in mine if not (0 <= x < n))
            report.add(f"{label}: access index {first_bad} out of range ({n} kernels)")
    return report


def validate_trace(trace: Trace) -> ValidationReport:
    return validate_arrays(trace.arrays())


# --------------------------------------------------------------------------
# file format (reference trace.py:160-311); the JSONL grammar is identical.

_KERNEL_KEYS = {"index", "name", "duration_us", "stage", "layer"}
_KERNEL_REQUIRED = {"index", "name", "duration_us"}
_TENSOR_KEYS = {"id", "size_bytes", "kind", "accesses", "layer"}
_TENSOR_REQUIRED = {"id", "size_bytes", "kind", "accesses"}


def _int_field(value, what: str, line: int, allow_none: bool = False):
    if value is None and allow_none:
        return None
    if isinstance(value, bool) or not isinstance(value, int):
        raise TraceParseError(f"{what} must be an integer, got {value!r}", line)
    return value


def _check_keys(obj: dict, allowed: set, required: set, what: str, line: int) -> None:
    extra = set(obj) - allowed
    if extra:
        raise TraceParseError(f"unknown {what} keys {sorted(extra)}", line)
    absent = required - set(obj)
    if absent:
        raise TraceParseError(f"{what} record missing keys {sorted(absent)}", line)


def _kernel_from(obj: dict, line: int) -> KernelRecord:
    _check_keys(obj, _KERNEL_KEYS, _KERNEL_REQUIRED, "kernel", line)
    if not isinstance(obj["name"], str):
        raise TraceParseError("kernel name must be a string", line)
    return KernelRecord(
        index=_int_field(obj["index"], "kernel index", line),
        name=obj["name"],
        duration_us=_int_field(obj["duration_us"], "kernel duration_us", line),
        stage=_int_field(obj.get("stage"), "kernel stage", line, allow_none=True),
        layer=_int_field(obj.get("layer"), "kernel layer", line, allow_none=True),
    )


def _tensor_from(obj: dict, line: int) -> TensorRecord:
    _check_keys(obj, _TENSOR_KEYS, _TENSOR_REQUIRED, "tensor", line)
    try:
        kind = TensorKind(obj["kind"])
    except ValueError:
        raise TraceParseError(f"unknown tensor kind {obj['kind']!r}", line) from None
    acc = obj["accesses"]
    if not isinstance(acc, list):
        raise TraceParseError("tensor accesses must be a list", line)
    return TensorRecord(
        id=_int_field(obj["id"], "tensor id", line),
        size_bytes=_int_field(obj["size_bytes"], "tensor size_bytes", line),
        kind=kind,
        accesses=tuple(_int_field(x, "tensor access", line) for x in acc),
        layer=_int_field(obj.get("layer"), "tensor layer", line, allow_none=True),
    )


def _as_text(data) -> str:
    if isinstance(data, bytes):
        return data.decode("utf-8")
    if isinstance(data, str):
        return data
    raw = data.read()
    return raw.decode("utf-8") if isinstance(raw, bytes) else raw


def _as_bytes(data) -> bytes:
    if isinstance(data, bytes):
        return data
    if isinstance(data, str):
        return data.encode("utf-8")
    raw = data.read()
    return raw if isinstance(raw, bytes) else raw.encode("utf-8")


def _fast_parse(raw: bytes):
    """Multi-threaded C++ parse (libtio csrc/jsonl.cu) into columns; None
    when the file is not in the writer's fast format (the exact parser then
    decides, with the reference's error messages)."""
    import ctypes
    from . import _native
    try:
        lib = _native.load()
    except Exception:
        return None
    h = ctypes.c_void_p()
    line = ctypes.c_int64()
    if lib.tio_trace_parse(raw, ctypes.c_size_t(len(raw)), ctypes.c_int(0), ctypes.byref(h),
                           ctypes.byref(line)) != 0:
        return None
    try:
        n = [ctypes.c_int64() for _ in range(6)]
        _native.check(lib.tio_parsed_sizes(h, *[ctypes.byref(x) for x in n]))
        N, T, E, NN, NB, MB = (x.value for x in n)
        k_index, k_dur, k_stage, k_layer = (np.empty(N, np.int64) for _ in range(4))
        k_code = np.empty(N, np.int32)
        t_id, t_size, t_layer = (np.empty(T, np.int64) for _ in range(3))
        t_kind = np.empty(T, np.int8)
        ptr = np.empty(T + 1, np.int64)
        acc = np.empty(E, np.int64)
        names = ctypes.create_string_buffer(max(1, NB))
        name_off = np.empty(NN + 1, np.int64)
        name_esc = np.empty(max(1, NN), np.uint8)
        meta = ctypes.create_string_buffer(max(1, MB))
        p = _native._ptr
        _native.check(lib.tio_parsed_copy(h, p(k_index), p(k_dur), p(k_code), p(k_stage), p(k_layer), p(t_id),
                                          p(t_size), p(t_kind), p(t_layer), p(ptr), p(acc), names,
                                          p(name_off), p(name_esc), meta))
    finally:
        lib.tio_parsed_destroy(h)
    table = []
    for i in range(NN):
        s = names.raw[name_off[i]:name_off[i + 1]]
        table.append(json.loads(b'"' + s + b'"') if name_esc[i] else s.decode("utf-8"))
    arrays = TraceArrays(duration_us=k_dur, kernel_index=k_index, kernel_name_code=k_code, name_table=table,
                         kernel_stage=k_stage, kernel_layer=k_layer, tensor_id=t_id, size_bytes=t_size,
                         kind=t_kind, tensor_layer=t_layer, access_ptr=ptr, accesses=acc)
    try:
        meta_obj = json.loads(meta.raw[:MB].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError):
        return None          # not valid JSON after all: the exact parser raises the reference's error
    return arrays, meta_obj


def parse_trace(data: bytes | str | IO) -> Trace:
    """Parse + validate a JSONL trace (reference trace.py:217-275).

    Valid files in the writer's format take the C++ multi-threaded parser
    (columns directly, no per-record objects); anything else goes through the
    exact parser below so errors carry the reference's messages and lines."""
    raw = _as_bytes(data)
    fast = _fast_parse(raw)
    if fast is not None:
        arrays, meta = fast
        report = validate_arrays(arrays)
        if not report.ok:
            raise TraceValidationError(report.violations)
        return Trace.from_arrays(arrays, meta)
    return _parse_exact(raw)


def _parse_exact(data) -> Trace:
    lines = _as_text(data).splitlines()
    if not lines or not lines[0].strip():
        raise TraceParseError("missing header line", 1)
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as exc:
        raise TraceParseError(f"invalid JSON: {exc.msg}", 1) from None
    if not isinstance(header, dict) or set(header) - {"version", "meta"}:
        raise TraceParseError("header must be {\"version\": ..., \"meta\": {...}}", 1)
    if header.get("version") != TRACE_FORMAT_VERSION:
        raise TraceParseError(f"unsupported version {header.get('version')!r}", 1)
    meta = header.get("meta", {})
    if not isinstance(meta, dict):
        raise TraceParseError("meta must be an object", 1)

    kernels: list[KernelRecord] = []
    tensors: list[TensorRecord] = []
    for lineno, text in enumerate(lines[1:], start=2):
        if not text.strip():
            continue
        try:
            obj = json.loads(text)
        except json.JSONDecodeError as exc:
            raise TraceParseError(f"invalid JSON: {exc.msg}", lineno) from None
        if not isinstance(obj, dict) or len(obj) != 1:
            raise TraceParseError("record must be a single-key object", lineno)
        (key, body), = obj.items()
        if not isinstance(body, dict):
            raise TraceParseError(f"{key} record body must be an object", lineno)
        if key == "kernel":
            if tensors:
                raise TraceParseError("kernel record after tensor records", lineno)
            kernels.append(_kernel_from(body, lineno))
        elif key == "tensor":
            tensors.append(_tensor_from(body, lineno))
        else:
            raise TraceParseError(f"unknown record type {key!r}", lineno)

    trace = Trace(kernels=kernels, tensors=tensors, meta=meta)
    report = validate_trace(trace)
    if not report.ok:
        raise TraceValidationError(report.violations)
    return trace


def _json_opt(v: int) -> str:
    return "null" if v == NONE_I64 else str(int(v))


def write_trace(trace: Trace) -> bytes:
    """Serialise byte-identically to the reference `write_trace`
    (trace.py:278-301: json.dumps default separators, one record per line).
    Integer columns are formatted directly from the arrays."""
    a = trace.arrays()
    out = io.StringIO()
    out.write(json.dumps({"version": TRACE_FORMAT_VERSION, "meta": trace.meta}))
    out.write("\n")
    names = [json.dumps(s) for s in a.name_table]
    for i, c, d, s, l in zip(a.kernel_index.tolist(), a.kernel_name_code.tolist(),
                             a.duration_us.tolist(), a.kernel_stage.tolist(),
                             a.kernel_layer.tolist()):
        out.write(f'{{"kernel": {{"index": {i}, "name": {names[c]}, "duration_us": {d}, '
                  f'"stage": {_json_opt(s)}, "layer": {_json_opt(l)}}}}}\n')
    acc = a.accesses.tolist()
    ptr = a.access_ptr.tolist()
    kinds = a.kind.tolist()
    for i, (tid, size, layer) in enumerate(zip(a.tensor_id.tolist(), a.size_bytes.tolist(),
                                               a.tensor_layer.tolist())):
        kc = kinds[i]
        kind = "global" if kc == KIND_GLOBAL else "intermediate" if kc == KIND_INTERMEDIATE \
            else a.bad_kinds[i].value
        body = ", ".join(map(str, acc[ptr[i]:ptr[i + 1]]))
        out.write(f'{{"tensor": {{"id": {tid}, "size_bytes": {size}, "kind": "{kind}", '
                  f'"accesses": [{body}], "layer": {_json_opt(layer)}}}}}\n')
    return out.getvalue().encode("utf-8")


def load_trace(path) -> Trace:
    with open(path, "rb") as fh:
        return parse_trace(fh)


def save_trace(trace: Trace, path) -> None:
    with open(path, "wb") as fh:
        fh.write(write_trace(trace))


def make_trace(kernels: Iterable[KernelRecord], tensors: Iterable[TensorRecord],
               meta: dict | None = None) -> Trace:
    """Build and validate (reference trace.py:314-321)."""
    trace = Trace(kernels=list(kernels), tensors=list(tensors), meta=meta or {})
    report = validate_trace(trace)
    if not report.ok:
        raise TraceValidationError(report.violations)
    return trace


def make_trace_from_arrays(arrays: TraceArrays, meta: dict | None = None) -> Trace:
    trace = Trace.from_arrays(arrays, meta or {})
    report = validate_arrays(arrays)
    if not report.ok:
        raise TraceValidationError(report.violations)
    return trace
