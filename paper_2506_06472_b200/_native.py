"""ctypes binding of libtio (include/tio.h).

The product path: every compute call goes through these entry points into
the sm_100a CUDA library.  There is no CPU fallback — if libtio.so is missing
or no CUDA device is visible the calls raise `NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import build as _build

_lock = threading.Lock()
_lib = None

TIO_OK = 0
TIO_ERR_INVALID = -1
TIO_ERR_UNSATISFIABLE = -2
TIO_ERR_CHANNEL_CONFIG = -3
TIO_ERR_CUDA = -4
TIO_ERR_NOMEM = -5
TIO_ERR_INTERNAL = -6
TIO_ERR_OVERFLOW = -7
TIO_ERR_SIMULATION = -8
TIO_ERR_CONFIG = -9

TIO_MEM_HOST = 0
TIO_MEM_DEVICE = 1
DEST_NAMES = {0: "GPU", 1: "SSD", 2: "CPU"}


class NativeUnavailable(RuntimeError):
    """libtio.so could not be loaded or no CUDA device is usable."""


class TioError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"libtio error {code}: {message}")
        self.code = code
        self.message = message


_i64 = ctypes.c_int64
_p = ctypes.c_void_p


class TraceDesc(ctypes.Structure):
    _fields_ = [("num_kernels", _i64), ("duration_us", _p), ("num_tensors", _i64),
                ("tensor_id", _p), ("size_bytes", _p), ("kind", _p), ("access_ptr", _p),
                ("num_events", _i64), ("accesses", _p)]


class Rates(ctypes.Structure):
    _fields_ = [("ssd_offload", ctypes.c_double), ("ssd_prefetch", ctypes.c_double),
                ("has_host", ctypes.c_int), ("host_offload", ctypes.c_double),
                ("host_prefetch", ctypes.c_double)]


class LifetimeView(ctypes.Structure):
    _fields_ = [("num_kernels", _i64), ("num_tensors", _i64), ("num_periods", _i64),
                ("iteration_us", _i64), ("starts", _p), ("timeline", _p), ("active", _p),
                ("period_tensor", _p), ("period_start", _p), ("period_end", _p),
                ("period_wraps", _p), ("tensor_period_ptr", _p)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, _i64) for n in ("num_commits", "num_entries", "num_over", "capacity_bytes",
                                    "residual_peak_bytes", "planned_host_bytes", "num_candidates",
                                    "rounds", "unsat_kernel", "unsat_bytes", "loop_ns")] + [
        ("dbg", _i64 * 14)]


class PlanOpts(ctypes.Structure):
    _fields_ = [("max_rounds", _i64), ("warp_refit_max", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("blocks", ctypes.c_int32),
                ("pad2", ctypes.c_int32), ("epoch", ctypes.c_uint64), ("mailbox", ctypes.c_void_p),
                ("peer_mailboxes", ctypes.POINTER(ctypes.c_void_p))]


class SimReportC(ctypes.Structure):
    _fields_ = [(n, _i64) for n in ("total_time", "ideal_time", "stall_time_total", "peak_resident_bytes",
                                    "emergency_offloads")] + [("channel_busy", _i64 * 4), ("num_transfers", _i64)]


class RooflineInfoC(ctypes.Structure):
    _fields_ = [(n, _i64) for n in ("ideal_us", "peak_bytes", "pressured", "num_periods", "max_period_bytes")]


COMMIT_DTYPE = np.dtype([("tensor_id", "<i8"), ("tensor_pos", "<i8"), ("start_kernel", "<i8"),
                         ("end_kernel", "<i8"), ("wraps", "<i8"), ("destination", "<i8"),
                         ("off_start", "<i8"), ("off_end", "<i8"), ("pre_start", "<i8"),
                         ("pre_end", "<i8"), ("benefit_lo", "<u8"), ("benefit_hi", "<u8"),
                         ("cost", "<i8"), ("rel0_lo", "<i8"), ("rel0_hi", "<i8"),
                         ("rel1_lo", "<i8"), ("rel1_hi", "<i8")])
TRANSFER_DTYPE = np.dtype([("tensor_pos", "<i8"), ("tensor_id", "<i8"), ("action", "<i4"), ("device", "<i4"),
                           ("urgent", "<i4"), ("emergency", "<i4"), ("start_us", "<i8"), ("end_us", "<i8"),
                           ("after_kernel", "<i8"), ("tail", "<i8"), ("seq", "<i8")])
ENTRY_DTYPE = np.dtype([("tensor_id", "<i8"), ("tensor_pos", "<i8"), ("trigger_us", "<i8"),
                        ("deadline_us", "<i8"), ("action", "<i4"), ("target", "<i4"),
                        ("urgent", "<i4"), ("pad", "<i4")])

# every exported symbol of include/tio.h
EXPORTS = ("tio_abi_version", "tio_kernel_launches", "tio_last_error", "tio_device_info", "tio_trace_create",
           "tio_trace_destroy", "tio_lifetime", "tio_lifetime_view_get", "tio_lifetime_copy_out",
           "tio_plan_create", "tio_plan_create2", "tio_plan_info_get", "tio_plan_copy_out", "tio_plan_write",
           "tio_plan_destroy", "tio_plan_host", "tio_transfer_duration", "tio_simulate", "tio_simulate_layers", "tio_roofline",
           "tio_engine_replay", "tio_pack", "tio_unpack", "tio_schedule", "tio_trace_parse",
           "tio_parsed_sizes", "tio_parsed_copy", "tio_parsed_destroy",
           "tio_engine_create", "tio_engine_info", "tio_engine_bind", "tio_engine_step_begin",
           "tio_engine_before_kernel", "tio_engine_after_kernel", "tio_engine_step_end", "tio_engine_stats_get",
           "tio_engine_destroy", "tio_checksum",
           "tio_engine_set_verify", "tio_engine_restore",
           "tio_engine_check_program", "tio_engine_step_abort", "tio_plan_create_virtual",
           "tio_mailbox_create", "tio_mailbox_destroy", "tio_mailbox_open", "tio_mailbox_close",
           "tio_channel_create", "tio_channel_destroy", "tio_channel_reserve_earliest", "tio_channel_reserve_latest",
           "tio_channel_record", "tio_channel_release", "tio_channel_size", "tio_channel_copy", "tio_channel_busy",
           "tio_candidate_window", "tio_host_peak_occupancy", "tio_candidate_benefit",
           "tio_period_interior")


def lib_path() -> str:
    # TIO_LIB_PATH: a variant build (tools/build_variant.sh) for experiments
    return os.environ.get("TIO_LIB_PATH") or _build.LIB


def load(build_if_missing: bool = True):
    """Load libtio.so (building it first if absent and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise NativeUnavailable(f"{path} not built")
            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                raise NativeUnavailable(f"cannot build libtio: {exc}") from exc
        lib = ctypes.CDLL(path)
        for name in EXPORTS:
            getattr(lib, name).restype = ctypes.c_int
        lib.tio_mailbox_bytes.restype = ctypes.c_size_t
        if lib.tio_abi_version() != 1:
            raise NativeUnavailable("libtio ABI mismatch")
        _lib = lib
        return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().tio_last_error(buf, ctypes.c_size_t(1024))
    return buf.value.decode("utf-8", "replace")


def check(rc: int) -> None:
    if rc != TIO_OK:
        raise TioError(rc, last_error())


_cuda_checked = False


def require_device() -> None:
    """Fail loudly when no CUDA device is usable (there is no CPU path)."""
    global _cuda_checked
    if _cuda_checked:
        return
    lib = load()
    buf = ctypes.create_string_buffer(256)
    rc = lib.tio_device_info(buf, ctypes.c_size_t(256))
    if rc != TIO_OK:
        raise NativeUnavailable("no usable CUDA device for libtio: " + last_error())
    _cuda_checked = True


def device_info() -> str:
    lib = load()
    buf = ctypes.create_string_buffer(256)
    check(lib.tio_device_info(buf, ctypes.c_size_t(256)))
    return buf.value.decode()


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


class HostColumns:
    """Contiguous host copies of the columns libtio reads (kept alive while in use)."""

    def __init__(self, arrays):
        self.dur = np.ascontiguousarray(arrays.duration_us, dtype=np.int64)
        self.tid = np.ascontiguousarray(arrays.tensor_id, dtype=np.int64)
        self.size = np.ascontiguousarray(arrays.size_bytes, dtype=np.int64)
        self.kind = np.ascontiguousarray(arrays.kind, dtype=np.int8)
        self.ptr = np.ascontiguousarray(arrays.access_ptr, dtype=np.int64)
        acc = np.asarray(arrays.accesses)
        if acc.size and (int(acc.min()) < np.iinfo(np.int32).min or int(acc.max()) > np.iinfo(np.int32).max):
            # an unvalidated trace: keep the value out of range instead of wrapping it
            # into a valid kernel index (libtio range-checks every access against N)
            acc = np.clip(acc, -1, np.iinfo(np.int32).max)
        self.acc = np.ascontiguousarray(acc, dtype=np.int32)

    def desc(self) -> TraceDesc:
        return TraceDesc(self.dur.shape[0], _ptr(self.dur), self.tid.shape[0], _ptr(self.tid),
                         _ptr(self.size), _ptr(self.kind), _ptr(self.ptr), self.acc.shape[0],
                         _ptr(self.acc))


class DeviceTrace:
    """A trace resident in HBM (libtio `tio_trace` handle, host-uploaded)."""

    def __init__(self, arrays, stream: int = 0):
        require_device()
        self._lib = load()
        self.cols = HostColumns(arrays)
        self.stream = ctypes.c_void_p(stream)
        self.handle = ctypes.c_void_p()
        d = self.cols.desc()
        check(self._lib.tio_trace_create(ctypes.byref(d), TIO_MEM_HOST, self.stream,
                                         ctypes.byref(self.handle)))
        self.num_kernels = d.num_kernels
        self.num_tensors = d.num_tensors

    def close(self) -> None:
        if self.handle:
            self._lib.tio_trace_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lifetime(self) -> dict:
        lib = self._lib
        check(lib.tio_lifetime(self.handle, self.stream))
        v = LifetimeView()
        check(lib.tio_lifetime_view_get(self.handle, self.stream, ctypes.byref(v)))
        n, p = v.num_kernels, v.num_periods
        out = {"starts": np.zeros(n + 1, np.int64), "timeline": np.zeros(n, np.int64),
               "active": np.zeros(n, np.int64), "period_tensor": np.zeros(p, np.int64),
               "period_start": np.zeros(p, np.int32), "period_end": np.zeros(p, np.int32),
               "period_wraps": np.zeros(p, np.int8)}
        check(lib.tio_lifetime_copy_out(
            self.handle, self.stream, _ptr(out["starts"]), _ptr(out["timeline"]), _ptr(out["active"]),
            _ptr(out["period_tensor"]), _ptr(out["period_start"]), _ptr(out["period_end"]),
            _ptr(out["period_wraps"])))
        out["iteration"] = v.iteration_us
        return out

    def plan(self, capacity: int, rates: Rates, host_cap: int, max_rounds: int = 0, shard=None) -> "DevicePlan":
        info = PlanInfo()
        h = ctypes.c_void_p()
        opts = PlanOpts(max_rounds, -1, 0)
        if shard is not None:
            # sharded planning: (rank, nranks, own mailbox ptr, [peer mailbox ptrs], epoch)
            rank, nranks, mb, peers, epoch = shard
            self._peers = (ctypes.c_void_p * nranks)(*peers)
            opts.nranks, opts.rank, opts.epoch, opts.mailbox = nranks, rank, epoch, mb
            opts.peer_mailboxes = ctypes.cast(self._peers, ctypes.POINTER(ctypes.c_void_p))
        rc = self._lib.tio_plan_create2(self.handle, _i64(capacity), ctypes.byref(rates), _i64(host_cap),
                                        ctypes.byref(opts), self.stream, ctypes.byref(h), ctypes.byref(info))
        if rc != TIO_OK:
            err = TioError(rc, last_error())
            err.info = info
            raise err
        return DevicePlan(self._lib, h, info, self.stream, self.num_kernels)

    def plan_virtual(self, capacity: int, rates: Rates, host_cap: int, nranks: int,
                     max_rounds: int = 0) -> list:
        """The sharded planner with `nranks` virtual ranks on this GPU
        (tio_plan_create_virtual): one DevicePlan per rank."""
        infos = (PlanInfo * nranks)()
        hs = (ctypes.c_void_p * nranks)()
        opts = PlanOpts(max_rounds, -1, 0)
        rc = self._lib.tio_plan_create_virtual(self.handle, _i64(capacity), ctypes.byref(rates), _i64(host_cap),
                                               ctypes.byref(opts), ctypes.c_int32(nranks), hs, infos)
        if rc != TIO_OK:
            raise TioError(rc, last_error())
        return [DevicePlan(self._lib, ctypes.c_void_p(hs[r]), infos[r], None, self.num_kernels)
                for r in range(nranks)]


class DevicePlan:
    def __init__(self, lib, handle, info: PlanInfo, stream, num_kernels: int):
        self._lib = lib
        self.handle = handle
        self.info = info
        self.stream = stream
        self.num_kernels = num_kernels

    def copy_out(self) -> dict:
        i = self.info
        commits = np.zeros(i.num_commits, COMMIT_DTYPE)
        entries = np.zeros(i.num_entries, ENTRY_DTYPE)
        resid = np.zeros(self.num_kernels, np.int64)
        over = np.zeros(i.num_over, np.int64)
        check(self._lib.tio_plan_copy_out(self.handle, self.stream, _ptr(commits), _ptr(entries),
                                          _ptr(resid), _ptr(over)))
        return {"commits": commits, "entries": entries, "residual": resid, "over": over}

    def write(self) -> bytes:
        n = ctypes.c_size_t(0)
        check(self._lib.tio_plan_write(self.handle, self.stream, None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        check(self._lib.tio_plan_write(self.handle, self.stream, buf, ctypes.byref(n)))
        return buf.raw[:n.value]

    def close(self) -> None:
        if self.handle:
            self._lib.tio_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


IPC_HANDLE_BYTES = 64


class Mailbox:
    """One rank's sharded-planning mailbox in device memory (tio_mailbox_create)
    and its CUDA IPC handle for the other ranks."""

    def __init__(self):
        require_device()
        self._lib = load()
        self.ptr = ctypes.c_void_p()
        buf = (ctypes.c_ubyte * IPC_HANDLE_BYTES)()
        check(self._lib.tio_mailbox_create(ctypes.byref(self.ptr), buf))
        self.handle = bytes(buf)

    def close(self) -> None:
        if self.ptr:
            self._lib.tio_mailbox_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mailbox_open(handle: bytes) -> int:
    """Map another process's mailbox (CUDA IPC, peer access over NVLink)."""
    lib = load()
    buf = (ctypes.c_ubyte * IPC_HANDLE_BYTES).from_buffer_copy(handle)
    out = ctypes.c_void_p()
    check(lib.tio_mailbox_open(buf, ctypes.byref(out)))
    return int(out.value)


def mailbox_close(ptr: int) -> None:
    check(load().tio_mailbox_close(ctypes.c_void_p(ptr)))


def kernel_launches() -> int:
    out = _i64()
    check(load().tio_kernel_launches(ctypes.byref(out)))
    return out.value


def transfer_duration(rate: float, nbytes: int) -> int:
    out = _i64()
    check(load().tio_transfer_duration(ctypes.c_double(rate), _i64(nbytes), ctypes.byref(out)))
    return out.value
