"""Python mirror of the reference's distributed-matrix API over the C ABI.

Names, argument meaning and error behaviour follow gridgemm::Session
(/root/reference/proj/include/gridgemm/session.hpp:53-485) and the layout
helpers of gridgemm/layout.hpp so parity tests read like the reference's own
tests.  Every call goes through libdmath_b200.so; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import Descriptor, Layout, PoolStats, SessionConfig, TransferRecord, WorkerStats, lib


# --------------------------------------------------------------- errors
class Error(RuntimeError):
    """gridgemm::Error (common.hpp:22-25)."""


class UsageError(Error): ...
class ConfigError(Error): ...
class ShapeError(Error): ...
class ProtocolError(Error): ...
class DeadlockError(Error): ...
class IntegrityError(Error): ...
class PlanError(Error): ...
class CudaError(Error): ...
class NcclError(Error): ...
class UnsupportedError(Error): ...


class CacheMissError(Error):
    """gridgemm::CacheMissError (common.hpp:72-78)."""

    def __init__(self, what: str, missing_coords):
        super().__init__(what)
        self.missing_coords = list(missing_coords)


_CODES = {1: UsageError, 2: ConfigError, 3: ShapeError, 4: ProtocolError, 5: DeadlockError,
          6: IntegrityError, 7: PlanError, 8: CacheMissError, 9: CudaError, 10: NcclError,
          11: UnsupportedError}


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib.dm_last_error() or b"").decode(errors="replace")
    cls = _CODES.get(rc, Error)
    if cls is CacheMissError:
        buf = (C.c_int32 * 4096)()
        n = lib.dm_last_error_missing(buf, 2048)
        raise CacheMissError(msg, [(buf[2 * i], buf[2 * i + 1]) for i in range(min(n, 2048))])
    raise cls(msg)


# --------------------------------------------------------------- enums
class LayoutKind(enum.IntEnum):
    """layout.hpp:69-75"""
    RowBlocks1D = 0
    ColBlocks1D = 1
    RowCyclic1D = 2
    Checkerboard2D = 3
    Custom = 4


class Precision(enum.IntEnum):
    """precision.hpp:14"""
    Half16 = 0
    Single32 = 1
    Double64 = 2


class Axis(enum.IntEnum):
    """kernels.hpp:16 (add_row_col_sum axis)"""
    Rows = 0
    Cols = 1


class FillKind(enum.IntEnum):
    """runtime_types.hpp:68"""
    Zeros = 0
    SeededRandom = 1
    FromHost = 2


# --------------------------------------------------------------- layouts
@dataclass
class LayoutSpec:
    """LayoutSpec (layout.hpp:116-142).  block_rows/cols are the nominal
    (un-clamped) sizes as given; the library clamps like make_grid."""
    kind: LayoutKind
    global_rows: int
    global_cols: int
    block_rows: int
    block_cols: int
    worker_count: int
    custom: Optional[Sequence[int]] = None
    _keep: list = field(default_factory=list, repr=False, compare=False)

    def _abi(self) -> Layout:
        l = Layout(int(self.kind), int(self.worker_count), int(self.global_rows),
                   int(self.global_cols), int(self.block_rows), int(self.block_cols), None, 0)
        if self.custom is not None:
            arr = (C.c_int32 * len(self.custom))(*self.custom)
            self._keep[:] = [arr]
            l.custom = C.cast(arr, C.POINTER(C.c_int32))
            l.custom_len = len(self.custom)
        return l

    def owner(self, row: int, col: int) -> int:
        o = C.c_int()
        _check(lib.dm_layout_owner(C.byref(self._abi()), row, col, C.byref(o)))
        return o.value

    def grid(self):
        r, c, cl = C.c_int(), C.c_int(), C.c_int()
        _check(lib.dm_layout_grid(C.byref(self._abi()), C.byref(r), C.byref(c), C.byref(cl)))
        return r.value, c.value, bool(cl.value)

    def block_extent(self, row: int, col: int):
        r, c = C.c_int64(), C.c_int64()
        _check(lib.dm_block_extent(C.byref(self._abi()), row, col, C.byref(r), C.byref(c)))
        return r.value, c.value

    def to_string(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        n = lib.dm_layout_to_string(C.byref(self._abi()), buf, len(buf))
        if n < 0:
            _check(-n)
        return buf.value.decode()


def make_layout(kind, global_rows, global_cols, block_rows, block_cols, worker_count) -> LayoutSpec:
    """make_layout (layout.hpp:146-156)."""
    spec = LayoutSpec(LayoutKind(kind), global_rows, global_cols, block_rows, block_cols, worker_count)
    spec.grid()  # validates (UsageError on non-positive sizes)
    return spec


def make_custom_layout(global_rows, global_cols, block_rows, block_cols, worker_count, table) -> LayoutSpec:
    """make_custom_layout (layout.hpp:158-171)."""
    spec = LayoutSpec(LayoutKind.Custom, global_rows, global_cols, block_rows, block_cols,
                      worker_count, list(table))
    spec.grid()
    return spec


def checkerboard_dims(workers: int):
    pr, pc = C.c_int(), C.c_int()
    _check(lib.dm_checkerboard_dims(workers, C.byref(pr), C.byref(pc)))
    return pr.value, pc.value


def pool_size_class(nbytes: int) -> int:
    return int(lib.dm_pool_size_class(nbytes))


def plan_general_gemm(la: LayoutSpec, ta: bool, lb: LayoutSpec, tb: bool, lc: LayoutSpec, worker: int):
    """Distinct peer blocks (and bytes) `worker` reads for general_gemm."""
    nb, by = C.c_int64(), C.c_int64()
    _check(lib.dm_plan_general_gemm(C.byref(la._abi()), int(ta), C.byref(lb._abi()), int(tb),
                                    C.byref(lc._abi()), worker, C.byref(nb), C.byref(by)))
    return nb.value, by.value


def presplit_panels(k: int, a_kblock: int, b_kblock: int, max_width: int = 16384) -> list:
    """K-panel starts (then K) of a presplit GEMM (dm_presplit_panels)."""
    cap = 4 * (k // 256 + 4) + 8
    out = (C.c_int64 * cap)()
    n = C.c_int()
    _check(lib.dm_presplit_panels(int(k), int(a_kblock), int(b_kblock), int(max_width), out, cap, C.byref(n)))
    return list(out[:n.value])


# --------------------------------------------------------------- session
@dataclass
class Config:
    """Session::Config (session.hpp:55-62) plus the B200 placement fields."""
    worker_count: int = 1
    root_seed: int = 0
    coherence_checks: bool = True
    mode: str = "local"              # "local" (one process, all workers) | "spmd" (one per GPU)
    rank: int = 0                    # spmd only
    devices: Optional[Sequence[int]] = None  # local: device per worker; spmd: [device]
    nccl_id: Optional[bytes] = None  # spmd only: 128-byte id from nccl_unique_id() on rank 0
    # Config::deterministic (session.hpp:60): the reference picks single-threaded
    # interleaving for reproducibility; here every command already runs in one
    # global order with fixed-order reductions (non-deterministic row/col sums
    # are chosen per call), so the flag is accepted and reported, never needed.
    deterministic: bool = True
    # Split-product scheme of the fp32 tensor-core GEMM (include/dmath_b200.h
    # dm_gemm_mode): "default" (env DM_GEMM_MODE, else auto), "auto" (f16x2
    # for fp32 operands), "f16x2" (3xTF32's 11+11-bit split on fp16 operands
    # with per-row power-of-two scales), "3xtf32" (the north star's 3xTF32),
    # "mixed" (tf32 hi*hi + bf16 cross terms).
    gemm_mode: str = "default"


GEMM_MODES = {"default": 0, "mixed": 1, "3xtf32": 2, "auto": 3, "f16x2": 4}  # dm_gemm_mode


def split_mode_for(mode: str, k: int, work: float = -1.0) -> str:
    """The scheme a product over K with `work` = 2 m n k flops per worker
    (< 0: large) runs in under `mode` -- the library's own rule
    (dm_split_mode_for; auto: f16x2, 3xTF32 below DM_F16X2_MIN_GFLOP)."""
    if mode not in GEMM_MODES:
        raise UsageError(f"unknown gemm_mode {mode!r}")
    out = C.c_int()
    _check(lib.dm_split_mode_for(GEMM_MODES[mode], int(k), float(work), C.byref(out)))
    return {1: "mixed", 2: "3xtf32", 4: "f16x2"}[out.value]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.dm_nccl_unique_id(buf))
    return buf.raw


@dataclass
class MatrixDescriptor:
    matrix_id: int
    precision: Precision
    replicated: bool
    version: int
    replica_version: int
    seed: int
    layout: LayoutSpec


def _host_ptr(arr: np.ndarray):
    return C.c_void_p(arr.ctypes.data)


_DTYPES = {Precision.Half16: np.float16, Precision.Single32: np.float32, Precision.Double64: np.float64}


def _dtype(p) -> np.dtype:
    return np.dtype(_DTYPES[Precision(p)])


def _make_config(cfg: "Config"):
    mode = {"local": 0, "spmd": 1}[cfg.mode]
    keep = []
    devs = None
    if cfg.devices is not None:
        devs = (C.c_int32 * len(cfg.devices))(*cfg.devices)
        keep.append(devs)
    nid = None
    if cfg.nccl_id is not None:
        nid = C.create_string_buffer(bytes(cfg.nccl_id), 128)
        keep.append(nid)
    if cfg.gemm_mode not in GEMM_MODES:
        raise ConfigError(f"unknown gemm_mode {cfg.gemm_mode!r} (one of {sorted(GEMM_MODES)})")
    c = SessionConfig(cfg.worker_count, mode, cfg.rank, int(cfg.coherence_checks),
                      cfg.root_seed & (2**64 - 1),
                      C.cast(devs, C.POINTER(C.c_int32)) if devs is not None else None,
                      C.cast(nid, C.c_void_p) if nid is not None else None,
                      GEMM_MODES[cfg.gemm_mode])
    return c, keep


class Session:
    """gridgemm::Session on B200 workers (one GPU each)."""

    def __init__(self, cfg: Config, _handle=None):
        self._cfg = cfg
        if _handle is not None:
            self._h = _handle
            return
        c, _keep = _make_config(cfg)
        h = C.c_void_p()
        _check(lib.dm_session_create(C.byref(c), C.byref(h)))
        self._h = h

    @classmethod
    def restore(cls, path: str, cfg: Optional[Config] = None) -> "Session":
        """Session::restore (session.hpp:425-465): worker count and root seed
        come from the image; `cfg` supplies placement (mode, devices, NCCL id)."""
        cfg = cfg or Config()
        c, _keep = _make_config(cfg)
        h = C.c_void_p()
        _check(lib.dm_restore(path.encode(), C.byref(c), C.byref(h)))
        return cls(cfg, _handle=h)

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib.dm_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def shutdown(self):
        _check(lib.dm_session_shutdown(self._h))

    # -- introspection
    def deterministic(self) -> bool:
        """Session::deterministic (session.hpp:91)."""
        return bool(self._cfg.deterministic)

    def gemm_mode(self) -> str:
        """Split-product scheme of this session: "mixed", "3xtf32", "f16x2" or "auto"."""
        v = C.c_int()
        _check(lib.dm_session_gemm_mode(self._h, C.byref(v)))
        return {1: "mixed", 2: "3xtf32", 3: "auto", 4: "f16x2"}[v.value]

    def root_seed(self) -> int:
        """Session::root_seed (session.hpp:92); follows seed_workers and restore."""
        v = C.c_uint64()
        _check(lib.dm_root_seed(self._h, C.byref(v)))
        return v.value

    def worker_count(self) -> int:
        n = C.c_int()
        _check(lib.dm_worker_count(self._h, C.byref(n)))
        return n.value

    def local_workers(self):
        buf = (C.c_int32 * 1024)()
        n = lib.dm_local_workers(self._h, buf, 1024)
        if n < 0:
            _check(-n)
        return list(buf[:n])

    def descriptor(self, mid: int) -> MatrixDescriptor:
        d = Descriptor()
        _check(lib.dm_descriptor_get(self._h, mid, C.byref(d)))
        l = d.layout
        custom = [l.custom[i] for i in range(l.custom_len)] if l.custom_len else None
        spec = LayoutSpec(LayoutKind(l.kind), l.global_rows, l.global_cols, l.block_rows,
                          l.block_cols, l.worker_count, custom)
        return MatrixDescriptor(d.matrix_id, Precision(d.precision), bool(d.replicated), d.version,
                                d.replica_version, d.seed, spec)

    def worker_pool_stats(self, w: int) -> PoolStats:
        s = PoolStats()
        _check(lib.dm_pool_stats_get(self._h, w, C.byref(s)))
        return s

    def pool_trim(self, w: int) -> int:
        f = C.c_uint64()
        _check(lib.dm_pool_trim(self._h, w, C.byref(f)))
        return f.value

    def worker_stats(self, w: int) -> WorkerStats:
        s = WorkerStats()
        _check(lib.dm_worker_stats_get(self._h, w, C.byref(s)))
        return s

    def reset_worker_stats(self):
        _check(lib.dm_worker_stats_reset(self._h))

    def set_gemm_timing(self, on: bool):
        _check(lib.dm_set_gemm_timing(self._h, int(on)))

    def worker_seed(self, w: int) -> int:
        v = C.c_uint64()
        _check(lib.dm_worker_seed(self._h, w, C.byref(v)))
        return v.value

    def trace(self):
        """Session::trace() (session.hpp:94; TraceLog, transport.hpp:56-71): the
        worker-to-worker block transfers this process's workers pulled, oldest
        first, as dicts {seq, src, dst, matrix_id, row, col, bytes, op}.  A GEMM
        logs one record per foreign block it read (bytes = the part it read)."""
        n = lib.dm_transfer_log(self._h, None, 0)
        if n < 0:
            _check(-n)
        buf = (TransferRecord * max(n, 1))()
        n = lib.dm_transfer_log(self._h, buf, n)
        if n < 0:
            _check(-n)
        return [{"seq": r.seq, "src": r.src, "dst": r.dst, "matrix_id": r.matrix_id, "row": r.row,
                 "col": r.col, "bytes": r.bytes, "op": r.op.decode()} for r in buf[:n]]

    def seed_workers(self, root: int):
        """Session::seed_workers (session.hpp:115-125): the new root seeds the
        workers and every matrix created afterwards; returns mix64(root, w)."""
        n = self.worker_count()
        buf = (C.c_uint64 * n)()
        _check(lib.dm_seed_workers(self._h, C.c_uint64(root & 0xFFFFFFFFFFFFFFFF), buf, n))
        return list(buf)

    def descriptor_digests(self):
        m = C.c_uint64()
        buf = (C.c_uint64 * 1024)()
        n = lib.dm_descriptor_digest(self._h, C.byref(m), buf, 1024)
        if n < 0:
            _check(-n)
        return [m.value] + list(buf[:n])

    def block_device_ptr(self, mid: int, row: int, col: int):
        p, d = C.c_void_p(), C.c_int()
        _check(lib.dm_block_device_ptr(self._h, mid, row, col, C.byref(p), C.byref(d)))
        return p.value, d.value

    def barrier(self):
        """Complete all outstanding (asynchronous) work on every worker/rank."""
        _check(lib.dm_barrier(self._h))
        self._async_keep = []

    def set_async(self, on: bool):
        """Asynchronous command mode (dm_set_async): scatter / gather /
        general_gemm return once enqueued; host buffers must stay alive and
        unmodified until barrier() or set_async(False)."""
        _check(lib.dm_set_async(self._h, int(on)))
        if not on:
            self._async_keep = []

    def marker_record(self, worker: int, slot: int):
        """Record device-time marker `slot` on the worker's GEMM stream."""
        _check(lib.dm_marker_record(self._h, worker, slot))

    def marker_elapsed(self, worker: int, a: int, b: int) -> float:
        ms = C.c_float()
        _check(lib.dm_marker_elapsed(self._h, worker, a, b, C.byref(ms)))
        return ms.value

    # -- matrices
    def create_matrix(self, layout: LayoutSpec, precision=Precision.Single32,
                      fill=FillKind.Zeros, host: Optional[np.ndarray] = None) -> int:
        """Session::create_matrix (session.hpp:129-150)."""
        hp = None
        if fill == FillKind.FromHost:
            if host is None:
                raise UsageError("create_matrix: FromHost requires host data")
            host = self._host_in(host, precision)
            if host.shape != (layout.global_rows, layout.global_cols):
                raise ShapeError("create_matrix: host data shape does not match the layout")
            hp = _host_ptr(host)
        out = C.c_uint64()
        _check(lib.dm_create_matrix(self._h, C.byref(layout._abi()), int(precision), int(fill), hp,
                                    C.byref(out)))
        return out.value

    def destroy_matrix(self, mid: int):
        _check(lib.dm_destroy_matrix(self._h, mid))

    def _keep_host(self, arr):
        """Async mode: keep converted host arrays alive until the next barrier."""
        keep = getattr(self, "_async_keep", None)
        if keep is None:
            keep = self._async_keep = []
        keep.append(arr)

    @staticmethod
    def _host_in(host: np.ndarray, precision) -> np.ndarray:
        """Host data at the matrix precision.  Other dtypes are converted with
        numpy's round-to-nearest-even, like the reference's scatter_payloads
        per-element conversion (session.hpp:568-576)."""
        return np.ascontiguousarray(host, dtype=_dtype(precision))

    def scatter(self, mid: int, host: np.ndarray):
        """Session::scatter (session.hpp:164-175); bit-exact."""
        host = self._host_in(host, self.descriptor(mid).precision)
        if host.ndim != 2:
            raise ShapeError("scatter: host data must be 2-D")
        self._keep_host(host)
        _check(lib.dm_scatter(self._h, mid, _host_ptr(host), host.shape[0], host.shape[1]))

    def gather(self, mid: int, out: Optional[np.ndarray] = None, root: int = 0) -> np.ndarray:
        """Session::gather (session.hpp:179-201); bit-exact, owned blocks only."""
        d = self.descriptor(mid)
        shape = (d.layout.global_rows, d.layout.global_cols)
        dt = _dtype(d.precision)
        if out is None:
            out = np.empty(shape, dtype=dt)
        if out.shape != shape or out.dtype != dt or not out.flags.c_contiguous:
            raise ShapeError("gather: output buffer shape does not match the matrix")
        _check(lib.dm_gather(self._h, mid, _host_ptr(out), shape[0], shape[1], root))
        return out

    def update_block(self, mid: int, row: int, col: int, data: np.ndarray):
        """Session::update_block (session.hpp:203-222)."""
        data = self._host_in(data, self.descriptor(mid).precision)
        if data.ndim != 2:
            raise ShapeError("update_block: data must be 2-D")
        _check(lib.dm_update_block(self._h, mid, row, col, _host_ptr(data), data.shape[0], data.shape[1]))

    # -- replication, reshape, row/col sums, checkpoint
    def replicate(self, mid: int, enable: bool):
        """Session::replicate (session.hpp:266-274)."""
        _check(lib.dm_replicate(self._h, mid, int(enable)))

    def replica_read(self, mid: int, reader: int) -> np.ndarray:
        """Session::replica_read (session.hpp:276-297)."""
        d = self.descriptor(mid)
        out = np.empty((d.layout.global_rows, d.layout.global_cols), dtype=_dtype(d.precision))
        _check(lib.dm_replica_read(self._h, mid, reader, _host_ptr(out), out.shape[0], out.shape[1]))
        return out

    def reshape(self, src: int, layout: LayoutSpec, precision=Precision.Single32) -> int:
        """Session::reshape (session.hpp:299-317)."""
        out = C.c_uint64()
        _check(lib.dm_reshape(self._h, src, C.byref(layout._abi()), int(precision), C.byref(out)))
        return out.value

    def add_row_col_sum(self, mid: int, axis: int, deterministic_reduce: bool = True) -> int:
        """Session::add_row_col_sum (session.hpp:321-348); axis 0 = rows, 1 = cols."""
        out = C.c_uint64()
        _check(lib.dm_add_row_col_sum(self._h, mid, int(axis), int(deterministic_reduce), C.byref(out)))
        return out.value

    def checkpoint(self, path: str):
        """Session::checkpoint (session.hpp:395-423), DMTH v1 file."""
        _check(lib.dm_checkpoint(self._h, path.encode()))

    # -- distributed operations
    def general_gemm(self, alpha, a, b, beta, c, trans_a=False, trans_b=False):
        """Session::general_gemm (session.hpp:244-250)."""
        _check(lib.dm_general_gemm(self._h, float(alpha), a, b, float(beta), c, int(trans_a), int(trans_b)))

    def cyclic_gemm(self, alpha, a, b, beta, c, trans_a=False, trans_b=False, cache_a=False):
        """Session::cyclic_gemm (session.hpp:226-234)."""
        _check(lib.dm_cyclic_gemm(self._h, float(alpha), a, b, float(beta), c, int(trans_a),
                                  int(trans_b), int(cache_a)))

    def broadcast_gemm_reference(self, alpha, a, b, beta, c, trans_a=False, trans_b=False):
        """Session::broadcast_gemm_reference (session.hpp:236-242)."""
        _check(lib.dm_broadcast_gemm_reference(self._h, float(alpha), a, b, float(beta), c,
                                               int(trans_a), int(trans_b)))

    def cached_backward_gemm(self, w, dy, dx):
        """Session::cached_backward_gemm (session.hpp:254-264)."""
        _check(lib.dm_cached_backward_gemm(self._h, w, dy, dx))


# --------------------------------------------------------------- device seam
def local_gemm(alpha, a, trans_a, b, trans_b, beta, c, cta_group: int = 0, stream=None,
               gemm_mode: str = "default", workspace=None):
    """local_gemm (kernels.hpp:81-89) on CUDA tensors (anything exposing
    data_ptr()/shape/stride, e.g. torch float32 CUDA tensors, row-major).
    Stream-ordered: enqueues on `stream` (a cudaStream_t as int, None = the
    legacy default stream) and returns.  `workspace` (a CUDA tensor of at
    least local_gemm_workspace_size() bytes) makes the call allocation-free
    and capturable in a CUDA graph."""
    def dims(t):
        r, cc = t.shape
        if t.stride(1) != 1:
            raise UsageError("local_gemm: operands must be row-major (unit column stride)")
        return r, cc, t.stride(0)
    ar, ac, lda = dims(a)
    br, bc, ldb = dims(b)
    cr, cc, ldc = dims(c)
    m, k = (ac, ar) if trans_a else (ar, ac)
    kb, n = (bc, br) if trans_b else (br, bc)
    if k != kb:
        raise ShapeError("local_gemm: inner dimensions do not conform")
    if (cr, cc) != (m, n):
        raise ShapeError("local_gemm: output dimensions do not conform")
    st = C.c_void_p(stream) if stream is not None else None
    if gemm_mode not in GEMM_MODES:
        raise UsageError(f"unknown gemm_mode {gemm_mode!r}")
    if workspace is not None:
        nbytes = workspace.numel() * workspace.element_size()
        _check(lib.dm_local_gemm_f32_ws(float(alpha), C.c_void_p(a.data_ptr()), lda, int(trans_a),
                                        C.c_void_p(b.data_ptr()), ldb, int(trans_b), float(beta),
                                        C.c_void_p(c.data_ptr()), ldc, m, n, k, cta_group,
                                        GEMM_MODES[gemm_mode], C.c_void_p(workspace.data_ptr()), nbytes, st))
        return
    _check(lib.dm_local_gemm_f32_ex(float(alpha), C.c_void_p(a.data_ptr()), lda, int(trans_a),
                                    C.c_void_p(b.data_ptr()), ldb, int(trans_b), float(beta),
                                    C.c_void_p(c.data_ptr()), ldc, m, n, k, cta_group,
                                    GEMM_MODES[gemm_mode], st))


def local_gemm_workspace_size(m: int, n: int, k: int, cta_group: int = 0, gemm_mode: str = "default") -> int:
    """Bytes of caller workspace local_gemm(..., workspace=) needs on the current device."""
    out = C.c_size_t()
    _check(lib.dm_local_gemm_f32_workspace_size(m, n, k, cta_group, GEMM_MODES[gemm_mode], C.byref(out)))
    return out.value


def fill_seeded(t, matrix_seed: int, block_row: int, block_col: int, stream=None):
    """WorkerContext::fill_seeded (runtime_types.hpp:208-218) into a CUDA tensor."""
    st = C.c_void_p(stream) if stream is not None else None
    _check(lib.dm_fill_seeded_f32(C.c_void_p(t.data_ptr()), t.numel(), matrix_seed & (2**64 - 1),
                                  block_row, block_col, st))
