"""TEST INFRASTRUCTURE ONLY -- the checkers for the dmath_b200 hot path.

  * `C` : plain-C restatement of the reference arithmetic (dmath_oracle.c),
          pinned bit-for-bit against the reference's own outputs
          (tests/golden/, tests/test_oracle.py).
  * `REF`: the unmodified reference implementation compiled from
          /root/reference/proj/include (oracle/_ref/libgridgemm_ref.so, built
          by oracle/Makefile in the build container and shipped prebuilt).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "liboracle_c.so")
REF_LIB = os.path.join(HERE, "_ref", "libgridgemm_ref.so")

i64, u64, f64, vp = C.c_int64, C.c_uint64, C.c_double, C.c_void_p
FP = C.POINTER(C.c_float)


def build() -> None:
    """Compile the C restatement and, where /root/reference exists, the reference."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(FP)


def _load_c():
    if not os.path.exists(C_LIB):
        build()
    lib = C.CDLL(C_LIB)
    lib.orc_mix64.restype = u64
    lib.orc_mix64.argtypes = [u64]
    lib.orc_mix64_2.restype = u64
    lib.orc_mix64_2.argtypes = [u64, u64]
    lib.orc_fnv1a.restype = u64
    lib.orc_fnv1a.argtypes = [vp, i64]
    lib.orc_matrix_seed.restype = u64
    lib.orc_matrix_seed.argtypes = [u64, u64]
    lib.orc_fill_block.restype = None
    lib.orc_fill_block.argtypes = [FP, i64, i64, u64, C.c_int, C.c_int]
    lib.orc_fill_range.restype = None
    lib.orc_fill_range.argtypes = [FP, i64, i64, u64, C.c_int, C.c_int]
    lib.orc_checkerboard_dims.restype = None
    lib.orc_checkerboard_dims.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.orc_owner.restype = C.c_int
    lib.orc_owner.argtypes = [C.c_int] * 6
    lib.orc_local_gemm_f32.restype = None
    lib.orc_local_gemm_f32.argtypes = [f64, FP, i64, i64, C.c_int, FP, i64, i64, C.c_int, f64, FP]
    lib.orc_rel_frobenius.restype = f64
    lib.orc_rel_frobenius.argtypes = [FP, FP, i64]
    return lib


class COracle:
    """Restated reference arithmetic (dmath_oracle.c)."""

    def __init__(self):
        self.lib = _load_c()

    def mix64_2(self, a: int, b: int) -> int:
        return self.lib.orc_mix64_2(a & (2**64 - 1), b & (2**64 - 1))

    def fnv1a(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        return self.lib.orc_fnv1a(arr.ctypes.data, arr.nbytes)

    def matrix_seed(self, root: int, mid: int) -> int:
        return self.lib.orc_matrix_seed(root & (2**64 - 1), mid)

    def fill_block(self, rows, cols, matrix_seed, brow, bcol) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        self.lib.orc_fill_block(_fp(out), rows, cols, matrix_seed & (2**64 - 1), brow, bcol)
        return out

    def fill_block_parallel(self, rows, cols, matrix_seed, brow, bcol, threads=8) -> np.ndarray:
        """fill_block split over host threads (ctypes releases the GIL)."""
        import threading
        out = np.empty(rows * cols, np.float32)
        n = out.size
        step = -(-n // threads)
        base = out.ctypes.data

        def work(e0):
            cnt = min(step, n - e0)
            if cnt > 0:
                self.lib.orc_fill_range(C.cast(base + 4 * e0, FP), e0, cnt, matrix_seed & (2**64 - 1),
                                        brow, bcol)
        ts = [threading.Thread(target=work, args=(t * step,)) for t in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return out.reshape(rows, cols)

    def checkerboard_dims(self, w):
        pr, pc = C.c_int(), C.c_int()
        self.lib.orc_checkerboard_dims(w, C.byref(pr), C.byref(pc))
        return pr.value, pc.value

    def owner(self, kind, nbr, nbc, workers, row, col) -> int:
        return self.lib.orc_owner(int(kind), nbr, nbc, workers, row, col)

    def seeded_matrix(self, root_seed, mid, kind, gr, gc, br, bc) -> np.ndarray:
        """Full matrix as the reference's SeededRandom create + gather produce it."""
        br, bc = min(br, gr), min(bc, gc)
        seed = self.matrix_seed(root_seed, mid)
        out = np.empty((gr, gc), np.float32)
        for r in range(-(-gr // br)):
            for c in range(-(-gc // bc)):
                rr, cc = min(br, gr - r * br), min(bc, gc - c * bc)
                out[r * br:r * br + rr, c * bc:c * bc + cc] = self.fill_block(rr, cc, seed, r, c)
        return out

    def local_gemm(self, alpha, a, ta, b, tb, beta, c0=None) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        c = np.zeros((m, n), np.float32) if c0 is None else np.array(c0, np.float32, copy=True)
        self.lib.orc_local_gemm_f32(float(alpha), _fp(a), a.shape[0], a.shape[1], int(ta), _fp(b),
                                    b.shape[0], b.shape[1], int(tb), float(beta), _fp(c))
        return c

    def rel_frobenius(self, got, want) -> float:
        got = np.ascontiguousarray(got, np.float32)
        want = np.ascontiguousarray(want, np.float32)
        return self.lib.orc_rel_frobenius(_fp(got), _fp(want), want.size)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


class RefOracle:
    """The reference implementation itself (oracle/_ref)."""

    def __init__(self):
        if not os.path.exists(REF_LIB):
            build()
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(REF_LIB)
        lib = C.CDLL(REF_LIB)
        P = C.POINTER
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_mix64_2": (u64, [u64, u64]),
            "ref_session_create": (C.c_int, [C.c_int, u64, C.c_int, P(vp)]),
            "ref_session_destroy": (C.c_int, [vp]),
            "ref_create_matrix": (C.c_int, [vp, C.c_int, i64, i64, i64, i64, C.c_int, C.c_int, FP, P(u64)]),
            "ref_gather": (C.c_int, [vp, u64, FP, i64]),
            "ref_scatter": (C.c_int, [vp, u64, FP, i64, i64]),
            "ref_general_gemm": (C.c_int, [vp, f64, u64, u64, f64, u64, C.c_int, C.c_int]),
            "ref_cyclic_gemm": (C.c_int, [vp, f64, u64, u64, f64, u64, C.c_int, C.c_int, C.c_int]),
            "ref_cached_backward_gemm": (C.c_int, [vp, u64, u64, u64]),
            "ref_broadcast_gemm": (C.c_int, [vp, f64, u64, u64, f64, u64, C.c_int, C.c_int]),
            "ref_trace_records": (C.c_int, [vp, u64, P(i64), C.c_char_p, C.c_int, P(C.c_int)]),
            "ref_descriptor": (C.c_int, [vp, u64, P(u64), P(u64)]),
            "ref_pool_stats": (C.c_int, [vp, C.c_int, P(u64)]),
            "ref_trace_count": (C.c_int, [vp, P(u64), P(u64)]),
            "ref_layout_owner": (C.c_int, [C.c_int, i64, i64, i64, i64, C.c_int, C.c_int, C.c_int, P(C.c_int)]),
            "ref_layout_string": (C.c_int, [C.c_int, i64, i64, i64, i64, C.c_int, C.c_char_p, C.c_int]),
            "ref_local_gemm_f32": (C.c_int, [f64, FP, i64, i64, C.c_int, FP, i64, i64, C.c_int, f64, FP, i64, i64]),
            "ref_sampled_rows": (C.c_int, [f64, FP, i64, i64, FP, i64, i64, C.c_int, f64, FP, FP, i64, C.c_int]),
            "ref_sampled_cols": (C.c_int, [f64, FP, i64, i64, C.c_int, FP, i64, i64, f64, FP, FP, i64, C.c_int]),
            "ref_fill_block": (C.c_int, [FP, i64, i64, u64, C.c_int, C.c_int]),
            "ref_fnv1a": (u64, [vp, i64]),
            "ref_create_matrix_p": (C.c_int, [vp, C.c_int, i64, i64, i64, i64, C.c_int, C.c_int, C.c_int, vp, P(u64)]),
            "ref_gather_bytes": (C.c_int, [vp, u64, vp, i64]),
            "ref_update_block": (C.c_int, [vp, u64, C.c_int, C.c_int, C.c_int, vp, i64, i64]),
            "ref_reshape": (C.c_int, [vp, u64, C.c_int, i64, i64, i64, i64, C.c_int, C.c_int, P(u64)]),
            "ref_add_row_col_sum": (C.c_int, [vp, u64, C.c_int, C.c_int, P(u64)]),
            "ref_replicate": (C.c_int, [vp, u64, C.c_int]),
            "ref_replica_read": (C.c_int, [vp, u64, C.c_int, vp, i64]),
            "ref_checkpoint": (C.c_int, [vp, C.c_char_p]),
            "ref_restore": (C.c_int, [C.c_char_p, P(vp)]),
            "ref_descriptor_full": (C.c_int, [vp, u64, P(u64), C.c_char_p, C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    def err(self) -> str:
        return (self.lib.ref_last_error() or b"").decode()

    def check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.err()}")

    def local_gemm(self, alpha, a, ta, b, tb, beta, c0=None) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        c = np.zeros((m, n), np.float32) if c0 is None else np.array(c0, np.float32, copy=True)
        self.check(self.lib.ref_local_gemm_f32(float(alpha), _fp(a), a.shape[0], a.shape[1], int(ta),
                                               _fp(b), b.shape[0], b.shape[1], int(tb), float(beta),
                                               _fp(c), m, n))
        return c

    def sampled_rows(self, alpha, a_rows, b, tb, beta, c0_rows, threads=1) -> np.ndarray:
        """Rows of alpha*opA*opB + beta*C0 for the given op(A) rows (bit-exact with
        the reference's distributed result for those rows)."""
        a_rows = np.ascontiguousarray(a_rows, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        n = b.shape[0] if tb else b.shape[1]
        out = np.zeros((a_rows.shape[0], n), np.float32)
        c0 = np.ascontiguousarray(c0_rows if c0_rows is not None else out, np.float32)
        self.check(self.lib.ref_sampled_rows(float(alpha), _fp(a_rows), a_rows.shape[0], a_rows.shape[1],
                                             _fp(b), b.shape[0], b.shape[1], int(tb), float(beta),
                                             _fp(c0), _fp(out), n, threads))
        return out

    def sampled_cols(self, alpha, a, ta, b_cols, beta, c0_cols, threads=1) -> np.ndarray:
        """Columns of alpha*opA*opB + beta*C0 for the given op(B) columns
        (`b_cols`: ncols x K, row j = op(B)[:, j]); returns ncols x m (row j =
        C[:, j]), bit-exact with the reference's distributed result."""
        a = np.ascontiguousarray(a, np.float32)
        b_cols = np.ascontiguousarray(b_cols, np.float32)
        m = a.shape[1] if ta else a.shape[0]
        out = np.zeros((b_cols.shape[0], m), np.float32)
        c0 = np.ascontiguousarray(c0_cols if c0_cols is not None else out, np.float32)
        self.check(self.lib.ref_sampled_cols(float(alpha), _fp(a), a.shape[0], a.shape[1], int(ta), _fp(b_cols),
                                             b_cols.shape[0], b_cols.shape[1], float(beta), _fp(c0), _fp(out), m,
                                             threads))
        return out

    def fill_block(self, rows, cols, matrix_seed, brow, bcol) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        self.check(self.lib.ref_fill_block(_fp(out), rows, cols, matrix_seed & (2**64 - 1), brow, bcol))
        return out

    def fnv1a(self, arr) -> int:
        arr = np.ascontiguousarray(arr)
        return self.lib.ref_fnv1a(arr.ctypes.data, arr.nbytes)

    def owner(self, kind, gr, gc, br, bc, w, row, col) -> int:
        o = C.c_int()
        self.check(self.lib.ref_layout_owner(int(kind), gr, gc, br, bc, w, row, col, C.byref(o)))
        return o.value

    def layout_string(self, kind, gr, gc, br, bc, w) -> str:
        buf = C.create_string_buffer(4096)
        self.check(self.lib.ref_layout_string(int(kind), gr, gc, br, bc, w, buf, 4096))
        return buf.value.decode()

    def session(self, workers, root_seed, deterministic=True):
        return RefSession(self, workers, root_seed, deterministic)


_NP = {0: np.float16, 1: np.float32, 2: np.float64}


class RefSession:
    def __init__(self, ro: RefOracle, workers, root_seed, deterministic=True, _handle=None):
        self.ro = ro
        self.shapes = {}
        if _handle is not None:
            self.h = _handle
            return
        h = vp()
        ro.check(ro.lib.ref_session_create(workers, root_seed & (2**64 - 1), int(deterministic), C.byref(h)))
        self.h = h

    @classmethod
    def restore(cls, ro: RefOracle, path: str) -> "RefSession":
        h = vp()
        ro.check(ro.lib.ref_restore(path.encode(), C.byref(h)))
        return cls(ro, 0, 0, _handle=h)

    def describe(self, mid):
        """(version, replica_version, replicated, precision, seed, layout string)"""
        buf = (u64 * 6)()
        ls = C.create_string_buffer(4096)
        self.ro.check(self.ro.lib.ref_descriptor_full(self.h, mid, buf, ls, 4096))
        rows, cols = buf[5] >> 32, buf[5] & 0xFFFFFFFF
        self.shapes[mid] = (rows, cols, buf[3])
        return buf[0], buf[1], bool(buf[2]), buf[3], buf[4], ls.value.decode()

    def create_p(self, kind, gr, gc, br, bc, workers, precision, fill=1, host=None) -> int:
        out = u64()
        hp = None
        if host is not None:
            host = np.ascontiguousarray(host, _NP[precision])
            hp = C.c_void_p(host.ctypes.data)
        self.ro.check(self.ro.lib.ref_create_matrix_p(self.h, int(kind), gr, gc, br, bc, workers, precision,
                                                      fill, hp, C.byref(out)))
        self.shapes[out.value] = (gr, gc, precision)
        return out.value

    def gather_p(self, mid) -> np.ndarray:
        if mid not in self.shapes or len(self.shapes[mid]) < 3:
            self.describe(mid)
        gr, gc, p = self.shapes[mid]
        out = np.empty((gr, gc), _NP[p])
        self.ro.check(self.ro.lib.ref_gather_bytes(self.h, mid, C.c_void_p(out.ctypes.data), out.nbytes))
        return out

    def update_block(self, mid, row, col, data):
        gr, gc, p = self.shapes[mid]
        data = np.ascontiguousarray(data, _NP[p])
        self.ro.check(self.ro.lib.ref_update_block(self.h, mid, row, col, p, C.c_void_p(data.ctypes.data),
                                                   data.shape[0], data.shape[1]))

    def reshape(self, src, kind, gr, gc, br, bc, workers, precision) -> int:
        out = u64()
        self.ro.check(self.ro.lib.ref_reshape(self.h, src, int(kind), gr, gc, br, bc, workers, precision,
                                              C.byref(out)))
        self.shapes[out.value] = (gr, gc, precision)
        return out.value

    def add_row_col_sum(self, mid, axis, deterministic=True) -> int:
        out = u64()
        self.ro.check(self.ro.lib.ref_add_row_col_sum(self.h, mid, axis, int(deterministic), C.byref(out)))
        self.describe(out.value)
        return out.value

    def replicate(self, mid, enable=True):
        self.ro.check(self.ro.lib.ref_replicate(self.h, mid, int(enable)))

    def replica_read(self, mid, reader) -> np.ndarray:
        if len(self.shapes.get(mid, ())) < 3:
            self.describe(mid)
        gr, gc, p = self.shapes[mid]
        out = np.empty((gr, gc), _NP[p])
        self.ro.check(self.ro.lib.ref_replica_read(self.h, mid, reader, C.c_void_p(out.ctypes.data), out.nbytes))
        return out

    def checkpoint(self, path):
        self.ro.check(self.ro.lib.ref_checkpoint(self.h, path.encode()))

    def close(self):
        if self.h:
            self.ro.lib.ref_session_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def create(self, kind, gr, gc, br, bc, workers, fill=1, host=None) -> int:
        out = u64()
        hp = _fp(np.ascontiguousarray(host, np.float32)) if host is not None else None
        self.ro.check(self.ro.lib.ref_create_matrix(self.h, int(kind), gr, gc, br, bc, workers, fill, hp,
                                                    C.byref(out)))
        self.shapes[out.value] = (gr, gc)
        return out.value

    def gather(self, mid) -> np.ndarray:
        gr, gc = self.shapes[mid]
        out = np.empty((gr, gc), np.float32)
        self.ro.check(self.ro.lib.ref_gather(self.h, mid, _fp(out), out.size))
        return out

    def scatter(self, mid, host):
        host = np.ascontiguousarray(host, np.float32)
        self.ro.check(self.ro.lib.ref_scatter(self.h, mid, _fp(host), host.shape[0], host.shape[1]))

    def general_gemm(self, alpha, a, b, beta, c, ta=False, tb=False) -> int:
        return self.ro.lib.ref_general_gemm(self.h, alpha, a, b, beta, c, int(ta), int(tb))

    def cyclic_gemm(self, alpha, a, b, beta, c, ta=False, tb=False, cache_a=False) -> int:
        return self.ro.lib.ref_cyclic_gemm(self.h, alpha, a, b, beta, c, int(ta), int(tb), int(cache_a))

    def cached_backward_gemm(self, w, dy, dx) -> int:
        return self.ro.lib.ref_cached_backward_gemm(self.h, w, dy, dx)

    def broadcast_gemm_reference(self, alpha, a, b, beta, c, ta=False, tb=False) -> int:
        return self.ro.lib.ref_broadcast_gemm(self.h, alpha, a, b, beta, c, int(ta), int(tb))

    def trace_records(self, start=0):
        """trace() records from index `start`: dicts {src, dst, bytes, op}."""
        cnt = C.c_int()
        self.ro.check(self.ro.lib.ref_trace_records(self.h, start, None, None, 0, C.byref(cnt)))
        n = cnt.value
        out = (i64 * (3 * max(n, 1)))()
        tags = C.create_string_buffer(48 * max(n, 1))
        self.ro.check(self.ro.lib.ref_trace_records(self.h, start, out, tags, n, C.byref(cnt)))
        return [{"src": out[3 * i], "dst": out[3 * i + 1], "bytes": out[3 * i + 2],
                 "op": tags.raw[48 * i:48 * (i + 1)].split(b"\0", 1)[0].decode()} for i in range(n)]

    def version(self, mid) -> int:
        v, s = u64(), u64()
        self.ro.check(self.ro.lib.ref_descriptor(self.h, mid, C.byref(v), C.byref(s)))
        return v.value

    def pool_stats(self, w):
        buf = (u64 * 5)()
        self.ro.check(self.ro.lib.ref_pool_stats(self.h, w, buf))
        return list(buf)

    def transfers(self):
        t, b = u64(), u64()
        self.ro.check(self.ro.lib.ref_trace_count(self.h, C.byref(t), C.byref(b)))
        return t.value, b.value
