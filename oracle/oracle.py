"""ctypes bindings for the parity checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module. The product package
(paper_2408_04093_b200) never does.

* ``Oracle``    -- oracle/liboracle.so, the C restatement of the reference
                   decode path (oracle/treedec_oracle.c).
* ``Reference`` -- oracle/_ref/libtreedec_ref.so, the reference's own
                   proj/core sources compiled by oracle/Makefile plus the
                   C-ABI wrapper oracle/ref_shim.cpp.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtreedec_ref.so")
REF_SRC = "/root/reference/proj/core"

F64, F32, BF16 = 0, 1, 2
TREE_BINARY, RING, HIER = 0, 1, 2
DTYPE_CODES = {"f64": F64, "f32": F32, "bf16": BF16}

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_c_double_p)


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (always) and oracle/_ref (when /root/reference exists)."""
    targets = ["all"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
        product = os.path.join(os.path.dirname(HERE), "paper_2408_04093_b200", "libtreedec_b200.so")
        if os.path.exists(product):
            targets.append("shim")  # the C++ drop-in check (tests/cpp/shim_parity.cpp)
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        lib = ctypes.CDLL(path)
        lib.orc_mix64.restype = ctypes.c_uint64
        lib.orc_mix64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.orc_uniform01.restype = ctypes.c_double
        lib.orc_uniform01.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.orc_round.restype = ctypes.c_double
        lib.orc_round.argtypes = [ctypes.c_double, ctypes.c_int]
        lib.orc_lse_combine.restype = ctypes.c_double
        lib.orc_lse_combine.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.orc_seeded_fill.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, _i64, _i64,
                                        _c_double_p]
        lib.orc_chunk_extents.argtypes = [_i64, ctypes.c_int, _c_i64_p]
        lib.orc_chunk_partial.argtypes = ([_c_double_p] * 3 + [_i64] * 6 + [_i64, ctypes.c_double,
                                          ctypes.c_int, ctypes.c_int] + [_c_double_p] * 3)
        lib.orc_combine_pair.argtypes = [_c_double_p] * 6 + [_i64, _i64, ctypes.c_int] + [_c_double_p] * 3
        lib.orc_combine_partials.argtypes = [ctypes.c_int, _c_double_p, _c_double_p, _i64, _i64,
                                             ctypes.c_int, _c_double_p]
        lib.orc_partial_to_numerator.argtypes = [_c_double_p] * 3 + [_i64, _i64, ctypes.c_int] + [_c_double_p] * 2
        lib.orc_schedule_rounds.argtypes = [ctypes.c_int] * 3 + [ctypes.POINTER(ctypes.c_int)] * 2
        lib.orc_tree_decode.argtypes = ([_c_double_p] * 3 + [_i64] * 5 + [ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_int, _c_double_p])
        lib.orc_ring_decode.argtypes = ([_c_double_p] * 3 + [_i64] * 5 + [ctypes.c_int, ctypes.c_double,
                                        ctypes.c_int, ctypes.c_int, _c_double_p])
        lib.orc_attention_naive.argtypes = ([_c_double_p] * 3 + [_i64] * 5 + [ctypes.c_double, ctypes.c_int,
                                            ctypes.c_int, _c_double_p])
        lib.orc_energy_forward_parallel.argtypes = ([_c_double_p] * 4 + [_i64] * 5 + [ctypes.c_int, ctypes.c_int]
                                                    + [_c_double_p] * 3)
        lib.orc_energy_grad_parallel.argtypes = ([_c_double_p] * 5 + [_i64] * 5 + [ctypes.c_int, ctypes.c_int,
                                                 _c_double_p])
        self.lib = lib

    # -- numerics ---------------------------------------------------------
    def mix64(self, seed: int, counter: int) -> int:
        return int(self.lib.orc_mix64(seed, counter))

    def round(self, x: float, dtype: int) -> float:
        return float(self.lib.orc_round(float(x), dtype))

    def seeded(self, seed: int, n: int, dtype: int = F64, scale: float = 1.0, offset: int = 0) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        rc = self.lib.orc_seeded_fill(seed, scale, dtype, offset, n, _dp(out))
        if rc != 0:
            raise ValueError("seeded_random_tensor: scale must be positive")
        return out

    def chunk_extents(self, n: int, p: int) -> list[int]:
        out = np.zeros(max(p, 1), dtype=np.int64)
        if self.lib.orc_chunk_extents(n, p, out.ctypes.data_as(_c_i64_p)) != 0:
            raise ValueError("chunk_extents: bad arguments")
        return [int(x) for x in out[:p]]

    def schedule_rounds(self, strategy: int, nodes: int, gpus: int) -> tuple[int, int]:
        r, t = ctypes.c_int(), ctypes.c_int()
        if self.lib.orc_schedule_rounds(strategy, nodes, gpus, ctypes.byref(r), ctypes.byref(t)) != 0:
            raise ValueError("bad topology")
        return r.value, t.value

    # -- attention --------------------------------------------------------
    def chunk_partial(self, q, k, v, start, length, scale=1.0, dtype=F64, nthreads=1):
        b, n_q, d = q.shape
        _, n_kv, seq, _ = k.shape
        rows = b * n_q
        m = np.empty(rows); lse = np.empty(rows); out = np.empty((b, n_q, d))
        rc = self.lib.orc_chunk_partial(_dp(q), _dp(k), _dp(v), b, n_q, n_kv, seq, start, length, d,
                                        scale, dtype, nthreads, _dp(m), _dp(lse), _dp(out))
        if rc != 0:
            raise ValueError("chunk_partial: bad arguments")
        return m.reshape(b, n_q), lse.reshape(b, n_q), out

    def combine_partials(self, lse: np.ndarray, out: np.ndarray, dtype=F64) -> np.ndarray:
        P = lse.shape[0]
        rows = int(np.prod(lse.shape[1:]))
        d = out.shape[-1]
        lse = np.ascontiguousarray(lse, dtype=np.float64)
        out = np.ascontiguousarray(out, dtype=np.float64)
        res = np.empty(rows * d)
        if self.lib.orc_combine_partials(P, _dp(lse), _dp(out), rows, d, dtype, _dp(res)) != 0:
            raise ValueError("combine_partials: no keys attended")
        return res.reshape(out.shape[1:])

    def tree_decode(self, q, k, v, p, strategy=HIER, scale=1.0, dtype=F64, nthreads=1):
        b, n_q, d = q.shape
        _, n_kv, seq, _ = k.shape
        out = np.empty((b, n_q, d))
        rc = self.lib.orc_tree_decode(_dp(q), _dp(k), _dp(v), b, n_q, n_kv, seq, d, p, strategy,
                                      scale, dtype, nthreads, _dp(out))
        if rc != 0:
            raise ValueError(f"tree_decode: invalid arguments (rc={rc})")
        return out

    def ring_decode(self, q, k, v, p, scale=1.0, dtype=F64, nthreads=1):
        b, n_q, d = q.shape
        _, n_kv, seq, _ = k.shape
        out = np.empty((b, n_q, d))
        rc = self.lib.orc_ring_decode(_dp(q), _dp(k), _dp(v), b, n_q, n_kv, seq, d, p, scale,
                                      dtype, nthreads, _dp(out))
        if rc != 0:
            raise ValueError(f"ring_decode: invalid arguments (rc={rc})")
        return out

    # -- energy formulation (energy.cpp:152-259) ---------------------------
    def energy_forward_parallel(self, q, k, v, source, chunks, dtype=F64):
        """q, source [b, h, nq, d] (source None: zero), k, v [b, h, n, d] ->
        (value, row_max, shifted_lse), each [b, h, nq]."""
        b, h, nq, d = q.shape
        n = k.shape[2]
        value, rmax, sh = (np.empty((b, h, nq)) for _ in range(3))
        src = None if source is None else np.ascontiguousarray(source, dtype=np.float64)
        rc = self.lib.orc_energy_forward_parallel(_dp(np.ascontiguousarray(q)), _dp(np.ascontiguousarray(k)),
                                                  _dp(np.ascontiguousarray(v)), None if src is None else _dp(src),
                                                  b, h, nq, n, d, chunks, dtype, _dp(value), _dp(rmax), _dp(sh))
        if rc != 0:
            raise ValueError("energy_forward_parallel: need 1 <= chunks <= N")
        return value, rmax, sh

    def energy_grad_parallel(self, q, k, v, row_max, shifted, chunks, dtype=F64):
        b, h, nq, d = q.shape
        n = k.shape[2]
        grad = np.empty((b, h, nq, d))
        rc = self.lib.orc_energy_grad_parallel(_dp(np.ascontiguousarray(q)), _dp(np.ascontiguousarray(k)),
                                               _dp(np.ascontiguousarray(v)), _dp(np.ascontiguousarray(row_max)),
                                               _dp(np.ascontiguousarray(shifted)), b, h, nq, n, d, chunks, dtype,
                                               _dp(grad))
        if rc != 0:
            raise ValueError("energy_grad_parallel: need 1 <= chunks <= N")
        return grad

    def attention_naive(self, q, k, v, scale=1.0, dtype=F64, nthreads=1):
        b, n_q, d = q.shape
        _, n_kv, seq, _ = k.shape
        out = np.empty((b, n_q, d))
        if self.lib.orc_attention_naive(_dp(q), _dp(k), _dp(v), b, n_q, n_kv, seq, d, scale, dtype,
                                        nthreads, _dp(out)) != 0:
            raise ValueError("attention_naive: empty key range")
        return out


class Reference:
    """The reference library itself (oracle/_ref/libtreedec_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = ctypes.CDLL(path)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_mix64.restype = ctypes.c_uint64
        lib.ref_mix64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.ref_round.restype = ctypes.c_double
        lib.ref_round.argtypes = [ctypes.c_double, ctypes.c_int]
        lib.ref_seeded_values.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, _i64, _c_double_p]
        lib.ref_chunk_extents.argtypes = [_i64, ctypes.c_int, _c_i64_p]
        lib.ref_chunk_partial.argtypes = [_c_double_p] * 3 + [_i64] * 4 + [ctypes.c_double, ctypes.c_int] + [_c_double_p] * 3
        lib.ref_combine_partials.argtypes = [ctypes.c_int, _c_double_p, _c_double_p, _i64, _i64, ctypes.c_int, _c_double_p]
        lib.ref_prepare.restype = ctypes.c_void_p
        lib.ref_prepare.argtypes = [_c_double_p] * 3 + [_i64] * 5 + [ctypes.c_int, ctypes.c_int]
        lib.ref_release.argtypes = [ctypes.c_void_p]
        lib.ref_energy_forward_parallel.argtypes = ([_c_double_p] * 4 + [_i64] * 5 + [ctypes.c_int, ctypes.c_int]
                                                    + [_c_double_p] * 3)
        lib.ref_energy_grad_parallel.argtypes = ([_c_double_p] * 6 + [_i64] * 5 + [ctypes.c_int, ctypes.c_int,
                                                 _c_double_p])
        lib.ref_decode.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                   _i64, _i64, ctypes.c_int, _c_double_p, _c_double_p, _c_double_p]
        self.lib = lib

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def mix64(self, seed: int, counter: int) -> int:
        return int(self.lib.ref_mix64(seed, counter))

    def round(self, x: float, dtype: int) -> float:
        return float(self.lib.ref_round(float(x), dtype))

    def seeded(self, seed: int, n: int, dtype: int = F64, scale: float = 1.0) -> np.ndarray:
        out = np.empty(n)
        if self.lib.ref_seeded_values(seed, scale, dtype, n, _dp(out)) != 0:
            raise ValueError(self.error())
        return out

    def chunk_extents(self, n: int, p: int) -> list[int]:
        out = np.zeros(max(p, 1), dtype=np.int64)
        if self.lib.ref_chunk_extents(n, p, out.ctypes.data_as(_c_i64_p)) != 0:
            raise ValueError(self.error())
        return [int(x) for x in out[:p]]

    def chunk_partial(self, q, k, v, scale=1.0, dtype=F64):
        """MHA only: q [b,h,d], k/v [b,h,t,d]."""
        b, h, d = q.shape
        t = k.shape[2]
        m = np.empty(b * h); lse = np.empty(b * h); out = np.empty((b, h, d))
        if self.lib.ref_chunk_partial(_dp(q), _dp(k), _dp(v), b, h, t, d, scale, dtype, _dp(m), _dp(lse), _dp(out)) != 0:
            raise ValueError(self.error())
        return m.reshape(b, h), lse.reshape(b, h), out

    def combine_partials(self, lse, out, dtype=F64):
        P = lse.shape[0]
        rows = int(np.prod(lse.shape[1:]))
        d = out.shape[-1]
        lse = np.ascontiguousarray(lse, dtype=np.float64)
        out = np.ascontiguousarray(out, dtype=np.float64)
        res = np.empty(rows * d)
        if self.lib.ref_combine_partials(P, _dp(lse), _dp(out), rows, d, dtype, _dp(res)) != 0:
            raise ValueError(self.error())
        return res.reshape(out.shape[1:])

    def prepare(self, q, k, v, p, dtype=F64):
        b, n_q, d = q.shape
        _, n_kv, seq, _ = k.shape
        h = self.lib.ref_prepare(_dp(q), _dp(k), _dp(v), b, n_q, n_kv, seq, d, p, dtype)
        if not h:
            raise ValueError(self.error())
        return PreparedRef(self, h, b * n_q, d, (b, n_q, d))

    def energy_forward_parallel(self, q, k, v, source, chunks, dtype=F64):
        b, h, nq, d = q.shape
        n = k.shape[2]
        value, rmax, sh = (np.empty((b, h, nq)) for _ in range(3))
        src = None if source is None else np.ascontiguousarray(source, dtype=np.float64)
        rc = self.lib.ref_energy_forward_parallel(_dp(np.ascontiguousarray(q)), _dp(np.ascontiguousarray(k)),
                                                  _dp(np.ascontiguousarray(v)), None if src is None else _dp(src),
                                                  b, h, nq, n, d, chunks, dtype, _dp(value), _dp(rmax), _dp(sh))
        if rc != 0:
            raise ValueError(self.error())
        return value, rmax, sh

    def energy_grad_parallel(self, q, k, v, value, row_max, shifted, chunks, dtype=F64):
        b, h, nq, d = q.shape
        n = k.shape[2]
        grad = np.empty((b, h, nq, d))
        rc = self.lib.ref_energy_grad_parallel(_dp(np.ascontiguousarray(q)), _dp(np.ascontiguousarray(k)),
                                               _dp(np.ascontiguousarray(v)), _dp(np.ascontiguousarray(value)),
                                               _dp(np.ascontiguousarray(row_max)), _dp(np.ascontiguousarray(shifted)),
                                               b, h, nq, n, d, chunks, dtype, _dp(grad))
        if rc != 0:
            raise ValueError(self.error())
        return grad

    def tree_decode(self, q, k, v, p, strategy=HIER, scale=1.0, dtype=F64, parallel=False):
        with self.prepare(q, k, v, p, dtype) as pr:
            return pr.decode(0, strategy, scale, parallel)[0]

    def ring_decode(self, q, k, v, p, scale=1.0, dtype=F64, parallel=False):
        with self.prepare(q, k, v, p, dtype) as pr:
            return pr.decode(1, HIER, scale, parallel)[0]


class PreparedRef:
    def __init__(self, ref: Reference, handle, rows, d, shape):
        self.ref, self.handle, self.rows, self.d, self.shape = ref, handle, rows, d, shape

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def close(self):
        if self.handle:
            self.ref.lib.ref_release(self.handle)
            self.handle = None

    def decode(self, algo, strategy=HIER, scale=1.0, parallel=False, row0=0, row1=None, nthreads=1):
        """Returns (out, seconds, counters); out covers rows [row0, row1)."""
        row1 = self.rows if row1 is None else row1
        out = np.empty((row1 - row0) * self.d)
        secs = ctypes.c_double()
        counters = np.zeros(4)
        rc = self.ref.lib.ref_decode(self.handle, algo, strategy, scale, int(parallel), row0, row1, nthreads, _dp(out),
                                     ctypes.byref(secs), _dp(counters))
        if rc != 0:
            raise ValueError(self.ref.error())
        if row0 == 0 and row1 == self.rows:
            out = out.reshape(self.shape)
        return out, secs.value, counters
