"""ctypes bindings to the CHECKERS -- TEST INFRASTRUCTURE ONLY.

Two libraries live under ``oracle/``:

* ``liboracle.so``          -- the plain-C restatement (``qtn_oracle.c``) of the
  reference's naive bucket contraction / ``contract_network`` / state vector.
* ``_ref/libqtnsim_ref.so`` -- the UNMODIFIED reference (``/root/reference/proj``)
  compiled by ``oracle/Makefile`` plus the marshalling shim ``ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs may import this module.  The product package
(``paper_2204_06045_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqtnsim_ref.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")

BACKENDS = {"naive": 0, "matmul": 1, "mixed": 2, "scale": 3}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# --------------------------------------------------------------- C restatement
_olib = None


def oracle_lib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = C.CDLL(ORACLE_SO)
        lib.qo_last_error.restype = C.c_char_p
        lib.qo_contract_bucket.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.c_int, _i32p,
                                           _i32p, _f64p, C.c_int64]
        lib.qo_contract_network.argtypes = [C.c_int, _i32p, _f64p, C.c_int, _f64p, _i32p,
                                            _i32p, C.c_int, C.POINTER(C.c_int),
                                            C.POINTER(C.c_uint64)]
        lib.qo_statevector_energy.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p,
                                              C.POINTER(C.c_double)]
        _olib = lib
    return _olib


def _flatten_bucket(tensors: Sequence[Tuple[Sequence[int], np.ndarray]]):
    ranks = np.array([len(v) for v, _ in tensors], dtype=np.int32)
    vars_ = np.array([x for v, _ in tensors for x in v], dtype=np.int32)
    if vars_.size == 0:
        vars_ = np.zeros(1, dtype=np.int32)
    data = np.concatenate([np.ascontiguousarray(d, dtype=np.complex128).view(np.float64)
                           for _, d in tensors]) if tensors else np.zeros(2)
    return ranks, vars_, np.ascontiguousarray(data)


def oracle_contract_bucket(tensors, sum_vars):
    """NaiveBackend::contract restated in C. tensors: [(vars, complex128 array)]."""
    lib = oracle_lib()
    ranks, vars_, data = _flatten_bucket(tensors)
    allv = sorted({x for v, _ in tensors for x in v})
    cap = 1 << max(len(allv), 0)
    out_vars = np.zeros(max(len(allv), 1), dtype=np.int32)
    out = np.zeros(2 * cap, dtype=np.float64)
    sv = np.array(list(sum_vars) or [0], dtype=np.int32)
    r = lib.qo_contract_bucket(len(tensors), ranks if ranks.size else np.zeros(1, np.int32),
                               vars_, data, len(sum_vars), sv, out_vars, out, cap)
    if r < 0:
        raise OracleError(-r, lib.qo_last_error().decode())
    return [int(x) for x in out_vars[:r]], out[: 2 << r].view(np.complex128).copy()


def oracle_contract_network(n_buckets: int, ints: np.ndarray, data: np.ndarray,
                            max_result_width: int = 30):
    """contract_network restated in C over a flattened schedule."""
    lib = oracle_lib()
    sc = np.zeros(2, dtype=np.float64)
    cap = max(n_buckets, 1)
    seq = np.zeros(cap, dtype=np.int32)
    wid = np.zeros(cap, dtype=np.int32)
    nrec = C.c_int(0)
    peak = C.c_uint64(0)
    st = lib.qo_contract_network(n_buckets, np.ascontiguousarray(ints, dtype=np.int32),
                                 np.ascontiguousarray(data, dtype=np.float64),
                                 max_result_width, sc, seq, wid, cap, C.byref(nrec),
                                 C.byref(peak))
    if st != 0:
        raise OracleError(st, lib.qo_last_error().decode())
    n = nrec.value
    return complex(sc[0], sc[1]), seq[:n].copy(), wid[:n].copy(), peak.value


def oracle_statevector_energy(n, edges, gammas, betas) -> float:
    lib = oracle_lib()
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1))
    out = C.c_double(0.0)
    st = lib.qo_statevector_energy(n, len(e) // 2, e, len(gammas),
                                   np.asarray(gammas, dtype=np.float64),
                                   np.asarray(betas, dtype=np.float64), C.byref(out))
    if st != 0:
        raise OracleError(st, lib.qo_last_error().decode())
    return out.value


# --------------------------------------------------------------- the reference
_rlib = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _rlib
    if _rlib is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_random_regular.argtypes = [C.c_int, C.c_int, C.c_uint64, _i32p, C.c_int]
        lib.ref_energy.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p, C.c_int,
                                   C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64)]
        lib.ref_edge_terms.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                       _f64p, C.POINTER(C.c_double)]
        lib.ref_statevector_energy.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p,
                                               C.POINTER(C.c_double)]
        lib.ref_edge_schedule.restype = C.c_long
        lib.ref_edge_schedule.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p,
                                          C.c_int, C.c_int, _i32p, C.c_long, _f64p, C.c_long,
                                          C.POINTER(C.c_long), C.POINTER(C.c_int)]
        lib.ref_simulate_widths.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p,
                                            C.c_int, C.c_int, _i32p, C.c_int]
        lib.ref_merge_counts.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f64p, _f64p, C.c_int,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_contract_bucket.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i32p, _f64p,
                                            C.c_int, _i32p, _i32p, _f64p, C.c_long]
        lib.ref_contract_bucket_capped.argtypes = [C.c_int, _i32p, _i32p, C.c_int, _i32p,
                                                   C.c_int]
        lib.ref_read_timing_csv.argtypes = [C.c_char_p, C.POINTER(C.c_long), C.POINTER(C.c_long),
                                            C.POINTER(C.c_double)]
        _rlib = lib
    return _rlib


def ref_read_timing_csv(text: str):
    """The reference's read_timing_csv on `text`: (n_records, sum width, sum ops)."""
    n, w, o = C.c_long(0), C.c_long(0), C.c_double(0)
    code = ref_lib().ref_read_timing_csv(text.encode(), C.byref(n), C.byref(w), C.byref(o))
    if code:
        _ref_err(code)
    return n.value, w.value, o.value


def _ref_err(code):
    raise OracleError(code, ref_lib().ref_last_error().decode())


def ref_random_regular(n: int, d: int, seed: int) -> np.ndarray:
    lib = ref_lib()
    buf = np.zeros(n * d + 2, dtype=np.int32)
    m = lib.ref_random_regular(n, d, seed, buf, len(buf) // 2)
    if m < 0:
        _ref_err(-m)
    return buf[: 2 * m].reshape(m, 2).copy()


def _g(edges):
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1))
    return e, len(e) // 2


def ref_energy(n, edges, gammas, betas, backend="matmul", threshold=15, merged=False,
               max_width=30, jobs=1):
    """energy_expectation (engine.cpp:503-563). Returns (energy, wall_s, n_records, peak)."""
    lib = ref_lib()
    e, m = _g(edges)
    en, wall = C.c_double(0), C.c_double(0)
    nrec, peak = C.c_uint64(0), C.c_uint64(0)
    st = lib.ref_energy(n, m, e, len(gammas), np.asarray(gammas, np.float64),
                        np.asarray(betas, np.float64), BACKENDS[backend], threshold,
                        int(merged), max_width, jobs, C.byref(en), C.byref(wall),
                        C.byref(nrec), C.byref(peak))
    if st != 0:
        _ref_err(st)
    return en.value, wall.value, nrec.value, peak.value


def ref_edge_terms(n, edges, gammas, betas, backend="naive", threshold=15, merged=False,
                   max_width=30, jobs=1, select: Optional[Sequence[int]] = None):
    """Per-edge e_jk (complex) via edge_schedule + contract_network."""
    lib = ref_lib()
    e, m = _g(edges)
    sel = np.arange(m, dtype=np.int32) if select is None else np.asarray(select, np.int32)
    out = np.zeros(2 * len(sel), dtype=np.float64)
    wall = C.c_double(0)
    st = lib.ref_edge_terms(n, m, e, len(gammas), np.asarray(gammas, np.float64),
                            np.asarray(betas, np.float64), BACKENDS[backend], threshold,
                            int(merged), max_width, jobs, len(sel), sel, out, C.byref(wall))
    if st != 0:
        _ref_err(st)
    return out.view(np.complex128).copy(), wall.value


def ref_statevector_energy(n, edges, gammas, betas) -> float:
    lib = ref_lib()
    e, m = _g(edges)
    out = C.c_double(0)
    st = lib.ref_statevector_energy(n, m, e, len(gammas), np.asarray(gammas, np.float64),
                                    np.asarray(betas, np.float64), C.byref(out))
    if st != 0:
        _ref_err(st)
    return out.value


def ref_edge_schedule(n, edges, gammas, betas, edge_index, merged=False):
    """Flattened schedule (ints, data, n_buckets) in the shared format."""
    lib = ref_lib()
    e, m = _g(edges)
    cap = 1 << 16
    while True:
        ints = np.zeros(cap, dtype=np.int32)
        data = np.zeros(cap, dtype=np.float64)
        dlen = C.c_long(0)
        nb = C.c_int(0)
        r = lib.ref_edge_schedule(n, m, e, len(gammas), np.asarray(gammas, np.float64),
                                  np.asarray(betas, np.float64), edge_index, int(merged),
                                  ints, cap, data, cap, C.byref(dlen), C.byref(nb))
        if r == -1:
            raise OracleError(99, lib.ref_last_error().decode())
        if r < 0:
            cap = int(-r) + 16
            continue
        return ints[:r].copy(), data[: dlen.value].copy(), nb.value


def ref_merge_counts(n, edges, gammas, betas, edge_index):
    """(merges_applied, merges_skipped) of one edge's merged schedule."""
    lib = ref_lib()
    e, m = _g(edges)
    ap, sk = C.c_int(0), C.c_int(0)
    st = lib.ref_merge_counts(n, m, e, len(gammas), np.asarray(gammas, np.float64),
                              np.asarray(betas, np.float64), edge_index, C.byref(ap),
                              C.byref(sk))
    if st != 0:
        _ref_err(st)
    return ap.value, sk.value


def ref_simulate_widths(n, edges, gammas, betas, edge_index, merged=False):
    lib = ref_lib()
    e, m = _g(edges)
    buf = np.zeros(1 << 16, dtype=np.int32)
    r = lib.ref_simulate_widths(n, m, e, len(gammas), np.asarray(gammas, np.float64),
                                np.asarray(betas, np.float64), edge_index, int(merged), buf,
                                len(buf))
    if r < 0:
        _ref_err(-r)
    return buf[:r].copy()


def ref_contract_bucket(tensors, sum_vars, backend="naive", threshold=15):
    lib = ref_lib()
    ranks, vars_, data = _flatten_bucket(tensors)
    allv = sorted({x for v, _ in tensors for x in v})
    cap = 1 << len(allv)
    out_vars = np.zeros(max(len(allv), 1), dtype=np.int32)
    out = np.zeros(2 * cap, dtype=np.float64)
    sv = np.array(list(sum_vars) or [0], dtype=np.int32)
    r = lib.ref_contract_bucket(BACKENDS[backend], threshold, len(tensors),
                                ranks if ranks.size else np.zeros(1, np.int32), vars_, data,
                                len(sum_vars), sv, out_vars, out, cap)
    if r < 0:
        _ref_err(-r)
    return [int(x) for x in out_vars[:r]], out[: 2 << r].view(np.complex128).copy()


def ref_contract_bucket_capped(var_lists, sum_vars, max_width):
    """contract_bucket's cap check; returns (code, message)."""
    lib = ref_lib()
    ranks = np.array([len(v) for v in var_lists], dtype=np.int32)
    vars_ = np.array([x for v in var_lists for x in v] or [0], dtype=np.int32)
    sv = np.array(list(sum_vars) or [0], dtype=np.int32)
    st = lib.ref_contract_bucket_capped(len(var_lists), ranks, vars_, len(sum_vars), sv,
                                        max_width)
    return st, (lib.ref_last_error().decode() if st else "")


# ------------------------------------------------------------------ fingerprints
FNV_OFFSET = 14695981039346656037
FNV_PRIME = 1099511628211


def fnv1a_int64(values) -> int:
    """FNV-1a 64 over int64 little-endian values."""
    h = FNV_OFFSET
    for v in values:
        b = int(v) & 0xFFFFFFFFFFFFFFFF
        for _ in range(8):
            h ^= b & 0xFF
            h = (h * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
            b >>= 8
    return h


def parse_schedule(ints: np.ndarray, n_buckets: int):
    """Flattened schedule -> [(sum_vars, [tensor var lists])]."""
    out = []
    i = 0
    for _ in range(n_buckets):
        ns = int(ints[i]); i += 1
        sums = [int(x) for x in ints[i:i + ns]]; i += ns
        nt = int(ints[i]); i += 1
        ts = []
        for _ in range(nt):
            r = int(ints[i]); i += 1
            ts.append([int(x) for x in ints[i:i + r]]); i += r
        out.append((sums, ts))
    return out
