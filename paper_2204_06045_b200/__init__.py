"""B200-native bucket-elimination contraction for QAOA MaxCut energies.

A from-scratch sm_100a implementation of the hot path of the reference
``qtnsim`` (arXiv 2204.06045's QTensor re-implementation, /root/reference/proj):
the per-lightcone bucket elimination behind ``ContractionBackend`` /
``contract_network`` / ``energy_expectation``.  This module mirrors that
interface in Python (names, argument meaning and error types follow
proj/include/qtnsim/*.hpp) on top of the C ABI in include/qtng.h; all compute
runs in the native library ``libqtng.so`` (host planner in C++, kernels in
CUDA for sm_100a).  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._native import EnergyReport, PlanInfo, Record, lib

__all__ = [
    "InvalidInputError", "GenerationError", "ResourceError", "ScheduleError", "NumericalError",
    "CudaError", "Graph", "Edge", "Angles", "Tensor", "Bucket", "ContractionSchedule",
    "TimingRecord", "write_timing_csv", "read_timing_csv", "ContractionReport", "EnergyResult", "EngineConfig", "Context",
    "GpuBackend", "Plan", "make_graph", "random_regular", "edge_schedule", "simulate_widths",
    "edge_costs", "validate_energy", "contract_bucket", "contract_network", "energy_expectation",
    "default_context", "version", "statevector_energy",
]


# ------------------------------------------------------------------ errors
# proj/include/qtnsim/errors.hpp:8-36
class InvalidInputError(RuntimeError):
    pass


class GenerationError(RuntimeError):
    pass


class ResourceError(RuntimeError):
    pass


class ScheduleError(RuntimeError):
    pass


class NumericalError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRORS = {1: InvalidInputError, 2: ResourceError, 3: ScheduleError, 4: NumericalError,
           5: CudaError, 6: GenerationError}


def _check(status: int) -> None:
    if status:
        raise _ERRORS.get(status, RuntimeError)(lib.qtng_last_error().decode())


def kernel_launches() -> int:
    """Kernel launches the native library has issued (eager + graph replays)."""
    return int(lib.qtng_kernel_launches())


def version() -> str:
    return lib.qtng_version().decode()


# ------------------------------------------------------------------ graph
@dataclass(frozen=True, order=True)
class Edge:
    u: int
    v: int


@dataclass
class Graph:
    """Undirected simple graph (graph.hpp:18-24); edges sorted, u < v."""

    n: int
    edges: np.ndarray  # (m, 2) int32

    @property
    def m(self) -> int:
        return int(self.edges.shape[0])

    def flat(self) -> np.ndarray:
        return np.ascontiguousarray(self.edges.reshape(-1), dtype=np.int32)

    def edge_list(self) -> List[Edge]:
        return [Edge(int(u), int(v)) for u, v in self.edges]


def make_graph(n: int, edges) -> Graph:
    """make_graph (graph.cpp:30-43): normalise endpoint order, sort, reject
    loops / out-of-range endpoints / duplicates."""
    if n < 0:
        raise InvalidInputError("vertex count must be non-negative")
    es = []
    for u, v in (tuple(e) for e in edges):
        u, v = int(u), int(v)
        if u > v:
            u, v = v, u
        if u == v:
            raise InvalidInputError(f"self-loop at vertex {u}")
        if u < 0 or v >= n:
            raise InvalidInputError(f"edge endpoint out of range: ({u}, {v})")
        es.append((u, v))
    es.sort()
    for a, b in zip(es, es[1:]):
        if a == b:
            raise InvalidInputError("duplicate edge")
    arr = np.array(es, dtype=np.int32).reshape(-1, 2)
    return Graph(n, arr)


def random_regular(n: int, d: int, seed: int) -> Graph:
    """random_regular (graph.cpp:45-76), identical edge set for a given seed."""
    buf = np.zeros(max(2, n * max(d, 0) + 2), dtype=np.int32)
    m = C.c_int(0)
    _check(lib.qtng_random_regular(n, d, seed, buf, len(buf) // 2, C.byref(m)))
    return Graph(n, buf[: 2 * m.value].reshape(-1, 2).copy())


# ------------------------------------------------------------------ angles / config
@dataclass
class Angles:
    """QAOA angles (circuit.hpp:14-20)."""

    gammas: Sequence[float]
    betas: Sequence[float]

    def depth(self) -> int:
        return len(self.gammas)

    def validate(self) -> None:
        if len(self.gammas) == 0 or len(self.gammas) != len(self.betas):
            raise InvalidInputError("angles: gammas and betas must have equal length p >= 1")
        if not all(np.isfinite(self.gammas)):
            raise InvalidInputError("angles: non-finite gamma")
        if not all(np.isfinite(self.betas)):
            raise InvalidInputError("angles: non-finite beta")

    def arrays(self):
        return (np.ascontiguousarray(self.gammas, dtype=np.float64),
                np.ascontiguousarray(self.betas, dtype=np.float64))


@dataclass
class EngineConfig:
    """EngineConfig (engine.hpp:16-20)."""

    max_result_width: int = 30
    # "c128" (default): bit-identical to the reference's naive backend;
    # "c64": complex64 arena and arithmetic (north_star tolerance 1e-5)
    dtype: str = "c128"

    def precision_bits(self) -> int:
        if self.dtype not in ("c128", "c64"):
            raise InvalidInputError("dtype must be 'c128' or 'c64'")
        return 128 if self.dtype == "c128" else 64

    @staticmethod
    def from_env() -> "EngineConfig":
        cfg = EngineConfig()
        v = os.environ.get("QTNSIM_MAX_WIDTH")
        if v is not None:
            try:
                cfg.max_result_width = int(v)
            except ValueError:
                cfg.max_result_width = 0  # std::atoi semantics
        return cfg


# ------------------------------------------------------------------ tensors / schedules
@dataclass
class Tensor:
    """Dense complex128 tensor over binary vars, first axis = MSB (tensor.hpp:13-25)."""

    label: str
    vars: List[int]
    data: np.ndarray

    def rank(self) -> int:
        return len(self.vars)


@dataclass
class Bucket:
    sum_vars: List[int]
    tensors: List[Tensor] = field(default_factory=list)


@dataclass
class ContractionSchedule:
    buckets: List[Bucket]
    merges_applied: int = 0
    merges_skipped: int = 0

    def flatten(self):
        ints: List[int] = []
        data = []
        for b in self.buckets:
            ints.append(len(b.sum_vars))
            ints.extend(int(v) for v in b.sum_vars)
            ints.append(len(b.tensors))
            for t in b.tensors:
                ints.append(len(t.vars))
                ints.extend(int(v) for v in t.vars)
                data.append(np.ascontiguousarray(t.data, dtype=np.complex128).view(np.float64))
        return (np.array(ints or [0], dtype=np.int32), len(ints),
                np.concatenate(data) if data else np.zeros(2))


@dataclass
class TimingRecord:
    """TimingRecord (engine.hpp:71-80)."""

    edge_u: int
    edge_v: int
    bucket_seq: int
    width: int
    backend: str
    elapsed_s: float
    ops: int
    flops_est: float


_CSV_HEADER = "edge_u,edge_v,bucket_seq,width,backend,elapsed_s,ops,flops_est"


def _fmt_g6(x: float) -> str:
    """std::ostream's default double formatting (%g, precision 6)."""
    return "%g" % x


def write_timing_csv(records: Sequence["TimingRecord"], f) -> None:
    """write_timing_csv (proj/src/engine.cpp:567-573): same header, field order
    and default stream formatting, so the reference's report tooling reads it."""
    f.write(_CSV_HEADER + "\n")
    for r in records:
        f.write(f"{r.edge_u},{r.edge_v},{r.bucket_seq},{r.width},{r.backend},"
                f"{_fmt_g6(r.elapsed_s)},{r.ops},{_fmt_g6(r.flops_est)}\n")


def read_timing_csv(f) -> List["TimingRecord"]:
    """read_timing_csv (proj/src/engine.cpp:575-601), same errors."""
    lines = f.read().split("\n")
    if not lines or lines == [""]:
        raise InvalidInputError("timing CSV: missing header")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        fields = line.split(",")
        if len(fields) < 8:
            raise InvalidInputError("timing CSV: short row: " + line)
        u, v, seq, w, backend, el, ops, fl = fields[:8]
        out.append(TimingRecord(int(u), int(v), int(seq), int(w), backend, float(el), int(ops),
                                float(fl)))
    return out


@dataclass
class ContractionReport:
    """ContractionReport (engine.hpp:82-88)."""

    scalar: complex
    records: List[TimingRecord]
    peak_tensor_bytes: int
    merges_applied: int = 0
    merges_skipped: int = 0


@dataclass
class EnergyResult:
    """EnergyResult (engine.hpp:136-139) plus the per-edge terms."""

    energy: float
    terms: np.ndarray  # complex e_jk per edge (edge order)
    report: Optional[ContractionReport] = None


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device's stream, HBM arena and staging buffers (qtng_ctx)."""

    def __init__(self, device: int = 0, arena_bytes: int = 0):
        h = C.c_void_p()
        _check(lib.qtng_create(device, arena_bytes, C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.qtng_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = {}
_ctx_lock = threading.Lock()


def default_context(device: Optional[int] = None) -> Context:
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0")) if "LOCAL_RANK" in os.environ else 0
    with _ctx_lock:
        if device not in _default_ctx:
            _default_ctx[device] = Context(device)
        return _default_ctx[device]


# ------------------------------------------------------------------ backend (drop-in)
def contract_bucket(bucket: Bucket, ctx: Optional[Context] = None) -> Tensor:
    """ContractionBackend::contract (engine.hpp:30) on the B200: sums
    bucket.sum_vars out of bucket.tensors; result axes ascending."""
    ctx = ctx or default_context()
    ranks = np.array([len(t.vars) for t in bucket.tensors] or [0], dtype=np.int32)
    vars_ = np.array([v for t in bucket.tensors for v in t.vars] or [0], dtype=np.int32)
    data = (np.concatenate([np.ascontiguousarray(t.data, dtype=np.complex128).view(np.float64)
                            for t in bucket.tensors]) if bucket.tensors else np.zeros(2))
    allv = {v for t in bucket.tensors for v in t.vars}
    cap = 1 << len(allv)
    out_vars = np.zeros(max(len(allv), 1), dtype=np.int32)
    out = np.zeros(2 * cap, dtype=np.float64)
    sv = np.array(list(bucket.sum_vars) or [0], dtype=np.int32)
    r = C.c_int(0)
    _check(lib.qtng_contract_bucket(ctx.handle, len(bucket.tensors), ranks, vars_,
                                    np.ascontiguousarray(data), len(bucket.sum_vars), sv,
                                    C.byref(r), out_vars, out, cap))
    k = r.value
    return Tensor("bucket_result", [int(v) for v in out_vars[:k]],
                  out[: 2 << k].view(np.complex128).copy())


class GpuBackend:
    """Drop-in for qtnsim::ContractionBackend (engine.hpp:22-31)."""

    def __init__(self, ctx: Optional[Context] = None):
        self._ctx = ctx

    @property
    def ctx(self) -> Context:
        return self._ctx or default_context()

    def name(self) -> str:
        return "b200"

    def select(self, width: int) -> "GpuBackend":
        return self

    def contract(self, bucket: Bucket) -> Tensor:
        return contract_bucket(bucket, self.ctx)


# ------------------------------------------------------------------ schedules
def _angles_arrays(angles: Angles):
    g, b = angles.arrays()
    return g, b


def edge_schedule(g: Graph, edge_index: int, angles: Angles,
                  merged: bool = False) -> ContractionSchedule:
    """edge_schedule (engine.cpp:493-501), built by the native host planner."""
    gam, bet = _angles_arrays(angles)
    n_ints, n_data, nb = C.c_int64(0), C.c_int64(0), C.c_int(0)
    probe_i = np.zeros(1, np.int32)
    probe_d = np.zeros(1, np.float64)
    merges = np.zeros(2, np.int32)
    _check(lib.qtng_edge_schedule(g.n, g.m, g.flat(), angles.depth(), gam, bet, edge_index,
                                  int(merged), probe_i, 0, probe_d, 0, C.byref(n_ints),
                                  C.byref(n_data), C.byref(nb), None))
    ints = np.zeros(max(1, n_ints.value), np.int32)
    data = np.zeros(max(1, n_data.value), np.float64)
    _check(lib.qtng_edge_schedule(g.n, g.m, g.flat(), angles.depth(), gam, bet, edge_index,
                                  int(merged), ints, len(ints), data, len(data),
                                  C.byref(n_ints), C.byref(n_data), C.byref(nb),
                                  merges.ctypes.data_as(C.c_void_p)))
    s = _parse_flat(ints[: n_ints.value], data[: n_data.value], nb.value)
    s.merges_applied, s.merges_skipped = int(merges[0]), int(merges[1])
    return s


def _parse_flat(ints, data, n_buckets) -> ContractionSchedule:
    cd = data.view(np.complex128)
    i = 0
    off = 0
    buckets = []
    for _ in range(n_buckets):
        ns = int(ints[i]); i += 1
        sums = [int(x) for x in ints[i:i + ns]]; i += ns
        nt = int(ints[i]); i += 1
        ts = []
        for _ in range(nt):
            r = int(ints[i]); i += 1
            vs = [int(x) for x in ints[i:i + r]]; i += r
            ts.append(Tensor("t", vs, cd[off:off + (1 << r)].copy()))
            off += 1 << r
        buckets.append(Bucket(sums, ts))
    return ContractionSchedule(buckets)


def merge_buckets(schedule: ContractionSchedule) -> ContractionSchedule:
    """merge_buckets (engine.cpp:306-358) of an explicit schedule: bucket A is
    folded into the first later bucket covering its kept vars when the
    schedule stays valid and no bucket grows past the widest one.  Tensors
    are moved, not copied; merges_applied / merges_skipped as the reference
    counts them."""
    ints, n_ints, _ = schedule.flatten()
    tensors = [t for b in schedule.buckets for t in b.tensors]
    n_out, nb = C.c_int64(0), C.c_int(0)
    merges = np.zeros(2, np.int32)
    _check(lib.qtng_merge_schedule(len(schedule.buckets), ints, n_ints, None, 0, C.byref(n_out),
                                   C.byref(nb), None))
    out = np.zeros(max(1, n_out.value), np.int32)
    _check(lib.qtng_merge_schedule(len(schedule.buckets), ints, n_ints,
                                   out.ctypes.data_as(C.c_void_p), len(out), C.byref(n_out),
                                   C.byref(nb), merges.ctypes.data_as(C.c_void_p)))
    buckets, i = [], 0
    for _ in range(nb.value):
        ns = int(out[i]); i += 1
        sums = [int(x) for x in out[i:i + ns]]; i += ns
        nt = int(out[i]); i += 1
        buckets.append(Bucket(sums, [tensors[int(k)] for k in out[i:i + nt]]))
        i += nt
    return ContractionSchedule(buckets, int(merges[0]), int(merges[1]))


def simulate_widths(g: Graph, edge_index: int, p: int, merged: bool = False) -> List[int]:
    """simulate_widths (engine.cpp:235-240) of one edge's schedule."""
    buf = np.zeros(1 << 16, dtype=np.int32)
    n = C.c_int(0)
    _check(lib.qtng_simulate_widths(g.n, g.m, g.flat(), p, edge_index, int(merged), buf,
                                    len(buf), C.byref(n)))
    return [int(x) for x in buf[: n.value]]


def edge_costs(g: Graph, p: int, merged: bool = False) -> np.ndarray:
    """Predicted algorithmic bytes per edge lightcone (sharding key)."""
    out = np.zeros(max(1, g.m), dtype=np.float64)
    _check(lib.qtng_edge_costs(g.n, g.m, g.flat(), p, int(merged), out))
    return out[: g.m]


def edge_work(g: Graph, p: int, merged: bool = False) -> np.ndarray:
    """Predicted device work per edge lightcone (complex products + adds of
    the reference loop): the multi-GPU sharding key."""
    out = np.zeros(max(1, g.m), dtype=np.float64)
    _check(lib.qtng_edge_work(g.n, g.m, g.flat(), p, int(merged), out))
    return out[: g.m]


def plan_dump(g: Graph, p: int, merged: bool = False, cfg: Optional[EngineConfig] = None,
              edges: Optional[Sequence[int]] = None) -> List[dict]:
    """Host-only description of the device program (one dict per device op,
    level-sorted): level, r, ns, nt, cb, recorded, width, inputs=[(rank,
    initial, src list)]."""
    cfg = cfg or EngineConfig()
    sel = None if edges is None else np.ascontiguousarray(edges, dtype=np.int32)
    k = g.m if sel is None else len(sel)
    sp = None if sel is None else sel.ctypes.data_as(C.c_void_p)
    n_ints, n_ops = C.c_int64(0), C.c_int(0)
    probe = np.zeros(1, np.int32)
    _check(lib.qtng_plan_dump(g.n, g.m, g.flat(), p, int(merged), cfg.max_result_width, k, sp,
                              probe, 0, C.byref(n_ints), C.byref(n_ops)))
    buf = np.zeros(max(1, n_ints.value), np.int32)
    _check(lib.qtng_plan_dump(g.n, g.m, g.flat(), p, int(merged), cfg.max_result_width, k, sp,
                              buf, len(buf), C.byref(n_ints), C.byref(n_ops)))
    out, i = [], 0
    for _ in range(n_ops.value):
        lv, r, ns, nt, cb, rec, w, outer = (int(x) for x in buf[i:i + 8])
        i += 8
        ins = []
        for _ in range(nt):
            rank, init = int(buf[i]), int(buf[i + 1])
            ins.append((rank, init, [int(x) for x in buf[i + 2:i + 2 + rank]]))
            i += 34
        out.append(dict(level=lv, r=r, ns=ns, nt=nt, cb=cb, recorded=rec, width=w, outer=outer,
                        inputs=ins))
    return out


def plan_stats(g: Graph, p: int, merged: bool = False, cfg: Optional[EngineConfig] = None,
               fuse: bool = True) -> PlanInfo:
    """Host-only: the PlanInfo Plan(g, p) would have (fuse=False: one device
    op per bucket, no fused-chain segments)."""
    cfg = cfg or EngineConfig()
    inf = PlanInfo()
    _check(lib.qtng_plan_stats(g.n, g.m, g.flat(), p, int(merged), cfg.max_result_width,
                               int(fuse), C.byref(inf)))
    return inf


def plan_segments(g: Graph, p: int, merged: bool = False,
                  cfg: Optional[EngineConfig] = None) -> List[dict]:
    """Host-only description of the fused-chain segments of Plan(g, p):
    level, L, ry, cy, nops, rb (paired rows' tile bit or None), rb2 (quad tiles:
    B's row bit, rb = A's; None otherwise),
    stages=[(nt, ns, main, [(rank, initial, codes)])]."""
    cfg = cfg or EngineConfig()
    n_ints = C.c_int64(0)
    probe = np.zeros(1, np.int32)
    _check(lib.qtng_plan_segments(g.n, g.m, g.flat(), p, int(merged), cfg.max_result_width,
                                  probe, 0, C.byref(n_ints)))
    buf = np.zeros(max(1, n_ints.value), np.int32)
    _check(lib.qtng_plan_segments(g.n, g.m, g.flat(), p, int(merged), cfg.max_result_width,
                                  buf, len(buf), C.byref(n_ints)))
    out, i = [], 0
    while i < n_ints.value:
        lv, L, ry, cy, nops, rb, rb2 = (int(x) for x in buf[i:i + 7])
        i += 7
        stages = []
        for _ in range(L):
            nt, ns, main = (int(x) for x in buf[i:i + 3])
            i += 3
            mem = []
            for _ in range(nt):
                rank, ini = int(buf[i]), int(buf[i + 1])
                mem.append((rank, ini, [int(x) for x in buf[i + 2:i + 2 + rank]]))
                i += 2 + rank
            stages.append((nt, ns, main, mem))
        out.append(dict(level=lv, L=L, ry=ry, cy=cy, nops=nops,
                        rb=None if rb == 0xff else rb, rb2=None if rb2 == 0xff else rb2,
                        stages=stages))
    return out


def statevector_energy(g: Graph, angles: Angles, cap: int = 24,
                       ctx: Optional[Context] = None):
    """The state-vector oracle on the device (run_ansatz + expectation_cost,
    proj/src/statevector.cpp:55-90): (energy, per-edge <Z_u Z_v>).  cap: the
    reference's qubit cap (default 24, StateVector::kDefaultCap); the device
    holds up to 33 qubits."""
    ctx = ctx or default_context()
    angles.validate()
    gam, bet = angles.arrays()
    e = C.c_double(0.0)
    zz = np.zeros(max(1, g.m), np.float64)
    _check(lib.qtng_statevector_energy(ctx.handle, g.n, g.m, g.flat(), angles.depth(), gam, bet,
                                       int(cap), C.byref(e), zz.ctypes.data_as(C.c_void_p)))
    return e.value, zz[: g.m]


def validate_energy(g: Graph, p: int, merged: bool = False,
                    cfg: Optional[EngineConfig] = None) -> None:
    """Host-only pre-flight of energy_expectation: raises the ScheduleError
    ("edge (u, v): contraction refused: ...") the reference would raise."""
    cfg = cfg or EngineConfig()
    _check(lib.qtng_validate_energy(g.n, g.m, g.flat(), p, int(merged), cfg.max_result_width))


def contract_network(schedule: ContractionSchedule, backend: Optional[GpuBackend] = None,
                     cfg: Optional[EngineConfig] = None) -> ContractionReport:
    """contract_network (engine.cpp:246-304) of a whole schedule on the device."""
    ctx = (backend.ctx if backend is not None else default_context())
    cfg = cfg or EngineConfig()
    ints, n_ints, data = schedule.flatten()
    n_b = len(schedule.buckets)
    recs = (Record * max(1, n_b))()
    nrec = C.c_int(0)
    peak = C.c_uint64(0)
    sc = np.zeros(2, np.float64)
    _check(lib.qtng_contract_schedule(ctx.handle, n_b, ints, n_ints, np.ascontiguousarray(data),
                                      cfg.max_result_width, sc, recs, len(recs), C.byref(nrec),
                                      C.byref(peak)))
    records = [TimingRecord(-1, -1, r.bucket_seq, r.width, "b200", r.elapsed_s, r.ops,
                            r.flops_est) for r in recs[: nrec.value]]
    return ContractionReport(complex(sc[0], sc[1]), records, peak.value)


def energy_expectation(g: Graph, angles: Angles, backend: Optional[GpuBackend] = None,
                       merged: bool = False, cfg: Optional[EngineConfig] = None,
                       edges: Optional[Sequence[int]] = None,
                       records: bool = False) -> EnergyResult:
    """energy_expectation (engine.cpp:503-563): <C> = |E|/2 - 1/2 sum_e Re e_jk,
    every lightcone contracted on the device in one level-batched program.
    With `edges` (a subset) the energy is NaN and the terms are the result.
    records=True also returns the TimingRecords in result.report."""
    angles.validate()
    ctx = backend.ctx if backend is not None else default_context()
    cfg = cfg or EngineConfig()
    gam, bet = _angles_arrays(angles)
    sel = None if edges is None else np.ascontiguousarray(edges, dtype=np.int32)
    k = g.m if sel is None else len(sel)
    terms = np.zeros(2 * max(1, k), np.float64)
    e = C.c_double(0)
    rep = EnergyReport()
    recs = None
    if records:
        # generous bound on the bucket count (the reference's lightcones hold
        # < 300 buckets at the benchmark sizes); re-run with the exact count
        # if it was not enough
        cap = 512 * max(1, k)
        recs = (Record * cap)()
        rep.records, rep.rec_cap = C.cast(recs, C.c_void_p), cap
    _check(lib.qtng_energy(ctx.handle, g.n, g.m, g.flat(), angles.depth(), gam, bet,
                           int(merged), cfg.max_result_width, cfg.precision_bits(), k,
                           None if sel is None else sel.ctypes.data_as(C.c_void_p),
                           C.byref(e), terms, C.byref(rep)))
    if records and rep.n_records > rep.rec_cap:
        recs = (Record * rep.n_records)()
        rep.records, rep.rec_cap = C.cast(recs, C.c_void_p), rep.n_records
        _check(lib.qtng_energy(ctx.handle, g.n, g.m, g.flat(), angles.depth(), gam, bet,
                               int(merged), cfg.max_result_width, cfg.precision_bits(), k,
                               None if sel is None else sel.ctypes.data_as(C.c_void_p),
                               C.byref(e), terms, C.byref(rep)))
    report = ContractionReport(
        complex(e.value, 0.0),
        [TimingRecord(r.edge_u, r.edge_v, r.bucket_seq, r.width, "b200", r.elapsed_s, r.ops,
                      r.flops_est) for r in recs[: rep.n_records]] if records else [],
        rep.peak_tensor_bytes, rep.merges_applied, rep.merges_skipped)
    return EnergyResult(e.value, terms[: 2 * k].view(np.complex128).copy(), report)


def fp64_peak(device: int = 0):
    """Measured FP64 rates of `device` (qtng_fp64_peak): (DMUL+DADD ops/s, DFMA flops/s)."""
    ma, fma = C.c_double(0), C.c_double(0)
    _check(lib.qtng_fp64_peak(int(device), C.byref(ma), C.byref(fma)))
    return ma.value, fma.value


def shard_edges(g: Graph, p: int, n_shards: int, merged: bool = False) -> np.ndarray:
    """The device (0..n_shards-1) energy_multi places each edge's lightcone on
    (LPT on the predicted work, host-only)."""
    out = np.zeros(max(1, g.m), np.int32)
    _check(lib.qtng_shard_edges(g.n, g.m, g.flat(), p, int(merged), int(n_shards), out))
    return out[: g.m]


def energy_multi(g: Graph, angles: Angles, contexts: Sequence[Context], merged: bool = False,
                 cfg: Optional[EngineConfig] = None):
    """energy_expectation over several GPUs from ONE process (qtng_energy_multi):
    LPT shards, one host thread per device, one ncclReduce of the term vector.
    Returns (EnergyResult, per-device shard ms)."""
    angles.validate()
    cfg = cfg or EngineConfig()
    gam, bet = _angles_arrays(angles)
    hs = (C.c_void_p * len(contexts))(*[c.handle.value for c in contexts])
    terms = np.zeros(2 * max(1, g.m), np.float64)
    ms = np.zeros(max(1, len(contexts)), np.float32)
    e = C.c_double(0)
    _check(lib.qtng_energy_multi(hs, len(contexts), g.n, g.m, g.flat(), angles.depth(), gam,
                                 bet, int(merged), cfg.max_result_width, cfg.precision_bits(),
                                 C.byref(e), terms, ms))
    return EnergyResult(e.value, terms[: 2 * g.m].view(np.complex128).copy()), ms[: len(contexts)]


# ------------------------------------------------------------------ plans
class Plan:
    """An angle-independent, device-resident plan of a set of lightcones.

    Build once per graph (host schedules, levels, arena placement, descriptor
    upload); each ``execute(angles)`` uploads only the gate table."""

    def __init__(self, g: Graph, p: int, merged: bool = False,
                 cfg: Optional[EngineConfig] = None, edges: Optional[Sequence[int]] = None,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        cfg = cfg or EngineConfig()
        self.graph = g
        self.p = p
        self.sel = (np.arange(g.m, dtype=np.int32) if edges is None
                    else np.ascontiguousarray(edges, dtype=np.int32))
        h = C.c_void_p()
        _check(lib.qtng_plan_create(self.ctx.handle, g.n, g.m, g.flat(), p, int(merged),
                                    cfg.max_result_width, cfg.precision_bits(), len(self.sel),
                                    self.sel.ctypes.data_as(C.c_void_p), C.byref(h)))
        self._h = h
        self.last_device_ms = 0.0

    def info(self) -> PlanInfo:
        inf = PlanInfo()
        _check(lib.qtng_plan_info_get(self._h, C.byref(inf)))
        return inf

    @classmethod
    def from_schedule(cls, schedule: ContractionSchedule, cfg: Optional[EngineConfig] = None,
                      ctx: Optional[Context] = None) -> "Plan":
        """Device-resident plan of one explicit schedule (e.g. a single wide
        bucket); execute() returns its scalar as a 1-element array."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        cfg = cfg or EngineConfig()
        self.graph, self.p, self.sel = None, 0, np.zeros(1, np.int32)
        ints, n_ints, data = schedule.flatten()
        h = C.c_void_p()
        _check(lib.qtng_plan_create_schedule(self.ctx.handle, len(schedule.buckets), ints, n_ints,
                                             np.ascontiguousarray(data), cfg.max_result_width,
                                             C.byref(h)))
        self._h = h
        self.last_device_ms = 0.0
        return self

    def execute(self, angles: Optional[Angles] = None) -> np.ndarray:
        """Per-edge complex e_jk of the selected edges (selection order): one
        CUDA-graph launch (gate-table upload + kernels + terms download)."""
        return self._run(lib.qtng_plan_execute, angles)

    def profile(self, angles: Optional[Angles] = None) -> np.ndarray:
        """execute() enqueued eagerly with CUDA events around every level and
        kernel; fills level_ms(), kernel_ms(), level_kernel_ms()."""
        return self._run(lib.qtng_plan_profile, angles)

    def _run(self, fn, angles) -> np.ndarray:
        if self.p:
            gam, bet = _angles_arrays(angles)
            if len(gam) != self.p or len(bet) != self.p:
                raise InvalidInputError("angles: gammas and betas must have equal length p >= 1")
            gp, bp = gam.ctypes.data_as(C.c_void_p), bet.ctypes.data_as(C.c_void_p)
        else:
            gp = bp = None
        out = np.zeros(2 * max(1, len(self.sel)), np.float64)
        ms = C.c_float(0)
        _check(fn(self._h, gp, bp, out.ctypes.data_as(C.c_void_p), C.byref(ms)))
        self.last_device_ms = ms.value
        return out[: 2 * len(self.sel)].view(np.complex128).copy()

    def run_device(self, n_runs: int = 1) -> float:
        """n_runs replays of the plan's captured CUDA graph (current angles);
        total device ms."""
        ms = C.c_float(0)
        _check(lib.qtng_plan_run_device(self._h, n_runs, C.byref(ms)))
        return ms.value

    def terms(self) -> np.ndarray:
        """The terms the last run (execute or a run_device replay) left on the device."""
        out = np.zeros(2 * max(1, len(self.sel)), np.float64)
        _check(lib.qtng_plan_terms(self._h, out))
        return out[: 2 * len(self.sel)].view(np.complex128).copy()

    def level_ms(self) -> np.ndarray:
        n = self.info().n_levels
        out = np.zeros(max(1, n), np.float32)
        _check(lib.qtng_plan_level_ms(self._h, out, n))
        return out[:n]

    def kernel_ms(self) -> dict:
        """Device ms of the last profile() per kernel kind (events on each kernel's stream)."""
        ms = np.zeros(4, np.float32)
        _check(lib.qtng_plan_kernel_ms(self._h, ms, None, 0))
        return {"level_kernel": float(ms[0]), "outer_kernel": float(ms[1]), "seg_kernel": float(ms[2]),
                "seg4_kernel": float(ms[3])}

    def level_kernel_ms(self) -> np.ndarray:
        """(n_levels, 4) device ms of the last profile(): level / outer / seg / seg4 kernel per level."""
        n = self.info().n_levels
        ms, per = np.zeros(4, np.float32), np.zeros(4 * max(1, n), np.float32)
        _check(lib.qtng_plan_kernel_ms(self._h, ms, per.ctypes.data_as(C.c_void_p), 4 * n))
        return per[:4 * n].reshape(n, 4)

    def time_level(self, level: int = -1, n_runs: int = 10):
        lv, by, ms = C.c_int(0), C.c_double(0), C.c_float(0)
        _check(lib.qtng_plan_time_level(self._h, level, n_runs, C.byref(lv), C.byref(by),
                                        C.byref(ms)))
        return lv.value, by.value, ms.value

    def records(self) -> List[TimingRecord]:
        n = C.c_int64(0)
        _check(lib.qtng_plan_records(self._h, None, 0, C.byref(n)))
        recs = (Record * max(1, n.value))()
        _check(lib.qtng_plan_records(self._h, recs, n.value, C.byref(n)))
        return [TimingRecord(r.edge_u, r.edge_v, r.bucket_seq, r.width, "b200", r.elapsed_s,
                             r.ops, r.flops_est) for r in recs[: n.value]]

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.qtng_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
