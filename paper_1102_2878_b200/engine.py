"""Host-side mirror of the reference's DFGT interface, over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/dfgt/{engine,cv,dataset}.hpp) so a caller of
``dfgt::DualTreeEngine`` / ``compute_sums`` / ``bandwidth_sweep`` can switch:

    reference (C++)                         here
    ------------------------------------    ----------------------------------------
    DualTreeEngine(refs, mode, cfg)         DualTreeEngine(refs, mode, config)
      .compute(queries, h)                    .compute(queries, h)     (None -> Q = R)
      .last_stats() / .p_max()                .last_stats() / .p_max()
      .reference_tree()                       .reference_tree()        (flat arrays)
    naive_kde / dfd_kde / dfgt_kde          naive_kde / dfd_kde / dfgt_kde  (GPU)
    compute_sums(Algorithm, Q, R, h, cfg)   compute_sums(algorithm, Q, R, h, config)
    lkcv_from_sums / lscv_from_sums         lkcv_from_sums / lscv_from_sums
    lkcv_score / lscv_score                 lkcv_score / lscv_score
    bandwidth_sweep(refs, scales, h0, ...)  bandwidth_sweep(refs, scales, h0, kind, options)
    verify_relative_error                   verify_relative_error
    gaussian_normalizer / pilot_bandwidth   gaussian_normalizer / pilot_bandwidth

std::invalid_argument -> ValueError; CUDA failures -> RuntimeError.
Points are (N, D) float64 arrays (PointSet, dataset.hpp:15-41).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import check, lib

_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)


def _pts(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("PointSet requires N >= 1 and D >= 1")
    return a


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


class CostModel(enum.IntEnum):
    exponential = 0
    term_count = 1


class Mode(enum.IntEnum):
    centroid = 0  # DFD
    series = 1    # DFGT


class Algorithm(enum.Enum):
    naive = "naive"
    dfd = "dfd"
    dfgt = "dfgt"


class CvScore(enum.Enum):
    likelihood = "likelihood"
    least_squares = "least_squares"


@dataclass
class EngineConfig:
    """EngineConfig (engine.hpp:17-26); gridfft fields are out of scope."""

    epsilon: float = 0.01
    leaf_threshold: int = 20
    p_max: Optional[int] = None
    cost_model: CostModel = CostModel.exponential
    # 0: direct evaluation of ancestors' local expansions (default, one kernel);
    # 1: the reference's L2L push-down chain (engine.cpp:294-304)
    local_pushdown: int = 0

    def _c(self, mode: Mode) -> _capi.Config:
        return _capi.Config(float(self.epsilon), int(self.leaf_threshold),
                            int(self.p_max or 0), int(self.cost_model), int(mode),
                            int(self.local_pushdown))


@dataclass
class TraversalStats:
    kernel_evaluations: int = 0
    pairs_visited: int = 0
    base_cases: int = 0
    prunes_finite_diff: int = 0
    prunes_farfield: int = 0
    prunes_direct_local: int = 0
    prunes_far_to_local: int = 0
    levels: int = 0
    pairs_covered: int = 0  # sum of |Q||R| over retired node pairs (== n_queries * n_refs)


@dataclass
class KdTreeArrays:
    """Flat KdTree arrays (kdtree.hpp:62-73), preorder node ids."""

    perm: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    centroid: np.ndarray
    max_side: np.ndarray
    left: np.ndarray
    right: np.ndarray
    split_dim: np.ndarray
    split_coord: np.ndarray
    begin: np.ndarray
    count: np.ndarray
    height: int = 0

    def fields(self):
        return ("perm", "lo", "hi", "centroid", "max_side", "left", "right", "split_dim",
                "split_coord", "begin", "count")


class DualTreeEngine:
    """GPU DualTreeEngine (engine.hpp:86-111).  Copies `refs` to the device and builds
    the reference kd-tree there (KdTree::build bit-exact)."""

    def __init__(self, refs, mode: Mode = Mode.series, config: EngineConfig | None = None):
        self.mode = Mode(mode)
        self.config = config or EngineConfig()
        h = C.c_void_p()
        cfg = self.config._c(self.mode)
        if isinstance(refs, np.ndarray) and refs.dtype == np.float32:
            # float32 points (BASELINE config 5): half the H2D bytes, widened exactly on
            # the device; the host mirror keeps the widened values
            r32 = np.ascontiguousarray(refs.reshape(-1, 1) if refs.ndim == 1 else refs)
            self.refs = _pts(r32)
            check(lib.dfgtb_create_f32(r32.ctypes.data_as(_F), r32.shape[0], r32.shape[1],
                                       C.byref(cfg), C.byref(h)))
        else:
            self.refs = _pts(refs)
            check(lib.dfgtb_create(_dp(self.refs), self.refs.shape[0], self.refs.shape[1],
                                   C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            try:
                lib.dfgtb_destroy(self._h)
            except (AttributeError, TypeError):  # interpreter shutdown: the library is gone
                pass
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def compute(self, queries, h: float) -> np.ndarray:
        """Per-query sums with |approx - exact| <= epsilon * exact (engine.hpp:93-95).
        queries=None (or the refs array itself) means Q = R."""
        if queries is None or queries is self.refs:
            out = np.empty(self.refs.shape[0])
            check(lib.dfgtb_compute(self._h, None, 0, float(h), _dp(out), None))
            return out
        q = _pts(queries)
        if q.shape[1] != self.refs.shape[1]:
            raise ValueError("query and reference dimensions differ")
        out = np.empty(q.shape[0])
        check(lib.dfgtb_compute(self._h, _dp(q), q.shape[0], float(h), _dp(out), None))
        return out

    def compute_batch(self, queries, hs, out: np.ndarray | None = None) -> np.ndarray:
        """Sums for several bandwidths through one lock-step GPU traversal:
        row b = compute(queries, hs[b]).  Returns (len(hs), n_queries), written into
        `out` when given (a C-contiguous float64 array of that shape, e.g. pinned host
        memory reused across calls)."""
        hv = np.ascontiguousarray(hs, dtype=np.float64).ravel()

        def _out(n):
            if out is None:
                return np.empty((hv.size, n))
            if out.dtype != np.float64 or out.shape != (hv.size, n) or not out.flags.c_contiguous:
                raise ValueError(f"out must be a C-contiguous float64 array of shape {(hv.size, n)}")
            return out
        if isinstance(queries, np.ndarray) and queries.dtype == np.float32:
            q32 = np.ascontiguousarray(queries.reshape(-1, 1) if queries.ndim == 1 else queries)
            if q32.ndim != 2 or q32.shape[1] != self.refs.shape[1]:
                raise ValueError("query and reference dimensions differ")
            res = _out(q32.shape[0])
            st = (_capi.Stats * max(1, hv.size))()
            check(lib.dfgtb_compute_batch_f32(self._h, q32.ctypes.data_as(_F), q32.shape[0],
                                              _dp(hv), hv.size, _dp(res), st))
            self._batch_stats = [TraversalStats(**s.as_dict()) for s in st[:hv.size]]
            return res
        if queries is None or queries is self.refs:
            q, nq, n_out = None, 0, self.refs.shape[0]
        else:
            q = _pts(queries)
            if q.shape[1] != self.refs.shape[1]:
                raise ValueError("query and reference dimensions differ")
            nq = n_out = q.shape[0]
        res = _out(n_out)
        st = (_capi.Stats * max(1, hv.size))()
        check(lib.dfgtb_compute_batch(self._h, _dp(q) if q is not None else None, nq, _dp(hv),
                                      hv.size, _dp(res), st))
        self._batch_stats = [TraversalStats(**s.as_dict()) for s in st[:hv.size]]
        return res

    def batch_stats(self):
        return list(getattr(self, "_batch_stats", []))

    def compute_device(self, d_queries: int, nq: int, h: float, d_out: int) -> None:
        """Device-pointer variant (inputs already resident in HBM)."""
        check(lib.dfgtb_compute_device(self._h, C.c_void_p(d_queries or 0), nq, float(h),
                                       C.c_void_p(d_out), None))

    def last_stats(self) -> TraversalStats:
        s = _capi.Stats()
        check(lib.dfgtb_last_stats(self._h, C.byref(s)))
        return TraversalStats(**s.as_dict())

    def last_timings(self) -> dict:
        t = _capi.Timings()
        check(lib.dfgtb_last_timings(self._h, C.byref(t)))
        return t.as_dict()

    def p_max(self) -> int:
        return lib.dfgtb_p_max(self._h)

    def reference_tree(self) -> KdTreeArrays:
        n, d = self.refs.shape
        k = lib.dfgtb_tree_nodes(self._h)
        t = KdTreeArrays(
            perm=np.zeros(n, np.int32), lo=np.zeros((k, d)), hi=np.zeros((k, d)),
            centroid=np.zeros((k, d)), max_side=np.zeros(k), left=np.zeros(k, np.int32),
            right=np.zeros(k, np.int32), split_dim=np.zeros(k, np.int32),
            split_coord=np.zeros(k), begin=np.zeros(k, np.int64), count=np.zeros(k, np.int32),
            height=lib.dfgtb_tree_height(self._h))
        I = C.POINTER(C.c_int)
        check(lib.dfgtb_export_tree(
            self._h, t.perm.ctypes.data_as(I), _dp(t.lo), _dp(t.hi), _dp(t.centroid),
            _dp(t.max_side), t.left.ctypes.data_as(I), t.right.ctypes.data_as(I),
            t.split_dim.ctypes.data_as(I), _dp(t.split_coord),
            t.begin.ctypes.data_as(C.POINTER(C.c_int64)), t.count.ctypes.data_as(I)))
        return t

    def cv(self, h: float, conv_h: float | None = None) -> _capi.CvRow:
        """Fused on-device CV at h (and conv_h, default 2h): sums never leave HBM."""
        row = _capi.CvRow()
        check(lib.dfgtb_cv(self._h, float(h), float(2.0 * h if conv_h is None else conv_h),
                           C.byref(row)))
        return row

    def sweep(self, scales: Sequence[float], base_h: float, sqrt2: bool = False):
        """bandwidth_sweep (cv.cpp:141-182) for both scores, every h and conv h in one
        batched GPU traversal.  Rows' `seconds` are shares of the batch's device time."""
        sc = np.ascontiguousarray(scales, dtype=np.float64)
        rows = (_capi.CvRow * len(sc))()
        check(lib.dfgtb_sweep(self._h, _dp(sc), len(sc), float(base_h), int(sqrt2), rows))
        return list(rows)

    @staticmethod
    def best(rows) -> tuple[int, int]:
        """h* of a sweep: (argmax lk_score, argmin ls_score), first index on ties."""
        arr = (_capi.CvRow * len(rows))(*rows)
        ik, il = C.c_size_t(), C.c_size_t()
        check(lib.dfgtb_sweep_best(arr, len(rows), C.byref(ik), C.byref(il)))
        return int(ik.value), int(il.value)


# ----------------------------------------------------------------- free functions
def gaussian_normalizer(dim: int, h: float) -> float:
    """(2 pi h^2)^(D/2) (dataset.cpp:32-39)."""
    if dim < 1 or not h > 0.0:
        raise ValueError("gaussian_normalizer requires D >= 1 and h > 0")
    return math.pow(6.283185307179586476925286766559 * h * h, 0.5 * dim)


def naive_kde(queries, refs, h: float) -> np.ndarray:
    """Exact FP64 sums on the GPU (engine.cpp:22-36)."""
    q, r = _pts(queries), _pts(refs)
    if q.shape[1] != r.shape[1]:
        raise ValueError("query and reference dimensions differ")
    out = np.empty(q.shape[0])
    check(lib.dfgtb_naive(_dp(q), q.shape[0], _dp(r), r.shape[0], r.shape[1], float(h), _dp(out)))
    return out


def dfgt_kde(queries, refs, h: float, config: EngineConfig | None = None) -> np.ndarray:
    """engine.cpp:436-441."""
    r = _pts(refs)
    q = _pts(queries)
    if q.shape[1] != r.shape[1]:
        raise ValueError("query and reference dimensions differ")
    with DualTreeEngine(r, Mode.series, config) as e:
        return e.compute(None if queries is refs else q, h)


def dfd_kde(queries, refs, h: float, epsilon: float, leaf_threshold: int = 20) -> np.ndarray:
    """engine.cpp:426-434."""
    r = _pts(refs)
    q = _pts(queries)
    if q.shape[1] != r.shape[1]:
        raise ValueError("query and reference dimensions differ")
    cfg = EngineConfig(epsilon=epsilon, leaf_threshold=leaf_threshold)
    with DualTreeEngine(r, Mode.centroid, cfg) as e:
        return e.compute(None if queries is refs else q, h)


def compute_sums(algorithm, queries, refs, h: float, config: EngineConfig | None = None):
    """engine.cpp:495-512 (gridfft is outside this path)."""
    algorithm = Algorithm(algorithm.value if isinstance(algorithm, Algorithm) else algorithm)
    config = config or EngineConfig()
    if algorithm is Algorithm.naive:
        return naive_kde(queries, refs, h)
    if algorithm is Algorithm.dfd:
        return dfd_kde(queries, refs, h, config.epsilon, config.leaf_threshold)
    return dfgt_kde(queries, refs, h, config)


@dataclass
class RelativeErrorReport:
    max_relative_error: float = 0.0
    worst_index: int = 0


def verify_relative_error(approx, exact) -> RelativeErrorReport:
    """engine.cpp:443-461."""
    a = np.asarray(approx, dtype=np.float64)
    e = np.asarray(exact, dtype=np.float64)
    if a.shape != e.shape:
        raise ValueError("approx and exact lengths differ")
    if not np.all(e > 0.0):
        raise ValueError("exact sums must be strictly positive")
    rel = np.abs(a - e) / e
    i = int(np.argmax(rel)) if rel.size else 0
    return RelativeErrorReport(float(rel[i]) if rel.size else 0.0, i)


@dataclass
class ScoreResult:
    score: float = 0.0
    clamped: int = 0


def lkcv_from_sums(refs, h: float, sums) -> ScoreResult:
    """cv.cpp:61-76 (leave-one-out by self-term subtraction, DBL_MIN clamp)."""
    r = _pts(refs)
    s = np.ascontiguousarray(sums, dtype=np.float64)
    sc, cl = C.c_double(), C.c_int()
    check(lib.dfgtb_lkcv_from_sums(r.shape[0], r.shape[1], float(h), _dp(s), C.byref(sc),
                                   C.byref(cl)))
    return ScoreResult(sc.value, cl.value)


def lscv_from_sums(refs, h: float, sums, conv_h: float, conv_sums) -> ScoreResult:
    """cv.cpp:78-97."""
    r = _pts(refs)
    s = np.ascontiguousarray(sums, dtype=np.float64)
    cs = np.ascontiguousarray(conv_sums, dtype=np.float64)
    sc = C.c_double()
    check(lib.dfgtb_lscv_from_sums(r.shape[0], r.shape[1], float(h), _dp(s), float(conv_h),
                                   _dp(cs), C.byref(sc)))
    return ScoreResult(sc.value, 0)


@dataclass
class CvOptions:
    """CvOptions (cv.hpp:14-23)."""

    algorithm: Algorithm = Algorithm.dfgt
    engine: EngineConfig = field(default_factory=EngineConfig)
    sqrt2_convolution: bool = False
    verify_against_naive: bool = False


def convolution_bandwidth(h: float, options: CvOptions) -> float:
    """cv.cpp:27-30."""
    return math.sqrt(2.0) * h if options.sqrt2_convolution else 2.0 * h


class _SumProvider:
    """cv.cpp:32-57: one engine reused across bandwidths."""

    def __init__(self, refs, options: CvOptions):
        self.refs = refs
        self.options = options
        self.engine = None
        if options.algorithm is Algorithm.dfd:
            self.engine = DualTreeEngine(refs, Mode.centroid, options.engine)
        elif options.algorithm is Algorithm.dfgt:
            self.engine = DualTreeEngine(refs, Mode.series, options.engine)

    def __call__(self, h: float) -> np.ndarray:
        if self.engine is not None:
            return self.engine.compute(None, h)
        return compute_sums(self.options.algorithm, self.refs, self.refs, h, self.options.engine)


def lkcv_score(refs, h: float, options: CvOptions | None = None) -> ScoreResult:
    options = options or CvOptions()
    return lkcv_from_sums(refs, h, _SumProvider(_pts(refs), options)(h))


def lscv_score(refs, h: float, options: CvOptions | None = None) -> ScoreResult:
    options = options or CvOptions()
    p = _SumProvider(_pts(refs), options)
    ch = convolution_bandwidth(h, options)
    return lscv_from_sums(refs, h, p(h), ch, p(ch))


def pilot_bandwidth(refs) -> float:
    """cv.cpp:112-139: mean per-dimension sample std * N^(-1/(D+4))."""
    r = _pts(refs)
    n, d = r.shape
    if n < 2:
        raise ValueError("pilot bandwidth requires at least 2 points")
    # the reference's summation order (sequential sums per dimension, two passes):
    # cumsum is a left-to-right sum, so h is bit-identical to cv.cpp's
    sigma_sum = 0.0
    for k in range(d):
        col = r[:, k]
        mean = float(np.cumsum(col)[-1]) / n
        t = col - mean
        var = float(np.cumsum(t * t)[-1])
        sigma_sum += math.sqrt(var / (n - 1))
    sigma = sigma_sum / d
    if not sigma > 0.0:
        raise ValueError("pilot bandwidth undefined for zero-variance data")
    return sigma * math.pow(float(n), -1.0 / (d + 4.0))


@dataclass
class CvRow:
    """cv.hpp:49-56."""

    scale: float = 0.0
    h: float = 0.0
    score: float = 0.0
    seconds: float = 0.0
    max_rel_err: Optional[float] = None
    clamped: int = 0


def bandwidth_sweep(refs, scales: Sequence[float], base_h: float, kind: CvScore,
                    options: CvOptions | None = None) -> list[CvRow]:
    """cv.cpp:141-182.  For the DFGT/DFD engines the sums stay on the device and the
    CV reductions run there (dfgtb_cv); `seconds` is device time of the computes."""
    options = options or CvOptions()
    if not base_h > 0.0:
        raise ValueError("base bandwidth must be positive")
    sc = list(scales)
    for a, b in zip(sc, sc[1:]):
        if not b > a:
            raise ValueError("scales must be strictly increasing")
    r = _pts(refs)
    p = _SumProvider(r, options)
    rows = []
    for s in sc:
        h = s * base_h
        row = CvRow(scale=s, h=h)
        if p.engine is not None and not options.verify_against_naive:
            ch = convolution_bandwidth(h, options) if kind is CvScore.least_squares else 0.0
            cr = _capi.CvRow()
            check(lib.dfgtb_cv(p.engine.handle, float(h), float(ch), C.byref(cr)))
            row.score = cr.lk_score if kind is CvScore.likelihood else cr.ls_score
            row.clamped = cr.lk_clamped if kind is CvScore.likelihood else 0
            row.seconds = cr.seconds
        else:
            sums = p(h)
            if kind is CvScore.likelihood:
                res = lkcv_from_sums(r, h, sums)
            else:
                ch = convolution_bandwidth(h, options)
                res = lscv_from_sums(r, h, sums, ch, p(ch))
            row.score, row.clamped = res.score, res.clamped
            if options.verify_against_naive and options.algorithm is not Algorithm.naive:
                row.max_rel_err = verify_relative_error(sums, naive_kde(r, r, h)).max_relative_error
        rows.append(row)
    return rows
