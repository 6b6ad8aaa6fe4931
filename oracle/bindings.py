"""ctypes bindings for the oracle restatement and the compiled reference.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_L = C.POINTER(C.c_longlong)
_U64 = C.POINTER(C.c_uint64)


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(_I)


def _c(x, dtype=np.float64):
    return np.ascontiguousarray(x, dtype=dtype)


@dataclass
class Tree:
    """Flat kd-tree arrays, node-major, preorder ids (kdtree.hpp:62-73)."""

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

    @property
    def nodes(self) -> int:
        return int(self.count.shape[0])

    def height(self) -> int:
        depth = np.zeros(self.nodes, dtype=np.int64)
        for n in range(self.nodes):  # preorder: parents precede children
            if self.left[n] >= 0:
                depth[self.left[n]] = depth[n] + 1
                depth[self.right[n]] = depth[n] + 1
        return int(depth.max()) + 1

    def fields(self):
        return ("perm", "lo", "hi", "centroid", "max_side", "left", "right", "split_dim",
                "split_coord", "begin", "count")


def _alloc_tree(n, d, nodes):
    return Tree(
        perm=np.zeros(n, np.int32),
        lo=np.zeros((nodes, d)), hi=np.zeros((nodes, d)), centroid=np.zeros((nodes, d)),
        max_side=np.zeros(nodes), left=np.zeros(nodes, np.int32), right=np.zeros(nodes, np.int32),
        split_dim=np.zeros(nodes, np.int32), split_coord=np.zeros(nodes),
        begin=np.zeros(nodes, np.int64), count=np.zeros(nodes, np.int32))


class _orc_tree(C.Structure):
    _fields_ = [("perm", _I), ("lo", _D), ("hi", _D), ("centroid", _D), ("max_side", _D),
                ("left", _I), ("right", _I), ("split_dim", _I), ("split_coord", _D),
                ("begin", _L), ("count", _I)]


def _make(path: str):
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=False,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    return C.CDLL(path) if os.path.exists(path) else None


class Oracle:
    """The C restatement (oracle/dfgt_oracle.c)."""

    def __init__(self, lib):
        self.lib = lib
        L = lib
        L.orc_gaussian_normalizer.restype = C.c_double
        L.orc_gaussian_normalizer.argtypes = [C.c_size_t, C.c_double]
        L.orc_farfield_error_bound.restype = C.c_double
        L.orc_f2l_error_bound.restype = C.c_double
        for f in ("orc_farfield_error_bound", "orc_f2l_error_bound"):
            getattr(L, f).argtypes = [C.c_double, C.c_double, C.c_int, C.c_int]
        L.orc_series_eval_farfield.restype = C.c_double
        L.orc_series_eval_local.restype = C.c_double
        L.orc_lkcv.restype = C.c_double
        L.orc_lscv.restype = C.c_double
        L.orc_pilot_bandwidth.restype = C.c_double

    # --- dataset / engine
    def gaussian_normalizer(self, d, h):
        return self.lib.orc_gaussian_normalizer(d, C.c_double(h))

    def naive_kde(self, q, r, h):
        q, r = _c(q), _c(r)
        out = np.empty(q.shape[0])
        self.lib.orc_naive_kde(_dp(q), C.c_size_t(q.shape[0]), _dp(r), C.c_size_t(r.shape[0]),
                               C.c_size_t(r.shape[1]), C.c_double(h), _dp(out))
        return out

    def box_bounds_sq(self, alo, ahi, blo, bhi):
        a, b, c, d = (_c(v) for v in (alo, ahi, blo, bhi))
        lo, hi = C.c_double(), C.c_double()
        self.lib.orc_box_bounds_sq(_dp(a), _dp(b), _dp(c), _dp(d), C.c_size_t(a.size),
                                   C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def tree(self, x, leaf):
        x = _c(x)
        n, d = x.shape
        t = _alloc_tree(n, d, max(1, 2 * n))
        s = _orc_tree(_ip(t.perm), _dp(t.lo), _dp(t.hi), _dp(t.centroid), _dp(t.max_side),
                      _ip(t.left), _ip(t.right), _ip(t.split_dim), _dp(t.split_coord),
                      t.begin.ctypes.data_as(_L), _ip(t.count))
        nodes = self.lib.orc_tree_build(_dp(x), C.c_size_t(n), C.c_size_t(d), C.c_int(leaf),
                                        C.byref(s))
        if nodes < 0:
            raise ValueError("leaf_threshold must be >= 1")
        for f in t.fields():
            if f != "perm":
                setattr(t, f, np.ascontiguousarray(getattr(t, f)[:nodes]))
        return t

    def dfgt(self, r, h, q=None, eps=0.01, leaf=20, p_max=0, cost_model=0, mode=1):
        r = _c(r)
        qq = _c(q) if q is not None else None
        nq = qq.shape[0] if qq is not None else r.shape[0]
        out = np.empty(nq)
        st = np.zeros(7, np.uint64)
        rc = self.lib.orc_dfgt(_dp(r), C.c_size_t(r.shape[0]), _dp(qq), C.c_size_t(nq),
                               C.c_size_t(r.shape[1]), C.c_double(h), C.c_double(eps), leaf,
                               p_max, cost_model, mode, _dp(out), st.ctypes.data_as(_U64))
        if rc != 0:
            raise ValueError("invalid argument")
        return out, st

    # --- truncation
    def farfield_error_bound(self, c, r, p, d):
        return self.lib.orc_farfield_error_bound(c, r, p, d)

    def f2l_error_bound(self, c, r, p, d):
        return self.lib.orc_f2l_error_bound(c, r, p, d)

    def choose_best_method(self, nq, nr, sq, sr, h, tau, p_max, d, cost_model=0):
        k, o = C.c_int(), C.c_int()
        self.lib.orc_choose_best_method(*(C.c_double(v) for v in (nq, nr, sq, sr, h, tau)),
                                        p_max, d, cost_model, C.byref(k), C.byref(o))
        return k.value, o.value

    def default_p_max(self, d):
        return self.lib.orc_default_p_max(d)

    # --- series
    def terms(self, d, p):
        T = p ** d
        pos, par, pd, deg = (np.zeros(T, np.int32) for _ in range(4))
        invf = np.zeros(T)
        self.lib.orc_series_terms(d, p, _ip(pos), _ip(par), _ip(pd), _ip(deg), _dp(invf))
        return pos, par, pd, deg, invf

    def moments(self, p_max, pts, center, h):
        pts = _c(pts)
        d = pts.shape[1]
        M = np.zeros(p_max ** d)
        self.lib.orc_series_moments(d, p_max, _dp(pts), C.c_size_t(pts.shape[0]), _dp(_c(center)),
                                    C.c_double(h), _dp(M))
        return M

    def f2f(self, p_max, src, sc, dc, h, dst=None):
        d = len(sc)
        dst = np.zeros(p_max ** d) if dst is None else _c(dst).copy()
        self.lib.orc_series_f2f(d, p_max, _dp(_c(src)), _dp(_c(sc)), _dp(_c(dc)), C.c_double(h),
                                _dp(dst))
        return dst

    def eval_farfield(self, p_max, M, c, q, h, order):
        return self.lib.orc_series_eval_farfield(len(c), p_max, _dp(_c(M)), _dp(_c(c)),
                                                 _dp(_c(q)), C.c_double(h), order)

    def direct_local(self, p_max, pts, c, h, order, L=None):
        pts = _c(pts)
        d = pts.shape[1]
        L = np.zeros(p_max ** d) if L is None else _c(L).copy()
        self.lib.orc_series_direct_local(d, p_max, _dp(pts), C.c_size_t(pts.shape[0]), _dp(_c(c)),
                                         C.c_double(h), order, _dp(L))
        return L

    def f2l(self, p_max, M, sc, dc, h, order, L=None):
        d = len(sc)
        L = np.zeros(p_max ** d) if L is None else _c(L).copy()
        self.lib.orc_series_f2l(d, p_max, _dp(_c(M)), _dp(_c(sc)), _dp(_c(dc)), C.c_double(h),
                                order, _dp(L))
        return L

    def l2l(self, p_max, src, sc, dc, h, order, dst=None):
        d = len(sc)
        dst = np.zeros(p_max ** d) if dst is None else _c(dst).copy()
        self.lib.orc_series_l2l(d, p_max, _dp(_c(src)), _dp(_c(sc)), _dp(_c(dc)), C.c_double(h),
                                order, _dp(dst))
        return dst

    def eval_local(self, p_max, L, c, q, h, order):
        return self.lib.orc_series_eval_local(len(c), p_max, _dp(_c(L)), _dp(_c(c)), _dp(_c(q)),
                                              C.c_double(h), order)

    # --- cv
    def lkcv(self, d, h, sums):
        s = _c(sums)
        cl = C.c_int()
        v = self.lib.orc_lkcv(C.c_size_t(s.size), C.c_size_t(d), C.c_double(h), _dp(s), C.byref(cl))
        return v, cl.value

    def lscv(self, d, h, sums, conv_h, conv_sums):
        s, cs = _c(sums), _c(conv_sums)
        return self.lib.orc_lscv(C.c_size_t(s.size), C.c_size_t(d), C.c_double(h), _dp(s),
                                 C.c_double(conv_h), _dp(cs))

    def pilot_bandwidth(self, x):
        x = _c(x)
        return self.lib.orc_pilot_bandwidth(_dp(x), C.c_size_t(x.shape[0]), C.c_size_t(x.shape[1]))


class Reference:
    """The unmodified reference, compiled from /root/reference (oracle/_ref)."""

    def __init__(self, lib):
        self.lib = lib
        L = lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_gaussian_normalizer.restype = C.c_double
        L.ref_gaussian_normalizer.argtypes = [C.c_size_t, C.c_double]
        L.ref_tree_build.restype = C.c_void_p
        L.ref_tree_build.argtypes = [_D, C.c_size_t, C.c_size_t, C.c_int]
        for f in ("ref_tree_node_count", "ref_tree_height", "ref_tree_free",
                  "ref_engine_p_max", "ref_engine_free", "ref_series_free",
                  "ref_series_table_size"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_tree_export.argtypes = [C.c_void_p, C.c_size_t, _I, _D, _D, _D, _D, _I, _I, _I, _D,
                                      _L, _I]
        L.ref_engine_create.restype = C.c_void_p
        L.ref_engine_create.argtypes = [_D, C.c_size_t, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                        C.c_int, C.c_int]
        L.ref_engine_compute.argtypes = [C.c_void_p, _D, C.c_size_t, C.c_double, _D, _U64]
        L.ref_farfield_error_bound.restype = C.c_double
        L.ref_f2l_error_bound.restype = C.c_double
        for f in ("ref_farfield_error_bound", "ref_f2l_error_bound"):
            getattr(L, f).argtypes = [C.c_double, C.c_double, C.c_int, C.c_int]
        L.ref_series_geometry.restype = C.c_void_p
        L.ref_series_eval_farfield.restype = C.c_double
        L.ref_series_eval_local.restype = C.c_double
        for f in ("ref_series_terms", "ref_series_moments", "ref_series_f2f",
                  "ref_series_eval_farfield", "ref_series_direct_local", "ref_series_f2l",
                  "ref_series_l2l", "ref_series_eval_local"):
            getattr(L, f).argtypes = None

    def _err(self, rc):
        if rc == 1:
            raise ValueError(self.lib.ref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def gaussian_normalizer(self, d, h):
        return self.lib.ref_gaussian_normalizer(d, h)

    def naive_kde(self, q, r, h):
        q, r = _c(q), _c(r)
        out = np.empty(q.shape[0])
        self._err(self.lib.ref_naive_kde(_dp(q), C.c_size_t(q.shape[0]), _dp(r),
                                         C.c_size_t(r.shape[0]), C.c_size_t(r.shape[1]),
                                         C.c_double(h), _dp(out)))
        return out

    def tree(self, x, leaf):
        x = _c(x)
        n, d = x.shape
        h = self.lib.ref_tree_build(_dp(x), n, d, leaf)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        try:
            nodes = self.lib.ref_tree_node_count(h)
            t = _alloc_tree(n, d, nodes)
            self.lib.ref_tree_export(h, n, _ip(t.perm), _dp(t.lo), _dp(t.hi), _dp(t.centroid),
                                     _dp(t.max_side), _ip(t.left), _ip(t.right), _ip(t.split_dim),
                                     _dp(t.split_coord), t.begin.ctypes.data_as(_L), _ip(t.count))
        finally:
            self.lib.ref_tree_free(h)
        return t

    def box_bounds_sq(self, alo, ahi, blo, bhi):
        a, b, c, d = (_c(v) for v in (alo, ahi, blo, bhi))
        out = np.zeros(2)
        self.lib.ref_box_bounds_sq(_dp(a), _dp(b), _dp(c), _dp(d), C.c_size_t(a.size), _dp(out))
        return out[0], out[1]

    def engine(self, r, eps=0.01, leaf=20, p_max=0, cost_model=0, mode=1):
        return RefEngine(self, r, eps, leaf, p_max, cost_model, mode)

    def dfgt(self, r, h, q=None, eps=0.01, leaf=20, p_max=0, cost_model=0, mode=1):
        e = self.engine(r, eps, leaf, p_max, cost_model, mode)
        try:
            return e.compute(h, q)
        finally:
            e.close()

    def lkcv(self, r, h, sums):
        r, s = _c(r), _c(sums)
        sc, cl = C.c_double(), C.c_int()
        self._err(self.lib.ref_lkcv(_dp(r), C.c_size_t(r.shape[0]), C.c_size_t(r.shape[1]),
                                    C.c_double(h), _dp(s), C.byref(sc), C.byref(cl)))
        return sc.value, cl.value

    def lscv(self, r, h, sums, conv_h, conv_sums):
        r, s, cs = _c(r), _c(sums), _c(conv_sums)
        sc = C.c_double()
        self._err(self.lib.ref_lscv(_dp(r), C.c_size_t(r.shape[0]), C.c_size_t(r.shape[1]),
                                    C.c_double(h), _dp(s), C.c_double(conv_h), _dp(cs),
                                    C.byref(sc)))
        return sc.value

    def pilot_bandwidth(self, x):
        x = _c(x)
        out = C.c_double()
        self._err(self.lib.ref_pilot_bandwidth(_dp(x), C.c_size_t(x.shape[0]),
                                               C.c_size_t(x.shape[1]), C.byref(out)))
        return out.value

    def farfield_error_bound(self, c, r, p, d):
        return self.lib.ref_farfield_error_bound(c, r, p, d)

    def f2l_error_bound(self, c, r, p, d):
        return self.lib.ref_f2l_error_bound(c, r, p, d)

    def choose_best_method(self, nq, nr, sq, sr, h, tau, p_max, d, cost_model=0):
        out = np.zeros(2, np.int32)
        self.lib.ref_choose_best_method(*(C.c_double(v) for v in (nq, nr, sq, sr, h, tau)),
                                        C.c_int(p_max), C.c_int(d), C.c_int(cost_model), _ip(out))
        return int(out[0]), int(out[1])

    def default_p_max(self, d):
        return self.lib.ref_default_p_max(d)

    def series(self, d, p_max):
        return RefSeries(self, d, p_max)


class RefEngine:
    def __init__(self, ref: Reference, r, eps, leaf, p_max, cost_model, mode):
        self.ref = ref
        self.r = _c(r)
        self.h = ref.lib.ref_engine_create(_dp(self.r), self.r.shape[0], self.r.shape[1], eps, leaf,
                                           p_max, cost_model, mode)
        if not self.h:
            raise ValueError(ref.lib.ref_last_error().decode())

    def compute(self, h, q=None):
        qq = _c(q) if q is not None else None
        nq = qq.shape[0] if qq is not None else self.r.shape[0]
        out = np.empty(nq)
        st = np.zeros(7, np.uint64)
        self.ref._err(self.ref.lib.ref_engine_compute(self.h, _dp(qq), nq, h, _dp(out),
                                                      st.ctypes.data_as(_U64)))
        return out, st

    def p_max(self):
        return self.ref.lib.ref_engine_p_max(self.h)

    def close(self):
        if self.h:
            self.ref.lib.ref_engine_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


class RefSeries:
    def __init__(self, ref: Reference, d, p_max):
        self.lib = ref.lib
        self.d, self.p = d, p_max
        self.g = C.c_void_p(ref.lib.ref_series_geometry(d, p_max))
        self.T = p_max ** d

    def __del__(self):
        self.lib.ref_series_free(self.g)

    def terms(self):
        pos, par, pd, deg = (np.zeros(self.T, np.int32) for _ in range(4))
        invf = np.zeros(self.T)
        self.lib.ref_series_terms(self.g, _ip(pos), _ip(par), _ip(pd), _ip(deg), _dp(invf))
        return pos, par, pd, deg, invf

    def moments(self, pts, center, h):
        pts = _c(pts)
        M = np.zeros(self.T)
        self.lib.ref_series_moments(self.g, _dp(pts), C.c_size_t(pts.shape[0]),
                                    C.c_size_t(self.d), _dp(_c(center)), C.c_double(h), _dp(M))
        return M

    def f2f(self, src, sc, dc, h, dst=None):
        dst = np.zeros(self.T) if dst is None else _c(dst).copy()
        self.lib.ref_series_f2f(self.g, _dp(_c(src)), _dp(_c(sc)), _dp(_c(dc)), C.c_size_t(self.d),
                                C.c_double(h), _dp(dst))
        return dst

    def eval_farfield(self, M, c, q, h, order):
        f = self.lib.ref_series_eval_farfield
        f.restype = C.c_double
        return f(self.g, _dp(_c(M)), _dp(_c(c)), _dp(_c(q)), C.c_size_t(self.d), C.c_double(h),
                 C.c_int(order))

    def direct_local(self, pts, c, h, order, L=None):
        pts = _c(pts)
        L = np.zeros(self.T) if L is None else _c(L).copy()
        self.lib.ref_series_direct_local(self.g, _dp(pts), C.c_size_t(pts.shape[0]),
                                         C.c_size_t(self.d), _dp(_c(c)), C.c_double(h),
                                         C.c_int(order), _dp(L))
        return L

    def f2l(self, M, sc, dc, h, order, L=None):
        L = np.zeros(self.T) if L is None else _c(L).copy()
        self.lib.ref_series_f2l(self.g, _dp(_c(M)), _dp(_c(sc)), _dp(_c(dc)), C.c_size_t(self.d),
                                C.c_double(h), C.c_int(order), _dp(L))
        return L

    def l2l(self, src, sc, dc, h, order, dst=None):
        dst = np.zeros(self.T) if dst is None else _c(dst).copy()
        self.lib.ref_series_l2l(self.g, _dp(_c(src)), _dp(_c(sc)), _dp(_c(dc)), C.c_size_t(self.d),
                                C.c_double(h), C.c_int(order), _dp(dst))
        return dst

    def eval_local(self, L, c, q, h, order):
        f = self.lib.ref_series_eval_local
        f.restype = C.c_double
        return f(self.g, _dp(_c(L)), _dp(_c(c)), _dp(_c(q)), C.c_size_t(self.d), C.c_double(h),
                 C.c_int(order))


_ORC = None
_REF = None


def load_oracle() -> Oracle:
    global _ORC
    if _ORC is None:
        lib = _make(os.path.join(ORACLE_DIR, "liboracle.so"))
        if lib is None:
            raise RuntimeError("oracle/liboracle.so missing and could not be built")
        _ORC = Oracle(lib)
    return _ORC


def load_reference():
    """The compiled reference, or None when oracle/_ref/libdfgt_ref.so is absent."""
    global _REF
    if _REF is None:
        p = os.path.join(ORACLE_DIR, "_ref", "libdfgt_ref.so")
        lib = _make(p)
        _REF = Reference(lib) if lib is not None else False
    return _REF or None
