"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (the parity checker).

ctypes front-end over the two CPU oracles that share oracle/oracle_api.h:

* ``Oracle("port")`` -> oracle/liblamg_oracle.so, the plain-C restatement
  (oracle/lamg_oracle.c);
* ``Oracle("ref")``  -> oracle/_ref/liblamg_ref.so, the unmodified reference
  core compiled from /root/reference (oracle/Makefile).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": (os.path.join(HERE, "liblamg_oracle.so"), "orc_"),
    "ref": (os.path.join(HERE, "_ref", "liblamg_ref.so"), "ref_"),
}

STATUS_NAMES = {
    0: "OK",
    1: "Error",
    2: "EmptyGraphError",
    3: "SingularDiagonalError",
    4: "InvalidLaplacianError",
    5: "DimensionMismatchError",
    6: "IncompatibleRhsError",
    7: "DivergedError",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))
        self.msg = msg


@dataclass
class CSR:
    """Host CSR Laplacian with the reference layout (sparse_laplacian.hpp:18-39)."""

    n: int
    m: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray  # int32[2m]
    val: np.ndarray  # float64[2m] (= -w)
    diag: np.ndarray  # float64[n]

    def args(self):
        return (
            C.c_int32(self.n),
            C.c_int64(self.m),
            _ptr(self.row_ptr, np.int64),
            _ptr(self.col, np.int32),
            _ptr(self.val, np.float64),
            _ptr(self.diag, np.float64),
        )

    @staticmethod
    def from_bag(d: dict, prefix: str = "") -> "CSR":
        return CSR(
            int(d[prefix + "n"][0]),
            int(d[prefix + "m"][0]),
            d[prefix + "row_ptr"],
            d[prefix + "col"],
            d[prefix + "val"],
            d[prefix + "diag"],
        )


def _ptr(a: np.ndarray, dtype):
    assert a.dtype == dtype and a.flags.c_contiguous, (a.dtype, dtype)
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


_DT = {0: np.int32, 1: np.int64, 2: np.float64}


def _csr(a):
    """CSR argument tuple for any object with the SparseLaplacian fields."""
    return CSR.args(a)


class Oracle:
    def __init__(self, which: str = "port"):
        path, prefix = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} missing: run `make -C oracle`")
        self.which = which
        self.lib = C.CDLL(path)
        self.p = prefix
        self._f("last_error").restype = C.c_char_p
        self._f("bag_len").restype = C.c_int64
        self._f("bag_name").restype = C.c_char_p
        self._f("rng_derive").restype = C.c_uint64
        self._f("rng_derive").argtypes = [C.c_uint64, C.c_uint64]
        self._f("flat_mu").restype = C.c_double
        self._f("flat_mu").argtypes = [C.c_double]
        self._f("level_cycle_index").restype = C.c_double
        for name in ("setup", "prepare"):
            self._f(name).restype = C.c_void_p
        for name in ("hier_free", "prepared_free", "hier_export", "prepared_export", "solve",
                     "solve_prepared", "solve_batch", "bag_free", "bag_count", "bag_get",
                     "bag_len", "bag_name", "bag_type", "level_cycle_index"):
            pass

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    # ----------------------------------------------------------------- utils
    def _check(self, code):
        if code != 0:
            raise OracleError(code, self._f("last_error")().decode())

    def _bag(self, bp) -> dict:
        out = {}
        b = C.c_void_p(bp)
        cnt = self._f("bag_count")(b)
        for i in range(cnt):
            name = self._f("bag_name")(b, C.c_int(i))
            ln = self._f("bag_len")(b, name)
            t = self._f("bag_type")(b, name)
            arr = np.empty(ln, dtype=_DT[t])
            self._f("bag_get")(b, name, arr.ctypes.data_as(C.c_void_p))
            out[name.decode()] = arr
        self._f("bag_free")(b)
        return out

    def _call_bag(self, name, *args):
        bp = C.c_void_p()
        code = self._f(name)(*args, C.byref(bp))
        try:
            self._check(code)
        finally:
            if code != 0 and bp.value:
                self._f("bag_free")(bp)
        return self._bag(bp.value)

    # ------------------------------------------------------------------ rng
    def rng_derive(self, seed: int, stream: int) -> int:
        return int(self._f("rng_derive")(C.c_uint64(seed), C.c_uint64(stream)))

    def rng_draws(self, seed: int, count: int, kind: str = "pm1") -> np.ndarray:
        k = {"u64": 0, "unit": 1, "pm1": 2}[kind]
        out = np.empty(count, dtype=np.uint64 if k == 0 else np.float64)
        self._f("rng_draws")(C.c_uint64(seed), C.c_int64(count), C.c_int(k), out.ctypes.data_as(C.c_void_p))
        return out

    # ----------------------------------------------------------- graph core
    def validate(self, a: CSR):
        self._check(self._f("validate")(*_csr(a)))

    def mvm(self, a: CSR, x):
        x = _f64(x)
        y = np.empty(a.n)
        self._check(self._f("mvm")(*_csr(a), _ptr(x, np.float64), _ptr(y, np.float64)))
        return y

    def residual(self, a: CSR, b, x):
        b, x = _f64(b), _f64(x)
        r = np.empty(a.n)
        self._check(self._f("residual")(*_csr(a), _ptr(b, np.float64), _ptr(x, np.float64), _ptr(r, np.float64)))
        return r

    def energy(self, a: CSR, x) -> float:
        x = _f64(x)
        e = C.c_double()
        self._check(self._f("energy")(*_csr(a), _ptr(x, np.float64), C.byref(e)))
        return e.value

    def vec_stats(self, x):
        x = _f64(x)
        s, n2 = C.c_double(), C.c_double()
        self._f("vec_stats")(C.c_int64(len(x)), _ptr(x, np.float64), C.byref(s), C.byref(n2))
        return s.value, n2.value

    def subtract_mean(self, x):
        x = _f64(x).copy()
        self._f("subtract_mean")(C.c_int64(len(x)), _ptr(x, np.float64))
        return x

    # ------------------------------------------------------------ smoothing
    def gs_sweep(self, a: CSR, b, x, backward=False):
        x = _f64(x).copy()
        bp = None if b is None else _f64(b)
        self._check(self._f("gs_sweep")(*_csr(a), None if bp is None else _ptr(bp, np.float64),
                                        _ptr(x, np.float64), C.c_int(int(backward))))
        return x

    def generate_tvs(self, a: CSR, count: int, sweeps: int, seed: int) -> np.ndarray:
        out = np.empty((count, a.n))
        self._check(self._f("generate_tvs")(*_csr(a), C.c_int(count), C.c_int(sweeps), C.c_uint64(seed),
                                            _ptr(out, np.float64)))
        return out

    def probe(self, a: CSR, sweeps: int = 8, seed: int = 7) -> float:
        f = C.c_double()
        self._check(self._f("probe")(*_csr(a), C.c_int(sweeps), C.c_uint64(seed), C.byref(f)))
        return f.value

    # ---------------------------------------------------------- aggregation
    def affinities(self, a: CSR, tvs: np.ndarray) -> dict:
        tvs = _f64(tvs)
        return self._call_bag("affinities", *_csr(a), C.c_int(tvs.shape[0]), _ptr(tvs, np.float64))

    def detect_hubs(self, a: CSR) -> np.ndarray:
        return self._call_bag("detect_hubs", *_csr(a))["hubs"]

    def energy_ratio_qus(self, a: CSR, tvs, u: int, s: int) -> float:
        tvs = _f64(tvs)
        q = C.c_double()
        self._check(self._f("energy_ratio_qus")(*_csr(a), C.c_int(tvs.shape[0]), _ptr(tvs, np.float64),
                                                C.c_int32(u), C.c_int32(s), C.byref(q)))
        return q.value

    def aggregate(self, a: CSR, tvs, gamma: float, hubs) -> dict:
        tvs, hubs = _f64(tvs), _i32(hubs)
        return self._call_bag("aggregate", *_csr(a), C.c_int(tvs.shape[0]), _ptr(tvs, np.float64),
                              C.c_double(gamma), _ptr(hubs, np.int32), C.c_int32(len(hubs)))

    def galerkin(self, a: CSR, aggregate_of, coarse_n: int) -> CSR:
        agg = _i32(aggregate_of)
        return CSR.from_bag(self._call_bag("galerkin", *_csr(a), _ptr(agg, np.int32), C.c_int32(coarse_n)))

    def restrict_residual(self, aggregate_of, coarse_n: int, r):
        agg, r = _i32(aggregate_of), _f64(r)
        rc = np.empty(coarse_n)
        self._f("restrict_residual")(_ptr(agg, np.int32), C.c_int32(len(agg)), C.c_int32(coarse_n),
                                     _ptr(r, np.float64), _ptr(rc, np.float64))
        return rc

    def add_interpolated(self, aggregate_of, ec, x):
        agg, ec = _i32(aggregate_of), _f64(ec)
        x = _f64(x).copy()
        self._f("add_interpolated")(_ptr(agg, np.int32), C.c_int32(len(agg)), _ptr(ec, np.float64),
                                    _ptr(x, np.float64))
        return x

    # ---------------------------------------------------------- elimination
    def select_low_degree(self, a: CSR, max_degree: int = 4):
        d = self._call_bag("select_low_degree", *_csr(a), C.c_int32(max_degree))
        return d["f"], d["c"]

    def schur(self, a: CSR, f, c) -> dict:
        f, c = _i32(f), _i32(c)
        return self._call_bag("schur", *_csr(a), _ptr(f, np.int32), C.c_int32(len(f)), _ptr(c, np.int32),
                              C.c_int32(len(c)))

    def eliminate_rounds(self, a: CSR) -> dict:
        return self._call_bag("eliminate_rounds", *_csr(a))

    @staticmethod
    def _stage_args(st: dict, p: str = ""):
        arrs = [
            _i32(st[p + "f_nodes"]), _f64(st[p + "f_diag"]), _i64(st[p + "f_ptr"]), _i32(st[p + "f_nbr"]),
            _f64(st[p + "f_val"]), _i32(st[p + "coarse_of_parent"]), _i32(st[p + "parent_of_coarse"]),
        ]
        dts = [np.int32, np.float64, np.int64, np.int32, np.float64, np.int32, np.int32]
        return arrs, (C.c_int32(int(st[p + "parent_n"][0])), C.c_int32(int(st[p + "coarse_n"][0])),
                      C.c_int32(len(arrs[0])), *[_ptr(x, t) for x, t in zip(arrs, dts)])

    def coarsen_rhs_stage(self, st: dict, b, p: str = ""):
        keep, args = self._stage_args(st, p)
        b = _f64(b)
        bc = np.empty(int(st[p + "coarse_n"][0]))
        self._check(self._f("coarsen_rhs_stage")(*args, _ptr(b, np.float64), _ptr(bc, np.float64)))
        return bc

    def backsub_stage(self, st: dict, xc, b, p: str = ""):
        keep, args = self._stage_args(st, p)
        xc, b = _f64(xc), _f64(b)
        x = np.empty(int(st[p + "parent_n"][0]))
        self._check(self._f("backsub_stage")(*args, _ptr(xc, np.float64), _ptr(b, np.float64), _ptr(x, np.float64)))
        return x

    # -------------------------------------------------------- coarse solver
    def coarsest_direct(self, a: CSR, b, x0=None):
        b = _f64(b)
        x = np.zeros(a.n) if x0 is None else _f64(x0).copy()
        self._check(self._f("coarsest_direct")(*_csr(a), _ptr(b, np.float64), _ptr(x, np.float64)))
        return x

    def coarsest_relax(self, a: CSR, b, x0=None):
        b = _f64(b)
        x = np.zeros(a.n) if x0 is None else _f64(x0).copy()
        self._check(self._f("coarsest_relax")(*_csr(a), _ptr(b, np.float64), _ptr(x, np.float64)))
        return x

    # ---------------------------------------------------------------- cycle
    def flat_mu(self, q: float) -> float:
        return float(self._f("flat_mu")(C.c_double(q)))

    def credit_takes(self, gamma: float, count: int):
        out = np.empty(count, dtype=np.int32)
        self._f("credit_takes")(C.c_double(gamma), C.c_int(count), _ptr(out, np.int32))
        return out

    def recombine(self, a: CSR, b, saved_x, saved_r, x):
        b = _f64(b)
        sx, sr = _f64(np.asarray(saved_x)), _f64(np.asarray(saved_r))
        x = _f64(x).copy()
        before, after = C.c_double(), C.c_double()
        self._check(self._f("recombine")(*_csr(a), _ptr(b, np.float64), C.c_int(sx.shape[0]), _ptr(sx, np.float64),
                                         _ptr(sr, np.float64), _ptr(x, np.float64), C.byref(before), C.byref(after)))
        return x, before.value, after.value

    # ------------------------------------------------------------- drivers
    def setup(self, a: CSR, gamma=1.5, seed=1, coarsest_n=150, tv_sweeps=3, tv_count_finest=4,
              tv_count_max=10) -> "OracleHierarchy":
        h = self._f("setup")(*_csr(a), C.c_double(gamma), C.c_uint64(seed), C.c_int32(coarsest_n),
                             C.c_int(tv_sweeps), C.c_int(tv_count_finest), C.c_int(tv_count_max))
        if not h:
            self._check(self._f("setup_status")() or 1)
        return OracleHierarchy(self, h, a.n)

    def prepare(self, a: CSR, gamma=1.5, seed=1, coarsest_n=150, tv_sweeps=3, tv_count_finest=4,
                tv_count_max=10, **cycle) -> "OraclePrepared":
        c = CycleCfg(**cycle)
        h = self._f("prepare")(*_csr(a), C.c_double(gamma), C.c_uint64(seed), C.c_int32(coarsest_n),
                               C.c_int(tv_sweeps), C.c_int(tv_count_finest), C.c_int(tv_count_max), *c.args())
        if not h:
            self._check(self._f("setup_status")() or 1)
        return OraclePrepared(self, h, a.n)


@dataclass
class CycleCfg:
    """lamg::CycleConfig (cycle.hpp:28-36)."""

    correction: int = 0  # 0 Flat, 1 AdaptiveRecombination
    mu: float = 4.0 / 3.0
    max_cycles: int = 300
    target_reduction: float = 1e10
    divergence_factor: float = 1e3
    gamma: float = 1.5
    seed: int = 1

    def args(self):
        return (C.c_int(self.correction), C.c_double(self.mu), C.c_int(self.max_cycles),
                C.c_double(self.target_reduction), C.c_double(self.divergence_factor), C.c_double(self.gamma),
                C.c_uint64(self.seed))


class OracleHierarchy:
    def __init__(self, o: Oracle, h, n: int):
        self.o, self.h, self.n = o, C.c_void_p(h), n

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.o._f("hier_free")(self.h)
            self.h = None

    def export(self) -> dict:
        bp = C.c_void_p()
        self.o._f("hier_export")(self.h, C.byref(bp))
        return self.o._bag(bp.value)

    def level_cycle_index(self, l: int, gamma: float) -> float:
        return float(self.o._f("level_cycle_index")(self.h, C.c_int32(l), C.c_double(gamma)))

    def solve(self, b, x0, **cycle):
        """Returns (x, stats dict). Raises OracleError; DivergedError carries .stats."""
        c = CycleCfg(**cycle)
        b, x0 = _f64(b), _f64(x0)
        x = np.empty(self.n)
        bp = C.c_void_p()
        code = self.o._f("solve")(self.h, _ptr(b, np.float64), _ptr(x0, np.float64), *c.args(),
                                  _ptr(x, np.float64), C.byref(bp))
        stats = self.o._bag(bp.value) if bp.value else {}
        if code != 0:
            err = OracleError(code, self.o._f("last_error")().decode())
            err.stats = stats
            raise err
        return x, stats

    def solve_batch(self, B, X0, nthreads: int, **cycle):
        c = CycleCfg(**cycle)
        B, X0 = _f64(B), _f64(X0)
        nrhs = B.shape[0]
        secs = C.c_double()
        cyc = np.empty(nrhs, dtype=np.int32)
        self.o._check(self.o._f("solve_batch")(self.h, C.c_int(nrhs), _ptr(B, np.float64), _ptr(X0, np.float64),
                                               *c.args(), C.c_int(nthreads), C.byref(secs), _ptr(cyc, np.int32)))
        return secs.value, cyc


class OraclePrepared:
    def __init__(self, o: Oracle, p, n: int):
        self.o, self.p, self.n = o, C.c_void_p(p), n

    def __del__(self):
        if getattr(self, "p", None) and self.p.value:
            self.o._f("prepared_free")(self.p)
            self.p = None

    def export(self) -> dict:
        bp = C.c_void_p()
        self.o._f("prepared_export")(self.p, C.byref(bp))
        return self.o._bag(bp.value)

    def solve(self, b, x0=None):
        b = _f64(b)
        x = np.empty(self.n)
        x0p = None if x0 is None else _f64(x0)
        bp = C.c_void_p()
        code = self.o._f("solve_prepared")(self.p, _ptr(b, np.float64),
                                           None if x0p is None else _ptr(x0p, np.float64),
                                           _ptr(x, np.float64), C.byref(bp))
        rep = self.o._bag(bp.value) if bp.value else {}
        if code != 0:
            err = OracleError(code, self.o._f("last_error")().decode())
            err.report = rep
            raise err
        return x, rep


def ref_generator(o: Oracle, name: str, p0: int, p1: float = 0.0, p2: float = 0.0, p3: int = 0) -> CSR:
    """Reference generator output (oracle/_ref only): pins graphs.py."""
    assert o.which == "ref"
    return CSR.from_bag(o._call_bag("gen", name.encode(), C.c_int32(p0), C.c_double(p1), C.c_double(p2),
                                    C.c_int32(p3)))


def ref_assemble(o: Oracle, n: int, u, v, w) -> CSR:
    assert o.which == "ref"
    u, v, w = _i32(u), _i32(v), _f64(w)
    return CSR.from_bag(o._call_bag("assemble", C.c_int32(n), C.c_int64(len(u)), _ptr(u, np.int32),
                                    _ptr(v, np.int32), _ptr(w, np.float64)))
