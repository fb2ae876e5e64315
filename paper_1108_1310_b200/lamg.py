"""Python mirror of the reference LAMG interface, backed by liblamg_b200.so.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/core/include/lamg/*.hpp):

* ``setup(a, SetupOptions)`` -> ``Hierarchy``            (hierarchy.hpp:65)
* ``solve(h, b, x0, CycleConfig)`` -> ``(x, SolveStats)`` (cycle.hpp:58-59)
* ``hierarchy_stats(h)``, ``level_cycle_index(h, l, g)``  (hierarchy.hpp:86,91)
* exceptions ``EmptyGraphError``, ``SingularDiagonalError``,
  ``InvalidLaplacianError``, ``DimensionMismatchError``,
  ``IncompatibleRhsError``, ``DivergedError`` (errors.hpp:13-42,
  cycle.hpp:50-53), raised with the reference's message text.

``Kernels`` exposes the per-kernel C-ABI entry points with the same method
names as the CPU oracle, so the parity tests drive both interchangeably.
Every call runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graphs import SparseLaplacian

MODE_VALIDATE = 0
MODE_THROUGHPUT = 1


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    kind = "Error"

    def __init__(self, msg: str):
        super().__init__(f"{self.kind}: {msg}")
        self.msg = msg


class EmptyGraphError(Error):
    kind = "EmptyGraphError"


class SingularDiagonalError(Error):
    kind = "SingularDiagonalError"


class InvalidLaplacianError(Error):
    kind = "InvalidLaplacianError"


class DimensionMismatchError(Error):
    kind = "DimensionMismatchError"


class IncompatibleRhsError(Error):
    kind = "IncompatibleRhsError"


class DivergedError(Error):
    kind = "DivergedError"

    def __init__(self, msg: str, stats=None):
        super().__init__(msg)
        self.stats = stats


class CudaError(Error):
    kind = "CudaError"


class ParseError(Error):
    kind = "ParseError"


class IoError(Error):
    kind = "IoError"


_CODES = {1: Error, 2: EmptyGraphError, 3: SingularDiagonalError, 4: InvalidLaplacianError,
          5: DimensionMismatchError, 6: IncompatibleRhsError, 7: DivergedError, 8: ParseError, 9: IoError,
          10: CudaError, 11: Error, 12: Error}


def _check(code: int):
    if code != 0:
        msg = _lib.lib().lamg_last_error().decode()
        raise _CODES.get(code, Error)(msg)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class _CSRArg:
    """Keeps the arrays alive while a lamg_csr points at them."""

    def __init__(self, a):
        self.rp, self.col = _i64(a.row_ptr), _i32(a.col)
        self.val, self.diag = _f64(a.val), _f64(a.diag)
        self.s = _lib.lamg_csr(int(a.n), int(a.m), _p(self.rp), _p(self.col), _p(self.val), _p(self.diag))

    def ref(self):
        return C.byref(self.s)


# ------------------------------------------------------------ public types
@dataclass
class SetupOptions:
    """lamg::SetupOptions (hierarchy.hpp:52-59)."""

    gamma: float = 1.5
    rng_seed: int = 1
    coarsest_n: int = 150
    tv_sweeps: int = 3
    tv_count_finest: int = 4
    tv_count_max: int = 10

    def c(self):
        return _lib.lamg_setup_opts(self.gamma, self.rng_seed, self.coarsest_n, self.tv_sweeps,
                                    self.tv_count_finest, self.tv_count_max)


FLAT, ADAPTIVE_RECOMBINATION = 0, 1


@dataclass
class CycleConfig:
    """lamg::CycleConfig (cycle.hpp:28-36); correction 0 Flat, 1 AdaptiveRecombination."""

    gamma: float = 1.5
    correction: int = FLAT
    mu: float = 4.0 / 3.0
    max_cycles: int = 300
    target_reduction: float = 1e10
    divergence_factor: float = 1e3
    rng_seed: int = 1

    def c(self):
        return _lib.lamg_cycle_cfg(self.gamma, self.correction, self.mu, self.max_cycles,
                                   self.target_reduction, self.divergence_factor, self.rng_seed)


@dataclass
class SolveStats:
    """lamg::SolveStats (cycle.hpp:38-46)."""

    residuals: list = field(default_factory=list)
    acf: float = 0.0
    solve_work: float = 0.0
    cycles: int = 0
    converged: bool = False
    recombinations: int = 0
    recomb_max_growth: float = 0.0
    relax_sweeps: int = 0

    def as_dict(self):
        return {"residuals": np.asarray(self.residuals, dtype=np.float64), "acf": np.array([self.acf]),
                "solve_work": np.array([self.solve_work]), "cycles": np.array([self.cycles], np.int32),
                "converged": np.array([int(self.converged)], np.int32),
                "recombinations": np.array([self.recombinations], np.int64),
                "recomb_max_growth": np.array([self.recomb_max_growth])}


class Context:
    """One device + one CUDA stream (lamg_ctx)."""

    def __init__(self, device: int = 0, mode: int = MODE_VALIDATE):
        self.lib = _lib.lib()
        self.p = C.c_void_p()
        _check(self.lib.lamg_ctx_create(C.c_int(device), C.c_int(mode), C.byref(self.p)))
        self.mode = mode

    def set_exact_levels(self, levels: int):
        """THROUGHPUT one-column solves: finest levels swept in the reference's exact order."""
        _check(self.lib.lamg_ctx_set_exact_levels(self.p, C.c_int32(levels)))

    def set_mode(self, mode: int):
        _check(self.lib.lamg_ctx_set_mode(self.p, C.c_int(mode)))
        self.mode = mode

    def close(self):
        if getattr(self, "p", None) and self.p.value:
            self.lib.lamg_ctx_destroy(self.p)
            self.p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0, MODE_VALIDATE)
    return _default_ctx


@dataclass
class LevelInfo:
    kind: int
    n: int
    m: int
    gamma: float
    nu_pre: int
    nu_post: int
    tv_count: int
    coarsest: int
    nstages: int
    coarse_n: int
    alpha: float
    stage_used: int
    dummy_aggregate: int
    gs_fronts: int
    colors: int = 0


class Hierarchy:
    """Device-resident lamg::Hierarchy (hierarchy.hpp:39-50)."""

    def __init__(self, ctx: Context, handle: C.c_void_p, n: int):
        self.ctx, self.h, self.n = ctx, handle, n
        lib = ctx.lib
        nl, nw = C.c_int32(), C.c_int32()
        sw, ss = C.c_double(), C.c_double()
        _check(lib.lamg_hier_info(self.h, C.byref(nl), C.byref(sw), C.byref(nw), C.byref(ss)))
        self.nlevels, self.setup_work, self.setup_seconds = nl.value, sw.value, ss.value
        self.warnings = []
        for i in range(nw.value):
            buf = C.create_string_buffer(512)
            _check(lib.lamg_hier_warning(self.h, C.c_int32(i), buf, C.c_int32(512)))
            self.warnings.append(buf.value.decode())
        self.levels = [self.level_info(l) for l in range(self.nlevels)]

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                self.ctx.lib.lamg_hier_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def level_info(self, l: int) -> LevelInfo:
        li = _lib.lamg_level_info()
        _check(self.ctx.lib.lamg_hier_level_info(self.h, C.c_int32(l), C.byref(li)))
        return LevelInfo(li.kind, li.n, li.m, li.gamma, li.nu_pre, li.nu_post, li.tv_count, li.coarsest,
                         li.nstages, li.coarse_n, li.alpha, li.stage_used, li.dummy_aggregate, li.gs_fronts,
                         li.colors)

    def op(self, l: int) -> SparseLaplacian:
        li = self.levels[l]
        rp = np.empty(li.n + 1, np.int64)
        col = np.empty(2 * li.m, np.int32)
        val = np.empty(2 * li.m)
        diag = np.empty(li.n)
        _check(self.ctx.lib.lamg_hier_download_op(self.h, C.c_int32(l), _p(rp), _p(col), _p(val), _p(diag)))
        return SparseLaplacian(li.n, li.m, rp, col, val, diag)

    def level_cycle_index(self, l: int, gamma: float) -> float:
        out = C.c_double()
        _check(self.ctx.lib.lamg_level_cycle_index(self.h, C.c_int32(l), C.c_double(gamma), C.byref(out)))
        return out.value

    def export(self) -> dict:
        """All artefacts with the oracle's key names (oracle_api.h hier_export)."""
        lib = self.ctx.lib
        d = {"nlevels": np.array([self.nlevels], np.int32), "setup_work": np.array([self.setup_work]),
             "nwarnings": np.array([len(self.warnings)], np.int32)}
        for l, li in enumerate(self.levels):
            p = f"L{l}."
            a = self.op(l)
            d[p + "kind"] = np.array([li.kind], np.int32)
            d[p + "n"] = np.array([a.n], np.int32)
            d[p + "m"] = np.array([a.m], np.int64)
            d[p + "row_ptr"], d[p + "col"], d[p + "val"], d[p + "diag"] = a.row_ptr, a.col, a.val, a.diag
            d[p + "gamma"] = np.array([li.gamma])
            d[p + "nu_pre"] = np.array([li.nu_pre], np.int32)
            d[p + "nu_post"] = np.array([li.nu_post], np.int32)
            d[p + "tv_count"] = np.array([li.tv_count], np.int32)
            d[p + "coarsest"] = np.array([li.coarsest], np.int32)
            if li.kind == 2:
                agg = np.empty(self.levels[l - 1].n, np.int32)
                seed = np.empty(max(li.coarse_n, 1), np.int32)
                _check(lib.lamg_hier_download_agg(self.h, C.c_int32(l), _p(agg), _p(seed)))
                d[p + "aggregate_of"], d[p + "seed_of"] = agg, seed[:li.coarse_n]
                d[p + "coarse_n"] = np.array([li.coarse_n], np.int32)
                d[p + "alpha"] = np.array([li.alpha])
                d[p + "stage_used"] = np.array([li.stage_used], np.int32)
                d[p + "dummy_aggregate"] = np.array([li.dummy_aggregate], np.int32)
            if li.kind == 1:
                d[p + "nstages"] = np.array([li.nstages], np.int32)
                for s in range(li.nstages):
                    pn, cn, nf, nz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
                    _check(lib.lamg_hier_stage_info(self.h, C.c_int32(l), C.c_int32(s), C.byref(pn), C.byref(cn),
                                                    C.byref(nf), C.byref(nz)))
                    arr = dict(f_nodes=np.empty(nf.value, np.int32), f_diag=np.empty(nf.value),
                               f_ptr=np.empty(nf.value + 1, np.int64), f_nbr=np.empty(nz.value, np.int32),
                               f_val=np.empty(nz.value), coarse_of_parent=np.empty(pn.value, np.int32),
                               parent_of_coarse=np.empty(cn.value, np.int32))
                    _check(lib.lamg_hier_download_stage(self.h, C.c_int32(l), C.c_int32(s),
                                                        *[_p(arr[k]) for k in ("f_nodes", "f_diag", "f_ptr", "f_nbr",
                                                                               "f_val", "coarse_of_parent",
                                                                               "parent_of_coarse")]))
                    ps = f"{p}S{s}."
                    d[ps + "parent_n"] = np.array([pn.value], np.int32)
                    d[ps + "coarse_n"] = np.array([cn.value], np.int32)
                    for k, v in arr.items():
                        d[ps + k] = v
        return d

    def prepare_throughput(self):
        """Builds the THROUGHPUT smoother data once (colourings, permuted copies)."""
        _check(self.ctx.lib.lamg_hier_prepare_throughput(self.ctx.p, self.h))
        self.levels = [self.level_info(l) for l in range(self.nlevels)]

    def colors(self, l: int):
        """(row_ids, color_ptr) of level l's coloured smoother: stored row -> natural row."""
        nc = C.c_int32()
        _check(self.ctx.lib.lamg_hier_color_count(self.h, C.c_int32(l), C.byref(nc)))
        rows = np.empty(self.levels[l].n, np.int32)
        ptr = np.empty(nc.value + 1, np.int32)
        _check(self.ctx.lib.lamg_hier_download_colors(self.h, C.c_int32(l), _p(rows), _p(ptr)))
        return rows, ptr

    def smooth(self, l: int, b, x, sweeps: int = 1):
        """`sweeps` THROUGHPUT coloured Gauss-Seidel sweeps on level l; b, x are [n] or node-major [n, K]."""
        b, x = np.ascontiguousarray(b, np.float64), np.array(x, np.float64, order="C")
        k = 1 if x.ndim == 1 else x.shape[1]
        _check(self.ctx.lib.lamg_hier_smooth(self.ctx.p, self.h, C.c_int32(l), C.c_int32(k), _p(b), _p(x),
                                             C.c_int32(sweeps)))
        return x

    def smooth_exact(self, l: int, b, x, sweeps: int = 1):
        """`sweeps` Gauss-Seidel sweeps on level l in the reference's row order; b, x are [n] or node-major [n, K]."""
        b, x = np.ascontiguousarray(b, np.float64), np.array(x, np.float64, order="C")
        k = 1 if x.ndim == 1 else x.shape[1]
        _check(self.ctx.lib.lamg_hier_smooth_exact(self.ctx.p, self.h, C.c_int32(l), C.c_int32(k), _p(b), _p(x),
                                                   C.c_int32(sweeps)))
        return x

    def solve(self, b, x0, **cycle):
        """Oracle-style solve: returns (x, stats dict); errors carry .stats."""
        cfg = CycleConfig(**{k: v for k, v in cycle.items() if k != "seed"})
        x, st = solve(self, b, x0, cfg)
        return x, st.as_dict()


# ---------------------------------------------------------------- drivers
def setup(a, opts: SetupOptions | None = None, ctx: Context | None = None, seed: int | None = None,
          **kw) -> Hierarchy:
    """lamg::setup (hierarchy.hpp:65) on the GPU. `a` is a host CSR or a
    DeviceGraph (already in HBM)."""
    ctx = ctx or default_context()
    opts = opts or SetupOptions(**kw)
    if seed is not None:
        opts.rng_seed = seed
    h = C.c_void_p()
    o = opts.c()
    if isinstance(a, DeviceGraph):
        _check(ctx.lib.lamg_setup(ctx.p, C.byref(a.csr), C.c_int(1), C.byref(o), C.byref(h)))
    else:
        arg = _CSRArg(a)
        _check(ctx.lib.lamg_setup(ctx.p, arg.ref(), C.c_int(0), C.byref(o), C.byref(h)))
    return Hierarchy(ctx, h, int(a.n))


class DeviceGraph:
    """A CSR Laplacian resident in HBM (lamg_graph): the output of the device
    generators / component extraction (gen.cu)."""

    def __init__(self, ctx: Context, g):
        self.ctx, self.g = ctx, g
        self.csr = _lib.lamg_csr()
        _check(ctx.lib.lamg_graph_csr(g, C.byref(self.csr)))
        self.n, self.m = int(self.csr.n), int(self.csr.m)

    def download(self):
        """Host copy with the SparseLaplacian field names."""
        from .graphs import SparseLaplacian
        rp = np.empty(self.n + 1, dtype=np.int64)
        col = np.empty(2 * self.m, dtype=np.int32)
        val = np.empty(2 * self.m)
        diag = np.empty(self.n)
        _check(self.ctx.lib.lamg_graph_download(self.g, _p(rp), _p(col), _p(val), _p(diag)))
        return SparseLaplacian(self.n, self.m, rp, col, val, diag)

    def close(self):
        if self.g:
            self.ctx.lib.lamg_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


def gen_rmat(scale: int, seed: int = 5, edge_factor: int = 16, abcd=(0.57, 0.19, 0.19, 0.05), lcc: bool = True,
             ctx: Context | None = None) -> DeviceGraph:
    """BASELINE config 5 generator on the device; bit-identical to graphs.rmat."""
    ctx = ctx or default_context()
    a, b, c, _ = abcd
    g = C.c_void_p()
    _check(ctx.lib.lamg_gen_rmat(ctx.p, C.c_int32(scale), C.c_int32(edge_factor), C.c_double(a), C.c_double(b),
                                 C.c_double(c), C.c_uint64(seed), C.c_int32(int(lcc)), C.byref(g)))
    return DeviceGraph(ctx, g)


def gen_chung_lu(n: int, seed: int = 4, beta: float = 2.1, mean_degree: float = 16.0, lcc: bool = True,
                 ctx: Context | None = None) -> DeviceGraph:
    """BASELINE config 4 generator on the device; bit-identical to graphs.chung_lu.

    The expected-degree CDF and the pair count are numpy's (pairwise mean,
    sequential cumsum), exactly as graphs.chung_lu forms them.
    """
    ctx = ctx or default_context()
    wi = (np.arange(n) + 1.0) ** (-1.0 / (beta - 1.0))
    wi *= mean_degree / wi.mean()
    wi = np.maximum(wi, 1.0)
    cdf = np.cumsum(wi)
    cdf /= cdf[-1]
    pairs = int(wi.sum() // 2)
    g = C.c_void_p()
    _check(ctx.lib.lamg_gen_chung_lu(ctx.p, C.c_int32(n), _p(cdf), C.c_int64(pairs), C.c_uint64(seed),
                                     C.c_int32(int(lcc)), C.byref(g)))
    return DeviceGraph(ctx, g)


def largest_component(a, ctx: Context | None = None) -> DeviceGraph:
    """graphs.largest_component on the device (union-find, ascending order)."""
    ctx = ctx or default_context()
    arg = _CSRArg(a)
    g = C.c_void_p()
    _check(ctx.lib.lamg_graph_lcc(ctx.p, arg.ref(), C.c_int(0), C.byref(g)))
    return DeviceGraph(ctx, g)


def solve(h: Hierarchy, b, x0, cfg: CycleConfig | None = None, ctx: Context | None = None):
    """lamg::solve (cycle.hpp:58-59): returns (x, SolveStats)."""
    ctx = ctx or h.ctx
    cfg = cfg or CycleConfig()
    b, x0 = _f64(b), _f64(x0)
    if len(b) != h.n or len(x0) != h.n:
        raise DimensionMismatchError("solve: vector length does not match the finest level")
    x = np.empty(h.n)
    st = _lib.lamg_solve_stats()
    cap = cfg.max_cycles + 2
    res = np.empty(cap)
    c = cfg.c()
    code = ctx.lib.lamg_solve(ctx.p, h.h, _p(b), _p(x0), C.byref(c), _p(x), C.byref(st), _p(res), C.c_int32(cap))
    stats = SolveStats(list(res[:min(st.nresiduals, cap)]), st.acf, st.solve_work, st.cycles, bool(st.converged),
                       st.recombinations, st.recomb_max_growth, st.relax_sweeps)
    if code == 7:
        raise DivergedError(_lib.lib().lamg_last_error().decode(), stats.as_dict())
    _check(code)
    return x, stats


def solve_batch(h: Hierarchy, B, X0, cfg: CycleConfig | None = None, ctx: Context | None = None):
    """nrhs independent solves (one lamg::solve per row of B, cycle.cpp:221-273).

    B and X0 are [nrhs, n]. THROUGHPUT mode runs blocks of up to 128 columns
    through one cycle schedule (lamg_solve_batch); VALIDATE mode solves each
    column in the reference's order. Returns (X [nrhs, n], [SolveStats]).
    """
    ctx = ctx or h.ctx
    cfg = cfg or CycleConfig()
    B, X0 = np.ascontiguousarray(B, dtype=np.float64), np.ascontiguousarray(X0, dtype=np.float64)
    if B.ndim != 2 or B.shape != X0.shape or B.shape[1] != h.n:
        raise DimensionMismatchError("solve_batch: B and X0 must be [nrhs, n] with n the finest size")
    nrhs = B.shape[0]
    X = np.empty_like(B)
    st = (_lib.lamg_solve_stats * max(nrhs, 1))()
    cap = cfg.max_cycles + 2
    res = np.empty((max(nrhs, 1), cap))
    c = cfg.c()
    code = ctx.lib.lamg_solve_batch(ctx.p, h.h, C.c_int32(nrhs), _p(B), _p(X0), C.byref(c), _p(X), st, _p(res),
                                    C.c_int32(cap))
    stats = [SolveStats(list(res[j, :min(st[j].nresiduals, cap)]), st[j].acf, st[j].solve_work, st[j].cycles,
                        bool(st[j].converged), st[j].recombinations, st[j].recomb_max_growth, st[j].relax_sweeps)
             for j in range(nrhs)]
    if code == 7:
        raise DivergedError(_lib.lib().lamg_last_error().decode(), [s.as_dict() for s in stats])
    _check(code)
    return X, stats


def level_cycle_index(h: Hierarchy, l: int, gamma: float) -> float:
    return h.level_cycle_index(l, gamma)


def hierarchy_stats(h: Hierarchy) -> dict:
    """lamg::hierarchy_stats (hierarchy.cpp:140-168)."""
    kinds = {0: "finest", 1: "elimination", 2: "aggregation", 3: "coarsest"}
    levels = []
    m1 = h.levels[0].m
    for l, li in enumerate(h.levels):
        coarsest = li.coarsest != 0
        kind = kinds[li.kind]
        if li.kind == 0 and coarsest:
            kind = "coarsest"
        nxt = h.levels[l + 1] if l + 1 < h.nlevels else None
        levels.append({"level": l + 1, "kind": kind, "coarsest": coarsest, "n": li.n, "m": li.m,
                       "gamma": nxt.gamma if nxt else 0.0, "nu_pre": 1 if nxt and nxt.kind == 2 else 0,
                       "nu_post": 2 if nxt and nxt.kind == 2 else 0, "tv_count": li.tv_count})
    edges = sum(li.m for li in h.levels)
    storage = sum(2.0 * li.m + li.n for li in h.levels)
    return {"levels": levels, "edge_ratio": edges / m1, "storage_per_edge": storage / m1,
            "setup_work": h.setup_work}


# ------------------------------------------------------- per-kernel API
class Kernels:
    """Per-kernel C-ABI entry points with the oracle's method names."""

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib

    def _c(self, code):
        _check(code)

    def validate(self, a):
        arg = _CSRArg(a)
        self._c(self.lib.lamg_k_validate(self.ctx.p, arg.ref()))

    def mvm(self, a, x):
        arg, x = _CSRArg(a), _f64(x)
        y = np.empty(a.n)
        self._c(self.lib.lamg_k_mvm(self.ctx.p, arg.ref(), _p(x), _p(y)))
        return y

    def residual(self, a, b, x):
        arg, b, x = _CSRArg(a), _f64(b), _f64(x)
        r = np.empty(a.n)
        self._c(self.lib.lamg_k_residual(self.ctx.p, arg.ref(), _p(b), _p(x), _p(r)))
        return r

    def energy(self, a, x) -> float:
        arg, x = _CSRArg(a), _f64(x)
        e = C.c_double()
        self._c(self.lib.lamg_k_energy(self.ctx.p, arg.ref(), _p(x), C.byref(e)))
        return e.value

    def gs_sweep(self, a, b, x, backward=False):
        arg = _CSRArg(a)
        x = _f64(x).copy()
        bb = None if b is None else _f64(b)
        self._c(self.lib.lamg_k_gs_sweep(self.ctx.p, arg.ref(), None if bb is None else _p(bb), _p(x),
                                         C.c_int(int(backward))))
        return x

    def generate_tvs(self, a, count, sweeps, seed):
        arg = _CSRArg(a)
        out = np.empty((count, a.n))
        self._c(self.lib.lamg_k_generate_tvs(self.ctx.p, arg.ref(), C.c_int32(count), C.c_int32(sweeps),
                                             C.c_uint64(seed), _p(out)))
        return out

    def probe(self, a, sweeps=8, seed=7):
        arg = _CSRArg(a)
        f = C.c_double()
        self._c(self.lib.lamg_k_probe(self.ctx.p, arg.ref(), C.c_int32(sweeps), C.c_uint64(seed), C.byref(f)))
        return f.value

    def affinities(self, a, tvs):
        arg, tvs = _CSRArg(a), _f64(tvs)
        K = tvs.shape[0]
        aff, nn = np.empty(2 * a.m), np.empty(a.n)
        deg, nd = np.empty(max(a.n, 1), np.int32), C.c_int32()
        self._c(self.lib.lamg_k_affinities(self.ctx.p, arg.ref(), C.c_int32(K), _p(tvs), _p(aff), _p(nn), _p(deg),
                                           C.byref(nd)))
        return {"edge_affinity": aff, "node_norm": nn, "degenerate": deg[:nd.value]}

    def detect_hubs(self, a):
        arg = _CSRArg(a)
        hubs, nh = np.empty(max(a.n, 1), np.int32), C.c_int32()
        self._c(self.lib.lamg_k_detect_hubs(self.ctx.p, arg.ref(), _p(hubs), C.byref(nh)))
        return hubs[:nh.value]

    def aggregate(self, a, tvs, gamma, hubs):
        arg, tvs, hubs = _CSRArg(a), _f64(tvs), _i32(hubs)
        agg, seed = np.empty(a.n, np.int32), np.empty(max(a.n, 1), np.int32)
        cn, al, su, dm = C.c_int32(), C.c_double(), C.c_int32(), C.c_int32()
        self._c(self.lib.lamg_k_aggregate(self.ctx.p, arg.ref(), C.c_int32(tvs.shape[0]), _p(tvs), C.c_double(gamma),
                                          _p(hubs), C.c_int32(len(hubs)), _p(agg), _p(seed), C.byref(cn),
                                          C.byref(al), C.byref(su), C.byref(dm)))
        return {"aggregate_of": agg, "seed_of": seed[:cn.value], "coarse_n": np.array([cn.value], np.int32),
                "alpha": np.array([al.value]), "stage_used": np.array([su.value], np.int32),
                "dummy_aggregate": np.array([dm.value], np.int32)}

    def _take_csr(self):
        n, m, nz = C.c_int32(), C.c_int64(), C.c_int64()
        self._c(self.lib.lamg_k_result_dims(self.ctx.p, C.byref(n), C.byref(m), C.byref(nz)))
        rp, col = np.empty(n.value + 1, np.int64), np.empty(2 * m.value, np.int32)
        val, diag = np.empty(2 * m.value), np.empty(n.value)
        self._c(self.lib.lamg_k_take_csr(self.ctx.p, _p(rp), _p(col), _p(val), _p(diag)))
        return SparseLaplacian(n.value, m.value, rp, col, val, diag), nz.value

    def galerkin(self, a, aggregate_of, coarse_n):
        arg, agg = _CSRArg(a), _i32(aggregate_of)
        self._c(self.lib.lamg_k_galerkin(self.ctx.p, arg.ref(), _p(agg), C.c_int32(coarse_n)))
        return self._take_csr()[0]

    def select_low_degree(self, a, max_degree=4):
        arg = _CSRArg(a)
        f, c = np.empty(max(a.n, 1), np.int32), np.empty(max(a.n, 1), np.int32)
        nf, nc = C.c_int32(), C.c_int32()
        self._c(self.lib.lamg_k_select_low_degree(self.ctx.p, arg.ref(), C.c_int32(max_degree), _p(f), C.byref(nf),
                                                  _p(c), C.byref(nc)))
        return f[:nf.value], c[:nc.value]

    def schur(self, a, f, c):
        arg, f, c = _CSRArg(a), _i32(f), _i32(c)
        self._c(self.lib.lamg_k_schur(self.ctx.p, arg.ref(), _p(f), C.c_int32(len(f)), _p(c), C.c_int32(len(c)),
                                      None))
        coarse, nnz = self._take_csr()
        nf = len(f)
        fd, fp = np.empty(max(nf, 1)), np.empty(nf + 1, np.int64)
        fn, fv, cop = np.empty(max(nnz, 1), np.int32), np.empty(max(nnz, 1)), np.empty(a.n, np.int32)
        self._c(self.lib.lamg_k_take_stage(self.ctx.p, _p(fd), _p(fp), _p(fn), _p(fv), _p(cop)))
        d = {"n": np.array([coarse.n], np.int32), "m": np.array([coarse.m], np.int64), "row_ptr": coarse.row_ptr,
             "col": coarse.col, "val": coarse.val, "diag": coarse.diag,
             "S.parent_n": np.array([a.n], np.int32), "S.coarse_n": np.array([len(c)], np.int32),
             "S.f_nodes": f.copy(), "S.f_diag": fd[:nf], "S.f_ptr": fp, "S.f_nbr": fn[:nnz], "S.f_val": fv[:nnz],
             "S.coarse_of_parent": cop, "S.parent_of_coarse": c.copy()}
        return d

    def eliminate_rounds(self, a):
        """Stage-by-stage restatement of eliminate_rounds through the kernels."""
        out = {"nstages": np.array([0], np.int32)}
        cur = a
        s = 0
        while cur.n > 1:
            f, c = self.select_low_degree(cur, 4)
            if len(f) < 0.01 * cur.n or len(f) == 0 or len(c) == 0:
                break
            d = self.schur(cur, f, c)
            for k, v in d.items():
                if k.startswith("S."):
                    out[f"S{s}." + k[2:]] = v
            cur = SparseLaplacian(int(d["n"][0]), int(d["m"][0]), d["row_ptr"], d["col"], d["val"], d["diag"])
            s += 1
        out["nstages"] = np.array([s], np.int32)
        if s:
            out.update({"n": np.array([cur.n], np.int32), "m": np.array([cur.m], np.int64),
                        "row_ptr": cur.row_ptr, "col": cur.col, "val": cur.val, "diag": cur.diag})
        return out

    def _stage_args(self, st, p=""):
        arrs = [_i32(st[p + "f_nodes"]), _f64(st[p + "f_diag"]), _i64(st[p + "f_ptr"]), _i32(st[p + "f_nbr"]),
                _f64(st[p + "f_val"]), _i32(st[p + "coarse_of_parent"]), _i32(st[p + "parent_of_coarse"])]
        return arrs, (C.c_int32(int(st[p + "parent_n"][0])), C.c_int32(int(st[p + "coarse_n"][0])),
                      C.c_int32(len(arrs[0])), *[_p(x) for x in arrs])

    def coarsen_rhs_stage(self, st, b, p=""):
        keep, args = self._stage_args(st, p)
        b = _f64(b)
        bc = np.empty(int(st[p + "coarse_n"][0]))
        self._c(self.lib.lamg_k_coarsen_rhs(self.ctx.p, *args, _p(b), _p(bc)))
        return bc

    def backsub_stage(self, st, xc, b, p=""):
        keep, args = self._stage_args(st, p)
        xc, b = _f64(xc), _f64(b)
        x = np.empty(int(st[p + "parent_n"][0]))
        self._c(self.lib.lamg_k_backsub(self.ctx.p, *args, _p(xc), _p(b), _p(x)))
        return x

    def restrict_residual(self, aggregate_of, coarse_n, r):
        agg, r = _i32(aggregate_of), _f64(r)
        rc = np.empty(coarse_n)
        self._c(self.lib.lamg_k_restrict(self.ctx.p, _p(agg), C.c_int32(len(agg)), C.c_int32(coarse_n), _p(r),
                                         _p(rc)))
        return rc

    def add_interpolated(self, aggregate_of, ec, x):
        agg, ec = _i32(aggregate_of), _f64(ec)
        x = _f64(x).copy()
        self._c(self.lib.lamg_k_interpolate(self.ctx.p, _p(agg), C.c_int32(len(agg)), C.c_int32(len(ec)), _p(ec),
                                            _p(x)))
        return x

    def coarsest_direct(self, a, b, x0=None):
        arg, b = _CSRArg(a), _f64(b)
        x = np.zeros(a.n) if x0 is None else _f64(x0).copy()
        self._c(self.lib.lamg_k_coarsest_direct(self.ctx.p, arg.ref(), _p(b), _p(x)))
        return x

    def coarsest_relax(self, a, b, x0=None):
        arg, b = _CSRArg(a), _f64(b)
        x = np.zeros(a.n) if x0 is None else _f64(x0).copy()
        self._c(self.lib.lamg_k_coarsest_relax(self.ctx.p, arg.ref(), _p(b), _p(x)))
        return x

    def recombine(self, a, b, saved_x, saved_r, x):
        arg, b = _CSRArg(a), _f64(b)
        sx, sr = _f64(np.asarray(saved_x)), _f64(np.asarray(saved_r))
        x = _f64(x).copy()
        before, after = C.c_double(), C.c_double()
        self._c(self.lib.lamg_k_recombine(self.ctx.p, arg.ref(), _p(b), C.c_int32(sx.shape[0]), _p(sx), _p(sr),
                                          _p(x), C.byref(before), C.byref(after)))
        return x, before.value, after.value

    def flat_mu(self, q):
        return float(self.lib.lamg_flat_mu(C.c_double(q)))

    def credit_takes(self, gamma, count):
        out = np.empty(count, np.int32)
        self.lib.lamg_credit_takes(C.c_double(gamma), C.c_int32(count), _p(out))
        return out

    def rng_derive(self, seed, stream):
        return int(self.lib.lamg_rng_derive(C.c_uint64(seed), C.c_uint64(stream)))

    def setup(self, a, gamma=1.5, seed=1, coarsest_n=150, tv_sweeps=3, tv_count_finest=4, tv_count_max=10):
        return setup(a, SetupOptions(gamma, seed, coarsest_n, tv_sweeps, tv_count_finest, tv_count_max), ctx=self.ctx)


# ------------------------------------------------ fine-level partition (8(e) mode 2)
def part_bounds(a, nparts: int) -> np.ndarray:
    """Contiguous row blocks balanced by rows + entries (host only)."""
    rp = _i64(a.row_ptr)
    out = np.empty(nparts + 1, np.int32)
    _check(_lib.lib().lamg_part_bounds(C.c_int32(a.n), _p(rp), C.c_int32(nparts), _p(out)))
    return out


def part_plan(a, bounds, part: int) -> dict:
    """Local CSR, ghosts and send/recv lists of one part (host only)."""
    arg, bounds = _CSRArg(a), _i32(bounds)
    P = len(bounds) - 1
    nloc, ngh, nsend, nnz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
    lib = _lib.lib()
    _check(lib.lamg_part_plan_sizes(arg.ref(), _p(bounds), C.c_int32(P), C.c_int32(part), C.byref(nloc),
                                    C.byref(ngh), C.byref(nnz), C.byref(nsend)))
    d = dict(row_ptr=np.empty(nloc.value + 1, np.int64), col=np.empty(nnz.value, np.int32),
             ghost_gid=np.empty(ngh.value, np.int32), recv_ptr=np.empty(P + 1, np.int32),
             send_ptr=np.empty(P + 1, np.int32), send_idx=np.empty(nsend.value, np.int32))
    _check(lib.lamg_part_plan(arg.ref(), _p(bounds), C.c_int32(P), C.c_int32(part),
                              *[_p(d[k]) for k in ("row_ptr", "col", "ghost_gid", "recv_ptr", "send_ptr",
                                                   "send_idx")]))
    d["lo"], d["hi"] = int(bounds[part]), int(bounds[part + 1])
    return d


class Comm:
    """NCCL communicator for the partitioned level (one rank per GPU)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib.lib().lamg_comm_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, uid: bytes, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.nranks, self.rank = nranks, rank
        self.p = C.c_void_p()
        _check(self.ctx.lib.lamg_comm_create(self.ctx.p, C.c_int32(nranks), C.c_int32(rank),
                                             C.create_string_buffer(uid, 128), C.byref(self.p)))

    def close(self):
        if self.p and self.p.value:
            self.ctx.lib.lamg_comm_destroy(self.p)
            self.p = C.c_void_p()


class PartLevel:
    """A level operator split into row blocks with halo exchange.

    Without `comm` this process owns every part (one device); with an NCCL
    `comm` it owns part `comm rank` of `nparts`.
    """

    def __init__(self, a, nparts: int, ctx: Context | None = None, bounds=None, comm: Comm | None = None):
        self.ctx = ctx or default_context()
        self.comm = comm  # the library keeps a pointer: the communicator must outlive the partition
        self.n = a.n
        self.bounds = _i32(bounds if bounds is not None else part_bounds(a, nparts))
        arg = _CSRArg(a)
        self.p = C.c_void_p()
        first, nown = (0, nparts) if comm is None else (comm.rank, 1)
        _check(self.ctx.lib.lamg_part_level_create(self.ctx.p, arg.ref(), _p(self.bounds), C.c_int32(nparts),
                                                   C.c_int32(first), C.c_int32(nown),
                                                   comm.p if comm is not None else None, C.byref(self.p)))

    @classmethod
    def from_hierarchy(cls, h: Hierarchy, nparts: int, comm: Comm | None = None):
        """The first smoothing level of `h` (level 0, or level 1 below a finest
        elimination) split into `nparts` row blocks (lamg_part_level_from_hier)."""
        self = cls.__new__(cls)
        self.ctx, self.n = h.ctx, h.n
        self.comm, self.hier = comm, h  # both must outlive the partition
        self.p = C.c_void_p()
        first, nown = (0, nparts) if comm is None else (comm.rank, 1)
        _check(self.ctx.lib.lamg_part_level_from_hier(self.ctx.p, h.h, C.c_int32(nparts), C.c_int32(first),
                                                      C.c_int32(nown), comm.p if comm is not None else None,
                                                      C.byref(self.p)))
        self.ctx.lib.lamg_part_level_n.restype = C.c_int32
        self.n = int(self.ctx.lib.lamg_part_level_n(self.p))  # the partitioned level's size
        return self

    def solve(self, h: Hierarchy, b, x0, cfg: CycleConfig | None = None):
        """lamg_part_solve: lamg::solve with this partitioned level (the hierarchy's first smoothing level)."""
        cfg = cfg or CycleConfig()
        b, x0 = _f64(b), _f64(x0)
        x = np.empty(h.n)
        st = _lib.lamg_solve_stats()
        cap = cfg.max_cycles + 2
        res = np.empty(cap)
        c = cfg.c()
        code = self.ctx.lib.lamg_part_solve(self.ctx.p, h.h, self.p, _p(b), _p(x0), C.byref(c), _p(x), C.byref(st),
                                            _p(res), C.c_int32(cap))
        stats = SolveStats(list(res[:min(st.nresiduals, cap)]), st.acf, st.solve_work, st.cycles, bool(st.converged),
                           st.recombinations, st.recomb_max_growth, st.relax_sweeps)
        if code == 7:
            raise DivergedError(_lib.lib().lamg_last_error().decode(), stats.as_dict())
        _check(code)
        return x, stats

    def smooth(self, b, x, sweeps: int = 1):
        b, x = _f64(b), _f64(x).copy()
        _check(self.ctx.lib.lamg_part_smooth(self.p, _p(b), _p(x), C.c_int32(sweeps)))
        return x

    def residual(self, b, x):
        b, x = _f64(b), _f64(x)
        r = np.zeros(self.n)
        _check(self.ctx.lib.lamg_part_residual(self.p, _p(b), _p(x), _p(r)))
        return r

    def time(self, sweeps: int) -> float:
        ms = C.c_float()
        _check(self.ctx.lib.lamg_part_time(self.p, C.c_int32(sweeps), C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "p", None) and self.p.value:
            self.ctx.lib.lamg_part_level_destroy(self.p)
            self.p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass



# ------------------------------------------------------------ Matrix Market
_MM_KIND = {"auto": 0, "adjacency": 1, "laplacian": 2}


def read_matrix_market(path: str, kind: str = "auto", absolute_weight_policy: bool = True):
    """read_matrix_market_file + assemble_problem (matrix_market.hpp:34-45).

    Returns (SparseLaplacian, was_laplacian, warnings). Host only.
    """
    lib = _lib.lib()
    mm = C.c_void_p()
    _check(lib.lamg_mm_read(str(path).encode(), C.c_int32(_MM_KIND[kind]), C.c_int32(int(absolute_weight_policy)),
                            C.byref(mm)))
    try:
        n, m, wl, nw = C.c_int32(), C.c_int64(), C.c_int32(), C.c_int32()
        _check(lib.lamg_mm_info(mm, C.byref(n), C.byref(m), C.byref(wl), C.byref(nw)))
        rp = np.empty(n.value + 1, np.int64)
        col = np.empty(2 * m.value, np.int32)
        val = np.empty(2 * m.value)
        diag = np.empty(n.value)
        _check(lib.lamg_mm_csr(mm, _p(rp), _p(col), _p(val), _p(diag)))
        warnings = []
        for i in range(nw.value):
            buf = C.create_string_buffer(1024)
            _check(lib.lamg_mm_warning(mm, C.c_int32(i), buf, C.c_int32(1024)))
            warnings.append(buf.value.decode())
        return SparseLaplacian(n.value, m.value, rp, col, val, diag), bool(wl.value), warnings
    finally:
        lib.lamg_mm_destroy(mm)


def write_matrix_market(path: str, a, as_laplacian: bool = False):
    """write_matrix_market_file (matrix_market.hpp:47-52)."""
    arg = _CSRArg(a)
    _check(_lib.lib().lamg_mm_write(str(path).encode(), arg.ref(), C.c_int32(int(as_laplacian))))
