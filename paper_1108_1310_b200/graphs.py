"""Host-side problem construction: seeded generators, Laplacian assembly, RHS.

This is layer L4 of the reference (problem I/O and generators) restated in
numpy so both the GPU path and the CPU oracles receive the SAME arrays. It is
input preparation, not part of the timed hot path.

* ``Rng`` / ``rng_u64`` reproduce ``lamg::Rng`` (include/lamg/rng.hpp:10-41)
  bit-exactly: draw i of ``Rng(s)`` is splitmix64 at state
  ``s' + (i + 3) * golden`` (s' = s, or golden if s == 0), so whole streams
  are generated vectorised.
* ``assemble_laplacian`` follows ``assemble_laplacian``/``assemble_canonical``
  (src/sparse_laplacian.cpp:12-45, 60-135): self-loops dropped, u<v, sorted,
  duplicates merged by summing, both triangles stored, rows ascending, and
  ``diag[x]`` folded over the row in ascending column order, which is the
  order the reference's edge-ordered fill produces.
* The small generators mirror src/generators.cpp:19-127 and the test fixture
  ``random_connected`` (tests/support/test_graphs.hpp:16-38); the five
  BASELINE.json configurations follow SURVEY.md 8(d).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


@dataclass
class SparseLaplacian:
    """lamg::SparseLaplacian (include/lamg/sparse_laplacian.hpp:18-39)."""

    n: int
    m: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray  # int32[2m], strictly ascending per row
    val: np.ndarray  # float64[2m], a_uv = -w_uv
    diag: np.ndarray  # float64[n]

    def degree(self, u: int) -> int:
        return int(self.row_ptr[u + 1] - self.row_ptr[u])

    def neighbors(self, u: int) -> np.ndarray:
        return self.col[self.row_ptr[u]: self.row_ptr[u + 1]]

    def weight(self, u: int, v: int) -> float:
        nb = self.neighbors(u)
        k = int(np.searchsorted(nb, v))
        if k == len(nb) or nb[k] != v:
            return 0.0
        return float(-self.val[self.row_ptr[u] + k])

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        a[rows, self.col] = self.val
        a[np.arange(self.n), np.arange(self.n)] = self.diag
        return a


# --------------------------------------------------------------------- rng
def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def rng_u64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start..start+count-1 of lamg::Rng(seed).next_u64() (counter form)."""
    s0 = seed if seed else GOLDEN
    idx = np.arange(start + 3, start + 3 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        state = np.uint64(s0) + idx * np.uint64(GOLDEN)
        return _mix(state)


def rng_unit(seed: int, start: int, count: int) -> np.ndarray:
    return (rng_u64(seed, start, count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def rng_pm1(seed: int, start: int, count: int) -> np.ndarray:
    return 2.0 * rng_unit(seed, start, count) - 1.0


class Rng:
    """Sequential lamg::Rng for streams with data-dependent draw counts."""

    def __init__(self, seed: int):
        self.state = (seed if seed else GOLDEN) & MASK
        self.next_u64()
        self.next_u64()

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def next_pm1(self) -> float:
        return 2.0 * self.next_unit() - 1.0

    @staticmethod
    def derive(seed: int, stream: int) -> int:
        return Rng((seed ^ ((0xD1342543DE82EF95 * (stream + 1)) & MASK)) & MASK).next_u64()


# ---------------------------------------------------------------- assembly
def assemble_laplacian(n: int, u, v, w) -> SparseLaplacian:
    """sparse_laplacian.cpp:106-135 with WeightPolicy::Keep."""
    if n <= 0:
        raise ValueError("cannot assemble a Laplacian with n = 0")
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    keep = u != v
    u, v, w = u[keep], v[keep], w[keep]
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    order = np.lexsort((hi, lo))
    lo, hi, w = lo[order], hi[order], w[order]
    if len(lo):
        new = np.ones(len(lo), dtype=bool)
        new[1:] = (lo[1:] != lo[:-1]) | (hi[1:] != hi[:-1])
        starts = np.flatnonzero(new)
        if len(starts) != len(lo):  # sequential merge of duplicates
            seg = np.cumsum(new) - 1
            merged = segmented_fold(seg, np.arange(len(lo)) - starts[seg], w, len(starts))
            lo, hi, w = lo[starts], hi[starts], merged
    return assemble_canonical(n, lo, hi, w)


def segmented_fold(seg, pos, w, nseg: int) -> np.ndarray:
    """out[s] = ((0.0 + w_0) + w_1) + ... over the entries of segment s in
    position order: the reference's sequential accumulation, vectorised by
    position (O(len) work)."""
    out = np.zeros(nseg)
    if len(w) == 0:
        return out
    order = np.argsort(pos, kind="stable")
    bounds = np.searchsorted(pos[order], np.arange(int(pos.max()) + 2))
    for j in range(len(bounds) - 1):
        sl = order[bounds[j]:bounds[j + 1]]
        out[seg[sl]] += w[sl]
    return out


def assemble_canonical(n: int, u, v, w) -> SparseLaplacian:
    """sparse_laplacian.cpp:60-104 for a sorted, merged u<v edge list."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    m = len(u)
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    vals = np.concatenate([-w, -w])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    counts = np.bincount(rows, minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    # diag[x] = ((0 + w_1) + w_2) + ... in ascending column order
    diag = segmented_fold(rows, np.arange(len(rows)) - row_ptr[rows], -vals, n)
    return SparseLaplacian(n, m, row_ptr, cols.astype(np.int32), vals.astype(np.float64), diag)


def largest_component(a: SparseLaplacian) -> tuple[SparseLaplacian, np.ndarray]:
    """Keeps the largest connected component (ascending node order, as
    components.cpp:35-56 extract_component does). Returns (sub, nodes)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    n = a.n
    g = csr_matrix((np.ones(len(a.col)), a.col, a.row_ptr), shape=(n, n))
    _, label = connected_components(g, directed=False)
    label = label.astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.row_ptr))
    cols = a.col.astype(np.int64)
    counts = np.bincount(label, minlength=n)
    big = int(np.argmax(counts))
    nodes = np.flatnonzero(label == big)
    if len(nodes) == n:
        return a, nodes
    local = np.full(n, -1, dtype=np.int64)
    local[nodes] = np.arange(len(nodes))
    sel = (label[rows] == big) & (rows < cols)
    lu, lv = local[rows[sel]], local[cols[sel]]
    w = -a.val[sel]
    order = np.lexsort((lv, lu))
    return assemble_canonical(len(nodes), lu[order], lv[order], w[order]), nodes


# -------------------------------------------------- reference generators
def from_stencil(n_side: int, legs) -> SparseLaplacian:
    """generators.cpp:19-33: node (i,j) -> i*N+j, half-space legs."""
    us, vs, ws = [], [], []
    i, j = np.meshgrid(np.arange(n_side), np.arange(n_side), indexing="ij")
    i, j = i.ravel(), j.ravel()
    for dx, dy, wt in legs:
        ii, jj = i + dx, j + dy
        ok = (ii >= 0) & (jj >= 0) & (ii < n_side) & (jj < n_side)
        us.append((i * n_side + j)[ok])
        vs.append((ii * n_side + jj)[ok])
        ws.append(np.full(ok.sum(), wt))
    return assemble_laplacian(n_side * n_side, np.concatenate(us), np.concatenate(vs), np.concatenate(ws))


def grid_5pt(n_side: int) -> SparseLaplacian:
    return from_stencil(n_side, [(1, 0, 1.0), (0, 1, 1.0)])


def grid_13pt_4th(n_side: int) -> SparseLaplacian:
    return from_stencil(n_side, [(1, 0, 16.0), (0, 1, 16.0), (2, 0, -1.0), (0, 2, -1.0)])


def grid_anis_rotated(n_side: int, alpha: float, eps: float, northeast: bool) -> SparseLaplacian:
    cx = math.cos(alpha) * math.cos(alpha) + eps * math.sin(alpha) * math.sin(alpha)
    cy = eps * math.cos(alpha) * math.cos(alpha) + math.sin(alpha) * math.sin(alpha)
    cxy = (1.0 - eps) * math.sin(2.0 * alpha)
    s = 0.5
    if not northeast:
        legs = [(1, 0, s * cx), (0, 1, s * cy), (1, 1, s * (cxy / 4.0)), (1, -1, s * (-cxy / 4.0))]
    else:
        legs = [(1, 0, s * (cx - cxy / 2.0)), (0, 1, s * (cy - cxy / 2.0)), (1, 1, s * (cxy / 2.0))]
    return from_stencil(n_side, [leg for leg in legs if leg[2] != 0.0])


def path(n: int) -> SparseLaplacian:
    i = np.arange(n - 1)
    return assemble_laplacian(n, i, i + 1, np.ones(n - 1))


def star(n: int) -> SparseLaplacian:
    i = np.arange(1, n)
    return assemble_laplacian(n, np.zeros(n - 1, dtype=np.int64), i, np.ones(n - 1))


def complete(n: int) -> SparseLaplacian:
    u, v = np.triu_indices(n, 1)
    return assemble_laplacian(n, u, v, np.ones(len(u)))


def two_hubs(leaves: int) -> SparseLaplacian:
    k = np.arange(leaves)
    u = np.concatenate([[0], np.zeros(leaves, dtype=np.int64), np.ones(leaves, dtype=np.int64)])
    v = np.concatenate([[1], 2 + k, 2 + leaves + k])
    return assemble_laplacian(2 + 2 * leaves, u, v, np.ones(len(u)))


def binary_tree(n: int) -> SparseLaplacian:
    i = np.arange(1, n)
    return assemble_laplacian(n, (i - 1) // 2, i, np.ones(n - 1))


def random_connected_edges(n: int, extra_per_node: float, seed: int, w_lo=0.5, w_hi=2.0):
    """tests/support/test_graphs.hpp:16-33 (sequential Rng stream)."""
    r = Rng(seed)
    us, vs, ws = [], [], []
    for v in range(1, n):
        us.append(r.next_u64() % v)
        vs.append(v)
        ws.append(w_lo + (w_hi - w_lo) * r.next_unit())
    for _ in range(int(extra_per_node * n)):
        a = r.next_u64() % n
        b = r.next_u64() % n
        if a == b:
            continue
        us.append(a)
        vs.append(b)
        ws.append(w_lo + (w_hi - w_lo) * r.next_unit())
    return us, vs, ws


def random_connected(n: int, extra_per_node: float, seed: int) -> SparseLaplacian:
    us, vs, ws = random_connected_edges(n, extra_per_node, seed)
    return assemble_laplacian(n, us, vs, ws)


def random_vector(n: int, seed: int, zero_mean: bool = False) -> np.ndarray:
    """tests/support/test_graphs.hpp:40-46."""
    x = rng_pm1(seed, 0, n)
    return subtract_mean_seq(x) if zero_mean else x


# ------------------------------------------------- BASELINE.json configs
def grid3d_7pt(N: int, seed: int = 2, log_uniform: bool = True) -> SparseLaplacian:
    """Config 2: node (i*N+j)*N+k; edges emitted per node in
    order (+x, +y, +z); w = 10^(-3 + 6U), U = next_unit() of one stream in
    emission order; assembled with assemble_laplacian."""
    i, j, k = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    node = ((i * N + j) * N + k).ravel()
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    nbrs = np.stack([node + N * N, node + N, node + 1], axis=1)
    ok = np.stack([i + 1 < N, j + 1 < N, k + 1 < N], axis=1)
    u = np.repeat(node, 3).reshape(-1, 3)[ok]
    v = nbrs[ok]
    if log_uniform:
        w = 10.0 ** (-3.0 + 6.0 * rng_unit(seed, 0, len(u)))
    else:
        w = np.ones(len(u))
    return assemble_laplacian(N * N * N, u, v, w)


def rgg(n: int, seed: int = 3, mean_degree: float = 10.0):
    """Config 3: n points uniform in [0,1)^2, edge iff 0 < d < r with
    r = sqrt(mean_degree/(pi n)), w = 1/d; largest component kept."""
    xy = rng_unit(seed, 0, 2 * n).reshape(n, 2)
    r = math.sqrt(mean_degree / (math.pi * n))
    cells = max(1, int(1.0 / r))
    cx = np.minimum((xy[:, 0] * cells).astype(np.int64), cells - 1)
    cy = np.minimum((xy[:, 1] * cells).astype(np.int64), cells - 1)
    cell = cx * cells + cy
    order = np.argsort(cell, kind="stable")
    start = np.searchsorted(cell[order], np.arange(cells * cells + 1))
    us, vs, ws = [], [], []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            ncx, ncy = cx + dx, cy + dy
            okc = (ncx >= 0) & (ncy >= 0) & (ncx < cells) & (ncy < cells)
            pts = np.flatnonzero(okc)
            nc = ncx[pts] * cells + ncy[pts]
            cnt = start[nc + 1] - start[nc]
            rep = np.repeat(pts, cnt)
            offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            other = order[np.repeat(start[nc], cnt) + offs]
            keep = rep < other
            a, b = rep[keep], other[keep]
            d = np.hypot(xy[a, 0] - xy[b, 0], xy[a, 1] - xy[b, 1])
            close = (d > 0) & (d < r)
            us.append(a[close])
            vs.append(b[close])
            ws.append(1.0 / d[close])
    full = assemble_laplacian(n, np.concatenate(us), np.concatenate(vs), np.concatenate(ws))
    return largest_component(full)[0]


def chung_lu(n: int, seed: int = 4, beta: float = 2.1, mean_degree: float = 16.0):
    """Config 4: w_i ~ (i+1)^(-1/(beta-1)) scaled to the mean degree, clamped
    >= 1; floor(sum w / 2) endpoint pairs drawn proportional to w by inverse
    CDF; self-loops dropped, duplicates merged to unit weight; LCC kept."""
    wi = (np.arange(n) + 1.0) ** (-1.0 / (beta - 1.0))
    wi *= mean_degree / wi.mean()
    wi = np.maximum(wi, 1.0)
    cdf = np.cumsum(wi)
    cdf /= cdf[-1]
    pairs = int(wi.sum() // 2)
    uu = np.searchsorted(cdf, rng_unit(seed, 0, pairs), side="right")
    vv = np.searchsorted(cdf, rng_unit(seed, pairs, pairs), side="right")
    uu, vv = np.minimum(uu, n - 1), np.minimum(vv, n - 1)
    keep = uu != vv
    lo, hi = np.minimum(uu[keep], vv[keep]), np.maximum(uu[keep], vv[keep])
    key = np.unique(lo.astype(np.int64) * n + hi)
    full = assemble_canonical(n, key // n, key % n, np.ones(len(key)))
    return largest_component(full)[0]


def rmat(scale: int, seed: int = 5, edge_factor: int = 16, abcd=(0.57, 0.19, 0.19, 0.05)):
    """Config 5: 2^scale nodes, edge_factor*2^scale samples with per-bit
    quadrant choice; self-loops dropped; duplicates summed into f64 weights
    (integer multiplicities); LCC kept."""
    n = 1 << scale
    samples = edge_factor * n
    a, b, c, _ = abcd
    u = np.zeros(samples, dtype=np.int64)
    v = np.zeros(samples, dtype=np.int64)
    for bit in range(scale):
        r = rng_unit(seed, bit * samples, samples)
        ubit = r >= a + b
        vbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= ubit.astype(np.int64) << bit
        v |= vbit.astype(np.int64) << bit
    keep = u != v
    lo, hi = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key, cnt = np.unique(lo * n + hi, return_counts=True)
    full = assemble_canonical(n, key // n, key % n, cnt.astype(np.float64))
    return largest_component(full)[0]


def gaussian_rhs(n: int, seed: int) -> np.ndarray:
    """Seeded N(0,1) by Box-Muller over lamg::Rng, then the reference's
    subtract_mean (sequential fold, sparse_laplacian.cpp:242-252)."""
    half = (n + 1) // 2
    u1 = rng_unit(seed, 0, half)
    u2 = rng_unit(seed, half, half)
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    z = np.concatenate([rad * np.cos(2 * np.pi * u2), rad * np.sin(2 * np.pi * u2)])[:n]
    return subtract_mean_seq(z)


def zero_sum(B: np.ndarray) -> np.ndarray:
    """At n ~ 1e7 the sequential mean subtraction of gaussian_rhs leaves |sum b|
    near the reference's 1e-10 * max|b| compatibility threshold
    (cycle.cpp:226-230): project again (twice) with numpy's pairwise sum.
    Used for the full-size configs 4 and 5 by bench.py, the GPU tests and
    tests/golden/make_golden_large.py alike."""
    for _ in range(2):
        B -= (B.sum(axis=-1, keepdims=True) / B.shape[-1])
    return B


def subtract_mean_seq(x: np.ndarray) -> np.ndarray:
    """subtract_mean with the reference's left-to-right fold."""
    s = sequential_sum(x)
    return x - s / len(x)


def sequential_sum(x: np.ndarray) -> float:
    """Exact left-to-right fold (numpy's sum is pairwise; its cumulative sum
    is the sequential recurrence, so the last prefix is the fold)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    return float(np.cumsum(x)[-1]) if x.size else 0.0


def default_x0(n: int, seed: int = 1) -> np.ndarray:
    """The reference's default initial guess: Rng(derive(cycle seed, 0x517))
    draws in node order (solver.cpp:74,90)."""
    return rng_pm1(Rng.derive(seed, 0x517), 0, n)


CONFIGS = {
    1: "2D 5-point grid 256x256, unit weights",
    2: "3D 7-point grid 128^3, log-uniform weights in [1e-3,1e3]",
    3: "random geometric graph, 4M points, mean degree 10, w=1/d, LCC",
    4: "Chung-Lu power law, 16M nodes, beta 2.1, mean degree 16, LCC",
    5: "R-MAT scale 25, edge factor 16, (.57,.19,.19,.05), LCC",
}


def make_config(cfg: int, scale_down: int = 0) -> SparseLaplacian:
    """Builds BASELINE.json config `cfg` (1-based); scale_down shrinks the
    linear size for parity tests (0 = full size)."""
    if cfg == 1:
        return grid_5pt(256 >> scale_down)
    if cfg == 2:
        return grid3d_7pt(128 >> scale_down)
    if cfg == 3:
        return rgg((1 << 22) >> (2 * scale_down))
    if cfg == 4:
        return chung_lu((1 << 24) >> (2 * scale_down))
    if cfg == 5:
        return rmat(25 - 2 * scale_down)
    raise ValueError(cfg)
