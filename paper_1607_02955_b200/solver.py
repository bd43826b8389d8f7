"""Multigrid Laplacian solver -- reference-compatible API, B200 solve path.

Mirrors pkg/src/cfcent/solver.py (names, signatures, defaults, exceptions):

* ``setup`` builds the hierarchy on the host with the reference's semantics
  (stage alternation and 10 % rule, solver.py:422-523).  The level matrices
  are produced by the same scipy operations as the reference (Schur
  complement, Galerkin product, Laplacian rebuild); the greedy O(n) loops
  (independent sets, affinity attachment, matching) run in C++
  (csrc/cf_setup.cpp).  The hierarchy is then uploaded once to the GPU as
  per-level int32/fp64 CSR operators, colour classes, aggregate maps and
  elimination transfer operators (csrc/cf_solve.cu, ``cf_hier_create``).
* ``solve`` / ``solve_many`` run entirely on the device: all right-hand sides
  of a call are solved together as one row-major block (up to 256 columns per
  device chunk), with per-column convergence, stagnation, freezing and the
  FCG / Jacobi-PCG fallback chain (solver.py:651-751) in CUDA.  There is no
  CPU fallback: without a CUDA device the solve raises.

Smoother change (stated as the north star requires): the reference smooths
aggregation levels with natural-order Gauss-Seidel (forward pre, backward
post; solver.py:545,559).  The device uses multicolour Gauss-Seidel: the same
forward/backward sweeps over colour classes of a greedy colouring, each class
updated in parallel.  Every other V-cycle step is the reference's.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field
from enum import Enum
from typing import Sequence

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components
from scipy.sparse.linalg import spsolve_triangular

from . import _native as N
from .errors import ConvergenceError, DomainError

__all__ = ["SolverConfig", "LevelKind", "Level", "MultigridHierarchy", "PotentialVector",
           "setup", "coarsen_eliminate", "coarsen_aggregate", "relaxed_test_vectors", "solve",
           "solve_many"]

# Fixed algorithm parameters (solver.py:48-58).
AFFINITY_THRESHOLD = 0.5
TEST_VECTOR_SWEEPS = 3
MAX_AGGREGATE_SIZE = 8
ATTACH_SWEEPS = 3
MIN_REDUCTION = 0.10
STAGNATION_FACTOR = 0.9
STAGNATION_CYCLES = 5
FCG_MAX_ITERS = 200
BLOCK_COLUMNS = 64     # reference block width; the device solves all columns of a call at once
STOP_MARGIN = 0.9
# Device hierarchy truncation (B200 design choice): the device copy
# of the hierarchy ends at the first level below the top with at most
# min(DEVICE_DIRECT_MAX, n0 * DEVICE_DIRECT_FRACTION) nodes; that level is
# solved exactly with its dense centred grounded inverse (one fp64 GEMM per
# V-cycle) instead of recursing through the deep tail of tiny levels.
DEVICE_DIRECT_MAX = 4096
DEVICE_DIRECT_FRACTION = 1.0 / 16.0
# Locality ordering of the device copy: every non-dense level is
# renumbered by reverse Cuthill-McKee so neighbour gathers of the row-major
# blocks hit L2; the permutation is applied at the API boundary.
DEVICE_REORDER = os.environ.get("CF_DEVICE_REORDER", "1") != "0"
# Stall breaker (B200 setup): on power-law graphs the reference's
# stages shrink a level by ~0.01-1 % for thousands of levels (R-MAT scale 20:
# 2,859 levels).  When both reference stages miss MIN_REDUCTION, the setup
# also tries exact elimination with off-degree cap STALL_ELIM_CAP and affinity
# aggregation with cap STALL_AGG_CAP / threshold STALL_AGG_THRESHOLD, and keeps
# the largest reduction.  Active on levels above DEVICE_DIRECT_MAX nodes, or on
# every level when n0 > STALL_BREAKER_MIN_N0; graphs whose hierarchies never
# stall there (C1-C3) keep the reference hierarchy exactly.
STALL_ELIM_CAP = 16
# escalation: the first cap (the reference's kind of low-degree set, one size
# up) is always a candidate; each larger cap only while its fill bound stays
# under the budget.  (Applying the budget to the first cap as well drops the
# elimination candidate on R-MAT hub levels -- the bound sum d_f^2 is a worst
# case -- and the C5 setup then runs for > 15 min into a many-level hierarchy.)
STALL_ELIM_CAPS = (16, 64, 256, 1024)
STALL_FILL_FACTOR = 2.0                 # min(sum d_f^2, |C|^2) <= factor * nnz
STALL_AGG_CAP = 64
STALL_AGG_THRESHOLD = 0.0
STALL_BREAKER_MIN_N0 = 262144
# Hub levels (B200 setup): on levels of a large graph (n0 >
# STALL_BREAKER_MIN_N0) whose maximum off-degree exceeds HUB_DEGREE_RATIO x the
# mean, the reference's aggregate cap of 8 leaves a hub's edges to its many
# small aggregates in the Galerkin operator (R-MAT: coarse levels with mean
# degree 90-280 and as many nonzeros as the fine level).  There the aggregate
# cap is HUB_AGG_CAP.  Geometric graphs (C3: max/mean 2.9) never qualify.
HUB_DEGREE_RATIO = 64.0
HUB_AGG_CAP = int(os.environ.get("CF_HUB_AGG_CAP", "512"))


@dataclass(frozen=True)
class SolverConfig:
    """Tuning knobs for hierarchy construction and solves (solver.py:61-88).

    ``smoothing_steps`` is (pre, post) Gauss-Seidel sweeps per V-cycle.
    """

    tau: float = 1e-5
    max_cycles: int = 100
    max_direct_size: int = 200
    smoothing_steps: tuple[int, int] = (1, 2)
    elimination_degree_cap: int = 4
    aggregation_test_vectors: int = 4
    seed: int = 0

    def __post_init__(self):
        if self.tau <= 0:
            raise DomainError("tau must be positive")
        if min(self.max_cycles, self.max_direct_size, self.smoothing_steps[0],
               self.smoothing_steps[1], self.elimination_degree_cap,
               self.aggregation_test_vectors) < 1:
            raise DomainError("all solver counts must be >= 1")


class LevelKind(Enum):
    ELIMINATION = "elimination"
    AGGREGATION = "aggregation"
    COARSEST = "coarsest"


@dataclass
class Level:
    """One hierarchy level (solver.py:97-120).  ``m_lower``/``m_upper`` (the
    reference's Gauss-Seidel triangles, solver.py:503-504) are built on first
    access for aggregation levels and cached; the device smoother itself uses
    ``colors`` (multicolour GS) and never needs them."""

    kind: LevelKind
    matrix: sp.csr_matrix
    f_nodes: np.ndarray | None = None
    c_nodes: np.ndarray | None = None
    f_degree: np.ndarray | None = None
    w_cf: sp.csr_matrix | None = None
    w_fc: sp.csr_matrix | None = None
    p: sp.csr_matrix | None = None
    aggregates: np.ndarray | None = None
    grounded_factor: tuple | None = None
    colors: np.ndarray | None = None
    _tri: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def size(self) -> int:
        return self.matrix.shape[0]

    def _triangle(self, which: str):
        if self.kind is not LevelKind.AGGREGATION:
            return None
        t = self._tri.get(which)
        if t is None:
            t = (sp.tril if which == "lower" else sp.triu)(self.matrix, 0, format="csr")
            self._tri[which] = t
        return t

    @property
    def m_lower(self) -> sp.csr_matrix | None:
        return self._triangle("lower")

    @property
    def m_upper(self) -> sp.csr_matrix | None:
        return self._triangle("upper")


@dataclass
class SolveStats:
    """solver.py:123-137, plus device counters.  ``fallback_solves`` keeps the
    reference meaning (columns that entered the FCG fallback after the
    stagnation rule, solver.py:717-720); ``krylov_solves`` counts columns the
    Krylov hand-off continued under V-cycle-preconditioned
    FCG before any stagnation."""

    solves: int = 0
    max_residual: float = 0.0
    fallback_solves: int = 0
    vcycles: int = 0
    krylov_solves: int = 0
    _lock: threading.Lock = field(default_factory=threading.Lock, repr=False)

    def record(self, residuals: np.ndarray, fallbacks: int, vcycles: int = 0,
               krylov: int = 0) -> None:
        with self._lock:
            self.solves += residuals.size
            if residuals.size:
                self.max_residual = max(self.max_residual, float(residuals.max()))
            self.fallback_solves += fallbacks
            self.vcycles += vcycles
            self.krylov_solves += krylov


_DEVICE: int | None = None


def set_device(index: int) -> None:
    """Select the CUDA device new hierarchies are uploaded to (one process
    per GPU; defaults to $LOCAL_RANK or 0)."""
    global _DEVICE
    _DEVICE = int(index)


def _device_index() -> int:
    if _DEVICE is not None:
        return _DEVICE
    import os
    return int(os.environ.get("LOCAL_RANK", "0"))


def device_levels(levels: list[Level]) -> list[Level]:
    """The level list uploaded to the device: the host hierarchy truncated at
    the first level j >= 1 with n_j <= min(DEVICE_DIRECT_MAX, n0/16), which
    becomes the (exactly solved) coarsest level."""
    n0 = levels[0].size
    cap = min(DEVICE_DIRECT_MAX, int(n0 * DEVICE_DIRECT_FRACTION))
    for j in range(1, len(levels) - 1):
        if levels[j].size <= cap:
            last = Level(kind=LevelKind.COARSEST, matrix=levels[j].matrix,
                         grounded_factor=_factor_coarsest(levels[j].matrix))
            return list(levels[:j]) + [last]
    return list(levels)


def _identity(n):
    return np.arange(n, dtype=np.int64)


def _inverse(p):
    inv = np.empty_like(p)
    inv[p] = np.arange(p.size, dtype=p.dtype)
    return inv


def _permute(A: sp.csr_matrix, rows: np.ndarray, cmap: np.ndarray, ncols: int) -> sp.csr_matrix:
    """A[rows][:, inverse(cmap)] with sorted rows (native, threaded)."""
    A = A.tocsr()
    ip, ix = _csr64(A)
    val = np.ascontiguousarray(A.data, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cmap = np.ascontiguousarray(cmap, dtype=np.int64)
    nnz = int(np.sum(ip[rows + 1] - ip[rows])) if rows.size else 0
    op = np.empty(rows.size + 1, dtype=np.int64)
    oi = np.empty(nnz, dtype=np.int64)
    ov = np.empty(nnz, dtype=np.float64)
    N.check(N.lib().cf_setup_permute(rows.size, N.ptr(ip, N.i64p), N.ptr(ix, N.i64p),
                                     N.ptr(val, N.f64p), N.ptr(rows, N.i64p),
                                     N.ptr(cmap, N.i64p), N.ptr(op, N.i64p), N.ptr(oi, N.i64p),
                                     N.ptr(ov, N.f64p)))
    out = sp.csr_matrix((ov, oi, op), shape=(rows.size, ncols))
    out.has_sorted_indices = True
    return out


def permute_levels(levels: list[Level]):
    """Renumber each non-dense level by RCM; returns (levels', perm0) with
    perm0[i'] = original node of device row i' on level 0.  Transfer
    operators are remapped so the permuted hierarchy is the same operator."""
    from scipy.sparse.csgraph import reverse_cuthill_mckee

    perms, classes = [], []
    for lvl in levels:
        classes.append(None)
        if lvl.kind is LevelKind.COARSEST or not DEVICE_REORDER:
            perms.append(_identity(lvl.size))
            continue
        A = lvl.matrix.tocsr()
        p = np.asarray(reverse_cuthill_mckee(A, symmetric_mode=True), dtype=np.int64)
        if lvl.kind is LevelKind.AGGREGATION:
            # colour classes of the RCM-ordered matrix become contiguous row
            # ranges (RCM order kept inside each class)
            col = _colour(_permute(A, p, _inverse(p), p.size))
            order = np.argsort(col, kind="stable")
            p = p[order]
            classes[-1] = col[order]
        perms.append(p)
    invs = []
    for p in perms:
        inv = np.empty_like(p)
        inv[p] = np.arange(p.size)
        invs.append(inv)
    out = []
    for j, lvl in enumerate(levels):
        p, inv = perms[j], invs[j]
        if lvl.kind is LevelKind.COARSEST:
            out.append(lvl)
            continue
        A = _permute(lvl.matrix, p, inv, p.size)
        pn, invn = perms[j + 1], invs[j + 1]
        if lvl.kind is LevelKind.AGGREGATION:
            agg = invn[lvl.aggregates[p]]
            col = classes[j] if classes[j] is not None else _colour(A)
            out.append(Level(kind=LevelKind.AGGREGATION, matrix=A, aggregates=agg, colors=col))
        else:
            f_new = inv[lvl.f_nodes]
            order = np.argsort(f_new, kind="stable")
            rank = np.empty_like(order)
            rank[order] = np.arange(order.size)
            w_cf = _permute(lvl.w_cf, pn, rank, order.size)
            out.append(Level(kind=LevelKind.ELIMINATION, matrix=A, f_nodes=f_new[order],
                             c_nodes=inv[lvl.c_nodes[pn]], f_degree=lvl.f_degree[order],
                             w_cf=w_cf, w_fc=w_cf.T.tocsr()))
    return out, perms[0]


class _DeviceHierarchy:
    """Owner of the C handle (device operators + workspace)."""

    def __init__(self, levels: list[Level], device: int | None = None):
        device = _device_index() if device is None else device
        L = N.lib()
        if L.cf_device_count() < 1:
            raise RuntimeError("cfcent_b200: no CUDA device visible; the solve path has no "
                               "CPU fallback")
        self._keep = []
        levels, perm0 = permute_levels(device_levels(levels))
        self.levels = levels
        self.perm0 = perm0                       # device row -> node
        self.inv0 = np.empty_like(perm0)         # node -> device row
        self.inv0[perm0] = np.arange(perm0.size)
        descs = (N.CfLevelDesc * len(levels))()
        for j, lvl in enumerate(levels):
            self._fill(descs[j], lvl, j)
        h = N.C.c_void_p()
        N.check(L.cf_hier_create(len(levels), descs, device, N.C.byref(h)))
        self.handle = h
        p32 = np.ascontiguousarray(perm0, dtype=np.int32)
        N.check(L.cf_hier_set_order(h, N.ptr(p32, N.i32p), p32.size))
        self._keep = None  # host arrays were copied to the device

    def _arr(self, a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        self._keep.append(a)
        return a

    def _fill(self, d, lvl: Level, j: int):
        A = lvl.matrix.tocsr()
        n = A.shape[0]
        d.kind = {LevelKind.ELIMINATION: 0, LevelKind.AGGREGATION: 1, LevelKind.COARSEST: 2}[lvl.kind]
        d.n = n
        need_matrix = j == 0 or lvl.kind is LevelKind.AGGREGATION
        if need_matrix:
            rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(A.indptr))
            off = A.indices != rows
            cnt = np.bincount(rows[off], minlength=n)
            rp = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(cnt, out=rp[1:])
            d.nnz_off = int(rp[-1])
            d.rowptr = N.ptr(self._arr(rp, np.int64), N.i64p)
            d.col = N.ptr(self._arr(A.indices[off], np.int32), N.i32p)
            d.val = N.ptr(self._arr(A.data[off], np.float64), N.f64p)
            d.diag = N.ptr(self._arr(A.diagonal(), np.float64), N.f64p)
        if lvl.kind is LevelKind.AGGREGATION:
            agg = lvl.aggregates
            nc = int(agg.max()) + 1
            d.n_coarse = nc
            col = lvl.colors
            order = np.argsort(col, kind="stable")
            cptr = np.zeros(int(col.max()) + 2, dtype=np.int64)
            np.cumsum(np.bincount(col, minlength=int(col.max()) + 1), out=cptr[1:])
            d.n_colors = int(col.max()) + 1
            d.color_ptr = N.ptr(self._arr(cptr, np.int32), N.i32p)
            d.color_rows = N.ptr(self._arr(order, np.int32), N.i32p)
            d.agg = N.ptr(self._arr(agg, np.int32), N.i32p)
            aptr = np.zeros(nc + 1, dtype=np.int64)
            np.cumsum(np.bincount(agg, minlength=nc), out=aptr[1:])
            d.agg_ptr = N.ptr(self._arr(aptr, np.int32), N.i32p)
            d.agg_members = N.ptr(self._arr(np.argsort(agg, kind="stable"), np.int32), N.i32p)
        elif lvl.kind is LevelKind.ELIMINATION:
            f, c = lvl.f_nodes, lvl.c_nodes
            d.n_coarse = c.size
            d.n_f = f.size
            d.f_nodes = N.ptr(self._arr(f, np.int32), N.i32p)
            d.c_nodes = N.ptr(self._arr(c, np.int32), N.i32p)
            d.f_degree = N.ptr(self._arr(lvl.f_degree, np.float64), N.f64p)
            wcf = lvl.w_cf.tocsr()
            wfc = lvl.w_fc.tocsr()
            d.wcf_ptr = N.ptr(self._arr(wcf.indptr, np.int64), N.i64p)
            d.wcf_col = N.ptr(self._arr(wcf.indices, np.int32), N.i32p)
            d.wcf_val = N.ptr(self._arr(wcf.data, np.float64), N.f64p)
            d.wfc_ptr = N.ptr(self._arr(wfc.indptr, np.int64), N.i64p)
            d.wfc_col = N.ptr(self._arr(wfc.indices, np.int32), N.i32p)
            d.wfc_val = N.ptr(self._arr(wfc.data, np.float64), N.f64p)
        else:
            d.n_coarse = 0
            if n > 1 and lvl.grounded_factor is not None:
                d.coarse_op = N.ptr(self._arr(_coarse_operator(lvl), np.float64), N.f64p)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            try:
                N.lib().cf_hier_destroy(self.handle)
            finally:
                self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class MultigridHierarchy:
    levels: list[Level]
    config: SolverConfig
    stats: SolveStats = field(default_factory=SolveStats)
    _dev: _DeviceHierarchy | None = field(default=None, repr=False, compare=False)
    _dev_lock: threading.Lock = field(default_factory=threading.Lock, repr=False,
                                      compare=False)
    _graphs: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def n(self) -> int:
        return self.levels[0].size

    @property
    def level_sizes(self) -> list[int]:
        return [lvl.size for lvl in self.levels]

    def device(self) -> _DeviceHierarchy:
        """Upload the hierarchy on first use (solve phase only)."""
        if self._dev is None:
            with self._dev_lock:
                if self._dev is None:
                    self._dev = _DeviceHierarchy(self.levels)
        return self._dev

    def device_bytes(self) -> int:
        return int(N.lib().cf_hier_device_bytes(self.device().handle))

    def stream_ptr(self) -> int:
        """cudaStream_t (as int) all kernels of this hierarchy run on."""
        return int(N.lib().cf_hier_stream(self.device().handle) or 0)

    def profile(self, enable: bool) -> None:
        N.check(N.lib().cf_profile(self.device().handle, 1 if enable else 0))

    def profile_report(self) -> list[tuple[str, int, int, float, float, float]]:
        """[(kind, level, launches, total_ms, algorithmic_bytes, gather_bytes)] of
        the launches recorded since ``profile(True)``."""
        need = np.zeros(1, dtype=np.int64)
        L = N.lib()
        N.check(L.cf_profile_report(self.device().handle, None, 0, N.ptr(need, N.i64p)))
        buf = N.C.create_string_buffer(int(need[0]) + 1)
        N.check(L.cf_profile_report(self.device().handle, buf, int(need[0]) + 1,
                                    N.ptr(need, N.i64p)))
        out = []
        for line in buf.value.decode().splitlines():
            k, lv, la, ms, by, gb = line.split()
            out.append((k, int(lv), int(la), float(ms), float(by), float(gb)))
        return out


@dataclass
class PotentialVector:
    """Solution of ``L p = b`` normalized to zero mean (solver.py:155-160)."""

    values: np.ndarray
    achieved_residual: float


# ---------------------------------------------------------------------------
# setup (host)
# ---------------------------------------------------------------------------

def _rebuild_laplacian(matrix: sp.spmatrix, unique: bool = False) -> sp.csr_matrix:
    """Symmetrise; keep strictly negative off-diagonals; diagonal = minus the
    off-diagonal row sum (solver.py:167-187).  Native (csrc/cf_setup.cpp) with
    the reference's arithmetic; duplicate-carrying inputs take the scipy path."""
    m = matrix.tocsr()
    if unique or m.has_canonical_format or _no_duplicates(m):
        n = m.shape[0]
        ip = np.ascontiguousarray(m.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(m.indices, dtype=np.int64)
        dv = np.ascontiguousarray(m.data, dtype=np.float64)
        cap = 2 * ix.size + n
        op = np.empty(n + 1, dtype=np.int64)
        oi = np.empty(cap, dtype=np.int64)
        ov = np.empty(cap, dtype=np.float64)
        nnz = np.zeros(1, dtype=np.int64)
        N.check(N.lib().cf_rebuild_laplacian(n, N.ptr(ip, N.i64p), N.ptr(ix, N.i64p),
                                             N.ptr(dv, N.f64p), N.ptr(op, N.i64p),
                                             N.ptr(oi, N.i64p), N.ptr(ov, N.f64p),
                                             N.ptr(nnz, N.i64p)))
        k = int(nnz[0])
        out = sp.csr_matrix((ov[:k].copy(), oi[:k].astype(np.int32), op.astype(np.int32)),
                            shape=(n, n))
        out.has_sorted_indices = True
        return out
    return _rebuild_laplacian_scipy(m)


def _no_duplicates(m: sp.csr_matrix) -> bool:
    c = m.copy()
    c.sum_duplicates()
    return c.nnz == m.nnz


def _rebuild_laplacian_scipy(matrix: sp.spmatrix) -> sp.csr_matrix:
    m = matrix.tocsr()
    m = (m + m.T) * 0.5
    t = m.tocoo()
    keep = (t.row != t.col) & (t.data < 0)
    r, c, v = t.row[keep], t.col[keep], t.data[keep]
    n = m.shape[0]
    dg = np.zeros(n)
    np.add.at(dg, r, -v)
    idx = np.arange(n)
    out = sp.csr_matrix((np.concatenate([v, dg]), (np.concatenate([r, idx]),
                                                   np.concatenate([c, idx]))), shape=(n, n))
    out.sort_indices()
    return out


def _validate_laplacian(matrix: sp.spmatrix) -> sp.csr_matrix:
    """solver.py:190-211."""
    if matrix.shape[0] != matrix.shape[1]:
        raise DomainError("matrix must be square")
    m = matrix.tocsr()
    n = m.shape[0]
    if (m.nnz >= DEVICE_SETUP_MIN_NNZ and os.environ.get("CF_DEVICE_SETUP", "1") != "0"
            and N.device_available()):
        # large inputs: the same checks as max-reductions on the GPU
        # (csrc/cf_setup_dev.cu); the transposes of the host route cost 14 s on C5
        if not m.has_canonical_format:
            m = m.copy()
            m.sum_duplicates()  # sorted rows without repeated entries (the caller's matrix is untouched)
        ip, ix = _csr64(m)
        dv = np.ascontiguousarray(m.data, dtype=np.float64)
        out = np.zeros(4)
        ncomp = np.zeros(1, dtype=np.int64)
        N.check(N.lib().cf_validate_laplacian_dev(_device_index(), n, N.ptr(ip, N.i64p),
                                                  N.ptr(ix, N.i64p), N.ptr(dv, N.f64p),
                                                  N.ptr(out, N.f64p), N.ptr(ncomp, N.i64p)))
        tol = 1e-12 * n * max(float(out[0]), 1.0)
        if out[1] > tol:
            raise DomainError("matrix is not symmetric")
        if out[2] > tol:
            raise DomainError("row sums are not zero; not a Laplacian")
        if out[3] > tol:
            raise DomainError("positive off-diagonal entry; not a Laplacian")
        if n > 1 and ncomp[0] > 1:
            raise DomainError("Laplacian graph is not connected")
        return _rebuild_laplacian(m)
    scale = float(np.abs(m.data).max()) if m.nnz else 0.0
    tol = 1e-12 * n * max(scale, 1.0)
    asym = abs(m - m.T)
    if asym.nnz and asym.data.max() > tol:
        raise DomainError("matrix is not symmetric")
    if np.abs(np.asarray(m.sum(axis=1)).ravel()).max(initial=0.0) > tol:
        raise DomainError("row sums are not zero; not a Laplacian")
    t = m.tocoo()
    off = t.row != t.col
    if off.any() and t.data[off].max() > tol:
        raise DomainError("positive off-diagonal entry; not a Laplacian")
    if n > 1 and connected_components(m, directed=False)[0] > 1:
        raise DomainError("Laplacian graph is not connected")
    return _rebuild_laplacian(m)


@dataclass
class EliminationRecord:
    f_nodes: np.ndarray
    c_nodes: np.ndarray
    f_degree: np.ndarray
    w_cf: sp.csr_matrix


def _csr64(matrix):
    m = matrix.tocsr()
    return (np.ascontiguousarray(m.indptr, dtype=np.int64),
            np.ascontiguousarray(m.indices, dtype=np.int64))


def coarsen_eliminate(matrix: sp.csr_matrix, degree_cap: int = 4):
    """Exact Schur elimination of a greedy independent low-degree set
    (solver.py:222-261).  Returns ``(schur, EliminationRecord | None)``."""
    matrix = matrix.tocsr()
    n = matrix.shape[0]
    ip, ix = _csr64(matrix)
    out = np.empty(max(n, 1), dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cf_setup_elim_select(n, N.ptr(ip, N.i64p), N.ptr(ix, N.i64p), degree_cap,
                                         N.ptr(out, N.i64p), N.ptr(cnt, N.i64p)))
    if cnt[0] == 0:
        return matrix, None
    return _eliminate_set(matrix, out[:cnt[0]].copy())


def _elim_select(matrix: sp.csr_matrix, cap: int) -> np.ndarray:
    """Greedy ascending-id independent set of off-degree <= cap (native)."""
    n = matrix.shape[0]
    ip, ix = _csr64(matrix)
    out = np.empty(max(n, 1), dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cf_setup_elim_select(n, N.ptr(ip, N.i64p), N.ptr(ix, N.i64p), int(cap),
                                         N.ptr(out, N.i64p), N.ptr(cnt, N.i64p)))
    return out[:cnt[0]].copy()


# Coarse operators on the GPU (csrc/cf_setup_dev.cu) for
# hub graphs above STALL_BREAKER_MIN_N0 nodes (maximum degree > HUB_DEGREE_RATIO
# x the mean on the finest level) -- exactly the graphs whose hierarchies
# already differ from the reference's (stall breaker, hub aggregates);
# everywhere else the host route keeps hierarchies bit-identical to the
# reference's goldens (C1-C3).  The device sums equal keys in sorted order, scipy in
# its SpGEMM order: values agree to rounding (tests/test_gpu_solver.py).
_native_relax_on = False  # set per setup() call: hub graphs only
DEVICE_SETUP_MIN_NNZ = 1 << 21
DEVICE_SETUP_MIN_N0 = STALL_BREAKER_MIN_N0
_device_setup_on = False


def _device_setup(nnz: int) -> bool:
    if not _device_setup_on or nnz < DEVICE_SETUP_MIN_NNZ:
        return False
    if os.environ.get("CF_DEVICE_SETUP", "1") == "0":
        return False
    return N.device_available()


def _coarse_operator_dev(matrix: sp.csr_matrix, cmap: np.ndarray, nc: int,
                         f: np.ndarray | None = None) -> sp.csr_matrix:
    """Galerkin product (f None) or Schur complement of the independent set f,
    rebuilt as a Laplacian, on the GPU."""
    m = matrix.tocsr()
    if not m.has_sorted_indices:
        m = m.sorted_indices()
    ip, ix = _csr64(m)
    dv = np.ascontiguousarray(m.data, dtype=np.float64)
    cmap = np.ascontiguousarray(cmap, dtype=np.int64)
    fn = np.ascontiguousarray(f if f is not None else np.zeros(0), dtype=np.int64)
    nnz = np.zeros(1, dtype=np.int64)
    L = N.lib()
    N.check(L.cf_coarse_operator_dev(_device_index(), m.shape[0], N.ptr(ip, N.i64p),
                                     N.ptr(ix, N.i64p), N.ptr(dv, N.f64p), N.ptr(cmap, N.i64p),
                                     int(nc), fn.size, N.ptr(fn, N.i64p), N.ptr(nnz, N.i64p)))
    k = int(nnz[0])
    op = np.empty(nc + 1, dtype=np.int64)
    oi = np.empty(max(k, 1), dtype=np.int64)
    ov = np.empty(max(k, 1), dtype=np.float64)
    N.check(L.cf_coarse_fetch_dev(N.ptr(op, N.i64p), N.ptr(oi, N.i64p), N.ptr(ov, N.f64p)))
    out = sp.csr_matrix((ov[:k], oi[:k].astype(np.int32), op.astype(np.int32)), shape=(nc, nc))
    out.has_sorted_indices = True
    return out


def _eliminate_set(matrix: sp.csr_matrix, f: np.ndarray):
    """Exact Schur complement of the independent set f (solver.py:251-261)."""
    n = matrix.shape[0]
    in_f = np.zeros(n, dtype=bool)
    in_f[f] = True
    c = np.flatnonzero(~in_f)
    d_f = matrix.diagonal()[f]
    w_cf = (-(matrix[c][:, f].tocsr())).tocsr()
    if _device_setup(matrix.nnz):
        cmap = np.full(n, -1, dtype=np.int64)
        cmap[c] = np.arange(c.size)
        schur = _coarse_operator_dev(matrix, cmap, c.size, np.asarray(f, dtype=np.int64))
        return schur, EliminationRecord(f_nodes=f, c_nodes=c, f_degree=d_f, w_cf=w_cf)
    schur = matrix[c][:, c] - w_cf @ sp.diags(1.0 / d_f) @ w_cf.T
    return _rebuild_laplacian(schur, unique=True), EliminationRecord(f_nodes=f, c_nodes=c, f_degree=d_f,
                                                        w_cf=w_cf)


def relaxed_test_vectors(matrix: sp.csr_matrix, count: int, rng: np.random.Generator):
    """Centred Gaussian vectors after 3 forward GS sweeps on Lx = 0
    (solver.py:264-275); same RNG draws and sweeps as the reference."""
    x = rng.standard_normal((matrix.shape[0], count))
    x -= x.mean(axis=0, keepdims=True)
    if _native_relax_on and matrix.has_sorted_indices and count <= 64:
        # hub graphs (hierarchies are this build's own): the same sweeps as a
        # native loop (csrc/cf_setup.cpp) instead of SuperLU triangular solves
        # (16 of the 36 s of the C5 host setup)
        ip, ix = _csr64(matrix)
        dv = np.ascontiguousarray(matrix.data, dtype=np.float64)
        x = np.ascontiguousarray(x)
        N.check(N.lib().cf_setup_relax(matrix.shape[0], N.ptr(ip, N.i64p), N.ptr(ix, N.i64p),
                                       N.ptr(dv, N.f64p), count, TEST_VECTOR_SWEEPS,
                                       N.ptr(x, N.f64p)))
        x -= x.mean(axis=0, keepdims=True)
        return x
    low = sp.tril(matrix, 0, format="csr")
    for _ in range(TEST_VECTOR_SWEEPS):
        x += spsolve_triangular(low, -(matrix @ x), lower=True)
    x -= x.mean(axis=0, keepdims=True)
    return x


def _galerkin(matrix: sp.csr_matrix, agg: np.ndarray, n_agg: int) -> sp.csr_matrix:
    if _device_setup(matrix.nnz):
        return _coarse_operator_dev(matrix, agg, n_agg)
    n = matrix.shape[0]
    p = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, n_agg))
    return _rebuild_laplacian(p.T @ matrix @ p, unique=True)


def coarsen_aggregate(matrix: sp.csr_matrix, test_vectors: np.ndarray,
                      cap: int = MAX_AGGREGATE_SIZE, threshold: float = AFFINITY_THRESHOLD):
    """Affinity aggregation + Galerkin coarse operator (solver.py:278-346).
    Returns ``(coarse, aggregates)``.  ``cap`` is the aggregate size limit
    (the reference's 8 by default)."""
    matrix = matrix.tocsr()
    n = matrix.shape[0]
    ip, ix = _csr64(matrix)
    tv = np.ascontiguousarray(test_vectors, dtype=np.float64)
    agg = np.empty(n, dtype=np.int64)
    na = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cf_setup_aggregate(n, N.ptr(ip, N.i64p), N.ptr(ix, N.i64p),
                                       N.ptr(tv, N.f64p), tv.shape[1], int(cap),
                                       float(threshold), N.ptr(agg, N.i64p), N.ptr(na, N.i64p)))
    return _galerkin(matrix, agg, int(na[0])), agg


def _matching_aggregation(matrix: sp.csr_matrix, test_vectors: np.ndarray):
    """Pair matching by descending affinity (solver.py:349-380)."""
    matrix = matrix.tocsr()
    n = matrix.shape[0]
    t = matrix.tocoo()
    up = t.row < t.col
    eu = np.ascontiguousarray(t.row[up], dtype=np.int64)
    ev = np.ascontiguousarray(t.col[up], dtype=np.int64)
    x = test_vectors
    nrm = np.einsum("ij,ij->i", x, x)
    dots = np.einsum("ij,ij->i", x[eu], x[ev])
    den = nrm[eu] * nrm[ev]
    aff = np.where(den > 0, dots * dots / den, 0.0)
    order = np.ascontiguousarray(np.lexsort((ev, eu, -aff)), dtype=np.int64)
    agg = np.empty(n, dtype=np.int64)
    na = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cf_setup_matching(n, eu.size, N.ptr(eu, N.i64p), N.ptr(ev, N.i64p),
                                      N.ptr(order, N.i64p), N.ptr(agg, N.i64p),
                                      N.ptr(na, N.i64p)))
    return _galerkin(matrix, agg, int(na[0])), agg


def _colour(matrix: sp.csr_matrix) -> np.ndarray:
    ip, ix = _csr64(matrix)
    n = matrix.shape[0]
    col = np.empty(n, dtype=np.int32)
    nc = np.zeros(1, dtype=np.int32)
    N.check(N.lib().cf_setup_colour(n, N.ptr(ip, N.i64p), N.ptr(ix, N.i64p),
                                    N.ptr(col, N.i32p), N.ptr(nc, N.i32p)))
    return col


def _factor_coarsest(matrix: sp.csr_matrix):
    """Dense factor of the node-0-grounded Laplacian (solver.py:394-403)."""
    n = matrix.shape[0]
    if n <= 1:
        return None
    dense = matrix.toarray()[1:, 1:]
    try:
        return ("cho", scipy.linalg.cho_factor(dense, lower=True, check_finite=False))
    except scipy.linalg.LinAlgError:
        return ("lu", scipy.linalg.lu_factor(dense, check_finite=False))


def _coarse_operator(level: Level) -> np.ndarray:
    """M = (I - 11^T/n) G+ with G+ the grounded inverse padded by a zero
    row/column: x = M b equals solver.py:406-419 (grounded solve of b[1:],
    x[0] = 0, then mean removal) as a single dense operator."""
    n = level.size
    kind, fac = level.grounded_factor
    eye = np.eye(n - 1)
    if kind == "cho":
        ginv = scipy.linalg.cho_solve(fac, eye, check_finite=False)
    else:
        ginv = scipy.linalg.lu_solve(fac, eye, check_finite=False)
    m = np.zeros((n, n))
    m[1:, 1:] = ginv
    return m - m.mean(axis=0, keepdims=True)


def setup(matrix: sp.spmatrix, config: SolverConfig | None = None,
          stall_breaker: bool | None = None) -> MultigridHierarchy:
    """Build the hierarchy with the reference's stage rule (solver.py:422-523).

    Elimination first; a stage shrinking the level by < 10 % yields to the
    other; if neither clears the bar the larger reduction is taken; the
    preferred stage alternates.  The result lives on the host until the first
    solve uploads it to the device.

    ``stall_breaker``: None (default) enables the stall breaker (see
    STALL_ELIM_CAP) on levels above DEVICE_DIRECT_MAX nodes or on graphs with
    more than STALL_BREAKER_MIN_N0 nodes; False reproduces the reference rule
    everywhere; True enables it on every level.
    """
    config = config or SolverConfig()
    current = _validate_laplacian(matrix)
    global _device_setup_on, _native_relax_on
    _device_setup_on = False
    _native_relax_on = False
    rng = np.random.default_rng(config.seed)
    levels: list[Level] = []
    preferred = LevelKind.ELIMINATION
    n0 = current.shape[0]
    tvecs: dict[int, np.ndarray] = {}

    def breaker_on(n_level: int) -> bool:
        if stall_breaker is not None:
            return bool(stall_breaker)
        return n0 > STALL_BREAKER_MIN_N0 or n_level > DEVICE_DIRECT_MAX
    def hub_level(mat) -> bool:
        if stall_breaker is False or n0 <= STALL_BREAKER_MIN_N0:
            return False
        offdeg = np.diff(mat.indptr) - 1
        return offdeg.max() > HUB_DEGREE_RATIO * max(offdeg.mean(), 1.0)
    # device coarse operators only on hub graphs (power-law: their hierarchies
    # already differ from the reference's); C3-like graphs keep the host
    # products and with them hierarchies identical to the reference's
    if stall_breaker is not False and n0 > DEVICE_SETUP_MIN_N0:
        od0 = np.diff(current.indptr) - 1
        _device_setup_on = bool(od0.max() > HUB_DEGREE_RATIO * max(od0.mean(), 1.0))
        _native_relax_on = _device_setup_on and os.environ.get("CF_NATIVE_RELAX", "1") != "0"
    while current.shape[0] > config.max_direct_size:
        n_cur = current.shape[0]
        need = MIN_REDUCTION * n_cur
        cand: dict[LevelKind, tuple] = {}

        def stage(kind: LevelKind):
            if kind not in cand:
                if kind is LevelKind.ELIMINATION:
                    schur, rec = coarsen_eliminate(current, config.elimination_degree_cap)
                    cand[kind] = (0 if rec is None else rec.f_nodes.size, schur, rec)
                else:
                    vec = relaxed_test_vectors(current, config.aggregation_test_vectors, rng)
                    tvecs[n_cur] = vec
                    cap = HUB_AGG_CAP if hub_level(current) else MAX_AGGREGATE_SIZE
                    coarse, agg = coarsen_aggregate(current, vec, cap)
                    red = n_cur - (int(agg.max()) + 1)
                    if red < need:
                        mc, ma = _matching_aggregation(current, vec)
                        mred = n_cur - (int(ma.max()) + 1)
                        if mred > red:
                            coarse, agg, red = mc, ma, mred
                    cand[kind] = (red, coarse, agg)
            return cand[kind]

        other = (LevelKind.AGGREGATION if preferred is LevelKind.ELIMINATION
                 else LevelKind.ELIMINATION)
        applied = next((k for k in (preferred, other) if stage(k)[0] >= need), None)
        if applied is None and breaker_on(n_cur):
            stage(LevelKind.AGGREGATION)
            offdeg = np.diff(current.indptr) - 1
            best_f = None
            for ecap in STALL_ELIM_CAPS:
                f = _elim_select(current, ecap)
                if f.size == n_cur and n_cur > 0:
                    f = f[:-1]
                # Schur fill is at most sum d_f^2 entries, and never more than the
                # remaining |C|^2 positions (duplicates merge)
                fill = min(float(np.sum(offdeg[f].astype(np.float64) ** 2)),
                           float(n_cur - f.size) ** 2)
                if fill > STALL_FILL_FACTOR * current.nnz and best_f is not None:
                    break  # escalation stops at the first cap over the budget
                if best_f is None or f.size > best_f.size:
                    best_f = f
            if best_f is not None and best_f.size:
                schur, rec = _eliminate_set(current, best_f)
            else:
                schur, rec = current, None
            alt = {"elim": (0 if rec is None else rec.f_nodes.size, schur, rec)}
            co, ag = coarsen_aggregate(current, tvecs[n_cur], STALL_AGG_CAP, STALL_AGG_THRESHOLD)
            alt["agg"] = (n_cur - (int(ag.max()) + 1), co, ag)
            best = max(alt, key=lambda k: alt[k][0])
            if alt[best][0] > max(c[0] for c in cand.values()):
                kind = LevelKind.ELIMINATION if best == "elim" else LevelKind.AGGREGATION
                cand[kind] = alt[best]
                applied = kind
        if applied is None:
            applied = max(cand, key=lambda k: cand[k][0])
            if cand[applied][0] <= 0:
                raise ConvergenceError("coarsening made no progress", best_residual=float("inf"))
        _, coarse, extra = cand[applied]
        if applied is LevelKind.ELIMINATION:
            levels.append(Level(kind=LevelKind.ELIMINATION, matrix=current, f_nodes=extra.f_nodes,
                                c_nodes=extra.c_nodes, f_degree=extra.f_degree, w_cf=extra.w_cf,
                                w_fc=extra.w_cf.T.tocsr()))
        else:
            n_agg = int(extra.max()) + 1
            levels.append(Level(kind=LevelKind.AGGREGATION, matrix=current,
                                p=sp.csr_matrix((np.ones(n_cur), (np.arange(n_cur), extra)),
                                                shape=(n_cur, n_agg)),
                                aggregates=extra, colors=_colour(current)))
        current = coarse
        preferred = (LevelKind.AGGREGATION if applied is LevelKind.ELIMINATION
                     else LevelKind.ELIMINATION)
    levels.append(Level(kind=LevelKind.COARSEST, matrix=current,
                        grounded_factor=_factor_coarsest(current)))
    sizes = [lvl.size for lvl in levels]
    assert all(a > b for a, b in zip(sizes, sizes[1:])), sizes
    return MultigridHierarchy(levels=levels, config=config)


# ---------------------------------------------------------------------------
# solve (device)
# ---------------------------------------------------------------------------

def _params(config: SolverConfig, n: int) -> N.CfSolveParams:
    p = N.CfSolveParams()
    p.tau = float(config.tau)
    p.max_cycles = int(config.max_cycles)
    p.nu1, p.nu2 = (int(s) for s in config.smoothing_steps)
    p.fcg_max_iters = FCG_MAX_ITERS
    p.jpcg_max_iters = max(2000, int(50 * np.sqrt(n)))
    p.stop_margin = STOP_MARGIN
    p.stagnation_factor = STAGNATION_FACTOR
    p.stagnation_cycles = STAGNATION_CYCLES
    return p


def _solve_rows(hierarchy: MultigridHierarchy, rows: np.ndarray, config: SolverConfig,
                out: np.ndarray | None = None):
    """rows: count x n (C-contiguous fp64) -> (values count x n, residuals)."""
    n = hierarchy.n
    count = rows.shape[0]
    if out is None:
        out = np.empty((count, n))
    elif (out.shape != (count, n) or out.dtype != np.float64
          or not out.flags.c_contiguous or not out.flags.writeable):
        raise DomainError(f"out must be a writeable C-contiguous float64 array of shape {(count, n)}")
    res = np.zeros(count)
    if count == 0:
        return out, res
    dev = hierarchy.device()
    st = N.CfSolveStats()
    N.check(N.lib().cf_solve_rows(dev.handle, N.ptr(rows, N.f64p), count,
                                  N.C.byref(_params(config, n)), N.ptr(out, N.f64p),
                                  N.ptr(res, N.f64p), N.C.byref(st)), st)
    hierarchy.stats.record(res, int(st.fallback_solves), int(st.vcycles),
                           int(st.krylov_solves))
    return out, res


def _as_rows(hierarchy: MultigridHierarchy, supplies) -> np.ndarray:
    s = np.asarray(supplies, dtype=np.float64)
    if s.ndim == 1:
        s = s.reshape(1, -1)
    if s.ndim != 2 or s.shape[1] != hierarchy.n:
        raise DomainError(f"right-hand side length {s.shape[-1]} != {hierarchy.n}")
    return np.ascontiguousarray(s)


def solve(hierarchy: MultigridHierarchy, b: Sequence[float] | np.ndarray,
          config: SolverConfig | None = None) -> PotentialVector:
    """Solve one Laplacian system to the configured relative residual
    (solver.py:754-768).  The supply must be balanced; the potential is
    mean-centred and its residual recomputed from the matrix."""
    config = config or hierarchy.config
    column = np.asarray(b, dtype=np.float64).reshape(-1)
    if column.size != hierarchy.n:
        raise DomainError(f"right-hand side length {column.size} != {hierarchy.n}")
    x, res = _solve_rows(hierarchy, np.ascontiguousarray(column.reshape(1, -1)), config)
    return PotentialVector(values=x[0], achieved_residual=float(res[0]))


def solve_many(hierarchy: MultigridHierarchy, supplies: Sequence[Sequence[float]] | np.ndarray,
               config: SolverConfig | None = None, threads: int = 1,
               out: np.ndarray | None = None) -> list[PotentialVector]:
    """Solve many systems over one hierarchy (solver.py:771-811).

    All rows are solved together on the device; every column is computed
    independently in a fixed order, so results do not depend on ``threads``
    (accepted for API compatibility), on batch composition or on order.

    ``out`` (extension, optional): a ``count x n`` float64 array that receives
    the potentials (the returned vectors are views of its rows).  Supplies and
    ``out`` in page-locked host memory are transferred by DMA directly.
    """
    config = config or hierarchy.config
    rows = _as_rows(hierarchy, supplies)
    x, res = _solve_rows(hierarchy, rows, config, out)
    return [PotentialVector(values=x[i], achieved_residual=float(res[i]))
            for i in range(rows.shape[0])]
