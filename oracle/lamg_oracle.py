"""Plain numpy/scipy restatement of the reference cfcent solve path (ORACLE).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  The product never
imports this module.

Everything here follows the reference package under
``pkg/src/cfcent`` (cited as ``solver.py:L``, ``graph.py:L`` ...).  The
restatement keeps the reference's numerical operations and their order
(scipy CSR products, ``spsolve_triangular`` Gauss-Seidel sweeps, LAPACK
Cholesky on the grounded coarsest matrix, numpy PCG64 streams), so for the
same inputs it reproduces the reference's hierarchies and solutions; the
pinning tests compare it to vectors produced by the reference itself.

Data model: a graph is a tuple ``(indptr, indices, weights)`` (each edge
stored twice, neighbours sorted, graph.py:30-98).  A hierarchy is a dict
``{"levels": [...], "cfg": OracleConfig}``, each level a dict with key
``kind`` in {"elim", "agg", "coarse"}.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components
from scipy.sparse.linalg import spsolve_triangular

# solver.py:48-58 (fixed algorithm constants)
AFF_THRESHOLD = 0.5
RELAX_SWEEPS = 3
AGG_CAP = 8
ATTACH_PASSES = 3
STAGE_MIN_REDUCTION = 0.10
STALL_FACTOR = 0.9
STALL_CYCLES = 5
FCG_ITERS = 200
COLUMN_BLOCK = 64
STOP_FRACTION = 0.9
# resistance.py:34
SKETCH_ROWS = 256


class OracleDomainError(ValueError):
    """Mirror of cfcent.errors.DomainError (errors.py:16-17)."""


class OracleConvergenceError(RuntimeError):
    """Mirror of cfcent.errors.ConvergenceError (errors.py:24-32)."""

    def __init__(self, msg: str, best_residual: float):
        super().__init__(f"{msg} (best relative residual {best_residual:.3e})")
        self.best_residual = best_residual


@dataclass(frozen=True)
class OracleConfig:
    """Same fields and defaults as SolverConfig (solver.py:61-74)."""

    tau: float = 1e-5
    max_cycles: int = 100
    max_direct_size: int = 200
    smoothing_steps: tuple = (1, 2)
    elimination_degree_cap: int = 4
    aggregation_test_vectors: int = 4
    seed: int = 0


# ----------------------------------------------------------------------------
# graph layer (graph.py)
# ----------------------------------------------------------------------------

def graph_from_edges(u, v, w=None, n=None):
    """Symmetrised CSR, loops dropped, duplicates summed (graph.py:100-147)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.ones(u.size) if w is None else np.asarray(w, dtype=np.float64)
    keep = u != v
    u, v, w = u[keep], v[keep], w[keep]
    if n is None:
        n = int(max(u.max(initial=-1), v.max(initial=-1)) + 1)
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    wt = np.concatenate([w, w])
    order = np.lexsort((dst, src))
    src, dst, wt = src[order], dst[order], wt[order]
    if src.size:
        first = np.ones(src.size, dtype=bool)
        first[1:] = (src[1:] != src[:-1]) | (dst[1:] != dst[:-1])
        starts = np.flatnonzero(first)
        wt = np.add.reduceat(wt, starts)
        src, dst = src[starts], dst[starts]
    counts = np.bincount(src, minlength=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, dst, wt


def canonical_edges(graph):
    """Edges (u<v) in (u, v) order (graph.py:78-86)."""
    indptr, indices, weights = graph
    n = indptr.size - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    sel = rows < indices
    return rows[sel], indices[sel], weights[sel]


def adjacency(graph):
    indptr, indices, weights = graph
    n = indptr.size - 1
    return sp.csr_matrix((weights, indices, indptr), shape=(n, n))


def laplacian(graph):
    """L = diag(A 1) - A (graph.py:253-258)."""
    a = adjacency(graph)
    deg = np.asarray(a.sum(axis=1)).ravel()
    return (sp.diags(deg, format="csr") - a).tocsr()


def largest_component(graph, labels=None):
    """LCC with smallest-label tie break (graph.py:217-250)."""
    indptr = graph[0]
    n = indptr.size - 1
    labels = np.arange(n, dtype=np.int64) if labels is None else labels
    ncomp, comp = connected_components(adjacency(graph), directed=False)
    if ncomp == 1:
        return graph, labels
    sizes = np.bincount(comp, minlength=ncomp)
    cands = np.flatnonzero(sizes == sizes.max())
    pick = cands[0] if cands.size == 1 else cands[
        int(np.argmin([labels[comp == c].min() for c in cands]))]
    keep = np.flatnonzero(comp == pick)
    newid = np.full(n, -1, dtype=np.int64)
    newid[keep] = np.arange(keep.size)
    eu, ev, ew = canonical_edges(graph)
    m = newid[eu] >= 0
    return graph_from_edges(newid[eu[m]], newid[ev[m]], ew[m], n=keep.size), labels[keep]


def grid_graph(rows, cols=None):
    """4-neighbour grid (generators.py:32-41)."""
    cols = rows if cols is None else cols
    ids = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    u = np.concatenate([ids[:, :-1].ravel(), ids[:-1, :].ravel()])
    v = np.concatenate([ids[:, 1:].ravel(), ids[1:, :].ravel()])
    return graph_from_edges(u, v, n=rows * cols)


def path_graph(n):
    """generators.py:24-29."""
    a = np.arange(n - 1, dtype=np.int64)
    return graph_from_edges(a, a + 1, n=n)


def barabasi_albert(n, m0, seed):
    """Urn-based preferential attachment (generators.py:94-127)."""
    rng = np.random.default_rng(seed)
    eu, ev, urn = [], [], []
    for i in range(m0 + 1):
        for j in range(i):
            eu.append(j)
            ev.append(i)
            urn.extend((i, j))
    for v in range(m0 + 1, n):
        picked = set()
        while len(picked) < m0:
            picked.add(urn[rng.integers(len(urn))])
        for u in sorted(picked):
            eu.append(u)
            ev.append(v)
            urn.extend((u, v))
    return graph_from_edges(np.asarray(eu), np.asarray(ev), n=n)


# ----------------------------------------------------------------------------
# hierarchy setup (solver.py:163-523)
# ----------------------------------------------------------------------------

def _restore_laplacian(mat):
    """Symmetrise, drop non-negative off-diagonals, rebuild the diagonal as
    minus the off-diagonal row sum (solver.py:167-187)."""
    mat = mat.tocsr()
    mat = (mat + mat.T) * 0.5
    t = mat.tocoo()
    sel = (t.row != t.col) & (t.data < 0)
    r, c, x = t.row[sel], t.col[sel], t.data[sel]
    n = mat.shape[0]
    d = np.zeros(n)
    np.add.at(d, r, -x)
    diag_idx = np.arange(n)
    out = sp.csr_matrix((np.concatenate([x, d]),
                         (np.concatenate([r, diag_idx]), np.concatenate([c, diag_idx]))),
                        shape=(n, n))
    out.sort_indices()
    return out


def _checked_laplacian(mat):
    """solver.py:190-211."""
    if mat.shape[0] != mat.shape[1]:
        raise OracleDomainError("matrix must be square")
    mat = mat.tocsr()
    n = mat.shape[0]
    big = float(np.abs(mat.data).max()) if mat.nnz else 0.0
    tol = 1e-12 * n * max(big, 1.0)
    skew = abs(mat - mat.T)
    if skew.nnz and skew.data.max() > tol:
        raise OracleDomainError("matrix is not symmetric")
    rs = np.asarray(mat.sum(axis=1)).ravel()
    if np.abs(rs).max(initial=0.0) > tol:
        raise OracleDomainError("row sums are not zero")
    t = mat.tocoo()
    off = t.row != t.col
    if off.any() and t.data[off].max() > tol:
        raise OracleDomainError("positive off-diagonal entry")
    if n > 1 and connected_components(mat, directed=False)[0] > 1:
        raise OracleDomainError("Laplacian graph is not connected")
    return _restore_laplacian(mat)


def eliminate_stage(mat, cap=4):
    """Greedy ascending-id independent set with off-degree <= cap, exact Schur
    complement (solver.py:222-261).  Returns (schur, record|None)."""
    mat = mat.tocsr()
    n = mat.shape[0]
    ptr, col = mat.indptr, mat.indices
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    offdeg = np.bincount(rows[col != rows], minlength=n)
    taken = np.zeros(n, dtype=bool)
    fine = []
    for i in np.flatnonzero(offdeg <= cap):
        if not taken[i]:
            fine.append(int(i))
            taken[col[ptr[i]:ptr[i + 1]]] = True
            taken[i] = True
    if n > 0 and len(fine) == n:
        fine.pop()
    if not fine:
        return mat, None
    f = np.asarray(fine, dtype=np.int64)
    is_f = np.zeros(n, dtype=bool)
    is_f[f] = True
    c = np.flatnonzero(~is_f)
    d_f = mat.diagonal()[f]
    w_cf = (-(mat[c][:, f].tocsr())).tocsr()
    schur = mat[c][:, c] - w_cf @ sp.diags(1.0 / d_f) @ w_cf.T
    rec = {"f": f, "c": c, "d_f": d_f, "w_cf": w_cf}
    return _restore_laplacian(schur), rec


def relax_test_vectors(mat, count, rng):
    """Centred Gaussian vectors after forward GS sweeps on Lx=0
    (solver.py:264-275)."""
    x = rng.standard_normal((mat.shape[0], count))
    x -= x.mean(axis=0, keepdims=True)
    low = sp.tril(mat, 0, format="csr")
    for _ in range(RELAX_SWEEPS):
        x += spsolve_triangular(low, -(mat @ x), lower=True)
    x -= x.mean(axis=0, keepdims=True)
    return x


def _galerkin_coarse(mat, agg, nagg):
    """P^T L P with piecewise-constant P (solver.py:383-386)."""
    n = mat.shape[0]
    p = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nagg))
    return _restore_laplacian(p.T @ mat @ p)


def affinity_aggregate(mat, tv):
    """Seeds by greedy independent set, then up to three attachment passes by
    maximal affinity > 0.5 with aggregate cap 8, leftovers as singletons
    (solver.py:278-346)."""
    mat = mat.tocsr()
    n = mat.shape[0]
    ptr, col = mat.indptr, mat.indices
    x = np.ascontiguousarray(tv)
    nrm = np.einsum("ij,ij->i", x, x)
    agg = np.full(n, -1, dtype=np.int64)
    size = []
    taken = np.zeros(n, dtype=bool)
    for u in range(n):
        if taken[u]:
            continue
        agg[u] = len(size)
        size.append(1)
        taken[col[ptr[u]:ptr[u + 1]]] = True
        taken[u] = True
    for _ in range(ATTACH_PASSES):
        moved = False
        for u in range(n):
            if agg[u] >= 0:
                continue
            nb = col[ptr[u]:ptr[u + 1]]
            nb = nb[nb != u]
            nb = nb[agg[nb] >= 0]
            if nb.size == 0 or nrm[u] <= 0:
                continue
            dots = x[nb] @ x[u]
            den = nrm[nb] * nrm[u]
            with np.errstate(divide="ignore", invalid="ignore"):
                aff = np.where(den > 0, dots * dots / den, 0.0)
            for k in np.argsort(-aff, kind="stable"):
                if aff[k] <= AFF_THRESHOLD:
                    break
                a = agg[nb[k]]
                if size[a] < AGG_CAP:
                    agg[u] = a
                    size[a] += 1
                    moved = True
                    break
        if not moved:
            break
    for u in np.flatnonzero(agg < 0):
        agg[u] = len(size)
        size.append(1)
    return _galerkin_coarse(mat, agg, len(size)), agg


def matching_aggregate(mat, tv):
    """Greedy pair matching by descending affinity (solver.py:349-380)."""
    mat = mat.tocsr()
    n = mat.shape[0]
    t = mat.tocoo()
    up = t.row < t.col
    eu, ev = t.row[up], t.col[up]
    nrm = np.einsum("ij,ij->i", tv, tv)
    dots = np.einsum("ij,ij->i", tv[eu], tv[ev])
    den = nrm[eu] * nrm[ev]
    aff = np.where(den > 0, dots * dots / den, 0.0)
    mate = np.full(n, -1, dtype=np.int64)
    for e in np.lexsort((ev, eu, -aff)):
        a, b = int(eu[e]), int(ev[e])
        if mate[a] < 0 and mate[b] < 0:
            mate[a], mate[b] = b, a
    agg = np.full(n, -1, dtype=np.int64)
    nxt = 0
    for u in range(n):
        if agg[u] >= 0:
            continue
        agg[u] = nxt
        if mate[u] > u:
            agg[mate[u]] = nxt
        nxt += 1
    return _galerkin_coarse(mat, agg, nxt), agg


def _coarsest_factor(mat):
    """Dense factor of the node-0-grounded matrix (solver.py:394-403)."""
    n = mat.shape[0]
    if n <= 1:
        return None
    g = mat.toarray()[1:, 1:]
    try:
        return ("cho", scipy.linalg.cho_factor(g, lower=True, check_finite=False))
    except scipy.linalg.LinAlgError:
        return ("lu", scipy.linalg.lu_factor(g, check_finite=False))


def build_hierarchy(lap, cfg: OracleConfig = OracleConfig()):
    """Stage alternation with the 10 % rule (solver.py:422-523)."""
    cur = _checked_laplacian(lap)
    rng = np.random.default_rng(cfg.seed)
    levels = []
    want = "elim"
    while cur.shape[0] > cfg.max_direct_size:
        n = cur.shape[0]
        need = STAGE_MIN_REDUCTION * n
        tried = {}

        def attempt(kind):
            if kind not in tried:
                if kind == "elim":
                    sc, rec = eliminate_stage(cur, cfg.elimination_degree_cap)
                    tried[kind] = (0 if rec is None else rec["f"].size, sc, rec)
                else:
                    tv = relax_test_vectors(cur, cfg.aggregation_test_vectors, rng)
                    co, agg = affinity_aggregate(cur, tv)
                    red = n - (int(agg.max()) + 1)
                    if red < need:
                        mco, magg = matching_aggregate(cur, tv)
                        mred = n - (int(magg.max()) + 1)
                        if mred > red:
                            co, agg, red = mco, magg, mred
                    tried[kind] = (red, co, agg)
            return tried[kind]

        alt = "agg" if want == "elim" else "elim"
        used = None
        for kind in (want, alt):
            if attempt(kind)[0] >= need:
                used = kind
                break
        if used is None:
            used = max(tried, key=lambda k: tried[k][0])
            if tried[used][0] <= 0:
                raise OracleConvergenceError("coarsening made no progress", float("inf"))
        _, coarse, extra = tried[used]
        if used == "elim":
            levels.append({"kind": "elim", "A": cur, "f": extra["f"], "c": extra["c"],
                           "d_f": extra["d_f"], "w_cf": extra["w_cf"],
                           "w_fc": extra["w_cf"].T.tocsr()})
        else:
            nagg = int(extra.max()) + 1
            levels.append({"kind": "agg", "A": cur, "agg": extra,
                           "P": sp.csr_matrix((np.ones(n), (np.arange(n), extra)),
                                              shape=(n, nagg)),
                           "lower": sp.tril(cur, 0, format="csr"),
                           "upper": sp.triu(cur, 0, format="csr")})
        cur = coarse
        want = "agg" if used == "elim" else "elim"
    levels.append({"kind": "coarse", "A": cur, "factor": _coarsest_factor(cur)})
    return {"levels": levels, "cfg": cfg, "stats": {"solves": 0, "max_residual": 0.0,
                                                     "fallback_solves": 0}}


# ----------------------------------------------------------------------------
# solve phase (solver.py:406-811)
# ----------------------------------------------------------------------------

def _coarse_direct(level, b):
    """Per-column grounded solve then re-centre (solver.py:406-419)."""
    out = np.zeros_like(b)
    if level["A"].shape[0] == 1 or level["factor"] is None:
        return out
    how, fac = level["factor"]
    for j in range(b.shape[1]):
        if how == "cho":
            out[1:, j] = scipy.linalg.cho_solve(fac, b[1:, j], check_finite=False)
        else:
            out[1:, j] = scipy.linalg.lu_solve(fac, b[1:, j], check_finite=False)
    out -= out.mean(axis=0, keepdims=True)
    return out


def vcycle(levels, j, b, nu1, nu2):
    """One V-cycle from zero (solver.py:526-560)."""
    lv = levels[j]
    if lv["kind"] == "coarse":
        return _coarse_direct(lv, b)
    if lv["kind"] == "elim":
        bf = b[lv["f"]]
        bc = b[lv["c"]] + lv["w_cf"] @ (bf / lv["d_f"][:, None])
        xc = vcycle(levels, j + 1, bc, nu1, nu2)
        x = np.empty_like(b)
        x[lv["c"]] = xc
        x[lv["f"]] = (bf + lv["w_fc"] @ xc) / lv["d_f"][:, None]
        return x
    A = lv["A"]
    x = spsolve_triangular(lv["lower"], b, lower=True)
    for _ in range(nu1 - 1):
        x += spsolve_triangular(lv["lower"], b - A @ x, lower=True)
    r = b - A @ x
    xc = vcycle(levels, j + 1, lv["P"].T @ r, nu1, nu2)
    d = lv["P"] @ xc
    ad = A @ d
    num = np.einsum("ij,ij->j", r, d)
    den = np.einsum("ij,ij->j", d, ad)
    x += d * np.divide(num, den, out=np.ones_like(num), where=den > 0)
    for _ in range(nu2):
        x += spsolve_triangular(lv["upper"], b - A @ x, lower=False)
    return x


def _cnorm(a):
    return np.sqrt(np.einsum("ij,ij->j", a, a))


def _cmean_removed(a):
    return a - a.mean(axis=0, keepdims=True)


def _flexible_cg(levels, x, b, bn, tau, nu1, nu2, iters):
    """V-cycle preconditioned FCG (solver.py:571-610)."""
    A = levels[0]["A"]
    cols = np.arange(b.shape[1])
    res = _cnorm(b - A @ x) / bn
    p = np.zeros_like(b)
    ap = np.zeros_like(b)
    seen = np.zeros(b.shape[1], dtype=bool)
    for _ in range(iters):
        cols = cols[res[cols] > tau]
        if cols.size == 0:
            break
        r = _cmean_removed(b[:, cols] - A @ x[:, cols])
        z = _cmean_removed(vcycle(levels, 0, r, nu1, nu2))
        old = seen[cols]
        if old.any():
            oc = cols[old]
            zl = np.einsum("ij,ij->j", z[:, old], ap[:, oc])
            dl = np.einsum("ij,ij->j", p[:, oc], ap[:, oc])
            z[:, old] -= p[:, oc] * np.divide(zl, dl, out=np.zeros_like(zl), where=dl > 0)
        p[:, cols] = z
        seen[cols] = True
        ap[:, cols] = A @ z
        dl = np.einsum("ij,ij->j", z, ap[:, cols])
        rd = np.einsum("ij,ij->j", r, z)
        x[:, cols] += z * np.divide(rd, dl, out=np.zeros_like(rd), where=dl > 0)
        x[:, cols] = _cmean_removed(x[:, cols])
        res[cols] = _cnorm(b[:, cols] - A @ x[:, cols]) / bn[cols]
    return x, res


def _jacobi_cg(A, x, b, bn, tau, iters):
    """Jacobi-preconditioned CG on the centred subspace (solver.py:613-648)."""
    dinv = 1.0 / np.maximum(A.diagonal(), np.finfo(float).tiny)
    r = _cmean_removed(b - A @ x)
    z = dinv[:, None] * r
    p = z.copy()
    rz = np.einsum("ij,ij->j", r, z)
    res = _cnorm(b - A @ x) / bn
    done = res <= tau
    for _ in range(iters):
        if done.all():
            break
        ap = A @ p
        pap = np.einsum("ij,ij->j", p, ap)
        a = np.divide(rz, pap, out=np.zeros_like(rz), where=pap > 0)
        a[done] = 0.0
        x += p * a
        r -= ap * a
        res = _cnorm(r) / bn
        done = done | (res <= tau)
        z = dinv[:, None] * r
        rz2 = np.einsum("ij,ij->j", r, z)
        beta = np.divide(rz2, rz, out=np.zeros_like(rz), where=rz > 0)
        beta[done] = 0.0
        p = z + p * beta
        rz = rz2
    x = _cmean_removed(x)
    return x, _cnorm(b - A @ x) / bn


def solve_columns(h, block, cfg: OracleConfig | None = None):
    """Per-column frozen V-cycle iteration + fallback chain
    (solver.py:651-751).  ``block`` is n x k.  Returns (x, res, n_fallback)."""
    cfg = cfg or h["cfg"]
    levels = h["levels"]
    A = levels[0]["A"]
    n = A.shape[0]
    if block.shape[0] != n:
        raise OracleDomainError(f"right-hand side length {block.shape[0]} != {n}")
    b = np.array(block, dtype=np.float64, copy=True)
    k = b.shape[1]
    x = np.zeros_like(b)
    if k == 0:
        return x, np.zeros(0), 0
    l1 = np.abs(b).sum(axis=0)
    unbalanced = np.abs(b.sum(axis=0)) > 1e-10 * np.maximum(l1, np.finfo(float).tiny)
    if unbalanced.any():
        raise OracleDomainError("supply vector columns are not balanced")
    bn = _cnorm(b)
    nz = bn > 0
    tau = cfg.tau
    stop = STOP_FRACTION * tau
    nu1, nu2 = cfg.smoothing_steps
    res = np.zeros(k)
    nfb = 0
    act = np.flatnonzero(nz)
    if act.size:
        safe = np.where(nz, bn, 1.0)
        stall = np.zeros(k, dtype=np.int64)
        prev = np.full(k, np.inf)
        rescue = []
        for _ in range(cfg.max_cycles):
            r = b[:, act] - A @ x[:, act]
            res[act] = _cnorm(r) / safe[act]
            ratio = res[act] / prev[act]
            stall[act] = np.where(ratio > STALL_FACTOR, stall[act] + 1, 0)
            prev[act] = res[act]
            ok = res[act] <= stop
            stuck = stall[act] >= STALL_CYCLES
            rescue.extend(act[stuck & ~ok].tolist())
            live = ~ok & ~stuck
            act = act[live]
            if act.size == 0:
                break
            x[:, act] += vcycle(levels, 0, _cmean_removed(r[:, live]), nu1, nu2)
            x[:, act] = _cmean_removed(x[:, act])
        else:
            r = b[:, act] - A @ x[:, act]
            res[act] = _cnorm(r) / safe[act]
            rescue.extend(act[~(res[act] <= stop)].tolist())
        if rescue:
            cols = np.asarray(sorted(rescue), dtype=np.int64)
            nfb = cols.size
            xf, rf = _flexible_cg(levels, x[:, cols].copy(), b[:, cols], bn[cols], stop,
                                  nu1, nu2, FCG_ITERS)
            x[:, cols] = xf
            res[cols] = rf
            left = cols[rf > stop]
            if left.size:
                xg, rg = _jacobi_cg(A, x[:, left].copy(), b[:, left], bn[left], stop,
                                    max(2000, int(50 * np.sqrt(n))))
                x[:, left] = xg
                res[left] = rg
            if (res[cols] > tau).any():
                raise OracleConvergenceError("solve(s) failed to reach tau",
                                             float(res[cols].max()))
    x = _cmean_removed(x)
    res = np.where(nz, _cnorm(b - A @ x) / np.where(nz, bn, 1.0), 0.0)
    st = h["stats"]
    st["solves"] += res.size
    if res.size:
        st["max_residual"] = max(st["max_residual"], float(res.max()))
    st["fallback_solves"] += nfb
    return x, res, nfb


def solve_rows(h, supplies, cfg: OracleConfig | None = None):
    """64-column blocks over row-wise supplies (solver.py:771-811).
    Returns (values count x n, residuals count)."""
    s = np.asarray(supplies, dtype=np.float64)
    if s.ndim == 1:
        s = s.reshape(1, -1)
    out = np.zeros((s.shape[0], h["levels"][0]["A"].shape[0]))
    res = np.zeros(s.shape[0])
    for lo in range(0, s.shape[0], COLUMN_BLOCK):
        hi = min(lo + COLUMN_BLOCK, s.shape[0])
        x, r, _ = solve_columns(h, s[lo:hi].T, cfg)
        out[lo:hi] = x.T
        res[lo:hi] = r
    return out, res


# ----------------------------------------------------------------------------
# estimators (resistance.py, centrality.py)
# ----------------------------------------------------------------------------

def sketch_rows(n, eps):
    """k = max(1, ceil(ln n / eps^2)) (resistance.py:156-158)."""
    return max(1, math.ceil(math.log(n) / eps ** 2))


def jl_rhs(graph, k, seed):
    """Rows of Q W^1/2 B with Q = +-1/sqrt(k) from default_rng(seed), drawn in
    256-row blocks, then row-centred (resistance.py:181-199).  Returns
    (rhs_uncentred, rhs_centred)."""
    n = graph[0].size - 1
    eu, ev, ew = canonical_edges(graph)
    m = eu.size
    inc = sp.csr_matrix((np.tile([1.0, -1.0], m),
                         (np.repeat(np.arange(m), 2), np.column_stack([eu, ev]).ravel())),
                        shape=(m, n))
    st = inc.multiply(np.sqrt(ew)[:, None]).T.tocsr()
    rng = np.random.default_rng(seed)
    s = 1.0 / math.sqrt(k)
    y = np.empty((k, n))
    for lo in range(0, k, SKETCH_ROWS):
        hi = min(lo + SKETCH_ROWS, k)
        q = (rng.integers(0, 2, size=(hi - lo, m)).astype(np.float64) * 2.0 - 1.0) * s
        y[lo:hi] = (st @ q.T).T
    raw = y.copy()
    y -= y.mean(axis=1, keepdims=True)
    return raw, y


def jl_sums(z, nodes):
    """Closed-form sum_w ||z_v - z_w||^2 (resistance.py:218-237)."""
    col_sq = np.einsum("ij,ij->j", z, z)
    idx = np.asarray(nodes, dtype=np.int64)
    return col_sq.sum() + z.shape[1] * col_sq[idx] - 2.0 * (z[:, idx].T @ z.sum(axis=1))


def closeness_projection(graph, h, query, eps, seed, cfg=None):
    """(n-1)/S_v (centrality.py:140-166).  Returns (scores, k, z)."""
    n = graph[0].size - 1
    k = sketch_rows(n, eps)
    _, rhs = jl_rhs(graph, k, seed)
    z, _ = solve_rows(h, rhs, cfg)
    sums = jl_sums(z, query)
    return (n - 1) / sums, k, z


def pivots(n, k, seed):
    """centrality.py:70-75."""
    return np.sort(np.random.default_rng(seed).choice(n, size=k, replace=False))


def node_potentials(h, nodes, cfg=None, cache=None):
    """Solutions of L z_x = e_x - 1/n (resistance.py:77-99)."""
    n = h["levels"][0]["A"].shape[0]
    cache = {} if cache is None else cache
    todo = sorted({int(x) for x in nodes} - cache.keys())
    if todo:
        rhs = np.full((len(todo), n), -1.0 / n)
        for i, x in enumerate(todo):
            rhs[i, x] += 1.0
        z, _ = solve_rows(h, rhs, cfg)
        for i, x in enumerate(todo):
            cache[x] = z[i]
    return cache


def resistances_from(h, v, targets, cfg=None, cache=None):
    """Four-term amortised formula (resistance.py:102-130)."""
    t = np.asarray(targets, dtype=np.int64)
    cache = node_potentials(h, np.r_[t, v], cfg, cache)
    zv = cache[int(v)]
    a = np.array([cache[int(w)][v] for w in t])
    b = np.array([cache[int(w)][w] for w in t])
    out = (zv[v] - zv[t]) - a + b
    out[t == v] = 0.0
    return out


def closeness_sampling(graph, h, query, k, seed, cfg=None):
    """(k/n)(n-1)/sum_t R(v,t) over shared pivots (centrality.py:104-137)."""
    n = graph[0].size - 1
    piv = pivots(n, k, seed)
    cache = {}
    out = []
    for v in query:
        out.append((k / n) * (n - 1) / float(resistances_from(h, v, piv, cfg, cache).sum()))
    return np.asarray(out)


def closeness_exact_pinv(graph):
    """Dense pseudo-inverse closeness (pkg/tests/conftest.py:35-45 oracle)."""
    L = laplacian(graph).toarray()
    pinv = np.linalg.pinv(L)
    d = np.diag(pinv)
    r = d[:, None] + d[None, :] - 2.0 * pinv
    return (L.shape[0] - 1) / r.sum(axis=1)


def jl_exact_pinv(graph, k, seed, query):
    """JL closeness with the same Q but exact solves (pinv)."""
    n = graph[0].size - 1
    _, rhs = jl_rhs(graph, k, seed)
    pinv = np.linalg.pinv(laplacian(graph).toarray())
    z = rhs @ pinv
    return (n - 1) / jl_sums(z, query)
