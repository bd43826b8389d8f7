// Host-side hierarchy setup helpers: the sequential greedy loops of the
// reference setup (pkg/src/cfcent/solver.py:222-380) in C++.  The algebra
// around them (Schur complement, Galerkin product, Laplacian rebuild) stays
// in scipy so every level matrix is produced by the same operations as the
// reference; only the O(n) Python loops are moved here.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "cfcent_b200.h"
#include "cf_common.h"

extern "C" int cf_setup_elim_select(int64_t n, const int64_t* indptr, const int64_t* indices,
                                    int32_t cap, int64_t* out_f, int64_t* n_f) {
    // solver.py:236-247: off-degree counts exclude the diagonal entry; nodes
    // with off-degree <= cap are taken in ascending id order unless a
    // previously taken node is adjacent; never every node.
    std::vector<uint8_t> blocked(n, 0);
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t off = 0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) off += (indices[p] != i);
        if (off > cap || blocked[i]) continue;
        out_f[cnt++] = i;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) blocked[indices[p]] = 1;
        blocked[i] = 1;
    }
    if (cnt == n && n > 0) --cnt;
    *n_f = cnt;
    return CF_OK;
}

extern "C" int cf_setup_aggregate(int64_t n, const int64_t* indptr, const int64_t* indices,
                                  const double* tv, int32_t nt, int32_t cap, double threshold,
                                  int64_t* out_agg, int64_t* n_agg) {
    // solver.py:297-346.  Affinity of u,v: <x_u,x_v>^2 / (|x_u|^2 |x_v|^2).
    // cap = MAX_AGGREGATE_SIZE (8) reproduces the reference; the stall breaker
    // of the B200 setup retries with larger caps.
    const double kThreshold = threshold;  // AFFINITY_THRESHOLD = 0.5 in the reference
    const int kCap = cap, kPasses = 3;
    std::vector<double> nrm(n);
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int t = 0; t < nt; ++t) s += tv[i * nt + t] * tv[i * nt + t];
        nrm[i] = s;
    }
    std::vector<int64_t> agg(n, -1);
    std::vector<int32_t> size;
    size.reserve(n);
    std::vector<uint8_t> blocked(n, 0);
    for (int64_t u = 0; u < n; ++u) {  // seeds: greedy independent set
        if (blocked[u]) continue;
        agg[u] = (int64_t)size.size();
        size.push_back(1);
        for (int64_t p = indptr[u]; p < indptr[u + 1]; ++p) blocked[indices[p]] = 1;
        blocked[u] = 1;
    }
    std::vector<int64_t> nb;
    std::vector<double> aff;
    std::vector<int32_t> ord;
    for (int pass = 0; pass < kPasses; ++pass) {
        bool moved = false;
        for (int64_t u = 0; u < n; ++u) {
            if (agg[u] >= 0) continue;
            nb.clear();
            for (int64_t p = indptr[u]; p < indptr[u + 1]; ++p) {
                int64_t v = indices[p];
                if (v != u && agg[v] >= 0) nb.push_back(v);
            }
            if (nb.empty() || nrm[u] <= 0.0) continue;
            aff.resize(nb.size());
            for (size_t q = 0; q < nb.size(); ++q) {
                int64_t v = nb[q];
                double d = 0.0;
                for (int t = 0; t < nt; ++t) d += tv[v * nt + t] * tv[u * nt + t];
                double den = nrm[v] * nrm[u];
                aff[q] = den > 0.0 ? d * d / den : 0.0;
            }
            ord.resize(nb.size());
            for (size_t q = 0; q < nb.size(); ++q) ord[q] = (int32_t)q;
            // np.argsort(-aff, kind="stable"): descending, ties by position
            std::stable_sort(ord.begin(), ord.end(),
                             [&](int32_t a, int32_t b) { return -aff[a] < -aff[b]; });
            for (int32_t q : ord) {
                if (aff[q] <= kThreshold) break;
                int64_t a = agg[nb[q]];
                if (size[a] < kCap) {
                    agg[u] = a;
                    size[a] += 1;
                    moved = true;
                    break;
                }
            }
        }
        if (!moved) break;
    }
    for (int64_t u = 0; u < n; ++u) {
        if (agg[u] < 0) {
            agg[u] = (int64_t)size.size();
            size.push_back(1);
        }
    }
    std::memcpy(out_agg, agg.data(), sizeof(int64_t) * n);
    *n_agg = (int64_t)size.size();
    return CF_OK;
}

extern "C" int cf_setup_matching(int64_t n, int64_t ne, const int64_t* eu, const int64_t* ev,
                                 const int64_t* order, int64_t* out_agg, int64_t* n_agg) {
    // solver.py:364-380: visit edges by (descending affinity, u, v); match
    // both endpoints if both are free; number aggregates by smallest member.
    std::vector<int64_t> mate(n, -1);
    for (int64_t q = 0; q < ne; ++q) {
        int64_t e = order[q];
        int64_t u = eu[e], v = ev[e];
        if (mate[u] < 0 && mate[v] < 0) {
            mate[u] = v;
            mate[v] = u;
        }
    }
    for (int64_t i = 0; i < n; ++i) out_agg[i] = -1;
    int64_t next = 0;
    for (int64_t u = 0; u < n; ++u) {
        if (out_agg[u] >= 0) continue;
        out_agg[u] = next;
        if (mate[u] > u) out_agg[mate[u]] = next;
        ++next;
    }
    *n_agg = next;
    return CF_OK;
}

extern "C" int cf_setup_colour(int64_t n, const int64_t* indptr, const int64_t* indices,
                               int32_t* colour, int32_t* n_colors) {
    // Greedy first-fit colouring in ascending node order.  The B200 smoother
    // sweeps colour classes in order (forward) / reverse order (backward)
    // instead of the reference's natural row order (solver.py:545,559).
    std::vector<int64_t> seen;  // seen[c] == i  <=> colour c used by a neighbour of i
    int32_t nc = 0;
    for (int64_t i = 0; i < n; ++i) colour[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            int64_t j = indices[p];
            if (j == i) continue;
            int32_t c = colour[j];
            if (c >= 0) {
                if ((size_t)c >= seen.size()) seen.resize(c + 1, -1);
                seen[c] = i;
            }
        }
        int32_t c = 0;
        while ((size_t)c < seen.size() && seen[c] == i) ++c;
        colour[i] = c;
        nc = std::max(nc, c + 1);
    }
    *n_colors = nc;
    return CF_OK;
}

extern "C" int cf_build_csr(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                            const double* w, int64_t* indptr, int64_t* indices, double* weights,
                            int64_t* nnz_out) {
    // graph.py:133-146: entries (u,v,w) then (v,u,w) in input order, stable
    // sort by (row, col), duplicates summed left to right.  Counting sort by
    // row keeps input order; a stable per-row sort by column follows.
    CF_API_BEGIN
    std::vector<int64_t> cnt(n + 1, 0);
    for (int64_t e = 0; e < m; ++e) {
        ++cnt[u[e] + 1];
        ++cnt[v[e] + 1];
    }
    for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    std::vector<int64_t> col(2 * m);
    std::vector<double> val(2 * m);
    for (int64_t e = 0; e < m; ++e) {  // first all (u -> v) entries, then all (v -> u)
        int64_t p = pos[u[e]]++;
        col[p] = v[e];
        val[p] = w[e];
    }
    for (int64_t e = 0; e < m; ++e) {
        int64_t p = pos[v[e]]++;
        col[p] = u[e];
        val[p] = w[e];
    }
    int64_t out = 0;
    indptr[0] = 0;
    std::vector<int64_t> ord;
    for (int64_t i = 0; i < n; ++i) {
        int64_t a = cnt[i], b = cnt[i + 1];
        ord.resize(b - a);
        for (int64_t q = 0; q < b - a; ++q) ord[q] = a + q;
        std::stable_sort(ord.begin(), ord.end(),
                         [&](int64_t x, int64_t y) { return col[x] < col[y]; });
        for (size_t q = 0; q < ord.size();) {
            int64_t c = col[ord[q]];
            double s = val[ord[q]];
            size_t r = q + 1;
            while (r < ord.size() && col[ord[r]] == c) s += val[ord[r++]];
            indices[out] = c;
            weights[out] = s;
            ++out;
            q = r;
        }
        indptr[i + 1] = out;
    }
    *nnz_out = out;
    CF_API_END
}

extern "C" int cf_rebuild_laplacian(int64_t n, const int64_t* indptr, const int64_t* indices,
                                    const double* data, int64_t* out_ptr, int64_t* out_idx,
                                    double* out_val, int64_t* nnz_out) {
    // solver.py:167-187 _rebuild_laplacian: (M + M^T) * 0.5, keep strictly
    // negative off-diagonals, diagonal = 0 - v_1 - v_2 - ... over the kept
    // off-diagonals of the row in column order (np.add.at order), sorted
    // indices.  Input: CSR without duplicate entries (any column order).
    CF_API_BEGIN
    const int64_t nnz = indptr[n];
    // transpose by counting sort
    std::vector<int64_t> tptr(n + 1, 0);
    for (int64_t p = 0; p < nnz; ++p) ++tptr[indices[p] + 1];
    for (int64_t i = 0; i < n; ++i) tptr[i + 1] += tptr[i];
    std::vector<int64_t> tpos(tptr.begin(), tptr.end() - 1), tidx(nnz);
    std::vector<double> tval(nnz);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            int64_t q = tpos[indices[p]]++;
            tidx[q] = i;
            tval[q] = data[p];
        }
    // scipy adds M + M^T with its canonical kernel (sorted output) when both
    // operands have sorted, duplicate-free rows, else with the general kernel
    // whose rows come out in reverse first-appearance order (M's row in
    // storage order, then M^T's); the diagonal is accumulated in that order.
    bool canonical = true;
    for (int64_t i = 0; i < n && canonical; ++i)
        for (int64_t p = indptr[i] + 1; p < indptr[i + 1]; ++p)
            if (indices[p] <= indices[p - 1]) {
                canonical = false;
                break;
            }
    std::vector<double> acc(n, 0.0);
    std::vector<int64_t> mark(n, -1), cols, appear;
    int64_t out = 0;
    out_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        appear.clear();
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            int64_t j = indices[p];
            if (mark[j] != i) {
                mark[j] = i;
                acc[j] = 0.0;
                appear.push_back(j);
            }
            acc[j] += data[p];
        }
        for (int64_t p = tptr[i]; p < tptr[i + 1]; ++p) {
            int64_t j = tidx[p];
            if (mark[j] != i) {
                mark[j] = i;
                acc[j] = 0.0;
                appear.push_back(j);
            }
            acc[j] += tval[p];
        }
        cols.assign(appear.begin(), appear.end());
        std::sort(cols.begin(), cols.end());
        double dg = 0.0;
        if (canonical) {
            for (int64_t j : cols) {
                double v = acc[j] * 0.5;
                if (j != i && v < 0.0) dg += -v;
            }
        } else {
            for (auto it = appear.rbegin(); it != appear.rend(); ++it) {
                int64_t j = *it;
                double v = acc[j] * 0.5;
                if (j != i && v < 0.0) dg += -v;
            }
        }
        bool placed = false;
        for (int64_t j : cols) {
            if (!placed && j > i) {
                out_idx[out] = i;
                out_val[out++] = dg;
                placed = true;
            }
            double v = acc[j] * 0.5;
            if (j != i && v < 0.0) {
                out_idx[out] = j;
                out_val[out++] = v;
            }
        }
        if (!placed) {
            out_idx[out] = i;
            out_val[out++] = dg;
        }
        out_ptr[i + 1] = out;
    }
    *nnz_out = out;
    CF_API_END
}
