// Host-side hierarchy setup helpers: the sequential greedy loops of the
// reference setup (pkg/src/cfcent/solver.py:222-380) in C++.  The algebra
// around them (Schur complement, Galerkin product, Laplacian rebuild) stays
// in scipy so every level matrix is produced by the same operations as the
// reference; only the O(n) Python loops are moved here.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
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
    // transpose by counting sort, threaded over row ranges: thread t scatters
    // its rows after the entries of threads < t in every column, so each
    // column lists its rows in ascending order (as a sequential pass would)
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 4096));
    std::vector<int64_t> cut(nt + 1, n);
    cut[0] = 0;
    for (int64_t t = 1; t < nt; ++t)
        cut[t] = std::upper_bound(indptr, indptr + n + 1, nnz * t / nt) - indptr - 1;
    for (int64_t t = 1; t <= nt; ++t) cut[t] = std::max(cut[t], cut[t - 1]);
    auto run = [&](auto&& fn) {
        std::vector<std::thread> th;
        for (int64_t t = 0; t < nt; ++t) th.emplace_back(fn, t);
        for (auto& x : th) x.join();
    };
    std::vector<std::vector<int64_t>> tcnt(nt, std::vector<int64_t>(n, 0));
    run([&](int64_t t) {
        auto& c = tcnt[t];
        for (int64_t p = indptr[cut[t]]; p < indptr[cut[t + 1]]; ++p) ++c[indices[p]];
    });
    std::vector<int64_t> tptr(n + 1, 0);
    for (int64_t c = 0; c < n; ++c) {
        int64_t s = tptr[c];
        for (int64_t t = 0; t < nt; ++t) {
            const int64_t k = tcnt[t][c];
            tcnt[t][c] = s;  // thread t's first slot in column c
            s += k;
        }
        tptr[c + 1] = s;
    }
    std::vector<int64_t> tidx(nnz);
    std::vector<double> tval(nnz);
    run([&](int64_t t) {
        auto& pos = tcnt[t];
        for (int64_t i = cut[t]; i < cut[t + 1]; ++i)
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                const int64_t q = pos[indices[p]]++;
                tidx[q] = i;
                tval[q] = data[p];
            }
    });
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
    // rows are independent given the transpose: threads take row ranges of
    // equal entry counts, write into local buffers, then concatenate in order
    std::vector<std::vector<int64_t>> lidx(nt), lcnt(nt);
    std::vector<std::vector<double>> lval(nt);
    auto work = [&](int64_t t) {
        std::vector<double> acc(n, 0.0);
        std::vector<int64_t> mark(n, -1), cols, appear;
        auto& oi = lidx[t];
        auto& ov = lval[t];
        auto& oc = lcnt[t];
        oc.reserve((size_t)(cut[t + 1] - cut[t]));
        for (int64_t i = cut[t]; i < cut[t + 1]; ++i) {
            const size_t start = oi.size();
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
                    oi.push_back(i);
                    ov.push_back(dg);
                    placed = true;
                }
                double v = acc[j] * 0.5;
                if (j != i && v < 0.0) {
                    oi.push_back(j);
                    ov.push_back(v);
                }
            }
            if (!placed) {
                oi.push_back(i);
                ov.push_back(dg);
            }
            oc.push_back((int64_t)(oi.size() - start));
        }
    };
    {
        std::vector<std::thread> th;
        for (int64_t t = 0; t < nt; ++t) th.emplace_back(work, t);
        for (auto& x : th) x.join();
    }

    int64_t out = 0;
    out_ptr[0] = 0;
    for (int64_t t = 0; t < nt; ++t) {
        std::memcpy(out_idx + out, lidx[t].data(), sizeof(int64_t) * lidx[t].size());
        std::memcpy(out_val + out, lval[t].data(), sizeof(double) * lval[t].size());
        for (size_t r = 0; r < lcnt[t].size(); ++r) {
            const int64_t i = cut[t] + (int64_t)r;
            out_ptr[i + 1] = out_ptr[i] + lcnt[t][r];
        }
        out += (int64_t)lidx[t].size();
    }
    *nnz_out = out;
    CF_API_END
}

// Permuted CSR for the device upload (solver.py permute_levels): output row r
// is input row rows[r]; an entry (j, v) becomes (cmap[j], v); every output row
// is sorted by column.  Equivalent to scipy's A[rows][:, order] + sort_indices
// with cmap = inverse of order, threaded over rows.  out_ptr: nrows + 1.
extern "C" int cf_setup_permute(int64_t nrows, const int64_t* indptr, const int64_t* indices,
                                const double* data, const int64_t* rows, const int64_t* cmap,
                                int64_t* out_ptr, int64_t* out_idx, double* out_val) {
    out_ptr[0] = 0;
    for (int64_t r = 0; r < nrows; ++r)
        out_ptr[r + 1] = out_ptr[r] + (indptr[rows[r] + 1] - indptr[rows[r]]);
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, nrows / 4096));
    auto work = [&](int64_t r0, int64_t r1) {
        std::vector<std::pair<int64_t, double>> tmp;
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t a = indptr[rows[r]], b = indptr[rows[r] + 1], o = out_ptr[r];
            tmp.resize((size_t)(b - a));
            for (int64_t p = a; p < b; ++p) tmp[(size_t)(p - a)] = {cmap[indices[p]], data[p]};
            std::sort(tmp.begin(), tmp.end(),
                      [](const std::pair<int64_t, double>& x, const std::pair<int64_t, double>& y) {
                          return x.first < y.first;
                      });
            for (int64_t q = 0; q < b - a; ++q) {
                out_idx[o + q] = tmp[(size_t)q].first;
                out_val[o + q] = tmp[(size_t)q].second;
            }
        }
    };
    // row ranges of equal entry counts (hub rows would unbalance equal row counts)
    std::vector<int64_t> cut(nt + 1, nrows);
    cut[0] = 0;
    for (int64_t t = 1; t < nt; ++t)
        cut[t] = std::upper_bound(out_ptr, out_ptr + nrows + 1, out_ptr[nrows] * t / nt) - out_ptr - 1;
    for (int64_t t = 1; t <= nt; ++t) cut[t] = std::max(cut[t], cut[t - 1]);
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t)
        th.emplace_back(work, cut[t], cut[t + 1]);
    for (auto& x : th) x.join();
    return CF_OK;
}

// Test-vector relaxation (solver.py:264-275): `sweeps` forward Gauss-Seidel
// sweeps on L x = 0 for the `count` columns of x (n x count, row-major),
// x <- x + tril(L)^-1 (-(L x)) per sweep: residual with the old iterate, then
// a forward substitution, all columns of a row together.  Used on hub graphs
// (whose hierarchies are this build's own) in place of scipy's SuperLU
// triangular solves; L has sorted rows with the diagonal stored.
extern "C" int cf_setup_relax(int64_t n, const int64_t* indptr, const int64_t* indices,
                              const double* data, int32_t count, int32_t sweeps, double* x) {
    CF_API_BEGIN
    if (count < 1 || count > 64) throw cf::CfError(CF_DOMAIN, "test vector count must be in [1, 64]");
    const int k = count;
    std::vector<double> r((size_t)n * k), y((size_t)n * k);
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 4096));
    const int64_t nnz = indptr[n];
    std::vector<int64_t> cut(nt + 1, n);
    cut[0] = 0;
    for (int64_t t = 1; t < nt; ++t)
        cut[t] = std::upper_bound(indptr, indptr + n + 1, nnz * t / nt) - indptr - 1;
    for (int64_t t = 1; t <= nt; ++t) cut[t] = std::max(cut[t], cut[t - 1]);
    for (int s = 0; s < sweeps; ++s) {
        // r = -(L x), rows in parallel (each row: entries in column order)
        std::vector<std::thread> th;
        for (int64_t t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                double acc[64];
                for (int64_t i = cut[t]; i < cut[t + 1]; ++i) {
                    for (int c = 0; c < k; ++c) acc[c] = 0.0;
                    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                        const double a = data[p];
                        const double* xj = x + (size_t)indices[p] * k;
                        for (int c = 0; c < k; ++c) acc[c] += a * xj[c];
                    }
                    for (int c = 0; c < k; ++c) r[(size_t)i * k + c] = -acc[c];
                }
            });
        for (auto& t : th) t.join();
        // forward substitution tril(L) y = r (sequential over rows)
        double acc[64];
        for (int64_t i = 0; i < n; ++i) {
            for (int c = 0; c < k; ++c) acc[c] = r[(size_t)i * k + c];
            double d = 0.0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                const int64_t j = indices[p];
                if (j > i) break;
                if (j == i) {
                    d = data[p];
                    break;
                }
                const double a = data[p];
                const double* yj = y.data() + (size_t)j * k;
                for (int c = 0; c < k; ++c) acc[c] -= a * yj[c];
            }
            if (d == 0.0) throw cf::CfError(CF_DOMAIN, "zero diagonal in the test-vector relaxation");
            for (int c = 0; c < k; ++c) y[(size_t)i * k + c] = acc[c] / d;
        }
        for (size_t q = 0; q < (size_t)n * k; ++q) x[q] += y[q];
    }
    CF_API_END
}
