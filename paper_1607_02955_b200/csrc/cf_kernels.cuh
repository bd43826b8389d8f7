// sm_100a kernels for the batched multigrid solve (reference: solver.py:526-751).
//
// Layout: a block of KC right-hand sides over n nodes is stored row-major,
// X[i * KC + j].  One "row group" of LPR = min(KC, 32) lanes owns a node row;
// each lane owns VEC = KC / LPR consecutive columns, so every gather of a
// neighbour row X[j, :] is one coalesced KC*8-byte load per row group and
// every column is computed by exactly one lane in a fixed order: results are
// bitwise independent of which other columns share the block.
//
// All reductions are deterministic: each CTA owns a fixed partition of
// kRowsPerPart rows, reduces its rows in a fixed order in shared memory and
// writes one partial per column; cf_finalize sums the partials in order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cf {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerPart = 256;

// One row group per warp for every width: the row -> (warp, pass) mapping and
// hence every reduction order is identical for all KC, so a column's result
// does not depend on the width of the block it was solved in.  For KC < 32
// only the first KC lanes work (narrow blocks are latency-bound anyway).
template <int KC>
struct Lay {
    static constexpr int LPR = KC < 32 ? KC : 32;  // working lanes per row group
    static constexpr int VEC = KC / LPR;           // doubles per lane
    static constexpr int RPW = 1;                  // row groups per warp
    static constexpr int RPB = kWarps;             // row groups per CTA pass
};

template <int V>
struct DV {
    double v[V];
};

template <int V>
__device__ __forceinline__ DV<V> ldv(const double* __restrict__ p) {
    DV<V> r;
    if constexpr (V % 2 == 0) {
#pragma unroll
        for (int t = 0; t < V / 2; ++t) {
            double2 q = __ldg(reinterpret_cast<const double2*>(p) + t);
            r.v[2 * t] = q.x;
            r.v[2 * t + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int t = 0; t < V; ++t) r.v[t] = __ldg(p + t);
    }
    return r;
}

// plain (coherent) load: for data written earlier in the same kernel by the same lane
template <int V>
__device__ __forceinline__ DV<V> ldv_c(const double* p) {
    DV<V> r;
    if constexpr (V % 2 == 0) {
#pragma unroll
        for (int t = 0; t < V / 2; ++t) {
            double2 q = reinterpret_cast<const double2*>(p)[t];
            r.v[2 * t] = q.x;
            r.v[2 * t + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int t = 0; t < V; ++t) r.v[t] = p[t];
    }
    return r;
}

template <int V>
__device__ __forceinline__ void stv(double* p, const DV<V>& r) {
    if constexpr (V % 2 == 0) {
#pragma unroll
        for (int t = 0; t < V / 2; ++t)
            reinterpret_cast<double2*>(p)[t] = make_double2(r.v[2 * t], r.v[2 * t + 1]);
    } else {
#pragma unroll
        for (int t = 0; t < V; ++t) p[t] = r.v[t];
    }
}

template <int V>
__device__ __forceinline__ void zero(DV<V>& r) {
#pragma unroll
    for (int t = 0; t < V; ++t) r.v[t] = 0.0;
}

// acc += sum_p val[p] * X[map(col[p]), c0 : c0+V]  over p in [beg, end), ascending p.
template <int KC, bool MAPPED>
__device__ __forceinline__ void gather_row(const int32_t* __restrict__ col,
                                           const double* __restrict__ val, int64_t beg,
                                           int64_t end, const int32_t* __restrict__ map,
                                           const double* __restrict__ X, int c0,
                                           DV<Lay<KC>::VEC>& acc) {
    constexpr int V = Lay<KC>::VEC;
    int64_t p = beg;
    for (; p + 4 <= end; p += 4) {
        int j[4];
        double a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            j[u] = __ldg(col + p + u);
            a[u] = __ldg(val + p + u);
        }
        if constexpr (MAPPED) {
#pragma unroll
            for (int u = 0; u < 4; ++u) j[u] = __ldg(map + j[u]);
        }
        DV<V> x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ldv<V>(X + (size_t)j[u] * KC + c0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int t = 0; t < V; ++t) acc.v[t] = fma(a[u], x[u].v[t], acc.v[t]);
    }
    for (; p < end; ++p) {
        int j = __ldg(col + p);
        double a = __ldg(val + p);
        if constexpr (MAPPED) j = __ldg(map + j);
        DV<V> x = ldv<V>(X + (size_t)j * KC + c0);
#pragma unroll
        for (int t = 0; t < V; ++t) acc.v[t] = fma(a, x.v[t], acc.v[t]);
    }
}

// ---------------------------------------------------------------------------
// CTA-level deterministic column reduction: every thread holds NQ partial
// vectors of VEC columns for its row slot; reduce over the RPB row slots in
// slot order and write parts[q][part][KC].
template <int KC, int NQ>
__device__ __forceinline__ void cta_reduce_store(DV<Lay<KC>::VEC> (&loc)[NQ], double* smem,
                                                 double* __restrict__ parts, int64_t nparts,
                                                 int64_t part) {
    using L = Lay<KC>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int slot = warp;
    const int c0 = lane * L::VEC;
    if (lane < L::LPR) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int t = 0; t < L::VEC; ++t)
                smem[((size_t)q * L::RPB + slot) * KC + c0 + t] = loc[q].v[t];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < NQ * KC; idx += blockDim.x) {
        int q = idx / KC, c = idx % KC;
        double s = 0.0;
        for (int r = 0; r < L::RPB; ++r) s += smem[((size_t)q * L::RPB + r) * KC + c];
        parts[((size_t)q * nparts + part) * KC + c] = s;
    }
}

}  // namespace cf
