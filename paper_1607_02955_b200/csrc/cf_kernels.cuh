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

#include <cstdlib>
#include <string>
#include <utility>

// Programmatic dependent launch (sm_90+): every kernel first waits for the
// grid it depends on (no-op without a programmatic dependency), then lets its
// own dependents start launching, so a dependent kernel's launch and prologue
// overlap the tail of this one.
#define CF_PDL_ENTRY()                                      \
    do {                                                    \
        asm volatile("griddepcontrol.wait;" ::: "memory");  \
        asm volatile("griddepcontrol.launch_dependents;");  \
    } while (0)

namespace cf {

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CF_PDL");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

// kernel launch with the programmatic-stream-serialization attribute
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef CF_ROWS_PER_PART
#define CF_ROWS_PER_PART 32
#endif
constexpr int kRowsPerPart = CF_ROWS_PER_PART;
#ifndef CF_GATHER_CTAS
#define CF_GATHER_CTAS 3
#endif
constexpr int kGatherCtas = CF_GATHER_CTAS;  // min CTAs per SM for sweep kernels (register cap)

// One row group per warp for every width: the row -> (warp, pass) mapping and
// hence every reduction order is identical for all KC, so a column's result
// does not depend on the width of the block it was solved in.  For KC < 32
// only the first KC lanes work (narrow blocks are latency-bound anyway).
template <int KC>
struct Lay {
    // working lanes per row group.  Widths 160 / 192 (remainder chunks) keep 32
    // lanes of 5 / 6 columns (64 / 128-bit accesses).  The alternative of 20 /
    // 24 lanes of 8 columns (two 256-bit accesses per lane) was measured slower
    // on C5 (block solve 818 vs 690 ms at 160, 844 vs 795 ms at 192): fewer
    // index entries per chunk and fewer neighbour rows in flight per warp.
    static constexpr int LPR = KC < 32 ? KC : 32;
    static constexpr int VEC = KC / LPR;           // doubles per lane
    static constexpr int RPW = 1;                  // row groups per warp
    static constexpr int RPB = kWarps;             // row groups per CTA pass
};

template <int V>
struct DV {
    double v[V];
};

// Row-slice loads/stores.  A lane's V consecutive doubles are 32-byte aligned
// when V % 4 == 0 (rows are KC * 8 bytes, KC >= 128), so one 256-bit access
// (LDG.E.256 / STG.E.256, sm_100) moves them; a warp then reads a 1 KB row
// with a single instruction.
#ifndef CF_LDG256
#define CF_LDG256 1
#endif
template <int V>
__device__ __forceinline__ DV<V> ldv(const double* __restrict__ p) {
    DV<V> r;
    if constexpr (CF_LDG256 && V % 4 == 0) {
#pragma unroll
        for (int t = 0; t < V / 4; ++t)
            asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(r.v[4 * t]), "=d"(r.v[4 * t + 1]), "=d"(r.v[4 * t + 2]),
                           "=d"(r.v[4 * t + 3])
                         : "l"(p + 4 * t));
    } else if constexpr (V % 2 == 0) {
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
    if constexpr (CF_LDG256 && V % 4 == 0) {
#pragma unroll
        for (int t = 0; t < V / 4; ++t)
            asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(r.v[4 * t]), "=d"(r.v[4 * t + 1]), "=d"(r.v[4 * t + 2]),
                           "=d"(r.v[4 * t + 3])
                         : "l"(p + 4 * t)
                         : "memory");
    } else if constexpr (V % 2 == 0) {
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
    if constexpr (CF_LDG256 && V % 4 == 0) {
#pragma unroll
        for (int t = 0; t < V / 4; ++t)
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * t),
                         "d"(r.v[4 * t]), "d"(r.v[4 * t + 1]), "d"(r.v[4 * t + 2]),
                         "d"(r.v[4 * t + 3])
                         : "memory");
    } else if constexpr (V % 2 == 0) {
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

// Gather modes: what the CSR entry (j, a) of a row multiplies.
enum GatherMode { G_PLAIN = 0, G_MAPPED = 1, G_ELIM = 2, G_DIV = 3 };

// acc += sum_p val[p] * Y(col[p]) over p in [beg, end), ascending p (one fma
// chain per column, identical for every block width), where
//   G_PLAIN : Y(j) = X[j, :]
//   G_MAPPED: Y(j) = X[map[j], :]                 (P xc gathers)
//   G_ELIM  : Y(j) = X[map[j], :] / div[j]        (W_cf (b_f / d_f))
//   G_DIV   : Y(j) = X[j, :] / div[p]             (G_ELIM with the map and the
//             divisor resolved per entry at upload: one dependent load less)
// The working lanes of the warp load LPR consecutive (col, val) pairs with one
// coalesced access and broadcast them by shuffle; up to 8 neighbour rows are
// then in flight per warp.
// Streaming loads of matrix entries (read once per launch): with
// CF_EVICT_FIRST they are marked L2::evict_first so they do not displace the
// neighbour rows of X that later rows gather again.
#ifndef CF_EVICT_FIRST
#define CF_EVICT_FIRST 0
#endif
#if CF_EVICT_FIRST
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
#endif
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
#if CF_EVICT_FIRST
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
        : "=r"(v) : "l"(p), "l"(evict_first_policy()));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double ld_stream(const double* p) {
#if CF_EVICT_FIRST
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
        : "=d"(v) : "l"(p), "l"(evict_first_policy()));
    return v;
#else
    return __ldg(p);
#endif
}

// A lane's share of one W-entry chunk of a CSR row: lane u < W holds entry
// p0 + u (column, value and, for G_ELIM, the divisor), or zeros past `end`.
template <int KC, int MODE>
__device__ __forceinline__ void fetch_chunk(const int32_t* __restrict__ col,
                                            const double* __restrict__ val,
                                            const int32_t* __restrict__ map,
                                            const double* __restrict__ div, int64_t p0,
                                            int64_t end, int& jj, double& aa, double& dd) {
    constexpr int W = Lay<KC>::LPR;
    const int lane = threadIdx.x & 31;
    jj = 0;
    aa = 0.0;
    dd = 1.0;
    if (p0 + lane < end && lane < W) {
        jj = ld_stream(col + p0 + lane);
        aa = ld_stream(val + p0 + lane);
        if constexpr (MODE == G_ELIM) dd = __ldg(div + jj);
        if constexpr (MODE == G_DIV) dd = ld_stream(div + p0 + lane);
        if constexpr (MODE == G_MAPPED || MODE == G_ELIM) jj = __ldg(map + jj);
    }
}

// acc += sum_p val[p] * Y(col[p]) over p in [beg, end), ascending p (one fma
// chain per column, identical for every block width), where
//   G_PLAIN : Y(j) = X[j, :]
//   G_MAPPED: Y(j) = X[map[j], :]                 (P xc gathers)
//   G_ELIM  : Y(j) = X[map[j], :] / div[j]        (W_cf (b_f / d_f))
//   G_DIV   : Y(j) = X[j, :] / div[p]             (G_ELIM with the map and the
//             divisor resolved per entry at upload: one dependent load less)
// The working lanes of the warp load LPR consecutive (col, val) pairs with one
// coalesced access and broadcast them by shuffle; up to G neighbour rows are
// then in flight per warp.  (jj, aa, dd) is the lane's share of the first chunk
// (fetch_chunk at beg), which a row pipeline loads one row ahead.
#ifndef CF_GATHER_DOUBLES
#define CF_GATHER_DOUBLES 16
#endif
#ifndef CF_GATHER_ROWS_MAX
#define CF_GATHER_ROWS_MAX 8
#endif
template <int KC, int MODE, int GD = CF_GATHER_DOUBLES>
__device__ __forceinline__ void gather_row_from(const int32_t* __restrict__ col,
                                                const double* __restrict__ val, int64_t beg,
                                                int64_t end, const int32_t* __restrict__ map,
                                                const double* __restrict__ div,
                                                const double* __restrict__ X, int c0,
                                                DV<Lay<KC>::VEC>& acc, int jj, double aa,
                                                double dd, int jlim = 0x7fffffff) {
    // jlim: neighbour rows j >= jlim are known to hold zero and are not read
    constexpr int V = Lay<KC>::VEC;
    constexpr int W = Lay<KC>::LPR;
    constexpr unsigned MASK = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
    // rows in flight per group: GD doubles of row data per lane (default
    // CF_GATHER_DOUBLES, so the gather kernels fit 3 CTAs of 256 threads per SM)
    // (at most 8 rows: 16 rows of narrow blocks spilled under the register cap)
    constexpr int G0 = GD / V > 0 ? (GD / V > CF_GATHER_ROWS_MAX ? CF_GATHER_ROWS_MAX : GD / V) : 1;
    constexpr int G = W < G0 ? W : G0;
    int jn = 0;
    double an = 0.0, dn = 1.0;
    for (int64_t p0 = beg; p0 < end; p0 += W) {
        const int cnt = (int)min((int64_t)W, end - p0);
        // next chunk's indices overlap this chunk's row loads
        if (p0 + W < end) fetch_chunk<KC, MODE>(col, val, map, div, p0 + W, end, jn, an, dn);
        for (int u0 = 0; u0 < cnt; u0 += G) {
            DV<V> x[G];
            double a[G], d[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                // source lanes are absolute (< W), so the full shuffle width also
                // serves row groups whose lane count is not a power of two
                int j = __shfl_sync(MASK, jj, u0 + u, 32);
                a[u] = __shfl_sync(MASK, aa, u0 + u, 32);
                if constexpr (MODE == G_ELIM || MODE == G_DIV) d[u] = __shfl_sync(MASK, dd, u0 + u, 32);
                if (u0 + u < cnt && j < jlim)
                    x[u] = ldv<V>(X + (size_t)j * KC + c0);
                else
                    zero(x[u]);
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                if (u0 + u < cnt) {
#pragma unroll
                    for (int t = 0; t < V; ++t) {
                        if constexpr (MODE == G_ELIM || MODE == G_DIV)
                            acc.v[t] = fma(a[u], x[u].v[t] / d[u], acc.v[t]);
                        else
                            acc.v[t] = fma(a[u], x[u].v[t], acc.v[t]);
                    }
                }
            }
        }
        jj = jn;
        aa = an;
        dd = dn;
    }
}

template <int KC, int MODE, int GD = CF_GATHER_DOUBLES>
__device__ __forceinline__ void gather_row(const int32_t* __restrict__ col,
                                           const double* __restrict__ val, int64_t beg,
                                           int64_t end, const int32_t* __restrict__ map,
                                           const double* __restrict__ div,
                                           const double* __restrict__ X, int c0,
                                           DV<Lay<KC>::VEC>& acc, int jlim = 0x7fffffff) {
    int jj;
    double aa, dd;
    fetch_chunk<KC, MODE>(col, val, map, div, beg, end, jj, aa, dd);
    gather_row_from<KC, MODE, GD>(col, val, beg, end, map, div, X, c0, acc, jj, aa, dd, jlim);
}

// Row pipeline: a warp visits the rows row_of(t) for t = first, first + stride,
// ... < cnt in that order, with the next row's first index chunk and the row
// after's row pointers in flight while the current row gathers, so a row costs
// one exposed memory latency instead of three (row pointer -> indices ->
// neighbour rows).  fn(t, i, beg, end, jj, aa, dd) processes row i (gathering
// via gather_row_from with the prefetched chunk).  Per-row arithmetic is
// unchanged; only the issue order of independent loads moves.
template <int KC, int MODE, class RowOf, class Fn>
__device__ __forceinline__ void row_pipeline(int64_t first, int64_t stride, int64_t cnt,
                                             RowOf row_of, const int64_t* __restrict__ rp,
                                             const int32_t* __restrict__ col,
                                             const double* __restrict__ val,
                                             const int32_t* __restrict__ map,
                                             const double* __restrict__ div, Fn fn) {
    int64_t t = first;
    if (t >= cnt) return;
    int64_t i0 = row_of(t), b0 = rp[i0], e0 = rp[i0 + 1];
    int jj0;
    double aa0, dd0;
    fetch_chunk<KC, MODE>(col, val, map, div, b0, e0, jj0, aa0, dd0);
    int64_t t1 = t + stride, i1 = 0, b1 = 0, e1 = 0;
    if (t1 < cnt) {
        i1 = row_of(t1);
        b1 = rp[i1];
        e1 = rp[i1 + 1];
    }
    while (true) {
        int jj1 = 0;
        double aa1 = 0.0, dd1 = 1.0;
        const int64_t t2 = t1 + stride;
        int64_t i2 = 0, b2 = 0, e2 = 0;
        if (t1 < cnt) {
            fetch_chunk<KC, MODE>(col, val, map, div, b1, e1, jj1, aa1, dd1);
            if (t2 < cnt) {
                i2 = row_of(t2);
                b2 = rp[i2];
                e2 = rp[i2 + 1];
            }
        }
        fn(t, i0, b0, e0, jj0, aa0, dd0);
        if (t1 >= cnt) break;
        t = t1;
        i0 = i1;
        b0 = b1;
        e0 = e1;
        jj0 = jj1;
        aa0 = aa1;
        dd0 = dd1;
        t1 = t2;
        i1 = i2;
        b1 = b2;
        e1 = e2;
    }
}

// Heavy rows (more than kHeavyNnz entries) are split into segments of at most
// kSegNnz entries; k_seg computes each segment's partial sum into P[seg][KC]
// and the row kernels add a heavy row's segment partials in segment order.
constexpr int kHeavyNnz = 64;
constexpr int kSegNnz = 64;

struct HeavyDev {
    const int32_t* hv = nullptr;   // row -> heavy index or -1
    const int64_t* hsp = nullptr;  // heavy index -> first segment (size nheavy+1)
    const double* P = nullptr;     // segment partials, [nseg][KC]
    // heavy index -> number of leading segments that hold a column below the
    // row's first-sweep bound (the start of its class range); the bounded
    // first sweep of a cycle computes and sums only those
    const int32_t* hlo = nullptr;
};

// In-kernel heavy rows for the smoother sweeps: the launch carries extra warps,
// one per segment [s_lo, s_hi); each writes its partial to SP, and the warp that
// completes a heavy row (per-row arrival counter) sums the row's partials in
// segment order and finalises the row.  The sum order is fixed; only which warp
// performs it varies.
struct SegWork {
    int64_t s_lo = 0, s_hi = 0;
    const int64_t* sbeg = nullptr;
    const int64_t* send = nullptr;
    const int32_t* seg_hv = nullptr;  // segment -> heavy index
    const int64_t* hsp = nullptr;
    const int32_t* h_row = nullptr;   // heavy index -> row
    const int32_t* h_pos = nullptr;   // heavy index -> position in the class-ordered row list
    int* cntr = nullptr;              // heavy index -> arrivals (kept zero between launches)
    double* SP = nullptr;
    const int32_t* sord = nullptr;    // launch position -> segment (nullptr: identity)
};

template <int KC>
__device__ __forceinline__ bool seg_item(const SegWork& w, int64_t s,
                                         const int32_t* __restrict__ col,
                                         const double* __restrict__ val,
                                         const double* __restrict__ X, int c0, int& hv_out,
                                         DV<Lay<KC>::VEC>& acc, int jlim = 0x7fffffff) {
    constexpr int V = Lay<KC>::VEC;
    constexpr int W = Lay<KC>::LPR;
    constexpr unsigned MASK = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
    const int lane = threadIdx.x & 31;
    zero(acc);
    gather_row<KC, G_PLAIN>(col, val, w.sbeg[s], w.send[s], nullptr, nullptr, X, c0, acc, jlim);
    stv<V>(w.SP + (size_t)s * KC + c0, acc);
    __threadfence();
    __syncwarp(MASK);
    const int hv = w.seg_hv[s];
    const int nsg = (int)(w.hsp[hv + 1] - w.hsp[hv]);
    int old = 0;
    if (lane == 0) old = atomicAdd(w.cntr + hv, 1);
    old = __shfl_sync(MASK, old, 0);
    if (old != nsg - 1) return false;
    __threadfence();
    zero(acc);
    for (int64_t sg = w.hsp[hv]; sg < w.hsp[hv + 1]; ++sg) {
        const double* q = w.SP + (size_t)sg * KC + c0;
#pragma unroll
        for (int t = 0; t < V; ++t) acc.v[t] += __ldcg(q + t);
    }
    if (lane == 0) w.cntr[hv] = 0;
    hv_out = hv;
    return true;
}

// acc += the segment partials of heavy row hv, in segment order
template <int KC>
__device__ __forceinline__ void heavy_partials(const HeavyDev& H, int hv, int c0,
                                               DV<Lay<KC>::VEC>& acc, bool lo_only = false) {
    constexpr int V = Lay<KC>::VEC;
    // a hub row has thousands of partials and one warp sums them: keep NB
    // loads in flight (same register budget as the gather loop); the adds stay
    // in segment order
    constexpr int NB0 = CF_GATHER_DOUBLES / V > 0 ? CF_GATHER_DOUBLES / V : 1;
    constexpr int NB = NB0 > 8 ? 8 : NB0;
    const int64_t s0 = H.hsp[hv], s1 = lo_only ? s0 + H.hlo[hv] : H.hsp[hv + 1];
    int64_t sgi = s0;
    for (; sgi + NB <= s1; sgi += NB) {
        DV<V> q[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) q[b] = ldv<V>(H.P + (size_t)(sgi + b) * KC + c0);
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int t = 0; t < V; ++t) acc.v[t] += q[b].v[t];
    }
    for (; sgi < s1; ++sgi) {
        DV<V> q = ldv<V>(H.P + (size_t)sgi * KC + c0);
#pragma unroll
        for (int t = 0; t < V; ++t) acc.v[t] += q.v[t];
    }
}

// Heavy rows use the partials of their segments (k_seg, summed in segment
// order); light rows gather from the prefetched first chunk.
template <int KC, int MODE>
__device__ __forceinline__ void row_sum_from(const HeavyDev& H, int64_t i,
                                             const int32_t* __restrict__ col,
                                             const double* __restrict__ val, int64_t beg,
                                             int64_t end, const int32_t* __restrict__ map,
                                             const double* __restrict__ div,
                                             const double* __restrict__ X, int c0,
                                             DV<Lay<KC>::VEC>& acc, int jj, double aa,
                                             double dd) {
    constexpr int V = Lay<KC>::VEC;
    // heavy <=> more than kHeavyNnz entries (how the plan was built), so the
    // row-to-heavy-index lookup is only paid by heavy rows
    const int hv = (H.hv && end - beg > kHeavyNnz) ? H.hv[i] : -1;
    if (hv >= 0) {
        heavy_partials<KC>(H, hv, c0, acc);
    } else {
        gather_row_from<KC, MODE>(col, val, beg, end, map, div, X, c0, acc, jj, aa, dd);
    }
}

template <int KC, int MODE>
__device__ __forceinline__ void row_sum(const HeavyDev& H, int64_t i,
                                        const int32_t* __restrict__ col,
                                        const double* __restrict__ val, int64_t beg, int64_t end,
                                        const int32_t* __restrict__ map,
                                        const double* __restrict__ div,
                                        const double* __restrict__ X, int c0,
                                        DV<Lay<KC>::VEC>& acc) {
    int jj;
    double aa, dd;
    fetch_chunk<KC, MODE>(col, val, map, div, beg, end, jj, aa, dd);
    row_sum_from<KC, MODE>(H, i, col, val, beg, end, map, div, X, c0, acc, jj, aa, dd);
}

// Row kernels process tiles of kTileRows rows per CTA; warp w of the CTA takes
// rows w, w + kWarps, ... of the tile through row_pipeline.
constexpr int kTileRows = 64;

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

// Fused deterministic reduction: after writing its part partial, a CTA counts
// its arrival in its 64-part segment; the segment's last CTA sums the segment's
// partials in part order, and the last segment finisher sums the segment sums
// in segment order into `out` (one segment: straight into `out`).  Same
// arithmetic as a separate two-stage finalize; no extra launches.
constexpr int kFinSeg = 64;
struct RedCtl {
    double* parts = nullptr;     // [q][nparts][KC]
    int64_t nparts = 0;
    double* segs = nullptr;      // [q][nseg][KC] scratch
    unsigned* seg_cnt = nullptr; // per-segment arrival counters (zero between uses)
    unsigned* glob_cnt = nullptr;
    double* out = nullptr;       // [q][KC]
};

template <int KC, int NQ>
__device__ __forceinline__ void cta_reduce_finish(DV<Lay<KC>::VEC> (&loc)[NQ], double* smem,
                                                  const RedCtl& r, int64_t part) {
    cta_reduce_store<KC, NQ>(loc, smem, r.parts, r.nparts, part);
    // arrival flags are broadcast with __syncthreads_or (no shared memory: the
    // widest reductions already use the whole default 48 KB)
    __threadfence();
    __syncthreads();
    const int64_t nseg = (r.nparts + kFinSeg - 1) / kFinSeg;
    const int64_t seg = part / kFinSeg;
    int flag = 0;
    if (threadIdx.x == 0) {
        const unsigned nin = (unsigned)min((int64_t)kFinSeg, r.nparts - seg * kFinSeg);
        flag = (atomicAdd(r.seg_cnt + seg, 1u) == nin - 1);
    }
    if (!__syncthreads_or(flag)) return;
    __threadfence();
    const int64_t p0 = seg * kFinSeg, p1 = min(r.nparts, p0 + kFinSeg);
    for (int idx = threadIdx.x; idx < NQ * KC; idx += blockDim.x) {
        const int q = idx / KC, c = idx % KC;
        double sum = 0.0;
        for (int64_t p = p0; p < p1; ++p) sum += __ldcg(r.parts + ((size_t)q * r.nparts + p) * KC + c);
        if (nseg == 1)
            r.out[q * KC + c] = sum;
        else
            r.segs[((size_t)q * nseg + seg) * KC + c] = sum;
    }
    if (threadIdx.x == 0) r.seg_cnt[seg] = 0;
    if (nseg == 1) return;
    __threadfence();
    __syncthreads();
    flag = 0;
    if (threadIdx.x == 0) flag = (atomicAdd(r.glob_cnt, 1u) == (unsigned)nseg - 1);
    if (!__syncthreads_or(flag)) return;
    __threadfence();
    for (int idx = threadIdx.x; idx < NQ * KC; idx += blockDim.x) {
        const int q = idx / KC, c = idx % KC;
        double t = 0.0;
        for (int64_t g = 0; g < nseg; ++g) t += __ldcg(r.segs + ((size_t)q * nseg + g) * KC + c);
        r.out[q * KC + c] = t;
    }
    if (threadIdx.x == 0) *r.glob_cnt = 0;
}

}  // namespace cf
