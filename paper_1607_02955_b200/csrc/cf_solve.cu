// Batched multigrid solve on the device (reference: pkg/src/cfcent/solver.py).
//
// One V-cycle (solver.py:526-560) is a fixed sequence of kernels per level:
//   aggregation level : multicolour forward GS (nu1 sweeps, first from zero)
//                       -> fused residual + restriction by aggregate
//                       -> coarse cycle -> line-search reductions
//                       -> correction x += alpha P xc -> nu2 backward sweeps
//   elimination level : exact restriction bc = b_c + W_cf D_f^-1 b_f
//                       -> coarse cycle -> exact interpolation
//   coarsest          : x = M b with M the centred grounded inverse
// The outer block iteration (solver.py:651-751) keeps per-column state on the
// device: residual norms, stagnation counters and the freeze mask.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cf_common.h"
#include "cf_hier.h"
#include "cf_kernels.cuh"
#include "cfcent_b200.h"

#ifndef CF_HOIST_OWN
// experiment knob: the row's own B / X / diagonal loads before the gather in the
// residual / restriction / line-search kernels.  Measured on C5: 1,612 vs
// 1,584 ms per step (more registers live across the gather, 128 -> 240 bytes
// of spills in k_residual<128>), so it stays off.
#define CF_HOIST_OWN 0
#endif
#ifndef CF_MANY_CTAS
#define CF_MANY_CTAS 4  // CTAs/SM of the k_seg launches of >= CF_MANY_SEG_CTAS CTAs
#endif
#ifndef CF_RED_CTAS
#define CF_RED_CTAS 3  // min CTAs/SM for the reduction / restriction gather kernels
#endif

// The kernels and the solve driver live in a variant namespace: this file is
// compiled twice, as itself (v_default: the launch bounds / rows-in-flight
// measured best on graphs whose levels fit the L2) and through
// cf_solve_hub.cu (v_hub: 4 CTAs/SM with half the rows in flight, measured
// 3.6 % faster on the L2-bound hub levels of power-law graphs and 5 % slower
// elsewhere; profiles/r02/occupancy_sweep_c5.txt).  Same arithmetic in both;
// solve_block picks by Hier::hub_profile.
#ifndef CF_VNS
#define CF_VNS v_default
#endif

namespace cf {

#ifndef CF_HUB_TU
static thread_local std::string g_last_error;
void set_error(const std::string& m) { g_last_error = m; }
#endif

// COL_KRYLOV: slowly converging column handed to V-cycle-preconditioned FCG
enum ColState { COL_ZERO = 0, COL_ACTIVE = 1, COL_CONV = 2, COL_FALLBACK = 3, COL_KRYLOV = 4 };

namespace CF_VNS {

// ============================================================================
// kernels
// ============================================================================

#define CF_LANE_SETUP(KC)                                     \
    using Lt = Lay<KC>;                                       \
    constexpr int V = Lt::VEC;                                \
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5; \
    const int slot = warp;                                    \
    const bool lane_ok = lane < Lt::LPR;                      \
    const int c0 = (lane_ok ? lane : 0) * V;                  \
    (void)slot;                                               \
    (void)c0;                                                 \
    (void)lane_ok;

// R = B - L X ; partials of sum(R), sum(R^2)  (solver.py:694-695)
template <int KC>
__global__ void __launch_bounds__(kThreads, (KC > 128 ? 2 : CF_RED_CTAS)) k_residual(int n, const int64_t* __restrict__ rp,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ diag,
                                                       const double* __restrict__ B,
                                                       const double* __restrict__ X,
                                                       double* __restrict__ R, RedCtl red,
                                                       HeavyDev H, int x_zero) {
    // x_zero: X is known to be all zeros (first check of a solve), so R = B
    // exactly (b - fma(d, 0, 0) = b) and no matrix entry or row of X is read
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    extern __shared__ double smem[];
    DV<V> loc[2];
    zero(loc[0]);
    zero(loc[1]);
    const int64_t part = blockIdx.x;
    for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
        int64_t i = part * kRowsPerPart + r;
        if (i >= n || !lane_ok) break;
        DV<V> acc, x;
        zero(acc);
        zero(x);
        double d = 0.0;
#if CF_HOIST_OWN
        // the row's own B / X / diagonal loads are issued before the gather so
        // they overlap its latency chain (indices -> neighbour rows)
        DV<V> b = ldv<V>(B + i * KC + c0);
        if (!x_zero) {
            x = ldv<V>(X + i * KC + c0);
            d = diag[i];
            row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, X, c0, acc);
        }
#else
        if (!x_zero) {
            row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, X, c0, acc);
            x = ldv<V>(X + i * KC + c0);
            d = diag[i];
        }
        DV<V> b = ldv<V>(B + i * KC + c0);
#endif
        DV<V> out;
#pragma unroll
        for (int t = 0; t < V; ++t) {
            double v = b.v[t] - fma(d, x.v[t], acc.v[t]);
            out.v[t] = v;
            loc[0].v[t] += v;
            loc[1].v[t] = fma(v, v, loc[1].v[t]);
        }
        if (R) stv<V>(R + i * KC + c0, out);
    }
    cta_reduce_finish<KC, 2>(loc, smem, red, part);
}

// Y = L X (full Laplacian product) -- fallback Krylov solvers (solver.py:571-648)
template <int KC>
__global__ void __launch_bounds__(kThreads, (KC > 128 ? 2 : CF_RED_CTAS)) k_spmm(int n, const int64_t* __restrict__ rp,
                                                   const int32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ diag,
                                                   const double* __restrict__ X,
                                                   double* __restrict__ Y, HeavyDev H) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> acc;
    zero(acc);
    row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, X, c0, acc);
    DV<V> x = ldv<V>(X + i * KC + c0);
    double d = diag[i];
#pragma unroll
    for (int t = 0; t < V; ++t) acc.v[t] = fma(d, x.v[t], acc.v[t]);
    stv<V>(Y + i * KC + c0, acc);
}

// partials of sum(b), sum|b|, sum(b^2) (balance check + norms, solver.py:672-679)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_colstats(int n, const double* __restrict__ B,
                                                       RedCtl red) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    extern __shared__ double smem[];
    DV<V> loc[3];
    zero(loc[0]);
    zero(loc[1]);
    zero(loc[2]);
    const int64_t part = blockIdx.x;
    for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
        int64_t i = part * kRowsPerPart + r;
        if (i >= n || !lane_ok) break;
        DV<V> b = ldv<V>(B + i * KC + c0);
#pragma unroll
        for (int t = 0; t < V; ++t) {
            loc[0].v[t] += b.v[t];
            loc[1].v[t] += fabs(b.v[t]);
            loc[2].v[t] = fma(b.v[t], b.v[t], loc[2].v[t]);
        }
    }
    cta_reduce_finish<KC, 3>(loc, smem, red, part);
}

// partials of sum(U1*V1), sum(U2*V2) (fallback dot products)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_dot2(int n, const double* __restrict__ U1,
                                                   const double* __restrict__ V1,
                                                   const double* __restrict__ U2,
                                                   const double* __restrict__ V2,
                                                   RedCtl red) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    extern __shared__ double smem[];
    DV<V> loc[2];
    zero(loc[0]);
    zero(loc[1]);
    const int64_t part = blockIdx.x;
    for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
        int64_t i = part * kRowsPerPart + r;
        if (i >= n || !lane_ok) break;
        DV<V> a = ldv<V>(U1 + i * KC + c0), b = ldv<V>(V1 + i * KC + c0);
        DV<V> c = ldv<V>(U2 + i * KC + c0), d = ldv<V>(V2 + i * KC + c0);
#pragma unroll
        for (int t = 0; t < V; ++t) {
            loc[0].v[t] = fma(a.v[t], b.v[t], loc[0].v[t]);
            loc[1].v[t] = fma(c.v[t], d.v[t], loc[1].v[t]);
        }
    }
    cta_reduce_finish<KC, 2>(loc, smem, red, part);
}

// partials of column sums of X (+ Y if given, formed as fl(X+Y))
template <int KC>
__global__ void __launch_bounds__(kThreads) k_colsum(int n, const double* __restrict__ X,
                                                     const double* __restrict__ Y,
                                                     RedCtl red) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    extern __shared__ double smem[];
    DV<V> loc[1];
    zero(loc[0]);
    const int64_t part = blockIdx.x;
    for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
        int64_t i = part * kRowsPerPart + r;
        if (i >= n || !lane_ok) break;
        DV<V> x = ldv<V>(X + i * KC + c0);
        if (Y) {
            DV<V> y = ldv<V>(Y + i * KC + c0);
#pragma unroll
            for (int t = 0; t < V; ++t) x.v[t] = x.v[t] + y.v[t];
        }
#pragma unroll
        for (int t = 0; t < V; ++t) loc[0].v[t] += x.v[t];
    }
    cta_reduce_finish<KC, 1>(loc, smem, red, part);
}

// Per-column outer-iteration bookkeeping (solver.py:693-715) on the device,
// plus the
// check counter, the V-cycle tallies and the while-condition of the solve
// graph.  Check c (0-based) is a regular check for c < max_cycles and the
// reference's loop-exhausted final check for c == max_cycles.
struct LoopCtl {
    const double* lp;        // stop, stagnation factor, stagnation cycles, max cycles
    int* iter;               // checks done
    long long* vcyc;         // column V-cycles executed
    int* ncyc;               // block V-cycles executed
};
template <int KC>
__global__ void k_status_loop(int n, const double* __restrict__ sums,
                              const double* __restrict__ bn, double* __restrict__ res,
                              double* __restrict__ prev, int* __restrict__ stall,
                              int* __restrict__ state, double* __restrict__ mean,
                              int* __restrict__ count, LoopCtl ctl,
                              cudaGraphConditionalHandle cond, int use_cond) {
    CF_PDL_ENTRY();
    // loop parameters live in device memory so a captured solve graph serves
    // every tolerance (they are not baked into the graph)
    const double stop = ctl.lp[0], sfac = ctl.lp[1], kfac = ctl.lp[5];
    const int scyc = (int)ctl.lp[2], max_cycles = (int)ctl.lp[3], kcheck = (int)ctl.lp[4];
    const int c = threadIdx.x;
    const int check = *ctl.iter;
    const bool final_check = check >= max_cycles;
    int a = 0;
    if (c < KC) {
        if (state[c] == COL_ACTIVE) {
            double r = sqrt(sums[KC + c]) / bn[c];
            res[c] = r;
            bool conv = r <= stop;
            if (!final_check) {
                double f = r / prev[c];
                stall[c] = f > sfac ? stall[c] + 1 : 0;
                prev[c] = r;
                if (conv)
                    state[c] = COL_CONV;
                else if (check == kcheck && f > kfac)
                    state[c] = COL_KRYLOV;
                else if (stall[c] >= scyc)
                    state[c] = COL_FALLBACK;
            } else {
                state[c] = conv ? COL_CONV : COL_FALLBACK;
            }
        }
        mean[c] = sums[c] / (double)n;
        a = (state[c] == COL_ACTIVE) ? 1 : 0;
    }
    a = __syncthreads_count(a);
    if (c == 0) {
        *count = a;
        *ctl.iter = check + 1;
        const bool go = a > 0;  // a == 0 after a final check
        if (go) {
            *ctl.vcyc += a;
            *ctl.ncyc += 1;
        }
        if (use_cond) cudaGraphSetConditional(cond, go ? 1u : 0u);
    }
}

template <int KC>
__global__ void __launch_bounds__(kThreads) k_zero_block(int64_t elems, double* __restrict__ X) {
    CF_PDL_ENTRY();
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < elems) X[t] = 0.0;
}

// R -= mean (per column)  (solver.py:567-568 _center)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_center(int n, double* __restrict__ R,
                                                     const double* __restrict__ mean) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> r = ldv_c<V>(R + i * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t) r.v[t] = r.v[t] - mean[c0 + t];
    stv<V>(R + i * KC + c0, r);
}

// X = fl(X + C) - mean for columns in state ACTIVE (solver.py:708-709)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_update(int n, double* __restrict__ X,
                                                     const double* __restrict__ C,
                                                     const double* __restrict__ csum,
                                                     const int* __restrict__ state) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> x = ldv_c<V>(X + i * KC + c0), c = ldv<V>(C + i * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t)
        if (state[c0 + t] == COL_ACTIVE) x.v[t] = (x.v[t] + c.v[t]) - csum[c0 + t] / (double)n;
    stv<V>(X + i * KC + c0, x);
}

// ---- Krylov hand-off: FCG preconditioned by one V-cycle (solver.py:571-611
// restated for the device; columns in state COL_KRYLOV).  Per iteration:
// centre r; z = V-cycle(r); zc = z - mean(z); beta = (zc.Ld)/(d.Ld) against
// the previous direction d; d = zc - beta d; Ld = L d; alpha = (r.d)/(d.Ld);
// x += alpha d; r = b - L x; status.
// (q0, q1) = (zc . AP, P . AP) with zc = C - csum / n
template <int KC>
__global__ void __launch_bounds__(kThreads) k_kry_beta(int n, const double* __restrict__ C,
                                                       const double* __restrict__ csum,
                                                       const double* __restrict__ P,
                                                       const double* __restrict__ AP,
                                                       RedCtl red) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    extern __shared__ double smem[];
    DV<V> loc[2];
    zero(loc[0]);
    zero(loc[1]);
    const int64_t part = blockIdx.x;
    for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
        int64_t i = part * kRowsPerPart + r;
        if (i >= n || !lane_ok) break;
        DV<V> z = ldv<V>(C + i * KC + c0), p = ldv<V>(P + i * KC + c0);
        DV<V> ap = ldv<V>(AP + i * KC + c0);
#pragma unroll
        for (int t = 0; t < V; ++t) {
            const double zc = z.v[t] - csum[c0 + t] / (double)n;
            loc[0].v[t] = fma(zc, ap.v[t], loc[0].v[t]);
            loc[1].v[t] = fma(p.v[t], ap.v[t], loc[1].v[t]);
        }
    }
    cta_reduce_finish<KC, 2>(loc, smem, red, part);
}
// P = zc - beta P  (beta = q0/q1 if q1 > 0, else 0)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_kry_dir(int n, const double* __restrict__ C,
                                                      const double* __restrict__ csum,
                                                      const double* __restrict__ q,
                                                      double* __restrict__ P) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> z = ldv<V>(C + i * KC + c0), p = ldv_c<V>(P + i * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t) {
        const int c = c0 + t;
        const double beta = q[KC + c] > 0.0 ? q[c] / q[KC + c] : 0.0;
        p.v[t] = (z.v[t] - csum[c] / (double)n) - beta * p.v[t];
    }
    stv<V>(P + i * KC + c0, p);
}
// X += alpha P for Krylov columns (alpha = (r.P)/(P.AP) if P.AP > 0); d = (P.AP, R.P)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_kry_step(int n, double* __restrict__ X,
                                                       const double* __restrict__ P,
                                                       const double* __restrict__ d,
                                                       const int* __restrict__ state) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> x = ldv_c<V>(X + i * KC + c0), p = ldv<V>(P + i * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t) {
        const int c = c0 + t;
        if (state[c] == COL_KRYLOV && d[c] > 0.0) x.v[t] = fma(d[KC + c] / d[c], p.v[t], x.v[t]);
    }
    stv<V>(X + i * KC + c0, x);
}
// status after an FCG iteration: residual norms of Krylov columns, stop at
// lp[0] (0.9 tau) or after lp[6] iterations (-> fallback chain); means of R
template <int KC>
__global__ void k_kry_status(int n, const double* __restrict__ sums,
                             const double* __restrict__ bn, double* __restrict__ res,
                             int* __restrict__ state, double* __restrict__ mean,
                             int* __restrict__ count, LoopCtl ctl, int* __restrict__ kiter,
                             cudaGraphConditionalHandle cond, int use_cond) {
    CF_PDL_ENTRY();
    const double stop = ctl.lp[0];
    const int kmax = (int)ctl.lp[6];
    const int c = threadIdx.x;
    const int it = *kiter + 1;
    int a = 0;
    if (c < KC) {
        if (state[c] == COL_KRYLOV) {
            const double r = sqrt(sums[KC + c]) / bn[c];
            res[c] = r;
            if (r <= stop)
                state[c] = COL_CONV;
            else if (it >= kmax)
                state[c] = COL_FALLBACK;
        }
        mean[c] = sums[c] / (double)n;
        a = (state[c] == COL_KRYLOV) ? 1 : 0;
    }
    a = __syncthreads_count(a);
    if (c == 0) {
        *count = a;
        *kiter = it;
        if (a > 0) *ctl.vcyc += a;
        if (use_cond) cudaGraphSetConditional(cond, a > 0 ? 1u : 0u);
    }
}

// Y = a*Y + b*U + d*W with per-column coefficients coef[0|1|2][KC]
template <int KC>
__global__ void __launch_bounds__(kThreads) k_lincomb(int n, double* __restrict__ Y,
                                                      const double* __restrict__ U,
                                                      const double* __restrict__ W,
                                                      const double* __restrict__ coef) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> y = ldv_c<V>(Y + i * KC + c0);
    DV<V> u, w;
    if (U) u = ldv_c<V>(U + i * KC + c0); else zero(u);
    if (W) w = ldv_c<V>(W + i * KC + c0); else zero(w);
#pragma unroll
    for (int t = 0; t < V; ++t) {
        int c = c0 + t;
        y.v[t] = fma(coef[c], y.v[t], fma(coef[KC + c], u.v[t], coef[2 * KC + c] * w.v[t]));
    }
    stv<V>(Y + i * KC + c0, y);
}

// Multicolour Gauss-Seidel sweep over one colour class:
// x_i = (b_i - sum_{j != i} L_ij x_j) / L_ii.  Rows of one colour are pairwise
// non-adjacent, so the class updates in parallel with exactly the values a
// sequential sweep in colour order would use.  from_zero: x_i = b_i / L_ii.
// Warps [0, cnt) take the class's rows (light rows only unless from_zero);
// warps [cnt, cnt + nseg) take heavy-row segments (SegWork).
// SHORT (classes of short rows): CTAs take tiles of RPB x rpw rows, each warp
// rpw rows through the row pipeline (next row's indices in flight), at 2
// CTAs/SM so the pipeline state does not spill; heavy-row segment CTAs follow
// the tiles.  Same per-row arithmetic as the warp-per-row form.
template <int KC, bool SHORT = false>
__global__ void __launch_bounds__(kThreads, SHORT ? 2 : (KC > 128 ? 2 : kGatherCtas)) k_gs(const int32_t* __restrict__ rows,
                                                              int base, int cnt,
                                                              const int64_t* __restrict__ rp,
                                                              const int32_t* __restrict__ col,
                                                              const double* __restrict__ val,
                                                              const double* __restrict__ diag,
                                                              const double* __restrict__ B,
                                                              double* __restrict__ X,
                                                              int from_zero, int jlim, int rpw,
                                                              HeavyDev H, SegWork w, int pre) {
    // pre: the heavy rows' segment partials were computed by a preceding k_seg
    // launch (H.P); otherwise the launch carries the segments itself (w)
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    if (!lane_ok) return;
    DV<V> acc;
    zero(acc);
    int64_t i;
    int64_t g;
    if constexpr (SHORT) {
        const int64_t tile = (int64_t)Lt::RPB * rpw;
        const int64_t ntile = ((int64_t)cnt + tile - 1) / tile;
        if ((int64_t)blockIdx.x < ntile) {
            const int64_t g0 = (int64_t)blockIdx.x * tile;
            const int64_t gend = min((int64_t)cnt, g0 + tile);
            auto row_of = [=](int64_t q) { return rows ? (int64_t)rows[q] : (int64_t)base + q; };
            if (from_zero) {
                for (int64_t q = g0 + slot; q < gend; q += Lt::RPB) {
                    const int64_t r = row_of(q);
                    DV<V> b = ldv<V>(B + r * KC + c0);
                    const double d = diag[r];
                    zero(acc);
#pragma unroll
                    for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
                    stv<V>(X + r * KC + c0, acc);
                }
                return;
            }
            row_pipeline<KC, G_PLAIN>(
                g0 + slot, Lt::RPB, gend, row_of, rp, col, val, nullptr, nullptr,
                [&](int64_t, int64_t r, int64_t beg, int64_t end, int jj, double aa, double dd) {
                    const bool heavy = H.hv && end - beg > kHeavyNnz;
                    if (heavy && !pre) return;  // finished by its last segment warp
                    DV<V> b = ldv<V>(B + r * KC + c0);
                    const double d = diag[r];
                    zero(acc);
                    if (heavy)
                        heavy_partials<KC>(H, H.hv[r], c0, acc, pre == 2);
                    else
                        gather_row_from<KC, G_PLAIN>(col, val, beg, end, nullptr, nullptr, X, c0,
                                                     acc, jj, aa, dd, jlim);
#pragma unroll
                    for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
                    stv<V>(X + r * KC + c0, acc);
                });
            return;
        }
        g = (int64_t)cnt + ((int64_t)blockIdx.x - ntile) * Lt::RPB + slot;
    } else {
        g = (int64_t)blockIdx.x * Lt::RPB + slot;
    }
    if (g < cnt) {
        i = rows ? (int64_t)rows[g] : base + g;
        if (!from_zero) {
            const int64_t beg = rp[i], end = rp[i + 1];
            const bool heavy = H.hv && end - beg > kHeavyNnz;
            if (heavy && !pre) return;  // finished by its last segment warp
            DV<V> b = ldv<V>(B + i * KC + c0);
            const double d = diag[i];
            if (heavy)
                heavy_partials<KC>(H, H.hv[i], c0, acc, pre == 2);
            else
                gather_row<KC, G_PLAIN>(col, val, beg, end, nullptr, nullptr, X, c0, acc, jlim);
#pragma unroll
            for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
            stv<V>(X + i * KC + c0, acc);
            return;
        }
    } else {
        int64_t sg = w.s_lo + (g - cnt);
        if (sg >= w.s_hi) return;
        if (w.sord) sg = w.sord[sg];
        int hv;
        if (!seg_item<KC>(w, sg, col, val, X, c0, hv, acc, jlim)) return;
        i = w.h_row[hv];
    }
    DV<V> b = ldv<V>(B + i * KC + c0);
    double d = diag[i];
#pragma unroll
    for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
    stv<V>(X + i * KC + c0, acc);
}

// Merged trailing colour classes, one Jacobi step: T[q] = (b_i - sum_j L_ij x_j) / L_ii
// for i = rows[q] with every x_j read before any row of the step is written
// (k_scatter_rows then writes T back).  Heavy rows as in k_gs.
template <int KC, bool SHORT = false>
__global__ void __launch_bounds__(kThreads, SHORT ? 2 : (KC > 128 ? 2 : kGatherCtas)) k_jacobi_rows(
    const int32_t* __restrict__ rows, int base, int cnt, const int64_t* __restrict__ rp,
    const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ diag, const double* __restrict__ B, const double* __restrict__ X,
    double* __restrict__ T, int jlim, int rpw, HeavyDev H, SegWork w, int pre) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    if (!lane_ok) return;
    int64_t i, q, g;
    DV<V> acc;
    zero(acc);
    if constexpr (SHORT) {
        const int64_t tile = (int64_t)Lt::RPB * rpw;
        const int64_t ntile = ((int64_t)cnt + tile - 1) / tile;
        if ((int64_t)blockIdx.x < ntile) {
            const int64_t g0 = (int64_t)blockIdx.x * tile;
            const int64_t gend = min((int64_t)cnt, g0 + tile);
            auto row_of = [=](int64_t t) { return rows ? (int64_t)rows[t] : (int64_t)base + t; };
            row_pipeline<KC, G_PLAIN>(
                g0 + slot, Lt::RPB, gend, row_of, rp, col, val, nullptr, nullptr,
                [&](int64_t qq, int64_t r, int64_t beg, int64_t end, int jj, double aa, double dd) {
                    const bool heavy = H.hv && end - beg > kHeavyNnz;
                    if (heavy && !pre) return;
                    DV<V> b = ldv<V>(B + r * KC + c0);
                    const double d = diag[r];
                    zero(acc);
                    if (heavy)
                        heavy_partials<KC>(H, H.hv[r], c0, acc, pre == 2);
                    else
                        gather_row_from<KC, G_PLAIN>(col, val, beg, end, nullptr, nullptr, X, c0,
                                                     acc, jj, aa, dd, jlim);
#pragma unroll
                    for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
                    stv<V>(T + qq * KC + c0, acc);
                });
            return;
        }
        g = (int64_t)cnt + ((int64_t)blockIdx.x - ntile) * Lt::RPB + slot;
    } else {
        g = (int64_t)blockIdx.x * Lt::RPB + slot;
    }
    if (g < cnt) {
        i = rows ? (int64_t)rows[g] : base + g;
        q = g;
        const int64_t beg = rp[i], end = rp[i + 1];
        const bool heavy = H.hv && end - beg > kHeavyNnz;
        if (heavy && !pre) return;
        DV<V> b = ldv<V>(B + i * KC + c0);
        const double d = diag[i];
        if (heavy)
            heavy_partials<KC>(H, H.hv[i], c0, acc, pre == 2);
        else
            gather_row<KC, G_PLAIN>(col, val, beg, end, nullptr, nullptr, X, c0, acc, jlim);
#pragma unroll
        for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
        stv<V>(T + q * KC + c0, acc);
        return;
    }
    int64_t sg = w.s_lo + (g - cnt);
    if (sg >= w.s_hi) return;
    if (w.sord) sg = w.sord[sg];
    int hv;
    if (!seg_item<KC>(w, sg, col, val, X, c0, hv, acc, jlim)) return;
    i = w.h_row[hv];
    q = w.h_pos[hv] - base;
    DV<V> b = ldv<V>(B + i * KC + c0);
    double d = diag[i];
#pragma unroll
    for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] - acc.v[t]) / d;
    stv<V>(T + q * KC + c0, acc);
}

template <int KC>
__global__ void __launch_bounds__(kThreads) k_scatter_rows(const int32_t* __restrict__ rows,
                                                           int base, int cnt,
                                                           const double* __restrict__ T,
                                                           double* __restrict__ X) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t g = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (g >= cnt || !lane_ok) return;
    const int64_t i = rows ? (int64_t)rows[g] : base + g;
    stv<V>(X + (size_t)i * KC + c0, ldv<V>(T + g * KC + c0));
}

// bc[a] = sum_{i in a} (b_i - L_i x)  (residual fused with P^T, solver.py:548-549)
// One warp per aggregate piece: pieces are runs of at most kAggPiece members of
// one aggregate (kAggPiece = the reference's aggregate cap, so reference-cap
// hierarchies have one piece per aggregate and a single member chain).  A
// split aggregate's pieces write partials to PP; the last-arriving piece sums
// them in piece order (fixed order, independent of scheduling).
constexpr int kAggPiece = 8;
template <int KC>
__global__ void __launch_bounds__(kThreads, (KC > 128 ? 2 : CF_RED_CTAS)) k_agg_restrict(
    int64_t np, const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
    const int32_t* __restrict__ pslot, int* __restrict__ acnt, double* __restrict__ PP,
    const int32_t* __restrict__ aptr, const int32_t* __restrict__ amem,
    const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ diag,
    const double* __restrict__ B, const double* __restrict__ X, double* __restrict__ Bc,
    HeavyDev H) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    const int64_t p = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (p >= np || !lane_ok) return;
    const int64_t a = pa ? pa[p] : p;
    const int a0 = aptr[a], a1 = aptr[a + 1];
    const int q0 = pb ? pb[p] : a0;
    const int q1 = pb ? min(a1, q0 + kAggPiece) : a1;
    DV<V> out;
    zero(out);
    for (int q = q0; q < q1; ++q) {
        int64_t i = amem[q];
        DV<V> acc;
        zero(acc);
#if CF_HOIST_OWN
        DV<V> b = ldv<V>(B + i * KC + c0), x = ldv<V>(X + i * KC + c0);
        double d = diag[i];
        row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, X, c0, acc);
#else
        row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, X, c0, acc);
        DV<V> b = ldv<V>(B + i * KC + c0), x = ldv<V>(X + i * KC + c0);
        double d = diag[i];
#endif
#pragma unroll
        for (int t = 0; t < V; ++t) out.v[t] += b.v[t] - fma(d, x.v[t], acc.v[t]);
    }
    if (q0 == a0 && q1 == a1) {
        stv<V>(Bc + a * KC + c0, out);
        return;
    }
    // split aggregate
    const int ps = pslot[p];
    constexpr unsigned MASK = Lt::LPR == 32 ? 0xffffffffu : ((1u << Lt::LPR) - 1u);
    stv<V>(PP + (size_t)ps * KC + c0, out);
    __threadfence();
    __syncwarp(MASK);
    const int npc = (a1 - a0 + kAggPiece - 1) / kAggPiece;
    int old = 0;
    if ((threadIdx.x & 31) == 0) old = atomicAdd(acnt + a, 1);
    old = __shfl_sync(MASK, old, 0);
    if (old != npc - 1) return;
    __threadfence();
    const int first = ps - (q0 - a0) / kAggPiece;
    zero(out);
    for (int k = 0; k < npc; ++k) {
        const double* q = PP + (size_t)(first + k) * KC + c0;
#pragma unroll
        for (int t = 0; t < V; ++t) out.v[t] += __ldcg(q + t);
    }
    if ((threadIdx.x & 31) == 0) acnt[a] = 0;
    stv<V>(Bc + a * KC + c0, out);
}

// Line-search partials (solver.py:550-556): den = d . L d with d = P xc over
// fine rows (CTAs [0, pf)), num = r . d = bc . xc over coarse rows (CTAs [pf, pf+pc)).
// agg == nullptr: the rows are the coarse level's own (den = xc . L_c xc with
// the Galerkin operator L_c = P^T L P, the same quantity over fewer nonzeros).
template <int KC>
__global__ void __launch_bounds__(kThreads, (KC > 128 ? 2 : CF_RED_CTAS)) k_agg_ls(
    int n, int nc, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ diag,
    const int32_t* __restrict__ agg, const double* __restrict__ Xc,
    const double* __restrict__ Bc, RedCtl rden, RedCtl rnum, HeavyDev H) {
    const int64_t pf = rden.nparts;
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    extern __shared__ double smem[];
    DV<V> loc[1];
    zero(loc[0]);
    if (blockIdx.x < pf) {
        const int64_t part = blockIdx.x;
        for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
            int64_t i = part * kRowsPerPart + r;
            if (i >= n || !lane_ok) break;
            DV<V> acc;
            zero(acc);
#if CF_HOIST_OWN
            DV<V> d = ldv<V>(Xc + (size_t)(agg ? agg[i] : i) * KC + c0);
            double dg = diag[i];
            row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, Xc, c0, acc);
#else
            row_sum<KC, G_PLAIN>(H, i, col, val, rp[i], rp[i + 1], nullptr, nullptr, Xc, c0, acc);
            DV<V> d = ldv<V>(Xc + (size_t)(agg ? agg[i] : i) * KC + c0);
            double dg = diag[i];
#endif
#pragma unroll
            for (int t = 0; t < V; ++t) {
                double ld = fma(dg, d.v[t], acc.v[t]);
                loc[0].v[t] = fma(d.v[t], ld, loc[0].v[t]);
            }
        }
        cta_reduce_finish<KC, 1>(loc, smem, rden, part);
    } else {
        const int64_t part = blockIdx.x - pf;
        for (int r = slot; r < kRowsPerPart; r += Lt::RPB) {
            int64_t a = part * kRowsPerPart + r;
            if (a >= nc || !lane_ok) break;
            DV<V> b = ldv<V>(Bc + a * KC + c0), x = ldv<V>(Xc + a * KC + c0);
#pragma unroll
            for (int t = 0; t < V; ++t) loc[0].v[t] = fma(b.v[t], x.v[t], loc[0].v[t]);
        }
        cta_reduce_finish<KC, 1>(loc, smem, rnum, part);
    }
}

// x += alpha * P xc, alpha = num/den (1 if den <= 0)  (solver.py:556-557)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_agg_correct(int n, const int32_t* __restrict__ agg,
                                                          double* __restrict__ X,
                                                          const double* __restrict__ Xc,
                                                          const double* __restrict__ ls) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> x = ldv_c<V>(X + i * KC + c0);
    DV<V> d = ldv<V>(Xc + (size_t)agg[i] * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t) {
        double den = ls[c0 + t], num = ls[KC + c0 + t];
        double alpha = den > 0.0 ? num / den : 1.0;
        x.v[t] = fma(d.v[t], alpha, x.v[t]);
    }
    stv<V>(X + i * KC + c0, x);
}

// bc_i = b[c_i] + sum_f W_cf(i,f) * (b_f / d_f)  (solver.py:534-536)
template <int KC>
__global__ void __launch_bounds__(kThreads, (KC > 128 ? 2 : CF_RED_CTAS)) k_elim_restrict(
    int nc, const int32_t* __restrict__ cn, const int64_t* __restrict__ wp,
    const int32_t* __restrict__ wc, const double* __restrict__ wv,
    const int32_t* __restrict__ fn, const double* __restrict__ fd,
    const double* __restrict__ B, double* __restrict__ Bc, HeavyDev H) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= nc || !lane_ok) return;
    DV<V> acc;
    zero(acc);
    row_sum<KC, G_DIV>(H, i, wc, wv, wp[i], wp[i + 1], nullptr, fd, B, c0, acc);
    DV<V> b = ldv<V>(B + (size_t)cn[i] * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t) acc.v[t] = b.v[t] + acc.v[t];
    stv<V>(Bc + i * KC + c0, acc);
}

// Partial sums of heavy-row segments: P[s] = sum over [sbeg[s], send[s]).
// DEEP: launches with few segments (a handful per SM) are latency-bound, so
// every warp keeps 4x the neighbour rows in flight (1 CTA/SM by registers).
// MANY: launches of tens of thousands of CTAs (the hub levels of power-law
// graphs) are bound by the L2 -> SM throughput, not by latency per warp: 4
// CTAs/SM with half the rows in flight per warp (C5 sweep, ms per estimate:
// 3 CTAs x 4 rows 1,454; 4 x 2 rows 1,399; 5 x 2 1,513; 6 x 1 1,497).  Levels
// that fit the L2 (C2, C3) prefer 3 x 4 (C2 12.14 vs 11.53 ms with 4 x 2
// everywhere), so only the large launches switch.
template <int KC, int MODE, bool DEEP = false, bool MANY = false>
__global__ void __launch_bounds__(kThreads, DEEP ? 1 : (KC > 128 ? 2 : (MANY ? CF_MANY_CTAS : kGatherCtas))) k_seg(int64_t s_lo, int64_t s_hi,
                                                  const int64_t* __restrict__ sbeg,
                                                  const int64_t* __restrict__ send,
                                                  const int32_t* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const int32_t* __restrict__ map,
                                                  const double* __restrict__ div,
                                                  const double* __restrict__ X,
                                                  double* __restrict__ P,
                                                  const int32_t* __restrict__ sord, int jlim) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t sg = s_lo + (int64_t)blockIdx.x * Lt::RPB + slot;
    if (sg >= s_hi || !lane_ok) return;
    if (sord) sg = sord[sg];
    DV<V> acc;
    zero(acc);
    gather_row<KC, MODE, DEEP ? 4 * CF_GATHER_DOUBLES
                               : (MANY && KC <= 128) ? CF_GATHER_DOUBLES / 2 : CF_GATHER_DOUBLES>(
        col, val, sbeg[sg], send[sg], map, div, X, c0, acc, jlim);
    stv<V>(P + (size_t)sg * KC + c0, acc);
}

// x[c_i] = xc_i ; x[f] = (b_f + sum W_fc xc) / d_f   (solver.py:538-541)
template <int KC>
__global__ void __launch_bounds__(kThreads, 2) k_elim_interp(
    int nf, int nc, const int32_t* __restrict__ cn, const int32_t* __restrict__ fn,
    const int64_t* __restrict__ wp, const int32_t* __restrict__ wc,
    const double* __restrict__ wv, const double* __restrict__ fd,
    const double* __restrict__ B, const double* __restrict__ Xc, double* __restrict__ X,
    int rpw) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    if (!lane_ok) return;
    const int64_t tile = (int64_t)Lt::RPB * rpw;
    const int64_t ctile = ((int64_t)nc + tile - 1) / tile;
    if ((int64_t)blockIdx.x < ctile) {
        const int64_t g0 = (int64_t)blockIdx.x * tile;
        const int64_t gend = min((int64_t)nc, g0 + tile);
        for (int64_t g = g0 + slot; g < gend; g += Lt::RPB)
            stv<V>(X + (size_t)cn[g] * KC + c0, ldv<V>(Xc + g * KC + c0));
        return;
    }
    const int64_t r0 = ((int64_t)blockIdx.x - ctile) * tile;
    row_pipeline<KC, G_PLAIN>(
        r0 + slot, Lt::RPB, min((int64_t)nf, r0 + tile), [](int64_t t) { return t; }, wp, wc,
        wv, nullptr, nullptr,
        [&](int64_t g, int64_t, int64_t beg, int64_t end, int jj, double aa, double dd) {
            DV<V> acc;
            zero(acc);
            gather_row_from<KC, G_PLAIN>(wc, wv, beg, end, nullptr, nullptr, Xc, c0, acc, jj, aa,
                                         dd);
            const int64_t i = fn[g];
            DV<V> b = ldv<V>(B + i * KC + c0);
            const double d = fd[g];
#pragma unroll
            for (int t = 0; t < V; ++t) acc.v[t] = (b.v[t] + acc.v[t]) / d;
            stv<V>(X + i * KC + c0, acc);
        });
}

// coarsest: x = M b, M dense n x n (solver.py:406-419 restated as one operator).
// The l range is cut into dense_splits(n) fixed chunks; every output is, per
// chunk, one fma chain over l ascending, and the chunk partials are summed in
// chunk order (k_dense_reduce) -- the same order for every block width.
// split count fills one wave of 148 SMs with the 128-row tiles (1 CTA/SM by
// registers); a function of n only, so every block width sums in one order
static inline int dense_splits(int n) {
    const int row_tiles = (n + 127) / 128;
    return n <= 256 ? 1 : std::max(1, std::min(16, 148 / row_tiles));
}
static inline int dense_chunk(int n, int S) { return (((n + S - 1) / S) + 15) / 16 * 16; }

// small widths: one thread per (row, column) output, per chunk
template <int KC>
__global__ void __launch_bounds__(kThreads) k_dense_small(int n, int chunk,
                                                          const double* __restrict__ M,
                                                          const double* __restrict__ B,
                                                          double* __restrict__ P) {
    CF_PDL_ENTRY();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (t >= (int64_t)n * KC) return;
    const int64_t i = t / KC;
    const int c = (int)(t % KC);
    const int l0 = s * chunk, l1 = min(n, l0 + chunk);
    double acc = 0.0;
    for (int l = l0; l < l1; ++l) acc = fma(__ldg(M + i * n + l), __ldg(B + (size_t)l * KC + c), acc);
    P[((size_t)s * n + i) * KC + c] = acc;
}

// wide blocks: 128 x TC output tile per CTA (TC = min(KC,128)), 16-deep l
// stages in shared memory, 8 x (TC/16) register tile per thread; the next
// stage's tiles are prefetched into registers while the current one is
// multiplied (global-load latency overlapped with the fp64 FMAs).
// Column-tile width (experiment knob; every output keeps its fma chain, so
// results do not depend on it).  64 (8 x 4 thread tile, 128 registers, 2
// CTAs/SM) was measured against 128 (8 x 8, 246 registers, 1 CTA/SM): C2
// 12.24 vs 12.07 ms per step, dense share 7.0 vs 6.0 % (profiles/r01/
// dense_tile_ab.txt), so the wider tile stays.
#ifndef CF_DENSE_TC
#define CF_DENSE_TC 128
#endif
constexpr int kGR = 128, kGL = 16, kDenseTC = CF_DENSE_TC;
template <int KC>
constexpr int dense_tc() {
    // column tile: the widest of kDenseTC / 64 / 32 that divides the block
    // (160 -> 32, 192 -> 64); the sum order per output does not depend on it
    return KC < kDenseTC ? KC : KC % kDenseTC == 0 ? kDenseTC : KC % 64 == 0 ? 64 : 32;
}
template <int KC>
__global__ void __launch_bounds__(kThreads) k_dense_tile(int n, int chunk,
                                                         const double* __restrict__ M,
                                                         const double* __restrict__ B,
                                                         double* __restrict__ P) {
    CF_PDL_ENTRY();
    constexpr int TC = dense_tc<KC>();
    constexpr int CT = TC / 16;
    constexpr int NA = kGR * kGL / kThreads;  // A elements per thread per stage
    constexpr int NB = kGL * TC / kThreads;   // B elements per thread per stage
    __shared__ __align__(16) double sA[kGL][kGR + 2];
    __shared__ __align__(16) double sB[kGL][TC];
    // thread (tx, ty) owns rows ty*8 .. ty*8+7 and, for even CT, the column
    // pairs 2tx + 32q, 2tx + 32q + 1 (q < CT/2) so both fragments load as
    // 128-bit shared-memory reads; odd CT keeps columns tx + 16c
    constexpr bool PAIR = CT % 2 == 0;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    auto colof = [&](int c) { return PAIR ? 2 * tx + 32 * (c >> 1) + (c & 1) : tx + 16 * c; };
    const int i0 = blockIdx.x * kGR, j0 = blockIdx.y * TC, s = blockIdx.z;
    const int l0 = s * chunk, l1 = min(n, l0 + chunk);
    double acc[8][CT];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < CT; ++c) acc[r][c] = 0.0;
    double ra[NA], rb[NB > 0 ? NB : 1];
    auto fetch = [&](int lb) {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int e = tid + q * kThreads, r = e / kGL, t = e % kGL;
            const int i = i0 + r, l = lb + t;
            ra[q] = (i < n && l < l1) ? __ldg(M + (size_t)i * n + l) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int e = tid + q * kThreads, t = e / TC, c = e % TC;
            const int l = lb + t;
            rb[q] = (l < l1) ? __ldg(B + (size_t)l * KC + j0 + c) : 0.0;
        }
    };
    if (l0 < l1) fetch(l0);
    for (int lb = l0; lb < l1; lb += kGL) {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int e = tid + q * kThreads;
            sA[e % kGL][e / kGL] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int e = tid + q * kThreads;
            sB[e / TC][e % TC] = rb[q];
        }
        __syncthreads();
        if (lb + kGL < l1) fetch(lb + kGL);
        const int tmax = min(kGL, l1 - lb);
        for (int t = 0; t < tmax; ++t) {
            double a[8], bb[CT];
#pragma unroll
            for (int r = 0; r < 8; r += 2) {
                const double2 v = *reinterpret_cast<const double2*>(&sA[t][ty * 8 + r]);
                a[r] = v.x;
                a[r + 1] = v.y;
            }
            if constexpr (PAIR) {
#pragma unroll
                for (int c = 0; c < CT; c += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(&sB[t][colof(c)]);
                    bb[c] = v.x;
                    bb[c + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int c = 0; c < CT; ++c) bb[c] = sB[t][colof(c)];
            }
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < CT; ++c) acc[r][c] = fma(a[r], bb[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int i = i0 + ty * 8 + r;
        if (i < n)
#pragma unroll
            for (int c = 0; c < CT; ++c) P[((size_t)s * n + i) * KC + j0 + colof(c)] = acc[r][c];
    }
}

// X = sum over chunks of P[s] in chunk order
template <int KC>
__global__ void __launch_bounds__(kThreads) k_dense_reduce(int n, int S,
                                                           const double* __restrict__ P,
                                                           double* __restrict__ X) {
    CF_PDL_ENTRY();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * KC) return;
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += P[(size_t)s * n * KC + t];
    X[t] = acc;
}

// rows layout (cnt x n) -> block (n x KC), zero padding for columns >= cnt
// device row i holds node perm[i] (perm == nullptr: identity)
template <int KC>
__global__ void k_rows_to_block(const double* __restrict__ S, int cnt, int n,
                                const int32_t* __restrict__ perm, double* __restrict__ B) {
    CF_PDL_ENTRY();
    __shared__ double tile[32][33];
    int i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int c = c0 + r, i = i0 + tx;
        int src = (i < n) ? (perm ? perm[i] : i) : 0;
        tile[r][tx] = (c < cnt && i < n) ? S[(size_t)c * n + src] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int i = i0 + r, c = c0 + tx;
        if (i < n && c < KC) B[(size_t)i * KC + c] = tile[tx][r];
    }
}

template <int KC>
__global__ void k_block_to_rows(const double* __restrict__ B, int cnt, int n,
                                const int32_t* __restrict__ perm, double* __restrict__ S) {
    CF_PDL_ENTRY();
    __shared__ double tile[32][33];
    int i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        int i = i0 + r, c = c0 + tx;
        tile[r][tx] = (i < n && c < KC) ? B[(size_t)i * KC + c] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int c = c0 + r, i = i0 + tx;
        if (c < cnt && i < n) S[(size_t)c * n + (perm ? perm[i] : i)] = tile[tx][r];
    }
}

// dst[i, :k] = src[perm[i], :k] (gather, to_dev) or dst[perm[i], :k] = src[i, :k]
// (scatter); src / dst row strides ks / kd.
__global__ void k_permute_rows(const double* __restrict__ src, int ks, double* __restrict__ dst,
                               int kd, int k, int n, const int32_t* __restrict__ perm,
                               int gather) {
    CF_PDL_ENTRY();
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * k) return;
    int64_t i = t / k;
    int c = (int)(t % k);
    int64_t p = perm ? perm[i] : i;
    if (gather)
        dst[i * kd + c] = src[p * ks + c];
    else
        dst[p * kd + c] = src[i * ks + c];
}

// ============================================================================
// host-side launch helpers
// ============================================================================

static inline int64_t nparts_of(int64_t n) { return (n + kRowsPerPart - 1) / kRowsPerPart; }
template <int KC>
static inline unsigned grid_rows(int64_t rows, int64_t at_least = 1) {
    return (unsigned)std::max<int64_t>(at_least, (rows + Lay<KC>::RPB - 1) / Lay<KC>::RPB);
}
#ifndef CF_DEEP_SEG_CTAS
#define CF_DEEP_SEG_CTAS 296
#endif
constexpr unsigned kDeepSegCtas = CF_DEEP_SEG_CTAS;  // <= 2 CTAs per SM: deep k_seg
#ifndef CF_MANY_SEG_CTAS
#define CF_MANY_SEG_CTAS 16384
#endif
constexpr unsigned kManySegCtas = CF_MANY_SEG_CTAS;  // L2-bound launches: 4 CTAs/SM k_seg
static inline unsigned grid_tiles(int64_t rows, int64_t at_least = 1, int rpw = kTileRows / kWarps) {
    const int64_t t = (int64_t)kWarps * rpw;
    return (unsigned)std::max<int64_t>(at_least, (rows + t - 1) / t);
}
// Rows per warp of the tiled row kernels: the row pipeline pays off with
// several rows per warp, but a launch must still fill the GPU several waves
// deep (148 SMs x 3 CTAs x kWaves), or small levels lose parallelism.
#ifndef CF_RPW_MAX
#define CF_RPW_MAX 8
#endif
// Short-row classes (mean off-degree <= CF_SHORT_DEG) with enough rows for
// several per warp use the tiled sweep kernels at 2 CTAs/SM; 0 = warp per row.
#ifndef CF_SHORT_DEG
#define CF_SHORT_DEG 12
#endif
static inline int short_rpw(int64_t rows, int64_t nnz) {
    static const int deg = [] {
        const char* e = std::getenv("CF_SHORT_DEG");
        return e ? std::atoi(e) : CF_SHORT_DEG;
    }();
    if (rows <= 0 || nnz > (int64_t)deg * rows) return 1;
    // 4 rows per warp and still >= 4 waves of 2-CTA slots, else warp per row
    // (measured: 2 rows per warp on C2's 20-30k-row classes is slower)
    constexpr int64_t kSlots = 148 * 2 * kWarps, kWaves = 4;
    return rows >= kSlots * kWaves * 4 ? 4 : 1;
}
static inline int pick_rpw(int64_t rows) {
    constexpr int64_t kSlots = 148 * 3 * kWarps, kWaves = 4;
    int r = CF_RPW_MAX;
    while (r > 1 && rows < kSlots * kWaves * r) r >>= 1;
    return r;
}
template <int KC, int NQ>
static inline size_t red_smem() {
    return sizeof(double) * NQ * Lay<KC>::RPB * KC;
}

// fused-reduction control for a reduction of np parts into out; region 0/1
// selects independent counter and scratch areas (two reductions per kernel)
static RedCtl redctl(Hier& h, double* parts, int64_t np, double* out, int region) {
    RedCtl r;
    r.parts = parts;
    r.nparts = np;
    r.out = out;
    r.segs = h.fin + (size_t)region * h.fin_region;
    r.seg_cnt = h.cnt + (size_t)region * h.cnt_region;
    r.glob_cnt = h.cnt + 2 * (size_t)h.cnt_region + region;
    return r;
}

template <int KC>
struct Ops {
    static double A(int64_t rows, int64_t nnz) { return 12.0 * nnz + 16.0 * rows; }
    static double Vb(int64_t rows) { return 8.0 * KC * rows; }
    static HeavyDev hd(const Hier& h, const Plan& pl) {
        HeavyDev d;
        if (pl.nheavy) {
            d.hv = pl.hv;
            d.hsp = pl.hsp;
            d.P = h.SP;
            d.hlo = pl.hlo;
        }
        return d;
    }
    static SegWork segwork(const Hier& h, const Plan& pl, int64_t lo, int64_t hi) {
        SegWork w;
        if (!pl.nheavy || hi <= lo) return w;
        w.sord = pl.sord_cls;
        w.s_lo = lo;
        w.s_hi = hi;
        w.sbeg = pl.sbeg;
        w.send = pl.send;
        w.seg_hv = pl.seg_hv;
        w.hsp = pl.hsp;
        w.h_row = pl.h_row;
        w.h_pos = pl.h_pos;
        w.cntr = pl.cntr;
        w.SP = h.SP;
        return w;
    }
    // segment partials of a plan's segments [lo, hi)
    // sweep = true: [lo, hi) is a sweep launch range (a Gauss-Seidel class or
    // the merged Jacobi classes; window order sord_cls), hnnz its entry count
    // (-1: the whole plan, window order sord_all)
    template <int MODE>
    static void seg(Hier& h, const Plan& pl, int64_t lo, int64_t hi, const int32_t* col,
                    const double* val, const int32_t* map, const double* div, const double* X,
                    int level, bool sweep = false, double hnnz = -1.0, int jlim = 0x7fffffff,
                    int64_t nbr = -1, int lo_range = -1) {
        if (lo_range >= 0) {
            // bounded first sweep: only the segments that hold a column below the
            // bound (listed per launch range in sord_lo)
            const int64_t a = pl.cseg_lo[(size_t)lo_range], b = pl.cseg_lo[(size_t)lo_range + 1];
            if (b <= a) return;
            ProfScope ps(h, "heavy_seg", level, 12.0 * hnnz + Vb(b - a) * 2, Vb(hnnz));
            const unsigned grid = (unsigned)((b - a + Lay<KC>::RPB - 1) / Lay<KC>::RPB);
            if (grid <= kDeepSegCtas)
                launch_k(k_seg<KC, MODE, true>, dim3(grid), dim3(kThreads), 0, h.s, a, b, pl.sbeg,
                         pl.send, col, val, map, div, X, h.SP, (const int32_t*)pl.sord_lo, jlim);
            else if (grid >= kManySegCtas)
                launch_k(k_seg<KC, MODE, false, true>, dim3(grid), dim3(kThreads), 0, h.s, a, b,
                         pl.sbeg, pl.send, col, val, map, div, X, h.SP,
                         (const int32_t*)pl.sord_lo, jlim);
            else
                launch_k(k_seg<KC, MODE, false>, dim3(grid), dim3(kThreads), 0, h.s, a, b, pl.sbeg,
                         pl.send, col, val, map, div, X, h.SP, (const int32_t*)pl.sord_lo, jlim);
            return;
        }
        if (hi <= lo) return;
        if (hnnz < 0)
            hnnz = (lo == 0 && hi == pl.nseg) ? (double)pl.heavy_nnz : (double)kSegNnz * (hi - lo);
        // compulsory bytes: matrix entries, one partial written (and read back by
        // the row kernel) per segment, every distinct neighbour row of X once
        if (nbr < 0) nbr = (lo == 0 && hi == pl.nseg && map == nullptr) ? pl.all_nbr : 0;
        ProfScope ps(h, "heavy_seg", level, 12.0 * hnnz + Vb(hi - lo) * 2 + Vb(nbr), Vb(hnnz));
        const unsigned grid = (unsigned)((hi - lo + Lay<KC>::RPB - 1) / Lay<KC>::RPB);
        const int32_t* ord = sweep ? pl.sord_cls
                                   : (lo == 0 && hi == pl.nseg) ? pl.sord_all : nullptr;
        if (grid <= kDeepSegCtas)
            launch_k(k_seg<KC, MODE, true>, dim3(grid), dim3(kThreads), 0, h.s, lo, hi, pl.sbeg,
                     pl.send, col, val, map, div, X, h.SP, ord, jlim);
        else if (grid >= kManySegCtas)
            launch_k(k_seg<KC, MODE, false, true>, dim3(grid), dim3(kThreads), 0, h.s, lo, hi,
                     pl.sbeg, pl.send, col, val, map, div, X, h.SP, ord, jlim);
        else
            launch_k(k_seg<KC, MODE, false>, dim3(grid), dim3(kThreads), 0, h.s, lo, hi, pl.sbeg,
                     pl.send, col, val, map, div, X, h.SP, ord, jlim);
    }
    // Sweeps over a launch range with at least this many heavy-row segments
    // compute the partials in a k_seg launch of their own (no fence / arrival
    // counter per segment: the same L1 matrix gathers at 10.9 TB/s in k_seg and
    // 6.3 TB/s inside the sweep kernel, profiles/r02); smaller ranges keep the
    // segments inside the sweep launch (one launch less on small levels).
    // Either way a heavy row is the sum of its partials in segment order.
    static int64_t pre_seg_min() {
        static const int64_t v = [] {
            const char* e = std::getenv("CF_PRE_SEG_MIN");
            return e ? (int64_t)std::atoll(e) : (int64_t)8192;
        }();
        return v;
    }
    static void residual(Hier& h, const double* B, const double* X, double* R, double* sums2,
                         bool x_zero = false) {
        DLevel& l = h.L[0];
        int64_t np = nparts_of(l.n);
        if (x_zero) {
            ProfScope ps(h, "residual0", 0, Vb(l.n) * (R ? 2 : 1));
            launch_k(k_residual<KC>, dim3((unsigned)np), dim3(kThreads), red_smem<KC, 2>(), h.s,
                     l.n, l.rp, l.col, l.val, l.diag, B, X, R, redctl(h, h.parts, np, sums2, 0),
                     HeavyDev{}, 1);
            return;
        }
        seg<G_PLAIN>(h, l.pm, 0, l.pm.nseg, l.col, l.val, nullptr, nullptr, X, 0);
        const int64_t light = l.nnz - l.pm.heavy_nnz;  // heavy rows: the k_seg launch above
        ProfScope ps(h, "residual", 0, A(l.n, light) + Vb(l.n) * (R ? 3 : 2), Vb(light));
        launch_k(k_residual<KC>, dim3((unsigned)np), dim3(kThreads), red_smem<KC, 2>(), h.s, l.n,
                 l.rp, l.col, l.val, l.diag, B, X, R, redctl(h, h.parts, np, sums2, 0),
                 hd(h, l.pm), 0);
    }
    static void colsum(Hier& h, const double* X, const double* Y, double* out) {
        int n = h.n0;
        int64_t np = nparts_of(n);
        ProfScope ps(h, "colsum", 0, Vb(n) * (Y ? 2 : 1));
        launch_k(k_colsum<KC>, dim3((unsigned)np), dim3(kThreads), red_smem<KC, 1>(), h.s, n, X, Y,
                 redctl(h, h.parts, np, out, 0));
    }
    static void dot2(Hier& h, const double* a, const double* b, const double* c, const double* d,
                     double* out) {
        int n = h.n0;
        int64_t np = nparts_of(n);
        ProfScope ps(h, "fallback", 0, 0.0);
        launch_k(k_dot2<KC>, dim3((unsigned)np), dim3(kThreads), red_smem<KC, 2>(), h.s, n, a, b,
                 c, d, redctl(h, h.parts, np, out, 0));
    }
    static void spmm(Hier& h, const double* X, double* Y) {
        DLevel& l = h.L[0];
        seg<G_PLAIN>(h, l.pm, 0, l.pm.nseg, l.col, l.val, nullptr, nullptr, X, 0);
        ProfScope ps(h, "fallback", 0, 0.0);
        launch_k(k_spmm<KC>, dim3(grid_rows<KC>(l.n)), dim3(kThreads), 0, h.s, l.n, l.rp, l.col, l.val, l.diag, X,
                                                             Y, hd(h, l.pm));
    }
    static void center(Hier& h, double* X, const double* mean) {
        ProfScope ps(h, "center", 0, 2 * Vb(h.n0));
        launch_k(k_center<KC>, dim3(grid_rows<KC>(h.n0)), dim3(kThreads), 0, h.s, h.n0, X, mean);
    }
    static void lincomb(Hier& h, double* Y, const double* U, const double* W, const double* coef) {
        ProfScope ps(h, "fallback", 0, 0.0);
        launch_k(k_lincomb<KC>, dim3(grid_rows<KC>(h.n0)), dim3(kThreads), 0, h.s, h.n0, Y, U, W, coef);
    }

    static void zero_block(Hier& h, double* x, int64_t elems) {
        launch_k(k_zero_block<KC>, dim3((unsigned)((elems + kThreads - 1) / kThreads)), dim3(kThreads), 0, h.s, elems,
                                                                                          x);
    }
    static bool coarse_ls() {
        static const bool on = [] {
            const char* e = std::getenv("CF_COARSE_LS");
            return !e || std::atoi(e) != 0;
        }();
        return on;
    }
    static double* bufb(Hier& h, int j) { return j == 0 ? h.R : h.L[j].b; }
    static double* bufx(Hier& h, int j) { return j == 0 ? h.C : h.L[j].x; }

    // One V-cycle from zero on level j: x_j = cycle(b_j)  (solver.py:526-560)
    static void cycle(Hier& h, int j, int nu1, int nu2) {
        DLevel& l = h.L[j];
        double* b = bufb(h, j);
        double* x = bufx(h, j);
        if (l.kind == CF_LEVEL_COARSEST) {
            if (l.n == 1 || !l.M) {
                ProfScope ps(h, "memset", j, Vb(l.n));
                zero_block(h, x, (int64_t)l.n * KC);
            } else {
                ProfScope ps(h, "dense", j, 8.0 * l.n * l.n + 2 * Vb(l.n));
                const int S = dense_splits(l.n), chunk = dense_chunk(l.n, S);
                if constexpr (KC >= 16) {
                    dim3 grd((unsigned)((l.n + kGR - 1) / kGR), KC / dense_tc<KC>(), S);
                    launch_k(k_dense_tile<KC>, dim3(grd), dim3(kThreads), 0, h.s, l.n, chunk, l.M, b, h.DP);
                } else {
                    dim3 grd((unsigned)(((int64_t)l.n * KC + kThreads - 1) / kThreads), S);
                    launch_k(k_dense_small<KC>, dim3(grd), dim3(kThreads), 0, h.s, l.n, chunk, l.M, b, h.DP);
                }
                launch_k(k_dense_reduce<KC>, dim3((unsigned)(((int64_t)l.n * KC + kThreads - 1) / kThreads)), dim3(kThreads), 0, h.s, l.n, S, h.DP, x);
            }
            return;
        }
        DLevel& c = h.L[j + 1];
        double* bc = bufb(h, j + 1);
        double* xc = bufx(h, j + 1);
        if (l.kind == CF_LEVEL_ELIMINATION) {
            {
                seg<G_DIV>(h, l.pw, 0, l.pw.nseg, l.wcm, l.wcv, nullptr, l.wcd, b, j);
                ProfScope ps(h, "elim_restrict", j,
                             12.0 * (l.w_nnz - l.pw.heavy_nnz) + 12.0 * l.nc + 12.0 * l.nf +
                                 Vb(2 * l.nc + l.nf));
                launch_k(k_elim_restrict<KC>, dim3(grid_rows<KC>(l.nc)), dim3(kThreads), 0, h.s,
                         l.nc, l.cn, l.wcp, l.wcm, l.wcv, nullptr, l.wcd, b, bc, hd(h, l.pw));
            }
            cycle(h, j + 1, nu1, nu2);
            ProfScope ps(h, "elim_interp", j,
                         12.0 * l.w_nnz + 24.0 * l.nf + 4.0 * l.nc + Vb(2 * l.nc + 2 * l.nf));
            const int rpw = pick_rpw(l.nf);
            launch_k(k_elim_interp<KC>,
                     dim3(std::max(1u, grid_tiles(l.nc, 0, rpw) + grid_tiles(l.nf, 0, rpw))),
                     dim3(kThreads), 0, h.s, l.nf, l.nc, l.cn, l.fn, l.wfp, l.wfc, l.wfv, l.fd, b,
                     xc, x, rpw);
            return;
        }
        // aggregation level.  The cycle starts from x = 0.  With contiguous
        // colour classes the first pre-smoothing sweep reads only rows of
        // classes it has already updated (j < first row of the class; the rest
        // are zero), so it needs no zeroed x and writes every row.
        const bool bounded = l.contig && nu1 > 0;
        if (!bounded) {
            ProfScope ps(h, "memset", j, Vb(l.n));
            zero_block(h, x, (int64_t)l.n * KC);
        }
        for (int s = 0; s < nu1; ++s) {
            const bool first = s == 0 && bounded;
            for (int col = 0; col < l.gs_classes; ++col)
                sweep(h, l, col, b, x, s == 0 && col == 0, first);
            if (l.merged) jacobi(h, l, b, x, first);
        }
        {
            seg<G_PLAIN>(h, l.pm, 0, l.pm.nseg, l.col, l.val, nullptr, nullptr, x, j);
            const int64_t light = l.nnz - l.pm.heavy_nnz;
            ProfScope ps(h, "agg_restrict", j,
                         A(l.n, light) + 4.0 * l.n + 4.0 * l.nc + Vb(2 * l.n + l.nc), Vb(light));
            launch_k(k_agg_restrict<KC>, dim3(grid_rows<KC>(l.npieces)), dim3(kThreads), 0, h.s,
                     (int64_t)l.npieces, l.pa, l.pb, l.pslot, l.acnt, h.PP, l.aptr, l.amem,
                     l.rp, l.col, l.val, l.diag, b, x, bc, hd(h, l.pm));
        }
        cycle(h, j + 1, nu1, nu2);
        int64_t pf = nparts_of(l.n), pc = nparts_of(l.nc);
        if (coarse_ls() && c.kind == CF_LEVEL_AGGREGATION && c.rp) {
            // d . L d = xc . (P^T L P) xc: the coarse level's Galerkin operator
            // gives the same denominator from nnz(L_c) instead of nnz(L) gathers
            pf = nparts_of(c.n);
            seg<G_PLAIN>(h, c.pm, 0, c.pm.nseg, c.col, c.val, nullptr, nullptr, xc, j + 1);
            const int64_t light = c.nnz - c.pm.heavy_nnz;
            ProfScope ps(h, "agg_linesearch", j, A(c.n, light) + Vb(2 * l.nc), Vb(light));
            launch_k(k_agg_ls<KC>, dim3((unsigned)(pf + pc)), dim3(kThreads), red_smem<KC, 1>(),
                     h.s, c.n, l.nc, c.rp, c.col, c.val, c.diag, (const int32_t*)nullptr, xc, bc,
                     redctl(h, h.parts, pf, l.ls, 0), redctl(h, h.parts + pf * KC, pc, l.ls + KC, 1),
                     hd(h, c.pm));
        } else {
            seg<G_PLAIN>(h, l.pm, 0, l.pm.nseg, l.cagg, l.val, nullptr, nullptr, xc, j);
            const int64_t light = l.nnz - l.pm.heavy_nnz;
            ProfScope ps(h, "agg_linesearch", j, A(l.n, light) + 4.0 * l.n + Vb(2 * l.nc),
                         Vb(light));
            launch_k(k_agg_ls<KC>, dim3((unsigned)(pf + pc)), dim3(kThreads), red_smem<KC, 1>(),
                     h.s, l.n, l.nc, l.rp, l.cagg, l.val, l.diag, l.agg, xc, bc,
                     redctl(h, h.parts, pf, l.ls, 0), redctl(h, h.parts + pf * KC, pc, l.ls + KC, 1),
                     hd(h, l.pm));
        }
        {
            ProfScope ps(h, "agg_correct", j, 4.0 * l.n + Vb(2 * l.n + l.nc));
            launch_k(k_agg_correct<KC>, dim3(grid_rows<KC>(l.n)), dim3(kThreads), 0, h.s, l.n, l.agg, x, xc, l.ls);
        }
        for (int s = 0; s < nu2; ++s) {
            if (l.merged) jacobi(h, l, b, x, false);
            for (int col = l.gs_classes - 1; col >= 0; --col) sweep(h, l, col, b, x, false, false);
        }
        (void)c;
    }
    // first: first sweep of a cycle from zero (bounded reads, see cycle())
    static void sweep(Hier& h, DLevel& l, int colr, const double* b, double* x, bool from_zero,
                      bool first) {
        int beg = l.cptr[colr], cnt = l.cptr[colr + 1] - beg;
        if (cnt <= 0) return;
        const int lev = (int)(&l - &h.L[0]);
        const int64_t s_lo = from_zero ? 0 : l.pm.cseg[colr], s_hi = from_zero ? 0 : l.pm.cseg[colr + 1];
        const int jlim = first ? beg : 0x7fffffff;
        int pre = (l.pm.nheavy && s_hi - s_lo >= pre_seg_min()) ? 1 : 0;
        if (pre && first && l.pm.hlo) {
            pre = 2;  // bounded: only the segments with a column below the bound
            seg<G_PLAIN>(h, l.pm, s_lo, s_hi, l.col, l.val, nullptr, nullptr, x, lev, true,
                         (double)std::min(l.pm.cheavy[colr], l.c_nnz_lo[colr]), jlim, 0, colr);
        } else if (pre)
            seg<G_PLAIN>(h, l.pm, s_lo, s_hi, l.col, l.val, nullptr, nullptr, x, lev, true,
                         (double)l.pm.cheavy[colr], jlim, first ? 0 : l.pm.cnbr[colr]);
        SegWork w = pre ? SegWork{} : segwork(h, l.pm, s_lo, s_hi);
        const int64_t hvy = pre ? l.pm.cheavy[colr] : 0;  // entries gathered by the k_seg launch
        const int64_t gnnz = from_zero ? 0 : first ? l.c_nnz_lo[colr] : l.c_nnz[colr] - hvy;
        // with the segments in their own launch the sweep kernel gathers for its
        // light rows only (the k_seg scope counts the heavy rows' neighbour rows)
        const int64_t gnbr = from_zero ? 0 : first ? l.c_nbr_lo[colr]
                                           : pre ? l.c_nbr_light[colr] : l.c_nbr[colr];
        ProfScope ps(h, "gs_sweep", lev,
                     12.0 * (l.c_nnz[colr] - hvy) + 20.0 * cnt + Vb(2 * cnt + gnbr), Vb(gnnz));
        const int rpw = short_rpw(cnt, l.c_nnz[colr]);
        if (rpw > 1)
            launch_k(k_gs<KC, true>,
                     dim3(grid_tiles(cnt, 1, rpw) + grid_rows<KC>(w.s_hi - w.s_lo, 0)),
                     dim3(kThreads), 0, h.s, l.contig ? nullptr : l.crows + beg, beg, cnt, l.rp,
                     l.col, l.val, l.diag, b, x, from_zero ? 1 : 0, jlim, rpw, hd(h, l.pm), w, pre);
        else
            launch_k(k_gs<KC, false>, dim3(grid_rows<KC>(cnt + (w.s_hi - w.s_lo))),
                     dim3(kThreads), 0, h.s, l.contig ? nullptr : l.crows + beg, beg, cnt, l.rp,
                     l.col, l.val, l.diag, b, x, from_zero ? 1 : 0, jlim, 1, hd(h, l.pm), w, pre);
    }

    static void jacobi(Hier& h, DLevel& l, const double* b, double* x, bool first) {
        const int K = l.gs_classes;
        int beg = l.cptr[K], cnt = l.cptr[l.ncolors] - beg;
        if (cnt <= 0) return;
        const int lev = (int)(&l - &h.L[0]);
        const int64_t s_lo = l.pm.cseg[K], s_hi = l.pm.cseg[l.ncolors];
        const int jlim = first ? beg : 0x7fffffff;
        int pre = (l.pm.nheavy && s_hi - s_lo >= pre_seg_min()) ? 1 : 0;
        int64_t nnz = 0, hvy = 0;
        for (int c = K; c < l.ncolors; ++c) {
            nnz += l.c_nnz[c];
            if (pre) hvy += l.pm.cheavy[c];
        }
        if (pre && first && l.pm.hlo) {
            pre = 2;  // bounded: only the segments with a column below the bound
            seg<G_PLAIN>(h, l.pm, s_lo, s_hi, l.col, l.val, nullptr, nullptr, x, lev, true,
                         (double)std::min(hvy, l.merged_nnz_lo), jlim, 0, K);
        } else if (pre)
            seg<G_PLAIN>(h, l.pm, s_lo, s_hi, l.col, l.val, nullptr, nullptr, x, lev, true,
                         (double)hvy, jlim, first ? 0 : l.pm.merged_nbr);
        SegWork w = pre ? SegWork{} : segwork(h, l.pm, s_lo, s_hi);
        const int64_t gnnz = first ? l.merged_nnz_lo : nnz - hvy;
        const int64_t gnbr = first ? l.merged_nbr_lo : pre ? l.merged_nbr_light : l.merged_nbr;
        {
            ProfScope ps(h, "jacobi_merged", lev,
                         12.0 * (nnz - hvy) + 20.0 * cnt + Vb(2 * cnt + gnbr), Vb(gnnz));
            const int rpw = short_rpw(cnt, nnz);
            if (rpw > 1)
                launch_k(k_jacobi_rows<KC, true>,
                         dim3(grid_tiles(cnt, 1, rpw) + grid_rows<KC>(w.s_hi - w.s_lo, 0)),
                         dim3(kThreads), 0, h.s, l.contig ? nullptr : l.crows + beg, beg, cnt,
                         l.rp, l.col, l.val, l.diag, b, x, h.T, jlim, rpw, hd(h, l.pm), w, pre);
            else
                launch_k(k_jacobi_rows<KC, false>, dim3(grid_rows<KC>(cnt + (w.s_hi - w.s_lo))),
                         dim3(kThreads), 0, h.s, l.contig ? nullptr : l.crows + beg, beg, cnt,
                         l.rp, l.col, l.val, l.diag, b, x, h.T, jlim, 1, hd(h, l.pm), w, pre);
        }
        ProfScope ps(h, "jacobi_scatter", lev, Vb(2 * cnt) + 4.0 * cnt);
        launch_k(k_scatter_rows<KC>, dim3(grid_rows<KC>(cnt)), dim3(kThreads), 0, h.s, 
            l.contig ? nullptr : l.crows + beg, beg, cnt, h.T, x);
    }

    // The whole outer iteration as one CUDA graph: a while node whose body is
    // centre -> V-cycle -> update -> residual -> status; the status kernel sets
    // the loop condition, so no host round trip happens between iterations.
    static cudaGraphExec_t loop_graph(Hier& h, const CfSolveParams& p) {
        const int key = KC * 1000000 + p.nu1 * 1000 + p.nu2;
        auto it = h.loop_graphs.find(key);
        if (it != h.loop_graphs.end()) return it->second;
        cudaGraph_t g;
        CF_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hc;
        CF_CUDA(cudaGraphConditionalHandleCreate(&hc, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hc;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CF_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CF_CUDA(cudaStreamBeginCaptureToGraph(h.s, body, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal));
        try {
            issue_iteration(h, p, hc, 1);
        } catch (...) {
            cudaGraph_t tmp;
            cudaStreamEndCapture(h.s, &tmp);
            cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t captured;
        CF_CUDA(cudaStreamEndCapture(h.s, &captured));
        cudaGraphExec_t ge;
        CF_CUDA(cudaGraphInstantiate(&ge, g, 0));
        CF_CUDA(cudaGraphDestroy(g));
        h.loop_graphs.emplace(key, ge);
        return ge;
    }
    // one outer iteration after a check: centre, cycle, update, next check
    static void issue_iteration(Hier& h, const CfSolveParams& p, cudaGraphConditionalHandle hc,
                                int use_cond) {
        const int n = h.n0;
        double* mean = h.sums + 2 * KC;
        double* csum = h.sums + 3 * KC;
        center(h, h.R, mean);
        cycle(h, 0, p.nu1, p.nu2);
        colsum(h, h.X, h.C, csum);
        {
            ProfScope ps(h, "update", 0, 3.0 * 8.0 * KC * n);
            launch_k(k_update<KC>, dim3(grid_rows<KC>(n)), dim3(kThreads), 0, h.s, n, h.X, h.C, csum, h.state);
        }
        residual(h, h.B, h.X, h.R, h.sums);
        status(h, p, hc, use_cond);
    }
    static void status(Hier& h, const CfSolveParams& p, cudaGraphConditionalHandle hc,
                       int use_cond) {
        ProfScope ps(h, "status", 0, 0.0);
        LoopCtl ctl{h.d_lp, h.d_iter, h.d_vcyc, h.d_ncyc};
        launch_k(k_status_loop<KC>, dim3(1), dim3(KC < 32 ? 32 : KC), 0, h.s, 
            h.n0, h.sums, h.bn, h.res, h.prev, h.stall, h.state, h.sums + 2 * KC, h.count, ctl, hc,
            use_cond);
    }

    static void run_cycle(Hier& h, int nu1, int nu2) {
        if (h.prof) {  // eager launches so every kernel can be bracketed by events
            cycle(h, 0, nu1, nu2);
            return;
        }
        auto it = h.cycle_graphs.find(KC * 1000000 + nu1 * 1000 + nu2);
        if (it == h.cycle_graphs.end()) {
            cudaGraph_t g;
            CF_CUDA(cudaStreamBeginCapture(h.s, cudaStreamCaptureModeThreadLocal));
            try {
                cycle(h, 0, nu1, nu2);
            } catch (...) {
                cudaStreamEndCapture(h.s, &g);
                throw;
            }
            CF_CUDA(cudaStreamEndCapture(h.s, &g));
            cudaGraphExec_t ge;
            CF_CUDA(cudaGraphInstantiate(&ge, g, 0));
            CF_CUDA(cudaGraphDestroy(g));
            it = h.cycle_graphs.emplace(KC * 1000000 + nu1 * 1000 + nu2, ge).first;
        }
        CF_CUDA(cudaGraphLaunch(it->second, h.s));
    }

    // --------------------------------------------------------------------
    // Fallback: V-cycle preconditioned flexible CG (solver.py:571-610) and
    // Jacobi-preconditioned CG (solver.py:613-648) on the masked columns.
    // Rare path: per-column scalars are formed on the host.
    static void host_sums(Hier& h, int nq, double* out) {
        CF_CUDA(cudaMemcpyAsync(out, h.sums, sizeof(double) * nq * KC, cudaMemcpyDeviceToHost,
                                h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
    }
    static void set_coef(Hier& h, const std::vector<double>& coef) {
        CF_CUDA(cudaMemcpyAsync(h.coef, coef.data(), sizeof(double) * 3 * KC,
                                cudaMemcpyHostToDevice, h.s));
    }
    static void center_cols(Hier& h, double* Xd, const std::vector<char>& mask) {
        // X[:, mask] -= mean(X[:, mask])
        colsum(h, Xd, nullptr, h.sums);
        std::vector<double> s(KC);
        host_sums(h, 1, s.data());
        std::vector<double> coef(3 * KC, 0.0);
        for (int c = 0; c < KC; ++c) {
            coef[c] = 1.0;
            coef[KC + c] = mask[c] ? -s[c] / (double)h.n0 : 0.0;
        }
        // Y = Y + (-mean) * ones : use W = nullptr, U = ones? implement via lincomb on a ones buffer
        set_coef(h, coef);
        k_add_const(h, Xd);
    }
    static void k_add_const(Hier& h, double* Xd);
    static void column_res(Hier& h, const double* Xd, const std::vector<double>& bn,
                           const std::vector<char>& mask, std::vector<double>& res) {
        residual(h, h.B, Xd, nullptr, h.sums);
        std::vector<double> s(2 * KC);
        host_sums(h, 2, s.data());
        for (int c = 0; c < KC; ++c)
            if (mask[c]) res[c] = std::sqrt(s[KC + c]) / bn[c];
    }

    // one FCG iteration of the Krylov hand-off (kernels above); R holds
    // b - L x with its sums, mean = column means of R, P / AP the direction
    static void krylov_iteration(Hier& h, int nu1, int nu2, cudaGraphConditionalHandle hc,
                                 int use_cond) {
        const int n = h.n0;
        const int64_t np = nparts_of(n);
        double* mean = h.sums + 2 * KC;
        double* csum = h.sums + 3 * KC;
        double* q = h.sums + 4 * KC;  // 2 x KC
        double* dd = h.sums + 6 * KC; // 2 x KC
        center(h, h.R, mean);
        cycle(h, 0, nu1, nu2);
        colsum(h, h.C, nullptr, csum);
        {
            ProfScope ps(h, "krylov", 0, 3.0 * Vb(n));
            launch_k(k_kry_beta<KC>, dim3((unsigned)np), dim3(kThreads), red_smem<KC, 2>(), h.s,
                     n, h.C, csum, h.P, h.AP, redctl(h, h.parts, np, q, 0));
        }
        {
            ProfScope ps(h, "krylov", 0, 3.0 * Vb(n));
            launch_k(k_kry_dir<KC>, dim3(grid_rows<KC>(n)), dim3(kThreads), 0, h.s, n, h.C, csum,
                     q, h.P);
        }
        spmm(h, h.P, h.AP);
        dot2(h, h.P, h.AP, h.R, h.P, dd);
        {
            ProfScope ps(h, "krylov", 0, 3.0 * Vb(n));
            launch_k(k_kry_step<KC>, dim3(grid_rows<KC>(n)), dim3(kThreads), 0, h.s, n, h.X, h.P,
                     dd, h.state);
        }
        residual(h, h.B, h.X, h.R, h.sums);
        ProfScope ps(h, "status", 0, 0.0);
        LoopCtl ctl{h.d_lp, h.d_iter, h.d_vcyc, h.d_ncyc};
        launch_k(k_kry_status<KC>, dim3(1), dim3(KC < 32 ? 32 : KC), 0, h.s, n, h.sums, h.bn,
                 h.res, h.state, mean, h.count, ctl, h.d_iter + 2, hc, use_cond);
    }
    static cudaGraphExec_t krylov_graph(Hier& h, int nu1, int nu2) {
        const int key = -(KC * 1000000 + nu1 * 1000 + nu2);
        auto it = h.loop_graphs.find(key);
        if (it != h.loop_graphs.end()) return it->second;
        cudaGraph_t g;
        CF_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hc;
        CF_CUDA(cudaGraphConditionalHandleCreate(&hc, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hc;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CF_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CF_CUDA(cudaStreamBeginCaptureToGraph(h.s, body, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal));
        try {
            krylov_iteration(h, nu1, nu2, hc, 1);
        } catch (...) {
            cudaGraph_t tmp;
            cudaStreamEndCapture(h.s, &tmp);
            cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t captured;
        CF_CUDA(cudaStreamEndCapture(h.s, &captured));
        cudaGraphExec_t ge;
        CF_CUDA(cudaGraphInstantiate(&ge, g, 0));
        CF_CUDA(cudaGraphDestroy(g));
        h.loop_graphs.emplace(key, ge);
        return ge;
    }
    // Krylov hand-off driver: columns in COL_KRYLOV (R / sums / mean current
    // for X) iterate until converged or kmax iterations; returns column cycles
    static int64_t krylov(Hier& h, int nu1, int nu2, int kmax, int nkry) {
        h.ensure_fallback(KC);
        CF_CUDA(cudaMemsetAsync(h.P, 0, sizeof(double) * (size_t)h.n0 * KC, h.s));
        CF_CUDA(cudaMemsetAsync(h.AP, 0, sizeof(double) * (size_t)h.n0 * KC, h.s));
        const double kx = (double)kmax;
        CF_CUDA(cudaMemcpyAsync(h.d_lp + 6, &kx, sizeof(double), cudaMemcpyHostToDevice, h.s));
        CF_CUDA(cudaMemsetAsync(h.d_iter + 2, 0, sizeof(int), h.s));
        CF_CUDA(cudaMemsetAsync(h.d_vcyc, 0, sizeof(long long), h.s));
        long long vc0 = nkry;  // the first iteration's cycles (counted at its end only if still active)
        if (h.prof || h.host_loop) {
            *h.h_count = nkry;
            for (int it = 0; it < kmax && *h.h_count > 0; ++it) {
                krylov_iteration(h, nu1, nu2, cudaGraphConditionalHandle{}, 0);
                CF_CUDA(cudaMemcpyAsync(h.h_count, h.count, sizeof(int), cudaMemcpyDeviceToHost,
                                        h.s));
                CF_CUDA(cudaStreamSynchronize(h.s));
            }
        } else {
            CF_CUDA(cudaGraphLaunch(krylov_graph(h, nu1, nu2), h.s));
        }
        long long vc = 0;
        CF_CUDA(cudaMemcpyAsync(&vc, h.d_vcyc, sizeof(long long), cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
        return vc0 + vc;
    }

    // returns the column V-cycles executed
    static int64_t fcg(Hier& h, const std::vector<double>& bn, double tau, int nu1, int nu2,
                       int iters, const std::vector<char>& mask0, std::vector<double>& res) {
        int64_t colcyc = 0;
        h.ensure_fallback(KC);
        std::vector<char> active = mask0, have(KC, 0);
        column_res(h, h.X, bn, active, res);
        CF_CUDA(cudaMemsetAsync(h.P, 0, sizeof(double) * (size_t)h.n0 * KC, h.s));
        CF_CUDA(cudaMemsetAsync(h.AP, 0, sizeof(double) * (size_t)h.n0 * KC, h.s));
        std::vector<double> s(2 * KC), coef(3 * KC);
        for (int it = 0; it < iters; ++it) {
            bool any = false;
            for (int c = 0; c < KC; ++c) {
                active[c] = active[c] && res[c] > tau;
                any = any || active[c];
            }
            if (!any) break;
            for (int c = 0; c < KC; ++c) colcyc += active[c] ? 1 : 0;
            // r = center(b - L x)
            residual(h, h.B, h.X, h.R, h.sums);
            host_sums(h, 2, s.data());
            for (int c = 0; c < KC; ++c) s[c] = s[c] / (double)h.n0;
            CF_CUDA(cudaMemcpyAsync(h.sums + 4 * KC, s.data(), sizeof(double) * KC,
                                    cudaMemcpyHostToDevice, h.s));
            center(h, h.R, h.sums + 4 * KC);
            // z = center(cycle(r))
            run_cycle(h, nu1, nu2);
            colsum(h, h.C, nullptr, h.sums);
            host_sums(h, 1, s.data());
            for (int c = 0; c < KC; ++c) s[c] = s[c] / (double)h.n0;
            CF_CUDA(cudaMemcpyAsync(h.sums + 4 * KC, s.data(), sizeof(double) * KC,
                                    cudaMemcpyHostToDevice, h.s));
            center(h, h.C, h.sums + 4 * KC);
            // beta for columns with a previous direction
            dot2(h, h.C, h.AP, h.P, h.AP, h.sums);
            host_sums(h, 2, s.data());
            for (int c = 0; c < KC; ++c) {
                double beta = 0.0;
                if (active[c] && have[c]) {
                    double zl = s[c], dl = s[KC + c];
                    beta = dl > 0 ? zl / dl : 0.0;
                }
                coef[c] = 1.0;
                coef[KC + c] = -beta;
                coef[2 * KC + c] = 0.0;
            }
            set_coef(h, coef);
            lincomb(h, h.C, h.P, nullptr, h.coef);  // z -= beta p
            // p = z (active), Lp = L z
            for (int c = 0; c < KC; ++c) {
                coef[c] = active[c] ? 0.0 : 1.0;
                coef[KC + c] = active[c] ? 1.0 : 0.0;
                coef[2 * KC + c] = 0.0;
            }
            set_coef(h, coef);
            lincomb(h, h.P, h.C, nullptr, h.coef);
            spmm(h, h.P, h.Z);
            lincomb(h, h.AP, h.Z, nullptr, h.coef);
            for (int c = 0; c < KC; ++c) have[c] = have[c] || active[c];
            // alpha = (r.z)/(z.Lz)
            dot2(h, h.C, h.AP, h.R, h.C, h.sums);
            host_sums(h, 2, s.data());
            for (int c = 0; c < KC; ++c) {
                double dl = s[c], rd = s[KC + c];
                double alpha = (active[c] && dl > 0) ? rd / dl : 0.0;
                coef[c] = 1.0;
                coef[KC + c] = active[c] ? alpha : 0.0;
                coef[2 * KC + c] = 0.0;
            }
            set_coef(h, coef);
            lincomb(h, h.X, h.C, nullptr, h.coef);
            center_cols(h, h.X, active);
            column_res(h, h.X, bn, active, res);
        }
        return colcyc;
    }

    static void jpcg(Hier& h, const std::vector<double>& bn, double tau, int iters,
                     const std::vector<char>& mask, std::vector<double>& res) {
        h.ensure_fallback(KC);
        // Z holds D^-1 (as a column-broadcast the kernel would need); use lincomb with
        // a diagonal-scaling pass instead: k_diag_scale.
        std::vector<double> s(2 * KC), coef(3 * KC), rz(KC), rz2(KC);
        // r = center(b - L x)
        residual(h, h.B, h.X, h.R, h.sums);
        host_sums(h, 2, s.data());
        for (int c = 0; c < KC; ++c) s[c] = s[c] / (double)h.n0;
        CF_CUDA(cudaMemcpyAsync(h.sums + 4 * KC, s.data(), sizeof(double) * KC,
                                cudaMemcpyHostToDevice, h.s));
        center(h, h.R, h.sums + 4 * KC);
        diag_scale(h, h.R, h.Z);  // z = D^-1 r
        CF_CUDA(cudaMemcpyAsync(h.P, h.Z, sizeof(double) * (size_t)h.n0 * KC,
                                cudaMemcpyDeviceToDevice, h.s));
        dot2(h, h.R, h.Z, h.R, h.Z, h.sums);
        host_sums(h, 2, s.data());
        for (int c = 0; c < KC; ++c) rz[c] = s[c];
        std::vector<char> all = mask;
        column_res(h, h.X, bn, all, res);
        std::vector<char> frozen(KC, 1);
        for (int c = 0; c < KC; ++c) frozen[c] = !mask[c] || res[c] <= tau;
        for (int it = 0; it < iters; ++it) {
            bool done = true;
            for (int c = 0; c < KC; ++c) done = done && frozen[c];
            if (done) break;
            spmm(h, h.P, h.AP);
            dot2(h, h.P, h.AP, h.P, h.AP, h.sums);
            host_sums(h, 2, s.data());
            std::vector<double> alpha(KC, 0.0);
            for (int c = 0; c < KC; ++c) {
                double plp = s[c];
                alpha[c] = (plp > 0 && !frozen[c]) ? rz[c] / plp : 0.0;
                coef[c] = 1.0;
                coef[KC + c] = alpha[c];
                coef[2 * KC + c] = 0.0;
            }
            set_coef(h, coef);
            lincomb(h, h.X, h.P, nullptr, h.coef);  // x += alpha p
            for (int c = 0; c < KC; ++c) coef[KC + c] = -alpha[c];
            set_coef(h, coef);
            lincomb(h, h.R, h.AP, nullptr, h.coef);  // r -= alpha Lp
            dot2(h, h.R, h.R, h.R, h.R, h.sums);
            host_sums(h, 2, s.data());
            for (int c = 0; c < KC; ++c) {
                if (mask[c]) res[c] = std::sqrt(s[c]) / bn[c];
                frozen[c] = frozen[c] || !mask[c] || res[c] <= tau;
            }
            diag_scale(h, h.R, h.Z);
            dot2(h, h.R, h.Z, h.R, h.Z, h.sums);
            host_sums(h, 2, s.data());
            for (int c = 0; c < KC; ++c) {
                rz2[c] = s[c];
                double beta = rz[c] > 0 ? rz2[c] / rz[c] : 0.0;
                if (frozen[c]) beta = 0.0;
                coef[c] = beta;  // p = z + beta p
                coef[KC + c] = 1.0;
                coef[2 * KC + c] = 0.0;
            }
            set_coef(h, coef);
            lincomb(h, h.P, h.Z, nullptr, h.coef);
            rz = rz2;
        }
        center_cols(h, h.X, mask);
        column_res(h, h.X, bn, mask, res);
    }
    static void diag_scale(Hier& h, const double* Rd, double* Zd);
};

template <int KC>
__global__ void __launch_bounds__(kThreads) k_diag_scale(int n, const double* __restrict__ diag,
                                                         const double* __restrict__ R,
                                                         double* __restrict__ Z) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> r = ldv_c<V>(R + i * KC + c0);
    double dinv = 1.0 / fmax(diag[i], 2.2250738585072014e-308);
#pragma unroll
    for (int t = 0; t < V; ++t) r.v[t] = dinv * r.v[t];
    stv<V>(Z + i * KC + c0, r);
}

// X[:, c] += coef[KC + c]  (coef[c] ignored)
template <int KC>
__global__ void __launch_bounds__(kThreads) k_addc(int n, double* __restrict__ X,
                                                   const double* __restrict__ coef) {
    CF_PDL_ENTRY();
    CF_LANE_SETUP(KC)
    int64_t i = (int64_t)blockIdx.x * Lt::RPB + slot;
    if (i >= n || !lane_ok) return;
    DV<V> x = ldv_c<V>(X + i * KC + c0);
#pragma unroll
    for (int t = 0; t < V; ++t) x.v[t] = x.v[t] + coef[KC + c0 + t];
    stv<V>(X + i * KC + c0, x);
}

template <int KC>
void Ops<KC>::diag_scale(Hier& h, const double* Rd, double* Zd) {
    ProfScope ps(h, "fallback", 0, 0.0);
    launch_k(k_diag_scale<KC>, dim3(grid_rows<KC>(h.n0)), dim3(kThreads), 0, h.s, h.n0, h.L[0].diag, Rd, Zd);
}
template <int KC>
void Ops<KC>::k_add_const(Hier& h, double* Xd) {
    ProfScope ps(h, "addc", 0, 16.0 * KC * h.n0);
    launch_k(k_addc<KC>, dim3(grid_rows<KC>(h.n0)), dim3(kThreads), 0, h.s, h.n0, Xd, h.coef);
}

// ============================================================================
// block solve driver (solver.py:651-751)
// ============================================================================

template <int KC>
static void solve_block_t(Hier& h, int ncols, const CfSolveParams& p, double* res_out,
                          CfSolveStats& st) {
    const int n = h.n0;
    using O = Ops<KC>;
    // column statistics of B: balance check and norms (solver.py:672-679)
    {
        int64_t np = nparts_of(n);
        {
            ProfScope ps(h, "colstats", 0, 8.0 * KC * n);
            launch_k(k_colstats<KC>, dim3((unsigned)np), dim3(kThreads), red_smem<KC, 3>(), h.s, n,
                     h.B, redctl(h, h.parts, np, h.sums, 0));
        }
        CF_CUDA(cudaMemcpyAsync(h.h_small, h.sums, sizeof(double) * 3 * KC,
                                cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
    }
    std::vector<double> bsum(KC), bl1(KC), bn(KC);
    std::vector<int> bad;
    for (int c = 0; c < KC; ++c) {
        bsum[c] = h.h_small[c];
        bl1[c] = h.h_small[KC + c];
        bn[c] = std::sqrt(h.h_small[2 * KC + c]);
        if (c < ncols && std::fabs(bsum[c]) > 1e-10 * std::max(bl1[c], 2.2250738585072014e-308))
            bad.push_back(c);
    }
    if (!bad.empty()) {
        std::string m = "supply vector columns [";
        for (size_t q = 0; q < bad.size(); ++q) m += (q ? ", " : "") + std::to_string(bad[q]);
        throw CfError(CF_DOMAIN, m + "] are not balanced");
    }
    // per-column state
    std::vector<int> state(KC, COL_ZERO);
    std::vector<double> safe(KC, 1.0), prev(KC, INFINITY), res(KC, 0.0);
    int nactive = 0;
    for (int c = 0; c < ncols; ++c)
        if (bn[c] > 0) {
            state[c] = COL_ACTIVE;
            safe[c] = bn[c];
            ++nactive;
        }
    CF_CUDA(cudaMemsetAsync(h.X, 0, sizeof(double) * (size_t)n * KC, h.s));
    const double tau = p.tau, stop = p.stop_margin * p.tau;
    std::vector<int> zeros(KC, 0);
    CF_CUDA(cudaMemcpyAsync(h.bn, safe.data(), sizeof(double) * KC, cudaMemcpyHostToDevice, h.s));
    CF_CUDA(cudaMemcpyAsync(h.prev, prev.data(), sizeof(double) * KC, cudaMemcpyHostToDevice, h.s));
    CF_CUDA(cudaMemcpyAsync(h.stall, zeros.data(), sizeof(int) * KC, cudaMemcpyHostToDevice, h.s));
    CF_CUDA(cudaMemcpyAsync(h.state, state.data(), sizeof(int) * KC, cudaMemcpyHostToDevice, h.s));
    CF_CUDA(cudaMemsetAsync(h.res, 0, sizeof(double) * KC, h.s));
    double* mean = h.sums + 2 * KC;
    double* csum = h.sums + 3 * KC;
    int64_t fallback_cols = 0;
    if (nactive > 0) {
        // check 0 on the host path, then the device-controlled loop
        // Krylov hand-off: a column whose residual shrank by less
        // than kKrylovFactor in the cycle before check kKrylovCheck continues
        // under FCG preconditioned by the same V-cycle (warm start)
        static const int kKrylovCheck = [] {
            const char* e = std::getenv("CF_KRYLOV_CHECK");
            return e ? std::atoi(e) : 3;
        }();
        static const double kKrylovFactor = [] {
            const char* e = std::getenv("CF_KRYLOV_FACTOR");
            return e ? std::atof(e) : 0.3;
        }();
        const double lp[6] = {stop, p.stagnation_factor, (double)p.stagnation_cycles,
                              (double)p.max_cycles,
                              kKrylovCheck > 0 && kKrylovCheck < p.max_cycles ? (double)kKrylovCheck : -1.0,
                              kKrylovFactor};
        CF_CUDA(cudaMemcpyAsync(h.d_lp, lp, sizeof lp, cudaMemcpyHostToDevice, h.s));
        CF_CUDA(cudaMemsetAsync(h.d_iter, 0, sizeof(int), h.s));
        CF_CUDA(cudaMemsetAsync(h.d_vcyc, 0, sizeof(long long), h.s));
        CF_CUDA(cudaMemsetAsync(h.d_ncyc, 0, sizeof(int), h.s));
        O::residual(h, h.B, h.X, h.R, h.sums, /*x_zero=*/true);
        O::status(h, p, cudaGraphConditionalHandle{}, 0);
        CF_CUDA(cudaMemcpyAsync(h.h_count, h.count, sizeof(int), cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
        if (*h.h_count > 0) {
            if (h.prof || h.host_loop) {
                // eager loop so every kernel is bracketed by events
                for (int it = 0; it <= p.max_cycles && *h.h_count > 0; ++it) {
                    O::issue_iteration(h, p, cudaGraphConditionalHandle{}, 0);
                    CF_CUDA(cudaMemcpyAsync(h.h_count, h.count, sizeof(int),
                                            cudaMemcpyDeviceToHost, h.s));
                    CF_CUDA(cudaStreamSynchronize(h.s));
                }
            } else {
                CF_CUDA(cudaGraphLaunch(O::loop_graph(h, p), h.s));
            }
        }
        long long vc = 0;
        int nc = 0;
        CF_CUDA(cudaMemcpyAsync(&vc, h.d_vcyc, sizeof(long long), cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaMemcpyAsync(&nc, h.d_ncyc, sizeof(int), cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
        st.vcycles += vc;
        st.outer_iterations += nc;
        CF_CUDA(cudaMemcpyAsync(state.data(), h.state, sizeof(int) * KC, cudaMemcpyDeviceToHost,
                                h.s));
        CF_CUDA(cudaMemcpyAsync(res.data(), h.res, sizeof(double) * KC, cudaMemcpyDeviceToHost,
                                h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
        {
            std::vector<char> kr(KC, 0);
            bool any = false;
            for (int c = 0; c < KC; ++c)
                if (state[c] == COL_KRYLOV) {
                    kr[c] = 1;
                    any = true;
                }
            if (any) {
                int nk = 0;
                for (int c = 0; c < KC; ++c) nk += kr[c];
                st.krylov_solves += nk;
                st.vcycles += O::krylov(h, p.nu1, p.nu2, std::max(1, p.max_cycles - kKrylovCheck),
                                        nk);
                CF_CUDA(cudaMemcpyAsync(state.data(), h.state, sizeof(int) * KC,
                                        cudaMemcpyDeviceToHost, h.s));
                CF_CUDA(cudaMemcpyAsync(res.data(), h.res, sizeof(double) * KC,
                                        cudaMemcpyDeviceToHost, h.s));
                CF_CUDA(cudaStreamSynchronize(h.s));
            }
        }
        std::vector<char> fb(KC, 0);
        for (int c = 0; c < KC; ++c)
            if (state[c] == COL_FALLBACK) {
                fb[c] = 1;
                ++fallback_cols;
            }
        if (fallback_cols) {
            std::vector<double> rf(KC, 0.0);
            O::fcg(h, safe, stop, p.nu1, p.nu2, p.fcg_max_iters, fb, rf);
            std::vector<char> still(KC, 0);
            bool any = false;
            for (int c = 0; c < KC; ++c)
                if (fb[c] && rf[c] > stop) {
                    still[c] = 1;
                    any = true;
                }
            if (any) {
                std::vector<double> rg(rf);
                O::jpcg(h, safe, stop, p.jpcg_max_iters, still, rg);
                for (int c = 0; c < KC; ++c)
                    if (still[c]) rf[c] = rg[c];
            }
            double worst = 0.0;
            int nbad = 0;
            for (int c = 0; c < KC; ++c)
                if (fb[c]) {
                    worst = std::max(worst, rf[c]);
                    if (rf[c] > tau) ++nbad;
                }
            if (nbad) {
                char buf[160];
                snprintf(buf, sizeof buf, "%d solve(s) failed to reach tau=%g", nbad, tau);
                throw CfError(CF_CONVERGENCE, buf, worst);
            }
        }
    }
    // final centring and independently recomputed residuals (solver.py:748-749)
    O::colsum(h, h.X, nullptr, csum);
    {
        // X -= mean(X) for all columns
        std::vector<double> s(KC);
        CF_CUDA(cudaMemcpyAsync(s.data(), csum, sizeof(double) * KC, cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaStreamSynchronize(h.s));
        std::vector<double> coef(3 * KC, 0.0);
        for (int c = 0; c < KC; ++c) coef[KC + c] = -(s[c] / (double)n);
        CF_CUDA(cudaMemcpyAsync(h.coef, coef.data(), sizeof(double) * 3 * KC,
                                cudaMemcpyHostToDevice, h.s));
        O::k_add_const(h, h.X);
    }
    O::residual(h, h.B, h.X, nullptr, h.sums);
    std::vector<double> s2(2 * KC);
    CF_CUDA(cudaMemcpyAsync(s2.data(), h.sums, sizeof(double) * 2 * KC, cudaMemcpyDeviceToHost,
                            h.s));
    CF_CUDA(cudaStreamSynchronize(h.s));
    for (int c = 0; c < ncols; ++c) {
        res_out[c] = bn[c] > 0 ? std::sqrt(s2[KC + c]) / bn[c] : 0.0;
        st.max_residual = std::max(st.max_residual, res_out[c]);
    }
    st.solves += ncols;
    st.fallback_solves += fallback_cols;
}

#define CF_DISPATCH(KCV, ...)                        \
    switch (KCV) {                                    \
        case 1: { constexpr int K_ = 1; __VA_ARGS__; } break;     \
        case 8: { constexpr int K_ = 8; __VA_ARGS__; } break;     \
        case 16: { constexpr int K_ = 16; __VA_ARGS__; } break;   \
        case 32: { constexpr int K_ = 32; __VA_ARGS__; } break;   \
        case 64: { constexpr int K_ = 64; __VA_ARGS__; } break;   \
        case 128: { constexpr int K_ = 128; __VA_ARGS__; } break; \
        case 160: { constexpr int K_ = 160; __VA_ARGS__; } break; \
        case 192: { constexpr int K_ = 192; __VA_ARGS__; } break; \
        case 256: { constexpr int K_ = 256; __VA_ARGS__; } break; \
        default: throw CfError(CF_RUNTIME, "unsupported block width"); \
    }

}  // namespace CF_VNS

#ifdef CF_HUB_TU
// hub-profile translation unit: only the block solve is exported
void solve_block_hub(Hier& h, int kc, int ncols, const CfSolveParams& p, double* res_out,
                     CfSolveStats& st) {
    CF_DISPATCH(kc, CF_VNS::solve_block_t<K_>(h, ncols, p, res_out, st));
}
}  // namespace cf
#else
using namespace CF_VNS;
void solve_block_hub(Hier& h, int kc, int ncols, const CfSolveParams& p, double* res_out,
                     CfSolveStats& st);

// Chunk width for the next `rem` columns.  Measured per-width block-solve
// cost (tools/kc_cost.py, profiles/r01/kc_cost_*.txt): 256 columns cost more
// than two chunks of 128 (the per-level X block of 256 columns leaves the L2),
// and widths 16..64 cost about the same as each other, so full chunks are 128
// wide and a tail takes the smallest width that holds it.
int pick_kc(int64_t rem) {
    // A remainder of 129..192 columns runs as ONE chunk of width 160 / 192
    // (5 / 6 columns per lane) instead of a full chunk plus a narrow tail: a
    // narrow chunk costs ~60 % of a full one (the per-nonzero index and
    // latency cost does not shrink with the width), a 25-50 % wider one
    // 25-50 % more.  CF_WIDE_TAIL=0 restores full chunk + tail.
    static const bool wide_tail = [] {
        const char* e = std::getenv("CF_WIDE_TAIL");
        return !e || std::atoi(e) != 0;
    }();
    static const int sizes[] = {1, 8, 16, 32, 64, 128, 256};
    static const int cap = [] {
        const char* e = std::getenv("CF_MAX_KC");
        int c = e ? std::atoi(e) : 128;
        int best = 1;
        for (int s : sizes)
            if (s <= c) best = s;
        return best;
    }();
    if (wide_tail && cap == 128 && rem > 128 && rem <= 192) return rem <= 160 ? 160 : 192;
    if (rem >= cap) return cap;
    for (int s : sizes)
        if (s >= rem) return s;
    return cap;
}

// widest chunk of the plan pick_kc makes for `total` columns (the workspace is
// sized once, before the first chunk, so it never regrows between chunks)
int plan_max_kc(int64_t total) {
    int kmax = 1;
    for (int64_t o = 0; o < total;) {
        const int kc = pick_kc(total - o);
        kmax = std::max(kmax, kc);
        o += std::min<int64_t>(kc, total - o);
    }
    return kmax;
}

static int kc_at_least(int k) {
    static const int sizes[] = {1, 8, 16, 32, 64, 128, 160, 192, 256};
    for (int s : sizes)
        if (s >= k) return s;
    return 256;
}

void solve_block(Hier& h, int kc, int ncols, const CfSolveParams& p, double* res_out,
                 CfSolveStats& st) {
    if (h.hub_profile) {
        solve_block_hub(h, kc, ncols, p, res_out, st);
        return;
    }
    CF_DISPATCH(kc, solve_block_t<K_>(h, ncols, p, res_out, st));
}

void rows_to_block(Hier& h, const double* S_dev, int cnt, int kc, double* B_dev) {
    dim3 blk(32, 8), grd((h.n0 + 31) / 32, (kc + 31) / 32);
    ProfScope ps(h, "transpose", 0, 16.0 * kc * h.n0);
    CF_DISPATCH(kc, (launch_k(k_rows_to_block<K_>, dim3(grd), dim3(blk), 0, h.s, S_dev, cnt, h.n0, h.perm0, B_dev)));
}
void block_to_rows(Hier& h, const double* B_dev, int cnt, int kc, double* S_dev) {
    dim3 blk(32, 8), grd((h.n0 + 31) / 32, (kc + 31) / 32);
    ProfScope ps(h, "transpose", 0, 16.0 * kc * h.n0);
    CF_DISPATCH(kc, (launch_k(k_block_to_rows<K_>, dim3(grd), dim3(blk), 0, h.s, B_dev, cnt, h.n0, h.perm0, S_dev)));
}
RedCtl redctl_dev(Hier& h, double* parts, int64_t np, double* out) {
    return redctl(h, parts, np, out, 0);
}
void colsum_dev(Hier& h, const double* X_dev, int kc, double* out_dev) {
    CF_DISPATCH(kc, Ops<K_>::colsum(h, X_dev, nullptr, out_dev));
}

// ============================================================================
// Hier lifetime
// ============================================================================

void* Hier::dalloc(size_t nb) {
    void* p = nullptr;
    if (nb == 0) nb = 8;
    CF_CUDA(cudaMalloc(&p, nb));
    owned.push_back(p);
    bytes += (int64_t)nb;
    return p;
}

Hier::~Hier() {
    cudaSetDevice(dev);
    for (auto& kv : cycle_graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : loop_graphs) cudaGraphExecDestroy(kv.second);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (void* p : owned) cudaFree(p);
    for (auto& l : L) {
        cudaFree(l.b);
        cudaFree(l.x);
    }
    cudaFree(B);
    cudaFree(X);
    cudaFree(R);
    cudaFree(C);
    cudaFree(Z);
    cudaFree(P);
    cudaFree(AP);
    cudaFree(parts);
    cudaFree(cnt);
    cudaFree(DP);
    cudaFree(fin);
    cudaFree(SP);
    cudaFree(T);
    cudaFree(S);
    cudaFree(PP);
    for (int i = 0; i < 2; ++i) {
        cudaFree(pin[i]);
        cudaFree(pout[i]);
        for (cudaEvent_t e : {ev_in[i], ev_in_free[i], ev_out_ready[i], ev_out_done[i]})
            if (e) cudaEventDestroy(e);
    }
    if (cs) cudaStreamDestroy(cs);
    if (h_count) cudaFreeHost(h_count);
    if (stage_host) cudaFreeHost(stage_host);
    for (auto& e : stage_ev)
        if (e) cudaEventDestroy(e);
    if (h_small) cudaFreeHost(h_small);
    if (s) cudaStreamDestroy(s);
}

void Hier::ensure_workspace(int kc) {
    if (kc <= kc_ws) return;
    for (auto& kv : cycle_graphs) cudaGraphExecDestroy(kv.second);
    cycle_graphs.clear();
    for (auto& kv : loop_graphs) cudaGraphExecDestroy(kv.second);
    loop_graphs.clear();
    CF_CUDA(cudaStreamSynchronize(s));
    auto re = [&](double*& p, size_t elems) {
        if (p) {
            CF_CUDA(cudaFree(p));
        }
        p = nullptr;
        CF_CUDA(cudaMalloc(&p, sizeof(double) * std::max<size_t>(elems, 1)));
    };
    for (size_t j = 1; j < L.size(); ++j) {
        re(L[j].b, (size_t)L[j].n * kc);
        re(L[j].x, (size_t)L[j].n * kc);
    }
    re(B, (size_t)n0 * kc);
    re(X, (size_t)n0 * kc);
    re(R, (size_t)n0 * kc);
    re(C, (size_t)n0 * kc);
    re(S, (size_t)n0 * kc);
    size_t np = 0;
    for (auto& l : L) np = std::max<size_t>(np, (size_t)(nparts_of(l.n) + nparts_of(l.nc) + 2));
    np = std::max<size_t>(np, 3 * (size_t)(nparts_of(n0) + 1));
    re(parts, np * kc);
    parts_cap = np * kc;
    re(SP, (size_t)std::max<int64_t>(max_nseg, 1) * kc);
    re(PP, (size_t)std::max<int64_t>(max_multi, 1) * kc);
    fin_region = (size_t)(3 * (np / kFinSeg + 2)) * kc;
    re(fin, 2 * fin_region);
    {
        const size_t creg = np / kFinSeg + 2;
        if (cnt) cudaFree(cnt);
        CF_CUDA(cudaMalloc(&cnt, sizeof(unsigned) * (2 * creg + 4)));
        CF_CUDA(cudaMemset(cnt, 0, sizeof(unsigned) * (2 * creg + 4)));
        cnt_region = creg;
    }
    re(T, (size_t)std::max<int64_t>(max_merged, 1) * kc);
    {
        int64_t nd = 1;
        for (auto& l : L)
            if (l.kind == CF_LEVEL_COARSEST && l.M) nd = std::max<int64_t>(nd, (int64_t)dense_splits(l.n) * l.n);
        re(DP, (size_t)nd * kc);
    }
    if (Z) {
        cudaFree(Z); cudaFree(P); cudaFree(AP);
        Z = P = AP = nullptr;
        kc_fb = 0;
    }
    kc_ws = kc;
}

void Hier::ensure_fallback(int kc) {
    if (kc <= kc_fb) return;
    auto re = [&](double*& p, size_t elems) {
        if (p) CF_CUDA(cudaFree(p));
        p = nullptr;
        CF_CUDA(cudaMalloc(&p, sizeof(double) * std::max<size_t>(elems, 1)));
    };
    re(Z, (size_t)n0 * kc_ws);
    re(P, (size_t)n0 * kc_ws);
    re(AP, (size_t)n0 * kc_ws);
    kc_fb = kc_ws;
}

int Hier::prof_begin(const char* kind, int level, double bytes_, double gbytes_) {
    if (ev_used + 2 > ev_pool.size()) {
        for (int t = 0; t < 64; ++t) {
            cudaEvent_t e;
            CF_CUDA(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
    }
    ProfRec r{kind, level, bytes_, gbytes_, ev_pool[ev_used], ev_pool[ev_used + 1]};
    ev_used += 2;
    CF_CUDA(cudaEventRecord(r.a, s));
    recs.push_back(r);
    return (int)recs.size() - 1;
}

void Hier::prof_end(int idx) { cudaEventRecord(recs[idx].b, s); }

}  // namespace cf

using namespace cf;

// ============================================================================
// Host <-> device transfers of pageable buffers: the bytes go through a
// persistent pinned staging ring; host-side memcpy is split over threads and
// overlapped with the DMA of the previous piece.
// ============================================================================

namespace cf {
static constexpr size_t kStagePiece = 16u << 20;  // bytes per piece
static constexpr int kStagePieces = 4;

static void par_memcpy(void* dst, const void* src, size_t bytes) {
    const size_t kMin = 4u << 20;
    unsigned nt = std::min<unsigned>(8, std::max<unsigned>(1, (unsigned)(bytes / kMin)));
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    size_t per = (bytes + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        size_t a = t * per, b = std::min(bytes, a + per);
        if (a >= b) break;
        th.emplace_back([=] { std::memcpy((char*)dst + a, (const char*)src + a, b - a); });
    }
    for (auto& x : th) x.join();
}

void Hier::ensure_pipe(int kc) {
    if (!cs) {
        CF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i)
            for (cudaEvent_t* e : {&ev_in[i], &ev_in_free[i], &ev_out_ready[i], &ev_out_done[i]}) {
                CF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
                CF_CUDA(cudaEventRecord(*e, s));  // "free" until first use
            }
    }
    if (kc <= pipe_kc) return;
    CF_CUDA(cudaStreamSynchronize(s));
    CF_CUDA(cudaStreamSynchronize(cs));
    for (int i = 0; i < 2; ++i) {
        cudaFree(pin[i]);
        cudaFree(pout[i]);
        pin[i] = pout[i] = nullptr;
        CF_CUDA(cudaMalloc(&pin[i], sizeof(double) * (size_t)n0 * kc));
        CF_CUDA(cudaMalloc(&pout[i], sizeof(double) * (size_t)n0 * kc));
    }
    pipe_kc = kc;
}

void Hier::ensure_stage() {
    if (stage_host) return;
    CF_CUDA(cudaMallocHost(&stage_host, kStagePiece * kStagePieces));
    for (int i = 0; i < kStagePieces; ++i) CF_CUDA(cudaEventCreateWithFlags(&stage_ev[i], cudaEventDisableTiming));
}

// Page-locked (cudaHostAlloc / cudaHostRegister) host buffers are copied by
// DMA directly; pageable ones go through the pinned staging ring.
static bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void h2d_staged(Hier& h, void* dst_dev, const void* src_host, size_t bytes) {
    if (host_pinned(src_host)) {
        CF_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, h.s));
        return;
    }
    h.ensure_stage();
    size_t off = 0;
    int slot = 0;
    std::vector<bool> used(kStagePieces, false);
    while (off < bytes) {
        size_t nb = std::min(kStagePiece, bytes - off);
        char* st = (char*)h.stage_host + (size_t)slot * kStagePiece;
        if (used[slot]) CF_CUDA(cudaEventSynchronize(h.stage_ev[slot]));
        par_memcpy(st, (const char*)src_host + off, nb);
        CF_CUDA(cudaMemcpyAsync((char*)dst_dev + off, st, nb, cudaMemcpyHostToDevice, h.s));
        CF_CUDA(cudaEventRecord(h.stage_ev[slot], h.s));
        used[slot] = true;
        off += nb;
        slot = (slot + 1) % kStagePieces;
    }
}

void d2h_staged(Hier& h, void* dst_host, const void* src_dev, size_t bytes) {
    if (host_pinned(dst_host)) {  // caller synchronises the stream
        CF_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, h.s));
        return;
    }
    h.ensure_stage();
    // issue up to kStagePieces DMAs ahead, drain in order
    const size_t npieces = (bytes + kStagePiece - 1) / kStagePiece;
    size_t issued = 0, drained = 0;
    auto issue = [&](size_t k) {
        size_t off = k * kStagePiece, nb = std::min(kStagePiece, bytes - off);
        int slot = (int)(k % kStagePieces);
        CF_CUDA(cudaMemcpyAsync((char*)h.stage_host + (size_t)slot * kStagePiece,
                                (const char*)src_dev + off, nb, cudaMemcpyDeviceToHost, h.s));
        CF_CUDA(cudaEventRecord(h.stage_ev[slot], h.s));
    };
    while (issued < npieces && issued < (size_t)kStagePieces) issue(issued++);
    while (drained < npieces) {
        int slot = (int)(drained % kStagePieces);
        size_t off = drained * kStagePiece, nb = std::min(kStagePiece, bytes - off);
        CF_CUDA(cudaEventSynchronize(h.stage_ev[slot]));
        par_memcpy((char*)dst_host + off, (const char*)h.stage_host + (size_t)slot * kStagePiece,
                   nb);
        ++drained;
        if (issued < npieces) issue(issued++);
    }
}
}  // namespace cf

// ============================================================================
// C-ABI
// ============================================================================

extern "C" const char* cf_last_error(void) { return g_last_error.c_str(); }
extern "C" int cf_version(void) { return 1; }
extern "C" int cf_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

template <typename T>
static T* upload(Hier& h, const T* src, size_t cnt);

// Column windows.  On a level whose X block is far
// larger than the L2, rows with at least win_deg() entries are cut into
// segments at multiples of win_rows() columns as well as every kSegNnz
// entries, and all segments of a launch are processed window by window: the
// warps in flight then gather from one window of X (win_rows x 8 KC bytes,
// 32 MB at KC = 128) that stays in the L2 while every hub row consumes it.
// Measured on C5 (ms per JL estimate, profiles/r02/window_sweep_c5.txt):
// windows off ~1,780; 32,768 rows with degree threshold 128 / 256 / 1,024:
// 1,661 / 1,584 / 1,527 (a lower threshold cuts medium rows into many short
// segments, each with a partial to write and read back; 2,048-16,384 are no
// better than 1,024); 16,384 / 65,536 rows at threshold 256: 1,673 / 1,560.
static int64_t win_rows() {
    static const int64_t w = [] {
        const char* e = std::getenv("CF_WIN_ROWS");
        return e ? (int64_t)std::atoll(e) : (int64_t)32768;
    }();
    return w;
}
static int64_t win_deg() {
    static const int64_t d = [] {
        const char* e = std::getenv("CF_WIN_DEG");
        return e ? (int64_t)std::atoll(e) : (int64_t)1024;
    }();
    return d;
}

// Build the heavy-row plan of a CSR operator: rows visited in class order
// (order == nullptr: natural order, one class).  col != nullptr (sorted rows)
// enables the column windows; merged_from = first class of the merged Jacobi
// range (the sweep launch ranges are the classes below it and the merged rest).
static Plan build_plan(Hier& h, int64_t n, const int64_t* rp, const int32_t* order,
                       const int32_t* cls_ptr, int ncls, const int32_t* col = nullptr,
                       int merged_from = 0x7fffffff) {
    Plan pl;
    std::vector<int32_t> hv(n, -1), shv, hrow, hpos;
    std::vector<int64_t> hsp{0}, sb, se;
    if (!order) ncls = 1;
    const int64_t W = win_rows();
    const bool windows = col && W > 0 && n >= 4 * W;
    for (int c = 0; c < ncls; ++c) {
        pl.cseg.push_back((int64_t)sb.size());
        pl.cheavy.push_back(0);
        int64_t lo = order ? cls_ptr[c] : 0, hi = order ? cls_ptr[c + 1] : n;
        for (int64_t q = lo; q < hi; ++q) {
            int64_t i = order ? order[q] : q;
            int64_t deg = rp[i + 1] - rp[i];
            if (deg <= kHeavyNnz) continue;
            hv[i] = (int32_t)pl.nheavy;
            hrow.push_back((int32_t)i);
            hpos.push_back((int32_t)q);
            pl.heavy_nnz += deg;
            pl.cheavy.back() += deg;
            if (windows && deg >= win_deg()) {
                int64_t b = rp[i];
                while (b < rp[i + 1]) {
                    const int64_t wnd = col[b] / W;
                    int64_t e = b + 1;
                    while (e < rp[i + 1] && e - b < kSegNnz && col[e] / W == wnd) ++e;
                    sb.push_back(b);
                    se.push_back(e);
                    shv.push_back((int32_t)pl.nheavy);
                    ++pl.nwin_seg;
                    b = e;
                }
            } else {
                for (int64_t b = rp[i]; b < rp[i + 1]; b += kSegNnz) {
                    sb.push_back(b);
                    se.push_back(std::min<int64_t>(b + kSegNnz, rp[i + 1]));
                    shv.push_back((int32_t)pl.nheavy);
                }
            }
            pl.nheavy++;
            hsp.push_back((int64_t)sb.size());
        }
    }
    pl.cseg.push_back((int64_t)sb.size());
    pl.nseg = (int64_t)sb.size();
    pl.cnbr.assign((size_t)ncls, 0);
    if (pl.nheavy && col) {
        // distinct neighbour rows per launch range (bytes model only)
        const int K = std::min(ncls, std::max(0, merged_from));
        std::vector<int32_t> stamp((size_t)n, -1);
        std::vector<uint8_t> seen_m((size_t)n, 0), seen_a((size_t)n, 0);
        int64_t hidx = 0;
        for (int c = 0; c < ncls; ++c) {
            int64_t lo = order ? cls_ptr[c] : 0, hi = order ? cls_ptr[c + 1] : n;
            for (int64_t q = lo; q < hi; ++q) {
                int64_t i = order ? order[q] : q;
                if (rp[i + 1] - rp[i] <= kHeavyNnz) continue;
                ++hidx;
                for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
                    const int32_t j = col[p];
                    if (stamp[(size_t)j] != c) {
                        stamp[(size_t)j] = c;
                        ++pl.cnbr[(size_t)c];
                    }
                    if (c >= K && !seen_m[(size_t)j]) {
                        seen_m[(size_t)j] = 1;
                        ++pl.merged_nbr;
                    }
                    if (!seen_a[(size_t)j]) {
                        seen_a[(size_t)j] = 1;
                        ++pl.all_nbr;
                    }
                }
            }
        }
        (void)hidx;
    }
    if (pl.nheavy) {
        pl.hv = upload(h, hv.data(), hv.size());
        pl.hsp = upload(h, hsp.data(), hsp.size());
        pl.sbeg = upload(h, sb.data(), sb.size());
        pl.send = upload(h, se.data(), se.size());
        pl.seg_hv = upload(h, shv.data(), shv.size());
        pl.h_row = upload(h, hrow.data(), hrow.size());
        pl.h_pos = upload(h, hpos.data(), hpos.size());
        pl.cntr = (int*)h.dalloc(sizeof(int) * pl.nheavy);
        CF_CUDA(cudaMemset(pl.cntr, 0, sizeof(int) * pl.nheavy));
        if (col && order) {
            // leading segments below the first-sweep bound of the row's class
            const int K = std::min(ncls, std::max(0, merged_from));
            std::vector<int32_t> hlo((size_t)pl.nheavy, 0), lo_list;
            std::vector<int32_t> key_lo;
            pl.cseg_lo.assign(1, 0);
            auto range_of = [&](int c) { return c < K ? c : K; };
            int cur = 0;
            for (int c = 0; c < ncls; ++c) {
                const int r = range_of(c);
                while (cur < r) {
                    pl.cseg_lo.push_back((int64_t)lo_list.size());
                    ++cur;
                }
                const int64_t bound = cls_ptr[r];
                for (int64_t sgi = pl.cseg[c]; sgi < pl.cseg[c + 1]; ++sgi)
                    if (col[sb[(size_t)sgi]] < bound) {
                        ++hlo[(size_t)shv[(size_t)sgi]];
                        lo_list.push_back((int32_t)sgi);
                        key_lo.push_back(W > 0 ? (int32_t)(col[sb[(size_t)sgi]] / W) : 0);
                    }
            }
            while ((int)pl.cseg_lo.size() < std::min(ncls, K + 1) + 1)
                pl.cseg_lo.push_back((int64_t)lo_list.size());
            pl.cseg_lo.back() = (int64_t)lo_list.size();
            // window order inside every launch range
            std::vector<int32_t> idx(lo_list.size());
            for (size_t t = 0; t < idx.size(); ++t) idx[t] = (int32_t)t;
            for (size_t r = 0; r + 1 < pl.cseg_lo.size(); ++r)
                std::stable_sort(idx.begin() + pl.cseg_lo[r], idx.begin() + pl.cseg_lo[r + 1],
                                 [&](int32_t x, int32_t y) { return key_lo[(size_t)x] < key_lo[(size_t)y]; });
            std::vector<int32_t> sorted(lo_list.size());
            for (size_t t = 0; t < idx.size(); ++t) sorted[t] = lo_list[(size_t)idx[t]];
            pl.hlo = upload(h, hlo.data(), hlo.size());
            if (!sorted.empty()) pl.sord_lo = upload(h, sorted.data(), sorted.size());
        }
        if (windows) {
            // processing orders: stable sort by the window of the first entry
            std::vector<int32_t> key((size_t)pl.nseg), ord((size_t)pl.nseg);
            // CF_SEG_SORT=col: order by first column (finer than the window: the
            // warps of a CTA then start at neighbouring columns)
            static const bool by_col = [] {
                const char* e = std::getenv("CF_SEG_SORT");
                return e && std::string(e) == "col";
            }();
            for (int64_t sgi = 0; sgi < pl.nseg; ++sgi)
                key[(size_t)sgi] = by_col ? col[sb[(size_t)sgi]] : (int32_t)(col[sb[(size_t)sgi]] / W);
            auto sort_range = [&](int64_t a, int64_t b) {
                for (int64_t t = a; t < b; ++t) ord[(size_t)t] = (int32_t)t;
                std::stable_sort(ord.begin() + a, ord.begin() + b,
                                 [&](int32_t x, int32_t y) { return key[(size_t)x] < key[(size_t)y]; });
            };
            const int K = std::min(ncls, std::max(0, merged_from));
            for (int c = 0; c < K; ++c) sort_range(pl.cseg[c], pl.cseg[c + 1]);
            sort_range(pl.cseg[K], pl.nseg);
            pl.sord_cls = upload(h, ord.data(), ord.size());
            sort_range(0, pl.nseg);
            pl.sord_all = upload(h, ord.data(), ord.size());
        }
    }
    h.max_nseg = std::max(h.max_nseg, pl.nseg);
    return pl;
}

template <typename T>
static T* upload(Hier& h, const T* src, size_t cnt) {
    if (!src || cnt == 0) return nullptr;
    T* d = (T*)h.dalloc(sizeof(T) * cnt);
    CF_CUDA(cudaMemcpy(d, src, sizeof(T) * cnt, cudaMemcpyHostToDevice));
    return d;
}

// Gauss-Seidel classes of a level with n rows (experiment knobs CF_GS_CLASSES,
// CF_GS_SMALL_ROWS)
static int gs_classes_for(int n) {
    static const int gs_env = [] {
        const char* e = std::getenv("CF_GS_CLASSES");
        return e ? std::max(0, std::atoi(e)) : kGsClasses;
    }();
    static const int gs_small = [] {  // levels below this many rows
        const char* e = std::getenv("CF_GS_SMALL_ROWS");
        return e ? std::atoi(e) : 0;
    }();
    return n < gs_small ? 0 : gs_env;
}

extern "C" int cf_hier_create(int32_t nlev, const CfLevelDesc* ds, int32_t device,
                              void** out) {
    CF_API_BEGIN
    if (nlev < 1) throw CfError(CF_DOMAIN, "hierarchy needs at least one level");
    CF_CUDA(cudaSetDevice(device));
    auto* h = new Hier();
    try {
        h->dev = device;
        CF_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
        h->n0 = ds[0].n;
        h->L.resize(nlev);
        for (int j = 0; j < nlev; ++j) {
            const CfLevelDesc& d = ds[j];
            DLevel& l = h->L[j];
            l.kind = d.kind;
            l.n = d.n;
            l.nc = d.n_coarse;
            l.nnz = d.nnz_off;
            bool need_matrix = (j == 0) || d.kind == CF_LEVEL_AGGREGATION;
            if (need_matrix && d.rowptr) {
                l.rp = upload(*h, d.rowptr, (size_t)d.n + 1);
                l.col = upload(*h, d.col, (size_t)d.nnz_off);
                l.val = upload(*h, d.val, (size_t)d.nnz_off);
                if (!l.col) l.col = (int32_t*)h->dalloc(8);
                if (!l.val) l.val = (double*)h->dalloc(8);
                l.diag = upload(*h, d.diag, (size_t)d.n);
                if (d.kind == CF_LEVEL_AGGREGATION)
                    l.pm = build_plan(*h, d.n, d.rowptr, d.color_rows, d.color_ptr, d.n_colors,
                                      d.col, std::min(d.n_colors, gs_classes_for(d.n)));
                else
                    l.pm = build_plan(*h, d.n, d.rowptr, nullptr, nullptr, 1, d.col);
            } else if (need_matrix) {
                throw CfError(CF_DOMAIN, "level matrix missing");
            }
            if (d.kind == CF_LEVEL_AGGREGATION) {
                l.ncolors = d.n_colors;
                const int gsk = gs_classes_for(d.n);
                l.gs_classes = std::min(d.n_colors, gsk);
                l.merged = d.n_colors > gsk;
                if (l.merged)
                    h->max_merged = std::max<int64_t>(
                        h->max_merged, d.color_ptr[d.n_colors] - d.color_ptr[l.gs_classes]);
                l.cptr.assign(d.color_ptr, d.color_ptr + d.n_colors + 1);
                l.crows = upload(*h, d.color_rows, (size_t)d.n);
                l.contig = true;
                for (int32_t q = 0; q < d.n && l.contig; ++q) l.contig = d.color_rows[q] == q;
                l.agg = upload(*h, d.agg, (size_t)d.n);
                {
                    // aggregate of every off-diagonal entry's column (line search
                    // gathers X_c[agg[j]] without the dependent map load)
                    std::vector<int32_t> ca((size_t)d.nnz_off);
                    for (int64_t q = 0; q < d.nnz_off; ++q) ca[(size_t)q] = d.agg[d.col[q]];
                    l.cagg = upload(*h, ca.data(), ca.size());
                    if (!l.cagg) l.cagg = (int32_t*)h->dalloc(8);
                }
                l.aptr = upload(*h, d.agg_ptr, (size_t)d.n_coarse + 1);
                l.amem = upload(*h, d.agg_members, (size_t)d.n);
                {
                    // restriction pieces: only when some aggregate exceeds kAggPiece
                    std::vector<int32_t> pa, pb, pslot;
                    bool split = false;
                    for (int32_t a = 0; a < d.n_coarse && !split; ++a)
                        split = d.agg_ptr[a + 1] - d.agg_ptr[a] > kAggPiece;
                    if (split) {
                        int32_t nm = 0;
                        for (int32_t a = 0; a < d.n_coarse; ++a) {
                            const int32_t a0 = d.agg_ptr[a], a1 = d.agg_ptr[a + 1];
                            const bool multi = a1 - a0 > kAggPiece;
                            for (int32_t q = a0; q < a1 || q == a0; q += kAggPiece) {
                                pa.push_back(a);
                                pb.push_back(q);
                                pslot.push_back(multi ? nm++ : -1);
                            }
                        }
                        l.npieces = (int64_t)pa.size();
                        l.nmulti = nm;
                        l.pa = upload(*h, pa.data(), pa.size());
                        l.pb = upload(*h, pb.data(), pb.size());
                        l.pslot = upload(*h, pslot.data(), pslot.size());
                        l.acnt = (int*)h->dalloc(sizeof(int) * (size_t)std::max(d.n_coarse, 1));
                        CF_CUDA(cudaMemset(l.acnt, 0, sizeof(int) * (size_t)std::max(d.n_coarse, 1)));
                        h->max_multi = std::max<int64_t>(h->max_multi, nm);
                    } else {
                        l.npieces = d.n_coarse;
                    }
                }
                l.ls = (double*)h->dalloc(sizeof(double) * 2 * kMaxKC);
                // colour-class sizes for the algorithmic-bytes model
                // (_lo: entries / distinct rows with j below the class's first
                // row, what the bounded first sweep reads on a contiguous level)
                std::vector<int64_t> stamp(d.n, -1), stamp_l(d.n, -1);
                for (int c = 0; c < d.n_colors; ++c) {
                    int64_t rows = d.color_ptr[c + 1] - d.color_ptr[c], nnz = 0, nbr = 0;
                    int64_t nnz_lo = 0, nbr_lo = 0, nbr_light = 0;
                    for (int32_t q = d.color_ptr[c]; q < d.color_ptr[c + 1]; ++q) {
                        int32_t i = d.color_rows[q];
                        const bool light = d.rowptr[i + 1] - d.rowptr[i] <= kHeavyNnz;
                        for (int64_t p = d.rowptr[i]; p < d.rowptr[i + 1]; ++p) {
                            ++nnz;
                            int32_t jn = d.col[p];
                            const bool lo = jn < d.color_ptr[c];
                            nnz_lo += lo;
                            if (stamp[jn] != c) {
                                stamp[jn] = c;
                                ++nbr;
                                nbr_lo += lo;
                            }
                            if (light && stamp_l[jn] != c) {
                                stamp_l[jn] = c;
                                ++nbr_light;
                            }
                        }
                    }
                    l.c_nbr_light.push_back(nbr_light);
                    l.c_rows.push_back(rows);
                    l.c_nnz.push_back(nnz);
                    l.c_nbr.push_back(nbr);
                    l.c_nnz_lo.push_back(nnz_lo);
                    l.c_nbr_lo.push_back(nbr_lo);
                }
                // distinct neighbour rows of the merged (Jacobi) classes, counted once
                if (l.merged) {
                    std::vector<uint8_t> seen(d.n, 0), seen_l(d.n, 0);
                    const int32_t mbeg = d.color_ptr[l.gs_classes];
                    for (int32_t q = mbeg; q < d.color_ptr[d.n_colors]; ++q) {
                        int32_t i = d.color_rows[q];
                        const bool light = d.rowptr[i + 1] - d.rowptr[i] <= kHeavyNnz;
                        for (int64_t p = d.rowptr[i]; p < d.rowptr[i + 1]; ++p) {
                            l.merged_nnz_lo += d.col[p] < mbeg;
                            if (!seen[d.col[p]]) {
                                seen[d.col[p]] = 1;
                                ++l.merged_nbr;
                                l.merged_nbr_lo += d.col[p] < mbeg;
                            }
                            if (light && !seen_l[d.col[p]]) {
                                seen_l[d.col[p]] = 1;
                                ++l.merged_nbr_light;
                            }
                        }
                    }
                }
            } else if (d.kind == CF_LEVEL_ELIMINATION) {
                l.nf = d.n_f;
                l.fn = upload(*h, d.f_nodes, (size_t)d.n_f);
                l.cn = upload(*h, d.c_nodes, (size_t)d.n_coarse);
                l.fd = upload(*h, d.f_degree, (size_t)d.n_f);
                l.wcp = upload(*h, d.wcf_ptr, (size_t)d.n_coarse + 1);
                l.wcc = upload(*h, d.wcf_col, (size_t)d.wcf_ptr[d.n_coarse]);
                l.wcv = upload(*h, d.wcf_val, (size_t)d.wcf_ptr[d.n_coarse]);
                {
                    // W_cf entries resolved to (fine node, its degree) at upload
                    const int64_t wn = d.wcf_ptr[d.n_coarse];
                    std::vector<int32_t> wm((size_t)wn);
                    std::vector<double> wd((size_t)wn);
                    for (int64_t q = 0; q < wn; ++q) {
                        wm[(size_t)q] = d.f_nodes[d.wcf_col[q]];
                        wd[(size_t)q] = d.f_degree[d.wcf_col[q]];
                    }
                    l.wcm = upload(*h, wm.data(), wm.size());
                    l.wcd = upload(*h, wd.data(), wd.size());
                    if (!l.wcm) l.wcm = (int32_t*)h->dalloc(8);
                    if (!l.wcd) l.wcd = (double*)h->dalloc(8);
                }
                l.wfp = upload(*h, d.wfc_ptr, (size_t)d.n_f + 1);
                l.w_nnz = d.wcf_ptr[d.n_coarse];
                l.pw = build_plan(*h, d.n_coarse, d.wcf_ptr, nullptr, nullptr, 1);
                l.wfc = upload(*h, d.wfc_col, (size_t)d.wfc_ptr[d.n_f]);
                l.wfv = upload(*h, d.wfc_val, (size_t)d.wfc_ptr[d.n_f]);
                if (!l.wcc) l.wcc = (int32_t*)h->dalloc(8);
                if (!l.wcv) l.wcv = (double*)h->dalloc(8);
                if (!l.wfc) l.wfc = (int32_t*)h->dalloc(8);
                if (!l.wfv) l.wfv = (double*)h->dalloc(8);
            } else {
                if (d.coarse_op && d.n > 1) l.M = upload(*h, d.coarse_op, (size_t)d.n * d.n);
            }
        }
        {
            // kernel profile: power-law graphs (hub levels bound by the L2 -> SM
            // throughput) run the v_hub build; CF_HUB_PROFILE=0/1 overrides
            const CfLevelDesc& d0 = ds[0];
            int64_t maxdeg = 0;
            if (d0.rowptr)
                for (int32_t i = 0; i < d0.n; ++i)
                    maxdeg = std::max<int64_t>(maxdeg, d0.rowptr[i + 1] - d0.rowptr[i]);
            const double mean = d0.n > 0 ? (double)d0.nnz_off / d0.n : 0.0;
            h->hub_profile = d0.n > 262144 && (double)maxdeg > 64.0 * std::max(mean, 1.0);
            if (const char* e = std::getenv("CF_HUB_PROFILE")) h->hub_profile = std::atoi(e) != 0;
        }
        h->sums = (double*)h->dalloc(sizeof(double) * 8 * kMaxKC);
        h->coef = (double*)h->dalloc(sizeof(double) * 4 * kMaxKC);
        h->bn = (double*)h->dalloc(sizeof(double) * kMaxKC);
        h->res = (double*)h->dalloc(sizeof(double) * kMaxKC);
        h->prev = (double*)h->dalloc(sizeof(double) * kMaxKC);
        h->stall = (int*)h->dalloc(sizeof(int) * kMaxKC);
        h->state = (int*)h->dalloc(sizeof(int) * kMaxKC);
        h->count = (int*)h->dalloc(sizeof(int) * 4);
        // CF_HOST_LOOP=1: drive the outer iteration from the host (profilers
        // cannot attribute kernels inside graphs with conditional nodes)
        if (const char* e = std::getenv("CF_HOST_LOOP")) h->host_loop = std::atoi(e) != 0;
        h->d_iter = (int*)h->dalloc(sizeof(int) * 4);
        h->d_lp = (double*)h->dalloc(sizeof(double) * 8);
        h->d_ncyc = (int*)h->dalloc(sizeof(int) * 4);
        h->d_vcyc = (long long*)h->dalloc(sizeof(long long) * 2);
        CF_CUDA(cudaMallocHost(&h->h_count, sizeof(int) * 4));
        CF_CUDA(cudaMallocHost(&h->h_small, sizeof(double) * 16 * kMaxKC));
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    CF_API_END
}

extern "C" int cf_hier_destroy(void* hp) {
    CF_API_BEGIN
    delete (Hier*)hp;
    CF_API_END
}

extern "C" int64_t cf_hier_device_bytes(void* hp) {
    Hier* h = (Hier*)hp;
    int64_t b = h->bytes;
    for (size_t j = 1; j < h->L.size(); ++j) b += 2 * (int64_t)h->L[j].n * h->kc_ws * 8;
    b += 5 * (int64_t)h->n0 * h->kc_ws * 8 + (int64_t)h->parts_cap * 8;
    return b;
}

extern "C" int cf_solve_rows(void* hp, const double* rows, int64_t count,
                             const CfSolveParams* p, double* out_rows, double* residuals,
                             CfSolveStats* st) {
    CF_API_BEGIN
    Hier& h = *(Hier*)hp;
    std::lock_guard<std::mutex> lk(h.mu);
    CF_CUDA(cudaSetDevice(h.dev));
    const int64_t n = h.n0;
    int64_t done = 0;
    if (count > pick_kc(count) && host_pinned(rows) && host_pinned(out_rows)) {
        // several blocks, page-locked host buffers: block b+1's supplies are
        // copied in and block b-1's solutions copied out on the copy stream
        // while block b solves (double-buffered rows-layout staging)
        std::vector<int64_t> off, num;
        std::vector<int> kcs;
        for (int64_t o = 0; o < count;) {
            const int kc = pick_kc(count - o);
            const int64_t c = std::min<int64_t>(kc, count - o);
            off.push_back(o);
            num.push_back(c);
            kcs.push_back(kc);
            o += c;
        }
        const int kmax = *std::max_element(kcs.begin(), kcs.end());
        h.ensure_workspace(kmax);
        h.ensure_pipe(kmax);
        const size_t nb = off.size();
        auto issue_in = [&](size_t b) {
            const int q = (int)(b & 1);
            CF_CUDA(cudaStreamWaitEvent(h.cs, h.ev_in_free[q], 0));
            CF_CUDA(cudaMemcpyAsync(h.pin[q], rows + off[b] * n, sizeof(double) * num[b] * n,
                                    cudaMemcpyHostToDevice, h.cs));
            CF_CUDA(cudaEventRecord(h.ev_in[q], h.cs));
        };
        // an exception (unbalanced column, convergence failure) must not
        // return while copies into / out of the caller's buffers are queued
        struct Drain {
            Hier& h;
            bool armed = true;
            ~Drain() {
                if (armed) {
                    cudaStreamSynchronize(h.s);
                    cudaStreamSynchronize(h.cs);
                }
            }
        } drain{h};
        issue_in(0);
        for (size_t b = 0; b < nb; ++b) {
            const int q = (int)(b & 1);
            if (b + 1 < nb) issue_in(b + 1);
            CF_CUDA(cudaStreamWaitEvent(h.s, h.ev_in[q], 0));
            rows_to_block(h, h.pin[q], (int)num[b], kcs[b], h.B);
            CF_CUDA(cudaEventRecord(h.ev_in_free[q], h.s));
            std::vector<double> res(kcs[b], 0.0);
            solve_block(h, kcs[b], (int)num[b], *p, res.data(), *st);
            CF_CUDA(cudaStreamWaitEvent(h.s, h.ev_out_done[q], 0));
            block_to_rows(h, h.X, (int)num[b], kcs[b], h.pout[q]);
            CF_CUDA(cudaEventRecord(h.ev_out_ready[q], h.s));
            CF_CUDA(cudaStreamWaitEvent(h.cs, h.ev_out_ready[q], 0));
            CF_CUDA(cudaMemcpyAsync(out_rows + off[b] * n, h.pout[q], sizeof(double) * num[b] * n,
                                    cudaMemcpyDeviceToHost, h.cs));
            CF_CUDA(cudaEventRecord(h.ev_out_done[q], h.cs));
            std::memcpy(residuals + off[b], res.data(), sizeof(double) * num[b]);
        }
        drain.armed = false;
        CF_CUDA(cudaStreamSynchronize(h.s));
        CF_CUDA(cudaStreamSynchronize(h.cs));
        done = count;
    }
    if (done < count) h.ensure_workspace(plan_max_kc(count - done));
    while (done < count) {
        int kc = pick_kc(count - done);
        int cnt = (int)std::min<int64_t>(kc, count - done);
        h2d_staged(h, h.S, rows + done * n, sizeof(double) * cnt * n);
        rows_to_block(h, h.S, cnt, kc, h.B);
        std::vector<double> res(kc, 0.0);
        solve_block(h, kc, cnt, *p, res.data(), *st);
        block_to_rows(h, h.X, cnt, kc, h.S);
        d2h_staged(h, out_rows + done * n, h.S, sizeof(double) * cnt * n);
        CF_CUDA(cudaStreamSynchronize(h.s));
        std::memcpy(residuals + done, res.data(), sizeof(double) * cnt);
        done += cnt;
    }
    CF_API_END_STATS(st)
}

// The library stream h.s is a non-blocking stream: device inputs produced on
// the caller's stream are ordered before this call's kernels by an event.
static void order_after(Hier& h, void* caller_stream) {
    cudaEvent_t ev;
    CF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaError_t e1 = cudaEventRecord(ev, (cudaStream_t)caller_stream);
    cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(h.s, ev, 0) : e1;
    cudaEventDestroy(ev);
    CF_CUDA(e2);
}

extern "C" int cf_solve_block_dev(void* hp, const double* B_dev, double* X_dev, int32_t k,
                                  const CfSolveParams* p, double* residuals, CfSolveStats* st,
                                  void* caller_stream) {
    CF_API_BEGIN
    Hier& h = *(Hier*)hp;
    std::lock_guard<std::mutex> lk(h.mu);
    CF_CUDA(cudaSetDevice(h.dev));
    order_after(h, caller_stream);
    if (k < 1 || k > kMaxKC) throw CfError(CF_DOMAIN, "k must be in [1, 256]");
    int kc = kc_at_least(k);
    h.ensure_workspace(kc);
    // B_dev is n x k row-major in node order; widen to kc columns in device order
    CF_CUDA(cudaMemsetAsync(h.B, 0, sizeof(double) * (size_t)h.n0 * kc, h.s));
    int64_t tot = (int64_t)h.n0 * k;
    launch_k(k_permute_rows, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, h.s, B_dev, k, h.B, kc, k, h.n0,
                                                                     h.perm0, 1);
    std::vector<double> res(kc, 0.0);
    solve_block(h, kc, k, *p, res.data(), *st);
    launch_k(k_permute_rows, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, h.s, h.X, kc, X_dev, k, k, h.n0,
                                                                     h.perm0, 0);
    CF_CUDA(cudaStreamSynchronize(h.s));
    std::memcpy(residuals, res.data(), sizeof(double) * k);
    CF_API_END_STATS(st)
}

extern "C" int cf_residual_dev(void* hp, const double* B_dev, const double* X_dev, double* R_dev,
                               int32_t k, double* colsq, void* caller_stream) {
    CF_API_BEGIN
    Hier& h = *(Hier*)hp;
    std::lock_guard<std::mutex> lk(h.mu);
    CF_CUDA(cudaSetDevice(h.dev));
    order_after(h, caller_stream);
    int kc = kc_at_least(k);
    if (kc != k) throw CfError(CF_DOMAIN, "k must be a supported block width");
    h.ensure_workspace(kc);
    int64_t tot = (int64_t)h.n0 * k;
    unsigned grd = (unsigned)((tot + 255) / 256);
    launch_k(k_permute_rows, dim3(grd), dim3(256), 0, h.s, B_dev, k, h.B, kc, k, h.n0, h.perm0, 1);
    launch_k(k_permute_rows, dim3(grd), dim3(256), 0, h.s, X_dev, k, h.X, kc, k, h.n0, h.perm0, 1);
    CF_DISPATCH(kc, Ops<K_>::residual(h, h.B, h.X, h.R, h.sums));
    launch_k(k_permute_rows, dim3(grd), dim3(256), 0, h.s, h.R, kc, R_dev, k, k, h.n0, h.perm0, 0);
    CF_CUDA(cudaMemcpyAsync(colsq, h.sums + k, sizeof(double) * k, cudaMemcpyDeviceToHost, h.s));
    CF_CUDA(cudaStreamSynchronize(h.s));
    CF_API_END
}

extern "C" void* cf_hier_stream(void* hp) { return (void*)((Hier*)hp)->s; }

extern "C" int cf_profile(void* hp, int32_t enable) {
    CF_API_BEGIN
    Hier& h = *(Hier*)hp;
    std::lock_guard<std::mutex> lk(h.mu);
    CF_CUDA(cudaStreamSynchronize(h.s));
    h.prof = enable != 0;
    h.recs.clear();
    h.ev_used = 0;
    CF_API_END
}

// One line per (kind, level): "kind level launches total_ms total_bytes\n".
// Returns the number of bytes needed (excluding NUL) through *needed.
extern "C" int cf_profile_report(void* hp, char* buf, int64_t cap, int64_t* needed) {
    CF_API_BEGIN
    Hier& h = *(Hier*)hp;
    std::lock_guard<std::mutex> lk(h.mu);
    CF_CUDA(cudaStreamSynchronize(h.s));
    struct Agg {
        int64_t launches = 0;
        double ms = 0, bytes = 0, gbytes = 0;
    };
    std::map<std::pair<std::string, int>, Agg> agg;
    for (auto& r : h.recs) {
        float ms = 0.f;
        CF_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        Agg& a = agg[{r.kind, r.level}];
        a.launches += 1;
        a.ms += ms;
        a.bytes += r.bytes;
        a.gbytes += r.gbytes;
    }
    std::string out;
    char line[256];
    for (auto& kv : agg) {
        snprintf(line, sizeof line, "%s %d %lld %.6f %.1f %.1f\n", kv.first.first.c_str(),
                 kv.first.second, (long long)kv.second.launches, kv.second.ms, kv.second.bytes,
                 kv.second.gbytes);
        out += line;
    }
    *needed = (int64_t)out.size();
    if (buf && cap > 0) {
        size_t nb = std::min<size_t>(out.size(), (size_t)cap - 1);
        std::memcpy(buf, out.data(), nb);
        buf[nb] = 0;
    }
    CF_API_END
}

extern "C" int cf_hier_set_order(void* hp, const int32_t* perm, int64_t n) {
    CF_API_BEGIN
    Hier& h = *(Hier*)hp;
    std::lock_guard<std::mutex> lk(h.mu);
    CF_CUDA(cudaSetDevice(h.dev));
    if (n != h.n0) throw CfError(CF_DOMAIN, "order length does not match the hierarchy");
    if (!h.perm0) h.perm0 = (int32_t*)h.dalloc(sizeof(int32_t) * std::max<int64_t>(n, 1));
    CF_CUDA(cudaMemcpy(h.perm0, perm, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    CF_API_END
}
#endif  // CF_HUB_TU
