// Device-side coarse operators of the multigrid setup:
// the Galerkin product P^T L P of an aggregation level (reference
// solver.py:383-386) and the Schur complement L_cc - W D_f^-1 W^T of an
// elimination level (solver.py:251-261), each followed by the Laplacian
// rebuild (solver.py:167-187: symmetrise, keep strictly negative
// off-diagonals, diagonal = minus the off-diagonal row sum).
//
// Both are "expand to (row, col, value) triples, sort by (row, col), sum equal
// keys": the off-diagonal triples are generated on the GPU, sorted with a
// stable radix sort and every run of equal keys is summed left to right by one
// thread, so the result is a pure function of the input (no atomics on values).
// The sums differ from scipy's SpGEMM in rounding only (different order); the
// host route stays the default wherever hierarchies are pinned bit-for-bit to
// the reference (n0 <= 262,144, C1-C3 and the golden graphs).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "cf_common.h"
#include "cfcent_b200.h"

namespace cf {
namespace {

struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    DBuf() = default;
    explicit DBuf(size_t bytes) { alloc(bytes); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    void alloc(size_t bytes) {
        release();
        CF_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        cap = bytes;
    }
    template <typename T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

constexpr int kT = 256;
constexpr uint64_t kNoKey = ~(uint64_t)0;
inline unsigned blocks_for(int64_t items) {
    return (unsigned)std::max<int64_t>(1, (items + kT - 1) / kT);
}

// row of CSR entry p (largest i with indptr[i] <= p)
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ indptr, int64_t n, int64_t p) {
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (indptr[mid] <= p)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Off-diagonal triples of P^T L P: entry (i, j, a) of L -> (agg[i], agg[j], a)
// when the aggregates differ (entries inside an aggregate only touch the
// diagonal, which the rebuild recomputes).
__global__ void __launch_bounds__(kT) k_galerkin_keys(int64_t n, int64_t nnz,
                                                      const int64_t* __restrict__ indptr,
                                                      const int64_t* __restrict__ indices,
                                                      const double* __restrict__ data,
                                                      const int64_t* __restrict__ map, int64_t nc,
                                                      uint64_t* __restrict__ key,
                                                      double* __restrict__ val) {
    const int64_t p = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (p >= nnz) return;
    const int64_t i = row_of(indptr, n, p);
    const int64_t a = map[i], b = map[indices[p]];
    const bool keep = a >= 0 && b >= 0 && a != b;
    key[p] = keep ? (uint64_t)a * (uint64_t)nc + (uint64_t)b : kNoKey;
    val[p] = keep ? data[p] : 0.0;
}

// Fill of the Schur complement: eliminated node f with neighbours c_1..c_d
// (all kept: the eliminated set is independent) and weights w_k = -L[f, c_k]
// contributes -(w_a / d_f) * w_b to (c_a, c_b), a != b.  One warp per f node;
// off[f] = first output slot of its d (d - 1) triples.
__global__ void __launch_bounds__(kT) k_schur_fill(int64_t nf, const int64_t* __restrict__ fnodes,
                                                   const int64_t* __restrict__ indptr,
                                                   const int64_t* __restrict__ indices,
                                                   const double* __restrict__ data,
                                                   const int64_t* __restrict__ map, int64_t nc,
                                                   const int64_t* __restrict__ off,
                                                   uint64_t* __restrict__ key,
                                                   double* __restrict__ val) {
    const int64_t w = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nf) return;
    const int64_t f = fnodes[w];
    const int64_t beg = indptr[f], end = indptr[f + 1];
    const int64_t d = end - beg - 1;  // off-diagonal entries (the diagonal is stored)
    if (d < 2) return;
    // the diagonal sits at the sorted position of f: entries after it shift by one
    int64_t dpos = beg;
    while (dpos < end && indices[dpos] != f) ++dpos;
    const double df = data[dpos];
    // pair index q = a * (d - 1) + b' over ordered pairs a != b
    const int64_t base = off[w];
    const int64_t pairs = d * (d - 1);
    for (int64_t q = lane; q < pairs; q += 32) {
        const int64_t a = q / (d - 1);
        int64_t b = q % (d - 1);
        if (b >= a) ++b;
        // a-th / b-th off-diagonal entry of row f (skip the diagonal position)
        int64_t pa = beg + a, pb = beg + b;
        if (pa >= dpos) ++pa;
        if (pb >= dpos) ++pb;
        const double wa = -data[pa], wb = -data[pb];
        const int64_t ca = map[indices[pa]], cb = map[indices[pb]];
        key[base + q] = (uint64_t)ca * (uint64_t)nc + (uint64_t)cb;
        val[base + q] = -((wa * (1.0 / df)) * wb);
    }
}

__global__ void __launch_bounds__(kT) k_heads(int64_t cnt, const uint64_t* __restrict__ key,
                                              int32_t* __restrict__ head) {
    const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (t >= cnt) return;
    head[t] = (key[t] != kNoKey && (t == 0 || key[t] != key[t - 1])) ? 1 : 0;
}

// one thread per run of equal keys: left-to-right sum (fixed order)
__global__ void __launch_bounds__(kT) k_sum_runs(int64_t cnt, const uint64_t* __restrict__ key,
                                                 const double* __restrict__ val,
                                                 const int32_t* __restrict__ head,
                                                 const int32_t* __restrict__ pos,
                                                 uint64_t* __restrict__ ukey,
                                                 double* __restrict__ uval) {
    const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (t >= cnt || !head[t]) return;
    const uint64_t k = key[t];
    double s = val[t];
    for (int64_t q = t + 1; q < cnt && key[q] == k; ++q) s += val[q];
    ukey[pos[t]] = k;
    uval[pos[t]] = s;
}

// symmetrise: v(I,J) = (s(I,J) + s(J,I)) * 0.5 (missing mirror = 0); keep v < 0
__global__ void __launch_bounds__(kT) k_symmetrise(int64_t U, int64_t nc,
                                                   const uint64_t* __restrict__ ukey,
                                                   const double* __restrict__ uval,
                                                   double* __restrict__ sval,
                                                   int32_t* __restrict__ keep) {
    const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (t >= U) return;
    const uint64_t k = ukey[t];
    const uint64_t I = k / (uint64_t)nc, J = k % (uint64_t)nc;
    const uint64_t mk = J * (uint64_t)nc + I;
    int64_t lo = 0, hi = U;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ukey[mid] < mk)
            lo = mid + 1;
        else
            hi = mid;
    }
    const double mirror = (lo < U && ukey[lo] == mk) ? uval[lo] : 0.0;
    const double v = (uval[t] + mirror) * 0.5;
    sval[t] = v;
    keep[t] = v < 0.0 ? 1 : 0;
}

// first unique entry of every coarse row (binary search), for the row loops
__global__ void __launch_bounds__(kT) k_urow_ptr(int64_t nc, int64_t U,
                                                 const uint64_t* __restrict__ ukey,
                                                 int64_t* __restrict__ urp) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i > nc) return;
    const uint64_t target = (uint64_t)i * (uint64_t)nc;
    int64_t lo = 0, hi = U;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ukey[mid] < target)
            lo = mid + 1;
        else
            hi = mid;
    }
    urp[i] = lo;
}

// kept entries per row (+ 1 for the diagonal); one warp per row
__global__ void __launch_bounds__(kT) k_row_counts(int64_t nc, const int64_t* __restrict__ urp,
                                                   const int32_t* __restrict__ keep,
                                                   int64_t* __restrict__ cnt) {
    const int64_t i = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nc) return;
    int64_t c = 0;
    for (int64_t t = urp[i] + lane; t < urp[i + 1]; t += 32) c += keep[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[i] = c + 1;
}

// write row i (one warp per row): kept off-diagonals in column order with the
// diagonal at its sorted position; diagonal = minus their sum, accumulated
// per 32-entry chunk by a fixed shuffle tree and over the chunks in column
// order (a fixed order for a given row)
__global__ void __launch_bounds__(kT) k_emit_rows(int64_t nc, const int64_t* __restrict__ urp,
                                                  const uint64_t* __restrict__ ukey,
                                                  const double* __restrict__ sval,
                                                  const int32_t* __restrict__ keep,
                                                  const int64_t* __restrict__ optr,
                                                  int64_t* __restrict__ oidx,
                                                  double* __restrict__ oval) {
    const int64_t i = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nc) return;
    const int64_t beg = urp[i], end = urp[i + 1];
    const int64_t o0 = optr[i];
    int64_t below = 0;  // kept entries left of the diagonal, found so far
    int64_t done = 0;   // kept entries written so far
    double dg = 0.0;
    for (int64_t base = beg; base < end; base += 32) {
        const int64_t t = base + lane;
        const bool k = t < end && keep[t];
        const int64_t j = k ? (int64_t)(ukey[t] % (uint64_t)nc) : 0;
        const double v = k ? sval[t] : 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, k);
        const unsigned lo = __ballot_sync(0xffffffffu, k && j < i);
        if (k) {
            const int r = __popc(m & ((1u << lane) - 1u));
            // entries right of the diagonal shift by one slot
            const int64_t slot = o0 + done + r + (j > i ? 1 : 0);
            oidx[slot] = j;
            oval[slot] = v;
        }
        double part = -v;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        dg += part;
        done += __popc(m);
        below += __popc(lo);
    }
    if (lane == 0) {
        oidx[o0 + below] = i;
        oval[o0 + below] = dg;
    }
}

// result kept on the device between cf_coarse_*_dev and cf_coarse_fetch_dev
struct CoarseCtx {
    int device = -1;
    int64_t nc = 0, nnz = 0;
    DBuf optr, oidx, oval;
};
thread_local CoarseCtx g_ctx;

// sort the (key, val) triples, sum runs, symmetrise, assemble the CSR Laplacian
void finish_coarse(int device, int64_t nc, int64_t cnt, DBuf& key, DBuf& val) {
    if (cnt >= (int64_t)1 << 31) throw CfError(CF_RUNTIME, "too many triples for one device sort");
    CoarseCtx& c = g_ctx;
    c.device = device;
    c.nc = nc;
    DBuf key2(sizeof(uint64_t) * std::max<int64_t>(cnt, 1)), val2(sizeof(double) * std::max<int64_t>(cnt, 1));
    int64_t U = 0;
    DBuf head, pos, ukey, uval;
    if (cnt > 0) {
        size_t tb = 0;
        int end_bit = 1;
        while (end_bit < 64 && (((uint64_t)nc * (uint64_t)nc) >> end_bit)) ++end_bit;
        // sentinel keys (all ones) must sort last: sort all 64 bits when present
        end_bit = 64;
        CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<uint64_t>(), key2.as<uint64_t>(),
                                                val.as<double>(), val2.as<double>(), (int)cnt, 0,
                                                end_bit));
        DBuf tmp(tb);
        CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.as<uint64_t>(), key2.as<uint64_t>(),
                                                val.as<double>(), val2.as<double>(), (int)cnt, 0,
                                                end_bit));
        head.alloc(sizeof(int32_t) * cnt);
        pos.alloc(sizeof(int32_t) * cnt);
        k_heads<<<blocks_for(cnt), kT>>>(cnt, key2.as<uint64_t>(), head.as<int32_t>());
        size_t sb = 0;
        CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, head.as<int32_t>(), pos.as<int32_t>(), (int)cnt));
        DBuf stmp(sb);
        CF_CUDA(cub::DeviceScan::ExclusiveSum(stmp.p, sb, head.as<int32_t>(), pos.as<int32_t>(), (int)cnt));
        int32_t lh = 0, lp = 0;
        CF_CUDA(cudaMemcpy(&lh, head.as<int32_t>() + (cnt - 1), sizeof(int32_t), cudaMemcpyDeviceToHost));
        CF_CUDA(cudaMemcpy(&lp, pos.as<int32_t>() + (cnt - 1), sizeof(int32_t), cudaMemcpyDeviceToHost));
        U = (int64_t)lh + lp;
        ukey.alloc(sizeof(uint64_t) * std::max<int64_t>(U, 1));
        uval.alloc(sizeof(double) * std::max<int64_t>(U, 1));
        k_sum_runs<<<blocks_for(cnt), kT>>>(cnt, key2.as<uint64_t>(), val2.as<double>(),
                                            head.as<int32_t>(), pos.as<int32_t>(),
                                            ukey.as<uint64_t>(), uval.as<double>());
        CF_CUDA(cudaGetLastError());
    } else {
        ukey.alloc(16);
        uval.alloc(16);
    }
    key.release();
    val.release();
    key2.release();
    val2.release();
    DBuf sval(sizeof(double) * std::max<int64_t>(U, 1)), keep(sizeof(int32_t) * std::max<int64_t>(U, 1));
    DBuf urp(sizeof(int64_t) * (nc + 1)), rcnt(sizeof(int64_t) * (nc + 1));
    if (U) k_symmetrise<<<blocks_for(U), kT>>>(U, nc, ukey.as<uint64_t>(), uval.as<double>(),
                                               sval.as<double>(), keep.as<int32_t>());
    k_urow_ptr<<<blocks_for(nc + 1), kT>>>(nc, U, ukey.as<uint64_t>(), urp.as<int64_t>());
    CF_CUDA(cudaMemset(rcnt.p, 0, sizeof(int64_t) * (nc + 1)));
    k_row_counts<<<blocks_for(nc * 32), kT>>>(nc, urp.as<int64_t>(), keep.as<int32_t>(), rcnt.as<int64_t>());
    c.optr.alloc(sizeof(int64_t) * (nc + 1));
    size_t sb = 0;
    CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, rcnt.as<int64_t>(), c.optr.as<int64_t>(), (int)(nc + 1)));
    DBuf stmp(sb);
    CF_CUDA(cub::DeviceScan::ExclusiveSum(stmp.p, sb, rcnt.as<int64_t>(), c.optr.as<int64_t>(), (int)(nc + 1)));
    int64_t total = 0;
    CF_CUDA(cudaMemcpy(&total, c.optr.as<int64_t>() + nc, sizeof(int64_t), cudaMemcpyDeviceToHost));
    c.nnz = total;
    c.oidx.alloc(sizeof(int64_t) * std::max<int64_t>(total, 1));
    c.oval.alloc(sizeof(double) * std::max<int64_t>(total, 1));
    k_emit_rows<<<blocks_for(nc * 32), kT>>>(nc, urp.as<int64_t>(), ukey.as<uint64_t>(), sval.as<double>(),
                                        keep.as<int32_t>(), c.optr.as<int64_t>(), c.oidx.as<int64_t>(),
                                        c.oval.as<double>());
    CF_CUDA(cudaGetLastError());
    CF_CUDA(cudaDeviceSynchronize());
}

}  // namespace
}  // namespace cf

using namespace cf;

// ---- Laplacian validation (solver.py:190-211) --------------------------------
namespace cf {
namespace {

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// out[0] = max |v|; out[1] = max |m - m^T|; out[3] = max off-diagonal value (if positive)
__global__ void __launch_bounds__(kT) k_validate_entries(int64_t n, int64_t nnz,
                                                         const int64_t* __restrict__ indptr,
                                                         const int64_t* __restrict__ indices,
                                                         const double* __restrict__ data,
                                                         double* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * kT + threadIdx.x;
    double m_abs = 0.0, m_asym = 0.0, m_pos = 0.0;
    if (p < nnz) {
        const int64_t i = row_of(indptr, n, p);
        const int64_t j = indices[p];
        const double v = data[p];
        m_abs = fabs(v);
        if (i != j) {
            if (v > 0.0) m_pos = v;
            // mirror entry (j, i): rows are sorted
            int64_t lo = indptr[j], hi = indptr[j + 1];
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (indices[mid] < i)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            const double t = (lo < indptr[j + 1] && indices[lo] == i) ? data[lo] : 0.0;
            m_asym = fabs(v - t);
        }
    }
    // one atomic per warp and quantity (max is order-independent)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m_abs = fmax(m_abs, __shfl_xor_sync(0xffffffffu, m_abs, o));
        m_asym = fmax(m_asym, __shfl_xor_sync(0xffffffffu, m_asym, o));
        m_pos = fmax(m_pos, __shfl_xor_sync(0xffffffffu, m_pos, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (m_abs > 0.0) atomic_max_nonneg(out + 0, m_abs);
        if (m_asym > 0.0) atomic_max_nonneg(out + 1, m_asym);
        if (m_pos > 0.0) atomic_max_nonneg(out + 3, m_pos);
    }
}
// out[2] = max |row sum|
__global__ void __launch_bounds__(kT) k_validate_rows(int64_t n, const int64_t* __restrict__ indptr,
                                                      const double* __restrict__ data,
                                                      double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += data[p];
    if (s != 0.0) atomic_max_nonneg(out + 2, fabs(s));
}
__global__ void __launch_bounds__(kT) k_cc_init32(int64_t n, int32_t* __restrict__ parent) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i < n) parent[i] = (int32_t)i;
}
// hooking over the CSR entries (i < j once per undirected edge)
__global__ void __launch_bounds__(kT) k_cc_hook_csr(int64_t n, int64_t nnz,
                                                    const int64_t* __restrict__ indptr,
                                                    const int64_t* __restrict__ indices,
                                                    int32_t* __restrict__ parent,
                                                    int* __restrict__ changed) {
    const int64_t p = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (p >= nnz) return;
    const int64_t j = indices[p];
    const int64_t i = row_of(indptr, n, p);
    if (i >= j) return;
    const int32_t a = parent[i], b = parent[j];
    if (a == b) return;
    const int32_t hi = a > b ? a : b, lo = a > b ? b : a;
    atomicMin(parent + hi, lo);
    *changed = 1;
}
__global__ void __launch_bounds__(kT) k_cc_jump32(int64_t n, int32_t* __restrict__ parent) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i >= n) return;
    int32_t p = parent[i];
    while (true) {
        const int32_t q = parent[p];
        if (q == p) break;
        p = q;
    }
    parent[i] = p;
}
__global__ void __launch_bounds__(kT) k_count_roots(int64_t n, const int32_t* __restrict__ parent,
                                                    unsigned long long* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i < n && parent[i] == (int32_t)i) atomicAdd(cnt, 1ull);
}

}  // namespace
}  // namespace cf

// The checks of _validate_laplacian (solver.py:190-211) on GPU `device` for an
// n x n CSR with sorted rows: out[0] = max |entry|, out[1] = max |m - m^T|,
// out[2] = max |row sum|, out[3] = largest positive off-diagonal (0 if none);
// *ncomp = connected components of the off-diagonal pattern.  Integer / max
// reductions only: the verdict equals the host route's.
extern "C" int cf_validate_laplacian_dev(int32_t device, int64_t n, const int64_t* indptr,
                                         const int64_t* indices, const double* data,
                                         double* out, int64_t* ncomp) {
    CF_API_BEGIN
    if (n < 0) throw cf::CfError(CF_DOMAIN, "negative size");
    if ((uint64_t)n >= ((uint64_t)1 << 31)) throw cf::CfError(CF_RUNTIME, "too many nodes");
    CF_CUDA(cudaSetDevice(device));
    const int64_t nnz = n ? indptr[n] : 0;
    cf::DBuf dp(sizeof(int64_t) * (n + 1)), di(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    cf::DBuf dd(sizeof(double) * std::max<int64_t>(nnz, 1)), dout(sizeof(double) * 4);
    cf::DBuf par(sizeof(int32_t) * std::max<int64_t>(n, 1)), chg(sizeof(int)), cnt(sizeof(unsigned long long));
    if (n) CF_CUDA(cudaMemcpy(dp.p, indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    if (nnz) {
        CF_CUDA(cudaMemcpy(di.p, indices, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice));
        CF_CUDA(cudaMemcpy(dd.p, data, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
    CF_CUDA(cudaMemset(dout.p, 0, sizeof(double) * 4));
    if (nnz)
        cf::k_validate_entries<<<cf::blocks_for(nnz), cf::kT>>>(n, nnz, dp.as<int64_t>(),
                                                                di.as<int64_t>(), dd.as<double>(),
                                                                dout.as<double>());
    if (n)
        cf::k_validate_rows<<<cf::blocks_for(n), cf::kT>>>(n, dp.as<int64_t>(), dd.as<double>(),
                                                           dout.as<double>());
    if (n) cf::k_cc_init32<<<cf::blocks_for(n), cf::kT>>>(n, par.as<int32_t>());
    for (int r = 0; nnz > 0 && r < 4096; ++r) {
        CF_CUDA(cudaMemset(chg.p, 0, sizeof(int)));
        cf::k_cc_hook_csr<<<cf::blocks_for(nnz), cf::kT>>>(n, nnz, dp.as<int64_t>(), di.as<int64_t>(),
                                                          par.as<int32_t>(), chg.as<int>());
        cf::k_cc_jump32<<<cf::blocks_for(n), cf::kT>>>(n, par.as<int32_t>());
        int h = 0;
        CF_CUDA(cudaMemcpy(&h, chg.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (!h) break;
    }
    CF_CUDA(cudaMemset(cnt.p, 0, sizeof(unsigned long long)));
    if (n) cf::k_count_roots<<<cf::blocks_for(n), cf::kT>>>(n, par.as<int32_t>(), cnt.as<unsigned long long>());
    CF_CUDA(cudaGetLastError());
    unsigned long long c = 0;
    CF_CUDA(cudaMemcpy(&c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost));
    CF_CUDA(cudaMemcpy(out, dout.p, sizeof(double) * 4, cudaMemcpyDeviceToHost));
    *ncomp = (int64_t)c;
    CF_API_END
}

// Coarse operator of one setup level on GPU `device`.  L: n x n CSR with its
// diagonal stored, sorted rows.  map[i] = coarse index of fine node i (the
// aggregate for a Galerkin product; the position among the kept nodes, or -1
// for an eliminated node, for a Schur complement).  nf = 0: Galerkin
// (solver.py:383-386); nf > 0: Schur complement of the independent set
// fnodes (solver.py:251-261).  *nnz_out = entries of the rebuilt coarse
// Laplacian (diagonal included), fetched with cf_coarse_fetch_dev.
extern "C" int cf_coarse_operator_dev(int32_t device, int64_t n, const int64_t* indptr,
                                      const int64_t* indices, const double* data,
                                      const int64_t* map, int64_t nc, int64_t nf,
                                      const int64_t* fnodes, int64_t* nnz_out) {
    CF_API_BEGIN
    if (n < 0 || nc < 0 || nf < 0) throw CfError(CF_DOMAIN, "negative sizes");
    if ((uint64_t)nc >= ((uint64_t)1 << 31)) throw CfError(CF_RUNTIME, "too many coarse nodes");
    CF_CUDA(cudaSetDevice(device));
    const int64_t nnz = indptr[n];
    DBuf dp(sizeof(int64_t) * (n + 1)), di(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    DBuf dd(sizeof(double) * std::max<int64_t>(nnz, 1)), dm(sizeof(int64_t) * std::max<int64_t>(n, 1));
    CF_CUDA(cudaMemcpy(dp.p, indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    if (nnz) {
        CF_CUDA(cudaMemcpy(di.p, indices, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice));
        CF_CUDA(cudaMemcpy(dd.p, data, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
    if (n) CF_CUDA(cudaMemcpy(dm.p, map, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    // fill triples of the eliminated nodes
    int64_t fill = 0;
    DBuf dfn, doff;
    if (nf > 0) {
        std::vector<int64_t> off((size_t)nf);
        for (int64_t w = 0; w < nf; ++w) {
            const int64_t f = fnodes[w];
            const int64_t d = indptr[f + 1] - indptr[f] - 1;
            off[(size_t)w] = fill;
            fill += d > 1 ? d * (d - 1) : 0;
        }
        dfn.alloc(sizeof(int64_t) * nf);
        doff.alloc(sizeof(int64_t) * nf);
        CF_CUDA(cudaMemcpy(dfn.p, fnodes, sizeof(int64_t) * nf, cudaMemcpyHostToDevice));
        CF_CUDA(cudaMemcpy(doff.p, off.data(), sizeof(int64_t) * nf, cudaMemcpyHostToDevice));
    }
    const int64_t cnt = nnz + fill;
    DBuf key(sizeof(uint64_t) * std::max<int64_t>(cnt, 1)), val(sizeof(double) * std::max<int64_t>(cnt, 1));
    if (nnz)
        k_galerkin_keys<<<blocks_for(nnz), kT>>>(n, nnz, dp.as<int64_t>(), di.as<int64_t>(),
                                                 dd.as<double>(), dm.as<int64_t>(), nc,
                                                 key.as<uint64_t>(), val.as<double>());
    if (fill)
        k_schur_fill<<<blocks_for(nf * 32), kT>>>(nf, dfn.as<int64_t>(), dp.as<int64_t>(),
                                                  di.as<int64_t>(), dd.as<double>(),
                                                  dm.as<int64_t>(), nc, doff.as<int64_t>(),
                                                  key.as<uint64_t>() + nnz, val.as<double>() + nnz);
    CF_CUDA(cudaGetLastError());
    CF_CUDA(cudaDeviceSynchronize());
    dp.release();
    di.release();
    dd.release();
    dm.release();
    finish_coarse(device, nc, cnt, key, val);
    *nnz_out = g_ctx.nnz;
    CF_API_END
}

// Copy out the coarse Laplacian computed by the last cf_coarse_operator_dev
// call of this thread (out_ptr: nc + 1; out_idx / out_val: *nnz_out entries)
// and release its device buffers.
extern "C" int cf_coarse_fetch_dev(int64_t* out_ptr, int64_t* out_idx, double* out_val) {
    CF_API_BEGIN
    CoarseCtx& c = g_ctx;
    if (c.device < 0) throw CfError(CF_DOMAIN, "no coarse operator pending");
    CF_CUDA(cudaSetDevice(c.device));
    CF_CUDA(cudaMemcpy(out_ptr, c.optr.p, sizeof(int64_t) * (c.nc + 1), cudaMemcpyDeviceToHost));
    if (c.nnz) {
        CF_CUDA(cudaMemcpy(out_idx, c.oidx.p, sizeof(int64_t) * c.nnz, cudaMemcpyDeviceToHost));
        CF_CUDA(cudaMemcpy(out_val, c.oval.p, sizeof(double) * c.nnz, cudaMemcpyDeviceToHost));
    }
    c.optr.release();
    c.oidx.release();
    c.oval.release();
    c.device = -1;
    CF_API_END
}
