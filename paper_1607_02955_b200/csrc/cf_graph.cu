// Device-side graph ingestion: the sort / merge of
// Graph.from_edges (reference graph.py:100-147) and the connected-component
// labelling behind largest_connected_component (graph.py:217-250), for edge
// lists large enough that the host O(m log m) passes dominate (R-MAT scale 22:
// 97 M adjacency entries).
//
// Integer / byte work throughout: results are exactly the host path's
// (paper_1607_02955_b200/graph.py, csrc/cf_setup.cpp cf_build_csr) -- same
// indptr, same sorted neighbour lists, same weights.  Duplicate edges are
// only DETECTED here (their weights would have to be summed in numpy's
// reduceat order to stay bit-identical with the reference); the caller then
// takes the host route, as the native host path already does.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "cf_common.h"
#include "cfcent_b200.h"

namespace cf {
namespace {

struct DBuf {
    void* p = nullptr;
    DBuf() = default;
    explicit DBuf(size_t bytes) { alloc(bytes); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t bytes) {
        if (p) cudaFree(p);
        p = nullptr;
        CF_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    }
    template <typename T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

constexpr int kT = 256;
inline unsigned blocks_for(int64_t items) { return (unsigned)std::max<int64_t>(1, (items + kT - 1) / kT); }

// Adjacency entries in the order the reference concatenates them
// (graph.py:133-135): entry e < m is (u_e -> v_e), entry m + e is (v_e -> u_e).
// key = src * n + dst; the radix sort is stable, so equal keys keep this order.
__global__ void __launch_bounds__(kT) k_edge_keys(int64_t m, int64_t n,
                                                  const int64_t* __restrict__ u,
                                                  const int64_t* __restrict__ v,
                                                  const double* __restrict__ w,
                                                  uint64_t* __restrict__ key,
                                                  double* __restrict__ val, int* __restrict__ bad) {
    const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (t >= 2 * m) return;
    const int64_t e = t < m ? t : t - m;
    const int64_t a = u[e], b = v[e];
    if (a < 0 || b < 0 || a >= n || b >= n || a == b) atomicExch(bad, 1);
    const int64_t s = t < m ? a : b, d = t < m ? b : a;
    key[t] = (uint64_t)s * (uint64_t)n + (uint64_t)d;
    val[t] = w[e];
}

// dup = 1 if any two consecutive sorted keys are equal
__global__ void __launch_bounds__(kT) k_any_duplicate(int64_t cnt, const uint64_t* __restrict__ key,
                                                      int* __restrict__ dup) {
    const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (t == 0 || t >= cnt) return;
    if (key[t] == key[t - 1]) atomicExch(dup, 1);
}

// indptr[i] = first sorted entry with src >= i (binary search); dst = key % n
__global__ void __launch_bounds__(kT) k_row_ptr(int64_t n, int64_t cnt,
                                                const uint64_t* __restrict__ key,
                                                int64_t* __restrict__ indptr) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i > n) return;
    const uint64_t target = (uint64_t)i * (uint64_t)n;
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] < target)
            lo = mid + 1;
        else
            hi = mid;
    }
    indptr[i] = lo;
}
__global__ void __launch_bounds__(kT) k_key_to_dst(int64_t cnt, int64_t n,
                                                   const uint64_t* __restrict__ key,
                                                   int64_t* __restrict__ dst) {
    const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (t < cnt) dst[t] = (int64_t)(key[t] % (uint64_t)n);
}

// ---- connected components: min-id hooking + full pointer jumping ------------
// parent[] holds roots at the start of every round (stars after k_cc_jump).
// Hooking the larger root under the smaller with atomicMin makes the final
// root of a component its smallest node id whatever the interleaving, so the
// labelling is deterministic.
__global__ void __launch_bounds__(kT) k_cc_init(int64_t n, int32_t* __restrict__ parent) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i < n) parent[i] = (int32_t)i;
}
__global__ void __launch_bounds__(kT) k_cc_hook(int64_t m, const int64_t* __restrict__ eu,
                                                const int64_t* __restrict__ ev,
                                                int32_t* __restrict__ parent,
                                                int* __restrict__ changed) {
    const int64_t e = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (e >= m) return;
    const int32_t a = parent[eu[e]], b = parent[ev[e]];
    if (a == b) return;
    const int32_t hi = a > b ? a : b, lo = a > b ? b : a;
    atomicMin(parent + hi, lo);
    *changed = 1;
}
__global__ void __launch_bounds__(kT) k_cc_jump(int64_t n, int32_t* __restrict__ parent) {
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
__global__ void __launch_bounds__(kT) k_widen(int64_t n, const int32_t* __restrict__ src,
                                              int64_t* __restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

int bits_for(uint64_t max_value) {
    int b = 1;
    while (b < 64 && (max_value >> b)) ++b;
    return b;
}

}  // namespace
}  // namespace cf

using namespace cf;

// Graph.from_edges core on the device (graph.py:133-146).  Same contract as
// cf_build_csr; *status = 0 ok, 1 duplicate edges present (nothing written:
// take the host route so the summed weights keep numpy's order), 2 an edge is
// a self-loop or out of range.
extern "C" int cf_csr_from_edges_dev(int32_t device, int64_t n, int64_t m, const int64_t* u,
                                     const int64_t* v, const double* w, int64_t* indptr,
                                     int64_t* indices, double* weights, int32_t* status) {
    CF_API_BEGIN
    *status = 0;
    if (n < 0 || m < 0) throw CfError(CF_DOMAIN, "negative sizes");
    if (2 * m >= (int64_t)1 << 31) throw CfError(CF_RUNTIME, "edge list too long for one device sort");
    if (n > 0 && (uint64_t)n > ((uint64_t)1 << 31)) throw CfError(CF_RUNTIME, "too many nodes");
    CF_CUDA(cudaSetDevice(device));
    const int64_t cnt = 2 * m;
    if (cnt == 0) {
        for (int64_t i = 0; i <= n; ++i) indptr[i] = 0;
        return CF_OK;
    }
    DBuf du(sizeof(int64_t) * m), dv(sizeof(int64_t) * m), dw(sizeof(double) * m);
    CF_CUDA(cudaMemcpy(du.p, u, sizeof(int64_t) * m, cudaMemcpyHostToDevice));
    CF_CUDA(cudaMemcpy(dv.p, v, sizeof(int64_t) * m, cudaMemcpyHostToDevice));
    CF_CUDA(cudaMemcpy(dw.p, w, sizeof(double) * m, cudaMemcpyHostToDevice));
    DBuf k0(sizeof(uint64_t) * cnt), k1(sizeof(uint64_t) * cnt);
    DBuf v0(sizeof(double) * cnt), v1(sizeof(double) * cnt), flag(sizeof(int) * 2);
    CF_CUDA(cudaMemset(flag.p, 0, sizeof(int) * 2));
    k_edge_keys<<<blocks_for(cnt), kT>>>(m, n, du.as<int64_t>(), dv.as<int64_t>(), dw.as<double>(),
                                         k0.as<uint64_t>(), v0.as<double>(), flag.as<int>());
    CF_CUDA(cudaGetLastError());
    const int end_bit = std::min(64, bits_for((uint64_t)n * (uint64_t)n));
    size_t tb = 0;
    CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                            v0.as<double>(), v1.as<double>(), (int)cnt, 0, end_bit));
    DBuf tmp(tb);
    CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                            v0.as<double>(), v1.as<double>(), (int)cnt, 0, end_bit));
    k_any_duplicate<<<blocks_for(cnt), kT>>>(cnt, k1.as<uint64_t>(), flag.as<int>() + 1);
    CF_CUDA(cudaGetLastError());
    int hf[2] = {0, 0};
    CF_CUDA(cudaMemcpy(hf, flag.p, sizeof(hf), cudaMemcpyDeviceToHost));
    if (hf[0]) {
        *status = 2;
        return CF_OK;
    }
    if (hf[1]) {
        *status = 1;
        return CF_OK;
    }
    // reuse the unsorted buffers for the outputs
    int64_t* d_ptr = du.as<int64_t>();
    DBuf dptr;
    if (n + 1 > m) {
        dptr.alloc(sizeof(int64_t) * (n + 1));
        d_ptr = dptr.as<int64_t>();
    }
    k_row_ptr<<<blocks_for(n + 1), kT>>>(n, cnt, k1.as<uint64_t>(), d_ptr);
    k_key_to_dst<<<blocks_for(cnt), kT>>>(cnt, n, k1.as<uint64_t>(),
                                          reinterpret_cast<int64_t*>(k0.p));
    CF_CUDA(cudaGetLastError());
    CF_CUDA(cudaMemcpy(indptr, d_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    CF_CUDA(cudaMemcpy(indices, k0.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost));
    CF_CUDA(cudaMemcpy(weights, v1.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    CF_API_END
}

// Component root of every node (the smallest node id of its component) for
// the undirected graph with edges (eu[e], ev[e]); graph.py:217-250 derives the
// largest component from these labels (ordering the roots ascending gives
// scipy's first-occurrence component numbering).
extern "C" int cf_components_dev(int32_t device, int64_t n, int64_t m, const int64_t* eu,
                                 const int64_t* ev, int64_t* root, int32_t* rounds) {
    CF_API_BEGIN
    if (n < 0 || m < 0) throw CfError(CF_DOMAIN, "negative sizes");
    if ((uint64_t)n >= ((uint64_t)1 << 31)) throw CfError(CF_RUNTIME, "too many nodes");
    if (n == 0) return CF_OK;
    CF_CUDA(cudaSetDevice(device));
    DBuf du(sizeof(int64_t) * m), dv(sizeof(int64_t) * m), par(sizeof(int32_t) * n), chg(sizeof(int));
    DBuf wide(sizeof(int64_t) * n);
    if (m) {
        CF_CUDA(cudaMemcpy(du.p, eu, sizeof(int64_t) * m, cudaMemcpyHostToDevice));
        CF_CUDA(cudaMemcpy(dv.p, ev, sizeof(int64_t) * m, cudaMemcpyHostToDevice));
    }
    k_cc_init<<<blocks_for(n), kT>>>(n, par.as<int32_t>());
    int r = 0;
    for (; m > 0 && r < 4096; ++r) {
        CF_CUDA(cudaMemset(chg.p, 0, sizeof(int)));
        k_cc_hook<<<blocks_for(m), kT>>>(m, du.as<int64_t>(), dv.as<int64_t>(), par.as<int32_t>(),
                                         chg.as<int>());
        k_cc_jump<<<blocks_for(n), kT>>>(n, par.as<int32_t>());
        int h = 0;
        CF_CUDA(cudaMemcpy(&h, chg.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (!h) break;
    }
    if (rounds) *rounds = r;
    k_widen<<<blocks_for(n), kT>>>(n, par.as<int32_t>(), wide.as<int64_t>());
    CF_CUDA(cudaGetLastError());
    CF_CUDA(cudaMemcpy(root, wide.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    CF_API_END
}
