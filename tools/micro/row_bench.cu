// Micro-benchmark of the solve kernels' CSR row gather (cf_kernels.cuh):
// Y_i = sum_j a_ij X_j over a random CSR with uniform degree D, X row-major
// n x KC fp64.  Variants: warp per row (gather_row) and tiled row pipelines
// with RPW rows per warp (row_pipeline), at 2 / 3 / 4 CTAs per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1607_02955_b200/csrc \
//        -I../../include -o row_bench row_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <stdexcept>
#include "cf_kernels.cuh"
using namespace cf;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
constexpr int KC = 128;
constexpr int V = KC / 32;

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_row(int n, const int64_t* rp, const int32_t* col, const double* val,
                                                   const double* X, double* Y) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= n) return;
    DV<V> acc; zero(acc);
    gather_row<KC, G_PLAIN>(col, val, rp[i], rp[i + 1], nullptr, nullptr, X, lane * V, acc);
    stv<V>(Y + i * KC + lane * V, acc);
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_tile(int n, int rpw, const int64_t* rp, const int32_t* col,
                                                    const double* val, const double* X, double* Y) {
    const int lane = threadIdx.x & 31, slot = threadIdx.x >> 5;
    const int64_t g0 = (int64_t)blockIdx.x * 8 * rpw;
    const int c0 = lane * V;
    row_pipeline<KC, G_PLAIN>(g0 + slot, 8, min((int64_t)n, g0 + 8 * rpw), [](int64_t t) { return t; },
        rp, col, val, nullptr, nullptr,
        [&](int64_t, int64_t i, int64_t beg, int64_t end, int jj, double aa, double dd) {
            DV<V> acc; zero(acc);
            gather_row_from<KC, G_PLAIN>(col, val, beg, end, nullptr, nullptr, X, c0, acc, jj, aa, dd);
            stv<V>(Y + i * KC + c0, acc);
        });
}

int main(int argc, char** argv) {
    for (int n : {18000, 66000, 100000, 1000000}) for (int D : {8, 16, 64}) {
        if ((int64_t)n * D > 64000000) continue;
        std::vector<int64_t> rp(n + 1);
        std::vector<int32_t> col((size_t)n * D);
        std::vector<double> val((size_t)n * D, 0.5);
        uint64_t st = 88172645463325252ull + n + D;
        for (int i = 0; i <= n; ++i) rp[i] = (int64_t)i * D;
        for (auto& c : col) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; c = (int32_t)(st % n); }
        int64_t *drp; int32_t* dcol; double *dval, *X, *Y;
        CK(cudaMalloc(&drp, 8 * (n + 1))); CK(cudaMalloc(&dcol, 4 * col.size())); CK(cudaMalloc(&dval, 8 * val.size()));
        CK(cudaMalloc(&X, 8ull * n * KC)); CK(cudaMalloc(&Y, 8ull * n * KC));
        CK(cudaMemcpy(drp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dcol, col.data(), 4 * col.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dval, val.data(), 8 * val.size(), cudaMemcpyHostToDevice));
        CK(cudaMemset(X, 0, 8ull * n * KC));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        auto run = [&](const char* name, auto launch) {
            for (int w = 0; w < 3; ++w) launch();
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int r = 0; r < 20; ++r) launch();
            cudaEventRecord(b); CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
            double gb = (double)n * D * KC * 8;
            printf("n=%7d D=%3d X=%6.1fMB %-16s %8.1f us  gather %7.0f GB/s\n", n, D, n * KC * 8 / 1e6, name,
                   ms * 1e3, gb / ms / 1e6);
        };
        run("row minb3", [&] { k_row<3><<<(n + 7) / 8, 256>>>(n, drp, dcol, dval, X, Y); });
        run("row minb4", [&] { k_row<4><<<(n + 7) / 8, 256>>>(n, drp, dcol, dval, X, Y); });
        for (int rpw : {2, 4, 8}) {
            char nm[32];
            snprintf(nm, 32, "tile%d minb3", rpw);
            run(nm, [&] { k_tile<3><<<(n + 8 * rpw - 1) / (8 * rpw), 256>>>(n, rpw, drp, dcol, dval, X, Y); });
            snprintf(nm, 32, "tile%d minb2", rpw);
            run(nm, [&] { k_tile<2><<<(n + 8 * rpw - 1) / (8 * rpw), 256>>>(n, rpw, drp, dcol, dval, X, Y); });
        }
        cudaFree(drp); cudaFree(dcol); cudaFree(dval); cudaFree(X); cudaFree(Y);
    }
    return 0;
}
