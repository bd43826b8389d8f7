// Micro-benchmark: random row gathers of a row-major fp64 block (rows of KC
// doubles) -- register LDG.256 with G rows in flight per warp vs. TMA bulk
// copies (cp.async.bulk + mbarrier) into a per-warp shared-memory ring of R
// rows.  Measures the ceiling of the solve kernels' neighbour gathers for an
// L2-resident and an HBM-resident block.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int KC = 128;
constexpr int V = KC / 32;

template <int G>
__global__ void __launch_bounds__(256) k_ldg(const double* __restrict__ X, const int* __restrict__ idx,
                                             int64_t per_warp, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * 256 + threadIdx.x) >> 5;
    const int* id = idx + w * per_warp;
    double acc[V] = {};
    for (int64_t p0 = 0; p0 < per_warp; p0 += 32) {
        int jj = id[p0 + lane];
        for (int u0 = 0; u0 < 32; u0 += G) {
            double x[G][V];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                int j = __shfl_sync(0xffffffffu, jj, u0 + u);
                const double* p = X + (size_t)j * KC + lane * V;
                asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x[u][0]), "=d"(x[u][1]), "=d"(x[u][2]), "=d"(x[u][3]) : "l"(p));
            }
#pragma unroll
            for (int u = 0; u < G; ++u)
#pragma unroll
                for (int t = 0; t < V; ++t) acc[t] += x[u][t];
        }
    }
    double s = 0; for (int t = 0; t < V; ++t) s += acc[t];
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_tma(const double* __restrict__ X, const int* __restrict__ idx,
                                                  int64_t per_warp, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* ring = reinterpret_cast<double*>(sm) + (size_t)wid * R * KC;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)WPB * R * KC * 8) + wid * R;
    const int64_t w = (int64_t)blockIdx.x * WPB + wid;
    const int* id = idx + w * per_warp;
    if (lane < R) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + lane)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    auto issue = [&](int64_t p) {  // lane-0 issues row idx[p] into slot p % R
        int s = (int)(p % R);
        int j = id[p];
        uint32_t b = smem_u32(bar + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(KC * 8) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(ring + (size_t)s * KC)), "l"(X + (size_t)j * KC), "r"(KC * 8), "r"(b) : "memory");
    };
    if (lane == 0)
        for (int64_t p = 0; p < R && p < per_warp; ++p) issue(p);
    double acc[V] = {};
    for (int64_t p = 0; p < per_warp; ++p) {
        const int s = (int)(p % R);
        const uint32_t par = (uint32_t)((p / R) & 1);
        uint32_t b = smem_u32(bar + s);
        asm volatile("{\n.reg .pred P;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra WAIT_%=;\n}" ::"r"(b), "r"(par) : "memory");
        const double* q = ring + (size_t)s * KC + lane * V;
        double4 v = *reinterpret_cast<const double4*>(q);
        acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
        __syncwarp();
        if (lane == 0 && p + R < per_warp) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(p + R);
        }
    }
    double s = 0; for (int t = 0; t < V; ++t) s += acc[t];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int64_t total = 1 << 24;  // gathers per launch (16M rows = 16 GB of row traffic)
    int* idx; CK(cudaMalloc(&idx, total * 4));
    double* out; CK(cudaMalloc(&out, 8));
    const size_t maxrows = (size_t)4 << 20;  // 4 GB block
    double* X; CK(cudaMalloc(&X, maxrows * KC * 8));
    CK(cudaMemset(X, 0, maxrows * KC * 8));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (size_t rows : {8192ul, 32768ul, 65536ul, 100000ul, 1ul << 22}) {
        std::vector<int> h(total);
        uint64_t st = 0x9e3779b97f4a7c15ull ^ rows;
        for (auto& v : h) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; v = (int)(st % rows); }
        CK(cudaMemcpy(idx, h.data(), total * 4, cudaMemcpyHostToDevice));
        auto run = [&](const char* name, auto launch) {
            launch(); CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) launch();
            cudaEventRecord(b); CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
            printf("rows=%8zu (%6.1f MB) %-22s %8.3f ms  %7.0f GB/s\n", rows, rows * KC * 8 / 1e6, name, ms,
                   total * KC * 8.0 / ms / 1e6);
        };
        const int64_t warps = 148 * 64;  // 64 warps per SM worth
        const int64_t pw = total / warps / 32 * 32;
        run("ldg G=4", [&] { k_ldg<4><<<warps / 8, 256>>>(X, idx, pw, out); });
        run("ldg G=8", [&] { k_ldg<8><<<warps / 8, 256>>>(X, idx, pw, out); });
        {
            constexpr int R = 8, WPB = 8;
            size_t sm = (size_t)WPB * R * KC * 8 + WPB * R * 8;
            CK(cudaFuncSetAttribute(k_tma<R, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            run("tma R=8 wpb=8", [&] { k_tma<R, WPB><<<warps / WPB, WPB * 32, sm>>>(X, idx, pw, out); });
        }
        {
            constexpr int R = 16, WPB = 8;
            size_t sm = (size_t)WPB * R * KC * 8 + WPB * R * 8;
            CK(cudaFuncSetAttribute(k_tma<R, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            run("tma R=16 wpb=8", [&] { k_tma<R, WPB><<<warps / WPB, WPB * 32, sm>>>(X, idx, pw, out); });
        }
        {
            constexpr int R = 24, WPB = 8;
            size_t sm = (size_t)WPB * R * KC * 8 + WPB * R * 8;
            CK(cudaFuncSetAttribute(k_tma<R, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            run("tma R=24 wpb=8", [&] { k_tma<R, WPB><<<warps / WPB, WPB * 32, sm>>>(X, idx, pw, out); });
        }
        {
            constexpr int R = 6, WPB = 16;
            size_t sm = (size_t)WPB * R * KC * 8 + WPB * R * 8;
            CK(cudaFuncSetAttribute(k_tma<R, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            run("tma R=6 wpb=16", [&] { k_tma<R, WPB><<<warps / WPB, WPB * 32, sm>>>(X, idx, pw, out); });
        }
    }
    return 0;
}
