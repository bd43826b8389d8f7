// Device-resident multigrid hierarchy and the batched solve driver (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdio>

#include <map>
#include <mutex>
#include <vector>

#include "cfcent_b200.h"

namespace cf {

// Heavy-row plan of one CSR operator (see cf_kernels.cuh): heavy rows of each
// colour class are numbered contiguously so one class's segments form a range.
struct Plan {
    int64_t nheavy = 0, nseg = 0, heavy_nnz = 0;
    int32_t* hv = nullptr;
    int64_t* hsp = nullptr;
    int64_t* sbeg = nullptr;
    int64_t* send = nullptr;
    std::vector<int64_t> cseg;  // class c -> segments [cseg[c], cseg[c+1])
    std::vector<int64_t> cheavy;  // class c -> entries in its heavy rows
    // distinct neighbour rows gathered by the heavy rows of: class c / the merged
    // Jacobi classes / the whole plan (compulsory X reads of a k_seg launch)
    std::vector<int64_t> cnbr;
    int64_t merged_nbr = 0, all_nbr = 0;
    int32_t* seg_hv = nullptr;  // segment -> heavy index
    int32_t* h_row = nullptr;   // heavy index -> row
    int32_t* h_pos = nullptr;   // heavy index -> position in class order
    int* cntr = nullptr;        // arrival counters (zero between launches)
    // Processing order of the segments (scheduling only; partials are still
    // indexed and summed by segment id): segments sorted by the column window
    // of their first entry, so the warps in flight gather from one L2-sized
    // window of X.  sord_cls: sorted inside every sweep launch range (each
    // Gauss-Seidel class, then the merged Jacobi classes as one range);
    // sord_all: sorted over the whole plan (k_seg launches).  nullptr: id order.
    int32_t* sord_cls = nullptr;
    int32_t* sord_all = nullptr;
    // bounded first sweeps (x = 0 above the class's first row): per heavy row
    // the leading segments with a column below that bound (hlo), and their
    // window-sorted order per launch range (sord_lo, ranges cseg_lo)
    int32_t* hlo = nullptr;
    int32_t* sord_lo = nullptr;
    std::vector<int64_t> cseg_lo;  // launch range r -> [cseg_lo[r], cseg_lo[r+1]) in sord_lo
    int64_t nwin_seg = 0;       // segments cut at column-window boundaries
};

struct DLevel {
    int kind = 0, n = 0, nc = 0, nf = 0, ncolors = 0;
    int64_t nnz = 0;
    int64_t* rp = nullptr;
    int32_t* col = nullptr;
    double* val = nullptr;
    double* diag = nullptr;
    std::vector<int32_t> cptr;  // host copy of colour offsets
    int32_t* crows = nullptr;
    bool contig = false;  // colour classes are contiguous row ranges (crows == identity)
    int32_t *agg = nullptr, *aptr = nullptr, *amem = nullptr;
    // aggregate pieces (restriction work items of <= kAggPiece members; an
    // aggregate with more members is split, its pieces combined in order)
    int64_t npieces = 0, nmulti = 0;  // pieces; pieces of split aggregates
    int32_t *pa = nullptr, *pb = nullptr, *pslot = nullptr;
    int* acnt = nullptr;  // split aggregate -> arrivals (zero between launches)
    int32_t *fn = nullptr, *cn = nullptr;
    int32_t* cagg = nullptr;  // aggregation: agg[col[p]] per off-diagonal entry
    int32_t* wcm = nullptr;   // elimination: fn[wcc[p]] per W_cf entry
    double* wcd = nullptr;    // elimination: fd[wcc[p]] per W_cf entry
    double* fd = nullptr;
    int64_t* wcp = nullptr;
    int32_t* wcc = nullptr;
    double* wcv = nullptr;
    int64_t* wfp = nullptr;
    int32_t* wfc = nullptr;
    double* wfv = nullptr;
    double* M = nullptr;
    // workspace, n x kc_ws row-major (level 0 uses Hier::R / Hier::C)
    double* b = nullptr;
    double* x = nullptr;
    double* ls = nullptr;  // 2 x 256 line-search sums
    // per colour class (host, for the algorithmic-bytes model): rows, nnz,
    // distinct neighbour rows
    std::vector<int64_t> c_rows, c_nnz, c_nbr, c_nnz_lo, c_nbr_lo;
    int64_t merged_nbr = 0;  // distinct neighbour rows of the merged Jacobi classes
    int64_t merged_nbr_lo = 0, merged_nnz_lo = 0;
    // the same counts over the light rows only (<= kHeavyNnz entries): what a
    // sweep kernel gathers itself when the heavy rows' segments run in k_seg
    std::vector<int64_t> c_nbr_light;
    int64_t merged_nbr_light = 0;
    int64_t w_nnz = 0;  // elimination: nnz(W_cf)
    int gs_classes = 0;  // colour classes swept one by one (<= kGsClasses)
    bool merged = false; // classes >= kGsClasses merged into one Jacobi step
    Plan pm;  // matrix rows (level 0 / aggregation levels)
    Plan pw;  // W_cf rows (elimination levels)
};

// Per-launch profiling (CUDA events around every launch; cycles run eagerly).
struct ProfRec {
    const char* kind;
    int level;
    double bytes;   // compulsory (algorithmic) HBM bytes
    double gbytes;  // neighbour-row gather volume (nnz * 8 * KC), served by L2/HBM
    cudaEvent_t a, b;
};

// Multicolour GS sweeps the first kGsClasses colour classes one by one; the
// remaining (small, hub-heavy) classes form one Jacobi step.
constexpr int kGsClasses = 2;

// Supported block widths (columns per device chunk).
constexpr int kMaxKC = 256;
int pick_kc(int64_t remaining);
int plan_max_kc(int64_t total);

struct Hier {
    int dev = 0;
    cudaStream_t s = nullptr;
    std::vector<DLevel> L;
    std::mutex mu;
    int kc_ws = 0;  // workspace width currently allocated
    int n0 = 0;
    int32_t* perm0 = nullptr;  // device row i holds node perm0[i] (nullptr: identity)
    // level-0 block buffers, n0 x kc_ws
    double *B = nullptr, *X = nullptr, *R = nullptr, *C = nullptr;
    // fallback buffers (lazily allocated)
    double *Z = nullptr, *P = nullptr, *AP = nullptr;
    int kc_fb = 0;
    double* parts = nullptr;
    size_t parts_cap = 0;  // doubles
    double* SP = nullptr;  // heavy-row segment partials, max_nseg x kc_ws
    double* PP = nullptr;  // aggregate-piece partials, max_multi x kc_ws
    int64_t max_multi = 0;
    double* fin = nullptr; // fused-reduction segment scratch (2 regions)
    size_t fin_region = 0;
    unsigned* cnt = nullptr;  // fused-reduction arrival counters (2 regions + 2 globals)
    size_t cnt_region = 0;
    double* DP = nullptr;  // dense coarse apply: per-chunk partials
    double* T = nullptr;   // merged-class Jacobi staging, max_merged x kc_ws
    int64_t max_merged = 0;
    int64_t max_nseg = 0;
    double* sums = nullptr;  // 8 x kMaxKC
    double* coef = nullptr;  // 4 x kMaxKC
    double *bn = nullptr, *res = nullptr, *prev = nullptr;
    int *stall = nullptr, *state = nullptr, *count = nullptr;
    int* h_count = nullptr;     // pinned
    double* h_small = nullptr;  // pinned, 16 x kMaxKC
    double* S = nullptr;        // staging for rows layout (kc_ws x n0)
    std::vector<void*> owned;   // operator allocations
    int64_t bytes = 0;
    std::map<int, cudaGraphExec_t> cycle_graphs;  // per KC
    std::map<int, cudaGraphExec_t> loop_graphs;   // whole outer iteration (while node)
    int *d_iter = nullptr, *d_ncyc = nullptr;
    double* d_lp = nullptr;  // solve-loop parameters read by the status kernel (6)
    long long* d_vcyc = nullptr;
    bool prof = false;
    bool host_loop = false;  // CF_HOST_LOOP=1
    // power-law graph (level-0 maximum degree > 64 x mean on > 262,144 nodes):
    // the solve runs the v_hub build of the kernels (cf_solve_hub.cu)
    bool hub_profile = false;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    int prof_begin(const char* kind, int level, double bytes, double gbytes);
    void prof_end(int idx);

    // multi-block pinned transfers overlapped with the solve (cf_solve_rows):
    // copy stream, double-buffered rows-layout staging in/out, n0 x pipe_kc
    cudaStream_t cs = nullptr;
    double* pin[2] = {nullptr, nullptr};
    double* pout[2] = {nullptr, nullptr};
    int pipe_kc = 0;
    cudaEvent_t ev_in[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_done[2] = {};
    void ensure_pipe(int kc);

    void* stage_host = nullptr;       // pinned staging ring for pageable transfers
    cudaEvent_t stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};
    void ensure_stage();

    ~Hier();
    void* dalloc(size_t bytes_);
    void ensure_workspace(int kc);
    void ensure_fallback(int kc);
};

// In profile mode each scope is also an NVTX range "cf:<kind>@L<level>", so an
// ncu capture can select one (kind, level) instance:
//   ncu --nvtx --nvtx-include "regex:cf:jacobi_merged@L1/" ...
struct ProfScope {
    Hier& h;
    int idx = -1;
    ProfScope(Hier& h_, const char* kind, int level, double bytes, double gbytes = 0.0) : h(h_) {
        if (h.prof) {
            idx = h.prof_begin(kind, level, bytes, gbytes);
            char name[64];
            std::snprintf(name, sizeof(name), "cf:%s@L%d", kind, level);
            nvtxRangePushA(name);
        }
    }
    ~ProfScope() {
        if (idx >= 0) {
            h.prof_end(idx);
            nvtxRangePop();
        }
    }
};

// Solve a device block B (n0 x kc row-major, already in h.B) into h.X.
// bnorm/state of columns are derived from h.B.  res_out: kc residuals (host).
void solve_block(Hier& h, int kc, int ncols, const CfSolveParams& p, double* res_out,
                 CfSolveStats& st);
// Transposes between rows layout (cnt x n) and block layout (n x kc).
void rows_to_block(Hier& h, const double* S_dev, int cnt, int kc, double* B_dev);
void block_to_rows(Hier& h, const double* B_dev, int cnt, int kc, double* S_dev);
// pageable host <-> device copies through the pinned staging ring (sync-free
// issue on h.s; d2h returns when the host buffer is filled)
void h2d_staged(Hier& h, void* dst_dev, const void* src_host, size_t bytes);
void d2h_staged(Hier& h, void* dst_host, const void* src_dev, size_t bytes);
// Column sums over level-0 n x kc block -> h.sums (device), one quantity.
void colsum_dev(Hier& h, const double* X_dev, int kc, double* out_dev);
// fused-reduction control (region 0) for kernels outside cf_solve.cu
struct RedCtl;
RedCtl redctl_dev(Hier& h, double* parts, int64_t np, double* out);

}  // namespace cf
