/*
 * cfcent_b200 -- C-ABI of the B200-native multi-RHS Laplacian multigrid path.
 *
 * The reference (cfcent 0.1.0, pure Python) has no FFI; its boundary is the
 * Python API of pkg/src/cfcent.  Each entry point below
 * replaces one reference call site and is bound from the Python mirror
 * (paper_1607_02955_b200/_native.py) with ctypes; INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / numpy types.
 *  - host pointers unless the name ends in _dev.
 *  - row-major blocks: a block of k right-hand sides over n nodes stored as
 *    X[i * k + j] (node i, column j) is called "n x k row-major".
 *  - "rows" layout (the reference's supplies / PotentialVector layout): one
 *    right-hand side per row, S[r * n + i].
 *  - every function returns a status: CF_OK, CF_DOMAIN (maps to DomainError),
 *    CF_CONVERGENCE (maps to ConvergenceError, *best_residual filled),
 *    CF_RUNTIME (CUDA / allocation failure).  cf_last_error() gives the message
 *    of the last failure on the calling thread.
 *  - handles are re-entrant: concurrent calls on one hierarchy serialise on a
 *    per-handle lock (reference contract SPEC.md:196).
 */
#ifndef CFCENT_B200_H
#define CFCENT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CF_OK = 0, CF_DOMAIN = 1, CF_CONVERGENCE = 2, CF_RUNTIME = 3 };
enum { CF_LEVEL_ELIMINATION = 0, CF_LEVEL_AGGREGATION = 1, CF_LEVEL_COARSEST = 2 };

/* One hierarchy level in host memory (copied to the device by
 * cf_hier_create).  Replaces solver.py:97-120 `Level`.
 * Matrix: off-diagonal CSR (int32 column, fp64 value = L_ij < 0) plus the
 * diagonal split out; required for level 0 and aggregation levels. */
typedef struct {
    int32_t kind;            /* CF_LEVEL_* */
    int32_t n;               /* rows at this level */
    int32_t n_coarse;        /* rows at the next level (0 for coarsest) */
    int64_t nnz_off;         /* off-diagonal entries (0 if no matrix) */
    const int64_t* rowptr;   /* n+1, offsets into col/val (NULL if no matrix) */
    const int32_t* col;
    const double* val;
    const double* diag;      /* n */
    /* aggregation (solver.py:110-114): colouring and aggregate map */
    int32_t n_colors;
    const int32_t* color_ptr;    /* n_colors+1 */
    const int32_t* color_rows;   /* n, rows grouped by colour, ascending */
    const int32_t* agg;          /* n, node -> aggregate */
    const int32_t* agg_ptr;      /* n_coarse+1 */
    const int32_t* agg_members;  /* n, members of each aggregate ascending */
    /* elimination (solver.py:104-108) */
    int32_t n_f;
    const int32_t* f_nodes;      /* n_f */
    const int32_t* c_nodes;      /* n_coarse */
    const double* f_degree;      /* n_f */
    const int64_t* wcf_ptr;      /* n_coarse+1; W_cf columns index f_nodes */
    const int32_t* wcf_col;
    const double* wcf_val;
    const int64_t* wfc_ptr;      /* n_f+1; W_fc = W_cf^T, columns index c_nodes */
    const int32_t* wfc_col;
    const double* wfc_val;
    /* coarsest (solver.py:115-116, 394-419): dense n x n operator
     * M = (I - 11^T/n) G^+ with G^+ the node-0-grounded inverse padded by a
     * zero row/column, so x = M b is the reference's direct solve. */
    const double* coarse_op;
} CfLevelDesc;

/* Solve parameters (SolverConfig, solver.py:61-74, plus module constants
 * solver.py:53-58). */
typedef struct {
    double tau;
    int32_t max_cycles;
    int32_t nu1, nu2;            /* smoothing_steps */
    int32_t fcg_max_iters;       /* FCG_MAX_ITERS = 200 */
    int32_t jpcg_max_iters;      /* max(2000, 50 sqrt(n)) */
    double stop_margin;          /* STOP_MARGIN = 0.9 */
    double stagnation_factor;    /* 0.9 */
    int32_t stagnation_cycles;   /* 5 */
} CfSolveParams;

/* Per-call statistics (SolveStats, solver.py:123-137). */
typedef struct {
    int64_t solves;              /* columns solved (nonzero and zero) */
    int64_t fallback_solves;     /* columns that entered FCG */
    int64_t vcycles;             /* V-cycle column-applications executed */
    int64_t outer_iterations;    /* block iterations executed */
    double max_residual;
    double best_residual;        /* on CF_CONVERGENCE: worst failing residual */
    int64_t krylov_solves;       /* columns continued under V-cycle-preconditioned FCG
                                    by the Krylov hand-off; NOT
                                    counted in fallback_solves, which keeps the
                                    reference meaning (solver.py:717-720) */
} CfSolveStats;

const char* cf_last_error(void);
int cf_device_count(void);
int cf_version(void);

/* --- hierarchy (replaces solver.py:422-523 `setup` output upload) ------ */
int cf_hier_create(int32_t n_levels, const CfLevelDesc* levels, int32_t device,
                   void** out_handle);
int cf_hier_destroy(void* handle);
/* Device node order: device row i of level 0 holds node perm[i] (a locality
 * ordering chosen at upload; level descriptors are given in that order).
 * All node-indexed host/device buffers of the API stay in node order; the
 * library permutes at the boundary.  Not calling it means identity. */
int cf_hier_set_order(void* handle, const int32_t* perm, int64_t n);
/* total device bytes owned by the hierarchy (operators + workspace) */
int64_t cf_hier_device_bytes(void* handle);

/* --- solves ------------------------------------------------------------- */
/* solver.py:771-811 `solve_many` (and :754 `solve` with count = 1):
 * supplies_rows (count x n, host) -> values_rows (count x n, host, centred)
 * and residuals (count).  Columns are processed in device chunks of up to
 * max_chunk columns; results never depend on chunking. */
int cf_solve_rows(void* handle, const double* supplies_rows, int64_t count,
                  const CfSolveParams* params, double* values_rows,
                  double* residuals, CfSolveStats* stats);

/* Same on device memory: B_dev, X_dev are n x k row-major (k <= 256).
 * caller_stream (a cudaStream_t, NULL = legacy default stream) is the stream
 * that produced B_dev: the library's stream waits on it (event) before reading
 * the inputs; outputs are complete when the call returns. */
int cf_solve_block_dev(void* handle, const double* B_dev, double* X_dev, int32_t k,
                       const CfSolveParams* params, double* residuals,
                       CfSolveStats* stats, void* caller_stream);

/* Exported for unit tests: R = B - L X and per-column sum(R^2) on level 0
 * (solver.py:694-695). Device pointers, n x k row-major; caller_stream as for
 * cf_solve_block_dev. */
int cf_residual_dev(void* handle, const double* B_dev, const double* X_dev, double* R_dev,
                    int32_t k, double* colsq_host, void* caller_stream);

/* --- estimators (resistance.py / centrality.py) ----------------------- */
/* Graph upload for the JL right-hand sides: adjacency (graph.py:30-98) with
 * per-entry canonical edge id (graph.py:78-86) and sqrt(w) per edge. */
int cf_graph_create(void* hier, int64_t n, int64_t m, const int64_t* adj_ptr,
                    const int32_t* adj_nbr, const int32_t* adj_edge,
                    const double* sqrt_w, void** out_graph);
int cf_graph_destroy(void* graph);

/* resistance.py:181-199: rows [row0, row0+k) of Q W^1/2 B for
 * Q = (default_rng(seed).integers(0,2,(K,m))*2-1)/sqrt(K), from the PCG64
 * state (state_hi/lo, inc_hi/lo) of a fresh default_rng(seed).
 * Output Y_rows (k x n host, UNcentred, bit-identical to the reference). */
int cf_jl_rhs_rows(void* graph, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                   uint64_t inc_lo, int64_t K, int64_t row0, int32_t k,
                   double* Y_rows);

/* Fused JL estimator (build_sketch + sketch_distance_sums,
 * resistance.py:161-237, centrality.py:140-166): generates Q on device,
 * forms and centres Y, solves, and reduces Z without downloading it.
 * out_sums[q] = sum_w ||z_v - z_w||^2 for query v = query[q].
 * If z_rows is not NULL, also returns Z (K x n host, the sketch's z). */
int cf_jl_sketch(void* graph, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                 uint64_t inc_lo, int64_t K, int64_t row0, int64_t n_rows, double inv_sqrt_k,
                 const int64_t* query, int64_t n_query, const CfSolveParams* params,
                 double* out_sums, double* row_parts, double* z_rows, double* residuals,
                 CfSolveStats* stats);
/* (cf_jl_sketch computes sketch rows [row0, row0 + n_rows) of the K-row
 * sketch; out_sums are the contributions of those rows.  If row_parts is not
 * NULL it receives, per row j, [T_j, C_j, Z[q_0, j], ..., Z[q_{nq-1}, j]]
 * (n_rows x (2 + n_query) host): ranks owning disjoint row ranges gather
 * their row parts and cf_jl_combine sums them in ascending row order, which
 * gives the same bits for every split -- SURVEY.md §8(e).) */
int cf_jl_combine(const double* row_parts, int64_t n_rows, int64_t n_query, int64_t n,
                  double* out_sums);

/* Amortised node solutions L z_x = e_x - 1/n (resistance.py:77-99) for the
 * given nodes, reduced on device to the |nodes| x |nodes| submatrix
 * sub[a * cnt + b] = z_{nodes[a]}[nodes[b]] (what resistances_from_node and
 * the sampling estimator read, resistance.py:124-129).  If z_rows is not
 * NULL the full solutions (cnt x n) are returned too. */
int cf_node_solutions(void* handle, const int64_t* nodes, int64_t cnt,
                      const CfSolveParams* params, double* sub, double* z_rows,
                      double* residuals, CfSolveStats* stats);

/* Exact current-flow closeness denominators (centrality.py:78-101): every node
 * is solved once (L z_t = e_t - 1/n, resistance.py:77-99) and, per query v
 * (device-order node ids), S_v = sum_t R(v, t) is accumulated on the device
 * without returning the n x n solutions.  max_residual (host, may be NULL)
 * receives the largest relative residual of the n solves. */
int cf_exact_sums(void* handle, const int64_t* query, int64_t n_query,
                  const CfSolveParams* params, double* out_sums, double* max_residual,
                  CfSolveStats* stats);

/* --- measurement ------------------------------------------------------- */
/* the cudaStream_t every kernel of this hierarchy is launched on */
void* cf_hier_stream(void* handle);
/* enable (1) / disable (0) per-launch CUDA-event profiling; clears records.
 * While enabled, V-cycles are launched eagerly instead of as a CUDA graph. */
int cf_profile(void* handle, int32_t enable);
/* aggregate of the recorded launches, one line per (kernel kind, level):
 * "kind level launches total_ms algorithmic_bytes\n"; *needed = length. */
int cf_profile_report(void* handle, char* buf, int64_t cap, int64_t* needed);

/* --- host setup helpers (solver.py greedy loops) ---------------------- */
/* solver.py:236-247: greedy ascending-id independent set of off-degree
 * <= cap; writes chosen ids to out_f, returns the count in *n_f. */
int cf_setup_elim_select(int64_t n, const int64_t* indptr, const int64_t* indices,
                         int32_t cap, int64_t* out_f, int64_t* n_f);
/* solver.py:297-346: seeds + affinity attachment with aggregate size cap
 * (8 in the reference) and affinity threshold (0.5 in the reference),
 * aggregate map in out_agg. */
int cf_setup_aggregate(int64_t n, const int64_t* indptr, const int64_t* indices,
                       const double* tv, int32_t n_tv, int32_t cap, double threshold,
                       int64_t* out_agg, int64_t* n_agg);
/* solver.py:364-380: greedy matching over a pre-sorted edge order. */
int cf_setup_matching(int64_t n, int64_t n_edges, const int64_t* eu, const int64_t* ev,
                      const int64_t* order, int64_t* out_agg, int64_t* n_agg);
/* solver.py:167-187 _rebuild_laplacian on a CSR without duplicates:
 * out capacity 2*nnz + n entries; *nnz = entries written (sorted rows). */
int cf_rebuild_laplacian(int64_t n, const int64_t* indptr, const int64_t* indices,
                         const double* data, int64_t* out_ptr, int64_t* out_idx,
                         double* out_val, int64_t* nnz);
/* graph.py:100-147 Graph.from_edges core: symmetric CSR of m (loop-free,
 * in-range) edges, neighbours sorted, duplicates summed in input order.
 * indptr: n+1; indices/weights: room for 2m entries; *nnz = entries written. */
int cf_build_csr(int64_t n, int64_t m, const int64_t* u, const int64_t* v, const double* w,
                 int64_t* indptr, int64_t* indices, double* weights, int64_t* nnz);
/* Device-side ingestion (csrc/cf_graph.cu).
 * cf_csr_from_edges_dev: the cf_build_csr contract computed on GPU `device`
 * (stable radix sort of the 2m adjacency entries by (row, col)); host arrays
 * in and out.  *status: 0 = written; 1 = duplicate edges present, nothing
 * written (the caller sums them on the host in the reference's order);
 * 2 = an edge is a self-loop or out of range.
 * cf_components_dev: root[i] = smallest node id of i's connected component
 * (graph.py:217-250 derives the largest component from these labels);
 * *rounds = hook/jump rounds used. */
int cf_csr_from_edges_dev(int32_t device, int64_t n, int64_t m, const int64_t* u,
                          const int64_t* v, const double* w, int64_t* indptr, int64_t* indices,
                          double* weights, int32_t* status);
int cf_components_dev(int32_t device, int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                      int64_t* root, int32_t* rounds);
/* solver.py:264-275 relaxed_test_vectors' sweeps: x (n x count row-major) <-
 * x + tril(L)^-1 (-(L x)), `sweeps` times; L sorted CSR with stored diagonal.
 * Native replacement of the SuperLU triangular solves on hub graphs. */
int cf_setup_relax(int64_t n, const int64_t* indptr, const int64_t* indices, const double* data,
                   int32_t count, int32_t sweeps, double* x);
/* Device-side coarse operators of the setup (
 * csrc/cf_setup_dev.cu).  L: n x n CSR with stored diagonal and sorted rows;
 * map[i] = coarse index of node i.  nf = 0: Galerkin product P^T L P of the
 * aggregation `map` (solver.py:383-386).  nf > 0: Schur complement of the
 * independent set fnodes[0..nf) (solver.py:251-261), map = position among the
 * kept nodes, -1 for eliminated ones.  Both are followed by the Laplacian
 * rebuild (solver.py:167-187).  *nnz_out = entries of the result; copy it out
 * (and free the device buffers) with cf_coarse_fetch_dev from the same thread:
 * out_ptr nc + 1, out_idx / out_val nnz entries, sorted rows, diagonal stored. */
int cf_coarse_operator_dev(int32_t device, int64_t n, const int64_t* indptr,
                           const int64_t* indices, const double* data, const int64_t* map,
                           int64_t nc, int64_t nf, const int64_t* fnodes, int64_t* nnz_out);
int cf_coarse_fetch_dev(int64_t* out_ptr, int64_t* out_idx, double* out_val);
/* The checks of _validate_laplacian (solver.py:190-211) on the GPU for an n x n
 * CSR with sorted rows: out[0] = max |entry|, out[1] = max |m - m^T|,
 * out[2] = max |row sum|, out[3] = largest positive off-diagonal (0 if none);
 * *ncomp = connected components of the pattern. */
int cf_validate_laplacian_dev(int32_t device, int64_t n, const int64_t* indptr,
                              const int64_t* indices, const double* data, double* out,
                              int64_t* ncomp);
/* greedy natural-order colouring of the off-diagonal graph (multicolour
 * Gauss-Seidel, the B200 smoother ordering). */
int cf_setup_colour(int64_t n, const int64_t* indptr, const int64_t* indices,
                    int32_t* out_colour, int32_t* n_colors);
/* locality renumbering for the device copy: output row r = input row
 * rows[r], columns mapped through cmap, rows sorted (scipy
 * A[rows][:, order].sort_indices() with cmap = inverse(order)), threaded. */
int cf_setup_permute(int64_t nrows, const int64_t* indptr, const int64_t* indices,
                     const double* data, const int64_t* rows, const int64_t* cmap,
                     int64_t* out_ptr, int64_t* out_idx, double* out_val);

#ifdef __cplusplus
}
#endif
#endif /* CFCENT_B200_H */
