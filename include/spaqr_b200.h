/*
 * spaqr_b200.h — C-ABI of the B200 (sm_100a) spaQR hot path.
 *
 * One context owns an HBM-resident block-sparse trailing matrix (dense fp64
 * blocks keyed by (row cluster, column cluster), column-major, ld = rows)
 * and the transform chains produced by factorizing it.  The host level
 * driver (Python, paper_2010_06807_b200/factor.py) calls these entry points
 * in exactly the order of the reference driver `nestqr.factor.factorize`
 * (pkg/src/nestqr/factor.py:771-911).  Plain pointers and sizes only.
 *
 * Status codes mirror the reference's exit codes (pkg/src/nestqr/errors.py:3-6):
 *   SPQ_OK 0, SPQ_ERR_SINGULAR 3 (SingularPivotError), SPQ_ERR_BAD_INPUT 4
 *   (NestqrError), SPQ_ERR_CUDA 5, SPQ_ERR_INTERNAL 6, SPQ_ERR_SPECULATION 7,
 *   SPQ_ERR_ILL_CONDITIONED 8 (IllConditionedInterfaceError)
 *   (speculative row flags were wrong: redo with speculate=0).  Details of the last
 *   failure via spq_last_error().
 * Ownership: the context owns all device memory; host arrays are borrowed
 * for the duration of a call.  Threading: one context per host thread; all
 * work is ordered on the context's CUDA stream.
 */
#ifndef SPAQR_B200_H
#define SPAQR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPQ_OK 0
#define SPQ_ERR_SINGULAR 3
#define SPQ_ERR_BAD_INPUT 4
#define SPQ_ERR_CUDA 5
#define SPQ_ERR_INTERNAL 6
#define SPQ_ERR_SPECULATION 7
#define SPQ_ERR_ILL_CONDITIONED 8   /* IllConditionedInterfaceError: index = interface,
                                       value = sigma_min, message = the floor */

typedef struct spq_ctx spq_ctx;

int spq_version(void);
/* device name / SM count / smem, for logs */
int spq_device_info(char* buf, int len);

/* ---------------------------------------------------------------- context */
int spq_create(spq_ctx** out, int device);
void spq_destroy(spq_ctx* ctx);
/* last error: code, pivot index, pivot value, message (context string) */
int spq_last_error(spq_ctx* ctx, int* code, int64_t* index, double* value,
                   char* msg, int msglen);
/* options (before spq_load):
 *   "speculate" (default 1): the host PREDICTS the per-row nonzero flags that
 *   decide panel row subsets and present column clusters (factor.py:422,
 *   454: np.any) from the symbolic effect of each update instead of reading
 *   them back after every factor wave; the device checks every prediction
 *   in stream order at the point it is used and spq_finish returns
 *   SPQ_ERR_SPECULATION if any was wrong (the host then redoes the
 *   factorization with speculate=0, which reads the flags back exactly). */
int spq_set_option(spq_ctx* ctx, const char* key, int64_t value);

/* -------------------------------------------------- (d) state construction
 * Replaces TrailingState.__init__ (factor.py:328-374) and
 * equilibrate_columns (sparse.py:142-166): uploads the CSC matrix, scales
 * columns to unit 2-norm on the device (recorded as W-chain[0],
 * factor.py:335-337) and scatters the entries into the depth-L blocks.
 * leaf_* describe the depth-L clusters (ids, and CSR-style row/col lists). */
int spq_load(spq_ctx* ctx, int64_t N, const int64_t* indptr,
             const int64_t* indices, const double* data, int equilibrate,
             int n_clusters_total, int n_leaf, const int32_t* leaf_ids,
             const int64_t* rows_ptr, const int64_t* rows,
             const int64_t* cols_ptr, const int64_t* cols);

/* ------------------------------------------------------ (a) interior elim
 * factor_interior for every id, in the given (ascending) order
 * (factor.py:402-493, loop :836-842).  Independent fronts are batched in
 * waves internally; results equal the sequential order. */
int spq_factor(spq_ctx* ctx, int n, const int32_t* ids);

/* ------------------------------------------------------ (b) scaling
 * scale_interface for every id (factor.py:504-532, loop :853-861).
 * out_done[i] = 1 when a record was produced. */
int spq_scale(spq_ctx* ctx, int n, const int32_t* ids, int32_t* out_done);

/* ------------------------------------------------------ (c) sparsification
 * sparsify_interface (scaled mode) for every id, in order
 * (factor.py:569-658, loop :864-878).  Per id: out_rank (accepted rank,
 * -1 when the interface was empty), out_before (|cols| before),
 * out_dropped (max spectral norm of the dropped blocks), out_done (record
 * produced). */
int spq_sparsify(spq_ctx* ctx, int n, const int32_t* ids, double eps,
                 int32_t* out_rank, int32_t* out_before, double* out_dropped,
                 int32_t* out_done);

/* sparsify_interface(p, eps, mode, scaled_now) for every id, in order
 * (factor.py:569-709): mode 0 'scaled', 1 'unscaled', 2 'variant1',
 * 3 'variant2'; scaled_now = whether this level was scaled (the driver's
 * do_scale, factor.py:849-850).  mode 0 with scaled_now runs the batched
 * wave path (= spq_sparsify); every other combination the reference's
 * sequential route, including the sigma-weighted unscaled target with its
 * IllConditionedInterfaceError (SPQ_ERR_ILL_CONDITIONED) and the
 * min_rank escalation loop. */
int spq_sparsify_ex(spq_ctx* ctx, int n, const int32_t* ids, double eps, int mode,
                    int scaled_now, int32_t* out_rank, int32_t* out_before,
                    double* out_dropped, int32_t* out_done);

/* ------------------------------------------------------ (d) merge
 * merge_level (factor.py:713-748): parent k takes the children
 * child_ids[child_ptr[k]:child_ptr[k+1]] in that order. */
int spq_merge(spq_ctx* ctx, int n_parents, const int32_t* parent_ids,
              const int32_t* child_ptr, const int32_t* child_ids);

/* closes the Q-chain with the row/column Permutation (factor.py:900-904)
 * and prepares the solve-phase chain programs. */
int spq_finish(spq_ctx* ctx);

/* ------------------------------------------------------ queries / stats */
int spq_cluster_size(spq_ctx* ctx, int id, int64_t* nrows, int64_t* ncols);
/* |cols| of n clusters in one call */
int spq_cluster_sizes(spq_ctx* ctx, int n, const int32_t* ids, int64_t* ncols);
int spq_total_cols(spq_ctx* ctx, int64_t* out);
/* trailing_blocks and trailing_nnz (exact nonzero count, device reduction) */
int spq_trailing_stats(spq_ctx* ctx, int64_t* nblocks, int64_t* nnz);
/* same statistics without a host round trip: trailing_blocks is returned at
 * once, trailing_nnz is counted on the device into `slot` (0..4095) and read
 * for slots [0, n) by spq_trailing_nnz (one synchronization). */
int spq_trailing_stats_async(spq_ctx* ctx, int slot, int64_t* nblocks);
int spq_trailing_nnz(spq_ctx* ctx, int n, int64_t* out);
/* keys (row cluster, column cluster) of the live trailing blocks -- the keys of
 * the reference's `TrailingState.trailing` dict (factor.py:349), which its
 * symbolic audit compares with `symbolic_fill_levels` (factor.py:1004-1050,
 * tests/test_factor.py:168-183).  At most `cap` pairs are written; *n
 * receives the full count. */
int spq_trailing_keys(spq_ctx* ctx, int64_t cap, int32_t* rows, int32_t* cols, int64_t* n);
int spq_row_of_col(spq_ctx* ctx, int64_t* out);
int spq_payload_scalars(spq_ctx* ctx, int64_t* out);
/* per kernel family [ms, algorithmic flops, launches, bytes] x 7 families
 * (copy, qr, wy, trsm, cpqr, flags, chain), then host counters
 * [alloc ms, sync ms, plan ms, api ms, allocs, syncs, pool bytes, kernels] */
int spq_timings(spq_ctx* ctx, double* out, int n);
int spq_reset_timings(spq_ctx* ctx);

/* ------------------------------------------------------ records (audit) */
int spq_num_records(spq_ctx* ctx);
/* info (8 slots): [kind(1 elim,2 scale,3 sparsify), m(rows), k, n(cols_n), rank,
 * cluster id, unscaled-sparsifier flag, fine count f] */
int spq_record_info(spq_ctx* ctx, int idx, int64_t* info8);
/* which: 0 rows, 1 cols_s/cols, 2 cols_n, 3 V, 4 tau, 5 T, 6 R (R_ss/R_pp;
 * R_ff f x f of an unscaled sparsifier), 7 R_sn (R_fc f x rank of an
 * unscaled sparsifier), 8/9/10 the H_f panel V (m x f) / tau / T (f x f).
 * Copies to host (int64 for index arrays, double otherwise). */
int spq_record_get(spq_ctx* ctx, int idx, int which, void* out);

/* ------------------------------------------------------ (e) solve chains
 * Factorization.apply_qt / solve_w / apply_w (factor.py:281-300) on an
 * N x nrhs column-major block.  *_host: host in/out (copies inside);
 * *_dev: device pointer, in place. */
/* ------------------------------------------------------- device GMRES
 * Right-preconditioned GMRES of pkg/src/nestqr/solve.py:66-209 on the device
 * (operator v -> apply_qt(A solve_w(v)), modified Gram-Schmidt with the
 * 1e-8 re-orthogonalisation test, Givens updates, the TRUE residual of every
 * iterate, best iterate returned).  spq_set_matrix uploads A (the original,
 * unscaled CSC matrix, stored as CSR on the device) once; spq_gmres takes
 * host b (N), optional host x0 (NULL = 0), writes x (N), the relative
 * residual history hist (room for maxit+1; its+1 entries written), the
 * iteration count, the converged flag and the best residual.
 * restart <= 0 means full GMRES. */
int spq_set_matrix(spq_ctx* ctx, int64_t N, const int64_t* indptr, const int64_t* indices,
                   const double* data);
int spq_gmres(spq_ctx* ctx, const double* b, const double* x0, double tol, int maxit,
              int restart, double* x, double* hist, int* its, int* converged,
              double* best_residual);

int spq_apply_qt_host(spq_ctx* ctx, const double* in, double* out, int nrhs);
int spq_solve_w_host(spq_ctx* ctx, const double* in, double* out, int nrhs);
int spq_apply_w_host(spq_ctx* ctx, const double* in, double* out, int nrhs);
int spq_apply_qt_dev(spq_ctx* ctx, double* d_inout, int nrhs);
int spq_solve_w_dev(spq_ctx* ctx, double* d_inout, int nrhs);
int spq_synchronize(spq_ctx* ctx);
/* compiled solve program (0 apply_qt, 1 solve_w, 2 apply_w): [waves, ops, max ops/wave, max k] */
int spq_chain_info(spq_ctx* ctx, int which, int64_t* info4);
/* CUDA events on the context stream (device timing of any call sequence) */
int spq_mark(spq_ctx* ctx, int slot);
int spq_mark_elapsed(spq_ctx* ctx, int slot_a, int slot_b, float* ms);

/* ------------------------------------------------------ kernel plugin API
 * The reference's backend contract (kernels/__init__.py:147-241), one
 * problem per call, host arrays (row-major as numpy hands them over):
 *   qr_house(B[m,k]) -> V[m,k], tau[k], T[k,k], R[k,k]      (m >= k)
 *   apply_panel(V,T, C[m,n], transpose) -> C in place
 *   rrqr(M[m,k], eps, min_rank) -> V[m,r], tau[r], Tred[m,k], perm[k], r
 *   tri_solve(R[k,k], C, side 0=left [k,n] / 1=right [n,k]) -> X
 * Errors: SPQ_ERR_SINGULAR with (index,value) for tri_solve pivots. */
int spq_qr_house(spq_ctx* ctx, int64_t m, int64_t k, const double* B,
                 double* V, double* tau, double* T, double* R);
int spq_apply_panel(spq_ctx* ctx, int64_t m, int64_t k, int64_t n,
                    const double* V, const double* T, double* C, int transpose);
int spq_rrqr(spq_ctx* ctx, int64_t m, int64_t k, const double* M, double eps,
             int64_t min_rank, double* V, double* tau, double* Tred,
             int64_t* perm, int64_t* rank);
int spq_tri_solve(spq_ctx* ctx, int64_t k, int64_t n, const double* R,
                  const double* C, int side, double* X);
/* build_t(V[m,k], tau[k]) -> T[k,k] (kernels/_numba.py:101-117) */
int spq_build_t(spq_ctx* ctx, int64_t m, int64_t k, const double* V,
                const double* tau, double* T);

/* raw DMMA GEMM timing, C(m x n) -= op(A) B, device-resident zeros; ms per call */
int spq_bench_gemm(spq_ctx* ctx, int m, int n, int k, int transA, int reps, float* ms);

/* ---------------------------------------- BASELINE config 2 (batched kernels)
 * batched_qr: nb blocks B_i (m_i x k_i, k_i <= m_i) + companions C_i
 * (m_i x nc_i), packed COLUMN-major back to back; R_i (k_i x k_i) out and
 * C_i <- H_i^T C_i; ms = device time of the batched QR + apply.
 * batched_rrqr: nb blocks (m x n) packed column-major; threshold CPQR with
 * the relative rule of rrqr_threshold; ranks[nb], rdiag[nb x min(m,n)]. */
int spq_batched_qr(spq_ctx* ctx, int nb, const int64_t* m, const int64_t* k,
                   const int64_t* nc, const double* B, double* R, double* C,
                   float* ms);
int spq_batched_rrqr(spq_ctx* ctx, int nb, int64_t m, int64_t n, const double* M,
                     double eps, int64_t* ranks, double* rdiag, float* ms);

#ifdef __cplusplus
}
#endif
#endif
