// Shared definitions of the sm_100a spaQR kernels.
//
// Storage convention for every dense operand: fp64, COLUMN-major, explicit
// leading dimension.  Index arrays are int64 on the host, int32 on the
// device where sizes allow.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define SPQ_HD __host__ __device__ __forceinline__

namespace spq {

// ----------------------------------------------------------- copy tasks
// dst[dr(i) + j*ldd] = src[sr(i) + j*lds]   (i < nr, j < nc)
//   sr(i) = src_rows ? src_rows[i] : i ;  dr(i) = dst_rows ? dst_rows[i] : i
// trans: dst[j + i*ldd] = src[sr(i) + j*lds]   (src rows -> dst columns)
// src == nullptr: zero fill of the destination rectangle.
// ident: write the identity into the (square) destination.
struct CopyTask {
  const double* src;
  double* dst;
  const int* src_rows;
  const int* dst_rows;
  int nr, nc;
  int lds, ldd;
  int trans;
  int ident;
  int cta0;   // first CTA of the task in a flattened (1-D) copy grid
  int ncta;   // CTAs of the task in that grid
};

// one interface of a sparsify wave: column norms, keep filter, compaction
struct PrepJob {
  const double* M;   // m x n candidates (ld m)
  double* sq;        // [n] squared column norms
  int* keep_idx;     // [n] kept column indices (ascending)
  int* nk;           // kept count
  double* ratio;     // min(eps / maxcol, 0.999999)
  double* maxcol;
  double* W;         // m x nk gathered columns (ld m)
  int m, n;
  int allow_filter, pad_;
};

// Householder scalars of a column step (kernels/_numba.py:15-35) from the pivot
// entry alpha and sigma = sum of squares below it (sigma > 0): beta, tau and
// 1 / v0.  The latency-bound kernels run this on ONE warp per step and a warp
// issues one fp64 instruction every ~14 cycles, so the instruction count is
// the cost: rsqrt + one Newton step gives beta and 1 / beta (tau = -v0 / beta
// becomes a product), and the alpha > 0 branch needs one reciprocal instead
// of two quotients.  Results are within ~2 ulp of sqrt / division (the parity
// tolerance is 1e-10); extreme magnitudes take the plain formulas.
#ifdef __CUDACC__
__device__ __forceinline__ void house_scalars(double alpha, double sigma, double& tau, double& beta,
                                              double& inv0) {
  const double s = fma(alpha, alpha, sigma);
#ifdef SPQ_PLAIN_SCALARS   // A/B builds
  const bool plain = true;
#else
  const bool plain = !(s > 1e-280 && s < 1e280 && sigma > 1e-280);
#endif
  if (plain) {
    beta = sqrt(s);
    if (alpha <= 0.0) {
      const double v0 = alpha - beta;
      inv0 = 1.0 / v0;
      tau = -v0 / beta;
    } else {
      const double ab = alpha + beta;
      inv0 = -ab / sigma;
      tau = sigma / (ab * beta);
    }
    return;
  }
  const double rb = rsqrt(s);
  double b = s * rb;
  b = fma(0.5 * rb, fma(-b, b, s), b);   // one Newton step: b = sqrt(s) to ~1 ulp
  beta = b;
  if (alpha <= 0.0) {
    const double v0 = alpha - b;
    inv0 = 1.0 / v0;
    tau = -v0 * rb;
  } else {
    const double ab = alpha + b;
    const double u = 1.0 / (ab * sigma);
    inv0 = -(ab * ab) * u;            // -ab / sigma
    tau = (sigma * rb) * (sigma * u); // sigma / (ab * beta)
  }
}
#endif

// ---------------------------------------------------- job lists in params
// Short job lists travel IN the kernel launch parameters (__grid_constant__,
// read through a generic pointer into parameter space) instead of through
// an H2D copy of the upload ring: a small pinned copy between two dependent
// kernels costs ~2.3 us of device time (measured, tools/memcpy_probe.py),
// and ~4000 launches per C3 factorization carried one or more.
template <class T, int N>
struct PList {
  T v[N];
};
constexpr int PL_GEMM = 24;
constexpr int PL_RED = 24;
constexpr int PL_COPY = 48;
constexpr int PL_WYF = 48;
constexpr int PL_SMALL = 8;   // panel / larft / CPQR job lists (one front or interface per wave, mostly)

// ------------------------------------------------------------- gemm
// C = alpha * op(A) * B + beta * C ; op(A) = A (m x k, lda) or A^T (A is k x m)
struct GemmProb {
  const double* A;
  const double* B;
  double* C;
  int m, n, k;
  int lda, ldb, ldc;
  double alpha, beta;
  int tile0;  // first CTA index of this problem in the launch
};

struct SplitRed {
  const double* P;   // splits x (m x n) partials
  double* C;
  int m, n, ldc, splits;
  double alpha, beta;
};

// -------------------------------------------------- panel QR (one nb-block)
// Factor columns [j0, j0+kb) (kb <= 32) of the m x k panel P (ld = m), rows
// j0..m-1.  On exit P holds V (unit lower trapezoidal, explicit, zeros
// above), R the upper triangle, tau the coefficients, and the block's
// compact-WY T_b in T[j0:j0+kb, j0:j0+kb].
struct PanelJob {
  double* P;
  double* R;     // k x k, ld = k
  double* tau;   // k
  double* T;     // k x k, ld = k (diagonal block written when want_T)
  int m, k, j0, kb;
  int want_T;
};

// ------------------------------------------- fused shallow compact-WY (k <= 64)
// C (m x n) <- C - V op(T) V^T C ; op(T) = T^T when trans (Q^T C), else T
struct WyfJob {
  const double* V;   // m x k (ldv), explicit (zeros above the unit diagonal)
  const double* T;   // k x k upper triangular (ldt)
  double* C;         // m x n (ldc)
  int ldv, ldt, ldc;
  int m, n, k;
  int trans;
  int tile0;         // first 32-column tile of this job in the launch
};

// ------------------------------------------------------ pivot check
struct PivotJob {
  const double* R;
  int k, ld;
  int slot;
};

// ------------------------------------------------------ right TRSM
// X R = B in place on B (n x k, ldb), R k x k upper (ldr)
struct TrsmJob {
  const double* R;
  double* B;
  int n, k, ldr, ldb;
  int tile0;
};

struct LarftJob {
  const double* G;   // k x k Gram V^T V (ld = ldg)
  const double* tau;
  double* T;         // k x k (ld = ldt)
  double* Y;         // scratch k x 32
  int k, ldg, ldt;
  int tile0;
};

struct CpqrArgs {
  double* W;            // m x ncols (ld m), compacted candidate columns, in/out
  int m, ncols_cap;     // ncols_cap: allocated columns; live count in *nk
  const int* nk;        // device: number of live columns
  const double* eps;    // device: threshold ratio
  int min_rank;
  double* V;            // m x kmax (ld m), pre-zeroed; explicit unit-lower out
  double* tau;          // kmax
  double* beta;         // kmax (R diagonal of accepted steps)
  int* rank;            // out
  int* perm;            // out: phys_at (logical -> physical), ncols_cap
  double* slot_val;     // [2][G]
  int* slot_pos;        // [2][G]
  int finalize;         // write beta/zeros into W's pivot columns (Tred)
  int* gmaps;           // per-CTA position maps [G][2][ncols] when shared memory is too small
  int force_gmaps;      // test switch: use gmaps even when shared memory would fit
};

// sigma_max of a dropped block through its Gram G = E E^T (f x f, ld f)
struct PowerJob {
  const double* G;
  int f;
  double* out;
};

// one record operation of a solve-chain wave
enum ChainKind { CH_WY_T = 1, CH_WY_N = 2, CH_TRI_SOLVE = 3, CH_TRI_MUL = 4 };
struct ChainOp {
  int kind;
  int m, k, n;          // WY: V is m x k on z[idx[0:m]]; TRI: R k x k on y[idx[0:k]], R_sn k x n on y[idx_n]
  const int* idx;
  const int* idx_n;
  const double* V;
  const double* T;
  const double* R;
  const double* Rsn;
  double* scratch;      // per chunk 3*k doubles of global scratch when k is too big for shared memory
  const double* W;      // WY: precomputed V T^T (WY_T) or V T (WY_N), m x k (ld m), or nullptr
  int* cnt;             // WY: chunk arrival counter (last chunk of phase A reduces)
  int64_t u_off;        // WY: offset of the reduced vector u (k) in the wave scratch (x nrhs)
  int nchunk;           // CTAs working on this op
  int per;              // rows (WY) or R_sn columns (TRI) per chunk
  int64_t part_off;     // offset of this op's partials in the wave scratch (x nrhs)
  const double* Dinv;   // TRI_SOLVE: inverses of the 32 x 32 diagonal blocks of R (block t covers
                        // columns k-32(t+1)..k-32t; 32 x 32, ld 32 each), or nullptr
  // a row block of a large TRI_SOLVE (compile_chains splits R_ss into row blocks so the
  // products with the already solved part run over many CTAs): R / R2 have leading
  // dimension ldr, R_sn ldn (0: k); R2 (k x n2) multiplies y[idx2], the columns of R_ss to
  // the right of this block
  int ldr, ldn, n2;
  const double* R2;
  const int* idx2;
};
constexpr size_t CHAIN_SMEM_MAX = 200 * 1024;

// one block of the batched one-sided Jacobi (k_svd.cu): A (m x n, lda) is
// overwritten; smax / smin receive the extreme singular values
struct SvJob {
  double* A;
  int m, n, lda;
  double* smax;
  double* smin;
};

// one problem of the batched CTA-resident CPQR
struct CpqrJob {
  double* W;           // m x n (ldw), candidate columns (compacted), read (and written back)
  int m, n, ncap, ldw; // n used when nk == nullptr; ncap sizes shared memory
  const int* nk;       // device live column count (sparsify) or nullptr
  const double* eps;   // device threshold
  int min_rank;
  double* V;           // m x kmax (ldv), pre-zeroed
  int ldv;
  double* tau;
  double* beta;
  int* rank;
  int* perm;
  int write_back;      // store the reduced matrix (Tred) back into W
};

}  // namespace spq

// ---------------------------------------------------------------- launchers
namespace spq {
// d_* == nullptr: the list is passed in the launch parameters from h_* (n <= PL_*)
void launch_copy(const CopyTask* d_tasks, const CopyTask* h_tasks, int ntasks, int64_t max_elems,
                 int64_t total_ctas, cudaStream_t st, int64_t gran = 2048);
void launch_rowflags(const double* const* d_ptrs, const int* d_nr, const int* d_nc,
                     const int64_t* d_off, unsigned char* d_out, int nblk, cudaStream_t st);
void launch_rowflags_verify(const double* const* d_ptrs, const int* d_nr, const int* d_nc,
                            const int64_t* d_off, const unsigned char* d_pred, int nblk, int* d_bad,
                            cudaStream_t st);
void launch_count_nnz(const double* const* d_ptrs, const int64_t* d_sizes, int nblk,
                      unsigned long long* d_count, cudaStream_t st);
void launch_colnorms_scale(const int64_t* indptr, const int64_t* indices, double* data,
                           int64_t N, double* scale, int* zero_col, int equilibrate, cudaStream_t st);
void launch_csc_scatter(const int64_t* indptr, const int64_t* indices, const double* data,
                        int64_t N, const int64_t* dest_off, double* const* blk_base,
                        const int* entry_blk, cudaStream_t st);
void launch_gemm(const GemmProb* d_probs, const GemmProb* h_probs, int nprob, int total_tiles,
                 bool transA, cudaStream_t st);
int gemm_tiles(int m, int n);
void gemm_set_variant(int v);   // 0 default, 1: 64x64 tiles, 2: 128x64 tiles
void launch_wyf(const WyfJob* d_jobs, const WyfJob* h_jobs, int njobs, int tiles, int kmax, int cl,
                cudaStream_t st);
int wyf_kmax();
int wyf_cluster(int m);
void launch_splitk_reduce(const SplitRed* d_tasks, const SplitRed* h_tasks, int ntasks,
                          int64_t max_mn, cudaStream_t st);
void launch_panel_qr(const PanelJob* d_jobs, int njobs, int cluster, int64_t slab_elems,
                     bool smem, int kbmax, cudaStream_t st);
void launch_panel_qr_reg(const PanelJob* d_jobs, const PanelJob* h_jobs, int njobs, int cluster, int rows_per_thread,
                         int kbmax, cudaStream_t st);
int panel_reg_kbmax(int kb);
void launch_larft(const LarftJob* d_jobs, int njobs, int total_tiles, cudaStream_t st);
int larft_tiles(int k);
void launch_larft_full(const LarftJob* d_jobs, const LarftJob* h_jobs, int njobs, int kmax,
                       cudaStream_t st);
int larft_full_max();
void launch_pivot_check(const PivotJob* d_jobs, int njobs, int64_t* d_err_idx,
                        double* d_err_val, cudaStream_t st);
void launch_trsm_right(const TrsmJob* d_jobs, int njobs, int total_tiles, cudaStream_t st);
int trsm_tiles(int n);
void launch_trsm_diag(const TrsmJob* d_jobs, int njobs, int total_tiles, int j0, cudaStream_t st);
size_t cpqr_cta_smem(int m, int ncap);
void launch_cpqr_cta(const CpqrJob* d_jobs, int njobs, size_t smem, cudaStream_t st);
void launch_power_iter(const PowerJob* d_jobs, int njobs, int fmax, cudaStream_t st);
int cpqr_cluster_size(int m, int ncap);
size_t cpqr_cluster_smem(int m, int ncap, int cl);
void launch_cpqr_cluster(const CpqrJob* d_jobs, int njobs, int cl, size_t smem, cudaStream_t st);
int cpqr_reg_plan(int m, int n, int variant, int* tpc, int* nt);
int cpqr_reg_nvar();
int cpqr_reg_rows(int variant);
int cpqr_reg_elems(int variant);
size_t cpqr_reg_smem(int padded_rows, int cl, int nt);
void launch_cpqr_reg(const CpqrJob* d_jobs, const CpqrJob* h_jobs, int njobs, int variant, int cl, int tpc, int nt, size_t smem,
                     cudaStream_t st);
extern cudaEvent_t g_chain_mid_event;
void launch_chain_dinv(const ChainOp* d_ops, int nops, cudaStream_t st);
void launch_chain_wave(const ChainOp* d_ops, const int2* d_tasks, int ntasks, int kmax, int slab_k,
                       bool has_wy, double* part, double* z, int64_t N, int nrhs,
                       cudaStream_t st);
}  // namespace spq

#define CUDA_TRY(x)                                                        \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      throw spq::CudaFailure(e_, #x, __FILE__, __LINE__);                  \
    }                                                                      \
  } while (0)

// every <<<>>> launch is followed by this: launch-configuration errors
// (grid limits, shared-memory attributes) must never pass silently
#define SPQ_LAUNCH_CHECK() CUDA_TRY(cudaGetLastError())

#include <stdexcept>
#include <string>
namespace spq {
struct CudaFailure : std::runtime_error {
  CudaFailure(cudaError_t e, const char* what, const char* f, int l)
      : std::runtime_error(std::string(cudaGetErrorString(e)) + " at " + f + ":" +
                           std::to_string(l) + " (" + what + ")") {}
};
// ---------------------------------------------------- Krylov (k_krylov.cu)
constexpr int KRY_G = 296;   // fixed grid of the deterministic reductions (2 x 148 SMs)
void kry_spmv(const int64_t* ptr, const int* idx, const double* val, const double* x,
              const double* b, double* y, int64_t n, int mode, cudaStream_t st);
void kry_dot_part(const double* x, const double* y, int64_t n, double* part, cudaStream_t st);
void kry_finish(const double* part, double* out, bool sqrt_it, cudaStream_t st);
void kry_mgs_step(const double* qi, const double* q_next, double* w, int64_t n,
                  const double* part_in, double* part_out, double* h_out, cudaStream_t st);
void kry_multi_dot(const double* Q, int64_t ldq, int j, const double* w, int64_t n, double* part,
                   double* cvec, cudaStream_t st);
void kry_reorth(const double* Q, int64_t ldq, int j, const double* cvec, const double* wn,
                double thr, double* w, int64_t n, double* Hcol, int* flag, double* part_out,
                cudaStream_t st);
void kry_scale_div(const double* src, const double* den, double* dst, int64_t n, cudaStream_t st);
void kry_gemv(const double* Q, int64_t ldq, int j, const double* y, double* out, int64_t n,
              cudaStream_t st);
void kry_add(const double* x, const double* y, double* z, int64_t n, cudaStream_t st);

}  // namespace spq
