// Householder panel factorization and its companions:
//
//  * panel_qr_kernel — factors one nb-column block [j0, j0+kb) of a
//    column-major m x k panel with the reference reflector convention
//    (kernels/_numba.py:14-35: beta >= 0, v0 = alpha-beta if alpha <= 0 else
//    -sigma/(alpha+beta), tau = -v0/beta, sigma == 0 -> tau 0 or 2).  The
//    rows j0..m-1 are split across the CTAs of a thread-block CLUSTER
//    (1..16 CTAs); each column step needs ONE cluster-wide reduction: every
//    CTA publishes (sigma_q, d_q[c] = sum x_i a_ic, pivot-row values) in
//    double-buffered shared memory, one barrier.cluster, then every CTA
//    sums the partials over DSMEM in rank order (bit-identical across CTAs)
//    and applies w_c = tau (a_pc + d_c / v0).  Row slabs live in shared
//    memory when they fit (227 KB/CTA), otherwise in global memory (L2).
//  * larft_kernel — T of the compact WY from the Gram G = V^T V, one
//    independent recurrence per ROW of T: T[a,i] = -tau_i sum_b T[a,b]G[b,i].
//  * pivot_check_kernel — `_check_pivots` (factor.py:57-68).
//  * trsm_right_kernel — X R = B (kernels/_numba.py:181-191), thread per row.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spq {

constexpr int QR_NT = 256;

template <bool SMEM>
__global__ void __launch_bounds__(QR_NT) panel_qr_kernel(const PanelJob* __restrict__ jobs,
                                                         int kbmax) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  const PanelJob J = jobs[blockIdx.x / CL];
  const int m = J.m, k = J.k, j0 = J.j0, kb = J.kb;
  const int mh = m - j0;
  const int rpc = (mh + CL - 1) / CL;
  const int r0 = min(mh, q * rpc);
  const int r1 = min(mh, r0 + rpc);
  const int nloc = r1 - r0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = QR_NT / 32;

  extern __shared__ double sm[];
  const int XCH = 1 + 2 * kbmax;
  double* xch = sm;                       // [2][XCH]
  double* dtot = xch + 2 * XCH;           // [kbmax]
  double* apiv = dtot + kbmax;            // [kbmax]
  double* wv = apiv + kbmax;              // [kbmax]
  double* scal = wv + kbmax;              // [4]
  double* gram = scal + 4;                // [kbmax*kbmax] only when want_T (kb <= 32)
  double* slab_s = gram + (kbmax <= 32 ? kbmax * kbmax : 0);

  double* P0 = J.P + (int64_t)j0 * m + j0 + r0;  // (row r0 of the block, col j0)
  double* S;
  int lds;
  if (SMEM) {
    S = slab_s;
    lds = nloc > 0 ? nloc : 1;
    for (int e = tid; e < nloc * kb; e += QR_NT) {
      const int i = e % nloc, c = e / nloc;
      S[i + c * lds] = P0[i + (int64_t)c * m];
    }
  } else {
    S = P0;
    lds = m;
  }
  // rows above the block in its columns are finished R entries: move them
  if (q == 0 && j0 > 0) {
    for (int e = tid; e < j0 * kb; e += QR_NT) {
      const int i = e % j0, c = e / j0;
      double* src = J.P + i + (int64_t)(j0 + c) * m;
      J.R[i + (int64_t)(j0 + c) * k] = *src;
      *src = 0.0;
    }
  }
  __syncthreads();

  for (int jj = 0; jj < kb; ++jj) {
    const int par = jj & 1;
    double* X = xch + par * XCH;
    const int ist = max(0, jj - r0 + 1);   // first local row strictly below the pivot
    const int ploc = jj - r0;              // local pivot row (owner iff 0 <= ploc < nloc)
    // ---- partial dots: column c = jj gives sigma, c > jj gives d_c
    for (int c = jj + warp; c < kb; c += NW) {
      double s = 0.0;
      for (int i = ist + lane; i < nloc; i += 32) s += S[i + jj * lds] * S[i + c * lds];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) X[1 + c] = s;
    }
    if (ploc >= 0 && ploc < nloc)
      for (int c = jj + tid; c < kb; c += QR_NT) X[1 + kbmax + c] = S[ploc + c * lds];
    cluster.sync();
    const int owner = min(CL - 1, jj / rpc);
    for (int c = jj + tid; c < kb; c += QR_NT) {
      double s = 0.0;
      for (int r = 0; r < CL; ++r) {
        const double* Xr = cluster.map_shared_rank(X, r);
        s += Xr[1 + c];
      }
      dtot[c] = s;
      apiv[c] = cluster.map_shared_rank(X, owner)[1 + kbmax + c];
    }
    __syncthreads();
    if (tid == 0) {
      const double sigma = dtot[jj], alpha = apiv[jj];
      double tau, beta, v0 = 1.0, zero = 0.0;
      if (sigma == 0.0) {
        zero = 1.0;
        if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
      } else {
        beta = sqrt(alpha * alpha + sigma);
        v0 = (alpha <= 0.0) ? alpha - beta : -sigma / (alpha + beta);
        tau = -v0 / beta;
      }
      scal[0] = tau; scal[1] = v0; scal[2] = beta; scal[3] = zero;
      if (q == 0) J.tau[j0 + jj] = tau;
    }
    __syncthreads();
    const double tau = scal[0], v0 = scal[1], beta = scal[2];
    const bool zero = scal[3] != 0.0;
    for (int c = jj + 1 + tid; c < kb; c += QR_NT)
      wv[c] = zero ? tau * apiv[c] : tau * (apiv[c] + dtot[c] / v0);
    // reflector entries below the pivot: v_i = x_i / v0
    for (int i = ist + tid; i < nloc; i += QR_NT)
      S[i + jj * lds] = zero ? 0.0 : S[i + jj * lds] / v0;
    __syncthreads();
    if (tau != 0.0) {
      const int ncol = kb - jj - 1;
      const int ibeg = (ploc >= 0 && ploc < nloc) ? ploc : ist;
      const int nr = nloc - ibeg;
      for (int e = tid; e < nr * ncol; e += QR_NT) {
        const int i = ibeg + e % nr, c = jj + 1 + e / nr;
        const double vi = (i == ploc) ? 1.0 : S[i + jj * lds];
        S[i + c * lds] -= wv[c] * vi;
      }
    }
    if (ploc >= 0 && ploc < nloc && tid == 0) S[ploc + jj * lds] = beta;
    __syncthreads();
  }

  // R entries of the diagonal block out, explicit unit-lower V in
  for (int e = tid; e < nloc * kb; e += QR_NT) {
    const int i = e % nloc, c = e / nloc;
    const int a = r0 + i;   // block-relative row
    if (a < kb && c >= a) {
      J.R[(j0 + a) + (int64_t)(j0 + c) * k] = S[i + c * lds];
      S[i + c * lds] = (c == a) ? 1.0 : 0.0;
    }
  }
  __syncthreads();

  if (J.want_T) {
    // partial Gram of this CTA's rows, cluster reduction into CTA 0, then
    // the row-parallel T recurrence (kb <= 32): T[a,i] = -tau_i sum T[a,b] G[b,i]
    for (int e = tid; e < kb * kb; e += QR_NT) {
      const int a = e % kb, b = e / kb;
      double s = 0.0;
      if (a <= b)
        for (int i = 0; i < nloc; ++i) s += S[i + a * lds] * S[i + b * lds];
      gram[e] = s;
    }
    cluster.sync();
    if (q == 0) {
      for (int e = tid; e < kb * kb; e += QR_NT) {
        double s = 0.0;
        for (int r = 0; r < CL; ++r) s += cluster.map_shared_rank(gram, r)[e];
        gram[e] = s;   // only CTA 0 reads CTA 0's partials: in-place is safe
      }
      __syncthreads();
      if (tid < kb) {
        const int a = tid;
        double trow[32];
        for (int b = 0; b < kb; ++b) trow[b] = 0.0;
        trow[a] = J.tau[j0 + a];
        for (int i = a + 1; i < kb; ++i) {
          const double ti = J.tau[j0 + i];
          double s = 0.0;
          for (int b = a; b < i; ++b) s += trow[b] * gram[b + i * kb];
          trow[i] = (ti != 0.0) ? -ti * s : 0.0;
        }
        double* Tg = J.T + j0 + (int64_t)j0 * k;
        for (int i = 0; i < kb; ++i) Tg[a + (int64_t)i * k] = trow[i];
      }
    }
  }

  if (SMEM) {
    for (int e = tid; e < nloc * kb; e += QR_NT) {
      const int i = e % nloc, c = e / nloc;
      P0[i + (int64_t)c * m] = S[i + c * lds];
    }
  }
  cluster.sync();   // no CTA leaves while others may still read its shared memory
}

static size_t panel_smem_bytes(int kbmax, bool want_T, int64_t slab_elems, bool smem) {
  size_t n = 2 * (1 + 2 * (size_t)kbmax) + 3 * (size_t)kbmax + 4;
  if (want_T) n += (size_t)kbmax * kbmax;
  if (smem) n += (size_t)slab_elems;
  return n * sizeof(double);
}

void launch_panel_qr(const PanelJob* d_jobs, int njobs, int cluster, int64_t slab_elems,
                     bool smem, int kbmax, cudaStream_t st) {
  if (njobs <= 0) return;
  const bool want_T = kbmax <= 32;
  const size_t bytes = panel_smem_bytes(kbmax, want_T, slab_elems, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * cluster));
  cfg.blockDim = dim3(QR_NT);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (smem) {
    static bool init = false;
    if (!init) {
      CUDA_TRY(cudaFuncSetAttribute(panel_qr_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(panel_qr_kernel<true>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      init = true;
    }
    CUDA_TRY(cudaLaunchKernelEx(&cfg, panel_qr_kernel<true>, d_jobs, kbmax));
  } else {
    static bool init = false;
    if (!init) {
      CUDA_TRY(cudaFuncSetAttribute(panel_qr_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(panel_qr_kernel<false>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      init = true;
    }
    CUDA_TRY(cudaLaunchKernelEx(&cfg, panel_qr_kernel<false>, d_jobs, kbmax));
  }
}

// ------------------------------------------------------------------ larft
constexpr int LARFT_NT = 128;

__global__ void __launch_bounds__(LARFT_NT) larft_kernel(const LarftJob* __restrict__ jobs,
                                                         int njobs) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const LarftJob J = jobs[lo];
  const int a = (blockIdx.x - J.tile0) * LARFT_NT + threadIdx.x;
  if (a >= J.k) return;
  const int k = J.k;
  double* T = J.T;
  for (int b = 0; b < a; ++b) T[a + (int64_t)b * J.ldt] = 0.0;
  T[a + (int64_t)a * J.ldt] = J.tau[a];
  for (int i = a + 1; i < k; ++i) {
    const double ti = J.tau[i];
    double s = 0.0;
    if (ti != 0.0)
      for (int b = a; b < i; ++b) s += T[a + (int64_t)b * J.ldt] * J.G[b + (int64_t)i * J.ldg];
    T[a + (int64_t)i * J.ldt] = (ti != 0.0) ? -ti * s : 0.0;
  }
}

int larft_tiles(int k) { return (k + LARFT_NT - 1) / LARFT_NT; }

void launch_larft(const LarftJob* d_jobs, int njobs, int total_tiles, cudaStream_t st) {
  if (njobs <= 0 || total_tiles <= 0) return;
  larft_kernel<<<total_tiles, LARFT_NT, 0, st>>>(d_jobs, njobs);
}

// ------------------------------------------------------------ pivot check
__global__ void pivot_check_kernel(const PivotJob* __restrict__ jobs, int njobs,
                                   int64_t* err_idx, double* err_val) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= njobs) return;
  const PivotJob J = jobs[j];
  int64_t bad = -1;
  double val = 0.0;
  if (J.k > 0) {
    const double d0 = fabs(J.R[0]);
    if (d0 == 0.0) {
      bad = 0;
    } else {
      const double floor = 1e-14 * d0;
      for (int i = 0; i < J.k; ++i) {
        const double r = J.R[i + (int64_t)i * J.ld];
        if (fabs(r) <= floor) { bad = i; val = r; break; }
      }
    }
  }
  err_idx[J.slot] = bad;
  err_val[J.slot] = val;
}

void launch_pivot_check(const PivotJob* d_jobs, int njobs, int64_t* d_err_idx, double* d_err_val,
                        cudaStream_t st) {
  if (njobs <= 0) return;
  pivot_check_kernel<<<(njobs + 127) / 128, 128, 0, st>>>(d_jobs, njobs, d_err_idx, d_err_val);
}

// ------------------------------------------------------------- right TRSM
constexpr int TRSM_NT = 128;

__global__ void __launch_bounds__(TRSM_NT) trsm_right_kernel(const TrsmJob* __restrict__ jobs,
                                                             int njobs) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const TrsmJob J = jobs[lo];
  const int row = (blockIdx.x - J.tile0) * TRSM_NT + threadIdx.x;
  if (row >= J.n) return;
  double* B = J.B + row;
  for (int j = 0; j < J.k; ++j) {
    double s = B[(int64_t)j * J.ldb];
    for (int i = 0; i < j; ++i) s -= B[(int64_t)i * J.ldb] * J.R[i + (int64_t)j * J.ldr];
    B[(int64_t)j * J.ldb] = s / J.R[j + (int64_t)j * J.ldr];
  }
}

int trsm_tiles(int n) { return (n + TRSM_NT - 1) / TRSM_NT; }

void launch_trsm_right(const TrsmJob* d_jobs, int njobs, int total_tiles, cudaStream_t st) {
  if (njobs <= 0 || total_tiles <= 0) return;
  trsm_right_kernel<<<total_tiles, TRSM_NT, 0, st>>>(d_jobs, njobs);
}

}  // namespace spq
