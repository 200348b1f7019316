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
constexpr int QR_NB = 32;   // columns per panel block (T_b is QR_NB x QR_NB)

// Shared-memory layout (doubles): exchange [2][XCH] | red [8][32] | dtot[32] |
// apiv[32] | wv[32] | scal[4] | Gs[32][33] | slab (nloc x kb, odd ld)
constexpr int XCH = 1 + 2 * QR_NB;
constexpr int SM_FIXED = 2 * XCH + 8 * QR_NB + 3 * QR_NB + 4 + QR_NB * (QR_NB + 1);

template <bool SMEM>
__global__ void __launch_bounds__(QR_NT) panel_qr_kernel(const PanelJob* __restrict__ jobs) {
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

  extern __shared__ __align__(16) double sm[];
  double* xch = sm;                        // [2][XCH]
  double* red = xch + 2 * XCH;             // [8][QR_NB]
  double* dtot = red + 8 * QR_NB;          // [QR_NB]
  double* apiv = dtot + QR_NB;             // [QR_NB]
  double* wv = apiv + QR_NB;               // [QR_NB]
  double* scal = wv + QR_NB;               // [4]
  double* Gs = scal + 4;                   // [QR_NB][QR_NB+1]  Gs[b + i*33] = V_b^T v_i
  double* slab_s = Gs + QR_NB * (QR_NB + 1);

  double* P0 = J.P + (int64_t)j0 * m + j0 + r0;  // (block row r0, col j0)
  double* S;
  int lds;
  if (SMEM) {
    S = slab_s;
    lds = nloc | 1;                         // odd: thread-per-column reads conflict-free
    for (int e = tid; e < nloc * kb; e += QR_NT) {
      const int i = e % nloc, c = e / nloc;
      S[i + c * lds] = P0[i + (int64_t)c * m];
    }
  } else {
    S = P0;
    lds = m;
  }
  if (q == 0 && j0 > 0) {   // finished R entries above the block
    for (int e = tid; e < j0 * kb; e += QR_NT) {
      const int i = e % j0, c = e / j0;
      double* src = J.P + i + (int64_t)(j0 + c) * m;
      J.R[i + (int64_t)(j0 + c) * k] = *src;
      *src = 0.0;
    }
  }
  __syncthreads();

  // thread -> (column c, row partition pr): kb <= 32 columns x NP partitions
  const int NP = QR_NT / QR_NB;            // 8
  const int c_of = tid % QR_NB, p_of = tid / QR_NB;

  for (int jj = 0; jj < kb; ++jj) {
    double* X = xch + (jj & 1) * XCH;
    const int ist = max(0, jj - r0 + 1);   // first local row strictly below the pivot
    const int ploc = jj - r0;
    const bool owner = ploc >= 0 && ploc < nloc;
    // dots of the pivot column (rows below the pivot) with EVERY block column:
    //   c == jj -> sigma, c > jj -> trailing d_c, c < jj -> Gram column for T
    if (c_of < kb) {
      double s = 0.0;
      const double* xc = S + jj * lds;
      const double* ac = S + c_of * lds;
      for (int i = ist + p_of; i < nloc; i += NP) s += xc[i] * ac[i];
      red[p_of * QR_NB + c_of] = s;
    }
    __syncthreads();
    if (tid < kb) {
      double s = 0.0;
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) s += red[pp * QR_NB + tid];
      X[1 + tid] = s;
      if (owner) X[1 + QR_NB + tid] = S[ploc + tid * lds];
    }
    cluster.sync();
    const int own = min(CL - 1, jj / rpc);
    // cluster totals: lane r of a warp loads CTA r's partial (parallel DSMEM
    // loads), fixed shuffle tree -> identical sums in every CTA
    const double* dsrc = X + 1;                 // CL == 1: the local exchange is the total
    const double* asrc = X + 1 + QR_NB;
    if (CL > 1) {
      for (int c = warp; c < kb; c += QR_NT / 32) {
        double v = lane < CL ? cluster.map_shared_rank(X, lane)[1 + c] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          dtot[c] = v;
          apiv[c] = cluster.map_shared_rank(X, own)[1 + QR_NB + c];
        }
      }
      __syncthreads();
      dsrc = dtot;
      asrc = apiv;
    }
    // every thread forms the reflector scalars itself
    const double sigma = dsrc[jj];
    const double alpha = asrc[jj];
    double tau, beta, v0 = 1.0;
    const bool zero = sigma == 0.0;
    if (zero) {
      if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
    } else {
      beta = sqrt(alpha * alpha + sigma);
      v0 = (alpha <= 0.0) ? alpha - beta : -sigma / (alpha + beta);
      tau = -v0 / beta;
    }
    if (q == 0 && tid == 0) J.tau[j0 + jj] = tau;
    if (tid < kb && tid != jj) {
      const double s = dsrc[tid];
      const double ap = asrc[tid];
      const double gv = zero ? ap : ap + s / v0;      // V_c^T v_jj
      if (tid < jj) Gs[tid + jj * (QR_NB + 1)] = gv;
      else wv[tid] = tau * gv;                        // w_c = tau v^T a_c
    }
    __syncthreads();
    // row-owned update: v_i = x_i / v0 stored in column jj, a_ic -= w_c v_i
    const int ibeg = owner ? ploc : ist;
    for (int i = ibeg + tid; i < nloc; i += QR_NT) {
      double vi;
      if (i == ploc) {
        vi = 1.0;
        S[i + jj * lds] = beta;
      } else {
        vi = zero ? 0.0 : S[i + jj * lds] / v0;
        S[i + jj * lds] = vi;
      }
      if (tau != 0.0)
        for (int c = jj + 1; c < kb; ++c) S[i + c * lds] -= wv[c] * vi;
    }
    __syncthreads();
  }

  // R entries of the diagonal block out, explicit unit-lower V in
  for (int e = tid; e < nloc * kb; e += QR_NT) {
    const int i = e % nloc, c = e / nloc;
    const int a = r0 + i;
    if (a < kb && c >= a) {
      J.R[(j0 + a) + (int64_t)(j0 + c) * k] = S[i + c * lds];
      S[i + c * lds] = (c == a) ? 1.0 : 0.0;
    }
  }
  // T_b from the Gram columns gathered above: row-parallel recurrence
  //   T[a,a] = tau_a,  T[a,i] = -tau_i sum_{b=a}^{i-1} T[a,b] G[b,i]
  if (q == 0 && tid < kb) {
    const int a = tid;
    double trow[QR_NB];
#pragma unroll
    for (int b = 0; b < QR_NB; ++b) trow[b] = 0.0;
    trow[a] = J.tau[j0 + a];
    for (int i = a + 1; i < kb; ++i) {
      const double ti = J.tau[j0 + i];
      double s = 0.0;
      for (int b = a; b < i; ++b) s += trow[b] * Gs[b + i * (QR_NB + 1)];
      trow[i] = (ti != 0.0) ? -ti * s : 0.0;
    }
    double* Tg = J.T + j0 + (int64_t)j0 * k;
    for (int i = 0; i < kb; ++i) Tg[a + (int64_t)i * k] = trow[i];
  }
  __syncthreads();
  if (SMEM) {
    for (int e = tid; e < nloc * kb; e += QR_NT) {
      const int i = e % nloc, c = e / nloc;
      P0[i + (int64_t)c * m] = S[i + c * lds];
    }
  }
  cluster.sync();   // no CTA leaves while others may still read its shared memory
}

size_t panel_smem_bytes(int64_t slab_elems, bool smem) {
  return (size_t)(SM_FIXED + (smem ? slab_elems : 0)) * sizeof(double);
}

void launch_panel_qr(const PanelJob* d_jobs, int njobs, int cluster, int64_t slab_elems,
                     bool smem, int /*kbmax*/, cudaStream_t st) {
  if (njobs <= 0) return;
  const size_t bytes = panel_smem_bytes(slab_elems, smem);
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
  static bool init = false;
  if (!init) {
    for (auto fn : {panel_qr_kernel<true>, panel_qr_kernel<false>}) {
      CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    init = true;
  }
  if (smem)
    CUDA_TRY(cudaLaunchKernelEx(&cfg, panel_qr_kernel<true>, d_jobs));
  else
    CUDA_TRY(cudaLaunchKernelEx(&cfg, panel_qr_kernel<false>, d_jobs));
}

// ------------------------------------------------------- register panel QR
// Same algorithm and conventions as panel_qr_kernel, with the 32-column
// block held in REGISTERS: thread t of CTA q owns local rows t + 256 r
// (r < R) of the CTA's row range, all 32 columns.  Per column step:
//   * partial dots x.a_c for all 32 columns are thread-local FMAs,
//   * a warp reduce-scatter (31 shuffles) leaves lane l with the warp sum of
//     column l, 8 warp partials are summed through shared memory, CTA
//     partials over DSMEM (one barrier.cluster),
//   * the rank-1 update is thread-local.
// No shared-memory traffic proportional to the panel (the smem kernel
// streams the slab through shared memory twice per column).  Requires
// rows-per-CTA >= 32 so every pivot row lives in CTA 0 (thread jj).
constexpr int QRR_NT = 256;
constexpr int QRR_CLMAX = 16;

// ---- DSMEM push exchange (st.async + mbarrier complete_tx): no cluster
// barrier per column step.  A cluster barrier with release/acquire
// semantics compiles to MEMBAR.ALL.GPU + L1 invalidation on sm_100a.
__device__ __forceinline__ uint32_t qrr_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t qrr_mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void qrr_st_async(uint32_t raddr, double v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :: "r"(raddr), "d"(v), "r"(rmbar) : "memory");
}
__device__ __forceinline__ void qrr_arm(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void qrr_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
  }
}

struct QrrShared {
  double XR[2][QRR_CLMAX][QR_NB];   // per source CTA: partial dots (pushed)
  double PR[2][QR_NB];              // pivot row (pushed by CTA 0)
  double Xp[QR_NB];                 // CTA 0: pivot row staging
  double red[QRR_NT / 32][QR_NB];
  double dtot[QR_NB], apiv[QR_NB];
  double Gs[QR_NB * (QR_NB + 1)];
  alignas(8) uint64_t mbar[2];
};

struct QrrCtx {
  int q, CL, nloc, tid, lane, warp, kb, j0;
  double* tau;
};

// One column step.  The loop over columns is NOT unrolled (a 32x unrolled
// step sequence overflows the instruction cache: ncu showed 58% of warp
// samples stalled on "no instructions"); the register block is indexed
// with compile-time columns only, so the dynamic column jj is selected
// with predicated moves.
#ifdef SPQ_TRACE
// diagnostic build only: clock64 stamps of thread 0 / CTA 0 per column step
__device__ long long g_panel_trace[32 * 8];
#define QRR_STAMP(slot) do { if (x.q == 0 && x.tid == 0) g_panel_trace[jj * 8 + (slot)] = clock64(); } while (0)
#else
#define QRR_STAMP(slot) do { } while (0)
#endif

template <int R>
__device__ __forceinline__ void qrr_step(const QrrCtx& x, double (&a)[R][QR_NB], QrrShared& sh,
                                         const int jj) {
  const int q = x.q, CL = x.CL, nloc = x.nloc, tid = x.tid, lane = x.lane, warp = x.warp;
  const int B = jj & 1;
  QRR_STAMP(0);
  // ---- this thread's entries of the pivot column
  double xv[R];
  bool part[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + QRR_NT * r;
    part[r] = i < nloc && (q > 0 || i > jj);
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < QR_NB; ++c) t = (c == jj) ? a[r][c] : t;
    xv[r] = t;
  }
  // ---- partial dots of the pivot column (rows strictly below the pivot),
  // in two halves of 16 columns (register pressure); a warp reduce-scatter
  // per half leaves lane l with the warp sum of column (l & 15) of the half
  double mine = 0.0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    double d[QR_NB / 2];
#pragma unroll
    for (int c = 0; c < QR_NB / 2; ++c) d[c] = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double xr = part[r] ? xv[r] : 0.0;
#pragma unroll
      for (int c = 0; c < QR_NB / 2; ++c) d[c] = fma(xr, a[r][half * (QR_NB / 2) + c], d[c]);
    }
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
      const bool hi = (lane & h) != 0;
#pragma unroll
      for (int t = 0; t < h; ++t) {
        const double send = hi ? d[t] : d[t + h];
        const double keep = hi ? d[t + h] : d[t];
        d[t] = keep + __shfl_xor_sync(0xffffffffu, send, h);
      }
    }
    const double tot = d[0] + __shfl_xor_sync(0xffffffffu, d[0], 16);
    if ((lane >> 4) == half) mine = tot;
  }
  QRR_STAMP(1);
  sh.red[warp][lane] = mine;
  if (q == 0 && tid == jj) {
#pragma unroll
    for (int c = 0; c < QR_NB; ++c) sh.Xp[c] = a[0][c];
  }
  __syncthreads();
  QRR_STAMP(2);
  // clock64 stamps (tools/panel_trace.py) showed this tail bound by fp64 ISSUE
  // (one fp64 instruction per warp every ~14 cycles): every thread repeated
  // the sqrt/div scalars and formed all 32 update coefficients itself (64
  // fp64 operations), and the totals took 20 shuffle+add rounds per warp.
  // Now warp 0 alone sums the CTA partials (lane c = column c, rank order),
  // forms the scalars once and publishes the 32 coefficients; the other
  // warps wait at one CTA barrier and read them.
  if (CL > 1) {
    // ---- push the CTA partials (and CTA 0's pivot row) to every CTA
    for (int t = tid; t < QR_NB * CL; t += QRR_NT) {
      const int dst = t >> 5, c = t & 31;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int w = 0; w < QRR_NT / 32; w += 2) { s0 += sh.red[w][c]; s1 += sh.red[w + 1][c]; }
      const uint32_t mb = qrr_mapa(qrr_smem(&sh.mbar[B]), dst);
      qrr_st_async(qrr_mapa(qrr_smem(&sh.XR[B][q][c]), dst), s0 + s1, mb);
      if (q == 0) qrr_st_async(qrr_mapa(qrr_smem(&sh.PR[B][c]), dst), sh.Xp[c], mb);
    }
  }
  QRR_STAMP(3);
  if (warp == 0) {
    double dt, ap;
    if (CL > 1) {
      qrr_wait(qrr_smem(&sh.mbar[B]), (uint32_t)((jj >> 1) & 1));
      QRR_STAMP(4);
      if (lane == 0)   // re-arm this buffer for step jj + 2 (before anyone can push it)
        qrr_arm(qrr_smem(&sh.mbar[B]), (uint32_t)((CL + 1) * QR_NB * sizeof(double)));
      // totals over the CTAs in rank order (identical in every CTA)
      double s0 = 0.0, s1 = 0.0;
      for (int p = 0; p + 1 < CL; p += 2) { s0 += sh.XR[B][p][lane]; s1 += sh.XR[B][p + 1][lane]; }
      if (CL & 1) s0 += sh.XR[B][CL - 1][lane];
      dt = s0 + s1;
      ap = sh.PR[B][lane];
    } else {
      QRR_STAMP(4);
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int w = 0; w < QRR_NT / 32; w += 2) { s0 += sh.red[w][lane]; s1 += sh.red[w + 1][lane]; }
      dt = s0 + s1;
      ap = sh.Xp[lane];
    }
    // ---- reflector scalars (kernels/_numba.py:15-35)
    const double sigma = __shfl_sync(0xffffffffu, dt, jj);
    const double alpha = __shfl_sync(0xffffffffu, ap, jj);
    // v0 = alpha - beta (alpha <= 0) or -sigma / (alpha + beta); 1 / v0 and
    // tau = -v0 / beta are formed from alpha, beta, sigma directly, so the two
    // quotients do not wait for each other (x * (1 / v0) instead of x / v0 and
    // these quotients are within an ulp or two of the reference's values, far
    // inside the parity tolerance)
    double tau, beta, inv0 = 0.0;
    if (sigma == 0.0) {
      if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
    } else {
      house_scalars(alpha, sigma, tau, beta, inv0);
    }
    const double g = fma(dt, inv0, ap);           // v_jj^T (column lane): G entry / update dot
    const double ts = tau != 0.0 ? tau : 0.0;
    sh.dtot[lane] = lane > jj ? ts * g : 0.0;     // update coefficient of column lane
    if (lane < jj) sh.Gs[lane + jj * (QR_NB + 1)] = g;
    if (lane == 0) {
      sh.apiv[0] = inv0;
      sh.apiv[1] = beta;
      if (q == 0 && jj < x.kb) x.tau[x.j0 + jj] = tau;
    }
  }
  __syncthreads();
  QRR_STAMP(5);
  const double inv0 = sh.apiv[0], beta = sh.apiv[1];
  // ---- v below the pivot, rank-1 update of the columns right of it
  double v[R], nj[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + QRR_NT * r;
    const bool piv = q == 0 && r == 0 && i == jj;
    v[r] = piv ? 1.0 : (part[r] ? xv[r] * inv0 : 0.0);
    nj[r] = piv ? beta : (part[r] ? v[r] : xv[r]);   // new value of column jj
  }
  QRR_STAMP(6);
#pragma unroll
  for (int c = 0; c < QR_NB; ++c) {
    const double wc = sh.dtot[c];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double u = fma(-wc, v[r], a[r][c]);
      a[r][c] = (c == jj) ? nj[r] : u;
    }
  }
  QRR_STAMP(7);
}

template <int R, int KBMAX>
__global__ void __launch_bounds__(QRR_NT, 1) panel_qr_reg_kernel(const PanelJob* __restrict__ jobs_g,
                                                                 const __grid_constant__ PList<PanelJob, PL_SMALL> pl) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  const PanelJob* jobs = jobs_g ? jobs_g : pl.v;
  const PanelJob J = jobs[blockIdx.x / CL];
  const int m = J.m, k = J.k, j0 = J.j0, kb = J.kb;
  const int mh = m - j0;
  const int rpc = (mh + CL - 1) / CL;
  const int r0 = min(mh, q * rpc);
  const int r1 = min(mh, r0 + rpc);
  const int nloc = r1 - r0;
  const int tid = threadIdx.x;
  __shared__ QrrShared sh;

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(qrr_smem(&sh.mbar[b])) : "memory");
      qrr_arm(qrr_smem(&sh.mbar[b]), (uint32_t)((CL + 1) * QR_NB * sizeof(double)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double* P0 = J.P + (int64_t)j0 * m + j0 + r0;
  double a[R][QR_NB];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + QRR_NT * r;
#pragma unroll
    for (int c = 0; c < QR_NB; ++c)
      a[r][c] = (i < nloc && c < kb) ? P0[i + (int64_t)c * m] : 0.0;
  }
  if (q == 0 && j0 > 0) {   // finished R entries above the block
    for (int e = tid; e < j0 * kb; e += QRR_NT) {
      const int i = e % j0, c = e / j0;
      double* src = J.P + i + (int64_t)(j0 + c) * m;
      J.R[i + (int64_t)(j0 + c) * k] = *src;
      *src = 0.0;
    }
  }
  cluster.sync();   // every CTA's barriers are initialised and armed before any push
  const QrrCtx x{q, CL, nloc, tid, tid & 31, tid >> 5, kb, j0, J.tau};
  // KBMAX steps run unconditionally (a data-dependent trip count would make
  // the compiler lower the shuffles as collectives); steps jj >= kb see an
  // all-zero column: tau = 0, no update, nothing stored
#pragma unroll 1
  for (int jj = 0; jj < KBMAX; ++jj) qrr_step<R>(x, a, sh, jj);

  // R entries of the diagonal block out, explicit unit-lower V in
  if (q == 0 && tid < kb) {
#pragma unroll
    for (int c = 0; c < QR_NB; ++c) {
      if (c >= tid && c < kb) {
        J.R[(j0 + tid) + (int64_t)(j0 + c) * k] = a[0][c];
        a[0][c] = (c == tid) ? 1.0 : 0.0;
      }
    }
  }
  __syncthreads();
  // T_b from the Gram columns: row-parallel recurrence
  if (q == 0 && tid < kb) {
    const int ar = tid;
    double tr[QR_NB];
#pragma unroll
    for (int b = 0; b < QR_NB; ++b) tr[b] = (b == ar) ? J.tau[j0 + ar] : 0.0;
#pragma unroll
    for (int i = 1; i < QR_NB; ++i) {
      if (i > ar && i < kb) {
        const double ti = J.tau[j0 + i];
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < i; ++b)
          if (b >= ar) s += tr[b] * sh.Gs[b + i * (QR_NB + 1)];
        tr[i] = (ti != 0.0) ? -ti * s : 0.0;
      }
    }
    double* Tg = J.T + j0 + (int64_t)j0 * k;
#pragma unroll
    for (int i = 0; i < QR_NB; ++i)
      if (i < kb) Tg[ar + (int64_t)i * k] = tr[i];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + QRR_NT * r;
    if (i < nloc) {
#pragma unroll
      for (int c = 0; c < QR_NB; ++c)
        if (c < kb) P0[i + (int64_t)c * m] = a[r][c];
    }
  }
  // every push addressed to this CTA has landed (waited above); a relaxed
  // cluster barrier keeps CTAs resident until all pushes were issued
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}

template <int R, int KBMAX>
void launch_qrr(const cudaLaunchConfig_t& cfg, const PanelJob* d_jobs,
                const PList<PanelJob, PL_SMALL>& pl) {
  static bool init = false;
  if (!init) {
    CUDA_TRY(cudaFuncSetAttribute(panel_qr_reg_kernel<R, KBMAX>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    init = true;
  }
  CUDA_TRY(cudaLaunchKernelEx(&cfg, panel_qr_reg_kernel<R, KBMAX>, d_jobs, pl));
}

int panel_reg_kbmax(int kb) { return kb <= 8 ? 8 : kb <= 16 ? 16 : kb <= 24 ? 24 : 32; }

void launch_panel_qr_reg(const PanelJob* d_jobs, const PanelJob* h_jobs, int njobs, int cluster,
                         int rows_per_thread, int kbmax, cudaStream_t st) {
  if (njobs <= 0) return;
  PList<PanelJob, PL_SMALL> pl;
  if (!d_jobs) {
    if (njobs > PL_SMALL) throw std::runtime_error("launch_panel_qr_reg: parameter list too long");
    for (int i = 0; i < njobs; ++i) pl.v[i] = h_jobs[i];
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * cluster));
  cfg.blockDim = dim3(QRR_NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int kc = panel_reg_kbmax(kbmax);
  if (rows_per_thread <= 1) {
    if (kc == 8) launch_qrr<1, 8>(cfg, d_jobs, pl);
    else if (kc == 16) launch_qrr<1, 16>(cfg, d_jobs, pl);
    else if (kc == 24) launch_qrr<1, 24>(cfg, d_jobs, pl);
    else launch_qrr<1, 32>(cfg, d_jobs, pl);
  } else {
    if (kc == 8) launch_qrr<2, 8>(cfg, d_jobs, pl);
    else if (kc == 16) launch_qrr<2, 16>(cfg, d_jobs, pl);
    else if (kc == 24) launch_qrr<2, 24>(cfg, d_jobs, pl);
    else launch_qrr<2, 32>(cfg, d_jobs, pl);
  }
}

// ------------------------------------------------------------------ larft
// Full compact-WY T (k x k) from G = V^T V and tau, one CTA per job, in
// 32-column block columns J:  T_JJ by the row recurrence (one warp),
// Y = G[0:j0,J] T_JJ (scratch), T[0:j0,J] = -T[0:j0,0:j0] Y.
constexpr int LARFT_NT = 256;

__global__ void __launch_bounds__(LARFT_NT) larft_kernel(const LarftJob* __restrict__ jobs) {
  const LarftJob J = jobs[blockIdx.x];
  const int k = J.k, tid = threadIdx.x;
  __shared__ double Tjj[32 * 33];
  __shared__ double Gjj[32 * 33];
  for (int j0 = 0; j0 < k; j0 += 32) {
    const int w = min(32, k - j0);
    for (int e = tid; e < w * w; e += LARFT_NT) {
      const int a = e % w, b = e / w;
      Gjj[a + b * 33] = J.G[(j0 + a) + (int64_t)(j0 + b) * J.ldg];
    }
    __syncthreads();
    if (tid < w) {
      const int a = tid;
      double trow[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) trow[b] = 0.0;
      trow[a] = J.tau[j0 + a];
      for (int i = a + 1; i < w; ++i) {
        const double ti = J.tau[j0 + i];
        double s = 0.0;
        for (int b = a; b < i; ++b) s += trow[b] * Gjj[b + i * 33];
        trow[i] = (ti != 0.0) ? -ti * s : 0.0;
      }
      for (int i = 0; i < w; ++i) Tjj[a + i * 33] = trow[i];
    }
    __syncthreads();
    for (int e = tid; e < w * w; e += LARFT_NT) {
      const int a = e % w, i = e / w;
      J.T[(j0 + a) + (int64_t)(j0 + i) * J.ldt] = (a <= i) ? Tjj[a + i * 33] : 0.0;
    }
    for (int e = tid; e < (k - j0 - w) * w; e += LARFT_NT) {   // strictly below: zeros
      const int a = j0 + w + e % (k - j0 - w), i = e / (k - j0 - w);
      J.T[a + (int64_t)(j0 + i) * J.ldt] = 0.0;
    }
    if (J.Y == nullptr)   // off-diagonal blocks are filled by the GEMM doubling
      for (int e = tid; e < j0 * w; e += LARFT_NT) {
        const int a = e % j0, i = e / j0;
        J.T[a + (int64_t)(j0 + i) * J.ldt] = 0.0;
      }
    if (j0 > 0 && J.Y != nullptr) {
      // Y[a,e] = sum_{f<=e} G[a, j0+f] T_JJ[f,e]   (a < j0)
      for (int t = tid; t < j0 * w; t += LARFT_NT) {
        const int a = t % j0, e = t / j0;
        double s = 0.0;
        for (int f = 0; f <= e; ++f) s += J.G[a + (int64_t)(j0 + f) * J.ldg] * Tjj[f + e * 33];
        J.Y[a + (int64_t)e * k] = s;
      }
      __syncthreads();
      // T[a, j0+e] = -sum_{b=a}^{j0-1} T[a,b] Y[b,e]
      for (int t = tid; t < j0 * w; t += LARFT_NT) {
        const int a = t % j0, e = t / j0;
        double s = 0.0;
        for (int b = a; b < j0; ++b) s += J.T[a + (int64_t)b * J.ldt] * J.Y[b + (int64_t)e * k];
        J.T[a + (int64_t)(j0 + e) * J.ldt] = -s;
      }
    }
    __syncthreads();
  }
}

// Full T in ONE launch for k <= LARFT_FULL_MAX (replaces the 32-block
// larft + 2 log2(k/32) doubling GEMM launches, ~15 us each, on the panels
// of the sequential upper-level fronts).  G is staged in shared memory; row
// a of T is an independent recurrence (thread a):
//   T[a,i] = -tau_i sum_{b=a}^{i-1} T[a,b] G[b,i]
// with T[a,b] (b > a) kept in the strictly LOWER triangle of the same
// buffer (G is only read above the diagonal): no second k x k array.
constexpr int LARFT_FULL_MAX = 160;

__global__ void __launch_bounds__(4 * LARFT_FULL_MAX) larft_full_kernel(const LarftJob* __restrict__ jobs_g,
                                                                       const __grid_constant__ PList<LarftJob, PL_SMALL> pl) {
  const LarftJob J = jobs_g ? jobs_g[blockIdx.x] : pl.v[blockIdx.x];
  const int k = J.k, tid = threadIdx.x, nt = blockDim.x;
  const int ld = (k + 1) & ~1;   // even: column reads and the (ld+1) row stride are conflict-free
  extern __shared__ double S[];
  // G (upper triangle) in batches of 8 independent loads per thread: their
  // latencies overlap (a plain strided loop serialises one L2 round trip
  // per iteration)
  for (int e0 = 0; e0 < k * k; e0 += 8 * nt) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * nt;
      const int a = e % k, b = e / k;
      t[u] = (e < k * k && a < b) ? __ldg(J.G + a + (int64_t)b * J.ldg) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * nt;
      const int a = e % k, b = e / k;
      if (e < k * k && a < b) S[a + b * ld] = t[u];
    }
  }
  __syncthreads();
  // row a of T by four lanes (the long rows near the top set the kernel's
  // duration): lane `sub` sums b = a+1+sub, a+5+sub, ...; two shuffles
  // combine; lane 0 stores and the group syncs before the next entry
  const int a = tid >> 2, sub = tid & 3;
  const unsigned gm = 0xFu << ((tid & 31) & 28);
  if (a < k) {
    const double ta = J.tau[a];
    double* Ta = S + a * ld;   // Ta[b] = T[a,b] for b > a (lower triangle, column a)
    for (int i = a + 1; i < k; ++i) {
      const double* Gi = S + i * ld;   // Gi[b] = G[b,i], b < i
      double s0 = sub == 0 ? ta * Gi[a] : 0.0, s1 = 0.0;
      int b = a + 1 + sub;
      for (; b + 4 < i; b += 8) {
        s0 = fma(Ta[b], Gi[b], s0);
        s1 = fma(Ta[b + 4], Gi[b + 4], s1);
      }
      if (b < i) s0 = fma(Ta[b], Gi[b], s0);
      double sv = s0 + s1;
      sv += __shfl_xor_sync(gm, sv, 1);
      sv += __shfl_xor_sync(gm, sv, 2);
      const double ti = J.tau[i];
      if (sub == 0) Ta[i] = (ti != 0.0) ? -ti * sv : 0.0;
      __syncwarp(gm);
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += nt) {
    const int a2 = e % k, i = e / k;
    J.T[a2 + (int64_t)i * J.ldt] = a2 < i ? S[i + a2 * ld] : (a2 == i ? J.tau[a2] : 0.0);
  }
}

// Blocked variant of the same launch (default): the long row recurrence above
// is a dependent chain of k steps (row 0: ~450 cycles per step, ~60 us at
// k = 130) on ONE SM.  Here
//   1. the 32 x 32 diagonal blocks T_JJ -- each depends only on G_JJ and
//      tau_J -- are built at the same time, four lanes per row (32 steps);
//   2. block column J (rows above it, j0 = 32, 64, ...) by two small
//      products, all in shared memory:
//        Y = G[0:j0, J] T_JJ                (in place over G[0:j0, J])
//        T[0:j0, J] = -T[0:j0, 0:j0] Y      (rows independent)
// T[a,b] (b > a) lives in the strictly lower triangle (S[b + a ld]), tau on
// the diagonal; ld is odd so a row read across 32 columns is conflict-free.
constexpr int LARFT_BLK_NT = 512;

__global__ void __launch_bounds__(LARFT_BLK_NT) larft_blk_kernel(const LarftJob* __restrict__ jobs_g,
                                                               const __grid_constant__ PList<LarftJob, PL_SMALL> pl) {
  const LarftJob J = jobs_g ? jobs_g[blockIdx.x] : pl.v[blockIdx.x];
  const int k = J.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = LARFT_BLK_NT, NW = NT / 32;
  const int ld = k | 1;
  extern __shared__ double S[];
  // G (strict upper triangle) and tau (diagonal), eight independent loads per thread
  for (int e0 = 0; e0 < k * k; e0 += 8 * NT) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * NT;
      const int a = e % k, b = e / k;
      t[u] = (e < k * k && a <= b) ? (a < b ? __ldg(J.G + a + (int64_t)b * J.ldg) : __ldg(J.tau + a)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * NT;
      const int a = e % k, b = e / k;
      if (e < k * k && a <= b) S[a + b * ld] = t[u];
    }
  }
  __syncthreads();
  // ---- 1. diagonal blocks: row f of block jb by four lanes
  const int nblk = (k + 31) / 32;
  for (int jb0 = 0; jb0 < nblk; jb0 += NT / 128) {
    const int jb = jb0 + tid / 128;
    const int f = (tid & 127) >> 2, sub = tid & 3;
    const int j0 = jb * 32, w = min(32, k - j0);
    const unsigned gm = 0xFu << (lane & 28);
    if (jb < nblk && f < w) {
      const int a = j0 + f;
      const double ta = S[a + a * ld];
      double* Ta = S + a * ld;   // Ta[b] = T[a,b], b > a
      for (int i = a + 1; i < j0 + w; ++i) {
        const double* Gi = S + i * ld;   // Gi[b] = G[b,i], b < i
        double s0 = sub == 0 ? ta * Gi[a] : 0.0, s1 = 0.0;
        int b = a + 1 + sub;
        for (; b + 4 < i; b += 8) {
          s0 = fma(Ta[b], Gi[b], s0);
          s1 = fma(Ta[b + 4], Gi[b + 4], s1);
        }
        if (b < i) s0 = fma(Ta[b], Gi[b], s0);
        double sv = s0 + s1;
        sv += __shfl_xor_sync(gm, sv, 1);
        sv += __shfl_xor_sync(gm, sv, 2);
        const double ti = Gi[i];
        if (sub == 0) Ta[i] = (ti != 0.0) ? -ti * sv : 0.0;
        __syncwarp(gm);
      }
    }
  }
  __syncthreads();
  // ---- 2. block columns above the diagonal blocks
  for (int j0 = 32; j0 < k; j0 += 32) {
    const int w = min(32, k - j0);
    // Y[b][e] = sum_{f<=e} G[b][j0+f] T_JJ[f][e]: warp per row b, lane e; in
    // place (every lane has read its G entries before any lane writes)
    for (int b = warp; b < j0; b += NW) {
      double y = 0.0;
      if (lane < w) {
        const int ce = j0 + lane;
        for (int f = 0; f < lane; ++f) y = fma(S[b + (j0 + f) * ld], S[ce + (j0 + f) * ld], y);
        y = fma(S[b + ce * ld], S[ce + ce * ld], y);   // f = e: T[e][e] = tau_e
      }
      __syncwarp();
      if (lane < w) S[b + (j0 + lane) * ld] = y;
    }
    __syncthreads();
    // T[a][j0+e] = -sum_{b=a}^{j0-1} T[a][b] Y[b][e]   (T[a][a] = tau_a)
    for (int a = warp; a < j0; a += NW) {
      if (lane < w) {
        const int ce = j0 + lane;
        double t0 = S[a + a * ld] * S[a + ce * ld], t1 = 0.0;
        int b = a + 1;
        for (; b + 1 < j0; b += 2) {
          t0 = fma(S[b + a * ld], S[b + ce * ld], t0);
          t1 = fma(S[b + 1 + a * ld], S[b + 1 + ce * ld], t1);
        }
        if (b < j0) t0 = fma(S[b + a * ld], S[b + ce * ld], t0);
        S[ce + a * ld] = -(t0 + t1);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < k * k; e += NT) {
    const int a2 = e % k, i = e / k;
    J.T[a2 + (int64_t)i * J.ldt] = a2 < i ? S[i + a2 * ld] : (a2 == i ? S[a2 + a2 * ld] : 0.0);
  }
}

int larft_full_max() { return LARFT_FULL_MAX; }

void launch_larft_full(const LarftJob* d_jobs, const LarftJob* h_jobs, int njobs, int kmax,
                       cudaStream_t st) {
  if (njobs <= 0) return;
  PList<LarftJob, PL_SMALL> pl;
  if (!d_jobs) {
    if (njobs > PL_SMALL) throw std::runtime_error("launch_larft_full: parameter list too long");
    for (int i = 0; i < njobs; ++i) pl.v[i] = h_jobs[i];
  }
  static const bool rowwise = getenv("SPQ_LARFT_ROWWISE") && getenv("SPQ_LARFT_ROWWISE")[0] == '1';
  if (!rowwise) {
    const size_t smem = (size_t)kmax * (kmax | 1) * sizeof(double);
    static size_t conf = 0;
    if (smem > conf) {
      CUDA_TRY(cudaFuncSetAttribute(larft_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      conf = smem;
    }
    larft_blk_kernel<<<njobs, LARFT_BLK_NT, smem, st>>>(d_jobs, pl); SPQ_LAUNCH_CHECK();
    return;
  }
  const size_t smem = (size_t)kmax * ((kmax + 1) & ~1) * sizeof(double);
  static size_t conf = 0;
  if (smem > conf) {
    CUDA_TRY(cudaFuncSetAttribute(larft_full_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    conf = smem;
  }
  const int nt = ((4 * kmax + 31) / 32) * 32;
  larft_full_kernel<<<njobs, nt, smem, st>>>(d_jobs, pl); SPQ_LAUNCH_CHECK();
}

int larft_tiles(int) { return 1; }

void launch_larft(const LarftJob* d_jobs, int njobs, int /*total_tiles*/, cudaStream_t st) {
  if (njobs <= 0) return;
  larft_kernel<<<njobs, LARFT_NT, 0, st>>>(d_jobs); SPQ_LAUNCH_CHECK();
}

// ------------------------------------------------------------ pivot check
__global__ void pivot_check_kernel(const PivotJob* __restrict__ jobs, int njobs,
                                   int64_t* err_idx, double* err_val) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
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
      for (int i0 = 0; i0 < J.k && bad < 0; i0 += 32) {   // first failing index wins
        const int i = i0 + lane;
        const double r = i < J.k ? J.R[i + (int64_t)i * J.ld] : 1.0;
        const unsigned b = __ballot_sync(0xffffffffu, i < J.k && fabs(r) <= floor);
        if (b) {
          const int first = __ffs(b) - 1;
          bad = i0 + first;
          val = __shfl_sync(0xffffffffu, r, first);
        }
      }
    }
  }
  if (lane == 0) {
    err_idx[J.slot] = bad;
    err_val[J.slot] = val;
  }
}

void launch_pivot_check(const PivotJob* d_jobs, int njobs, int64_t* d_err_idx, double* d_err_val,
                        cudaStream_t st) {
  if (njobs <= 0) return;
  pivot_check_kernel<<<(njobs * 32 + 255) / 256, 256, 0, st>>>(d_jobs, njobs, d_err_idx, d_err_val); SPQ_LAUNCH_CHECK();
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

// diagonal-block step of the blocked right TRSM: columns [j0, j0+w) of
// X R = B, the contributions of columns < j0 already subtracted (GEMM)
__global__ void __launch_bounds__(TRSM_NT) trsm_diag_kernel(const TrsmJob* __restrict__ jobs,
                                                           int njobs, int j0) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const TrsmJob J = jobs[lo];
  const int row = (blockIdx.x - J.tile0) * TRSM_NT + threadIdx.x;
  if (row >= J.n || j0 >= J.k) return;
  const int w = min(32, J.k - j0);
  double* B = J.B + row;
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (j >= w) break;
    double s = B[(int64_t)(j0 + j) * J.ldb];
    for (int i = 0; i < j; ++i) s -= x[i] * J.R[(j0 + i) + (int64_t)(j0 + j) * J.ldr];
    x[j] = s / J.R[(j0 + j) + (int64_t)(j0 + j) * J.ldr];
    B[(int64_t)(j0 + j) * J.ldb] = x[j];
  }
}

void launch_trsm_diag(const TrsmJob* d_jobs, int njobs, int total_tiles, int j0, cudaStream_t st) {
  if (njobs <= 0 || total_tiles <= 0) return;
  trsm_diag_kernel<<<total_tiles, TRSM_NT, 0, st>>>(d_jobs, njobs, j0); SPQ_LAUNCH_CHECK();
}

void launch_trsm_right(const TrsmJob* d_jobs, int njobs, int total_tiles, cudaStream_t st) {
  if (njobs <= 0 || total_tiles <= 0) return;
  trsm_right_kernel<<<total_tiles, TRSM_NT, 0, st>>>(d_jobs, njobs); SPQ_LAUNCH_CHECK();
}

}  // namespace spq

#ifdef SPQ_TRACE
extern "C" int spq_debug_panel_trace(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, spq::g_panel_trace, sizeof(long long) * (size_t)(n < 32 * 8 ? n : 32 * 8));
}
#endif
