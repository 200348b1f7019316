// Fused compact-WY application for SHALLOW reflector blocks (k <= 64):
//
//     C  <-  C - V op(T) (V^T C)        op(T) = T^T (Q^T C) or T (Q C)
//
// in ONE launch, instead of the three batched GEMMs (+ split-K reduce) the
// generic path issues (`wy_batch` / the per-block panel update of
// `qr_batch`).  Those launches each cost ~10-20 us for the thin shapes of
// the panel updates (k = 32 reflectors against <= ~100 trailing columns over
// thousands of rows) and of the sparsifier applications (k = rank against a
// few hundred rows): latency, not flops, is the bound (reference
// `apply_panel_left` / `_apply_sparsify_scaled`, `kernels/__init__.py:
// 140-171`, `factor.py:600-616`).
//
// Decomposition: a job's C is cut into 32-column tiles; each tile is owned by
// one thread-block CLUSTER of CL CTAs that split the rows.  CTA q:
//   1. W_q = V[rows_q]^T C[rows_q, tile]          (k x 32, shared memory)
//   2. W = sum_q W_q  over DSMEM, rank order      (identical in every CTA)
//   3. W2 = op(T) W
//   4. C[rows_q, tile] -= V[rows_q] W2
// Rows are streamed through shared memory in chunks of WYF_RC; when a CTA's
// rows fit one chunk (m <= CL * WYF_RC) the chunk stays resident between
// steps 1 and 4 and C is read once.  Summation order over rows is fixed per
// CTA and the cluster reduction runs in rank order: results are
// deterministic.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spq {

constexpr int WYF_NT = 256;
constexpr int WYF_TC = 32;    // columns per tile
constexpr int WYF_RC = 128;   // rows per shared-memory chunk
constexpr int WYF_LDS = WYF_RC + 1;

template <int KM>
struct WyfSmem {
  double Vs[KM][WYF_LDS];        // V chunk, column-major (row index fastest)
  double Cs[WYF_TC][WYF_LDS];    // C tile chunk
  double Wp[KM][WYF_TC];         // this CTA's partial V^T C (read remotely)
  double W2[KM][WYF_TC];         // reduced W, then op(T) W
};

__device__ __forceinline__ const WyfJob* wyf_find(const WyfJob* jobs, int njobs, int tile) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {   // last job with tile0 <= tile
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return jobs + lo;
}

// Chunk loads: all global loads of a chunk are issued before any shared
// store (a fully unrolled register batch), so their latencies overlap
// instead of serialising one ~1 us HBM/L2 round trip per loop iteration.
template <int NR, int LD>
__device__ __forceinline__ void wyf_load_mat(double (*dst)[LD], const double* src, int64_t ld,
                                             int r0, int nr, int ncols) {
  constexpr int PER = NR * WYF_RC / WYF_NT;
  double t[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * WYF_NT;
    const int r = e % WYF_RC, i = e / WYF_RC;
    t[u] = (r < nr && i < ncols) ? __ldg(src + (int64_t)(r0 + r) + (int64_t)i * ld) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * WYF_NT;
    dst[e / WYF_RC][e % WYF_RC] = t[u];
  }
}

template <int KM>
__device__ __forceinline__ void wyf_load(WyfSmem<KM>& sh, const WyfJob& J, int r0, int nr, int c0,
                                         int nc, bool loadV) {
  if (loadV) {
    if (KM <= 32) {
      wyf_load_mat<KM, WYF_LDS>(sh.Vs, J.V, J.ldv, r0, nr, J.k);
    } else {   // two halves: bounded register batch
      wyf_load_mat<KM / 2, WYF_LDS>(sh.Vs, J.V, J.ldv, r0, nr, J.k);
      wyf_load_mat<KM / 2, WYF_LDS>(sh.Vs + KM / 2, J.V + (int64_t)(KM / 2) * J.ldv, J.ldv, r0, nr,
                                    J.k - KM / 2);
    }
  }
  wyf_load_mat<WYF_TC, WYF_LDS>(sh.Cs, J.C + (int64_t)c0 * J.ldc, J.ldc, r0, nr, nc);
}

template <int KM, int NP>
__global__ void __launch_bounds__(WYF_NT, 1) wyf_kernel(const WyfJob* __restrict__ jobs_g, int njobs,
                                                        const __grid_constant__ PList<WyfJob, NP> pl) {
  const WyfJob* jobs = NP > 1 ? pl.v : jobs_g;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  const int tile = blockIdx.x / CL;
  const WyfJob J = *wyf_find(jobs, njobs, tile);
  const int c0 = (tile - J.tile0) * WYF_TC;
  const int nc = min(WYF_TC, J.n - c0);
  const int k = J.k;
  // rows of this CTA: contiguous, balanced
  const int per = (J.m + CL - 1) / CL;
  const int rb = min(J.m, q * per), re = min(J.m, rb + per);
  const int nchunks = (re - rb + WYF_RC - 1) / WYF_RC;
  extern __shared__ __align__(16) unsigned char wyf_raw[];
  WyfSmem<KM>& sh = *reinterpret_cast<WyfSmem<KM>*>(wyf_raw);
  const int tid = threadIdx.x;
  const int j = tid & 31;        // tile column of this thread
  const int ig = tid >> 5;       // warp: reflector rows ig, ig+8, ...
  constexpr int NI = KM / 8;

  // ---- 1. partial W over this CTA's rows
  double w[NI];
#pragma unroll
  for (int s = 0; s < NI; ++s) w[s] = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int r0 = rb + ch * WYF_RC, nr = min(WYF_RC, re - r0);
    if (ch > 0) __syncthreads();
    wyf_load<KM>(sh, J, r0, nr, c0, nc, true);
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
      const double cv = sh.Cs[j][r];
#pragma unroll
      for (int s = 0; s < NI; ++s) w[s] = fma(sh.Vs[ig + 8 * s][r], cv, w[s]);
    }
  }
#pragma unroll
  for (int s = 0; s < NI; ++s) sh.Wp[ig + 8 * s][j] = w[s];

  // ---- 2. cluster sum in rank order (every CTA computes the same W)
  if (CL > 1) {
    cluster.sync();
#pragma unroll
    for (int s = 0; s < NI; ++s) w[s] = 0.0;
    for (int src = 0; src < CL; ++src) {
      const double* Wr = cluster.map_shared_rank(&sh.Wp[0][0], src);
#pragma unroll
      for (int s = 0; s < NI; ++s) w[s] += Wr[(ig + 8 * s) * WYF_TC + j];
    }
    // remote reads done: arrive now, wait before exiting (step 4 overlaps)
    asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
#pragma unroll
    for (int s = 0; s < NI; ++s) sh.W2[ig + 8 * s][j] = w[s];
  } else {
#pragma unroll
    for (int s = 0; s < NI; ++s) sh.W2[ig + 8 * s][j] = w[s];
  }
  __syncthreads();

  // ---- 3. W2 = op(T) W  (T upper triangular, k x k, ld ldt)
  double t2[NI];
#pragma unroll
  for (int s = 0; s < NI; ++s) {
    const int i = ig + 8 * s;
    double acc = 0.0;
    if (i < k) {
      if (J.trans) {   // (T^T W)[i] = sum_{l <= i} T[l, i] W[l]
        for (int l = 0; l <= i; ++l) acc = fma(J.T[l + (int64_t)i * J.ldt], sh.W2[l][j], acc);
      } else {         // (T W)[i] = sum_{l >= i} T[i, l] W[l]
        for (int l = i; l < k; ++l) acc = fma(J.T[i + (int64_t)l * J.ldt], sh.W2[l][j], acc);
      }
    }
    t2[s] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NI; ++s) sh.W2[ig + 8 * s][j] = t2[s];
  __syncthreads();
  double w2[KM];
#pragma unroll
  for (int i = 0; i < KM; ++i) w2[i] = sh.W2[i][j];

  // ---- 4. C -= V W2 over this CTA's rows
  for (int ch = 0; ch < nchunks; ++ch) {
    const int r0 = rb + ch * WYF_RC, nr = min(WYF_RC, re - r0);
    if (nchunks > 1) {   // chunk no longer resident: reload V and C
      __syncthreads();
      wyf_load<KM>(sh, J, r0, nr, c0, nc, true);
      __syncthreads();
    }
    for (int r = ig; r < nr; r += 8) {
      double cv = sh.Cs[j][r];
#pragma unroll
      for (int i = 0; i < KM; ++i) cv = fma(-sh.Vs[i][r], w2[i], cv);
      sh.Cs[j][r] = cv;
    }
    __syncthreads();
    for (int e = tid; e < WYF_TC * WYF_RC; e += WYF_NT) {
      const int r = e % WYF_RC, jj = e / WYF_RC;
      if (r < nr && jj < nc) J.C[(int64_t)(r0 + r) + (int64_t)(c0 + jj) * J.ldc] = sh.Cs[jj][r];
    }
  }
  if (CL > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

int wyf_kmax() { return 64; }

int wyf_cluster(int m) {   // CTAs per tile: rows resident in one chunk when possible
  int cl = (m + WYF_RC - 1) / WYF_RC;
  return cl < 1 ? 1 : (cl > 16 ? 16 : cl);
}

template <int KM, int NP>
static void launch_wyf_t(const WyfJob* d_jobs, const PList<WyfJob, NP>& pl, int njobs, int tiles,
                         int cl, cudaStream_t st) {
  const size_t smem = sizeof(WyfSmem<KM>);
  static bool init = false;
  if (!init) {
    CUDA_TRY(cudaFuncSetAttribute(wyf_kernel<KM, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_TRY(cudaFuncSetAttribute(wyf_kernel<KM, NP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles * cl));
  cfg.blockDim = dim3(WYF_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, wyf_kernel<KM, NP>, d_jobs, njobs, pl));
}

template <int KM>
static void launch_wyf_k(const WyfJob* d_jobs, const WyfJob* h_jobs, int njobs, int tiles, int cl,
                         cudaStream_t st) {
  if (d_jobs == nullptr) {
    if (njobs > PL_WYF) throw std::runtime_error("launch_wyf: parameter list too long");
    PList<WyfJob, PL_WYF> pl;
    for (int i = 0; i < njobs; ++i) pl.v[i] = h_jobs[i];
    launch_wyf_t<KM, PL_WYF>(nullptr, pl, njobs, tiles, cl, st);
  } else {
    launch_wyf_t<KM, 1>(d_jobs, PList<WyfJob, 1>{}, njobs, tiles, cl, st);
  }
}

void launch_wyf(const WyfJob* d_jobs, const WyfJob* h_jobs, int njobs, int tiles, int kmax, int cl,
                cudaStream_t st) {
  if (njobs <= 0 || tiles <= 0) return;
  if (kmax <= 32) launch_wyf_k<32>(d_jobs, h_jobs, njobs, tiles, cl, st);
  else if (kmax <= 64) launch_wyf_k<64>(d_jobs, h_jobs, njobs, tiles, cl, st);
  else throw std::runtime_error("wyf: k > 64");
}

}  // namespace spq
