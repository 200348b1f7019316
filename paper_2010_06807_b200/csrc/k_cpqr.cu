// Threshold column-pivoted Householder QR, the
// sparsification kernel: `cpqr_threshold` (kernels/_numba.py:120-167) with
// the reference's exact rules — trailing column norms RECOMPUTED every step
// (here fused into the update pass), argmax with the LOWEST current
// position winning ties, stop at step i >= 1 once max norm < eps * norm0
// (and i >= min_rank), swap, reflect, rank-1 update.
//
// One cooperative launch per interface: CTAs own contiguous ranges of
// physical columns; swaps are logical (every CTA keeps identical copies of
// the position <-> column maps in shared memory), so each step costs one
// grid-wide barrier: publish local argmax -> sync -> every CTA reduces the
// G candidates identically, recomputes the pivot reflector from the pivot
// column (deterministic block reduction) and updates its own columns.
//
// Also here: the sparsify preamble (`factor.py:583-604`: column norms of
// M = [A_np^T, A_pn], maxcol, ratio = min(eps/maxcol, 0.999999), the
// `ncols > 4|p|` column filter and its compaction) kept on the device so
// the host syncs once per interface, for the accepted rank.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace spq {

constexpr int CP_NT = 256;



__host__ __device__ __forceinline__ bool cpqr_maps_in_smem(int ncols_cap, int m) {
  return ncols_cap >= 0 && (size_t)(2 * ncols_cap + 2) * 4 + (size_t)m * 8 + 16 <= 200 * 1024;
}

__device__ __forceinline__ bool better(double v, int pos, double bv, int bpos) {
  // strict '>' scan in position order == max value, lowest position on ties
  return v > bv || (v == bv && pos < bpos);
}

__global__ void __launch_bounds__(CP_NT) cpqr_kernel(CpqrArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = CP_NT / 32;
  const int m = a.m;
  const int nk = *a.nk;
  const double eps = *a.eps;
  const int kmax = min(m, nk);
  const int cpc = (nk + G - 1) / G;
  const int c0 = min(nk, g * cpc), c1 = min(nk, c0 + cpc);

  extern __shared__ __align__(16) unsigned char smraw[];
  const bool smaps = !a.force_gmaps && cpqr_maps_in_smem(a.ncols_cap, m);
  int* pos_of = smaps ? reinterpret_cast<int*>(smraw)
                      : a.gmaps + (size_t)blockIdx.x * 2 * a.ncols_cap;   // [ncols_cap]
  int* phys_at = pos_of + a.ncols_cap;                                  // [ncols_cap]
  double* v = reinterpret_cast<double*>(smaps ? (void*)(phys_at + a.ncols_cap) : (void*)smraw);  // [m]
  __shared__ double red_v[NW];
  __shared__ int red_p[NW];
  __shared__ double sc[4];
  __shared__ int colpos_s[1];

  for (int j = tid; j < nk; j += CP_NT) { pos_of[j] = j; phys_at[j] = j; }

  // initial norms (rows 0..m-1), warp per column, then local best
  double bv = -1.0;
  int bp = 0x7fffffff;
  for (int j = c0 + warp; j < c1; j += NW) {
    const double* col = a.W + (int64_t)j * m;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += col[r] * col[r];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double nv = sqrt(s);
    if (better(nv, j, bv, bp)) { bv = nv; bp = j; }
  }
  if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; }
  __syncthreads();
  if (tid == 0) {
    double v0 = -1.0; int p0 = 0x7fffffff;
    for (int w = 0; w < NW; ++w) if (better(red_v[w], red_p[w], v0, p0)) { v0 = red_v[w]; p0 = red_p[w]; }
    a.slot_val[g] = v0;
    a.slot_pos[g] = p0;
  }

  double norm0 = 0.0;
  int r = kmax;
  for (int i = 0; i < kmax; ++i) {
    const int par = i & 1;
    grid.sync();
    // ---- global argmax (identical in every CTA): each thread loads one
    // CTA's candidate, then a fixed shuffle/shared-memory tree
    {
      double v0 = -1.0;
      int p0 = 0x7fffffff;
      for (int h = tid; h < G; h += CP_NT) {
        const double hv = a.slot_val[par * G + h];
        const int hp = a.slot_pos[par * G + h];
        if (better(hv, hp, v0, p0)) { v0 = hv; p0 = hp; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v0, o);
        const int op = __shfl_xor_sync(0xffffffffu, p0, o);
        if (better(ov, op, v0, p0)) { v0 = ov; p0 = op; }
      }
      if (lane == 0) { red_v[warp] = v0; red_p[warp] = p0; }
      __syncthreads();
      if (tid == 0) {
        double v1 = -1.0; int p1 = 0x7fffffff;
        for (int w = 0; w < NW; ++w) if (better(red_v[w], red_p[w], v1, p1)) { v1 = red_v[w]; p1 = red_p[w]; }
        sc[0] = v1;
        colpos_s[0] = p1;
      }
    }
    __syncthreads();
    const double nrm = sc[0];
    const int lp = colpos_s[0];     // logical position of the pivot
    if (i == 0) {
      norm0 = nrm;
      if (norm0 == 0.0) { r = 0; break; }
    } else if (nrm < eps * norm0 && i >= a.min_rank) {
      r = i;
      break;
    }
    // ---- logical swap of positions i and lp
    const int phys_p = phys_at[lp];
    const int phys_i = phys_at[i];
    __syncthreads();
    if (tid == 0) {
      phys_at[i] = phys_p; phys_at[lp] = phys_i;
      pos_of[phys_p] = i; pos_of[phys_i] = lp;
    }
    // ---- reflector from the pivot column (rows i..m-1)
    const double* x = a.W + (int64_t)phys_p * m;
    double s = 0.0;
    for (int rr = i + 1 + tid; rr < m; rr += CP_NT) s += x[rr] * x[rr];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red_v[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double sigma = 0.0;
      for (int w = 0; w < NW; ++w) sigma += red_v[w];
      const double alpha = x[i];
      double tau, beta, v0 = 1.0, zero = 0.0;
      if (sigma == 0.0) {
        zero = 1.0;
        if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
      } else {
        beta = sqrt(alpha * alpha + sigma);
        v0 = (alpha <= 0.0) ? alpha - beta : -sigma / (alpha + beta);
        tau = -v0 / beta;
      }
      sc[1] = tau; sc[2] = v0; sc[3] = zero;
      if (g == 0) { a.tau[i] = tau; a.beta[i] = beta; }
    }
    __syncthreads();
    const double tau = sc[1], v0 = sc[2];
    const bool zero = sc[3] != 0.0;
    for (int rr = i + tid; rr < m; rr += CP_NT)
      v[rr] = (rr == i) ? 1.0 : (zero ? 0.0 : x[rr] / v0);
    __syncthreads();
    if (g == 0)
      for (int rr = i + tid; rr < m; rr += CP_NT) a.V[rr + (int64_t)i * m] = v[rr];
    // ---- update own trailing columns, fused norm over rows i+1..m-1
    bv = -1.0;
    bp = 0x7fffffff;
    for (int j = c0 + warp; j < c1; j += NW) {
      const int pj = pos_of[j];
      if (pj <= i) continue;       // retired pivot columns (incl. this step's)
      double* col = a.W + (int64_t)j * m;
      double ns = 0.0;
      if (tau != 0.0) {
        double d = 0.0;
        for (int rr = i + lane; rr < m; rr += 32) d += v[rr] * col[rr];
#pragma unroll
        for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const double w = tau * d;
        for (int rr = i + lane; rr < m; rr += 32) {
          const double nv = col[rr] - w * v[rr];
          col[rr] = nv;
          if (rr > i) ns += nv * nv;
        }
      } else {
        for (int rr = i + 1 + lane; rr < m; rr += 32) ns += col[rr] * col[rr];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
      const double nv = sqrt(ns);
      if (better(nv, pj, bv, bp)) { bv = nv; bp = pj; }
    }
    if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; }
    __syncthreads();
    if (tid == 0) {
      double v1 = -1.0; int p1 = 0x7fffffff;
      for (int w = 0; w < NW; ++w) if (better(red_v[w], red_p[w], v1, p1)) { v1 = red_v[w]; p1 = red_p[w]; }
      a.slot_val[(par ^ 1) * G + g] = v1;
      a.slot_pos[(par ^ 1) * G + g] = p1;
    }
    // the pivot column's rows stay intact until every CTA has read x: the
    // owner writes beta/zeros in the finalize pass below
  }
  if (g == 0 && tid == 0) *a.rank = r;
  if (g == 0)
    for (int j = tid; j < nk; j += CP_NT) a.perm[j] = phys_at[j];
  if (a.finalize) {
    grid.sync();
    for (int j = c0 + warp; j < c1; j += NW) {
      const int pj = pos_of[j];
      if (pj >= r) continue;
      double* col = a.W + (int64_t)j * m;
      for (int rr = pj + lane; rr < m; rr += 32) col[rr] = (rr == pj) ? a.beta[pj] : 0.0;
    }
  }
}

size_t cpqr_smem_bytes(int ncols_cap, int m, bool force_gmaps) {
  if (!force_gmaps && cpqr_maps_in_smem(ncols_cap, m))
    return (size_t)(2 * ncols_cap + 2) * sizeof(int) + (size_t)m * sizeof(double) + 16;
  return (size_t)m * sizeof(double) + 16;
}

int cpqr_grid(int ncols, int nsm) {
  static int gmax = -1, per = -1;
  if (gmax < 0) {
    const char* e = getenv("SPQ_CPQR_GMAX");
    gmax = e ? atoi(e) : 0;
    const char* f = getenv("SPQ_CPQR_COLS_PER_CTA");
    per = f ? atoi(f) : 8;
    if (per < 1) per = 8;
  }
  int g = (ncols + per - 1) / per;
  if (g > nsm) g = nsm;
  if (gmax > 0 && g > gmax) g = gmax;
  if (g < 1) g = 1;
  return g;
}

void launch_cpqr(const CpqrArgs& a, int G, cudaStream_t st) {
  const size_t bytes = cpqr_smem_bytes(a.ncols_cap, a.m, a.force_gmaps != 0);
  static size_t configured = 0;
  if (bytes > configured) {   // the default 48 KB cap counts static + dynamic
    CUDA_TRY(cudaFuncSetAttribute(cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bytes));
    configured = bytes;
  }
  CpqrArgs args = a;
  void* params[] = {&args};
  CUDA_TRY(cudaLaunchCooperativeKernel((void*)cpqr_kernel, dim3(G), dim3(CP_NT), params, bytes,
                                       st));
}

// ------------------------------------------------------ sparsify preamble
// warp per column: squared norm of column j of M (m x n, ld m)
__global__ void colsq_kernel(const double* __restrict__ M, int m, int n, double* __restrict__ sq) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const double* col = M + (int64_t)w * m;
  double s = 0.0;
  for (int r = lane; r < m; r += 32) s += col[r] * col[r];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sq[w] = s;
}

// single CTA: maxcol, ratio, keep filter, compaction list
__global__ void __launch_bounds__(1024) sparsify_select_kernel(const double* __restrict__ sq,
                                                               int m, int n, double eps_user,
                                                               int* __restrict__ keep_idx,
                                                               int* nk, double* ratio_out,
                                                               double* maxcol_out, int allow_filter) {
  __shared__ double red[32];
  __shared__ int cnt[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double mx = 0.0;
  for (int j = tid; j < n; j += blockDim.x) mx = fmax(mx, sqrt(sq[j]));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    red[0] = v;
  }
  __syncthreads();
  const double maxcol = red[0];
  const double ratio = (maxcol == 0.0) ? 0.0 : fmin(eps_user / maxcol, 0.999999);
  // scaled route only (factor.py:600-604); the unscaled route runs the CPQR
  // on the full target (factor.py:606-611)
  const bool filter = allow_filter && maxcol > 0.0 && n > 4 * m;
  const double thr = ratio * maxcol;
  // ordered compaction in chunks of blockDim
  int base = 0;
  for (int j0 = 0; j0 < n; j0 += blockDim.x) {
    const int j = j0 + tid;
    const bool keep = j < n && (!filter || sqrt(sq[j]) >= thr);
    const unsigned ball = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) cnt[warp] = __popc(ball);
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const int c = cnt[w]; cnt[w] = acc; acc += c; }
      cnt[32] = acc;
    }
    __syncthreads();
    if (keep) keep_idx[base + cnt[warp] + __popc(ball & ((1u << lane) - 1u))] = j;
    base += cnt[32];
    __syncthreads();
  }
  if (tid == 0) { *nk = base; *ratio_out = ratio; *maxcol_out = maxcol; }
}

// W[:, t] = M[:, keep_idx[t]] for t < *nk
// (column index on grid x: candidate counts exceed gridDim.y's 65535 limit
// on 3D problems)
__global__ void gather_cols_kernel(const double* __restrict__ M, int m, const int* __restrict__ idx,
                                   const int* nk, double* __restrict__ W) {
  const int t = blockIdx.x;
  if (t >= *nk) return;
  const double* src = M + (int64_t)idx[t] * m;
  double* dst = W + (int64_t)t * m;
  for (int r = blockIdx.y * blockDim.x + threadIdx.x; r < m; r += gridDim.y * blockDim.x)
    dst[r] = src[r];
}

void launch_sparsify_prep(const double* M, int m, int n, double eps, double* sq, int* keep_idx,
                          int* nk, double* ratio, double* maxcol, double* W, cudaStream_t st,
                          int allow_filter) {
  if (n > 0) colsq_kernel<<<(n * 32 + 255) / 256, 256, 0, st>>>(M, m, n, sq); SPQ_LAUNCH_CHECK();
  sparsify_select_kernel<<<1, 1024, 0, st>>>(sq, m, n, eps, keep_idx, nk, ratio, maxcol, allow_filter); SPQ_LAUNCH_CHECK();
  if (n > 0) gather_cols_kernel<<<dim3(n, (unsigned)std::min((m + 255) / 256, 64)), 256, 0, st>>>(M, m, keep_idx, nk, W); SPQ_LAUNCH_CHECK();
}

// ---- the same three steps for every interface of a wave in three launches
// (a wave launched them per interface: 3 dependent ~5 us launches each).
// Per column / per interface the arithmetic is that of the kernels above.
constexpr int PL_PREP = 16;

__global__ void colsq_batch_kernel(const PrepJob* __restrict__ jobs_g,
                                   const __grid_constant__ PList<PrepJob, PL_PREP> pl) {
  const PrepJob& J = (jobs_g ? jobs_g : pl.v)[blockIdx.y];
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= J.n) return;
  const double* col = J.M + (int64_t)w * J.m;
  double s = 0.0;
  for (int r = lane; r < J.m; r += 32) s += col[r] * col[r];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) J.sq[w] = s;
}

__global__ void __launch_bounds__(1024) select_batch_kernel(const PrepJob* __restrict__ jobs_g,
                                                            double eps_user,
                                                            const __grid_constant__ PList<PrepJob, PL_PREP> pl) {
  const PrepJob& J = (jobs_g ? jobs_g : pl.v)[blockIdx.x];
  const double* sq = J.sq;
  const int m = J.m, n = J.n;
  __shared__ double red[32];
  __shared__ int cnt[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double mx = 0.0;
  for (int j = tid; j < n; j += blockDim.x) mx = fmax(mx, sqrt(sq[j]));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    red[0] = v;
  }
  __syncthreads();
  const double maxcol = red[0];
  const double ratio = (maxcol == 0.0) ? 0.0 : fmin(eps_user / maxcol, 0.999999);
  const bool filter = J.allow_filter && maxcol > 0.0 && n > 4 * m;
  const double thr = ratio * maxcol;
  int base = 0;
  for (int j0 = 0; j0 < n; j0 += blockDim.x) {
    const int j = j0 + tid;
    const bool keep = j < n && (!filter || sqrt(sq[j]) >= thr);
    const unsigned ball = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) cnt[warp] = __popc(ball);
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const int c = cnt[w]; cnt[w] = acc; acc += c; }
      cnt[32] = acc;
    }
    __syncthreads();
    if (keep) J.keep_idx[base + cnt[warp] + __popc(ball & ((1u << lane) - 1u))] = j;
    base += cnt[32];
    __syncthreads();
  }
  if (tid == 0) { *J.nk = base; *J.ratio = ratio; *J.maxcol = maxcol; }
}

__global__ void gather_cols_batch_kernel(const PrepJob* __restrict__ jobs_g,
                                         const __grid_constant__ PList<PrepJob, PL_PREP> pl) {
  const PrepJob& J = (jobs_g ? jobs_g : pl.v)[blockIdx.z];
  const int t = blockIdx.x;
  if (t >= *J.nk) return;
  const int m = J.m;
  const double* src = J.M + (int64_t)J.keep_idx[t] * m;
  double* dst = J.W + (int64_t)t * m;
  for (int r = blockIdx.y * blockDim.x + threadIdx.x; r < m; r += gridDim.y * blockDim.x)
    dst[r] = src[r];
}

int sparsify_prep_plist_max() { return PL_PREP; }

// d_jobs == nullptr: the list travels in the launch parameters (njobs <= PL_PREP)
void launch_sparsify_prep_batch(const PrepJob* d_jobs, const PrepJob* h_jobs, int njobs, double eps,
                                cudaStream_t st) {
  if (njobs <= 0) return;
  PList<PrepJob, PL_PREP> pl;
  if (!d_jobs) {
    if (njobs > PL_PREP) throw std::runtime_error("launch_sparsify_prep_batch: parameter list too long");
    for (int i = 0; i < njobs; ++i) pl.v[i] = h_jobs[i];
  }
  constexpr int CHUNK = 16384;   // grid y / z limits (65535)
  for (int j0 = 0; j0 < njobs; j0 += CHUNK) {
    const int nj = std::min(CHUNK, njobs - j0);
    const PrepJob* dj = d_jobs ? d_jobs + j0 : nullptr;
    int nmax = 0, mmax = 0;
    for (int i = j0; i < j0 + nj; ++i) {
      nmax = std::max(nmax, h_jobs[i].n);
      mmax = std::max(mmax, h_jobs[i].m);
    }
    if (nmax > 0) {
      colsq_batch_kernel<<<dim3((nmax * 32 + 255) / 256, nj), 256, 0, st>>>(dj, pl);
      SPQ_LAUNCH_CHECK();
    }
    select_batch_kernel<<<nj, 1024, 0, st>>>(dj, eps, pl); SPQ_LAUNCH_CHECK();
    if (nmax > 0) {
      gather_cols_batch_kernel<<<dim3(nmax, (unsigned)std::min((mmax + 255) / 256, 64), nj), 256, 0, st>>>(dj, pl);
      SPQ_LAUNCH_CHECK();
    }
  }
}

}  // namespace spq

// ===================================================================== batched
// CTA-resident threshold CPQR: one CTA per problem, the m x n candidate
// matrix held in shared memory (physical column swaps, exactly the
// reference's sequence), __syncthreads-only steps.  Used for every
// interface whose M fits (and for BASELINE config 2's 4096 x (64x192)
// batch).  Same semantics as cpqr_kernel / kernels/_numba.py:120-167.
namespace spq {

constexpr int CB_NT = 512;
constexpr int CB_NW = CB_NT / 32;

__device__ __forceinline__ void argmax_merge(double& v, int& p, double ov, int op) {
  if (ov > v || (ov == v && op < p)) { v = ov; p = op; }
}

struct CbLayout {
  int lds, n1, m1;
  __host__ __device__ CbLayout(int m, int n) : lds(m | 1), n1(n > 0 ? n : 1), m1(m > 0 ? m : 1) {}
  // doubles: S (lds*n1) | nrm (n1) | v (m1) | dpart (8*n1) | npart (8*n1) | redv (CB_NW)
  // ints after: perm (n1) | redp (CB_NW)
  __host__ __device__ size_t doubles() const {
    return (size_t)lds * n1 + n1 + m1 + 16 * (size_t)n1 + CB_NW;
  }
  __host__ __device__ size_t bytes() const { return doubles() * 8 + ((size_t)n1 + CB_NW) * 4; }
};

__global__ void __launch_bounds__(CB_NT) cpqr_cta_kernel(const CpqrJob* __restrict__ jobs) {
  const CpqrJob J = jobs[blockIdx.x];
  const int m = J.m;
  const int n = J.nk ? *J.nk : J.n;
  const double eps = *J.eps;
  const int kmax = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) double cs[];
  const CbLayout L(m, J.ncap);
  const int lds = L.lds;
  double* S = cs;
  double* nrm = S + (size_t)lds * L.n1;
  double* v = nrm + L.n1;
  double* dpart = v + L.m1;
  double* npart = dpart + 8 * L.n1;
  double* redv = npart + 8 * L.n1;
  int* perm = reinterpret_cast<int*>(redv + CB_NW);
  int* redp = perm + L.n1;
  __shared__ double sc[4];
  __shared__ int sp[1];

  for (int e = tid; e < m * n; e += CB_NT) {
    const int a = e % m, j = e / m;
    S[a + j * lds] = J.W[a + (int64_t)j * J.ldw];
  }
  for (int j = tid; j < n; j += CB_NT) perm[j] = j;
  int P = CB_NT / (n > 0 ? n : 1);
  P = P >= 8 ? 8 : (P >= 4 ? 4 : (P >= 2 ? 2 : 1));
  __syncthreads();
  for (int t = tid; t < n * P; t += CB_NT) {
    const int j = t % n, pr = t / n;
    double s = 0.0;
    for (int a = pr; a < m; a += P) s += S[a + j * lds] * S[a + j * lds];
    npart[pr * L.n1 + j] = s;
  }
  __syncthreads();
  for (int j = tid; j < n; j += CB_NT) {
    double s = 0.0;
    for (int pr = 0; pr < P; ++pr) s += npart[pr * L.n1 + j];
    nrm[j] = sqrt(s);
  }
  __syncthreads();

  double norm0 = 0.0;
  int r = kmax;
  for (int i = 0; i < kmax; ++i) {
    double bv = -1.0;
    int bp = 0x7fffffff;
    for (int j = i + tid; j < n; j += CB_NT) argmax_merge(bv, bp, nrm[j], j);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      argmax_merge(bv, bp, ov, op);
    }
    if (lane == 0) { redv[warp] = bv; redp[warp] = bp; }
    __syncthreads();
    if (tid == 0) {
      double v1 = -1.0; int p1 = 0x7fffffff;
      for (int w = 0; w < CB_NW; ++w) argmax_merge(v1, p1, redv[w], redp[w]);
      sc[0] = v1;
      sp[0] = p1;
    }
    __syncthreads();
    const double best = sc[0];
    const int p = sp[0];
    if (i == 0) {
      norm0 = best;
      if (norm0 == 0.0) { r = 0; break; }
    } else if (best < eps * norm0 && i >= J.min_rank) {
      r = i;
      break;
    }
    if (p != i) {   // physical swap, like the reference
      for (int a = tid; a < m; a += CB_NT) {
        const double t0 = S[a + i * lds];
        S[a + i * lds] = S[a + p * lds];
        S[a + p * lds] = t0;
      }
      if (tid == 0) {
        const double tn = nrm[i]; nrm[i] = nrm[p]; nrm[p] = tn;
        const int tp = perm[i]; perm[i] = perm[p]; perm[p] = tp;
      }
    }
    __syncthreads();
    double s = 0.0;
    for (int a = i + 1 + tid; a < m; a += CB_NT) s += S[a + i * lds] * S[a + i * lds];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) redv[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double sigma = 0.0;
      for (int w = 0; w < CB_NW; ++w) sigma += redv[w];
      const double alpha = S[i + i * lds];
      double tau, beta, v0 = 1.0, zero = 0.0;
      if (sigma == 0.0) {
        zero = 1.0;
        if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
      } else {
        beta = sqrt(alpha * alpha + sigma);
        v0 = (alpha <= 0.0) ? alpha - beta : -sigma / (alpha + beta);
        tau = -v0 / beta;
      }
      sc[1] = tau; sc[2] = v0; sc[3] = zero;
      J.tau[i] = tau;
      J.beta[i] = beta;
    }
    __syncthreads();
    const double tau = sc[1], v0 = sc[2];
    const bool zero = sc[3] != 0.0;
    for (int a = i + tid; a < m; a += CB_NT) {
      const double va = (a == i) ? 1.0 : (zero ? 0.0 : S[a + i * lds] / v0);
      v[a] = va;
      J.V[a + (int64_t)i * J.ldv] = va;
    }
    __syncthreads();
    const int nt = n - i - 1;
    if (tau != 0.0 && nt > 0) {
      for (int t = tid; t < nt * P; t += CB_NT) {
        const int j = i + 1 + t % nt, pr = t / nt;
        double d = 0.0;
        for (int a = i + pr; a < m; a += P) d += v[a] * S[a + j * lds];
        dpart[pr * L.n1 + j] = d;
      }
      __syncthreads();
      for (int t = tid; t < nt * P; t += CB_NT) {
        const int j = i + 1 + t % nt, pr = t / nt;
        double d = 0.0;
        for (int q = 0; q < P; ++q) d += dpart[q * L.n1 + j];
        const double w = tau * d;
        double ns = 0.0;
        for (int a = i + pr; a < m; a += P) {
          const double nv = S[a + j * lds] - w * v[a];
          S[a + j * lds] = nv;
          if (a > i) ns += nv * nv;
        }
        npart[pr * L.n1 + j] = ns;
      }
    } else {
      for (int t = tid; t < nt * P; t += CB_NT) {
        const int j = i + 1 + t % nt, pr = t / nt;
        double ns = 0.0;
        for (int a = i + 1 + pr; a < m; a += P) ns += S[a + j * lds] * S[a + j * lds];
        npart[pr * L.n1 + j] = ns;
      }
    }
    __syncthreads();
    for (int j = i + 1 + tid; j < n; j += CB_NT) {
      double ns = 0.0;
      for (int q = 0; q < P; ++q) ns += npart[q * L.n1 + j];
      nrm[j] = sqrt(ns);
    }
    if (tid == 0) S[i + i * lds] = J.beta[i];
    for (int a = i + 1 + tid; a < m; a += CB_NT) S[a + i * lds] = 0.0;
    __syncthreads();
  }
  if (tid == 0) *J.rank = r;
  for (int j = tid; j < n; j += CB_NT) J.perm[j] = perm[j];
  if (J.write_back)
    for (int e = tid; e < m * n; e += CB_NT) {
      const int a = e % m, j = e / m;
      J.W[a + (int64_t)j * J.ldw] = S[a + j * lds];
    }
}

size_t cpqr_cta_smem(int m, int ncap) { return CbLayout(m, ncap).bytes() + 64; }

void launch_cpqr_cta(const CpqrJob* d_jobs, int njobs, size_t smem, cudaStream_t st) {
  if (njobs <= 0) return;
  static size_t conf = 0;
  if (smem > conf) {
    CUDA_TRY(cudaFuncSetAttribute(cpqr_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(smem, 48 * 1024)));
    conf = smem;
  }
  cpqr_cta_kernel<<<njobs, CB_NT, smem, st>>>(d_jobs); SPQ_LAUNCH_CHECK();
}

}  // namespace spq

// ===================================================================== cluster
// Cluster-resident threshold CPQR: one thread-block cluster (CL <= 16 CTAs)
// per problem; CTA q owns physical columns [q*cpc, (q+1)*cpc) of the
// compacted candidate matrix in SHARED memory.  Per pivot step: one
// barrier.cluster; the CL local candidates and the winning column travel
// over DSMEM; swaps are logical (identical position maps in every CTA), so
// ties go to the lowest current position exactly as in the reference.
namespace spq {

constexpr int CC_NT = 512;
constexpr int CC_NW = CC_NT / 32;

struct CcLayout {
  int lds, cpc, n1, m1;
  __host__ __device__ CcLayout(int m, int ncap, int CL)
      : lds(m | 1), cpc((ncap + CL - 1) / CL), n1(ncap > 0 ? ncap : 1), m1(m > 0 ? m : 1) {}
  // doubles: S (lds*cpc) | x (m1) | dpart (8*cpc) | npart (8*cpc) | arow (cpc) | red (CC_NW) | xch (2*2)
  // ints:    lpos (cpc) | phys (n1) | redp (CC_NW)
  __host__ __device__ size_t doubles() const {
    return (size_t)lds * cpc + m1 + 17 * (size_t)cpc + CC_NW + 4;
  }
  __host__ __device__ size_t bytes() const {
    return doubles() * 8 + ((size_t)cpc + n1 + CC_NW) * 4 + 16;
  }
};

__global__ void __launch_bounds__(CC_NT) cpqr_cluster_kernel(const CpqrJob* __restrict__ jobs) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  const CpqrJob J = jobs[blockIdx.x / CL];
  const int m = J.m;
  const int n = J.nk ? *J.nk : J.n;
  const double eps = *J.eps;
  const int kmax = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const CcLayout L(m, J.ncap, CL);
  const int lds = L.lds, cpc = L.cpc;
  const int c0 = min(n, q * cpc), c1 = min(n, c0 + cpc), nloc = c1 - c0;
  extern __shared__ __align__(16) double cs[];
  double* S = cs;
  double* x = S + (size_t)lds * cpc;           // raw pivot column (rows i..m-1)
  double* dpart = x + L.m1;
  double* npart = dpart + 8 * (size_t)cpc;
  double* arow = npart + 8 * (size_t)cpc;      // row i of the own columns, this step
  double* red = arow + cpc;
  double* xch = red + CC_NW;                   // [2][2]: best value, best position
  int* lpos = reinterpret_cast<int*>(xch + 4);
  int* phys = lpos + cpc;
  int* redp = phys + L.n1;

  for (int e = tid; e < m * nloc; e += CC_NT) {
    const int a = e % m, j = e / m;
    S[a + j * lds] = J.W[a + (int64_t)(c0 + j) * J.ldw];
  }
  for (int j = tid; j < nloc; j += CC_NT) lpos[j] = c0 + j;
  for (int j = tid; j < n; j += CC_NT) phys[j] = j;
  int P = CC_NT / max(nloc, 1);
  P = P >= 8 ? 8 : (P >= 4 ? 4 : (P >= 2 ? 2 : 1));
  __syncthreads();
  // initial column norms -> local candidate
  for (int t = tid; t < nloc * P; t += CC_NT) {
    const int j = t % nloc, pr = t / nloc;
    double s = 0.0;
    for (int a = pr; a < m; a += P) s += S[a + j * lds] * S[a + j * lds];
    npart[pr * cpc + j] = s;
  }
  __syncthreads();
  auto publish_best = [&](int from, int parity, int pp_over, int pi_over, int i_over, int lp_over) {
    double bv = -1.0;
    int bp = 0x7fffffff;
    for (int j = tid; j < nloc; j += CC_NT) {
      int pj = lpos[j];
      if (c0 + j == pp_over) pj = i_over;
      else if (c0 + j == pi_over) pj = lp_over;
      if (pj < from) continue;
      double s = 0.0;
      for (int pr = 0; pr < P; ++pr) s += npart[pr * cpc + j];
      const double nv = sqrt(s);
      if (better(nv, pj, bv, bp)) { bv = nv; bp = pj; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
    }
    if (lane == 0) { red[warp] = bv; redp[warp] = bp; }
    __syncthreads();
    if (tid == 0) {
      double b1 = -1.0; int p1 = 0x7fffffff;
      for (int w = 0; w < CC_NW; ++w) if (better(red[w], redp[w], b1, p1)) { b1 = red[w]; p1 = redp[w]; }
      xch[parity * 2] = b1;
      xch[parity * 2 + 1] = (double)p1;
    }
  };
  publish_best(0, 0, -1, -1, 0, 0);

  double norm0 = 0.0;
  int r = kmax;
  for (int i = 0; i < kmax; ++i) {
    const int par = i & 1;
    cluster.sync();
    // every warp: argmax over the CL candidates (DSMEM), identical everywhere
    double best = -1.0;
    int lp = 0x7fffffff;
    if (lane < CL) {
      const double* X = cluster.map_shared_rank(xch, lane);
      best = X[par * 2];
      lp = (int)X[par * 2 + 1];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, lp, o);
      if (better(ov, op, best, lp)) { best = ov; lp = op; }
    }
    if (i == 0) {
      norm0 = best;
      if (norm0 == 0.0) { r = 0; break; }
    } else if (best < eps * norm0 && i >= J.min_rank) {
      r = i;
      break;
    }
    const int pp = phys[lp], pi = phys[i];
    const int qo = pp / cpc, jo = pp - qo * cpc;
    // raw pivot column from its owner (DSMEM), partial sigma
    const double* Xo = cluster.map_shared_rank(S, qo) + (size_t)jo * lds;
    double s = 0.0;
    for (int a = i + tid; a < m; a += CC_NT) {
      const double xa = Xo[a];
      x[a] = xa;
      if (a > i) s += xa * xa;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();                                           // (1)
    double sigma = 0.0;
    for (int w = 0; w < CC_NW; ++w) sigma += red[w];
    const double alpha = x[i];
    double tau, beta, v0 = 1.0;
    const bool zero = sigma == 0.0;
    if (zero) {
      if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
    } else {
      beta = sqrt(alpha * alpha + sigma);
      v0 = (alpha <= 0.0) ? alpha - beta : -sigma / (alpha + beta);
      tau = -v0 / beta;
    }
    if (q == 0) {
      for (int a = i + tid; a < m; a += CC_NT)
        J.V[a + (int64_t)i * J.ldv] = (a == i) ? 1.0 : (zero ? 0.0 : x[a] / v0);
      if (tid == 0) { J.tau[i] = tau; J.beta[i] = beta; }
    }
    // dot partials over rows > i with the raw pivot column
    for (int t = tid; t < nloc * P; t += CC_NT) {
      const int j = t % nloc, pr = t / nloc;
      int pj = lpos[j];
      if (c0 + j == pp) pj = i; else if (c0 + j == pi) pj = lp;
      if (pj <= i) continue;
      double d = 0.0;
      for (int a = i + 1 + pr; a < m; a += P) d += x[a] * S[a + j * lds];
      dpart[pr * cpc + j] = d;
      if (pr == 0) arow[j] = S[i + j * lds];
    }
    __syncthreads();                                           // (2)
    if (tid == 0) {   // logical swap of positions i and lp (identical in every CTA)
      phys[i] = pp;
      phys[lp] = pi;
      if (pp >= c0 && pp < c1) lpos[pp - c0] = i;
      if (pi >= c0 && pi < c1 && pi != pp) lpos[pi - c0] = lp;
    }
    // update + norm partials over rows > i
    for (int t = tid; t < nloc * P; t += CC_NT) {
      const int j = t % nloc, pr = t / nloc;
      int pj = lpos[j];
      if (c0 + j == pp) pj = i; else if (c0 + j == pi) pj = lp;
      if (pj <= i) continue;
      double* col = S + j * lds;
      double ns = 0.0;
      if (tau != 0.0) {
        double D = 0.0;
        for (int u = 0; u < P; ++u) D += dpart[u * cpc + j];
        const double aij = arow[j];
        const double w = zero ? tau * aij : tau * (aij + D / v0);   // w = tau v^T a_j
        const double coef = zero ? 0.0 : w / v0;                      // v_a = x_a / v0
        if (pr == 0) col[i] = aij - w;
        for (int a = i + 1 + pr; a < m; a += P) {
          const double nv = col[a] - coef * x[a];
          col[a] = nv;
          ns += nv * nv;
        }
      } else {
        for (int a = i + 1 + pr; a < m; a += P) ns += col[a] * col[a];
      }
      npart[pr * cpc + j] = ns;
    }
    __syncthreads();                                           // (3)
    publish_best(i + 1, par ^ 1, pp, pi, i, lp);               // (4) inside
  }
  if (q == 0 && tid == 0) *J.rank = r;
  __syncthreads();
  if (q == 0)
    for (int j = tid; j < n; j += CC_NT) J.perm[j] = phys[j];
  cluster.sync();   // no CTA leaves while others may read its shared memory
}

int cpqr_cluster_size(int m, int ncap) {
  static int clmax = -1;
  if (clmax < 0) {
    const char* e = getenv("SPQ_CPQR_CLMAX");
    clmax = e ? atoi(e) : 16;
  }
  for (int cl = 1; cl <= clmax; cl *= 2)
    if (CcLayout(m, ncap, cl).bytes() <= (size_t)200 * 1024) return cl;
  return 0;
}

size_t cpqr_cluster_smem(int m, int ncap, int cl) { return CcLayout(m, ncap, cl).bytes() + 64; }

void launch_cpqr_cluster(const CpqrJob* d_jobs, int njobs, int cl, size_t smem, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool init = false;
  if (!init) {
    CUDA_TRY(cudaFuncSetAttribute(cpqr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    CUDA_TRY(cudaFuncSetAttribute(cpqr_cluster_kernel,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * cl));
  cfg.blockDim = dim3(CC_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, cpqr_cluster_kernel, d_jobs));
}

}  // namespace spq

// ============================================================ spectral norms
// sigma_max of dropped blocks (`spectral_norm`, kernels/__init__.py:236-241;
// stats only, factor.py:643): power iteration on the Gram G = E E^T
// (f x f, ld f), one CTA per matrix, Rayleigh quotient to relative 1e-14.
namespace spq {

constexpr int PI_NT = 256;

__global__ void __launch_bounds__(PI_NT) power_iter_kernel(const PowerJob* __restrict__ jobs) {
  const PowerJob J = jobs[blockIdx.x];
  const int f = J.f, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) double pv[];
  double* x = pv;          // f
  double* y = pv + f;      // f
  __shared__ double red[PI_NT / 32];
  __shared__ double sc[3];
  if (f <= 0) { if (tid == 0) *J.out = 0.0; return; }
  for (int a = tid; a < f; a += PI_NT) x[a] = 1.0 + 0.001 * (a % 7);
  __syncthreads();
  double lam_prev = -1.0, lam = 0.0;
  for (int it = 0; it < 1000; ++it) {
    // y = G x ; lam = x^T y / x^T x ; x = y / ||y||
    double xy = 0.0, xx = 0.0, yy = 0.0;
    for (int a = tid; a < f; a += PI_NT) {
      double s = 0.0;
      for (int b = 0; b < f; ++b) s += J.G[a + (int64_t)b * f] * x[b];
      y[a] = s;
      xy += x[a] * s; xx += x[a] * x[a]; yy += s * s;
    }
    double vals[3] = {xy, xx, yy};
    for (int t = 0; t < 3; ++t) {
      double v = vals[t];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      if (tid == 0) {
        double sum = 0.0;
        for (int w = 0; w < PI_NT / 32; ++w) sum += red[w];
        sc[t] = sum;
      }
      __syncthreads();
    }
    lam = sc[1] > 0.0 ? sc[0] / sc[1] : 0.0;
    const double ny = sqrt(sc[2]);
    if (ny == 0.0) { lam = 0.0; break; }
    for (int a = tid; a < f; a += PI_NT) x[a] = y[a] / ny;
    __syncthreads();
    if (fabs(lam - lam_prev) <= 1e-14 * fabs(lam)) break;
    lam_prev = lam;
  }
  if (tid == 0) *J.out = sqrt(fmax(lam, 0.0));
}

void launch_power_iter(const PowerJob* d_jobs, int njobs, int fmax, cudaStream_t st) {
  if (njobs <= 0) return;
  const size_t smem = 2 * (size_t)(fmax > 0 ? fmax : 1) * sizeof(double);
  static size_t conf = 0;
  if (smem > conf) {   // the default 48 KB cap counts static + dynamic
    CUDA_TRY(cudaFuncSetAttribute(power_iter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    conf = smem;
  }
  power_iter_kernel<<<njobs, PI_NT, smem, st>>>(d_jobs); SPQ_LAUNCH_CHECK();
}

}  // namespace spq

// ============================================================ register-resident
// Cluster threshold CPQR with the candidate matrix held in REGISTERS.
//
// The smem-resident kernels stream the whole m x n matrix through shared
// memory three times per pivot step (dot, update, norm), which bounds a
// sparsify wave at ~2 us per step.  Here a group of TPC lanes owns C
// columns, lane s of the group holding rows s, s+TPC, ... (R per lane):
// the per-step work is register FMAs plus log2(TPC) shuffles per column.
// One step:
//   cluster.sync -> every warp reads the CL per-CTA candidates (DSMEM) and
//   picks the winner identically -> the CTA copies the winner's column
//   (published by its owner at the end of the previous step) from the
//   winning CTA into shared memory -> every warp forms sigma, alpha, tau,
//   v0 identically -> v = x / v0 (a thread per row) -> each group updates
//   its columns and their norms -> CTA argmax -> the owner group publishes
//   the CTA's best column for the next step.
// Logical swaps as in the other kernels (owners update the position of
// the pivot and of the column it displaces).  Semantics: `cpqr_threshold`
// (kernels/_numba.py:120-167), v = x / v0 like the reference.
namespace spq {

constexpr int RG_NT = 512;

__device__ __forceinline__ unsigned long long rg_pack(int pos, int phys) {
  return ((unsigned long long)(unsigned)pos << 32) | (unsigned)phys;
}
__device__ __forceinline__ bool rg_better(double v, unsigned long long k, double bv,
                                          unsigned long long bk) {
  return v > bv || (v == bv && (int)(k >> 32) < (int)(bk >> 32));
}

// DSMEM push exchange: at the end of every step each CTA pushes its best
// candidate (value, key, column) with ONE bulk copy per destination
// (cp.async.bulk shared::cta -> shared::cluster, completing on the
// destination's mbarrier).  After its wait, every CTA holds all CL
// candidates locally: no cluster barrier (which compiles to MEMBAR.GPU +
// L1 invalidation per step on sm_100a) and no remote loads.
__device__ __forceinline__ uint32_t rg_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t rg_mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void rg_arm(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void rg_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
  }
}

// clock64 stamps of the first versions of this kernel (512-thread CTAs,
// every warp repeating the scalar work; tools/cpqr_trace.py, profiles/r02c)
// showed a pivot step of ~7800 cycles that
// is bound by one SM's ISSUE throughput, not by the exchange (the mbarrier
// wait was ~200 cycles): 16 warps each repeated the winner scan, sigma, the
// sqrt/div scalars and the CTA-winner scan (fp64 division and 64-bit
// shuffles at 16x redundancy), and every CTA carried 16K matrix entries.
// Here:
//   * the CTA size is a launch parameter (128/256/512 threads, still 32
//     entries per thread): the planner spreads a problem over up to 16 CTAs
//     so each SM issues ~4x fewer fp64 / shuffle instructions per step;
//   * warp 0 alone waits for the candidates, picks the winner, forms sigma,
//     tau, v0 and writes v: the other warps sleep at the CTA barrier;
//   * every argmax (across column groups of a warp, across the warp
//     records of a CTA, across the CTA candidates) is three integer warp
//     reductions (redux.sync on the norm's high word, low word, position)
//     and a ballot instead of a 5-stage butterfly of 64-bit shuffles;
//   * cluster problems push the winner record with st.async from a few
//     warps (8-byte remote stores completing on the destination's mbarrier);
//   * norms over rows > i by predicated FMAs (no mask multiply);
//   * v = x * (1 / v0): one division per step instead of one per row
//     (within an ulp of the reference's x / v0, like the panel QR kernel).
__device__ __forceinline__ void rg_st_async(uint32_t raddr, double v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :: "r"(raddr), "d"(v), "r"(rmbar) : "memory");
}
// lane holding the best candidate of the warp: largest norm v (v < 0: none),
// then lowest position.  Every lane takes part; identical in every lane.
__device__ __forceinline__ int rg_argbest(double v, int pos) {
  const unsigned hi = v < 0.0 ? 0u : (unsigned)__double2hiint(v) + 1u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned lo = hi == mh ? (unsigned)__double2loint(v) : 0u;
  const unsigned ml = __reduce_max_sync(0xffffffffu, lo);
  const bool cand = hi == mh && lo == ml;
  const unsigned mp = __reduce_min_sync(0xffffffffu, cand ? (unsigned)pos : 0xffffffffu);
  return __ffs(__ballot_sync(0xffffffffu, cand && (unsigned)pos == mp)) - 1;
}

// records at least this long travel as cp.async.bulk copies (SPQ_CPQR_BULK_BYTES)
__constant__ uint32_t RG_BULK_BYTES = 512;

struct Rg3Layout {   // shared memory in doubles; rows padded to mp = tpc * R
  int m1, cl, rec, nw;  // rec = one candidate record: [value, key, column (m1)]
  __host__ __device__ Rg3Layout(int mp, int cl_, int nw_)
      : m1(mp > 0 ? ((mp + 1) & ~1) : 2), cl(cl_), rec(m1 + 2), nw(nw_) {}
  // vbuf (m1) | ST [nw][rec] | RX [2][cl][rec] | sc [4] | mbar [2]
  __host__ __device__ size_t sx() const { return (size_t)m1; }
  __host__ __device__ size_t rx() const { return sx() + (size_t)nw * rec; }
  __host__ __device__ size_t sco() const { return rx() + 2 * (size_t)cl * rec; }
  __host__ __device__ size_t bytes() const { return (sco() + 4 + 2) * 8 + 64; }
};

#ifdef SPQ_TRACE
// diagnostic build only (SPQ_TRACE=1 python -m paper_2010_06807_b200.build):
// per-step clock64 stamps of thread 0 / CTA 0, read by spq_debug_cpqr_trace
__device__ long long g_cpqr_trace[64 * 12];
#ifndef SPQ_TRACE_MMAX
#define SPQ_TRACE_MMAX 1000000   // -DSPQ_TRACE_MMAX=64: stamps of the small (typical 2D) interfaces only
#endif
#define RG_STAMP(slot) do { if (q == 0 && tid == 0 && i < 64 && m <= SPQ_TRACE_MMAX) g_cpqr_trace[i * 12 + (slot)] = clock64(); } while (0)
#else
#define RG_STAMP(slot) do { } while (0)
#endif

template <int R, int C>
__global__ void __launch_bounds__(RG_NT, 1) cpqr_reg_kernel(const CpqrJob* __restrict__ jobs_g,
                                                             int tpc,
                                                             const __grid_constant__ PList<CpqrJob, PL_SMALL> pl) {
  const CpqrJob* jobs = jobs_g ? jobs_g : pl.v;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  const bool multi = CL > 1;
  const int NT = (int)blockDim.x, NW = NT >> 5;
  const CpqrJob J = jobs[blockIdx.x / CL];
  const int m = J.m;
  const int n = J.nk ? *J.nk : J.n;
  const double eps = *J.eps;
  const int kmax = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = tid % tpc;
  const int grp = tid / tpc;
  const int cpc = (NT / tpc) * C;
  const int mp = tpc * R;
  const int ph0 = q * cpc + grp * C;
  extern __shared__ __align__(16) double rs[];
  const Rg3Layout L(mp, CL, NW);
  double* vbuf = rs;
  double* ST = rs + L.sx();
  double* RX = rs + L.rx();
  double* sc = rs + L.sco();   // [0] tau, [1] (lp << 32 | pp), [2] stop
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sc + 4);
  const uint32_t rec_bytes = (uint32_t)(L.rec * sizeof(double));
  const bool bulk = multi && rec_bytes >= RG_BULK_BYTES;   // exchange by bulk copies

  if (multi && tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(rg_smem(&mbar[b])) : "memory");
      rg_arm(rg_smem(&mbar[b]), rec_bytes * CL);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double x[C][R];
  int pos[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    pos[c] = ph0 + c;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int a = sub + tpc * r;
      x[c][r] = (ph0 + c < n && a < m) ? J.W[a + (int64_t)(ph0 + c) * J.ldw] : 0.0;
    }
  }
  for (int a = tid; a < L.m1; a += NT) vbuf[a] = 0.0;
  if (multi) cluster.sync(); else __syncthreads();

  // Every warp stages its best candidate record [value, key, column]; one
  // CTA barrier.  A record is rewritten only by the next step's stage(),
  // after that step's vbuf barrier, which every warp reaches after its reads
  // of this step's records (winner scan and reflector in warp 0, pushes).
  auto stage = [&](double bv, unsigned long long bk) {
    const int bl = rg_argbest(bv, (int)(bk >> 32));   // lanes of a group agree already
    double* st = ST + (size_t)warp * L.rec;
    if (lane / tpc == bl / tpc && bv >= 0.0) {       // the winning group writes its column
      const int cph = (int)(bk & 0xffffffffu);
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (ph0 + c == cph)
#pragma unroll
          for (int r = 0; r < R; ++r) st[2 + sub + tpc * r] = x[c][r];
    }
    if (lane == bl) { st[0] = bv; st[1] = __longlong_as_double((long long)bk); }
    if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> bulk copy
    __syncthreads();
  };
  // cluster problems: warp w pushes the CTA winner's record to the CTAs
  // w, w + NW, ...
  auto push = [&](int slot) {
    if (warp >= CL) return;
    const int w = lane < NW ? lane : 0;
    const double v = lane < NW ? ST[(size_t)w * L.rec] : -1.0;
    const unsigned long long k = (unsigned long long)__double_as_longlong(ST[(size_t)w * L.rec + 1]);
    const int cw = rg_argbest(v, lane < NW ? (int)(k >> 32) : 0x7fffffff);
    const double* src = ST + (size_t)cw * L.rec;
    for (int d = warp; d < CL; d += NW) {
      const uint32_t dst = rg_mapa(rg_smem(RX + ((size_t)slot * CL + q) * L.rec), d);
      const uint32_t mb = rg_mapa(rg_smem(&mbar[slot]), d);
      if (bulk) {   // long records: one bulk copy per destination (~21 B/cycle; st.async ~7 B/cycle)
        if (lane == 0) {
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes "
                       "[%0], [%1], %2, [%3];" :: "r"(dst), "r"(rg_smem(src)), "r"(rec_bytes), "r"(mb)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // staging reusable
        }
      } else {
        for (int idx = lane; idx < L.rec; idx += 32) rg_st_async(dst + 8u * (uint32_t)idx, src[idx], mb);
      }
    }
  };

  {   // initial norms (all rows)
    double bv = -1.0;
    unsigned long long bk = rg_pack(0x7fffffff, 0);
    double ns[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      ns[c] = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) ns[c] = fma(x[c][r], x[c][r], ns[c]);
    }
    for (int o = tpc >> 1; o; o >>= 1)
#pragma unroll
      for (int c = 0; c < C; ++c) ns[c] += __shfl_xor_sync(0xffffffffu, ns[c], o);
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (ph0 + c < n) {
        const double nv = sqrt(ns[c]);
        const unsigned long long k = rg_pack(pos[c], ph0 + c);
        if (rg_better(nv, k, bv, bk)) { bv = nv; bk = k; }
      }
    if (kmax > 0) {
      stage(bv, bk);
      if (multi) push(0);
    }
  }

  double norm0 = 0.0;   // warp 0
  int r_out = kmax;
  for (int i = 0; i < kmax; ++i) {
    RG_STAMP(0);
    if (warp == 0) {
      // ---- candidates -> winner -> reflector scalars -> v (warp 0 only)
      const double* recs;
      int nrec;
      if (multi) {
        const int slot = i & 1;
        rg_wait(rg_smem(&mbar[slot]), (uint32_t)((i >> 1) & 1));
        if (lane == 0) rg_arm(rg_smem(&mbar[slot]), rec_bytes * CL);   // for step i + 2
        recs = RX + (size_t)slot * CL * L.rec;
        nrec = CL;
      } else {
        recs = ST;
        nrec = NW;
      }
      RG_STAMP(1);
      const int w = lane < nrec ? lane : 0;
      const double cv = lane < nrec ? recs[(size_t)w * L.rec] : -1.0;
      const unsigned long long ck = (unsigned long long)__double_as_longlong(recs[(size_t)w * L.rec + 1]);
      const int wl = rg_argbest(cv, lane < nrec ? (int)(ck >> 32) : 0x7fffffff);
      const double best = __shfl_sync(0xffffffffu, cv, wl);
      const unsigned long long bk = __shfl_sync(0xffffffffu, ck, wl);
      RG_STAMP(2);
      bool stop = false;
      if (i == 0) {
        norm0 = best;
        if (norm0 == 0.0) { r_out = 0; stop = true; }
      } else if (best < eps * norm0 && i >= J.min_rank) {
        r_out = i;
        stop = true;
      }
      if (!stop) {
        const double* Xr = recs + (size_t)wl * L.rec + 2;
        double sg = 0.0;
        for (int a = i + 1 + lane; a < m; a += 32) sg = fma(Xr[a], Xr[a], sg);
#pragma unroll
        for (int o = 16; o; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
        RG_STAMP(3);
        const double alpha = Xr[i];
        // v0 = alpha - beta (alpha <= 0) or -sigma / (alpha + beta); 1 / v0 and
        // tau = -v0 / beta are formed from alpha, beta, sigma directly so the
        // two quotients do not wait for each other (within an ulp or two of
        // the reference's values, kernels/_numba.py:15-35)
        double tau, beta, inv0 = 0.0;
        if (sg == 0.0) {
          if (alpha >= 0.0) { tau = 0.0; beta = alpha; } else { tau = 2.0; beta = -alpha; }
        } else {
          house_scalars(alpha, sg, tau, beta, inv0);
        }
        // v (zero outside rows i..m-1: row i-1 is cleared, rows < i-1 were)
        for (int a = i + lane; a < m; a += 32) {
          const double va = (a == i) ? 1.0 : Xr[a] * inv0;
          vbuf[a] = va;
          if (q == 0) J.V[a + (int64_t)i * J.ldv] = va;
        }
        if (lane == 0) {
          if (i > 0) vbuf[i - 1] = 0.0;
          sc[0] = tau;
          sc[1] = __longlong_as_double((long long)bk);
          if (q == 0) { J.tau[i] = tau; J.beta[i] = beta; }
        }
      }
      if (lane == 0) sc[2] = stop ? 1.0 : 0.0;
    }
    RG_STAMP(4);
    __syncthreads();
    RG_STAMP(5);
    if (sc[2] != 0.0) break;
    const double tau = sc[0];
    const unsigned long long bk = (unsigned long long)__double_as_longlong(sc[1]);
    const int lp = (int)(bk >> 32), pp = (int)(bk & 0xffffffffu);
    // ---- own columns: swap bookkeeping, update, norms over rows > i
    double vr[R];
    bool below[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      vr[r] = vbuf[sub + tpc * r];
      below[r] = sub + tpc * r > i;
    }
    bool act[C];
    double d[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (ph0 + c == pp) pos[c] = i;                 // the pivot retires at position i
      else if (pos[c] == i) pos[c] = lp;             // displaced by the swap
      act[c] = ph0 + c < n && ph0 + c != pp && pos[c] > i;
      d[c] = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) d[c] = fma(vr[r], x[c][r], d[c]);
    }
    for (int o = tpc >> 1; o; o >>= 1)
#pragma unroll
      for (int c = 0; c < C; ++c) d[c] += __shfl_xor_sync(0xffffffffu, d[c], o);
    RG_STAMP(6);
    double ns[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double w = act[c] ? tau * d[c] : 0.0;
      ns[c] = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[c][r] = fma(-w, vr[r], x[c][r]);
        if (below[r]) ns[c] = fma(x[c][r], x[c][r], ns[c]);
      }
    }
    for (int o = tpc >> 1; o; o >>= 1)
#pragma unroll
      for (int c = 0; c < C; ++c) ns[c] += __shfl_xor_sync(0xffffffffu, ns[c], o);
    double bv = -1.0;
    unsigned long long bkk = rg_pack(0x7fffffff, 0);
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (act[c]) {
        const double nv = sqrt(ns[c]);
        const unsigned long long k = rg_pack(pos[c], ph0 + c);
        if (rg_better(nv, k, bv, bkk)) { bv = nv; bkk = k; }
      }
    RG_STAMP(7);
    // no push after the last step: nobody would wait for it, and a remote
    // store still in flight when its destination CTA exits lands in shared
    // memory that may already belong to another CTA
    if (i + 1 < kmax) {
      stage(bv, bkk);
      RG_STAMP(8);
      if (multi) push((i & 1) ^ 1);
      RG_STAMP(9);
    }
  }
  if (q == 0 && tid == 0) *J.rank = r_out;
  if (sub == 0)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (ph0 + c < n) J.perm[pos[c]] = ph0 + c;
  // every push addressed to this CTA was waited for; keep the CTAs resident
  // until all of them issued theirs
  if (multi)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}

// variant v: (R, C) = (16,2), (8,4), (4,8).  Plan of one problem: lanes per
// column tpc (power of two, tpc * R >= m), CTA size nt and cluster size (0:
// no plan).  The smallest CTA (128, 256, 512 threads) whose cluster still
// holds all n columns wins: a pivot step is bound by one SM's issue rate, so
// the columns are spread as widely as the cluster limit allows
// (SPQ_CPQR_NTMIN / SPQ_CPQR_CLMAX narrow the choice for A/B runs).
constexpr int RG_NVAR = 5;
static const int RG_R[RG_NVAR] = {16, 8, 4, 16, 8}, RG_C[RG_NVAR] = {2, 4, 8, 1, 2};
int cpqr_reg_nvar() { return RG_NVAR; }
int cpqr_reg_rows(int v) { return RG_R[v]; }
int cpqr_reg_elems(int v) { return RG_R[v] * RG_C[v]; }

int cpqr_reg_plan(int m, int n, int v, int* tpc_out, int* nt_out) {
  const int* RR = RG_R;
  const int* CC = RG_C;
  static int clmax = -1, ntmin = 128;
  if (clmax < 0) {
    const char* e = getenv("SPQ_CPQR_CLMAX");
    clmax = e ? atoi(e) : 16;
    const char* f = getenv("SPQ_CPQR_NTMIN");
    if (f) ntmin = std::max(32, std::min(RG_NT, atoi(f)));
  }
  if (m <= 0 || n <= 0) return 0;
  const int R = RR[v], C = CC[v];
  int tpc = 1;
  while (tpc * R < m) tpc *= 2;
  if (tpc > 32) return 0;
  // every CTA sends its candidate column to all CL CTAs each step (8-byte
  // remote stores): prefer plans whose exchange cl * rows stays <= 2048
  for (int pass = 0; pass < 2; ++pass)
    for (int nt = ntmin; nt <= RG_NT; nt *= 2) {
      if (nt < tpc || nt < 32) continue;
      const int cpc = (nt / tpc) * C;
      int cl = 1;
      while (cl * cpc < n) cl *= 2;
      if (cl > clmax || cl > 16) continue;
      if (pass == 0 && cl * tpc * R > 2048) continue;
      *tpc_out = tpc;
      *nt_out = nt;
      return cl;
    }
  return 0;
}

size_t cpqr_reg_smem(int mp, int cl, int nt) {   // mp = tpc * R
  return Rg3Layout(mp, cl, nt / 32).bytes();
}

template <int R, int C>
static void launch_rg(const CpqrJob* d_jobs, const PList<CpqrJob, PL_SMALL>& pl, int njobs, int cl,
                      int tpc, int nt, size_t smem, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    CUDA_TRY(cudaFuncSetAttribute(cpqr_reg_kernel<R, C>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CUDA_TRY(cudaFuncSetAttribute(cpqr_reg_kernel<R, C>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (const char* e = getenv("SPQ_CPQR_BULK_BYTES")) {   // A/B runs
      const uint32_t v = (uint32_t)strtoul(e, nullptr, 10);
      CUDA_TRY(cudaMemcpyToSymbol(RG_BULK_BYTES, &v, sizeof v));
    }
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * cl));
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, cpqr_reg_kernel<R, C>, d_jobs, tpc, pl));
}

void launch_cpqr_reg(const CpqrJob* d_jobs, const CpqrJob* h_jobs, int njobs, int v, int cl, int tpc,
                     int nt, size_t smem, cudaStream_t st) {
  if (njobs <= 0) return;
  PList<CpqrJob, PL_SMALL> pl;
  if (!d_jobs) {
    if (njobs > PL_SMALL) throw std::runtime_error("launch_cpqr_reg: parameter list too long");
    for (int i = 0; i < njobs; ++i) pl.v[i] = h_jobs[i];
  }
  switch (v) {
    case 0: launch_rg<16, 2>(d_jobs, pl, njobs, cl, tpc, nt, smem, st); break;
    case 1: launch_rg<8, 4>(d_jobs, pl, njobs, cl, tpc, nt, smem, st); break;
    case 2: launch_rg<4, 8>(d_jobs, pl, njobs, cl, tpc, nt, smem, st); break;
    case 3: launch_rg<16, 1>(d_jobs, pl, njobs, cl, tpc, nt, smem, st); break;
    case 4: launch_rg<8, 2>(d_jobs, pl, njobs, cl, tpc, nt, smem, st); break;
    default: throw std::runtime_error("cpqr_reg: bad variant");
  }
}

}  // namespace spq

#ifdef SPQ_TRACE
extern "C" int spq_debug_cpqr_trace(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, spq::g_cpqr_trace, sizeof(long long) * (size_t)(n < 64 * 12 ? n : 64 * 12));
}
#endif
