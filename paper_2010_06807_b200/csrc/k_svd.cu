// Extreme singular values of small dense blocks: one-sided (Hestenes) Jacobi.
//
// The unscaled sparsification route (reference factor.py:557-566, 660-709)
// needs three LAPACK-SVD numbers per interface:
//   * sigma_min / sigma_max of the column stack [A_pp; A_np] — sigma_min sets
//     the weight 1/sigma_min of the coupling block in the CPQR target and
//     must carry full relative accuracy (it moves every pivot decision);
//   * ||R_fn||_2 — compared with eps (1 + 1e-8) to decide rank escalation;
//   * ||E1||_2 — the `dropped` statistic.
// The host reduces the first to the R factor of a QR (same singular values),
// the others to Gram matrices (their largest eigenvalue carries full relative
// accuracy).  One-sided Jacobi on the columns of such an n x n block yields
// singular values with high relative accuracy (column-scaled rotations,
// Demmel-Veselic), which a Gram / eigenvalue route would not give sigma_min.
//
// Layout: one CTA per job, the block in global memory (col-major, lda; it is
// small and L2-resident), modified in place.  Round-robin (circle-method)
// ordering: every round rotates n/2 disjoint column pairs, one warp per
// pair, dot products by warp shuffles; a sweep is n-1 rounds; sweeps repeat
// until no pair is rotated.  Outputs: the largest and smallest column norm.
#include "common.cuh"

namespace spq {

constexpr int SV_NT = 512;
constexpr int SV_NW = SV_NT / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(SV_NT) jacobi_sv_kernel(const SvJob* __restrict__ jobs) {
  const SvJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n, lda = J.lda;
  double* A = J.A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int rotated;
  __shared__ double red[SV_NW][2];
  if (n <= 0 || m <= 0) {
    if (threadIdx.x == 0) { *J.smax = 0.0; *J.smin = 0.0; }
    return;
  }
  const int np2 = n + (n & 1);      // even player count (one bye when n is odd)
  const int nr = np2 - 1;            // rounds per sweep
  const double tol = 1e-15 * sqrt((double)m);
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int t = 0; t < nr; ++t) {
      for (int k = warp; k < np2 / 2; k += SV_NW) {
        int a, b;
        if (k == 0) { a = t % nr; b = nr; }
        else { a = (t + k) % nr; b = (t - k + nr) % nr; }
        if (a > b) { const int x = a; a = b; b = x; }
        if (b >= n) continue;                       // the bye
        double* ca = A + (size_t)a * lda;
        double* cb = A + (size_t)b * lda;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double x = ca[i], y = cb[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + tt * tt);
        const double sn = cs * tt;
        for (int i = lane; i < m; i += 32) {
          const double x = ca[i], y = cb[i];
          ca[i] = cs * x - sn * y;
          cb[i] = sn * x + cs * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  // extreme column norms
  double mx = 0.0, mn = 1.0 / 0.0;
  for (int j = warp; j < n; j += SV_NW) {
    const double* cj = A + (size_t)j * lda;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(cj[i], cj[i], s);
    s = sqrt(warp_sum(s));
    mx = fmax(mx, s);
    mn = fmin(mn, s);
  }
  if (lane == 0) { red[warp][0] = mx; red[warp][1] = mn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < SV_NW; ++w) { mx = fmax(mx, red[w][0]); mn = fmin(mn, red[w][1]); }
    mx = fmax(mx, red[0][0]);
    mn = fmin(mn, red[0][1]);
    *J.smax = mx;
    *J.smin = mn;
  }
}

void launch_jacobi_sv(const SvJob* d_jobs, int n, cudaStream_t st) {
  if (n <= 0) return;
  jacobi_sv_kernel<<<n, SV_NT, 0, st>>>(d_jobs);
  SPQ_LAUNCH_CHECK();
}

}  // namespace spq
