// Device kernels of the right-preconditioned GMRES (the
// caller of the solve-phase chains; reference pkg/src/nestqr/solve.py:66-209
// and the CSR matrix-vector product sparse.py:110-113).
//
// Every reduction is deterministic: a fixed grid of KRY_G blocks, each block
// owning the same grid-stride slice of the vector in every kernel, writes one
// partial per block; consumers sum the KRY_G partials in block order.  Because
// a block owns its slice, the modified Gram-Schmidt step "h = q_i.w ;
// w -= h q_i ; partial of q_{i+1}.w" runs as ONE launch per step: each block
// first reduces the previous step's partials (redundantly, identical in every
// block), updates its own slice, then produces its partial of the next dot.
#include <algorithm>

#include "common.cuh"

namespace spq {

constexpr int KRY_NT = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < KRY_NT / 32; ++i) s += sh[i];
  return s;   // valid in thread 0
}

// sum of the G partials in block order (every thread gets the same value)
__device__ __forceinline__ double reduce_partials(const double* __restrict__ part, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < KRY_G; i += KRY_NT) v += part[i];
  // fixed tree over the block: identical result in every block
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < KRY_NT / 32; ++i) s += sh[i];
  __syncthreads();
  return s;
}

// y = A x  (mode 0)   or   y = b - A x  (mode 1); one warp per row
__global__ void __launch_bounds__(KRY_NT) csr_spmv_kernel(const int64_t* __restrict__ ptr,
                                                          const int* __restrict__ idx,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ b,
                                                          double* __restrict__ y, int64_t n,
                                                          int mode) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = ((int64_t)blockIdx.x * KRY_NT + threadIdx.x) >> 5; row < n;
       row += ((int64_t)gridDim.x * KRY_NT) >> 5) {
    const int64_t a = ptr[row], e = ptr[row + 1];
    double s = 0.0;
    for (int64_t k = a + lane; k < e; k += 32) s = fma(val[k], x[idx[k]], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[row] = mode ? b[row] - s : s;
  }
}

// partial[blk] of x.y over the block's slice
__global__ void __launch_bounds__(KRY_NT) dot_part_kernel(const double* __restrict__ x,
                                                          const double* __restrict__ y, int64_t n,
                                                          double* __restrict__ part) {
  __shared__ double sh[KRY_NT / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * KRY_NT + threadIdx.x; i < n; i += (int64_t)KRY_G * KRY_NT)
    s = fma(x[i], y[i], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out[0] = sum of partials (single block)
__global__ void __launch_bounds__(KRY_NT) finish_sum_kernel(const double* __restrict__ part,
                                                            double* __restrict__ out, int sqrt_it) {
  __shared__ double sh[KRY_NT / 32];
  const double s = reduce_partials(part, sh);
  if (threadIdx.x == 0) *out = sqrt_it ? sqrt(s) : s;
}

// One modified Gram-Schmidt step (solve.py:154-157):
//   h = sum(part_in) (= q_i . w) ; H_i = h ; w -= h q_i ; part_out = q_{i+1} . w
// q_next == nullptr: produce the partials of w . w instead (the norm).
__global__ void __launch_bounds__(KRY_NT) mgs_step_kernel(const double* __restrict__ qi,
                                                          const double* __restrict__ q_next,
                                                          double* __restrict__ w, int64_t n,
                                                          const double* __restrict__ part_in,
                                                          double* __restrict__ part_out,
                                                          double* __restrict__ h_out) {
  __shared__ double sh[KRY_NT / 32];
  const double h = reduce_partials(part_in, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) *h_out = h;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * KRY_NT + threadIdx.x; i < n; i += (int64_t)KRY_G * KRY_NT) {
    const double wi = fma(-h, qi[i], w[i]);
    w[i] = wi;
    s = fma(q_next ? q_next[i] : wi, wi, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part_out[blockIdx.x] = s;
}

// partials of Q[:, 0:j]^T w: part[c * G + blk] (re-orthogonalisation test)
__global__ void __launch_bounds__(KRY_NT) multi_dot_part_kernel(const double* __restrict__ Q,
                                                                int64_t ldq, int j,
                                                                const double* __restrict__ w,
                                                                int64_t n, double* __restrict__ part) {
  __shared__ double sh[KRY_NT / 32];
  for (int c = blockIdx.y; c < j; c += gridDim.y) {
    const double* q = Q + (int64_t)c * ldq;
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * KRY_NT + threadIdx.x; i < n; i += (int64_t)KRY_G * KRY_NT)
      s = fma(q[i], w[i], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[(int64_t)c * KRY_G + blockIdx.x] = s;
  }
}

// c[col] = sum of the column's partials; one block per column
__global__ void __launch_bounds__(KRY_NT) multi_finish_kernel(const double* __restrict__ part,
                                                              double* __restrict__ cvec) {
  __shared__ double sh[KRY_NT / 32];
  const double s = reduce_partials(part + (int64_t)blockIdx.x * KRY_G, sh);
  if (threadIdx.x == 0) cvec[blockIdx.x] = s;
}

// Conditional re-orthogonalisation (solve.py:158-163), decided on the device:
// if max|c| / wn > thr: H[0:j] += c ; w -= Q c ; flag = 1.  Also produces the
// partials of the (possibly updated) w . w.
__global__ void __launch_bounds__(KRY_NT) reorth_kernel(const double* __restrict__ Q, int64_t ldq,
                                                        int j, const double* __restrict__ cvec,
                                                        const double* __restrict__ wn_ptr,
                                                        double thr, double* __restrict__ w,
                                                        int64_t n, double* __restrict__ Hcol,
                                                        int* __restrict__ flag,
                                                        double* __restrict__ part_out) {
  __shared__ double sh[KRY_NT / 32];
  const double wn = *wn_ptr;
  double cmax = 0.0;
  for (int c = 0; c < j; ++c) cmax = fmax(cmax, fabs(cvec[c]));
  const bool doit = wn > 0.0 && cmax / wn > thr;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *flag = doit ? 1 : 0;
    if (doit)
      for (int c = 0; c < j; ++c) Hcol[c] += cvec[c];
  }
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * KRY_NT + threadIdx.x; i < n; i += (int64_t)KRY_G * KRY_NT) {
    double wi = w[i];
    if (doit) {
      double t = 0.0;
      for (int c = 0; c < j; ++c) t = fma(Q[(int64_t)c * ldq + i], cvec[c], t);
      wi -= t;
      w[i] = wi;
    }
    s = fma(wi, wi, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part_out[blockIdx.x] = s;
}

// dst = src * (1 / *den)  (q_{j+1} = w / wn; z / beta)
__global__ void scale_div_kernel(const double* __restrict__ src, const double* __restrict__ den,
                                 double* __restrict__ dst, int64_t n) {
  const double d = *den;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] / d;
}

// out = Q[:, 0:j] y  (GEMV, y on the device)
__global__ void gemv_kernel(const double* __restrict__ Q, int64_t ldq, int j,
                            const double* __restrict__ y, double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int c = 0; c < j; ++c) t = fma(Q[(int64_t)c * ldq + i], y[c], t);
    out[i] = t;
  }
}

// z = x + y
__global__ void add_kernel(const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ z, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = x[i] + y[i];
}

// ------------------------------------------------------------ launchers
static unsigned elt_grid(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 4 * 148); }

void kry_spmv(const int64_t* ptr, const int* idx, const double* val, const double* x,
              const double* b, double* y, int64_t n, int mode, cudaStream_t st) {
  const int64_t warps = n;
  const unsigned g = (unsigned)std::min<int64_t>((warps * 32 + KRY_NT - 1) / KRY_NT, 16 * 148);
  csr_spmv_kernel<<<g, KRY_NT, 0, st>>>(ptr, idx, val, x, b, y, n, mode); SPQ_LAUNCH_CHECK();
}
void kry_dot_part(const double* x, const double* y, int64_t n, double* part, cudaStream_t st) {
  dot_part_kernel<<<KRY_G, KRY_NT, 0, st>>>(x, y, n, part); SPQ_LAUNCH_CHECK();
}
void kry_finish(const double* part, double* out, bool sqrt_it, cudaStream_t st) {
  finish_sum_kernel<<<1, KRY_NT, 0, st>>>(part, out, sqrt_it ? 1 : 0); SPQ_LAUNCH_CHECK();
}
void kry_mgs_step(const double* qi, const double* q_next, double* w, int64_t n,
                  const double* part_in, double* part_out, double* h_out, cudaStream_t st) {
  mgs_step_kernel<<<KRY_G, KRY_NT, 0, st>>>(qi, q_next, w, n, part_in, part_out, h_out);
  SPQ_LAUNCH_CHECK();
}
void kry_multi_dot(const double* Q, int64_t ldq, int j, const double* w, int64_t n, double* part,
                   double* cvec, cudaStream_t st) {
  if (j <= 0) return;
  dim3 g(KRY_G, (unsigned)std::min(j, 64));
  multi_dot_part_kernel<<<g, KRY_NT, 0, st>>>(Q, ldq, j, w, n, part); SPQ_LAUNCH_CHECK();
  multi_finish_kernel<<<j, KRY_NT, 0, st>>>(part, cvec); SPQ_LAUNCH_CHECK();
}
void kry_reorth(const double* Q, int64_t ldq, int j, const double* cvec, const double* wn,
                double thr, double* w, int64_t n, double* Hcol, int* flag, double* part_out,
                cudaStream_t st) {
  reorth_kernel<<<KRY_G, KRY_NT, 0, st>>>(Q, ldq, j, cvec, wn, thr, w, n, Hcol, flag, part_out);
  SPQ_LAUNCH_CHECK();
}
void kry_scale_div(const double* src, const double* den, double* dst, int64_t n, cudaStream_t st) {
  scale_div_kernel<<<elt_grid(n), 256, 0, st>>>(src, den, dst, n); SPQ_LAUNCH_CHECK();
}
void kry_gemv(const double* Q, int64_t ldq, int j, const double* y, double* out, int64_t n,
              cudaStream_t st) {
  gemv_kernel<<<elt_grid(n), 256, 0, st>>>(Q, ldq, j, y, out, n); SPQ_LAUNCH_CHECK();
}
void kry_add(const double* x, const double* y, double* z, int64_t n, cudaStream_t st) {
  add_kernel<<<elt_grid(n), 256, 0, st>>>(x, y, z, n); SPQ_LAUNCH_CHECK();
}

}  // namespace spq
