// Solve-phase transform-chain kernels: the per-record
// applications behind Factorization.apply_qt / solve_w / apply_w
// (factor.py:97-241, 281-300) on an N x nrhs column-major block z.
//
//   WY on an index subset:  z[rows] <- z[rows] - V T^T V^T z[rows]   (or T)
//     wy_dot    : w = V^T z[rows]        warp per reflector column
//     tri_mv    : w2 = T^T w (or T w)    one CTA, k x k upper triangle
//     wy_update : z[rows] -= V w2        thread per row (coalesced V rows)
//   BlockHouseholder.solve_w: rhs = y[cols_s] - R_sn y[cols_n] (column-chunk
//     partial sums + one reduction CTA), then R_ss back substitution.
//   apply_w: y_s = R_ss x_s + R_sn x_n ; DiagonalScaling ; Permutation.
// All HBM-bound (~0.4 flop/byte).
#include <algorithm>
#include <string>

#include "common.cuh"

namespace spq {

// w[c + r*k] = sum_i V[i + c*m] * z[rows[i] + r*N]
__global__ void wy_dot_kernel(const double* __restrict__ V, int m, int k,
                              const double* __restrict__ z, const int* __restrict__ rows,
                              int64_t N, int nrhs, double* __restrict__ w) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= k) return;
  const double* v = V + (int64_t)c * m;
  for (int r = 0; r < nrhs; ++r) {
    const double* zr = z + (int64_t)r * N;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s += v[i] * zr[rows[i]];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) w[c + (int64_t)r * k] = s;
  }
}

// w2 = T^T w (trans) or T w ; one CTA; T upper (k x k, ld k)
__global__ void tri_mv_kernel(const double* __restrict__ T, int k, const double* __restrict__ w,
                              int nrhs, int trans, double* __restrict__ w2) {
  for (int r = 0; r < nrhs; ++r)
    for (int a = threadIdx.x; a < k; a += blockDim.x) {
      double s = 0.0;
      if (trans) {   // (T^T w)_a = sum_{b <= a} T[b,a] w_b
        for (int b = 0; b <= a; ++b) s += T[b + (int64_t)a * k] * w[b + (int64_t)r * k];
      } else {       // (T w)_a = sum_{b >= a} T[a,b] w_b
        for (int b = a; b < k; ++b) s += T[a + (int64_t)b * k] * w[b + (int64_t)r * k];
      }
      w2[a + (int64_t)r * k] = s;
    }
}

// z[rows[i]] -= sum_c V[i + c*m] w2[c]
__global__ void wy_update_kernel(const double* __restrict__ V, int m, int k,
                                 double* __restrict__ z, const int* __restrict__ rows, int64_t N,
                                 int nrhs, const double* __restrict__ w2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int r = 0; r < nrhs; ++r) {
    double s = 0.0;
    for (int c = 0; c < k; ++c) s += V[i + (int64_t)c * m] * w2[c + (int64_t)r * k];
    z[rows[i] + (int64_t)r * N] -= s;
  }
}

// part[chunk*k + a + r*k*nchunk] = sum_{j in chunk} Rsn[a + j*k] y[cols_n[j]]
__global__ void rsn_partial_kernel(const double* __restrict__ Rsn, int k, int n,
                                   const double* __restrict__ y, const int* __restrict__ cols_n,
                                   int64_t N, int nrhs, int chunk, double* __restrict__ part) {
  const int ch = blockIdx.y;
  const int j0 = ch * chunk, j1 = min(n, j0 + chunk);
  const int nch = gridDim.y;
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < k; a += gridDim.x * blockDim.x)
    for (int r = 0; r < nrhs; ++r) {
      double s = 0.0;
      for (int j = j0; j < j1; ++j) s += Rsn[a + (int64_t)j * k] * y[cols_n[j] + (int64_t)r * N];
      part[(int64_t)ch * k + a + (int64_t)r * k * nch] = s;
    }
}

// mode 0 (solve_w of BlockHouseholder / InterfaceScaling):
//   b = y[cols] - sum_chunks part ; y[cols] = R^{-1} b      (back substitution)
// mode 1 (apply_w): y[cols] = R y[cols] + sum_chunks part
__global__ void __launch_bounds__(1024) tri_solve_vec_kernel(const double* __restrict__ R, int k,
                                                             double* __restrict__ y,
                                                             const int* __restrict__ cols,
                                                             int64_t N, int nrhs,
                                                             const double* __restrict__ part,
                                                             int nch, int mode) {
  extern __shared__ double b[];   // k
  for (int r = 0; r < nrhs; ++r) {
    double* yr = y + (int64_t)r * N;
    for (int a = threadIdx.x; a < k; a += blockDim.x) {
      double s = 0.0;
      if (part)
        for (int ch = 0; ch < nch; ++ch) s += part[(int64_t)ch * k + a + (int64_t)r * k * nch];
      if (mode == 0) {
        b[a] = yr[cols[a]] - s;
      } else {
        double t = 0.0;
        for (int c = a; c < k; ++c) t += R[a + (int64_t)c * k] * yr[cols[c]];
        b[a] = t + s;
      }
    }
    __syncthreads();
    if (mode == 0) {
      for (int i = k - 1; i >= 0; --i) {
        if (threadIdx.x == 0) b[i] = b[i] / R[i + (int64_t)i * k];
        __syncthreads();
        const double xi = b[i];
        for (int a = threadIdx.x; a < i; a += blockDim.x) b[a] -= R[a + (int64_t)i * k] * xi;
        __syncthreads();
      }
    }
    for (int a = threadIdx.x; a < k; a += blockDim.x) yr[cols[a]] = b[a];
    __syncthreads();
  }
}

__global__ void diag_scale_kernel(double* __restrict__ y, const double* __restrict__ s, int64_t N,
                                  int nrhs, int divide) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * nrhs) return;
  const double d = s[t % N];
  y[t] = divide ? y[t] / d : y[t] * d;
}

__global__ void permute_kernel(const double* __restrict__ z, const int* __restrict__ roc,
                               int64_t N, int nrhs, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * nrhs) return;
  const int64_t j = t % N, r = t / N;
  out[t] = z[roc[j] + r * N];
}

// ------------------------------------------------------------- launchers
void chain_wy(const double* V, const double* T, int m, int k, double* z, const int* rows,
              int64_t N, int nrhs, bool transpose, double* w, double* w2, cudaStream_t st) {
  if (k <= 0 || m <= 0) return;
  wy_dot_kernel<<<(k * 32 + 255) / 256, 256, 0, st>>>(V, m, k, z, rows, N, nrhs, w); SPQ_LAUNCH_CHECK();
  tri_mv_kernel<<<1, 256, 0, st>>>(T, k, w, nrhs, transpose ? 1 : 0, w2); SPQ_LAUNCH_CHECK();
  wy_update_kernel<<<(m + 127) / 128, 128, 0, st>>>(V, m, k, z, rows, N, nrhs, w2); SPQ_LAUNCH_CHECK();
}

int chain_rsn_chunks(int n) { return n <= 0 ? 0 : (n + 127) / 128; }

void chain_tri(const double* R, int k, const double* Rsn, int n, double* y, const int* cols_s,
               const int* cols_n, int64_t N, int nrhs, int mode, double* part, cudaStream_t st) {
  if (k <= 0) return;
  const int nch = chain_rsn_chunks(n);
  if (nch > 0)
    rsn_partial_kernel<<<dim3((k + 127) / 128, nch), 128, 0, st>>>(Rsn, k, n, y, cols_n, N, nrhs,
                                                                   128, part); SPQ_LAUNCH_CHECK();
  const size_t smem = (size_t)k * sizeof(double);
  static size_t conf = 0;
  if (smem > conf) {   // the default 48 KB cap counts static + dynamic
    CUDA_TRY(cudaFuncSetAttribute(tri_solve_vec_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    conf = smem;
  }
  tri_solve_vec_kernel<<<1, 1024, smem, st>>>(R, k, y, cols_s, N, nrhs, nch ? part : nullptr, nch,
                                              mode); SPQ_LAUNCH_CHECK();
}

void chain_diag(double* y, const double* s, int64_t N, int nrhs, bool divide, cudaStream_t st) {
  const int64_t t = N * nrhs;
  if (t <= 0) return;
  diag_scale_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(y, s, N, nrhs, divide ? 1 : 0); SPQ_LAUNCH_CHECK();
}

void chain_perm(const double* z, const int* roc, int64_t N, int nrhs, double* out,
                cudaStream_t st) {
  const int64_t t = N * nrhs;
  if (t <= 0) return;
  permute_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(z, roc, N, nrhs, out); SPQ_LAUNCH_CHECK();
}

}  // namespace spq

// ======================================================= wave-batched chain
// Two launches per wave of data-independent record operations (disjoint
// index sets, planned at spq_finish).  Large operations are split into
// chunks, one CTA per (op, chunk):
//   phase A: partial products  w_chunk = V[rows_chunk]^T z[rows_chunk]  (WY)
//                              s_chunk = R_sn[:, cols_chunk] y[cols_chunk] (TRI)
//   phase B: every chunk-CTA of a WY op reduces the partials (fixed order),
//            forms T^T w / T w and updates its rows; the TRI ops finish in
//            chunk 0 (R_ss back substitution with 32x32 diagonal blocks staged
//            in shared memory, or the R y product).
namespace spq {

constexpr int CW_NT = 512;
constexpr int CW_NW = CW_NT / 32;

// out[c] = sum_q part[q*k + c], q < nq: g lanes per column (g = power of two
// ~ nq/4, so each lane has a few independent loads), fixed shuffle tree
__device__ __forceinline__ void chain_reduce_partials(const double* part, int nq, int k,
                                                      double* out) {
  int g = 1;
  while (g < 32 && g * 4 < nq) g <<= 1;
  const int tid = threadIdx.x, sub = tid & (g - 1);
  const int per_pass = CW_NT / g;
  for (int c0 = 0; c0 < k; c0 += per_pass) {
    const int c = c0 + tid / g;
    double s0 = 0.0, s1 = 0.0;
    if (c < k) {
      int q = sub;
      for (; q + g < nq; q += 2 * g) {
        s0 += __ldcg(part + (int64_t)q * k + c);
        s1 += __ldcg(part + (int64_t)(q + g) * k + c);
      }
      if (q < nq) s0 += __ldcg(part + (int64_t)q * k + c);
    }
    double s = s0 + s1;
    for (int sh = g >> 1; sh; sh >>= 1) s += __shfl_xor_sync(0xffffffffu, s, sh);
    if (sub == 0 && c < k) out[c] = s;
  }
}

__global__ void __launch_bounds__(CW_NT) chain_phaseA_kernel(const ChainOp* __restrict__ ops,
                                                             const int2* __restrict__ tasks,
                                                             double* __restrict__ part,
                                                             const double* __restrict__ z,
                                                             int64_t N, int nrhs) {
  const int2 tk = tasks[blockIdx.x];
  const ChainOp o = ops[tk.x];
  const int chunk = tk.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = o.k;
  if (o.kind == CH_WY_T || o.kind == CH_WY_N) {
    const int i0 = chunk * o.per, i1 = min(o.m, i0 + o.per);
    for (int r = 0; r < nrhs; ++r) {
      const double* zr = z + (int64_t)r * N;
      // z rows of the chunk staged once in shared memory (gathered)
      __shared__ double zs[CW_NT * 2];
      const int nrow = i1 - i0;
      const bool staged = nrow <= CW_NT * 2;
      if (staged)
        for (int i = tid; i < nrow; i += CW_NT) zs[i] = zr[o.idx[i0 + i]];
      __syncthreads();
      // two columns per warp pass, four independent accumulators (the loads
      // are latency-bound: keep several in flight per lane)
      for (int c = warp; c < k; c += 2 * CW_NW) {
        const int c2 = c + CW_NW;
        const double* vc = o.V + (int64_t)c * o.m;
        const double* vd = o.V + (int64_t)(c2 < k ? c2 : c) * o.m;
        double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
        int i = i0 + lane;
        for (; i + 32 < i1; i += 64) {
          const double z0 = staged ? zs[i - i0] : zr[o.idx[i]];
          const double z1 = staged ? zs[i + 32 - i0] : zr[o.idx[i + 32]];
          s0 = fma(vc[i], z0, s0);
          s1 = fma(vc[i + 32], z1, s1);
          t0 = fma(vd[i], z0, t0);
          t1 = fma(vd[i + 32], z1, t1);
        }
        if (i < i1) {
          const double z0 = staged ? zs[i - i0] : zr[o.idx[i]];
          s0 = fma(vc[i], z0, s0);
          t0 = fma(vd[i], z0, t0);
        }
        double s = s0 + s1, t = t0 + t1;
#pragma unroll
        for (int q = 16; q; q >>= 1) {
          s += __shfl_xor_sync(0xffffffffu, s, q);
          t += __shfl_xor_sync(0xffffffffu, t, q);
        }
        if (lane == 0) {
          part[o.part_off * nrhs + ((int64_t)r * o.nchunk + chunk) * k + c] = s;
          if (c2 < k) part[o.part_off * nrhs + ((int64_t)r * o.nchunk + chunk) * k + c2] = t;
        }
      }
      __syncthreads();
    }
    // the last chunk to arrive reduces the partials (fixed chunk order) and
    // forms u = w (W precomputed) or T^T w / T w, once per operation
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(o.cnt, 1) == o.nchunk - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    __shared__ double wred[CW_NT * 2];
    for (int r = 0; r < nrhs; ++r) {
      const double* pr = part + o.part_off * nrhs + (int64_t)r * o.nchunk * k;
      double* u = part + o.u_off * nrhs + (int64_t)r * 2 * k;   // u (k) | global w (k)
      const bool sm = k <= CW_NT * 2;
      double* wv = o.W ? u : (sm ? wred : u + k);
      chain_reduce_partials(pr, o.nchunk, k, wv);
      __syncthreads();
      if (!o.W && o.kind == CH_WY_T) {   // (T^T w)_a = sum_{b<=a} T[b,a] w_b: warp per a (coalesced)
        for (int a = warp; a < k; a += CW_NW) {
          double s = 0.0;
          for (int b = lane; b <= a; b += 32) s = fma(o.T[b + (int64_t)a * k], sm ? wv[b] : __ldcg(wv + b), s);
#pragma unroll
          for (int q = 16; q; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
          if (lane == 0) u[a] = s;
        }
      } else if (!o.W) {                 // (T w)_a = sum_{b>=a} T[a,b] w_b: warp per a, lanes over b
        for (int a = warp; a < k; a += CW_NW) {
          double s = 0.0;
          for (int b = a + lane; b < k; b += 32) s = fma(o.T[a + (int64_t)b * k], sm ? wv[b] : __ldcg(wv + b), s);
#pragma unroll
          for (int q = 16; q; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
          if (lane == 0) u[a] = s;
        }
      }
      __syncthreads();
    }
    if (tid == 0) *o.cnt = 0;   // ready for the next application
    return;
  } else if (o.n > 0 || o.kind == CH_TRI_MUL) {
    // [R | R_sn][:, chunk] [y_s; y_n][chunk] (TRI_MUL: the whole product, R
    // upper triangular; TRI_SOLVE: the R_sn part only): rows a split over
    // threads, columns over P partitions
    __shared__ double redA[CW_NT];
    const bool mul = o.kind == CH_TRI_MUL;
    const int ncol = mul ? k + o.n : o.n;
    const int j0 = chunk * o.per, j1 = min(ncol, j0 + o.per);
    int P = CW_NT / max(k, 1);
    P = P >= 16 ? 16 : (P >= 8 ? 8 : (P >= 4 ? 4 : (P >= 2 ? 2 : 1)));
    const int rows_per_pass = CW_NT / P;
    for (int r = 0; r < nrhs; ++r) {
      const double* zr = z + (int64_t)r * N;
      for (int a0 = 0; a0 < k; a0 += rows_per_pass) {
        const int a = a0 + tid % rows_per_pass, jp = tid / rows_per_pass;
        double s = 0.0;
        if (a < k) {
          if (mul) {
            for (int j = j0 + jp; j < j1; j += P) {
              if (j < k) {
                if (a <= j) s += o.R[a + (int64_t)j * k] * zr[o.idx[j]];
              } else {
                s += o.Rsn[a + (int64_t)(j - k) * k] * zr[o.idx_n[j - k]];
              }
            }
          } else {
            for (int j = j0 + jp; j < j1; j += P) s += o.Rsn[a + (int64_t)j * k] * zr[o.idx_n[j]];
          }
        }
        redA[tid] = s;
        __syncthreads();
        if (tid < rows_per_pass && a0 + tid < k) {
          double t = 0.0;
          for (int q = 0; q < P; ++q) t += redA[tid + q * rows_per_pass];
          part[o.part_off * nrhs + ((int64_t)r * o.nchunk + chunk) * k + a0 + tid] = t;
        }
        __syncthreads();
      }
    }
  }
}

// Back substitution of one (wd <= 32) upper-triangular diagonal block by a
// single warp: lane l holds row l of the block in registers and its
// reciprocal pivot, so each of the wd sequential steps is one shuffle and one
// FMA (the pivot division -- a long multi-instruction sequence -- is off the
// dependency chain; x * (1/d) differs from x / d by at most one rounding).
__device__ __forceinline__ void tri32_backsolve(const double* D, int ldd, int wd, double* wv,
                                                int lane) {
  double rrow[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) rrow[j] = (j < wd && lane < j) ? D[lane + (int64_t)j * ldd] : 0.0;
  const double dinv = lane < wd ? 1.0 / D[lane + (int64_t)lane * ldd] : 0.0;
  double wl = lane < wd ? wv[lane] : 0.0;
#pragma unroll
  for (int i = 31; i >= 0; --i) {
    if (i < wd) {
      if (lane == i) wl *= dinv;
      const double xi = __shfl_sync(0xffffffffu, wl, i);
      if (lane < i) wl = fma(-rrow[i], xi, wl);
    }
  }
  if (lane < wd) wv[lane] = wl;
}

__global__ void __launch_bounds__(CW_NT) chain_phaseB_kernel(const ChainOp* __restrict__ ops,
                                                             const int2* __restrict__ tasks,
                                                             const double* __restrict__ part,
                                                             double* __restrict__ z, int64_t N,
                                                             int nrhs, int slab_k) {
  const int2 tk = tasks[blockIdx.x];
  const ChainOp o = ops[tk.x];
  const int chunk = tk.y;
  extern __shared__ __align__(16) double cw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = o.k;
  double* w = o.scratch ? o.scratch + (int64_t)chunk * 3 * k : cw;   // k
  double* w2 = w + k;                                                   // k
  __shared__ double Rd[32 * 33];
  for (int r = 0; r < nrhs; ++r) {
    double* zr = z + (int64_t)r * N;
    const double* pr = part + o.part_off * nrhs + (int64_t)r * o.nchunk * k;
    if (o.kind == CH_WY_T || o.kind == CH_WY_N) {
      // u (reduced by the last chunk of phase A) into shared memory, then
      // z[rows] -= M u with M = W (= V T^T / V T, precomputed) or V
      const double* u = part + o.u_off * nrhs + (int64_t)r * 2 * k;
      for (int c = tid; c < k; c += CW_NT) w[c] = __ldcg(u + c);
      __syncthreads();
      const double* M = o.W ? o.W : o.V;
      const int i0 = chunk * o.per, i1 = min(o.m, i0 + o.per), nrow = i1 - i0;
      if (nrow <= CW_NT / 2) {
        // few rows: TPR threads per row split the k columns (every thread
        // keeps independent loads in flight; rows stay coalesced per column),
        // partial sums reduced in a fixed order through shared memory
        __shared__ double redB[CW_NT];
        int rp = 1;
        while (rp < nrow) rp <<= 1;
        const int tpr = CW_NT / rp, row = tid % rp, cs = tid / rp;
        double s0 = 0.0, s1 = 0.0;
        if (row < nrow) {
          const double* Mi = M + i0 + row;
          int c = cs;
          for (; c + tpr < k; c += 2 * tpr) {
            s0 = fma(Mi[(int64_t)c * o.m], w[c], s0);
            s1 = fma(Mi[(int64_t)(c + tpr) * o.m], w[c + tpr], s1);
          }
          if (c < k) s0 = fma(Mi[(int64_t)c * o.m], w[c], s0);
        }
        redB[tid] = s0 + s1;
        __syncthreads();
        if (cs == 0 && row < nrow) {
          double t = 0.0;
          for (int q = 0; q < tpr; ++q) t += redB[row + q * rp];
          zr[o.idx[i0 + row]] -= t;
        }
        __syncthreads();
      } else {
        for (int i = i0 + tid; i < i1; i += CW_NT) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int c = 0;
          for (; c + 3 < k; c += 4) {
            s0 = fma(M[i + (int64_t)c * o.m], w[c], s0);
            s1 = fma(M[i + (int64_t)(c + 1) * o.m], w[c + 1], s1);
            s2 = fma(M[i + (int64_t)(c + 2) * o.m], w[c + 2], s2);
            s3 = fma(M[i + (int64_t)(c + 3) * o.m], w[c + 3], s3);
          }
          for (; c < k; ++c) s0 = fma(M[i + (int64_t)c * o.m], w[c], s0);
          zr[o.idx[i]] -= (s0 + s1) + (s2 + s3);
        }
        __syncthreads();
      }
    } else {
      if (chunk != 0) return;
      if (o.n > 0 || o.kind == CH_TRI_MUL) {
        // R_sn y_n partials (TRI_SOLVE) / R y_s + R_sn y_n partials (TRI_MUL)
        chain_reduce_partials(pr, o.nchunk, k, w);
      } else {
        for (int a = tid; a < k; a += CW_NT) w[a] = 0.0;
      }
      __syncthreads();
      if (o.kind == CH_TRI_SOLVE)
        for (int a = tid; a < k; a += CW_NT) w[a] = zr[o.idx[a]] - w[a];
      __syncthreads();
      if (o.kind == CH_TRI_SOLVE && k > 32 && k <= slab_k) {
        // blocked back substitution, 32 columns per block from the bottom;
        // the R slab of the next block (rows 0..i1, its 32 columns) streams
        // into shared memory (cp.async, double buffered) while the current
        // block is solved, so the solve never waits on a global load
        double* slab = cw + 2 * (int64_t)slab_k;     // two buffers of slab_k x 32
        const int nb = (k + 31) / 32;
        auto issue = [&](int t) {
          const int i1 = k - 32 * t, i0 = max(0, i1 - 32), wd = i1 - i0;
          double* dst = slab + (int64_t)(t & 1) * slab_k * 32;
          for (int e = tid; e < i1 * wd; e += CW_NT) {
            const int a = e % i1, b = e / i1;
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + a + (int64_t)b * i1);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa),
                         "l"(o.R + (i0 + b) * (int64_t)k + a) : "memory");
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        };
        issue(0);
        for (int t = 0; t < nb; ++t) {
          if (t + 1 < nb) {
            issue(t + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
          __syncthreads();
          const int i1 = k - 32 * t, i0 = max(0, i1 - 32), wd = i1 - i0;
          const double* S = slab + (int64_t)(t & 1) * slab_k * 32;   // i1 x wd, ld i1
          if (warp == 0) tri32_backsolve(S + i0, i1, wd, w + i0, lane);
          __syncthreads();
          for (int a = tid; a < i0; a += CW_NT) {
            double s = 0.0;
            for (int b = 0; b < wd; ++b) s = fma(S[a + (int64_t)b * i1], w[i0 + b], s);
            w[a] -= s;
          }
          __syncthreads();
        }
      } else if (o.kind == CH_TRI_SOLVE) {
        for (int i1 = k; i1 > 0; i1 -= 32) {
          const int i0 = max(0, i1 - 32), wd = i1 - i0;
          for (int e = tid; e < wd * wd; e += CW_NT) {     // stage the diagonal block
            const int a = e % wd, b = e / wd;
            Rd[a + b * 33] = o.R[(i0 + a) + (int64_t)(i0 + b) * k];
          }
          __syncthreads();
          if (warp == 0) tri32_backsolve(Rd, 33, wd, w + i0, lane);
          __syncthreads();
          for (int a = tid; a < i0; a += CW_NT) {
            double s = 0.0;
            for (int b = i0; b < i1; ++b) s += o.R[a + (int64_t)b * k] * w[b];
            w[a] -= s;
          }
          __syncthreads();
        }
      }
      for (int a = tid; a < k; a += CW_NT) zr[o.idx[a]] = w[a];
      __syncthreads();
    }
  }
}

size_t chain_wave_smem(int kmax, int slab_k) {
  const size_t b = (size_t)2 * (kmax > 0 ? kmax : 1) * sizeof(double) +
                   (size_t)64 * slab_k * sizeof(double);
  return b <= CHAIN_SMEM_MAX ? b : 0;
}

void launch_chain_wave(const ChainOp* d_ops, const int2* d_tasks, int ntasks, int kmax, int slab_k,
                       double* part, double* z, int64_t N, int nrhs, cudaStream_t st) {
  if (ntasks <= 0) return;
  const size_t smem = chain_wave_smem(std::max(kmax, slab_k), slab_k);
  static size_t conf = 0;
  if (smem > conf) {   // the default 48 KB cap counts static + dynamic
    CUDA_TRY(cudaFuncSetAttribute(chain_phaseB_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    conf = smem;
  }
  auto fail = [&](const char* where) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
      throw std::runtime_error(std::string(cudaGetErrorString(e)) + " " + where +
                               " (ntasks=" + std::to_string(ntasks) + " kmax=" +
                               std::to_string(kmax) + " smem=" + std::to_string(smem) +
                               " conf=" + std::to_string(conf) + ")");
  };
  fail("pending before chain wave");
  chain_phaseA_kernel<<<ntasks, CW_NT, 0, st>>>(d_ops, d_tasks, part, z, N, nrhs);
  fail("at chain phase A launch");
  chain_phaseB_kernel<<<ntasks, CW_NT, smem, st>>>(d_ops, d_tasks, part, z, N, nrhs, slab_k);
  fail("at chain phase B launch");
}

}  // namespace spq
