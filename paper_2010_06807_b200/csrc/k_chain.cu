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
#include <cstdlib>
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

// out[c] = sum_q part[q*k + c], q < nq: columns over adjacent threads (the
// loads of a warp are contiguous), the nq partials over S thread groups with
// independent loads, groups combined in a fixed order through red (CW_NT)
__device__ __forceinline__ void chain_reduce_partials(const double* part, int nq, int k,
                                                      double* out, double* red) {
  int cwid = 32;
  while (cwid < k && cwid < CW_NT) cwid <<= 1;
  const int S = CW_NT / cwid, tid = threadIdx.x, cl = tid % cwid, g = tid / cwid;
  for (int c0 = 0; c0 < k; c0 += cwid) {
    const int c = c0 + cl;
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (c < k) {
      const double* p = part + c;
      int q = g;
      for (; q + 7 * S < nq; q += 8 * S) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (int64_t)(q + u * S) * k);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += v[u];
      }
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = q + u * S < nq ? __ldcg(p + (int64_t)(q + u * S) * k) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += v[u];
    }
    red[tid] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    __syncthreads();
    if (g == 0 && c < k) {
      double t = red[cl];
      for (int j = 1; j < S; ++j) t += red[cl + j * cwid];
      out[c] = t;
    }
    __syncthreads();
  }
}

// Back substitution of one (wd <= 32) upper-triangular diagonal block by a
// single warp: lane l holds row l of the block in registers and its
// reciprocal pivot, so each of the wd sequential steps is one shuffle and one
// FMA (the pivot division -- a long multi-instruction sequence -- is off the
// dependency chain; x * (1/d) differs from x / d by at most one rounding).
__device__ __forceinline__ void tri32_backsolve(const double* D, int ldd, int wd, double* wv,
                                                int lane) {
  // the block's entries are read from shared memory a few steps ahead of the
  // dependency chain (addresses do not depend on it), not held in registers:
  // the caller's kernel keeps two CTAs per SM
  const double dinv = lane < wd ? 1.0 / D[lane + (int64_t)lane * ldd] : 0.0;
  double wl = lane < wd ? wv[lane] : 0.0;
#pragma unroll 8
  for (int i = wd - 1; i >= 0; --i) {
    const double rv = lane < i ? D[lane + (int64_t)i * ldd] : 0.0;
    if (lane == i) wl *= dinv;
    const double xi = __shfl_sync(0xffffffffu, wl, i);
    wl = fma(-rv, xi, wl);
  }
  if (lane < wd) wv[lane] = wl;
}

// The rest of a TRI op once all its partial products are in global memory
// (run by the op's last phase-A chunk): fixed-order reduction of the partials,
// then R_ss back substitution (32-column blocks, R slabs streamed through
// shared memory) or the finished R y product, scattered back into z.
__device__ void chain_tri_finish(const ChainOp& o, const double* __restrict__ part,
                                 double* __restrict__ z, int64_t N, int nrhs, int slab_k,
                                 double* cw, double* Rd, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = o.k;
  const int64_t ldr = o.ldr ? o.ldr : k;
  const bool has_part = o.n + o.n2 > 0 || o.kind == CH_TRI_MUL;
  double* w = o.scratch ? o.scratch : cw;   // k
  double* w2 = w + k;                       // k
  for (int r = 0; r < nrhs; ++r) {
    double* zr = z + (int64_t)r * N;
    const double* pr = part + o.part_off * nrhs + (int64_t)r * o.nchunk * k;
    // the first R slab and the gathered right-hand side are requested before
    // the partials are reduced: three independent memory latencies overlap
    const bool slabbed = o.kind == CH_TRI_SOLVE && k > 32 && k <= slab_k;
    double* slab = cw + 2 * (int64_t)slab_k;     // two buffers of slab_k x 32
    const int nb = (k + 31) / 32;
    const bool inv = slabbed && o.Dinv != nullptr;
    auto issue = [&](int t) {
      const int i1 = k - 32 * t, i0 = max(0, i1 - 32), wd = i1 - i0;
      double* dst = slab + (int64_t)(t & 1) * slab_k * 32;
      if (inv) {
        // inverse diagonal block (1024 doubles, 16-byte copies), then the
        // panel above it: rows 0..i0 of the block's columns (ld i0)
        for (int e = tid * 2; e < 1024; e += CW_NT * 2) {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + e);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa),
                       "l"(o.Dinv + (int64_t)t * 1024 + e) : "memory");
        }
        for (int e = tid; e < i0 * wd; e += CW_NT) {
          const int a = e % i0, b = e / i0;
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + 1024 + a + (int64_t)b * i0);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa),
                       "l"(o.R + (i0 + b) * ldr + a) : "memory");
        }
      } else {
        for (int e = tid; e < i1 * wd; e += CW_NT) {
          const int a = e % i1, b = e / i1;
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + a + (int64_t)b * i1);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa),
                       "l"(o.R + (i0 + b) * ldr + a) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (slabbed) issue(0);
    if (o.kind == CH_TRI_SOLVE)
      for (int a = tid; a < k; a += CW_NT) w2[a] = zr[o.idx[a]];
    if (has_part) {
      // R_sn y_n partials (TRI_SOLVE) / R y_s + R_sn y_n partials (TRI_MUL)
      chain_reduce_partials(pr, o.nchunk, k, w, red);
    } else {
      for (int a = tid; a < k; a += CW_NT) w[a] = 0.0;
    }
    __syncthreads();
    if (o.kind == CH_TRI_SOLVE)
      for (int a = tid; a < k; a += CW_NT) w[a] = w2[a] - w[a];
    __syncthreads();
    if (slabbed) {
      // blocked back substitution, 32 columns per block from the bottom;
      // the R slab of the next block (rows 0..i1, its 32 columns) streams
      // into shared memory (cp.async, double buffered) while the current
      // block is solved, so the solve never waits on a global load
      for (int t = 0; t < nb; ++t) {
        if (t + 1 < nb) {
          issue(t + 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int i1 = k - 32 * t, i0 = max(0, i1 - 32), wd = i1 - i0;
        const double* S = slab + (int64_t)(t & 1) * slab_k * 32;
        if (inv) {
          // x_block = Dinv w_block: four warps take eight columns each
          if (warp < 4) {
            double acc = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int cc = warp * 8 + u;
              if (cc < wd) acc = fma(S[lane + cc * 32], w[i0 + cc], acc);
            }
            red[tid] = acc;
          }
          __syncthreads();
          if (tid < wd) w[i0 + tid] = (red[tid] + red[32 + tid]) + (red[64 + tid] + red[96 + tid]);
          __syncthreads();
          const double* Pn = S + 1024;   // i0 x wd, ld i0
          for (int a = tid; a < i0; a += CW_NT) {
            double s0 = 0.0, s1 = 0.0;
            int b = 0;
            for (; b + 1 < wd; b += 2) {
              s0 = fma(Pn[a + (int64_t)b * i0], w[i0 + b], s0);
              s1 = fma(Pn[a + (int64_t)(b + 1) * i0], w[i0 + b + 1], s1);
            }
            if (b < wd) s0 = fma(Pn[a + (int64_t)b * i0], w[i0 + b], s0);
            w[a] -= s0 + s1;
          }
          __syncthreads();
          continue;
        }
        // S: i1 x wd, ld i1
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
          Rd[a + b * 33] = o.R[(i0 + a) + (i0 + b) * ldr];
        }
        __syncthreads();
        if (warp == 0) tri32_backsolve(Rd, 33, wd, w + i0, lane);
        __syncthreads();
        for (int a = tid; a < i0; a += CW_NT) {
          double s = 0.0;
          for (int b = i0; b < i1; ++b) s += o.R[a + b * ldr] * w[b];
          w[a] -= s;
        }
        __syncthreads();
      }
    }
    for (int a = tid; a < k; a += CW_NT) zr[o.idx[a]] = w[a];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(CW_NT, 2) chain_phaseA_kernel(const ChainOp* __restrict__ ops,
                                                             const int2* __restrict__ tasks,
                                                             double* __restrict__ part,
                                                             double* z, int64_t N, int nrhs,
                                                             int slab_k) {
  const int2 tk = tasks[blockIdx.x];
  const ChainOp o = ops[tk.x];
  const int chunk = tk.y;
  // programmatic dependent launch: the next wave's CTAs may start and fetch
  // their (static) task and op descriptors while this grid runs; everything
  // that touches z or the partials comes after the wait
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = o.k;
  extern __shared__ __align__(16) double cw[];
  __shared__ int last;
  // one static buffer, carved per branch: gathered z / y entries (then the
  // reduced w) | WY: per-warp 8 x 33 product tiles, TRI: reduction scratch and
  // the staged diagonal block
  __shared__ double sraw[CW_NT * 2 + CW_NW * 8 * 33];
  double* sbuf = sraw;
  double* redA = sraw + CW_NT * 2;
  if (o.kind == CH_WY_T || o.kind == CH_WY_N) {
    const int i0 = chunk * o.per, i1 = min(o.m, i0 + o.per);
    for (int r = 0; r < nrhs; ++r) {
      const double* zr = z + (int64_t)r * N;
      // z rows of the chunk staged once in shared memory (gathered)
      double* zs = sbuf;
      const int nrow = i1 - i0;
      const bool staged = nrow <= CW_NT * 2;
      if (staged)
        for (int i = tid; i < nrow; i += CW_NT) zs[i] = zr[o.idx[i0 + i]];
      __syncthreads();
      if (nrow <= 64 && staged) {
        // eight columns per warp pass: every lane loads its one or two rows of
        // the eight columns (up to 16 independent loads), multiplies by its z
        // entries and parks the products in the warp's 8 x 33 tile; lane j then
        // adds eight tile entries of column j % 8 and two shuffles combine the
        // four quarters -- 10 additions per eight columns instead of 40
        double* tile = sraw + CW_NT * 2 + warp * (8 * 33);
        const bool r0 = lane < nrow, r1 = lane + 32 < nrow;
        const double z0 = r0 ? zs[lane] : 0.0, z1 = r1 ? zs[lane + 32] : 0.0;
        const double* vbase = o.V + i0 + lane;
        double* pw = part + o.part_off * nrhs + ((int64_t)r * o.nchunk + chunk) * k;
        for (int c = warp * 8; c < k; c += 8 * CW_NW) {
          double a0[8], a1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double* vc = vbase + (int64_t)min(c + u, k - 1) * o.m;
            a0[u] = r0 ? vc[0] : 0.0;
            a1[u] = r1 ? vc[32] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) tile[u * 33 + lane] = fma(a1[u], z1, a0[u] * z0);
          __syncwarp();
          const int cu = lane & 7, q = lane >> 3;
          double sacc = 0.0;
#pragma unroll
          for (int e = 0; e < 8; ++e) sacc += tile[cu * 33 + q * 8 + e];
          sacc += __shfl_xor_sync(0xffffffffu, sacc, 8);
          sacc += __shfl_xor_sync(0xffffffffu, sacc, 16);
          if (lane < 8 && c + lane < k) pw[c + lane] = sacc;
          __syncwarp();
        }
      } else
      // four columns per warp pass; all loads of a pass are issued before the
      // shuffle reductions (the loads are latency-bound: a chunk is a few
      // dozen rows, so every lane keeps up to eight loads in flight)
      for (int c = warp; c < k; c += 4 * CW_NW) {
        const double* vc[4];
        bool on[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cu = c + u * CW_NW;
          on[u] = cu < k;
          vc[u] = o.V + (int64_t)(on[u] ? cu : c) * o.m;
        }
        double s[4] = {0.0, 0.0, 0.0, 0.0}, t[4] = {0.0, 0.0, 0.0, 0.0};
        int i = i0 + lane;
        for (; i + 32 < i1; i += 64) {
          const double z0 = staged ? zs[i - i0] : zr[o.idx[i]];
          const double z1 = staged ? zs[i + 32 - i0] : zr[o.idx[i + 32]];
          double a0[4], a1[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            a0[u] = vc[u][i];
            a1[u] = vc[u][i + 32];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            s[u] = fma(a0[u], z0, s[u]);
            t[u] = fma(a1[u], z1, t[u]);
          }
        }
        if (i < i1) {
          const double z0 = staged ? zs[i - i0] : zr[o.idx[i]];
          double a0[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) a0[u] = vc[u][i];
#pragma unroll
          for (int u = 0; u < 4; ++u) s[u] = fma(a0[u], z0, s[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] += t[u];
#pragma unroll
        for (int q = 16; q; q >>= 1) {
#pragma unroll
          for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], q);
        }
        if (lane == 0) {
          double* pw = part + o.part_off * nrhs + ((int64_t)r * o.nchunk + chunk) * k;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (on[u]) pw[c + u * CW_NW] = s[u];
        }
      }
      __syncthreads();
    }
    // the last chunk to arrive reduces the partials (fixed chunk order) and
    // forms u = w (W precomputed) or T^T w / T w, once per operation
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(o.cnt, 1) == o.nchunk - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double* wred = sbuf;
    for (int r = 0; r < nrhs; ++r) {
      const double* pr = part + o.part_off * nrhs + (int64_t)r * o.nchunk * k;
      double* u = part + o.u_off * nrhs + (int64_t)r * 2 * k;   // u (k) | global w (k)
      const bool sm = k <= CW_NT * 2;
      double* wv = o.W ? u : (sm ? wred : u + k);
      chain_reduce_partials(pr, o.nchunk, k, wv, redA);
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
  } else {
    double* Rd = sraw + CW_NT * 3;
    if (o.n + o.n2 > 0 || o.kind == CH_TRI_MUL) {
      // [R | R_sn][:, chunk] [y_s; y_n][chunk] (TRI_MUL: the whole product, R
      // upper triangular; TRI_SOLVE: the R_sn part only): rows a split over
      // threads, columns over P partitions; the chunk's y entries are gathered
      // into shared memory first so the matrix loads are all independent
      double* ys = sbuf;
      const bool mul = o.kind == CH_TRI_MUL;
      const int n2 = o.n2;   // TRI_SOLVE row block: columns of R_ss right of the block first
      const int64_t ldr = o.ldr ? o.ldr : k, ldn = o.ldn ? o.ldn : k;
      const int ncol = mul ? k + o.n : n2 + o.n;
      const int j0 = chunk * o.per, j1 = min(ncol, j0 + o.per), nj = j1 - j0;
      const bool staged = nj <= CW_NT * 2;
      int P = CW_NT / max(k, 1);
      P = P >= 16 ? 16 : (P >= 8 ? 8 : (P >= 4 ? 4 : (P >= 2 ? 2 : 1)));
      const int rows_per_pass = CW_NT / P;
      for (int r = 0; r < nrhs; ++r) {
        const double* zr = z + (int64_t)r * N;
        auto yv = [&](int j) {
          return mul ? (j < k ? zr[o.idx[j]] : zr[o.idx_n[j - k]])
                     : (j < n2 ? zr[o.idx2[j]] : zr[o.idx_n[j - n2]]);
        };
        if (staged) {
          for (int i = tid; i < nj; i += CW_NT) ys[i] = yv(j0 + i);
          __syncthreads();
        }
        for (int a0 = 0; a0 < k; a0 += rows_per_pass) {
          const int a = a0 + tid % rows_per_pass, jp = tid / rows_per_pass;
          double s0 = 0.0, s1 = 0.0;
          if (a < k) {
            if (mul) {
              for (int j = j0 + jp; j < j1; j += P) {
                const double yj = staged ? ys[j - j0] : yv(j);
                if (j < k) {
                  if (a <= j) s0 = fma(o.R[a + (int64_t)j * k], yj, s0);
                } else {
                  s1 = fma(o.Rsn[a + (int64_t)(j - k) * k], yj, s1);
                }
              }
            } else {
              // two column segments: R_ss right of a row block (split ops only), then R_sn
              int j = j0 + jp;
              const int je = min(j1, n2);
              const double* R2a = o.R2 + a;
#pragma unroll 4
              for (; j + P < je; j += 2 * P) {
                s0 = fma(R2a[j * ldr], staged ? ys[j - j0] : yv(j), s0);
                s1 = fma(R2a[(j + P) * ldr], staged ? ys[j + P - j0] : yv(j + P), s1);
              }
              if (j < je) {
                s0 = fma(R2a[j * ldr], staged ? ys[j - j0] : yv(j), s0);
                j += P;
              }
              const double* Rna = o.Rsn + a - n2 * ldn;
#pragma unroll 4
              for (; j + P < j1; j += 2 * P) {
                s0 = fma(Rna[j * ldn], staged ? ys[j - j0] : yv(j), s0);
                s1 = fma(Rna[(j + P) * ldn], staged ? ys[j + P - j0] : yv(j + P), s1);
              }
              if (j < j1) s0 = fma(Rna[j * ldn], staged ? ys[j - j0] : yv(j), s0);
            }
          }
          redA[tid] = s0 + s1;
          __syncthreads();
          if (tid < rows_per_pass && a0 + tid < k) {
            double t = 0.0;
            for (int q = 0; q < P; ++q) t += redA[tid + q * rows_per_pass];
            part[o.part_off * nrhs + ((int64_t)r * o.nchunk + chunk) * k + a0 + tid] = t;
          }
          __syncthreads();
        }
      }
      // the last chunk to arrive finishes the operation
      __threadfence();
      __syncthreads();
      if (tid == 0) last = atomicAdd(o.cnt, 1) == o.nchunk - 1;
      __syncthreads();
      if (!last) return;
      __threadfence();
      if (tid == 0) *o.cnt = 0;
    }
    chain_tri_finish(o, part, z, N, nrhs, slab_k, cw, Rd, redA);
  }
}

__global__ void __launch_bounds__(CW_NT) chain_phaseB_kernel(const ChainOp* __restrict__ ops,
                                                             const int2* __restrict__ tasks,
                                                             const double* __restrict__ part,
                                                             double* __restrict__ z, int64_t N,
                                                             int nrhs) {
  const int2 tk = tasks[blockIdx.x];
  const ChainOp o = ops[tk.x];
  const int chunk = tk.y;
  // programmatic dependent launch: the next wave's CTAs may start and fetch
  // their (static) task and op descriptors while this grid runs; everything
  // that touches z or the partials comes after the wait
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) double cw[];
  const int tid = threadIdx.x;
  const int k = o.k;
  double* w = o.scratch ? o.scratch + (int64_t)chunk * 3 * k : cw;   // k
  for (int r = 0; r < nrhs; ++r) {
    double* zr = z + (int64_t)r * N;
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
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (row < nrow) {
          const double* Mi = M + i0 + row;
          for (int c = cs; c < k; c += 4 * tpr) {   // four independent loads per round (eight measured slower)
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = c + u * tpr < k ? Mi[(int64_t)(c + u * tpr) * o.m] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(v[u], c + u * tpr < k ? w[c + u * tpr] : 0.0, acc[u]);
          }
        }
        redB[tid] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
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
      return;   // TRI ops are finished by their last chunk in phase A
    }
  }
}

size_t chain_wave_smem(int kmax, int slab_k) {
  const size_t b = (size_t)2 * (kmax > 0 ? kmax : 1) * sizeof(double) +
                   (size_t)64 * slab_k * sizeof(double);
  return b <= CHAIN_SMEM_MAX ? b : 0;
}

// Inverses of the 32 x 32 diagonal blocks of R_ss (chain compile time, like
// the W = V T^T products): the blocked back substitution then multiplies by
// the inverse block instead of running 32 dependent substitution steps.
// One warp per block, lane j solves R_block x = e_j by back substitution.
__global__ void __launch_bounds__(64) chain_dinv_kernel(const ChainOp* __restrict__ ops) {
  const ChainOp o = ops[blockIdx.x];
  if (o.kind != CH_TRI_SOLVE || !o.Dinv) return;
  __shared__ double D[2][32 * 33], X[2][32 * 33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, k = o.k, nb = (k + 31) / 32;
  const int64_t ldr = o.ldr ? o.ldr : k;
  double* out = const_cast<double*>(o.Dinv);
  for (int t = warp; t < nb; t += 2) {
    const int i1 = k - 32 * t, i0 = max(0, i1 - 32), wd = i1 - i0;
    double* Dw = D[warp];
    double* Xw = X[warp];
    for (int b = 0; b < 32; ++b)   // identity padding beyond wd
      Dw[lane + b * 33] = (lane < wd && b < wd) ? (lane <= b ? o.R[(i0 + lane) + (i0 + b) * ldr] : 0.0)
                                                : (lane == b ? 1.0 : 0.0);
    __syncwarp();
    for (int i = 31; i >= 0; --i) {   // X[i, lane]
      double x = 0.0;
      if (i == lane) {
        x = 1.0 / Dw[i + i * 33];
      } else if (i < lane) {
        double s = 0.0;
        for (int l = i + 1; l <= lane; ++l) s = fma(Dw[i + l * 33], Xw[l + lane * 33], s);
        x = -s / Dw[i + i * 33];
      }
      Xw[i + lane * 33] = x;
    }
    __syncwarp();
    for (int b = 0; b < 32; ++b) out[(int64_t)t * 1024 + lane + b * 32] = Xw[lane + b * 33];
    __syncwarp();
  }
}

void launch_chain_dinv(const ChainOp* d_ops, int nops, cudaStream_t st) {
  if (nops <= 0) return;
  chain_dinv_kernel<<<nops, 64, 0, st>>>(d_ops);
  SPQ_LAUNCH_CHECK();
}

cudaEvent_t g_chain_mid_event = nullptr;   // diagnostics: recorded between the two phases

void launch_chain_wave(const ChainOp* d_ops, const int2* d_tasks, int ntasks, int kmax, int slab_k,
                       bool has_wy, double* part, double* z, int64_t N, int nrhs,
                       cudaStream_t st) {
  if (ntasks <= 0) return;
  const size_t smem = chain_wave_smem(std::max(kmax, slab_k), slab_k);
  const size_t smemB = (size_t)std::max(kmax, 1) * sizeof(double);
  static size_t conf = 0;
  if (smem > conf) {   // the default 48 KB cap counts static + dynamic
    CUDA_TRY(cudaFuncSetAttribute(chain_phaseA_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
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
  static const bool pdl = getenv("SPQ_CHAIN_NO_PDL") == nullptr;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ntasks);
  cfg.blockDim = dim3(CW_NT);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cfg.dynamicSmemBytes = smem;
  const double* cpart = part;
  cudaLaunchKernelEx(&cfg, chain_phaseA_kernel, d_ops, d_tasks, part, z, N, nrhs, slab_k);
  fail("at chain phase A launch");
  if (g_chain_mid_event) cudaEventRecord(g_chain_mid_event, st);
  if (!has_wy) return;   // TRI ops finish inside phase A (their last chunk)
  cfg.dynamicSmemBytes = smemB;
  cudaLaunchKernelEx(&cfg, chain_phaseB_kernel, d_ops, d_tasks, cpart, z, N, nrhs);
  fail("at chain phase B launch");
}

}  // namespace spq
