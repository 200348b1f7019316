// Batched fp64 tensor-core GEMM for the compact-WY updates
//   W = V^T C,  W = T^T W,  C -= V W        (kernels/__init__.py:100-118)
// and the Gram products V^T V behind the T factor (kernels/_numba.py:101-117).
//
// sm_100a has no fp64 tcgen05 kind (ptxas rejects .kind::f64),
// so the fp64 tensor path is the warp-level DMMA `mma.sync.m8n8k4.f64`.
// Tile 64x64x16, 4 warps each owning 32x32 (4x4 DMMA tiles, 32 fp64
// accumulators per thread), register-prefetched double-buffered shared
// memory with a 68-double row pitch (conflict-free fragment loads: the 4
// k-rows of a fragment land on disjoint 8-bank groups).  One launch covers
// every problem of a wave; each CTA finds its problem by binary search over
// the per-problem first-tile prefix.
#include <cstdlib>

#include "common.cuh"

namespace spq {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, PITCH = 68, NT = 128;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
}  // namespace

// Epilogue C = alpha acc + beta C for a thread's 4 x 4 x 2 fragment (rows
// r0 + 8i, columns c0 + 8j + h).  All C loads are issued before any store:
// with loads and stores interleaved the compiler cannot hoist a load past a
// store that may alias it, and every element paid a full L2/HBM round trip
// (ncu: 78% of the v2 kernel's stall samples on this line).
__device__ __forceinline__ void gemm_epilogue(const GemmProb& p, const double (&acc)[4][4][2],
                                              int r0, int c0) {
  double cv[4][4][2];
  if (p.beta != 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = r0 + i * 8, col = c0 + j * 8 + h;
          cv[i][j][h] = (row < p.m && col < p.n) ? __ldg(p.C + row + (int64_t)col * p.ldc) : 0.0;
        }
  }
  // the two shapes of the compact-WY products get their own (uniform) branch:
  // one fp64 add, or none, per element instead of a multiply and an FMA (a
  // warp issues one fp64 instruction every ~14 cycles; on the short-K updates
  // C -= V W the epilogue was 40% of the kernel's stall samples)
  if (p.alpha == -1.0 && p.beta == 1.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = r0 + i * 8, col = c0 + j * 8 + h;
          if (row < p.m && col < p.n) p.C[row + (int64_t)col * p.ldc] = cv[i][j][h] - acc[i][j][h];
        }
    return;
  }
  if (p.alpha == 1.0 && p.beta == 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = r0 + i * 8, col = c0 + j * 8 + h;
          if (row < p.m && col < p.n) p.C[row + (int64_t)col * p.ldc] = acc[i][j][h];
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = r0 + i * 8, col = c0 + j * 8 + h;
        if (row < p.m && col < p.n) {
          const double v = p.alpha * acc[i][j][h];
          p.C[row + (int64_t)col * p.ldc] = (p.beta == 0.0) ? v : fma(p.beta, cv[i][j][h], v);
        }
      }
}

template <bool TA, int NP>
__global__ void __launch_bounds__(NT) gemm_dmma_kernel(const GemmProb* __restrict__ probs_g,
                                                       int nprob,
                                                       const __grid_constant__ PList<GemmProb, NP> pl) {
  const GemmProb* probs = NP > 1 ? pl.v : probs_g;
  int lo = 0, hi = nprob - 1;
  const int bid = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (probs[mid].tile0 <= bid) lo = mid; else hi = mid - 1;
  }
  const GemmProb p = probs[lo];
  const int tm = (p.m + BM - 1) / BM;
  const int t = bid - p.tile0;
  const int m0 = (t % tm) * BM, n0 = (t / tm) * BN;

  __shared__ double As[2][BK][PITCH];
  __shared__ double Bs[2][BK][PITCH];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int g = lane >> 2, q = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int l = tid + e * NT;
      int mi, ki;
      if (TA) { ki = l & 15; mi = l >> 4; } else { mi = l & 63; ki = l >> 6; }
      const int gm = m0 + mi, gk = k0 + ki;
      double v = 0.0;
      if (gm < p.m && gk < p.k)
        v = TA ? p.A[gk + (int64_t)gm * p.lda] : p.A[gm + (int64_t)gk * p.lda];
      ra[e] = v;
      const int kb = l & 15, nb = l >> 4;
      const int gk2 = k0 + kb, gn = n0 + nb;
      rb[e] = (gk2 < p.k && gn < p.n) ? p.B[gk2 + (int64_t)gn * p.ldb] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int l = tid + e * NT;
      int mi, ki;
      if (TA) { ki = l & 15; mi = l >> 4; } else { mi = l & 63; ki = l >> 6; }
      As[buf][ki][mi] = ra[e];
      Bs[buf][l & 15][l >> 4] = rb[e];
    }
  };

  const int nk = (p.k + BK - 1) / BK;
  if (nk > 0) {
    load(0);
    store(0);
    __syncthreads();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk + q][wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk + q][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    if (kt + 1 < nk) {
      store(buf ^ 1);
      __syncthreads();
    }
  }

  gemm_epilogue(p, acc, m0 + wm + g, n0 + wn + 2 * q);
}

// C = alpha * sum_s P_s + beta * C over split-K partials P_s (m x n, ld m,
// stride m*n), fixed summation order -> deterministic
template <int NP>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const SplitRed* __restrict__ tasks_g,
                                                            const __grid_constant__ PList<SplitRed, NP> pl) {
  const SplitRed t = NP > 1 ? pl.v[blockIdx.x] : tasks_g[blockIdx.x];
  const int64_t mn = (int64_t)t.m * t.n;
  for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < mn;
       e += (int64_t)gridDim.y * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < t.splits; ++q) s += t.P[e + q * mn];
    const int i = (int)(e % t.m), j = (int)(e / t.m);
    double* c = t.C + i + (int64_t)j * t.ldc;
    const double v = t.alpha * s;
    *c = (t.beta == 0.0) ? v : v + t.beta * (*c);
  }
}

void launch_splitk_reduce(const SplitRed* d_tasks, const SplitRed* h_tasks, int ntasks,
                          int64_t max_mn, cudaStream_t st) {
  if (ntasks <= 0) return;
  int64_t y = (max_mn + 2047) / 2048;
  if (y < 1) y = 1;
  if (y > 256) y = 256;
  const dim3 grid(ntasks, (unsigned)y);
  if (d_tasks == nullptr) {
    if (ntasks > PL_RED) throw std::runtime_error("launch_splitk_reduce: parameter list too long");
    PList<SplitRed, PL_RED> pl;
    for (int i = 0; i < ntasks; ++i) pl.v[i] = h_tasks[i];
    splitk_reduce_kernel<PL_RED><<<grid, 256, 0, st>>>(nullptr, pl);
  } else {
    splitk_reduce_kernel<1><<<grid, 256, 0, st>>>(d_tasks, PList<SplitRed, 1>{});
  }
  SPQ_LAUNCH_CHECK();
}


// ---------------------------------------------------------------- v2
// 128x64x16 CTA tile, 8 warps (4 along M x 2 along N, 32x32 each), 3-stage
// cp.async pipeline (8-byte copies with zero-fill for the ragged edges, any
// leading dimension), same conflict-free k-major shared layout.
namespace {
constexpr int BK2 = 16, NT2 = 256, ST2 = 3;
constexpr int TILE2_M = 128, TILE2_N = 64;   // variant 2; variant 3 swaps them

__device__ __forceinline__ void cp8(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(ok ? src : nullptr), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
}  // namespace

// BMx x BNx = 128 x 64 (variant 2) or 64 x 128 (variant 3: few rows, e.g. the
// k x n products W = V^T C, where a 128-row tile pads k = 300 to 384)
template <bool TA, int NP, int BMx, int BNx>
__global__ void __launch_bounds__(NT2, 2) gemm_dmma2_kernel(const GemmProb* __restrict__ probs_g,
                                                         int nprob,
                                                         const __grid_constant__ PList<GemmProb, NP> pl) {
  constexpr int BM2 = BMx, BN2 = BNx, PA2 = BMx + 4, PB2 = BNx + 4, WM = BMx / 32;
  const GemmProb* probs = NP > 1 ? pl.v : probs_g;
  int lo = 0, hi = nprob - 1;
  const int bid = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (probs[mid].tile0 <= bid) lo = mid; else hi = mid - 1;
  }
  const GemmProb p = probs[lo];
  const int tm = (p.m + BM2 - 1) / BM2;
  const int t = bid - p.tile0;
  const int m0 = (t % tm) * BM2, n0 = (t / tm) * BN2;

  extern __shared__ __align__(16) double smem2[];
  double* As = smem2;                       // [ST2][BK2][PA2]
  double* Bs = smem2 + ST2 * BK2 * PA2;     // [ST2][BK2][PB2]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % WM) * 32, wn = (warp / WM) * 32;
  const int g = lane >> 2, q = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto issue = [&](int stage, int k0) {
    double* a = As + stage * BK2 * PA2;
    double* b = Bs + stage * BK2 * PB2;
#pragma unroll
    for (int e = 0; e < BM2 * BK2 / NT2; ++e) {      // A: BM2 x 16 elements
      const int l = tid + e * NT2;
      int mi, ki;
      if (TA) { ki = l & 15; mi = l >> 4; } else { mi = l % BM2; ki = l / BM2; }
      const int gm = m0 + mi, gk = k0 + ki;
      const bool ok = gm < p.m && gk < p.k;
      const double* src = TA ? p.A + gk + (int64_t)gm * p.lda : p.A + gm + (int64_t)gk * p.lda;
      cp8(a + ki * PA2 + mi, src, ok);
    }
#pragma unroll
    for (int e = 0; e < BN2 * BK2 / NT2; ++e) {      // B: 16 x BN2 elements
      const int l = tid + e * NT2;
      const int kb = l & 15, nb = l >> 4;
      const int gk = k0 + kb, gn = n0 + nb;
      const bool ok = gk < p.k && gn < p.n;
      cp8(b + kb * PB2 + nb, p.B + gk + (int64_t)gn * p.ldb, ok);
    }
  };

  const int nk = (p.k + BK2 - 1) / BK2;
#pragma unroll
  for (int s = 0; s < ST2 - 1; ++s) {
    if (s < nk) issue(s, s * BK2);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<ST2 - 2>();
    __syncthreads();
    const int nxt = kt + ST2 - 1;
    if (nxt < nk) issue(nxt % ST2, nxt * BK2);
    cp_commit();
    const double* a = As + (kt % ST2) * BK2 * PA2;
    const double* b = Bs + (kt % ST2) * BK2 * PB2;
#pragma unroll
    for (int kk = 0; kk < BK2; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = a[(kk + q) * PA2 + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = b[(kk + q) * PB2 + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
  }
  cp_wait<0>();

  gemm_epilogue(p, acc, m0 + wm + g, n0 + wn + 2 * q);
}

static int gemm_env_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPQ_GEMM");
    v = (e && e[0] == '1') ? 1 : 2;
  }
  return v;
}
// per-batch choice (set by the host before tiling a batch): small batches use
// the 64x64 kernel so more CTAs cover the SMs
static thread_local int g_variant = 0;
static int gemm_variant() { return g_variant ? g_variant : gemm_env_variant(); }
void gemm_set_variant(int v) { g_variant = v; }

int gemm_tiles(int m, int n) {
  if (m <= 0 || n <= 0) return 0;
  if (gemm_variant() == 2) return ((m + TILE2_M - 1) / TILE2_M) * ((n + TILE2_N - 1) / TILE2_N);
  if (gemm_variant() == 3) return ((m + TILE2_N - 1) / TILE2_N) * ((n + TILE2_M - 1) / TILE2_M);
  return ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
}

template <int NP>
static void launch_gemm_t(const GemmProb* d_probs, const PList<GemmProb, NP>& pl, int nprob,
                          int total_tiles, bool transA, cudaStream_t st) {
  if (gemm_variant() == 2 || gemm_variant() == 3) {
    const size_t smem = (size_t)ST2 * BK2 * (TILE2_M + 4 + TILE2_N + 4) * sizeof(double);
    static bool init = false;
    if (!init) {
      CUDA_TRY(cudaFuncSetAttribute(gemm_dmma2_kernel<true, NP, TILE2_M, TILE2_N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CUDA_TRY(cudaFuncSetAttribute(gemm_dmma2_kernel<false, NP, TILE2_M, TILE2_N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CUDA_TRY(cudaFuncSetAttribute(gemm_dmma2_kernel<true, NP, TILE2_N, TILE2_M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CUDA_TRY(cudaFuncSetAttribute(gemm_dmma2_kernel<false, NP, TILE2_N, TILE2_M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      init = true;
    }
    if (gemm_variant() == 2) {
      if (transA)
        gemm_dmma2_kernel<true, NP, TILE2_M, TILE2_N><<<total_tiles, NT2, smem, st>>>(d_probs, nprob, pl);
      else
        gemm_dmma2_kernel<false, NP, TILE2_M, TILE2_N><<<total_tiles, NT2, smem, st>>>(d_probs, nprob, pl);
    } else {
      if (transA)
        gemm_dmma2_kernel<true, NP, TILE2_N, TILE2_M><<<total_tiles, NT2, smem, st>>>(d_probs, nprob, pl);
      else
        gemm_dmma2_kernel<false, NP, TILE2_N, TILE2_M><<<total_tiles, NT2, smem, st>>>(d_probs, nprob, pl);
    }
    SPQ_LAUNCH_CHECK();
    return;
  }
  if (transA)
    gemm_dmma_kernel<true, NP><<<total_tiles, NT, 0, st>>>(d_probs, nprob, pl);
  else
    gemm_dmma_kernel<false, NP><<<total_tiles, NT, 0, st>>>(d_probs, nprob, pl);
  SPQ_LAUNCH_CHECK();
}

void launch_gemm(const GemmProb* d_probs, const GemmProb* h_probs, int nprob, int total_tiles,
                 bool transA, cudaStream_t st) {
  if (nprob <= 0 || total_tiles <= 0) return;
  if (d_probs == nullptr) {
    if (nprob > PL_GEMM) throw std::runtime_error("launch_gemm: parameter list too long");
    PList<GemmProb, PL_GEMM> pl;
    for (int i = 0; i < nprob; ++i) pl.v[i] = h_probs[i];
    launch_gemm_t<PL_GEMM>(nullptr, pl, nprob, total_tiles, transA, st);
  } else {
    launch_gemm_t<1>(d_probs, PList<GemmProb, 1>{}, nprob, total_tiles, transA, st);
  }
}

}  // namespace spq
