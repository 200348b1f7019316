// Data-movement kernels of the block-sparse store (SURVEY §8a rows a2, a3,
// a13, a14): batched gather/scatter/transposed copies between blocks and
// front buffers, zero fills, identity writes, row-nonzero flags for the host
// planner (the device twin of `np.any(blk, axis=1)` at factor.py:422 and
// `np.any(sub)` at factor.py:454), the CSC equilibration + block scatter of
// TrailingState.__init__ (factor.py:335-374, sparse.py:142-166), and the
// exact nonzero count behind the `trailing_nnz` statistic (factor.py:887).
//
// All of these are HBM-bound byte movers: coalesced along the contiguous
// (row) dimension of the column-major blocks, grid-strided.
#include "common.cuh"

namespace spq {

// Element e of a task maps to (row i, column j) = (e mod nr, e div nr).  A
// 64-bit division per element was the kernel's top stall (ncu: 34% of
// samples); tasks below 2^32 elements use a per-CTA magic-number division
// (Granlund-Montgomery, round-up variant): three integer ops per element.
struct FastDiv {
  uint32_t d, m, s;
  __device__ explicit FastDiv(uint32_t dd) : d(dd), m(0), s(0) {
    if (d > 1) {
      uint32_t l = 32 - __clz(d - 1);   // ceil(log2 d)
      m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << l) - d)) / d) + 1;
      s = l;
    }
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d == 1) return n;
    const uint32_t t = __umulhi(m, n);
    return (t + ((n - t) >> 1)) >> (s - 1);
  }
};

// Element loop of one task: CTA `cb` of `nb` CTAs assigned to it.  Four
// elements per thread and pass with the loads issued before the stores: the
// one-element loop kept a single load in flight per thread (the copies ran
// at ~1.07 TB/s, 16% of the HBM peak, bench r02).
__device__ __forceinline__ void copy_task_elems(const CopyTask& t, int64_t cb, int64_t nb) {
  const int64_t total = (int64_t)t.nr * t.nc;
  const int64_t stride = nb * blockDim.x;
  const bool small = total + 4 * stride < ((int64_t)1 << 32);
  const FastDiv fd((uint32_t)(t.nr > 0 ? t.nr : 1));
  constexpr int U = 4;
  for (int64_t e0 = cb * blockDim.x + threadIdx.x; e0 < total; e0 += U * stride) {
    int ii[U], jj[U];
    double v[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      ok[u] = e < total;
      if (small) {
        const uint32_t q = fd.div((uint32_t)e);
        jj[u] = (int)q;
        ii[u] = (int)((uint32_t)e - q * (uint32_t)t.nr);
      } else {
        ii[u] = (int)(e % t.nr);
        jj[u] = (int)(e / t.nr);
      }
    }
    if (t.ident) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = (ii[u] == jj[u]) ? 1.0 : 0.0;
    } else if (t.src == nullptr) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = 0.0;
    } else {
      int si[U];
#pragma unroll
      for (int u = 0; u < U; ++u) si[u] = (ok[u] && t.src_rows) ? t.src_rows[ii[u]] : ii[u];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ok[u] ? t.src[si[u] + (int64_t)jj[u] * t.lds] : 0.0;
    }
    if (t.trans) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) t.dst[jj[u] + (int64_t)ii[u] * t.ldd] = v[u];
    } else {
      int di[U];
#pragma unroll
      for (int u = 0; u < U; ++u) di[u] = (ok[u] && t.dst_rows) ? t.dst_rows[ii[u]] : ii[u];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) t.dst[di[u] + (int64_t)jj[u] * t.ldd] = v[u];
    }
  }
}

// Rectangular grid (task, CTA within task): used when the tasks have similar
// sizes (the rectangle wastes at most a few empty CTAs per task).
template <int NP>
__global__ void __launch_bounds__(256) copy_tasks_kernel(const CopyTask* __restrict__ tasks_g,
                                                         const __grid_constant__ PList<CopyTask, NP> pl) {
  const CopyTask t = NP > 1 ? pl.v[blockIdx.x] : tasks_g[blockIdx.x];
  copy_task_elems(t, blockIdx.y, gridDim.y);
}

// Flattened grid: task k owns CTAs [cta0, cta0 + ncta).  Mixed batches (one
// huge front buffer among 10^5 small blocks) would otherwise launch
// ntasks x max-CTAs mostly empty CTAs (C5 level 8: seconds of empty CTA
// scheduling).  Warp 0 finds the task by a 32-ary search over cta0.
__global__ void __launch_bounds__(256) copy_tasks_flat_kernel(const CopyTask* __restrict__ tasks,
                                                              int ntasks) {
  __shared__ int s_task;
  const int bid = (int)blockIdx.x;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int lo = 0, n = ntasks;   // invariant: tasks[lo].cta0 <= bid
    while (n > 1) {
      const int seg = (n + 31) / 32;
      const int idx = lo + lane * seg;
      const bool ok = lane * seg < n && tasks[idx].cta0 <= bid;
      const unsigned msk = __ballot_sync(0xffffffffu, ok);
      const int last = 31 - __clz(msk);
      lo += last * seg;
      n = min(seg, n - last * seg);
    }
    if (lane == 0) s_task = lo;
  }
  __syncthreads();
  const CopyTask t = tasks[s_task];
  copy_task_elems(t, bid - t.cta0, t.ncta);
}

// h_tasks carry cta0/ncta (set by the caller for the flattened grid);
// total_ctas = their sum; max_elems = the largest task.
void launch_copy(const CopyTask* d_tasks, const CopyTask* h_tasks, int ntasks, int64_t max_elems,
                 int64_t total_ctas, cudaStream_t st, int64_t gran) {
  if (ntasks <= 0) return;
  if (gran < 256) gran = 256 * 8;
  int64_t y = (max_elems + gran - 1) / gran;
  if (y < 1) y = 1;
  if (y > 512) y = 512;
  if (d_tasks != nullptr && total_ctas > 0 && (int64_t)ntasks * y > 4 * total_ctas + 4096) {
    copy_tasks_flat_kernel<<<(unsigned)total_ctas, 256, 0, st>>>(d_tasks, ntasks);
    SPQ_LAUNCH_CHECK();
    return;
  }
  // grid.x limit is 2^31-1; y <= 512 stays far below the 65535 limit
  dim3 grid((unsigned)ntasks, (unsigned)y);
  if (d_tasks == nullptr) {
    if (ntasks > PL_COPY) throw std::runtime_error("launch_copy: parameter list too long");
    PList<CopyTask, PL_COPY> pl;
    for (int i = 0; i < ntasks; ++i) pl.v[i] = h_tasks[i];
    copy_tasks_kernel<PL_COPY><<<grid, 256, 0, st>>>(nullptr, pl);
  } else {
    copy_tasks_kernel<1><<<grid, 256, 0, st>>>(d_tasks, PList<CopyTask, 1>{});
  }
  SPQ_LAUNCH_CHECK();
}

// one CTA per block; thread per row; flag = any nonzero in the row
__global__ void __launch_bounds__(256) rowflags_kernel(const double* const* __restrict__ ptrs,
                                                       const int* __restrict__ nr,
                                                       const int* __restrict__ nc,
                                                       const int64_t* __restrict__ off,
                                                       unsigned char* __restrict__ out) {
  const int b = blockIdx.x;
  const double* p = ptrs[b];
  const int R = nr[b], C = nc[b];
  unsigned char* o = out + off[b];
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    bool f = false;   // eight columns per round, loads issued together
    for (int j = 0; j < C && !f; j += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (j + u < C) ? p[i + (int64_t)(j + u) * R] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) f = f || (v[u] != 0.0);
    }
    o[i] = (unsigned char)f;
  }
}

void launch_rowflags(const double* const* d_ptrs, const int* d_nr, const int* d_nc,
                     const int64_t* d_off, unsigned char* d_out, int nblk, cudaStream_t st) {
  if (nblk <= 0) return;
  rowflags_kernel<<<nblk, 128, 0, st>>>(d_ptrs, d_nr, d_nc, d_off, d_out); SPQ_LAUNCH_CHECK();
}

// Speculative-mode check: the row flags the host PREDICTED (pred) against
// the block values; every mismatching row adds one to *bad.
__global__ void __launch_bounds__(128) rowflags_verify_kernel(const double* const* __restrict__ ptrs,
                                                              const int* __restrict__ nr,
                                                              const int* __restrict__ nc,
                                                              const int64_t* __restrict__ off,
                                                              const unsigned char* __restrict__ pred,
                                                              int* bad) {
  const int b = blockIdx.x;
  const double* p = ptrs[b];
  const int R = nr[b], C = nc[b];
  const unsigned char* q = pred + off[b];
  int miss = 0;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    // eight columns per round, loads issued together (a zero row walks all C
    // columns: one dependent load per column cost ~0.3 us each)
    bool f = false;
    for (int j = 0; j < C && !f; j += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (j + u < C) ? p[i + (int64_t)(j + u) * R] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) f = f || (v[u] != 0.0);
    }
    miss += ((unsigned char)f != q[i]);
  }
  for (int o = 16; o; o >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, o);
  if ((threadIdx.x & 31) == 0 && miss) atomicAdd(bad, miss);
}

void launch_rowflags_verify(const double* const* d_ptrs, const int* d_nr, const int* d_nc,
                            const int64_t* d_off, const unsigned char* d_pred, int nblk, int* d_bad,
                            cudaStream_t st) {
  if (nblk <= 0) return;
  rowflags_verify_kernel<<<nblk, 128, 0, st>>>(d_ptrs, d_nr, d_nc, d_off, d_pred, d_bad);
  SPQ_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) count_nnz_kernel(const double* const* __restrict__ ptrs,
                                                        const int64_t* __restrict__ sizes,
                                                        unsigned long long* count) {
  const double* p = ptrs[blockIdx.x];
  const int64_t n = sizes[blockIdx.x];
  unsigned long long c = 0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) c += (p[e] != 0.0);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

void launch_count_nnz(const double* const* d_ptrs, const int64_t* d_sizes, int nblk,
                      unsigned long long* d_count, cudaStream_t st) {
  if (nblk <= 0) return;
  count_nnz_kernel<<<nblk, 256, 0, st>>>(d_ptrs, d_sizes, d_count); SPQ_LAUNCH_CHECK();
}

// Column 2-norms accumulated sequentially in CSC entry order, no FMA
// contraction: bit-identical to `np.add.at(sq, col_of, data**2)` followed by
// sqrt and division (sparse.py:96-106, 158-166).
__global__ void colnorms_scale_kernel(const int64_t* __restrict__ indptr, double* data, int64_t N,
                                      double* scale, int* zero_col, int equilibrate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const int64_t a = indptr[j], b = indptr[j + 1];
  double s = 0.0;
  for (int64_t e = a; e < b; ++e) s = __dadd_rn(s, __dmul_rn(data[e], data[e]));
  const double nrm = sqrt(s);
  if (nrm == 0.0) atomicMin(zero_col, (int)j);
  if (equilibrate) {
    scale[j] = nrm;
    if (nrm != 0.0)
      for (int64_t e = a; e < b; ++e) data[e] = data[e] / nrm;
  }
}

void launch_colnorms_scale(const int64_t* indptr, const int64_t* /*indices*/, double* data,
                           int64_t N, double* scale, int* zero_col, int equilibrate,
                           cudaStream_t st) {
  if (N <= 0) return;
  colnorms_scale_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(indptr, data, N, scale,
                                                                      zero_col, equilibrate); SPQ_LAUNCH_CHECK();
}

// entry e of the CSC goes to blk_base[entry_blk[e]][dest_off[e]]
__global__ void csc_scatter_kernel(const double* __restrict__ data, int64_t nnz,
                                   const int64_t* __restrict__ dest_off,
                                   double* const* __restrict__ blk_base,
                                   const int* __restrict__ entry_blk) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  blk_base[entry_blk[e]][dest_off[e]] = data[e];
}

void launch_csc_scatter(const int64_t* indptr, const int64_t* /*indices*/, const double* data,
                        int64_t nnz, const int64_t* dest_off, double* const* blk_base,
                        const int* entry_blk, cudaStream_t st) {
  (void)indptr;
  if (nnz <= 0) return;
  csc_scatter_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(data, nnz, dest_off,
                                                                     blk_base, entry_blk); SPQ_LAUNCH_CHECK();
}

}  // namespace spq
