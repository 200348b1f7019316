// Native runtime of the B200 spaQR path: the HBM-resident block store, the
// wave planner that batches independent eliminations, the level operations
// (a) factor, (b) scale, (c) sparsify, (d) merge, the transform records and
// the solve-phase chains (e), exported through the C-ABI in
// include/spaqr_b200.h.
//
// Semantics follow the reference TrailingState (pkg/src/nestqr/factor.py):
// the host keeps the block STRUCTURE (which (row cluster, col cluster)
// blocks exist, their row/col index sets, row_of_col) exactly as the
// reference's dicts do; every VALUE lives in device memory.  Data-dependent
// structure decisions (`np.any` row subsets and present-column filters,
// factor.py:422,454) read per-row nonzero flags computed on the device.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <malloc.h>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/spaqr_b200.h"
#include "common.cuh"

namespace spq {
// launchers defined in other translation units

void launch_cpqr(const CpqrArgs& a, int G, cudaStream_t st);
int cpqr_grid(int ncols, int nsm);
void launch_sparsify_prep(const double* M, int m, int n, double eps, double* sq, int* keep_idx,
                          int* nk, double* ratio, double* maxcol, double* W, cudaStream_t st,
                          int allow_filter = 1);
void launch_sparsify_prep_batch(const PrepJob* d_jobs, const PrepJob* h_jobs, int njobs, double eps,
                                cudaStream_t st);
int sparsify_prep_plist_max();
void launch_jacobi_sv(const SvJob* d_jobs, int n, cudaStream_t st);
void chain_wy(const double* V, const double* T, int m, int k, double* z, const int* rows,
              int64_t N, int nrhs, bool transpose, double* w, double* w2, cudaStream_t st);
void chain_tri(const double* R, int k, const double* Rsn, int n, double* y, const int* cols_s,
               const int* cols_n, int64_t N, int nrhs, int mode, double* part, cudaStream_t st);
int chain_rsn_chunks(int n);
void chain_diag(double* y, const double* s, int64_t N, int nrhs, bool divide, cudaStream_t st);
void chain_perm(const double* z, const int* roc, int64_t N, int nrhs, double* out,
                cudaStream_t st);
constexpr int CHAIN_SLAB_KMAX = 320;
}  // namespace spq

using namespace spq;

namespace {

struct SpqError : std::runtime_error {
  int code;
  int64_t index;
  double value;
  SpqError(int c, const std::string& m, int64_t i = -1, double v = 0.0)
      : std::runtime_error(m), code(c), index(i), value(v) {}
};

inline uint64_t bkey(int i, int j) { return ((uint64_t)(uint32_t)i << 32) | (uint32_t)j; }

// Per-row flags of one block with inline storage for short blocks: the
// planner creates ~10^4 blocks per level on the leaf levels, most with
// fewer than 56 rows -- no heap allocation for those.
class RowFlags {
  static constexpr int INL = 56;
  uint8_t* p_ = inl_;
  int n_ = 0, cap_ = INL;
  uint8_t inl_[INL];
  void reserve_(int n) {
    if (n <= cap_) return;
    uint8_t* q = new uint8_t[n];
    if (p_ != inl_) delete[] p_;
    p_ = q;
    cap_ = n;
  }

 public:
  RowFlags() = default;
  RowFlags(const RowFlags& o) { assign(o.begin(), o.end()); }
  RowFlags& operator=(const RowFlags& o) {
    if (this != &o) assign(o.begin(), o.end());
    return *this;
  }
  RowFlags(RowFlags&& o) noexcept { *this = std::move(o); }
  RowFlags& operator=(RowFlags&& o) noexcept {
    if (this == &o) return *this;
    if (o.p_ != o.inl_) {   // steal the heap buffer
      if (p_ != inl_) delete[] p_;
      p_ = o.p_; cap_ = o.cap_; n_ = o.n_;
      o.p_ = o.inl_; o.cap_ = INL; o.n_ = 0;
    } else {
      n_ = 0;
      assign(o.begin(), o.end());
      o.n_ = 0;
    }
    return *this;
  }
  ~RowFlags() { if (p_ != inl_) delete[] p_; }
  void assign(size_t n, uint8_t v) {
    reserve_((int)n);
    n_ = (int)n;
    std::memset(p_, v, n);
  }
  template <class It, class = typename std::enable_if<!std::is_integral<It>::value>::type>
  void assign(It a, It b) {
    const int n = (int)(b - a);
    reserve_(n);
    n_ = n;
    std::copy(a, b, p_);
  }
  void clear() { n_ = 0; }
  bool empty() const { return n_ == 0; }
  size_t size() const { return (size_t)n_; }
  uint8_t& operator[](size_t i) { return p_[i]; }
  const uint8_t& operator[](size_t i) const { return p_[i]; }
  const uint8_t* begin() const { return p_; }
  const uint8_t* end() const { return p_ + n_; }
};

struct Block {
  double* p = nullptr;
  void* base = nullptr;        // shared (refcounted) allocation this block lives in
  size_t abytes = 0;           // own allocation (base == nullptr): bytes requested from the pool
  int nr = 0, nc = 0;
  RowFlags flags;              // per row: 0 zero, 1 nonzero, 2 unknown (written)
  bool clean = false;
  // flags PREDICTED by the symbolic rules (speculative mode), not yet
  // checked against the device values; checked at the next query
  bool unverified = false;
  uint8_t origin = 0;   // last predicting site (SPQ_SPEC_DEBUG reports)
};

// 64-bit key -> small value, open addressing with linear probing (the
// allocator's pointer tables: one probe instead of a node allocation and two
// cache misses per dalloc/dfree)
template <class V>
class FlatMap {
  static constexpr uint64_t EMPTY = ~0ull, TOMB = ~1ull;
  std::vector<uint64_t> keys_;
  std::vector<V> vals_;
  size_t live_ = 0, used_ = 0;
  static size_t mix(uint64_t k) {
    k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
    return (size_t)k;
  }
  void rehash(size_t cap) {
    std::vector<uint64_t> ok;
    std::vector<V> ov;
    ok.swap(keys_);
    ov.swap(vals_);
    keys_.assign(cap, EMPTY);
    vals_.assign(cap, V());
    used_ = live_;
    for (size_t t = 0; t < ok.size(); ++t)
      if (ok[t] < TOMB) {
        size_t h = mix(ok[t]) & (cap - 1);
        while (keys_[h] != EMPTY) h = (h + 1) & (cap - 1);
        keys_[h] = ok[t];
        vals_[h] = ov[t];
      }
  }
  size_t slot_of(uint64_t k) const {
    const size_t m = keys_.size() - 1;
    for (size_t h = mix(k) & m;; h = (h + 1) & m) {
      if (keys_[h] == k) return h;
      if (keys_[h] == EMPTY) return SIZE_MAX;
    }
  }

 public:
  FlatMap() { rehash(1024); }
  size_t size() const { return live_; }
  V* find(uint64_t k) {
    const size_t h = slot_of(k);
    return h == SIZE_MAX ? nullptr : &vals_[h];
  }
  V& operator[](uint64_t k) {
    if (V* v = find(k)) return *v;
    if (2 * (used_ + 1) > keys_.size()) rehash(keys_.size() * (2 * (live_ + 1) > keys_.size() / 2 ? 2 : 1));
    const size_t m = keys_.size() - 1;
    size_t h = mix(k) & m;
    while (keys_[h] < TOMB) h = (h + 1) & m;
    if (keys_[h] == EMPTY) ++used_;
    keys_[h] = k;
    vals_[h] = V();
    ++live_;
    return vals_[h];
  }
  bool erase(uint64_t k) {
    const size_t h = slot_of(k);
    if (h == SIZE_MAX) return false;
    keys_[h] = TOMB;
    --live_;
    return true;
  }
  void clear() { keys_.assign(keys_.size(), EMPTY); live_ = used_ = 0; }
};
inline uint64_t pkey(const void* p) { return (uint64_t)(uintptr_t)p; }

// Block objects live in a deque (stable references across inserts) recycled
// through a free list.  There is no (row, col) -> Block hash table any more:
// every lookup goes through the sorted row adjacency list of the row cluster
// (FlatSet below carries the Block pointers), which the planner had at hand
// anyway; the hash insert / erase per block was ~3 ms of host time per C3
// factorization.
class BlockMap {
  std::deque<Block> pool_;
  std::vector<Block*> free_;
  size_t live_ = 0;

 public:
  size_t size() const { return live_; }
  bool empty() const { return live_ == 0; }
  void reserve(size_t) {}
  Block& create() {
    ++live_;
    if (!free_.empty()) {
      Block* b = free_.back();
      free_.pop_back();
      return *b;
    }
    pool_.emplace_back();
    return pool_.back();
  }
  void destroy(Block* b) {
    *b = Block();
    free_.push_back(b);
    --live_;
  }
  void swap(BlockMap& o) {
    pool_.swap(o.pool_); free_.swap(o.free_);
    std::swap(live_, o.live_);
  }
};

// sorted small-vector set (cluster adjacency lists are short; iteration
// must be ascending like the reference's sorted(...) calls).  Each entry
// also carries the Block it stands for, so the planner's block lookups are a
// binary search in a short, cache-resident row list instead of a hash probe.
struct FlatSet {
  std::vector<int> v;
  std::vector<Block*> b;
  void insert(int x, Block* blk = nullptr) {
    if (v.empty() || x > v.back()) {   // ascending arrival (merge, load): append, no search
      v.push_back(x);
      b.push_back(blk);
      return;
    }
    auto it = std::lower_bound(v.begin(), v.end(), x);
    const size_t i = (size_t)(it - v.begin());
    if (it == v.end() || *it != x) {
      v.insert(it, x);
      b.insert(b.begin() + i, blk);
    } else if (blk) {
      b[i] = blk;
    }
  }
  void erase(int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it != v.end() && *it == x) {
      b.erase(b.begin() + (it - v.begin()));
      v.erase(it);
    }
  }
  Block* find(int x) const {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    return (it != v.end() && *it == x) ? b[it - v.begin()] : nullptr;
  }
  void clear() { v.clear(); b.clear(); }
  std::vector<int>::const_iterator begin() const { return v.begin(); }
  std::vector<int>::const_iterator end() const { return v.end(); }
};

// pivot checks (factor.py:57-68) queued on the device, raised in order at
// the next synchronization point
struct PivotSet {
  std::vector<PivotJob> jobs;
  std::vector<std::string> ctx;
  size_t launched = 0;   // jobs[0, launched) already checked on the device
};

enum RecKind { REC_ELIM = 1, REC_SCALE = 2, REC_SPARSIFY = 3 };

struct Record {
  int kind = 0;
  int m = 0, k = 0, n = 0, rank = 0;
  int cid = -1;          // cluster the record eliminates / scales / compresses
  // unscaled sparsifier (factor.py:660-709): H_f panel (m x f) + R_ff (f x f, in R)
  // + R_fc (f x rank, in Rsn); fine / coarse column lists for the W-side ops
  bool unscaled = false;
  int f = 0;
  double *hV = nullptr, *htau = nullptr, *hT = nullptr;
  std::vector<int64_t> cols_f, cols_c;
  int *d_cols_f = nullptr, *d_cols_c = nullptr;
  std::vector<int64_t> rows, cols_s, cols_n;
  double* payload = nullptr;
  double *V = nullptr, *tau = nullptr, *T = nullptr, *R = nullptr, *Rsn = nullptr;
  int *d_rows = nullptr, *d_cols_s = nullptr, *d_cols_n = nullptr;
  int64_t payload_scalars = 0;
  bool full_T = false;   // T already complete (built for a target update)
  double* WT = nullptr;  // chain: V T^T (m x k), built at chain compile time
  double* WN = nullptr;  // chain: V T (sparsifiers, solve_w direction)
};

// families for device timing / flop accounting
enum Fam { F_COPY = 0, F_QR, F_WY, F_TRSM, F_CPQR, F_FLAGS, F_CHAIN, F_NFAM };

struct FamTimer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[F_NFAM];
  std::vector<std::string> tag[F_NFAM];   // SPQ_SCOPE_LOG only
  double ms[F_NFAM] = {0};
  double flops[F_NFAM] = {0};
  double bytes[F_NFAM] = {0};
  int64_t launches[F_NFAM] = {0};
};


}  // namespace

struct spq_ctx {
  int dev = 0;
  int nsm = 148;
  cudaStream_t st = nullptr;
  // pinned upload ring
  char* pin = nullptr;
  char* dring = nullptr;
  size_t ring_cap = 0, ring_off = 0;
  // error
  int err_code = 0;
  int64_t err_index = -1;
  double err_value = 0.0;
  std::string err_msg;
  // structure
  int64_t N = 0;
  int ncl = 0;
  std::vector<std::vector<int64_t>> rows_of, cols_of;
  std::vector<char> active;
  std::vector<FlatSet> rix, cix;
  BlockMap blk;
  std::vector<int64_t> row_of_col;
  std::vector<double*> deferred;
  std::vector<std::pair<void*, size_t>> deferred_blk;   // block memory: (pointer, bytes), see dfree_block
  std::vector<std::pair<void*, size_t>> side_free_blk;
  // transform chain
  std::vector<Record> recs;
  double* d_scale = nullptr;
  double* d_dropped = nullptr;
  bool equil = false;
  int* d_roc = nullptr;
  int* d_index_pack = nullptr;
  bool finished = false;
  bool compiled = false;
  // speculative row flags (no host sync per factor wave); mismatches found
  // by the device verification are counted in d_spec_bad (mapped pinned)
  bool spec = true;
  int* h_spec_bad = nullptr;
  int* d_spec_bad = nullptr;
  int64_t n_verified = 0;
  int64_t n_sparsify_waves = 0;
  PivotSet piv;   // speculative mode: checks pending across calls
  unsigned long long* d_nnz_slots = nullptr;   // per-level trailing_nnz counters
  // device GMRES: the original (unscaled) matrix in CSR
  int64_t* d_csr_ptr = nullptr;
  int* d_csr_idx = nullptr;
  double* d_csr_val = nullptr;
  // device error slots for pivot checks
  int64_t* d_err_idx = nullptr;
  double* d_err_val = nullptr;
  int err_slots = 0;
  // timing
  bool timing = true;
  FamTimer tm;
  // scratch for chains
  double* d_vec = nullptr;
  double* d_vec2 = nullptr;
  double* d_w = nullptr;
  double* d_w2 = nullptr;
  double* d_part = nullptr;
  size_t vec_cap = 0, w_cap = 0, part_cap = 0;
  // device memory pool
  // free lists by size class (flat: class sizes grow in quarter-octave steps, ~100 classes
  // below 8 MB): kv.first = class bytes, kv.second = (ptr, slab) entries
  struct ClassFree {
    std::vector<std::pair<size_t, std::vector<std::pair<void*, int>>>> v;
    std::vector<std::pair<void*, int>>& operator[](size_t cls) {
      const size_t i = index_of(cls);
      if (i >= v.size()) v.resize(i + 1);
      v[i].first = cls;
      return v[i].second;
    }
    static size_t index_of(size_t cls) {   // cls is a size_class() value: 256-byte multiples
      const size_t u = cls >> 8;
      const int l = 63 - __builtin_clzll((unsigned long long)u);
      return l < 2 ? u : (size_t)4 * l + ((u >> (l - 2)) & 3);
    }
    std::vector<std::pair<size_t, std::vector<std::pair<void*, int>>>>::iterator begin() { return v.begin(); }
    std::vector<std::pair<size_t, std::vector<std::pair<void*, int>>>>::iterator end() { return v.end(); }
  } pool_free;
  bool counted = false;   // included in gcache().n_ctx
  // side stream: work off the critical path whose result is only read at a
  // later join (the sparsifiers' dropped-norm statistic).  While `on_side`,
  // launches go to the side stream, uploads bypass the ring and every free
  // is held in side_free until side_join() orders it after the side work.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_side_a = nullptr, ev_side_b = nullptr;
  bool on_side = false, side_pending = false;
  std::vector<void*> side_free;
  static constexpr int NAUX = 4;
  cudaStream_t aux[NAUX] = {};               // fork-join streams for independent launches
  cudaEvent_t ev_fork = nullptr, ev_join[NAUX] = {};
  const char* stage = "";   // innermost runtime stage (OOM reports)
  struct PoolEnt { size_t cls; int slab; };
  FlatMap<PoolEnt> pool_size;
  std::vector<void*> slabs;          // nullptr once reclaimed
  std::vector<size_t> slab_caps;
  std::vector<int64_t> slab_live;    // live pool buffers per slab
  int cur_slab = -1;
  FlatMap<int> refcnt;   // shared block allocations
  std::set<void*> big;                      // large buffers (arena)
  std::vector<void*> big_pending;           // freed, awaiting a stream sync
  std::unordered_map<void*, size_t> big_size;
  size_t live_bytes = 0, peak_bytes = 0;
  char* slab_ptr = nullptr;
  size_t slab_off = 0, slab_cap = 0, pool_bytes = 0;
  // host-side accounting: [alloc, sync-wait, plan, api]
  double host_ms[16] = {0};
  int64_t n_allocs = 0, n_syncs = 0, n_kernels = 0, n_ring_overflow = 0;
  std::vector<cudaEvent_t> marks;
  std::vector<cudaEvent_t> ev_pool;
  // compiled solve-chain programs: 0 apply_qt, 1 solve_w, 2 apply_w
  struct Prog {
    ChainOp* d_ops = nullptr;
    int2* d_tasks = nullptr;
    std::vector<int> toff, tcnt;          // per wave: task range
    std::vector<int64_t> part_sz;         // per wave: partial-sum doubles (x nrhs)
    std::map<int, double*> part_buf;      // nrhs -> wave scratch (max over waves)
    std::vector<int> off, cnt, kmax, slabk;   // slabk: back-substitution slab width (0: none)
    std::vector<char> has_wy;                 // per wave: any WY op (phase B launched)
    std::map<int, cudaGraphExec_t> graphs;   // nrhs -> executable graph (z = d_vec)
    std::vector<ChainOp> hops;               // host copy of the ordered ops (diagnostics)
  } prog[3];
};

namespace {

// ------------------------------------------------------------ utilities
// Process-wide caches: device slabs and the pinned upload ring outlive a
// context, so repeated factorizations do not pay cudaMalloc/cudaMallocHost.
// Best-fit arena with coalescing for large buffers (one reservation per
// process; no driver calls in steady state).
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  std::map<size_t, size_t> free_off;             // offset -> size
  std::multimap<size_t, size_t> free_size;       // size -> offset
  std::unordered_map<size_t, size_t> used;       // offset -> size
  void add_free(size_t off, size_t sz) {
    auto nx = free_off.lower_bound(off);
    if (nx != free_off.end() && off + sz == nx->first) {   // merge with the next block
      erase_size(nx->second, nx->first);
      sz += nx->second;
      nx = free_off.erase(nx);
    }
    if (nx != free_off.begin()) {                            // merge with the previous block
      auto pv = std::prev(nx);
      if (pv->first + pv->second == off) {
        erase_size(pv->second, pv->first);
        off = pv->first;
        sz += pv->second;
        free_off.erase(pv);
      }
    }
    free_off[off] = sz;
    free_size.emplace(sz, off);
  }
  void erase_size(size_t sz, size_t off) {
    auto range = free_size.equal_range(sz);
    for (auto it = range.first; it != range.second; ++it)
      if (it->second == off) { free_size.erase(it); return; }
  }
  void* alloc(size_t bytes) {
    bytes = (bytes + 4095) & ~(size_t)4095;
    auto it = free_size.lower_bound(bytes);
    if (it == free_size.end()) return nullptr;
    const size_t sz = it->first, off = it->second;
    free_size.erase(it);
    free_off.erase(off);
    if (sz > bytes) add_free(off + bytes, sz - bytes);
    used[off] = bytes;
    return base + off;
  }
  bool owns(void* p) const { return base && (char*)p >= base && (char*)p < base + cap; }
  size_t size_of(void* p) const { return used.at((size_t)((char*)p - base)); }
  void release(void* p) {
    const size_t off = (size_t)((char*)p - base);
    auto it = used.find(off);
    if (it == used.end()) return;
    const size_t sz = it->second;
    used.erase(it);
    add_free(off, sz);
  }
};

// streams and synchronisation events of a closed context: creating (and
// destroying) six streams per factorization showed up as an occasional
// 30-75 ms host stall at the first fork of a factorization (the first
// multi-group CPQR wave), and the side stream used to leak
struct StreamSet {
  cudaStream_t st = nullptr, side = nullptr, aux[spq_ctx::NAUX] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[spq_ctx::NAUX] = {}, ev_side_a = nullptr, ev_side_b = nullptr;
};

struct GlobalCache {
  std::mutex mu;
  std::vector<StreamSet> stream_sets;            // idle (synchronized) sets of closed contexts
  std::vector<std::pair<void*, size_t>> slabs;   // (ptr, bytes)
  Arena arena;
  std::vector<std::pair<char*, char*>> rings;    // (pinned, device) of RING_BYTES
  std::vector<int*> spec_flags;                  // mapped pinned ints of closed contexts
  std::vector<cudaEvent_t> events;               // timing events of closed contexts
  int events_dev = -1;                           // device those events belong to
  int n_ctx = 0;                                 // live contexts (1 => frees reusable at once)
};
// One cache per device: slabs, arena ranges, rings, mapped flags and events
// belong to the device they were allocated on, and a context only ever draws
// from its own device's cache.
constexpr int kMaxDevices = 64;
GlobalCache& gcache(int dev) {
  static std::mutex mu;
  static GlobalCache* g[kMaxDevices] = {};   // leaked on purpose (process lifetime)
  if (dev < 0 || dev >= kMaxDevices) throw SpqError(SPQ_ERR_BAD_INPUT, "device ordinal out of range");
  std::lock_guard<std::mutex> lk(mu);
  if (!g[dev]) g[dev] = new GlobalCache();
  return *g[dev];
}

size_t arena_free_bytes(int dev) {
  auto& g = gcache(dev);
  std::lock_guard<std::mutex> lk(g.mu);
  size_t t = 0;
  for (auto& kv : g.arena.free_off) t += kv.second;
  return t;
}

struct HostTimer {
  double* acc;
  std::chrono::steady_clock::time_point t0;
  explicit HostTimer(double* a) : acc(a), t0(std::chrono::steady_clock::now()) {}
  ~HostTimer() {
    *acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};
struct Stage {   // tags allocations with the runtime stage making them
  spq_ctx* c;
  const char* prev;
  Stage(spq_ctx* cc, const char* name) : c(cc), prev(cc->stage) { c->stage = name; }
  ~Stage() { c->stage = prev; }
};

// Size-class pool over large cudaMalloc slabs.  All device work of a context
// is ordered on ONE stream, so a buffer released after its last use has been
// enqueued can be handed out again immediately (the same guarantee
// cudaFreeAsync gives) without the per-call driver cost.
size_t size_class(size_t b) {
  if (b <= 256) return 256;
  const size_t p = (size_t)1 << (63 - __builtin_clzll((unsigned long long)b));   // largest power of two <= b
  const size_t q = p >> 2;  // quarter steps: <= 25% waste
  const size_t c = p + ((b - p + q - 1) / q) * q;
  return (c + 255) & ~(size_t)255;
}

constexpr size_t BIG_ALLOC = (size_t)8 << 20;   // >= 8 MB: driver stream-ordered pool

// out-of-memory: report where the memory is (live vs. pooled vs. arena
// fragmentation) instead of a bare cudaMalloc failure
[[noreturn]] void throw_oom(spq_ctx* c, size_t bytes, const char* what) {
  (void)cudaGetLastError();
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  size_t afree = 0, alarge = 0, anfree = 0;
  {
    auto& g = gcache(c->dev);
    std::lock_guard<std::mutex> lk(g.mu);
    for (auto& kv : g.arena.free_off) { afree += kv.second; alarge = std::max(alarge, kv.second); ++anfree; }
  }
  size_t pooled_free = 0;
  for (auto& kv : c->pool_free) pooled_free += kv.first * kv.second.size();
  const double G = 1.0 / (1 << 30);
  char buf[768];
  snprintf(buf, sizeof buf,
           "out of memory (%s, %.3f GB requested): live %.2f GB, peak %.2f GB, slabs %.2f GB "
           "(%.2f GB in free lists), arena %.2f GB with %.2f GB free in %zu ranges (largest %.3f GB), "
           "device free %.2f of %.2f GB, stage %s",
           what, bytes * G, c->live_bytes * G, c->peak_bytes * G, c->pool_bytes * G,
           pooled_free * G, gcache(c->dev).arena.cap * G, afree * G, anfree, alarge * G, fr * G, tot * G,
           c->stage);
  throw spq::CudaFailure(cudaErrorMemoryAllocation, buf, __FILE__, __LINE__);
}

void publish_big(spq_ctx* c);

constexpr size_t kSlabBytes = (size_t)32 << 20;

// Pool slabs whose buffers are all free go back to the arena (after one
// stream sync, so no queued work still touches them), together with the
// process cache of slabs left by destroyed contexts.  The recovery path of
// an arena miss: a level's merge frees most small blocks at once, leaving
// whole slabs empty.  Returns the bytes reclaimed.
size_t reclaim_slabs(spq_ctx* c) {
  std::vector<char> dead(c->slabs.size(), 0);
  bool any = false;
  for (size_t i = 0; i < c->slabs.size(); ++i)
    if (c->slabs[i] && c->slab_live[i] == 0) { dead[i] = 1; any = true; }
  auto& g = gcache(c->dev);
  {
    std::lock_guard<std::mutex> lk(g.mu);
    any = any || !g.slabs.empty();
  }
  // large frees deferred while other contexts live (published at a stream
  // sync) are the other recoverable reserve
  size_t pending = 0;
  for (void* p : c->big_pending) {
    auto it = c->big_size.find(p);
    pending += it != c->big_size.end() ? it->second : 1;
  }
  if (!any && pending == 0) return 0;
  // not sync(): that also recycles the upload ring, and this runs inside
  // dalloc, possibly between an upload and the launch that reads it
  CUDA_TRY(cudaStreamSynchronize(c->st));
  publish_big(c);
  for (auto& kv : c->pool_free) {
    auto& v = kv.second;
    v.erase(std::remove_if(v.begin(), v.end(), [&](const std::pair<void*, int>& e) { return dead[e.second] != 0; }),
            v.end());
  }
  size_t freed = 0;
  std::lock_guard<std::mutex> lk(g.mu);
  for (size_t i = 0; i < c->slabs.size(); ++i) {
    if (!dead[i]) continue;
    if ((int)i == c->cur_slab) { c->slab_ptr = nullptr; c->cur_slab = -1; }
    if (g.arena.owns(c->slabs[i])) g.arena.release(c->slabs[i]);
    else cudaFree(c->slabs[i]);
    freed += c->slab_caps[i];
    c->pool_bytes -= c->slab_caps[i];
    c->slabs[i] = nullptr;
    c->slab_caps[i] = 0;
  }
  for (auto& e : g.slabs) {
    if (g.arena.owns(e.first)) g.arena.release(e.first);
    else cudaFree(e.first);
    freed += e.second;
  }
  g.slabs.clear();
  return freed + pending;
}

// The process-wide arena takes all free HBM but a reserve (for torch and
// other libraries in the process) at first use; SPQ_ARENA_RESERVE_GB
// overrides the reserve.  Caller holds g.mu.
void ensure_arena(GlobalCache& g) {
  if (g.arena.base) return;
  size_t fr = 0, tot = 0;
  CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  const char* e = getenv("SPQ_ARENA_RESERVE_GB");
  size_t reserve = e ? (size_t)(atof(e) * (double)(1ull << 30))
                     : std::max<size_t>((size_t)6 << 30, fr / 20);
  size_t cap = fr > reserve ? fr - reserve : fr / 2;
  cap &= ~(((size_t)1 << 21) - 1);
  void* b = nullptr;
  if (cudaMalloc(&b, cap) != cudaSuccess) { (void)cudaGetLastError(); cap = 0; b = nullptr; }
  g.arena.base = (char*)b;
  g.arena.cap = cap;
  if (cap) g.arena.add_free(0, cap);
}

// tracked = false (block memory, new_block_mem): the pointer is not entered in
// the pointer -> class table; its owner frees it with its size (dfree_block).
// The table's insert / find / erase per block was ~3 ms of host time per C3
// factorization (two cache misses per operation, 10^5 operations).
double* dalloc(spq_ctx* c, size_t bytes, bool tracked = true) {
  if (bytes >= BIG_ALLOC) {
    auto t0 = std::chrono::steady_clock::now();
    // large buffers: process-wide best-fit arena
    void* p = nullptr;
    size_t got = 0;
    {
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      ensure_arena(g);
      if (g.arena.base) {
        p = g.arena.alloc(bytes);
        if (p) got = g.arena.size_of(p);
      }
    }
    if (!p && reclaim_slabs(c) > 0) {   // empty pool slabs back to the arena, retry
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      p = g.arena.alloc(bytes);
      if (p) got = g.arena.size_of(p);
    }
    if (!p) {   // arena exhausted: dedicated allocation
      if (cudaMalloc(&p, bytes) != cudaSuccess) throw_oom(c, bytes, "large buffer");
      got = bytes;
    }
    c->big.insert(p);
    c->big_size[p] = got;
    c->live_bytes += got;
    c->peak_bytes = std::max(c->peak_bytes, c->live_bytes);
    c->n_allocs++;
    c->host_ms[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return (double*)p;
  }
  const size_t cls = size_class(bytes == 0 ? 8 : bytes);
  void* p = nullptr;
  int sid = -1;
  auto& fl = c->pool_free[cls];
  if (!fl.empty()) {
    p = fl.back().first;
    sid = fl.back().second;
    fl.pop_back();
  } else {
    if (c->slab_ptr == nullptr || c->slab_off + cls > c->slab_cap) {
      size_t cap = std::max<size_t>(cls, kSlabBytes);
      void* s = nullptr;
      for (int attempt = 0; attempt < 2 && !s; ++attempt) {
        if (attempt == 1 && reclaim_slabs(c) == 0) break;
        auto& g = gcache(c->dev);
        std::lock_guard<std::mutex> lk(g.mu);
        for (size_t i = 0; i < g.slabs.size(); ++i)
          if (g.slabs[i].second >= cap) {
            s = g.slabs[i].first;
            cap = g.slabs[i].second;
            g.slabs.erase(g.slabs.begin() + i);
            break;
          }
        if (!s) {   // carve the slab from the arena
          ensure_arena(g);
          if (g.arena.base) s = g.arena.alloc(cap);
        }
      }
      if (!s && cudaMalloc(&s, cap) != cudaSuccess) throw_oom(c, cap, "pool slab");
      c->slabs.push_back(s);
      c->slab_caps.push_back(cap);
      c->slab_live.push_back(0);
      c->cur_slab = (int)c->slabs.size() - 1;
      c->slab_ptr = (char*)s;
      c->slab_off = 0;
      c->slab_cap = cap;
      c->pool_bytes += cap;
    }
    p = c->slab_ptr + c->slab_off;
    sid = c->cur_slab;
    c->slab_off += cls;
  }
  if (tracked) c->pool_size[pkey(p)] = spq_ctx::PoolEnt{cls, sid};
  c->slab_live[sid]++;
  c->live_bytes += cls;
  c->peak_bytes = std::max(c->peak_bytes, c->live_bytes);
  c->n_allocs++;   // (small path untimed: two clock reads would cost as much as the pool op)
  return (double*)p;
}
// Scratch whose size is a free parameter (chunk widths, WY batches): the
// largest power-of-two fraction of `want` (>= `floor`) the arena can give
// right now; `got` receives the size.  Falls back to dalloc at the floor.
double* dalloc_flex(spq_ctx* c, size_t want, size_t floor, size_t* got) {
  floor = std::min(floor, want);
  if (want < BIG_ALLOC) {
    *got = std::max<size_t>(want, 8);
    return dalloc(c, *got);
  }
  {
    auto& g = gcache(c->dev);
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (attempt == 1 && reclaim_slabs(c) == 0) break;
      std::lock_guard<std::mutex> lk(g.mu);
      ensure_arena(g);
      if (!g.arena.base) break;
      for (size_t b = want; b >= std::max(floor, BIG_ALLOC); b /= 2) {
        void* p = g.arena.alloc(b);
        if (!p) continue;
        const size_t sz = g.arena.size_of(p);
        c->big.insert(p);
        c->big_size[p] = sz;
        c->live_bytes += sz;
        c->peak_bytes = std::max(c->peak_bytes, c->live_bytes);
        c->n_allocs++;
        *got = b;
        return (double*)p;
      }
    }
  }
  *got = std::max<size_t>(floor, 8);
  return dalloc(c, *got);
}

void dfree(spq_ctx* c, void* p) {
  if (!p) return;
  if (c->on_side) {   // still used by queued side work: released at side_join
    c->side_free.push_back(p);
    return;
  }
  auto bi = c->big.find(p);
  if (bi != c->big.end()) {
    c->big.erase(bi);
    c->live_bytes -= c->big_size[p];
    c->big_size.erase(p);
    {
      // sole context: all device work is ordered on its one stream, so the
      // range can be handed out again at once (stream-ordered reuse);
      // otherwise it is published at this context's next stream sync
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      if (g.n_ctx <= 1 && g.arena.owns(p)) {
        g.arena.release(p);
        return;
      }
    }
    c->big_pending.push_back(p);
    return;
  }
  spq_ctx::PoolEnt* it = c->pool_size.find(pkey(p));
  if (!it) throw std::runtime_error("dfree of unknown pointer");
  const spq_ctx::PoolEnt e = *it;
  c->pool_size.erase(pkey(p));
  c->pool_free[e.cls].push_back({p, e.slab});
  c->slab_live[e.slab]--;
  c->live_bytes -= e.cls;
}

int env_flag(const char* name);
inline bool blocks_untracked() {   // SPQ_ALLOC_TRACK_ALL=1: block memory through the pointer table (A/B runs)
  static const bool v = !env_flag("SPQ_ALLOC_TRACK_ALL");
  return v;
}

// free of untracked block memory (dalloc(..., tracked = false)) by size
void dfree_block(spq_ctx* c, void* p, size_t bytes) {
  if (!p) return;
  if (bytes >= BIG_ALLOC) { dfree(c, p); return; }   // large buffers are tracked in c->big
  if (c->on_side) {   // still used by queued side work: released at side_join
    c->side_free_blk.push_back({p, bytes});
    return;
  }
  const size_t cls = size_class(bytes == 0 ? 8 : bytes);
  int slab = -1;
  for (size_t i = 0; i < c->slabs.size(); ++i)
    if (c->slabs[i] && (char*)p >= (char*)c->slabs[i] && (char*)p < (char*)c->slabs[i] + c->slab_caps[i]) {
      slab = (int)i;
      break;
    }
  if (slab < 0) throw std::runtime_error("dfree_block of unknown pointer");
  c->pool_free[cls].push_back({p, slab});
  c->slab_live[slab]--;
  c->live_bytes -= cls;
}

// stream-ordered release of a block's memory (shared allocations refcounted)
void release_mem(spq_ctx* c, Block& b) {
  if (b.base) {
    int* rc = c->refcnt.find(pkey(b.base));
    if (rc && --*rc == 0) {
      c->deferred.push_back((double*)b.base);
      c->refcnt.erase(pkey(b.base));
    }
  } else if (b.p) {
    if (blocks_untracked()) c->deferred_blk.push_back({b.p, b.abytes});
    else c->deferred.push_back(b.p);
  }
  b.p = nullptr;
  b.base = nullptr;
  b.abytes = 0;
}

double* shared_alloc(spq_ctx* c, size_t elems, int nref) {
  double* base = dalloc(c, std::max<size_t>(elems, 1) * sizeof(double));
  c->refcnt[pkey(base)] = nref;
  return base;
}

void publish_big(spq_ctx* c) {
  if (c->big_pending.empty()) return;
  auto& g = gcache(c->dev);
  std::lock_guard<std::mutex> lk(g.mu);
  for (void* p : c->big_pending) {
    if (g.arena.owns(p)) g.arena.release(p);
    else cudaFree(p);
  }
  c->big_pending.clear();
}

void sync(spq_ctx* c) {
  auto t0 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(c->st));
  publish_big(c);
  c->ring_off = 0;
  c->n_syncs++;
  c->host_ms[1] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// enter/leave the side stream (see spq_ctx::side)
struct SideScope {
  spq_ctx* c;
  cudaStream_t main;
  explicit SideScope(spq_ctx* cc) : c(cc), main(cc->st) {
    if (!c->side) {
      CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_side_a, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_side_b, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(c->ev_side_a, main));
    CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_side_a, 0));
    c->st = c->side;
    c->on_side = true;
  }
  ~SideScope() {
    c->st = main;
    c->on_side = false;
    c->side_pending = true;
  }
};

void dfree(spq_ctx* c, void* p);
// the main stream waits for all side work; its buffers are released in
// stream order after that point
void side_join(spq_ctx* c) {
  if (!c->side_pending) return;
  CUDA_TRY(cudaEventRecord(c->ev_side_b, c->side));
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_side_b, 0));
  c->side_pending = false;
  std::vector<void*> f;
  f.swap(c->side_free);
  for (void* p : f) dfree(c, p);
  std::vector<std::pair<void*, size_t>> fb;
  fb.swap(c->side_free_blk);
  for (auto& e : fb) dfree_block(c, e.first, e.second);
}

template <class T>
T* upload(spq_ctx* c, const T* src, size_t n) {
  const size_t bytes = n * sizeof(T);
  if (bytes == 0) return nullptr;
  size_t aligned = (bytes + 255) & ~(size_t)255;
  if (c->on_side) {   // the ring is recycled at main-stream syncs: side work owns its buffers
    T* d = (T*)dalloc(c, bytes);
    CUDA_TRY(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, c->st));
    c->side_free.push_back(d);
    return d;
  }
  if (aligned > c->ring_cap) {
    // oversize: dedicated allocation, freed stream-ordered after use by caller
    T* d = (T*)dalloc(c, bytes);
    CUDA_TRY(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, c->st));
    c->deferred.push_back((double*)d);
    return d;
  }
  if (c->ring_off + aligned > c->ring_cap) {
    // never wrap mid-sequence: later launches may still reference earlier
    // uploads, so overflow goes to a dedicated stream-ordered buffer
    T* d = (T*)dalloc(c, bytes);
    CUDA_TRY(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, c->st));
    c->deferred.push_back((double*)d);
    c->n_ring_overflow++;
    return d;
  }
  std::memcpy(c->pin + c->ring_off, src, bytes);
  T* d = (T*)(c->dring + c->ring_off);
  CUDA_TRY(cudaMemcpyAsync(d, c->pin + c->ring_off, bytes, cudaMemcpyHostToDevice, c->st));
  c->ring_off += aligned;
  return d;
}
template <class T>
T* upload(spq_ctx* c, const std::vector<T>& v) {
  return upload(c, v.data(), v.size());
}
// nullptr (the launcher carries the list in its parameters) for short
// lists, an uploaded copy otherwise; SPQ_NO_PARAM_LISTS=1 always uploads
int env_flag(const char* name);
template <class T>
const T* up_or_param(spq_ctx* c, const std::vector<T>& v, int pmax) {
  static const bool off = env_flag("SPQ_NO_PARAM_LISTS");
  if (!off && (int)v.size() <= pmax) return nullptr;
  return upload(c, v);
}

void flush_deferred(spq_ctx* c) {
  for (double* p : c->deferred) dfree(c, p);
  c->deferred.clear();
  for (auto& e : c->deferred_blk) dfree_block(c, e.first, e.second);
  c->deferred_blk.clear();
}

// fork-join: independent launches on auxiliary streams that start after
// everything queued so far on the context stream and are joined back
// before anything after them (all buffers they touch stay stream-ordered)
struct Fork {
  spq_ctx* c;
  int used = 0;
  bool single = false;   // one launch only: it goes straight to the context stream
  explicit Fork(spq_ctx* cc, int nlaunch = 2) : c(cc), single(nlaunch <= 1) {
    if (single) return;
    if (!c->ev_fork) {
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      for (int k = 0; k < spq_ctx::NAUX; ++k) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming));
      }
    }
    CUDA_TRY(cudaEventRecord(c->ev_fork, c->st));
  }
  cudaStream_t next() {
    if (single) return c->st;
    const int k = used % spq_ctx::NAUX;
    if (used < spq_ctx::NAUX) CUDA_TRY(cudaStreamWaitEvent(c->aux[k], c->ev_fork, 0));
    ++used;
    return c->aux[k];
  }
  void join() {
    if (single) return;
    for (int k = 0; k < std::min(used, spq_ctx::NAUX); ++k) {
      CUDA_TRY(cudaEventRecord(c->ev_join[k], c->aux[k]));
      CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_join[k], 0));
    }
    used = 0;
  }
};

struct Scope {
  spq_ctx* c;
  int fam;
  cudaEvent_t a, b;
  static cudaEvent_t get(spq_ctx* c) {
    if (!c->ev_pool.empty()) {
      cudaEvent_t e = c->ev_pool.back();
      c->ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    return e;
  }
  Scope(spq_ctx* c_, int f, std::string tag = std::string()) : c(c_), fam(f) {
    if (c->timing) {
      a = get(c);
      CUDA_TRY(cudaEventRecord(a, c->st));
      if (scope_log()) c->tm.tag[fam].push_back(std::move(tag));
    }
  }
  ~Scope() {
    if (c->timing) {
      b = get(c);
      cudaEventRecord(b, c->st);
      c->tm.ev[fam].push_back({a, b});
    }
  }
  // SPQ_SCOPE_LOG=<path>: every timed scope (family, ms, tag) appended at
  // the next timing collection (diagnostic)
  static FILE* scope_log() {
    static FILE* f = [] {
      const char* e = getenv("SPQ_SCOPE_LOG");
      return (e && *e) ? fopen(e, "a") : (FILE*)nullptr;
    }();
    return f;
  }
};

void collect_timings(spq_ctx* c) {
  for (int f = 0; f < F_NFAM; ++f) {
    FILE* lg = Scope::scope_log();
    for (size_t t = 0; t < c->tm.ev[f].size(); ++t) {
      auto& e = c->tm.ev[f][t];
      float ms = 0.f;
      CUDA_TRY(cudaEventSynchronize(e.second));
      CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
      c->tm.ms[f] += ms;
      if (lg) {
        float t0 = -1.f;   // start, relative to mark 0 (the factorization start) when recorded
        if (!c->marks.empty() && cudaEventElapsedTime(&t0, c->marks[0], e.first) != cudaSuccess) {
          (void)cudaGetLastError();
          t0 = -1.f;
        }
        fprintf(lg, "%d %.4f %.4f %s\n", f, ms, t0, t < c->tm.tag[f].size() ? c->tm.tag[f][t].c_str() : "");
      }
      c->ev_pool.push_back(e.first);
      c->ev_pool.push_back(e.second);
    }
    c->tm.ev[f].clear();
    c->tm.tag[f].clear();
  }
}

void ensure_err_slots(spq_ctx* c, int n) {
  if (n <= c->err_slots) return;
  int cap = std::max(n, 2 * c->err_slots + 64);
  int64_t* idx = (int64_t*)dalloc(c, cap * sizeof(int64_t));
  double* val = dalloc(c, cap * sizeof(double));
  if (c->err_slots > 0) {   // results of checks not yet raised survive the growth
    CUDA_TRY(cudaMemcpyAsync(idx, c->d_err_idx, c->err_slots * sizeof(int64_t),
                             cudaMemcpyDeviceToDevice, c->st));
    CUDA_TRY(cudaMemcpyAsync(val, c->d_err_val, c->err_slots * sizeof(double),
                             cudaMemcpyDeviceToDevice, c->st));
  }
  dfree(c, c->d_err_idx);
  dfree(c, c->d_err_val);
  c->d_err_idx = idx;
  c->d_err_val = val;
  c->err_slots = cap;
}

// --------------------------------------------------------- copy batches
// task vectors are recycled through a per-thread pool: a batch of 10^4 tasks
// written into freshly allocated (cache-cold) memory costs ~65 ns per task in
// write-allocate misses (host profile r02: 4 ms per C3 factorization)
inline std::vector<std::vector<CopyTask>>& copy_task_pool() {
  static thread_local std::vector<std::vector<CopyTask>> pool;
  return pool;
}

struct CopyBatch {
  std::vector<CopyTask> t;
  int64_t maxe = 0;
  int64_t tot_e = 0;   // elements of all tasks
  double by = 0;       // bytes moved (read + write)
  void account(const CopyTask& x) {
    const int64_t e = (int64_t)std::max(x.nr, 0) * std::max(x.nc, 0);
    maxe = std::max(maxe, e);
    tot_e += e;
    by += (double)e * ((x.src && !x.ident) ? 16.0 : 8.0);
  }
  CopyBatch() {
    auto& pool = copy_task_pool();
    if (!pool.empty()) { t.swap(pool.back()); pool.pop_back(); }
  }
  ~CopyBatch() {
    auto& pool = copy_task_pool();
    if (t.capacity() > 0 && pool.size() < 8) { t.clear(); pool.emplace_back(); pool.back().swap(t); }
  }
  CopyBatch(const CopyBatch&) = delete;
  CopyBatch& operator=(const CopyBatch&) = delete;
  // callers that know their task count reserve it: growing a 10^4-task vector
  // by doubling was ~4 ms of memmove per C3 factorization (host profile r02)
  void reserve(size_t n) {
    if (t.empty() && t.capacity() < n)   // a recycled vector that is already large enough?
      for (auto& v : copy_task_pool())
        if (v.capacity() >= n) { t.swap(v); break; }
    t.reserve(t.size() + n);
  }
  void add(const CopyTask& x) {
    if (x.nr <= 0 || x.nc <= 0) return;
    t.push_back(x);
    account(x);
  }
  void zero(double* dst, int64_t n) {
    if (n <= 0) return;
    // split very long fills into columns of 1<<20 for the 2D grid
    const int64_t col = 1 << 20;
    CopyTask x{};
    x.dst = dst;
    if (n <= col) {
      x.nr = (int)n; x.nc = 1; x.ldd = (int)n;
      add(x);
    } else {
      const int64_t full = n / col;
      x.nr = (int)col; x.nc = (int)full; x.ldd = (int)col;
      add(x);
      if (n - full * col > 0) zero(dst + full * col, n - full * col);
    }
  }
  void run(spq_ctx* c) {
    if (t.empty()) return;
    std::string tag;
    if (Scope::scope_log()) {
      char b[160];
      snprintf(b, sizeof b, "copy %s nt=%zu maxe=%lld gb=%.4f", c->stage, t.size(), (long long)maxe, by / 1e9);
      tag = b;
    }
    Scope s(c, F_COPY, tag);
    // elements per CTA: 2048 (eight per thread) while that still fills the
    // machine, up to 8192 for the big batches -- a CTA's task lookup and launch
    // cost amortised over more elements (SPQ_COPY_GRAN overrides)
    static const int64_t gran_env = getenv("SPQ_COPY_GRAN") ? atoll(getenv("SPQ_COPY_GRAN")) : 0;
    int64_t gran = 2048;
    while (gran < 8192 && tot_e / (2 * gran) >= (int64_t)c->nsm * 8) gran *= 2;
    if (gran_env > 0) gran = gran_env;
    // flattened-grid assignment (used for mixed task sizes), written in the
    // same pass that stages a long list in the pinned upload ring
    static const bool no_param = env_flag("SPQ_NO_PARAM_LISTS");
    const size_t bytes = t.size() * sizeof(CopyTask), aligned = (bytes + 255) & ~(size_t)255;
    const bool in_param = !no_param && (int)t.size() <= PL_COPY;
    const bool in_ring = !in_param && !c->on_side && aligned <= c->ring_cap &&
                         c->ring_off + aligned <= c->ring_cap;
    CopyTask* stage = in_ring ? reinterpret_cast<CopyTask*>(c->pin + c->ring_off) : nullptr;
    int64_t ctas = 0;
    for (size_t i = 0; i < t.size(); ++i) {
      CopyTask& x = t[i];
      const int64_t nb = std::min<int64_t>(512, std::max<int64_t>(1, ((int64_t)x.nr * x.nc + gran - 1) / gran));
      x.cta0 = (int)ctas;
      x.ncta = (int)nb;
      ctas += nb;
      if (stage) stage[i] = x;
    }
    const CopyTask* d_tasks = nullptr;
    if (in_ring) {
      CopyTask* d = reinterpret_cast<CopyTask*>(c->dring + c->ring_off);
      CUDA_TRY(cudaMemcpyAsync(d, stage, bytes, cudaMemcpyHostToDevice, c->st));
      c->ring_off += aligned;
      d_tasks = d;
    } else if (!in_param) {
      d_tasks = upload(c, t);
    }
    launch_copy(d_tasks, t.data(), (int)t.size(), maxe, ctas, c->st, gran);
    c->tm.launches[F_COPY]++;
    c->n_kernels++;
    c->tm.bytes[F_COPY] += by;
    t.clear();
    maxe = 0;
    tot_e = 0;
    by = 0;
  }
};

// (Host threads were tried for the per-front task construction of the large
// leaf-level waves -- every front fills its own slice -- and measured SLOWER
// on the GPU boxes: 133.9 ms per C3 factorization with 1 thread, 141.5 with 4,
// 154.7 with 8, every host phase slowing down, profiles/r02g/host_threads.txt.
// The loops below therefore run on the calling thread.)
template <class F>
void parallel_fronts(size_t n, size_t, F&& fn) { fn((size_t)0, n); }

// --------------------------------------------------------- gemm batches
// A batch whose output tiles cannot fill the machine splits long-K problems
// (K >= 1024) into partial products reduced in a fixed order.
struct GemmBatch {
  std::vector<GemmProb> p;
  int tiles = 0;
  void add(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int m, int n,
           int k, double alpha, double beta) {
    const int t = gemm_tiles(m, n);
    if (t == 0) return;
    GemmProb g{A, B, C, m, n, k, lda, ldb, ldc, alpha, beta, 0};
    p.push_back(g);
    tiles += t;
  }
  void run(spq_ctx* c, bool transA, double flops) {
    if (p.empty()) return;
    // few output tiles: switch to the 64x64 kernel (4x the CTAs per area)
    int small = 0;
    gemm_set_variant(2);
    for (auto& g : p) small += gemm_tiles(g.m, g.n);
    // few output tiles: the 64 x 64 kernel covers the SMs with 4x the CTAs per
    // area (large tiles + split-K for long-K problems measured no better on C3
    // and worse on the small shapes, profiles/r02i/gemm_longk_rule.txt)
    int variant = small < c->nsm ? 1 : 2;
    if (variant == 2) {
      // 64 x 128 tiles when they pad noticeably less than 128 x 64 (few rows:
      // the k x n products W = V^T C of the 3D fronts, k = 100..600)
      static const bool no_v3 = env_flag("SPQ_GEMM_NO_V3");
      double a2 = 0, a3 = 0;
      for (auto& g : p) {
        a2 += (double)((g.m + 127) / 128) * 128 * ((g.n + 63) / 64) * 64 * g.k;
        a3 += (double)((g.m + 63) / 64) * 64 * ((g.n + 127) / 128) * 128 * g.k;
      }
      if (!no_v3 && a3 < 0.93 * a2) variant = 3;
    }
    gemm_set_variant(variant);
    tiles = 0;
    for (auto& g : p) tiles += gemm_tiles(g.m, g.n);
    const int target = 2 * c->nsm;
    std::vector<GemmProb> q;
    std::vector<SplitRed> red;
    int64_t red_max = 0;
    size_t part_tot = 0;
    std::vector<int> splits(p.size(), 1);
    if (tiles < target) {
      for (size_t i = 0; i < p.size(); ++i) {
        const GemmProb& g = p[i];
        if (g.k < 512) continue;
        int sp = std::min((g.k + 255) / 256, std::max(1, target / std::max(tiles, 1)));
        splits[i] = std::max(1, sp);
        if (splits[i] > 1) part_tot += (size_t)splits[i] * g.m * g.n;
      }
    }
    double* part = part_tot ? dalloc(c, part_tot * sizeof(double)) : nullptr;
    size_t poff = 0;
    int t0 = 0;
    for (size_t i = 0; i < p.size(); ++i) {
      GemmProb g = p[i];
      const int nt = gemm_tiles(g.m, g.n);
      if (splits[i] == 1) {
        g.tile0 = t0;
        t0 += nt;
        q.push_back(g);
        continue;
      }
      const int S = splits[i];
      const int kc = (g.k + S - 1) / S;
      double* P = part + poff;
      for (int sidx = 0; sidx < S; ++sidx) {
        const int k0 = sidx * kc;
        const int kk = std::min(kc, g.k - k0);
        GemmProb h = g;
        h.A = transA ? g.A + k0 : g.A + (int64_t)k0 * g.lda;
        h.B = g.B + k0;
        h.C = P + (size_t)sidx * g.m * g.n;
        h.ldc = g.m;
        h.k = std::max(kk, 0);
        h.alpha = 1.0;
        h.beta = 0.0;
        h.tile0 = t0;
        t0 += nt;
        q.push_back(h);
      }
      red.push_back(SplitRed{P, g.C, g.m, g.n, g.ldc, S, g.alpha, g.beta});
      red_max = std::max<int64_t>(red_max, (int64_t)g.m * g.n);
      poff += (size_t)S * g.m * g.n;
    }
    {
      std::string tag;
      if (Scope::scope_log()) {
        int mm = 0, nn = 0, kk = 0;
        double fl = 0;
        for (auto& g : p) {
          mm = std::max(mm, g.m); nn = std::max(nn, g.n); kk = std::max(kk, g.k);
          fl += 2.0 * g.m * g.n * (double)g.k;
        }
        char b[200];
        snprintf(b, sizeof b, "gemm %s np=%zu tiles=%d split=%zu tA=%d max_mnk=%d,%d,%d gflop=%.4f",
                 c->stage, p.size(), t0, red.size(), (int)transA, mm, nn, kk, fl / 1e9);
        tag = b;
      }
      Scope s(c, F_WY, tag);
      launch_gemm(up_or_param(c, q, PL_GEMM), q.data(), (int)q.size(), t0, transA, c->st);
      if (!red.empty())
        launch_splitk_reduce(up_or_param(c, red, PL_RED), red.data(), (int)red.size(), red_max, c->st);
    }
    c->tm.launches[F_WY] += 1 + (red.empty() ? 0 : 1);
    c->n_kernels += 1 + (red.empty() ? 0 : 1);
    gemm_set_variant(0);
    c->tm.flops[F_WY] += flops;
    if (part) dfree(c, part);
    p.clear();
    tiles = 0;
  }
};

// ----------------------------------------------------------- QR engine
// Blocked Householder QR of a batch of panels (nb = 32 columns per block).
// After each block's panel kernel, its compact WY (V_b, T_b) is applied to
// the rest of the panel AND to every extra target C (rows j0..m-1):
//   W = V_b^T X,  W = T_b^T W,  X -= V_b W      (batched DMMA GEMMs)
// so the factorization never needs the full k x k T; records get it in one
// batched build at spq_finish (build_full_T).
struct CTarget {
  double* C;
  int ldc, n;
};

struct QrProb {
  double* P;  // m x k, ld m -> V on exit
  int m, k;
  double* R;  // k x k
  double* tau;
  double* T;  // k x k (diagonal 32-blocks written)
  std::vector<CTarget> targets;
  bool want_T = false;   // full T even without targets (targets applied later, in chunks)
};

// full k x k T for a batch of (V, tau, T) triples: G = V^T V, blocked larft
struct TProb {
  const double* V;
  int m, k;
  const double* tau;
  double* T;
};

int env_flag(const char* name);

void build_full_T(spq_ctx* c, const std::vector<TProb>& tp) {
  Stage stage_(c, "build_full_T");
  // G = V^T V (batched DMMA), the 32x32 diagonal blocks of T by the row
  // recurrence (one CTA per job), then recursive doubling over block pairs
  // A=[x, x+s), B=[x+s, x+2s):  T_AB = -T_AA (G_AB T_BB)   (batched GEMMs)
  size_t gsz = 0;
  int maxk = 0;
  for (auto& t : tp) {
    gsz += 2 * (size_t)t.k * t.k;
    maxk = std::max(maxk, t.k);
  }
  if (gsz == 0) return;
  double* scr = dalloc(c, gsz * sizeof(double));
  GemmBatch gg;
  std::vector<LarftJob> lj;
  std::vector<double*> Gp(tp.size()), Yp(tp.size());
  size_t off = 0;
  for (size_t i = 0; i < tp.size(); ++i) {
    const auto& t = tp[i];
    if (t.k <= 0) continue;
    Gp[i] = scr + off;
    Yp[i] = Gp[i] + (size_t)t.k * t.k;
    off += 2 * (size_t)t.k * t.k;
    gg.add(t.V, t.m, t.V, t.m, Gp[i], t.k, t.k, t.k, t.m, 1.0, 0.0);
    lj.push_back(LarftJob{Gp[i], t.tau, t.T, nullptr, t.k, t.k, t.k, 0});
  }
  gg.run(c, true, 0);
  if (maxk <= larft_full_max() && !env_flag("SPQ_LARFT_DOUBLING")) {   // whole T in one launch
    Scope s(c, F_QR);
    launch_larft_full(up_or_param(c, lj, PL_SMALL), lj.data(), (int)lj.size(), maxk, c->st);
    c->tm.launches[F_QR]++;
    c->n_kernels++;
    dfree(c, scr);
    return;
  }
  {
    Scope s(c, F_QR);
    launch_larft(upload(c, lj), (int)lj.size(), 0, c->st);
    c->tm.launches[F_QR]++;
    c->n_kernels++;
  }
  for (int sz = 32; sz < maxk; sz *= 2) {
    GemmBatch g1, g2;
    for (size_t i = 0; i < tp.size(); ++i) {
      const auto& t = tp[i];
      for (int x = 0; x + sz < t.k; x += 2 * sz) {
        const int na = sz, nb = std::min(sz, t.k - x - sz);
        const int xa = x, xb = x + sz;
        double* Y = Yp[i] + (size_t)xa;                        // na x nb, ld k
        // Y = G[A, B] T[B, B]
        g1.add(Gp[i] + xa + (int64_t)xb * t.k, t.k, t.T + xb + (int64_t)xb * t.k, t.k,
               Y + (int64_t)xb * t.k, t.k, na, nb, nb, 1.0, 0.0);
        // T[A, B] = -T[A, A] Y
        g2.add(t.T + xa + (int64_t)xa * t.k, t.k, Y + (int64_t)xb * t.k, t.k,
               t.T + xa + (int64_t)xb * t.k, t.k, na, nb, na, -1.0, 0.0);
      }
    }
    g1.run(c, false, 0);
    g2.run(c, false, 0);
  }
  dfree(c, scr);
}

// C <- C - V T^T V^T C (transpose) or C - V T V^T C
struct WyProb {
  const double* V;
  const double* T;
  int m, k;
  double* C;
  int ldc, n;
};

// fused shallow-WY kernel on (SPQ_NO_WYF=1: the three-GEMM path, A/B tests)
bool use_wyf() {
  static const bool v = !env_flag("SPQ_NO_WYF");
  return v;
}

std::string wyf_tag(spq_ctx* c, const std::vector<WyfJob>& wj, int tiles, int cl) {
  if (!Scope::scope_log()) return std::string();
  int mm = 0, nn = 0, kk = 0;
  double fl = 0;
  for (auto& w : wj) {
    mm = std::max(mm, w.m); nn = std::max(nn, w.n); kk = std::max(kk, w.k);
    fl += 4.0 * w.m * (double)w.n * w.k;
  }
  char b[200];
  snprintf(b, sizeof b, "wyf %s np=%zu tiles=%d cl=%d max_mnk=%d,%d,%d gflop=%.4f", c->stage,
           wj.size(), tiles, cl, mm, nn, kk, fl / 1e9);
  return b;
}

size_t chunk_bytes() {   // SPQ_CHUNK_BYTES overrides (tests force the chunked path)
  static size_t v = 0;
  if (!v) {
    const char* e = getenv("SPQ_CHUNK_BYTES");
    v = e ? std::max<size_t>(4096, strtoull(e, nullptr, 10)) : ((size_t)2 << 30);
  }
  return v;
}

// The (W, W2) scratch of a batch is bounded by chunk_bytes(): problems are
// split by columns (the update is column-independent) and the batch runs in
// consecutive groups that reuse one scratch buffer (stream order).  A level
// of interface scalings otherwise needs 2 k n doubles for ALL its targets
// at once (~100 GB at 64^3).
// join_side: the T factors of this batch are still being built on the side
// stream (build_full_T under a SideScope).  Only T^T W needs them, so the
// first product W = V^T C -- the long one -- runs beside G = V^T V and the
// larft recurrence; the main stream joins the side stream just before the
// first kernel that reads T.
void wy_batch(spq_ctx* c, const std::vector<WyProb>& probs_in, bool transpose, int fam = F_WY,
              bool join_side = false) {
  Stage stage_(c, "wy_batch");
  (void)fam;
  struct Joiner {   // whatever path returns, the side stream is joined
    spq_ctx* c;
    bool* pending;
    ~Joiner() { if (*pending) side_join(c); }
  } joiner_{c, &join_side};
  const size_t budget = std::max<size_t>(chunk_bytes() / sizeof(double), 2);
  std::vector<WyProb> probs;
  size_t tot = 0;
  for (auto& p : probs_in) {
    if (p.k <= 0 || p.n <= 0 || p.m <= 0) continue;
    const int64_t maxn = (int64_t)std::max<size_t>(1, budget / (2 * (size_t)p.k));
    for (int64_t j0 = 0; j0 < p.n; j0 += maxn) {
      WyProb q = p;
      q.C = p.C + j0 * (int64_t)p.ldc;
      q.n = (int)std::min<int64_t>(maxn, p.n - j0);
      probs.push_back(q);
      tot += 2 * (size_t)q.k * q.n;
    }
  }
  if (tot == 0) return;
  for (auto& p : probs)   // algorithmic bytes of the WY apply: 8(2mn + mk + k^2)
    c->tm.bytes[F_WY] += 8.0 * (2.0 * p.m * (double)p.n + (double)p.m * p.k + (double)p.k * p.k);
  {
    // shallow reflector blocks (every k <= 64) with little total work: one
    // fused launch (k_wyf.cu) instead of three GEMM launches + split-K
    // (big batches -- the leaf levels' thousands of fronts -- stay on the
    // GEMM engine, which runs several CTAs per SM)
    bool shallow = use_wyf();
    double fl = 0;
    int64_t ctas = 0;
    int clm = 1;
    for (auto& p : probs) {
      shallow = shallow && p.k <= wyf_kmax();
      fl += 4.0 * p.m * (double)p.n * p.k;
      ctas += (p.n + 31) / 32;
      clm = std::max(clm, wyf_cluster(p.m));
    }
    if (shallow && fl <= 8e9 && ctas * clm <= 4 * c->nsm) {
      std::vector<WyfJob> wj;
      int tiles = 0, cl = 1, kmax = 1;
      for (auto& p : probs) {
        WyfJob w{};
        w.V = p.V; w.ldv = p.m; w.T = p.T; w.ldt = p.k; w.C = p.C; w.ldc = p.ldc;
        w.m = p.m; w.n = p.n; w.k = p.k; w.trans = transpose ? 1 : 0; w.tile0 = tiles;
        tiles += (p.n + 31) / 32;
        cl = std::max(cl, wyf_cluster(p.m));
        kmax = std::max(kmax, p.k);
        c->tm.flops[F_WY] += 4.0 * p.m * (double)p.n * p.k - (double)p.n * p.k * p.k;
        wj.push_back(w);
      }
      if (join_side) { side_join(c); join_side = false; }
      Scope s(c, F_WY, wyf_tag(c, wj, tiles, cl));
      launch_wyf(up_or_param(c, wj, PL_WYF), wj.data(), (int)wj.size(), tiles, kmax, cl, c->st);
      c->tm.launches[F_WY]++;
      c->n_kernels++;
      return;
    }
  }
  size_t need1 = 0;   // the largest single (split) problem
  for (auto& p : probs) need1 = std::max(need1, 2 * (size_t)p.k * p.n);
  size_t got = 0;
  double* scr = dalloc_flex(c, std::min(tot, std::max(budget, need1)) * sizeof(double),
                            need1 * sizeof(double), &got);
  const size_t cap = got / sizeof(double);
  size_t i = 0;
  while (i < probs.size()) {
    GemmBatch g1, g2, g3;
    size_t off = 0;
    double flops = 0;
    for (; i < probs.size(); ++i) {
      const WyProb& p = probs[i];
      const size_t need = 2 * (size_t)p.k * p.n;
      if (off > 0 && off + need > cap) break;
      double* W = scr + off;
      double* W2 = W + (size_t)p.k * p.n;
      off += need;
      flops += 4.0 * p.m * (double)p.n * p.k - (double)p.n * p.k * p.k;
      g1.add(p.V, p.m, p.C, p.ldc, W, p.k, p.k, p.n, p.m, 1.0, 0.0);
      g2.add(p.T, p.k, W, p.k, W2, p.k, p.k, p.n, p.k, 1.0, 0.0);
      g3.add(p.V, p.m, W2, p.k, p.C, p.ldc, p.m, p.n, p.k, -1.0, 1.0);
    }
    g1.run(c, true, flops);
    if (join_side) { side_join(c); join_side = false; }
    g2.run(c, transpose, 0);
    g3.run(c, false, 0);
  }
  dfree(c, scr);
}

constexpr int NB = 32;

// debug/test switch: SPQ_PANEL_GLOBAL=1 forces the L2-resident panel path
int env_flag(const char* name) {
  const char* e = getenv(name);
  return (e && e[0] == '1') ? 1 : 0;
}

bool force_global_panel() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPQ_PANEL_GLOBAL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
constexpr size_t SLAB_BYTES = 200 * 1024;
bool legacy_panel() {
  static const bool v = env_flag("SPQ_PANEL_LEGACY") || force_global_panel();
  return v;
}
int panel_rows() {   // target rows per CTA of the register panel kernel
  static const int v = [] {
    const char* e = getenv("SPQ_PANEL_ROWS");
    const int r = e ? atoi(e) : 256;
    return std::max(32, std::min(512, r));
  }();
  return v;
}

void qr_batch(spq_ctx* c, const std::vector<QrProb>& probs) {
  Stage stage_(c, "qr_batch");
  if (probs.empty()) return;
  double qr_flops = 0;
  int maxk = 0;
  for (auto& q : probs) {
    qr_flops += 2.0 * q.m * (double)q.k * q.k - 2.0 * q.k * (double)q.k * q.k / 3.0;
    c->tm.bytes[F_QR] += 8.0 * (2.0 * q.m * (double)q.k + (double)q.k * q.k);
    maxk = std::max(maxk, q.k);
  }
  c->tm.flops[F_QR] += qr_flops;
  for (int j0 = 0; j0 < maxk; j0 += NB) {
    std::map<std::pair<int, int>, std::pair<std::vector<PanelJob>, int64_t>> groups;
    std::map<std::tuple<int, int, int>, std::vector<PanelJob>> rgroups;   // (cl, R, kbmax)
    size_t wtot = 0;
    // the register kernel (1 CTA/SM, 255 registers) minimises the latency of
    // few large panels; many small panels run at higher occupancy in the
    // shared-memory kernel (throughput: BASELINE config 2's 4096 blocks)
    int njobs = 0;
    for (auto& q : probs) njobs += j0 < q.k;
    const bool many = njobs > 2 * c->nsm;
    for (auto& q : probs) {
      if (j0 >= q.k) continue;
      const int kb = std::min(NB, q.k - j0);
      const int mh = q.m - j0;
      if (!legacy_panel() && !many && mh <= 16 * 2 * 256) {
        // register-resident block: ~panel_rows() rows per CTA, R rows per thread
        int cl = std::max(1, std::min(16, (mh + panel_rows() - 1) / panel_rows()));
        int rpc = (mh + cl - 1) / cl;
        while (cl > 1 && rpc < 32) { --cl; rpc = (mh + cl - 1) / cl; }
        const int R = rpc <= 256 ? 1 : 2;
        rgroups[{cl, R, panel_reg_kbmax(kb)}].push_back(PanelJob{q.P, q.R, q.tau, q.T, q.m, q.k, j0, kb, 1});
        const int j1 = j0 + kb;
        if (j1 < q.k) wtot += 2 * (size_t)kb * (q.k - j1);
        continue;
      }
      int cl = (int)(((size_t)mh * kb * 8 + SLAB_BYTES - 1) / SLAB_BYTES);
      cl = std::max(1, cl);
      int smem = 1;
      if (cl > 16 || force_global_panel()) { cl = std::min(cl, 16); smem = 0; }
      while (cl > 1 && (mh + cl - 1) / cl < 64) --cl;
      const int rpc = (mh + cl - 1) / cl;
      auto& grp = groups[{cl, smem}];
      grp.first.push_back(PanelJob{q.P, q.R, q.tau, q.T, q.m, q.k, j0, kb, 1});
      grp.second = std::max<int64_t>(grp.second, (int64_t)(rpc | 1) * kb);
      const int j1 = j0 + kb;
      if (j1 < q.k) wtot += 2 * (size_t)kb * (q.k - j1);
    }
    {
      Scope s(c, F_QR);
      for (auto& kv : groups) {
        launch_panel_qr(upload(c, kv.second.first), (int)kv.second.first.size(), kv.first.first,
                        kv.second.second, kv.first.second != 0, NB, c->st);
        c->tm.launches[F_QR]++;
        c->n_kernels++;
      }
      for (auto& kv : rgroups) {
        launch_panel_qr_reg(up_or_param(c, kv.second, PL_SMALL), kv.second.data(),
                            (int)kv.second.size(), std::get<0>(kv.first),
                            std::get<1>(kv.first), std::get<2>(kv.first), c->st);
        c->tm.launches[F_QR]++;
        c->n_kernels++;
      }
    }
    if (wtot == 0) continue;
    if (use_wyf()) {   // the block's compact WY on the trailing panel columns: one fused launch
      std::vector<WyfJob> wj;
      int tiles = 0, cl = 1;
      for (auto& q : probs) {
        if (j0 >= q.k) continue;
        const int kb = std::min(NB, q.k - j0);
        const int j1 = j0 + kb;
        if (j1 >= q.k) continue;
        WyfJob w{};
        w.V = q.P + j0 + (int64_t)j0 * q.m; w.ldv = q.m;
        w.T = q.T + j0 + (int64_t)j0 * q.k; w.ldt = q.k;
        w.C = q.P + j0 + (int64_t)j1 * q.m; w.ldc = q.m;
        w.m = q.m - j0; w.n = q.k - j1; w.k = kb; w.trans = 1; w.tile0 = tiles;
        tiles += (w.n + 31) / 32;
        cl = std::max(cl, wyf_cluster(w.m));
        c->tm.flops[F_WY] += 4.0 * w.m * (double)w.n * w.k - (double)w.n * w.k * w.k;
        c->tm.bytes[F_WY] += 8.0 * (2.0 * w.m * (double)w.n + (double)w.m * w.k + (double)w.k * w.k);
        wj.push_back(w);
      }
      Scope s(c, F_WY, wyf_tag(c, wj, tiles, cl));
      launch_wyf(up_or_param(c, wj, PL_WYF), wj.data(), (int)wj.size(), tiles, NB, cl, c->st);
      c->tm.launches[F_WY]++;
      c->n_kernels++;
      continue;
    }
    double* Ws = dalloc(c, wtot * sizeof(double));
    size_t off = 0;
    GemmBatch g1, g2, g3;
    for (auto& q : probs) {
      if (j0 >= q.k) continue;
      const int kb = std::min(NB, q.k - j0);
      const int mh = q.m - j0;
      const int j1 = j0 + kb;
      double* Vb = q.P + j0 + (int64_t)j0 * q.m;
      const double* Tb = q.T + j0 + (int64_t)j0 * q.k;
      auto add = [&](double* X, int ldx, int nx) {
        if (nx <= 0 || mh <= 0) return;
        double* W = Ws + off;
        double* W2 = W + (size_t)kb * nx;
        off += 2 * (size_t)kb * nx;
        g1.add(Vb, q.m, X, ldx, W, kb, kb, nx, mh, 1.0, 0.0);
        g2.add(Tb, q.k, W, kb, W2, kb, kb, nx, kb, 1.0, 0.0);
        g3.add(Vb, q.m, W2, kb, X, ldx, mh, nx, kb, -1.0, 1.0);
      };
      if (j1 < q.k) add(q.P + j0 + (int64_t)j1 * q.m, q.m, q.k - j1);
    }
    g1.run(c, true, 0);
    g2.run(c, true, 0);
    g3.run(c, false, 0);
    dfree(c, Ws);
  }
  // targets: one pass with the full compact WY (k-deep GEMMs, C read once)
  std::vector<TProb> tp;
  std::vector<WyProb> wp;
  for (auto& q : probs) {
    if (q.k <= 0 || (q.targets.empty() && !q.want_T)) continue;
    tp.push_back(TProb{q.P, q.m, q.k, q.tau, q.T});
    for (auto& t : q.targets) wp.push_back(WyProb{q.P, q.T, q.m, q.k, t.C, t.ldc, t.n});
  }
  if (!tp.empty()) {
    static const bool overlap_T = !env_flag("SPQ_NO_T_OVERLAP");
    const bool ov = overlap_T && !wp.empty() && !c->on_side && !c->side_pending;
    if (ov) {
      SideScope side_(c);
      build_full_T(c, tp);
    } else {
      build_full_T(c, tp);
    }
    wy_batch(c, wp, true, F_WY, ov);
  }
}

// pivot checks for a batch; returns the first failing job (in order) or -1
// checks the jobs added since the last launch; results accumulate in the
// error slots until pivot_raise reads them (one read per set, in order)
void pivot_launch(spq_ctx* c, PivotSet& ps) {
  if (ps.jobs.size() <= ps.launched) return;
  ensure_err_slots(c, (int)ps.jobs.size());
  for (size_t i = ps.launched; i < ps.jobs.size(); ++i) ps.jobs[i].slot = (int)i;
  const int n = (int)(ps.jobs.size() - ps.launched);
  launch_pivot_check(upload(c, ps.jobs.data() + ps.launched, n), n, c->d_err_idx, c->d_err_val,
                     c->st);
  ps.launched = ps.jobs.size();
  c->n_kernels++;
}

// after a stream sync: raise SPQ_ERR_SPECULATION if the device found a
// predicted row flag wrong (speculative mode only)
void spec_raise(spq_ctx* c) {
  if (c->spec && c->h_spec_bad && *c->h_spec_bad)
    throw SpqError(SPQ_ERR_SPECULATION, std::to_string(*c->h_spec_bad) +
                   " predicted row flags differed from the device values; "
                   "re-run with speculation off");
}

void pivot_raise(spq_ctx* c, PivotSet& ps) {
  if (ps.jobs.empty()) return;
  HostTimer ht(&c->host_ms[12]);
  const int n = (int)ps.jobs.size();
  std::vector<int64_t> idx(n);
  std::vector<double> val(n);
  CUDA_TRY(cudaMemcpyAsync(idx.data(), c->d_err_idx, n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           c->st));
  CUDA_TRY(cudaMemcpyAsync(val.data(), c->d_err_val, n * sizeof(double), cudaMemcpyDeviceToHost,
                           c->st));
  sync(c);
  // a pivot failure that follows a wrong row-flag prediction is an artefact
  // of the speculation: report that first, so the host retries exactly
  spec_raise(c);
  for (int i = 0; i < n; ++i)
    if (idx[i] >= 0) throw SpqError(SPQ_ERR_SINGULAR, ps.ctx[i], idx[i], val[i]);
  ps.jobs.clear();
  ps.ctx.clear();
  ps.launched = 0;
}

// ----------------------------------------------------- block bookkeeping
inline Block* find_block(spq_ctx* c, int i, int j) { return c->rix[i].find(j); }

Block& put_block(spq_ctx* c, int i, int j, double* p, int nr, int nc, void* base = nullptr) {
  Block* have = c->rix[i].find(j);
  Block& b = have ? *have : c->blk.create();
  b.p = p;
  b.base = base;
  b.abytes = base ? 0 : (size_t)std::max(1, nr) * std::max(1, nc) * sizeof(double);   // = new_block_mem(nr, nc)
  b.nr = nr;
  b.nc = nc;
  c->rix[i].insert(j, &b);
  c->cix[j].insert(i, &b);
  return b;
}

// same for a key the caller knows to be absent (no lookup)
Block& put_block_new(spq_ctx* c, int i, int j, double* p, int nr, int nc, void* base = nullptr) {
  Block& b = c->blk.create();
  b.p = p;
  b.base = base;
  b.abytes = base ? 0 : (size_t)std::max(1, nr) * std::max(1, nc) * sizeof(double);
  b.nr = nr;
  b.nc = nc;
  c->rix[i].insert(j, &b);
  c->cix[j].insert(i, &b);
  return b;
}

void drop_block(spq_ctx* c, int i, int j) {
  if (Block* b = c->rix[i].find(j)) {
    release_mem(c, *b);
    c->blk.destroy(b);
  }
  c->rix[i].erase(j);
  c->cix[j].erase(i);
}

// every live block with its key, rows ascending, columns ascending within a row
template <class F>
void for_each_block(spq_ctx* c, F&& f) {
  for (int i = 0; i < c->ncl; ++i) {
    const FlatSet& row = c->rix[i];
    for (size_t t = 0; t < row.v.size(); ++t)
      if (row.b[t]) f(bkey(i, row.v[t]), *row.b[t]);
  }
}

void retire(spq_ctx* c, int s) {
  c->active[s] = 0;
  c->rows_of[s].clear();
  c->cols_of[s].clear();
  c->rix[s].clear();
  c->cix[s].clear();
}

double* new_block_mem(spq_ctx* c, int nr, int nc) {
  return dalloc(c, (size_t)std::max(1, nr) * std::max(1, nc) * sizeof(double), /*tracked=*/!blocks_untracked());
}

// refresh row flags of every non-clean block in the given row clusters.
// Speculative mode: blocks whose flags were PREDICTED (clean, unverified)
// are checked on the device in stream order -- the check sees exactly the
// values the prediction describes -- without a host round trip; only
// blocks with unknown flags still need the synchronous exact refresh.
void refresh_flags(spq_ctx* c, const std::vector<int>& row_clusters) {
  Stage stage_(c, "refresh_flags");
  HostTimer ht(&c->host_ms[4]);
  std::vector<const double*> ptrs, vptrs;
  std::vector<int> nr, nc, vnr, vnc;
  std::vector<int64_t> off, voff;
  std::vector<unsigned char> vpred;
  std::vector<Block*> which;
  int64_t tot = 0;
  for (int r : row_clusters) {
    const FlatSet& row = c->rix[r];
    for (size_t t = 0; t < row.v.size(); ++t) {
      Block* b = row.b[t] ? row.b[t] : find_block(c, r, row.v[t]);
      if (!b) continue;
      if (b->clean) {
        if (b->unverified) {
          b->unverified = false;
          if ((int64_t)b->nr * b->nc == 0) continue;
          vptrs.push_back(b->p);
          vnr.push_back(b->nr);
          vnc.push_back(b->nc);
          voff.push_back((int64_t)vpred.size());
          vpred.insert(vpred.end(), b->flags.begin(), b->flags.end());
        }
        continue;
      }
      b->unverified = false;
      if (b->nr == 0) { b->flags.clear(); b->clean = true; continue; }
      if (b->nc == 0) { b->flags.assign(b->nr, 0); b->clean = true; continue; }
      ptrs.push_back(b->p);
      nr.push_back(b->nr);
      nc.push_back(b->nc);
      off.push_back(tot);
      which.push_back(b);
      tot += b->nr;
    }
  }
  static const bool spec_debug = env_flag("SPQ_SPEC_DEBUG");
  if (spec_debug && !vptrs.empty()) {   // exact read-back of every prediction, report mismatches
    std::vector<int64_t> noff(vptrs.size());
    for (size_t t = 0; t < vptrs.size(); ++t) noff[t] = voff[t];
    unsigned char* d_o = (unsigned char*)dalloc(c, vpred.size());
    launch_rowflags(upload(c, vptrs), upload(c, vnr), upload(c, vnc), upload(c, noff), d_o,
                    (int)vptrs.size(), c->st);
    std::vector<unsigned char> hh(vpred.size());
    CUDA_TRY(cudaMemcpyAsync(hh.data(), d_o, hh.size(), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    dfree(c, d_o);
    for (size_t t = 0; t < vptrs.size(); ++t) {
      int bad = 0, first = -1;
      for (int i = 0; i < vnr[t]; ++i)
        if (hh[voff[t] + i] != vpred[voff[t] + i]) { ++bad; if (first < 0) first = i; }
      if (bad) {
        Block* hit = nullptr;
        int hr = -1, hc = -1;
        for_each_block(c, [&](uint64_t key, Block& bb) {
          if (bb.p == vptrs[t]) { hit = &bb; hr = (int)(key >> 32); hc = (int)(key & 0xffffffffu); }
        });
        fprintf(stderr, "[spec] block (%d,%d) %dx%d origin %d: %d rows differ, first %d pred %d actual %d\n",
                hr, hc, vnr[t], vnc[t], hit ? hit->origin : -1, bad, first,
                (int)vpred[voff[t] + first], (int)hh[voff[t] + first]);
      }
    }
  }
  if (!vptrs.empty()) {
    static const bool sabotage = env_flag("SPQ_SPEC_TEST_FAIL");   // tests: force the retry path
    if (sabotage) vpred[0] ^= 1;
    Scope s(c, F_FLAGS);
    launch_rowflags_verify(upload(c, vptrs), upload(c, vnr), upload(c, vnc), upload(c, voff),
                           upload(c, vpred), (int)vptrs.size(), c->d_spec_bad, c->st);
    c->tm.launches[F_FLAGS]++;
    c->n_kernels++;
    c->n_verified += (int64_t)vptrs.size();
  }
  if (which.empty()) return;
  unsigned char* d_out = (unsigned char*)dalloc(c, tot);
  {
    Scope s(c, F_FLAGS);
    launch_rowflags(upload(c, ptrs), upload(c, nr), upload(c, nc), upload(c, off), d_out,
                    (int)which.size(), c->st);
    c->tm.launches[F_FLAGS]++;
    c->n_kernels++;
  }
  std::vector<unsigned char> h(tot);
  {
    HostTimer hw(&c->host_ms[5]);
    CUDA_TRY(cudaMemcpyAsync(h.data(), d_out, tot, cudaMemcpyDeviceToHost, c->st));
    dfree(c, d_out);
    sync(c);
  }
  for (size_t t = 0; t < which.size(); ++t) {
    Block* b = which[t];
    b->flags.assign(h.begin() + off[t], h.begin() + off[t] + b->nr);
    b->clean = true;
  }
}

// speculative-mode prediction helpers
inline bool any_nonzero(const Block& b) {
  for (uint8_t f : b.flags) if (f == 1) return true;
  return false;
}
// every row becomes a combination of all rows (left orthogonal transform)
void predict_mixed_rows(spq_ctx* c, Block& b, bool nonzero, int new_nr) {
  if (!c->spec) { b.clean = false; b.flags.clear(); return; }
  b.flags.assign(new_nr, nonzero ? 1 : 0);
  b.clean = true;
  b.unverified = true;
}
// rows keep their zero/nonzero pattern (right transform by a nonsingular factor)
void predict_same_rows(spq_ctx* c, Block& b) {
  if (!c->spec || !b.clean) { b.clean = false; return; }
  b.unverified = true;
}
// exact identity
void set_identity_flags(spq_ctx* c, Block& b, int n) {
  if (!c->spec) { b.clean = false; b.flags.clear(); return; }
  b.flags.assign(n, 1);
  b.clean = true;
  b.unverified = false;
}

int* upload_idx32(spq_ctx* c, const std::vector<int64_t>& v) {
  std::vector<int> t(v.begin(), v.end());
  return upload(c, t);
}

// ================================================================ (a) factor
struct Part {
  int r;
  std::vector<int> ix;  // local rows (empty => all rows when full)
  bool full;
  int o0, o1;
};

struct Front {
  int s = -1;
  int m = 0, k = 0, n = 0;
  std::vector<Part> parts;
  std::vector<int> cols_t;
  std::vector<int> woff;
  std::vector<int64_t> stack_rows;
  // captured gather sources (pre-update pointers)
  struct Src { const double* p; int nr; int part; int col_off; int ncols; bool full; };
  std::vector<Src> gsrc;       // C gather
  std::vector<Src> psrc;       // panel gather
  // scatter destinations (post-update pointers)
  struct Dst { double* p; int nr; int part; int col_off; int ncols; bool full; };
  std::vector<Dst> dsts;
  std::vector<const int*> d_ix;  // per part: device local-row list (nullptr = all rows)
  int rec = -1;
};

// plan front s from the current structure; returns false if a queried row
// is not known yet (written earlier in this wave)
bool plan_front(spq_ctx* c, int s, Front& f) {
  f = Front();
  f.s = s;
  const auto& rows_s = c->rows_of[s];
  const auto& cols_s = c->cols_of[s];
  f.k = (int)cols_s.size();
  Part p0;
  p0.r = s;
  p0.full = true;
  p0.o0 = 0;
  p0.o1 = (int)rows_s.size();
  f.parts.push_back(p0);
  const FlatSet& col_s = c->cix[s];   // (plan_front does not change the structure)
  int off = p0.o1;
  for (size_t q = 0; q < col_s.v.size(); ++q) {
    const int r = col_s.v[q];
    if (r == s) continue;
    Block* b = col_s.b[q];
    if (!b) continue;
    Part p;
    p.r = r;
    if (b->nr > 0) {
      if (!b->clean && b->flags.empty()) return false;   // unknown flags
      const uint8_t* fl = b->flags.begin();
      p.ix.reserve(b->nr);
      for (int i = 0; i < b->nr; ++i) {
        if (fl[i] == 2) return false;
        if (fl[i] == 1) p.ix.push_back(i);
      }
    }
    if (p.ix.empty()) continue;
    p.full = (int)p.ix.size() == b->nr;
    p.o0 = off;
    off += (int)p.ix.size();
    p.o1 = off;
    f.parts.push_back(std::move(p));
  }
  f.m = off;
  // candidate trailing columns (sorted, unique)
  static thread_local std::vector<int> cand;
  cand.clear();
  {
    static thread_local std::vector<int> mark;   // epoch stamps per cluster
    static thread_local int epoch = 0;
    if ((int)mark.size() < c->ncl) mark.assign(c->ncl, 0), epoch = 0;
    if (++epoch == 0x7fffffff) { std::fill(mark.begin(), mark.end(), 0); epoch = 1; }
    for (auto& p : f.parts)
      for (int cc : c->rix[p.r])
        if (cc != s && mark[cc] != epoch) { mark[cc] = epoch; cand.push_back(cc); }
    std::sort(cand.begin(), cand.end());
  }
  // presence of each candidate (factor.py:454): parts in order until a
  // nonzero row is found.  Walked part-major over each part's row list
  // (block pointers at hand, no lookups); for every candidate the parts and
  // rows examined -- hence the unknown-flag bail-out -- are exactly those of
  // the candidate-major loop.
  static thread_local std::vector<char> present;
  present.assign(cand.size(), 0);
  for (auto& p : f.parts) {
    const FlatSet& row = c->rix[p.r];
    size_t q = 0;
    for (size_t t = 0; t < row.v.size(); ++t) {
      const int cc = row.v[t];
      if (cc == s) continue;
      while (q < cand.size() && cand[q] < cc) ++q;
      if (q == cand.size()) break;
      if (present[q]) continue;
      const Block* b = row.b[t];
      if (!b || b->nr == 0 || b->nc == 0) continue;
      const auto& fl = b->flags;
      const bool known = b->clean || !fl.empty();
      if (p.full) {
        for (int i = 0; i < b->nr; ++i) {
          const uint8_t v = known ? fl[i] : 2;
          if (v == 2) return false;
          if (v == 1) { present[q] = 1; break; }
        }
      } else {
        for (int i : p.ix) {
          const uint8_t v = known ? fl[i] : 2;
          if (v == 2) return false;
          if (v == 1) { present[q] = 1; break; }
        }
      }
    }
  }
  int w = 0;
  for (size_t q = 0; q < cand.size(); ++q) {
    if (present[q]) {
      const int cc = cand[q];
      f.cols_t.push_back(cc);
      f.woff.push_back(w);
      w += (int)c->cols_of[cc].size();
    }
  }
  f.n = w;
  for (auto& p : f.parts) {
    const auto& rr = c->rows_of[p.r];
    if (p.r == s || p.full)
      f.stack_rows.insert(f.stack_rows.end(), rr.begin(), rr.end());
    else
      for (int i : p.ix) f.stack_rows.push_back(rr[i]);
  }
  return true;
}

void apply_front_structure(spq_ctx* c, Front& f, CopyBatch& zeros) {
  Stage stage_(c, "apply_front_structure");
  HostTimer ht(&c->host_ms[6]);
  const int s = f.s;
  f.psrc.reserve(f.parts.size());
  f.gsrc.reserve(f.parts.size() * f.cols_t.size());
  f.dsts.reserve(f.parts.size() * (f.cols_t.size() + 1));
  // gather sources (current blocks, before any replacement); the same walk
  // records which (part, target column) blocks exist, so the structure loop
  // below needs no lookups
  const int nct = (int)f.cols_t.size();
  static thread_local std::vector<Block*> exist;
  exist.assign(f.parts.size() * (size_t)std::max(nct, 1), nullptr);
  for (int pi = 0; pi < (int)f.parts.size(); ++pi) {
    auto& p = f.parts[pi];
    Block* b = find_block(c, p.r, s);
    if (b && b->nc > 0 && b->nr > 0) f.psrc.push_back({b->p, b->nr, pi, 0, b->nc, p.full});
    // blocks (p.r, cols_t[ci]): merge-walk of the sorted row list and cols_t
    const FlatSet& row = c->rix[p.r];
    size_t t = 0;
    for (int ci = 0; ci < nct; ++ci) {
      const int cc = f.cols_t[ci];
      while (t < row.v.size() && row.v[t] < cc) ++t;
      if (t == row.v.size()) break;
      if (row.v[t] != cc) continue;
      Block* bc = row.b[t];
      exist[(size_t)pi * nct + ci] = bc;
      if (bc && bc->nr > 0 && bc->nc > 0)
        f.gsrc.push_back({bc->p, bc->nr, pi, f.woff[ci], bc->nc, p.full});
    }
  }
  // trailing blocks of the neighbour rows (factor.py:467-480).  A fully
  // covered row cluster gets ONE allocation holding all its new blocks
  // side by side (block (r,c) = slab + woff_c * nr, ld nr) and one scatter.
  std::vector<double*> full_slab(f.parts.size(), nullptr);
  for (int pi = 1; pi < (int)f.parts.size(); ++pi) {
    auto& p = f.parts[pi];
    if (!p.full || f.cols_t.empty()) continue;
    const int nr = (int)c->rows_of[p.r].size();
    full_slab[pi] = shared_alloc(c, (size_t)nr * f.n, (int)f.cols_t.size());
    f.dsts.push_back({full_slab[pi], nr, pi, 0, f.n, true});
  }
  for (int ci = 0; ci < (int)f.cols_t.size(); ++ci) {
    const int cc = f.cols_t[ci];
    const int ncol = (int)c->cols_of[cc].size();
    for (int pi = 1; pi < (int)f.parts.size(); ++pi) {
      auto& p = f.parts[pi];
      const int nr = (int)c->rows_of[p.r].size();
      if (p.full) {
        Block* old = exist[(size_t)pi * nct + ci];
        double* mem = full_slab[pi] + (int64_t)f.woff[ci] * nr;
        if (old) {   // replaced in place: the map and adjacency entries stay
          release_mem(c, *old);
          old->p = mem;
          old->base = full_slab[pi];
          old->nr = nr;
          old->nc = ncol;
        }
        Block& b = old ? *old : put_block_new(c, p.r, cc, mem, nr, ncol, full_slab[pi]);
        // speculative: every row is a panel row and receives a row of
        // H^T C_all with cc present -- nonzero (verified at the next query)
        b.flags.assign(nr, c->spec ? 1 : 2);
        b.clean = c->spec;
        b.unverified = c->spec;
        b.origin = 1;
      } else {
        Block* b = exist[(size_t)pi * nct + ci];
        if (!b) {
          double* mem = new_block_mem(c, nr, ncol);
          zeros.zero(mem, (int64_t)nr * ncol);
          Block& nb = put_block_new(c, p.r, cc, mem, nr, ncol);
          nb.flags.assign(nr, 0);
          nb.clean = true;
          b = &nb;
        } else if (b->flags.size() != (size_t)nr) {
          b->flags.assign(nr, 2);
          b->clean = false;
        }
        const uint8_t w = c->spec ? 1 : 2;
        for (int i : p.ix) b->flags[i] = w;
        b->origin = 2;
        if (c->spec) {
          b->unverified = true;   // rows outside the panel keep their (known or unknown) flags
        } else {
          b->clean = false;
        }
        f.dsts.push_back({b->p, nr, pi, f.woff[ci], ncol, false});
      }
    }
  }
  // delete row/col s (factor.py:481-484): the blocks leave the map and the
  // NEIGHBOURS' adjacency lists; the lists of s itself are cleared by retire()
  {
    const FlatSet& col = c->cix[s];
    for (size_t t = 0; t < col.v.size(); ++t) {
      const int r = col.v[t];
      if (Block* b = col.b[t]) {
        release_mem(c, *b);
        c->blk.destroy(b);
      }
      if (r != s) c->rix[r].erase(s);
    }
    const FlatSet& row = c->rix[s];
    for (size_t t = 0; t < row.v.size(); ++t) {
      const int cc = row.v[t];
      if (cc == s) continue;   // (s, s) went with the column
      if (Block* b = row.b[t]) {
        release_mem(c, *b);
        c->blk.destroy(b);
      }
      c->cix[cc].erase(s);
    }
  }
  // record + bookkeeping (factor.py:486-492)
  Record rec;
  rec.kind = REC_ELIM;
  rec.cid = s;
  rec.m = f.m;
  rec.k = f.k;
  rec.n = f.n;
  rec.rows = std::move(f.stack_rows);   // (the planner stamped its rows before this call)
  rec.cols_s = c->cols_of[s];
  for (int cc : f.cols_t) rec.cols_n.insert(rec.cols_n.end(), c->cols_of[cc].begin(), c->cols_of[cc].end());
  const size_t mk = (size_t)f.m * f.k, kk = (size_t)f.k * f.k, kn = (size_t)f.k * f.n;
  rec.payload = dalloc(c, (mk + f.k + 2 * kk + kn) * sizeof(double));
  rec.V = rec.payload;
  rec.tau = rec.V + mk;
  rec.T = rec.tau + f.k;
  rec.R = rec.T + kk;
  rec.Rsn = rec.R + kk;
  rec.payload_scalars = (int64_t)(mk + f.k + kk) + (int64_t)kk + (int64_t)kn;
  zeros.zero(rec.payload, (int64_t)(mk + f.k + 2 * kk));
  for (size_t i = 0; i < c->cols_of[s].size(); ++i) c->row_of_col[c->cols_of[s][i]] = c->rows_of[s][i];
  f.rec = (int)c->recs.size();
  c->recs.push_back(std::move(rec));
  retire(c, s);
}

// Fronts whose target scratch C (m x n) would exceed kChunkBytes stream
// their targets in column chunks after the panel QR (gather -> compact-WY
// Q^T -> scatter per chunk).  Q^T acts column by column, so the result is
// the same as the one-shot C_all path; chunks follow column-cluster
// boundaries, so no block is both written by one chunk and read by another.
bool front_chunked(const Front& f) { return (size_t)f.m * f.n * sizeof(double) > chunk_bytes(); }
size_t front_scratch_bytes(const Front& f) {
  return front_chunked(f) ? chunk_bytes() : (size_t)f.m * f.n * sizeof(double);
}

void run_front_chunked(spq_ctx* c, Front& f) {
  Stage stage_(c, "run_front_chunked");
  Record& rec = c->recs[f.rec];
  const int nct = (int)f.cols_t.size();
  auto cend = [&](int ci) { return ci + 1 < nct ? f.woff[ci + 1] : f.n; };
  // one chunk buffer for the whole front, as large as the arena allows
  // (>= the widest column cluster); chunks are packed to its width
  size_t wmin = 1;
  for (int ci = 0; ci < nct; ++ci) wmin = std::max<size_t>(wmin, cend(ci) - f.woff[ci]);
  const size_t colb = sizeof(double) * (size_t)f.m;
  size_t got = 0;
  double* Cbuf = dalloc_flex(c, std::max(chunk_bytes(), wmin * colb), wmin * colb, &got);
  const size_t maxw = std::max<size_t>(wmin, got / colb);
  int ci0 = 0;
  while (ci0 < nct) {
    int ci1 = ci0 + 1;
    while (ci1 < nct && (size_t)(cend(ci1) - f.woff[ci0]) <= maxw) ++ci1;
    const int a = f.woff[ci0], b = cend(ci1 - 1), w = b - a;
    ci0 = ci1;
    if (w <= 0) continue;
    double* C = Cbuf;
    CopyBatch g;
    g.zero(C, (int64_t)f.m * w);
    g.run(c);
    CopyBatch g2;
    for (auto& sg : f.gsrc) {
      if (sg.col_off < a || sg.col_off >= b) continue;
      auto& p = f.parts[sg.part];
      CopyTask t{};
      t.src = sg.p; t.dst = C + p.o0 + (int64_t)(sg.col_off - a) * f.m; t.src_rows = f.d_ix[sg.part];
      t.nr = p.o1 - p.o0; t.nc = sg.ncols; t.lds = sg.nr; t.ldd = f.m;
      g2.add(t);
    }
    g2.run(c);
    wy_batch(c, {WyProb{rec.V, rec.T, f.m, f.k, C, f.m, w}}, true);
    CopyBatch sc;
    CopyTask t{};
    t.src = C; t.dst = rec.Rsn + (int64_t)a * f.k; t.nr = f.k; t.nc = w; t.lds = f.m; t.ldd = f.k;
    sc.add(t);
    for (auto& d : f.dsts) {
      const int x0 = std::max(d.col_off, a), x1 = std::min(d.col_off + d.ncols, b);
      if (x0 >= x1) continue;
      auto& p = f.parts[d.part];
      CopyTask u{};
      u.src = C + p.o0 + (int64_t)(x0 - a) * f.m;
      u.dst = d.p + (int64_t)(x0 - d.col_off) * d.nr;
      u.nr = p.o1 - p.o0;
      u.nc = x1 - x0;
      u.lds = f.m;
      u.ldd = d.nr;
      u.dst_rows = d.full ? nullptr : f.d_ix[d.part];
      sc.add(u);
    }
    sc.run(c);
  }
  dfree(c, Cbuf);
}

void execute_wave(spq_ctx* c, std::vector<Front>& wave, CopyBatch& zeros, PivotSet& ps) {
  Stage stage_(c, "execute_wave");
  HostTimer ht(&c->host_ms[7]);
  // scratch per (one-shot) front: C (m x n)
  size_t tot = 0;
  std::vector<size_t> coff(wave.size());
  for (size_t i = 0; i < wave.size(); ++i) {
    coff[i] = tot;
    if (!front_chunked(wave[i])) tot += (size_t)wave[i].m * wave[i].n;
  }
  double* scr = tot ? dalloc(c, tot * sizeof(double)) : nullptr;
  for (size_t i = 0; i < wave.size(); ++i)
    if (!front_chunked(wave[i])) zeros.zero(scr + coff[i], (int64_t)wave[i].m * wave[i].n);
  zeros.run(c);
  // all partial row lists of the wave in ONE upload
  std::vector<int> ixpack;
  std::vector<std::vector<size_t>> ixoff(wave.size());
  for (size_t fi = 0; fi < wave.size(); ++fi) {
    Front& f = wave[fi];
    ixoff[fi].assign(f.parts.size(), (size_t)-1);
    for (size_t pi = 0; pi < f.parts.size(); ++pi) {
      auto& p = f.parts[pi];
      if (p.r != f.s && !p.full) {
        ixoff[fi][pi] = ixpack.size();
        ixpack.insert(ixpack.end(), p.ix.begin(), p.ix.end());
      }
    }
  }
  const int* d_ixpack = ixpack.empty() ? nullptr : upload(c, ixpack);
  // gather: every front's tasks at a precomputed offset (empty tasks stay in
  // the list as no-ops), filled by a few host threads on the large waves
  CopyBatch g;
  {
    std::vector<size_t> goff(wave.size() + 1, 0);
    for (size_t fi = 0; fi < wave.size(); ++fi)
      goff[fi + 1] = goff[fi] + wave[fi].psrc.size() + (front_chunked(wave[fi]) ? 0 : wave[fi].gsrc.size());
    g.reserve(goff.back());
    g.t.resize(goff.back());
    parallel_fronts(wave.size(), goff.back(), [&](size_t f0, size_t f1) {
      for (size_t fi = f0; fi < f1; ++fi) {
        Front& f = wave[fi];
        Record& rec = c->recs[f.rec];
        double* C = scr + coff[fi];
        f.d_ix.assign(f.parts.size(), nullptr);
        for (size_t pi = 0; pi < f.parts.size(); ++pi)
          if (ixoff[fi][pi] != (size_t)-1) f.d_ix[pi] = d_ixpack + ixoff[fi][pi];
        CopyTask* out = g.t.data() + goff[fi];
        for (auto& sp : f.psrc) {
          auto& p = f.parts[sp.part];
          CopyTask t{};
          t.src = sp.p; t.dst = rec.V + p.o0; t.src_rows = f.d_ix[sp.part];
          t.nr = p.o1 - p.o0; t.nc = sp.ncols; t.lds = sp.nr; t.ldd = f.m;
          g.account(t);
          *out++ = t;
        }
        if (!front_chunked(f))
          for (auto& sg : f.gsrc) {
            auto& p = f.parts[sg.part];
            CopyTask t{};
            t.src = sg.p; t.dst = C + p.o0 + (int64_t)sg.col_off * f.m; t.src_rows = f.d_ix[sg.part];
            t.nr = p.o1 - p.o0; t.nc = sg.ncols; t.lds = sg.nr; t.ldd = f.m;
            g.account(t);
            *out++ = t;
          }
      }
    });
  }
  g.run(c);
  // QR of every panel, its reflectors applied block by block to C_all
  std::vector<QrProb> qp;
  for (size_t fi = 0; fi < wave.size(); ++fi) {
    Front& f = wave[fi];
    Record& rec = c->recs[f.rec];
    QrProb q{rec.V, f.m, f.k, rec.R, rec.tau, rec.T, {}};
    if (f.n > 0 && !front_chunked(f)) q.targets.push_back(CTarget{scr + coff[fi], f.m, f.n});
    q.want_T = f.n > 0 && front_chunked(f);
    rec.full_T = f.n > 0;
    qp.push_back(std::move(q));
  }
  qr_batch(c, qp);
  for (auto& f : wave) {
    Record& rec = c->recs[f.rec];
    ps.jobs.push_back(PivotJob{rec.R, f.k, f.k, 0});
    ps.ctx.push_back("pivot block of cluster " + std::to_string(f.s));
  }
  // scatter: R_sn = C[:k], neighbour rows back into blocks
  CopyBatch sc;
  {
    std::vector<size_t> soff(wave.size() + 1, 0);
    for (size_t fi = 0; fi < wave.size(); ++fi)
      soff[fi + 1] = soff[fi] + (front_chunked(wave[fi]) ? 0 : wave[fi].dsts.size() + 1);
    sc.reserve(soff.back());
    sc.t.resize(soff.back());
    parallel_fronts(wave.size(), soff.back(), [&](size_t f0, size_t f1) {
      for (size_t fi = f0; fi < f1; ++fi) {
        Front& f = wave[fi];
        if (front_chunked(f)) continue;
        Record& rec = c->recs[f.rec];
        double* C = scr + coff[fi];
        CopyTask* out = sc.t.data() + soff[fi];
        CopyTask t{};
        t.src = C; t.dst = rec.Rsn; t.nr = f.k; t.nc = f.n; t.lds = f.m; t.ldd = f.k;
        sc.account(t);
        *out++ = t;
        for (auto& d : f.dsts) {
          auto& p = f.parts[d.part];
          CopyTask u{};
          u.src = C + p.o0 + (int64_t)d.col_off * f.m;
          u.dst = d.p;
          u.nr = p.o1 - p.o0;
          u.nc = d.ncols;
          u.lds = f.m;
          u.ldd = d.nr;
          u.dst_rows = d.full ? nullptr : f.d_ix[d.part];
          sc.account(u);
          *out++ = u;
        }
      }
    });
  }
  sc.run(c);
  if (scr) dfree(c, scr);
  for (auto& f : wave)
    if (front_chunked(f)) run_front_chunked(c, f);
  pivot_launch(c, ps);
  flush_deferred(c);
}

constexpr size_t kWaveBudget = (size_t)12 << 30;   // front scratch per wave

void do_factor(spq_ctx* c, const std::vector<int>& ids) {
  size_t pos = 0;
  std::vector<int> stamp(c->N, -1);
  int wave_id = 0;
  PivotSet& ps = c->piv;
  if (!c->spec) pivot_raise(c, ps);
  while (pos < ids.size()) {
    // refresh flags of every row cluster any pending op may query
    // (ascending cluster ids, each once)
    std::vector<int> rows;
    {
      static thread_local std::vector<char> seen;
      seen.assign(c->ncl, 0);
      auto take = [&](int r) { if (!seen[r]) { seen[r] = 1; rows.push_back(r); } };
      for (size_t t = pos; t < ids.size(); ++t) {
        const int s = ids[t];
        take(s);
        for (int r : c->cix[s]) take(r);
      }
      std::sort(rows.begin(), rows.end());
    }
    refresh_flags(c, rows);
    // exact mode: the refresh synchronized, so reading the previous waves'
    // pivot checks is free; speculative mode defers them to the end of the call
    if (!c->spec) pivot_raise(c, ps);
    ++wave_id;
    std::vector<Front> wave;
    wave.reserve(ids.size() - pos);
    CopyBatch zeros;
    zeros.reserve(2 * (ids.size() - pos) + 64);
    size_t wave_bytes = 0;
    while (pos < ids.size()) {
      const int s = ids[pos];
      if (!c->active[s]) throw SpqError(SPQ_ERR_BAD_INPUT, "factor of inactive cluster " + std::to_string(s));
      if (c->cols_of[s].empty()) {  // factor.py:413-415
        retire(c, s);
        ++pos;
        continue;
      }
      Front f;
      auto tp = std::chrono::steady_clock::now();
      const bool ok = plan_front(c, s, f);
      c->host_ms[2] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp).count();
      if (!ok) break;
      bool clash = false;
      for (int64_t r : f.stack_rows)
        if (stamp[r] == wave_id) { clash = true; break; }
      if (clash) break;
      // memory budget for the wave's front scratch (C_all) and payloads
      const size_t fbytes = front_scratch_bytes(f) + 8 * ((size_t)f.m * f.k + (size_t)f.k * f.n);
      if (!wave.empty() && wave_bytes + fbytes > kWaveBudget) break;
      wave_bytes += fbytes;
      for (int64_t r : f.stack_rows) stamp[r] = wave_id;
      apply_front_structure(c, f, zeros);
      wave.push_back(std::move(f));
      ++pos;
    }
    if (wave.empty()) {
      if (pos < ids.size()) throw SpqError(SPQ_ERR_INTERNAL, "wave planner made no progress");
      break;
    }
    execute_wave(c, wave, zeros, ps);
  }
  if (!c->spec) pivot_raise(c, ps);
  flush_deferred(c);
}

// ================================================================ (b) scale
void do_scale(spq_ctx* c, const std::vector<int>& ids, int32_t* done) {
  Stage stage_(c, "do_scale");
  HostTimer ht(&c->host_ms[11]);
  std::vector<int> todo;
  for (size_t t = 0; t < ids.size(); ++t) {
    done[t] = 0;
    const int p = ids[t];
    if (!c->active[p]) throw SpqError(SPQ_ERR_BAD_INPUT, "scale of inactive cluster");
    if (!c->cols_of[p].empty()) { todo.push_back(p); done[t] = 1; }
  }
  if (todo.empty()) return;
  CopyBatch zeros, g;
  std::vector<QrProb> qp;
  std::vector<int> recid;
  for (int p : todo) {
    const int np = (int)c->cols_of[p].size();
    Record rec;
    rec.kind = REC_SCALE;
    rec.cid = p;
    rec.m = np; rec.k = np; rec.n = 0;
    rec.rows = c->rows_of[p];
    rec.cols_s = c->cols_of[p];
    const size_t kk = (size_t)np * np;
    rec.payload = dalloc(c, (kk + np + 2 * kk) * sizeof(double));
    rec.V = rec.payload; rec.tau = rec.V + kk; rec.T = rec.tau + np; rec.R = rec.T + kk;
    rec.payload_scalars = (int64_t)(kk + np + kk) + (int64_t)kk;
    zeros.zero(rec.payload, (int64_t)(3 * kk + np));
    Block* b = find_block(c, p, p);
    if (b && b->nr == np && b->nc == np) {
      CopyTask t{};
      t.src = b->p; t.dst = rec.V; t.nr = np; t.nc = np; t.lds = np; t.ldd = np;
      g.add(t);
    }
    // left application U_pp^T to every (p, c) block rides on the QR (factor.py:512-520)
    QrProb q{rec.V, np, np, rec.R, rec.tau, rec.T, {}};
    for (int cc : c->rix[p]) {
      if (cc == p) continue;
      Block* bc = find_block(c, p, cc);
      if (bc && bc->nc > 0 && bc->nr == np) {
        q.targets.push_back(CTarget{bc->p, bc->nr, bc->nc});
        // U_pp^T mixes rows only within the coupled groups of A_pp (merged
        // child fragments can be decoupled: block-diagonal U) -- no
        // prediction, the next query reads these flags back exactly
        bc->origin = 3;
        bc->clean = false;
        bc->unverified = false;
        bc->flags.clear();
      }
    }
    rec.full_T = !q.targets.empty();
    qp.push_back(std::move(q));
    recid.push_back((int)c->recs.size());
    c->recs.push_back(std::move(rec));
  }
  zeros.run(c);
  g.run(c);
  qr_batch(c, qp);
  PivotSet& ps = c->piv;
  for (size_t t = 0; t < todo.size(); ++t) {
    Record& rec = c->recs[recid[t]];
    ps.jobs.push_back(PivotJob{rec.R, rec.k, rec.k, 0});
    ps.ctx.push_back("diagonal block of interface " + std::to_string(todo[t]));
  }
  pivot_launch(c, ps);
  // right: R_pp^{-1} on every (r, p) block (factor.py:521-529)
  std::vector<TrsmJob> tj;
  int ttiles = 0;
  double trsm_flops = 0;
  for (size_t t = 0; t < todo.size(); ++t) {
    const int p = todo[t];
    Record& rec = c->recs[recid[t]];
    for (int r : c->cix[p]) {
      if (r == p) continue;
      Block* b = find_block(c, r, p);
      if (b && b->nr > 0) {
        tj.push_back(TrsmJob{rec.R, b->p, b->nr, rec.k, rec.k, b->nr, ttiles});
        ttiles += trsm_tiles(b->nr);
        trsm_flops += (double)b->nr * rec.k * rec.k;
        b->origin = 4;
        predict_same_rows(c, *b);
      }
    }
  }
  // blocked right TRSM: per 32-column block, DMMA update from the solved
  // columns then the diagonal-block substitution (thread per row)
  if (!tj.empty()) {
    int kmax = 0;
    for (auto& t : tj) kmax = std::max(kmax, t.k);
    const TrsmJob* dj = upload(c, tj);
    for (int j0 = 0; j0 < kmax; j0 += 32) {
      if (j0 > 0) {
        GemmBatch gb;
        for (auto& t : tj) {
          if (j0 >= t.k) continue;
          const int w = std::min(32, t.k - j0);
          gb.add(t.B, t.ldb, t.R + (int64_t)j0 * t.ldr, t.ldr, t.B + (int64_t)j0 * t.ldb, t.ldb,
                 t.n, w, j0, -1.0, 1.0);
        }
        gb.run(c, false, 0);
      }
      Scope s(c, F_TRSM);
      launch_trsm_diag(dj, (int)tj.size(), ttiles, j0, c->st);
      c->tm.launches[F_TRSM]++;
      c->n_kernels++;
    }
    c->tm.flops[F_TRSM] += trsm_flops;
  }
  CopyBatch id;
  for (int p : todo) {
    const int np = (int)c->cols_of[p].size();
    Block* b = find_block(c, p, p);
    double* mem;
    if (b && b->nr == np && b->nc == np) {
      mem = b->p;
    } else {
      mem = new_block_mem(c, np, np);
      Block& nb = put_block(c, p, p, mem, np, np);
      (void)nb;
      b = find_block(c, p, p);
    }
    set_identity_flags(c, *b, np);
    CopyTask t{};
    t.dst = mem; t.nr = np; t.nc = np; t.ldd = np; t.ident = 1;
    id.add(t);
  }
  id.run(c);
  if (!c->spec) pivot_raise(c, ps);
  flush_deferred(c);
}

// ============================================================ (c) sparsify
struct SparsifyOut {
  int rank;
  int before;
  double dropped;
  int done;
};

// One sparsification job (an interface of a wave).
struct SpJob {
  int p = -1;
  std::vector<int64_t> cols_p, rows_p;
  int np = 0;
  std::vector<int> us, cs, hu, wc;
  int nu = 0, ncols = 0, kmax = 0;
  double *M = nullptr, *Wm = nullptr, *sq = nullptr, *pay = nullptr;
  double *V = nullptr, *tau = nullptr, *beta = nullptr, *T = nullptr;
  int *keep = nullptr, *perm = nullptr;
  bool m_on_side = false;   // M read by queued side-stream work (freed at side_join)
  bool cta = false;
  int cl = 0;        // cluster size for the cluster-resident CPQR (0: cooperative)
  int rank = -1;
};

struct SpScal { int nk; int rank; double ratio; double maxcol; };

constexpr size_t CPQR_CTA_MAX_SMEM = 220 * 1024;

// Threshold CPQR of a list of independent problems (job.ncap = column
// capacity, job.nk = device live column count).  Per problem: the
// register-resident cluster kernel when a plan exists (smallest cluster,
// then least row padding), else the CTA shared-memory kernel, the cluster
// shared-memory kernel, or the cooperative grid kernel.  Everything but the
// cooperative jobs runs concurrently on the fork streams.
void run_cpqr_jobs(spq_ctx* c, const std::vector<CpqrJob>& jobs) {
  const bool coop_only = env_flag("SPQ_CPQR_COOP"), no_ws = env_flag("SPQ_CPQR_NOWS");
  std::map<std::tuple<int, int, int, int>, std::pair<std::vector<CpqrJob>, size_t>> rg_groups;   // (variant, cl, tpc, nt)
  std::map<int, std::pair<std::vector<CpqrJob>, size_t>> by_cl;
  std::vector<CpqrJob> cj;
  std::vector<CpqrJob> coop;
  size_t cta_smem = 0;
  for (const CpqrJob& q : jobs) {
    const int np = q.m, ncap = std::max(q.ncap, 1);
    // register plan: smallest CTA (widest spread), then fewest lanes per
    // column (fewest shuffles per reduction), then least row padding
    int bv = -1, bcl = 0, btpc = 0, bnt = 0;
    static const int only_var = getenv("SPQ_CPQR_VAR") ? atoi(getenv("SPQ_CPQR_VAR")) : -1;   // A/B runs
    static const int nvar = getenv("SPQ_CPQR_NVAR") ? atoi(getenv("SPQ_CPQR_NVAR")) : 3;
    if (!coop_only && !no_ws)
      for (int v = 0; v < std::min(nvar, cpqr_reg_nvar()); ++v) {
        if (only_var >= 0 && v != only_var) continue;
        int tpc = 0, nt = 0;
        const int cl = cpqr_reg_plan(np, ncap, v, &tpc, &nt);
        if (cl == 0) continue;
        const auto key = std::make_tuple(nt, tpc * cpqr_reg_rows(v), tpc, cl);
        if (bv < 0 || key < std::make_tuple(bnt, btpc * cpqr_reg_rows(bv), btpc, bcl)) { bv = v; bcl = cl; btpc = tpc; bnt = nt; }
      }
    static const bool cpqr_log = env_flag("SPQ_CPQR_LOG");   // diagnostics: problem sizes and plans
    if (cpqr_log) fprintf(stderr, "[cpqr] m=%d ncap=%d n=%d variant=%d cl=%d tpc=%d nt=%d\n", np, ncap, q.n, bv, bcl, btpc, bnt);
    if (bv >= 0) {
      auto& g = rg_groups[std::make_tuple(bv, bcl, btpc, bnt)];
      g.first.push_back(q);
      g.second = std::max(g.second, cpqr_reg_smem(btpc * cpqr_reg_rows(bv), bcl, bnt));
      continue;
    }
    if (!coop_only && !env_flag("SPQ_CPQR_CLUSTER") && cpqr_cta_smem(np, ncap) <= CPQR_CTA_MAX_SMEM) {
      cj.push_back(q);
      cta_smem = std::max(cta_smem, cpqr_cta_smem(np, ncap));
      continue;
    }
    const int cl = coop_only ? 0 : cpqr_cluster_size(np, ncap);
    if (cl > 0) {
      auto& g2 = by_cl[cl];
      g2.first.push_back(q);
      g2.second = std::max(g2.second, cpqr_cluster_smem(np, ncap, cl));
      continue;
    }
    coop.push_back(q);
  }
  std::string cq_tag;
  if (Scope::scope_log()) {
    char b[200];
    int m0 = 0, n0 = 0;
    for (auto& q : jobs) { m0 = std::max(m0, q.m); n0 = std::max(n0, q.ncap); }
    snprintf(b, sizeof b, "cpqr jobs=%zu reg_groups=%zu cta=%zu cluster=%zu coop=%zu max_m=%d max_n=%d",
             jobs.size(), rg_groups.size(), cj.size(), by_cl.size(), coop.size(), m0, n0);
    cq_tag = b;
  }
  Scope s(c, F_CPQR, cq_tag);
  // upload every job list first (the ring), then fork
  std::vector<std::tuple<const CpqrJob*, int, std::tuple<int, int, int, int>, size_t, const CpqrJob*>> wl;
  for (auto& kv : rg_groups)
    wl.emplace_back(up_or_param(c, kv.second.first, PL_SMALL), (int)kv.second.first.size(), kv.first,
                    kv.second.second, kv.second.first.data());
  std::vector<std::tuple<const CpqrJob*, int, int, size_t>> cl_l;
  for (auto& kv : by_cl)
    cl_l.emplace_back(upload(c, kv.second.first), (int)kv.second.first.size(), kv.first,
                      kv.second.second);
  const CpqrJob* d_cj = cj.empty() ? nullptr : upload(c, cj);
  {
    Fork fk(c, (int)(wl.size() + cl_l.size() + (d_cj ? 1 : 0)));
    for (auto& w : wl) {
      const auto& key = std::get<2>(w);
      launch_cpqr_reg(std::get<0>(w), std::get<4>(w), std::get<1>(w), std::get<0>(key), std::get<1>(key),
                      std::get<2>(key), std::get<3>(key), std::get<3>(w), fk.next());
      c->tm.launches[F_CPQR]++;
      c->n_kernels++;
    }
    for (auto& w : cl_l) {
      launch_cpqr_cluster(std::get<0>(w), std::get<1>(w), std::get<2>(w), std::get<3>(w), fk.next());
      c->tm.launches[F_CPQR]++;
      c->n_kernels++;
    }
    if (d_cj) {
      launch_cpqr_cta(d_cj, (int)cj.size(), cta_smem, fk.next());
      c->tm.launches[F_CPQR]++;
      c->n_kernels++;
    }
    fk.join();
  }
  for (const CpqrJob& q : coop) {
    const int ncap = std::max(q.ncap, 1);
    const int G = cpqr_grid(ncap, c->nsm);
    double* slots = dalloc(c, 2 * G * sizeof(double));
    int* slotp = (int*)dalloc(c, 2 * G * sizeof(int));
    CpqrArgs a{};
    a.gmaps = (int*)dalloc(c, (size_t)G * 2 * ncap * sizeof(int));
    a.force_gmaps = env_flag("SPQ_CPQR_GMAPS");
    c->deferred.push_back((double*)a.gmaps);
    a.W = q.W; a.m = q.m; a.ncols_cap = ncap; a.nk = q.nk;
    a.eps = q.eps; a.min_rank = q.min_rank; a.V = q.V; a.tau = q.tau; a.beta = q.beta;
    a.rank = q.rank; a.perm = q.perm; a.slot_val = slots; a.slot_pos = slotp;
    a.finalize = 0;
    launch_cpqr(a, G, c->st);
    c->tm.launches[F_CPQR]++;
    c->n_kernels++;
    dfree(c, slots);
    dfree(c, slotp);
  }
}

// sparsify_interface for a WAVE of mutually independent interfaces (no
// shared block): identical to running them one after another in order.
void do_sparsify_wave(spq_ctx* c, const std::vector<int>& wave, double eps,
                      std::vector<SparsifyOut>& outs, const std::vector<int>& drop_idx) {
  Stage stage_(c, "do_sparsify_wave");
  HostTimer ht(&c->host_ms[8]);
  const int nw = (int)wave.size();
  std::vector<SpJob> J(nw);
  CopyBatch g;
  for (int t = 0; t < nw; ++t) {
    SpJob& j = J[t];
    j.p = wave[t];
    j.cols_p = c->cols_of[j.p];
    j.rows_p = c->rows_of[j.p];
    j.np = (int)j.cols_p.size();
    outs[t] = SparsifyOut{-1, j.np, 0.0, 0};
    if (j.np == 0) continue;
    for (int u : c->cix[j.p]) if (u != j.p) j.us.push_back(u);
    for (int cc : c->rix[j.p]) if (cc != j.p) j.cs.push_back(cc);
    for (int u : j.us) { j.hu.push_back(find_block(c, u, j.p)->nr); j.nu += j.hu.back(); }
    int ncl = 0;
    for (int cc : j.cs) { j.wc.push_back(find_block(c, j.p, cc)->nc); ncl += j.wc.back(); }
    j.ncols = j.nu + ncl;
    j.kmax = std::min(j.np, j.ncols);
    const size_t Msz = (size_t)j.np * std::max(j.ncols, 1);
    j.M = dalloc(c, Msz * sizeof(double));
    j.Wm = dalloc(c, Msz * sizeof(double));
    j.sq = dalloc(c, std::max(j.ncols, 1) * sizeof(double));
    j.keep = (int*)dalloc(c, std::max(j.ncols, 1) * sizeof(int));
    j.perm = (int*)dalloc(c, std::max(j.ncols, 1) * sizeof(int));
    const size_t vsz = (size_t)j.np * std::max(j.kmax, 1);
    const int k1 = std::max(j.kmax, 1);
    j.pay = dalloc(c, (vsz + 2 * (size_t)k1 + (size_t)k1 * k1) * sizeof(double));
    j.V = j.pay;
    j.tau = j.V + vsz;
    j.beta = j.tau + k1;
    j.T = j.beta + k1;
    g.zero(j.V, (int64_t)vsz);
    int off = 0;
    for (size_t q = 0; q < j.us.size(); ++q) {
      Block* b = find_block(c, j.us[q], j.p);
      CopyTask x{};
      x.src = b->p; x.dst = j.M + (int64_t)off * j.np; x.nr = b->nr; x.nc = j.np; x.lds = b->nr;
      x.ldd = j.np; x.trans = 1;
      g.add(x);
      off += b->nr;
    }
    for (size_t q = 0; q < j.cs.size(); ++q) {
      Block* b = find_block(c, j.p, j.cs[q]);
      CopyTask x{};
      x.src = b->p; x.dst = j.M + (int64_t)off * j.np; x.nr = j.np; x.nc = b->nc; x.lds = j.np;
      x.ldd = j.np;
      g.add(x);
      off += b->nc;
    }
  }
  g.run(c);
  SpScal* dsc = (SpScal*)dalloc(c, std::max(nw, 1) * sizeof(SpScal));
  {
    Scope s(c, F_CPQR, Scope::scope_log() ? std::string("prep") : std::string());
    std::vector<PrepJob> pj;
    for (int t = 0; t < nw; ++t) {
      SpJob& j = J[t];
      if (j.np == 0) continue;
      pj.push_back(PrepJob{j.M, j.sq, j.keep, &dsc[t].nk, &dsc[t].ratio, &dsc[t].maxcol, j.Wm,
                           j.np, j.ncols, 1, 0});
    }
    if (!pj.empty()) {
      const PrepJob* d_pj = (int)pj.size() <= sparsify_prep_plist_max() ? nullptr : upload(c, pj);
      launch_sparsify_prep_batch(d_pj, pj.data(), (int)pj.size(), eps, c->st);
      c->tm.launches[F_CPQR] += 3;
      c->n_kernels += 3;
    }
  }
  // the kept column counts (one read per wave) size every CPQR exactly.
  // SPQ_SPARSIFY_NO_NKSYNC=1 sizes them by the pre-filter count instead (no
  // read-back; measured slower on C3: the larger clusters cost more per
  // pivot step than the sync saves)
  std::vector<SpScal> hk(std::max(nw, 1));
  static const bool nk_sync = !env_flag("SPQ_SPARSIFY_NO_NKSYNC");
  if (nk_sync) {
    HostTimer hw(&c->host_ms[9]);
    CUDA_TRY(cudaMemcpyAsync(hk.data(), dsc, nw * sizeof(SpScal), cudaMemcpyDeviceToHost, c->st));
    sync(c);
  } else {
    for (int t = 0; t < nw; ++t) hk[t].nk = J[t].ncols;
  }
  pivot_raise(c, c->piv);   // checks queued by this level's factor/scale calls
  auto job_of = [&](int t, int ncap) {
    SpJob& j = J[t];
    CpqrJob q{};
    q.W = j.Wm; q.m = j.np; q.n = j.ncols; q.ncap = ncap; q.ldw = j.np;
    q.nk = &dsc[t].nk; q.eps = &dsc[t].ratio; q.min_rank = 0; q.V = j.V; q.ldv = j.np;
    q.tau = j.tau; q.beta = j.beta; q.rank = &dsc[t].rank; q.perm = j.perm; q.write_back = 0;
    return q;
  };
  std::vector<CpqrJob> jobs;
  for (int t = 0; t < nw; ++t)
    if (J[t].np > 0) jobs.push_back(job_of(t, std::max(hk[t].nk, 1)));
  run_cpqr_jobs(c, jobs);
  std::vector<SpScal> h(std::max(nw, 1));
  {
    HostTimer hw(&c->host_ms[9]);
    CUDA_TRY(cudaMemcpyAsync(h.data(), dsc, nw * sizeof(SpScal), cudaMemcpyDeviceToHost, c->st));
    sync(c);
  }
  dfree(c, dsc);
  // T of the accepted reflectors + Q^T M for every compressed interface
  std::vector<TProb> tp;
  std::vector<WyProb> wp;
  for (int t = 0; t < nw; ++t) {
    SpJob& j = J[t];
    if (j.np == 0) continue;
    j.rank = h[t].rank;
    outs[t].rank = j.rank;
    const double mm = j.np, nn = h[t].nk, rr = j.rank;
    c->tm.flops[F_CPQR] += 4.0 * mm * nn * rr - 2.0 * rr * rr * (mm + nn) + 4.0 * rr * rr * rr / 3.0;
    c->tm.bytes[F_CPQR] += 16.0 * mm * nn;
    if (j.rank >= j.np || j.rank <= 0) continue;
    tp.push_back(TProb{j.V, j.np, j.rank, j.tau, j.T});
    wp.push_back(WyProb{j.V, j.T, j.np, j.rank, j.M, j.np, j.ncols});
  }
  // (no T / W overlap here: the side stream still carries the previous
  // wave's dropped-norm statistics, which must stay off the critical path)
  build_full_T(c, tp);
  wy_batch(c, wp, true);
  // dropped = max(||E1||_2, ||E2||_2), E1^T = QtM[r:, :nu], E2 = QtM[r:, nu:]
  // (factor.py:634-643): Gram matrices by DMMA, batched power iteration
  {
    std::vector<size_t> eoff;
    size_t etot = 0, gtot = 0;
    for (int t = 0; t < nw; ++t) {
      SpJob& j = J[t];
      if (j.np == 0 || j.rank >= j.np || j.rank <= 0) continue;
      const int fdim = j.np - j.rank;
      etot += (size_t)fdim * std::max(j.ncols, 1);
      gtot += 2 * (size_t)fdim * fdim;
    }
    if (gtot > 0) {
      // only the level's statistic reads the result (after side_join at the
      // end of do_sparsify): off the critical path, on the side stream
      SideScope side_(c);
      double* Et = dalloc(c, etot * sizeof(double));
      double* Gs = dalloc(c, gtot * sizeof(double));
      CopyBatch tcb;
      GemmBatch gg;
      std::vector<PowerJob> pj;
      size_t eo = 0, go = 0;
      int fmax = 0;
      for (int t = 0; t < nw; ++t) {
        SpJob& j = J[t];
        if (j.np == 0 || j.rank >= j.np || j.rank <= 0) continue;
        const int fdim = j.np - j.rank;
        fmax = std::max(fmax, fdim);
        double* E = Et + eo;              // E^T: ncols x fdim (ld ncols)
        eo += (size_t)fdim * std::max(j.ncols, 1);
        CopyTask x{};
        x.src = j.M + j.rank; x.dst = E; x.nr = fdim; x.nc = j.ncols; x.lds = j.np;
        x.ldd = std::max(j.ncols, 1); x.trans = 1;
        tcb.add(x);
        const int nu = j.nu, nc = j.ncols - j.nu;
        double* G1 = Gs + go;
        double* G2 = G1 + (size_t)fdim * fdim;
        go += 2 * (size_t)fdim * fdim;
        // G = E E^T = (E^T)^T (E^T) over the column ranges [0,nu) and [nu,ncols)
        gg.add(E, std::max(j.ncols, 1), E, std::max(j.ncols, 1), G1, fdim, fdim, fdim, nu, 1.0, 0.0);
        gg.add(E + nu, std::max(j.ncols, 1), E + nu, std::max(j.ncols, 1), G2, fdim, fdim, fdim,
               nc, 1.0, 0.0);
        pj.push_back(PowerJob{G1, fdim, c->d_dropped + 2 * drop_idx[t]});
        pj.push_back(PowerJob{G2, fdim, c->d_dropped + 2 * drop_idx[t] + 1});
      }
      tcb.run(c);
      gg.run(c, true, 0);
      launch_power_iter(upload(c, pj), (int)pj.size(), fmax, c->st);
      c->n_kernels++;
      c->side_free.push_back(Et);
      c->side_free.push_back(Gs);
      // the side work reads M (= Q^T M): keep every M of this wave until the join
      for (int t = 0; t < nw; ++t)
        if (J[t].np > 0 && J[t].rank > 0 && J[t].rank < J[t].np) J[t].m_on_side = true;
    }
  }
  // split back + structure, in order (factor.py:617-658)
  CopyBatch sc;
  for (int t = 0; t < nw; ++t) {
    SpJob& j = J[t];
    if (j.np == 0) continue;
    const int p = j.p, r = j.rank, np = j.np;
    // M is still read by the queued split-back copies: free after sc.run
    auto release = [&]() {
      for (void* q : {(void*)j.Wm, (void*)j.sq, (void*)j.keep, (void*)j.perm})
        c->deferred.push_back((double*)q);
      if (j.m_on_side) c->side_free.push_back(j.M);
      else c->deferred.push_back(j.M);
    };
    if (r >= np) {   // factor.py:630-631
      release();
      dfree(c, j.pay);
      continue;
    }
    int off = 0;
    for (size_t q = 0; q < j.us.size(); ++q) {
      const int u = j.us[q], h_u = j.hu[q];
      Block* old = find_block(c, u, p);
      // rows of u keep their zero pattern under the right rotation
      RowFlags keep_fl;
      const bool known = c->spec && old && old->clean && old->flags.size() == (size_t)h_u;
      if (known) keep_fl = old->flags;
      if (old) release_mem(c, *old);
      if ((int64_t)h_u * r > 0) {
        double* mem = new_block_mem(c, h_u, r);
        CopyTask x{};
        x.src = j.M + (int64_t)off * np; x.dst = mem; x.nr = r; x.nc = h_u; x.lds = np;
        x.ldd = h_u; x.trans = 1;
        sc.add(x);
        Block& b = put_block(c, u, p, mem, h_u, r);
        b.origin = 5;
        if (known) {
          b.flags = std::move(keep_fl);
          b.clean = true;
          b.unverified = true;
        } else {
          b.clean = false;
          b.flags.clear();
        }
      } else {
        drop_block(c, u, p);
      }
      off += h_u;
    }
    for (size_t q = 0; q < j.cs.size(); ++q) {
      const int cc = j.cs[q], w = j.wc[q];
      Block* old = find_block(c, p, cc);
      const bool known = c->spec && old && old->clean;
      const bool nz = known && any_nonzero(*old);
      if (old) release_mem(c, *old);
      if ((int64_t)w * r > 0) {
        double* mem = new_block_mem(c, r, w);
        CopyTask x{};
        x.src = j.M + (int64_t)off * np; x.dst = mem; x.nr = r; x.nc = w; x.lds = np; x.ldd = r;
        sc.add(x);
        Block& b = put_block(c, p, cc, mem, r, w);
        b.origin = 6;
        if (known) {
          predict_mixed_rows(c, b, nz, r);
        } else {
          b.clean = false;
          b.flags.clear();
        }
      } else {
        drop_block(c, p, cc);
      }
      off += w;
    }
    Block* dp = find_block(c, p, p);
    if (dp) release_mem(c, *dp);
    if (r > 0) {
      double* mem = new_block_mem(c, r, r);
      CopyTask x{};
      x.dst = mem; x.nr = r; x.nc = r; x.ldd = r; x.ident = 1;
      sc.add(x);
      Block& b = put_block(c, p, p, mem, r, r);
      set_identity_flags(c, b, r);
    } else {
      drop_block(c, p, p);
      for (int u : j.us) drop_block(c, u, p);
      for (int cc : j.cs) drop_block(c, p, cc);
    }
    Record rec;
    rec.kind = REC_SPARSIFY;
    rec.cid = p;
    rec.m = np; rec.k = r; rec.n = 0; rec.rank = r;
    rec.rows = j.rows_p;
    rec.cols_s = j.cols_p;
    rec.payload = j.pay;
    rec.V = j.V; rec.tau = j.tau; rec.T = j.T;
    rec.payload_scalars = (int64_t)np * r + r + (int64_t)r * r;
    for (int i = r; i < np; ++i) c->row_of_col[j.cols_p[i]] = j.rows_p[i];
    c->rows_of[p].assign(j.rows_p.begin(), j.rows_p.begin() + r);
    c->cols_of[p].assign(j.cols_p.begin(), j.cols_p.begin() + r);
    c->recs.push_back(std::move(rec));
    outs[t].done = 1;
    release();   // M etc. are read by the queued copies: stream order keeps them valid
  }
  sc.run(c);
  flush_deferred(c);
}

// ------------------------------------------------------------------------
// Sequential route for the sparsification variants the wave path does not
// cover (factor.py:536-709): the UNSCALED route (mode 'unscaled', and every
// level on which scale_every > 1 skips the scaling) and the one-sided /
// Gram targets of 'variant1' / 'variant2'.  One interface at a time in the
// reference's ascending order; every numeric step runs on the device, the
// host reads only the scalars that steer the control flow (sigma_min, the
// accepted rank, ||R_fn||_2).
enum SpMode { SPM_SCALED = 0, SPM_UNSCALED = 1, SPM_VARIANT1 = 2, SPM_VARIANT2 = 3 };
constexpr double SIGMA_FLOOR = 1e-14;   // factor.py:53

// extreme singular values of A (m x n, lda) by one-sided Jacobi on a copy
void jacobi_extremes(spq_ctx* c, const double* A, int m, int n, int lda, double* smax,
                     double* smin) {
  *smax = 0.0;
  *smin = 0.0;
  if ((int64_t)m * n == 0) return;
  double* W = dalloc(c, ((size_t)m * n + 2) * sizeof(double));
  CopyBatch cb;
  CopyTask x{};
  x.src = A; x.dst = W; x.nr = m; x.nc = n; x.lds = lda; x.ldd = m;
  cb.add(x);
  cb.run(c);
  SvJob j{W, m, n, m, W + (size_t)m * n, W + (size_t)m * n + 1};
  launch_jacobi_sv(upload(c, &j, 1), 1, c->st);
  c->n_kernels++;
  double h[2];
  CUDA_TRY(cudaMemcpyAsync(h, W + (size_t)m * n, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  *smax = h[0];
  *smin = h[1];
  dfree(c, W);
}

// ||X||_2 (X rows x cols, ldx): the largest eigenvalue of the smaller Gram
// matrix (full relative accuracy for the largest singular value)
double spectral_norm_dev(spq_ctx* c, const double* X, int rows, int cols, int ldx) {
  if ((int64_t)rows * cols == 0) return 0.0;
  const int g = std::min(rows, cols);
  double* G = dalloc(c, (size_t)g * g * sizeof(double));
  double* Xt = nullptr;
  GemmBatch gb;
  if (cols <= rows) {   // X^T X
    gb.add(X, ldx, X, ldx, G, g, g, g, rows, 1.0, 0.0);
  } else {              // X X^T = (X^T)^T (X^T)
    Xt = dalloc(c, (size_t)rows * cols * sizeof(double));
    CopyBatch cb;
    CopyTask x{};
    x.src = X; x.dst = Xt; x.nr = rows; x.nc = cols; x.lds = ldx; x.ldd = cols; x.trans = 1;
    cb.add(x);
    cb.run(c);
    gb.add(Xt, cols, Xt, cols, G, g, g, g, cols, 1.0, 0.0);
  }
  gb.run(c, true, 2.0 * g * g * (double)std::max(rows, cols));
  double smax, smin;
  jacobi_extremes(c, G, g, g, g, &smax, &smin);
  dfree(c, G);
  if (Xt) dfree(c, Xt);
  return std::sqrt(smax);
}

void do_sparsify_seq(spq_ctx* c, int p, double eps, int mode, bool scaled_now,
                     SparsifyOut& out) {
  Stage stage_(c, "do_sparsify_seq");
  HostTimer ht(&c->host_ms[8]);
  const std::vector<int64_t> rows_p = c->rows_of[p], cols_p = c->cols_of[p];
  const int np = (int)cols_p.size();
  out = SparsifyOut{-1, np, 0.0, 0};
  if (np == 0) return;
  std::vector<int> us, cs, hu, wc;
  for (int u : c->cix[p]) if (u != p) us.push_back(u);
  for (int cc : c->rix[p]) if (cc != p) cs.push_back(cc);
  int nu = 0, ncl = 0;
  for (int u : us) { hu.push_back(find_block(c, u, p)->nr); nu += hu.back(); }
  for (int cc : cs) { wc.push_back(find_block(c, p, cc)->nc); ncl += wc.back(); }
  const size_t pp = (size_t)np * np;
  // ---- operands: A_pp (np x np), A_np^T (np x nu), A_pn (np x ncl); col-major
  double* App = dalloc(c, std::max<size_t>(pp, 1) * sizeof(double));
  double* AnpT = dalloc(c, std::max<size_t>((size_t)np * nu, 1) * sizeof(double));
  double* Apn = dalloc(c, std::max<size_t>((size_t)np * ncl, 1) * sizeof(double));
  {
    CopyBatch g;
    Block* bp = find_block(c, p, p);
    if (bp && bp->nr == np && bp->nc == np) {
      CopyTask x{};
      x.src = bp->p; x.dst = App; x.nr = np; x.nc = np; x.lds = np; x.ldd = np;
      g.add(x);
    } else {
      g.zero(App, (int64_t)pp);   // a missing block reads as zeros (factor.py:389-392)
    }
    int off = 0;
    for (size_t q = 0; q < us.size(); ++q) {
      Block* b = find_block(c, us[q], p);
      CopyTask x{};
      x.src = b->p; x.dst = AnpT + (int64_t)off * np; x.nr = b->nr; x.nc = np; x.lds = b->nr;
      x.ldd = np; x.trans = 1;
      g.add(x);
      off += b->nr;
    }
    off = 0;
    for (size_t q = 0; q < cs.size(); ++q) {
      Block* b = find_block(c, p, cs[q]);
      CopyTask x{};
      x.src = b->p; x.dst = Apn + (int64_t)off * np; x.nr = np; x.nc = b->nc; x.lds = np;
      x.ldd = np;
      g.add(x);
      off += b->nc;
    }
    g.run(c);
  }
  // ---- compression target M (factor.py:536-567)
  int mcols = 0;
  double* M = nullptr;
  if (mode == SPM_VARIANT1) {
    mcols = nu;
    M = AnpT;
  } else if (mode == SPM_VARIANT2) {
    // M = [sum_{r in col_index[p] & col_index[c]} A_rp^T A_rc  for c in c_list]
    mcols = ncl;
    M = dalloc(c, std::max<size_t>((size_t)np * ncl, 1) * sizeof(double));
    CopyBatch z;
    z.zero(M, (int64_t)np * ncl);
    z.run(c);
    int off = 0;
    for (size_t q = 0; q < cs.size(); ++q) {
      const int cc = cs[q];
      for (int r : c->cix[p]) {
        Block* brc = find_block(c, r, cc);
        if (!brc) continue;
        Block* brp = find_block(c, r, p);
        GemmBatch gb;
        gb.add(brp->p, brp->nr, brc->p, brc->nr, M + (int64_t)off * np, np, np, brc->nc, brp->nr,
               1.0, 1.0);
        gb.run(c, true, 2.0 * np * brc->nc * (double)brp->nr);
      }
      off += wc[q];
    }
  } else if (scaled_now) {
    mcols = nu + ncl;
    M = dalloc(c, std::max<size_t>((size_t)np * mcols, 1) * sizeof(double));
    CopyBatch g;
    CopyTask x{};
    x.src = AnpT; x.dst = M; x.nr = np; x.nc = nu; x.lds = np; x.ldd = np;
    g.add(x);
    x.src = Apn; x.dst = M + (int64_t)nu * np; x.nc = ncl;
    g.add(x);
    g.run(c);
  } else {
    // sigma-weighted route: sigma_min of [A_pp; A_np] from the R of its QR
    const int ms = np + nu;
    double* CS = dalloc(c, ((size_t)ms * np + 2 * pp + np) * sizeof(double));
    double* Rcs = CS + (size_t)ms * np;
    double* tcs = Rcs + pp;
    double* Tcs = tcs + np;
    CopyBatch g;
    g.zero(Rcs, (int64_t)(2 * pp + np));
    CopyTask x{};
    x.src = App; x.dst = CS; x.nr = np; x.nc = np; x.lds = np; x.ldd = ms;
    g.add(x);
    x.src = AnpT; x.dst = CS + np; x.nr = np; x.nc = nu; x.lds = np; x.ldd = ms; x.trans = 1;
    g.add(x);
    g.run(c);
    qr_batch(c, {QrProb{CS, ms, np, Rcs, tcs, Tcs, {}}});
    double smax, smin;
    jacobi_extremes(c, Rcs, np, np, np, &smax, &smin);
    dfree(c, CS);
    if (smin <= SIGMA_FLOOR * std::max(smax, 1e-300)) {
      char fl[64];
      snprintf(fl, sizeof fl, "%.17g", SIGMA_FLOOR * smax);
      throw SpqError(SPQ_ERR_ILL_CONDITIONED, fl, p, smin);
    }
    const double sigma = 1.0 / smin;
    mcols = nu + ncl;
    M = dalloc(c, std::max<size_t>((size_t)np * mcols, 1) * sizeof(double));
    CopyBatch g2;
    CopyTask y{};
    y.src = AnpT; y.dst = M; y.nr = np; y.nc = nu; y.lds = np; y.ldd = np;
    g2.add(y);
    g2.run(c);
    GemmBatch gb;   // sigma * A_pp^T A_pn
    gb.add(App, np, Apn, np, M + (int64_t)nu * np, np, np, ncl, np, sigma, 0.0);
    gb.run(c, true, 2.0 * np * ncl * (double)np);
  }
  // ---- threshold CPQR (scaled: column filter; unscaled: full target)
  const int kmax = std::min(np, mcols);
  const int rank_max = kmax;
  const size_t msz = (size_t)np * std::max(mcols, 1);
  double* Wm = dalloc(c, msz * sizeof(double));
  double* sq = dalloc(c, std::max(mcols, 1) * sizeof(double));
  int* keep = (int*)dalloc(c, std::max(mcols, 1) * sizeof(int));
  int* perm = (int*)dalloc(c, std::max(mcols, 1) * sizeof(int));
  const int k1 = std::max(kmax, 1);
  double* Vq = dalloc(c, ((size_t)np * k1 + 2 * (size_t)k1) * sizeof(double));
  double* tq = Vq + (size_t)np * k1;
  double* bq = tq + k1;
  SpScal* dsc = (SpScal*)dalloc(c, sizeof(SpScal));
  auto cpqr = [&](int min_rank) {
    CopyBatch z;
    z.zero(Vq, (int64_t)np * k1 + 2 * k1);
    z.run(c);
    {
      Scope s(c, F_CPQR);
      launch_sparsify_prep(M, np, mcols, eps, sq, keep, &dsc->nk, &dsc->ratio, &dsc->maxcol, Wm,
                           c->st, scaled_now ? 1 : 0);
      c->tm.launches[F_CPQR] += 3;
      c->n_kernels += 3;
    }
    SpScal h{};
    CUDA_TRY(cudaMemcpyAsync(&h, dsc, sizeof(SpScal), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    CpqrJob q{};
    q.W = Wm; q.m = np; q.n = mcols; q.ncap = std::max(h.nk, 1); q.ldw = np;
    q.nk = &dsc->nk; q.eps = &dsc->ratio; q.min_rank = std::min(min_rank, kmax); q.V = Vq;
    q.ldv = np; q.tau = tq; q.beta = bq; q.rank = &dsc->rank; q.perm = perm; q.write_back = 0;
    if (mcols > 0) run_cpqr_jobs(c, {q});
    else CUDA_TRY(cudaMemsetAsync(&dsc->rank, 0, sizeof(int), c->st));
    CUDA_TRY(cudaMemcpyAsync(&h, dsc, sizeof(SpScal), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    const double mm = np, nn = h.nk, rr = h.rank;
    c->tm.flops[F_CPQR] += 4.0 * mm * nn * rr - 2.0 * rr * rr * (mm + nn) + 4.0 * rr * rr * rr / 3.0;
    c->tm.bytes[F_CPQR] += 16.0 * mm * nn;
    return h.rank;
  };
  int r = cpqr(0);
  auto free_all = [&]() {
    for (void* q : {(void*)App, (void*)AnpT, (void*)Apn, (void*)Wm, (void*)sq, (void*)keep,
                    (void*)perm, (void*)Vq, (void*)dsc})
      dfree(c, q);
    if (M && M != AnpT) dfree(c, M);
  };
  out.rank = r;
  CopyBatch sc;            // split-back copies, in order
  std::vector<std::pair<int, int>> drops;
  auto put_new = [&](int i, int j, int nr, int nc, const double* src, int lds, bool trans) {
    Block* old = find_block(c, i, j);
    if (old) release_mem(c, *old);
    if ((int64_t)nr * nc <= 0) {
      drop_block(c, i, j);
      return;
    }
    double* mem = new_block_mem(c, nr, nc);
    CopyTask x{};
    x.src = src; x.dst = mem; x.lds = lds;
    if (trans) { x.nr = nc; x.nc = nr; x.ldd = nr; x.trans = 1; }
    else { x.nr = nr; x.nc = nc; x.ldd = nr; }
    sc.add(x);
    Block& b = put_block(c, i, j, mem, nr, nc);
    b.clean = false;            // values of a new rotation: flags read back on demand
    b.unverified = false;
    b.flags.clear();
  };
  auto drop_all = [&]() {
    drop_block(c, p, p);
    for (int u : us) drop_block(c, u, p);
    for (int cc : cs) drop_block(c, p, cc);
  };
  Record rec;
  rec.kind = REC_SPARSIFY;
  rec.cid = p;
  rec.rows = rows_p;
  rec.cols_s = cols_p;
  if (scaled_now) {
    // ---------------- scaled apply (factor.py:627-658) on [A_np^T, A_pn]
    if (r >= np) { free_all(); return; }
    double* X = dalloc(c, std::max<size_t>((size_t)np * (nu + ncl), 1) * sizeof(double));
    {
      CopyBatch g;
      CopyTask x{};
      x.src = AnpT; x.dst = X; x.nr = np; x.nc = nu; x.lds = np; x.ldd = np;
      g.add(x);
      x.src = Apn; x.dst = X + (int64_t)nu * np; x.nc = ncl;
      g.add(x);
      g.run(c);
    }
    const int rk = std::max(r, 1);
    rec.m = np; rec.k = r; rec.rank = r;
    rec.payload = dalloc(c, ((size_t)np * rk + 2 * (size_t)rk + (size_t)rk * rk) * sizeof(double));
    rec.V = rec.payload; rec.tau = rec.V + (size_t)np * rk; rec.T = rec.tau + rk;
    {
      CopyBatch g;
      g.zero(rec.T, (int64_t)rk * rk);
      CopyTask x{};
      x.src = Vq; x.dst = rec.V; x.nr = np; x.nc = r; x.lds = np; x.ldd = np;
      g.add(x);
      x.src = tq; x.dst = rec.tau; x.nr = r; x.nc = 1; x.lds = r; x.ldd = r;
      g.add(x);
      g.run(c);
    }
    if (r > 0) {
      build_full_T(c, {TProb{rec.V, np, r, rec.tau, rec.T}});
      wy_batch(c, {WyProb{rec.V, rec.T, np, r, X, np, nu + ncl}}, true);
    }
    rec.full_T = true;
    rec.payload_scalars = (int64_t)np * r + r + (int64_t)r * r;
    const double e1 = spectral_norm_dev(c, X + r, np - r, nu, np);
    const double e2 = spectral_norm_dev(c, X + r + (int64_t)nu * np, np - r, ncl, np);
    out.dropped = std::max(e1, e2);
    int off = 0;
    for (size_t q = 0; q < us.size(); ++q) {   // (u,p) <- (X[:r, u cols])^T
      put_new(us[q], p, hu[q], r, X + (int64_t)off * np, np, true);
      off += hu[q];
    }
    for (size_t q = 0; q < cs.size(); ++q) {   // (p,c) <- X[:r, c cols]
      put_new(p, cs[q], r, wc[q], X + (int64_t)off * np, np, false);
      off += wc[q];
    }
    {
      Block* dp = find_block(c, p, p);
      if (dp) release_mem(c, *dp);
      if (r > 0) {
        double* mem = new_block_mem(c, r, r);
        CopyTask x{};
        x.dst = mem; x.nr = r; x.nc = r; x.ldd = r; x.ident = 1;
        sc.add(x);
        Block& b = put_block(c, p, p, mem, r, r);
        set_identity_flags(c, b, r);
      } else {
        drop_all();
      }
    }
    for (int i = r; i < np; ++i) c->row_of_col[cols_p[i]] = rows_p[i];
    c->rows_of[p].assign(rows_p.begin(), rows_p.begin() + r);
    c->cols_of[p].assign(cols_p.begin(), cols_p.begin() + r);
    sc.run(c);
    c->recs.push_back(std::move(rec));
    out.done = 1;
    dfree(c, X);
    free_all();
    flush_deferred(c);
    return;
  }
  // ---------------- unscaled apply with rank escalation (factor.py:660-709)
  const bool enforce = mode == SPM_SCALED || mode == SPM_UNSCALED;
  double* G = dalloc(c, std::max<size_t>(pp, 1) * sizeof(double));
  double* Gt = dalloc(c, std::max<size_t>(pp, 1) * sizeof(double));
  double* ApnT = dalloc(c, std::max<size_t>((size_t)np * ncl, 1) * sizeof(double));
  double* Tq = dalloc(c, (size_t)k1 * k1 * sizeof(double));
  double* Rff = dalloc(c, (std::max<size_t>(pp, 1) * 2 + np) * sizeof(double));
  double* Tf = Rff + pp;
  double* tf = Tf + pp;
  double nrm_fn = 0.0;
  int f = 0;
  for (;;) {
    f = np - r;
    if (f == 0) {   // factor.py:665-666: every direction coarse, no transform
      for (void* q : {(void*)G, (void*)Gt, (void*)ApnT, (void*)Tq, (void*)Rff}) dfree(c, q);
      free_all();
      out.rank = r;
      return;
    }
    CopyBatch g;
    g.zero(Tq, (int64_t)k1 * k1);
    g.zero(Rff, (int64_t)2 * pp + np);
    CopyTask x{};
    x.src = App; x.dst = Gt; x.nr = np; x.nc = np; x.lds = np; x.ldd = np; x.trans = 1;
    g.add(x);   // Gt = A_pp^T
    CopyTask y{};
    y.src = Apn; y.dst = ApnT; y.nr = np; y.nc = ncl; y.lds = np; y.ldd = np;
    g.add(y);
    g.run(c);
    if (r > 0) {   // Gt <- Q^T A_pp^T = (A_pp Q)^T
      build_full_T(c, {TProb{Vq, np, r, tq, Tq}});
      wy_batch(c, {WyProb{Vq, Tq, np, r, Gt, np, np}}, true);
    }
    CopyBatch g2;
    CopyTask z{};
    z.src = Gt; z.dst = G; z.nr = np; z.nc = np; z.lds = np; z.ldd = np; z.trans = 1;
    g2.add(z);   // G = A_pp Q
    g2.run(c);
    // H_f, R_ff = qr_house(G[:, r:]); H_f^T on G[:, :r] and on A_pn
    QrProb qf{G + (int64_t)r * np, np, f, Rff, tf, Tf, {}};
    if (r > 0) qf.targets.push_back(CTarget{G, np, r});
    if (ncl > 0) qf.targets.push_back(CTarget{ApnT, np, ncl});
    qr_batch(c, {qf});
    nrm_fn = spectral_norm_dev(c, ApnT, f, ncl, np);    // ||R_fn||_2, R_fn = (H_f^T A_pn)[:f]
    if (!enforce || nrm_fn <= eps * (1.0 + 1e-8) || r >= rank_max) break;
    r = cpqr(r + 1);                                       // rank escalation (factor.py:676)
  }
  out.rank = r;
  // pivot floor of R_ff (factor.py:677)
  {
    PivotSet ps;
    ps.jobs.push_back(PivotJob{Rff, f, f, 0});
    ps.ctx.push_back("fine block of interface " + std::to_string(p));
    pivot_launch(c, ps);
    pivot_raise(c, ps);
  }
  // A_np Q: (A_np Q)^T = Q^T A_np^T in place of AnpT (factor.py:679-680)
  double* Tqr = Tq;
  if (r > 0) {
    CopyBatch g;
    g.zero(Tq, (int64_t)k1 * k1);
    g.run(c);
    build_full_T(c, {TProb{Vq, np, r, tq, Tq}});
    wy_batch(c, {WyProb{Vq, Tq, np, r, AnpT, np, nu}}, true);
  }
  const double e1 = spectral_norm_dev(c, AnpT + r, f, nu, np);   // E1^T = rows r: of (A_np Q)^T
  out.dropped = std::max(e1, nrm_fn);
  // record: Q panel | H_f panel | R_ff | R_fc
  const int rk = std::max(r, 1);
  const size_t nq = (size_t)np * rk + 2 * (size_t)rk + (size_t)rk * rk;
  const size_t nh = (size_t)np * f + f + (size_t)f * f;
  const size_t nr_ = (size_t)f * f + (size_t)f * rk;
  rec.m = np; rec.k = r; rec.rank = r; rec.unscaled = true; rec.f = f;
  rec.payload = dalloc(c, (nq + nh + nr_) * sizeof(double));
  rec.V = rec.payload; rec.tau = rec.V + (size_t)np * rk; rec.T = rec.tau + 2 * (size_t)rk;
  rec.hV = rec.payload + nq; rec.htau = rec.hV + (size_t)np * f; rec.hT = rec.htau + f;
  rec.R = rec.hT + (size_t)f * f; rec.Rsn = rec.R + (size_t)f * f;
  {
    CopyBatch g;
    g.zero(rec.payload, (int64_t)(nq + nh + nr_));
    g.run(c);
    CopyTask x{};
    x.src = Vq; x.dst = rec.V; x.nr = np; x.nc = r; x.lds = np; x.ldd = np;
    g.add(x);
    x.src = tq; x.dst = rec.tau; x.nr = r; x.nc = 1; x.lds = r; x.ldd = r;
    g.add(x);
    x.src = Tqr; x.dst = rec.T; x.nr = r; x.nc = r; x.lds = r; x.ldd = r;
    g.add(x);
    x.src = G + (int64_t)r * np; x.dst = rec.hV; x.nr = np; x.nc = f; x.lds = np; x.ldd = np;
    g.add(x);
    x.src = tf; x.dst = rec.htau; x.nr = f; x.nc = 1; x.lds = f; x.ldd = f;
    g.add(x);
    x.src = Rff; x.dst = rec.R; x.nr = f; x.nc = f; x.lds = f; x.ldd = f;
    g.add(x);
    x.src = G; x.dst = rec.Rsn; x.nr = f; x.nc = r; x.lds = np; x.ldd = f;   // R_fc = G2[:f, :r]
    g.add(x);
    g.run(c);
    build_full_T(c, {TProb{rec.hV, np, f, rec.htau, rec.hT}});
  }
  rec.n = 0;
  rec.full_T = true;
  rec.payload_scalars = (int64_t)np * r + r + (int64_t)r * r + (int64_t)np * f + f +
                        (int64_t)f * f + (int64_t)f * f + (int64_t)f * r;
  rec.cols_c.assign(cols_p.begin(), cols_p.begin() + r);
  rec.cols_f.assign(cols_p.begin() + r, cols_p.end());
  // split back (factor.py:682-685) and the new diagonal block G2[f:, :r]
  int off = 0;
  for (size_t q = 0; q < us.size(); ++q) {
    put_new(us[q], p, hu[q], r, AnpT + (int64_t)off * np, np, true);
    off += hu[q];
  }
  off = 0;
  for (size_t q = 0; q < cs.size(); ++q) {
    put_new(p, cs[q], r, wc[q], ApnT + f + (int64_t)off * np, np, false);
    off += wc[q];
  }
  if (r > 0) {
    put_new(p, p, r, r, G + f, np, false);
  } else {
    Block* dp = find_block(c, p, p);
    if (dp) release_mem(c, *dp);
    drop_all();
  }
  // fine rows are the first f slots after H_f; they pair with the fine
  // columns (last f slots after the basis rotation), factor.py:690-693
  for (int i = 0; i < f; ++i) c->row_of_col[cols_p[r + i]] = rows_p[i];
  c->rows_of[p].assign(rows_p.begin() + f, rows_p.end());
  c->cols_of[p].assign(cols_p.begin(), cols_p.begin() + r);
  sc.run(c);
  c->recs.push_back(std::move(rec));
  out.done = 1;
  sync(c);   // the scratch below is read by the queued split-back copies
  for (void* q : {(void*)G, (void*)Gt, (void*)ApnT, (void*)Tq, (void*)Rff}) dfree(c, q);
  free_all();
  flush_deferred(c);
}

void do_sparsify(spq_ctx* c, const std::vector<int>& ids, double eps,
                 std::vector<SparsifyOut>& outs, int mode = SPM_SCALED, bool scaled_now = true) {
  outs.assign(ids.size(), SparsifyOut{-1, 0, 0.0, 0});
  if (mode != SPM_SCALED || !scaled_now) {
    // unscaled route / variant targets: the reference's sequential loop
    for (size_t t = 0; t < ids.size(); ++t) {
      if (!c->active[ids[t]]) throw SpqError(SPQ_ERR_BAD_INPUT, "sparsify of inactive cluster");
      do_sparsify_seq(c, ids[t], eps, mode, scaled_now, outs[t]);
    }
    return;
  }
  c->d_dropped = dalloc(c, 2 * std::max<size_t>(ids.size(), 1) * sizeof(double));
  CUDA_TRY(cudaMemsetAsync(c->d_dropped, 0, 2 * std::max<size_t>(ids.size(), 1) * sizeof(double), c->st));
  // Waves of pairwise non-adjacent interfaces (no shared block).  The
  // reference sparsifies in ascending id; two interfaces commute unless
  // they share a block, so each interface goes one wave after the latest
  // EARLIER (in id order) interface adjacent to it: every adjacent pair
  // keeps its order, everything else is batched (fewer waves than a greedy
  // prefix split, hence fewer rank read-backs).  SPQ_SPARSIFY_PREFIX=1:
  // the greedy prefix split.
  const int nid = (int)ids.size();
  std::vector<int> lvl(nid, 0);
  {
    std::unordered_map<int, int> where;
    where.reserve(nid * 2);
    for (int t = 0; t < nid; ++t) where[ids[t]] = t;
    static const bool prefix = env_flag("SPQ_SPARSIFY_PREFIX");
    int cur = 0;
    std::set<int> members;
    for (int t = 0; t < nid; ++t) {
      const int p = ids[t];
      if (!c->active[p]) throw SpqError(SPQ_ERR_BAD_INPUT, "sparsify of inactive cluster");
      int L = 0;
      if (prefix) {
        bool clash = false;
        for (int q : c->cix[p]) if (q != p && members.count(q)) { clash = true; break; }
        if (!clash) for (int q : c->rix[p]) if (q != p && members.count(q)) { clash = true; break; }
        if (clash) { ++cur; members.clear(); }
        members.insert(p);
        L = cur;
      } else {
        auto dep = [&](int q) {
          if (q == p) return;
          auto it = where.find(q);
          if (it != where.end() && it->second < t) L = std::max(L, lvl[it->second] + 1);
        };
        for (int q : c->cix[p]) dep(q);
        for (int q : c->rix[p]) dep(q);
      }
      lvl[t] = L;
    }
  }
  int nlev = 0;
  for (int t = 0; t < nid; ++t) nlev = std::max(nlev, lvl[t] + 1);
  for (int L = 0; L < nlev; ++L) {
    std::vector<int> members_t;
    for (int t = 0; t < nid; ++t) if (lvl[t] == L) members_t.push_back(t);
    size_t pos = 0;
    while (pos < members_t.size()) {   // memory-bounded groups, ascending id
      std::vector<int> wave, didx;
      size_t wave_bytes = 0;
      while (pos < members_t.size()) {
        const int t = members_t[pos];
        const int p = ids[t];
        // device scratch of the job (M and its compacted copy, np x ncols each)
        size_t nc = 0;
        for (int q : c->rix[p]) if (q != p) nc += c->cols_of[q].size();
        for (int q : c->cix[p]) if (q != p) nc += c->rows_of[q].size();
        const size_t est = 2 * sizeof(double) * c->cols_of[p].size() * nc;
        if (!wave.empty() && wave_bytes + est > 4 * chunk_bytes()) break;
        wave_bytes += est;
        wave.push_back(p);
        didx.push_back(t);
        ++pos;
      }
      std::vector<SparsifyOut> wo(wave.size());
      do_sparsify_wave(c, wave, eps, wo, didx);
      for (size_t u = 0; u < wave.size(); ++u) outs[didx[u]] = wo[u];
      c->n_sparsify_waves++;
    }
  }
  // dropped norms of all compressed interfaces: one read at the end
  side_join(c);
  std::vector<double> hd(2 * ids.size());
  CUDA_TRY(cudaMemcpyAsync(hd.data(), c->d_dropped, hd.size() * 8, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  for (size_t t = 0; t < ids.size(); ++t)
    if (outs[t].done) outs[t].dropped = std::max(hd[2 * t], hd[2 * t + 1]);
  dfree(c, c->d_dropped);
  c->d_dropped = nullptr;
}

// ================================================================ (d) merge
void do_merge(spq_ctx* c, int np_, const int32_t* pid, const int32_t* cptr, const int32_t* cid) {
  Stage stage_(c, "do_merge");
  HostTimer ht(&c->host_ms[10]);
  std::vector<int> parent_of(c->ncl, -1), roff(c->ncl, 0), coff(c->ncl, 0);
  std::vector<std::vector<int64_t>> nrows(np_), ncols(np_);
  for (int t = 0; t < np_; ++t) {
    int ro = 0, co = 0;
    for (int q = cptr[t]; q < cptr[t + 1]; ++q) {
      const int k = cid[q];
      if (k < 0 || k >= c->ncl) throw SpqError(SPQ_ERR_BAD_INPUT, "merge: bad child id");
      parent_of[k] = pid[t];
      roff[k] = ro;
      coff[k] = co;
      ro += (int)c->rows_of[k].size();
      co += (int)c->cols_of[k].size();
      nrows[t].insert(nrows[t].end(), c->rows_of[k].begin(), c->rows_of[k].end());
      ncols[t].insert(ncols[t].end(), c->cols_of[k].begin(), c->cols_of[k].end());
    }
  }
  // old blocks in ascending (i, j) key order: the row adjacency lists are
  // sorted by column and carry the block pointers, so walking rows in
  // ascending id yields the sorted key list without a sort.  Any mismatch
  // with the map (a list entry without its block) falls back to sorting.
  std::vector<std::pair<uint64_t, Block*>> keys;   // (key, block): no lookups below
  keys.reserve(c->blk.size());
  for (int i = 0; i < c->ncl; ++i) {
    const FlatSet& row = c->rix[i];
    for (size_t t = 0; t < row.v.size(); ++t) keys.push_back({bkey(i, row.v[t]), row.b[t]});
  }
  if (keys.size() != c->blk.size()) throw SpqError(SPQ_ERR_INTERNAL, "merge: adjacency lists and block count disagree");
  for (auto& kb : keys)
    if (!kb.second) throw SpqError(SPQ_ERR_INTERNAL, "merge: adjacency entry without a block");
  BlockMap old;   // the children's Block objects stay alive (their pool) until the copies are planned
  old.swap(c->blk);
  for (int s = 0; s < c->ncl; ++s) {
    if (c->active[s]) { c->rows_of[s].clear(); c->cols_of[s].clear(); }
    c->active[s] = 0;
    c->rix[s].clear();
    c->cix[s].clear();
  }
  for (int t = 0; t < np_; ++t) {
    const int P = pid[t];
    c->rows_of[P] = std::move(nrows[t]);
    c->cols_of[P] = std::move(ncols[t]);
    c->active[P] = 1;
  }
  CopyBatch zeros, cp;
  // parent blocks needed, grouped by parent row: one zeroed allocation per row
  std::vector<std::vector<int>> prow_v(c->ncl);   // Pi -> Pj list
  for (auto& kb : keys) {
    const uint64_t key = kb.first;
    Block& B = *kb.second;
    if ((int64_t)B.nr * B.nc == 0) continue;
    const int i = (int)(key >> 32), j = (int)(key & 0xffffffffu);
    const int Pi = parent_of[i], Pj = parent_of[j];
    if (Pi < 0 || Pj < 0) throw SpqError(SPQ_ERR_BAD_INPUT, "merge: block of unmerged cluster");
    prow_v[Pi].push_back(Pj);
  }
  size_t nparent_blocks = 0;
  for (auto& v : prow_v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    nparent_blocks += v.size();
  }
  c->blk.reserve(nparent_blocks * 2 + 16);
  // old blocks by parent row; a shared slab only ever holds blocks of one
  // row cluster, so releasing a parent row's children frees whole slabs
  std::vector<std::vector<std::pair<uint64_t, Block*>>> by_prow(c->ncl);
  for (auto& kb : keys) {
    Block& B = *kb.second;
    if ((int64_t)B.nr * B.nc == 0) { release_mem(c, B); continue; }
    by_prow[parent_of[(int)(kb.first >> 32)]].push_back(kb);
  }
  flush_deferred(c);
  // parent rows in groups of bounded new storage: allocate + zero the
  // group's slabs, copy its children in, release them (reused by the next
  // group in stream order) -- the transient is one group, not the level
  const size_t budget = 4 * chunk_bytes();
  int Pi = 0;
  while (Pi < c->ncl) {
    CopyBatch zeros, cp;
    size_t group = 0;
    const int g0 = Pi;
    for (; Pi < c->ncl; ++Pi) {
      auto& v = prow_v[Pi];
      if (v.empty()) continue;
      const int R = (int)c->rows_of[Pi].size();
      size_t tot = 0;
      for (int Pj : v) tot += (size_t)R * c->cols_of[Pj].size();
      if (Pi > g0 && group > 0 && (group + tot) * sizeof(double) > budget) break;
      group += tot;
      double* slab = shared_alloc(c, tot, (int)v.size());
      zeros.zero(slab, (int64_t)tot);
      size_t off = 0;
      for (int Pj : v) {
        const int C = (int)c->cols_of[Pj].size();
        Block& nb = put_block_new(c, Pi, Pj, slab + off, R, C, slab);   // the lists were cleared: every parent key is new
        // merged values are copies: the parent's row flags are the OR of its
        // children's (exact given theirs; unverified if any child is)
        if (c->spec) nb.flags.assign(R, 0);
        else nb.flags.clear();
        nb.clean = c->spec;
        nb.unverified = false;
        nb.origin = 7;
        off += (size_t)R * C;
      }
    }
    {
      size_t ncp = 0;
      for (int q = g0; q < Pi; ++q) ncp += by_prow[q].size();
      cp.reserve(ncp);
    }
    for (int q = g0; q < Pi; ++q)
      for (auto& kb : by_prow[q]) {
        const uint64_t key = kb.first;
        Block& B = *kb.second;
        const int i = (int)(key >> 32), j = (int)(key & 0xffffffffu);
        const int Pj = parent_of[j];
        Block* tgt = find_block(c, q, Pj);
        const int R = (int)c->rows_of[q].size();
        CopyTask x{};
        x.src = B.p; x.dst = tgt->p + roff[i] + (int64_t)coff[j] * R; x.nr = B.nr; x.nc = B.nc;
        x.lds = B.nr; x.ldd = R;
        cp.add(x);
        if (tgt->clean) {
          if (B.clean && B.flags.size() == (size_t)B.nr) {
            {   // clean flags are 0/1: a byte-wise OR (vectorised) instead of a branch per row
              const uint8_t* src = B.flags.begin();
              uint8_t* dst = &tgt->flags[roff[i]];
              for (int t = 0; t < B.nr; ++t) dst[t] |= (uint8_t)(src[t] & 1);
            }
            if (B.unverified && !tgt->unverified) tgt->origin = (uint8_t)(10 + B.origin % 10);
            tgt->unverified = tgt->unverified || B.unverified;
          } else {
            tgt->clean = false;
            tgt->unverified = false;
            tgt->flags.clear();
          }
        }
        release_mem(c, B);
      }
    zeros.run(c);
    cp.run(c);
    flush_deferred(c);
  }
}

// ================================================================== load
void do_load(spq_ctx* c, int64_t N, const int64_t* indptr, const int64_t* indices,
             const double* data, int equilibrate, int ncl, int nleaf, const int32_t* leaf_ids,
             const int64_t* rptr, const int64_t* rows, const int64_t* cptr, const int64_t* cols) {
  Stage stage_(c, "do_load");
  c->N = N;
  c->ncl = ncl;
  c->rows_of.assign(ncl, {});
  c->cols_of.assign(ncl, {});
  c->active.assign(ncl, 0);
  c->rix.assign(ncl, {});
  c->cix.assign(ncl, {});
  c->row_of_col.assign(N, -1);
  const int64_t nnz = indptr[N];
  for (int64_t j = 0; j < N; ++j) {
    bool nz = false;   // the column's squared norm is positive (same products as the device sum)
    for (int64_t e = indptr[j]; e < indptr[j + 1]; ++e) {
      if (indices[e] < 0 || indices[e] >= N) throw SpqError(SPQ_ERR_BAD_INPUT, "row index out of range");
      if (e > indptr[j] && indices[e] <= indices[e - 1])
        throw SpqError(SPQ_ERR_BAD_INPUT, "CSC row indices must be strictly increasing per column");
      nz = nz || data[e] * data[e] > 0.0;
    }
    // sparse.py:158-166: a zero column cannot be equilibrated.  Decided on the
    // host (no read-back of the device's column norms: the load used to end
    // with a stream synchronization for this one integer)
    if (equilibrate && !nz)
      throw SpqError(SPQ_ERR_BAD_INPUT, "cannot equilibrate: column " + std::to_string(j) + " has zero norm");
  }
  std::vector<int> rown(N, -1), coln(N, -1), rpos(N), cpos(N);
  for (int t = 0; t < nleaf; ++t) {
    const int id = leaf_ids[t];
    if (id < 0 || id >= ncl) throw SpqError(SPQ_ERR_BAD_INPUT, "leaf id out of range");
    c->rows_of[id].assign(rows + rptr[t], rows + rptr[t + 1]);
    c->cols_of[id].assign(cols + cptr[t], cols + cptr[t + 1]);
    c->active[id] = 1;
    for (size_t i = 0; i < c->rows_of[id].size(); ++i) {
      rown[c->rows_of[id][i]] = id;
      rpos[c->rows_of[id][i]] = (int)i;
    }
    for (size_t i = 0; i < c->cols_of[id].size(); ++i) {
      coln[c->cols_of[id][i]] = id;
      cpos[c->cols_of[id][i]] = (int)i;
    }
  }
  for (int64_t i = 0; i < N; ++i)
    if (rown[i] < 0 || coln[i] < 0) throw SpqError(SPQ_ERR_BAD_INPUT, "leaf clusters do not cover all rows/columns");
  // block structure of the entries
  FlatMap<int> bidx;
  std::vector<std::pair<int, int>> bkeys;
  std::vector<int> eb(nnz);
  std::vector<int64_t> eoff(nnz);
  uint64_t last_key = ~0ull;
  int last_b = -1;
  for (int64_t j = 0; j < N; ++j) {
    const int cj = coln[j];
    for (int64_t e = indptr[j]; e < indptr[j + 1]; ++e) {
      const int64_t r = indices[e];
      const int ri = rown[r];
      const uint64_t key = bkey(ri, cj);
      int b;
      if (key == last_key) {   // runs of entries of one block: no probe
        b = last_b;
      } else {
        const int* hit = bidx.find(key);
        if (!hit) {
          b = (int)bkeys.size();
          bidx[key] = b;
          bkeys.push_back({ri, cj});
        } else {
          b = *hit;
        }
        last_key = key;
        last_b = b;
      }
      eb[e] = b;
      eoff[e] = rpos[r] + (int64_t)cpos[j] * (int64_t)c->rows_of[ri].size();
    }
  }
  std::vector<double*> bases(bkeys.size());
  CopyBatch zeros;
  for (size_t b = 0; b < bkeys.size(); ++b) {
    const int i = bkeys[b].first, j = bkeys[b].second;
    const int nr = (int)c->rows_of[i].size(), nc = (int)c->cols_of[j].size();
    double* mem = new_block_mem(c, nr, nc);
    zeros.zero(mem, (int64_t)nr * nc);
    Block& B = put_block_new(c, i, j, mem, nr, nc);   // bkeys are unique
    B.clean = false;
    bases[b] = mem;
  }
  // exact initial row flags from the stored values (equilibration divides
  // by positive norms: zero stays zero, nonzero stays nonzero)
  if (c->spec) {
    std::vector<Block*> bp(bkeys.size());
    for (size_t b = 0; b < bkeys.size(); ++b) {
      bp[b] = find_block(c, bkeys[b].first, bkeys[b].second);
      bp[b]->flags.assign(bp[b]->nr, 0);
      bp[b]->clean = true;
      bp[b]->unverified = true;
      bp[b]->origin = 8;
    }
    for (int64_t j = 0; j < N; ++j)
      for (int64_t e = indptr[j]; e < indptr[j + 1]; ++e)
        if (data[e] != 0.0) bp[eb[e]]->flags[rpos[indices[e]]] = 1;
  }
  zeros.run(c);
  // CSC arrays and the per-entry block map through the pinned upload ring: a
  // host memcpy into pinned memory plus an asynchronous DMA each, instead of
  // pageable cudaMemcpyAsync calls (staged synchronously, ~8 MB at C3)
  int64_t* d_indptr = upload(c, indptr, (size_t)N + 1);
  double* d_data = nnz ? upload(c, data, (size_t)nnz) : dalloc(c, sizeof(double));
  c->equil = equilibrate != 0;
  c->d_scale = dalloc(c, N * sizeof(double));
  int* d_zero = (int*)dalloc(c, sizeof(int));
  const int big = 0x7fffffff;
  CUDA_TRY(cudaMemcpyAsync(d_zero, &big, sizeof(int), cudaMemcpyHostToDevice, c->st));
  {
    Scope s(c, F_COPY);
    launch_colnorms_scale(d_indptr, nullptr, d_data, N, c->d_scale, d_zero, equilibrate, c->st);
    if (nnz) {
      int64_t* d_off = upload(c, eoff);
      int* d_eb = upload(c, eb);
      double** d_bases = upload(c, bases);
      launch_csc_scatter(d_indptr, nullptr, d_data, nnz, d_off, d_bases, d_eb, c->st);
    }
  }
  if (!nnz) dfree(c, d_data);
  dfree(c, d_zero);
}

// ================================================================ chains
void ensure_chain_scratch(spq_ctx* c, int nrhs) {
  size_t maxk = 1, maxp = 1;
  for (auto& r : c->recs) {
    maxk = std::max<size_t>(maxk, (size_t)std::max(r.k, r.m));
    maxp = std::max<size_t>(maxp, (size_t)chain_rsn_chunks(r.n) * std::max(r.k, 1));
    if (r.unscaled)   // TRI op with R_ff (f x f) and R_fc (f x rank)
      maxp = std::max<size_t>(maxp, (size_t)chain_rsn_chunks(r.k) * std::max(r.f, 1));
  }
  const size_t vneed = (size_t)c->N * nrhs;
  if (vneed > c->vec_cap) {
    for (auto& P : c->prog) {
      for (auto& kv : P.graphs) cudaGraphExecDestroy(kv.second);
      P.graphs.clear();
    }
    dfree(c, c->d_vec);
    dfree(c, c->d_vec2);
    c->d_vec = dalloc(c, vneed * sizeof(double));
    c->d_vec2 = dalloc(c, vneed * sizeof(double));
    c->vec_cap = vneed;
  }
  if (maxk * nrhs > c->w_cap) {
    dfree(c, c->d_w);
    dfree(c, c->d_w2);
    c->d_w = dalloc(c, maxk * nrhs * sizeof(double));
    c->d_w2 = dalloc(c, maxk * nrhs * sizeof(double));
    c->w_cap = maxk * nrhs;
  }
  if (maxp * nrhs > c->part_cap) {
    dfree(c, c->d_part);
    c->d_part = dalloc(c, maxp * nrhs * sizeof(double));
    c->part_cap = maxp * nrhs;
  }
}

// ---------------------------------------------------- chain programs (e)
// Record operations in chain order grouped into waves of mutually
// independent ops (no op writes an index another op of the wave reads or
// writes): one launch per wave, one CTA per op.
void build_prog(spq_ctx* c, int which, const std::vector<ChainOp>& ops,
                const std::vector<std::vector<int>>& wr, const std::vector<std::vector<int>>& rd) {
  auto& P = c->prog[which];
  // dependency levels: an op goes one wave after the latest earlier op it
  // conflicts with (read-after-write, write-after-read, write-after-write on
  // any index); ops of one level commute, so the chain is applied level by
  // level -- the critical path of the record DAG, not a greedy in-order split
  std::vector<int> lw(c->N, -1), lr(c->N, -1), lev(ops.size(), 0);
  int nlev = 0;
  for (size_t t = 0; t < ops.size(); ++t) {
    int L = 0;
    for (int i : wr[t]) L = std::max(L, std::max(lw[i], lr[i]) + 1);
    for (int i : rd[t]) L = std::max(L, lw[i] + 1);
    for (int i : wr[t]) lw[i] = L;
    for (int i : rd[t]) lr[i] = std::max(lr[i], L);
    lev[t] = L;
    nlev = std::max(nlev, L + 1);
  }
  std::vector<ChainOp> ordered;
  P.off.clear(); P.cnt.clear(); P.kmax.clear();
  {
    std::vector<std::vector<int>> by(nlev);
    for (size_t t = 0; t < ops.size(); ++t) by[lev[t]].push_back((int)t);
    for (int L = 0; L < nlev; ++L) {
      P.off.push_back((int)ordered.size());
      P.cnt.push_back(0);
      P.kmax.push_back(0);
      for (int t : by[L]) {
        ordered.push_back(ops[t]);
        P.cnt.back()++;
        P.kmax.back() = std::max(P.kmax.back(), ops[t].k);
      }
    }
  }
  // chunking: per wave, the operations split into chunks so the wave fills
  // ~4 CTAs per SM (the chain is latency-bound wave by wave), at least 32
  // rows (WY) / columns (R_sn) per chunk
  std::vector<int2> tasks;
  P.toff.clear(); P.tcnt.clear(); P.part_sz.clear(); P.slabk.clear(); P.has_wy.clear();
  size_t scr = 0;
  for (size_t w = 0; w < P.off.size(); ++w) {
    double wave_work = 0;
    for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
      const ChainOp& o = ordered[t];
      const bool wy = o.kind == CH_WY_T || o.kind == CH_WY_N;
      const int64_t len = wy ? o.m : (o.kind == CH_TRI_MUL ? (int64_t)o.k + o.n : (int64_t)o.n + o.n2);
      wave_work += (double)std::max<int64_t>(len, 1) * std::max(o.k, 1);
    }
    static const int min_chunk = std::max(8, getenv("SPQ_CHAIN_MINCHUNK") ? atoi(getenv("SPQ_CHAIN_MINCHUNK")) : 32);
    const double per_cta = std::max(64.0 * min_chunk, wave_work / (4.0 * c->nsm));
    for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
      ChainOp& o = ordered[t];
      const bool wy = o.kind == CH_WY_T || o.kind == CH_WY_N;
      // the dimension that is split: WY rows; TRI_MUL the columns of [R | R_sn];
      // TRI_SOLVE the R_sn columns (the back substitution stays in one CTA)
      const int64_t len = wy ? o.m : (o.kind == CH_TRI_MUL ? (int64_t)o.k + o.n : (int64_t)o.n + o.n2);
      const double work = (double)std::max(len, (int64_t)1) * std::max(o.k, 1);
      int64_t nch = (int64_t)std::ceil(work / per_cta);
      nch = std::max<int64_t>(1, std::min<int64_t>(nch, (len + min_chunk - 1) / min_chunk));
      nch = std::min<int64_t>(nch, 512);
      if (!wy && len == 0) nch = 1;
      o.per = (int)std::max<int64_t>(1, (len + nch - 1) / nch);
      o.nchunk = (int)std::max<int64_t>(1, (len + o.per - 1) / o.per);
      if ((size_t)2 * o.k * sizeof(double) > CHAIN_SMEM_MAX) scr += 3 * (size_t)o.k * o.nchunk;
    }
  }
  if (scr) {   // ops too large for shared memory: private global scratch per chunk
    double* base = dalloc(c, scr * sizeof(double));
    size_t off = 0;
    for (auto& o : ordered)
      if ((size_t)2 * o.k * sizeof(double) > CHAIN_SMEM_MAX) {
        o.scratch = base + off;
        off += 3 * (size_t)o.k * o.nchunk;
      }
  }
  // arrival counters of the WY operations (reset by the last chunk)
  int* cnts = ordered.empty() ? nullptr : (int*)dalloc(c, ordered.size() * sizeof(int));
  if (cnts) CUDA_TRY(cudaMemsetAsync(cnts, 0, ordered.size() * sizeof(int), c->st));
  for (size_t w = 0; w < P.off.size(); ++w) {
    int km = 0;
    int64_t psz = 0;
    P.toff.push_back((int)tasks.size());
    for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
      ChainOp& o = ordered[t];
      if (!o.scratch) km = std::max(km, o.k);
      o.part_off = psz;
      psz += (int64_t)o.nchunk * std::max(o.k, 1);
      o.cnt = cnts + t;
      for (int q = 0; q < o.nchunk; ++q) tasks.push_back(make_int2(t - P.off[w], q));
    }
    for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {   // reduced vectors after the partials
      ChainOp& o = ordered[t];
      o.u_off = psz;
      psz += 2 * (int64_t)std::max(o.k, 1);
    }
    P.tcnt.push_back((int)tasks.size() - P.toff.back());
    P.kmax[w] = km;
    int sk = 0;   // TRI_SOLVE ops whose R slabs stream through shared memory
    char wy_any = 0;
    for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t)
      if (ordered[t].kind == CH_WY_T || ordered[t].kind == CH_WY_N) wy_any = 1;
    P.has_wy.push_back(wy_any);
    for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
      const ChainOp& o = ordered[t];
      if (o.kind == CH_TRI_SOLVE && !o.scratch && o.k > 32 && o.k <= CHAIN_SLAB_KMAX) sk = std::max(sk, o.k);
    }
    if ((size_t)(2 * std::max(km, sk) + 64 * sk) * sizeof(double) > CHAIN_SMEM_MAX) sk = 0;
    P.slabk.push_back(sk);
    P.part_sz.push_back(psz);
  }
  // inverse diagonal blocks for the slab-streamed back substitutions
  bool any_dinv = false;
  if (!env_flag("SPQ_CHAIN_NO_DINV")) {
    size_t nd = 0;
    for (size_t w = 0; w < P.off.size(); ++w)
      for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
        const ChainOp& o = ordered[t];
        if (o.kind == CH_TRI_SOLVE && !o.scratch && o.k > 32 && o.k <= P.slabk[w]) nd += (size_t)((o.k + 31) / 32) * 1024;
      }
    if (nd) {
      double* base = dalloc(c, nd * sizeof(double));
      size_t off = 0;
      for (size_t w = 0; w < P.off.size(); ++w)
        for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
          ChainOp& o = ordered[t];
          if (o.kind == CH_TRI_SOLVE && !o.scratch && o.k > 32 && o.k <= P.slabk[w]) {
            o.Dinv = base + off;
            off += (size_t)((o.k + 31) / 32) * 1024;
          }
        }
      any_dinv = true;
    }
  }
  if (env_flag("SPQ_CHAIN_PROFILE")) P.hops = ordered;
  if (!ordered.empty()) {
    P.d_ops = (ChainOp*)dalloc(c, ordered.size() * sizeof(ChainOp));
    CUDA_TRY(cudaMemcpyAsync(P.d_ops, ordered.data(), ordered.size() * sizeof(ChainOp),
                             cudaMemcpyHostToDevice, c->st));
    P.d_tasks = (int2*)dalloc(c, std::max<size_t>(tasks.size(), 1) * sizeof(int2));
    CUDA_TRY(cudaMemcpyAsync(P.d_tasks, tasks.data(), tasks.size() * sizeof(int2),
                             cudaMemcpyHostToDevice, c->st));
    if (any_dinv) launch_chain_dinv(P.d_ops, (int)ordered.size(), c->st);
    sync(c);
  }
}

// W = V T^T (transposed) or V T for every WY record: the chain update
// becomes z -= W (V^T z) with no triangular product per chunk.  Built with
// the batched DMMA GEMM at chain compile time; skipped (kernels fall back
// to the T path) when the extra payload would not fit comfortably.
constexpr int CHAIN_W_KMIN = 32;   // below: T w in the reducing chunk is cheap (one short pass)
void build_chain_W(spq_ctx* c) {
  const int kmin = env_flag("SPQ_CHAIN_W") ? 1 : CHAIN_W_KMIN;
  size_t need = 0;
  for (auto& r : c->recs)
    if (r.k >= kmin && !r.unscaled) need += (size_t)r.m * r.k * (r.kind == REC_SPARSIFY ? 2 : 1);
  if (need == 0 || env_flag("SPQ_CHAIN_NO_W")) return;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  if (need * sizeof(double) * 3 > fr + arena_free_bytes(c->dev)) return;
  CopyBatch cp;
  GemmBatch gT, gN;
  std::vector<double*> tts;
  for (auto& r : c->recs) {
    if (r.k < kmin || r.unscaled) continue;
    const size_t mk = (size_t)r.m * r.k, kk = (size_t)r.k * r.k;
    const bool sp = r.kind == REC_SPARSIFY;
    r.WT = dalloc(c, mk * sizeof(double));
    double* Tt = dalloc(c, kk * sizeof(double));
    tts.push_back(Tt);
    CopyTask x{};
    x.src = r.T; x.dst = Tt; x.nr = r.k; x.nc = r.k; x.lds = r.k; x.ldd = r.k; x.trans = 1;
    cp.add(x);
    gT.add(r.V, r.m, Tt, r.k, r.WT, r.m, r.m, r.k, r.k, 1.0, 0.0);
    if (sp) {
      r.WN = dalloc(c, mk * sizeof(double));
      gN.add(r.V, r.m, r.T, r.k, r.WN, r.m, r.m, r.k, r.k, 1.0, 0.0);
    }
  }
  cp.run(c);
  gT.run(c, false, 0);
  gN.run(c, false, 0);
  for (double* p : tts) dfree(c, p);
}

void compile_chains(spq_ctx* c) {
  build_chain_W(c);
  std::vector<ChainOp> ops;
  std::vector<std::vector<int>> wr, rd;
  auto to_int = [](const std::vector<int64_t>& v) { return std::vector<int>(v.begin(), v.end()); };
  // apply_qt: every record's panel on its rows, in chain order (an unscaled
  // sparsifier's Q-side is its H_f panel, factor.py:183-186)
  for (auto& r : c->recs) {
    if (r.unscaled) {
      ops.push_back(ChainOp{CH_WY_T, r.m, r.f, 0, r.d_rows, nullptr, r.hV, r.hT, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 1, 1, 0});
      wr.push_back(to_int(r.rows));
      rd.push_back({});
      continue;
    }
    if (r.k <= 0) continue;
    ops.push_back(ChainOp{CH_WY_T, r.m, r.k, 0, r.d_rows, nullptr, r.V, r.T, nullptr, nullptr, nullptr, r.WT, nullptr, 0, 1, 1, 0});
    wr.push_back(to_int(r.rows));
    rd.push_back({});
  }
  build_prog(c, 0, ops, wr, rd);
  // solve_w: reversed W-chain
  ops.clear(); wr.clear(); rd.clear();
  // A back substitution runs in one CTA; R_ss larger than the shared-memory
  // slab limit is split into row blocks from the bottom, each its own op
  // whose product with the already solved unknowns (the columns of R_ss to
  // the right of the block, then R_sn) is spread over many CTAs
  // (SPQ_CHAIN_SPLIT_K=s: split everything larger than s into blocks of s)
  const int split_env = getenv("SPQ_CHAIN_SPLIT_K") ? std::max(32, atoi(getenv("SPQ_CHAIN_SPLIT_K"))) : 0;
  const int split_thr = split_env ? split_env : CHAIN_SLAB_KMAX, split_sz = split_env ? split_env : 256;
  auto push_tri_solve = [&](int k, int n, const int* d_idx, const int* d_idx_n, const double* R,
                            const double* Rsn, const std::vector<int>& cols,
                            const std::vector<int>& cols_n) {
    if (k <= split_thr || env_flag("SPQ_CHAIN_NO_SPLIT")) {
      ops.push_back(ChainOp{CH_TRI_SOLVE, k, k, n, d_idx, d_idx_n, nullptr, nullptr, R, Rsn, nullptr,
                            nullptr, nullptr, 0, 1, 1, 0});
      wr.push_back(cols);
      rd.push_back(cols_n);
      return;
    }
    const int nblk = (k + split_sz - 1) / split_sz;
    const int bs = (((k + nblk - 1) / nblk) + 31) / 32 * 32;
    for (int r1 = k; r1 > 0; r1 -= bs) {
      const int r0 = std::max(0, r1 - bs), kk = r1 - r0;
      ChainOp o{};
      o.kind = CH_TRI_SOLVE;
      o.m = kk; o.k = kk; o.n = n;
      o.idx = d_idx + r0;
      o.idx_n = d_idx_n;
      o.R = R + r0 + (int64_t)r0 * k;
      o.Rsn = Rsn ? Rsn + r0 : nullptr;
      o.nchunk = 1; o.per = 1;
      o.ldr = k; o.ldn = k;
      o.n2 = k - r1;
      o.R2 = R + r0 + (int64_t)r1 * k;
      o.idx2 = d_idx + r1;
      ops.push_back(o);
      wr.push_back(std::vector<int>(cols.begin() + r0, cols.begin() + r1));
      std::vector<int> rdv(cols.begin() + r1, cols.end());
      rdv.insert(rdv.end(), cols_n.begin(), cols_n.end());
      rd.push_back(std::move(rdv));
    }
  };
  for (auto it = c->recs.rbegin(); it != c->recs.rend(); ++it) {
    Record& r = *it;
    if (r.unscaled) {
      // v = y[cols]; v[r:] = R_ff^{-1}(v[r:] - R_fc v[:r]); y[cols] = Q v  (factor.py:195-203)
      push_tri_solve(r.f, r.k, r.d_cols_f, r.d_cols_c, r.R, r.Rsn, to_int(r.cols_f), to_int(r.cols_c));
      if (r.k > 0) {
        ops.push_back(ChainOp{CH_WY_N, r.m, r.k, 0, r.d_cols_s, nullptr, r.V, r.T, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 1, 1, 0});
        wr.push_back(to_int(r.cols_s));
        rd.push_back({});
      }
      continue;
    }
    if (r.kind == REC_SPARSIFY) {
      if (r.k <= 0) continue;
      ops.push_back(ChainOp{CH_WY_N, r.m, r.k, 0, r.d_cols_s, nullptr, r.V, r.T, nullptr, nullptr, nullptr, r.WN, nullptr, 0, 1, 1, 0});
      wr.push_back(to_int(r.cols_s));
      rd.push_back({});
    } else {
      if (r.k <= 0) continue;
      const bool bh = r.kind == REC_ELIM;
      push_tri_solve(r.k, bh ? r.n : 0, r.d_cols_s, bh ? r.d_cols_n : nullptr, r.R,
                     bh ? r.Rsn : nullptr, to_int(r.cols_s),
                     bh ? to_int(r.cols_n) : std::vector<int>());
    }
  }
  build_prog(c, 1, ops, wr, rd);
  // apply_w: forward W-chain (after the diagonal scaling)
  ops.clear(); wr.clear(); rd.clear();
  for (auto& r : c->recs) {
    if (r.unscaled) {
      // v = Q^T x[cols]; v[r:] = R_ff v[r:] + R_fc v[:r]  (factor.py:188-193)
      if (r.k > 0) {
        ops.push_back(ChainOp{CH_WY_T, r.m, r.k, 0, r.d_cols_s, nullptr, r.V, r.T, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 1, 1, 0});
        wr.push_back(to_int(r.cols_s));
        rd.push_back({});
      }
      ops.push_back(ChainOp{CH_TRI_MUL, r.f, r.f, r.k, r.d_cols_f, r.d_cols_c, nullptr, nullptr,
                            r.R, r.Rsn, nullptr, nullptr, nullptr, 0, 1, 1, 0});
      wr.push_back(to_int(r.cols_f));
      rd.push_back(to_int(r.cols_c));
      continue;
    }
    if (r.k <= 0) continue;
    if (r.kind == REC_SPARSIFY) {
      ops.push_back(ChainOp{CH_WY_T, r.m, r.k, 0, r.d_cols_s, nullptr, r.V, r.T, nullptr, nullptr, nullptr, r.WT, nullptr, 0, 1, 1, 0});
      wr.push_back(to_int(r.cols_s));
      rd.push_back({});
    } else {
      const bool bh = r.kind == REC_ELIM;
      ops.push_back(ChainOp{CH_TRI_MUL, r.k, r.k, bh ? r.n : 0, r.d_cols_s,
                            bh ? r.d_cols_n : nullptr, nullptr, nullptr, r.R, bh ? r.Rsn : nullptr, nullptr, nullptr, nullptr, 0, 1, 1, 0});
      wr.push_back(to_int(r.cols_s));
      rd.push_back(bh ? to_int(r.cols_n) : std::vector<int>());
    }
  }
  build_prog(c, 2, ops, wr, rd);
}

double* ensure_part(spq_ctx* c, int which, int nrhs) {   // call outside graph capture
  auto& P = c->prog[which];
  auto it = P.part_buf.find(nrhs);
  if (it == P.part_buf.end()) {
    int64_t mx = 1;
    for (auto v : P.part_sz) mx = std::max(mx, v);
    it = P.part_buf.emplace(nrhs, dalloc(c, (size_t)mx * nrhs * sizeof(double))).first;
  }
  return it->second;
}

void run_prog(spq_ctx* c, int which, double* z, int nrhs) {
  auto& P = c->prog[which];
  auto it = P.part_buf.find(nrhs);
  if (it == P.part_buf.end()) throw SpqError(SPQ_ERR_INTERNAL, "chain scratch missing");
  for (size_t w = 0; w < P.off.size(); ++w)
    launch_chain_wave(P.d_ops + P.off[w], P.d_tasks + P.toff[w], P.tcnt[w], P.kmax[w], P.slabk[w],
                      P.has_wy[w] != 0, it->second, z, c->N, nrhs, c->st);
}

// full application on c->d_vec (result in d_vec), captured once per nrhs
void run_chain(spq_ctx* c, int which, int nrhs) {
  if (!c->compiled) {   // solve programs are built on first use (not part of factorize)
    compile_chains(c);
    c->compiled = true;
  }
  auto& P = c->prog[which];
  if (env_flag("SPQ_CHAIN_PROFILE")) {
    // diagnostics: every wave timed on its own (no graph), one line per wave
    double* part = ensure_part(c, which, nrhs);
    if (which == 2 && c->equil) chain_diag(c->d_vec, c->d_scale, c->N, nrhs, false, c->st);
    cudaEvent_t e0, e1, em;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventCreate(&em));
    g_chain_mid_event = em;
    for (size_t w = 0; w < P.off.size(); ++w) {
      CUDA_TRY(cudaEventRecord(e0, c->st));
      launch_chain_wave(P.d_ops + P.off[w], P.d_tasks + P.toff[w], P.tcnt[w], P.kmax[w], P.slabk[w],
                        P.has_wy[w] != 0, part, c->d_vec, c->N, nrhs, c->st);
      CUDA_TRY(cudaEventRecord(e1, c->st));
      CUDA_TRY(cudaEventSynchronize(e1));
      float ms = 0, msa = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
      CUDA_TRY(cudaEventElapsedTime(&msa, e0, em));
      int nwy = 0, ntri = 0, kmx = 0, mmx = 0, nmx = 0;
      for (int t = P.off[w]; t < P.off[w] + P.cnt[w]; ++t) {
        const ChainOp& o = P.hops[t];
        (o.kind == CH_WY_T || o.kind == CH_WY_N ? nwy : ntri)++;
        kmx = std::max(kmx, o.k); mmx = std::max(mmx, o.m); nmx = std::max(nmx, o.n);
      }
      fprintf(stderr, "chain %d wave %zu: %.1f us (A %.1f) ops %d (wy %d tri %d) tasks %d kmax %d mmax %d nmax %d\n",
              which, w, 1e3 * ms, 1e3 * msa, P.cnt[w], nwy, ntri, P.tcnt[w], kmx, mmx, nmx);
    }
    if (which == 1 && c->equil) chain_diag(c->d_vec, c->d_scale, c->N, nrhs, true, c->st);
    if (which == 0) {
      chain_perm(c->d_vec, c->d_roc, c->N, nrhs, c->d_vec2, c->st);
      CUDA_TRY(cudaMemcpyAsync(c->d_vec, c->d_vec2, (size_t)c->N * nrhs * sizeof(double),
                               cudaMemcpyDeviceToDevice, c->st));
    }
    g_chain_mid_event = nullptr;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(em);
    return;
  }
  auto it = P.graphs.find(nrhs);
  if (it == P.graphs.end()) {
    ensure_part(c, which, nrhs);
    cudaGraph_t g;
    CUDA_TRY(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    if (which == 0) {
      run_prog(c, 0, c->d_vec, nrhs);
      chain_perm(c->d_vec, c->d_roc, c->N, nrhs, c->d_vec2, c->st);
      CUDA_TRY(cudaMemcpyAsync(c->d_vec, c->d_vec2, (size_t)c->N * nrhs * sizeof(double),
                               cudaMemcpyDeviceToDevice, c->st));
    } else if (which == 1) {
      run_prog(c, 1, c->d_vec, nrhs);
      if (c->equil) chain_diag(c->d_vec, c->d_scale, c->N, nrhs, true, c->st);
    } else {
      if (c->equil) chain_diag(c->d_vec, c->d_scale, c->N, nrhs, false, c->st);
      run_prog(c, 2, c->d_vec, nrhs);
    }
    CUDA_TRY(cudaStreamEndCapture(c->st, &g));
    cudaGraphExec_t ex;
    CUDA_TRY(cudaGraphInstantiate(&ex, g, 0));
    CUDA_TRY(cudaGraphDestroy(g));
    it = P.graphs.emplace(nrhs, ex).first;
  }
  Scope s(c, F_CHAIN);
  CUDA_TRY(cudaGraphLaunch(it->second, c->st));
  c->tm.launches[F_CHAIN]++;
}

template <class F>
int guarded(spq_ctx* c, F&& fn) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    fn();
    if (c) c->host_ms[3] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return SPQ_OK;
  } catch (const SpqError& e) {
    if (c) {
      c->err_code = e.code;
      c->err_index = e.index;
      c->err_value = e.value;
      c->err_msg = e.what();
    }
    return e.code;
  } catch (const CudaFailure& e) {
    if (c) {
      c->err_code = SPQ_ERR_CUDA;
      c->err_msg = e.what();
    }
    return SPQ_ERR_CUDA;
  } catch (const std::exception& e) {
    if (c) {
      c->err_code = SPQ_ERR_INTERNAL;
      c->err_msg = e.what();
    }
    return SPQ_ERR_INTERNAL;
  }
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int spq_version(void) { return 1; }

int spq_device_info(char* buf, int len) {
  int dev = 0;
  cudaDeviceProp p;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess)
    return SPQ_ERR_CUDA;
  snprintf(buf, len, "%s sm_%d%d SMs=%d smem/block=%zu", p.name, p.major, p.minor,
           p.multiProcessorCount, p.sharedMemPerBlockOptin);
  return SPQ_OK;
}

int spq_create(spq_ctx** out, int device) {
  *out = nullptr;
  spq_ctx* c = new spq_ctx();
  int rc = guarded(c, [&] {
    c->dev = device;
    // The planner builds and drops multi-megabyte task vectors many times per
    // factorization; with glibc's defaults each of them is a fresh mmap (page
    // faults on first touch, munmap on free).  Keep them in the heap.
    // SPQ_NO_MALLOPT=1 leaves the process's malloc policy alone.
    static const bool tuned = [] {
      if (!env_flag("SPQ_NO_MALLOPT")) {
        mallopt(M_MMAP_THRESHOLD, 256 << 20);
        mallopt(M_TRIM_THRESHOLD, 512 << 20);
        mallopt(M_TOP_PAD, 64 << 20);
      }
      return true;
    }();
    (void)tuned;
    CUDA_TRY(cudaSetDevice(device));
    // two attribute queries (cudaGetDeviceProperties fills the whole struct:
    // milliseconds per context)
    int major = 0, nsm = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    if (major < 10) throw SpqError(SPQ_ERR_CUDA, "sm_100a device required");
    c->nsm = nsm;
    {
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      if (!g.stream_sets.empty()) {
        const StreamSet ss = g.stream_sets.back();
        g.stream_sets.pop_back();
        c->st = ss.st;
        c->side = ss.side;
        c->ev_side_a = ss.ev_side_a;
        c->ev_side_b = ss.ev_side_b;
        c->ev_fork = ss.ev_fork;
        for (int k = 0; k < spq_ctx::NAUX; ++k) { c->aux[k] = ss.aux[k]; c->ev_join[k] = ss.ev_join[k]; }
      }
    }
    if (!c->st) CUDA_TRY(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    c->ring_cap = env_flag("SPQ_RING_SMALL") ? (1u << 16) : (64u << 20);
    bool others_live = false;
    {
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      others_live = g.n_ctx > 0;
      ++g.n_ctx;
      c->counted = true;
      if (!g.rings.empty() && !env_flag("SPQ_RING_SMALL")) {
        c->pin = g.rings.back().first;
        c->dring = g.rings.back().second;
        g.rings.pop_back();
      }
    }
    // A sole live context hands freed arena ranges back at once, ordered only
    // by its own stream (dfree).  Once this context is counted, the others
    // defer their frees to a stream sync; ranges they released before that
    // may still be read by their queued kernels, so drain the device once
    // before this context can allocate any of them.
    if (others_live) CUDA_TRY(cudaDeviceSynchronize());
    if (!c->pin) {
      CUDA_TRY(cudaMallocHost(&c->pin, c->ring_cap));
      CUDA_TRY(cudaMalloc(&c->dring, c->ring_cap));
    }
    c->spec = !env_flag("SPQ_NO_SPEC");
    {   // mapped speculation flag, reused across contexts (pinned allocations
        // and their frees cost milliseconds and cudaFreeHost synchronizes)
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      if (!g.spec_flags.empty()) {
        c->h_spec_bad = g.spec_flags.back();
        g.spec_flags.pop_back();
      }
      if (g.events_dev == device) c->ev_pool.swap(g.events);
    }
    if (!c->h_spec_bad)
      CUDA_TRY(cudaHostAlloc(&c->h_spec_bad, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    *c->h_spec_bad = 0;
    CUDA_TRY(cudaHostGetDevicePointer(&c->d_spec_bad, c->h_spec_bad, 0));
  });
  if (rc != SPQ_OK) {
    *out = c;  // caller may query the error, then destroy
    return rc;
  }
  *out = c;
  return SPQ_OK;
}

void spq_destroy(spq_ctx* c) {
  if (!c) return;
  try {
    if (c->side) cudaStreamSynchronize(c->side);
    if (c->st) cudaStreamSynchronize(c->st);
    // scope events go back to the process pool (the streams are drained:
    // every recorded event has completed); the next context reuses them
    // instead of creating ~5000 events per factorization
    for (int f = 0; f < F_NFAM; ++f)
      for (auto& e : c->tm.ev[f]) { c->ev_pool.push_back(e.first); c->ev_pool.push_back(e.second); }
    {
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      if (g.events.empty()) g.events_dev = c->dev;
      while (!c->ev_pool.empty() && g.events_dev == c->dev && g.events.size() < ((size_t)1 << 16)) {
        g.events.push_back(c->ev_pool.back());
        c->ev_pool.pop_back();
      }
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->st) cudaStreamSynchronize(c->st);
    for (void* p : c->big) c->big_pending.push_back(p);
    c->big.clear();
    publish_big(c);
    for (auto e : c->marks) cudaEventDestroy(e);
    for (auto& P : c->prog)
      for (auto& kv : P.graphs) cudaGraphExecDestroy(kv.second);
    {
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      for (size_t i = 0; i < c->slabs.size(); ++i)
        if (c->slabs[i]) g.slabs.push_back({c->slabs[i], c->slab_caps[i]});
      if (c->pin && c->dring) g.rings.push_back({c->pin, c->dring});
      if (c->counted) --g.n_ctx;
    }
    {   // every stream drained: the whole set goes back to the device's cache
      StreamSet ss;
      for (int k = 0; k < spq_ctx::NAUX; ++k) {
        if (c->aux[k]) cudaStreamSynchronize(c->aux[k]);
        ss.aux[k] = c->aux[k];
        ss.ev_join[k] = c->ev_join[k];
      }
      if (c->side) cudaStreamSynchronize(c->side);
      if (c->st) cudaStreamSynchronize(c->st);
      ss.st = c->st;
      ss.side = c->side;
      ss.ev_side_a = c->ev_side_a;
      ss.ev_side_b = c->ev_side_b;
      ss.ev_fork = c->ev_fork;
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      if (ss.st && g.stream_sets.size() < 16) {
        g.stream_sets.push_back(ss);
      } else {
        for (int k = 0; k < spq_ctx::NAUX; ++k) {
          if (ss.aux[k]) cudaStreamDestroy(ss.aux[k]);
          if (ss.ev_join[k]) cudaEventDestroy(ss.ev_join[k]);
        }
        if (ss.ev_fork) cudaEventDestroy(ss.ev_fork);
        if (ss.side) cudaStreamDestroy(ss.side);
        if (ss.ev_side_a) cudaEventDestroy(ss.ev_side_a);
        if (ss.ev_side_b) cudaEventDestroy(ss.ev_side_b);
        if (ss.st) cudaStreamDestroy(ss.st);
      }
    }
    if (c->h_spec_bad) {   // every stream of the context is drained: back to the pool
      auto& g = gcache(c->dev);
      std::lock_guard<std::mutex> lk(g.mu);
      g.spec_flags.push_back(c->h_spec_bad);
      c->h_spec_bad = nullptr;
    }
  } catch (...) {
  }
  delete c;
}

int spq_last_error(spq_ctx* c, int* code, int64_t* index, double* value, char* msg, int msglen) {
  if (!c) return SPQ_ERR_BAD_INPUT;
  if (code) *code = c->err_code;
  if (index) *index = c->err_index;
  if (value) *value = c->err_value;
  if (msg && msglen > 0) snprintf(msg, msglen, "%s", c->err_msg.c_str());
  return SPQ_OK;
}

int spq_load(spq_ctx* c, int64_t N, const int64_t* indptr, const int64_t* indices,
             const double* data, int equilibrate, int n_clusters_total, int n_leaf,
             const int32_t* leaf_ids, const int64_t* rows_ptr, const int64_t* rows,
             const int64_t* cols_ptr, const int64_t* cols) {
  return guarded(c, [&] {
    HostTimer ht(&c->host_ms[14]);
    do_load(c, N, indptr, indices, data, equilibrate, n_clusters_total, n_leaf, leaf_ids,
            rows_ptr, rows, cols_ptr, cols);
  });
}

int spq_factor(spq_ctx* c, int n, const int32_t* ids) {
  return guarded(c, [&] { do_factor(c, std::vector<int>(ids, ids + n)); });
}

int spq_scale(spq_ctx* c, int n, const int32_t* ids, int32_t* out_done) {
  return guarded(c, [&] { do_scale(c, std::vector<int>(ids, ids + n), out_done); });
}

int spq_sparsify(spq_ctx* c, int n, const int32_t* ids, double eps, int32_t* out_rank,
                 int32_t* out_before, double* out_dropped, int32_t* out_done) {
  return spq_sparsify_ex(c, n, ids, eps, SPM_SCALED, 1, out_rank, out_before, out_dropped,
                         out_done);
}

int spq_sparsify_ex(spq_ctx* c, int n, const int32_t* ids, double eps, int mode, int scaled_now,
                    int32_t* out_rank, int32_t* out_before, double* out_dropped,
                    int32_t* out_done) {
  return guarded(c, [&] {
    if (mode < SPM_SCALED || mode > SPM_VARIANT2) throw SpqError(SPQ_ERR_BAD_INPUT, "sparsify mode");
    for (int t = 0; t < n; ++t) {
      out_rank[t] = -1; out_before[t] = 0; out_dropped[t] = 0.0; out_done[t] = 0;
    }
    std::vector<SparsifyOut> outs;
    do_sparsify(c, std::vector<int>(ids, ids + n), eps, outs, mode, scaled_now != 0);
    for (int t = 0; t < n; ++t) {
      out_rank[t] = outs[t].rank;
      out_before[t] = outs[t].before;
      out_dropped[t] = outs[t].dropped;
      out_done[t] = outs[t].done;
    }
  });
}

int spq_merge(spq_ctx* c, int n_parents, const int32_t* parent_ids, const int32_t* child_ptr,
              const int32_t* child_ids) {
  return guarded(c, [&] { do_merge(c, n_parents, parent_ids, child_ptr, child_ids); });
}

int spq_finish(spq_ctx* c) {
  return guarded(c, [&] {
    HostTimer ht(&c->host_ms[15]);
    pivot_raise(c, c->piv);
    for (int64_t j = 0; j < c->N; ++j)
      if (c->row_of_col[j] < 0) {
        sync(c);
        spec_raise(c);
        int64_t miss = 0;
        for (int64_t t = 0; t < c->N; ++t) miss += c->row_of_col[t] < 0;
        throw SpqError(SPQ_ERR_BAD_INPUT, std::to_string(miss) + " columns were never factored (inconsistent tree?)");
      }
    // one packed device array for row_of_col and every record's index sets
    std::vector<int> pack(c->row_of_col.begin(), c->row_of_col.end());
    std::vector<size_t> offs;
    for (auto& r : c->recs)
      for (auto* v : {&r.rows, &r.cols_s, &r.cols_n, &r.cols_f, &r.cols_c}) {
        offs.push_back(pack.size());
        pack.insert(pack.end(), v->begin(), v->end());
      }
    int* d = (int*)dalloc(c, std::max<size_t>(pack.size(), 1) * sizeof(int));
    CUDA_TRY(cudaMemcpyAsync(d, pack.data(), pack.size() * sizeof(int), cudaMemcpyHostToDevice, c->st));
    c->d_roc = d;
    c->d_index_pack = d;
    size_t q = 0;
    for (auto& r : c->recs) {
      r.d_rows = d + offs[q++];
      r.d_cols_s = d + offs[q++];
      r.d_cols_n = d + offs[q++];
      r.d_cols_f = d + offs[q++];
      r.d_cols_c = d + offs[q++];
    }
    std::vector<TProb> tp;
    for (auto& r : c->recs)
      if (r.kind != REC_SPARSIFY && r.k > 0 && !r.full_T) tp.push_back(TProb{r.V, r.m, r.k, r.tau, r.T});
    build_full_T(c, tp);
    c->finished = true;
    sync(c);
    spec_raise(c);
  });
}

int spq_set_option(spq_ctx* c, const char* key, int64_t value) {
  return guarded(c, [&] {
    const std::string k = key ? key : "";
    if (k == "speculate") {
      if (!c->blk.empty() || !c->recs.empty())
        throw SpqError(SPQ_ERR_BAD_INPUT, "speculate must be set before spq_load");
      c->spec = value != 0;
    } else {
      throw SpqError(SPQ_ERR_BAD_INPUT, "unknown option '" + k + "'");
    }
  });
}

int spq_cluster_size(spq_ctx* c, int id, int64_t* nr, int64_t* nc) {
  return guarded(c, [&] {
    if (id < 0 || id >= c->ncl) throw SpqError(SPQ_ERR_BAD_INPUT, "cluster id out of range");
    *nr = (int64_t)c->rows_of[id].size();
    *nc = (int64_t)c->cols_of[id].size();
  });
}

int spq_cluster_sizes(spq_ctx* c, int n, const int32_t* ids, int64_t* ncols) {
  return guarded(c, [&] {
    for (int t = 0; t < n; ++t) {
      if (ids[t] < 0 || ids[t] >= c->ncl) throw SpqError(SPQ_ERR_BAD_INPUT, "cluster id out of range");
      ncols[t] = (int64_t)c->cols_of[ids[t]].size();
    }
  });
}

int spq_total_cols(spq_ctx* c, int64_t* out) {
  return guarded(c, [&] {
    int64_t t = 0;
    for (int s = 0; s < c->ncl; ++s) if (c->active[s]) t += (int64_t)c->cols_of[s].size();
    *out = t;
  });
}

int spq_trailing_stats(spq_ctx* c, int64_t* nblocks, int64_t* nnz) {
  return guarded(c, [&] {
    HostTimer ht(&c->host_ms[13]);
    *nblocks = (int64_t)c->blk.size();
    std::vector<const double*> ptrs;
    std::vector<int64_t> sizes;
    for_each_block(c, [&](uint64_t, Block& b) {
      const int64_t n = (int64_t)b.nr * b.nc;
      if (n > 0) { ptrs.push_back(b.p); sizes.push_back(n); }
    });
    unsigned long long* d = (unsigned long long*)dalloc(c, sizeof(unsigned long long));
    CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->st));
    if (!ptrs.empty())
      launch_count_nnz(upload(c, ptrs), upload(c, sizes), (int)ptrs.size(), d, c->st);
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    dfree(c, d);
    *nnz = (int64_t)h;
  });
}

// trailing_blocks now, trailing_nnz counted on the device into a slot read
// later (spq_trailing_nnz): no host round trip per level
int spq_trailing_stats_async(spq_ctx* c, int slot, int64_t* nblocks) {
  return guarded(c, [&] {
    HostTimer ht(&c->host_ms[13]);
    if (slot < 0 || slot >= 4096) throw SpqError(SPQ_ERR_BAD_INPUT, "stats slot out of range");
    if (!c->d_nnz_slots) {
      c->d_nnz_slots = (unsigned long long*)dalloc(c, 4096 * sizeof(unsigned long long));
      CUDA_TRY(cudaMemsetAsync(c->d_nnz_slots, 0, 4096 * sizeof(unsigned long long), c->st));
    }
    *nblocks = (int64_t)c->blk.size();
    std::vector<const double*> ptrs;
    std::vector<int64_t> sizes;
    for_each_block(c, [&](uint64_t, Block& b) {
      const int64_t n = (int64_t)b.nr * b.nc;
      if (n > 0) { ptrs.push_back(b.p); sizes.push_back(n); }
    });
    unsigned long long* d = c->d_nnz_slots + slot;
    CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->st));
    if (!ptrs.empty())
      launch_count_nnz(upload(c, ptrs), upload(c, sizes), (int)ptrs.size(), d, c->st);
    c->n_kernels++;
  });
}

int spq_trailing_nnz(spq_ctx* c, int n, int64_t* out) {
  return guarded(c, [&] {
    if (n < 0 || n > 4096) throw SpqError(SPQ_ERR_BAD_INPUT, "stats slot count out of range");
    if (!c->d_nnz_slots || n == 0) { std::fill(out, out + n, 0); return; }
    std::vector<unsigned long long> h(n);
    CUDA_TRY(cudaMemcpyAsync(h.data(), c->d_nnz_slots, n * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int i = 0; i < n; ++i) out[i] = (int64_t)h[i];
  });
}

int spq_trailing_keys(spq_ctx* c, int64_t cap, int32_t* rows, int32_t* cols, int64_t* n) {
  return guarded(c, [&] {
    int64_t t = 0;
    for (int i = 0; i < c->ncl; ++i) {   // ascending (row, column): the sorted adjacency lists
      const FlatSet& row = c->rix[i];
      for (size_t q = 0; q < row.v.size(); ++q) {
        const Block* b = row.b[q];
        if (!b || (int64_t)b->nr * b->nc == 0) continue;
        if (t < cap) { rows[t] = i; cols[t] = row.v[q]; }
        ++t;
      }
    }
    *n = t;
  });
}

int spq_row_of_col(spq_ctx* c, int64_t* out) {
  return guarded(c, [&] { std::copy(c->row_of_col.begin(), c->row_of_col.end(), out); });
}

int spq_payload_scalars(spq_ctx* c, int64_t* out) {
  return guarded(c, [&] {
    int64_t t = c->equil ? c->N : 0;
    for (auto& r : c->recs) t += r.payload_scalars;
    *out = t;
  });
}

int spq_timings(spq_ctx* c, double* out, int n) {
  return guarded(c, [&] {
    collect_timings(c);
    // layout: [ms, flops, launches] per family
    for (int f = 0; f < F_NFAM && 4 * f + 3 < n; ++f) {
      out[4 * f] = c->tm.ms[f];
      out[4 * f + 1] = c->tm.flops[f];
      out[4 * f + 2] = (double)c->tm.launches[f];
      out[4 * f + 3] = c->tm.bytes[f];
    }
    const double extra[8] = {c->host_ms[0], c->host_ms[1], c->host_ms[2], c->host_ms[3],
                             (double)c->n_allocs, (double)c->n_syncs, (double)c->pool_bytes,
                             (double)c->n_kernels};
    for (int i = 0; i < 8 && 4 * F_NFAM + i < n; ++i) out[4 * F_NFAM + i] = extra[i];
    for (int i = 4; i < 16 && 4 * F_NFAM + 8 + (i - 4) < n; ++i) out[4 * F_NFAM + 8 + (i - 4)] = c->host_ms[i];
    if (4 * F_NFAM + 21 < n) {
      out[4 * F_NFAM + 20] = (double)c->live_bytes;
      out[4 * F_NFAM + 21] = (double)c->peak_bytes;
    }
    if (4 * F_NFAM + 24 < n) {
      out[4 * F_NFAM + 22] = c->spec ? 1.0 : 0.0;
      out[4 * F_NFAM + 23] = (double)c->n_verified;
      out[4 * F_NFAM + 24] = c->h_spec_bad ? (double)*c->h_spec_bad : 0.0;
    }
    if (4 * F_NFAM + 25 < n) out[4 * F_NFAM + 25] = (double)c->n_sparsify_waves;
  });
}

int spq_reset_timings(spq_ctx* c) {
  return guarded(c, [&] {
    collect_timings(c);
    for (int f = 0; f < F_NFAM; ++f) {
      c->tm.ms[f] = 0; c->tm.flops[f] = 0; c->tm.launches[f] = 0; c->tm.bytes[f] = 0;
    }
    for (double& h : c->host_ms) h = 0;
    c->n_allocs = c->n_syncs = c->n_kernels = 0;
  });
}

int spq_num_records(spq_ctx* c) { return c ? (int)c->recs.size() : 0; }

int spq_record_info(spq_ctx* c, int idx, int64_t* info) {
  return guarded(c, [&] {
    if (idx < 0 || idx >= (int)c->recs.size()) throw SpqError(SPQ_ERR_BAD_INPUT, "record index");
    Record& r = c->recs[idx];
    info[0] = r.kind; info[1] = r.m; info[2] = r.k; info[3] = r.n; info[4] = r.rank;
    info[5] = r.cid;
    info[6] = r.unscaled ? 1 : 0;
    info[7] = r.f;
  });
}

int spq_record_get(spq_ctx* c, int idx, int which, void* out) {
  return guarded(c, [&] {
    if (idx < 0 || idx >= (int)c->recs.size()) throw SpqError(SPQ_ERR_BAD_INPUT, "record index");
    Record& r = c->recs[idx];
    auto cp = [&](const double* d, size_t n) {
      if (n) CUDA_TRY(cudaMemcpyAsync(out, d, n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      sync(c);
    };
    switch (which) {
      case 0: std::copy(r.rows.begin(), r.rows.end(), (int64_t*)out); break;
      case 1: std::copy(r.cols_s.begin(), r.cols_s.end(), (int64_t*)out); break;
      case 2: std::copy(r.cols_n.begin(), r.cols_n.end(), (int64_t*)out); break;
      case 3: cp(r.V, (size_t)r.m * r.k); break;
      case 4: cp(r.tau, r.k); break;
      case 5: cp(r.T, (size_t)r.k * r.k); break;
      case 6:
        if (r.unscaled) cp(r.R, (size_t)r.f * r.f);        // R_ff
        else if (r.R) cp(r.R, (size_t)r.k * r.k);
        break;
      case 7:
        if (r.unscaled) cp(r.Rsn, (size_t)r.f * r.k);      // R_fc
        else if (r.Rsn) cp(r.Rsn, (size_t)r.k * r.n);
        break;
      case 8: if (r.unscaled) cp(r.hV, (size_t)r.m * r.f); break;
      case 9: if (r.unscaled) cp(r.htau, r.f); break;
      case 10: if (r.unscaled) cp(r.hT, (size_t)r.f * r.f); break;
      default: throw SpqError(SPQ_ERR_BAD_INPUT, "record field");
    }
  });
}

static int chain_host(spq_ctx* c, const double* in, double* out, int nrhs, int which) {
  return guarded(c, [&] {
    if (!c->finished) throw SpqError(SPQ_ERR_BAD_INPUT, "factorization not finished");
    ensure_chain_scratch(c, nrhs);
    const size_t bytes = (size_t)c->N * nrhs * sizeof(double);
    CUDA_TRY(cudaMemcpyAsync(c->d_vec, in, bytes, cudaMemcpyHostToDevice, c->st));
    run_chain(c, which, nrhs);
    CUDA_TRY(cudaMemcpyAsync(out, c->d_vec, bytes, cudaMemcpyDeviceToHost, c->st));
    sync(c);
  });
}

int spq_apply_qt_host(spq_ctx* c, const double* in, double* out, int nrhs) { return chain_host(c, in, out, nrhs, 0); }
int spq_solve_w_host(spq_ctx* c, const double* in, double* out, int nrhs) { return chain_host(c, in, out, nrhs, 1); }
int spq_apply_w_host(spq_ctx* c, const double* in, double* out, int nrhs) { return chain_host(c, in, out, nrhs, 2); }

static int chain_dev(spq_ctx* c, double* d, int nrhs, int which) {
  return guarded(c, [&] {
    if (!c->finished) throw SpqError(SPQ_ERR_BAD_INPUT, "factorization not finished");
    ensure_chain_scratch(c, nrhs);
    const size_t bytes = (size_t)c->N * nrhs * sizeof(double);
    CUDA_TRY(cudaMemcpyAsync(c->d_vec, d, bytes, cudaMemcpyDeviceToDevice, c->st));
    run_chain(c, which, nrhs);
    CUDA_TRY(cudaMemcpyAsync(d, c->d_vec, bytes, cudaMemcpyDeviceToDevice, c->st));
  });
}

int spq_apply_qt_dev(spq_ctx* c, double* d, int nrhs) { return chain_dev(c, d, nrhs, 0); }
int spq_solve_w_dev(spq_ctx* c, double* d, int nrhs) { return chain_dev(c, d, nrhs, 1); }

// ================================================================ GMRES
// Right-preconditioned GMRES entirely on the device (reference
// pkg/src/nestqr/solve.py:66-209): the operator v -> apply_qt(A solve_w(v))
// runs as chain graphs + a CSR SpMV, Arnoldi with modified Gram-Schmidt (one
// fused launch per step) and the conditional re-orthogonalisation test on
// the device; only the Hessenberg column (j+2 scalars) and the true residual
// norm come back per iteration for the Givens / least-squares update, which
// the host does exactly like the reference.
int spq_set_matrix(spq_ctx* c, int64_t N, const int64_t* indptr, const int64_t* indices,
                   const double* data) {
  return guarded(c, [&] {
    if (N != c->N) throw SpqError(SPQ_ERR_BAD_INPUT, "matrix size does not match the factorization");
    const int64_t nnz = indptr[N];
    std::vector<int64_t> rp(N + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) {
      if (indices[e] < 0 || indices[e] >= N) throw SpqError(SPQ_ERR_BAD_INPUT, "row index out of range");
      rp[indices[e] + 1]++;
    }
    for (int64_t i = 0; i < N; ++i) rp[i + 1] += rp[i];
    std::vector<int> ci(std::max<int64_t>(nnz, 1));
    std::vector<double> cv(std::max<int64_t>(nnz, 1));
    std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
    for (int64_t j = 0; j < N; ++j)
      for (int64_t e = indptr[j]; e < indptr[j + 1]; ++e) {
        const int64_t at = fill[indices[e]]++;
        ci[at] = (int)j;
        cv[at] = data[e];
      }
    dfree(c, c->d_csr_ptr);
    dfree(c, c->d_csr_idx);
    dfree(c, c->d_csr_val);
    c->d_csr_ptr = (int64_t*)dalloc(c, (N + 1) * sizeof(int64_t));
    c->d_csr_idx = (int*)dalloc(c, ci.size() * sizeof(int));
    c->d_csr_val = dalloc(c, cv.size() * sizeof(double));
    CUDA_TRY(cudaMemcpyAsync(c->d_csr_ptr, rp.data(), (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaMemcpyAsync(c->d_csr_idx, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaMemcpyAsync(c->d_csr_val, cv.data(), cv.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
    sync(c);
  });
}

int spq_gmres(spq_ctx* c, const double* b_h, const double* x0_h, double tol, int maxit,
              int restart, double* x_h, double* hist_h, int* its_out, int* conv_out,
              double* best_out) {
  return guarded(c, [&] {
    if (!c->finished) throw SpqError(SPQ_ERR_BAD_INPUT, "factorization not finished");
    if (!c->d_csr_ptr) throw SpqError(SPQ_ERR_BAD_INPUT, "spq_set_matrix was not called");
    if (maxit < 0) throw SpqError(SPQ_ERR_BAD_INPUT, "maxit must be >= 0");
    const int64_t n = c->N;
    const size_t vb = (size_t)n * sizeof(double);
    const double thr = 1e-8;   // solve.py:25
    ensure_chain_scratch(c, 1);
    const int mcap = std::max(1, restart > 0 ? std::min(restart, std::max(maxit, 1)) : std::max(maxit, 1));
    // device workspace: Q (n x (mcap+1)) | b | x | xn | best | w | t
    double* Q = dalloc(c, (size_t)n * (mcap + 1) * sizeof(double));
    double* vecs = dalloc(c, 6 * vb);
    double *b = vecs, *x = b + n, *xn = x + n, *best = xn + n, *w = best + n, *t = w + n;
    double* part = dalloc(c, (size_t)(mcap + 3) * KRY_G * sizeof(double));
    double* scal = dalloc(c, (size_t)(3 * (mcap + 2) + 8) * sizeof(double));
    double* Hcol = scal;                  // mcap + 2
    double* cvec = Hcol + (mcap + 2);     // mcap + 2
    double* ydev = cvec + (mcap + 2);     // mcap + 2
    double* sc = ydev + (mcap + 2);       // [0] norm, [1] norm2
    int* flag = (int*)dalloc(c, sizeof(int));
    double* partA = part;
    double* partB = part + KRY_G;
    double* partM = part + 2 * KRY_G;
    auto norm_of = [&](const double* v, double* out) {
      kry_dot_part(v, v, n, partA, c->st);
      kry_finish(partA, out, true, c->st);
    };
    auto fetch = [&](const double* d, double* h, int cnt) {
      CUDA_TRY(cudaMemcpyAsync(h, d, cnt * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      sync(c);
    };
    // preconditioned operator pieces on c->d_vec
    auto apply_qt_into = [&](const double* src, double* dst) {
      CUDA_TRY(cudaMemcpyAsync(c->d_vec, src, vb, cudaMemcpyDeviceToDevice, c->st));
      run_chain(c, 0, 1);
      CUDA_TRY(cudaMemcpyAsync(dst, c->d_vec, vb, cudaMemcpyDeviceToDevice, c->st));
    };
    CUDA_TRY(cudaMemcpyAsync(b, b_h, vb, cudaMemcpyHostToDevice, c->st));
    if (x0_h) CUDA_TRY(cudaMemcpyAsync(x, x0_h, vb, cudaMemcpyHostToDevice, c->st));
    else CUDA_TRY(cudaMemsetAsync(x, 0, vb, c->st));
    double h2[2];
    norm_of(b, sc);
    fetch(sc, h2, 1);
    const double bnorm = h2[0];
    int nh = 0;
    if (bnorm == 0.0) {
      std::fill(x_h, x_h + n, 0.0);
      hist_h[0] = 0.0;
      *its_out = 0;
      *conv_out = 1;
      *best_out = 0.0;
    } else {
      kry_spmv(c->d_csr_ptr, c->d_csr_idx, c->d_csr_val, x, b, t, n, 1, c->st);
      norm_of(t, sc);
      fetch(sc, h2, 1);
      hist_h[nh++] = h2[0] / bnorm;
      bool done = hist_h[0] <= tol;
      double best_r = hist_h[0];
      CUDA_TRY(cudaMemcpyAsync(best, x, vb, cudaMemcpyDeviceToDevice, c->st));
      int its = 0;
      std::vector<double> H, cs, sn, g, hc(mcap + 2), y;
      while (!done && its < maxit) {
        // z = apply_qt(b - A x), beta = ||z||
        kry_spmv(c->d_csr_ptr, c->d_csr_idx, c->d_csr_val, x, b, t, n, 1, c->st);
        apply_qt_into(t, Q);
        norm_of(Q, sc);
        fetch(sc, h2, 1);
        const double beta = h2[0];
        if (beta == 0.0) { done = true; break; }
        const int m = restart > 0 ? std::min(restart, maxit - its) : maxit - its;
        H.assign((size_t)(m + 1) * m, 0.0);   // column-major (m+1) x m
        cs.assign(m, 0.0); sn.assign(m, 0.0); g.assign(m + 1, 0.0);
        g[0] = beta;
        kry_scale_div(Q, sc, Q, n, c->st);
        CUDA_TRY(cudaMemcpyAsync(xn, x, vb, cudaMemcpyDeviceToDevice, c->st));
        auto Hij = [&](int i, int j) -> double& { return H[(size_t)j * (m + 1) + i]; };
        for (int j = 0; j < m; ++j) {
          const double* qj = Q + (size_t)j * n;
          // w = apply_qt(A solve_w(q_j))
          CUDA_TRY(cudaMemcpyAsync(c->d_vec, qj, vb, cudaMemcpyDeviceToDevice, c->st));
          run_chain(c, 1, 1);
          kry_spmv(c->d_csr_ptr, c->d_csr_idx, c->d_csr_val, c->d_vec, nullptr, t, n, 0, c->st);
          apply_qt_into(t, w);
          // modified Gram-Schmidt, one fused launch per step
          kry_dot_part(Q, w, n, partA, c->st);
          for (int i = 0; i <= j; ++i) {
            const double* qn = i < j ? Q + (size_t)(i + 1) * n : nullptr;
            kry_mgs_step(Q + (size_t)i * n, qn, w, n, (i & 1) ? partB : partA,
                         (i & 1) ? partA : partB, Hcol + i, c->st);
          }
          double* pw = ((j + 1) & 1) ? partB : partA;   // w.w partials of the last step
          kry_finish(pw, sc, true, c->st);
          // conditional re-orthogonalisation against Q[:, 0:j+1]
          kry_multi_dot(Q, n, j + 1, w, n, partM, cvec, c->st);
          kry_reorth(Q, n, j + 1, cvec, sc, thr, w, n, Hcol, flag, partA, c->st);
          kry_finish(partA, sc + 1, true, c->st);
          CUDA_TRY(cudaMemcpyAsync(hc.data(), Hcol, (j + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->st));
          fetch(sc, h2, 2);
          for (int i = 0; i <= j; ++i) Hij(i, j) = hc[i];
          const double wn = h2[1];
          Hij(j + 1, j) = wn;
          for (int i = 0; i < j; ++i) {     // previous rotations
            const double a = Hij(i, j), bb = Hij(i + 1, j);
            Hij(i, j) = cs[i] * a + sn[i] * bb;
            Hij(i + 1, j) = -sn[i] * a + cs[i] * bb;
          }
          const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
          if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
          else { cs[j] = Hij(j, j) / den; sn[j] = Hij(j + 1, j) / den; }
          Hij(j, j) = cs[j] * Hij(j, j) + sn[j] * Hij(j + 1, j);
          Hij(j + 1, j) = 0.0;
          g[j + 1] = -sn[j] * g[j];
          g[j] = cs[j] * g[j];
          // y = H[0:j+1, 0:j+1]^{-1} g[0:j+1] (upper triangular)
          y.assign(j + 1, 0.0);
          for (int i = j; i >= 0; --i) {
            double s = g[i];
            for (int l = i + 1; l <= j; ++l) s -= Hij(i, l) * y[l];
            y[i] = s / Hij(i, i);
          }
          // x_new = x + solve_w(Q y); true residual
          CUDA_TRY(cudaMemcpyAsync(ydev, y.data(), (j + 1) * sizeof(double), cudaMemcpyHostToDevice, c->st));
          kry_gemv(Q, n, j + 1, ydev, c->d_vec, n, c->st);
          run_chain(c, 1, 1);
          kry_add(x, c->d_vec, xn, n, c->st);
          kry_spmv(c->d_csr_ptr, c->d_csr_idx, c->d_csr_val, xn, b, t, n, 1, c->st);
          norm_of(t, sc);
          fetch(sc, h2, 1);
          ++its;
          hist_h[nh++] = h2[0] / bnorm;
          if (hist_h[nh - 1] < best_r) {
            best_r = hist_h[nh - 1];
            CUDA_TRY(cudaMemcpyAsync(best, xn, vb, cudaMemcpyDeviceToDevice, c->st));
          }
          if (std::fabs(g[j + 1]) / bnorm <= tol || hist_h[nh - 1] <= tol) { done = true; break; }
          if (wn <= 1e-300) break;
          kry_scale_div(w, sc + 1, Q + (size_t)(j + 1) * n, n, c->st);
        }
        CUDA_TRY(cudaMemcpyAsync(x, xn, vb, cudaMemcpyDeviceToDevice, c->st));
      }
      CUDA_TRY(cudaMemcpyAsync(x_h, best, vb, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      *its_out = its;
      *conv_out = done ? 1 : 0;
      *best_out = best_r;
    }
    dfree(c, Q);
    dfree(c, vecs);
    dfree(c, part);
    dfree(c, scal);
    dfree(c, flag);
    sync(c);
  });
}

int spq_mark(spq_ctx* c, int slot) {
  return guarded(c, [&] {
    if (slot < 0 || slot > 63) throw SpqError(SPQ_ERR_BAD_INPUT, "mark slot");
    while ((int)c->marks.size() <= slot) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      c->marks.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(c->marks[slot], c->st));
  });
}

int spq_mark_elapsed(spq_ctx* c, int a, int b, float* ms) {
  return guarded(c, [&] {
    if (a < 0 || b < 0 || a >= (int)c->marks.size() || b >= (int)c->marks.size())
      throw SpqError(SPQ_ERR_BAD_INPUT, "mark slot");
    CUDA_TRY(cudaEventSynchronize(c->marks[b]));
    CUDA_TRY(cudaEventElapsedTime(ms, c->marks[a], c->marks[b]));
  });
}

int spq_chain_info(spq_ctx* c, int which, int64_t* info4) {
  return guarded(c, [&] {
    if (which < 0 || which > 2) throw SpqError(SPQ_ERR_BAD_INPUT, "chain index");
    if (!c->compiled) { compile_chains(c); c->compiled = true; }
    auto& P = c->prog[which];
    int64_t ops = 0, maxw = 0, kmax = 0;
    for (size_t w = 0; w < P.cnt.size(); ++w) {
      ops += P.cnt[w];
      maxw = std::max<int64_t>(maxw, P.cnt[w]);
      kmax = std::max<int64_t>(kmax, P.kmax[w]);
    }
    info4[0] = (int64_t)P.cnt.size(); info4[1] = ops; info4[2] = maxw; info4[3] = kmax;
  });
}

int spq_synchronize(spq_ctx* c) {
  return guarded(c, [&] { sync(c); });
}

// ------------------------------------------------------ kernel plugin API
// host row-major (numpy) <-> device column-major via transposing copies
static double* to_dev_colmajor(spq_ctx* c, const double* h, int64_t m, int64_t k, CopyBatch& cb) {
  double* raw = dalloc(c, (size_t)std::max<int64_t>(m * k, 1) * sizeof(double));
  double* cm = dalloc(c, (size_t)std::max<int64_t>(m * k, 1) * sizeof(double));
  if (m * k) CUDA_TRY(cudaMemcpyAsync(raw, h, m * k * sizeof(double), cudaMemcpyHostToDevice, c->st));
  CopyTask t{};
  t.src = raw; t.dst = cm; t.nr = (int)k; t.nc = (int)m; t.lds = (int)std::max<int64_t>(k, 1);
  t.ldd = (int)std::max<int64_t>(m, 1); t.trans = 1;
  cb.add(t);
  c->deferred.push_back(raw);
  return cm;
}

static void to_host_rowmajor(spq_ctx* c, const double* d, int64_t m, int64_t k, int64_t ld,
                             double* h) {
  if (m * k == 0) return;
  double* raw = dalloc(c, (size_t)(m * k) * sizeof(double));
  CopyBatch cb;
  CopyTask t{};
  t.src = d; t.dst = raw; t.nr = (int)m; t.nc = (int)k; t.lds = (int)ld; t.ldd = (int)k; t.trans = 1;
  cb.add(t);
  cb.run(c);
  CUDA_TRY(cudaMemcpyAsync(h, raw, m * k * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  dfree(c, raw);
}

int spq_qr_house(spq_ctx* c, int64_t m, int64_t k, const double* B, double* V, double* tau,
                 double* T, double* R) {
  return guarded(c, [&] {
    if (m < k) throw SpqError(SPQ_ERR_BAD_INPUT, "qr_house needs m >= k");
    if (k == 0) return;
    CopyBatch cb;
    double* P = to_dev_colmajor(c, B, m, k, cb);
    double* aux = dalloc(c, (size_t)(k + 2 * k * k) * sizeof(double));
    cb.zero(aux, k + 2 * k * k);
    cb.run(c);
    double* dtau = aux;
    double* dT = aux + k;
    double* dR = dT + k * k;
    qr_batch(c, {QrProb{P, (int)m, (int)k, dR, dtau, dT, {}}});
    build_full_T(c, {TProb{P, (int)m, (int)k, dtau, dT}});
    to_host_rowmajor(c, P, m, k, m, V);
    to_host_rowmajor(c, dT, k, k, k, T);
    to_host_rowmajor(c, dR, k, k, k, R);
    CUDA_TRY(cudaMemcpyAsync(tau, dtau, k * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    dfree(c, P);
    dfree(c, aux);
    flush_deferred(c);
  });
}

int spq_apply_panel(spq_ctx* c, int64_t m, int64_t k, int64_t n, const double* V, const double* T,
                    double* C, int transpose) {
  return guarded(c, [&] {
    if (k == 0 || n == 0 || m == 0) return;
    CopyBatch cb;
    double* dV = to_dev_colmajor(c, V, m, k, cb);
    double* dT = to_dev_colmajor(c, T, k, k, cb);
    double* dC = to_dev_colmajor(c, C, m, n, cb);
    cb.run(c);
    wy_batch(c, {WyProb{dV, dT, (int)m, (int)k, dC, (int)m, (int)n}}, transpose != 0);
    to_host_rowmajor(c, dC, m, n, m, C);
    dfree(c, dV); dfree(c, dT); dfree(c, dC);
    flush_deferred(c);
  });
}

int spq_rrqr(spq_ctx* c, int64_t m, int64_t k, const double* M, double eps, int64_t min_rank,
             double* V, double* tau, double* Tred, int64_t* perm, int64_t* rank) {
  return guarded(c, [&] {
    const int kmax = (int)std::min(m, k);
    CopyBatch cb;
    double* W = to_dev_colmajor(c, M, m, k, cb);
    const int G = cpqr_grid((int)std::max<int64_t>(k, 1), c->nsm);
    const size_t vsz = (size_t)std::max<int64_t>(m, 1) * std::max(kmax, 1);
    double* aux = dalloc(c, (vsz + 2 * (size_t)std::max(kmax, 1) + 2 * G + 2) * sizeof(double));
    double* dV = aux;
    double* dtau = dV + vsz;
    double* dbeta = dtau + std::max(kmax, 1);
    double* slots = dbeta + std::max(kmax, 1);
    double* deps = slots + 2 * G;
    cb.zero(dV, vsz);
    cb.run(c);
    int* ints = (int*)dalloc(c, (2 * G + 2 + std::max<int64_t>(k, 1)) * sizeof(int));
    int* slotp = ints;
    int* dnk = ints + 2 * G;
    int* drank = dnk + 1;
    int* dperm = drank + 1;
    int hk[1] = {(int)k};
    CUDA_TRY(cudaMemcpyAsync(dnk, hk, sizeof(int), cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaMemcpyAsync(deps, &eps, sizeof(double), cudaMemcpyHostToDevice, c->st));
    sync(c);
    CpqrArgs a{};
    a.gmaps = (int*)dalloc(c, (size_t)G * 2 * std::max<int64_t>(k, 1) * sizeof(int));
    c->deferred.push_back((double*)a.gmaps);
    a.W = W; a.m = (int)m; a.ncols_cap = (int)std::max<int64_t>(k, 1); a.nk = dnk; a.eps = deps;
    a.min_rank = (int)min_rank; a.V = dV; a.tau = dtau; a.beta = dbeta; a.rank = drank;
    a.perm = dperm; a.slot_val = slots; a.slot_pos = slotp; a.finalize = 1;
    if (m > 0 && k > 0) {
      launch_cpqr(a, G, c->st);
    } else {
      int z = 0;
      CUDA_TRY(cudaMemcpyAsync(drank, &z, sizeof(int), cudaMemcpyHostToDevice, c->st));
    }
    int hr = 0;
    CUDA_TRY(cudaMemcpyAsync(&hr, drank, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    *rank = hr;
    std::vector<int> hp(std::max<int64_t>(k, 1));
    if (k) CUDA_TRY(cudaMemcpyAsync(hp.data(), dperm, k * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int64_t j = 0; j < k; ++j) perm[j] = hp[j];
    // Tred in pivoted order: column l = W[:, perm[l]]
    if (m * k) {
      double* Tp = dalloc(c, (size_t)(m * k) * sizeof(double));
      CopyBatch g;
      for (int64_t l = 0; l < k; ++l) {
        CopyTask t{};
        t.src = W + (int64_t)hp[l] * m; t.dst = Tp + l * m; t.nr = (int)m; t.nc = 1;
        t.lds = (int)m; t.ldd = (int)m;
        g.add(t);
      }
      g.run(c);
      to_host_rowmajor(c, Tp, m, k, m, Tred);
      dfree(c, Tp);
    }
    if (hr > 0) {
      to_host_rowmajor(c, dV, m, hr, m, V);
      CUDA_TRY(cudaMemcpyAsync(tau, dtau, hr * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    }
    sync(c);
    dfree(c, W); dfree(c, aux); dfree(c, ints);
    flush_deferred(c);
  });
}

int spq_tri_solve(spq_ctx* c, int64_t k, int64_t n, const double* R, const double* Cm, int side,
                  double* X) {
  return guarded(c, [&] {
    if (k == 0) return;
    // pivot rule (kernels/__init__.py:211-223) evaluated on the device
    CopyBatch cb;
    double* dR = to_dev_colmajor(c, R, k, k, cb);
    cb.run(c);
    PivotSet ps;
    ps.jobs.push_back(PivotJob{dR, (int)k, (int)k, 0});
    ps.ctx.push_back("");
    pivot_launch(c, ps);
    pivot_raise(c, ps);
    if (n == 0) { dfree(c, dR); flush_deferred(c); return; }
    if (side == 1) {
      // X R = C with C (n x k) row-major
      CopyBatch cb2;
      double* dC = to_dev_colmajor(c, Cm, n, k, cb2);
      cb2.run(c);
      std::vector<TrsmJob> tj{TrsmJob{dR, dC, (int)n, (int)k, (int)k, (int)n, 0}};
      launch_trsm_right(upload(c, tj), 1, trsm_tiles((int)n), c->st);
      to_host_rowmajor(c, dC, n, k, n, X);
      dfree(c, dC);
    } else {
      // R X = C  <=>  X^T R^T = C^T : solve column by column with the chain kernel
      CopyBatch cb2;
      double* dC = to_dev_colmajor(c, Cm, k, n, cb2);
      cb2.run(c);
      std::vector<int64_t> ids(k);
      std::iota(ids.begin(), ids.end(), 0);
      int* dids = upload_idx32(c, ids);
      chain_tri(dR, (int)k, nullptr, 0, dC, dids, nullptr, k, (int)n, 0, nullptr, c->st);
      to_host_rowmajor(c, dC, k, n, k, X);
      dfree(c, dC);
    }
    dfree(c, dR);
    flush_deferred(c);
  });
}

int spq_build_t(spq_ctx* c, int64_t m, int64_t k, const double* V, const double* tau,
                double* T) {
  return guarded(c, [&] {
    if (k == 0) return;
    CopyBatch cb;
    double* dV = to_dev_colmajor(c, V, m, k, cb);
    double* aux = dalloc(c, (size_t)(k + 2 * k * k) * sizeof(double));
    cb.run(c);
    double* dtau = aux;
    double* G = aux + k;
    double* dT = G + k * k;
    CUDA_TRY(cudaMemcpyAsync(dtau, tau, k * sizeof(double), cudaMemcpyHostToDevice, c->st));
    (void)G;
    build_full_T(c, {TProb{dV, (int)m, (int)k, dtau, dT}});
    to_host_rowmajor(c, dT, k, k, k, T);
    dfree(c, dV);
    dfree(c, aux);
    flush_deferred(c);
  });
}

int spq_bench_gemm(spq_ctx* c, int m, int n, int k, int transA, int reps, float* ms) {
  return guarded(c, [&] {
    const size_t na = (size_t)m * k, nb = (size_t)k * n, nc = (size_t)m * n;
    double* buf = dalloc(c, (na + nb + nc) * sizeof(double));
    CUDA_TRY(cudaMemsetAsync(buf, 0, (na + nb + nc) * sizeof(double), c->st));
    double* A = buf;
    double* B = A + na;
    double* C = B + nb;
    const int lda = transA ? k : m;
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    for (int r = -1; r < reps; ++r) {
      if (r == 0) CUDA_TRY(cudaEventRecord(e0, c->st));
      GemmBatch g;
      g.add(A, lda, B, k, C, m, m, n, k, -1.0, 1.0);
      g.run(c, transA != 0, 0);
    }
    CUDA_TRY(cudaEventRecord(e1, c->st));
    sync(c);
    CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
    *ms /= std::max(reps, 1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(c, buf);
  });
}

// BASELINE config 2: nb independent blocks B_i (m_i x k_i, k_i <= m_i) and
// companions C_i (m_i x c_i), all packed column-major; R_i (k_i x k_i) out,
// C_i <- H_i^T C_i in place.  ms = device time of QR + apply.
int spq_batched_qr(spq_ctx* c, int nb, const int64_t* m, const int64_t* k, const int64_t* nc,
                   const double* B, double* R, double* C, float* ms) {
  return guarded(c, [&] {
    size_t nB = 0, nR = 0, nC = 0, nT = 0, nt = 0;
    for (int i = 0; i < nb; ++i) {
      if (k[i] > m[i]) throw SpqError(SPQ_ERR_BAD_INPUT, "batched_qr needs m >= k");
      nB += m[i] * k[i]; nR += k[i] * k[i]; nC += m[i] * nc[i]; nT += k[i] * k[i]; nt += k[i];
    }
    double* dB = dalloc(c, std::max<size_t>(nB, 1) * 8);
    double* dR = dalloc(c, std::max<size_t>(nR, 1) * 8);
    double* dC = dalloc(c, std::max<size_t>(nC, 1) * 8);
    double* dT = dalloc(c, std::max<size_t>(nT + nt, 1) * 8);
    CUDA_TRY(cudaMemcpyAsync(dB, B, nB * 8, cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaMemcpyAsync(dC, C, nC * 8, cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaMemsetAsync(dR, 0, std::max<size_t>(nR, 1) * 8, c->st));
    CUDA_TRY(cudaMemsetAsync(dT, 0, std::max<size_t>(nT + nt, 1) * 8, c->st));
    std::vector<QrProb> qp;
    size_t ob = 0, orr = 0, oc = 0, ot = 0;
    for (int i = 0; i < nb; ++i) {
      QrProb q{dB + ob, (int)m[i], (int)k[i], dR + orr, dT + nT + ot, dT + orr, {}};
      if (nc[i] > 0) q.targets.push_back(CTarget{dC + oc, (int)m[i], (int)nc[i]});
      qp.push_back(std::move(q));
      ob += m[i] * k[i]; orr += k[i] * k[i]; oc += m[i] * nc[i]; ot += k[i];
    }
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, c->st));
    qr_batch(c, qp);
    CUDA_TRY(cudaEventRecord(e1, c->st));
    CUDA_TRY(cudaMemcpyAsync(R, dR, nR * 8, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaMemcpyAsync(C, dC, nC * 8, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(c, dB); dfree(c, dR); dfree(c, dC); dfree(c, dT);
  });
}

// BASELINE config 2 (RRQR set): nb blocks M_i (m x n, packed column-major),
// threshold CPQR with the relative rule nrm < eps*norm0 (rrqr_threshold).
// ranks out; rdiag (nb x min(m,n)) |R_ii| of the accepted steps; ms device.
int spq_batched_rrqr(spq_ctx* c, int nb, int64_t m, int64_t n, const double* M, double eps,
                     int64_t* ranks, double* rdiag, float* ms) {
  return guarded(c, [&] {
    const int kmax = (int)std::min(m, n);
    const size_t blk = (size_t)m * n;
    if (cpqr_cta_smem((int)m, (int)n) > CPQR_CTA_MAX_SMEM)
      throw SpqError(SPQ_ERR_BAD_INPUT, "batched_rrqr block too large for the CTA-resident kernel");
    double* dM = dalloc(c, std::max<size_t>(nb * blk, 1) * 8);
    double* dV = dalloc(c, std::max<size_t>((size_t)nb * m * kmax, 1) * 8);
    double* dtb = dalloc(c, std::max<size_t>((size_t)nb * 2 * kmax + 1, 1) * 8);
    int* di = (int*)dalloc(c, std::max<size_t>((size_t)nb * (n + 1), 1) * 4);
    CUDA_TRY(cudaMemcpyAsync(dM, M, nb * blk * 8, cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaMemsetAsync(dV, 0, std::max<size_t>((size_t)nb * m * kmax, 1) * 8, c->st));
    double* deps = dtb + (size_t)nb * 2 * kmax;
    CUDA_TRY(cudaMemcpyAsync(deps, &eps, 8, cudaMemcpyHostToDevice, c->st));
    std::vector<CpqrJob> jobs(nb);
    for (int i = 0; i < nb; ++i) {
      CpqrJob& q = jobs[i];
      q.W = dM + i * blk; q.m = (int)m; q.n = (int)n; q.ncap = (int)n; q.ldw = (int)m;
      q.nk = nullptr; q.eps = deps; q.min_rank = 0; q.V = dV + (size_t)i * m * kmax;
      q.ldv = (int)m; q.tau = dtb + (size_t)i * 2 * kmax; q.beta = q.tau + kmax;
      q.rank = di + (size_t)nb * n + i; q.perm = di + (size_t)i * n; q.write_back = 0;
    }
    const CpqrJob* dj = upload(c, jobs);
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, c->st));
    launch_cpqr_cta(dj, nb, cpqr_cta_smem((int)m, (int)n), c->st);
    CUDA_TRY(cudaEventRecord(e1, c->st));
    std::vector<int> hr(nb);
    std::vector<double> htb((size_t)nb * 2 * kmax);
    CUDA_TRY(cudaMemcpyAsync(hr.data(), di + (size_t)nb * n, nb * 4, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaMemcpyAsync(htb.data(), dtb, htb.size() * 8, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int i = 0; i < nb; ++i) {
      ranks[i] = hr[i];
      for (int j = 0; j < kmax; ++j)
        rdiag[(size_t)i * kmax + j] = j < hr[i] ? htb[(size_t)i * 2 * kmax + kmax + j] : 0.0;
    }
    dfree(c, dM); dfree(c, dV); dfree(c, dtb); dfree(c, di);
  });
}

}  // extern "C"
