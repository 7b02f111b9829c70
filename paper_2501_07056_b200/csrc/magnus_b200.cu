// Host side of the C-ABI (include/magnus_b200.h): plans, launches, workspace.
//
// Reference boundary: spgemm_magnus / magnus_symbolic / magnus_numeric
// (magnus.py:420-583).  One context holds the per-call device state between
// the symbolic and numeric phases, like the reference keeps `stats`, `cats`
// and the plans between the two calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/magnus_b200.h"
#include "baselines.cuh"
#include <nvtx3/nvToolsExt.h>

#include "big_direct.cuh"
#include "fused_big.cuh"
#include "coarse_rows.cuh"
#include "radix_sort.cuh"
#include "binned_rows.cuh"
#include "microbench.cuh"
#include "common.cuh"
#include "dense_rows.cuh"
#include "direct_rows.cuh"
#include "heavy_rows.cuh"
#include "setup_kernels.cuh"
#include "small_rows.cuh"
#include "symbolic_rows.cuh"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#ifdef MG_DIR_DEBUG
#define DIR_SYNC(what)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = cudaStreamSynchronize(s);                                                \
    fprintf(stderr, "[dir] %s: %s\n", what, cudaGetErrorString(e_));                           \
  } while (0)
#else
#define DIR_SYNC(what) do { } while (0)
#endif

// NVTX ranges around the phases and the heavy-row batches (visible in Nsight Systems / Compute;
// nvtx3 is header-only and a no-op without an attached tool).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// MAGNUS_TRACE=1: host timestamps of magnus_setup's steps on stderr (synchronising)
static void trace_point(cudaStream_t s, const char* what) {
  static const bool on = [] { const char* e = std::getenv("MAGNUS_TRACE"); return e && std::strcmp(e, "1") == 0; }();
  if (!on) return;
  static auto t0 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  fprintf(stderr, "[trace] %10.3f ms  %s\n", ms, what);
}

#define MG_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return set_err(MAGNUS_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

// The library's device workspace comes from a private stream-ordered pool per device (never
// the default pool: the process's other allocators are left alone).  Freed workspace stays
// reserved in the pool between calls (no re-mapping of tens of GB per call) until
// magnus_release_workspace() trims it.
cudaMemPool_t workspace_pool() {
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[dev] = p;
  }
  return pools[dev];
}

cudaError_t mg_malloc_async(void** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = workspace_pool();
  if (!pool) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

int64_t ceil_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
int64_t exact_log2(int64_t x) {
  int64_t k = 0;
  while ((int64_t(1) << k) < x) ++k;
  return k;
}
// util.py:28-44
int64_t round_pow2_of_sqrt(unsigned __int128 num, unsigned __int128 den) {
  if (num < den) return 1;
  int k = 0;
  while (num >= (den << (2 * (k + 1)))) ++k;
  if (num >= (den << (2 * k + 1))) ++k;
  return int64_t(1) << k;
}

mg::DevCsr dev_csr(const magnus_csr& m) {
  mg::DevCsr d;
  d.n_rows = m.n_rows;
  d.n_cols = m.n_cols;
  d.nnz = m.nnz;
  d.rp64 = m.rp_bytes == 8 ? static_cast<const int64_t*>(m.row_ptr) : nullptr;
  d.rp32 = m.rp_bytes == 4 ? static_cast<const int32_t*>(m.row_ptr) : nullptr;
  d.col = m.col;
  d.val = m.val;
  d.skip = nullptr;
  return d;
}

}  // namespace

struct magnus_ctx {
  int device = 0;
  int sm_count = 148;
  int64_t launches = 0;
  std::vector<void*> allocs;   // per-setup device allocations
  cudaStream_t stream = nullptr;

  mg::DevCsr A{}, B{};
  magnus_sys sys{};
  magnus_thresholds th{};
  magnus_chunk_plan plan_sym{}, plan_num{};
  int force_fine_only = 0;
  bool ready = false;
  bool have_symbolic = false;

  int64_t* inter = nullptr;
  int64_t* mn = nullptr;
  int64_t* mx = nullptr;
  int8_t* cat = nullptr;
  int32_t* listW = nullptr;
  int32_t* listB = nullptr;
  int32_t* listH = nullptr;
  int32_t* listCoarse = nullptr;
  int32_t* listD = nullptr;
  unsigned long long* stats = nullptr;   // kStatLen
  unsigned long long* work = nullptr;    // work counters (4)
  unsigned long long* err = nullptr;
  int64_t* counts = nullptr;
  int64_t* tile_sums = nullptr;
  uint32_t* skip = nullptr;
  uint32_t* modebits = nullptr;
  uint32_t* gk = nullptr;
  uint32_t* gchunk = nullptr;
  int64_t gk_stride = 0;
  // binned heavy path (binned_rows.cuh)
  bool binned = false;
  int gshift = 0;        // column bin shift (bins nest in the numeric-plan chunks)
  int64_t ncnt = 0;      // per-CTA chunk/bin counters of the heavy symbolic kernel
  int64_t* choff = nullptr;   // per heavy row: first chunk-table entry (nH + 1)
  int64_t* hbase = nullptr;   // per heavy row: exclusive prefix of the stream sizes (nH + 1)
  int64_t* nent = nullptr;
  int64_t* hinter = nullptr;
  uint32_t* ce = nullptr;     // chunk tables: element prefix / distinct-column prefix
  // direct big-chunk path (big_direct.cuh, MAGNUS_BIG_PATH=direct)
  bool big_direct = false;
  bool big_fused = false;     // big chunks by k_fu_sweep (fused_big.cuh, MAGNUS_BIG_PATH=fused)
  bool coarse_dev = false;    // Coarse-category heavy rows through the device coarse level (coarse_rows.cuh)
  int64_t c4_rows = 0, c4_batches = 0, c4_brows = 0;   // last numeric call: coarse rows / batches / CSC entries
  uint32_t* cs = nullptr;     // numeric phase: small-chunk element prefix (big chunks excluded)
  int64_t* hbase_s = nullptr;   // numeric phase: exclusive prefix of the heavy rows' small-chunk products
  std::vector<int64_t> h_small;
  // caller-owned workspace for the heavy rows' reorder buffer (magnus_set_workspace)
  unsigned char* ws_ptr = nullptr;
  int64_t ws_bytes = 0;
  // fused warp rows (k_rows_warp Mode 2 in the symbolic pass, k_rows_copy in the numeric pass)
  bool fused = false;
  int64_t* fused_ub = nullptr;
  uint32_t* fused_col = nullptr;
  double* fused_val = nullptr;
  uint32_t* cd = nullptr;
  uint32_t* cbm_slot = nullptr;   // per chunk entry: slot of its column bitmap in cbm_pool (big chunks)
  uint32_t* cbm_pool = nullptr;
  uint64_t cbm_cap = 0;
  std::vector<int64_t> h_hinter, h_nent;
  std::vector<int32_t> h_rows;   // heavy rows, ascending
  // host readback overlapped with the numeric phase (magnus_numeric_host)
  uint32_t* host_col = nullptr;
  double* host_val = nullptr;
  int64_t host_done = 0;
  int64_t total_ent = 0;
  // direct heavy path (direct_rows.cuh)
  bool direct = false;
  bool sym2 = false;   // heavy symbolic: k_heavy_sym2 (symbolic_rows.cuh)
  int sym2_occ = 1;
  int dir_wlog = 0;
  int dir_occ = 1;
  int64_t dir_nwin1 = 0, dir_min_len = 0, dir_nidx = 0, kst_stride = 0;
  int32_t* bslot = nullptr;
  uint32_t* bidx = nullptr;
  unsigned long long* kst = nullptr;
  cudaStream_t aux = nullptr, aux2 = nullptr, aux3 = nullptr;   // concurrent pipelines
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_e[2] = {nullptr, nullptr}, ev_r[2] = {nullptr, nullptr}, ev_b[2] = {nullptr, nullptr};
  cudaEvent_t ev_pl[2] = {nullptr, nullptr}, ev_it[2] = {nullptr, nullptr};   // batch plan done / plan consumed
  int64_t host_stats[mg::kStatLen] = {0};
  int64_t coarse_batches = 0;
  mg::Sem sem{};
  // profiling telemetry
  bool profile = false;
  struct Mark { int kernel; cudaEvent_t a, b; };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> event_pool;

  cudaEvent_t get_event() {
    if (!event_pool.empty()) { cudaEvent_t e = event_pool.back(); event_pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
  }
  // bracket one launch: call begin() before and end() after (on the launch's stream)
  int pending = -1; cudaEvent_t pend_a = nullptr;
  void begin(int kernel) {
    ++launches;
    if (!profile) return;
    pend_a = get_event(); pending = kernel;
    cudaEventRecord(pend_a, stream);
  }
  void end() {
    if (!profile || pending < 0) return;
    cudaEvent_t b = get_event();
    cudaEventRecord(b, stream);
    marks.push_back({pending, pend_a, b});
    pending = -1;
  }
  // the same for a launch on another stream (concurrent pipelines)
  cudaEvent_t begin_on(int kernel, cudaStream_t st) {
    ++launches;
    if (!profile) return nullptr;
    cudaEvent_t a = get_event();
    cudaEventRecord(a, st);
    (void)kernel;
    return a;
  }
  void end_on(int kernel, cudaEvent_t a, cudaStream_t st) {
    if (!profile || !a) return;
    cudaEvent_t b = get_event();
    cudaEventRecord(b, st);
    marks.push_back({kernel, a, b});
  }

  void free_all() {
    for (void* p : allocs) cudaFreeAsync(p, stream);
    allocs.clear();
  }
  // B-derived state (validation, skip list, window index) kept across setups with the same B:
  // the row waves of one product (waves.py) re-run setup per block of A against one B
  std::vector<void*> b_allocs;
  struct BKey {
    const void* rp = nullptr;
    const void* col = nullptr;
    const void* val = nullptr;
    int64_t n_rows = -1, n_cols = -1, nnz = -1;
    int32_t rp_bytes = 0;
    bool operator==(const BKey& o) const {
      return rp == o.rp && col == o.col && val == o.val && n_rows == o.n_rows && n_cols == o.n_cols && nnz == o.nnz &&
             rp_bytes == o.rp_bytes;
    }
  } bkey;
  bool b_validated = false;
  int bidx_wlog = -1;
  int64_t bidx_minreq = -1;
  void free_b() {
    for (void* p : b_allocs) cudaFreeAsync(p, stream);
    b_allocs.clear();
    b_validated = false;
    bidx_wlog = -1;
    bidx_minreq = -1;
    skip = nullptr;
    bslot = nullptr;
    bidx = nullptr;
  }
  template <class T>
  cudaError_t balloc(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = mg_malloc_async(&q, std::max<size_t>(count, 1) * sizeof(T), stream);
    if (e == cudaSuccess) b_allocs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }
  template <class T>
  cudaError_t alloc(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = mg_malloc_async(&q, std::max<size_t>(count, 1) * sizeof(T), stream);
    if (e == cudaSuccess) allocs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }
};

extern "C" {

const char* magnus_last_error(void) { return g_err.c_str(); }
const char* magnus_version(void) { return "magnus_b200 0.1 (sm_100a)"; }
int64_t magnus_launch_count(magnus_ctx* ctx) { return ctx ? ctx->launches : 0; }

int magnus_workspace_bytes(magnus_ctx* ctx, int64_t* preferred, int64_t* minimum) {
  if (!ctx || !preferred || !minimum) return set_err(MAGNUS_INPUT, "null argument");
  if (!ctx->ready || !ctx->have_symbolic) return set_err(MAGNUS_CONTRACT, "magnus_workspace_bytes needs magnus_symbolic first");
  int64_t total = 0, max_row = 0;
  if (ctx->binned && !ctx->direct && !ctx->big_direct)
    for (int64_t h : ctx->h_hinter) {
      total += h;
      max_row = std::max(max_row, h);
    }
  *preferred = total ? total * 10 + 256 : 0;   // one batch: u16 column + f64 product per heavy-row product
  *minimum = max_row ? max_row * 10 + 256 : 0;
  return MAGNUS_OK;
}

int magnus_set_workspace(magnus_ctx* ctx, void* ws, int64_t bytes) {
  if (!ctx) return set_err(MAGNUS_INPUT, "null argument");
  if ((ws == nullptr) != (bytes == 0) || bytes < 0) return set_err(MAGNUS_INPUT, "workspace pointer and size disagree");
  ctx->ws_ptr = static_cast<unsigned char*>(ws);
  ctx->ws_bytes = bytes;
  return MAGNUS_OK;
}

int magnus_release_workspace(void) {
  cudaMemPool_t pool = workspace_pool();
  if (!pool) return set_err(MAGNUS_CUDA, "no workspace pool");
  MG_CUDA(cudaDeviceSynchronize());
  MG_CUDA(cudaMemPoolTrimTo(pool, 0));
  return MAGNUS_OK;
}

int64_t magnus_workspace_reserved(void) {
  cudaMemPool_t pool = workspace_pool();
  uint64_t r = 0;
  if (pool) cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r);
  return (int64_t)r;
}

int magnus_profile_enable(magnus_ctx* ctx, int enable) {
  if (!ctx) return set_err(MAGNUS_INPUT, "null argument");
  ctx->profile = enable != 0;
  return MAGNUS_OK;
}

int magnus_profile_read(magnus_ctx* ctx, double* ms, int64_t* launches) {
  if (!ctx || !ms || !launches) return set_err(MAGNUS_INPUT, "null argument");
  for (int k = 0; k < MAGNUS_K_COUNT; ++k) { ms[k] = 0.0; launches[k] = 0; }
  for (auto& m : ctx->marks) {
    MG_CUDA(cudaEventSynchronize(m.b));
    float t = 0.f;
    MG_CUDA(cudaEventElapsedTime(&t, m.a, m.b));
    ms[m.kernel] += t;
    launches[m.kernel] += 1;
    ctx->event_pool.push_back(m.a);
    ctx->event_pool.push_back(m.b);
  }
  ctx->marks.clear();
  return MAGNUS_OK;
}

int magnus_coarse_level_stats(magnus_ctx* ctx, int64_t* out3) {
  if (!ctx || !out3) return set_err(MAGNUS_INPUT, "null argument");
  out3[0] = ctx->c4_rows;
  out3[1] = ctx->c4_batches;
  out3[2] = ctx->c4_brows;
  return MAGNUS_OK;
}

int magnus_heavy_stats(magnus_ctx* ctx, int64_t* out4) {
  if (!ctx || !out4) return set_err(MAGNUS_INPUT, "null argument");
  for (int q = 0; q < 4; ++q) out4[q] = 0;
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  if (!ctx->ready || !ctx->have_symbolic || !ctx->binned || nH == 0) return MAGNUS_OK;
  unsigned long long* d = nullptr;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&d), 32, ctx->stream));
  MG_CUDA(cudaMemsetAsync(d, 0, 32, ctx->stream));
  mg::k_heavy_stats<<<(unsigned)std::min<int64_t>((nH + 7) / 8, (int64_t)ctx->sm_count * 8), 256, 0, ctx->stream>>>(
      ctx->listH, nH, ctx->mn, ctx->mx, (int)ctx->sem.shift_num, ctx->choff, ctx->ce, ctx->cd, d);
  MG_CUDA(cudaGetLastError());
  unsigned long long h[4];
  MG_CUDA(cudaMemcpyAsync(h, d, 32, cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaFreeAsync(d, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int q = 0; q < 4; ++q) out4[q] = (int64_t)h[q];
  return MAGNUS_OK;
}

// compute_chunk_plan planner.py:106-152
int magnus_compute_chunk_plan(const magnus_sys* sys, int64_t m_c, int numeric, int allow_coarse, magnus_chunk_plan* out) {
  if (!sys || !out) return set_err(MAGNUS_INPUT, "null argument");
  if (m_c < 1) return set_err(MAGNUS_INPUT, "m_c must be >= 1");
  if (sys->cache_line_bytes <= 0 || sys->l2_bytes <= 0 || sys->memory_budget_bytes <= 0 || sys->histo_type_bytes <= 0 ||
      sys->prefix_sum_type_bytes <= 0 || sys->val_bytes <= 0)
    return set_err(MAGNUS_INPUT, "SystemParams fields must be positive");
  if (sys->cache_line_bytes & (sys->cache_line_bytes - 1)) return set_err(MAGNUS_INPUT, "cache_line_bytes must be a power of two");
  const int64_t plan_cols = ceil_pow2(m_c);
  const int64_t sda = numeric ? sys->val_bytes + 1 : 1;
  const int64_t scf = sys->histo_type_bytes + sys->prefix_sum_type_bytes + 2 * sys->cache_line_bytes;
  const unsigned __int128 raw =
      (unsigned __int128)sys->l2_bytes * (unsigned __int128)sys->l2_bytes / (unsigned __int128)(4 * scf);
  int64_t m_max = 1;
  if (raw >= 1) {
    unsigned __int128 p = 1;
    while ((p << 1) <= raw) p <<= 1;
    m_max = (int64_t)p;
  }
  const int use_coarse = allow_coarse && plan_cols > m_max;
  const int64_t span = use_coarse ? m_max : plan_cols;
  int64_t n_fine = round_pow2_of_sqrt((unsigned __int128)span * sda, scf);
  const int64_t min_len = std::max<int64_t>(1, sys->cache_line_bytes / 4);
  n_fine = std::min(n_fine, std::max<int64_t>(1, span / min_len));
  n_fine = std::max<int64_t>(1, std::min(n_fine, span));
  const int64_t len = span / n_fine;
  out->plan_cols = plan_cols;
  out->s_dense_accum = sda;
  out->s_chunk_fine = scf;
  out->n_chunks_fine = n_fine;
  out->chunk_len_fine = len;
  out->shift_fine = exact_log2(len);
  out->m_max_l2 = m_max;
  out->use_coarse = use_coarse;
  out->n_chunks_coarse = use_coarse ? plan_cols / m_max : 1;
  out->chunk_len_coarse = use_coarse ? m_max : plan_cols;
  out->shift_coarse = exact_log2(out->chunk_len_coarse);
  return MAGNUS_OK;
}

int magnus_ctx_create(magnus_ctx** out) {
  if (!out) return set_err(MAGNUS_INPUT, "null argument");
  auto* c = new magnus_ctx();
  MG_CUDA(cudaGetDevice(&c->device));
  MG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
  if (!workspace_pool()) return set_err(MAGNUS_CUDA, "cudaMemPoolCreate failed");
  MG_CUDA(cudaFuncSetAttribute(mg::k_rows_block<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mg::kBSmem));
  MG_CUDA(cudaFuncSetAttribute(mg::k_rows_block<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mg::kBSmem));
  MG_CUDA(cudaFuncSetAttribute(mg::k_rows_dense<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::DenseRowSmem::kTotal));
  MG_CUDA(cudaFuncSetAttribute(mg::k_rows_dense<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::DenseRowSmem::kTotal));
  MG_CUDA(cudaFuncSetAttribute(mg::k_heavy_symbolic, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::HeavySymSmem::kTotal));
  MG_CUDA(cudaFuncSetAttribute(mg::k_heavy_numeric, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::HeavyNumSmem::kTotal));
  MG_CUDA(cudaFuncSetAttribute(mg::k_bin_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(mg::bin_reduce_warp_smem(mg::kBinMaxShift) * (mg::kBinT / 32))));
  MG_CUDA(cudaFuncSetAttribute(mg::k_bin_big<mg::kBigD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::bin_big_smem(mg::kBinMaxShift, mg::kBigD)));
  MG_CUDA(cudaFuncSetAttribute(mg::k_bin_big<mg::kBigDWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::bin_big_smem(mg::kBinMaxShift, mg::kBigDWide)));
  MG_CUDA(cudaFuncSetAttribute(mg::k_bd_num<mg::kBigD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(mg::bd_warp_smem(mg::kBinMaxShift, mg::kBigD) * mg::kBdW)));
  MG_CUDA(cudaFuncSetAttribute(mg::k_bd_num<mg::kBigDWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(mg::bd_warp_smem(mg::kBinMaxShift, mg::kBigDWide) * mg::kBdW)));
  MG_CUDA(cudaFuncSetAttribute(mg::k_c4_fine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(4 * sizeof(uint32_t) << mg::kC4MaxFineLog)));
  MG_CUDA(cudaFuncSetAttribute(mg::k_fu_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mg::FuSmem::kTotal));
  MG_CUDA(cudaFuncSetAttribute(mg::k_bin_expand2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::Exp2Smem::kTotal));
  MG_CUDA(cudaFuncSetAttribute(mg::k_heavy_sym2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)mg::Sym2Smem::kTotal));
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->sym2_occ, mg::k_heavy_sym2, mg::kS2T, mg::Sym2Smem::kTotal));
  c->sym2_occ = std::max(1, std::min(c->sym2_occ, 7));
  MG_CUDA(cudaFuncSetAttribute(mg::k_dir_num, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(mg::DirSmem::kWarp * mg::kDirNW)));


  {
    // the pairwise summation keeps an explicit recursion stack (common.cuh)
    size_t stack = 0;
    MG_CUDA(cudaDeviceGetLimit(&stack, cudaLimitStackSize));
    if (stack < 2048) MG_CUDA(cudaDeviceSetLimit(cudaLimitStackSize, 2048));
  }
  MG_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  MG_CUDA(cudaStreamCreateWithFlags(&c->aux2, cudaStreamNonBlocking));
  MG_CUDA(cudaStreamCreateWithFlags(&c->aux3, cudaStreamNonBlocking));
  MG_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  MG_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  for (int q = 0; q < 2; ++q) {
    MG_CUDA(cudaEventCreateWithFlags(&c->ev_e[q], cudaEventDisableTiming));
    MG_CUDA(cudaEventCreateWithFlags(&c->ev_r[q], cudaEventDisableTiming));
    MG_CUDA(cudaEventCreateWithFlags(&c->ev_b[q], cudaEventDisableTiming));
    MG_CUDA(cudaEventCreateWithFlags(&c->ev_pl[q], cudaEventDisableTiming));
    MG_CUDA(cudaEventCreateWithFlags(&c->ev_it[q], cudaEventDisableTiming));
  }
  *out = c;
  return MAGNUS_OK;
}

void magnus_ctx_destroy(magnus_ctx* ctx) {
  if (!ctx) return;
  ctx->free_all();
  ctx->free_b();
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& m : ctx->marks) { cudaEventDestroy(m.a); cudaEventDestroy(m.b); }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->aux2) cudaStreamDestroy(ctx->aux2);
  if (ctx->aux3) cudaStreamDestroy(ctx->aux3);
  for (int q = 0; q < 2; ++q) {
    if (ctx->ev_e[q]) cudaEventDestroy(ctx->ev_e[q]);
    if (ctx->ev_r[q]) cudaEventDestroy(ctx->ev_r[q]);
    if (ctx->ev_b[q]) cudaEventDestroy(ctx->ev_b[q]);
    if (ctx->ev_pl[q]) cudaEventDestroy(ctx->ev_pl[q]);
    if (ctx->ev_it[q]) cudaEventDestroy(ctx->ev_it[q]);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

int magnus_row_stats(const magnus_csr* A, const magnus_csr* B, int64_t* inter, int64_t* min_col, int64_t* max_col,
                     void* stream) {
  if (!A || !B) return set_err(MAGNUS_INPUT, "null argument");
  if (A->n_cols != B->n_rows) return set_err(MAGNUS_INPUT, "dimension mismatch");
  if (A->n_rows == 0) return MAGNUS_OK;
  int dev = 0, sms = 148;
  MG_CUDA(cudaGetDevice(&dev));
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // four rows per warp when A's rows are short (<= 12 nonzeros on average)
  const bool short_rows = A->nnz <= 12 * A->n_rows;
  const int64_t lanes = std::min<int64_t>(A->n_rows * (short_rows ? 8 : 32), (int64_t)sms * 64 * 32);
  const unsigned grid = (unsigned)((lanes + 255) / 256);
  if (short_rows)
    mg::k_row_stats<8><<<grid, 256, 0, (cudaStream_t)stream>>>(dev_csr(*A), dev_csr(*B), inter, min_col, max_col);
  else
    mg::k_row_stats<32><<<grid, 256, 0, (cudaStream_t)stream>>>(dev_csr(*A), dev_csr(*B), inter, min_col, max_col);
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

// Direct heavy path: B window index (long rows) and per-warp cursor scratch.
// B window index (direct_rows.cuh k_didx_*): for B rows of at least kDirIdxMinLen entries,
// the position of the first column >= g << wlog for every g.  Replaces the binary searches
// of segment bounds at window / unit boundaries by one load.
static int setup_bidx(magnus_ctx* ctx, int wlog, int64_t min_len_req) {
  cudaStream_t s = ctx->stream;
  const mg::DevCsr& B = ctx->B;
  if (ctx->bidx && ctx->bidx_wlog == wlog && ctx->bidx_minreq == min_len_req) return MAGNUS_OK;   // same B
  if (ctx->bidx) {   // same B, other granularity: rebuild
    for (void* q : {static_cast<void*>(ctx->bslot), static_cast<void*>(ctx->bidx)}) {
      auto it = std::find(ctx->b_allocs.begin(), ctx->b_allocs.end(), q);
      if (it != ctx->b_allocs.end()) ctx->b_allocs.erase(it);
      MG_CUDA(cudaFreeAsync(q, s));
    }
    ctx->bslot = nullptr;
    ctx->bidx = nullptr;
  }
  ctx->bidx_wlog = wlog;
  ctx->bidx_minreq = min_len_req;
  ctx->dir_wlog = wlog;
  const int64_t W = int64_t(1) << ctx->dir_wlog;
  ctx->dir_nwin1 = (std::max<int64_t>(B.n_cols, 1) + W - 1) / W + 1;
  unsigned long long* dbuf = nullptr;
  MG_CUDA(ctx->alloc(&dbuf, 48));
  MG_CUDA(cudaMemsetAsync(dbuf, 0, 48 * 8, s));
  const unsigned g = (unsigned)std::min<int64_t>((B.n_rows + 255) / 256 + 1, (int64_t)ctx->sm_count * 8);
  ctx->begin(MAGNUS_K_DIR_INDEX);
  mg::k_didx_hist<<<g, 256, 0, s>>>(B, dbuf);
  ctx->end();
  unsigned long long hist[40];
  MG_CUDA(cudaMemcpyAsync(hist, dbuf, sizeof hist, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  // shortest indexed row: >= kDirIdxMinLen, and the index within ~1 GB
  const int64_t cap_bytes = int64_t(1) << 30;
  int b = 0;
  while ((int64_t(1) << b) < min_len_req) ++b;
  for (;; ++b) {
    int64_t rows_ge = 0;
    for (int q = b; q < 40; ++q) rows_ge += (int64_t)hist[q];
    if (rows_ge * ctx->dir_nwin1 * 4 <= cap_bytes || b >= 39) break;
  }
  ctx->dir_min_len = int64_t(1) << b;
  MG_CUDA(ctx->balloc(&ctx->bslot, B.n_rows + 1));
  ctx->begin(MAGNUS_K_DIR_INDEX);
  mg::k_didx_slots<<<g, 256, 0, s>>>(B, ctx->dir_min_len, ctx->bslot, dbuf + 40);
  ctx->end();
  unsigned long long nidx = 0;
  MG_CUDA(cudaMemcpyAsync(&nidx, dbuf + 40, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  ctx->dir_nidx = (int64_t)nidx;
  MG_CUDA(ctx->balloc(&ctx->bidx, (size_t)std::max<int64_t>(1, ctx->dir_nidx) * ctx->dir_nwin1));
  if (nidx > 0) {
    ctx->begin(MAGNUS_K_DIR_INDEX);
    mg::k_didx_fill<<<(unsigned)std::min<int64_t>(((int64_t)nidx * 32 + 255) / 256, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
        B, ctx->bslot, ctx->dir_wlog, ctx->dir_nwin1, ctx->bidx);
    ctx->end();
    DIR_SYNC("index fill");
    MG_CUDA(cudaGetLastError());
  }
  return MAGNUS_OK;
}

static int setup_direct(magnus_ctx* ctx) {
  int rc = setup_bidx(ctx, std::min(mg::kDirLog, (int)ctx->sem.shift_num), mg::kDirIdxMinLen);
  if (rc) return rc;
  const size_t smem = mg::DirSmem::kWarp * mg::kDirNW;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->dir_occ, mg::k_dir_num, 32 * mg::kDirNW, smem));
  ctx->dir_occ = std::max(ctx->dir_occ, 1);
  const int64_t maxnk = ctx->host_stats[mg::kStatMaxNk];
  ctx->kst_stride = ((std::max<int64_t>(maxnk, 1) + 31) / 32) * 32;
  const size_t warps = (size_t)ctx->sm_count * ctx->dir_occ * mg::kDirNW;
  MG_CUDA(ctx->alloc(&ctx->kst, warps * (size_t)ctx->kst_stride * 2));
  return MAGNUS_OK;
}

// Heavy rows, numeric phase, direct path.
static int launch_direct(magnus_ctx* ctx, const int64_t* c_rp, uint32_t* c_col, double* c_val) {
  cudaStream_t s = ctx->stream;
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  const int64_t cap = std::max<int64_t>(ctx->total_ent, 1);
  void* items = nullptr;
  unsigned long long* cnt = nullptr;
  MG_CUDA(mg_malloc_async(&items, (size_t)cap * sizeof(mg::DirItem), s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&cnt), 64, s));
  MG_CUDA(cudaMemsetAsync(cnt, 0, 64, s));
  ctx->begin(MAGNUS_K_DIR_PLAN);
  mg::k_dir_plan<<<(unsigned)std::min<int64_t>((nH + 7) / 8, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
      ctx->listH, nH, ctx->mn, ctx->mx, ctx->sem.shift_num, ctx->choff, ctx->ce, mg::kDirItem,
      static_cast<mg::DirItem*>(items), cnt, cap);
  ctx->end();
  DIR_SYNC("plan");
  ctx->begin(MAGNUS_K_DIR_NUM);
  mg::k_dir_num<<<(unsigned)(ctx->sm_count * ctx->dir_occ), 32 * mg::kDirNW, mg::DirSmem::kWarp * mg::kDirNW, s>>>(
      ctx->A, ctx->B, ctx->listH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->dir_wlog, ctx->choff, ctx->ce, ctx->cd,
      static_cast<const mg::DirItem*>(items), cnt, cnt + 2, cap, ctx->bslot, ctx->bidx, ctx->dir_nwin1, ctx->kst,
      ctx->kst_stride, c_rp, c_col, c_val, ctx->err);
  ctx->end();
  DIR_SYNC("num");
  MG_CUDA(cudaGetLastError());
  MG_CUDA(cudaFreeAsync(items, s));
  MG_CUDA(cudaFreeAsync(cnt, s));
  return MAGNUS_OK;
}

// Device check of both operands (k_validate); err[1] collects the flags.  Out-of-range columns
// of B are the reference's ContractViolation (magnus.py:208-209, 245-246); malformed row_ptr,
// A columns outside B's rows and non-canonical rows are InputError (validate_csr).
static int validate_inputs(magnus_ctx* ctx, const magnus_csr& A, const magnus_csr& B, cudaStream_t s) {
  const bool same = A.row_ptr == B.row_ptr && A.col == B.col && A.n_rows == B.n_rows;
  auto launch = [&](const magnus_csr& m, unsigned long long* f) {
    const bool short_rows = m.nnz <= 12 * m.n_rows;   // four rows per warp
    const int64_t lanes =
        std::max<int64_t>(32, std::min<int64_t>(m.n_rows * (short_rows ? 8 : 32), (int64_t)ctx->sm_count * 64 * 32));
    const unsigned grid = (unsigned)((lanes + 255) / 256);
    if (short_rows) mg::k_validate<8><<<grid, 256, 0, s>>>(dev_csr(m), f);
    else mg::k_validate<32><<<grid, 256, 0, s>>>(dev_csr(m), f);
    ++ctx->launches;
  };
  unsigned long long* fb = nullptr;
  MG_CUDA(ctx->alloc(&fb, 2));
  MG_CUDA(cudaMemsetAsync(fb, 0, 16, s));
  launch(A, fb);
  if (!same && !ctx->b_validated) launch(B, fb + 1);
  MG_CUDA(cudaGetLastError());
  unsigned long long h[2] = {0, 0};
  MG_CUDA(cudaMemcpyAsync(h, fb, 16, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  if (same) h[1] = h[0];
  auto bad = [](const char* which, unsigned long long f) -> std::string {
    std::string m = std::string(which) + ": ";
    if (f & 1) return m + "row_ptr is not a valid CSR row pointer (row_ptr[0] != 0, decreasing, or row_ptr[-1] != nnz)";
    if (f & 2) return m + "column index out of range";
    return m + "columns not strictly increasing within a row (non-canonical input: sort each row and sum "
               "duplicates first; the device path requires canonical rows)";
  };
  if (h[0] & 1) return set_err(MAGNUS_INPUT, bad("A", h[0]));
  if (h[1] & 1) return set_err(MAGNUS_INPUT, bad("B", h[1]));
  if (h[0] & 2) return set_err(MAGNUS_INPUT, bad("A", 2) + " (A column >= B.n_rows)");
  if (h[1] & 2) return set_err(MAGNUS_CONTRACT, "column index outside the planned fine-level span (B column >= n_cols)");
  if (h[0] & 4) return set_err(MAGNUS_INPUT, bad("A", 4));
  if (h[1] & 4) return set_err(MAGNUS_INPUT, bad("B", 4));
  ctx->b_validated = true;
  return MAGNUS_OK;
}

int magnus_setup(magnus_ctx* ctx, const magnus_csr* A, const magnus_csr* B, const magnus_sys* sys,
                 const magnus_thresholds* th, int force_fine_only, void* stream) {
  if (!ctx || !A || !B || !sys || !th) return set_err(MAGNUS_INPUT, "null argument");
  NvtxRange nvtx_range("magnus_setup");
  if (A->n_cols != B->n_rows)   // _check_dims gustavson.py:39-41
    return set_err(MAGNUS_INPUT, "dimension mismatch: A is " + std::to_string(A->n_rows) + "x" + std::to_string(A->n_cols) +
                                     ", B is " + std::to_string(B->n_rows) + "x" + std::to_string(B->n_cols));
  if ((A->rp_bytes != 4 && A->rp_bytes != 8) || (B->rp_bytes != 4 && B->rp_bytes != 8))
    return set_err(MAGNUS_INPUT, "row_ptr must be int32 or int64");
  if (B->nnz >= (int64_t(1) << 32) || A->n_rows >= (int64_t(1) << 31))
    return set_err(MAGNUS_INPUT, "device limits: nnz(B) < 2^32 and n_rows(A) < 2^31");
  if (B->n_cols > (int64_t(1) << 32)) return set_err(MAGNUS_INPUT, "more than 2^32 columns needs 8-byte column indices");
  if (th->sort_dense_crossover < 1 || th->sort_sweet_spot > th->sort_dense_crossover)
    return set_err(MAGNUS_INPUT, "invalid AccumThresholds");
  if (th->sort_dense_crossover > mg::kCap)
    return set_err(MAGNUS_INPUT, "sort_dense_crossover above the device batch capacity (" + std::to_string(mg::kCap) + ")");
  trace_point(ctx->stream ? ctx->stream : (cudaStream_t)stream, "setup: enter");
  ctx->free_all();
  // per-setup allocations are gone: no pointer may survive into this setup
  ctx->cbm_slot = ctx->cbm_pool = nullptr;
  ctx->cbm_cap = 0;
  ctx->kst = nullptr;
  {
    magnus_ctx::BKey k;
    k.rp = B->row_ptr;
    k.col = B->col;
    k.val = B->val;
    k.n_rows = B->n_rows;
    k.n_cols = B->n_cols;
    k.nnz = B->nnz;
    k.rp_bytes = B->rp_bytes;
    if (!(k == ctx->bkey)) {
      ctx->stream = (cudaStream_t)stream;
      ctx->free_b();
      ctx->bkey = k;
    }
  }
  ctx->ce = ctx->cd = nullptr;
  ctx->direct = ctx->binned = false;
  ctx->fused = false;
  ctx->fused_ub = nullptr;
  ctx->fused_col = nullptr;
  ctx->fused_val = nullptr;
  ctx->stream = (cudaStream_t)stream;
  cudaStream_t s = ctx->stream;
  ctx->A = dev_csr(*A);
  ctx->B = dev_csr(*B);
  ctx->sys = *sys;
  ctx->th = *th;
  ctx->force_fine_only = force_fine_only;
  ctx->ready = false;
  ctx->have_symbolic = false;
  const int64_t m_c = std::max<int64_t>(B->n_cols, 1);   // magnus.py:565
  int rc = magnus_compute_chunk_plan(sys, m_c, 0, !force_fine_only, &ctx->plan_sym);
  if (rc) return rc;
  rc = magnus_compute_chunk_plan(sys, m_c, 1, !force_fine_only, &ctx->plan_num);
  if (rc) return rc;
  const int64_t n = A->n_rows;
  MG_CUDA(ctx->alloc(&ctx->inter, n + 1));
  MG_CUDA(ctx->alloc(&ctx->mn, n + 1));
  MG_CUDA(ctx->alloc(&ctx->mx, n + 1));
  MG_CUDA(ctx->alloc(&ctx->cat, n + 1));
  MG_CUDA(ctx->alloc(&ctx->listW, n + 1));
  MG_CUDA(ctx->alloc(&ctx->listB, n + 1));
  MG_CUDA(ctx->alloc(&ctx->listH, n + 1));
  MG_CUDA(ctx->alloc(&ctx->listCoarse, n + 1));
  MG_CUDA(ctx->alloc(&ctx->listD, n + 1));
  MG_CUDA(ctx->alloc(&ctx->stats, mg::kStatLen));
  MG_CUDA(ctx->alloc(&ctx->work, 8));
  MG_CUDA(ctx->alloc(&ctx->err, 2));
  MG_CUDA(cudaMemsetAsync(ctx->stats, 0, mg::kStatLen * 8, s));
  MG_CUDA(cudaMemsetAsync(ctx->err, 0, 16, s));
  {
    // input contract before anything indexes through A or B (validate_csr matrix.py:119-150)
    int rc0 = validate_inputs(ctx, *A, *B, s);
    if (rc0) return rc0;
  }
  if (!ctx->skip) {
    const int64_t nskip = (B->nnz + 31) / 32;
    MG_CUDA(ctx->balloc(&ctx->skip, nskip + 1));
    if (nskip > 0) {
      mg::k_build_skip<<<(unsigned)std::min<int64_t>((nskip + 255) / 256, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
          B->col, B->nnz, ctx->skip);
      MG_CUDA(cudaGetLastError());
      ++ctx->launches;
    }
  }
  ctx->B.skip = ctx->skip;
  if (A->row_ptr == B->row_ptr && A->col == B->col) ctx->A.skip = ctx->skip;
  if (n > 0) {
    ctx->begin(MAGNUS_K_ROW_STATS);
    rc = magnus_row_stats(A, B, ctx->inter, ctx->mn, ctx->mx, stream);
    ctx->end();
    if (rc) return rc;
    mg::CatParams cp{th->sort_dense_crossover, sys->l2_bytes, sys->val_bytes, (int32_t)ctx->plan_sym.use_coarse};
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sm_count * 16);
    ctx->begin(MAGNUS_K_CATEGORIZE);
    mg::k_categorize<<<grid, 256, 0, s>>>(n, ctx->A, ctx->inter, ctx->mn, ctx->mx, cp, ctx->cat, ctx->listW, ctx->listB,
                                          ctx->listH, ctx->listCoarse, ctx->listD, ctx->stats);
    ctx->end();
    MG_CUDA(cudaGetLastError());
  }
  trace_point(s, "setup: stats + categorize");
  unsigned long long hs[mg::kStatLen];
  MG_CUDA(cudaMemcpyAsync(hs, ctx->stats, sizeof hs, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  for (int j = 0; j < mg::kStatLen; ++j) ctx->host_stats[j] = (int64_t)hs[j];
  // build_coarse_batches (magnus.py:277-314): batch count and the over-budget error.
  ctx->coarse_batches = 0;
  const int64_t ncoarse = ctx->host_stats[mg::kStatNCoarse];
  if (ncoarse > 0) {
    // (row, inter) of every coarse row: one device gather + two copies, then the reference's
    // ascending row order on the host
    std::vector<int32_t> rows(ncoarse);
    std::vector<int64_t> inter(ncoarse);
    {
      int64_t* g = nullptr;
      MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&g), (size_t)ncoarse * 8, s));
      mg::k_gather_i64<<<(unsigned)std::min<int64_t>((ncoarse + 255) / 256, (int64_t)ctx->sm_count * 8), 256, 0, s>>>(
          ctx->inter, ctx->listCoarse, ncoarse, g);
      ++ctx->launches;
      MG_CUDA(cudaGetLastError());
      std::vector<int64_t> gi(ncoarse);
      MG_CUDA(cudaMemcpyAsync(rows.data(), ctx->listCoarse, ncoarse * 4, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaMemcpyAsync(gi.data(), g, ncoarse * 8, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaFreeAsync(g, s));
      MG_CUDA(cudaStreamSynchronize(s));
      std::vector<int64_t> order(ncoarse);
      for (int64_t j = 0; j < ncoarse; ++j) order[j] = j;
      std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return rows[x] < rows[y]; });
      std::vector<int32_t> r2(ncoarse);
      for (int64_t j = 0; j < ncoarse; ++j) { r2[j] = rows[order[j]]; inter[j] = gi[order[j]]; }
      rows.swap(r2);
    }
    const int64_t ncc = ctx->plan_sym.n_chunks_coarse, budget = sys->memory_budget_bytes;
    const int64_t bpe = (B->n_cols <= (int64_t(1) << 32) ? 4 : 8) + sys->val_bytes;   // magnus.py:414-417
    int64_t cur_n = 0, cur_bytes = 0, cur_meta = 0, nb = 0;
    for (int64_t j = 0; j < ncoarse; ++j) {
      const int64_t isz = inter[j], row_bytes = isz * bpe;
      if (row_bytes > budget)
        return set_err(MAGNUS_OVER_BUDGET, "row " + std::to_string(rows[j]) + ": buffering " + std::to_string(isz) +
                                               " intermediate elements needs " + std::to_string(row_bytes) +
                                               " bytes, over the " + std::to_string(budget) + "-byte memory budget");
      const int64_t meta = ncc * sys->histo_type_bytes + (ncc + 1) * sys->prefix_sum_type_bytes +
                           2 * sys->cache_line_bytes * std::min(ncc, isz);
      if (cur_n && (cur_bytes + row_bytes > budget || cur_meta + meta > sys->l2_bytes)) {
        ++nb;
        cur_n = cur_bytes = cur_meta = 0;
      }
      ++cur_n;
      cur_bytes += row_bytes;
      cur_meta += meta;
    }
    if (cur_n) ++nb;
    ctx->coarse_batches = nb;
  }
  // device semantics
  ctx->sem.crossover = th->sort_dense_crossover;
  ctx->sem.shift_num = (int32_t)ctx->plan_num.shift_fine;
  // numeric-plan fine chunks over the whole column span (n_fine per coarse chunk x n_coarse):
  // the chunk of column c is c >> shift_fine in both the fine and the coarse level.
  const int64_t n_chunks_global = ctx->plan_num.plan_cols >> ctx->plan_num.shift_fine;
  ctx->sem.n_chunks_num = n_chunks_global;
  ctx->sem.mode_words = (int32_t)((n_chunks_global + 31) / 32);
  trace_point(s, "setup: coarse batches");
  // heavy-row workspace
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  MG_CUDA(ctx->alloc(&ctx->counts, n + 1));
  MG_CUDA(ctx->alloc(&ctx->tile_sums, (n + mg::kScanTile - 1) / mg::kScanTile + 1));
  if (nH > 1) {
    // heavy rows in ascending row order (stable compaction instead of k_categorize's atomic
    // order): batches then complete contiguous row ranges (the host readback overlaps them)
    // and their contents do not depend on atomic order
    int64_t* pos = nullptr;
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&pos), (size_t)(n + 1) * 8, s));
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sm_count * 16);
    mg::k_heavy_flags<<<g, 256, 0, s>>>(ctx->inter, n, ctx->counts);
    const int64_t tiles = (n + mg::kScanTile - 1) / mg::kScanTile;
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->counts, n, ctx->tile_sums);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(ctx->tile_sums, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->counts, n, ctx->tile_sums, pos);
    mg::k_heavy_scatter<<<g, 256, 0, s>>>(ctx->inter, pos, n, ctx->listH);
    ctx->launches += 5;
    MG_CUDA(cudaGetLastError());
    MG_CUDA(cudaFreeAsync(pos, s));
  }
  ctx->h_rows.resize(nH);
  if (nH > 0) {
    MG_CUDA(cudaMemcpyAsync(ctx->h_rows.data(), ctx->listH, nH * 4, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
  }
  trace_point(s, "setup: heavy rows sorted");
  MG_CUDA(ctx->alloc(&ctx->modebits, std::max<int64_t>(1, nH) * ctx->sem.mode_words));
  const int64_t maxnk = ctx->host_stats[mg::kStatMaxNk];
  ctx->gk_stride = maxnk > mg::kKSN ? ((maxnk + 8) / 4) * 4 : 4;
  MG_CUDA(ctx->alloc(&ctx->gk, (size_t)2 * ctx->sm_count * ctx->gk_stride * 7));
  // binned heavy path: chunk width <= 2^14 and every big chunk dense (crossover <= kBinE)
  ctx->binned = nH > 0 && ctx->sem.shift_num <= mg::kBinMaxShift && th->sort_dense_crossover <= mg::kBinE;
  {
    // the binned path by default; MAGNUS_HEAVY_PATH=direct selects the direct path (no reorder
    // buffer; bit-identical results, slower on skewed inputs -- DESIGN.md)
    const char* hp = std::getenv("MAGNUS_HEAVY_PATH");
    const bool want_direct = hp && std::strcmp(hp, "direct") == 0;
    ctx->direct = ctx->binned && want_direct && ctx->sem.shift_num <= mg::kDirMaxShift &&
                  th->sort_dense_crossover <= mg::kDirList && B->n_cols < (int64_t(1) << 32);
  }
  {
    const char* sp = std::getenv("MAGNUS_HEAVY_SYMBOLIC");
    ctx->sym2 = ctx->binned && !(sp && std::strcmp(sp, "window") == 0) &&
                (ctx->plan_num.plan_cols >> ctx->sem.shift_num) + 1 <= mg::kS2Chunks;
  }
  {
    // big chunks straight from B (big_direct.cuh) instead of through the reorder buffer:
    // opt-in (MAGNUS_BIG_PATH=direct; bit-identical, measured slower on cfg3 -- DESIGN.md)
    const char* bp = std::getenv("MAGNUS_BIG_PATH");
    const bool want_fused = bp && std::strcmp(bp, "fused") == 0;
    ctx->big_fused = ctx->binned && !ctx->direct && want_fused && ctx->sem.shift_num <= mg::kFuMaxShift;
    ctx->big_direct = ctx->binned && !ctx->direct && ((bp && std::strcmp(bp, "direct") == 0) || ctx->big_fused);
  }
  {
    // Coarse-category rows: the coarse level (Alg. 4, coarse_rows.cuh) ahead of the chunk reducers;
    // MAGNUS_COARSE_PATH=fine sends them through the fine-level expand like every other heavy row
    const char* cp = std::getenv("MAGNUS_COARSE_PATH");
    const int64_t csl = ctx->plan_num.shift_coarse - ctx->plan_num.shift_fine;
    ctx->coarse_dev = ctx->binned && !ctx->direct && !ctx->big_direct && ctx->plan_sym.use_coarse && !force_fine_only &&
                      !(cp && std::strcmp(cp, "fine") == 0) && ctx->plan_num.n_chunks_coarse <= mg::kC4MaxCoarse &&
                      csl >= 0 && csl <= mg::kC4MaxFineLog && ctx->plan_num.shift_coarse < 32 &&
                      ctx->host_stats[mg::kStatNCoarse] > 0;
  }
  ctx->gshift = mg::bin_shift_of(ctx->sem.shift_num);
  ctx->ncnt = ctx->binned ? (ctx->plan_num.plan_cols >> ctx->gshift) : n_chunks_global;
  const bool chunk_global = ctx->ncnt > mg::kChunkSmem;
  const size_t gchunk_n = (size_t)ctx->sm_count * mg::kSymCtas * ctx->ncnt * 2;
  MG_CUDA(ctx->alloc(&ctx->gchunk, chunk_global ? gchunk_n : 1));
  if (chunk_global) MG_CUDA(cudaMemsetAsync(ctx->gchunk, 0, gchunk_n * 4, s));
  if (ctx->binned) {
    MG_CUDA(ctx->alloc(&ctx->nent, nH));
    MG_CUDA(ctx->alloc(&ctx->hinter, nH));
    MG_CUDA(ctx->alloc(&ctx->choff, nH + 1));
    MG_CUDA(ctx->alloc(&ctx->hbase, nH + 1));
    mg::k_bin_prep<<<(unsigned)std::min<int64_t>((nH + 255) / 256, (int64_t)ctx->sm_count * 8), 256, 0, s>>>(
        ctx->listH, nH, ctx->inter, ctx->mn, ctx->mx, ctx->gshift, ctx->nent, ctx->hinter);
    const int64_t tiles = (nH + mg::kScanTile - 1) / mg::kScanTile;
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->nent, nH, ctx->tile_sums);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(ctx->tile_sums, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->nent, nH, ctx->tile_sums, ctx->choff);
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->hinter, nH, ctx->tile_sums);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(ctx->tile_sums, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->hinter, nH, ctx->tile_sums, ctx->hbase);
    ctx->launches += 7;
    MG_CUDA(cudaGetLastError());
    ctx->h_hinter.resize(nH);
    ctx->h_nent.resize(nH);
    int64_t total_ent = 0;
    MG_CUDA(cudaMemcpyAsync(ctx->h_hinter.data(), ctx->hinter, nH * 8, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(ctx->h_nent.data(), ctx->nent, nH * 8, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(&total_ent, ctx->choff + nH, 8, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    ctx->total_ent = total_ent;
    MG_CUDA(ctx->alloc(&ctx->ce, total_ent));
    MG_CUDA(ctx->alloc(&ctx->cd, total_ent));
    // column bitmaps of big chunks (> kBinE elements), written by the symbolic pass: at most
    // sum(inter) / (kBinE + 1) of them; the pool is capped (chunks beyond it are marked again)
    // (only where the symbolic kernel writes them: chunks wider than 32 bitmap words)
    if (!ctx->direct && ctx->gshift == ctx->sem.shift_num && ctx->sem.shift_num > 10) {
      int64_t tot_inter = 0;
      for (int64_t h = 0; h < nH; ++h) tot_inter += ctx->h_hinter[h];
      const int64_t wpc = int64_t(1) << (ctx->sem.shift_num - 5);
      ctx->cbm_cap = (uint64_t)std::min<int64_t>(tot_inter / (mg::kBinE + 1) + 1, (int64_t(4) << 30) / (wpc * 4));
      MG_CUDA(ctx->alloc(&ctx->cbm_slot, total_ent));
      MG_CUDA(ctx->alloc(&ctx->cbm_pool, (size_t)ctx->cbm_cap * wpc));
    }
  }
  trace_point(s, "setup: chunk tables allocated");
  if (ctx->direct) {
    int rc2 = setup_direct(ctx);
    if (rc2) return rc2;
  } else if (ctx->binned) {
    // expand units start and end on sub-bin boundaries; the direct big-chunk kernel looks up
    // every (k, chunk) segment here: there rows down to 2 entries are indexed
    int rc2 = setup_bidx(ctx, ctx->gshift, ctx->big_direct && !ctx->big_fused ? 2 : mg::kDirIdxMinLen);
    if (rc2) return rc2;
  }
  trace_point(s, "setup: B window index");
  ctx->ready = true;
  return MAGNUS_OK;
}

int magnus_categories(magnus_ctx* ctx, int8_t* dst, void* stream) {
  if (!ctx || !ctx->ready) return set_err(MAGNUS_CONTRACT, "magnus_setup has not run");
  if (ctx->A.n_rows) MG_CUDA(cudaMemcpyAsync(dst, ctx->cat, ctx->A.n_rows, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return MAGNUS_OK;
}

// Coarse level of one batch of heavy rows [h0, h1) (coarse_level_batch magnus.py:379-406): the
// Coarse-category rows' products, reordered by (row, coarse chunk) from a CSC view of their A
// rows with every referenced B row read once (build_coarse_chunks magnus.py:317-376), then the
// fine level per bucket into the reorder buffer (bcol, bval) the chunk reducers read.
static int coarse_level_batch(magnus_ctx* ctx, int64_t h0, int64_t h1, int64_t batch_base, int64_t batch_elems,
                              uint16_t* bcol, double* bval, bool* handled) {
  *handled = false;
  cudaStream_t s = ctx->stream;
  const mg::DevCsr& A = ctx->A;
  const mg::DevCsr& B = ctx->B;
  const int64_t nB = B.n_rows;
  mg::C4Geom g;
  g.sf = (int)ctx->plan_num.shift_fine;
  g.sc = (int)ctx->plan_num.shift_coarse;
  g.ncc = (int)ctx->plan_num.n_chunks_coarse;
  g.h0 = h0;
  int32_t* list = nullptr;
  int64_t *apos = nullptr, *colcnt = nullptr, *colptr = nullptr;
  unsigned long long *colcur = nullptr, *cnt = nullptr;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&list), (size_t)(h1 - h0 + 1) * 4, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&apos), (size_t)(h1 - h0 + 1) * 8, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&colcnt), (size_t)(nB + 1) * 8, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&colptr), (size_t)(nB + 2) * 8, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&colcur), (size_t)(nB + 1) * 8, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&cnt), 64, s));
  MG_CUDA(cudaMemsetAsync(colcnt, 0, (size_t)(nB + 1) * 8, s));
  MG_CUDA(cudaMemsetAsync(colcur, 0, (size_t)(nB + 1) * 8, s));
  MG_CUDA(cudaMemsetAsync(cnt, 0, 64, s));
  const unsigned gw = (unsigned)std::min<int64_t>((h1 - h0 + 7) / 8, (int64_t)ctx->sm_count * 16);
  ctx->begin(MAGNUS_K_BIN_PLAN);
  mg::k_c4_rows<<<gw, 256, 0, s>>>(A, ctx->listH, ctx->cat, h0, h1, list, apos, cnt, colcnt);
  ctx->end();
  unsigned long long hc[2] = {0, 0};
  MG_CUDA(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  const int64_t nlist = (int64_t)hc[0], nnz_a = (int64_t)hc[1];
  int rc = MAGNUS_OK;
  // (A nonzeros are numbered in 32 bits, and the segment-position table holds one entry per
  // (A nonzero, coarse chunk): beyond 4 GB of it the fine-level expand takes the batch)
  const bool fits = nnz_a < (int64_t(1) << 32) && nnz_a * (int64_t)g.ncc * 4 <= (int64_t(4) << 30);
  if (nlist > 0 && nnz_a > 0 && fits) {
    *handled = true;
    ctx->c4_rows += nlist;
    ctx->c4_brows += nnz_a;
    ++ctx->c4_batches;
    const int64_t tiles = (nB + mg::kScanTile - 1) / mg::kScanTile;
    int64_t* tsum = nullptr;
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&tsum), (size_t)(tiles + 1) * 8, s));
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(colcnt, nB, tsum);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(tsum, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(colcnt, nB, tsum, colptr);
    ctx->launches += 3;
    int32_t* csc_h = nullptr;
    uint32_t *csc_q = nullptr, *koff = nullptr, *ccol = nullptr;
    double *csc_a = nullptr, *cval = nullptr;
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&csc_h), (size_t)nnz_a * 4, s));
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&csc_q), (size_t)nnz_a * 4, s));
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&csc_a), (size_t)nnz_a * 8, s));
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&koff), (size_t)nnz_a * g.ncc * 4, s));
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&ccol), (size_t)std::max<int64_t>(batch_elems, 1) * 4, s));
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&cval), (size_t)std::max<int64_t>(batch_elems, 1) * 8, s));
    const unsigned gl = (unsigned)std::min<int64_t>((nlist + 7) / 8, (int64_t)ctx->sm_count * 16);
    ctx->begin(MAGNUS_K_BIN_PLAN);
    mg::k_c4_fill<<<gl, 256, 0, s>>>(A, ctx->listH, list, nlist, apos, h0, colptr, colcur, csc_h, csc_q, csc_a);
    mg::k_c4_koff<<<gl, 256, (size_t)8 * g.ncc * 4, s>>>(A, B, ctx->listH, list, nlist, apos, g, ctx->mn, ctx->mx, ctx->choff, ctx->ce,
                                     ctx->bslot, ctx->bidx, ctx->dir_nwin1, ctx->dir_wlog, koff, ctx->err);
    ctx->end();
    ++ctx->launches;
    // work items of the outer-product pass: (B row, 256 CSC entries); item pointers reuse colcnt / colcur
    int64_t* icnt = colcnt;
    int64_t* iptr = reinterpret_cast<int64_t*>(colcur);
    mg::k_c4_icount<<<(unsigned)std::min<int64_t>((nB + 255) / 256, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(B, colptr, icnt);
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(icnt, nB, tsum);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(tsum, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(icnt, nB, tsum, iptr);
    ctx->launches += 4;
    ctx->begin(MAGNUS_K_BIN_EXPAND);
    mg::k_c4_scatter<<<(unsigned)(ctx->sm_count * 4), mg::kC4T, mg::C4Smem::kTotal, s>>>(
        B, ctx->listH, g, ctx->mn, ctx->mx, ctx->choff, ctx->ce, ctx->hbase, batch_base, colptr, iptr, csc_h, csc_q, csc_a,
        koff, cnt + 2, ccol, cval);
    const size_t fsm = (size_t)4 * sizeof(uint32_t) << (g.sc - g.sf);
    mg::k_c4_fine<<<(unsigned)(ctx->sm_count * 8), 128, fsm, s>>>(ctx->listH, list, nlist, g, ctx->mn, ctx->mx, ctx->choff,
                                                                  ctx->ce, ctx->hbase, batch_base, ccol, cval, cnt + 3, bcol,
                                                                  bval);
    ctx->end();
    ++ctx->launches;
    if (cudaGetLastError() != cudaSuccess) rc = set_err(MAGNUS_CUDA, "coarse level launch failed");
    for (void* q : {(void*)tsum, (void*)csc_h, (void*)csc_q, (void*)csc_a, (void*)koff, (void*)ccol, (void*)cval})
      MG_CUDA(cudaFreeAsync(q, s));
  }
  for (void* q : {(void*)list, (void*)apos, (void*)colcnt, (void*)colptr, (void*)colcur, (void*)cnt})
    MG_CUDA(cudaFreeAsync(q, s));
  return rc;
}

// Heavy rows, numeric phase, binned path: batches of rows whose products fit the reorder buffer.
#ifndef MG_BATCH_FRAC_SERIAL
#define MG_BATCH_FRAC_SERIAL 0.3
#endif
static constexpr double kBatchFracSerial = MG_BATCH_FRAC_SERIAL;
static int launch_binned(magnus_ctx* ctx, const int64_t* c_rp, uint32_t* c_col, double* c_val) {
  cudaStream_t s = ctx->stream;
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  ctx->c4_rows = ctx->c4_batches = ctx->c4_brows = 0;
  int64_t max_row = 0, total = 0;
  for (int64_t h = 0; h < nH; ++h) {
    max_row = std::max(max_row, ctx->h_hinter[h]);
    total += ctx->h_hinter[h];
  }
  size_t free_b = 0, tot_b = 0;
  MG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
  {
    // memory the pool holds but does not use is available too
    cudaMemPool_t pool = workspace_pool();
    uint64_t reserved = 0, used = 0;
    MG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    MG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
    if (reserved > used) free_b += (size_t)(reserved - used);
  }
  const int64_t per_elem = 10;   // u16 local column + f64 product
  // the reducers run on the main stream after each batch's expand (measured faster than
  // overlapping them on side streams); MAGNUS_SERIAL=0 restores the concurrent pipeline,
  // which needs a second buffer set
  const char* serial_env = std::getenv("MAGNUS_SERIAL");
  const bool serial = !(serial_env && std::strcmp(serial_env, "0") == 0);
  // fraction of free HBM per buffer set (MAGNUS_BATCH_FRAC overrides; measured on cfg3)
  double frac = serial ? kBatchFracSerial : 0.2;
  if (const char* bf = std::getenv("MAGNUS_BATCH_FRAC")) {
    const double v = std::atof(bf);
    if (v > 0.0 && v < 0.9) frac = v;
  }
  int64_t cap = std::min<int64_t>(total, std::min<int64_t>((int64_t)(free_b * frac) / per_elem, int64_t(3) << 30));
  if (const char* ce = std::getenv("MAGNUS_BATCH_ELEMS")) {   // testing: force many heavy-row batches
    const long long v = std::atoll(ce);
    if (v > 0) cap = std::min<int64_t>(cap, (int64_t)v);
  }
  const bool own_ws = ctx->ws_ptr != nullptr && serial;   // caller-owned reorder buffer
  if (own_ws) {
    const int64_t ws_cap = (ctx->ws_bytes - 256) / per_elem;
    if (ws_cap < max_row)
      return set_err(MAGNUS_INPUT, "workspace of " + std::to_string(ctx->ws_bytes) + " bytes is below the minimum " +
                                       std::to_string(max_row * per_elem + 256) + " (magnus_workspace_bytes)");
    cap = std::min(total, ws_cap);
  }
  cap = std::max(cap, max_row);
  // batches [h0, h1) and the largest chunk-table span of a batch
  std::vector<int64_t> cuts{0};
  int64_t acc = 0, ent = 0, max_ent = 0;
  for (int64_t h = 0; h < nH; ++h) {
    if (acc + ctx->h_hinter[h] > cap && h > cuts.back()) {
      cuts.push_back(h);
      max_ent = std::max(max_ent, ent);
      acc = ent = 0;
    }
    acc += ctx->h_hinter[h];
    ent += ctx->h_nent[h];
  }
  cuts.push_back(nH);
  max_ent = std::max(max_ent, ent);
  int64_t buf_elems = 0;
  {
    int64_t a = 0;
    for (size_t b = 0; b + 1 < cuts.size(); ++b, a = 0) {
      for (int64_t h = cuts[b]; h < cuts[b + 1]; ++h) a += ctx->h_hinter[h];
      buf_elems = std::max(buf_elems, a);
    }
  }
  // two buffer sets when the expand of batch b+1 overlaps the reducers of batch b
  const int nbuf = (cuts.size() > 2 && !serial) ? 2 : 1;
  // two plan sets: batch b+1 is planned on a side stream while batch b computes
  const int nitem = cuts.size() > 2 ? 2 : 1;
  const int64_t max_big = std::max<int64_t>(max_ent, 1) * MG_BIG_WIDE_PARTS + buf_elems / mg::kBigSplit + 1;
  void *bcol[2] = {nullptr, nullptr}, *bval[2] = {nullptr, nullptr}, *items[2] = {nullptr, nullptr},
       *cnts[2] = {nullptr, nullptr};
  for (int q = 0; q < nbuf; ++q) {
    // (+64 bytes: bulk copies read 16-byte aligned supersets of a slice)
    if (own_ws) {   // values first (16-byte aligned), then the columns; 64 bytes slack each
      const uintptr_t base = (reinterpret_cast<uintptr_t>(ctx->ws_ptr) + 15) & ~uintptr_t(15);
      bval[q] = reinterpret_cast<void*>(base);
      bcol[q] = reinterpret_cast<void*>((base + (size_t)std::max<int64_t>(buf_elems, 1) * 8 + 64 + 15) & ~uintptr_t(15));
      continue;
    }
    MG_CUDA(mg_malloc_async(&bcol[q], (size_t)std::max<int64_t>(buf_elems, 1) * 2 + 64, s));
    MG_CUDA(mg_malloc_async(&bval[q], (size_t)std::max<int64_t>(buf_elems, 1) * 8 + 64, s));
  }
  for (int q = 0; q < nitem; ++q) {
    // windows and units: <= one per chunk entry; big-chunk parts: <= entries + elements / kBigSplit
    MG_CUDA(mg_malloc_async(&items[q], (size_t)std::max<int64_t>(max_ent, 1) * 3 * sizeof(mg::BinItem) +
                                           (size_t)max_big * 2 * sizeof(mg::BigItem), s));
    MG_CUDA(mg_malloc_async(&cnts[q], 128, s));
  }
  const size_t big_smem = mg::bin_big_smem(ctx->sem.shift_num, mg::kBigD);
  const size_t big_smem_w = mg::bin_big_smem(ctx->sem.shift_num, mg::kBigDWide);
  int occ_b = 1, occ_bw = 1;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, mg::k_bin_big<mg::kBigD>, 32, big_smem));
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_bw, mg::k_bin_big<mg::kBigDWide>, 32, big_smem_w));
  occ_b = std::max(occ_b, 1);
  occ_bw = std::max(occ_bw, 1);
  const size_t red_smem = mg::bin_reduce_warp_smem(ctx->sem.shift_num) * (mg::kBinT / 32);
  int occ = 1;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mg::k_bin_reduce, mg::kBinT, red_smem));
  int occ_e2 = 1;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_e2, mg::k_bin_expand2, mg::kE2T, mg::Exp2Smem::kTotal));
  occ_e2 = std::max(occ_e2, 1);
  uint32_t* e2scr = nullptr;   // per-CTA segment tables of units with more than kE2K k's
  const int64_t e2_stride = ((ctx->host_stats[mg::kStatMaxNk] + 8 + 3) / 4) * 4;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&e2scr), (size_t)ctx->sm_count * occ_e2 * 5 * e2_stride * 4, s));
  std::vector<int64_t> hb(cuts.size());
  {
    int64_t a = 0;
    size_t b = 0;
    for (int64_t h = 0; h <= nH; ++h) {
      while (b < cuts.size() && cuts[b] == h) hb[b++] = a;
      if (h < nH) a += ctx->h_hinter[h];
    }
  }
  // host readback: C offset of each batch's end row (the next batch's first heavy row)
  std::vector<int64_t> batch_end(cuts.size(), -1);
  if (ctx->host_col) {
    for (size_t b = 0; b + 2 < cuts.size(); ++b)
      MG_CUDA(cudaMemcpyAsync(&batch_end[b], c_rp + ctx->h_rows[cuts[b + 1]], 8, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
  }
  cudaStream_t sr = ctx->aux, sbig = ctx->aux2;
  if (serial) sr = sbig = s;
  bool used[2] = {false, false};
  // plan of batch b into plan set b % nitem, on stream st
  auto plan_batch = [&](size_t b, cudaStream_t st) {
    const int qi = (int)(b % nitem);
    const int64_t h0 = cuts[b], h1 = cuts[b + 1];
    mg::BinItem* wins = static_cast<mg::BinItem*>(items[qi]);
    mg::BinItem* units = wins + std::max<int64_t>(max_ent, 1);
    mg::BinItem* wins_t = units + std::max<int64_t>(max_ent, 1);
    mg::BigItem* bigs = reinterpret_cast<mg::BigItem*>(wins_t + std::max<int64_t>(max_ent, 1));
    auto* nwin = static_cast<unsigned long long*>(cnts[qi]);
    cudaMemsetAsync(cnts[qi], 0, 128, st);
    cudaEvent_t m0 = ctx->begin_on(MAGNUS_K_BIN_PLAN, st);
    mg::k_bin_plan<<<(unsigned)std::min<int64_t>((h1 - h0 + 7) / 8, (int64_t)ctx->sm_count * 16), 256, 0, st>>>(
        ctx->listH, h0, h1, ctx->mn, ctx->mx, ctx->sem.shift_num, ctx->choff, ctx->ce, wins, nwin, wins_t, bigs, nwin + 2,
        units, nwin + 1, std::max<int64_t>(max_ent, 1), max_big, ctx->cd, ctx->hbase, hb[b], c_rp, ctx->cbm_slot);
    ctx->end_on(MAGNUS_K_BIN_PLAN, m0, st);
  };
  plan_batch(0, s);
  for (size_t b = 0; b + 1 < cuts.size(); ++b) {
    NvtxRange nvtx_batch("magnus heavy-row batch");
    const int q = (int)(b % nbuf);
    const int qi = (int)(b % nitem);
    mg::BinItem* wins = static_cast<mg::BinItem*>(items[qi]);
    mg::BinItem* units = wins + std::max<int64_t>(max_ent, 1);
    mg::BinItem* wins_t = units + std::max<int64_t>(max_ent, 1);   // windows of tiny chunks (k_bin_reduce_tiny)
    mg::BigItem* bigs = reinterpret_cast<mg::BigItem*>(wins_t + std::max<int64_t>(max_ent, 1));
    auto* nwin = static_cast<unsigned long long*>(cnts[qi]);
    auto* nunit = nwin + 1;
    auto* nbig = nwin + 2;
    if (used[q]) {   // the reducers of batch b - nbuf still read this buffer set
      MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_r[q], 0));
      MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_b[q], 0));
    }
    used[q] = true;
    if (b > 0) MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_pl[qi], 0));   // this batch's plan (side stream)
    if (b + 2 < cuts.size()) {
      // plan batch b+1 beside this batch, once batch b-1 (the previous user of that set) is done
      const int qn = (int)((b + 1) % nitem);
      if (b > 0) MG_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_it[qn], 0));
      plan_batch(b + 1, ctx->aux);
      MG_CUDA(cudaEventRecord(ctx->ev_pl[qn], ctx->aux));
    }
    bool coarse_done = false;
    if (ctx->coarse_dev) {
      int rc4 = coarse_level_batch(ctx, cuts[b], cuts[b + 1], hb[b], hb[b + 1] - hb[b], static_cast<uint16_t*>(bcol[q]),
                                   static_cast<double*>(bval[q]), &coarse_done);
      if (rc4) return rc4;
    }
    ctx->begin(MAGNUS_K_BIN_EXPAND);
    mg::k_bin_expand2<<<(unsigned)(ctx->sm_count * occ_e2), mg::kE2T, mg::Exp2Smem::kTotal, s>>>(
        ctx->A, ctx->B, ctx->listH, ctx->mn, ctx->mx, ctx->sem.shift_num, ctx->choff, ctx->ce, ctx->hbase, hb[b], units,
        nunit, nwin + 3, std::max<int64_t>(max_ent, 1), static_cast<uint16_t*>(bcol[q]), static_cast<double*>(bval[q]),
        ctx->bslot, ctx->bidx, ctx->dir_nwin1, ctx->dir_wlog, e2scr, e2_stride, ctx->err,
        coarse_done ? ctx->cat : nullptr);
    ctx->end();
    MG_CUDA(cudaEventRecord(ctx->ev_e[q], s));
    // the big-chunk and small-chunk reducers of this batch run on their own streams
    MG_CUDA(cudaStreamWaitEvent(sbig, ctx->ev_e[q], 0));
    cudaEvent_t m1 = ctx->begin_on(MAGNUS_K_BIN_BIG, sbig);
    mg::k_bin_big<mg::kBigD><<<(unsigned)(ctx->sm_count * occ_b), 32, big_smem, sbig>>>(
        ctx->sem, bigs, nbig, nwin + 5, max_big, ctx->cbm_pool, static_cast<const uint16_t*>(bcol[q]),
        static_cast<const double*>(bval[q]), c_col, c_val, ctx->err);
    // chunks with more than kBigD distinct columns: one pass with a 4096-rank accumulator
    mg::k_bin_big<mg::kBigDWide><<<(unsigned)(ctx->sm_count * occ_bw), 32, big_smem_w, sbig>>>(
        ctx->sem, bigs + max_big, nwin + 10, nwin + 12, max_big, ctx->cbm_pool, static_cast<const uint16_t*>(bcol[q]),
        static_cast<const double*>(bval[q]), c_col, c_val, ctx->err);
    ctx->end_on(MAGNUS_K_BIN_BIG, m1, sbig);
    MG_CUDA(cudaEventRecord(ctx->ev_b[q], sbig));
    MG_CUDA(cudaStreamWaitEvent(sr, ctx->ev_e[q], 0));
    cudaEvent_t m2 = ctx->begin_on(MAGNUS_K_BIN_REDUCE, sr);
    mg::k_bin_reduce<<<(unsigned)(ctx->sm_count * occ), mg::kBinT, red_smem, sr>>>(
        ctx->listH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->choff, ctx->ce, ctx->cd, ctx->hbase, hb[b], wins, nwin,
        nwin + 4, static_cast<const uint16_t*>(bcol[q]), static_cast<const double*>(bval[q]), c_rp, c_col, c_val, ctx->err);
    ctx->end_on(MAGNUS_K_BIN_REDUCE, m2, sr);
    cudaEvent_t m3 = ctx->begin_on(MAGNUS_K_BIN_REDUCE, sr);
    mg::k_bin_reduce_tiny<<<(unsigned)(ctx->sm_count * 8), 256, 0, sr>>>(
        ctx->listH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->choff, ctx->ce, ctx->cd, ctx->hbase, hb[b], wins_t, nwin + 8,
        nwin + 9, static_cast<const uint16_t*>(bcol[q]), static_cast<const double*>(bval[q]), c_rp, c_col, c_val, ctx->err);
    ctx->end_on(MAGNUS_K_BIN_REDUCE, m3, sr);
    MG_CUDA(cudaEventRecord(ctx->ev_r[q], sr));
    MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_b[q], 0));
    MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_r[q], 0));
    MG_CUDA(cudaEventRecord(ctx->ev_it[qi], s));   // plan set qi free again
    MG_CUDA(cudaGetLastError());
    if (ctx->host_col && sr == s && sbig == s) {
      // rows below the next batch's first heavy row are complete (light rows ran first):
      // read that prefix of C back on the copy stream while the next batch computes
      const int64_t end = b + 2 < cuts.size() ? batch_end[b] : -1;
      if (end > ctx->host_done) {
        MG_CUDA(cudaEventRecord(ctx->ev_fork, s));
        MG_CUDA(cudaStreamWaitEvent(ctx->aux3, ctx->ev_fork, 0));
        MG_CUDA(cudaMemcpyAsync(ctx->host_col + ctx->host_done, c_col + ctx->host_done, (end - ctx->host_done) * 4,
                                cudaMemcpyDeviceToHost, ctx->aux3));
        MG_CUDA(cudaMemcpyAsync(ctx->host_val + ctx->host_done, c_val + ctx->host_done, (end - ctx->host_done) * 8,
                                cudaMemcpyDeviceToHost, ctx->aux3));
        ctx->host_done = end;
      }
    }
  }
  for (int q = 0; q < nbuf; ++q) {
    if (!used[q]) continue;
    MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_r[q], 0));
    MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_b[q], 0));
  }
  MG_CUDA(cudaFreeAsync(e2scr, s));
  for (int q = 0; q < nbuf; ++q) {
    if (own_ws) continue;
    MG_CUDA(cudaFreeAsync(bcol[q], s));
    MG_CUDA(cudaFreeAsync(bval[q], s));
  }
  for (int q = 0; q < nitem; ++q) {
    MG_CUDA(cudaFreeAsync(items[q], s));
    MG_CUDA(cudaFreeAsync(cnts[q], s));
  }
  return MAGNUS_OK;
}

// Big chunks of all heavy rows, straight from B (big_direct.cuh); also the small-chunk tables
// (cs, per-row small totals -> ctx->h_small, ctx->hbase_s) the binned small-chunk path uses.
static int launch_big_direct(magnus_ctx* ctx, const int64_t* c_rp, uint32_t* c_col, double* c_val) {
  cudaStream_t s = ctx->stream;
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  const int shift = ctx->sem.shift_num;
  const int64_t nchunks = std::max<int64_t>(ctx->sem.n_chunks_num, 1);
  unsigned long long* bucket = nullptr;   // 2 * nchunks counters + total
  int64_t* hsmall = nullptr;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&bucket), (size_t)(2 * nchunks + 8) * 8, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&hsmall), (size_t)std::max<int64_t>(nH, 1) * 8, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&ctx->cs), (size_t)std::max<int64_t>(ctx->total_ent, 1) * 4, s));
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&ctx->hbase_s), (size_t)(nH + 1) * 8, s));
  MG_CUDA(cudaMemsetAsync(bucket, 0, (size_t)(2 * nchunks + 8) * 8, s));
  const unsigned gp = (unsigned)std::min<int64_t>((nH + 7) / 8, (int64_t)ctx->sm_count * 16);
  // items chunk-major (default) or in arrival order (MAGNUS_BD_ORDER=arrival; tuning)
  const char* bo = std::getenv("MAGNUS_BD_ORDER");
  const bool bd_chunk_major = !(bo && std::strcmp(bo, "arrival") == 0);
  ctx->begin(MAGNUS_K_BIN_PLAN);
  mg::k_bd_plan<0><<<gp, 256, 0, s>>>(ctx->listH, nH, ctx->mn, ctx->mx, shift, ctx->choff, ctx->ce, ctx->cd,
                                      ctx->cbm_slot, c_rp, ctx->cs, hsmall, bucket, nchunks, nullptr, bd_chunk_major, ctx->big_fused);
  mg::k_bd_bucket_scan<<<1, 1024, 0, s>>>(bucket, 2 * nchunks, bucket + 2 * nchunks);
  {
    const int64_t tiles = (nH + mg::kScanTile - 1) / mg::kScanTile;
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(hsmall, nH, ctx->tile_sums);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(ctx->tile_sums, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(hsmall, nH, ctx->tile_sums, ctx->hbase_s);
  }
  ctx->end();
  ctx->launches += 4;
  MG_CUDA(cudaGetLastError());
  unsigned long long tots[2] = {0, 0};   // first wide item, all items
  ctx->h_small.resize(nH);
  MG_CUDA(cudaMemcpyAsync(&tots[0], bucket + nchunks, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaMemcpyAsync(&tots[1], bucket + 2 * nchunks, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaMemcpyAsync(ctx->h_small.data(), hsmall, nH * 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  const uint64_t n_narrow = tots[0], n_all = tots[1];
  if (n_all > 0) {
    mg::BdItem* items = nullptr;
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&items), (size_t)n_all * sizeof(mg::BdItem), s));
    int32_t* aslot = nullptr;   // B index slot per A nonzero (k_bd_aprep)
    uint32_t* abase = nullptr;  // B row start per A nonzero
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&aslot), (size_t)std::max<int64_t>(ctx->A.nnz, 1) * 4, s));
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&abase), (size_t)std::max<int64_t>(ctx->A.nnz, 1) * 4, s));
    if (ctx->big_fused) {
      mg::k_fu_aprep<<<(unsigned)std::min<int64_t>((ctx->A.nnz + 255) / 256 + 1, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
          ctx->A, ctx->B, ctx->bslot, aslot, abase);
    } else {
      mg::k_bd_aprep<<<(unsigned)std::min<int64_t>((ctx->A.nnz + 255) / 256 + 1, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
          ctx->A, ctx->B, ctx->bslot, aslot, abase);
    }
    ++ctx->launches;
    ctx->begin(MAGNUS_K_BIN_PLAN);
    mg::k_bd_plan<1><<<gp, 256, 0, s>>>(ctx->listH, nH, ctx->mn, ctx->mx, shift, ctx->choff, ctx->ce, ctx->cd,
                                        ctx->cbm_slot, c_rp, ctx->cs, hsmall, bucket, nchunks, items, bd_chunk_major,
                                        ctx->big_fused);
    ctx->end();
    MG_CUDA(cudaMemsetAsync(bucket + 2 * nchunks + 2, 0, 16, s));   // tickets
    if (ctx->big_fused) {
      int occ_f = 1;
      MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, mg::k_fu_sweep, mg::kFuT, mg::FuSmem::kTotal));
      occ_f = std::max(occ_f, 1);
      const unsigned grid_f = (unsigned)(ctx->sm_count * occ_f);
      // units: chunk ranges of ~kFuUnit big-chunk products
      int64_t tot_inter = 0;
      for (int64_t h = 0; h < nH; ++h) tot_inter += ctx->h_hinter[h];
      const int64_t cap_u = nH + tot_inter / mg::kFuUnit + 1;
      mg::BinItem* units = nullptr;
      unsigned long long* ucnt = nullptr;
      uint32_t* gst = nullptr;
      const int64_t maxnk = ctx->host_stats[mg::kStatMaxNk];
      const int64_t gst_stride = maxnk > mg::kFuKS ? ((maxnk + 31) / 32) * 32 : 0;
      MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&units), (size_t)cap_u * sizeof(mg::BinItem), s));
      MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&ucnt), 64, s));
      MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&gst), std::max<size_t>((size_t)grid_f * gst_stride * 2 * 4, 16), s));
      MG_CUDA(cudaMemsetAsync(ucnt, 0, 64, s));
      ctx->begin(MAGNUS_K_BIN_PLAN);
      mg::k_fu_plan<<<gp, 256, 0, s>>>(ctx->listH, nH, ctx->mn, ctx->mx, shift, ctx->choff, ctx->ce, units, ucnt, cap_u);
      ctx->end();
      ctx->begin(MAGNUS_K_BIN_BIG);
      mg::k_fu_sweep<<<grid_f, mg::kFuT, mg::FuSmem::kTotal, s>>>(
          ctx->A, ctx->B, ctx->listH, ctx->mn, ctx->mx, ctx->sem, ctx->choff, ctx->ce, ctx->cd, ctx->cbm_slot, ctx->cbm_pool,
          units, ucnt, cap_u, ucnt + 2, aslot, abase, ctx->bidx, ctx->dir_nwin1, ctx->dir_wlog, gst, gst_stride, c_rp, c_col,
          c_val, ctx->err);
      ctx->end();
      MG_CUDA(cudaGetLastError());
      MG_CUDA(cudaFreeAsync(units, s));
      MG_CUDA(cudaFreeAsync(ucnt, s));
      MG_CUDA(cudaFreeAsync(gst, s));
    } else {
    const size_t sm_n = mg::bd_warp_smem(shift, mg::kBigD) * mg::kBdW;
    const size_t sm_w = mg::bd_warp_smem(shift, mg::kBigDWide) * mg::kBdW;
    int occ_n = 1, occ_w = 1;
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_n, mg::k_bd_num<mg::kBigD>, 32 * mg::kBdW, sm_n));
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, mg::k_bd_num<mg::kBigDWide>, 32 * mg::kBdW, sm_w));
    occ_n = std::max(occ_n, 1);
    occ_w = std::max(occ_w, 1);
    ctx->begin(MAGNUS_K_BIN_BIG);
    if (n_narrow > 0)
      mg::k_bd_num<mg::kBigD><<<(unsigned)(ctx->sm_count * occ_n), 32 * mg::kBdW, sm_n, s>>>(
          ctx->A, ctx->B, ctx->listH, ctx->sem, items, n_narrow, bucket + 2 * nchunks + 2, ctx->cbm_pool, aslot, abase,
          ctx->bidx, ctx->dir_nwin1, ctx->dir_wlog, c_col, c_val, ctx->err);
    if (n_all > n_narrow)
      mg::k_bd_num<mg::kBigDWide><<<(unsigned)(ctx->sm_count * occ_w), 32 * mg::kBdW, sm_w, s>>>(
          ctx->A, ctx->B, ctx->listH, ctx->sem, items + n_narrow, n_all - n_narrow, bucket + 2 * nchunks + 3,
          ctx->cbm_pool, aslot, abase, ctx->bidx, ctx->dir_nwin1, ctx->dir_wlog, c_col, c_val, ctx->err);
    ctx->end();
    if (n_all > n_narrow) ++ctx->launches;
    MG_CUDA(cudaGetLastError());
    }
#ifdef MG_BD_STATS
    {
      unsigned long long h[2][16];
      MG_CUDA(cudaStreamSynchronize(s));
      MG_CUDA(cudaMemcpyFromSymbol(h, mg::g_bd_stats, sizeof h));
      const char* nm[9] = {"items", "k_lookups", "pieces", "subbatches", "waves", "single_waves", "products", "runs", "passes"};
      for (int l = 0; l < 2; ++l) {
        fprintf(stderr, "[bd] list %d:", l);
        for (int q = 0; q < 9; ++q) fprintf(stderr, " %s=%llu", nm[q], h[l][q]);
        fprintf(stderr, "\n");
      }
      unsigned long long z[2][16] = {};
      MG_CUDA(cudaMemcpyToSymbol(mg::g_bd_stats, z, sizeof z));
    }
#endif
    MG_CUDA(cudaFreeAsync(items, s));
    MG_CUDA(cudaFreeAsync(aslot, s));
    MG_CUDA(cudaFreeAsync(abase, s));
  }
  MG_CUDA(cudaFreeAsync(bucket, s));
  MG_CUDA(cudaFreeAsync(hsmall, s));
  return MAGNUS_OK;
}

// Heavy rows, numeric phase, direct big-chunk path: big chunks straight from B, then the small
// chunks through the binned path in batches of rows whose small-chunk products fit the reorder buffer.
static int launch_binned_direct(magnus_ctx* ctx, const int64_t* c_rp, uint32_t* c_col, double* c_val) {
  cudaStream_t s = ctx->stream;
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  {
    int rc = launch_big_direct(ctx, c_rp, c_col, c_val);
    if (rc) return rc;
  }
  const std::vector<int64_t>& hsz = ctx->h_small;   // small-chunk products per heavy row
  int64_t max_row = 0, total = 0;
  for (int64_t h = 0; h < nH; ++h) {
    max_row = std::max(max_row, hsz[h]);
    total += hsz[h];
  }
  size_t free_b = 0, tot_b = 0;
  MG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
  {
    // memory the pool holds but does not use is available too
    cudaMemPool_t pool = workspace_pool();
    uint64_t reserved = 0, used = 0;
    MG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    MG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
    if (reserved > used) free_b += (size_t)(reserved - used);
  }
  const int64_t per_elem = 10;   // u16 local column + f64 product
  double frac = kBatchFracSerial;
  if (const char* bf = std::getenv("MAGNUS_BATCH_FRAC")) {
    const double v = std::atof(bf);
    if (v > 0.0 && v < 0.9) frac = v;
  }
  int64_t cap = std::min<int64_t>(total, std::min<int64_t>((int64_t)(free_b * frac) / per_elem, int64_t(3) << 30));
  if (const char* ce = std::getenv("MAGNUS_BATCH_ELEMS")) {   // testing: force many heavy-row batches
    const long long v = std::atoll(ce);
    if (v > 0) cap = std::min<int64_t>(cap, (int64_t)v);
  }
  cap = std::max<int64_t>(cap, std::max<int64_t>(max_row, 1));
  // batches [h0, h1) and the largest chunk-table span of a batch
  std::vector<int64_t> cuts{0};
  int64_t acc = 0, ent = 0, max_ent = 0;
  for (int64_t h = 0; h < nH; ++h) {
    if (acc + hsz[h] > cap && h > cuts.back()) {
      cuts.push_back(h);
      max_ent = std::max(max_ent, ent);
      acc = ent = 0;
    }
    acc += hsz[h];
    ent += ctx->h_nent[h];
  }
  cuts.push_back(nH);
  max_ent = std::max(max_ent, ent);
  int64_t buf_elems = 0;
  std::vector<int64_t> hb(cuts.size());
  {
    int64_t a = 0;
    size_t b = 0;
    for (int64_t h = 0; h <= nH; ++h) {
      while (b < cuts.size() && cuts[b] == h) hb[b++] = a;
      if (h < nH) a += hsz[h];
    }
    for (size_t q = 0; q + 1 < cuts.size(); ++q) buf_elems = std::max(buf_elems, hb[q + 1] - hb[q]);
  }
  void *bcol = nullptr, *bval = nullptr, *items = nullptr, *cnts = nullptr;
  MG_CUDA(mg_malloc_async(&bcol, (size_t)std::max<int64_t>(buf_elems, 1) * 2 + 64, s));
  MG_CUDA(mg_malloc_async(&bval, (size_t)std::max<int64_t>(buf_elems, 1) * 8 + 64, s));
  // windows and units: <= one per chunk entry each
  MG_CUDA(mg_malloc_async(&items, (size_t)std::max<int64_t>(max_ent, 1) * 3 * sizeof(mg::BinItem), s));
  MG_CUDA(mg_malloc_async(&cnts, 128, s));
  const size_t red_smem = mg::bin_reduce_warp_smem(ctx->sem.shift_num) * (mg::kBinT / 32);
  int occ = 1;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mg::k_bin_reduce, mg::kBinT, red_smem));
  occ = std::max(occ, 1);
  int occ_e2 = 1;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_e2, mg::k_bin_expand2, mg::kE2T, mg::Exp2Smem::kTotal));
  occ_e2 = std::max(occ_e2, 1);
  uint32_t* e2scr = nullptr;   // per-CTA segment tables of units with more than kE2K k's
  const int64_t e2_stride = ((ctx->host_stats[mg::kStatMaxNk] + 8 + 3) / 4) * 4;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&e2scr), (size_t)ctx->sm_count * occ_e2 * 5 * e2_stride * 4, s));
  // host readback: C offset of each batch's end row (the next batch's first heavy row)
  std::vector<int64_t> batch_end(cuts.size(), -1);
  if (ctx->host_col) {
    for (size_t b = 0; b + 2 < cuts.size(); ++b)
      MG_CUDA(cudaMemcpyAsync(&batch_end[b], c_rp + ctx->h_rows[cuts[b + 1]], 8, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t me = std::max<int64_t>(max_ent, 1);
  for (size_t b = 0; b + 1 < cuts.size(); ++b) {
    const int64_t h0 = cuts[b], h1 = cuts[b + 1];
    if (hb[b + 1] == hb[b]) continue;   // no small-chunk products in this batch
    mg::BinItem* wins = static_cast<mg::BinItem*>(items);
    mg::BinItem* units = wins + me;
    mg::BinItem* wins_t = units + me;   // windows of tiny chunks (k_bin_reduce_tiny)
    auto* nwin = static_cast<unsigned long long*>(cnts);
    auto* nunit = nwin + 1;
    MG_CUDA(cudaMemsetAsync(cnts, 0, 128, s));
    ctx->begin(MAGNUS_K_BIN_PLAN);
    mg::k_bin_plan_small<<<(unsigned)std::min<int64_t>((h1 - h0 + 7) / 8, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
        ctx->listH, h0, h1, ctx->mn, ctx->mx, ctx->sem.shift_num, ctx->choff, ctx->ce, ctx->cs, wins, nwin, wins_t, units,
        nunit, me);
    ctx->end();
    ctx->begin(MAGNUS_K_BIN_EXPAND);
    mg::k_bin_expand2<<<(unsigned)(ctx->sm_count * occ_e2), mg::kE2T, mg::Exp2Smem::kTotal, s>>>(
        ctx->A, ctx->B, ctx->listH, ctx->mn, ctx->mx, ctx->sem.shift_num, ctx->choff, ctx->cs, ctx->hbase_s, hb[b], units,
        nunit, nwin + 3, me, static_cast<uint16_t*>(bcol), static_cast<double*>(bval), ctx->bslot, ctx->bidx,
        ctx->dir_nwin1, ctx->dir_wlog, e2scr, e2_stride, ctx->err);
    ctx->end();
    ctx->begin(MAGNUS_K_BIN_REDUCE);
    mg::k_bin_reduce<<<(unsigned)(ctx->sm_count * occ), mg::kBinT, red_smem, s>>>(
        ctx->listH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->choff, ctx->cs, ctx->cd, ctx->hbase_s, hb[b], wins, nwin,
        nwin + 4, static_cast<const uint16_t*>(bcol), static_cast<const double*>(bval), c_rp, c_col, c_val, ctx->err);
    mg::k_bin_reduce_tiny<<<(unsigned)(ctx->sm_count * 8), 256, 0, s>>>(
        ctx->listH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->choff, ctx->cs, ctx->cd, ctx->hbase_s, hb[b], wins_t,
        nwin + 8, nwin + 9, static_cast<const uint16_t*>(bcol), static_cast<const double*>(bval), c_rp, c_col, c_val,
        ctx->err);
    ctx->end();
    ++ctx->launches;
    MG_CUDA(cudaGetLastError());
    if (ctx->host_col) {
      // rows below the next batch's first heavy row are complete (light rows and big chunks
      // ran first): read that prefix of C back on the copy stream while the next batch computes
      const int64_t end = b + 2 < cuts.size() ? batch_end[b] : -1;
      if (end > ctx->host_done) {
        MG_CUDA(cudaEventRecord(ctx->ev_fork, s));
        MG_CUDA(cudaStreamWaitEvent(ctx->aux3, ctx->ev_fork, 0));
        MG_CUDA(cudaMemcpyAsync(ctx->host_col + ctx->host_done, c_col + ctx->host_done, (end - ctx->host_done) * 4,
                                cudaMemcpyDeviceToHost, ctx->aux3));
        MG_CUDA(cudaMemcpyAsync(ctx->host_val + ctx->host_done, c_val + ctx->host_done, (end - ctx->host_done) * 8,
                                cudaMemcpyDeviceToHost, ctx->aux3));
        ctx->host_done = end;
      }
    }
  }
  MG_CUDA(cudaFreeAsync(e2scr, s));
  MG_CUDA(cudaFreeAsync(bcol, s));
  MG_CUDA(cudaFreeAsync(bval, s));
  MG_CUDA(cudaFreeAsync(items, s));
  MG_CUDA(cudaFreeAsync(cnts, s));
  MG_CUDA(cudaFreeAsync(ctx->cs, s));
  MG_CUDA(cudaFreeAsync(ctx->hbase_s, s));
  ctx->cs = nullptr;
  ctx->hbase_s = nullptr;
  return MAGNUS_OK;
}

static int launch_light(magnus_ctx* ctx, bool numeric, const int64_t* c_rp, uint32_t* c_col, double* c_val);

static int launch_rows(magnus_ctx* ctx, bool numeric, const int64_t* c_rp, uint32_t* c_col, double* c_val) {
  cudaStream_t s = ctx->stream;
  const int64_t nH = ctx->host_stats[mg::kStatNH];
  // the light row classes run on a side stream, concurrently with the heavy rows
  const char* serial_env = std::getenv("MAGNUS_SERIAL");
  // (light rows on a side stream while the heavy rows compute; MAGNUS_LIGHT_SIDE=0 serialises)
  const char* light_env = std::getenv("MAGNUS_LIGHT_SIDE");
  const bool side = nH > 0 && ((serial_env && std::strcmp(serial_env, "0") == 0) || !(light_env && std::strcmp(light_env, "0") == 0));
  if (side) {
    MG_CUDA(cudaEventRecord(ctx->ev_fork, s));
    MG_CUDA(cudaStreamWaitEvent(ctx->aux3, ctx->ev_fork, 0));
    ctx->stream = ctx->aux3;
  }
  int rc = launch_light(ctx, numeric, c_rp, c_col, c_val);
  ctx->stream = s;
  if (rc) return rc;
  if (side) MG_CUDA(cudaEventRecord(ctx->ev_join, ctx->aux3));
  if (nH > 0 && numeric && ctx->direct) {
    int rc = launch_direct(ctx, c_rp, c_col, c_val);
    if (rc) return rc;
  } else if (nH > 0 && numeric && ctx->binned) {
    int rc = ctx->big_direct ? launch_binned_direct(ctx, c_rp, c_col, c_val) : launch_binned(ctx, c_rp, c_col, c_val);
    if (rc) return rc;
  } else if (nH > 0) {
    MG_CUDA(cudaMemsetAsync(ctx->work, 0, 24, s));
    const unsigned grid = (unsigned)std::min<int64_t>(nH, (int64_t)ctx->sm_count * (numeric ? 2 : mg::kSymCtas));
    ctx->begin(numeric ? MAGNUS_K_NUM_HEAVY : MAGNUS_K_SYM_HEAVY);
    if (numeric)
      mg::k_heavy_numeric<<<grid, mg::kNT, mg::HeavyNumSmem::kTotal, s>>>(
          ctx->A, ctx->B, ctx->listH, nH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->modebits, c_rp, c_col, c_val, ctx->gk,
          ctx->gk_stride, ctx->work, ctx->err);
    else if (ctx->binned && ctx->sym2)
      mg::k_heavy_sym2<<<(unsigned)std::min<int64_t>(nH, (int64_t)ctx->sm_count * ctx->sym2_occ), mg::kS2T,
                         mg::Sym2Smem::kTotal, s>>>(
          ctx->A, ctx->B, ctx->listH, nH, ctx->mn, ctx->mx, (int)ctx->sem.shift_num, ctx->counts, ctx->choff, ctx->ce,
          ctx->cd, ctx->cbm_pool, ctx->cbm_slot, ctx->cbm_cap, ctx->work, ctx->bslot, ctx->bidx, ctx->dir_nwin1,
          ctx->dir_wlog, ctx->gk, ctx->gk_stride);
    else
      mg::k_heavy_symbolic<<<grid, mg::kHT, mg::HeavySymSmem::kTotal, s>>>(
          ctx->A, ctx->B, ctx->listH, nH, ctx->cat, ctx->mn, ctx->mx, ctx->sem, ctx->counts, ctx->modebits, ctx->gk,
          ctx->gk_stride, ctx->gchunk, ctx->work, ctx->binned ? 1 : 0, ctx->ncnt, ctx->choff, ctx->ce, ctx->cd,
          ctx->cbm_pool, ctx->cbm_slot, ctx->cbm_cap);
    ctx->end();
    MG_CUDA(cudaGetLastError());
  }
  if (side) MG_CUDA(cudaStreamWaitEvent(s, ctx->ev_join, 0));
  return MAGNUS_OK;
}

static int launch_light(magnus_ctx* ctx, bool numeric, const int64_t* c_rp, uint32_t* c_col, double* c_val) {
  cudaStream_t s = ctx->stream;
  const int64_t nW = ctx->host_stats[mg::kStatNW], nB = ctx->host_stats[mg::kStatNB];
  if (nB > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(nB, (int64_t)ctx->sm_count * 3);
    ctx->begin(numeric ? MAGNUS_K_NUM_BLOCK : MAGNUS_K_SYM_BLOCK);
    if (numeric)
      mg::k_rows_block<true><<<grid, mg::kBT, mg::kBSmem, s>>>(ctx->A, ctx->B, ctx->listB, nB, ctx->cat, ctx->sem,
                                                                ctx->counts, c_rp, c_col, c_val, ctx->err);
    else
      mg::k_rows_block<false><<<grid, mg::kBT, mg::kBSmem, s>>>(ctx->A, ctx->B, ctx->listB, nB, ctx->cat, ctx->sem,
                                                                 ctx->counts, c_rp, c_col, c_val, ctx->err);
    ctx->end();
    MG_CUDA(cudaGetLastError());
  }
  const int64_t nD = ctx->host_stats[mg::kStatND];
  if (nD > 0) {
    const int64_t blocks = (nD + mg::kDT / 32 - 1) / (mg::kDT / 32);
    const unsigned grid = (unsigned)std::min<int64_t>(blocks, (int64_t)ctx->sm_count * 2 * 4);
    ctx->begin(numeric ? MAGNUS_K_NUM_DENSE : MAGNUS_K_SYM_DENSE);
    if (numeric)
      mg::k_rows_dense<true><<<grid, mg::kDT, mg::DenseRowSmem::kTotal, s>>>(ctx->A, ctx->B, ctx->listD, nD, ctx->mn,
                                                                           ctx->mx, ctx->counts, c_rp, c_col, c_val,
                                                                           ctx->err);
    else
      mg::k_rows_dense<false><<<grid, mg::kDT, mg::DenseRowSmem::kTotal, s>>>(ctx->A, ctx->B, ctx->listD, nD, ctx->mn,
                                                                            ctx->mx, ctx->counts, c_rp, c_col, c_val,
                                                                            ctx->err);
    ctx->end();
    MG_CUDA(cudaGetLastError());
  }
  if (nW > 0) {
    const int64_t blocks = (nW + mg::kWT / 32 - 1) / (mg::kWT / 32);
    const unsigned grid = (unsigned)std::min<int64_t>(blocks, (int64_t)ctx->sm_count * 8);
    const bool key32 = ctx->B.n_cols <= (int64_t(1) << 24);
    if (!numeric) {
      // fused warp rows: the symbolic pass also computes the values, into the rows' upper-bound
      // slots of a buffer (<= 256 products per row); the numeric pass copies them into C.
      // Used when that buffer fits a quarter of the free HBM (MAGNUS_FUSED_ROWS=0 disables it).
      ctx->fused = false;
      const char* fe = std::getenv("MAGNUS_FUSED_ROWS");
      if (!(fe && std::strcmp(fe, "0") == 0)) {
        MG_CUDA(ctx->alloc(&ctx->fused_ub, nW + 1));
        mg::k_gather_inter<<<(unsigned)std::min<int64_t>((nW + 255) / 256, (int64_t)ctx->sm_count * 8), 256, 0, s>>>(
            ctx->listW, nW, ctx->inter, ctx->fused_ub);
        int64_t* ts = nullptr;
        const int64_t tiles = (nW + mg::kScanTile - 1) / mg::kScanTile;
        MG_CUDA(ctx->alloc(&ts, tiles + 1));
        mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->fused_ub, nW, ts);
        mg::k_scan_tiles<<<1, 1024, 0, s>>>(ts, tiles);
        mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->fused_ub, nW, ts, ctx->fused_ub);
        ctx->launches += 4;
        int64_t tot = 0;
        MG_CUDA(cudaMemcpyAsync(&tot, ctx->fused_ub + nW, 8, cudaMemcpyDeviceToHost, s));
        MG_CUDA(cudaStreamSynchronize(s));
        size_t fr = 0, to = 0;
        MG_CUDA(cudaMemGetInfo(&fr, &to));
        if ((size_t)tot * 12 <= fr / 4) {
          MG_CUDA(ctx->alloc(&ctx->fused_col, tot));
          MG_CUDA(ctx->alloc(&ctx->fused_val, tot));
          ctx->fused = true;
        }
      }
    }
    ctx->begin(numeric ? MAGNUS_K_NUM_WARP : MAGNUS_K_SYM_WARP);
    if (numeric && ctx->fused)
      mg::k_rows_copy<<<grid, 256, 0, s>>>(ctx->listW, nW, ctx->fused_ub, ctx->fused_col, ctx->fused_val, c_rp, c_col, c_val);
    else if (numeric && key32)
      mg::k_rows_warp<1, true><<<grid, mg::kWT, 0, s>>>(ctx->A, ctx->B, ctx->listW, nW, ctx->cat, ctx->sem, ctx->counts,
                                                         c_rp, c_col, c_val, ctx->err);
    else if (numeric)
      mg::k_rows_warp<1, false><<<grid, mg::kWT, 0, s>>>(ctx->A, ctx->B, ctx->listW, nW, ctx->cat, ctx->sem, ctx->counts,
                                                          c_rp, c_col, c_val, ctx->err);
    else if (ctx->fused && key32)
      mg::k_rows_warp<2, true><<<grid, mg::kWT, 0, s>>>(ctx->A, ctx->B, ctx->listW, nW, ctx->cat, ctx->sem, ctx->counts,
                                                         nullptr, ctx->fused_col, ctx->fused_val, ctx->err, ctx->fused_ub);
    else if (ctx->fused)
      mg::k_rows_warp<2, false><<<grid, mg::kWT, 0, s>>>(ctx->A, ctx->B, ctx->listW, nW, ctx->cat, ctx->sem, ctx->counts,
                                                          nullptr, ctx->fused_col, ctx->fused_val, ctx->err, ctx->fused_ub);
    else if (key32)
      mg::k_rows_warp<0, true><<<grid, mg::kWT, 0, s>>>(ctx->A, ctx->B, ctx->listW, nW, ctx->cat, ctx->sem, ctx->counts,
                                                         c_rp, c_col, c_val, ctx->err);
    else
      mg::k_rows_warp<0, false><<<grid, mg::kWT, 0, s>>>(ctx->A, ctx->B, ctx->listW, nW, ctx->cat, ctx->sem, ctx->counts,
                                                          c_rp, c_col, c_val, ctx->err);
    ctx->end();
    MG_CUDA(cudaGetLastError());
  }
  return MAGNUS_OK;
}

int magnus_symbolic(magnus_ctx* ctx, int64_t* c_row_ptr, int64_t* nnz_out, void* stream) {
  if (!ctx || !ctx->ready) return set_err(MAGNUS_CONTRACT, "magnus_setup has not run");
  NvtxRange nvtx_range("magnus_symbolic");
  ctx->stream = (cudaStream_t)stream;
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->A.n_rows;
  if (n == 0) {
    MG_CUDA(cudaMemsetAsync(c_row_ptr, 0, 8, s));
    if (nnz_out) *nnz_out = 0;
    ctx->have_symbolic = true;
    return MAGNUS_OK;
  }
  MG_CUDA(cudaMemsetAsync(ctx->counts, 0, n * 8, s));   // rows with an empty product stay 0
  int rc = launch_rows(ctx, false, nullptr, nullptr, nullptr);
  if (rc) return rc;
  // row_ptr = cumsum(counts)  (magnus.py:454-456)
  const int64_t tiles = (n + mg::kScanTile - 1) / mg::kScanTile;
  ctx->begin(MAGNUS_K_SCAN);
  mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->counts, n, ctx->tile_sums);
  mg::k_scan_tiles<<<1, 1024, 0, s>>>(ctx->tile_sums, tiles);
  mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(ctx->counts, n, ctx->tile_sums, c_row_ptr);
  ctx->end();
  ctx->launches += 2;
  MG_CUDA(cudaGetLastError());
  int64_t nnz = 0;
  MG_CUDA(cudaMemcpyAsync(&nnz, c_row_ptr + n, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  if (nnz_out) *nnz_out = nnz;
  ctx->have_symbolic = true;
  return MAGNUS_OK;
}

int magnus_numeric(magnus_ctx* ctx, const int64_t* c_row_ptr, uint32_t* c_col, double* c_val, magnus_counters* counters,
                   void* stream) {
  if (!ctx || !ctx->ready) return set_err(MAGNUS_CONTRACT, "magnus_setup has not run");
  if (!ctx->have_symbolic) return set_err(MAGNUS_CONTRACT, "row_ptr does not come from a symbolic pass of (A, B)");
  NvtxRange nvtx_range("magnus_numeric");
  ctx->stream = (cudaStream_t)stream;
  cudaStream_t s = ctx->stream;
  if (ctx->A.n_rows > 0) {
    int rc = launch_rows(ctx, true, c_row_ptr, c_col, c_val);
    if (rc) return rc;
  }
  unsigned long long e = 0;
  MG_CUDA(cudaMemcpyAsync(&e, ctx->err, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  if (e) {
    char buf[32];
    snprintf(buf, sizeof buf, "%llx", e);
    // flags: 1 light rows, 2 windowed heavy rows, 4 binned heavy rows, 8 direct heavy rows
    return set_err(MAGNUS_CONTRACT, std::string("numeric phase count differs from the symbolic count (flags 0x") + buf + ")");
  }
  if (counters) {
    int64_t nnz = 0;
    if (ctx->A.n_rows > 0) MG_CUDA(cudaMemcpy(&nnz, c_row_ptr + ctx->A.n_rows, 8, cudaMemcpyDeviceToHost));
    counters->nnz_c = nnz;
    counters->inter_prod_size = ctx->host_stats[mg::kStatInter];
    counters->coarse_batches = ctx->coarse_batches;
    counters->rows_sort = ctx->host_stats[mg::kStatCat + 0];
    counters->rows_dense = ctx->host_stats[mg::kStatCat + 1];
    counters->rows_fine = ctx->host_stats[mg::kStatCat + 2];
    counters->rows_coarse = ctx->host_stats[mg::kStatCat + 3];
  }
  return MAGNUS_OK;
}

int magnus_numeric_host(magnus_ctx* ctx, const int64_t* c_row_ptr, uint32_t* c_col, double* c_val, uint32_t* c_col_host,
                        double* c_val_host, magnus_counters* counters, void* stream) {
  if (!ctx || !c_col_host || !c_val_host) return set_err(MAGNUS_INPUT, "null argument");
  ctx->host_col = c_col_host;
  ctx->host_val = c_val_host;
  ctx->host_done = 0;
  int rc = magnus_numeric(ctx, c_row_ptr, c_col, c_val, counters, stream);
  const int64_t done = ctx->host_done;
  ctx->host_col = nullptr;
  ctx->host_val = nullptr;
  if (rc) {
    cudaStreamSynchronize(ctx->aux3);
    return rc;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nnz = 0;
  if (ctx->A.n_rows > 0) MG_CUDA(cudaMemcpyAsync(&nnz, c_row_ptr + ctx->A.n_rows, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  if (nnz > done) {
    MG_CUDA(cudaMemcpyAsync(c_col_host + done, c_col + done, (nnz - done) * 4, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(c_val_host + done, c_val + done, (nnz - done) * 8, cudaMemcpyDeviceToHost, s));
  }
  MG_CUDA(cudaStreamSynchronize(ctx->aux3));
  MG_CUDA(cudaStreamSynchronize(s));
  return MAGNUS_OK;
}

// internal debug hook (not part of the public header): phase cycle counters of
// k_heavy_numeric when built with -DMG_PROFILE_PHASES, else zeros.
int magnus_debug_phases(unsigned long long* out16, int reset) {
#ifdef MG_PROFILE_PHASES
  MG_CUDA(cudaDeviceSynchronize());
  MG_CUDA(cudaMemcpyFromSymbol(out16, mg::g_phase, 16 * 8));
  if (reset) {
    unsigned long long z[32] = {0};
    MG_CUDA(cudaMemcpyToSymbol(mg::g_phase, z, sizeof z));
  }
#else
  for (int i = 0; i < 16; ++i) out16[i] = 0;
  (void)reset;
#endif
  return MAGNUS_OK;
}

// ---------------------------------------------------------------- Gustavson baselines (gustavson.py:155-268)
size_t magnus_gd_scratch_bytes(int64_t n_cols, int64_t ctas) {
  const int64_t nwords = (std::max<int64_t>(n_cols, 1) + 31) / 32;
  return (size_t)ctas * (size_t)nwords * (4 + 32 * 8);
}

static int gd_launch(const magnus_csr* A, const magnus_csr* B, int numeric, const int64_t* c_rp, int64_t* rp_out,
                     uint32_t* c_col, double* c_val, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (!A || !B || (!scratch && A->n_rows)) return set_err(MAGNUS_INPUT, "null argument");
  if (A->n_cols != B->n_rows)
    return set_err(MAGNUS_INPUT, "dimension mismatch: A is " + std::to_string(A->n_rows) + "x" + std::to_string(A->n_cols) +
                                     ", B is " + std::to_string(B->n_rows) + "x" + std::to_string(B->n_cols));
  if (B->n_cols > (int64_t(1) << 32)) return set_err(MAGNUS_INPUT, "more than 2^32 columns needs 8-byte column indices");
  const int64_t n = A->n_rows;
  if (n == 0) {
    if (!numeric) MG_CUDA(cudaMemsetAsync(rp_out, 0, 8, s));
    return MAGNUS_OK;
  }
  int dev = 0, sms = 148;
  MG_CUDA(cudaGetDevice(&dev));
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t nwords = (std::max<int64_t>(B->n_cols, 1) + 31) / 32;
  const size_t per = magnus_gd_scratch_bytes(B->n_cols, 1);
  const int64_t ctas = std::min<int64_t>({(int64_t)sms * 4, (int64_t)(scratch_bytes / per), n});
  if (ctas < 1)
    return set_err(MAGNUS_OVER_BUDGET, "scratch of " + std::to_string(scratch_bytes) + " bytes holds no " +
                                           std::to_string(per) + "-byte dense accumulator");
  uint32_t* bm = static_cast<uint32_t*>(scratch);
  double* acc = reinterpret_cast<double*>(bm + (size_t)ctas * nwords + ((size_t)ctas * nwords & 1));
  unsigned long long* flags = nullptr;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&flags), 16, s));
  MG_CUDA(cudaMemsetAsync(flags, 0, 16, s));
  MG_CUDA(cudaMemsetAsync(bm, 0, (size_t)ctas * nwords * 4, s));
  const mg::DevCsr dA = dev_csr(*A), dB = dev_csr(*B);
  if (numeric)
    mg::k_gd_rows<true><<<(unsigned)ctas, mg::kGdT, 0, s>>>(dA, dB, c_rp, c_col, c_val, nullptr, bm, acc, nwords, flags,
                                                            flags + 1);
  else
    mg::k_gd_rows<false><<<(unsigned)ctas, mg::kGdT, 0, s>>>(dA, dB, nullptr, nullptr, nullptr, rp_out, bm, nullptr,
                                                             nwords, flags, flags + 1);
  MG_CUDA(cudaGetLastError());
  unsigned long long err = 0;
  if (!numeric) {
    // row_ptr = exclusive scan of the per-row counts, in place (k_scan_apply reads and writes each index
    // from the same thread)
    const int64_t tiles = (n + mg::kScanTile - 1) / mg::kScanTile;
    int64_t* tile_sums = nullptr;
    MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&tile_sums), (size_t)(tiles + 1) * 8, s));
    mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(rp_out, n, tile_sums);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(tile_sums, tiles);
    mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(rp_out, n, tile_sums, rp_out);
    MG_CUDA(cudaGetLastError());
    MG_CUDA(cudaFreeAsync(tile_sums, s));
  } else {
    MG_CUDA(cudaMemcpyAsync(&err, flags + 1, 8, cudaMemcpyDeviceToHost, s));
  }
  MG_CUDA(cudaFreeAsync(flags, s));
  MG_CUDA(cudaStreamSynchronize(s));
  if (err) return set_err(MAGNUS_CONTRACT, "numeric phase count differs from the symbolic count");
  return MAGNUS_OK;
}

int magnus_gd_symbolic(const magnus_csr* A, const magnus_csr* B, int64_t* c_row_ptr, void* scratch, size_t scratch_bytes,
                       void* stream) {
  if (!c_row_ptr) return set_err(MAGNUS_INPUT, "null argument");
  return gd_launch(A, B, 0, nullptr, c_row_ptr, nullptr, nullptr, scratch, scratch_bytes, (cudaStream_t)stream);
}

int magnus_gd_numeric(const magnus_csr* A, const magnus_csr* B, const int64_t* c_row_ptr, uint32_t* c_col, double* c_val,
                      void* scratch, size_t scratch_bytes, void* stream) {
  if (!c_row_ptr) return set_err(MAGNUS_INPUT, "null argument");
  return gd_launch(A, B, 1, c_row_ptr, nullptr, c_col, c_val, scratch, scratch_bytes, (cudaStream_t)stream);
}

int magnus_esc_expand(const magnus_csr* A, const magnus_csr* B, int64_t r0, int64_t r1, const int64_t* inter_off,
                      uint64_t* keys, double* vals, void* stream) {
  if (!A || !B || !inter_off) return set_err(MAGNUS_INPUT, "null argument");
  if (A->n_cols != B->n_rows) return set_err(MAGNUS_INPUT, "dimension mismatch");
  if (r0 < 0 || r1 > A->n_rows || r0 > r1) return set_err(MAGNUS_INPUT, "row range outside A");
  if (r1 - r0 > (int64_t(1) << 31)) return set_err(MAGNUS_INPUT, "row range wider than 2^31");
  if (r1 == r0) return MAGNUS_OK;
  int dev = 0, sms = 148;
  MG_CUDA(cudaGetDevice(&dev));
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t blocks = std::min<int64_t>((r1 - r0 + 7) / 8, (int64_t)sms * 8);
  mg::k_esc_expand<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dev_csr(*A), dev_csr(*B), r0, r1, inter_off, keys,
                                                                       vals);
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

int magnus_esc_compress(const uint64_t* keys, const int64_t* perm, const double* vals, int64_t n, int64_t out0,
                        uint32_t* c_col, double* c_val, int64_t* run_scratch, int64_t* runs_out, void* stream) {
  if (n < 0 || (n && (!keys || !perm || !vals || !run_scratch))) return set_err(MAGNUS_INPUT, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (runs_out) *runs_out = 0;
    return MAGNUS_OK;
  }
  int dev = 0, sms = 148;
  MG_CUDA(cudaGetDevice(&dev));
  MG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16);
  mg::k_esc_heads<<<g, 256, 0, s>>>(keys, n, run_scratch);
  const int64_t tiles = (n + mg::kScanTile - 1) / mg::kScanTile;
  int64_t* tile_sums = nullptr;
  MG_CUDA(mg_malloc_async(reinterpret_cast<void**>(&tile_sums), (size_t)(tiles + 1) * 8, s));
  mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(run_scratch, n, tile_sums);
  mg::k_scan_tiles<<<1, 1024, 0, s>>>(tile_sums, tiles);
  mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(run_scratch, n, tile_sums, run_scratch);
  MG_CUDA(cudaFreeAsync(tile_sums, s));
  int64_t runs = 0;
  MG_CUDA(cudaMemcpyAsync(&runs, run_scratch + n, 8, cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  if (runs_out) *runs_out = runs;
  if (c_col && c_val) {
    mg::k_esc_reduce<<<g, 256, 0, s>>>(keys, perm, vals, n, run_scratch, out0, c_col, c_val);
    MG_CUDA(cudaGetLastError());
  }
  return MAGNUS_OK;
}

// ---------------------------------------------------------------- building-block microbenchmarks (bench.py:88-196)
static int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

int magnus_mb_histogram(const uint32_t* idx, int64_t n, int shift, int n_chunks, int64_t* counts, void* stream) {
  if (n_chunks < 1 || n_chunks > 16384 || shift < 0 || shift > 31 || (n && !idx) || !counts)
    return set_err(MAGNUS_INPUT, "histogram: 1 <= n_chunks <= 16384, 0 <= shift < 32");
  cudaStream_t s = (cudaStream_t)stream;
  MG_CUDA(cudaMemsetAsync(counts, 0, (size_t)n_chunks * 8, s));
  if (!n) return MAGNUS_OK;
  const int64_t g = std::min<int64_t>((n + 1023) / 1024, (int64_t)sm_count() * 4);
  mg::k_mb_hist<<<(unsigned)g, 512, (size_t)n_chunks * 4, s>>>(idx, n, shift, n_chunks,
                                                               reinterpret_cast<unsigned long long*>(counts));
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

size_t magnus_mb_reorder_scratch_bytes(int64_t n, int n_chunks) {
  const int64_t ntiles = (n + mg::kMbTile - 1) / mg::kMbTile;
  const int64_t tiles = (n_chunks * ntiles + mg::kScanTile - 1) / mg::kScanTile;
  return (size_t)(n_chunks * ntiles + 1 + tiles + 1) * 8;
}

int magnus_mb_reorder(const uint32_t* idx, const double* val, int64_t n, int shift, int n_chunks, void* scratch,
                      size_t scratch_bytes, uint32_t* out_col, double* out_val, void* stream) {
  if (n_chunks < 1 || n_chunks > mg::kMbMaxChunks || shift < 0 || shift > 31)
    return set_err(MAGNUS_INPUT, "reorder: 1 <= n_chunks <= 4096, 0 <= shift < 32");
  if (n >= (int64_t(1) << 32)) return set_err(MAGNUS_INPUT, "reorder: stream longer than 2^32");
  if (scratch_bytes < magnus_mb_reorder_scratch_bytes(n, n_chunks)) return set_err(MAGNUS_INPUT, "reorder: scratch too small");
  if (!n) return MAGNUS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ntiles = (n + mg::kMbTile - 1) / mg::kMbTile, m = (int64_t)n_chunks * ntiles;
  int64_t* toff = static_cast<int64_t*>(scratch);
  int64_t* tile_sums = toff + m + 1;
  const size_t sh = (size_t)mg::kMbWarps * n_chunks * 4;
  MG_CUDA(cudaFuncSetAttribute(mg::k_mb_tile_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  MG_CUDA(cudaFuncSetAttribute(mg::k_mb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  const unsigned g = (unsigned)((ntiles + mg::kMbWarps - 1) / mg::kMbWarps);
  mg::k_mb_tile_hist<<<g, mg::kMbWarps * 32, sh, s>>>(idx, n, shift, n_chunks, ntiles, toff);
  const int64_t tiles = (m + mg::kScanTile - 1) / mg::kScanTile;
  mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(toff, m, tile_sums);
  mg::k_scan_tiles<<<1, 1024, 0, s>>>(tile_sums, tiles);
  mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(toff, m, tile_sums, toff);
  mg::k_mb_scatter<<<g, mg::kMbWarps * 32, sh, s>>>(idx, val, n, shift, n_chunks, ntiles, toff, out_col, out_val);
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

int magnus_mb_dense(const uint32_t* col, const double* val, const int64_t* offsets, int n_chunks, int chunk_len,
                    uint32_t* out_col, double* out_val, int64_t* distinct, void* stream) {
  if (n_chunks < 1 || chunk_len < 1 || chunk_len > (1 << 14)) return set_err(MAGNUS_INPUT, "dense: 1 <= chunk_len <= 16384");
  const size_t sh = (size_t)chunk_len * 8 + (size_t)((chunk_len + 63) / 64) * 8 + 32 * 8;
  MG_CUDA(cudaFuncSetAttribute(mg::k_mb_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  mg::k_mb_dense<<<(unsigned)n_chunks, 32, sh, (cudaStream_t)stream>>>(col, val, offsets, n_chunks, chunk_len, out_col,
                                                                       out_val, distinct);
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

// Stable LSD radix sort of (key, position): the sort stage of the sort-accumulator microbenchmark.
size_t magnus_sort_pairs_scratch_bytes(int64_t n) {
  const int64_t ntiles = (std::max<int64_t>(n, 1) + mg::kRsTile - 1) / mg::kRsTile;
  const int64_t nh = 256 * ntiles;
  return (size_t)std::max<int64_t>(n, 1) * 16 + (size_t)(2 * nh + 2) * 8 + (size_t)((nh + mg::kScanTile - 1) / mg::kScanTile + 2) * 8 + 64;
}

int magnus_sort_pairs(const uint64_t* keys, int64_t n, uint64_t key_mask, uint64_t* keys_out, int64_t* perm_out,
                      void* scratch, void* stream) {
  if (n < 0 || (n && (!keys || !keys_out || !perm_out || !scratch))) return set_err(MAGNUS_INPUT, "sort_pairs: bad argument");
  if (!n) return MAGNUS_OK;
  if (!key_mask) key_mask = 0xffull;   // nothing to order by: one pass copies the keys and writes the identity
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ntiles = (n + mg::kRsTile - 1) / mg::kRsTile, nh = 256 * ntiles;
  unsigned char* sp = static_cast<unsigned char*>(scratch);
  uint64_t* tk = reinterpret_cast<uint64_t*>(sp); sp += (size_t)n * 8;
  int64_t* tp = reinterpret_cast<int64_t*>(sp); sp += (size_t)n * 8;
  int64_t* hist = reinterpret_cast<int64_t*>(sp); sp += (size_t)nh * 8;
  int64_t* base = reinterpret_cast<int64_t*>(sp); sp += (size_t)(nh + 2) * 8;
  int64_t* tsum = reinterpret_cast<int64_t*>(sp);
  // one pass per key byte that has a significant bit
  int shifts[8], passes = 0;
  for (int b = 0; b < 8; ++b)
    if ((key_mask >> (8 * b)) & 0xffull) shifts[passes++] = 8 * b;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count() * 16);
  const int64_t stiles = (nh + mg::kScanTile - 1) / mg::kScanTile;
  const uint64_t* src_k = keys;
  const int64_t* src_p = nullptr;
  for (int p = 0; p < passes; ++p) {
    // the last pass writes the caller's arrays: out on passes with the parity of passes - 1
    const bool to_out = ((passes - 1 - p) & 1) == 0;
    uint64_t* dk = to_out ? keys_out : tk;
    int64_t* dp = to_out ? perm_out : tp;
    mg::k_rs_hist<<<grid, mg::kRsT, 0, s>>>(src_k, n, shifts[p], ntiles, hist);
    mg::k_scan_reduce<<<(unsigned)stiles, mg::kScanT, 0, s>>>(hist, nh, tsum);
    mg::k_scan_tiles<<<1, 1024, 0, s>>>(tsum, stiles);
    mg::k_scan_apply<<<(unsigned)stiles, mg::kScanT, 0, s>>>(hist, nh, tsum, base);
    mg::k_rs_scatter<<<grid, mg::kRsT, 0, s>>>(src_k, src_p, n, shifts[p], ntiles, base, dk, dp);
    src_k = dk;
    src_p = dp;
  }
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

size_t magnus_mb_scan_scratch_bytes(int64_t n) { return (size_t)((n + mg::kScanTile - 1) / mg::kScanTile + 1) * 8; }

int magnus_mb_scan(const int64_t* in, int64_t n, int64_t* out, void* scratch, void* stream) {
  if (n < 0 || !out || (n && (!in || !scratch))) return set_err(MAGNUS_INPUT, "scan: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (!n) {
    MG_CUDA(cudaMemsetAsync(out, 0, 8, s));
    return MAGNUS_OK;
  }
  const int64_t tiles = (n + mg::kScanTile - 1) / mg::kScanTile;
  int64_t* tile_sums = static_cast<int64_t*>(scratch);
  mg::k_scan_reduce<<<(unsigned)tiles, mg::kScanT, 0, s>>>(in, n, tile_sums);
  mg::k_scan_tiles<<<1, 1024, 0, s>>>(tile_sums, tiles);
  mg::k_scan_apply<<<(unsigned)tiles, mg::kScanT, 0, s>>>(in, n, tile_sums, out);
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

int magnus_mb_stream(const void* src, void* dst, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes & 15) || (((uintptr_t)src | (uintptr_t)dst) & 15))
    return set_err(MAGNUS_INPUT, "stream: 16-byte aligned buffers and sizes");
  if (!bytes) return MAGNUS_OK;
  const int64_t n16 = bytes / 16;
  const unsigned g = (unsigned)std::min<int64_t>((n16 + 255) / 256, (int64_t)sm_count() * 8);
  mg::k_mb_stream<<<g, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), n16);
  MG_CUDA(cudaGetLastError());
  return MAGNUS_OK;
}

}  // extern "C"
