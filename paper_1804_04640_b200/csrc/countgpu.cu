// countgpu.cu -- host side of libcountgpu.so: the C ABI declared in include/countstream_gpu.h.
//
// Planning (which kernel class, replica count, SIMD lane mode and row segmentation each
// query gets) happens here on the host in C++; the hot loops are the kernels in
// cs_kernels.cuh.  See DESIGN.md for the kernel classes and their rooflines.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/countstream_gpu.h"
#include "cs_common.cuh"
#include "cs_kernels.cuh"
#include "cs_itemsets.cuh"
#include "cs_radix.cuh"
#include "cs_spill.cuh"
#include "cs_ingest.cuh"
#include "cs_itemsets_sel.cuh"
#include "cs_bitmapq.cuh"
#include "cs_one.cuh"
#include "cs_comm.cuh"

using namespace cs;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CS_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      return fail(e_ == cudaErrorMemoryAllocation ? CS_ERR_OOM : CS_ERR_CUDA,          \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,    \
                  __LINE__);                                                           \
    }                                                                                  \
  } while (0)

#define CS_TRY(expr)          \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != CS_OK) return rc_; \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

double now_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s && *s ? atoi(s) : dflt;
}

}  // namespace

// K1 variants: kHist[k-1][path][column layout: uint8 / 4-bit / 2-bit] (nullptr where a path needs fewer digits)
using HistFn = void (*)(const QDesc*, const WItem*, int, int*, uint32_t*, uint32_t*, double*, double*,
                        int64_t*, uint32_t, double);
#define CS_HK3(K, P) {k_hist<K, P, 0>, k_hist<K, P, 1>, k_hist<K, P, 2>}
#define CS_HK(K)                                                                           \
  {CS_HK3(K, P_LANE16),                                                                    \
   {K <= 5 ? k_hist<(K <= 5 ? K : 5), P_PACK2, 0> : nullptr,                               \
    K <= 5 ? k_hist<(K <= 5 ? K : 5), P_PACK2, 1> : nullptr,                               \
    K <= 5 ? k_hist<(K <= 5 ? K : 5), P_PACK2, 2> : nullptr},                              \
   {K <= 5 ? k_hist<(K <= 5 ? K : 5), P_PACK4, 0> : nullptr,                               \
    K <= 5 ? k_hist<(K <= 5 ? K : 5), P_PACK4, 1> : nullptr,                               \
    K <= 5 ? k_hist<(K <= 5 ? K : 5), P_PACK4, 2> : nullptr},                              \
   CS_HK3(K, P_ROWS), CS_HK3(K, P_HALF), CS_HK3(K, P_SLICE),                                \
   {nullptr, K >= 2 ? k_hist<(K >= 2 ? K : 2), P_NARROW8, 1> : nullptr, nullptr},             \
   {nullptr, K >= 2 ? k_hist<(K >= 2 ? K : 2), P_NARROW16, 1> : nullptr, nullptr}}
static const HistFn kHist[CS_MAXK][8][3] = {CS_HK(1), CS_HK(2), CS_HK(3), CS_HK(4),
                                            CS_HK(5), CS_HK(6), CS_HK(7), CS_HK(8)};
#undef CS_HK3
#undef CS_HK

// K1r partition kernels per digit count (k >= 2)
using RadixPartFn = void (*)(const RDesc*, int, int, int64_t, char*);
using SpillHistFn = void (*)(const SDesc*, const SItem*, int, int*, uint32_t*, char*, int);
static const SpillHistFn kSpillHist[CS_MAXK] = {nullptr,         k_spill_hist<2>, k_spill_hist<3>,
                                                k_spill_hist<4>, k_spill_hist<5>, k_spill_hist<6>,
                                                k_spill_hist<7>, k_spill_hist<8>};
static const RadixPartFn kRadixPart[CS_MAXK] = {nullptr,         k_radix_part<2>, k_radix_part<3>,
                                                k_radix_part<4>, k_radix_part<5>, k_radix_part<6>,
                                                k_radix_part<7>, k_radix_part<8>};

// K7 bitmap class per digit count
using BitmapQFn = void (*)(const BDesc*, const BItem*, int, int*, int64_t, uint32_t*);
static const BitmapQFn kBitmapQ[BQ_MAXK] = {k_bitmap_query<1>, k_bitmap_query<2>, k_bitmap_query<3>,
                                            k_bitmap_query<4>};
static int bq_smem_bytes(int k) { return BQ_STAGES * k * BQ_TILE * 4; }

static int hist_path(const QDesc& d) {
  if (d.narrow == 8) return P_NARROW8;
  if (d.narrow == 16) return P_NARROW16;
  if (d.pack == 4) return P_PACK4;
  if (d.pack == 2) return P_PACK2;
  if (d.half) return P_HALF;
  if (d.scells) return P_SLICE;
  return d.mode == 0 ? P_LANE16 : P_ROWS;
}

// ------------------------------------------------------------------------------------------
// handles

struct cs_ctx {
  // every entry point that touches the context's stream, scratch, staging, pipelining bank or
  // events holds this (recursive: cs_query_batch re-enters cs_plan_execute); a context shared by
  // several databases / strategies / threads therefore serialises their calls
  std::recursive_mutex mu;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 0;
  int hist_smem = 0;      // dynamic SMEM bytes per K1 CTA
  int hist_ctas = 0;      // resident K1 CTAs (persistent grid)
  int hist_threads = CS_HIST_THREADS;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // bracket the last K1 launch
  bool ev_valid = false;
  int64_t launches = 0;
  int32_t itemset_class = 0;  // class of the last cs_itemset_supports call (CS_ITEMSETS_*)
  int smem_optin = 0;         // max dynamic SMEM per block (opt-in)
  // grow-only device scratch for host-bound outputs
  std::map<int, std::pair<void*, size_t>> scratch;
  // grow-only pinned staging
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // pipelined cs_query_batch: chunk j plans into scratch bank j&1 while chunk j-1's kernels run;
  // bank 1 has its own device scratch slots and pinned staging, each bank's staging upload is
  // guarded by an event instead of a stream sync, and per-chunk output syncs are deferred
  int bank = 0;
  bool pipe = false;
  void* pinned1 = nullptr;
  size_t pinned1_bytes = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  bool stage_ev_valid[2] = {false, false};
  // cs_query_one mailbox: page-locked, device-mapped host memory the K8 kernel stores into
  // (3 scalars, then up to ONE_MAX_CELLS table cells)
  char* mbox = nullptr;
  char* mbox_dev = nullptr;
  uint32_t one_seq = 0;
  // instance-shard merge (cs_comm_init): NCCL communicator of this context's device
  ncclComm_t comm = nullptr;
  int comm_rank = 0, comm_size = 1;
  // side streams of the histogram phase (cs_plan_execute): the per-variant persistent kernels of
  // one plan are spread over the context stream and these, forked and joined with events, so a
  // kernel's tail (SMs idle while its last items finish) is filled by the next kernel's CTAs
  static constexpr int NSIDE = 3;
  cudaStream_t side[NSIDE] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[NSIDE] = {nullptr, nullptr, nullptr};

  int scratch_get(int slot, size_t bytes, void** out) {
    auto& s = scratch[slot + 1000 * bank];
    if (s.second < bytes) {
      if (s.first) cudaFree(s.first);
      s.first = nullptr;
      s.second = 0;
      size_t want = std::max<size_t>(bytes, 256);
      CS_CUDA(cudaMalloc(&s.first, want));
      s.second = want;
    }
    *out = s.first;
    return CS_OK;
  }
  int pinned_get(size_t bytes, void** out) {
    void*& pb = bank ? pinned1 : pinned;
    size_t& pn = bank ? pinned1_bytes : pinned_bytes;
    if (pn < bytes) {
      if (pb) cudaFreeHost(pb);
      pb = nullptr;
      pn = 0;
      size_t want = std::max<size_t>(bytes, 1 << 20);
      CS_CUDA(cudaHostAlloc(&pb, want, cudaHostAllocDefault));
      pn = want;
    }
    *out = pb;
    return CS_OK;
  }
};

struct cs_db {
  cs_ctx* ctx = nullptr;
  int32_t n = 0;
  int64_t m = 0, ld = 0, m_total = 0;
  uint8_t* cols = nullptr;
  uint8_t* nib = nullptr;  // 4-bit copy (all arities <= 16), ldn bytes per column
  int64_t ldn = 0;
  uint8_t* crumb = nullptr;  // 2-bit copy (all arities <= 4), ldc bytes per column
  bool pooled = false;       // buffers from the stream-ordered pool (text ingest)
  int64_t ldc = 0;
  int32_t* d_arity = nullptr;
  std::vector<int32_t> arity;
  // bitmap index
  uint32_t* planes = nullptr;
  int64_t words = 0;
  std::vector<int64_t> plane_off;  // per var, first plane (state 0) offset in words, -1 = none
  std::vector<int64_t> plane_count;  // popcount of every plane (BitmapIndex.state_counts, bitmap.py:62)
};

struct cs_plan {
  cs_db* db = nullptr;
  int32_t nq = 0;
  uint32_t flags = 0;
  std::vector<QDesc> hq;
  std::vector<int64_t> cells, table_off;
  int64_t total_cells = 0;
  bool needs_global = false;   // some query accumulates into a global table
  bool needs_zero = false;     // tables must be zeroed before K1
  bool transient = false;      // one-shot plan (cs_query_batch): buffers come from ctx scratch
  std::vector<int32_t> score_list;    // queries scored by K2 after K1 (kind 1/2)
  struct SparseQ {  // kind 3: hash-counted queries (no dense table)
    int32_t q = 0, k = 0, rt = 0;
    uint64_t C = 0, H = 0;
    std::vector<int32_t> vars;
    std::vector<unsigned long long> stride;
    char* blob = nullptr;  // [vars | stride | keys | pkeys | cnt | pcnt | part]
    int32_t* d_vars = nullptr;
    unsigned long long *d_stride = nullptr, *keys = nullptr, *pkeys = nullptr;
    uint32_t *cnt = nullptr, *pcnt = nullptr;
    double* part = nullptr;
    int nparts = 0;
  };
  std::vector<SparseQ> sparse;
  std::vector<int32_t> generic_list;  // kind 2 queries
  // kind 4 (partition class, cs_radix.cuh): queries in wave order, processed in waves whose
  // partition buffers share one context scratch (slot 23)
  struct RadixLaunch {
    int k, first, count;  // k_radix_part<k> over RDescs [first, first + count)
  };
  struct RadixWave {
    std::vector<RadixLaunch> parts;
    int item0 = 0, nitems = 0;  // k_radix_count items
  };
  std::vector<RDesc> rdesc;
  std::vector<RadixWave> waves;
  int rx_nchunks = 0;
  size_t rx_scratch = 0;  // bytes of wave scratch
  RDesc* d_rdesc = nullptr;
  RItem* d_ritems = nullptr;
  int* d_rhead = nullptr;  // one work-queue head per wave
  // kind 6 (spill class, cs_spill.cuh): waves sharing context scratch slot 24
  struct SpillWave {
    std::vector<RadixLaunch> parts;  // k_spill_hist<k> over SItems [first, first + count)
    int item0 = 0, nitems = 0;       // k_spill_count items
  };
  std::vector<SDesc> sdesc;
  std::vector<SpillWave> swaves;
  size_t sp_scratch = 0;
  int sp_heads = 0;  // work-queue heads: one per k_spill_hist launch and one per wave
  SDesc* d_sdesc = nullptr;
  SItem* d_sitems = nullptr;
  CItem* d_citems = nullptr;
  int* d_shead = nullptr;
  struct Group {
    int key, first, count;
  };
  std::vector<Group> groups;  // SMEM-class item groups, one K1 launch each
  // kind 5 (bitmap class, cs_bitmapq.cuh): descriptors grouped by digit count, one launch per group
  struct BLaunch {
    int k, item0, nitems;
  };
  std::vector<BDesc> bdesc;
  std::vector<BLaunch> blaunch;
  BDesc* d_bdesc = nullptr;
  BItem* d_bitems = nullptr;
  int* d_bhead = nullptr;
  int nitems = 0;   // SMEM-class items (k_hist)
  int ngitems = 0;  // global-class items (k_hist_global), stored after the SMEM items
  // device
  QDesc* d_q = nullptr;
  WItem* d_items = nullptr;
  int32_t* d_score_list = nullptr;
  int32_t* d_generic_list = nullptr;
  int32_t* d_gvars = nullptr;
  uint32_t* d_gstride = nullptr;
  int* d_head = nullptr;
  uint32_t* d_done = nullptr;
  uint32_t* d_tables = nullptr;  // plan-owned table buffer when the caller gives none
  size_t d_tables_cells = 0;
  const uint32_t* last_dtab = nullptr;  // device tables of the last execute
  // chunked K2 work lists (built lazily): [0] = global-class queries, [1] = every query
  struct ScoreList {
    bool built = false;
    int nlist = 0, nitems = 0;
    char* blob = nullptr;  // [qlist | first | items | partials]
    int32_t* qlist = nullptr;
    int32_t* first = nullptr;
    ScoreItem* items = nullptr;
    double* part = nullptr;
  } sl[2];
};

struct CtxLock {  // RAII hold of cs_ctx::mu (NULL handles are reported by the callee)
  cs_ctx* c;
  explicit CtxLock(cs_ctx* x) : c(x) {
    if (c) c->mu.lock();
  }
  ~CtxLock() {
    if (c) c->mu.unlock();
  }
  CtxLock(const CtxLock&) = delete;
  CtxLock& operator=(const CtxLock&) = delete;
};

// ------------------------------------------------------------------------------------------
// library / context

extern "C" int cs_abi_version(void) { return CS_ABI_VERSION; }
extern "C" const char* cs_last_error(void) { return g_err.c_str(); }

extern "C" int cs_device_count(int32_t* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  if (count) *count = c;
  return CS_OK;
}

extern "C" int cs_ctx_create(int32_t device, cs_ctx** out) {
  if (!out) return fail(CS_ERR_INVALID, "cs_ctx_create: out is NULL");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(CS_ERR_CUDA, "cs_ctx_create: no CUDA device visible");
  }
  if (device < 0 || device >= ndev) return fail(CS_ERR_INVALID, "cs_ctx_create: bad device %d", device);
  CS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  CS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(CS_ERR_UNSUPPORTED, "libcountgpu is built for sm_100a; device %d is sm_%d%d",
                device, prop.major, prop.minor);
  cs_ctx* c = new cs_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  CS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  // K1: one 1024-thread CTA per SM with ~220 KB of dynamic SMEM (32 conflict-free replicas up
  // to C = 1760 cells, or a cp.async ring for narrow queries); measured best on cfg2
  // (profiles/README.md).  The attribute is per function (process-wide): raise it once.
  const int smem_cap = (int)prop.sharedMemPerBlockOptin - (int)sizeof(ScoreSmem) - 1024;
  c->hist_smem = std::min(env_int("CS_HIST_SMEM_KB", 220) * 1024, smem_cap);
  for (auto& a : kHist)
    for (auto& b : a)
      for (HistFn f : b)
        if (f) CS_CUDA(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap));
  int per_sm = 0;
  CS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kHist[7][0][0], CS_HIST_THREADS,
                                                        c->hist_smem));
  if (per_sm < 1) return fail(CS_ERR_CUDA, "k_hist does not fit on an SM with %d B smem", c->hist_smem);
  for (RadixPartFn f : kRadixPart)
    if (f) CS_CUDA(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, RX_SMEM));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_radix_count, cudaFuncAttributeMaxDynamicSharedMemorySize, RC_SMEM));
  for (SpillHistFn f : kSpillHist)
    if (f) CS_CUDA(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_spill_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               SP_COUNT_SMEM));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_query_one, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(ONE_MAX_CELLS * 4)));
  for (int k = 1; k <= BQ_MAXK; ++k)
    CS_CUDA(cudaFuncSetAttribute((const void*)kBitmapQ[k - 1], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 bq_smem_bytes(k)));
  {  // keep freed ingest scratch in the device's stream-ordered pool between loads
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  // the other large-SMEM kernels (function attributes are per device: set them per context)
  c->smem_optin = (int)prop.sharedMemPerBlockOptin;
  CS_CUDA(cudaFuncSetAttribute((const void*)k_itemsets_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               c->smem_optin - 2048));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_sel_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_txt_parse<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_txt_parse<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024));
  CS_CUDA(cudaFuncSetAttribute((const void*)k_txt_parse_thr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024));
  CS_CUDA(cudaEventCreate(&c->ev0));
  CS_CUDA(cudaEventCreate(&c->ev1));
  CS_CUDA(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
  for (int i = 0; i < cs_ctx::NSIDE; ++i) {
    CS_CUDA(cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking));
    CS_CUDA(cudaEventCreateWithFlags(&c->join_ev[i], cudaEventDisableTiming));
  }
  c->hist_ctas = per_sm * c->num_sms;
  *out = c;
  return CS_OK;
}

extern "C" int cs_ctx_destroy(cs_ctx* ctx) {
  if (!ctx) return CS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->scratch)
    if (kv.second.first) cudaFree(kv.second.first);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->pinned1) cudaFreeHost(ctx->pinned1);
  if (ctx->mbox) cudaFreeHost(ctx->mbox);
  if (ctx->comm) nccl_api().CommDestroy(ctx->comm);
  for (auto& e : ctx->stage_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  for (int i = 0; i < cs_ctx::NSIDE; ++i) {
    if (ctx->side[i]) {
      cudaStreamSynchronize(ctx->side[i]);
      cudaStreamDestroy(ctx->side[i]);
    }
    if (ctx->join_ev[i]) cudaEventDestroy(ctx->join_ev[i]);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return CS_OK;
}

extern "C" int cs_ctx_set_stream(cs_ctx* ctx, void* stream) {
  CtxLock lk_(ctx);
  if (!ctx) return fail(CS_ERR_INVALID, "cs_ctx_set_stream: NULL ctx");
  if (ctx->own_stream && ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
    ctx->own_stream = false;
  } else {
    CS_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  return CS_OK;
}

extern "C" int cs_ctx_sync(cs_ctx* ctx) {
  if (!ctx) return fail(CS_ERR_INVALID, "cs_ctx_sync: NULL ctx");
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

extern "C" int cs_ctx_launch_count(cs_ctx* ctx, int64_t* launches) {
  if (!ctx || !launches) return fail(CS_ERR_INVALID, "cs_ctx_launch_count: NULL argument");
  *launches = ctx->launches;
  return CS_OK;
}

extern "C" int cs_ctx_last_kernel_ms(cs_ctx* ctx, float* ms) {
  CtxLock lk_(ctx);
  if (!ctx || !ms) return fail(CS_ERR_INVALID, "cs_ctx_last_kernel_ms: NULL argument");
  *ms = 0.f;
  if (!ctx->ev_valid) return CS_OK;
  CS_CUDA(cudaEventSynchronize(ctx->ev1));
  CS_CUDA(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  return CS_OK;
}

extern "C" int cs_ctx_itemset_class(cs_ctx* ctx, int32_t* cls) {
  if (!ctx || !cls) return fail(CS_ERR_INVALID, "cs_ctx_itemset_class: NULL argument");
  *cls = ctx->itemset_class;
  return CS_OK;
}

extern "C" int cs_ctx_info(cs_ctx* ctx, int32_t* num_sms, int32_t* hist_smem_bytes,
                           int32_t* hist_ctas) {
  if (!ctx) return fail(CS_ERR_INVALID, "cs_ctx_info: NULL ctx");
  if (num_sms) *num_sms = ctx->num_sms;
  if (hist_smem_bytes) *hist_smem_bytes = ctx->hist_smem;
  if (hist_ctas) *hist_ctas = ctx->hist_ctas;
  return CS_OK;
}

// ------------------------------------------------------------------------------------------
// database

// Database buffers: cudaMalloc, or (databases parsed from text) the device's stream-ordered
// pool, whose freed blocks are kept for the next load instead of a cudaMalloc / cudaFree pair
static cudaError_t db_malloc(cs_db* db, void** p, size_t bytes) {
  return db->pooled ? cudaMallocAsync(p, bytes, db->ctx->stream) : cudaMalloc(p, bytes);
}
static void db_free(cs_db* db, void* p) {
  if (!p) return;
  if (db->pooled) cudaFreeAsync(p, db->ctx->stream);
  else cudaFree(p);
}

// 4-bit / 2-bit column copies for the bandwidth-bound histogram kernels, from db->arity
static int db_alloc_copies(cs_db* db) {
  cs_ctx* ctx = db->ctx;
  const int n = db->n;
  const int64_t m = db->m;
  const std::vector<int32_t>& arities = db->arity;
  // 4-bit copy for the bandwidth-bound histogram kernels when every arity fits a nibble
  bool small = env_int("CS_NIBBLE", 1) != 0;
  for (int i = 0; i < n && small; ++i) small = arities[i] <= 16;
  if (small) {
    db->ldn = round_up((m + 1) / 2, 256);
    if (db_malloc(db, (void**)&db->nib, (size_t)n * db->ldn) != cudaSuccess) {
      cudaGetLastError();  // not enough memory: the kernels read the uint8 columns instead
      db->nib = nullptr;
      db->ldn = 0;
    } else {
      CS_CUDA(cudaMemsetAsync(db->nib, 0, (size_t)n * db->ldn, ctx->stream));
    }
  }
  // 2-bit copy when every arity <= 4 (the histogram kernels' smallest row footprint)
  bool tiny = env_int("CS_CRUMB", 1) != 0;
  for (int i = 0; i < n && tiny; ++i) tiny = arities[i] <= 4;
  if (tiny) {
    db->ldc = round_up((m + 3) / 4, 256);
    if (db_malloc(db, (void**)&db->crumb, (size_t)n * db->ldc) != cudaSuccess) {
      cudaGetLastError();
      db->crumb = nullptr;
      db->ldc = 0;
    } else {
      CS_CUDA(cudaMemsetAsync(db->crumb, 0, (size_t)n * db->ldc, ctx->stream));
    }
  }
  return CS_OK;
}

static int db_alloc(cs_ctx* ctx, int32_t n, int64_t m, const int32_t* arities, cs_db** out,
                    bool copies = true, bool pooled = false) {
  if (!ctx || !out) return fail(CS_ERR_INVALID, "cs_db: NULL argument");
  if (n < 1 || m < 1)
    return fail(CS_ERR_INVALID, "database must have at least one variable and one row, got n=%d m=%lld",
                n, (long long)m);
  if (!arities) return fail(CS_ERR_INVALID, "cs_db: arities is NULL");
  if (m > (int64_t)UINT32_MAX)
    return fail(CS_ERR_UNSUPPORTED, "database has %lld rows; the uint32 count tables hold at most 2^32-1 records",
                (long long)m);
  for (int i = 0; i < n; ++i) {
    if (arities[i] < 1) return fail(CS_ERR_INVALID, "every arity must be at least 1 (variable %d)", i);
    if (arities[i] > CS_MAX_ARITY)
      return fail(CS_ERR_UNSUPPORTED,
                  "variable %d has arity %d; the uint8 column layout supports arity <= 256", i,
                  arities[i]);
  }
  CS_CUDA(cudaSetDevice(ctx->device));
  cs_db* db = new cs_db();
  db->ctx = ctx;
  db->n = n;
  db->m = m;
  db->m_total = m;
  db->ld = round_up(m, 256);
  db->arity.assign(arities, arities + n);
  db->plane_off.assign(n, -1);
  db->pooled = pooled;
  cudaError_t e = db_malloc(db, (void**)&db->cols, (size_t)n * db->ld);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete db;
    return fail(CS_ERR_OOM, "cs_db: cannot allocate %lld bytes of columns: %s",
                (long long)n * db->ld, cudaGetErrorString(e));
  }
  CS_CUDA(db_malloc(db, (void**)&db->d_arity, sizeof(int32_t) * n));
  CS_CUDA(cudaMemcpyAsync(db->d_arity, arities, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                          ctx->stream));
  // zero padding (and everything: generated DBs fill columns later)
  CS_CUDA(cudaMemsetAsync(db->cols, 0, (size_t)n * db->ld, ctx->stream));
  if (copies) CS_TRY(db_alloc_copies(db));
  *out = db;
  return CS_OK;
}

// (re)pack columns [var0, var0 + nvars) into the 4-bit copy
static int db_pack(cs_db* db, int32_t var0, int32_t nvars) {
  if (db->crumb && nvars > 0) {
    const int64_t w16 = (db->m + 15) >> 4;
    dim3 g2((unsigned)std::min<int64_t>((w16 + 255) / 256, 2048), (unsigned)std::min(nvars, 1024));
    k_pack2<<<g2, 256, 0, db->ctx->stream>>>(db->cols, db->ld, db->crumb, db->ldc, db->m, var0, nvars);
    db->ctx->launches++;
    CS_CUDA(cudaGetLastError());
  }
  if (!db->nib || nvars <= 0) return CS_OK;
  cs_ctx* ctx = db->ctx;
  const int64_t words = (db->m + 7) >> 3;
  dim3 grid((unsigned)std::min<int64_t>((words + 255) / 256, 2048), (unsigned)std::min(nvars, 1024));
  k_pack4<<<grid, 256, 0, ctx->stream>>>(db->cols, db->ld, db->nib, db->ldn, db->m, var0, nvars);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  return CS_OK;
}

extern "C" int cs_db_create_empty(cs_ctx* ctx, int32_t n, int64_t m, const int32_t* arities,
                                  cs_db** out) {
  CtxLock lk_(ctx);
  return db_alloc(ctx, n, m, arities, out);
}

extern "C" int cs_db_create(cs_ctx* ctx, const uint8_t* cols, int32_t n, int64_t m, int64_t ld,
                            const int32_t* arities, cs_db** out) {
  CtxLock lk_(ctx);
  if (!cols) return fail(CS_ERR_INVALID, "cs_db_create: cols is NULL");
  if (ld < m) return fail(CS_ERR_INVALID, "cs_db_create: ld %lld < m %lld", (long long)ld, (long long)m);
  cs_db* db = nullptr;
  CS_TRY(db_alloc(ctx, n, m, arities, &db));
  const cudaMemcpyKind kind = is_device_ptr(cols) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CS_CUDA(cudaMemcpy2DAsync(db->cols, db->ld, cols, ld, m, n, kind, ctx->stream));
  // validate states against declared arities (Database.__init__, database.py:61-77)
  unsigned long long* d_bad = nullptr;
  CS_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long) * n));
  CS_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long) * n, ctx->stream));
  dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 1024), (unsigned)std::min(n, 65535));
  k_check_states<<<grid, 256, 0, ctx->stream>>>(db->cols, db->ld, m, db->d_arity, d_bad, n);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  std::vector<unsigned long long> bad(n);
  CS_CUDA(cudaMemcpyAsync(bad.data(), d_bad, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost,
                          ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_bad);
  for (int i = 0; i < n; ++i) {
    if (bad[i] != ~0ull) {
      uint8_t st = 0;
      cudaMemcpy(&st, db->cols + (int64_t)i * db->ld + (int64_t)bad[i], 1, cudaMemcpyDeviceToHost);
      int rc = fail(CS_ERR_INVALID, "row %lld: variable %d has state %d, exceeding declared arity %d",
                    (long long)bad[i] + 1, i, (int)st, db->arity[i]);
      cudaFree(db->cols);
      cudaFree(db->d_arity);
      delete db;
      return rc;
    }
  }
  CS_TRY(db_pack(db, 0, n));
  *out = db;
  return CS_OK;
}

extern "C" int cs_db_generate(cs_db* db, int32_t var, uint64_t seed, int64_t row_offset,
                              int32_t nparents, const int32_t* parents, const uint32_t* thresholds,
                              int64_t nthresholds) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db) return fail(CS_ERR_INVALID, "cs_db_generate: NULL db");
  if (var < 0 || var >= db->n) return fail(CS_ERR_INVALID, "cs_db_generate: bad var %d", var);
  if (nparents < 0 || nparents > CS_MAXK) return fail(CS_ERR_INVALID, "cs_db_generate: nparents %d", nparents);
  const int r = db->arity[var];
  int64_t q = 1;
  std::vector<const uint8_t*> pcols(nparents);
  std::vector<uint32_t> pstride(nparents);
  for (int t = 0; t < nparents; ++t) {
    const int p = parents[t];
    if (p < 0 || p >= db->n || p == var) return fail(CS_ERR_INVALID, "cs_db_generate: bad parent %d", p);
    pcols[t] = db->cols + (int64_t)p * db->ld;
    pstride[t] = (uint32_t)q;
    q *= db->arity[p];
    if (q > (1 << 24)) return fail(CS_ERR_INVALID, "cs_db_generate: parent space too large");
  }
  if (nthresholds != q * (r - 1))
    return fail(CS_ERR_INVALID, "cs_db_generate: expected %lld thresholds, got %lld",
                (long long)(q * (r - 1)), (long long)nthresholds);
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  // one small device blob: [pcols][pstride][thr]
  size_t bytes = sizeof(void*) * std::max(nparents, 1) + sizeof(uint32_t) * std::max(nparents, 1) +
                 sizeof(uint32_t) * std::max<int64_t>(nthresholds, 1);
  char* blob = nullptr;
  CS_CUDA(cudaMalloc(&blob, bytes));
  std::vector<char> h(bytes, 0);
  size_t o1 = sizeof(void*) * std::max(nparents, 1);
  size_t o2 = o1 + sizeof(uint32_t) * std::max(nparents, 1);
  if (nparents) {
    memcpy(h.data(), pcols.data(), sizeof(void*) * nparents);
    memcpy(h.data() + o1, pstride.data(), sizeof(uint32_t) * nparents);
  }
  if (nthresholds) memcpy(h.data() + o2, thresholds, sizeof(uint32_t) * nthresholds);
  CS_CUDA(cudaMemcpyAsync(blob, h.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  const int64_t m = db->m;
  unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_generate<<<grid, 256, 0, ctx->stream>>>(db->cols + (int64_t)var * db->ld, m, column_key(seed, var),
                                            row_offset, nparents, (const uint8_t* const*)blob,
                                            (const uint32_t*)(blob + o1), (const uint32_t*)(blob + o2),
                                            r - 1);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  CS_TRY(db_pack(db, var, 1));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(blob);
  return CS_OK;
}

extern "C" int cs_db_destroy(cs_db* db) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db) return CS_OK;
  cudaSetDevice(db->ctx->device);
  cudaStreamSynchronize(db->ctx->stream);
  db_free(db, db->cols);
  db_free(db, db->nib);
  db_free(db, db->crumb);
  db_free(db, db->d_arity);
  if (db->pooled) cudaStreamSynchronize(db->ctx->stream);
  if (db->planes) cudaFree(db->planes);
  delete db;
  return CS_OK;
}

extern "C" int cs_db_shape(cs_db* db, int32_t* n, int64_t* m, int64_t* ld) {
  if (!db) return fail(CS_ERR_INVALID, "cs_db_shape: NULL db");
  if (n) *n = db->n;
  if (m) *m = db->m;
  if (ld) *ld = db->ld;
  return CS_OK;
}

extern "C" int cs_db_columns(cs_db* db, const uint8_t** dev, int64_t* ld) {
  if (!db) return fail(CS_ERR_INVALID, "cs_db_columns: NULL db");
  if (dev) *dev = db->cols;
  if (ld) *ld = db->ld;
  return CS_OK;
}

extern "C" int cs_db_download(cs_db* db, int32_t var, int64_t row0, int64_t nrows, uint8_t* host) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db || !host) return fail(CS_ERR_INVALID, "cs_db_download: NULL argument");
  if (var < 0 || var >= db->n || row0 < 0 || nrows < 0 || row0 + nrows > db->m)
    return fail(CS_ERR_INVALID, "cs_db_download: out of range");
  CS_CUDA(cudaSetDevice(db->ctx->device));
  CS_CUDA(cudaMemcpyAsync(host, db->cols + (int64_t)var * db->ld + row0, nrows, cudaMemcpyDeviceToHost,
                          db->ctx->stream));
  CS_CUDA(cudaStreamSynchronize(db->ctx->stream));
  return CS_OK;
}

extern "C" int cs_db_arities(cs_db* db, int32_t* arities) {
  if (!db || !arities) return fail(CS_ERR_INVALID, "cs_db_arities: NULL argument");
  std::copy(db->arity.begin(), db->arity.end(), arities);
  return CS_OK;
}

extern "C" int cs_db_set_total_rows(cs_db* db, int64_t m_total) {
  if (!db || m_total < db->m) return fail(CS_ERR_INVALID, "cs_db_set_total_rows: bad argument");
  if (m_total > (int64_t)UINT32_MAX)
    return fail(CS_ERR_UNSUPPORTED, "%lld total rows: merged uint32 count tables hold at most 2^32-1 records",
                (long long)m_total);
  db->m_total = m_total;
  return CS_OK;
}

// ------------------------------------------------------------------------------------------
// text ingest (cs_ingest.cuh; reference load_csv, database.py:160-207)

namespace {

// RAII bag of stream-ordered temporaries
struct TmpBag {
  cudaStream_t st;
  std::vector<void*> p;
  explicit TmpBag(cudaStream_t s) : st(s) {}
  ~TmpBag() {
    for (void* x : p) cudaFreeAsync(x, st);
  }
  template <class T>
  int get(size_t count, T** out) {
    void* x = nullptr;
    cudaError_t e = cudaMallocAsync(&x, std::max<size_t>(count * sizeof(T), 16), st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(e == cudaErrorMemoryAllocation ? CS_ERR_OOM : CS_ERR_CUDA, "ingest scratch (%zu B): %s",
                  count * sizeof(T), cudaGetErrorString(e));
    }
    p.push_back(x);
    *out = static_cast<T*>(x);
    return CS_OK;
  }
};

// exclusive scan of n int64 on the context stream (tiles of TX_SCAN_TILE, recursive on totals)
int scan64(cs_ctx* ctx, TmpBag& bag, int64_t* d, int64_t n) {
  const int64_t tiles = (n + TX_SCAN_TILE - 1) / TX_SCAN_TILE;
  if (tiles <= 1) {
    k_scan64_tiles<<<1, 1024, 0, ctx->stream>>>(d, n, nullptr);
    ctx->launches++;
    CS_CUDA(cudaGetLastError());
    return CS_OK;
  }
  int64_t* sums = nullptr;
  CS_TRY(bag.get(tiles, &sums));
  k_scan64_tiles<<<(unsigned)tiles, 1024, 0, ctx->stream>>>(d, n, sums);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  CS_TRY(scan64(ctx, bag, sums, tiles));
  k_scan64_add<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(d, n, sums);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  return CS_OK;
}

template <class T>
int d2h(cs_ctx* ctx, T* host, const T* dev, size_t count = 1) {
  CS_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

// host -> device copy of a large pageable buffer: pinned in place when the driver allows it,
// else staged through the context's pinned buffer (two halves, event-guarded)
int h2d_large(cs_ctx* ctx, void* dst, const void* src, size_t bytes) {
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
    CS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));  // pinned: DMA directly
    return CS_OK;
  }
  cudaGetLastError();
  if (bytes >= (1u << 30) &&
      cudaHostRegister(const_cast<void*>(src), bytes, cudaHostRegisterReadOnly) == cudaSuccess) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
    cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
    cudaHostUnregister(const_cast<void*>(src));
    CS_CUDA(e);
    CS_CUDA(e2);
    return CS_OK;
  }
  cudaGetLastError();
  const size_t CH = 32u << 20;
  void* pin = nullptr;
  CS_TRY(ctx->pinned_get(2 * CH, &pin));
  cudaEvent_t ev[2];
  CS_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CS_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  int rc = CS_OK;
  for (size_t off = 0, i = 0; off < bytes && rc == CS_OK; off += CH, ++i) {
    const size_t len = std::min(CH, bytes - off);
    char* stage = static_cast<char*>(pin) + (i & 1) * CH;
    if (i >= 2 && cudaEventSynchronize(ev[i & 1]) != cudaSuccess) rc = fail(CS_ERR_CUDA, "h2d stage wait");
    if (rc != CS_OK) break;
    // pageable -> pinned with several host threads (one memcpy thread moves ~10 GB/s)
    const char* from = static_cast<const char*>(src) + off;
    const int nt = (int)std::min<size_t>(8, std::max<size_t>(1, len >> 22));
    std::vector<std::thread> pool;
    const size_t per = (len + nt - 1) / nt;
    for (int t = 1; t < nt; ++t) {
      const size_t a = t * per, b = std::min(len, a + per);
      if (a < b) pool.emplace_back([=] { memcpy(stage + a, from + a, b - a); });
    }
    memcpy(stage, from, std::min(len, per));
    for (auto& th : pool) th.join();
    if (cudaMemcpyAsync(static_cast<char*>(dst) + off, stage, len, cudaMemcpyHostToDevice, ctx->stream) !=
            cudaSuccess ||
        cudaEventRecord(ev[i & 1], ctx->stream) != cudaSuccess)
      rc = fail(CS_ERR_CUDA, "h2d staged copy failed");
  }
  cudaStreamSynchronize(ctx->stream);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  return rc;
}

}  // namespace

extern "C" int cs_db_load_text(cs_ctx* ctx, const char* text, int64_t nbytes, int32_t delim,
                               const int32_t* arities, int32_t n_arities, cs_db** out, int64_t* info) {
  CtxLock lk_(ctx);
  if (!ctx || !out || !info || (!text && nbytes > 0) || nbytes < 0)
    return fail(CS_ERR_INVALID, "cs_db_load_text: bad argument");
  if (delim < CS_DELIM_WHITESPACE || delim > 255)
    return fail(CS_ERR_INVALID, "cs_db_load_text: delimiter must be a byte, CS_DELIM_SNIFF or CS_DELIM_WHITESPACE");
  for (int i = 0; i < 8; ++i) info[i] = 0;
  *out = nullptr;
  if (nbytes == 0) {
    info[0] = CS_LOAD_NO_RECORDS;
    return fail(CS_ERR_PARSE, "no records found");
  }
  CS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  TmpBag bag(st);
  // 1. text on the device, zero padded (vector loads and the look-ahead byte stay in bounds)
  const int64_t tbytes = round_up(nbytes, 64) + TX_PAD;
  uint8_t* dt = nullptr;
  CS_TRY(bag.get(tbytes, &dt));
  CS_CUDA(cudaMemsetAsync(dt + nbytes, 0, tbytes - nbytes, st));
  if (is_device_ptr(text)) {
    CS_CUDA(cudaMemcpyAsync(dt, text, nbytes, cudaMemcpyDeviceToDevice, st));
  } else {
    CS_TRY(h2d_large(ctx, dt, text, nbytes));
  }
  // 2. line boundaries
  const int64_t nch = (nbytes + TX_CHUNK - 1) / TX_CHUNK;
  if (nch > INT32_MAX) return fail(CS_ERR_UNSUPPORTED, "text too large");
  int64_t* cnt = nullptr;
  CS_TRY(bag.get(nch + 1, &cnt));
  CS_CUDA(cudaMemsetAsync(cnt + nch, 0, sizeof(int64_t), st));
  k_txt_breaks<false><<<(unsigned)nch, TX_THREADS, 0, st>>>(dt, nbytes, cnt, nullptr, nullptr);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  CS_TRY(scan64(ctx, bag, cnt, nch + 1));
  int64_t nbrk = 0;
  CS_TRY(d2h(ctx, &nbrk, cnt + nch));
  int64_t* brk = nullptr;
  CS_TRY(bag.get(nbrk + 1, &brk));
  k_txt_breaks<true><<<(unsigned)nch, TX_THREADS, 0, st>>>(dt, nbytes, nullptr, cnt, brk);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  // 3. lines -> stripped bounds, non-empty flags -> record map
  const int64_t nl = nbrk + 1;
  int64_t *la = nullptr, *lb = nullptr, *ne = nullptr, *rank = nullptr;
  CS_TRY(bag.get(nl, &la));
  CS_TRY(bag.get(nl, &lb));
  CS_TRY(bag.get(nl + 1, &ne));
  CS_TRY(bag.get(nl + 1, &rank));
  const unsigned lgrid = (unsigned)std::min<int64_t>((nl + 7) / 8, (int64_t)ctx->num_sms * 16);
  k_txt_lines<<<lgrid, 256, 0, st>>>(dt, nbytes, brk, nl, la, lb, ne);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  CS_CUDA(cudaMemsetAsync(ne + nl, 0, sizeof(int64_t), st));
  CS_CUDA(cudaMemcpyAsync(rank, ne, sizeof(int64_t) * (nl + 1), cudaMemcpyDeviceToDevice, st));
  CS_TRY(scan64(ctx, bag, rank, nl + 1));
  int64_t nrec = 0;
  CS_TRY(d2h(ctx, &nrec, rank + nl));
  if (nrec == 0) {
    info[0] = CS_LOAD_NO_RECORDS;
    return fail(CS_ERR_PARSE, "no records found");
  }
  if (nrec > INT32_MAX) return fail(CS_ERR_UNSUPPORTED, "more than 2^31-1 records");
  int64_t* rec_line = nullptr;
  CS_TRY(bag.get(nrec, &rec_line));
  k_txt_compact<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(ne, rank, nl, rec_line);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  // 4. delimiter sniff and record width from the first record (reference: `"," in lines[0]`)
  int64_t* dhead = nullptr;
  CS_TRY(bag.get(4, &dhead));
  k_txt_head<<<1, 32, 0, st>>>(dt, la, lb, rec_line, delim >= 0 ? delim : ',', dhead);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  int64_t head[4];
  CS_TRY(d2h(ctx, head, dhead, 4));
  int32_t kd = delim;  // kernel delimiter: < 0 = whitespace
  if (delim == CS_DELIM_SNIFF) kd = head[0] ? ',' : -1;
  if (kd == CS_DELIM_WHITESPACE) kd = -1;
  const int64_t width = kd < 0 ? head[1] : head[2];
  info[1] = width;
  info[2] = nrec;
  info[3] = kd;
  if (width > 50000) return fail(CS_ERR_UNSUPPORTED, "records of %lld values: the loader supports <= 50000", (long long)width);
  // 5. database with placeholder arities (fixed below), then the parse
  std::vector<int32_t> ones(width, 1);
  cs_db* db = nullptr;
  CS_TRY(db_alloc(ctx, (int32_t)width, nrec, ones.data(), &db, /*copies=*/false, /*pooled=*/true));
  int rc = CS_OK;
  auto drop = [&](int code) {
    cs_db_destroy(db);
    return code;
  };
  int *colmax = nullptr, *gmin = nullptr;
  unsigned long long* bad = nullptr;
  if ((rc = bag.get(width, &colmax)) || (rc = bag.get(1, &gmin)) || (rc = bag.get(1, &bad))) return drop(rc);
  cudaMemsetAsync(colmax, 0x80, sizeof(int) * width, st);  // 0x80808080 < -TX_SAT
  cudaMemsetAsync(gmin, 0x7f, sizeof(int), st);            // 0x7f7f7f7f > TX_SAT
  cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st);
  if (width <= 256) {
    // thread per record, SMEM tile [W][256]
    const unsigned pgrid = (unsigned)((nrec + TX_THREADS - 1) / TX_THREADS);
    k_txt_parse_thr<<<pgrid, TX_THREADS, width * TX_THREADS, st>>>(dt, la, lb, rec_line, nrec, (int32_t)width, kd,
                                                                   db->cols, db->ld, colmax, gmin, bad);
  } else {
    // warp per record (long records), SMEM tile [W][tr]
    int tr = 256;
    while (tr > 32 && 4 * width + width * (int64_t)tr > 48 * 1024) tr >>= 1;
    const bool direct = 4 * width + width * (int64_t)tr > 200 * 1024;
    const size_t smem = 4 * width + (direct ? 0 : width * (int64_t)tr);
    const unsigned pgrid = (unsigned)((nrec + tr - 1) / tr);
    if (direct)
      k_txt_parse<true><<<pgrid, TX_THREADS, smem, st>>>(dt, la, lb, rec_line, nrec, (int32_t)width, kd, tr,
                                                         db->cols, db->ld, colmax, gmin, bad);
    else
      k_txt_parse<false><<<pgrid, TX_THREADS, smem, st>>>(dt, la, lb, rec_line, nrec, (int32_t)width, kd, tr,
                                                          db->cols, db->ld, colmax, gmin, bad);
  }
  ctx->launches++;
  if (cudaGetLastError() != cudaSuccess) return drop(fail(CS_ERR_CUDA, "k_txt_parse launch failed"));
  unsigned long long hbad = 0;
  int hmin = 0;
  std::vector<int> cmax(width);
  if ((rc = d2h(ctx, &hbad, bad)) || (rc = d2h(ctx, &hmin, gmin)) || (rc = d2h(ctx, cmax.data(), colmax, width)))
    return drop(rc);
  // 6. the reference's error order: first bad record, negative states, then Database checks
  if (hbad != ~0ull) {
    int64_t ln = 0;
    if ((rc = d2h(ctx, &ln, rec_line + hbad)) || (rc = d2h(ctx, &info[5], la + ln)) || (rc = d2h(ctx, &info[6], lb + ln)))
      return drop(rc);
    info[0] = CS_LOAD_BAD_RECORD;
    info[4] = (int64_t)hbad;
    return drop(fail(CS_ERR_PARSE, "record %llu is ragged or holds a non-integer token", hbad));
  }
  if (hmin < 0) {
    info[0] = CS_LOAD_NEGATIVE;
    info[4] = hmin;
    return drop(fail(CS_ERR_PARSE, "negative state %d; states must be >= 0", hmin));
  }
  const bool shift = hmin == 1;
  if (shift) {
    dim3 g((unsigned)std::min<int64_t>((nrec / 4 + 255) / 256 + 1, 1024), (unsigned)std::min<int64_t>(width, 65535));
    k_txt_shift<<<g, 256, 0, st>>>(db->cols, db->ld, nrec, (int)width);
    ctx->launches++;
    if (cudaGetLastError() != cudaSuccess) return drop(fail(CS_ERR_CUDA, "k_txt_shift launch failed"));
  }
  info[7] = shift;
  std::vector<int32_t> ar(width);
  for (int64_t i = 0; i < width; ++i) ar[i] = cmax[i] - (shift ? 1 : 0) + 1;  // observed arity
  // states above 255 do not fit the uint8 layout (Database.columns_u8's check, raised before the
  // declared-arity checks because the stored bytes no longer hold them)
  const int32_t amax = *std::max_element(ar.begin(), ar.end());
  if (amax > CS_MAX_ARITY)
    return drop(fail(CS_ERR_UNSUPPORTED,
                     "the GPU engine stores states as uint8; arities above 256 are unsupported (max arity %d)",
                     amax));
  if (arities) {
    if (n_arities != width) {
      info[0] = CS_LOAD_ARITY_COUNT;
      info[4] = n_arities;
      return drop(fail(CS_ERR_PARSE, "expected %lld arities, got %d", (long long)width, n_arities));
    }
    for (int64_t i = 0; i < width; ++i) {
      if (arities[i] < ar[i]) {  // first short variable, then its first offending row
        const int32_t ai = std::max(0, arities[i]);
        unsigned long long* dbad = nullptr;
        if ((rc = bag.get(1, &dbad))) return drop(rc);
        cudaMemcpyAsync(db->d_arity + i, &ai, sizeof(int32_t), cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(dbad, 0xff, sizeof(unsigned long long), st);
        dim3 g((unsigned)std::min<int64_t>((nrec + 255) / 256, 1024), 1);
        k_check_states<<<g, 256, 0, st>>>(db->cols + i * db->ld, db->ld, nrec, db->d_arity + i, dbad, 1);
        ctx->launches++;
        unsigned long long row = 0;
        uint8_t state = 0;
        if ((rc = d2h(ctx, &row, dbad)) || (rc = d2h(ctx, &state, db->cols + i * db->ld + row))) return drop(rc);
        info[0] = CS_LOAD_ARITY_SHORT;
        info[4] = (int64_t)row;
        info[5] = i;
        info[6] = state;
        return drop(fail(CS_ERR_PARSE, "row %llu: variable %lld has state %d, exceeding declared arity %d",
                         row + 1, (long long)i, (int)state, arities[i]));
      }
    }
    for (int64_t i = 0; i < width; ++i) ar[i] = arities[i];
    for (int64_t i = 0; i < width; ++i)
      if (ar[i] < 1) {
        info[0] = CS_LOAD_ARITY_ZERO;
        return drop(fail(CS_ERR_PARSE, "every arity must be at least 1"));
      }
    if (*std::max_element(ar.begin(), ar.end()) > CS_MAX_ARITY)
      return drop(fail(CS_ERR_UNSUPPORTED,
                       "the GPU engine stores states as uint8; arities above 256 are unsupported (max arity %d)",
                       *std::max_element(ar.begin(), ar.end())));
  }
  db->arity = ar;
  CS_CUDA(cudaMemcpyAsync(db->d_arity, ar.data(), sizeof(int32_t) * width, cudaMemcpyHostToDevice, st));
  if ((rc = db_alloc_copies(db))) return drop(rc);  // now that the arities are known
  if ((rc = db_pack(db, 0, db->n))) return drop(rc);
  CS_CUDA(cudaStreamSynchronize(st));
  *out = db;
  return CS_OK;
}

// ------------------------------------------------------------------------------------------
// bitmap index

extern "C" int cs_bitmap_build(cs_db* db, int32_t nvars, const int32_t* vars) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db) return fail(CS_ERR_INVALID, "cs_bitmap_build: NULL db");
  std::vector<int32_t> list;
  if (!vars || nvars < 0) {
    list.resize(db->n);
    std::iota(list.begin(), list.end(), 0);
  } else {
    for (int i = 0; i < nvars; ++i) {
      if (vars[i] < 0 || vars[i] >= db->n) return fail(CS_ERR_INVALID, "cs_bitmap_build: bad var %d", vars[i]);
      list.push_back(vars[i]);
    }
  }
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  // (re)build the whole pool: planes of previously indexed vars are kept by re-adding them
  for (int v = 0; v < db->n; ++v)
    if (db->plane_off[v] >= 0 && std::find(list.begin(), list.end(), v) == list.end()) list.push_back(v);
  std::sort(list.begin(), list.end());
  list.erase(std::unique(list.begin(), list.end()), list.end());
  const int64_t words = round_up((db->m + 31) / 32, 32);
  int64_t total = 0;
  std::vector<int64_t> off(list.size());
  for (size_t i = 0; i < list.size(); ++i) {
    off[i] = total;
    total += words * db->arity[list[i]];
  }
  if (db->planes) {
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(db->planes);
    db->planes = nullptr;
  }
  CS_CUDA(cudaMalloc(&db->planes, sizeof(uint32_t) * std::max<int64_t>(total, 1)));
  db->words = words;
  std::fill(db->plane_off.begin(), db->plane_off.end(), -1);
  for (size_t i = 0; i < list.size(); ++i) db->plane_off[list[i]] = off[i];
  if (list.empty()) return CS_OK;
  int32_t* d_vars = nullptr;
  int64_t* d_off = nullptr;
  CS_CUDA(cudaMalloc(&d_vars, sizeof(int32_t) * list.size()));
  CS_CUDA(cudaMalloc(&d_off, sizeof(int64_t) * list.size()));
  CS_CUDA(cudaMemcpyAsync(d_vars, list.data(), sizeof(int32_t) * list.size(), cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * list.size(), cudaMemcpyHostToDevice, ctx->stream));
  dim3 grid((unsigned)std::min<int64_t>((words + 255) / 256, 4096), (unsigned)std::min<size_t>(list.size(), 65535));
  k_bitmap_build<<<grid, 256, 0, ctx->stream>>>(db->cols, db->ld, db->m, d_vars, db->d_arity, d_off,
                                                 db->planes, words, (int)list.size());
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  // per-plane record counts (the index's state counts): the itemset planner ranks items by them
  const int64_t nplanes = total / words;
  unsigned long long* d_cnt = nullptr;
  CS_CUDA(cudaMalloc(&d_cnt, sizeof(unsigned long long) * nplanes));
  CS_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * nplanes, ctx->stream));
  k_plane_popc<<<dim3(8, (unsigned)std::min<int64_t>(nplanes, 65535)), 256, 0, ctx->stream>>>(db->planes, words,
                                                                                               d_cnt, nplanes);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  db->plane_count.assign(nplanes, 0);
  CS_CUDA(cudaMemcpyAsync(db->plane_count.data(), d_cnt, sizeof(int64_t) * nplanes, cudaMemcpyDeviceToHost,
                          ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_cnt);
  cudaFree(d_vars);
  cudaFree(d_off);
  return CS_OK;
}

extern "C" int cs_bitmap_plane(cs_db* db, int32_t var, int32_t state, const uint32_t** dev,
                               int64_t* words) {
  if (!db) return fail(CS_ERR_INVALID, "cs_bitmap_plane: NULL db");
  if (var < 0 || var >= db->n || state < 0 || state >= db->arity[var])
    return fail(CS_ERR_INVALID, "cs_bitmap_plane: bad (var, state) (%d, %d)", var, state);
  if (dev) *dev = db->plane_off[var] < 0 ? nullptr : db->planes + db->plane_off[var] + (int64_t)state * db->words;
  if (words) *words = db->words;
  return CS_OK;
}

// ------------------------------------------------------------------------------------------
// planning

static int plan_build(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                      uint32_t flags, cs_plan** out, bool transient = false, int32_t qbase = 0) {
  if (!db || !out) return fail(CS_ERR_INVALID, "cs_plan_create: NULL argument");
  if (nq < 0) return fail(CS_ERR_INVALID, "cs_plan_create: nq < 0");
  if (nq > 0 && (!var_off || !vars)) return fail(CS_ERR_INVALID, "cs_plan_create: NULL query arrays");
  const double trc = now_ms();
  cs_ctx* ctx = db->ctx;
  const int smem_words = ctx->hist_smem / 4;
  const int64_t m = db->m;
  cs_plan* p = new cs_plan();
  p->db = db;
  p->nq = nq;
  p->flags = flags;
  p->hq.resize(nq);
  p->cells.resize(nq);
  p->table_off.resize(nq);
  std::vector<int32_t> gvars;
  std::vector<uint32_t> gstride;
  int64_t total = 0;
  // tuning knobs, read once per plan (getenv per query cost milliseconds on 10K-query plans)
  const int64_t max_dense = (int64_t)env_int("CS_MAX_DENSE_LOG2", 30);
  const bool knob_pack = env_int("CS_PACK", 1) != 0;
  const bool knob_half = env_int("CS_HALF", 0) != 0;  // measured slower on cfg2: opt-in
  const bool knob_stages = env_int("CS_STAGES", 1) != 0;
  const bool knob_nibble = env_int("CS_NIBBLE", 1) != 0;
  const bool knob_slice = env_int("CS_SLICE", 1) != 0;
  const bool knob_radix = env_int("CS_RADIX", 1) != 0;
  // spill class (cs_spill.cuh): the first hist_smem cells counted in SMEM, the other rows' indices
  // moved once and counted per 192K-cell group (<= CS_SPILL_GROUPS groups)
  const bool knob_spill = env_int("CS_SPILL", 1) != 0;
  const int64_t spill_t1 = (int64_t)(ctx->hist_smem / 4) * 4;
  const int64_t spill_max =
      spill_t1 + (int64_t)SP_GROUP_CELLS * std::max(1, std::min(SP_MAXG, env_int("CS_SPILL_GROUPS", 2)));
  // narrow-counter SMEM class (8 / 16-bit counters with exact wrap repair) for tables of up to
  // 4x the 32-bit SMEM capacity
  const bool knob_narrow = env_int("CS_NARROW", 1) != 0;
  const int64_t knob_narrow_seg = (int64_t)env_int("CS_NARROW_SEG_ROWS", 1 << 24);
  // more than 4x the capacity: several passes (cell ranges) over each L2-resident row segment
  const int64_t knob_narrow_passes = std::max(1, env_int("CS_NARROW_MAX_PASSES", 1));
  const int64_t knob_narrow_pass_seg = (int64_t)env_int("CS_NARROW_PASS_SEG_ROWS", 1 << 22);
  // bitmap class (K7): -1 auto (cost model), 0 never, 1 whenever a query is eligible
  const int knob_bitmap = env_int("CS_BITMAP", -1);
  const int64_t knob_seg_max = (int64_t)env_int("CS_SEG_MAX_ROWS", 1 << 22);
  // tables above SMEM: the slice class (columns re-read once per pass, from L2) when it needs at
  // most this many passes over a row segment, else the partition class
  const int knob_slice_passes = env_int("CS_SLICE_MAX_PASSES", 0);
  auto slice_passes = [&](int64_t c, int rlast) -> int64_t {
    const int64_t sc = c / rlast;
    int rl = 0;
    while (rl < 5 && (sc << (rl + 1)) <= smem_words) ++rl;
    const int64_t spc = std::max<int64_t>(1, smem_words / (sc << rl));
    return (rlast + spc - 1) / spc;
  };
  // classification of every query (independent per query)
  const double trs = now_ms();
  auto classify = [&](int q) -> int {
    const int b = var_off[q], e = var_off[q + 1];
    const int k = e - b;
    if (k < 1) {
      return fail(CS_ERR_INVALID, "query %d has no target variable", qbase + q);
    }
    QDesc d;
    memset(&d, 0, sizeof d);
    int64_t c = 1;
    int nbyte = 0;
    for (int i = 0; i < k; ++i) {
      const int v = vars[b + i];
      if (v < 0 || v >= db->n) {
        return fail(CS_ERR_INVALID, "variable %d out of range for a database with n=%d", v, db->n);
      }
      for (int j = 0; j < i; ++j)
        if (vars[b + j] == v) {
          return fail(CS_ERR_INVALID, "query %d repeats variable %d", qbase + q, v);
        }
      if (i < CS_MAXK) {
        d.coff[i] = (uint32_t)((int64_t)v * (db->ld / 256));
        d.stride[i] = (uint32_t)c;
      }
      if (c > (int64_t)(((uint64_t)1 << 63) - 1) / db->arity[v]) {
        return fail(CS_ERR_UNSUPPORTED, "query %d: joint state space exceeds 2^63 cells", qbase + q);
      }
      c *= db->arity[v];
      if (c <= 256) nbyte = i + 1;
    }
    d.base = db->cols;
    if (k >= 4 && k <= CS_MAXK) {
      // digits in groups of three, each combined in byte lanes when its arity product fits a byte
      bool ok = true;
      for (int g0 = 0; g0 < k; g0 += 3) {
        int64_t gp = 1;
        for (int i = g0; i < std::min(k, g0 + 3); ++i) {
          d.gstride[i] = (uint32_t)gp;
          gp *= db->arity[vars[b + i]];
        }
        ok = ok && gp <= 256;
      }
      d.g3 = ok ? 1 : 0;
    }
    const bool sparse = c > ((int64_t)1 << max_dense);
    if (sparse && (flags & F_PARTIAL)) {
      return fail(CS_ERR_UNSUPPORTED, "query %d: sparse (hash) queries cannot be instance-sharded", qbase + q);
    }
    d.k = k;
    d.cells = sparse ? 0u : (uint32_t)c;
    d.nbyte = std::max(nbyte, 1);
    d.mode = c <= 65536 ? 1 : 2;
    d.r_target = db->arity[vars[b]];
    // bitmap class: every digit binary with a state-1 plane, <= 4 digits.  The planes are half
    // the bytes of the 2-bit column copy and a word of 32 records costs 2^k - 1 POPC, no SMEM
    // atomics: measured 2.1-2.8x the histogram classes for k = 1..4 (tools/bitmap_compare.py,
    // profiles/r02/bitmap_compare.txt), so every eligible query takes it
    bool bitmap_ok = knob_bitmap != 0 && !sparse && db->planes && k <= BQ_MAXK;
    for (int i = 0; i < k && bitmap_ok; ++i) {
      const int v = vars[b + i];
      bitmap_ok = db->arity[v] == 2 && db->plane_off[v] >= 0;
    }
    if (sparse) {
      d.kind = 3;  // hash class: descriptor built in the serial pass below
    } else if (bitmap_ok) {
      d.kind = 5;  // bitmap class: descriptor built in the serial pass below
    } else if (k > CS_MAXK) {
      d.kind = 2;  // generic class: variable list appended in the serial pass below
    } else if (c <= 6 && c * c * c * c * 32 <= smem_words && knob_pack) {
      d.kind = 0;  // 4 rows per atomic (hist_smem_packed<K, 4>)
      d.pack = 4;
      d.rlog = 5;
    } else if (c <= 41 && c * c * 32 <= smem_words && knob_pack) {
      d.kind = 0;  // 2 rows per atomic (hist_smem_packed<K, 2>)
      d.pack = 2;
      d.rlog = 5;
    } else if (c <= smem_words) {
      d.kind = 0;
      d.pack = 1;
      // replicas: as many as fit (<= 32; R = 32 makes every ATOMS wavefront conflict-free).
      // When C*R*4 <= 64 KB the byte offsets fit 16-bit SIMD lanes (mode 0, hist_smem_lane16).
      int rl = 0;
      while (rl < 5 && (c << (rl + 1)) <= smem_words) ++rl;
      d.rlog = rl;
      d.mode = (c << rl) <= 16384 ? 0 : (c <= 65536 ? 1 : 2);
      // 16-bit counters (two cells per word) double the replicas when 32-bit ones are short of
      // 32; counters cannot overflow while every replica serves <= 65535 rows of an item
      const int64_t seg_cap = std::min<int64_t>(round_up(m, 256), knob_seg_max);
      if (d.rlog < 5 && c <= 65536 && knob_half) {
        int rh = 0;
        while (rh < 5 && (((c + 1) / 2) << (rh + 1)) <= smem_words) ++rh;
        // the busiest replica: thread t takes vectors t, t + 1024, ... (RPV rows each, padding
        // included), so a replica of 1024 / R threads counts up to ceil(nvec / 1024) * (1024 / R)
        // * RPV rows -- for every column layout the query may read
        int64_t busiest = 0;
        for (int64_t rpv = 16; rpv <= 64; rpv *= 2) {
          const int64_t nvec = (seg_cap + rpv - 1) / rpv;
          busiest = std::max(busiest, (nvec + CS_HIST_THREADS - 1) / CS_HIST_THREADS * (CS_HIST_THREADS >> rh) * rpv);
        }
        if (rh > d.rlog && busiest <= 65535) {
          d.half = 1;
          d.rlog = rh;
        }
      }
    } else if (knob_narrow && db->nib && k >= 2 && k <= CS_MAXK &&
               c <= 4 * (int64_t)smem_words * knob_narrow_passes) {
      // narrow-counter SMEM class (cs_kernels.cuh hist_smem_narrow): 16-bit counters up to 2x,
      // 8-bit up to 4x the 32-bit capacity; reads the 4-bit columns
      d.kind = 0;
      d.pack = 1;
      d.rlog = 0;
      d.mode = 2;
      d.narrow = c <= 2 * (int64_t)smem_words ? 16 : 8;
      d.npass = (int32_t)((c + 4 * (int64_t)smem_words - 1) / (4 * (int64_t)smem_words));
      d.pcells = (uint32_t)round_up((c + d.npass - 1) / d.npass, 4);
      d.nib = 1;
      d.base = db->nib;
      uint32_t r8[8];
      for (int v = 0; v < 8; ++v) r8[v] = v < k ? (uint32_t)db->arity[vars[b + v]] : 1u;
      for (int p2 = 0; p2 < 4; ++p2) d.rpair[p2] = r8[2 * p2];
      d.R0 = r8[0] * r8[1];
      d.R2 = r8[4] * r8[5];
      d.P01 = r8[0] * r8[1] * r8[2] * r8[3];
      for (int i = 0; i < k; ++i) d.coff[i] = (uint32_t)((int64_t)vars[b + i] * (db->ldn / 256));
    } else if (knob_spill && db->nib && k >= 2 && k <= CS_MAXK && c > spill_t1 && c <= spill_max) {
      d.kind = 6;
      d.mode = 2;
      d.nib = 1;
      d.base = db->nib;
      for (int i = 0; i < k; ++i) d.coff[i] = (uint32_t)((int64_t)vars[b + i] * (db->ldn / 256));
    } else if (knob_radix && db->nib && k >= 2 && c <= ((int64_t)1 << 24) &&
               !(knob_slice && c / db->arity[vars[e - 1]] <= smem_words &&
                 slice_passes(c, db->arity[vars[e - 1]]) <= knob_slice_passes)) {
      // partition class (cs_radix.cuh): one counting-sort pass by the high bits of the joint
      // index, then SMEM histograms per 32K-cell group; reads the 4-bit columns
      d.kind = 4;
      d.mode = 2;
      d.nib = 1;
      d.base = db->nib;
      for (int i = 0; i < k; ++i) d.coff[i] = (uint32_t)((int64_t)vars[b + i] * (db->ldn / 256));
    } else if (k >= 2 && c / db->arity[vars[e - 1]] <= smem_words && knob_slice) {
      // slice class: one CTA per value of the most significant digit, C / r_last cells each
      d.kind = 0;
      d.scells = (uint32_t)(c / db->arity[vars[e - 1]]);
      int rl = 0;
      while (rl < 5 && ((int64_t)d.scells << (rl + 1)) <= smem_words) ++rl;
      d.rlog = rl;
      d.mode = 1;
    } else {
      d.kind = 1;
      d.mode = c <= 65536 ? 1 : 2;
    }
    if (d.kind == 0) {
      // cp.async ring for the row stream: up to 4 stages in the SMEM left after the table
      // (K <= 4 only: higher K keeps its SMEM for conflict-free replicas instead)
      const int64_t smem_bytes = (int64_t)ctx->hist_smem;
      const int64_t per_stage = (int64_t)k * 16 * ctx->hist_threads;
      auto table_bytes = [&](const QDesc& x) {
        int64_t ct = x.cells;
        for (int i = 1; i < x.pack; ++i) ct *= x.cells;
        if (x.half) ct = (ct + 1) / 2;
        return round_up((ct << x.rlog) * 4, 128);
      };
      if (k <= 4 && knob_stages && !d.scells && !d.narrow) {
        // shrink packing first if it is what keeps the ring from fitting 3 stages
        while (d.pack > 1 && table_bytes(d) + 3 * per_stage > smem_bytes) {
          d.pack = d.pack == 4 ? 2 : 1;
          if (d.pack == 1) {
            int rl = 0;
            while (rl < 5 && (c << (rl + 1)) <= smem_words) ++rl;
            d.rlog = rl;
            d.mode = (c << rl) <= 16384 ? 0 : (c <= 65536 ? 1 : 2);
          }
        }
        const int64_t left = smem_bytes - table_bytes(d);
        const int st = (int)std::min<int64_t>(4, left / std::max<int64_t>(per_stage, 1));
        if (st >= 3 && (d.pack > 1 || d.mode <= 1)) {
          d.stages = st;
          d.stage_off = (uint32_t)table_bytes(d);
        }
      }
    }
    if (d.kind == 0 && db->crumb && (d.pack > 1 || d.mode <= 1) && knob_nibble) {
      d.nib = 2;  // 2-bit columns: 64 rows per 16 B
      d.base = db->crumb;
      for (int i = 0; i < k; ++i) d.coff[i] = (uint32_t)((int64_t)vars[b + i] * (db->ldc / 256));
    } else if (d.kind == 0 && db->nib && (d.pack > 1 || d.mode <= 1) && knob_nibble) {
      d.nib = 1;
      d.base = db->nib;
      for (int i = 0; i < k; ++i) d.coff[i] = (uint32_t)((int64_t)vars[b + i] * (db->ldn / 256));
    }
    p->hq[q] = d;
    p->cells[q] = c;
    return CS_OK;
  };
  {
    // host threads for the classification (CS_PLAN_THREADS, default 1): the parallel part
    // scales (74.5K queries: 2.95 -> 0.75 ms on 8 threads) but the passes after it then read
    // descriptors written on other cores and lose more than that (measured, tools/plan_probe.py)
    const int nt = std::max(1, std::min(nq, env_int("CS_PLAN_THREADS", 1)));
    std::vector<int> rc(nt, CS_OK), first_bad(nt, -1);
    std::vector<std::string> msg(nt);
    auto run = [&](int t) {
      const int q0 = (int)((int64_t)nq * t / nt), q1 = (int)((int64_t)nq * (t + 1) / nt);
      for (int q = q0; q < q1; ++q) {
        const int r = classify(q);
        if (r != CS_OK) {
          rc[t] = r;
          first_bad[t] = q;
          msg[t] = g_err;  // thread-local message of this worker
          return;
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(run, t);
    run(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < nt; ++t)
      if (rc[t] != CS_OK) {  // the lowest query's error, as a serial pass would report it
        delete p;
        g_err = msg[t];
        return rc[t];
      }
  }
  const double trp = now_ms();
  // serial pass: table offsets, hash-class descriptors, generic-class variable lists
  int64_t nkind[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // queries per class: later passes skip empty ones
  for (int q = 0; q < nq; ++q) {
    QDesc& d = p->hq[q];
    nkind[d.kind & 7]++;
    const int b = var_off[q], k = var_off[q + 1] - b;
    d.table_off = total;
    if (d.kind == 3) {
      cs_plan::SparseQ sq;
      sq.q = q;
      sq.k = k;
      sq.rt = db->arity[vars[b]];
      sq.C = (uint64_t)p->cells[q];
      uint64_t st = 1;
      for (int i = 0; i < k; ++i) {
        sq.vars.push_back(vars[b + i]);
        sq.stride.push_back(st);
        st *= (uint64_t)db->arity[vars[b + i]];
      }
      uint64_t H = 1024;
      while (H < 2 * std::min<uint64_t>((uint64_t)m, sq.C)) H <<= 1;
      sq.H = H;
      p->sparse.push_back(sq);
      p->cells[q] = 0;  // no dense table
    } else if (d.kind == 5) {
      BDesc bq;
      memset(&bq, 0, sizeof bq);
      for (int i = 0; i < k; ++i) bq.plane[i] = db->planes + db->plane_off[vars[b + i]] + db->words;
      bq.table_off = total;
      bq.k = k;
      d.var_base = (int32_t)p->bdesc.size();  // BDesc index
      p->bdesc.push_back(bq);
    } else if (d.kind == 2) {
      d.var_base = (int32_t)gvars.size();
      int64_t s2 = 1;
      for (int i = 0; i < k; ++i) {
        gvars.push_back(vars[b + i]);
        gstride.push_back((uint32_t)s2);
        s2 *= db->arity[vars[b + i]];
      }
    }
    p->table_off[q] = total;
    total += p->cells[q];
  }
  p->total_cells = total;
  const bool trace = env_int("CS_TRACE", 0) != 0;
  const double tr0 = trace ? now_ms() : 0.0;
  // row segmentation: >= 4 work items per resident CTA, segments of 64K..4M rows
  const int64_t seg_min = 1 << 16, seg_max = knob_seg_max;
  const int64_t target_items = 4LL * ctx->hist_ctas;
  std::vector<WItem> items;
  std::vector<double> cost;
  items.reserve((size_t)nq * 2);
  cost.reserve((size_t)nq * 2);
  for (int q = 0; q < nq; ++q) {
    QDesc& d = p->hq[q];
    if (d.kind == 3) {
      d.nseg = 1;
      continue;
    }
    if (d.kind == 4 || d.kind == 5 || d.kind == 6) {
      p->score_list.push_back(q);
      p->needs_global = p->needs_zero = true;
      d.nseg = 1;
      continue;
    }
    if (d.kind == 2) {
      p->generic_list.push_back(q);
      p->score_list.push_back(q);
      p->needs_global = p->needs_zero = true;
      d.nseg = 1;
      continue;
    }
    const int64_t smax = d.narrow ? (d.npass > 1 ? knob_narrow_pass_seg : std::max(seg_max, knob_narrow_seg)) : seg_max;
    int64_t nseg = std::max<int64_t>(1, (m + smax - 1) / smax);
    const int64_t want = (target_items + nq - 1) / std::max(nq, 1);
    nseg = std::max(nseg, std::min<int64_t>(want, (m + seg_min - 1) / seg_min));
    int64_t L = round_up((m + nseg - 1) / nseg, 256);
    nseg = (m + L - 1) / L;
    d.nseg = (int32_t)nseg;
    if (d.kind == 1) {
      p->score_list.push_back(q);
      p->needs_global = p->needs_zero = true;
    } else if (d.narrow) {
      p->needs_global = p->needs_zero = true;  // always merged with global atomics (wrap repairs)
    } else if (d.scells) {
      p->score_list.push_back(q);
      p->needs_global = true;
      if (nseg > 1) p->needs_zero = true;
    } else if (nseg > 1) {
      p->needs_global = p->needs_zero = true;
    }
    // slice class: a CTA owns as many consecutive last-digit values as its SMEM holds
    const int rlast = d.scells ? (int)(d.cells / d.scells) : (d.narrow ? d.npass : 1);
    const int spc = d.scells ? std::max(1, (int)(smem_words / ((int64_t)d.scells << d.rlog))) : 1;
    for (int64_t s = 0; s < nseg; ++s) {
      for (int sl = 0; sl < rlast; sl += spc) {
        WItem w;
        memset(&w, 0, sizeof w);
        w.q = q;
        w.seg = (int32_t)s;
        w.r0 = s * L;
        w.r1 = std::min(m, (s + 1) * L);
        w.slice = sl;
        w.nsl = std::min(spc, rlast - sl);
        items.push_back(w);
        const double rows = (double)(w.r1 - w.r0);
        cost.push_back(rows * (1.0 + d.k) + (d.kind == 0 ? (double)(d.cells << d.rlog) * 2.0 : 0.0));
      }
    }
  }
  const double tr1 = trace ? now_ms() : 0.0;
  // longest-processing-time-first order for the persistent CTAs
  std::vector<int> order(items.size());
  std::iota(order.begin(), order.end(), 0);
  // Segment-major (CS_SEG_ORDER=1, default): all items of row segment 0 first, then 1, ...;
  // LPT within a segment.  Concurrently running CTAs then share one row window of the
  // columns, which stays L2-resident (the L2 is split per die, so a 100 MB database does not).
  const bool seg_major = env_int("CS_SEG_ORDER", 1) != 0;
  {
    // LPT needs only an approximate cost order: a stable counting sort on (segment, 1/16-octave
    // cost bucket, descending) is O(items) -- a comparison sort of 10K items cost ~0.7 ms of a
    // ~4 ms one-shot call
    constexpr int NB = 1024;
    int32_t nsegs = 1;
    for (const WItem& w : items) nsegs = std::max(nsegs, w.seg + 1);
    if (!seg_major) nsegs = 1;
    std::vector<int32_t> bucket(items.size());
    std::vector<int32_t> count((size_t)nsegs * NB + 1, 0);
    for (size_t i = 0; i < items.size(); ++i) {
      const int cb = std::max(0, std::min(NB - 1, (int)(std::log2(std::max(cost[i], 1.0)) * 16.0)));
      bucket[i] = (seg_major ? items[i].seg : 0) * NB + (NB - 1 - cb);
      count[bucket[i] + 1]++;
    }
    for (size_t b = 1; b < count.size(); ++b) count[b] += count[b - 1];
    for (size_t i = 0; i < items.size(); ++i) order[count[bucket[i]]++] = (int)i;
  }
  // SMEM-class items grouped by K1 variant (k, path, layout), groups by descending total cost,
  // LPT order inside a group; then the global-class items.
  std::vector<std::vector<int>> groups(CS_MAXK * 24);  // key = (k-1)*24 + path*3 + layout
  std::vector<double> gcost(CS_MAXK * 24, 0.0);
  {
    std::vector<int32_t> qkey(nq);
    std::vector<int32_t> gsize(CS_MAXK * 24, 0);
    for (int q = 0; q < nq; ++q) {
      const QDesc& d = p->hq[q];
      qkey[q] = d.kind == 0 ? (d.k - 1) * 24 + hist_path(d) * 3 + d.nib : -1;
    }
    for (const WItem& w : items)
      if (qkey[w.q] >= 0) gsize[qkey[w.q]]++;
    for (int k = 0; k < CS_MAXK * 24; ++k) groups[k].reserve(gsize[k]);
    for (size_t i = 0; i < order.size(); ++i) {
      const int key = qkey[items[order[i]].q];
      if (key < 0) continue;
      groups[key].push_back(order[i]);
      gcost[key] += cost[order[i]];
    }
  }
  std::vector<int> keys;
  for (int k = 0; k < (int)groups.size(); ++k)
    if (!groups[k].empty()) keys.push_back(k);
  std::stable_sort(keys.begin(), keys.end(), [&](int a, int b) { return gcost[a] > gcost[b]; });
  std::vector<WItem> sorted;
  sorted.reserve(items.size());
  for (int key : keys) {
    auto& g = groups[key];
    if ((key % 24) / 3 == P_SLICE) {
      // slices of one segment back to back (they share its columns through L2), queries LPT
      std::map<int, double> qc;
      for (int i : g) qc[items[i].q] += cost[i];
      std::stable_sort(g.begin(), g.end(), [&](int a, int b) {
        const WItem &x = items[a], &y = items[b];
        if (x.q != y.q) return qc[x.q] != qc[y.q] ? qc[x.q] > qc[y.q] : x.q < y.q;
        if (x.seg != y.seg) return x.seg < y.seg;
        return x.slice < y.slice;
      });
    }
    p->groups.push_back({key, (int)sorted.size(), (int)g.size()});
    for (int i : g) sorted.push_back(items[i]);
  }
  p->nitems = (int)sorted.size();
  // global class: query-major (all segments of a query back to back, queries LPT by total
  // cost) so concurrently running CTAs share one L2-resident table -- RED.ADD throughput
  // collapses when they spray many >SMEM tables at once
  if (nkind[1]) {
    std::map<int, double> qcost;
    std::vector<int> gq;
    for (size_t i = 0; i < items.size(); ++i)
      if (p->hq[items[i].q].kind == 1) {
        if (!qcost.count(items[i].q)) gq.push_back(items[i].q);
        qcost[items[i].q] += cost[i];
      }
    std::stable_sort(gq.begin(), gq.end(), [&](int a, int b) { return qcost[a] > qcost[b]; });
    std::map<int, std::vector<int>> byq;
    for (size_t i = 0; i < items.size(); ++i)
      if (p->hq[items[i].q].kind == 1) byq[items[i].q].push_back((int)i);
    for (int qq : gq)
      for (int i : byq[qq]) sorted.push_back(items[i]);
  }
  p->ngitems = (int)sorted.size() - p->nitems;
  // partition class (kind 4): descriptors in wave order (waves grouped by digit count), count
  // items per (query, 32K-cell group, chunk range)
  std::vector<RItem> ritems;
  if (nkind[4]) {
    std::vector<int> rq;
    for (int q = 0; q < nq; ++q)
      if (p->hq[q].kind == 4) rq.push_back(q);
    if (!rq.empty()) {
      std::stable_sort(rq.begin(), rq.end(), [&](int a, int b) { return p->hq[a].k < p->hq[b].k; });
      const int64_t nchunks = (m + RX_CH - 1) / RX_CH;
      p->rx_nchunks = (int)nchunks;
      const size_t buf_b = (size_t)round_up(nchunks * RX_CH * 2, 256);
      const size_t choff_b = (size_t)round_up(nchunks * (RX_MAX_NB + 1) * 4, 256);
      const size_t slot = std::max<size_t>(buf_b + choff_b, 256);
      size_t budget = (size_t)env_int("CS_RADIX_MB", 4096) << 20;
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min(budget, fr / 2);
      else cudaGetLastError();
      const int W = (int)std::max<size_t>(1, std::min<size_t>(budget / slot, rq.size()));
      p->rx_scratch = slot * (size_t)W;
      const int64_t cpi = std::max(1, env_int("CS_RADIX_CPI", 2048 * (8192 / RX_CH)));  // 16M rows per count item
      const int64_t G = std::max<int64_t>(1, (nchunks + cpi - 1) / cpi);
      const int64_t cper = std::max<int64_t>(1, (nchunks + G - 1) / G);
      for (size_t w0 = 0; w0 < rq.size(); w0 += (size_t)W) {
        cs_plan::RadixWave wave;
        wave.item0 = (int)ritems.size();
        for (size_t i = w0; i < std::min(rq.size(), w0 + (size_t)W); ++i) {
          const int q = rq[i];
          const QDesc& d = p->hq[q];
          RDesc r;
          memset(&r, 0, sizeof r);
          const size_t s = i - w0;
          r.buf_off = (int64_t)(s * slot);
          r.choff_off = (int64_t)(s * slot + buf_b);
          r.q = q;
          r.base = d.base;
          const int64_t C = d.cells;
          int bb = 10;  // >= 32 buckets where possible (SMEM bucket counters contend less)
          while (bb < RX_GROUP_BITS && (C >> (bb + 1)) >= 32) ++bb;
          r.bb = bb;
          r.nb = (int)((C + (1LL << bb) - 1) >> bb);
          {
            uint32_t r8[8];
            for (int v = 0; v < 8; ++v) r8[v] = v < d.k ? (uint32_t)db->arity[vars[var_off[q] + v]] : 1u;
            for (int p2 = 0; p2 < 4; ++p2) r.rpair[p2] = r8[2 * p2];
            r.R0 = r8[0] * r8[1];
            r.R2 = r8[4] * r8[5];
            r.P01 = r8[0] * r8[1] * r8[2] * r8[3];
            for (int v = 0; v < d.k; ++v) r.coff[v] = d.coff[v];
          }
          // count sub-group width: ~2 16-B vectors per lane of a chunk's run in one group
          const double vec = (double)RX_CH * (double)std::min<int64_t>(C, 1LL << RX_GROUP_BITS) / (double)C / 8.0;
          int wl = 2;
          while (wl < 5 && (double)(4 << wl) <= vec) ++wl;
          r.wlog = wl;
          const int ri = (int)p->rdesc.size();
          p->rdesc.push_back(r);
          if (wave.parts.empty() || wave.parts.back().k != d.k) wave.parts.push_back({d.k, ri, 0});
          wave.parts.back().count++;
          const int ngrp = (int)((C + (1LL << RX_GROUP_BITS) - 1) >> RX_GROUP_BITS);
          for (int g = 0; g < ngrp; ++g)
            for (int64_t c0 = 0; c0 < nchunks; c0 += cper)
              ritems.push_back(RItem{ri, g, (int32_t)c0, (int32_t)std::min<int64_t>(nchunks, c0 + cper)});
        }
        wave.nitems = (int)ritems.size() - wave.item0;
        p->waves.push_back(wave);
      }
    }
  }
  // spill class (kind 6): waves of queries whose spill regions share one context scratch; per
  // wave one k_spill_hist launch per digit count over (query, row segment) items, then
  // k_spill_count over (query, range group, row segment) items
  std::vector<SItem> sitems;
  std::vector<CItem> citems;
  if (nkind[6]) {
    std::vector<int> sq;
    for (int q = 0; q < nq; ++q)
      if (p->hq[q].kind == 6) sq.push_back(q);
    std::stable_sort(sq.begin(), sq.end(), [&](int a, int b) { return p->hq[a].k < p->hq[b].k; });
    const double slack = std::max(0, env_int("CS_SPILL_SLACK", 125)) / 100.0;
    const int64_t seg_rows = std::max<int64_t>(1 << 16, env_int("CS_SPILL_SEG_ROWS", 1 << 23));
    const int64_t n0 = std::max<int64_t>(1, (m + seg_rows - 1) / seg_rows);
    size_t budget = (size_t)env_int("CS_SPILL_MB", 4096) << 20;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min(budget, fr / 2);
    else cudaGetLastError();
    // scratch of one query split into nseg segments: one stream of cap entries per (segment, warp)
    struct Lay {
      int64_t L, nseg, cap, regions;
      size_t reg_b, cnt_b;
    };
    auto layout = [&](int64_t C, int64_t nseg) {
      Lay y;
      y.L = round_up((m + nseg - 1) / nseg, 256);
      y.nseg = (m + y.L - 1) / y.L;
      const int64_t nvec = (y.L + 31) / 32;
      const int64_t rows_warp = (nvec + SP_THREADS - 1) / SP_THREADS * 1024;  // 32 lanes x 32 rows per iteration
      // the uniform expectation times the slack, plus the 1024 entries one vector may append
      const double expect = (double)rows_warp * (double)(C - spill_t1) / (double)C;
      y.cap = slack > 0 ? round_up(std::min<int64_t>(rows_warp, (int64_t)std::ceil(expect * slack)) + 1024, 4) : 0;
      y.regions = y.nseg * SP_WARPS;
      y.reg_b = (size_t)round_up(y.regions * y.cap * 4, 256);
      y.cnt_b = (size_t)round_up(y.regions * 4, 256);
      return y;
    };
    size_t i0 = 0;
    while (i0 < sq.size()) {
      // greedy wave under the budget, sized with the finest segmentation it may get
      size_t i1 = i0, bytes = 0;
      while (i1 < sq.size()) {
        const Lay y = layout(p->cells[sq[i1]], 2 * n0);
        if (i1 > i0 && bytes + y.reg_b + y.cnt_b > budget) break;
        bytes += y.reg_b + y.cnt_b;
        ++i1;
      }
      // segments per query: n0 .. 2 n0, whichever fills the persistent grid's rounds best
      const int64_t W = (int64_t)(i1 - i0);
      int64_t nseg = n0;
      double best = -1.0;
      for (int64_t c = n0; c <= 2 * n0; ++c) {
        const int64_t it = W * c, rounds = (it + ctx->num_sms - 1) / ctx->num_sms;
        const double eff = (double)it / (double)(rounds * ctx->num_sms);
        if (eff > best + 1e-9) {
          best = eff;
          nseg = c;
        }
      }
      cs_plan::SpillWave wave;
      wave.item0 = (int)citems.size();
      size_t off = 0;
      for (size_t i = i0; i < i1; ++i) {
        const int q = sq[i];
        const QDesc& d = p->hq[q];
        const Lay y = layout(p->cells[q], nseg);
        SDesc r;
        memset(&r, 0, sizeof r);
        r.base = d.base;
        r.table_off = d.table_off;
        r.reg_off = (int64_t)off;
        r.cnt_off = (int64_t)(off + y.reg_b);
        off += y.reg_b + y.cnt_b;
        uint32_t r8[8];
        for (int v = 0; v < 8; ++v) r8[v] = v < d.k ? (uint32_t)db->arity[vars[var_off[q] + v]] : 1u;
        for (int p2 = 0; p2 < 4; ++p2) r.rpair[p2] = r8[2 * p2];
        r.R0 = r8[0] * r8[1];
        r.R2 = r8[4] * r8[5];
        r.P01 = r8[0] * r8[1] * r8[2] * r8[3];
        for (int v = 0; v < d.k; ++v) r.coff[v] = d.coff[v];
        r.cells = d.cells;
        r.t1 = (uint32_t)spill_t1;
        r.cap = (uint32_t)y.cap;
        r.ng = (int32_t)((p->cells[q] - spill_t1 + SP_GROUP_CELLS - 1) / SP_GROUP_CELLS);
        r.nseg = (int32_t)y.nseg;
        r.q = q;
        const int si = (int)p->sdesc.size();
        p->sdesc.push_back(r);
        if (wave.parts.empty() || wave.parts.back().k != d.k) wave.parts.push_back({d.k, (int)sitems.size(), 0});
        for (int64_t g = 0; g < y.nseg; ++g) {
          sitems.push_back(SItem{si, (int32_t)g, g * y.L, std::min(m, (g + 1) * y.L)});
          wave.parts.back().count++;
        }
        for (int grp = 0; grp < r.ng; ++grp)
          for (int64_t g = 0; g < y.nseg; ++g) citems.push_back(CItem{si, grp, (int32_t)g, 0});
      }
      p->sp_scratch = std::max(p->sp_scratch, off);
      p->sp_heads += (int)wave.parts.size() + 1;
      wave.nitems = (int)citems.size() - wave.item0;
      p->swaves.push_back(wave);
      i0 = i1;
    }
  }
  // bitmap class (kind 5): (query, tile range) items grouped by digit count
  std::vector<BItem> bitems;
  if (!p->bdesc.empty()) {
    const int64_t tiles = (db->words + BQ_TILE - 1) / BQ_TILE;
    for (int k = 1; k <= BQ_MAXK; ++k) {
      int64_t nqk = 0;
      for (const BDesc& x : p->bdesc) nqk += x.k == k;
      if (!nqk) continue;
      // ~4 items per CTA of the launch, <= 16 tiles (512K records) each
      const int64_t per = std::max<int64_t>(1, std::min<int64_t>(16, nqk * tiles / (4LL * ctx->num_sms)));
      cs_plan::BLaunch L{k, (int)bitems.size(), 0};
      for (size_t i = 0; i < p->bdesc.size(); ++i) {
        if (p->bdesc[i].k != k) continue;
        for (int64_t t0 = 0; t0 < tiles; t0 += per)
          bitems.push_back(BItem{(int32_t)i, (int32_t)t0, (int32_t)std::min(tiles, t0 + per)});
      }
      L.nitems = (int)bitems.size() - L.item0;
      p->blaunch.push_back(L);
    }
  }
  const double tr2 = trace ? now_ms() : 0.0;
  if (trace)
    fprintf(stderr,
            "plan_build: classes smem=%lld global=%lld generic=%lld hash=%lld partition=%lld bitmap=%lld spill=%lld\n",
            (long long)nkind[0], (long long)nkind[1], (long long)nkind[2], (long long)nkind[3], (long long)nkind[4],
            (long long)nkind[5], (long long)nkind[6]);
  if (trace)
    fprintf(stderr, "plan_build: setup %.3f ms, classify %.3f ms (parallel part %.3f), items %.3f ms, order %.3f ms\n",
            trs - trc, tr0 - trs, trp - trs, tr1 - tr0,
            tr2 - tr1);
  // upload descriptors (one blob through pinned staging)
  CS_CUDA(cudaSetDevice(ctx->device));
  const size_t bq = sizeof(QDesc) * std::max(nq, 1);
  const size_t bi = sizeof(WItem) * std::max<size_t>(sorted.size(), 1);
  const size_t bs = sizeof(int32_t) * std::max<size_t>(p->score_list.size(), 1);
  const size_t bg = sizeof(int32_t) * std::max<size_t>(p->generic_list.size(), 1);
  const size_t bv = sizeof(int32_t) * std::max<size_t>(gvars.size(), 1);
  const size_t bst = sizeof(uint32_t) * std::max<size_t>(gstride.size(), 1);
  size_t off = 0;
  auto place = [&](size_t bytes) {
    size_t o = off;
    off = round_up(off + bytes, 256);
    return o;
  };
  const size_t oq = place(bq), oi = place(bi), os = place(bs), og = place(bg), ov = place(bv),
               ost = place(bst), oh = place(1024), od = place(sizeof(uint32_t) * std::max(nq, 1)),
               ord = place(sizeof(RDesc) * std::max<size_t>(p->rdesc.size(), 1)),
               ori = place(sizeof(RItem) * std::max<size_t>(ritems.size(), 1)),
               orh = place(sizeof(int) * std::max<size_t>(p->waves.size(), 1)),
               obd = place(sizeof(BDesc) * std::max<size_t>(p->bdesc.size(), 1)),
               obi = place(sizeof(BItem) * std::max<size_t>(bitems.size(), 1)),
               obh = place(sizeof(int) * BQ_MAXK),
               osd = place(sizeof(SDesc) * std::max<size_t>(p->sdesc.size(), 1)),
               osi = place(sizeof(SItem) * std::max<size_t>(sitems.size(), 1)),
               oci = place(sizeof(CItem) * std::max<size_t>(citems.size(), 1)),
               osh = place(sizeof(int) * std::max(p->sp_heads, 1));
  char* dblob = nullptr;
  p->transient = transient;
  if (transient) {
    // grow-only context scratch: no cudaMalloc/cudaFree (and their device syncs) per call;
    // stream order keeps a later plan's upload behind this plan's kernels
    void* b = nullptr;
    int rc = ctx->scratch_get(18, off, &b);
    if (rc != CS_OK) {
      delete p;
      return rc;
    }
    dblob = (char*)b;
  } else {
    cudaError_t e = cudaMalloc(&dblob, off);
    if (e != cudaSuccess) {
      cudaGetLastError();
      delete p;
      return fail(CS_ERR_OOM, "cs_plan_create: cannot allocate %zu bytes", off);
    }
  }
  void* stage = nullptr;
  CS_TRY(ctx->pinned_get(off, &stage));
  if (ctx->pipe) {
    // only this bank's previous upload can still be reading its staging buffer
    if (ctx->stage_ev_valid[ctx->bank]) CS_CUDA(cudaEventSynchronize(ctx->stage_ev[ctx->bank]));
  } else {
    CS_CUDA(cudaStreamSynchronize(ctx->stream));  // staging buffer may be in flight
  }
  char* hs = (char*)stage;
  memcpy(hs + oq, p->hq.data(), sizeof(QDesc) * nq);
  memcpy(hs + oi, sorted.data(), sizeof(WItem) * sorted.size());
  memcpy(hs + os, p->score_list.data(), sizeof(int32_t) * p->score_list.size());
  memcpy(hs + og, p->generic_list.data(), sizeof(int32_t) * p->generic_list.size());
  memcpy(hs + ov, gvars.data(), sizeof(int32_t) * gvars.size());
  memcpy(hs + ost, gstride.data(), sizeof(uint32_t) * gstride.size());
  memcpy(hs + ord, p->rdesc.data(), sizeof(RDesc) * p->rdesc.size());
  memcpy(hs + ori, ritems.data(), sizeof(RItem) * ritems.size());
  memcpy(hs + obd, p->bdesc.data(), sizeof(BDesc) * p->bdesc.size());
  memcpy(hs + obi, bitems.data(), sizeof(BItem) * bitems.size());
  memcpy(hs + osd, p->sdesc.data(), sizeof(SDesc) * p->sdesc.size());
  memcpy(hs + osi, sitems.data(), sizeof(SItem) * sitems.size());
  memcpy(hs + oci, citems.data(), sizeof(CItem) * citems.size());
  CS_CUDA(cudaMemcpyAsync(dblob, hs, oh, cudaMemcpyHostToDevice, ctx->stream));
  if (!p->rdesc.empty())
    CS_CUDA(cudaMemcpyAsync(dblob + ord, hs + ord, orh - ord, cudaMemcpyHostToDevice, ctx->stream));
  if (!p->bdesc.empty())
    CS_CUDA(cudaMemcpyAsync(dblob + obd, hs + obd, obh - obd, cudaMemcpyHostToDevice, ctx->stream));
  if (!p->sdesc.empty())
    CS_CUDA(cudaMemcpyAsync(dblob + osd, hs + osd, osh - osd, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->pipe) {
    auto& ev = ctx->stage_ev[ctx->bank];
    if (!ev) CS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CS_CUDA(cudaEventRecord(ev, ctx->stream));
    ctx->stage_ev_valid[ctx->bank] = true;
  }
  p->d_q = (QDesc*)(dblob + oq);
  p->d_items = (WItem*)(dblob + oi);
  p->d_score_list = (int32_t*)(dblob + os);
  p->d_generic_list = (int32_t*)(dblob + og);
  p->d_gvars = (int32_t*)(dblob + ov);
  p->d_gstride = (uint32_t*)(dblob + ost);
  p->d_head = (int*)(dblob + oh);
  p->d_done = (uint32_t*)(dblob + od);
  p->d_rdesc = (RDesc*)(dblob + ord);
  p->d_ritems = (RItem*)(dblob + ori);
  p->d_rhead = (int*)(dblob + orh);
  p->d_bdesc = (BDesc*)(dblob + obd);
  p->d_bitems = (BItem*)(dblob + obi);
  p->d_bhead = (int*)(dblob + obh);
  p->d_sdesc = (SDesc*)(dblob + osd);
  p->d_sitems = (SItem*)(dblob + osi);
  p->d_citems = (CItem*)(dblob + oci);
  p->d_shead = (int*)(dblob + osh);
  if (trace) fprintf(stderr, "plan_build: upload %.3f ms\n", now_ms() - tr2);
  *out = p;
  return CS_OK;
}

extern "C" int cs_plan_create(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                              uint32_t flags, cs_plan** out) {
  CtxLock lk_(db ? db->ctx : nullptr);
  int rc = plan_build(db, nq, var_off, vars, flags, out);
  if (rc == CS_OK) {
    // the staging copy must land before the caller may reuse the pinned buffer
    CS_CUDA(cudaStreamSynchronize(db->ctx->stream));
  }
  return rc;
}

extern "C" int cs_plan_info(cs_plan* p, int64_t* cells, int64_t* table_off, int64_t* total_cells) {
  if (!p) return fail(CS_ERR_INVALID, "cs_plan_info: NULL plan");
  if (cells) memcpy(cells, p->cells.data(), sizeof(int64_t) * p->nq);
  if (table_off) memcpy(table_off, p->table_off.data(), sizeof(int64_t) * p->nq);
  if (total_cells) *total_cells = p->total_cells;
  return CS_OK;
}

extern "C" int cs_plan_destroy(cs_plan* p) {
  CtxLock lk_(p ? p->db->ctx : nullptr);
  if (!p) return CS_OK;
  cudaSetDevice(p->db->ctx->device);
  for (auto& sq : p->sparse)
    if (sq.blob) {
      cudaStreamSynchronize(p->db->ctx->stream);
      cudaFree(sq.blob);
    }
  for (auto& L : p->sl)
    if (L.blob) {
      cudaStreamSynchronize(p->db->ctx->stream);
      cudaFree(L.blob);
    }
  if (!p->transient) {
    cudaStreamSynchronize(p->db->ctx->stream);
    if (p->d_q) cudaFree((void*)p->d_q);  // blob base
    if (p->d_tables) cudaFree(p->d_tables);
  }
  delete p;
  return CS_OK;
}

// output routing: device pointers are written in place; host pointers go through scratch
struct OutBuf {
  void* user = nullptr;
  void* dev = nullptr;
  size_t bytes = 0;
  bool host = false;    // device scratch, copied to the user's host buffer at the end
  bool mapped = false;  // the user's page-locked host buffer, written in place by the kernels
};

static int route(cs_ctx* ctx, int slot, void* user, size_t bytes, OutBuf& ob) {
  ob.user = user;
  ob.bytes = bytes;
  if (!user) return CS_OK;
  if (is_device_ptr(user)) {
    ob.dev = user;
    return CS_OK;
  }
  ob.host = true;
  return ctx->scratch_get(slot, bytes, &ob.dev);
}

static int plan_tables(cs_plan* p, uint32_t* user_tables, OutBuf& tb, uint32_t** dtab) {
  const size_t bytes = sizeof(uint32_t) * std::max<int64_t>(p->total_cells, 1);
  *dtab = nullptr;
  tb = OutBuf();
  const bool user_dev = user_tables && is_device_ptr(user_tables);
  // page-locked host tables that the kernels only ever store to (no zeroing, no global
  // accumulation): the K1 epilogues write them directly over the bus, overlapped with the
  // remaining histogram work, instead of a scratch table plus a D2H copy after the last kernel
  void* mapped = nullptr;
  if (user_tables && !user_dev && !p->needs_zero && !p->needs_global && env_int("CS_ZEROCOPY", 1)) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, user_tables) == cudaSuccess && a.type == cudaMemoryTypeHost)
      mapped = a.devicePointer;
    cudaGetLastError();
  }
  if (user_dev) {
    tb.user = tb.dev = user_tables;
    tb.bytes = bytes;
    *dtab = user_tables;
  } else if (mapped) {
    tb.user = user_tables;
    tb.dev = mapped;
    tb.bytes = bytes;
    tb.mapped = true;
    *dtab = (uint32_t*)mapped;
  } else if (user_tables || (p->flags & F_TABLES) || p->needs_global) {
    if (p->transient) {
      void* b = nullptr;
      CS_TRY(p->db->ctx->scratch_get(17, bytes, &b));
      p->d_tables = (uint32_t*)b;
      p->d_tables_cells = std::max<int64_t>(p->total_cells, 1);
    } else if (p->d_tables_cells < (size_t)std::max<int64_t>(p->total_cells, 1)) {
      if (p->d_tables) cudaFree(p->d_tables);
      p->d_tables = nullptr;
      CS_CUDA(cudaMalloc(&p->d_tables, bytes));
      p->d_tables_cells = std::max<int64_t>(p->total_cells, 1);
    }
    *dtab = p->d_tables;
    if (user_tables) {
      tb.user = user_tables;
      tb.dev = p->d_tables;
      tb.bytes = sizeof(uint32_t) * p->total_cells;
      tb.host = true;
    }
  }
  p->last_dtab = *dtab;
  return CS_OK;
}

// tables argument of score/compact: NULL = the device tables of the last execute
static int input_tables(cs_plan* p, const uint32_t* tables, const uint32_t** out) {
  cs_ctx* ctx = p->db->ctx;
  if (!tables) {
    if (!p->last_dtab) return fail(CS_ERR_INVALID, "no device tables: execute with CS_WANT_TABLES first");
    *out = p->last_dtab;
    return CS_OK;
  }
  if (is_device_ptr(tables)) {
    *out = tables;
    return CS_OK;
  }
  void* d = nullptr;
  CS_TRY(ctx->scratch_get(1, sizeof(uint32_t) * std::max<int64_t>(p->total_cells, 1), &d));
  CS_CUDA(cudaMemcpyAsync(d, tables, sizeof(uint32_t) * p->total_cells, cudaMemcpyHostToDevice, ctx->stream));
  *out = (const uint32_t*)d;
  return CS_OK;
}

static int finish_outputs(cs_ctx* ctx, OutBuf* obs, int nob) {
  bool any_host = false;
  for (int i = 0; i < nob; ++i) {
    any_host = any_host || obs[i].mapped;  // written in place by the kernels: wait for them
    if (obs[i].host) {
      CS_CUDA(cudaMemcpyAsync(obs[i].user, obs[i].dev, obs[i].bytes, cudaMemcpyDeviceToHost, ctx->stream));
      any_host = true;
    }
  }
  if (any_host && !ctx->pipe) CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

// sparse (hash) query: count into the two hash tables, then score from them
static int run_sparse(cs_plan* p, cs_plan::SparseQ& sq, uint32_t flags, double* ll, double* mi,
                      int64_t* nnz) {
  cs_db* db = p->db;
  cs_ctx* ctx = db->ctx;
  const int nparts = (int)std::min<uint64_t>((sq.H + 255) / 256, (uint64_t)ctx->num_sms * 8);
  if (!sq.blob) {
    const size_t bv = round_up(sizeof(int32_t) * sq.k, 256), bs = round_up(sizeof(uint64_t) * sq.k, 256);
    const size_t bk = round_up(8 * sq.H, 256), bc = round_up(4 * sq.H, 256), bp = round_up(24 * nparts, 256);
    cudaError_t e = cudaMalloc(&sq.blob, bv + bs + 2 * bk + 2 * bc + bp);
    if (e != cudaSuccess) {
      cudaGetLastError();
      sq.blob = nullptr;
      return fail(CS_ERR_OOM, "sparse query %d: cannot allocate hash tables of %llu slots", sq.q,
                  (unsigned long long)sq.H);
    }
    char* o = sq.blob;
    sq.d_vars = (int32_t*)o;
    o += bv;
    sq.d_stride = (unsigned long long*)o;
    o += bs;
    sq.keys = (unsigned long long*)o;
    o += bk;
    sq.pkeys = (unsigned long long*)o;
    o += bk;
    sq.cnt = (uint32_t*)o;
    o += bc;
    sq.pcnt = (uint32_t*)o;
    o += bc;
    sq.part = (double*)o;
    sq.nparts = nparts;
    CS_CUDA(cudaMemcpy(sq.d_vars, sq.vars.data(), sizeof(int32_t) * sq.k, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(sq.d_stride, sq.stride.data(), sizeof(uint64_t) * sq.k, cudaMemcpyHostToDevice));
  }
  CS_CUDA(cudaMemsetAsync(sq.keys, 0xff, 2 * round_up(8 * sq.H, 256), ctx->stream));
  CS_CUDA(cudaMemsetAsync(sq.cnt, 0, 2 * round_up(4 * sq.H, 256), ctx->stream));
  const unsigned grid = (unsigned)std::min<int64_t>((db->m + 255) / 256, (int64_t)ctx->num_sms * 8);
  k_sparse_count<<<grid, 256, 0, ctx->stream>>>(db->cols, db->ld, db->m, sq.d_vars, sq.d_stride, sq.k, sq.rt,
                                                sq.keys, sq.cnt, sq.pkeys, sq.pcnt, sq.H - 1);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  if ((flags & F_PARTIAL) || !(flags & (F_LOGLIK | F_MI | F_NNZ))) return CS_OK;
  unsigned long long* qmarg = nullptr;
  if (flags & F_MI) {
    void* d = nullptr;
    CS_TRY(ctx->scratch_get(20, sizeof(unsigned long long) * CS_MAX_ARITY, &d));
    qmarg = (unsigned long long*)d;
    CS_CUDA(cudaMemsetAsync(qmarg, 0, sizeof(unsigned long long) * CS_MAX_ARITY, ctx->stream));
    k_sparse_marg<<<sq.nparts, 256, 0, ctx->stream>>>(sq.keys, sq.cnt, sq.H, sq.rt, qmarg);
    ctx->launches++;
  }
  const double m_total = (double)db->m_total;
  k_sparse_part<<<sq.nparts, 256, 0, ctx->stream>>>(sq.keys, sq.cnt, sq.pkeys, sq.pcnt, sq.H, sq.rt, qmarg,
                                                    flags, m_total, sq.part);
  k_sparse_reduce<<<1, 32, 0, ctx->stream>>>(sq.part, sq.nparts, sq.q, ll, mi, nnz, m_total);
  ctx->launches += 2;
  CS_CUDA(cudaGetLastError());
  return CS_OK;
}

// chunked K2 over a query list (which = 0: global-class score_list, 1: all queries)
static int run_chunked_score(cs_plan* p, int which, const uint32_t* dtab, uint32_t flags, double* ll,
                             double* mi, int64_t* nnz) {
  cs_ctx* ctx = p->db->ctx;
  auto& L = p->sl[which];
  if (!L.built) {
    std::vector<int32_t> qlist;
    if (which == 0) qlist = p->score_list;
    else {
      qlist.resize(p->nq);
      std::iota(qlist.begin(), qlist.end(), 0);
    }
    const uint32_t CH = 2048;  // configurations per CTA
    std::vector<int32_t> first(1, 0);
    std::vector<ScoreItem> items;
    for (size_t i = 0; i < qlist.size(); ++i) {
      const QDesc& d = p->hq[qlist[i]];
      const uint32_t J = d.cells / (uint32_t)d.r_target;
      for (uint32_t j0 = 0; j0 < J || (J == 0 && j0 == 0); j0 += CH) {
        items.push_back(ScoreItem{qlist[i], (int32_t)i, j0, std::min(J, j0 + CH)});
        if (J == 0) break;
      }
      first.push_back((int32_t)items.size());
    }
    const size_t b0 = sizeof(int32_t) * std::max<size_t>(qlist.size(), 1);
    const size_t b1 = sizeof(int32_t) * first.size();
    const size_t b2 = sizeof(ScoreItem) * std::max<size_t>(items.size(), 1);
    const size_t b3 = sizeof(double) * 3 * std::max<size_t>(items.size(), 1);
    const size_t o1 = round_up(b0, 256), o2 = o1 + round_up(b1, 256), o3 = o2 + round_up(b2, 256);
    CS_CUDA(cudaMalloc(&L.blob, o3 + b3));
    CS_CUDA(cudaMemcpy(L.blob, qlist.data(), sizeof(int32_t) * qlist.size(), cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(L.blob + o1, first.data(), b1, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(L.blob + o2, items.data(), sizeof(ScoreItem) * items.size(), cudaMemcpyHostToDevice));
    L.qlist = (int32_t*)L.blob;
    L.first = (int32_t*)(L.blob + o1);
    L.items = (ScoreItem*)(L.blob + o2);
    L.part = (double*)(L.blob + o3);
    L.nlist = (int)qlist.size();
    L.nitems = (int)items.size();
    L.built = true;
  }
  if (L.nlist == 0) return CS_OK;
  unsigned long long* qmarg = nullptr;
  if (flags & F_MI) {
    void* d = nullptr;
    CS_TRY(ctx->scratch_get(19, sizeof(unsigned long long) * CS_MAX_ARITY * L.nlist, &d));
    qmarg = (unsigned long long*)d;
    CS_CUDA(cudaMemsetAsync(qmarg, 0, sizeof(unsigned long long) * CS_MAX_ARITY * L.nlist, ctx->stream));
    k_score_marg<<<L.nitems, 256, 0, ctx->stream>>>(p->d_q, L.items, dtab, qmarg);
    ctx->launches++;
    CS_CUDA(cudaGetLastError());
  }
  const double m_total = (double)p->db->m_total;
  k_score_part<<<L.nitems, 256, 0, ctx->stream>>>(p->d_q, L.items, dtab, qmarg, L.part, flags, m_total);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  k_score_reduce<<<(L.nlist + 255) / 256, 256, 0, ctx->stream>>>(L.qlist, L.first, L.nlist, L.part, ll, mi,
                                                                  nnz, m_total);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  return CS_OK;
}

extern "C" int cs_plan_execute(cs_plan* p, uint32_t* tables, double* loglik, double* mi,
                               int64_t* nnz) {
  CtxLock lk_(p ? p->db->ctx : nullptr);
  if (!p) return fail(CS_ERR_INVALID, "cs_plan_execute: NULL plan");
  cs_db* db = p->db;
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  if (p->nq == 0) return CS_OK;
  uint32_t flags = p->flags;
  if (env_int("CS_NARROW_FAST", 1) == 0) flags |= F_NARROW_EXACT;
  if (loglik) flags |= F_LOGLIK;
  if (mi) flags |= F_MI;
  if (nnz) flags |= F_NNZ;
  OutBuf tb, lb, mb, nb;
  uint32_t* dtab = nullptr;
  CS_TRY(plan_tables(p, tables, tb, &dtab));
  const bool partial = (flags & F_PARTIAL) != 0;
  if (!partial) {
    CS_TRY(route(ctx, 2, loglik, sizeof(double) * p->nq, lb));
    CS_TRY(route(ctx, 3, mi, sizeof(double) * p->nq, mb));
    CS_TRY(route(ctx, 4, nnz, sizeof(int64_t) * p->nq, nb));
  }
  if (p->needs_zero && dtab)
    CS_CUDA(cudaMemsetAsync(dtab, 0, sizeof(uint32_t) * p->total_cells, ctx->stream));
  CS_CUDA(cudaMemsetAsync(p->d_head, 0, 1024, ctx->stream));
  CS_CUDA(cudaMemsetAsync(p->d_done, 0, sizeof(uint32_t) * p->nq, ctx->stream));
  const double m_total = (double)db->m_total;
  // ev0/ev1 bracket the whole histogram phase (K1 global + K1 SMEM + K1g) on this stream
  CS_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  // fork: launches of the histogram phase rotate over the context stream and the side streams
  // (CS_STREAMS = 1 keeps everything on the context stream)
  const int nlaunch = (int)p->groups.size() + (p->ngitems > 0) + !p->generic_list.empty() + !p->waves.empty() +
                      !p->blaunch.empty() + !p->swaves.empty();
  const int nstreams = nlaunch > 1 ? std::max(1, std::min(1 + cs_ctx::NSIDE, env_int("CS_STREAMS", 4))) : 1;
  int rr = 0;  // next stream of the rotation
  auto pick = [&]() -> cudaStream_t {
    const int s = rr++ % nstreams;
    return s == 0 ? ctx->stream : ctx->side[s - 1];
  };
  if (nstreams > 1) {
    CS_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
    for (int i = 0; i + 1 < nstreams; ++i) CS_CUDA(cudaStreamWaitEvent(ctx->side[i], ctx->fork_ev, 0));
  }
  if (p->ngitems > 0) {
    const int grid = std::min(2 * ctx->num_sms, p->ngitems);
    k_hist_global<<<grid, 512, 0, pick()>>>(p->d_q, p->d_items + p->nitems, p->ngitems,
                                                 p->d_head + 1, dtab);
    ctx->launches++;
    CS_CUDA(cudaGetLastError());
  }
  if (p->nitems > 0) {
    for (size_t g = 0; g < p->groups.size(); ++g) {
      const auto& G = p->groups[g];
      const int k = G.key / 24 + 1, path = (G.key % 24) / 3, nib = G.key % 3;
      HistFn f = kHist[k - 1][path][nib];
      if (!f) return fail(CS_ERR_INVALID, "internal: no K1 variant for k=%d path=%d", k, path);
      const int grid = std::min(ctx->hist_ctas, G.count);
      f<<<grid, CS_HIST_THREADS, ctx->hist_smem, pick()>>>(
          p->d_q, p->d_items + G.first, G.count, p->d_head + 2 + (int)g, dtab, p->d_done,
          (double*)lb.dev, (double*)mb.dev, (int64_t*)nb.dev, flags, m_total);
      ctx->launches++;
      CS_CUDA(cudaGetLastError());
    }
  }
  if (!p->generic_list.empty()) {
    dim3 grid((unsigned)std::min<int64_t>((db->m + 255) / 256, 1024),
              (unsigned)std::min<size_t>(p->generic_list.size(), 65535));
    k_hist_generic<<<grid, 256, 0, pick()>>>(p->d_q, p->d_generic_list, p->d_gvars, p->d_gstride,
                                                  db->cols, db->ld, db->m, dtab, (int)p->generic_list.size());
    ctx->launches++;
    CS_CUDA(cudaGetLastError());
  }
  if (!p->waves.empty()) {
    // partition class: per wave, k_radix_part per digit count, then k_radix_count
    void* scr = nullptr;
    CS_TRY(ctx->scratch_get(23, p->rx_scratch, &scr));
    const cudaStream_t ws = pick();  // waves share the scratch: one stream for all of them
    CS_CUDA(cudaMemsetAsync(p->d_rhead, 0, sizeof(int) * p->waves.size(), ws));
    for (size_t w = 0; w < p->waves.size(); ++w) {
      const auto& wv = p->waves[w];
      for (const auto& L : wv.parts) {
        const int total = L.count * p->rx_nchunks;
        if (total == 0) continue;
        const int grid = std::min(total, (1024 / RX_THREADS) * ctx->num_sms);
        kRadixPart[L.k - 1]<<<grid, RX_THREADS, RX_SMEM, ws>>>(p->d_rdesc + L.first, L.count,
                                                                         p->rx_nchunks, db->m, (char*)scr);
        ctx->launches++;
        CS_CUDA(cudaGetLastError());
      }
      if (wv.nitems > 0 && p->rx_nchunks > 0) {
        const int grid = std::min(wv.nitems, ctx->num_sms);
        k_radix_count<<<grid, RC_THREADS, RC_SMEM, ws>>>(p->d_q, p->d_rdesc, p->d_ritems + wv.item0,
                                                                  wv.nitems, p->d_rhead + w, dtab, (const char*)scr);
        ctx->launches++;
        CS_CUDA(cudaGetLastError());
      }
    }
  }
  if (!p->swaves.empty()) {
    // spill class: per wave, k_spill_hist per digit count, then k_spill_count
    void* scr = nullptr;
    CS_TRY(ctx->scratch_get(24, p->sp_scratch, &scr));
    const cudaStream_t ss = pick();  // waves share the scratch: one stream for all of them
    CS_CUDA(cudaMemsetAsync(p->d_shead, 0, sizeof(int) * p->sp_heads, ss));
    int hd = 0;
    const int sp_exact = (flags & F_NARROW_EXACT) ? 1 : 0;  // CS_NARROW_FAST=0: always recount exactly
    for (const auto& wv : p->swaves) {
      for (const auto& L : wv.parts) {
        const int grid = std::min(L.count, ctx->hist_ctas);
        kSpillHist[L.k - 1]<<<grid, SP_THREADS, ctx->hist_smem, ss>>>(p->d_sdesc, p->d_sitems + L.first, L.count,
                                                                      p->d_shead + hd++, dtab, (char*)scr, sp_exact);
        ctx->launches++;
        CS_CUDA(cudaGetLastError());
      }
      const int grid = std::min(wv.nitems, ctx->num_sms);
      k_spill_count<<<grid, SP_THREADS, SP_COUNT_SMEM, ss>>>(p->d_sdesc, p->d_citems + wv.item0, wv.nitems,
                                                            p->d_shead + hd++, dtab, (const char*)scr, sp_exact);
      ctx->launches++;
      CS_CUDA(cudaGetLastError());
    }
  }
  if (!p->blaunch.empty()) {
    // bitmap class: subset popcounts per digit count, then the in-place superset -> cell transform
    const cudaStream_t bs = pick();  // subset popcounts, then their in-place transform: one stream
    CS_CUDA(cudaMemsetAsync(p->d_bhead, 0, sizeof(int) * BQ_MAXK, bs));
    for (size_t i = 0; i < p->blaunch.size(); ++i) {
      const auto& L = p->blaunch[i];
      const int per_sm = bq_smem_bytes(L.k) <= 100 * 1024 ? 2 : 1;
      const int grid = std::min(L.nitems, per_sm * ctx->num_sms);
      kBitmapQ[L.k - 1]<<<grid, BQ_THREADS, bq_smem_bytes(L.k), bs>>>(
          p->d_bdesc, p->d_bitems + L.item0, L.nitems, p->d_bhead + i, db->words, dtab);
      ctx->launches++;
      CS_CUDA(cudaGetLastError());
    }
    const int nb = (int)p->bdesc.size();
    k_bitmap_mobius<<<(nb + 127) / 128, 128, 0, bs>>>(p->d_bdesc, nb, (uint32_t)db->m, dtab);
    ctx->launches++;
    CS_CUDA(cudaGetLastError());
  }
  if (nstreams > 1) {  // join
    for (int i = 0; i + 1 < nstreams; ++i) {
      CS_CUDA(cudaEventRecord(ctx->join_ev[i], ctx->side[i]));
      CS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev[i], 0));
    }
  }
  for (auto& sq : p->sparse) CS_TRY(run_sparse(p, sq, flags, (double*)lb.dev, (double*)mb.dev, (int64_t*)nb.dev));
  CS_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->ev_valid = true;
  if (!partial && !p->score_list.empty() && (flags & (F_LOGLIK | F_MI | F_NNZ)))
    CS_TRY(run_chunked_score(p, 0, dtab, flags, (double*)lb.dev, (double*)mb.dev, (int64_t*)nb.dev));
  OutBuf obs[4] = {tb, lb, mb, nb};
  return finish_outputs(ctx, obs, 4);
}

extern "C" int cs_plan_score(cs_plan* p, const uint32_t* tables, double* loglik, double* mi,
                             int64_t* nnz) {
  CtxLock lk_(p ? p->db->ctx : nullptr);
  if (!p) return fail(CS_ERR_INVALID, "cs_plan_score: NULL plan");
  cs_ctx* ctx = p->db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  if (p->nq == 0) return CS_OK;
  uint32_t flags = p->flags & F_NLOGN;
  if (loglik) flags |= F_LOGLIK;
  if (mi) flags |= F_MI;
  if (nnz) flags |= F_NNZ;
  if (!(flags & (F_LOGLIK | F_MI | F_NNZ))) return CS_OK;
  const uint32_t* dtab = nullptr;
  CS_TRY(input_tables(p, tables, &dtab));
  OutBuf lb, mb, nb;
  CS_TRY(route(ctx, 2, loglik, sizeof(double) * p->nq, lb));
  CS_TRY(route(ctx, 3, mi, sizeof(double) * p->nq, mb));
  CS_TRY(route(ctx, 4, nnz, sizeof(int64_t) * p->nq, nb));
  CS_TRY(run_chunked_score(p, 1, dtab, flags, (double*)lb.dev, (double*)mb.dev, (int64_t*)nb.dev));
  OutBuf obs[3] = {lb, mb, nb};
  return finish_outputs(ctx, obs, 3);
}

extern "C" int cs_plan_compact(cs_plan* p, const uint32_t* tables, const int64_t* out_off,
                               int64_t total_nnz, int64_t* cell_idx, int64_t* n_ijk, int64_t* n_ij) {
  CtxLock lk_(p ? p->db->ctx : nullptr);
  if (!p || !out_off || !cell_idx || !n_ijk || !n_ij)
    return fail(CS_ERR_INVALID, "cs_plan_compact: NULL argument");
  cs_ctx* ctx = p->db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  if (p->nq == 0 || total_nnz == 0) return CS_OK;
  const uint32_t* dtab = nullptr;
  CS_TRY(input_tables(p, tables, &dtab));
  void* d_off = nullptr;
  CS_TRY(ctx->scratch_get(5, sizeof(int64_t) * p->nq, &d_off));
  CS_CUDA(cudaMemcpyAsync(d_off, out_off, sizeof(int64_t) * p->nq, cudaMemcpyHostToDevice, ctx->stream));
  OutBuf a, b, c;
  CS_TRY(route(ctx, 6, cell_idx, sizeof(int64_t) * total_nnz, a));
  CS_TRY(route(ctx, 7, n_ijk, sizeof(int64_t) * total_nnz, b));
  CS_TRY(route(ctx, 8, n_ij, sizeof(int64_t) * total_nnz, c));
  k_compact<<<(unsigned)p->nq, 256, 0, ctx->stream>>>(p->d_q, dtab, (const int64_t*)d_off,
                                                       (int64_t*)a.dev, (int64_t*)b.dev, (int64_t*)c.dev);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  if (!p->sparse.empty()) {
    void* dpos = nullptr;
    CS_TRY(ctx->scratch_get(21, sizeof(unsigned long long) * p->sparse.size(), &dpos));
    CS_CUDA(cudaMemsetAsync(dpos, 0, sizeof(unsigned long long) * p->sparse.size(), ctx->stream));
    for (size_t i = 0; i < p->sparse.size(); ++i) {
      auto& sq = p->sparse[i];
      if (!sq.blob) return fail(CS_ERR_INVALID, "cs_plan_compact: execute the plan first");
      k_sparse_compact<<<(unsigned)std::max(sq.nparts, 1), 256, 0, ctx->stream>>>(
          sq.keys, sq.cnt, sq.pkeys, sq.pcnt, sq.H, sq.rt, out_off[sq.q], (unsigned long long*)dpos + i,
          (int64_t*)a.dev, (int64_t*)b.dev, (int64_t*)c.dev);
      ctx->launches++;
      CS_CUDA(cudaGetLastError());
    }
  }
  OutBuf obs[3] = {a, b, c};
  CS_TRY(finish_outputs(ctx, obs, 3));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));  // out_off staging reused next call
  return CS_OK;
}

// batched learn_parents: family LL / MDL from the N ln N sums of the distinct variable subsets
extern "C" int cs_family_scores(cs_ctx* ctx, int64_t nfam, const double* nlogn, int64_t nsub,
                                const int32_t* s_idx, const int32_t* p_idx, const double* penalty,
                                double m_ln_m, double* ll, double* mdl) {
  CtxLock lk_(ctx);
  if (!ctx || nfam < 0 || nsub < 0) return fail(CS_ERR_INVALID, "cs_family_scores: bad argument");
  if (nfam == 0) return CS_OK;
  if (!nlogn || !s_idx || !p_idx || (mdl && !penalty))
    return fail(CS_ERR_INVALID, "cs_family_scores: NULL input");
  CS_CUDA(cudaSetDevice(ctx->device));
  auto dev_in = [&](const void* src, size_t bytes, int slot, const void** out) -> int {
    if (is_device_ptr(src)) {
      *out = src;
      return CS_OK;
    }
    void* d = nullptr;
    CS_TRY(ctx->scratch_get(slot, bytes, &d));
    CS_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *out = d;
    return CS_OK;
  };
  const void *dn = nullptr, *ds = nullptr, *dp = nullptr, *dpen = nullptr;
  CS_TRY(dev_in(nlogn, sizeof(double) * std::max<int64_t>(nsub, 1), 11, &dn));
  CS_TRY(dev_in(s_idx, sizeof(int32_t) * nfam, 12, &ds));
  CS_TRY(dev_in(p_idx, sizeof(int32_t) * nfam, 13, &dp));
  if (mdl) CS_TRY(dev_in(penalty, sizeof(double) * nfam, 14, &dpen));
  OutBuf lb, mb;
  CS_TRY(route(ctx, 15, ll, sizeof(double) * nfam, lb));
  CS_TRY(route(ctx, 16, mdl, sizeof(double) * nfam, mb));
  const unsigned grid = (unsigned)std::min<int64_t>((nfam + 255) / 256, 65535);
  k_family<<<grid, 256, 0, ctx->stream>>>(nfam, (const double*)dn, (const int32_t*)ds, (const int32_t*)dp,
                                          (const double*)dpen, m_ln_m, (double*)lb.dev, (double*)mb.dev);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  OutBuf obs[2] = {lb, mb};
  return finish_outputs(ctx, obs, 2);
}

static int query_batch_pipelined(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                                 uint32_t flags, uint32_t* tables, double* loglik, double* mi, int64_t* nnz,
                                 int nchunks, bool trace) {
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  if (!var_off || !vars) return fail(CS_ERR_INVALID, "cs_plan_create: NULL query arrays");
  nchunks = std::min(nchunks, 8);
  // chunk j holds a growth^j share of the batch (growth 4: 1/5 + 4/5, 1/21 + 4/21 + 16/21, ...)
  const int64_t growth = std::min(std::max(env_int("CS_QB_GROWTH", 2), 1), 8);
  std::vector<int64_t> gp(nchunks + 1, 1);
  for (int j = 1; j <= nchunks; ++j) gp[j] = gp[j - 1] * growth;
  int64_t wsum = 0;
  for (int j = 0; j < nchunks; ++j) wsum += gp[j];
  struct Restore {  // leave the context in single-bank, synchronous mode on every exit
    cs_ctx* c;
    ~Restore() {
      c->bank = 0;
      c->pipe = false;
      cudaStreamSynchronize(c->stream);
    }
  } restore{ctx};
  {
    // validate the whole batch before the first chunk launches, so a bad query leaves every
    // output untouched (the per-chunk plans would otherwise fail after earlier chunks wrote)
    const int64_t max_dense = (int64_t)env_int("CS_MAX_DENSE_LOG2", 30);
    for (int32_t q = 0; q < nq; ++q) {
      const int b = var_off[q], e = var_off[q + 1];
      if (e - b < 1) return fail(CS_ERR_INVALID, "query %d has no target variable", q);
      uint64_t c = 1;
      for (int i = b; i < e; ++i) {
        const int v = vars[i];
        if (v < 0 || v >= db->n)
          return fail(CS_ERR_INVALID, "variable %d out of range for a database with n=%d", v, db->n);
        for (int j = b; j < i; ++j)
          if (vars[j] == v) return fail(CS_ERR_INVALID, "query %d repeats variable %d", q, v);
        if (c > (((uint64_t)1 << 63) - 1) / (uint64_t)db->arity[v])
          return fail(CS_ERR_UNSUPPORTED, "query %d: joint state space exceeds 2^63 cells", q);
        c *= (uint64_t)db->arity[v];
      }
      if ((flags & F_PARTIAL) && c > ((uint64_t)1 << max_dense))
        return fail(CS_ERR_UNSUPPORTED, "query %d: sparse (hash) queries cannot be instance-sharded", q);
    }
  }
  ctx->pipe = true;
  int64_t cell_off = 0, wcum = 0;
  int32_t q0 = 0;
  double tplan = 0.0;
  for (int j = 0; j < nchunks; ++j) {
    wcum += gp[j];
    const int32_t q1 = j == nchunks - 1 ? nq : (int32_t)((int64_t)nq * wcum / wsum);
    if (q1 <= q0) continue;
    ctx->bank = j & 1;
    cs_plan* p = nullptr;
    const double t0 = trace ? now_ms() : 0.0;
    CS_TRY(plan_build(db, q1 - q0, var_off + q0, vars, flags, &p, /*transient=*/true, q0));
    if (trace) tplan += now_ms() - t0;
    const int rc = cs_plan_execute(p, tables ? tables + cell_off : nullptr, loglik ? loglik + q0 : nullptr,
                                   mi ? mi + q0 : nullptr, nnz ? nnz + q0 : nullptr);
    cell_off += p->total_cells;
    cs_plan_destroy(p);
    if (rc != CS_OK) return rc;
    q0 = q1;
  }
  if (trace) fprintf(stderr, "cs_query_batch: %d chunks, plan %.3f ms (host, overlapped after the first)\n",
                     nchunks, tplan);
  ctx->pipe = false;
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

extern "C" int cs_query_batch(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                              uint32_t flags, uint32_t* tables, double* loglik, double* mi,
                              int64_t* nnz) {
  CtxLock lk_(db ? db->ctx : nullptr);
  cs_plan* p = nullptr;
  const bool trace = env_int("CS_TRACE", 0) != 0;
  // big batches: plan chunk j+1 on the host while chunk j's kernels run (chunk sizes double,
  // so each chunk's execution covers the next chunk's planning; only the first plan is exposed).
  // Chunk j holds a CS_QB_GROWTH^j share; a first chunk below ~1.4K queries loses more to K1
  // launch tails than its planning costs.  Round 1 kernels (cfg2 e2e, 10K queries): one plan
  // 4.08 ms; 2 chunks at growth 2/3/4: 3.89/3.85/3.81.  Round 2 kernels are ~20% faster, a chunk
  // covers less planning, and growth 2 wins: cfg2 growth 2 (3-4 chunks) 3.19-3.24 ms against
  // growth 4 (2 chunks) 3.28-3.42; cfg3 (74.5K subsets) 21.9-22.3 against 23.4-29.4 ms.
  // Score-only batches of cfg2's size lose (LL-only 10K queries: 4.20 ms one plan, 4.62 ms
  // chunked; the kernels skip the table stores, so chunk j no longer covers chunk j+1's plan):
  // they are chunked only from 32K queries (cfg3's 289K LL+MDL batch gains 30.7 -> 25 ms).
  int nchunks = env_int("CS_QB_CHUNKS", 0);
  if (nchunks <= 0 && !tables && nq < env_int("CS_QB_SCORE_MIN", 32768)) nchunks = 1;
  if (nchunks <= 0) {
    const int64_t min_chunk = std::max(env_int("CS_QB_MIN_CHUNK", 1400), 1);
    const int64_t growth = std::min(std::max(env_int("CS_QB_GROWTH", 2), 1), 8);
    int64_t w = 1, wsum = 1;
    nchunks = 1;
    while (nchunks < 4) {
      w *= growth;
      if ((int64_t)nq / (wsum + w) < min_chunk) break;
      wsum += w;
      ++nchunks;
    }
  }
  if (db && nchunks > 1 && nq >= 2) return query_batch_pipelined(db, nq, var_off, vars, flags, tables,
                                                                         loglik, mi, nnz, nchunks, trace);
  const double t0 = trace ? now_ms() : 0.0;
  CS_TRY(plan_build(db, nq, var_off, vars, flags, &p, /*transient=*/true));
  const double t1 = trace ? now_ms() : 0.0;
  int rc = cs_plan_execute(p, tables, loglik, mi, nnz);
  const double t2 = trace ? now_ms() : 0.0;
  cs_plan_destroy(p);
  if (trace) fprintf(stderr, "cs_query_batch: plan %.3f ms, execute+copy %.3f ms\n", t1 - t0, t2 - t1);
  return rc;
}

// one query, latency class (K8, cs_one.cuh)
static int query_one(cs_db* db, int32_t k, const int32_t* vars, uint32_t flags, uint32_t* table, double* loglik,
                     double* mi, int64_t* nnz, int64_t* cell_idx, int64_t* n_ijk, int64_t* n_ij);

extern "C" int cs_query_one(cs_db* db, int32_t k, const int32_t* vars, uint32_t flags, uint32_t* table,
                            double* loglik, double* mi, int64_t* nnz) {
  return query_one(db, k, vars, flags, table, loglik, mi, nnz, nullptr, nullptr, nullptr);
}

extern "C" int cs_query_one_cells(cs_db* db, int32_t k, const int32_t* vars, int64_t* cell_idx, int64_t* n_ijk,
                                  int64_t* n_ij, int64_t* nnz) {
  if (!cell_idx || !n_ijk || !n_ij || !nnz) return fail(CS_ERR_INVALID, "cs_query_one_cells: NULL output");
  return query_one(db, k, vars, 0, nullptr, nullptr, nullptr, nnz, cell_idx, n_ijk, n_ij);
}

static int query_one(cs_db* db, int32_t k, const int32_t* vars, uint32_t flags, uint32_t* table, double* loglik,
                     double* mi, int64_t* nnz, int64_t* cell_idx, int64_t* n_ijk, int64_t* n_ij) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db) return fail(CS_ERR_INVALID, "cs_query_one: NULL db");
  if (k < 1) return fail(CS_ERR_INVALID, "query 0 has no target variable");
  if (!vars) return fail(CS_ERR_INVALID, "cs_query_one: vars is NULL");
  uint64_t C = 1;
  for (int i = 0; i < k; ++i) {
    const int v = vars[i];
    if (v < 0 || v >= db->n) return fail(CS_ERR_INVALID, "variable %d out of range for a database with n=%d", v, db->n);
    for (int j = 0; j < i; ++j)
      if (vars[j] == v) return fail(CS_ERR_INVALID, "query 0 repeats variable %d", v);
    if (C > (((uint64_t)1 << 63) - 1) / (uint64_t)db->arity[v])
      return fail(CS_ERR_UNSUPPORTED, "query 0: joint state space exceeds 2^63 cells");
    C *= (uint64_t)db->arity[v];
  }
  const int64_t max_rows = env_int("CS_ONE_MAX_ROWS", 1 << 18);
  const bool one = k <= CS_MAXK && C <= ONE_MAX_CELLS && db->m <= max_rows && !(flags & (F_PARTIAL | F_NLOGN)) &&
                   env_int("CS_ONE", 1) != 0;
  if (!one) {  // the batch path (transient plan) answers everything else
    if (cell_idx)
      return fail(CS_ERR_UNSUPPORTED, "cs_query_one_cells: query outside the single-query class (use a plan + "
                                      "cs_plan_compact)");
    const int32_t off[2] = {0, k};
    return cs_query_batch(db, 1, off, vars, flags, table, loglik, mi, nnz);
  }
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  if (!ctx->mbox) {
    CS_CUDA(cudaHostAlloc((void**)&ctx->mbox, 64 + (size_t)ONE_MAX_CELLS * 4 + (size_t)ONE_MAX_CELLS * 24,
                          cudaHostAllocMapped));
    CS_CUDA(cudaHostGetDevicePointer((void**)&ctx->mbox_dev, ctx->mbox, 0));
  }
  OneQ q;
  memset(&q, 0, sizeof q);
  uint32_t s = 1;
  for (int i = 0; i < k; ++i) {
    q.col[i] = db->cols + (int64_t)vars[i] * db->ld;
    q.stride[i] = s;
    s *= (uint32_t)db->arity[vars[i]];
  }
  q.k = k;
  q.r_t = db->arity[vars[0]];
  q.cells = (uint32_t)C;
  q.flags = flags | (loglik ? F_LOGLIK : 0u) | (mi ? F_MI : 0u) | (nnz ? F_NNZ : 0u);
  q.m = db->m;
  q.m_total = (double)db->m_total;
  const bool table_dev = table && is_device_ptr(table);
  q.table = table ? (table_dev ? table : (uint32_t*)(ctx->mbox_dev + 64)) : nullptr;
  q.out = (double*)ctx->mbox_dev;
  q.cells_out = cell_idx ? (int64_t*)(ctx->mbox_dev + 64 + (size_t)ONE_MAX_CELLS * 4) : nullptr;
  q.done = (volatile uint32_t*)(ctx->mbox_dev + 32);
  q.seq = ++ctx->one_seq;
  volatile uint32_t* done = (volatile uint32_t*)(ctx->mbox + 32);
  k_query_one<<<1, ONE_THREADS, (size_t)C * 4, ctx->stream>>>(q);
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  // poll the mapped completion word (a stream sync costs several microseconds more); after
  // ~2 ms fall back to the stream sync, which also reports a failed kernel
  const double t0 = now_ms();
  bool seen = false;
  for (int spin = 0; !seen; ++spin) {
    seen = *done == q.seq;
    if (!seen && (spin & 1023) == 1023 && now_ms() - t0 > 2.0) break;
  }
  if (!seen) CS_CUDA(cudaStreamSynchronize(ctx->stream));
  std::atomic_thread_fence(std::memory_order_acquire);
  const double* o = (const double*)ctx->mbox;
  auto put = [&](void* user, const void* src, size_t bytes) -> int {
    if (!user) return CS_OK;
    if (is_device_ptr(user)) {
      CS_CUDA(cudaMemcpy(user, src, bytes, cudaMemcpyHostToDevice));
    } else {
      memcpy(user, src, bytes);
    }
    return CS_OK;
  };
  CS_TRY(put(loglik, o, 8));
  CS_TRY(put(mi, o + 1, 8));
  CS_TRY(put(nnz, o + 2, 8));
  if (table && !table_dev) memcpy(table, ctx->mbox + 64, (size_t)C * 4);
  if (cell_idx) {
    const int64_t nz = ((const int64_t*)ctx->mbox)[2];
    const int64_t* src = (const int64_t*)(ctx->mbox + 64 + (size_t)ONE_MAX_CELLS * 4);
    memcpy(cell_idx, src, sizeof(int64_t) * nz);
    memcpy(n_ijk, src + C, sizeof(int64_t) * nz);
    memcpy(n_ij, src + 2 * C, sizeof(int64_t) * nz);
  }
  return CS_OK;
}

// ------------------------------------------------------------------------------------------
// instance-shard merge (NCCL; cs_comm.cuh)

#define CS_NCCL(call)                                                                         \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      return fail(CS_ERR_CUDA, "%s failed: %s", #call, nccl_api().GetErrorString(r_));        \
  } while (0)

extern "C" int cs_comm_unique_id(void* id) {
  if (!id) return fail(CS_ERR_INVALID, "cs_comm_unique_id: NULL id");
  NcclApi& a = nccl_api();
  if (!a.ok) return fail(CS_ERR_UNSUPPORTED, "%s", a.err.c_str());
  ncclUniqueId u;
  CS_NCCL(a.GetUniqueId(&u));
  memcpy(id, &u, sizeof u);
  return CS_OK;
}

extern "C" int cs_comm_init(cs_ctx* ctx, const void* id, int32_t rank, int32_t nranks) {
  CtxLock lk_(ctx);
  if (!ctx || !id) return fail(CS_ERR_INVALID, "cs_comm_init: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CS_ERR_INVALID, "cs_comm_init: rank %d of %d", rank, nranks);
  NcclApi& a = nccl_api();
  if (!a.ok) return fail(CS_ERR_UNSUPPORTED, "%s", a.err.c_str());
  CS_CUDA(cudaSetDevice(ctx->device));
  if (ctx->comm) {
    a.CommDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  CS_NCCL(a.CommInitRank(&ctx->comm, nranks, u, rank));
  ctx->comm_rank = rank;
  ctx->comm_size = nranks;
  return CS_OK;
}

extern "C" int cs_comm_destroy(cs_ctx* ctx) {
  CtxLock lk_(ctx);
  if (!ctx) return fail(CS_ERR_INVALID, "cs_comm_destroy: NULL ctx");
  if (ctx->comm) {
    CS_CUDA(cudaSetDevice(ctx->device));
    CS_NCCL(nccl_api().CommDestroy(ctx->comm));
    ctx->comm = nullptr;
  }
  ctx->comm_rank = 0;
  ctx->comm_size = 1;
  return CS_OK;
}

extern "C" int cs_reduce_tables(cs_ctx* ctx, uint32_t* tables, int64_t cells, int32_t op, uint32_t* out) {
  CtxLock lk_(ctx);
  if (!ctx || !tables) return fail(CS_ERR_INVALID, "cs_reduce_tables: NULL argument");
  if (!ctx->comm) return fail(CS_ERR_INVALID, "cs_reduce_tables: call cs_comm_init first");
  if (cells < 0) return fail(CS_ERR_INVALID, "cs_reduce_tables: cells < 0");
  if (!is_device_ptr(tables) || (out && !is_device_ptr(out)))
    return fail(CS_ERR_INVALID, "cs_reduce_tables: tables must be device memory");
  CS_CUDA(cudaSetDevice(ctx->device));
  NcclApi& a = nccl_api();
  // uint32 counts summed as uint32 (m < 2^32 keeps every merged count exact)
  if (op == CS_REDUCE_ALLREDUCE) {
    CS_NCCL(a.AllReduce(tables, out ? out : tables, (size_t)cells, ncclUint32, ncclSum, ctx->comm, ctx->stream));
  } else if (op == CS_REDUCE_SCATTER) {
    if (cells % ctx->comm_size) return fail(CS_ERR_INVALID, "cs_reduce_tables: %lld cells not a multiple of %d ranks",
                                            (long long)cells, ctx->comm_size);
    if (!out) return fail(CS_ERR_INVALID, "cs_reduce_tables: REDUCE_SCATTER needs an output buffer");
    CS_NCCL(a.ReduceScatter(tables, out, (size_t)(cells / ctx->comm_size), ncclUint32, ncclSum, ctx->comm, ctx->stream));
  } else {
    return fail(CS_ERR_INVALID, "cs_reduce_tables: bad op %d", op);
  }
  return CS_OK;
}

extern "C" int cs_comm_all_gather(cs_ctx* ctx, const void* send, int64_t bytes, void* recv) {
  CtxLock lk_(ctx);
  if (!ctx || !send || !recv) return fail(CS_ERR_INVALID, "cs_comm_all_gather: NULL argument");
  if (!ctx->comm) return fail(CS_ERR_INVALID, "cs_comm_all_gather: call cs_comm_init first");
  if (!is_device_ptr(send) || !is_device_ptr(recv))
    return fail(CS_ERR_INVALID, "cs_comm_all_gather: buffers must be device memory");
  CS_CUDA(cudaSetDevice(ctx->device));
  CS_NCCL(nccl_api().AllGather(send, recv, (size_t)bytes, ncclUint8, ctx->comm, ctx->stream));
  return CS_OK;
}

// ------------------------------------------------------------------------------------------
// point counts

extern "C" int cs_count_points(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                               const int32_t* states, int64_t* counts) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db || !counts) return fail(CS_ERR_INVALID, "cs_count_points: NULL argument");
  if (nq < 0) return fail(CS_ERR_INVALID, "cs_count_points: nq < 0");
  if (nq == 0) return CS_OK;
  if (!var_off || !vars || !states) return fail(CS_ERR_INVALID, "cs_count_points: NULL query arrays");
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  bool all_planes = db->planes != nullptr;
  for (int q = 0; q < nq; ++q) {
    for (int j = var_off[q]; j < var_off[q + 1]; ++j) {
      const int v = vars[j], s = states[j];
      if (v < 0 || v >= db->n)
        return fail(CS_ERR_INVALID, "variable %d out of range for a database with n=%d", v, db->n);
      if (s < 0 || s >= db->arity[v])
        return fail(CS_ERR_INVALID, "state %d out of range for variable %d with arity %d", s, v, db->arity[v]);
      if (db->plane_off[v] < 0) all_planes = false;
    }
  }
  // queries with no variables count every record (Assignment((), ()) -> m)
  std::vector<int32_t> qmap;  // non-empty queries
  std::vector<int32_t> poff(1, 0);
  std::vector<int64_t> plist;
  std::vector<int32_t> pvar, pstate;
  for (int q = 0; q < nq; ++q) {
    if (var_off[q + 1] == var_off[q]) continue;
    qmap.push_back(q);
    for (int j = var_off[q]; j < var_off[q + 1]; ++j) {
      if (all_planes) plist.push_back(db->plane_off[vars[j]] + (int64_t)states[j] * db->words);
      pvar.push_back(vars[j]);
      pstate.push_back(states[j]);
    }
    poff.push_back((int32_t)pvar.size());
  }
  const int nne = (int)qmap.size();
  std::vector<int64_t> out(nq, db->m);
  if (nne > 0) {
    const size_t b0 = sizeof(int32_t) * poff.size();
    const size_t b1 = sizeof(int64_t) * std::max<size_t>(plist.size(), 1);
    const size_t b2 = sizeof(int32_t) * pvar.size();
    const size_t b3 = sizeof(unsigned long long) * nne;
    const size_t o1 = round_up(b0, 256), o2 = o1 + round_up(b1, 256), o3 = o2 + round_up(b2, 256),
                 o4 = o3 + round_up(b2, 256), tot = o4 + round_up(b3, 256);
    void* blob = nullptr;
    CS_TRY(ctx->scratch_get(9, tot, &blob));
    char* d = (char*)blob;
    CS_CUDA(cudaMemcpyAsync(d, poff.data(), b0, cudaMemcpyHostToDevice, ctx->stream));
    if (all_planes) CS_CUDA(cudaMemcpyAsync(d + o1, plist.data(), b1, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaMemcpyAsync(d + o2, pvar.data(), b2, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaMemcpyAsync(d + o3, pstate.data(), b2, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaMemsetAsync(d + o4, 0, b3, ctx->stream));
    unsigned long long* dc = (unsigned long long*)(d + o4);
    if (all_planes) {
      const int64_t wpc = 32768;
      dim3 grid((unsigned)((db->words + wpc - 1) / wpc), (unsigned)std::min(nne, 65535));
      k_points_bitmap<<<grid, 256, 0, ctx->stream>>>((const int32_t*)d, (const int64_t*)(d + o1),
                                                      db->planes, db->words, wpc, dc, nne);
    } else {
      const int64_t rpc = 1 << 20;
      dim3 grid((unsigned)((db->m + rpc - 1) / rpc), (unsigned)std::min(nne, 65535));
      k_points_scan<<<grid, 256, 0, ctx->stream>>>((const int32_t*)d, (const int32_t*)(d + o2),
                                                    (const int32_t*)(d + o3), db->cols, db->ld, db->m,
                                                    rpc, dc, nne);
    }
    ctx->launches++;
    CS_CUDA(cudaGetLastError());
    std::vector<unsigned long long> hc(nne);
    CS_CUDA(cudaMemcpyAsync(hc.data(), dc, b3, cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < nne; ++i) out[qmap[i]] = (int64_t)hc[i];
  }
  if (is_device_ptr(counts)) {
    CS_CUDA(cudaMemcpyAsync(counts, out.data(), sizeof(int64_t) * nq, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    memcpy(counts, out.data(), sizeof(int64_t) * nq);
  }
  return CS_OK;
}

// K4d (cs_itemsets_sel.cuh): supports by rarest-item selection.  Returns 1 (declined, nothing
// written) when the cost model prefers the dense bit-GEMM for this data, CS_OK when done.
static int itemsets_selector(cs_db* db, int n, const std::vector<const uint32_t*>& hp, int64_t* pairs,
                             int64_t* triples, int mode) {
  cs_ctx* ctx = db->ctx;
  const int64_t W = db->words;  // multiple of 32 words
  const int64_t ntri = (int64_t)n * (n - 1) * (n - 2) / 6;
  // 1. item supports: the state-1 plane counts recorded when the bitmap index was built
  size_t off = 0;
  auto place = [&](size_t b) {
    size_t o = off;
    off = round_up(off + b, 256);
    return o;
  };
  const size_t bp = sizeof(void*) * n;
  const size_t ors = place(bp), ori = place(sizeof(int16_t) * SEL_MAXN), ohd = place(sizeof(int));
  const size_t meta_end = off;
  std::vector<unsigned long long> supp(n);
  for (int i = 0; i < n; ++i) supp[i] = (unsigned long long)db->plane_count[(hp[i] - db->planes) / db->words];
  // 2. ranks (support descending, ties by position) and the cost model
  std::vector<int> rank_item(n);
  std::iota(rank_item.begin(), rank_item.end(), 0);
  std::stable_sort(rank_item.begin(), rank_item.end(), [&](int a, int b) { return supp[a] > supp[b]; });
  const double m = (double)db->m;
  // cost model: k_sel_gram issues ~r^2/64 popcounts per selected record of rank r (8 x 4
  // register blocks over 32-record batches), plus the record gathers
  std::vector<double> cost(n, 0.0);
  std::vector<char> dmode(n, 0);
  double total = 0.0, gathered = 0.0;
  for (int r = 1; r < n; ++r) {
    const double sr = (double)supp[rank_item[r]];
    const int nby = (r + 7) / 8, nbz = (r + 3) / 4;
    double nblk = 0;
    for (int y = 0; y < nby && 2 * y < nbz; ++y) nblk += nbz - 2 * y;
    // warp instructions: Gram 3 x 32 popc-steps per block per 32-record batch, the batch
    // transposes ~30 per mask word per batch, the selector-plane scan ~1.25 per word
    const double compact = sr * (0.094 * nblk + (r + 31) / 32 + 1.0) + 1.25 * (double)W;
    // dense selectors: every plane word is a batch (Y = P_y & P_s), no list / gather / transpose
    const double direct = (double)W * (3.0 * nblk + 0.19 * r + 1.0);
    dmode[r] = direct < compact;
    cost[r] = std::min(compact, direct);
    total += cost[r];
    gathered += sr;
  }
  // measured rates (B200): POPC ~16/clk/SM at ~60% issue; the tcgen05 bit-GEMM ~7e14 MAC/s
  const double sparse_s = total / (ctx->num_sms * 4.0 * 1.9e9 * 0.5) + gathered * 32.0 / 3e12 +
                          (double)W * 32 * 32 / 5e12;
  const double dense_s = ((double)ntri + 0.5 * n * (n - 1)) * m / 7e14;
  if (mode < 0 && sparse_s > dense_s) return 1;
  // 3. record-major rank masks
  const int wr = n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8;
  // units: (rank, word range) with ~equal cost, ranges in multiples of 512 words (16 warps x 32)
  const double target = std::max(1.0, total / (ctx->num_sms * (double)env_int("CS_SEL_UNITS", 48)));
  std::vector<SelUnit> units;
  std::vector<double> ucost;
  for (int r = 1; r < n; ++r) {
    if (!cost[r]) continue;
    const int nby = (r + 7) / 8, nbz = (r + 3) / 4;
    int nblk = 0;
    for (int y = 0; y < nby && 2 * y < nbz; ++y) nblk += nbz - 2 * y;
    const int nsplit = (nblk + SEL_THREADS - 1) / SEL_THREADS;  // block ranges of <= SEL_THREADS
    int64_t chunks = std::max<int64_t>(1, (int64_t)std::ceil(cost[r] / target / nsplit));
    const int64_t per = round_up((W + chunks - 1) / chunks, 128 * SEL_WARPS);  // A1 chunk stride
    for (int sp = 0; sp < nsplit; ++sp) {
      const int b0 = (int)((int64_t)nblk * sp / nsplit), b1 = (int)((int64_t)nblk * (sp + 1) / nsplit);
      for (int64_t w0 = 0; w0 < W; w0 += per) {
        units.push_back(SelUnit{r | (dmode[r] ? 1 << 30 : 0), (int16_t)b0, (int16_t)b1, w0, std::min(W, w0 + per)});
        ucost.push_back(cost[r] / nsplit * (double)(std::min(W, w0 + per) - w0) / (double)W + 2.0 * (b1 - b0));
      }
    }
  }
  std::vector<int> order(units.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ucost[a] > ucost[b]; });
  std::vector<SelUnit> sorted(units.size());
  for (size_t i = 0; i < order.size(); ++i) sorted[i] = units[order[i]];
  const size_t bu = sizeof(SelUnit) * std::max<size_t>(1, sorted.size());
  const size_t bpairs = sizeof(uint64_t) * (size_t)n * n, btri = sizeof(uint64_t) * std::max<int64_t>(ntri, 1);
  const size_t brm = sizeof(uint32_t) * (size_t)W * 32 * wr;
  const size_t ou = place(bu), opr = place(bpairs), otr = place(btri), orm = place(brm);
  void* blob = nullptr;
  CS_TRY(ctx->scratch_get(11, off, &blob));
  char* d = (char*)blob;
  std::vector<const uint32_t*> rp(n);
  std::vector<int16_t> ri(SEL_MAXN, 0);
  for (int r = 0; r < n; ++r) rp[r] = hp[rank_item[r]], ri[r] = (int16_t)rank_item[r];
  void* hst = nullptr;
  const size_t hbytes = meta_end + bu;
  CS_TRY(ctx->pinned_get(hbytes, &hst));
  char* h = (char*)hst;
  memcpy(h + ors, rp.data(), bp);
  memcpy(h + ori, ri.data(), sizeof(int16_t) * SEL_MAXN);
  if (!sorted.empty()) memcpy(h + ou, sorted.data(), sizeof(SelUnit) * sorted.size());
  CS_CUDA(cudaMemcpyAsync(d, h, ohd, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemcpyAsync(d + ou, h + ou, bu, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemsetAsync(d + ohd, 0, sizeof(int), ctx->stream));
  CS_CUDA(cudaMemsetAsync(d + opr, 0, otr - opr + btri, ctx->stream));
  const int Rw = (int)round_up(n - 1, 8);  // Y row stride (ranks < rmax = n - 1)
  const size_t smem = sizeof(uint32_t) * (SEL_LCAP + (size_t)SEL_MAXB * Rw);
  ctx->itemset_class = CS_ITEMSETS_SELECTOR;
  CS_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  k_sel_rowmask<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>((const uint32_t* const*)(d + ors), n, W, wr,
                                                          (uint32_t*)(d + orm));
  ctx->launches++;
  if (!sorted.empty()) {
    k_sel_gram<<<2 * ctx->num_sms, SEL_THREADS, smem, ctx->stream>>>(
        (const uint32_t* const*)(d + ors), (const uint32_t*)(d + orm), wr, (const int16_t*)(d + ori), n,
        (const SelUnit*)(d + ou), (int)sorted.size(), (int*)(d + ohd), Rw, (unsigned long long*)(d + opr),
        (unsigned long long*)(d + otr), env_int("CS_SEL_DEBUG", 0));  // diagnostic: skip phases (wrong results)
    ctx->launches++;
  }
  CS_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->ev_valid = true;
  CS_CUDA(cudaGetLastError());
  const cudaMemcpyKind kp = is_device_ptr(pairs) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const cudaMemcpyKind kt = is_device_ptr(triples) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (pairs) CS_CUDA(cudaMemcpyAsync(pairs, d + opr, bpairs, kp, ctx->stream));
  if (triples && ntri) CS_CUDA(cudaMemcpyAsync(triples, d + otr, sizeof(uint64_t) * ntri, kt, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

extern "C" int cs_itemset_supports(cs_db* db, int32_t nitems, const int32_t* items, int64_t* pairs,
                                   int64_t* triples) {
  CtxLock lk_(db ? db->ctx : nullptr);
  if (!db) return fail(CS_ERR_INVALID, "cs_itemset_supports: NULL db");
  if (nitems < 0 || nitems > 30000) return fail(CS_ERR_INVALID, "cs_itemset_supports: nitems %d", nitems);
  if (nitems == 0 || (!pairs && !triples)) return CS_OK;
  if (!items) return fail(CS_ERR_INVALID, "cs_itemset_supports: items is NULL");
  cs_ctx* ctx = db->ctx;
  CS_CUDA(cudaSetDevice(ctx->device));
  const int n = nitems;
  std::vector<const uint32_t*> hp(n);
  for (int i = 0; i < n; ++i) {
    const int v = items[i];
    if (v < 0 || v >= db->n) return fail(CS_ERR_INVALID, "variable %d out of range for a database with n=%d", v, db->n);
    if (db->arity[v] < 2) return fail(CS_ERR_INVALID, "item %d has no state 1 (arity %d)", v, db->arity[v]);
    if (db->plane_off[v] < 0)
      return fail(CS_ERR_INVALID, "item %d has no bit planes; call cs_bitmap_build first", v);
    hp[i] = db->planes + db->plane_off[v] + db->words;  // state-1 plane
  }
  // rows: singles (a, a) -> pair supports, pairs (a, b) -> triple supports; sorted by b
  std::vector<ISRow> rows;
  rows.reserve((size_t)n * (n + 1) / 2);
  for (int b = 0; b < n; ++b) {
    rows.push_back(ISRow{(int16_t)b, (int16_t)b});
    for (int a = 0; a < b; ++a) rows.push_back(ISRow{(int16_t)a, (int16_t)b});
  }
  const int nrows = (int)rows.size();
  const int64_t W = db->words;  // multiple of 32 words
  const int64_t ntri = (int64_t)n * (n - 1) * (n - 2) / 6;
  const size_t bpairs = sizeof(uint64_t) * (size_t)n * n, btri = sizeof(uint64_t) * std::max<int64_t>(ntri, 1);
  // sparse data: count every itemset under its rarest item (K4d) when the cost model says so
  const int sel_mode = env_int("CS_ITEMSETS_SEL", -1);  // -1 auto, 0 never, 1 always (read per call)
  if (sel_mode != 0 && n <= SEL_MAXN && n >= 2) {
    const int rc = itemsets_selector(db, n, hp, pairs, triples, sel_mode);
    if (rc != 1) return rc;
  }
  static const int use_tc = env_int("CS_ITEMSETS_TC", 1);
  if (use_tc) {
    // tensor-core path (K4c, cs_itemsets.cuh).  Tiles = (128-row block, <= 256-column chunk
    // starting at the block's smallest b + 1).  The step axis is cut into windows whose planes
    // fit in L2 (~24 MB); inside a window the tiles' costs are laid end to end and cut into one
    // equal piece per CTA, so every SM works on the same window at the same time.
    const int64_t nsteps = W / 8;
    struct Tile {
      int row0, col0, ncols;
    };
    std::vector<Tile> tiles;
    for (int r0 = 0; r0 < nrows; r0 += 128)
      for (int c0 = rows[r0].b + 1; c0 < n; c0 += TC_NMAX)
        tiles.push_back(Tile{r0, c0, (int)std::min<int64_t>(TC_NMAX, round_up(n - c0, 16))});
    int maxN = 16;
    for (const Tile& t : tiles) maxN = std::max(maxN, t.ncols);
    // per row block: the items its rows touch (merged ranges) and each row's two raw slots
    const int nblocks = (nrows + 127) / 128;
    std::vector<TCSeg> segs(nblocks);
    std::vector<TCSlot> slots(nrows);
    for (int bk = 0; bk < nblocks; ++bk) {
      std::vector<int> it;
      for (int r = bk * 128; r < std::min(nrows, bk * 128 + 128); ++r) {
        it.push_back(rows[r].a);
        it.push_back(rows[r].b);
      }
      std::sort(it.begin(), it.end());
      it.erase(std::unique(it.begin(), it.end()), it.end());
      // contiguous copy ranges over the sorted items (one bulk copy per range per step): exact
      // runs, then the smallest gaps (< 64 items) merged while the copied span stays <= 256 slots
      // (gap items are copied and ignored)
      std::vector<std::pair<int, int>> rg;  // [lo, hi]
      for (size_t k = 0; k < it.size(); ++k) {
        if (k == 0 || it[k] != it[k - 1] + 1) rg.emplace_back(it[k], it[k]);
        rg.back().second = it[k];
      }
      int span = (int)it.size();
      for (;;) {
        int best = -1, gap = 64;
        for (size_t k = 0; k + 1 < rg.size(); ++k) {
          const int g2 = rg[k + 1].first - rg[k].second - 1;
          if (g2 < gap && span + g2 <= TC_RAWA / 32) gap = g2, best = (int)k;
        }
        if (best < 0) break;
        span += gap;
        rg[best].second = rg[best + 1].second;
        rg.erase(rg.begin() + best + 1);
      }
      TCSeg& sg = segs[bk];
      if ((int)rg.size() > TC_MAXSEG)
        return fail(CS_ERR_UNSUPPORTED, "itemsets: row block %d has %zu item ranges (max %d)", bk, rg.size(), TC_MAXSEG);
      sg.nseg = (int)rg.size();
      for (int k = 0, slot = 0; k < sg.nseg; ++k) {
        sg.src[k] = rg[k].first;
        sg.len[k] = rg[k].second - rg[k].first + 1;
        sg.dst[k] = slot;
        slot += sg.len[k];
      }
      if ((sg.dst[sg.nseg - 1] + sg.len[sg.nseg - 1]) * 32 > TC_RAWA)
        return fail(CS_ERR_UNSUPPORTED, "itemsets: row block %d spans too many items", bk);
      auto slot_of = [&](int item) {
        for (int k = 0; k < sg.nseg; ++k)
          if (item >= sg.src[k] && item < sg.src[k] + sg.len[k]) return sg.dst[k] + item - sg.src[k];
        return 0;
      };
      for (int r = bk * 128; r < std::min(nrows, bk * 128 + 128); ++r)
        slots[r] = TCSlot{(int16_t)slot_of(rows[r].a), (int16_t)slot_of(rows[r].b)};
    }
    // One launch per column-width class (N <= 64, <= 128, <= 256), each with stage geometry
    // sized for its widest tile: nb operand stages of maxN x 256 B (TMEM A stages packed right
    // after the accumulator's columns), released in commit groups of cpc stages (a commit costs
    // short MMAs ~200 issue cycles, tools/microbench6.cu), and a raw ring of nr slots of
    // (the blocks' item slots + maxN) x 32 B.
    const int smem_optin = ctx->smem_optin;
    static const int tc_dbg = env_int("CS_TC_DEBUG", 0);  // diagnostic: skip work per role (wrong results)
#ifdef CS_TC_PROFILE
    static const int tc_prof = env_int("CS_TC_PROF", 0);   // diagnostic: per-role wait cycles to stderr
#else
    const int tc_prof = 0;  // build with -DCS_TC_PROFILE for per-role wait cycles
#endif
    static const double costk = env_int("CS_TC_COSTK", 250);  // fixed per-step cost, in columns (measured)
    int maxslots = 1;
    for (const TCSeg& sg : segs) maxslots = std::max(maxslots, sg.dst[sg.nseg - 1] + sg.len[sg.nseg - 1]);
    const int budget = smem_optin - 2048, rawa_bytes = maxslots * 32;
    const int grid = ctx->num_sms;
    const double plane_bytes = 4.0 * (double)W * n;
    const int64_t nwin = std::max<int64_t>(1, std::min<int64_t>(nsteps / 64, (int64_t)(plane_bytes / 24e6)));
    struct Launch {
      size_t unit0;
      std::vector<int32_t> cta_off;
      int ga, nb, cpc, a_col, nr, stage_bytes, rawb_bytes, dyn_smem;
    };
    std::vector<TCUnit> all_units;
    std::vector<Launch> launches;
    static const int tc_classes = env_int("CS_TC_CLASSES", 1);
    static const int tc_cpc = env_int("CS_TC_CPC", 0);  // 0 = automatic
    static const int tc_only = env_int("CS_TC_ONLY", 0);
    static const int tc_sync = env_int("CS_TC_SYNC", 0);  // diagnostic: synchronize after each launch  // diagnostic: launch only class k (1..3)
    int lo = 0;
    for (const int hi : {64, 128, 256}) {
      if (!tc_classes && hi < 256) continue;
      if (tc_only && hi != (tc_only == 1 ? 64 : tc_only == 2 ? 128 : 256)) {
        lo = hi;
        continue;
      }
      std::vector<Tile> sub;
      int maxN = 16;
      for (const Tile& t : tiles)
        if (t.ncols > lo && t.ncols <= hi) {
          sub.push_back(t);
          maxN = std::max(maxN, t.ncols);
        }
      lo = hi;
      if (sub.empty()) continue;
      Launch L;
      L.a_col = (int)round_up(maxN, 64);
      L.stage_bytes = maxN * TC_KT;
      L.rawb_bytes = maxN * 32;
      const int raw_slot = rawa_bytes + L.rawb_bytes;
      int nb = std::min(TC_MAXNB, (512 - L.a_col) / 64);
      // nb >= the B group count; the A group count ga <= nb (parity waits on the stage ring stay
      // unambiguous when a group's previous step is at least nb steps back)
      while (nb > 2 && nb * L.stage_bytes + 6 * raw_slot > budget) --nb;
      if (nb >= 4) nb &= ~1;
      L.nb = nb;
      L.ga = std::min(TC_GA, nb >= 4 ? 4 : 2);  // divides nr (a multiple of 4): raw-slot parity waits stay unambiguous
      L.cpc = nb >= 4 ? nb / 2 : 1;
      if (tc_cpc) L.cpc = nb % tc_cpc == 0 ? tc_cpc : 1;
      // nr is a multiple of the loader count (4): raw slot s is then always refilled by the same
      // loader warp, in order, so its parity waits cannot alias a phase two cycles back (loaders
      // run independently; with nr % TC_LOADERS != 0 a fast loader could re-arm a slot early).
      // It is also a multiple of the A / B group counts, so a slot's consumers are always the
      // same groups, which have consumed its previous fill.
      L.nr = std::min(TC_MAXNR, (budget - nb * L.stage_bytes) / raw_slot) / TC_LOADERS * TC_LOADERS;
      if (L.nr < TC_LOADERS) return fail(CS_ERR_UNSUPPORTED, "itemsets: SMEM plan does not fit (N %d)", maxN);
      L.dyn_smem = nb * L.stage_bytes + L.nr * raw_slot;
      // step axis cut into L2-sized windows; inside a window the tiles' costs are laid end to
      // end and cut into one equal piece per CTA
      std::vector<std::vector<TCUnit>> per(grid);
      for (int64_t wi = 0; wi < nwin; ++wi) {
        const int64_t s0 = nsteps * wi / nwin, s1 = nsteps * (wi + 1) / nwin, len = s1 - s0;
        if (len <= 0) continue;
        double T = 0;
        for (const Tile& t : sub) T += (double)(t.ncols + costk) * len;
        double C = 0;
        for (const Tile& t : sub) {
          const double c = t.ncols + costk;
          auto cut = [&](int k) {  // step of this tile where CTA k's share begins
            const double B = T * k / grid;
            return (int64_t)std::min<double>((double)len, std::max(0.0, std::floor((B - C) / c + 0.5)));
          };
          for (int k = std::max(0, (int)std::floor(C * grid / T) - 1); k < grid; ++k) {
            const int64_t a = cut(k), b = cut(k + 1);
            if (a >= len) break;
            if (b > a)
              per[k].push_back(
                  TCUnit{t.row0, (int16_t)t.col0, (int16_t)t.ncols, (int32_t)(s0 + a), (int32_t)(s0 + b)});
          }
          C += c * len;
        }
      }
      L.unit0 = all_units.size();
      L.cta_off.assign(grid + 1, 0);
      for (int b = 0; b < grid; ++b) {
        for (const TCUnit& u : per[b]) all_units.push_back(u);
        L.cta_off[b + 1] = (int32_t)(all_units.size() - L.unit0);
      }
      launches.push_back(std::move(L));
    }
    const size_t bp = sizeof(void*) * n, br = sizeof(ISRow) * nrows, bsl = sizeof(TCSlot) * nrows,
                 bsg = sizeof(TCSeg) * nblocks, bu = sizeof(TCUnit) * std::max<size_t>(all_units.size(), 1),
                 bo = sizeof(int32_t) * (grid + 1) * std::max<size_t>(launches.size(), 1),
                 bpmt = (size_t)nsteps * n * 32;
    size_t off = 0;
    auto place = [&](size_t b) {
      size_t o = off;
      off = round_up(off + b, 256);
      return o;
    };
    const size_t op = place(bp), orr = place(br), osl = place(bsl), osg = place(bsg), ou = place(bu),
                 oo = place(bo), opr = place(bpairs), otr = place(btri), opm = place(bpmt), opf = place(1024);
    void* blob = nullptr;
    CS_TRY(ctx->scratch_get(10, off, &blob));
    char* d = (char*)blob;
    // one pinned upload of the plan tables
    const size_t meta = oo + bo;
    void* hst = nullptr;
    CS_TRY(ctx->pinned_get(meta, &hst));
    char* h = (char*)hst;
    memcpy(h + op, hp.data(), bp);
    memcpy(h + orr, rows.data(), br);
    memcpy(h + osl, slots.data(), bsl);
    memcpy(h + osg, segs.data(), bsg);
    if (!all_units.empty()) memcpy(h + ou, all_units.data(), sizeof(TCUnit) * all_units.size());
    for (size_t li = 0; li < launches.size(); ++li)
      memcpy(h + oo + sizeof(int32_t) * (grid + 1) * li, launches[li].cta_off.data(), sizeof(int32_t) * (grid + 1));
    CS_CUDA(cudaMemcpyAsync(d, h, meta, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaMemsetAsync(d + opr, 0, otr - opr + btri, ctx->stream));
    if (tc_prof) CS_CUDA(cudaMemsetAsync(d + opf, 0, 1024, ctx->stream));
    ctx->itemset_class = CS_ITEMSETS_TENSOR;
    CS_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    k_pmt_transpose<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>((const uint32_t* const*)(d + op), n, nsteps,
                                                              (uint4*)(d + opm));
    ctx->launches++;
    for (size_t li = 0; li < launches.size(); ++li) {
      const Launch& L = launches[li];
      k_itemsets_tc<<<grid, TC_THREADS, L.dyn_smem, ctx->stream>>>(
          (const uint4*)(d + opm), n, (const ISRow*)(d + orr), (const TCSlot*)(d + osl), nrows,
          (const TCSeg*)(d + osg), (const TCUnit*)(d + ou) + L.unit0,
          (const int32_t*)(d + oo) + (grid + 1) * li, L.ga, L.nb, L.cpc, L.a_col, L.nr, L.stage_bytes, rawa_bytes,
          L.rawb_bytes, (unsigned long long*)(d + opr), (unsigned long long*)(d + otr), tc_dbg,
          tc_prof ? (long long*)(d + opf) + 16 * li : nullptr);
      ctx->launches++;
      if (tc_sync) {
        const cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return fail(CS_ERR_CUDA, "itemsets launch %zu (N<=%d nb %d cpc %d nr %d): %s", li,
                                          L.stage_bytes / TC_KT, L.nb, L.cpc, L.nr, cudaGetErrorString(e));
      }
    }
    CS_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->ev_valid = true;
    CS_CUDA(cudaGetLastError());
    const cudaMemcpyKind kp = is_device_ptr(pairs) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const cudaMemcpyKind kt = is_device_ptr(triples) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (pairs) CS_CUDA(cudaMemcpyAsync(pairs, d + opr, bpairs, kp, ctx->stream));
    if (triples && ntri) CS_CUDA(cudaMemcpyAsync(triples, d + otr, sizeof(uint64_t) * ntri, kt, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (tc_prof) {
      long long pr[16 * 3];
      CS_CUDA(cudaMemcpy(pr, d + opf, sizeof(long long) * 16 * launches.size(), cudaMemcpyDeviceToHost));
      const double g = grid;
      for (size_t li = 0; li < launches.size(); ++li) {
        const long long* q = pr + 16 * li;
        const Launch& L = launches[li];
        fprintf(stderr,
                "[tc prof] launch %zu (N<=%d nb %d cpc %d nr %d units %d): per-CTA Mcycles total avg %.2f max %.2f | "
                "A wait raw %.2f empty %.2f dfull %.2f epi %.2f lds %.2f st %.2f | B wait raw %.2f empty %.2f | "
                "MMA wait full %.2f dempty %.2f issue %.2f | loader wait %.2f issue %.2f\n",
                li, L.stage_bytes / TC_KT, L.nb, L.cpc, L.nr, L.cta_off[grid], q[11] / g / 1e6, q[12] / 1e6,
                q[0] / g / 1e6, q[1] / g / 1e6, q[2] / g / 1e6, q[3] / g / 1e6, q[13] / g / 1e6, q[14] / g / 1e6,
                q[4] / g / 1e6, q[5] / g / 1e6,
                q[6] / g / 1e6, q[7] / g / 1e6, q[8] / g / 1e6, q[9] / g / 1e6, q[10] / g / 1e6);
      }
    }
    return CS_OK;
  }
  ctx->itemset_class = CS_ITEMSETS_BITGEMM;
  std::vector<std::pair<int, int>> tiles;
  for (int r0 = 0; r0 < nrows; r0 += IS_ROWS) {
    const int minb = rows[r0].b;
    // columns start right after the block's smallest b (unaligned): 1.25x computed/useful
    // outputs instead of 1.6x with 32-aligned column blocks
    for (int c0 = minb + 1; c0 < n; c0 += IS_COLS) tiles.emplace_back(r0, c0);
  }
  const int64_t target = 4LL * 2 * ctx->num_sms;
  int64_t S = std::max<int64_t>(1, (target + (int64_t)tiles.size() - 1) / std::max<int64_t>(1, tiles.size()));
  S = std::min<int64_t>(S, W / IS_TW);
  const int64_t slice = ((W / S + IS_TW - 1) / IS_TW) * IS_TW;
  std::vector<ISUnit> units;
  for (int64_t w0 = 0; w0 < W; w0 += slice)
    for (auto& t : tiles) units.push_back(ISUnit{t.first, t.second, w0, std::min(W, w0 + slice)});
  const size_t bp = sizeof(void*) * n, br = sizeof(ISRow) * nrows, bu = sizeof(ISUnit) * units.size();
  size_t off = 0;
  auto place = [&](size_t b) {
    size_t o = off;
    off = round_up(off + b, 256);
    return o;
  };
  const size_t op = place(bp), orr = place(br), ou = place(bu), oh = place(256), opr = place(bpairs),
               otr = place(btri);
  void* blob = nullptr;
  CS_TRY(ctx->scratch_get(10, off, &blob));
  char* d = (char*)blob;
  CS_CUDA(cudaMemcpyAsync(d + op, hp.data(), bp, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemcpyAsync(d + orr, rows.data(), br, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemcpyAsync(d + ou, units.data(), bu, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemsetAsync(d + oh, 0, 256, ctx->stream));
  CS_CUDA(cudaMemsetAsync(d + opr, 0, bpairs + (otr - opr - bpairs) + btri, ctx->stream));
  const int grid = (int)std::min<int64_t>((int64_t)units.size(), 2LL * ctx->num_sms);
  CS_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  k_itemsets<<<grid, IS_THREADS, 0, ctx->stream>>>((const uint32_t* const*)(d + op), (const ISRow*)(d + orr),
                                                   nrows, n, (const ISUnit*)(d + ou), (int)units.size(),
                                                   (int*)(d + oh), (unsigned long long*)(d + opr),
                                                   (unsigned long long*)(d + otr));
  CS_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->ev_valid = true;
  ctx->launches++;
  CS_CUDA(cudaGetLastError());
  const cudaMemcpyKind kp = is_device_ptr(pairs) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const cudaMemcpyKind kt = is_device_ptr(triples) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (pairs) CS_CUDA(cudaMemcpyAsync(pairs, d + opr, bpairs, kp, ctx->stream));
  if (triples && ntri) CS_CUDA(cudaMemcpyAsync(triples, d + otr, sizeof(uint64_t) * ntri, kt, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}
