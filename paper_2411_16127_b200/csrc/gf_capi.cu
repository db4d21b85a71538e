#include <atomic>
#include <cstring>
#include <thread>
#include <initializer_list>
#include <algorithm>
#include <mutex>
#include <cstdlib>
// C-ABI entry points of libgraphfuse_cuda (see include/gf_cuda.h).
#include <string>

#include "gf_internal.cuh"

namespace gfb {
namespace {
thread_local std::string t_err;
}
void set_error(const std::string& msg) { t_err = msg; }

namespace {
std::once_flag pool_once[64];
cudaMemPool_t pools[64];
}  // namespace

cudaError_t scratch_alloc_raw(void** p, size_t bytes, cudaStream_t s) {
  // Library-private stream-ordered pool per device: freed scratch stays
  // mapped for the next call (with a release threshold of 0 every
  // synchronisation returned it and the next call re-mapped it: +5.6 ms per
  // unfused AGNN backward on C3), without touching the device's default pool
  // that the host application (e.g. PyTorch) allocates from.
  // gf_scratch_trim() gives the cached bytes back.
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  std::call_once(pool_once[dev], [dev] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t keep = uint64_t(8) << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = pool;
    } else {
      cudaGetLastError();
    }
  });
  if (!pools[dev]) return cudaMallocAsync(p, bytes, s);
  return cudaMallocFromPoolAsync(p, bytes, pools[dev], s);
}

cudaMemPool_t scratch_pool(int dev) { return dev >= 0 && dev < 64 ? pools[dev] : nullptr; }
}  // namespace gfb


namespace gfb {
bool l2_prefetch_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GF_L2_PREFETCH");
    return !(e && *e == '0');
  }();
  return on;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GF_PDL");
    return !(e && *e == '0');
  }();
  return on;
}
}  // namespace gfb

extern "C" int gf_scratch_trim(void) {
  int dev = 0;
  GF_CHECK_CUDA(cudaGetDevice(&dev));
  if (cudaMemPool_t pool = gfb::scratch_pool(dev)) {
    GF_CHECK_CUDA(cudaDeviceSynchronize());
    GF_CHECK_CUDA(cudaMemPoolTrimTo(pool, 0));
  }
  return GF_OK;
}

extern "C" const char* gf_last_error(void) { return gfb::t_err.c_str(); }

extern "C" int gf_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return 0;
  return p.major == 10 && p.minor == 0;  // built for sm_100a only
}

// Device buffers of the host API layer come from the library's private
// stream-ordered pool on the legacy default stream (which orders them against
// every blocking stream): cudaMalloc / cudaFree per operator call cost
// milliseconds each (cudaFree synchronises the device) on the drop-in path.
extern "C" int gf_malloc(size_t bytes, void** out) {
  if (!out) {
    gfb::set_error("gf_malloc: null out");
    return GF_ERR_INVALID;
  }
  *out = nullptr;
  if (bytes == 0) return GF_OK;
  GF_CHECK_CUDA(gfb::scratch_alloc_raw(out, bytes, cudaStreamLegacy));
  return GF_OK;
}

extern "C" int gf_free(void* p) {
  if (p) GF_CHECK_CUDA(cudaFreeAsync(p, cudaStreamLegacy));
  return GF_OK;
}

namespace {
// Large copies between PAGEABLE host memory and the device (the drop-in C++
// API's std::vector operands, e.g. the E-length P of run_strategy) go through
// a persistent pinned staging ring: the DMA of chunk i overlaps the host
// memcpy of chunk i-1 (4 threads), instead of the driver's pageable path.
constexpr size_t kStageChunk = size_t(32) << 20;
constexpr size_t kStageMin = size_t(64) << 20;

struct Stage {
  std::mutex mu;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool ok = false;
  bool init() {
    if (ok) return true;
    for (int i = 0; i < 2; ++i)
      if (cudaHostAlloc(&buf[i], kStageChunk, cudaHostAllocDefault) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
    ok = true;
    return true;
  }
};

Stage& stage() {
  static Stage st;
  return st;
}

bool is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

void par_memcpy(void* dst, const void* src, size_t n) {
  constexpr int kThreads = 4;
  if (n < (size_t(4) << 20)) {
    std::memcpy(dst, src, n);
    return;
  }
  std::thread th[kThreads - 1];
  const size_t part = (n / kThreads + 63) / 64 * 64;
  for (int t = 1; t < kThreads; ++t) {
    const size_t b = std::min(n, part * t), e = std::min(n, part * (t + 1));
    th[t - 1] = std::thread([=] {
      if (e > b) std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
    });
  }
  std::memcpy(dst, src, std::min(n, part));
  for (auto& x : th) x.join();
}

int staged_copy(void* dst, const void* src, size_t bytes, bool d2h, cudaStream_t s) {
  Stage& st = stage();
  std::lock_guard<std::mutex> lock(st.mu);
  if (!st.init()) return -1;  // caller falls back to the plain copy
  const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
  auto len = [&](size_t i) { return std::min(kStageChunk, bytes - i * kStageChunk); };
  if (d2h) {
    for (size_t i = 0; i <= nch; ++i) {
      if (i < nch) {
        GF_CHECK_CUDA(cudaMemcpyAsync(st.buf[i % 2], static_cast<const char*>(src) + i * kStageChunk,
                                      len(i), cudaMemcpyDeviceToHost, s));
        GF_CHECK_CUDA(cudaEventRecord(st.ev[i % 2], s));
      }
      if (i > 0) {  // chunk i-1 landed: copy it out while chunk i is in flight
        GF_CHECK_CUDA(cudaEventSynchronize(st.ev[(i - 1) % 2]));
        par_memcpy(static_cast<char*>(dst) + (i - 1) * kStageChunk, st.buf[(i - 1) % 2], len(i - 1));
      }
    }
  } else {
    for (size_t i = 0; i < nch; ++i) {
      if (i >= 2) GF_CHECK_CUDA(cudaEventSynchronize(st.ev[i % 2]));  // buffer free again
      par_memcpy(st.buf[i % 2], static_cast<const char*>(src) + i * kStageChunk, len(i));
      GF_CHECK_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + i * kStageChunk, st.buf[i % 2], len(i),
                                    cudaMemcpyHostToDevice, s));
      GF_CHECK_CUDA(cudaEventRecord(st.ev[i % 2], s));
    }
    for (int b = 0; b < 2; ++b) GF_CHECK_CUDA(cudaEventSynchronize(st.ev[b]));
  }
  return GF_OK;
}
}  // namespace

extern "C" int gf_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream) {
  if (bytes == 0) return GF_OK;
  auto s = static_cast<cudaStream_t>(stream);
  if ((kind == 0 || kind == 1) && bytes >= kStageMin && is_pageable(kind == 0 ? src : dst)) {
    const int rc = staged_copy(dst, src, bytes, kind == 1, s);
    if (rc >= 0) return rc;
  }
  const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                           : kind == 1 ? cudaMemcpyDeviceToHost
                                       : cudaMemcpyDeviceToDevice;
  GF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, k, s));
  return GF_OK;
}

extern "C" int gf_memset(void* dst, int32_t value, size_t bytes, void* stream) {
  if (bytes == 0) return GF_OK;
  GF_CHECK_CUDA(cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream)));
  return GF_OK;
}

extern "C" int gf_stream_sync(void* stream) {
  GF_CHECK_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  GF_CHECK_CUDA(cudaGetLastError());
  return GF_OK;
}

namespace {

int check_desc(const gf_attn_desc* d, const char* who) {
  if (!d) {
    gfb::set_error(std::string(who) + ": null descriptor");
    return GF_ERR_INVALID;
  }
  if ((d->dtype != GF_F32 && d->dtype != GF_F64) || (d->variant != GF_DOT && d->variant != GF_ADD) ||
      d->heads < 1 || d->head_dim < 1 || (d->variant == GF_ADD && d->l2)) {
    gfb::set_error(std::string(who) + ": invalid descriptor (dtype/variant/heads/head_dim/l2)");
    return GF_ERR_INVALID;
  }
  if ((d->reserved & ~GF_FLAG_LOGITS_FROM_V) != 0 ||
      ((d->reserved & GF_FLAG_LOGITS_FROM_V) && d->variant != GF_ADD)) {
    gfb::set_error(std::string(who) + ": invalid descriptor flags (GF_FLAG_LOGITS_FROM_V needs GF_ADD)");
    return GF_ERR_INVALID;
  }
  return GF_OK;
}

// GF_FLAG_LOGITS_FROM_V resolution for one call: the fused fast kernels take
// a_l / a_r directly (kernel variant GF_ADDV); every other path gets el / er
// tables computed once (gf_gat_logits) into stream-ordered scratch and runs
// the table form.  Without the flag: pass-through.
struct Logits {
  int variant = GF_ADD;
  const void* Q = nullptr;
  const void* K = nullptr;
  void* tables = nullptr;
  cudaStream_t s = nullptr;
  Logits() = default;
  Logits(const Logits&) = delete;
  ~Logits() {
    if (tables) cudaFreeAsync(tables, s);
  }
};

int resolve_logits(const gf_graph_s* g, const gf_attn_desc& d, const void* Q, const void* K,
                   const void* V, bool fast_path, std::initializer_list<const void*> vec_ptrs,
                   cudaStream_t s, Logits& out) {
  out.variant = d.variant;
  out.Q = Q;
  out.K = K;
  out.s = s;
  if (!(d.reserved & GF_FLAG_LOGITS_FROM_V)) return GF_OK;
  const int elem = d.dtype == GF_F32 ? 4 : 8;
  const int64_t F = static_cast<int64_t>(d.heads) * d.head_dim;
  bool fast = fast_path && gfb::fast_shape(d.heads, d.head_dim, elem, g->e).ok &&
              static_cast<int64_t>(g->n) * F < (int64_t(1) << 31);
  for (const void* p : vec_ptrs) fast = fast && (reinterpret_cast<uintptr_t>(p) % 32) == 0;
  fast = fast && (reinterpret_cast<uintptr_t>(Q) % 32) == 0 && (reinterpret_cast<uintptr_t>(K) % 32) == 0;
  if (fast) {
    out.variant = gfb::GF_ADDV;
    return GF_OK;
  }
  const size_t nb = static_cast<size_t>(g->n) * d.heads * elem;
  GF_CHECK_CUDA(gfb::scratch_alloc_raw(&out.tables, 2 * nb + 64, s));
  char* el = static_cast<char*>(out.tables);
  char* er = el + (nb + 31) / 32 * 32;
  if (int rc = gf_gat_logits(d.dtype, g->n, d.heads, d.head_dim, V, Q, K, el, er, s)) return rc;
  out.Q = el;
  out.K = er;
  return GF_OK;
}

template <typename T>
gfb::FwdArgs<T> fwd_args(const gfb::DevGraph& g, const gf_attn_desc& d, const void* Q,
                         const void* K, const void* V, void* O, void* lse) {
  gfb::FwdArgs<T> a{};
  a.ptr = g.row_ptr;
  a.idx = g.col;
  a.order = g.row_order;
  a.sched = g.row_sched;
  a.n_small = g.n_small_rows;
  a.n_empty = g.n_empty_rows;
  a.e = g.e;
  a.n = g.active_rows();
  a.n_cta = g.n_cta_rows;
  a.cta_tab = g.row_cta;
  a.cta_blocks = g.row_cta_blocks;
  a.parts = g.row_parts;
  a.H = d.heads;
  a.D = d.head_dim;
  a.F = d.heads * d.head_dim;
  a.LPH = 1;
  a.l2 = d.l2;
  a.scale = static_cast<T>(d.scale);
  a.slope = static_cast<T>(d.slope);
  a.Q = static_cast<const T*>(Q);
  a.K = static_cast<const T*>(K);
  a.V = static_cast<const T*>(V);
  a.O = static_cast<T*>(O);
  a.stats = static_cast<T*>(lse);
  return a;
}

template <typename T>
int fwd_impl(gf_graph_t g, const gf_attn_desc& d, const void* Q, const void* K, const void* V,
             void* O, void* lse, void* P, cudaStream_t s) {
  Logits lg;  // P materialisation reads el / er tables
  if (int rc = resolve_logits(g, d, Q, K, V, P == nullptr, {V, O, lse}, s, lg)) return rc;
  auto a = fwd_args<T>(*g, d, lg.Q, lg.K, V, O, lse);
  int rc = gfb::launch_fwd<T>(*g, a, lg.variant, s);
  if (rc || !P) return rc;
  return gfb::launch_materialize_p<T>(*g, a, lg.variant, static_cast<T*>(P), s);
}

template <typename T>
int bwd_impl(gf_graph_t g, const gf_attn_desc& d, const void* Q, const void* K, const void* V,
             const void* O, void* stats, const void* dO, void* dQ, void* dK, void* dV, int passes,
             cudaStream_t s) {
  gfb::BwdArgs<T> a{};
  a.n = g->n;
  a.H = d.heads;
  a.D = d.head_dim;
  a.F = d.heads * d.head_dim;
  a.LPH = 1;
  a.l2 = d.l2;
  a.scale = static_cast<T>(d.scale);
  a.slope = static_cast<T>(d.slope);
  a.Q = static_cast<const T*>(Q);
  a.K = static_cast<const T*>(K);
  a.V = static_cast<const T*>(V);
  a.O = static_cast<const T*>(O);
  a.dO = static_cast<const T*>(dO);
  a.stats = static_cast<T*>(stats);
  a.dQ = static_cast<T*>(dQ);
  a.dK = static_cast<T*>(dK);
  a.dV = static_cast<T*>(dV);
  Logits lg;
  if (int rc = resolve_logits(g, d, Q, K, V, true, {V, O, dO, dV, dK, dQ, stats}, s, lg)) return rc;
  a.Q = static_cast<const T*>(lg.Q);
  a.K = static_cast<const T*>(lg.K);
  return gfb::launch_bwd<T>(*g, a, lg.variant, passes, s);
}

bool bad_graph(gf_graph_t g, const char* who) {
  if (g) return false;
  gfb::set_error(std::string(who) + ": null graph");
  return true;
}

}  // namespace

// L2 carve-out for the evict-last node tables (opt-in).  The kernels mark the
// gathered tables (V, Q|el, dO, K) L2::evict_last and the streamed ids
// evict_first; measured on B200, that priority only protects lines while a
// persisting-L2 set-aside exists (cudaLimitPersistingL2CacheSize; 0 by
// default).  With a 64 MiB set-aside C4 (gathered tables 67-90 MB) gains
// ~2-3 %; with tables far beyond L2 (C5) it is neutral
// (profiles/ab_r1_l2_persist.txt).  The set-aside is a device-wide limit, so
// the library never changes it on its own: a caller opts in with
// gf_l2_persist(bytes) (bench.py does) or GF_L2_SETASIDE=<MiB> in the
// environment, and gf_l2_persist(0) / gf_l2_reset_persisting() give the
// lines back.
static void ensure_l2_setaside() {
  static const long env = [] {
    const char* e = std::getenv("GF_L2_SETASIDE");
    return e && *e ? std::atol(e) : 0L;
  }();
  if (env <= 0) return;
  static std::atomic<uint32_t> applied{0};  // bit d: device d done
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) {
    cudaGetLastError();
    return;
  }
  if (applied.fetch_or(1u << dev) >> dev & 1u) return;
  gf_l2_persist(static_cast<size_t>(env) << 20);
}

extern "C" int gf_l2_persist(size_t bytes) {
  int dev = 0, max_persist = 0;
  GF_CHECK_CUDA(cudaFree(nullptr));  // the context calls below need a current context
  GF_CHECK_CUDA(cudaGetDevice(&dev));
  GF_CHECK_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  if (bytes == 0) GF_CHECK_CUDA(cudaCtxResetPersistingL2Cache());
  GF_CHECK_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                                   std::min(bytes, static_cast<size_t>(max_persist))));
  return GF_OK;
}

extern "C" int gf_l2_persist_get(size_t* bytes) {
  if (!bytes) {
    gfb::set_error("gf_l2_persist_get: null out");
    return GF_ERR_INVALID;
  }
  GF_CHECK_CUDA(cudaDeviceGetLimit(bytes, cudaLimitPersistingL2CacheSize));
  return GF_OK;
}

extern "C" int gf_l2_reset_persisting(void) {
  GF_CHECK_CUDA(cudaFree(nullptr));
  GF_CHECK_CUDA(cudaCtxResetPersistingL2Cache());
  return GF_OK;
}

extern "C" int gf_attn_fwd(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                           const void* V, void* O, void* stats, void* P, void* stream) {
  if (int rc = check_desc(desc, "gf_attn_fwd")) return rc;
  if (bad_graph(g, "gf_attn_fwd")) return GF_ERR_INVALID;
  if (g->n > 0 && (!Q || !K || !V || !O || !stats)) {
    gfb::set_error("gf_attn_fwd: null operand");
    return GF_ERR_INVALID;
  }
  ensure_l2_setaside();
  auto s = static_cast<cudaStream_t>(stream);
  return desc->dtype == GF_F32 ? fwd_impl<float>(g, *desc, Q, K, V, O, stats, P, s)
                               : fwd_impl<double>(g, *desc, Q, K, V, O, stats, P, s);
}

extern "C" int gf_attn_fwd_workspace(gf_graph_t g, const gf_attn_desc* desc, int32_t strategy,
                                     int32_t have_p, size_t* bytes) {
  if (int rc = check_desc(desc, "gf_attn_fwd_workspace")) return rc;
  if (bad_graph(g, "gf_attn_fwd_workspace")) return GF_ERR_INVALID;
  if (!bytes || strategy < GF_STRAT_SMMF || strategy > GF_STRAT_BASELINE) {
    gfb::set_error("gf_attn_fwd_workspace: invalid arguments");
    return GF_ERR_INVALID;
  }
  *bytes = gfb::strategy_workspace_bytes(*g, desc->heads, desc->dtype == GF_F32 ? 4 : 8, strategy,
                                         have_p != 0);
  return GF_OK;
}

extern "C" int gf_attn_fwd_strategy(gf_graph_t g, const gf_attn_desc* desc, int32_t strategy,
                                    const void* Q, const void* K, const void* V, void* O,
                                    void* stats, void* P, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (int rc = check_desc(desc, "gf_attn_fwd_strategy")) return rc;
  if (bad_graph(g, "gf_attn_fwd_strategy")) return GF_ERR_INVALID;
  if (strategy < GF_STRAT_SMMF || strategy > GF_STRAT_BASELINE) {
    gfb::set_error("gf_attn_fwd_strategy: unknown strategy");
    return GF_ERR_INVALID;
  }
  if (g->n > 0 && (!Q || !K || !V || !O || !stats)) {
    gfb::set_error("gf_attn_fwd_strategy: null operand");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  const int elem = desc->dtype == GF_F32 ? 4 : 8;
  const size_t need = gfb::strategy_workspace_bytes(*g, desc->heads, elem, strategy, P != nullptr);
  void* ws = workspace;
  bool own = false;
  if (need > 0 && !ws) {
    GF_CHECK_CUDA(gfb::scratch_alloc(&ws, need, s));
    own = true;
  } else if (need > workspace_bytes) {
    gfb::set_error("gf_attn_fwd_strategy: workspace too small (see gf_attn_fwd_workspace)");
    return GF_ERR_INVALID;
  }
  int rc;
  Logits lg;
  if ((rc = resolve_logits(g, *desc, Q, K, V, strategy == GF_STRAT_SMMF && !P, {V, O, stats}, s,
                           lg))) {
    if (own) cudaFreeAsync(ws, s);
    return rc;
  }
  if (desc->dtype == GF_F32)
    rc = gfb::launch_fwd_strategy<float>(*g, fwd_args<float>(*g, *desc, lg.Q, lg.K, V, O, stats),
                                         lg.variant, strategy, static_cast<float*>(P),
                                         static_cast<float*>(ws), s);
  else
    rc = gfb::launch_fwd_strategy<double>(*g, fwd_args<double>(*g, *desc, lg.Q, lg.K, V, O, stats),
                                          lg.variant, strategy, static_cast<double*>(P),
                                          static_cast<double*>(ws), s);
  if (own) cudaFreeAsync(ws, s);
  return rc;
}

extern "C" int gf_time_fwd_strategy(gf_graph_t g, const gf_attn_desc* desc, int32_t strategy,
                                    const void* Q, const void* K, const void* V, void* O,
                                    void* stats, int32_t reps, float* ms_out, void* stream) {
  if (!ms_out || reps < 1) {
    gfb::set_error("gf_time_fwd_strategy: invalid arguments");
    return GF_ERR_INVALID;
  }
  auto s = static_cast<cudaStream_t>(stream);
  size_t need = 0;
  if (int rc = gf_attn_fwd_workspace(g, desc, strategy, 0, &need)) return rc;
  void* ws = nullptr;
  if (need) GF_CHECK_CUDA(gfb::scratch_alloc(&ws, need, s));
  cudaEvent_t a = nullptr, b = nullptr;
  int rc = GF_OK;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) {
    gfb::set_error("gf_time_fwd_strategy: cudaEventCreate failed");
    rc = GF_ERR_CUDA;
  }
  if (!rc) rc = gf_attn_fwd_strategy(g, desc, strategy, Q, K, V, O, stats, nullptr, ws, need, stream);
  if (!rc && cudaEventRecord(a, s) != cudaSuccess) rc = GF_ERR_CUDA;
  for (int i = 0; i < reps && !rc; ++i)
    rc = gf_attn_fwd_strategy(g, desc, strategy, Q, K, V, O, stats, nullptr, ws, need, stream);
  if (!rc && cudaEventRecord(b, s) != cudaSuccess) rc = GF_ERR_CUDA;
  if (!rc && cudaEventSynchronize(b) != cudaSuccess) rc = GF_ERR_CUDA;
  float ms = 0.f;
  if (!rc && cudaEventElapsedTime(&ms, a, b) != cudaSuccess) rc = GF_ERR_CUDA;
  if (rc == GF_ERR_CUDA) gfb::set_error("gf_time_fwd_strategy: CUDA event failure");
  *ms_out = ms / reps;
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  if (ws) cudaFreeAsync(ws, s);
  return rc;
}

extern "C" int gf_attn_bwd(gf_graph_t g, const gf_attn_desc* desc, const void* Q, const void* K,
                           const void* V, const void* O, void* stats, const void* dO, void* dQ,
                           void* dK, void* dV, void* stream) {
  if (int rc = check_desc(desc, "gf_attn_bwd")) return rc;
  if (bad_graph(g, "gf_attn_bwd")) return GF_ERR_INVALID;
  if (g->n > 0 && (!Q || !K || !V || !O || !stats || !dO || !dQ || !dK || !dV)) {
    gfb::set_error("gf_attn_bwd: null operand");
    return GF_ERR_INVALID;
  }
  ensure_l2_setaside();
  auto s = static_cast<cudaStream_t>(stream);
  return desc->dtype == GF_F32
             ? bwd_impl<float>(g, *desc, Q, K, V, O, stats, dO, dQ, dK, dV, 3, s)
             : bwd_impl<double>(g, *desc, Q, K, V, O, stats, dO, dQ, dK, dV, 3, s);
}

extern "C" int gf_attn_bwd_rows(gf_graph_t g, const gf_attn_desc* desc, const void* Q,
                                const void* K, const void* V, const void* O, void* stats,
                                const void* dO, void* dK, void* stream) {
  if (int rc = check_desc(desc, "gf_attn_bwd_rows")) return rc;
  if (bad_graph(g, "gf_attn_bwd_rows")) return GF_ERR_INVALID;
  if (g->n > 0 && (!Q || !K || !V || !O || !stats || !dO || !dK)) {
    gfb::set_error("gf_attn_bwd_rows: null operand");
    return GF_ERR_INVALID;
  }
  ensure_l2_setaside();
  auto s = static_cast<cudaStream_t>(stream);
  return desc->dtype == GF_F32
             ? bwd_impl<float>(g, *desc, Q, K, V, O, stats, dO, nullptr, dK, nullptr, 1, s)
             : bwd_impl<double>(g, *desc, Q, K, V, O, stats, dO, nullptr, dK, nullptr, 1, s);
}

extern "C" int gf_attn_bwd_cols(gf_graph_t g, const gf_attn_desc* desc, const void* Q,
                                const void* K, const void* V, const void* stats, const void* dO,
                                void* dQ, void* dV, void* stream) {
  if (int rc = check_desc(desc, "gf_attn_bwd_cols")) return rc;
  if (bad_graph(g, "gf_attn_bwd_cols")) return GF_ERR_INVALID;
  if (g->n > 0 && (!Q || !K || !V || !stats || !dO || !dQ || !dV)) {
    gfb::set_error("gf_attn_bwd_cols: null operand");
    return GF_ERR_INVALID;
  }
  ensure_l2_setaside();
  auto s = static_cast<cudaStream_t>(stream);
  void* st = const_cast<void*>(stats);
  return desc->dtype == GF_F32
             ? bwd_impl<float>(g, *desc, Q, K, V, nullptr, st, dO, dQ, nullptr, dV, 2, s)
             : bwd_impl<double>(g, *desc, Q, K, V, nullptr, st, dO, dQ, nullptr, dV, 2, s);
}
