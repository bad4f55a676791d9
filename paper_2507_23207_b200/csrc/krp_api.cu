// krp_api.cu — the C ABI (include/krp.h): validation, workspace layout, launch
// sequencing of the sketch / CholeskyQR / TTM / truncation kernels, and the
// NCCL-based slab-sharded variants.  Every step of the path runs in this
// library's kernels; there is no host or CPU fallback.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstring>
#include <vector>

#include "krp_common.cuh"
#include "krp_internal.h"

namespace krp {

// ------------------------------------------------------------------ errors / counters
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }

// ---- kernel profiling
struct ProfRec {
  cudaEvent_t a, b;
  double bytes, flops;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;
static std::atomic<int> g_prof_on{0};
static cudaEvent_t g_prof_pending = nullptr;
bool prof_on() { return g_prof_on.load() != 0; }
void prof_begin(cudaStream_t s) {
  if (!prof_on()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEventCreate(&g_prof_pending);
  cudaEventRecord(g_prof_pending, s);
}
void prof_end(cudaStream_t s, double bytes, double flops) {
  if (!prof_on()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_pending) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, s);
  g_prof.push_back(ProfRec{g_prof_pending, b, bytes, flops});
  g_prof_pending = nullptr;
}

// ------------------------------------------------------------------ validation
static int validate_common(const void* X, int d, const int64_t* dims, int R) {
  if (!X || !dims) {
    set_error("null pointer argument");
    return KRP_EINVAL;
  }
  if (d < 2 || d > kMaxD) {
    set_error("d=%d not in [2,%d]", d, kMaxD);
    return KRP_EINVAL;
  }
  if (R < 1 || R > kMaxR) {
    set_error("R=%d not in [1,%d]", R, kMaxR);
    return KRP_EINVAL;
  }
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) {
      set_error("dims[%d]=%lld < 1", k, static_cast<long long>(dims[k]));
      return KRP_EINVAL;
    }
  return KRP_OK;
}

static int validate_ptrs(const float* const* p, int count, int skip, const char* what) {
  if (!p) {
    set_error("%s is NULL", what);
    return KRP_EINVAL;
  }
  for (int k = 0; k < count; ++k)
    if (k != skip && !p[k]) {
      set_error("%s[%d] is NULL", what, k);
      return KRP_EINVAL;
    }
  return KRP_OK;
}

// R must not exceed min(I_n, N/I_n) for the thin QR
static int validate_ranks(const Dims& g, const int* ranks, int R) {
  if (!ranks) {
    set_error("ranks is NULL");
    return KRP_EINVAL;
  }
  if (R > kMaxRDecomp) {  // reading R20: the decompositions take R <= 64
    set_error("rhosvd/sthosvd support R <= %d (got %d)", kMaxRDecomp, R);
    return KRP_EINVAL;
  }
  for (int k = 0; k < g.d; ++k) {
    if (ranks[k] < 1 || ranks[k] > R) {
      set_error("ranks[%d]=%d not in [1, R=%d]", k, ranks[k], R);
      return KRP_ESHAPE;
    }
    if (R > g.n[k] || R > g.N / g.n[k]) {
      set_error("R=%d > min(I_%d, N/I_%d) (SPEC S:329)", R, k + 1, k + 1);
      return KRP_ESHAPE;
    }
  }
  return KRP_OK;
}

// ------------------------------------------------------------------ workspace helpers
struct WsGuard {
  void* owned = nullptr;
  cudaStream_t s = nullptr;
  ~WsGuard() {
    if (owned) cudaFreeAsync(owned, s);
  }
};

static int setup_arena(size_t need, void* ws, size_t ws_bytes, cudaStream_t s, Arena& ar, WsGuard& guard) {
  if (ws == nullptr) {
    if (need > 0) {
      cudaError_t e = cudaMallocAsync(&guard.owned, need, s);
      if (e != cudaSuccess) {
        set_error("cudaMallocAsync(%zu) failed: %s", need, cudaGetErrorString(e));
        return KRP_ENOMEM;
      }
      guard.s = s;
    }
    ar.base = static_cast<char*>(guard.owned);
    ar.cap = need;
  } else {
    if (ws_bytes < need) {
      set_error("workspace too small: %zu < %zu bytes", ws_bytes, need);
      return KRP_ENOMEM;
    }
    if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) {
      set_error("workspace must be 256-byte aligned");
      return KRP_EINVAL;
    }
    ar.base = static_cast<char*>(ws);
    ar.cap = ws_bytes;
  }
  ar.off = 0;
  return KRP_OK;
}

static OmegaPtrs make_om(const float* const* omega, int d, int skip) {
  OmegaPtrs om{};
  for (int k = 0; k < d; ++k) om.p[k] = (k == skip) ? nullptr : omega[k];
  return om;
}

// ------------------------------------------------------------------ rHOSVD building blocks
// Sizes of the TTM chain X x_1 A_1 x_2 ... (ascending modes): returns the largest intermediate.
static int64_t chain_max(const Dims& g, const int* newdims) {
  int64_t cur = g.N, mx = 0;
  for (int k = 0; k < g.d; ++k) {
    cur = cur / g.n[k] * newdims[k];
    mx = std::max(mx, cur);
  }
  return mx;
}

// Y = X x_1 A_1 ... x_d A_d with A_k = Qt_k (J_k x I_k, row stride sj, col stride si); ping-pong bufs.
struct TtmOp {
  const float* A;
  int J;
  int64_t sj, si;
};
static int ttm_chain(const float* X, Dims g, const TtmOp* ops, float* bufA, float* bufB, float* out,
                     cudaStream_t s, Arena* ar = nullptr) {
  const float* src = X;
  int last = -1;
  for (int k = 0; k < g.d; ++k)
    if (ops[k].A) last = k;
  if (last < 0) {
    KRP_CHECK_CUDA(cudaMemcpyAsync(out, X, g.N * sizeof(float), cudaMemcpyDeviceToDevice, s));
    return KRP_OK;
  }
  bool use_a = true;
  int k_begin = 0;
  // modes 1 and 2 both contracted on the tensor cores: the first product is written mode-permuted,
  // (I_2, J_1, I_3..), so the second is again a mode-0 product, written permuted back to (J_1, J_2, I_3..)
  if (ar && g.d >= 2 && ops[0].A && ops[1].A && last >= 1 && g.n[1] % 4 == 0 && ops[1].J <= 64 &&
      ttm0_tc_ok(X, g.n[0], g.N / g.n[0], ops[0].J) &&
      (ar->cap - ar->off) >= std::max(ttm0_tc_ws_bytes(g.n[0], ops[0].J), ttm0_tc_ws_bytes(g.n[1], ops[1].J))) {
    const int64_t rest = g.N / (g.n[0] * g.n[1]);
    float* t1 = bufA;
    KRP_TRY(ttm0_tc(X, g.n[0], g.N / g.n[0], ops[0].A, ops[0].J, ops[0].sj, ops[0].si, t1, *ar, s, g.n[1]));
    float* t2 = (last == 1) ? out : bufB;
    KRP_TRY(ttm0_tc(t1, g.n[1], static_cast<int64_t>(ops[0].J) * rest, ops[1].A, ops[1].J, ops[1].sj, ops[1].si, t2,
                    *ar, s, ops[0].J));
    int64_t nd[kMaxD];
    for (int m = 0; m < g.d; ++m) nd[m] = g.n[m];
    nd[0] = ops[0].J;
    nd[1] = ops[1].J;
    g = make_dims(g.d, nd);
    src = t2;
    use_a = true;
    k_begin = 2;
    if (last == 1) return KRP_OK;
  }
  for (int k = k_begin; k < g.d; ++k) {
    if (!ops[k].A) continue;
    float* dst = (k == last) ? out : (use_a ? bufA : bufB);
    KRP_TRY(ttm(src, g, k, ops[k].A, ops[k].J, ops[k].sj, ops[k].si, dst, s, ar));
    int64_t nd[kMaxD];
    for (int m = 0; m < g.d; ++m) nd[m] = g.n[m];
    nd[k] = ops[k].J;
    g = make_dims(g.d, nd);
    src = dst;
    use_a = !use_a;
  }
  return KRP_OK;
}

// Orchestrates RHOSVD for a (possibly sharded) tensor.  When comm != nullptr, the local core and
// the error sums are all-reduced across ranks (slab sharding along the last mode; Y is global).
struct DistCtx;
// Per-device side streams for independent per-mode work (the d CholeskyQR2 factorisations of rHOSVD):
// forked from and joined back into the caller's stream with events, so the caller sees one ordered
// stream (and a captured graph gets parallel branches).  The fork / join events are shared, so a caller
// holds the per-device lock from the fork record until its stream has waited on every join event
// (concurrent rhosvd calls from several host threads on one device serialise only that enqueue section).
struct SideStreams {
  cudaStream_t st[kMaxD];
  cudaEvent_t fork, join[kMaxD];
  bool ok = false;
};
static std::mutex g_side_mu[64];
static int side_streams(SideStreams** out, std::unique_lock<std::mutex>& lk) {
  static SideStreams per_dev[64];
  int dev = 0;
  KRP_CHECK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("device ordinal %d out of range", dev);
    return KRP_EINVAL;
  }
  lk = std::unique_lock<std::mutex>(g_side_mu[dev]);
  SideStreams& ss = per_dev[dev];
  if (!ss.ok) {
    for (int k = 0; k < kMaxD; ++k) {
      KRP_CHECK_CUDA(cudaStreamCreateWithFlags(&ss.st[k], cudaStreamNonBlocking));
      KRP_CHECK_CUDA(cudaEventCreateWithFlags(&ss.join[k], cudaEventDisableTiming));
    }
    KRP_CHECK_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    ss.ok = true;
  }
  *out = &ss;
  return KRP_OK;
}

static int allreduce_sum_f32(DistCtx* c, float* buf, size_t count, cudaStream_t s);
static int allreduce_sum_f64(DistCtx* c, double* buf, size_t count, cudaStream_t s);

// Which sketch feeds the decomposition (NEXT-2): the memoized KRP sketch (one shared set), Alg. 7
// read literally (a fresh KRP sequence per mode, steps[n*d + j]), or the dense-Gaussian baseline (Table 1:
// dense[n] is (N/I_n) x R, or for STHOSVD the step's (N_i/I_i) x R).  Single-GPU only for the latter two.
struct SketchVariant {
  int kind = 0;  // 0 memoized KRP, 1 fresh KRP per mode, 2 dense Gaussian
  const float* const* steps = nullptr;
  const float* const* dense = nullptr;
};

static int rhosvd_impl(const float* X, const Dims& g /*local*/, int64_t Id_global, int64_t slab_begin,
                       const int* ranks, int R, const float* const* omega, float* const* Q, float* core,
                       double* rel_err, Arena& ar, cudaStream_t s, DistCtx* dc, bool measure_only,
                       const SketchVariant* sv = nullptr);

}  // namespace krp

using namespace krp;

// ================================================================== distributed context (NCCL via dlopen)
namespace krp {
typedef struct {
  char internal[128];
} nccl_uid_t;
typedef void* nccl_comm_t;
typedef int (*fn_get_uid)(nccl_uid_t*);
typedef int (*fn_init_rank)(nccl_comm_t*, int, nccl_uid_t, int);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_destroy)(nccl_comm_t);
typedef const char* (*fn_errstr)(int);
struct NcclApi {
  void* h = nullptr;
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_allreduce allreduce = nullptr;
  fn_destroy destroy = nullptr;
  fn_errstr errstr = nullptr;
};
static NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (api.h) {
      api.get_uid = reinterpret_cast<fn_get_uid>(dlsym(api.h, "ncclGetUniqueId"));
      api.init_rank = reinterpret_cast<fn_init_rank>(dlsym(api.h, "ncclCommInitRank"));
      api.allreduce = reinterpret_cast<fn_allreduce>(dlsym(api.h, "ncclAllReduce"));
      api.destroy = reinterpret_cast<fn_destroy>(dlsym(api.h, "ncclCommDestroy"));
      api.errstr = reinterpret_cast<fn_errstr>(dlsym(api.h, "ncclGetErrorString"));
    }
  }
  if (!api.h || !api.get_uid || !api.init_rank || !api.allreduce || !api.destroy) return nullptr;
  return &api;
}
struct DistCtx {
  nccl_comm_t comm = nullptr;
  int nranks = 1, rank = 0;
};
enum { kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0 };
static int allreduce_sum_f32(DistCtx* c, float* buf, size_t count, cudaStream_t s) {
  if (!c || c->nranks == 1 || count == 0) return KRP_OK;
  NcclApi* api = nccl();
  int r = api->allreduce(buf, buf, count, kNcclFloat32, kNcclSum, c->comm, s);
  if (r != 0) {
    set_error("ncclAllReduce failed: %s", api->errstr ? api->errstr(r) : "?");
    return KRP_ENCCL;
  }
  return KRP_OK;
}
static int allreduce_sum_f64(DistCtx* c, double* buf, size_t count, cudaStream_t s) {
  if (!c || c->nranks == 1 || count == 0) return KRP_OK;
  NcclApi* api = nccl();
  int r = api->allreduce(buf, buf, count, kNcclFloat64, kNcclSum, c->comm, s);
  if (r != 0) {
    set_error("ncclAllReduce failed: %s", api->errstr ? api->errstr(r) : "?");
    return KRP_ENCCL;
  }
  return KRP_OK;
}
}  // namespace krp

struct krp_comm_s {
  krp::DistCtx ctx;
};

// ================================================================== rHOSVD implementation
namespace krp {

static int rhosvd_impl(const float* X, const Dims& g, int64_t Id_global, int64_t slab_begin, const int* ranks, int R,
                       const float* const* omega, float* const* Q, float* core, double* rel_err, Arena& ar,
                       cudaStream_t s, DistCtx* dc, bool measure_only, const SketchVariant* sv) {
  const int d = g.d;
  const int kind = sv ? sv->kind : 0;
  const bool dist = dc != nullptr;
  int64_t gd[kMaxD];  // global dims
  for (int k = 0; k < d; ++k) gd[k] = g.n[k];
  gd[d - 1] = Id_global;
  const Dims gg = make_dims(d, gd);

  // ---- buffers
  float* Ybuf[kMaxD];
  float* Qfull[kMaxD];
  int64_t ysum = 0;
  for (int k = 0; k < d; ++k) ysum += gd[k] * R;
  float* Ypack = ar.take<float>(ysum);  // packed [Y_1 .. Y_d] (global sizes): one all-reduce
  {
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
      Ybuf[k] = measure_only ? nullptr : Ypack + off;
      off += gd[k] * R;
    }
  }
  for (int k = 0; k < d; ++k) Qfull[k] = ar.take<float>(gd[k] * R);
  int* flag = ar.take<int>(kMaxD);  // one CholeskyQR status word per mode (the chains run concurrently)
  double* errsum = ar.take<double>(2);
  const int64_t coreR = [&] {
    int64_t c = 1;
    for (int k = 0; k < d; ++k) c *= R;
    return c;
  }();
  float* G0 = ar.take<float>(coreR);  // R^d core
  float* G1 = ar.take<float>(coreR);
  double* H = ar.take<double>(static_cast<size_t>(d) * R * R);  // one Gram per mode (HOSVD of the core)
  float* U = ar.take<float>(static_cast<size_t>(d) * R * R);
  int rdims_all[kMaxD];
  for (int k = 0; k < d; ++k) rdims_all[k] = R;
  const int64_t cmax = chain_max(g, rdims_all);
  float* CA = ar.take<float>(cmax);
  float* CB = ar.take<float>(cmax);
  // the local Y_d rows live inside the packed global buffer at the slab offset
  // scratch for the sketch / QR / gram / error (max of all)
  bool want[kMaxD];
  for (int k = 0; k < d; ++k) want[k] = true;
  size_t scratch = kind == 0 ? sketch_ws_bytes(g, R, want) : 0;
  for (int k = 0; k < d && kind != 0; ++k) {  // per-mode sketches of the variants
    bool w1[kMaxD] = {};
    w1[k] = true;
    scratch = std::max(scratch, kind == 1 ? sketch_ws_bytes(g, R, w1) : gaussian_sketch_ws_bytes(g, k));
  }
  {  // the d CholeskyQR2 run concurrently: disjoint scratch per mode
    size_t qr = 0;
    for (int k = 0; k < d; ++k) qr += cholqr_ws_bytes(gd[k], R);
    scratch = std::max(scratch, qr);
  }
  {
    int64_t cd[kMaxD];
    for (int k = 0; k < d; ++k) cd[k] = R;
    Dims cg = make_dims(d, cd);
    for (int k = 0; k < d; ++k) scratch = std::max(scratch, mode_gram_ws_bytes(cg, k));
  }
  // the first two core contractions on the tensor cores (ttm_chain)
  scratch = std::max(scratch, std::max(ttm_ws_bytes(g, 0, R), ttm0_tc_ws_bytes(g.n[1], R)));
  // error pass buffers: slab chunks of the last mode
  const int64_t inner = g.N / g.n[d - 1];
  int64_t chunk = std::max<int64_t>(1, (int64_t(1) << 25) / std::max<int64_t>(inner, 1));
  chunk = std::min<int64_t>(chunk, g.n[d - 1]);
  float* EA = nullptr;
  float* EB = nullptr;
  float* Xh = nullptr;
  if (rel_err) {
    int64_t ed[kMaxD];
    for (int k = 0; k < d; ++k) ed[k] = ranks[k];
    ed[d - 1] = chunk;
    // expansion chain from (r_1..r_{d-1}, chunk) up to (I_1..I_{d-1}, chunk)
    int64_t mx = 0, cur = 1;
    for (int k = 0; k < d; ++k) cur *= ed[k];
    mx = cur;
    for (int k = d - 2; k >= 0; --k) {
      cur = cur / ed[k] * g.n[k];
      mx = std::max(mx, cur);
    }
    EA = ar.take<float>(mx);
    EB = ar.take<float>(mx);
    Xh = ar.take<float>(inner * chunk);
    scratch = std::max(scratch, sqdiff_ws_bytes(inner * chunk));
  }
  const size_t scratch_mark = ar.off;
  ar.take<char>(scratch);
  if (measure_only) return KRP_OK;
  if (ar.overflow()) {
    set_error("workspace too small for rhosvd");
    return KRP_ENOMEM;
  }
  ar.off = scratch_mark;

  KRP_CHECK_CUDA(cudaMemsetAsync(flag, 0, kMaxD * sizeof(int), s));
  // ---- 1. memoized all-mode sketch of the local slab (Alg. 7 line 3 with memoization)
  OmegaPtrs om{};
  if (kind == 0) {
    om = make_om(omega, d, -1);
    if (dist) om.p[d - 1] = omega[d - 1] + slab_begin * R;  // local rows of the global Omega_d
  }
  float* Yloc[kMaxD];
  for (int k = 0; k < d; ++k) Yloc[k] = Ybuf[k];
  if (dist) {
    Yloc[d - 1] = Ybuf[d - 1] + slab_begin * R;
    KRP_CHECK_CUDA(cudaMemsetAsync(Ypack, 0, ysum * sizeof(float), s));
  }
  if (kind == 0) {
    KRP_TRY(sketch(X, g, om, R, want, Yloc, ar, s));
  } else {
    for (int n = 0; n < d; ++n) {
      if (kind == 1) {  // Alg. 7 line 3 with this mode's own fresh sequence
        OmegaPtrs on{};
        for (int j = 0; j < d; ++j) on.p[j] = (j == n) ? nullptr : sv->steps[n * d + j];
        bool w1[kMaxD] = {};
        w1[n] = true;
        float* Y1[kMaxD] = {};
        Y1[n] = Yloc[n];
        KRP_TRY(sketch(X, g, on, R, w1, Y1, ar, s));
      } else {  // the dense-Gaussian baseline (Table 1)
        KRP_TRY(gaussian_sketch_mode(X, g, n, sv->dense[n], R, Yloc[n], ar, s));
      }
      ar.off = scratch_mark;
    }
  }
  ar.off = scratch_mark;
  // ---- multi-GPU: one all-reduce(sum) of the packed sketches (the zero-padded Y_d doubles as the gather)
  if (dist) KRP_TRY(allreduce_sum_f32(dc, Ypack, static_cast<size_t>(ysum), s));
  // ---- 2. thin QR of every Y_n, replicated; the d factorisations are independent and run on
  //      side streams (each is a chain of small latency-bound kernels)
  {
    SideStreams* ss = nullptr;
    std::unique_lock<std::mutex> side_lock;  // held until s has waited on every join event
    KRP_TRY(side_streams(&ss, side_lock));
    KRP_CHECK_CUDA(cudaEventRecord(ss->fork, s));
    size_t off = scratch_mark;
    for (int k = 0; k < d; ++k) {
      KRP_CHECK_CUDA(cudaStreamWaitEvent(ss->st[k], ss->fork, 0));
      ar.off = off;
      KRP_TRY(cholqr(Ybuf[k], gd[k], R, Qfull[k], nullptr, flag + k, ar, ss->st[k]));
      off += cholqr_ws_bytes(gd[k], R);
      KRP_CHECK_CUDA(cudaEventRecord(ss->join[k], ss->st[k]));
      KRP_CHECK_CUDA(cudaStreamWaitEvent(s, ss->join[k], 0));
    }
    ar.off = scratch_mark;
  }
  // ---- 3. core G = X x_1 Q_1^T ... x_d Q_d^T on the local slab, then all-reduce
  TtmOp ops[kMaxD];
  for (int k = 0; k < d; ++k) ops[k] = TtmOp{Qfull[k], R, 1, R};  // A = Q^T: (j,i) at Q[i*R + j]
  if (dist) ops[d - 1].A = Qfull[d - 1] + slab_begin * R;
  KRP_TRY(ttm_chain(X, g, ops, CA, CB, G0, s, &ar));
  if (dist) KRP_TRY(allreduce_sum_f32(dc, G0, static_cast<size_t>(coreR), s));
  // ---- 4. truncation R -> r_n by HOSVD of the small core (reading R4): every U_n comes from the
  //      untruncated core G0, so the d Gram matrices and eigenproblems are independent (one batched
  //      eigensolver launch); then G = G0 x_1 U_1^T ... x_d U_d^T and Q_n <- Qfull_n U_n
  int64_t cd[kMaxD];
  for (int k = 0; k < d; ++k) cd[k] = R;
  const Dims c0g = make_dims(d, cd);
  const double* Hk[kMaxD];
  float* Uk[kMaxD];
  int rk[kMaxD];
  int neig = 0;
  for (int k = 0; k < d; ++k) {
    if (ranks[k] < R) {
      double* Hm = H + static_cast<size_t>(k) * R * R;
      KRP_TRY(mode_gram(G0, c0g, k, Hm, ar, s));
      ar.off = scratch_mark;
      Hk[neig] = Hm;
      Uk[neig] = U + static_cast<size_t>(k) * R * R;
      rk[neig] = ranks[k];
      ++neig;
    }
  }
  if (neig > 0) KRP_TRY(sym_eig_top_batched(Hk, neig, R, rk, Uk, s));
  float* Gc = G0;
  float* Gn = G1;
  for (int k = 0; k < d; ++k) {
    const Dims cg = make_dims(d, cd);
    if (ranks[k] < R) {
      const float* Um = U + static_cast<size_t>(k) * R * R;
      // Q_k <- Qfull_k U  (Qfull as dims (R, I_k): mode-0 TTM with A = U^T, (j,i) at U[i*r + j])
      int64_t qd[2] = {R, gd[k]};
      KRP_TRY(ttm(Qfull[k], make_dims(2, qd), 0, Um, ranks[k], 1, ranks[k], Q[k], s));
      // G <- G x_k U^T
      KRP_TRY(ttm(Gc, cg, k, Um, ranks[k], 1, ranks[k], Gn, s));
      std::swap(Gc, Gn);
      cd[k] = ranks[k];
    } else {
      KRP_CHECK_CUDA(cudaMemcpyAsync(Q[k], Qfull[k], gd[k] * R * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }
  }
  int64_t csz = 1;
  for (int k = 0; k < d; ++k) csz *= cd[k];
  KRP_CHECK_CUDA(cudaMemcpyAsync(core, Gc, csz * sizeof(float), cudaMemcpyDeviceToDevice, s));
  // ---- 5. optional relative error ||X - X̂|| / ||X||, reconstructed slab chunk by chunk
  if (rel_err) {
    KRP_CHECK_CUDA(cudaMemsetAsync(errsum, 0, 2 * sizeof(double), s));
    for (int64_t k0 = 0; k0 < g.n[d - 1]; k0 += chunk) {
      const int64_t k1 = std::min<int64_t>(g.n[d - 1], k0 + chunk);
      // T = core x_d Q_d[rows]  (core dims cd; A = Q_d rows: (j, i) at Q[(j)*r + i])
      const float* qd_rows = Q[d - 1] + (slab_begin + k0) * ranks[d - 1];
      const Dims c0 = make_dims(d, cd);
      KRP_TRY(ttm(core, c0, d - 1, qd_rows, static_cast<int>(k1 - k0), ranks[d - 1], 1, EA, s));
      int64_t ed[kMaxD];
      for (int m = 0; m < d; ++m) ed[m] = cd[m];
      ed[d - 1] = k1 - k0;
      float* src = EA;
      for (int m = d - 2; m >= 0; --m) {
        float* o = (m == 0) ? Xh : (src == EA ? EB : EA);
        KRP_TRY(ttm(src, make_dims(d, ed), m, Q[m], static_cast<int>(g.n[m]), ranks[m], 1, o, s));
        ed[m] = g.n[m];
        src = o;
      }
      KRP_TRY(sqdiff_accumulate(X + k0 * inner, Xh, (k1 - k0) * inner, errsum, ar, s));
      ar.off = scratch_mark;
    }
    if (dist) KRP_TRY(allreduce_sum_f64(dc, errsum, 2, s));
  }
  // ---- status
  int hflag[kMaxD] = {};
  double herr[2] = {0.0, 0.0};
  KRP_CHECK_CUDA(cudaMemcpyAsync(hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, s));
  if (rel_err) KRP_CHECK_CUDA(cudaMemcpyAsync(herr, errsum, sizeof(herr), cudaMemcpyDeviceToHost, s));
  KRP_CHECK_CUDA(cudaStreamSynchronize(s));
  int fl = 0;
  for (int k = 0; k < d; ++k) fl |= hflag[k];
  if (fl & 2) {
    set_error("CholeskyQR breakdown (shifted fallback failed)");
    return KRP_ENUMERIC;
  }
  if (rel_err) *rel_err = herr[1] > 0 ? sqrt(herr[0] / herr[1]) : 0.0;
  return KRP_OK;
}

// ================================================================== STHOSVD
// RSTHOSVD-KRP (Alg. 8) on a (possibly slab-sharded) tensor.  g = local dims (the last mode is the
// local slab [slab_begin, slab_begin + g.n[d-1]) of Id_global rows); dc != nullptr combines across ranks
// (SURVEY §8(e)): steps i < d-1 keep the slab layout — their sketch and the mode Gram of B_(i) are sums over
// slabs (all-reduce) and the TTMs are local; the last step sketches complete rows of Y_d, gathered by the
// zero-padded all-reduce, contracts the sharded mode locally and all-reduces the (small) partial core.
static int sthosvd_impl(const float* X, const Dims& g, int64_t Id_global, int64_t slab_begin, const int* ranks, int R,
                        const float* const* omega, float* const* Q, float* core, double* rel_err, Arena& ar,
                        cudaStream_t s, DistCtx* dc, bool measure_only, const float* const* dense = nullptr) {
  const int d = g.d;
  const bool dist = dc != nullptr;
  int64_t gd[kMaxD];  // global dims
  for (int k = 0; k < d; ++k) gd[k] = g.n[k];
  gd[d - 1] = Id_global;
  int64_t imax = 0;
  for (int k = 0; k < d; ++k) imax = std::max(imax, gd[k]);
  float* Y = ar.take<float>(imax * R);
  float* Qf = ar.take<float>(imax * R);
  double* H = ar.take<double>(static_cast<size_t>(R) * R);
  float* U = ar.take<float>(static_cast<size_t>(R) * R);
  int* flag = ar.take<int>(4);
  double* errsum = ar.take<double>(2);
  // step buffers: B_i = G x_i Q^T has dims (r_<i, R, I_>i); G_i has (r_<=i, I_>i)  (local last mode)
  int64_t bmax = 0;
  for (int i = 0; i < d; ++i) {
    int64_t b = 1;
    for (int k = 0; k < d; ++k) b *= (k < i) ? ranks[k] : (k == i ? R : g.n[k]);
    bmax = std::max(bmax, b);
  }
  float* B = ar.take<float>(bmax);
  float* GA = ar.take<float>(bmax);
  size_t scratch = 0;
  {
    int64_t cur[kMaxD];
    for (int k = 0; k < d; ++k) cur[k] = g.n[k];
    for (int i = 0; i < d; ++i) {
      const Dims cg = make_dims(d, cur);
      bool want[kMaxD] = {};
      want[i] = true;
      scratch = std::max(scratch, dense ? gaussian_sketch_ws_bytes(cg, i) : sketch_ws_bytes(cg, R, want));
      scratch = std::max(scratch, cholqr_ws_bytes(gd[i], R));
      scratch = std::max(scratch, ttm_ws_bytes(cg, i, R));
      if (i == 0)  // the fused first step: B = X x_1 Q^T with its mode-1 Gram partials (4 per CTA)
        scratch = std::max(scratch, ttm_ws_bytes(cg, 0, R) +
                                        align_up(static_cast<size_t>(4 * 148) * R * R * sizeof(double), 256));
      cur[i] = R;
      scratch = std::max(scratch, mode_gram_ws_bytes(make_dims(d, cur), i));
      cur[i] = ranks[i];
    }
  }
  // error pass (full reconstruction of the local slab, chunked over the last mode) reuses B/GA-sized buffers
  const int64_t inner = g.N / g.n[d - 1];
  int64_t chunk = std::max<int64_t>(1, (int64_t(1) << 25) / std::max<int64_t>(inner, 1));
  chunk = std::min<int64_t>(chunk, g.n[d - 1]);
  float *EA = nullptr, *EB = nullptr, *Xh = nullptr;
  if (rel_err) {
    int64_t mx = 1, cur = 1;
    for (int k = 0; k < d - 1; ++k) cur *= ranks[k];
    cur *= chunk;
    mx = cur;
    for (int k = d - 2; k >= 0; --k) {
      cur = cur / ranks[k] * g.n[k];
      mx = std::max(mx, cur);
    }
    EA = ar.take<float>(mx);
    EB = ar.take<float>(mx);
    Xh = ar.take<float>(inner * chunk);
    scratch = std::max(scratch, sqdiff_ws_bytes(inner * chunk));
  }
  const size_t mark = ar.off;
  ar.take<char>(scratch);
  if (measure_only) return KRP_OK;
  if (ar.overflow()) {
    set_error("workspace too small for sthosvd");
    return KRP_ENOMEM;
  }
  ar.off = mark;
  KRP_CHECK_CUDA(cudaMemsetAsync(flag, 0, 4 * sizeof(int), s));

  int64_t cur[kMaxD];
  for (int k = 0; k < d; ++k) cur[k] = g.n[k];
  const float* G = X;
  for (int i = 0; i < d; ++i) {
    const bool last = i == d - 1;
    const Dims cg = make_dims(d, cur);
    // 1. Y_i = G_(i) (⊙_{j != i} Omega^{(i)}_j), compressed modes read only their leading r_j rows; the
    //    sharded mode reads its slab rows
    OmegaPtrs om{};
    if (!dense) {
      for (int j = 0; j < d; ++j) om.p[j] = (j == i) ? nullptr : omega[i * d + j];
      if (dist && !last) om.p[d - 1] = omega[i * d + d - 1] + slab_begin * R;
    }
    bool want[kMaxD] = {};
    want[i] = true;
    float* Yp[kMaxD] = {};
    const int64_t yrows = last ? gd[d - 1] : cur[i];
    if (dist && last) {  // complete local rows of Y_d at their global offset, zero elsewhere: the sum gathers
      KRP_CHECK_CUDA(cudaMemsetAsync(Y, 0, yrows * R * sizeof(float), s));
      Yp[i] = Y + slab_begin * R;
    } else {
      Yp[i] = Y;
    }
    if (dense) KRP_TRY(gaussian_sketch_mode(G, cg, i, dense[i], R, Y, ar, s));  // the Table 1 baseline
    else KRP_TRY(sketch(G, cg, om, R, want, Yp, ar, s));
    ar.off = mark;
    if (dist) KRP_TRY(allreduce_sum_f32(dc, Y, static_cast<size_t>(yrows * R), s));
    // 2. thin QR, replicated
    KRP_TRY(cholqr(Y, yrows, R, Qf, nullptr, flag, ar, s));
    ar.off = mark;
    // 3. B = G x_i Q^T: local; on the sharded mode the slab rows of Q, and the partial B is summed
    const float* Qrows = (dist && last) ? Qf + slab_begin * R : Qf;
    // NEXT-3, the fused step: for the first mode (a mode-1 product on the tensor cores) the truncation's
    // Gram B_(1) B_(1)^T is formed in the same pass, from the product's output tile in shared memory
    const int64_t H0 = cg.N / cg.n[0];
    const bool fused = i == 0 && ranks[i] < R && R <= 32 && ttm0_tc_ok(G, cg.n[0], H0, R) && ttm0_tc_grid(H0) <= 148;
    if (fused) {
      const int P = 4 * ttm0_tc_grid(H0);
      double* gp = ar.take<double>(static_cast<size_t>(P) * R * R);
      KRP_TRY(ttm0_tc(G, cg.n[0], H0, Qrows, R, 1, R, B, ar, s, 0, gp));
      KRP_TRY(sum_partials_f64(gp, P, static_cast<int64_t>(R) * R, H, s));
    } else {
      KRP_TRY(ttm(G, cg, i, Qrows, R, 1, R, B, s, &ar));
    }
    ar.off = mark;
    int64_t bd[kMaxD];
    for (int k = 0; k < d; ++k) bd[k] = cur[k];
    bd[i] = R;
    const Dims bg = make_dims(d, bd);
    if (dist && last) KRP_TRY(allreduce_sum_f32(dc, B, static_cast<size_t>(bg.N), s));
    float* Gout = last ? core : GA;
    if (ranks[i] < R) {
      // 4. U = leading r_i left singular vectors of B_(i) (its Gram sums over the slabs for i < d-1);
      //    G <- B x_i U^T; Q_i = Q U
      if (!fused) KRP_TRY(mode_gram(B, bg, i, H, ar, s));
      ar.off = mark;
      if (dist && !last) KRP_TRY(allreduce_sum_f64(dc, H, static_cast<size_t>(R) * R, s));
      KRP_TRY(sym_eig_top(H, R, ranks[i], U, s));
      KRP_TRY(ttm(B, bg, i, U, ranks[i], 1, ranks[i], Gout, s));
      int64_t qd[2] = {R, yrows};
      KRP_TRY(ttm(Qf, make_dims(2, qd), 0, U, ranks[i], 1, ranks[i], Q[i], s));
    } else {
      KRP_CHECK_CUDA(cudaMemcpyAsync(Gout, B, bg.N * sizeof(float), cudaMemcpyDeviceToDevice, s));
      KRP_CHECK_CUDA(cudaMemcpyAsync(Q[i], Qf, yrows * R * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }
    cur[i] = ranks[i];
    // the next step reads GA (B is free again: it is rewritten from GA before GA is overwritten)
    if (!last) G = GA;
  }
  if (rel_err) {
    KRP_CHECK_CUDA(cudaMemsetAsync(errsum, 0, 2 * sizeof(double), s));
    int64_t cd[kMaxD];
    for (int k = 0; k < d; ++k) cd[k] = ranks[k];
    for (int64_t k0 = 0; k0 < g.n[d - 1]; k0 += chunk) {
      const int64_t k1 = std::min<int64_t>(g.n[d - 1], k0 + chunk);
      KRP_TRY(ttm(core, make_dims(d, cd), d - 1, Q[d - 1] + (slab_begin + k0) * ranks[d - 1],
                  static_cast<int>(k1 - k0), ranks[d - 1], 1, EA, s));
      int64_t ed[kMaxD];
      for (int m = 0; m < d; ++m) ed[m] = cd[m];
      ed[d - 1] = k1 - k0;
      float* src = EA;
      for (int m = d - 2; m >= 0; --m) {
        float* o = (m == 0) ? Xh : (src == EA ? EB : EA);
        KRP_TRY(ttm(src, make_dims(d, ed), m, Q[m], static_cast<int>(g.n[m]), ranks[m], 1, o, s));
        ed[m] = g.n[m];
        src = o;
      }
      KRP_TRY(sqdiff_accumulate(X + k0 * inner, Xh, (k1 - k0) * inner, errsum, ar, s));
      ar.off = mark;
    }
    if (dist) KRP_TRY(allreduce_sum_f64(dc, errsum, 2, s));
  }
  int hflag[4] = {0, 0, 0, 0};
  double herr[2] = {0.0, 0.0};
  KRP_CHECK_CUDA(cudaMemcpyAsync(hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, s));
  if (rel_err) KRP_CHECK_CUDA(cudaMemcpyAsync(herr, errsum, sizeof(herr), cudaMemcpyDeviceToHost, s));
  KRP_CHECK_CUDA(cudaStreamSynchronize(s));
  if (hflag[0] & 2) {
    set_error("CholeskyQR breakdown (shifted fallback failed)");
    return KRP_ENUMERIC;
  }
  if (rel_err) *rel_err = herr[1] > 0 ? sqrt(herr[0] / herr[1]) : 0.0;
  return KRP_OK;
}

}  // namespace krp

// ================================================================== C ABI
extern "C" {

const char* krp_status_string(int st) {
  switch (st) {
    case KRP_OK: return "ok";
    case KRP_EINVAL: return "invalid argument";
    case KRP_ESHAPE: return "inconsistent shape or rank";
    case KRP_ECUDA: return "CUDA error";
    case KRP_ENCCL: return "NCCL error";
    case KRP_ENUMERIC: return "numerical breakdown (CholeskyQR)";
    case KRP_ENOMEM: return "workspace too small / out of memory";
    case KRP_EUNSUPPORTED: return "unsupported shape or device";
    default: return "unknown status";
  }
}

const char* krp_last_error_message(void) { return krp::last_error(); }
int krp_version(void) { return 10000; }
uint64_t krp_launch_count(void) { return krp::g_launches.load(); }

int krp_profile_enable(int on) {
  krp::g_prof_on.store(on ? 1 : 0);
  return KRP_OK;
}

void krp_profile_reset(void) {
  std::lock_guard<std::mutex> lk(krp::g_prof_mu);
  for (auto& r : krp::g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  krp::g_prof.clear();
}

int krp_profile_read(double* kernel_ms, uint64_t* launches, double* alg_bytes, double* alg_flops) {
  std::lock_guard<std::mutex> lk(krp::g_prof_mu);
  double ms = 0.0, by = 0.0, fl = 0.0;
  for (auto& r : krp::g_prof) {
    KRP_CHECK_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    KRP_CHECK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    by += r.bytes;
    fl += r.flops;
  }
  if (kernel_ms) *kernel_ms = ms;
  if (launches) *launches = krp::g_prof.size();
  if (alg_bytes) *alg_bytes = by;
  if (alg_flops) *alg_flops = fl;
  return KRP_OK;
}
void krp_reset_launch_count(void) { krp::g_launches.store(0); }

static size_t ws_bytes_impl(int op, int d, const int64_t* dims, int64_t Id_global, int R, const int* ranks) {
  if (op == KRP_OP_TTM && dims && d >= 2 && d <= kMaxD && R >= 1) {  // R = J; only mode 0 takes workspace
    for (int k = 0; k < d; ++k)
      if (dims[k] < 1) return 0;
    return ttm_ws_bytes(make_dims(d, dims), 0, R) + 256;
  }
  if (!dims || d < 2 || d > kMaxD || R < 1 || R > kMaxR) return 0;
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) return 0;
  const Dims g = make_dims(d, dims);
  Arena ar;
  ar.measuring = true;
  switch (op) {
    case KRP_OP_SKETCH_ALL: {
      bool want[kMaxD];
      for (int k = 0; k < d; ++k) want[k] = true;
      return align_up(sketch_ws_bytes(g, R, want), 256) + 256;
    }
    case KRP_OP_SKETCH_ALL_HOST: {
      bool want[kMaxD];
      for (int k = 0; k < d; ++k) want[k] = true;
      size_t b = align_up(g.N * sizeof(float), 256);
      for (int k = 0; k < d; ++k) b += 2 * align_up(g.n[k] * R * sizeof(float), 256);
      return b + align_up(sketch_ws_bytes(g, R, want), 256) + 256;
    }
    case KRP_OP_SKETCH_MODE: {
      size_t b = 0;
      for (int n = 0; n < d; ++n) {
        bool want[kMaxD] = {};
        want[n] = true;
        b = std::max(b, sketch_ws_bytes(g, R, want));
      }
      return align_up(b, 256) + 256;
    }
    case KRP_OP_RHOSVD:
    case KRP_OP_RHOSVD_ERR: {
      if (!ranks) return 0;
      double dummy;
      rhosvd_impl(nullptr, g, Id_global, 0, ranks, R, nullptr, nullptr, nullptr,
                  op == KRP_OP_RHOSVD_ERR ? &dummy : nullptr, ar, nullptr, nullptr, true);
      return ar.off + 256;
    }
    case KRP_OP_STHOSVD:
    case KRP_OP_STHOSVD_GAUSSIAN: {
      if (!ranks) return 0;
      double dummy;
      const float* const dummy_dense[kMaxD] = {};
      sthosvd_impl(nullptr, g, Id_global, 0, ranks, R, nullptr, nullptr, nullptr, &dummy, ar, nullptr, nullptr, true,
                   op == KRP_OP_STHOSVD_GAUSSIAN ? dummy_dense : nullptr);
      return ar.off + 256;
    }
    case KRP_OP_RHOSVD_FRESH:
    case KRP_OP_RHOSVD_GAUSSIAN: {
      if (!ranks) return 0;
      double dummy;
      SketchVariant v;
      v.kind = op == KRP_OP_RHOSVD_FRESH ? 1 : 2;
      rhosvd_impl(nullptr, g, Id_global, 0, ranks, R, nullptr, nullptr, nullptr, &dummy, ar, nullptr, nullptr, true, &v);
      return ar.off + 256;
    }
    default:
      return 0;
  }
}

size_t krp_workspace_bytes(int op, int d, const int64_t* dims, int R, const int* ranks) {
  if (!dims || d < 2 || d > kMaxD) return 0;
  return ws_bytes_impl(op, d, dims, dims[d - 1], R, ranks);
}

size_t krp_workspace_bytes_dist(int op, int d, const int64_t* dims_local, int64_t I_d_global, int R,
                                const int* ranks) {
  size_t b = ws_bytes_impl(op, d, dims_local, I_d_global, R, ranks);
  if (op == KRP_OP_SKETCH_ALL && b) {
    // packed send buffer of the global sketches
    int64_t ysum = 0;
    for (int k = 0; k < d - 1; ++k) ysum += dims_local[k] * R;
    ysum += I_d_global * R;
    b += align_up(ysum * sizeof(float), 256);
  }
  return b;
}

int krp_sketch_all_modes(const float* X, int d, const int64_t* dims, const float* const* omega, int R,
                         float* const* Y, void* ws, size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  KRP_TRY(validate_ptrs(omega, d, -1, "omega"));
  KRP_TRY(validate_ptrs(Y, d, -1, "Y"));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims);
  bool want[kMaxD];
  for (int k = 0; k < d; ++k) want[k] = true;
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_SKETCH_ALL, d, dims, R, nullptr), ws, ws_bytes, s, ar, guard));
  return sketch(X, g, make_om(omega, d, -1), R, want, Y, ar, s);
}

int krp_sketch_all_modes_host(const float* X_host, int d, const int64_t* dims, const float* const* omega_host, int R,
                              float* const* Y_host, void* ws, size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X_host, d, dims, R));
  KRP_TRY(validate_ptrs(omega_host, d, -1, "omega"));
  KRP_TRY(validate_ptrs(Y_host, d, -1, "Y"));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_SKETCH_ALL_HOST, d, dims, R, nullptr), ws, ws_bytes, s, ar, guard));
  float* Xd = ar.take<float>(g.N);
  float* Od[kMaxD];
  float* Yd[kMaxD];
  for (int k = 0; k < d; ++k) Od[k] = ar.take<float>(g.n[k] * R);
  for (int k = 0; k < d; ++k) Yd[k] = ar.take<float>(g.n[k] * R);
  KRP_CHECK_CUDA(cudaMemcpyAsync(Xd, X_host, g.N * sizeof(float), cudaMemcpyHostToDevice, s));
  for (int k = 0; k < d; ++k)
    KRP_CHECK_CUDA(cudaMemcpyAsync(Od[k], omega_host[k], g.n[k] * R * sizeof(float), cudaMemcpyHostToDevice, s));
  bool want[kMaxD];
  for (int k = 0; k < d; ++k) want[k] = true;
  OmegaPtrs om{};
  for (int k = 0; k < d; ++k) om.p[k] = Od[k];
  KRP_TRY(sketch(Xd, g, om, R, want, Yd, ar, s));
  for (int k = 0; k < d; ++k)
    KRP_CHECK_CUDA(cudaMemcpyAsync(Y_host[k], Yd[k], g.n[k] * R * sizeof(float), cudaMemcpyDeviceToHost, s));
  KRP_CHECK_CUDA(cudaStreamSynchronize(s));
  return KRP_OK;
}

int krp_sketch_mode(const float* X, int d, const int64_t* dims, int n, const float* const* omega, int R, float* Y,
                    void* ws, size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  if (n < 0 || n >= d) {
    set_error("mode n=%d not in [0,%d)", n, d);
    return KRP_EINVAL;
  }
  KRP_TRY(validate_ptrs(omega, d, n, "omega"));
  if (!Y) {
    set_error("Y is NULL");
    return KRP_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims);
  bool want[kMaxD] = {};
  want[n] = true;
  float* Yp[kMaxD] = {};
  Yp[n] = Y;
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_SKETCH_MODE, d, dims, R, nullptr), ws, ws_bytes, s, ar, guard));
  return sketch(X, g, make_om(omega, d, n), R, want, Yp, ar, s);
}

int krp_ttm(const float* X, int d, const int64_t* dims, int n, const float* A, int J, float* Y, void* ws,
            size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, 1));
  if (n < 0 || n >= d) {
    set_error("mode n=%d not in [0,%d)", n, d);
    return KRP_EINVAL;
  }
  if (!A || !Y || J < 1 || J > (1 << 24)) {
    set_error("krp_ttm: A / Y NULL or J=%d not in [1, 2^24]", J);
    return KRP_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_TTM, d, dims, J, nullptr), ws, ws_bytes, s, ar, guard));
  return ttm(X, g, n, A, J, g.n[n], 1, Y, s, &ar);
}

int krp_rhosvd(const float* X, int d, const int64_t* dims, const int* ranks, int R, const float* const* omega,
               float* const* Q, float* core, double* rel_err, void* ws, size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  KRP_TRY(validate_ptrs(omega, d, -1, "omega"));
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core) {
    set_error("core is NULL");
    return KRP_EINVAL;
  }
  const Dims g = make_dims(d, dims);
  KRP_TRY(validate_ranks(g, ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Arena ar;
  WsGuard guard;
  const size_t need = krp_workspace_bytes(rel_err ? KRP_OP_RHOSVD_ERR : KRP_OP_RHOSVD, d, dims, R, ranks);
  KRP_TRY(setup_arena(need, ws, ws_bytes, s, ar, guard));
  return rhosvd_impl(X, g, dims[d - 1], 0, ranks, R, omega, Q, core, rel_err, ar, s, nullptr, false);
}

int krp_sthosvd(const float* X, int d, const int64_t* dims, const int* ranks, int R, const float* const* omega,
                float* const* Q, float* core, double* rel_err, void* ws, size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  if (!omega) {
    set_error("omega is NULL");
    return KRP_EINVAL;
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (i != j && !omega[i * d + j]) {
        set_error("omega[%d*d+%d] is NULL", i, j);
        return KRP_EINVAL;
      }
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core) {
    set_error("core is NULL");
    return KRP_EINVAL;
  }
  const Dims g = make_dims(d, dims);
  KRP_TRY(validate_ranks(g, ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_STHOSVD, d, dims, R, ranks), ws, ws_bytes, s, ar, guard));
  return sthosvd_impl(X, g, dims[d - 1], 0, ranks, R, omega, Q, core, rel_err, ar, s, nullptr, false);
}

static int validate_steps(const float* const* steps, int d, const char* what) {
  if (!steps) {
    set_error("%s is NULL", what);
    return KRP_EINVAL;
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (i != j && !steps[i * d + j]) {
        set_error("%s[%d*d+%d] is NULL", what, i, j);
        return KRP_EINVAL;
      }
  return KRP_OK;
}

int krp_rhosvd_fresh(const float* X, int d, const int64_t* dims, const int* ranks, int R,
                     const float* const* omega_steps, float* const* Q, float* core, double* rel_err, void* ws,
                     size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  KRP_TRY(validate_steps(omega_steps, d, "omega_steps"));
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core) {
    set_error("core is NULL");
    return KRP_EINVAL;
  }
  const Dims g = make_dims(d, dims);
  KRP_TRY(validate_ranks(g, ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_RHOSVD_FRESH, d, dims, R, ranks), ws, ws_bytes, s, ar, guard));
  SketchVariant v;
  v.kind = 1;
  v.steps = omega_steps;
  return rhosvd_impl(X, g, dims[d - 1], 0, ranks, R, nullptr, Q, core, rel_err, ar, s, nullptr, false, &v);
}

int krp_rhosvd_gaussian(const float* X, int d, const int64_t* dims, const int* ranks, int R,
                        const float* const* omega_dense, float* const* Q, float* core, double* rel_err, void* ws,
                        size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  KRP_TRY(validate_ptrs(omega_dense, d, -1, "omega_dense"));
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core) {
    set_error("core is NULL");
    return KRP_EINVAL;
  }
  const Dims g = make_dims(d, dims);
  KRP_TRY(validate_ranks(g, ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_RHOSVD_GAUSSIAN, d, dims, R, ranks), ws, ws_bytes, s, ar, guard));
  SketchVariant v;
  v.kind = 2;
  v.dense = omega_dense;
  return rhosvd_impl(X, g, dims[d - 1], 0, ranks, R, nullptr, Q, core, rel_err, ar, s, nullptr, false, &v);
}

int krp_sthosvd_gaussian(const float* X, int d, const int64_t* dims, const int* ranks, int R,
                         const float* const* omega_dense, float* const* Q, float* core, double* rel_err, void* ws,
                         size_t ws_bytes, void* stream) {
  KRP_TRY(validate_common(X, d, dims, R));
  KRP_TRY(validate_ptrs(omega_dense, d, -1, "omega_dense"));
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core) {
    set_error("core is NULL");
    return KRP_EINVAL;
  }
  const Dims g = make_dims(d, dims);
  KRP_TRY(validate_ranks(g, ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes(KRP_OP_STHOSVD_GAUSSIAN, d, dims, R, ranks), ws, ws_bytes, s, ar, guard));
  return sthosvd_impl(X, g, dims[d - 1], 0, ranks, R, nullptr, Q, core, rel_err, ar, s, nullptr, false, omega_dense);
}

static int validate_hadamard(const int64_t* n, const int64_t* q, const int64_t* s, const int* ranks, const int* ls) {
  if (!n || !q || !s || !ranks || !ls) {
    set_error("null size argument");
    return KRP_EINVAL;
  }
  for (int k = 0; k < 3; ++k) {
    if (n[k] < 1 || q[k] < 1 || s[k] < 1 || q[k] > n[k] || s[k] > n[k]) {
      set_error("mode %d: n=%lld q=%lld s=%lld (need 1 <= q, s <= n)", k, static_cast<long long>(n[k]),
                static_cast<long long>(q[k]), static_cast<long long>(s[k]));
      return KRP_EINVAL;
    }
    if (ls[k] < 1 || ls[k] > kMaxRDecomp || ranks[k] < 1 || ranks[k] > ls[k] || ls[k] > n[k]) {
      set_error("mode %d: l=%d, r=%d (need 1 <= r <= l <= min(n, %d))", k, ls[k], ranks[k], kMaxRDecomp);
      return KRP_ESHAPE;
    }
  }
  return KRP_OK;
}

size_t krp_hadamard_workspace_bytes(const int64_t* n, const int64_t* q, const int64_t* s, const int* ranks,
                                    const int* ls) {
  if (validate_hadamard(n, q, s, ranks, ls) != KRP_OK) return 0;
  Arena ar;
  ar.measuring = true;
  hadamard_tucker_impl(nullptr, q, nullptr, nullptr, s, nullptr, n, ranks, ls, nullptr, nullptr, nullptr, ar, nullptr,
                       true);
  return ar.off + 256;
}

int krp_hadamard_tucker(const float* F, const int64_t* q, const float* const* A, const float* G, const int64_t* s,
                        const float* const* U, const int64_t* n, const int* ranks, const int* ls,
                        const float* const* omega, float* const* Q, float* core, void* ws, size_t ws_bytes,
                        void* stream) {
  KRP_TRY(validate_hadamard(n, q, s, ranks, ls));
  if (!F || !G || !core) {
    set_error("F, G or core is NULL");
    return KRP_EINVAL;
  }
  KRP_TRY(validate_ptrs(A, 3, -1, "A"));
  KRP_TRY(validate_ptrs(U, 3, -1, "U"));
  KRP_TRY(validate_ptrs(Q, 3, -1, "Q"));
  KRP_TRY(validate_steps(omega, 3, "omega"));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_hadamard_workspace_bytes(n, q, s, ranks, ls), ws, ws_bytes, st, ar, guard));
  return hadamard_tucker_impl(F, q, A, G, s, U, n, ranks, ls, omega, Q, core, ar, st, false);
}

// ------------------------------------------------------------------ distributed
size_t krp_comm_id_bytes(void) { return sizeof(krp::nccl_uid_t); }

int krp_comm_get_unique_id(void* id_out) {
  if (!id_out) {
    set_error("id_out is NULL");
    return KRP_EINVAL;
  }
  NcclApi* api = nccl();
  if (!api) {
    set_error("libnccl.so.2 could not be loaded");
    return KRP_ENCCL;
  }
  nccl_uid_t uid;
  int r = api->get_uid(&uid);
  if (r != 0) {
    set_error("ncclGetUniqueId failed (%d)", r);
    return KRP_ENCCL;
  }
  memcpy(id_out, &uid, sizeof(uid));
  return KRP_OK;
}

int krp_comm_init(krp_comm* comm, int nranks, int rank, const void* id) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("bad krp_comm_init arguments");
    return KRP_EINVAL;
  }
  auto* c = new krp_comm_s();
  c->ctx.nranks = nranks;
  c->ctx.rank = rank;
  if (nranks > 1) {
    NcclApi* api = nccl();
    if (!api) {
      delete c;
      set_error("libnccl.so.2 could not be loaded");
      return KRP_ENCCL;
    }
    nccl_uid_t uid;
    memcpy(&uid, id, sizeof(uid));
    int r = api->init_rank(&c->ctx.comm, nranks, uid, rank);
    if (r != 0) {
      delete c;
      set_error("ncclCommInitRank failed: %s", api->errstr ? api->errstr(r) : "?");
      return KRP_ENCCL;
    }
  }
  *comm = c;
  return KRP_OK;
}

int krp_comm_destroy(krp_comm comm) {
  if (!comm) return KRP_OK;
  if (comm->ctx.comm) {
    NcclApi* api = nccl();
    if (api) api->destroy(comm->ctx.comm);
  }
  delete comm;
  return KRP_OK;
}

static int validate_slab(int d, const int64_t* dims_local, int64_t Id_global, int64_t slab_begin) {
  if (!dims_local || d < 2) return KRP_EINVAL;
  if (Id_global < 1 || slab_begin < 0 || slab_begin + dims_local[d - 1] > Id_global) {
    set_error("inconsistent slab: begin=%lld len=%lld global=%lld", static_cast<long long>(slab_begin),
              static_cast<long long>(dims_local[d - 1]), static_cast<long long>(Id_global));
    return KRP_ESHAPE;
  }
  return KRP_OK;
}

int krp_slab_range(int64_t I_d, int nranks, int rank, int64_t* begin, int64_t* len) {
  if (I_d < 1 || nranks < 1 || rank < 0 || rank >= nranks || !begin || !len) {
    set_error("krp_slab_range: bad arguments");
    return KRP_EINVAL;
  }
  if (nranks > I_d) {  // every rank must own a non-empty slab (all ranks take this branch together)
    set_error("krp_slab_range: %d ranks > I_d = %lld (empty slabs)", nranks, static_cast<long long>(I_d));
    return KRP_ESHAPE;
  }
  const int64_t b = I_d * rank / nranks, e = I_d * (rank + 1) / nranks;
  *begin = b;
  *len = e - b;
  return KRP_OK;
}

int krp_pack_layout(int d, const int64_t* dims_local, int64_t I_d_global, int64_t slab_begin, int R,
                    int64_t* offsets, int64_t* slab_offset) {
  if (!dims_local || !offsets || !slab_offset || d < 2 || d > krp::kMaxD || R < 1) {
    set_error("krp_pack_layout: bad arguments");
    return KRP_EINVAL;
  }
  KRP_TRY(validate_slab(d, dims_local, I_d_global, slab_begin));
  int64_t off = 0;
  for (int k = 0; k < d; ++k) {
    offsets[k] = off;
    off += ((k == d - 1) ? I_d_global : dims_local[k]) * R;
  }
  offsets[d] = off;
  *slab_offset = offsets[d - 1] + slab_begin * R;
  return KRP_OK;
}

int krp_sketch_all_modes_dist(const float* X_slab, int d, const int64_t* dims_local, int64_t I_d_global,
                              int64_t slab_begin, const float* const* omega, int R, float* const* Y, void* ws,
                              size_t ws_bytes, krp_comm comm, void* stream) {
  KRP_TRY(validate_common(X_slab, d, dims_local, R));
  KRP_TRY(validate_slab(d, dims_local, I_d_global, slab_begin));
  KRP_TRY(validate_ptrs(omega, d, -1, "omega"));
  KRP_TRY(validate_ptrs(Y, d, -1, "Y"));
  if (!comm) {
    set_error("comm is NULL");
    return KRP_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims_local);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes_dist(KRP_OP_SKETCH_ALL, d, dims_local, I_d_global, R, nullptr), ws,
                      ws_bytes, s, ar, guard));
  int64_t poff[kMaxD + 1], slab_off = 0;
  KRP_TRY(krp_pack_layout(d, dims_local, I_d_global, slab_begin, R, poff, &slab_off));
  const int64_t ysum = poff[d];
  float* pack = ar.take<float>(ysum);
  float* Yl[kMaxD];
  for (int k = 0; k < d - 1; ++k) Yl[k] = pack + poff[k];
  Yl[d - 1] = pack + slab_off;
  KRP_CHECK_CUDA(cudaMemsetAsync(pack, 0, ysum * sizeof(float), s));
  OmegaPtrs om = make_om(omega, d, -1);
  om.p[d - 1] = omega[d - 1] + slab_begin * R;
  bool want[kMaxD];
  for (int k = 0; k < d; ++k) want[k] = true;
  KRP_TRY(sketch(X_slab, g, om, R, want, Yl, ar, s));
  // one all-reduce(sum): partial Y_1..Y_{d-1} summed, zero-padded Y_d rows gathered
  KRP_TRY(allreduce_sum_f32(&comm->ctx, pack, static_cast<size_t>(ysum), s));
  for (int k = 0; k < d; ++k)
    KRP_CHECK_CUDA(cudaMemcpyAsync(Y[k], pack + poff[k], (poff[k + 1] - poff[k]) * sizeof(float),
                                   cudaMemcpyDeviceToDevice, s));
  return KRP_OK;
}

int krp_sthosvd_dist(const float* X_slab, int d, const int64_t* dims_local, int64_t I_d_global, int64_t slab_begin,
                     const int* ranks, int R, const float* const* omega, float* const* Q, float* core,
                     double* rel_err, void* ws, size_t ws_bytes, krp_comm comm, void* stream) {
  KRP_TRY(validate_common(X_slab, d, dims_local, R));
  KRP_TRY(validate_slab(d, dims_local, I_d_global, slab_begin));
  if (!omega) {
    set_error("omega is NULL");
    return KRP_EINVAL;
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (i != j && !omega[i * d + j]) {
        set_error("omega[%d*d+%d] is NULL", i, j);
        return KRP_EINVAL;
      }
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core || !comm) {
    set_error("core/comm is NULL");
    return KRP_EINVAL;
  }
  int64_t gd[kMaxD];
  for (int k = 0; k < d; ++k) gd[k] = dims_local[k];
  gd[d - 1] = I_d_global;
  KRP_TRY(validate_ranks(make_dims(d, gd), ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims_local);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes_dist(KRP_OP_STHOSVD, d, dims_local, I_d_global, R, ranks), ws, ws_bytes, s,
                      ar, guard));
  return sthosvd_impl(X_slab, g, I_d_global, slab_begin, ranks, R, omega, Q, core, rel_err, ar, s, &comm->ctx, false);
}

int krp_rhosvd_dist(const float* X_slab, int d, const int64_t* dims_local, int64_t I_d_global, int64_t slab_begin,
                    const int* ranks, int R, const float* const* omega, float* const* Q, float* core,
                    double* rel_err, void* ws, size_t ws_bytes, krp_comm comm, void* stream) {
  KRP_TRY(validate_common(X_slab, d, dims_local, R));
  KRP_TRY(validate_slab(d, dims_local, I_d_global, slab_begin));
  KRP_TRY(validate_ptrs(omega, d, -1, "omega"));
  KRP_TRY(validate_ptrs(Q, d, -1, "Q"));
  if (!core || !comm) {
    set_error("core/comm is NULL");
    return KRP_EINVAL;
  }
  int64_t gd[kMaxD];
  for (int k = 0; k < d; ++k) gd[k] = dims_local[k];
  gd[d - 1] = I_d_global;
  KRP_TRY(validate_ranks(make_dims(d, gd), ranks, R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims g = make_dims(d, dims_local);
  Arena ar;
  WsGuard guard;
  KRP_TRY(setup_arena(krp_workspace_bytes_dist(rel_err ? KRP_OP_RHOSVD_ERR : KRP_OP_RHOSVD, d, dims_local,
                                               I_d_global, R, ranks),
                      ws, ws_bytes, s, ar, guard));
  return rhosvd_impl(X_slab, g, I_d_global, slab_begin, ranks, R, omega, Q, core, rel_err, ar, s, &comm->ctx, false);
}

}  // extern "C"
