// rbffd_b200.cu -- host driver + C ABI (include/rbffd_b200.h) of the B200-native
// explicit RBF-FD time loop.  Replaces rbffd.solver._step_kernel and the step
// loop of rbffd.solver.run_time_loop (pkg/src/rbffd/solver.py:168-311).
//
// Design (DESIGN.md has the long form):
//  * plan_create packs the reference's row-major ShapeStore into SELL-32 on the
//    device (pack_rows_kernel) and renumbers nodes so interior row r updates
//    node B + r.  The renumbering never touches the per-row j order, so the
//    arithmetic, and therefore every bit, is unchanged.
//  * small problems (whole working set <= ~220 KB) run the entire loop inside
//    one CTA's shared memory (resident_loop_kernel): one launch per run.
//  * everything else runs one streaming launch per step, captured into CUDA
//    graphs of kGraphSteps steps and chained with programmatic dependent launch
//    so step s+1 streams its weights while step s drains.  The non-finite
//    flag, the residual max and the steady-state decision are fused into the
//    step (last-CTA ticket), so the host only polls a 64-byte status per chunk.
#include "../../include/rbffd_b200.h"
#include "step_kernels.cuh"
#include "pair.h"
#include "weights_kernels.cuh"
#include "knn_kernels.cuh"

#include <cub/cub.cuh>

#include <cuda_runtime.h>
#include <emmintrin.h>
#include <omp.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace rbf_detail {
// error entry for the host-only translation units (nodes.cpp)
int fail_c(int code, const char* msg) { return fail(code, msg ? msg : ""); }
}  // namespace rbf_detail

namespace {

#define RBF_CK(call)                                                                         \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(RBF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define RBF_TRY(expr)          \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != RBF_OK) return rc_; \
  } while (0)

constexpr int kGraphSteps = 64;  // steps per captured graph (even: keeps buffer parity)
constexpr int kStreamBlock = 256;
constexpr size_t kResidentSmemMax = 227 * 1024;
constexpr int64_t kPairAutoEntries = 1000000;  // N_i*n up to which fixed-step runs use the pair kernel

using StreamFn = void (*)(rbf::StepArgs, const double*, double*, int);
using TmaFn = void (*)(rbf::StepArgs, const double*, double*, int, rbf::TmaGeom);
using ResidentFn = void (*)(rbf::ResidentArgs);
using ClusterFn = void (*)(rbf::ClusterArgs);
using GridFn = void (*)(rbf::GridArgs);
using LoopFn = void (*)(rbf::StepArgs, rbf::LoopArgs, rbf::TmaGeom);
using PartLoopFn = void (*)(const rbf::PartLoop*, int, long long, rbf::TmaGeom);

template <int NJ>
struct KernelSet {
  static StreamFn stream() { return rbf::step_stream_kernel<NJ>; }
  static ResidentFn resident() { return rbf::resident_loop_kernel<NJ>; }
  static ClusterFn cluster(bool small) {
    return small ? rbf::cluster_loop_kernel<NJ, 256> : rbf::cluster_loop_kernel<NJ, 1024>;
  }
  // consumer warps: 15 (512-thread CTA, <= 128 registers) for narrow
  // stencils; 8 (<= 168 registers) for wide ones, which keep all NJ gathers in
  // flight (measured 1 % faster at n=56 than 15 warps gathering in two halves).
  // kCWide: the most consumer warps the register file holds for the widths the
  // benchmarks use (n=15: 23 at <= 80 registers, n=30: 18 at <= 104, n=56: 11
  // at <= 160); chosen with RBFFD_TMA_CW=<kCWide>.
  static constexpr int kCW = NJ <= 32 ? 15 : 8;
  static constexpr int kCWide = NJ == 15 ? 23 : (NJ == 30 ? 18 : (NJ == 56 ? 11 : kCW));
  static TmaFn tma(int cw_req, bool idx16) {
    if constexpr (NJ > 0) {
      if constexpr (kCWide != kCW) {
        if (cw_req == kCWide)
          return idx16 ? rbf::step_tma_kernel<NJ, kCWide, 1, 2> : rbf::step_tma_kernel<NJ, kCWide, 1, 4>;
      }
      return idx16 ? rbf::step_tma_kernel<NJ, kCW, 1, 2> : rbf::step_tma_kernel<NJ, kCW, 1, 4>;
    } else {
      (void)cw_req;
      (void)idx16;
      return nullptr;
    }
  }
  static int cw(int cw_req) { return (NJ > 0 && cw_req == kCWide) ? kCWide : kCW; }
  // persistent streaming loop (one cooperative launch per run)
  static LoopFn loop(bool idx16) {
    if constexpr (NJ > 0) {
      return idx16 ? rbf::stream_loop_kernel<NJ, kCW, 2> : rbf::stream_loop_kernel<NJ, kCW, 4>;
    } else {
      (void)idx16;
      return nullptr;
    }
  }
  // partitioned persistent loop of a push-mode group (group.inc.cuh)
  static PartLoopFn part_loop(bool idx16) {
    if constexpr (NJ > 0) {
      return idx16 ? rbf::part_loop_kernel<NJ, kCW, 2> : rbf::part_loop_kernel<NJ, kCW, 4>;
    } else {
      (void)idx16;
      return nullptr;
    }
  }
  static GridFn grid(bool two) {
    if constexpr (NJ > 0) return two ? rbf::grid_loop_kernel<NJ, true> : rbf::grid_loop_kernel<NJ, false>;
    else {
      (void)two;
      return nullptr;
    }
  }
};

// Support sizes with a fully unrolled instantiation; others use the generic
// runtime-n kernel (same arithmetic, same order).
#define RBF_SPECIALISED(X) \
  X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(12) X(15) X(16) X(20) X(21) X(24) X(28) X(30) X(32) \
  X(36) X(40) X(42) X(45) X(48) X(56) X(60) X(64)

bool pick_kernels(int n, int cw_req, bool idx16, StreamFn* s, ResidentFn* r, TmaFn* t, int* kn,
                  int* rpl, int* cw) {
  switch (n) {
#define RBF_CASE(K)                        \
  case K:                                  \
    *s = KernelSet<K>::stream();           \
    *r = KernelSet<K>::resident();         \
    *t = KernelSet<K>::tma(cw_req, idx16); \
    *rpl = 1;                              \
    *cw = KernelSet<K>::cw(cw_req);        \
    *kn = K;                               \
    return true;
    RBF_SPECIALISED(RBF_CASE)
#undef RBF_CASE
    default:
      *s = KernelSet<0>::stream();
      *r = KernelSet<0>::resident();
      *t = nullptr;
      *kn = 0;
      *rpl = 1;
      *cw = 8;
      return false;
  }
}

// RBFFD_VERBOSE=1: phase timings of plan construction on stderr
struct PhaseTimer {
  bool on = std::getenv("RBFFD_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rbffd] %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

// The dynamic shared-memory cap is per-function global state: raise it once to
// the device maximum (never to a plan's own size, or a later, smaller plan
// would invalidate the launches of an earlier, larger one).
template <typename F>
cudaError_t set_max_smem(F fn) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - static_cast<int>(fa.sharedSizeBytes));
}


}  // namespace

struct rbf_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t N = 0, N_i = 0, B = 0, S = 0;
  int n = 0;
  double* W = nullptr;
  int* C = nullptr;
  double* F = nullptr;
  double* U[2] = {nullptr, nullptr};
  double* tmp = nullptr;      // N doubles for permuted field transfers
  // error norms (rbf_error_norms): numpy's pairwise-sum blocks of [0, N)
  std::vector<long long> norm_start;  // block starts + N
  long long* d_norm_start = nullptr;
  double* d_norm_sum = nullptr;       // [blocks] block sums, then [blocks] = max bits slot
  double* norm_exact = nullptr;       // N doubles (tmp when the plan is renumbered)
  int* new_id = nullptr;      // [N] original -> plan node id; nullptr = identity
  long long* row_of_k = nullptr;  // [N_i] reference row k -> plan row; nullptr = identity
  rbf::DevStatus* st = nullptr;
  rbf::DevStatus* h_st = nullptr;  // pinned
  StreamFn stream_fn = nullptr;
  ResidentFn resident_fn = nullptr;
  TmaFn tma_fn = nullptr;          // non-null: TMA-pipelined streaming step is used
  rbf::TmaGeom tma_geom = {1, 2};
  size_t tma_smem = 0;
  int tma_block = 0;
  int variant = 1;                 // 0 resident, 1 LDG streaming, 2 TMA streaming, 3 cluster loop
  ClusterFn cluster_fn = nullptr;  // non-null: the loop runs in one thread-block cluster
  GridFn grid_fn = nullptr;        // non-null: the loop runs in one cooperative grid (rows in smem)
  LoopFn loop_fn = nullptr;        // non-null: streaming runs go through the persistent loop
  size_t loop_smem = 0;
  int loop_grid = 0;
  rbf::TmaGeom loop_geom = {1, 2, 0, 0};
  unsigned long long* loop_red = nullptr;  // [7] residual slots + arrival counter
  int grid_ctas = 0, grid_spc = 0, grid_spr = 0;
  size_t grid_smem = 0;
  unsigned long long* grid_red = nullptr;  // [3][2] per-step partial slots
  rbf::PairPlan grid_pair;                 // two steps per barrier: halo / local-id tables
  bool grid_two = false;
  int cluster_q = 0, cluster_rpc = 0, cluster_threads = 0;
  size_t cluster_smem = 0;
  unsigned int* cluster_dest = nullptr;
  unsigned short* C16 = nullptr;   // 16-bit two-window ids (index_bits == 16)
  int4* meta = nullptr;            // per-slice {base0, base1, ok, 0}
  int index_bits = 32;
  int64_t overflow_slices = 0;
  double* u_init = nullptr;        // start field kept for the exact re-run after a failure (pair path)
  // two steps per launch (pair_kernels.cu): fixed-step runs of TMA plans
  rbf::PairPlan pair;
  bool pair_ok = false;
  bool pair_forced = false;        // RBF_PAIR / RBFFD_PAIR=1: ahead of the persistent loop
  cudaGraphExec_t pair_graph = nullptr;
  int kernel_n = 0;
  bool resident = false;
  size_t resident_smem = 0;
  bool renumbered = false;
  bool pdl = true;
  int grid = 1;
  int cur = 0;                // buffer holding the current field
  cudaGraphExec_t graphs[4] = {nullptr, nullptr, nullptr, nullptr};  // [copy_back*2 + steady]
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t launches = 0;
  int64_t device_bytes = 0;
  // partitioned runs (group.inc.cuh): exchange lists of this part
  std::vector<int> halo_peers;
  std::vector<int64_t> halo_send_count, halo_send_off, halo_recv_count, halo_recv_off;
  // push-mode groups (group.inc.cuh): field buffers from cudaMalloc (IPC-exportable),
  // this part's arrival counters (indexed by part id) and the neighbours to wait for
  bool u_legacy = false;
  bool push = false;
  unsigned long long* push_flags = nullptr;
  int wait_ids[rbf::kMaxPushPeers] = {};
  int wait_n = 0;
  int64_t push_base = 0;
  int* halo_send_idx = nullptr;     // [halo_send_total] local ids of owned nodes to send
  std::vector<int32_t> halo_send_idx_h;  // host copy (the part loop's per-slice push lists)
  double* halo_sendbuf = nullptr;   // packed values, segments per peer
  int64_t halo_send_total = 0;
  int64_t halo_row0 = 0;            // first row that reads a halo node (rbf_plan_set_halo)
  unsigned long long* trace = nullptr;  // RBFFD_TRACE=<file>: per-step CTA timestamps of the TMA step
  int trace_cap = 0;

  rbf::StepArgs args() const {
    rbf::StepArgs a;
    a.W = W;
    a.C = C;
    a.F = F;
    a.n_rows = N_i;
    a.dst_base = B;
    a.n = n;
    a.st = st;
    a.C16 = C16;
    a.meta = meta;
    a.wait_flags = push ? push_flags : nullptr;
    a.wait_mask = 0;
    for (int i = 0; push && i < wait_n; ++i) a.wait_mask |= 1ull << wait_ids[i];
    static const unsigned long long wait_ns = [] {
      const char* e = std::getenv("RBFFD_WAIT_TIMEOUT_MS");
      const long long ms = e ? std::atoll(e) : 20000;
      return static_cast<unsigned long long>(ms > 0 ? ms : 20000) * 1000000ull;
    }();
    a.wait_ns = wait_ns;
    a.halo_row0 = push ? halo_row0 : 0;
    a.trace = trace;
    a.trace_cap = trace_cap;
    return a;
  }
};

namespace {

// Device memory comes from the stream-ordered default pool of the device,
// with the release threshold raised so freed plan memory stays mapped and the
// next plan reuses it (cudaMalloc/cudaFree of hundreds of MB cost 10-1000 ms
// per plan on B200; profiles/README.md).
int prepare_pool(int device) {
  static bool done[64] = {false};
  if (device >= 0 && device < 64 && !done[device]) {
    cudaMemPool_t pool;
    RBF_CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    RBF_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done[device] = true;
  }
  return RBF_OK;
}

template <typename T>
int pool_alloc(T** ptr, size_t count, cudaStream_t s) {
  if (count == 0) count = 1;
  RBF_CK(cudaMallocAsync(reinterpret_cast<void**>(ptr), count * sizeof(T), s));
  return RBF_OK;
}

template <typename T>
void pool_free(T*& ptr, cudaStream_t s) {
  if (ptr) cudaFreeAsync(ptr, s);
  ptr = nullptr;
}

template <typename T>
int dev_alloc(rbf_plan* p, T** ptr, size_t count) {
  RBF_TRY(pool_alloc(ptr, count, p->stream));
  p->device_bytes += static_cast<int64_t>((count ? count : 1) * sizeof(T));
  return RBF_OK;
}

// Pinned host status slots for all plans of the process: one pinned slab,
// handed out from a free list (cudaMallocHost / cudaFreeHost per plan cost up
// to ~40 ms at plan teardown, profiles/README.md).
struct StatusSlab {
  std::mutex mu;
  std::vector<rbf::DevStatus*> free_list;
  std::vector<void*> slabs;
};

StatusSlab& status_slab() {
  static StatusSlab s;
  return s;
}

cudaError_t status_alloc(rbf::DevStatus** out) {
  StatusSlab& sl = status_slab();
  std::lock_guard<std::mutex> lock(sl.mu);
  if (sl.free_list.empty()) {
    constexpr int kSlots = 256;
    void* mem = nullptr;
    cudaError_t e = cudaMallocHost(&mem, sizeof(rbf::DevStatus) * kSlots);
    if (e != cudaSuccess) return e;
    sl.slabs.push_back(mem);
    for (int i = kSlots - 1; i >= 0; --i) sl.free_list.push_back(static_cast<rbf::DevStatus*>(mem) + i);
  }
  *out = sl.free_list.back();
  sl.free_list.pop_back();
  return cudaSuccess;
}

void status_free(rbf::DevStatus* p) {
  if (!p) return;
  StatusSlab& sl = status_slab();
  std::lock_guard<std::mutex> lock(sl.mu);
  sl.free_list.push_back(p);
}

// Staging copies with non-temporal (streaming) stores: the pinned staging
// buffer is written once and read only by the DMA engine.
void copy_f64_nt(double* dst, const double* src, int64_t count) {
  int64_t i = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) && count > 0) {
    dst[0] = src[0];
    i = 1;
  }
  for (; i + 2 <= count; i += 2) _mm_stream_pd(dst + i, _mm_loadu_pd(src + i));
  for (; i < count; ++i) dst[i] = src[i];
}
int narrow_ids_nt(int32_t* dst, const int64_t* src, int64_t count, int64_t N) {
  int bad = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t v = src[i];
    bad |= (v < 0 || v >= N);
    _mm_stream_si32(dst + i, static_cast<int32_t>(v));
  }
  return bad;
}

// Pinned, double-buffered staging for plan uploads: the host copies (and
// int64 -> int32 id conversion) of chunk c+1 run while chunk c is on the bus.
struct Staging {
  std::mutex mu;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  size_t cap = 0;
  int device = -1;
};

Staging& staging() {
  static Staging s;
  return s;
}

int staging_acquire(Staging& sg, int device) {
  size_t kCap = size_t(16) << 20;  // 16 MB chunks pipeline the host copy with the DMA (8 / 64 MB: slower)
  if (const char* e = std::getenv("RBFFD_STAGING_MB")) kCap = std::max<size_t>(1, std::atoll(e)) << 20;
  if (sg.cap == kCap && sg.device == device) return RBF_OK;
  for (int b = 0; b < 2; ++b) {
    if (sg.buf[b]) cudaFreeHost(sg.buf[b]);
    if (sg.ev[b]) cudaEventDestroy(sg.ev[b]);
    sg.buf[b] = nullptr;
    sg.ev[b] = nullptr;
  }
  sg.cap = 0;
  for (int b = 0; b < 2; ++b) {
    RBF_CK(cudaMallocHost(reinterpret_cast<void**>(&sg.buf[b]), kCap));
    RBF_CK(cudaEventCreateWithFlags(&sg.ev[b], cudaEventDisableTiming));
  }
  sg.cap = kCap;
  sg.device = device;
  return RBF_OK;
}


// Field transfers through the pinned staging pair: pageable copies of a
// whole field run at a fraction of the link rate (the driver stages them
// through its own small bounce buffers); here the DMA of chunk c overlaps the
// host copy of chunk c-1, and the host copies use every core.
constexpr size_t kFieldStagedMin = size_t(4) << 20;  // bytes; below this a plain copy is faster

// Host memory already page-locked (cudaMallocHost / rbf_host_alloc /
// registered): the DMA reads or writes it directly, no staging copy.
bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int staged_d2h(double* dst, const double* dsrc, size_t count, cudaStream_t st, int device) {
  if (is_pinned(dst)) {
    RBF_CK(cudaMemcpyAsync(dst, dsrc, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBF_CK(cudaStreamSynchronize(st));
    return RBF_OK;
  }
  Staging& sg = staging();
  std::lock_guard<std::mutex> lk(sg.mu);
  RBF_TRY(staging_acquire(sg, device));
  const size_t chunk = sg.cap / sizeof(double);
  const size_t nchunks = (count + chunk - 1) / chunk;
  for (size_t c = 0; c <= nchunks; ++c) {
    if (c < nchunks) {  // start the DMA of chunk c
      const int b = static_cast<int>(c & 1);
      const size_t lo = c * chunk, n = std::min(chunk, count - lo);
      RBF_CK(cudaMemcpyAsync(sg.buf[b], dsrc + lo, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      RBF_CK(cudaEventRecord(sg.ev[b], st));
    }
    if (c > 0) {  // drain chunk c-1 into the caller's buffer
      const int b = static_cast<int>((c - 1) & 1);
      const size_t lo = (c - 1) * chunk, n = std::min(chunk, count - lo);
      RBF_CK(cudaEventSynchronize(sg.ev[b]));
      const double* src = reinterpret_cast<const double*>(sg.buf[b]);
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < static_cast<int64_t>(n); ++e) dst[lo + e] = src[e];
    }
  }
  return RBF_OK;
}

int staged_h2d(double* ddst, const double* src, size_t count, cudaStream_t st, int device) {
  if (is_pinned(src)) {
    RBF_CK(cudaMemcpyAsync(ddst, src, count * sizeof(double), cudaMemcpyHostToDevice, st));
    RBF_CK(cudaStreamSynchronize(st));
    return RBF_OK;
  }
  Staging& sg = staging();
  std::lock_guard<std::mutex> lk(sg.mu);
  RBF_TRY(staging_acquire(sg, device));
  const size_t chunk = sg.cap / sizeof(double);
  for (size_t lo = 0, c = 0; lo < count; lo += chunk, ++c) {
    const int b = static_cast<int>(c & 1);
    const size_t n = std::min(chunk, count - lo);
    RBF_CK(cudaEventSynchronize(sg.ev[b]));  // the previous DMA out of this buffer is done
    double* hb = reinterpret_cast<double*>(sg.buf[b]);
#pragma omp parallel
    {
      const int64_t T = omp_get_num_threads(), t = omp_get_thread_num();
      const int64_t a = static_cast<int64_t>(n) * t / T, e = static_cast<int64_t>(n) * (t + 1) / T;
      copy_f64_nt(hb + a, src + lo + a, e - a);
      _mm_sfence();
    }
    RBF_CK(cudaMemcpyAsync(ddst + lo, hb, n * sizeof(double), cudaMemcpyHostToDevice, st));
    RBF_CK(cudaEventRecord(sg.ev[b], st));
  }
  RBF_CK(cudaStreamSynchronize(st));
  return RBF_OK;
}

// One streaming step: reads U[in], writes U[1-in].
int launch_step(rbf_plan* p, int in, int flags) {
  if (p->N_i == 0) return RBF_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->grid);
  cfg.blockDim = dim3(p->tma_fn ? p->tma_block : kStreamBlock);
  cfg.dynamicSmemBytes = p->tma_fn ? p->tma_smem : 0;
  cfg.stream = p->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p->pdl ? 1 : 0;
  if (p->tma_fn) {
    RBF_CK(cudaLaunchKernelEx(&cfg, p->tma_fn, p->args(), static_cast<const double*>(p->U[in]),
                              p->U[1 - in], flags, p->tma_geom));
  } else {
    RBF_CK(cudaLaunchKernelEx(&cfg, p->stream_fn, p->args(), static_cast<const double*>(p->U[in]),
                              p->U[1 - in], flags));
  }
  ++p->launches;
  return RBF_OK;
}

// Two steps in one launch (pair_kernels.cu): U[in] -> U[1-in].
int launch_pair(rbf_plan* p, int in, int flags) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->pair.grid);
  cfg.blockDim = dim3(p->pair.block);
  cfg.dynamicSmemBytes = p->pair.smem;
  cfg.stream = p->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p->pdl ? 1 : 0;
  RBF_CK(cudaLaunchKernelEx(&cfg, p->pair.fn, p->pair.args, static_cast<const double*>(p->U[in]),
                            p->U[1 - in], flags, p->pair.geom));
  ++p->launches;
  return RBF_OK;
}

// A copy-back step (paper Listing 1, solver.py:213): U[0] -> U[1], then U[0] = U[1].
int launch_copy_back_step(rbf_plan* p, int flags) {
  RBF_TRY(launch_step(p, 0, flags));
  RBF_CK(cudaMemcpyAsync(p->U[0], p->U[1], sizeof(double) * p->N, cudaMemcpyDeviceToDevice,
                         p->stream));
  return RBF_OK;
}

int get_graph(rbf_plan* p, bool copy_back, bool steady, cudaGraphExec_t* out) {
  const int slot = (copy_back ? 2 : 0) + (steady ? 1 : 0);
  if (p->graphs[slot]) {
    *out = p->graphs[slot];
    return RBF_OK;
  }
  const int flags = steady ? (rbf::kNeedResidual | rbf::kSteady) : 0;
  RBF_CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  int rc = RBF_OK;
  const int64_t before = p->launches;
  for (int i = 0; i < kGraphSteps && rc == RBF_OK; ++i)
    rc = copy_back ? launch_copy_back_step(p, flags) : launch_step(p, i & 1, flags);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(p->stream, &g);
  p->launches = before;  // captured launches are counted when the graph runs
  if (rc != RBF_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(RBF_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  cudaGraphExec_t ge = nullptr;
  e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(RBF_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  p->graphs[slot] = ge;
  *out = ge;
  return RBF_OK;
}

int reset_status(rbf_plan* p, double dt, double tol) {
  rbf::DevStatus s = {};
  s.res_bits = 0;
  s.last_res_bits = 0;
  s.last_res_step = -1;
  s.bad_step = -1;
  s.conv_step = -1;
  s.step = 0;
  s.ticket = 0;
  s.dt = dt;
  s.tol = tol;
  s.push_base = p->push_base;
  s.push_count = 0;
  *p->h_st = s;
  RBF_CK(cudaMemcpyAsync(p->st, p->h_st, sizeof(s), cudaMemcpyHostToDevice, p->stream));
  return RBF_OK;
}

int read_status(rbf_plan* p) {
  RBF_CK(cudaMemcpyAsync(p->h_st, p->st, sizeof(rbf::DevStatus), cudaMemcpyDeviceToHost, p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

// Make U[0] hold the current field so graph parity (step s reads U[s % 2]) holds.
int normalise_current(rbf_plan* p) {
  if (p->cur != 0) {
    RBF_CK(cudaMemcpyAsync(p->U[0], p->U[1], sizeof(double) * p->N, cudaMemcpyDeviceToDevice,
                           p->stream));
    p->cur = 0;
  }
  return RBF_OK;
}

int run_streaming(rbf_plan* p, int64_t limit, bool steady, bool copy_back) {
  const int step_flags = steady ? (rbf::kNeedResidual | rbf::kSteady) : 0;
  cudaGraphExec_t graph = nullptr;
  PhaseTimer timer;
  if (limit > kGraphSteps) RBF_TRY(get_graph(p, copy_back, steady, &graph));
  timer.mark("graph capture/instantiate");
  RBF_CK(cudaEventRecord(p->ev0, p->stream));
  int64_t launched = 0;
  if (!steady) {
    const int64_t chunks = (limit - 1) / kGraphSteps;
    for (int64_t c = 0; c < chunks; ++c) {
      RBF_CK(cudaGraphLaunch(graph, p->stream));
      p->launches += kGraphSteps;
    }
    launched = chunks * kGraphSteps;
    for (; launched < limit; ++launched) {
      const int fl = (launched == limit - 1) ? rbf::kNeedResidual : 0;
      if (copy_back) RBF_TRY(launch_copy_back_step(p, fl));
      else RBF_TRY(launch_step(p, static_cast<int>(launched & 1), fl));
    }
    RBF_CK(cudaEventRecord(p->ev1, p->stream));
    timer.mark("enqueue");
    return RBF_OK;
  }
  // Steady: poll the device status once per chunk, keeping two chunks in
  // flight; steps issued after convergence are no-ops on the device.
  int in_flight = 0;
  cudaEvent_t evs[2];
  RBF_CK(cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming));
  RBF_CK(cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming));
  int which = 0;
  int rc = RBF_OK;
  while (launched < limit && rc == RBF_OK) {
    if (graph && limit - launched >= kGraphSteps) {
      if (cudaGraphLaunch(graph, p->stream) != cudaSuccess) { rc = fail(RBF_ERR_CUDA, "graph launch"); break; }
      p->launches += kGraphSteps;
      launched += kGraphSteps;
    } else {
      for (; launched < limit && rc == RBF_OK; ++launched)
        rc = copy_back ? launch_copy_back_step(p, step_flags)
                       : launch_step(p, static_cast<int>(launched & 1), step_flags);
      if (rc != RBF_OK) break;
    }
    cudaEventRecord(evs[which], p->stream);
    ++in_flight;
    which ^= 1;
    if (in_flight == 2 && launched < limit) {
      // wait for the older chunk, then peek at the status
      cudaEventSynchronize(evs[which]);
      --in_flight;
      rbf::DevStatus s;
      if (cudaMemcpy(&s, p->st, sizeof(s), cudaMemcpyDeviceToHost) != cudaSuccess) {
        rc = fail(RBF_ERR_CUDA, "status poll");
        break;
      }
      if (s.bad_step >= 0 || s.conv_step >= 0) break;
    }
  }
  cudaEventRecord(p->ev1, p->stream);
  cudaStreamSynchronize(p->stream);
  cudaEventDestroy(evs[0]);
  cudaEventDestroy(evs[1]);
  return rc;
}

// Fixed-step loop two steps per launch (pair_kernels.cu), CUDA graphs of
// kGraphSteps/2 launches, an odd last step on the single-step kernel.  The
// start field is kept; if any step produced a non-finite value the caller
// replays the run on the single-step path, which stops at the exact step
// (*fallback = true).  *final_buf = buffer holding the result.
int run_pair(rbf_plan* p, int64_t limit, bool* fallback, int* final_buf) {
  *fallback = false;
  if (!p->u_init) RBF_CK(cudaMallocAsync(reinterpret_cast<void**>(&p->u_init), sizeof(double) * p->N, p->stream));
  RBF_CK(cudaMemcpyAsync(p->u_init, p->U[0], sizeof(double) * p->N, cudaMemcpyDeviceToDevice, p->stream));
  const int64_t pairs = limit / 2;
  const bool odd = (limit & 1) != 0;
  constexpr int kPairGraph = kGraphSteps / 2;
  if (pairs > kPairGraph && !p->pair_graph) {
    RBF_CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t before = p->launches;
    int rc = RBF_OK;
    for (int i = 0; i < kPairGraph && rc == RBF_OK; ++i) rc = launch_pair(p, i & 1, 0);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(p->stream, &g);
    p->launches = before;
    if (rc != RBF_OK) return rc;
    if (e != cudaSuccess) return fail(RBF_ERR_CUDA, std::string("pair graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&p->pair_graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(RBF_ERR_CUDA, std::string("pair graph instantiate: ") + cudaGetErrorString(e));
  }
  RBF_CK(cudaEventRecord(p->ev0, p->stream));
  int64_t done = 0;
  const int64_t graphed = pairs > kPairGraph ? ((pairs - 1) / kPairGraph) * kPairGraph : 0;
  for (; done < graphed; done += kPairGraph) {
    RBF_CK(cudaGraphLaunch(p->pair_graph, p->stream));
    p->launches += kPairGraph;
  }
  for (; done < pairs; ++done)
    RBF_TRY(launch_pair(p, static_cast<int>(done & 1), (!odd && done == pairs - 1) ? rbf::kNeedResidual : 0));
  if (odd) RBF_TRY(launch_step(p, static_cast<int>(pairs & 1), rbf::kNeedResidual));
  RBF_CK(cudaEventRecord(p->ev1, p->stream));
  *final_buf = static_cast<int>((pairs + (odd ? 1 : 0)) & 1);
  RBF_CK(cudaStreamSynchronize(p->stream));
  RBF_TRY(read_status(p));
  if (p->h_st->bad_step >= 0) {
    RBF_CK(cudaMemcpyAsync(p->U[0], p->u_init, sizeof(double) * p->N, cudaMemcpyDeviceToDevice, p->stream));
    RBF_CK(cudaMemcpyAsync(p->U[1], p->u_init, sizeof(double) * p->N, cudaMemcpyDeviceToDevice, p->stream));
    *fallback = true;
  }
  return RBF_OK;
}

int run_resident(rbf_plan* p, int64_t limit, bool steady, bool copy_back) {
  RBF_CK(cudaEventRecord(p->ev0, p->stream));
  if (limit > 0 && p->N_i > 0 && p->cluster_fn) {
    // buffer discipline makes copy-back and swap value-identical;
    // the cluster loop always swaps
    rbf::ClusterArgs a;
    a.W = p->W;
    a.C = p->C;
    a.F = p->F;
    a.dest = p->cluster_dest;
    a.U0 = p->U[0];
    a.U1 = p->U[1];
    a.n_rows = p->N_i;
    a.N = p->N;
    a.dst_base = p->B;
    a.limit = limit;
    a.n = p->n;
    a.flags = steady ? rbf::kSteady : 0;
    a.rpc = p->cluster_rpc;
    a.st = p->st;
    a.phase_cycles = nullptr;
    static unsigned long long* d_phase = nullptr;  // RBFFD_CLUSTER_PHASES=1: per-phase cycles to stderr
    const bool phases = std::getenv("RBFFD_CLUSTER_PHASES") != nullptr;
    if (phases) {
      if (!d_phase) RBF_CK(cudaMalloc(&d_phase, 4 * sizeof(unsigned long long)));
      RBF_CK(cudaMemsetAsync(d_phase, 0, 4 * sizeof(unsigned long long), p->stream));
      a.phase_cycles = d_phase;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p->cluster_q);
    cfg.blockDim = dim3(p->cluster_threads);
    cfg.dynamicSmemBytes = p->cluster_smem;
    cfg.stream = p->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p->cluster_q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RBF_CK(cudaLaunchKernelEx(&cfg, p->cluster_fn, a));
    ++p->launches;
    if (phases) {
      unsigned long long h[4];
      RBF_CK(cudaMemcpyAsync(h, d_phase, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
      RBF_CK(cudaStreamSynchronize(p->stream));
      std::fprintf(stderr, "[rbffd] cluster q=%d cycles/step: compute %.0f partials %.0f barrier %.0f decide %.0f\n",
                   p->cluster_q, double(h[0]) / limit, double(h[1]) / limit, double(h[2]) / limit,
                   double(h[3]) / limit);
    }
  } else if (limit > 0 && p->N_i > 0 && p->grid_fn) {
    rbf::GridArgs a;
    a.W = p->W;
    a.C = p->C;
    a.F = p->F;
    a.U0 = p->U[0];
    a.U1 = p->U[1];
    a.n_rows = p->N_i;
    a.dst_base = p->B;
    a.limit = limit;
    a.spc = p->grid_spc;
    a.spr = p->grid_spr;
    a.flags = steady ? rbf::kSteady : 0;
    a.st = p->st;
    a.red = p->grid_red;
    const rbf::PairArgs& gp = p->grid_pair.args;
    a.HW = p->grid_two ? gp.HW : nullptr;
    a.HC = gp.HC;
    a.HF = gp.HF;
    a.HR = gp.HR;
    a.L16 = gp.L16;
    a.hoff = gp.hoff;
    a.hsl = gp.hsl;
    a.u1_cap = gp.u1_cap;
    RBF_CK(cudaMemsetAsync(p->grid_red, 0, 7 * sizeof(unsigned long long), p->stream));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p->grid_ctas);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = p->grid_smem;
    cfg.stream = p->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: grid barrier per step
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RBF_CK(cudaLaunchKernelEx(&cfg, p->grid_fn, a));
    ++p->launches;
  } else if (limit > 0 && p->N_i > 0) {
    rbf::ResidentArgs a;
    a.W = p->W;
    a.C = p->C;
    a.F = p->F;
    a.U0 = p->U[0];
    a.U1 = p->U[1];
    a.n_rows = p->N_i;
    a.N = p->N;
    a.dst_base = p->B;
    a.limit = limit;
    a.n = p->n;
    a.flags = steady ? rbf::kSteady : 0;
    a.copy_back = copy_back ? 1 : 0;
    a.st = p->st;
    const int threads = static_cast<int>(std::min<int64_t>(1024, ((p->N_i + 31) / 32) * 32));
    p->resident_fn<<<1, threads, p->resident_smem, p->stream>>>(a);
    RBF_CK(cudaGetLastError());
    ++p->launches;
  }
  RBF_CK(cudaEventRecord(p->ev1, p->stream));
  return RBF_OK;
}

// The whole run in one cooperative launch of the persistent streaming loop;
// with kPublish (copy-back runs) the final field is published into both buffers.
int run_loop(rbf_plan* p, int64_t limit, bool steady, bool publish) {
  RBF_CK(cudaMemsetAsync(p->loop_red, 0, 7 * sizeof(unsigned long long), p->stream));
  rbf::LoopArgs L;
  L.U0 = p->U[0];
  L.U1 = p->U[1];
  L.limit = limit;
  L.flags = (steady ? rbf::kSteady : 0) | (publish ? rbf::kPublish : 0);
  L.red = p->loop_red;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->loop_grid);
  cfg.blockDim = dim3(p->tma_block);
  cfg.dynamicSmemBytes = p->loop_smem;
  cfg.stream = p->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: grid barrier per step
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RBF_CK(cudaEventRecord(p->ev0, p->stream));
  RBF_CK(cudaLaunchKernelEx(&cfg, p->loop_fn, p->args(), L, p->loop_geom));
  ++p->launches;
  RBF_CK(cudaEventRecord(p->ev1, p->stream));
  return RBF_OK;
}

}  // namespace

extern "C" {

int rbf_version(void) { return 1; }

int rbf_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(RBF_ERR_PARAM, "bad arguments");
  *out = nullptr;
  RBF_CK(cudaMallocHost(out, static_cast<size_t>(std::max<int64_t>(bytes, 1))));
  return RBF_OK;
}

void rbf_host_free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

const char* rbf_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace {

// Monomial table of degree m (graded lex, x-exponent descending; weights.py:35-68).
int fill_monomials(int degree, rbf::WeightArgs* wa) {
  if (degree < 0 || degree > 6) return fail(RBF_ERR_PARAM, "degree must be in [0, 6]");
  int k = 0;
  for (int t = 0; t <= degree; ++t)
    for (int ax = t; ax >= 0; --ax) {
      wa->ex[k] = ax;
      wa->ey[k] = t - ax;
      wa->lap0[k] = ((ax == 2 && t == 2) || (ax == 0 && t == 2)) ? 2.0 : 0.0;
      ++k;
    }
  wa->M = k;
  return RBF_OK;
}

// Launch the weight assembly for `cnt` rows (device arrays); returns the
// shared-memory size actually needed or an error.
int launch_assemble(const double* d_pos, const int* d_rows, long long cnt, long long k0, int n,
                    const rbf::WeightArgs& proto, double* d_w, long long* d_bad, unsigned char* d_status,
                    unsigned long long* d_nflag, cudaStream_t stream) {
  rbf::WeightArgs wa = proto;
  wa.pos = d_pos;
  wa.rows = d_rows;
  wa.cnt = cnt;
  wa.k0 = k0;
  wa.n = n;
  wa.w_out = d_w;
  wa.bad_row = d_bad;
  wa.status = d_status;
  wa.n_flagged = d_nflag;
  const size_t per_warp = rbf::assemble_smem_doubles(n, wa.M) * sizeof(double);
  int warps = static_cast<int>(std::min<size_t>(8, (200 * 1024) / per_warp));
  if (warps < 1) return fail(RBF_ERR_PARAM, "support too large for on-chip weight assembly");
  const size_t smem = per_warp * warps;
  RBF_CK(set_max_smem(rbf::assemble_weights_kernel));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long blocks = std::min<long long>((cnt + warps - 1) / warps, static_cast<long long>(sms) * 8);
  rbf::assemble_weights_kernel<<<static_cast<int>(std::max<long long>(blocks, 1)), 32 * warps, smem, stream>>>(wa);
  RBF_CK(cudaGetLastError());
  return RBF_OK;
}

// Kernel / loop selection shared by rbf_plan_create and rbf_plan_load: 16-bit
// ids, the resident / cluster loops, the TMA ring geometry.
int finish_plan(std::unique_ptr<rbf_plan>& p, uint32_t flags) {
  const int64_t N = p->N, N_i = p->N_i, B = p->B;
  const int n = p->n;
  const int device = p->device;
  const size_t sell = static_cast<size_t>(p->S) * 32 * n;
  // ---- kernel selection -----------------------------------------------------
  int cw = 8;         // consumer warps of the TMA ring kernel (per width, KernelSet::kCW)
  int cw_req = 0;     // RBFFD_TMA_CW=<KernelSet::kCWide>: the wide-CTA instantiation
  if (const char* e = std::getenv("RBFFD_TMA_CW")) cw_req = std::atoi(e);
  TmaFn tma_fn = nullptr;
  int rpl = 1;
  // 16-bit two-window ids for the TMA ring (only worth it when almost every
  // slice fits; the rest fall back to int32 ids read from HBM)
  bool idx16 = false;
  {
    StreamFn sf;
    ResidentFn rf;
    TmaFn tf = nullptr;
    int kn, r1, c1;
    pick_kernels(n, 1, false, &sf, &rf, &tf, &kn, &r1, &c1);
    const char* e = std::getenv("RBFFD_IDX16");
    // wide stencils (n > 32) run consumer-bound: the decode costs more than
    // the saved bytes (C4: 9.40e9 vs 9.72e9 upd/s, profiles/README.md)
    const bool want16 = (n <= 32) || (e && std::atoi(e) == 2);
    if (p->C16) {  // loaded from a plan file: already compressed
      idx16 = !(flags & RBF_NO_IDX16) && !(flags & RBF_STREAM_LDG);
    } else if (tf && want16 && N_i >= 4096 && !(flags & RBF_NO_IDX16) && !(flags & RBF_STREAM_LDG) &&
        !(e && std::atoi(e) == 0)) {
      RBF_TRY(dev_alloc(p.get(), &p->C16, sell));
      RBF_TRY(dev_alloc(p.get(), &p->meta, static_cast<size_t>(p->S)));
      unsigned long long* d_over = nullptr;
      RBF_TRY(pool_alloc(&d_over, 1, p->stream));
      RBF_CK(cudaMemsetAsync(d_over, 0, sizeof(unsigned long long), p->stream));
      const int blocks = static_cast<int>(std::min<int64_t>((p->S * 32 + 255) / 256, 148 * 16));
      rbf::compress_ids_kernel<<<blocks, 256, 0, p->stream>>>(p->C, N_i, n, p->C16, p->meta, d_over);
      RBF_CK(cudaGetLastError());
      unsigned long long over = 0;
      RBF_CK(cudaMemcpyAsync(&over, d_over, sizeof(over), cudaMemcpyDeviceToHost, p->stream));
      RBF_CK(cudaStreamSynchronize(p->stream));
      pool_free(d_over, p->stream);
      const bool force = e && std::atoi(e) == 2;  // tests: exercise the overflow path
      if (force || over * 20 <= static_cast<unsigned long long>(p->S)) {  // <= 5 % of the slices overflow
        idx16 = true;
        p->overflow_slices = static_cast<int64_t>(over);
      } else {
        pool_free(p->C16, p->stream);
        pool_free(p->meta, p->stream);
        p->device_bytes -= static_cast<int64_t>(sell * sizeof(unsigned short) + p->S * sizeof(int4));
      }
    }
  }
  pick_kernels(n, cw_req, idx16, &p->stream_fn, &p->resident_fn, &tma_fn, &p->kernel_n, &rpl, &cw);
  p->index_bits = idx16 ? 16 : 32;
  const int64_t rows_pad = ((N_i + 31) / 32) * 32;
  const size_t smem = static_cast<size_t>(rows_pad) * n * (sizeof(double) + sizeof(int)) +
                      static_cast<size_t>(rows_pad) * sizeof(double) +
                      2 * static_cast<size_t>(N) * sizeof(double);
  if (!(flags & RBF_NO_RESIDENT) && N_i > 0 && smem <= kResidentSmemMax - 1024) {
    if (set_max_smem(p->resident_fn) == cudaSuccess) {
      p->resident = true;
      p->resident_smem = smem;
    } else {
      cudaGetLastError();
    }
  }
  // cluster-resident loop: rows spread over Q SMs of one cluster (DSMEM halo)
  if (!(flags & RBF_NO_RESIDENT) && !(flags & RBF_NO_CLUSTER) && N_i >= 256) {
    // 4-8 CTAs measured best on the paper's Fig. 1 case (1.01 / 1.04 us/step vs
    // 1.30 at 16, profiles/README.md); more when a CTA would own more than 256
    // rows (register-resident variant) or its rows would not fit
    const size_t NU = static_cast<size_t>(((B + 1) & ~int64_t(1)) + N_i + 2);
    auto smem_for = [&](int qq) {
      const int rpc_ = static_cast<int>(((N_i + qq - 1) / qq + 1) & ~int64_t(1));
      return 2 * NU * 8 + 2 * 16 * 32 * 2 * 8 + static_cast<size_t>(n) * rpc_ * 12 + rpc_ * 8 + rpc_ * 4;
    };
    int q = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(4, (N_i + 255) / 256)));
    while (q < 16 && smem_for(q) > 200 * 1024) ++q;
    if (const char* e = std::getenv("RBFFD_CLUSTER")) q = std::max(2, std::min(16, std::atoi(e)));
    const int rpc = static_cast<int>(((N_i + q - 1) / q + 1) & ~int64_t(1));
    const size_t csmem = smem_for(q);
    ClusterFn cfn = nullptr;
    switch (n) {
#define RBF_CCASE(K) \
  case K:            \
    cfn = KernelSet<K>::cluster(rpc <= 256); \
    break;
      RBF_SPECIALISED(RBF_CCASE)
#undef RBF_CCASE
      default:
        cfn = KernelSet<0>::cluster(rpc <= 256);
    }
    const int threads = std::min(1024, ((rpc + 31) / 32) * 32);
    if (csmem <= 200 * 1024 && rpc <= 1024 &&
        set_max_smem(cfn) == cudaSuccess &&
        (q <= 8 || cudaFuncSetAttribute(cfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(q);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = csmem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = q;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, cfn, &cfg) == cudaSuccess && nclusters >= 1) {
        RBF_TRY(dev_alloc(p.get(), &p->cluster_dest, static_cast<size_t>(N_i)));
        RBF_CK(cudaMemsetAsync(p->cluster_dest, 0, sizeof(unsigned int) * N_i, p->stream));
        const int blocks = static_cast<int>(std::min<int64_t>((N_i * n + 255) / 256, 148 * 16));
        rbf::cluster_dest_kernel<<<blocks, 256, 0, p->stream>>>(p->C, N_i, n, B, rpc, p->cluster_dest);
        RBF_CK(cudaGetLastError());
        p->cluster_fn = cfn;
        p->cluster_q = q;
        p->cluster_rpc = rpc;
        p->cluster_threads = threads;
        p->cluster_smem = csmem;
        p->resident = true;
      }
    }
    cudaGetLastError();
  }
  int sms = 148, per_sm = 1;
  RBF_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // grid-resident loop: every SM holds its share of the rows in shared memory
  const char* grid_env = std::getenv("RBFFD_GRID");
  if (!p->resident && !(flags & RBF_NO_RESIDENT) && N_i > 0 && !(grid_env && std::atoi(grid_env) == 0)) {
    GridFn gfn = nullptr, gfn2 = nullptr;
    switch (n) {
#define RBF_GCASE(K) \
  case K:            \
    gfn = KernelSet<K>::grid(false); \
    gfn2 = KernelSet<K>::grid(true); \
    break;
      RBF_SPECIALISED(RBF_GCASE)
#undef RBF_GCASE
      default:
        break;
    }
    // rows beyond what shared memory holds are re-read every step from L2
    // (evict_last); allowed while that part stays well inside the L2
    const int64_t spc = (p->S + sms - 1) / sms;
    const size_t slice_bytes = static_cast<size_t>(n) * 32 * 12 + 32 * 8;
    int optin = 0;
    RBF_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    const int64_t spr = std::min<int64_t>(spc, static_cast<int64_t>((static_cast<size_t>(optin) - 2048) / slice_bytes));
    const size_t gsmem = static_cast<size_t>(spr) * slice_bytes;
    const double l2_part = static_cast<double>(std::max<int64_t>(0, p->S - spr * sms)) * slice_bytes;
    double l2_cap = 88.0e6;  // measured crossover ~90-100 MB (profiles/README.md)
    if (const char* e = std::getenv("RBFFD_GRID_L2_MB")) l2_cap = std::atof(e) * 1.0e6;
    if (gfn && spr >= 1 && l2_part <= l2_cap && set_max_smem(gfn) == cudaSuccess) {
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gfn, 512, gsmem) == cudaSuccess && occ >= 1) {
        RBF_TRY(dev_alloc(p.get(), &p->grid_red, 7));
        p->grid_fn = gfn;
        p->grid_spc = static_cast<int>(spc);
        p->grid_spr = static_cast<int>(spr);
        p->grid_smem = gsmem;
        // two steps per grid barrier when every row is on chip: the pair
        // tables with one tile per CTA (pair_kernels.cu), U1 after the rows
        // (measured: 1.1-1.2x up to ~1.3e6 stencil entries, where the grid
        // barrier dominates a step; even or slower above; RBFFD_GRID_PAIR=0/1
        // forces it off / on)
        const char* gp_env = std::getenv("RBFFD_GRID_PAIR");
        const bool gp_want = gp_env ? std::atoi(gp_env) == 1 : N_i * static_cast<int64_t>(n) <= 1300000;
        if (spr == spc && gp_want) {
          bool tok = false;
          RBF_TRY(rbf::pair_build(p->args(), 1, 1, sms, 0, p->stream, &p->grid_pair, &tok, static_cast<int>(spc),
                                  true));
          const size_t u1b = static_cast<size_t>(p->grid_pair.args.u1_cap) * sizeof(double);
          if (tok && gsmem + u1b + 2048 <= static_cast<size_t>(optin) && set_max_smem(gfn2) == cudaSuccess &&
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gfn2, 512, gsmem + u1b) == cudaSuccess && occ >= 1) {
            p->grid_two = true;
            p->grid_fn = gfn2;
            p->grid_smem = gsmem + u1b;
          } else if (tok) {
            rbf::pair_free(&p->grid_pair, p->stream);
          }
        }
        p->grid_ctas = static_cast<int>((p->S + spc - 1) / spc);
        p->resident = true;
      }
    }
    cudaGetLastError();
  }
  p->variant = p->grid_fn ? 4 : (p->cluster_fn ? 3 : (p->resident ? 0 : 1));
  if (tma_fn && !(flags & RBF_STREAM_LDG) && N_i > 0) {
    // ring geometry: ~24 KB stages (~30 KB for 16-bit ids at n=30), as many
    // as fit in ~200 KB of shared memory.  Slices per stage, measured: n=15 4 >
    // 5 (0.4 %) > 8; n=30 3 = +9 % over 2; n=56 1 > 2 (profiles/README.md).
    // Only the measured widths get the larger stage.
    const int slice = n * 32 * (8 + p->index_bits / 8) + 32 * 8 + (p->index_bits == 16 ? 16 : 0);
    int sps = std::max(1, (p->index_bits == 16 && n == 30 ? 30000 : 24576) / slice);
    if (const char* e = std::getenv("RBFFD_TMA_SPS")) sps = std::max(1, std::atoi(e));
    sps = std::max(rpl, (sps / rpl) * rpl);
    const int stage = sps * slice;
    // as many stages as the shared memory holds: a deeper ring covers more HBM
    // latency (C2: 8 -> 11 stages +2.2 %, C3 +1 %, C4 8 -> 10 +1.5 %;
    // profiles/README.md)
    int optin_s = 0;
    RBF_CK(cudaDeviceGetAttribute(&optin_s, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    cudaFuncAttributes tfa;
    RBF_CK(cudaFuncGetAttributes(&tfa, tma_fn));
    const size_t ring_room = static_cast<size_t>(optin_s) - tfa.sharedSizeBytes - 2 * 16 * sizeof(uint64_t) - 256;
    int stages = std::max(2, std::min(16, static_cast<int>(ring_room / stage)));
    if (const char* e = std::getenv("RBFFD_TMA_STAGES")) stages = std::max(2, std::min(16, std::atoi(e)));
    const size_t smem_t = 2 * 16 * sizeof(uint64_t) + static_cast<size_t>(stages) * stage;
    if (smem_t <= kResidentSmemMax && set_max_smem(tma_fn) == cudaSuccess) {
      p->tma_fn = tma_fn;
      p->tma_geom = rbf::TmaGeom{sps, stages, 0, 0};
      // ring-fill chunks stay L2-resident (TmaGeom::res): 8 for n <= 20 (C2
      // 29.5 -> 28.4 us with the round-2 kernel, profiles/r02/c2_geom_sweep.log),
      // 1.5 x stages above (round-1 sweep)
      p->tma_geom.res = n <= 20 ? 8 : (3 * stages) / 2;
      if (const char* e = std::getenv("RBFFD_L2_RES_CHUNKS")) p->tma_geom.res = std::atoll(e);
      p->tma_smem = smem_t;
      p->tma_block = 32 * (cw + 1);
      const int64_t chunks = (p->S + sps - 1) / sps;
      int occ = 1;
      RBF_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_fn, p->tma_block, smem_t));
      p->grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(chunks, int64_t(sms) * std::max(occ, 1))));
      if (!p->resident && !p->cluster_fn) p->variant = 2;
    } else {
      cudaGetLastError();
    }
  }
  // persistent streaming loop (stream_loop_kernel): the TMA step's ring in one
  // cooperative launch per run; RBFFD_PERSIST=0 keeps the graph + PDL loop
  const char* persist_env = std::getenv("RBFFD_PERSIST");
  if (p->tma_fn && !p->resident && !(flags & RBF_NO_PERSIST) && !(persist_env && std::atoi(persist_env) == 0)) {
    LoopFn lfn = nullptr;
    switch (n) {
#define RBF_LCASE(K) \
  case K:            \
    lfn = KernelSet<K>::loop(p->index_bits == 16); \
    break;
      RBF_SPECIALISED(RBF_LCASE)
#undef RBF_LCASE
      default:
        break;
    }
    int optin_l = 0;
    RBF_CK(cudaDeviceGetAttribute(&optin_l, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    if (lfn && set_max_smem(lfn) == cudaSuccess) {
      cudaFuncAttributes lfa;
      RBF_CK(cudaFuncGetAttributes(&lfa, lfn));
      const int slice = n * 32 * (8 + p->index_bits / 8) + 32 * 8 + (p->index_bits == 16 ? 16 : 0);
      // slices per stage of the persistent loop: its ring never drains, so
      // larger stages pay (C2: 5 -> 24.7 us per step vs 4 -> 25.7; C4: 2 ->
      // 2.592 ms vs 1 -> 2.707; profiles/r02/loop_geom_sweep.log)
      int lsps = p->tma_geom.sps;
      if (p->index_bits == 16 && n <= 20) lsps = std::max(1, 30000 / slice);
      if (p->index_bits == 32) lsps = std::max(1, 45000 / slice);
      if (const char* e = std::getenv("RBFFD_LOOP_SPS")) lsps = std::max(1, std::atoi(e));
      const int stage = lsps * slice;
      const size_t room = static_cast<size_t>(optin_l) - lfa.sharedSizeBytes - 2 * 16 * sizeof(uint64_t) - 256;
      int stages = std::min(16, static_cast<int>(room / stage));
      if (const char* e = std::getenv("RBFFD_LOOP_STAGES")) stages = std::max(2, std::min(stages, std::atoi(e)));
      const size_t lsmem = 2 * 16 * sizeof(uint64_t) + static_cast<size_t>(stages) * stage;
      int occ = 0;
      if (stages >= 2 &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lfn, p->tma_block, lsmem) == cudaSuccess &&
          occ >= 1) {
        RBF_TRY(dev_alloc(p.get(), &p->loop_red, 7));
        p->loop_fn = lfn;
        p->loop_smem = lsmem;
        p->loop_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((p->S + lsps - 1) / lsps,
                                                                                 int64_t(sms) * occ)));
        int lres = 0;
        if (const char* e = std::getenv("RBFFD_LOOP_RES")) lres = std::max(0, std::atoi(e));
        // L2 policy of the stream: evict_first keeps the field buffers
        // L2-resident while they fit (C2: 24.7 us vs 29.3 with evict_normal);
        // once they do not, evict_normal is 0.7 % faster with 16-bit ids
        // (m=2 N=1e7 260.0 vs 261.8 us, C3 480.0 vs 483.5) and 0.9 % slower
        // with int32 ids (C4 2.600 vs 2.576 ms): profiles/r02/loop_policy_ab.log
        int lpol = (p->index_bits == 16 && 16 * N > (int64_t(64) << 20)) ? 1 : 0;
        if (const char* e = std::getenv("RBFFD_LOOP_POLICY")) lpol = std::max(0, std::min(2, std::atoi(e)));
        p->loop_geom = rbf::TmaGeom{lsps, stages, lpol, lres};
      }
    }
    cudaGetLastError();
  }
  // two-step tile kernel for fixed-step runs (pair_kernels.cu)
  // (Runs only when no on-chip loop applies: the grid-resident loop wins at
  // these sizes.)  Measured (profiles/README.md, tools/pair_sweep.py): 1.1-1.5x faster up to
  // ~1e6 stencil entries, where the per-launch grid dependency dominates;
  // even or slower above, where both are bound by the streamed bytes and the
  // pair kernel's extra phase-2 work.  RBF_PAIR / RBFFD_PAIR=1 force it on.
  const char* pair_env = std::getenv("RBFFD_PAIR");
  const bool pair_force = (flags & RBF_PAIR) || (pair_env && std::atoi(pair_env) == 1);
  const bool pair_off = (flags & RBF_NO_PAIR) || (pair_env && std::atoi(pair_env) == 0);
  const bool pair_auto = N_i * static_cast<int64_t>(n) <= kPairAutoEntries;
  if (p->tma_fn && p->index_bits == 16 && !pair_off && (pair_force || (pair_auto && !p->resident))) {
    int tpc = 4;
    if (const char* e = std::getenv("RBFFD_PAIR_TILES")) tpc = std::max(1, std::atoi(e));
    int optin = 0;
    RBF_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    bool ok = false;
    RBF_TRY(rbf::pair_build(p->args(), p->tma_geom.sps, tpc, sms, static_cast<size_t>(optin) - 2048,
                            p->stream, &p->pair, &ok));
    if (ok && set_max_smem(p->pair.fn) == cudaSuccess) {
      p->pair_ok = true;
      p->pair_forced = pair_force;
      p->device_bytes += p->pair.halo_slices * 32LL * (12LL * n + 12) + p->S * 32LL * n * 2;
    } else {
      if (ok) rbf::pair_free(&p->pair, p->stream);
      cudaGetLastError();
    }
  }
  if (p->tma_fn && std::getenv("RBFFD_TRACE")) {  // diagnostics: CTA timelines of up to 4096 steps
    p->trace_cap = 4096;
    const int tg = std::max(p->grid, p->loop_grid);
    RBF_TRY(dev_alloc(p.get(), &p->trace, static_cast<size_t>(p->trace_cap) * tg * 4));
    RBF_CK(cudaMemsetAsync(p->trace, 0, sizeof(unsigned long long) * p->trace_cap * tg * 4, p->stream));
  }
  if (!p->tma_fn) {
    RBF_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p->stream_fn, kStreamBlock, 0));
    per_sm = std::max(per_sm, 1);
    const int64_t need = (N_i + kStreamBlock - 1) / kStreamBlock;
    p->grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sms) * per_sm)));
  }
  RBF_CK(cudaStreamSynchronize(p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

int plan_create_impl(rbf_plan** out, int64_t N, int64_t N_i, int32_t n, const int64_t* interior,
                     const int64_t* rows, const double* weights, const double* f_int,
                     const double* positions, int32_t device, uint32_t flags, int32_t degree,
                     uint8_t* row_status = nullptr) {
  const bool assemble = degree >= 0;
  if (!out) return fail(RBF_ERR_PARAM, "out is NULL");
  *out = nullptr;
  if (N < 1 || N > std::numeric_limits<int32_t>::max())
    return fail(RBF_ERR_PARAM, "N must be in [1, 2^31-1]");
  if (N_i < 0 || N_i > N) return fail(RBF_ERR_PARAM, "need 0 <= N_i <= N");
  if (n < 1) return fail(RBF_ERR_PARAM, "support size n must be >= 1");
  if (N_i > 0 && (!interior || !rows || (!weights && !assemble)))
    return fail(RBF_ERR_PARAM, "interior/rows/weights must be non-NULL");
  const bool morton = (flags & RBF_RENUMBER_MORTON) != 0;
  if ((morton || assemble) && !positions)
    return fail(RBF_ERR_PARAM, "RBF_RENUMBER_MORTON / weight assembly need positions");
  rbf::WeightArgs wproto = {};
  if (assemble) RBF_TRY(fill_monomials(degree, &wproto));
  if (assemble && n < wproto.M) return fail(RBF_ERR_PARAM, "support size below the monomial count");

  // ---- validation (host, parallel: parameter errors before any CUDA call) ----
  PhaseTimer timer;
  const int64_t B = N - N_i;
  // range check + membership marks with plain stores; the ids are distinct
  // iff exactly N_i marks end up set (a duplicate marks one entry twice)
  std::vector<uint8_t> seen(static_cast<size_t>(N), 0);
  int bad_range = 0, ident = morton ? 0 : 1;
#pragma omp parallel for schedule(static) reduction(| : bad_range) reduction(& : ident)
  for (int64_t k = 0; k < N_i; ++k) {
    const int64_t v = interior[k];
    if (v < 0 || v >= N) bad_range = 1;
    else seen[v] = 1;
    if (v != B + k) ident = 0;
  }
  if (bad_range) return fail(RBF_ERR_PARAM, "interior node id out of range");
  int64_t marked = 0;
#pragma omp parallel for schedule(static) reduction(+ : marked)
  for (int64_t i = 0; i < N; ++i) marked += seen[i];
  if (marked != N_i) return fail(RBF_ERR_PARAM, "interior node ids must be distinct");
  const bool identity = ident != 0;
  timer.mark("validate (host)");
  timer.mark("validate + renumber (host)");

  std::unique_ptr<rbf_plan> p(new rbf_plan());
  p->device = device;
  p->N = N;
  p->N_i = N_i;
  p->B = B;
  p->n = n;
  p->S = (N_i + 31) / 32;
  p->renumbered = !identity;
  p->pdl = (flags & RBF_NO_PDL) == 0;
  RBF_CK(cudaSetDevice(device));
  RBF_TRY(prepare_pool(device));
  RBF_CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  RBF_CK(cudaEventCreate(&p->ev0));
  RBF_CK(cudaEventCreate(&p->ev1));
  RBF_CK(status_alloc(&p->h_st));
  RBF_TRY(dev_alloc(p.get(), &p->st, 1));
  const size_t sell = static_cast<size_t>(p->S) * 32 * n;
  RBF_TRY(dev_alloc(p.get(), &p->W, sell));
  RBF_TRY(dev_alloc(p.get(), &p->C, sell));
  RBF_TRY(dev_alloc(p.get(), &p->F, static_cast<size_t>(p->S) * 32));
  RBF_TRY(dev_alloc(p.get(), &p->U[0], static_cast<size_t>(N)));
  RBF_TRY(dev_alloc(p.get(), &p->U[1], static_cast<size_t>(N)));
  // padding lanes of the last slice are never consumed (every kernel masks
  // r >= N_i), so only the field buffers are cleared
  RBF_CK(cudaMemsetAsync(p->U[0], 0, static_cast<size_t>(N) * sizeof(double), p->stream));
  RBF_CK(cudaMemsetAsync(p->U[1], 0, static_cast<size_t>(N) * sizeof(double), p->stream));
  timer.mark("alloc");

  // ---- device-side SELL-32 packing, in row chunks through pinned staging ----
  long long* d_row_of_k = nullptr;
  if (!identity) {
    // ---- renumbering on the device: Morton keys, stable radix sort, maps ----
    RBF_TRY(dev_alloc(p.get(), &p->new_id, static_cast<size_t>(N)));
    RBF_TRY(dev_alloc(p.get(), &p->tmp, static_cast<size_t>(N)));
    RBF_TRY(dev_alloc(p.get(), &p->row_of_k, static_cast<size_t>(std::max<int64_t>(1, N_i))));
    d_row_of_k = p->row_of_k;
    long long* d_int = nullptr;
    unsigned char* d_seen = nullptr;
    int* d_flag = nullptr;
    RBF_TRY(pool_alloc(&d_int, static_cast<size_t>(std::max<int64_t>(1, N_i)), p->stream));
    RBF_TRY(pool_alloc(&d_seen, static_cast<size_t>(N), p->stream));
    RBF_TRY(pool_alloc(&d_flag, static_cast<size_t>(N), p->stream));
    // 8-byte elements through the pinned staging pair (pageable copies run at
    // ~11 GB/s and block the host); doubles here are only bit copies
    RBF_TRY(staged_h2d(reinterpret_cast<double*>(d_int), reinterpret_cast<const double*>(interior),
                       static_cast<size_t>(N_i), p->stream, device));
    RBF_CK(cudaMemcpyAsync(d_seen, seen.data(), N, cudaMemcpyHostToDevice, p->stream));
    const int blocks = static_cast<int>(std::min<int64_t>((std::max(N, N_i) + 255) / 256, 148 * 16));
    long long* d_order = nullptr;
    RBF_TRY(pool_alloc(&d_order, static_cast<size_t>(std::max<int64_t>(1, N_i)), p->stream));
    if (morton && N_i > 1) {
      double* d_pos = nullptr;
      unsigned long long *d_key = nullptr, *d_key2 = nullptr;
      long long* d_val = nullptr;
      RBF_TRY(pool_alloc(&d_pos, static_cast<size_t>(2 * N), p->stream));
      RBF_TRY(pool_alloc(&d_key, static_cast<size_t>(N_i), p->stream));
      RBF_TRY(pool_alloc(&d_key2, static_cast<size_t>(N_i), p->stream));
      RBF_TRY(pool_alloc(&d_val, static_cast<size_t>(N_i), p->stream));
      RBF_TRY(staged_h2d(d_pos, positions, static_cast<size_t>(2 * N), p->stream, device));
      // bounding box on the device (the host pass over 16 B/node was ~0.3 ms at C2)
      const int nbb = static_cast<int>(std::min<int64_t>((N + 255) / 256, 148 * 4));
      double* d_bb = nullptr;
      RBF_TRY(pool_alloc(&d_bb, static_cast<size_t>(4 * nbb), p->stream));
      rbf::bounds_partial_kernel<<<nbb, 256, 0, p->stream>>>(d_pos, N, d_bb);
      RBF_CK(cudaGetLastError());
      rbf::morton_keys_dev_kernel<<<blocks, 256, 0, p->stream>>>(d_pos, d_int, N_i, d_bb, nbb, d_key, d_val);
      RBF_CK(cudaGetLastError());
      pool_free(d_bb, p->stream);
      size_t tb = 0;
      RBF_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, d_key, d_key2, d_val, d_order, N_i, 0, 42, p->stream));
      void* d_tb = nullptr;
      RBF_TRY(pool_alloc(reinterpret_cast<unsigned char**>(&d_tb), std::max<size_t>(tb, 16), p->stream));
      RBF_CK(cub::DeviceRadixSort::SortPairs(d_tb, tb, d_key, d_key2, d_val, d_order, N_i, 0, 42, p->stream));
      pool_free(d_tb, p->stream);
      pool_free(d_pos, p->stream);
      pool_free(d_key, p->stream);
      pool_free(d_key2, p->stream);
      pool_free(d_val, p->stream);
    } else {
      rbf::iota_kernel<<<blocks, 256, 0, p->stream>>>(d_order, N_i);
      RBF_CK(cudaGetLastError());
    }
    // row_of_k[order[r]] = r;  new_id: non-interior nodes keep their relative
    // order at 0..B-1 (exclusive scan of !seen), interior node k -> B + row_of_k[k]
    rbf::invert_order_kernel<<<blocks, 256, 0, p->stream>>>(d_order, N_i, d_row_of_k);
    rbf::not_seen_kernel<<<blocks, 256, 0, p->stream>>>(d_seen, N, d_flag);
    RBF_CK(cudaGetLastError());
    size_t tb = 0;
    RBF_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_flag, p->new_id, static_cast<int>(N), p->stream));
    void* d_tb = nullptr;
    RBF_TRY(pool_alloc(reinterpret_cast<unsigned char**>(&d_tb), std::max<size_t>(tb, 16), p->stream));
    RBF_CK(cub::DeviceScan::ExclusiveSum(d_tb, tb, d_flag, p->new_id, static_cast<int>(N), p->stream));
    rbf::interior_ids_kernel<<<blocks, 256, 0, p->stream>>>(d_int, d_row_of_k, N_i, B, p->new_id);
    RBF_CK(cudaGetLastError());
    pool_free(d_tb, p->stream);
    pool_free(d_order, p->stream);
    pool_free(d_int, p->stream);
    pool_free(d_seen, p->stream);
    pool_free(d_flag, p->stream);
  }
  seen.clear();
  seen.shrink_to_fit();
  int* d_err = nullptr;
  RBF_TRY(pool_alloc(&d_err, 1, p->stream));
  RBF_CK(cudaMemsetAsync(d_err, 0, sizeof(int), p->stream));
  double* d_pos = nullptr;
  long long* d_bad = nullptr;           // {first flagged row, flagged-row count}
  unsigned char* d_status = nullptr;    // per reference row: 0 ok, 1 host check, 2 degenerate
  if (assemble && N_i > 0) {
    RBF_TRY(pool_alloc(&d_pos, static_cast<size_t>(2 * N), p->stream));
    RBF_CK(cudaMemcpyAsync(d_pos, positions, sizeof(double) * 2 * N, cudaMemcpyHostToDevice, p->stream));
    RBF_TRY(pool_alloc(&d_bad, 2, p->stream));
    RBF_TRY(pool_alloc(&d_status, static_cast<size_t>(N_i), p->stream));
    const long long init[2] = {std::numeric_limits<long long>::max(), 0};
    RBF_CK(cudaMemcpyAsync(d_bad, init, sizeof(init), cudaMemcpyHostToDevice, p->stream));
    RBF_CK(cudaStreamSynchronize(p->stream));  // `init` lives on this stack frame
  }
  bool ids_ok = true;
  if (N_i > 0) {
    Staging& sg = staging();
    std::lock_guard<std::mutex> lock(sg.mu);
    RBF_TRY(staging_acquire(sg, device));
    const size_t row_bytes = static_cast<size_t>(n) * (assemble ? 4 : 12) + 8;
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(N_i, static_cast<int64_t>(sg.cap / row_bytes)));
    double* d_w = nullptr;
    int* d_c = nullptr;
    double* d_f = nullptr;
    RBF_TRY(pool_alloc(&d_w, static_cast<size_t>(cap) * n, p->stream));
    RBF_TRY(pool_alloc(&d_c, static_cast<size_t>(cap) * n, p->stream));
    RBF_TRY(pool_alloc(&d_f, static_cast<size_t>(cap), p->stream));
    int64_t c = 0;
    for (int64_t k0 = 0; k0 < N_i && ids_ok; k0 += cap, ++c) {
      const int b = static_cast<int>(c & 1);
      const int64_t cnt = std::min<int64_t>(cap, N_i - k0);
      const int64_t total = cnt * n;
      RBF_CK(cudaEventSynchronize(sg.ev[b]));  // the previous DMA out of this buffer is done
      unsigned char* hb = sg.buf[b];
      int32_t* hc = reinterpret_cast<int32_t*>(hb);
      double* hf = reinterpret_cast<double*>(hb + ((static_cast<size_t>(total) * 4 + 15) & ~size_t(15)));
      double* hw = hf + cnt;
      int bad = 0;
      const int64_t* src_c = rows + k0 * n;
      const double* src_w = assemble ? nullptr : weights + k0 * n;
      // one pass per thread over a contiguous range: ids range-checked and
      // narrowed, weights copied, both with non-temporal stores (the staging
      // buffer is only read again by the DMA: no read-for-ownership traffic)
#pragma omp parallel reduction(| : bad)
      {
        const int64_t T = omp_get_num_threads(), t = omp_get_thread_num();
        const int64_t lo = total * t / T, hi = total * (t + 1) / T;
        bad |= narrow_ids_nt(hc + lo, src_c + lo, hi - lo, N);
        if (src_w) copy_f64_nt(hw + lo, src_w + lo, hi - lo);
        _mm_sfence();
      }
      if (bad) {
        ids_ok = false;
        break;
      }
      if (f_int) std::memcpy(hf, f_int + k0, sizeof(double) * cnt);
      else std::memset(hf, 0, sizeof(double) * cnt);  // forcing set later (rbf_set_forcing)
      RBF_CK(cudaMemcpyAsync(d_c, hc, sizeof(int32_t) * total, cudaMemcpyHostToDevice, p->stream));
      RBF_CK(cudaMemcpyAsync(d_f, hf, sizeof(double) * cnt, cudaMemcpyHostToDevice, p->stream));
      if (assemble) {  // weights computed on the device, never on the host
        RBF_TRY(launch_assemble(d_pos, d_c, cnt, k0, n, wproto, d_w, d_bad, d_status,
                                reinterpret_cast<unsigned long long*>(d_bad + 1), p->stream));
      } else {
        RBF_CK(cudaMemcpyAsync(d_w, hw, sizeof(double) * total, cudaMemcpyHostToDevice, p->stream));
      }
      RBF_CK(cudaEventRecord(sg.ev[b], p->stream));
      const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 32));
      rbf::pack_rows_kernel<<<blocks, 256, 0, p->stream>>>(d_w, d_c, d_f, k0, cnt, n, d_row_of_k,
                                                           p->new_id, N, p->W, p->C, p->F, d_err);
      RBF_CK(cudaGetLastError());
    }
    RBF_CK(cudaStreamSynchronize(p->stream));
    pool_free(d_w, p->stream);
    pool_free(d_c, p->stream);
    pool_free(d_f, p->stream);
  }
  if (!ids_ok) {
    pool_free(d_err, p->stream);
    pool_free(d_pos, p->stream);
    pool_free(d_bad, p->stream);
    pool_free(d_status, p->stream);
    rbf_plan_destroy(p.release());
    return fail(RBF_ERR_PARAM, "stencil node id out of range");
  }
  timer.mark("upload + pack");
  int h_err = 0;
  RBF_CK(cudaMemcpy(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  pool_free(d_err, p->stream);
  if (d_bad) {
    long long hb[2] = {0, 0};
    RBF_CK(cudaMemcpy(hb, d_bad, sizeof(hb), cudaMemcpyDeviceToHost));
    int verdict = RBF_OK;
    std::string msg;
    if (hb[1] != 0) {  // flagged rows: the caller decides on the status-1 rows (exact 2-norm check)
      std::vector<uint8_t> local;
      uint8_t* stv = row_status;
      if (!stv) {
        local.resize(static_cast<size_t>(N_i));
        stv = local.data();
      }
      RBF_CK(cudaMemcpy(stv, d_status, static_cast<size_t>(N_i), cudaMemcpyDeviceToHost));
      int64_t first_deg = -1;
      for (int64_t k = 0; k < N_i && first_deg < 0; ++k)
        if (stv[k] == 2) first_deg = k;
      if (!(flags & RBF_ACCEPT_ILLCOND) || first_deg >= 0) {
        verdict = RBF_ERR_ILLCOND;
        msg = "weight assembly flagged " + std::to_string(hb[1]) + " stencil(s), first at interior row " +
              std::to_string(hb[0]) + (first_deg >= 0 ? " (degenerate: zero pivot, non-finite weights or "
                                                        "condition estimate above n * 1e14)"
                                                      : " (condition estimate above 1e10: needs the exact check)");
      }
    }
    pool_free(d_bad, p->stream);
    pool_free(d_status, p->stream);
    pool_free(d_pos, p->stream);
    if (verdict != RBF_OK) {
      pool_free(d_err, p->stream);
      rbf_plan_destroy(p.release());
      return fail(verdict, msg);
    }
  }
  if (h_err) {
    rbf_plan_destroy(p.release());
    return fail(RBF_ERR_PARAM, "stencil node id out of range");
  }

  RBF_TRY(finish_plan(p, flags));
  timer.mark("kernel selection");
  *out = p.release();
  return RBF_OK;
}

}  // namespace

extern "C" {

int rbf_plan_create(rbf_plan** out, int64_t N, int64_t N_i, int32_t n, const int64_t* interior,
                    const int64_t* rows, const double* weights, const double* f_int,
                    const double* positions, int32_t device, uint32_t flags) {
  return plan_create_impl(out, N, N_i, n, interior, rows, weights, f_int, positions, device, flags, -1);
}

int rbf_plan_create_assembled(rbf_plan** out, int64_t N, int64_t N_i, int32_t n, int32_t degree,
                              const int64_t* interior, const int64_t* rows, const double* positions,
                              const double* f_int, int32_t device, uint32_t flags, uint8_t* row_status) {
  if (degree < 0) return fail(RBF_ERR_PARAM, "degree must be >= 0");
  return plan_create_impl(out, N, N_i, n, interior, rows, nullptr, f_int, positions, device, flags,
                          degree, row_status);
}

int rbf_assemble_weights(const double* positions, int64_t N, const int64_t* rows, int64_t N_i,
                         int32_t n, int32_t degree, double* weights_out, int64_t* bad_row,
                         uint8_t* row_status, int32_t device) {
  if (!positions || (N_i > 0 && (!rows || !weights_out)) || n < 1 || N < 1)
    return fail(RBF_ERR_PARAM, "bad arguments");
  rbf::WeightArgs wproto = {};
  RBF_TRY(fill_monomials(degree, &wproto));
  if (n < wproto.M) return fail(RBF_ERR_PARAM, "support size below the monomial count");
  if (bad_row) *bad_row = -1;
  if (N_i == 0) return RBF_OK;
  for (int64_t e = 0; e < N_i * n; ++e)
    if (rows[e] < 0 || rows[e] >= N) return fail(RBF_ERR_PARAM, "stencil node id out of range");
  RBF_CK(cudaSetDevice(device));
  RBF_TRY(prepare_pool(device));
  cudaStream_t st;
  RBF_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double* d_pos = nullptr;
  int* d_rows = nullptr;
  double* d_w = nullptr;
  long long* d_bad = nullptr;  // {first flagged row, flagged-row count}
  unsigned char* d_status = nullptr;
  const int64_t cap = std::min<int64_t>(N_i, std::max<int64_t>(1, (int64_t(1) << 24) / n));
  const long long none[2] = {std::numeric_limits<long long>::max(), 0};
  std::vector<int32_t> ids(static_cast<size_t>(cap) * n);
  int rc = RBF_OK;
  if (pool_alloc(&d_pos, static_cast<size_t>(2 * N), st) != RBF_OK ||
      pool_alloc(&d_rows, static_cast<size_t>(cap) * n, st) != RBF_OK ||
      pool_alloc(&d_w, static_cast<size_t>(cap) * n, st) != RBF_OK || pool_alloc(&d_bad, 2, st) != RBF_OK ||
      pool_alloc(&d_status, static_cast<size_t>(N_i), st) != RBF_OK)
    rc = RBF_ERR_CUDA;
  if (rc == RBF_OK && (cudaMemcpyAsync(d_bad, none, sizeof(none), cudaMemcpyHostToDevice, st) != cudaSuccess ||
                       cudaMemcpyAsync(d_pos, positions, sizeof(double) * 2 * N, cudaMemcpyHostToDevice, st) != cudaSuccess))
    rc = fail(RBF_ERR_CUDA, "upload positions");
  for (int64_t k0 = 0; k0 < N_i && rc == RBF_OK; k0 += cap) {
    const int64_t cnt = std::min<int64_t>(cap, N_i - k0);
    if (cudaStreamSynchronize(st) != cudaSuccess) {  // `ids` is reused below
      rc = fail(RBF_ERR_CUDA, "assembly");
      break;
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < cnt * n; ++e) ids[e] = static_cast<int32_t>(rows[k0 * n + e]);
    if (cudaMemcpyAsync(d_rows, ids.data(), sizeof(int32_t) * cnt * n, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      rc = fail(RBF_ERR_CUDA, "upload rows");
      break;
    }
    rc = launch_assemble(d_pos, d_rows, cnt, k0, n, wproto, d_w, d_bad, d_status,
                         reinterpret_cast<unsigned long long*>(d_bad + 1), st);
    if (rc == RBF_OK && cudaMemcpyAsync(weights_out + k0 * n, d_w, sizeof(double) * cnt * n,
                                        cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = fail(RBF_ERR_CUDA, "download weights");
  }
  if (rc == RBF_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(RBF_ERR_CUDA, "assembly");
  long long hb[2] = {none[0], 0};
  if (rc == RBF_OK && cudaMemcpy(hb, d_bad, sizeof(hb), cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(RBF_ERR_CUDA, "assembly status");
  if (rc == RBF_OK && hb[1] != 0 && row_status &&
      cudaMemcpy(row_status, d_status, static_cast<size_t>(N_i), cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(RBF_ERR_CUDA, "assembly status");
  if (rc == RBF_OK && hb[1] == 0 && row_status) std::memset(row_status, 0, static_cast<size_t>(N_i));
  pool_free(d_pos, st);
  pool_free(d_rows, st);
  pool_free(d_w, st);
  pool_free(d_bad, st);
  pool_free(d_status, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != RBF_OK) return rc;
  if (hb[1] != 0) {
    if (bad_row) *bad_row = hb[0];
    return fail(RBF_ERR_ILLCOND, "weight assembly flagged " + std::to_string(hb[1]) +
                                     " stencil(s), first at interior row " + std::to_string(hb[0]));
  }
  return RBF_OK;
}

int rbf_knn(const double* positions, int64_t N, int32_t n, int64_t* neighbors_out, int32_t device) {
  return rbf_knn_subset(positions, N, n, nullptr, N, neighbors_out, device);
}

int rbf_knn_subset(const double* positions, int64_t N, int32_t n, const int64_t* query_ids, int64_t n_query,
                   int64_t* neighbors_out, int32_t device) {
  if (!positions || !neighbors_out) return fail(RBF_ERR_PARAM, "NULL argument");
  if (n_query < 0 || (!query_ids && n_query != N)) return fail(RBF_ERR_PARAM, "bad query set");
  if (query_ids)
    for (int64_t q = 0; q < n_query; ++q)
      if (query_ids[q] < 0 || query_ids[q] >= N) return fail(RBF_ERR_PARAM, "query node id out of range");
  if (N < 1 || N > std::numeric_limits<int32_t>::max()) return fail(RBF_ERR_PARAM, "N must be in [1, 2^31-1]");
  if (n < 1 || n > N) return fail(RBF_ERR_PARAM, "support size n=" + std::to_string(n) + " outside [1, N]");
  if (n > 128) return fail(RBF_ERR_PARAM, "support size above 128 is not supported on the GPU path");
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (int64_t i = 0; i < N; ++i) {
    const double x = positions[2 * i], y = positions[2 * i + 1];
    if (!std::isfinite(x) || !std::isfinite(y)) return fail(RBF_ERR_PARAM, "non-finite node position");
    xmin = std::min(xmin, x);
    xmax = std::max(xmax, x);
    ymin = std::min(ymin, y);
    ymax = std::max(ymax, y);
  }
  rbf::KnnGrid g;
  const double w = std::max(xmax - xmin, 1e-300), h = std::max(ymax - ymin, 1e-300);
  double c = std::sqrt(2.0 * w * h / static_cast<double>(N));  // ~2 points per cell
  if (!(c > 0)) c = std::max(w, h);
  c = std::max(c, std::max(w, h) / 32768.0);
  g.c = c;
  g.inv_c = 1.0 / c;
  g.x0 = xmin;
  g.y0 = ymin;
  g.nx = static_cast<int>(w / c) + 1;
  g.ny = static_cast<int>(h / c) + 1;
  const int64_t cells = static_cast<int64_t>(g.nx) * g.ny;
  RBF_CK(cudaSetDevice(device));
  RBF_TRY(prepare_pool(device));
  cudaStream_t st;
  RBF_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double* d_pos = nullptr;
  int* d_cell = nullptr;
  int* d_sorted = nullptr;
  unsigned int* d_count = nullptr;
  unsigned int* d_start = nullptr;
  long long* d_out = nullptr;
  long long* d_q = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(n_query, 1), (int64_t(1) << 25) / n));
  int rc = RBF_OK;
  auto ck = [&](cudaError_t e, const char* what) {
    if (rc == RBF_OK && e != cudaSuccess) rc = fail(RBF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  ck(cudaMallocAsync(&d_pos, sizeof(double) * 2 * N, st), "alloc");
  ck(cudaMallocAsync(&d_cell, sizeof(int) * N, st), "alloc");
  ck(cudaMallocAsync(&d_sorted, sizeof(int) * N, st), "alloc");
  ck(cudaMallocAsync(&d_count, sizeof(unsigned int) * (cells + 1), st), "alloc");
  ck(cudaMallocAsync(&d_start, sizeof(unsigned int) * (cells + 1), st), "alloc");
  ck(cudaMallocAsync(&d_out, sizeof(long long) * chunk * n, st), "alloc");
  ck(cudaMemcpyAsync(d_pos, positions, sizeof(double) * 2 * N, cudaMemcpyHostToDevice, st), "upload");
  if (query_ids && n_query > 0) {
    ck(cudaMallocAsync(&d_q, sizeof(long long) * n_query, st), "alloc");
    ck(cudaMemcpyAsync(d_q, query_ids, sizeof(long long) * n_query, cudaMemcpyHostToDevice, st), "upload");
  }
  ck(cudaMemsetAsync(d_count, 0, sizeof(unsigned int) * (cells + 1), st), "memset");
  const int blocks = static_cast<int>(std::min<int64_t>((N + 255) / 256, 148 * 16));
  if (rc == RBF_OK) {
    rbf::knn_count_kernel<<<blocks, 256, 0, st>>>(d_pos, N, g, d_cell, d_count);
    ck(cudaGetLastError(), "count");
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_count, d_start, static_cast<int>(cells + 1), st), "scan");
    ck(cudaMallocAsync(&d_tmp, std::max<size_t>(tmp_bytes, 16), st), "alloc");
    ck(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_count, d_start, static_cast<int>(cells + 1), st), "scan");
    ck(cudaMemcpyAsync(d_count, d_start, sizeof(unsigned int) * (cells + 1), cudaMemcpyDeviceToDevice, st), "copy");
    rbf::knn_fill_kernel<<<blocks, 256, 0, st>>>(d_cell, N, d_count, d_sorted);
    ck(cudaGetLastError(), "fill");
  }
  for (int64_t q0 = 0; q0 < n_query && rc == RBF_OK; q0 += chunk) {
    const int64_t nq = std::min<int64_t>(chunk, n_query - q0);
    const int qb = static_cast<int>(std::min<int64_t>((nq + 127) / 128, 148 * 32));
    if (n <= 16) rbf::knn_query_kernel<16><<<qb, 128, 0, st>>>(d_pos, N, g, d_start, d_sorted, n, q0, nq, d_out, d_q);
    else if (n <= 32) rbf::knn_query_kernel<32><<<qb, 128, 0, st>>>(d_pos, N, g, d_start, d_sorted, n, q0, nq, d_out, d_q);
    else if (n <= 64) rbf::knn_query_kernel<64><<<qb, 128, 0, st>>>(d_pos, N, g, d_start, d_sorted, n, q0, nq, d_out, d_q);
    else rbf::knn_query_kernel<128><<<qb, 128, 0, st>>>(d_pos, N, g, d_start, d_sorted, n, q0, nq, d_out, d_q);
    ck(cudaGetLastError(), "query");
    ck(cudaMemcpyAsync(neighbors_out + q0 * n, d_out, sizeof(long long) * nq * n, cudaMemcpyDeviceToHost, st),
       "download");
    ck(cudaStreamSynchronize(st), "knn");
  }
  cudaFreeAsync(d_pos, st);
  cudaFreeAsync(d_cell, st);
  cudaFreeAsync(d_sorted, st);
  cudaFreeAsync(d_count, st);
  cudaFreeAsync(d_start, st);
  cudaFreeAsync(d_out, st);
  if (d_q) cudaFreeAsync(d_q, st);
  if (d_tmp) cudaFreeAsync(d_tmp, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}

int rbf_plan_weight_row_sum_max(rbf_plan* p, double* out) {
  if (!p || !out) return fail(RBF_ERR_PARAM, "NULL argument");
  RBF_CK(cudaSetDevice(p->device));
  double* d = nullptr;
  RBF_TRY(pool_alloc(&d, 1, p->stream));
  RBF_CK(cudaMemsetAsync(d, 0, sizeof(double), p->stream));
  const int blocks = static_cast<int>(std::min<int64_t>((p->N_i + 255) / 256, 148 * 8));
  if (p->N_i > 0) {
    rbf::row_abs_sum_max_kernel<<<blocks, 256, 0, p->stream>>>(p->W, p->N_i, p->n, d);
    RBF_CK(cudaGetLastError());
  }
  RBF_CK(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  pool_free(d, p->stream);
  return RBF_OK;
}

// ---- plan files: the packed device layout on disk ------
struct PlanFileHeader {
  char magic[8];  // "RBFPLAN1"
  int32_t version, n;
  int64_t N, N_i, B, S;
  int32_t index_bits, renumbered;
  int64_t overflow_slices;
  int64_t reserved[4];
};

// One staging chunk <-> the file at byte offset `off`, as kFilePieces
// positional reads/writes on host threads: a single fread/fwrite is one memcpy
// stream out of the page cache (~4.5 GB/s); several in parallel are not.
static constexpr int kFilePieces = 8;
static bool chunk_io(int fd, unsigned char* buf, size_t len, off_t off, bool save) {
  const size_t piece = (len + kFilePieces - 1) / kFilePieces;
  int ok = 1;
#pragma omp parallel for schedule(static, 1) num_threads(kFilePieces) reduction(& : ok)
  for (int t = 0; t < kFilePieces; ++t) {
    size_t a = std::min(len, t * piece), e = std::min(len, a + piece);
    while (a < e) {
      const ssize_t r = save ? ::pwrite(fd, buf + a, e - a, off + static_cast<off_t>(a))
                             : ::pread(fd, buf + a, e - a, off + static_cast<off_t>(a));
      if (r <= 0) { ok = 0; break; }
      a += static_cast<size_t>(r);
    }
  }
  return ok != 0;
}

// Device <-> file through the two pinned staging buffers: the disk read of
// chunk k+1 overlaps the H2D copy of chunk k (load), the D2H copy of chunk k+1
// overlaps the write of chunk k (save).  Reads and writes are positional on
// the FILE's descriptor from its current offset; the FILE is repositioned past
// the section at the end (fflush first so no buffered header bytes are lost).
static int file_io(std::FILE* f, void* dev, size_t bytes, bool save, cudaStream_t stream) {
  if (std::fflush(f) != 0) return fail(RBF_ERR_PARAM, "plan file: flush failed");
  const int fd = fileno(f);
  const off_t base = ftello(f);
  if (base < 0) return fail(RBF_ERR_PARAM, "plan file: not seekable");
  Staging& sg = staging();
  std::lock_guard<std::mutex> lock(sg.mu);
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  RBF_TRY(staging_acquire(sg, dev_id));
  unsigned char* d = static_cast<unsigned char*>(dev);
  const size_t nchunks = (bytes + sg.cap - 1) / sg.cap;
  auto len_of = [&](size_t c) { return std::min(sg.cap, bytes - c * sg.cap); };
  if (save) {
    if (nchunks) {
      RBF_CK(cudaMemcpyAsync(sg.buf[0], d, len_of(0), cudaMemcpyDeviceToHost, stream));
      RBF_CK(cudaEventRecord(sg.ev[0], stream));
    }
    for (size_t c = 0; c < nchunks; ++c) {
      const int b = static_cast<int>(c & 1);
      if (c + 1 < nchunks) {  // start the next D2H into the other buffer
        RBF_CK(cudaMemcpyAsync(sg.buf[b ^ 1], d + (c + 1) * sg.cap, len_of(c + 1), cudaMemcpyDeviceToHost, stream));
        RBF_CK(cudaEventRecord(sg.ev[b ^ 1], stream));
      }
      RBF_CK(cudaEventSynchronize(sg.ev[b]));
      if (!chunk_io(fd, static_cast<unsigned char*>(sg.buf[b]), len_of(c), base + static_cast<off_t>(c * sg.cap), true)) {
        cudaStreamSynchronize(stream);
        return fail(RBF_ERR_PARAM, "plan file: write failed");
      }
    }
    RBF_CK(cudaStreamSynchronize(stream));
    if (fseeko(f, base + static_cast<off_t>(bytes), SEEK_SET) != 0) return fail(RBF_ERR_PARAM, "plan file: seek failed");
    return RBF_OK;
  }
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = static_cast<int>(c & 1);
    RBF_CK(cudaEventSynchronize(sg.ev[b]));  // the H2D out of this buffer (chunk c-2) is done
    if (!chunk_io(fd, static_cast<unsigned char*>(sg.buf[b]), len_of(c), base + static_cast<off_t>(c * sg.cap), false)) {
      cudaStreamSynchronize(stream);
      return fail(RBF_ERR_PARAM, "plan file: truncated");
    }
    RBF_CK(cudaMemcpyAsync(d + c * sg.cap, sg.buf[b], len_of(c), cudaMemcpyHostToDevice, stream));
    RBF_CK(cudaEventRecord(sg.ev[b], stream));
  }
  RBF_CK(cudaStreamSynchronize(stream));
  if (fseeko(f, base + static_cast<off_t>(bytes), SEEK_SET) != 0) return fail(RBF_ERR_PARAM, "plan file: seek failed");
  return RBF_OK;
}

int rbf_plan_save(const rbf_plan* cp, const char* path) {
  if (!cp || !path) return fail(RBF_ERR_PARAM, "NULL argument");
  rbf_plan* p = const_cast<rbf_plan*>(cp);
  RBF_CK(cudaSetDevice(p->device));
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return fail(RBF_ERR_PARAM, std::string("cannot open ") + path);
  PlanFileHeader h = {};
  std::memcpy(h.magic, "RBFPLAN1", 8);
  h.version = 1;
  h.n = p->n;
  h.N = p->N;
  h.N_i = p->N_i;
  h.B = p->B;
  h.S = p->S;
  h.index_bits = p->C16 ? 16 : 32;
  h.renumbered = p->renumbered ? 1 : 0;
  h.overflow_slices = p->overflow_slices;
  int rc = std::fwrite(&h, sizeof(h), 1, f) == 1 ? RBF_OK : fail(RBF_ERR_PARAM, "plan file: write failed");
  const size_t sell = static_cast<size_t>(p->S) * 32 * p->n;
  if (rc == RBF_OK) rc = file_io(f, p->W, sell * sizeof(double), true, p->stream);
  if (rc == RBF_OK) rc = file_io(f, p->C, sell * sizeof(int), true, p->stream);
  if (rc == RBF_OK) rc = file_io(f, p->F, static_cast<size_t>(p->S) * 32 * sizeof(double), true, p->stream);
  if (rc == RBF_OK && p->C16) {
    rc = file_io(f, p->C16, sell * sizeof(unsigned short), true, p->stream);
    if (rc == RBF_OK) rc = file_io(f, p->meta, static_cast<size_t>(p->S) * sizeof(int4), true, p->stream);
  }
  if (rc == RBF_OK && p->renumbered) {
    rc = file_io(f, p->new_id, static_cast<size_t>(p->N) * sizeof(int), true, p->stream);
    if (rc == RBF_OK) rc = file_io(f, p->row_of_k, static_cast<size_t>(p->N_i) * sizeof(long long), true, p->stream);
  }
  if (std::fclose(f) != 0 && rc == RBF_OK) rc = fail(RBF_ERR_PARAM, "plan file: close failed");
  return rc;
}

int rbf_plan_load(rbf_plan** out, const char* path, int32_t device, uint32_t flags) {
  if (!out || !path) return fail(RBF_ERR_PARAM, "NULL argument");
  *out = nullptr;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail(RBF_ERR_PARAM, std::string("cannot open ") + path);
  PlanFileHeader h = {};
  if (std::fread(&h, sizeof(h), 1, f) != 1 || std::memcmp(h.magic, "RBFPLAN1", 8) != 0 || h.version != 1 ||
      h.n < 1 || h.N < 1 || h.N_i < 0 || h.N_i > h.N || h.S != (h.N_i + 31) / 32 || h.B != h.N - h.N_i) {
    std::fclose(f);
    return fail(RBF_ERR_PARAM, "not an rbffd_b200 plan file (or a different version)");
  }
  std::unique_ptr<rbf_plan> p(new rbf_plan());
  p->device = device;
  p->N = h.N;
  p->N_i = h.N_i;
  p->B = h.B;
  p->n = h.n;
  p->S = h.S;
  p->renumbered = h.renumbered != 0;
  p->pdl = (flags & RBF_NO_PDL) == 0;
  p->overflow_slices = h.overflow_slices;
  int rc = RBF_OK;
  auto step = [&](int r) { if (rc == RBF_OK) rc = r; };
  step(cudaSetDevice(device) == cudaSuccess ? RBF_OK : fail(RBF_ERR_CUDA, "cudaSetDevice"));
  step(prepare_pool(device));
  if (rc == RBF_OK) {
    step(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) == cudaSuccess ? RBF_OK : fail(RBF_ERR_CUDA, "stream"));
    step(cudaEventCreate(&p->ev0) == cudaSuccess ? RBF_OK : fail(RBF_ERR_CUDA, "event"));
    step(cudaEventCreate(&p->ev1) == cudaSuccess ? RBF_OK : fail(RBF_ERR_CUDA, "event"));
    step(status_alloc(&p->h_st) == cudaSuccess
             ? RBF_OK : fail(RBF_ERR_CUDA, "host status"));
  }
  const size_t sell = static_cast<size_t>(p->S) * 32 * p->n;
  if (rc == RBF_OK) step(dev_alloc(p.get(), &p->st, 1));
  if (rc == RBF_OK) step(dev_alloc(p.get(), &p->W, sell));
  if (rc == RBF_OK) step(dev_alloc(p.get(), &p->C, sell));
  if (rc == RBF_OK) step(dev_alloc(p.get(), &p->F, static_cast<size_t>(p->S) * 32));
  if (rc == RBF_OK) step(dev_alloc(p.get(), &p->U[0], static_cast<size_t>(p->N)));
  if (rc == RBF_OK) step(dev_alloc(p.get(), &p->U[1], static_cast<size_t>(p->N)));
  if (rc == RBF_OK) step(file_io(f, p->W, sell * sizeof(double), false, p->stream));
  if (rc == RBF_OK) step(file_io(f, p->C, sell * sizeof(int), false, p->stream));
  if (rc == RBF_OK) step(file_io(f, p->F, static_cast<size_t>(p->S) * 32 * sizeof(double), false, p->stream));
  if (rc == RBF_OK && h.index_bits == 16) {
    step(dev_alloc(p.get(), &p->C16, sell));
    step(dev_alloc(p.get(), &p->meta, static_cast<size_t>(p->S)));
    step(file_io(f, p->C16, sell * sizeof(unsigned short), false, p->stream));
    step(file_io(f, p->meta, static_cast<size_t>(p->S) * sizeof(int4), false, p->stream));
  }
  if (rc == RBF_OK && p->renumbered) {
    step(dev_alloc(p.get(), &p->new_id, static_cast<size_t>(p->N)));
    step(dev_alloc(p.get(), &p->tmp, static_cast<size_t>(p->N)));
    step(dev_alloc(p.get(), &p->row_of_k, static_cast<size_t>(std::max<int64_t>(1, p->N_i))));
    step(file_io(f, p->new_id, static_cast<size_t>(p->N) * sizeof(int), false, p->stream));
    step(file_io(f, p->row_of_k, static_cast<size_t>(p->N_i) * sizeof(long long), false, p->stream));
  }
  // the file must end exactly here (a longer file is not what save wrote)
  if (rc == RBF_OK && std::fgetc(f) != EOF) rc = fail(RBF_ERR_PARAM, "plan file: trailing bytes after the payload");
  std::fclose(f);
  // payload range check on the device before any step kernel can gather with it
  if (rc == RBF_OK && p->N_i > 0) {
    unsigned int* d_err = nullptr;
    step(pool_alloc(&d_err, 1, p->stream));
    unsigned int h_err = 0;
    auto ck = [&](cudaError_t e, const char* what) {
      if (rc == RBF_OK && e != cudaSuccess) rc = fail(RBF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    if (rc == RBF_OK) {
      ck(cudaMemsetAsync(d_err, 0, sizeof(unsigned int), p->stream), "memset");
      const int blocks = static_cast<int>(std::min<int64_t>((p->S * 32 * p->n + 255) / 256, 148 * 16));
      rbf::validate_plan_kernel<<<blocks, 256, 0, p->stream>>>(p->C, p->C16, p->meta, p->N_i, p->n, p->N,
                                                               p->new_id, p->row_of_k, d_err);
      ck(cudaGetLastError(), "validate_plan_kernel");
      ck(cudaMemcpyAsync(&h_err, d_err, sizeof(h_err), cudaMemcpyDeviceToHost, p->stream), "d2h");
      ck(cudaStreamSynchronize(p->stream), "validate plan");
      pool_free(d_err, p->stream);
      if (rc == RBF_OK && h_err)
        rc = fail(RBF_ERR_PARAM, "plan file: corrupt payload (node ids / renumbering out of range, code " +
                                     std::to_string(h_err) + ")");
    }
  }
  if (rc == RBF_OK) {
    RBF_CK(cudaMemsetAsync(p->U[0], 0, sizeof(double) * p->N, p->stream));
    RBF_CK(cudaMemsetAsync(p->U[1], 0, sizeof(double) * p->N, p->stream));
    step(finish_plan(p, flags));
  }
  if (rc != RBF_OK) {
    rbf_plan_destroy(p.release());
    return rc;
  }
  *out = p.release();
  return RBF_OK;
}

int rbf_set_forcing(rbf_plan* p, const double* f_int) {
  if (!p || (p->N_i > 0 && !f_int)) return fail(RBF_ERR_PARAM, "NULL argument");
  if (p->N_i == 0) return RBF_OK;
  RBF_CK(cudaSetDevice(p->device));
  const bool staged = static_cast<size_t>(p->N_i) * sizeof(double) >= kFieldStagedMin;
  double* dst = p->renumbered ? p->tmp : p->F;
  if (staged) RBF_TRY(staged_h2d(dst, f_int, static_cast<size_t>(p->N_i), p->stream, p->device));
  else RBF_CK(cudaMemcpyAsync(dst, f_int, sizeof(double) * p->N_i, cudaMemcpyHostToDevice, p->stream));
  if (p->renumbered) {
    // Renumbered: F[row_of_k[k]] = f_int[k].
    const int blocks = static_cast<int>(std::min<int64_t>((p->N_i + 255) / 256, 148 * 16));
    rbf::scatter_rows_kernel<<<blocks, 256, 0, p->stream>>>(p->tmp, p->row_of_k, p->N_i, p->F);
    RBF_CK(cudaGetLastError());
  }
  // the two-step tables carry a copy of the halo rows' forcing
  if (p->pair_ok) RBF_TRY(rbf::pair_refresh_forcing(&p->pair, p->stream));
  if (p->grid_two) RBF_TRY(rbf::pair_refresh_forcing(&p->grid_pair, p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

int rbf_set_field(rbf_plan* p, const double* u) {
  if (!p || !u) return fail(RBF_ERR_PARAM, "NULL argument");
  RBF_CK(cudaSetDevice(p->device));
  const size_t bytes = sizeof(double) * p->N;
  const bool staged = bytes >= kFieldStagedMin;
  if (!p->new_id) {
    if (staged) RBF_TRY(staged_h2d(p->U[0], u, static_cast<size_t>(p->N), p->stream, p->device));
    else RBF_CK(cudaMemcpyAsync(p->U[0], u, bytes, cudaMemcpyHostToDevice, p->stream));
    RBF_CK(cudaMemcpyAsync(p->U[1], p->U[0], bytes, cudaMemcpyDeviceToDevice, p->stream));
  } else {
    if (staged) RBF_TRY(staged_h2d(p->tmp, u, static_cast<size_t>(p->N), p->stream, p->device));
    else RBF_CK(cudaMemcpyAsync(p->tmp, u, bytes, cudaMemcpyHostToDevice, p->stream));
    const int blocks = static_cast<int>(std::min<int64_t>((p->N + 255) / 256, 148 * 16));
    rbf::scatter_field_kernel<<<blocks, 256, 0, p->stream>>>(p->tmp, p->new_id, p->N, p->U[0], p->U[1]);
    RBF_CK(cudaGetLastError());
  }
  p->cur = 0;
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

int rbf_get_field(rbf_plan* p, double* u) {
  if (!p || !u) return fail(RBF_ERR_PARAM, "NULL argument");
  RBF_CK(cudaSetDevice(p->device));
  const size_t bytes = sizeof(double) * p->N;
  const double* src = p->U[p->cur];
  if (p->new_id) {
    const int blocks = static_cast<int>(std::min<int64_t>((p->N + 255) / 256, 148 * 16));
    rbf::gather_field_kernel<<<blocks, 256, 0, p->stream>>>(p->U[p->cur], p->new_id, p->N, p->tmp);
    RBF_CK(cudaGetLastError());
    src = p->tmp;
  }
  if (bytes >= kFieldStagedMin) return staged_d2h(u, src, static_cast<size_t>(p->N), p->stream, p->device);
  RBF_CK(cudaMemcpyAsync(u, src, bytes, cudaMemcpyDeviceToHost, p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

}  // extern "C"

namespace {
// numpy's pairwise summation tree over [lo, lo+n) (loops_utils.h.src):
// blocks of <= 128 elements are leaves, larger ranges split at n/2 rounded
// down to a multiple of 8.
constexpr long long kPwBlock = 128;
void pw_blocks(long long lo, long long n, std::vector<long long>& starts) {
  if (n <= kPwBlock) {
    starts.push_back(lo);
    return;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  pw_blocks(lo, n2, starts);
  pw_blocks(lo + n2, n - n2, starts);
}
double pw_combine(long long n, const double* sums, size_t& next) {
  if (n <= kPwBlock) return sums[next++];
  long long n2 = n / 2;
  n2 -= n2 % 8;
  const double a = pw_combine(n2, sums, next);
  const double b = pw_combine(n - n2, sums, next);
  return a + b;
}
}  // namespace

extern "C" {

int rbf_error_norms(rbf_plan* p, const double* exact, double* linf, double* l2) {
  if (!p || !exact || !linf || !l2) return fail(RBF_ERR_PARAM, "NULL argument");
  RBF_CK(cudaSetDevice(p->device));
  const long long N = p->N;
  if (p->norm_start.empty()) {
    pw_blocks(0, N, p->norm_start);
    p->norm_start.push_back(N);
    const size_t nb = p->norm_start.size() - 1;
    RBF_TRY(pool_alloc(&p->d_norm_start, nb + 1, p->stream));
    RBF_TRY(pool_alloc(&p->d_norm_sum, nb + 1, p->stream));
    RBF_CK(cudaMemcpyAsync(p->d_norm_start, p->norm_start.data(), sizeof(long long) * (nb + 1),
                           cudaMemcpyHostToDevice, p->stream));
    RBF_CK(cudaStreamSynchronize(p->stream));  // the host vector may be reallocated later
  }
  const long long nb = static_cast<long long>(p->norm_start.size()) - 1;
  double* ex = p->tmp ? p->tmp : p->norm_exact;
  if (!ex) {
    RBF_TRY(pool_alloc(&p->norm_exact, static_cast<size_t>(N), p->stream));
    ex = p->norm_exact;
  }
  if (static_cast<size_t>(N) * sizeof(double) >= kFieldStagedMin)
    RBF_TRY(staged_h2d(ex, exact, static_cast<size_t>(N), p->stream, p->device));
  else
    RBF_CK(cudaMemcpyAsync(ex, exact, sizeof(double) * N, cudaMemcpyHostToDevice, p->stream));
  unsigned long long* d_max = reinterpret_cast<unsigned long long*>(p->d_norm_sum + nb);
  RBF_CK(cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), p->stream));
  const int eblocks = static_cast<int>(std::max<long long>(1, std::min<long long>((N + 255) / 256, 148 * 16)));
  rbf::norm_diff_kernel<<<eblocks, 256, 0, p->stream>>>(p->U[p->cur], p->new_id, ex, N, d_max);
  const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>((nb + 127) / 128, 148 * 8)));
  rbf::norm_blocks_kernel<<<blocks, 128, 0, p->stream>>>(ex, p->d_norm_start, nb, p->d_norm_sum);
  RBF_CK(cudaGetLastError());
  std::vector<double> sums(static_cast<size_t>(nb) + 1);
  RBF_CK(cudaMemcpyAsync(sums.data(), p->d_norm_sum, sizeof(double) * (nb + 1), cudaMemcpyDeviceToHost,
                         p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  size_t next = 0;
  const double total = pw_combine(N, sums.data(), next);  // np.add.reduce(diff**2)
  unsigned long long mb;
  std::memcpy(&mb, &sums[nb], sizeof(mb));
  double mx;
  std::memcpy(&mx, &mb, sizeof(mx));
  *linf = mx;                          // np.max(np.abs(diff))
  *l2 = std::sqrt(total / static_cast<double>(N));  // math.sqrt(mean)
  return RBF_OK;
}

int rbf_run(rbf_plan* p, double dt, int64_t steps, int32_t mode, double tol, int64_t max_steps,
            int32_t copy_back, int64_t* steps_done, double* residual, int32_t* has_residual,
            int64_t* bad_step, double* device_seconds) {
  if (!p) return fail(RBF_ERR_PARAM, "plan is NULL");
  if (mode != RBF_MODE_FIXED && mode != RBF_MODE_STEADY) return fail(RBF_ERR_PARAM, "bad mode");
  const bool steady = mode == RBF_MODE_STEADY;
  const int64_t limit = steady ? max_steps : steps;  // solver.py:192
  if (limit < 0) return fail(RBF_ERR_PARAM, "steps/max_steps must be >= 0");
  RBF_CK(cudaSetDevice(p->device));
  RBF_TRY(normalise_current(p));
  RBF_TRY(reset_status(p, dt, tol));
  int rc;
  int pair_buf = -1;  // >= 0: the pair path ran and left the field in U[pair_buf]
  PhaseTimer timer;
  bool published = p->resident;  // the loop publishes the final field into both buffers
  bool looped = false;            // the persistent streaming loop ran
  if (p->resident) {
    rc = run_resident(p, limit, steady, copy_back != 0);
  } else if (p->loop_fn && limit >= 1 && !(p->pair_forced && !steady && limit >= 2)) {
    rc = run_loop(p, limit, steady, copy_back != 0);
    published = copy_back != 0;  // else the final field is in U[st.step & 1]
    looped = true;
  } else if (p->pair_ok && !steady && limit >= 2) {
    bool fallback = false;
    int final_buf = 0;
    rc = run_pair(p, limit, &fallback, &final_buf);
    if (rc == RBF_OK && fallback) {
      RBF_TRY(reset_status(p, dt, tol));
      rc = run_streaming(p, limit, steady, copy_back != 0);
    } else if (rc == RBF_OK) {
      pair_buf = final_buf;
      if (copy_back && final_buf != 0) {  // copy-back runs end with the field in U[0]
        RBF_CK(cudaMemcpyAsync(p->U[0], p->U[1], sizeof(double) * p->N, cudaMemcpyDeviceToDevice, p->stream));
        pair_buf = 0;
      }
    }
  } else {
    rc = run_streaming(p, limit, steady, copy_back != 0);
  }
  if (rc != RBF_OK) return rc;
  RBF_CK(cudaStreamSynchronize(p->stream));
  timer.mark("run total (incl. sync)");
  RBF_TRY(read_status(p));
  float ms = 0.f;
  RBF_CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  const rbf::DevStatus s = *p->h_st;
  if (p->trace && limit > 0) {  // RBFFD_TRACE: append {grid, steps, [steps][grid][4] ns} to the file
    const int64_t n_tr = std::min<int64_t>(limit, p->trace_cap);
    const int tg = looped ? p->loop_grid : p->grid;
    std::vector<unsigned long long> h(static_cast<size_t>(n_tr) * tg * 4);
    RBF_CK(cudaMemcpy(h.data(), p->trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (std::FILE* f = std::fopen(std::getenv("RBFFD_TRACE"), "ab")) {
      const int64_t hdr[2] = {looped ? -tg : tg, n_tr};  // negative: persistent-loop layout
      std::fwrite(hdr, sizeof(hdr), 1, f);
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      std::fclose(f);
    }
  }

  int64_t done = limit > 0 && p->N_i > 0 ? s.step : limit;
  bool have_res = false;
  double res = 0.0;
  if (p->N_i == 0 && limit > 0) {
    // no interior rows: every step is the identity, residual 0
    done = steady ? 1 : limit;
    have_res = true;
    res = 0.0 / dt;
  } else if (s.last_res_step >= 0 && s.last_res_step == done - 1) {
    double m;
    std::memcpy(&m, &s.last_res_bits, sizeof(m));
    res = m / dt;  // solver.py:209/:211, same IEEE division as numpy
    have_res = true;
  }
  if (device_seconds) *device_seconds = ms * 1e-3;
  if (bad_step) *bad_step = s.bad_step;
  if (s.bad_step >= 0) {
    // field of the failing step's u2 (solver.py:201)
    p->cur = copy_back ? 0 : static_cast<int>((s.bad_step + 1) & 1);
    if (published) p->cur = 0;  // resident / cluster / persistent loops publish into both buffers
    if (steps_done) *steps_done = s.bad_step;
    if (has_residual) *has_residual = 0;
    return fail(RBF_ERR_INSTABILITY, "time loop unstable at step " + std::to_string(s.bad_step));
  }
  p->cur = (copy_back || published) ? 0 : static_cast<int>(done & 1);
  if (pair_buf >= 0) p->cur = pair_buf;
  if (steps_done) *steps_done = done;
  if (residual) *residual = have_res ? res : 0.0;
  if (has_residual) *has_residual = have_res ? 1 : 0;
  if (steady && done == max_steps && (!have_res || !(res <= tol))) {
    return fail(RBF_ERR_TIMEOUT, "no steady state after " + std::to_string(done) + " steps");
  }
  return RBF_OK;
}

int rbf_step(rbf_plan* p, double dt) {
  if (!p) return fail(RBF_ERR_PARAM, "plan is NULL");
  RBF_CK(cudaSetDevice(p->device));
  RBF_TRY(reset_status(p, dt, 0.0));
  RBF_TRY(launch_step(p, p->cur, 0));
  RBF_TRY(read_status(p));
  p->cur ^= 1;
  if (p->h_st->bad_step >= 0) return fail(RBF_ERR_INSTABILITY, "explicit step produced non-finite values");
  return RBF_OK;
}

int rbf_step_kernel(const double* u1, double* u2, int64_t N, const int64_t* interior,
                    const int64_t* rows, const double* weights, const double* f_int, int64_t N_i,
                    int32_t n, double dt, int64_t chunk, uint8_t* flags, int32_t device) {
  if (!u1 || !u2 || (N_i > 0 && !flags)) return fail(RBF_ERR_PARAM, "NULL argument");
  if (chunk < 1) return fail(RBF_ERR_PARAM, "chunk must be >= 1");
  rbf_plan* p = nullptr;
  int rc = rbf_plan_create(&p, N, N_i, n, interior, rows, weights, f_int, nullptr, device,
                           RBF_NO_RESIDENT);
  if (rc != RBF_OK) return rc;
  rc = rbf_set_field(p, u1);
  if (rc == RBF_OK) {
    rc = rbf_step(p, dt);
    if (rc == RBF_ERR_INSTABILITY) rc = RBF_OK;  // reported through flags, like the numba kernel
  }
  std::vector<double> out;
  if (rc == RBF_OK) {
    out.resize(static_cast<size_t>(N));
    rc = rbf_get_field(p, out.data());
  }
  rbf_plan_destroy(p);
  if (rc != RBF_OK) return rc;
  const int64_t n_chunks = std::max<int64_t>(1, (N_i + chunk - 1) / chunk);
  for (int64_t c = 0; c < n_chunks; ++c) flags[c] = 0;
  for (int64_t k = 0; k < N_i; ++k) {
    const double v = out[interior[k]];
    u2[interior[k]] = v;  // the numba kernel writes u2[interior] only (solver.py:308)
    if (!std::isfinite(v)) flags[k / chunk] = 1;
  }
  return RBF_OK;
}

int rbf_plan_get_info(const rbf_plan* p, rbf_plan_info* info) {
  if (!p || !info) return fail(RBF_ERR_PARAM, "NULL argument");
  info->N = p->N;
  info->N_i = p->N_i;
  info->n = p->n;
  info->device = p->device;
  info->resident = p->resident ? 1 : 0;
  info->renumbered = p->renumbered ? 1 : 0;
  info->kernel_n = p->kernel_n;
  info->grid = p->grid;
  info->block = p->tma_fn ? p->tma_block : kStreamBlock;
  info->variant = p->variant;
  info->device_bytes = p->device_bytes;
  info->bytes_per_step = p->N_i * (12LL * p->n + 24);
  info->launches = p->launches;
  info->index_bits = p->index_bits;
  // bytes the streaming step actually moves: 16-bit ids, the per-slice window
  // bases, and int32 ids of the overflow slices
  info->pair = p->pair_ok ? 1 : 0;
  info->pair_tiles = p->pair_ok ? p->pair.args.n_tiles : 0;
  info->pair_halo_rows = p->pair_ok ? p->pair.halo_entries : 0;
  info->persist = p->loop_fn ? 1 : 0;
  info->persist_grid = p->loop_fn ? p->loop_grid : 0;
  info->stream_bytes_per_step = (p->index_bits == 16 && !p->resident)
      ? p->N_i * (10LL * p->n + 24) + p->S * 16 + p->overflow_slices * 32LL * p->n * 4
      : info->bytes_per_step;
  return RBF_OK;
}

int rbf_time_step_kernel(rbf_plan* p, double dt, int32_t iters, double* seconds_per_launch) {
  if (!p || iters < 1 || !seconds_per_launch) return fail(RBF_ERR_PARAM, "bad argument");
  RBF_CK(cudaSetDevice(p->device));
  RBF_TRY(normalise_current(p));
  RBF_TRY(reset_status(p, dt, 0.0));
  RBF_CK(cudaEventRecord(p->ev0, p->stream));
  for (int i = 0; i < iters; ++i) RBF_TRY(launch_step(p, i & 1, 0));
  RBF_CK(cudaEventRecord(p->ev1, p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  float ms = 0.f;
  RBF_CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  p->cur = iters & 1;
  *seconds_per_launch = ms * 1e-3 / iters;
  return RBF_OK;
}

void rbf_plan_destroy(rbf_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  for (auto& g : p->graphs)
    if (g) cudaGraphExecDestroy(g);
  if (p->pair_graph) cudaGraphExecDestroy(p->pair_graph);
  cudaStream_t s = p->stream;
  if (p->pair_ok) rbf::pair_free(&p->pair, s);
  if (p->grid_two) rbf::pair_free(&p->grid_pair, s);
  pool_free(p->W, s);
  pool_free(p->C, s);
  pool_free(p->F, s);
  if (p->u_legacy) {
    if (s) cudaStreamSynchronize(s);
    cudaFree(p->U[0]);
    cudaFree(p->U[1]);
    cudaFree(p->push_flags);
  } else {
    pool_free(p->U[0], s);
    pool_free(p->U[1], s);
  }
  pool_free(p->tmp, s);
  pool_free(p->trace, s);
  pool_free(p->d_norm_start, s);
  pool_free(p->d_norm_sum, s);
  pool_free(p->norm_exact, s);
  pool_free(p->new_id, s);
  pool_free(p->row_of_k, s);
  pool_free(p->halo_send_idx, s);
  pool_free(p->cluster_dest, s);
  pool_free(p->grid_red, s);
  pool_free(p->loop_red, s);
  pool_free(p->C16, s);
  pool_free(p->meta, s);
  pool_free(p->u_init, s);
  pool_free(p->halo_sendbuf, s);
  pool_free(p->st, s);
  if (s) cudaStreamSynchronize(s);
  status_free(p->h_st);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

}  // extern "C"

// ---- partitioned (multi-GPU) loop ------------------------------------------
#include "group.inc.cuh"
