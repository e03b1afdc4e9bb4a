// group.inc.cuh -- partitioned (multi-GPU) time loop; included by rbffd_b200.cu.
//
// nodes are partitioned across GPUs (paper_2107_03632_b200/
// multigpu.py builds the parts); every part is an ordinary plan whose local
// numbering is [replicated boundary | halo grouped by owner | owned rows].
// Per step:  pack owned values the peers read -> exchange (NCCL send/recv,
// or device copies when all parts live in this process) -> step kernel
// (kDistributed epilogue: only red[] is accumulated) -> all-reduce(max) of
// red[] = {residual bits, non-finite flag} -> decide_kernel applies the
// reference's flag check / residual / steady break (solver.py:200-217)
// identically on every part.  The j-order of every row is untouched: the
// partitioned run is bitwise identical to a single-GPU run.
//
// NCCL is loaded at run time (dlopen) so the single-GPU library has no hard
// dependency on it; the torch-bundled libnccl.so.2 (2.28.x) is used.
#include <dlfcn.h>
#include <nccl.h>

#include <map>

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

int load_nccl() {
  if (g_nccl.h) return RBF_OK;
  const char* env = std::getenv("RBFFD_NCCL_LIB");
  void* h = env ? dlopen(env, RTLD_NOW | RTLD_GLOBAL) : nullptr;
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(RBF_ERR_CUDA, std::string("cannot load NCCL: ") + dlerror());
#define RBF_SYM(name, field)                                                         \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));          \
  if (!g_nccl.field) return fail(RBF_ERR_CUDA, std::string("NCCL symbol missing: ") + name);
  RBF_SYM("ncclGetUniqueId", GetUniqueId)
  RBF_SYM("ncclCommInitRank", CommInitRank)
  RBF_SYM("ncclCommDestroy", CommDestroy)
  RBF_SYM("ncclSend", Send)
  RBF_SYM("ncclRecv", Recv)
  RBF_SYM("ncclGroupStart", GroupStart)
  RBF_SYM("ncclGroupEnd", GroupEnd)
  RBF_SYM("ncclAllReduce", AllReduce)
  RBF_SYM("ncclGetErrorString", GetErrorString)
#undef RBF_SYM
  g_nccl.h = h;
  return RBF_OK;
}

#define RBF_NCK(call)                                                                      \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(RBF_ERR_CUDA, std::string(#call) + ": " + g_nccl.GetErrorString(r_));  \
  } while (0)

}  // namespace

struct rbf_group {
  std::vector<rbf_plan*> parts;   // parts living in this process
  std::vector<int> ids;           // their global part ids
  std::map<int, int> local_of;    // global id -> index in parts (local mode)
  bool nccl = false;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int device = 0;
  cudaStream_t stream = nullptr;  // every launch of the group runs here
  rbf::DevStatus** d_status = nullptr;  // device array of the parts' status pointers
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaGraphExec_t fast_graph = nullptr;  // kGroupGraph fixed-mode steps (pack, exchange, step)
  std::vector<int64_t> graph_launches;   // per part: kernel launches inside fast_graph
  long long* d_red = nullptr;            // [2] end-of-run reduction: {first bad step key, residual bits}
  // push mode (fixed-step fast path): halos stored straight into the peers'
  // buffers by push_halo_kernel, arrivals signalled through per-part counters
  bool push = false;
  std::vector<rbf::PushArgs> push_args;  // per local part
  std::vector<unsigned int*> tickets;
  std::vector<void*> ipc_opened;         // IPC mappings to close on destroy
  // host-paced push mode (rbf_group_set_step_barrier): every fixed-mode step
  // is followed by a stream sync and this callback (a barrier across the
  // ranks), so no step kernel ever waits on a kernel of another process that
  // may not be running -- the cross-process path on ranks sharing one GPU
  void (*step_barrier)(void*) = nullptr;
  void* step_barrier_ctx = nullptr;
  // partitioned persistent loop (part_loop_kernel): all local parts in one
  // cooperative launch, halo pushes fused into the consumers
  int part_loop_state = 0;               // 0 not prepared, 1 ready, -1 not applicable
  PartLoopFn part_fn = nullptr;
  size_t part_smem = 0;
  int part_grid = 0, part_block = 0;
  rbf::TmaGeom part_geom = {1, 2, 0, 0};
  rbf::PartLoop* d_parts = nullptr;
  std::vector<rbf::PartLoop> h_parts;
  unsigned long long* d_bars = nullptr;  // [16] per part (one line each): arrivals, first bad step, residual
  std::vector<void*> part_bufs;          // push lists
};

// What one part publishes so that its peers can push into it (IPC mode).
struct PushBlob {
  int magic;
  int part_id;
  cudaIpcMemHandle_t u0, u1, flags;
  int n_peers;
  int peer_ids[rbf::kMaxPushPeers];
  long long recv_off[rbf::kMaxPushPeers];
  long long recv_count[rbf::kMaxPushPeers];
};
constexpr int kPushMagic = 0x52424650;  // "RBFP"

namespace {

int group_pack(rbf_group* g, rbf_plan* p, int cur) {
  if (p->halo_send_total == 0) return RBF_OK;
  const int blocks = static_cast<int>(std::min<int64_t>((p->halo_send_total + 255) / 256, 148 * 8));
  rbf::pack_halo_kernel<<<blocks, 256, 0, g->stream>>>(p->U[cur], p->halo_send_idx,
                                                       p->halo_send_total, p->halo_sendbuf);
  RBF_CK(cudaGetLastError());
  ++p->launches;
  return RBF_OK;
}

int group_exchange(rbf_group* g, int cur) {
  if (g->nccl) {
    rbf_plan* p = g->parts[0];
    RBF_NCK(g_nccl.GroupStart());
    for (size_t i = 0; i < p->halo_peers.size(); ++i) {
      const int peer = p->halo_peers[i];
      if (p->halo_send_count[i] > 0)
        RBF_NCK(g_nccl.Send(p->halo_sendbuf + p->halo_send_off[i], p->halo_send_count[i],
                            ncclFloat64, peer, g->comm, g->stream));
      if (p->halo_recv_count[i] > 0)
        RBF_NCK(g_nccl.Recv(p->U[cur] + p->halo_recv_off[i], p->halo_recv_count[i], ncclFloat64,
                            peer, g->comm, g->stream));
    }
    RBF_NCK(g_nccl.GroupEnd());
    return RBF_OK;
  }
  // in-process: copy each peer's packed segment straight into the halo slice
  for (size_t a = 0; a < g->parts.size(); ++a) {
    rbf_plan* p = g->parts[a];
    for (size_t i = 0; i < p->halo_peers.size(); ++i) {
      if (p->halo_recv_count[i] == 0) continue;
      auto it = g->local_of.find(p->halo_peers[i]);
      if (it == g->local_of.end()) return fail(RBF_ERR_PARAM, "peer part not in this group");
      rbf_plan* q = g->parts[it->second];
      int j = -1;
      for (size_t k = 0; k < q->halo_peers.size(); ++k)
        if (q->halo_peers[k] == g->ids[a]) j = static_cast<int>(k);
      if (j < 0 || q->halo_send_count[j] != p->halo_recv_count[i])
        return fail(RBF_ERR_PARAM, "halo lists of two parts disagree");
      // parts of an in-process group share one device (rbf_group_create):
      // a plain device-to-device copy, capturable into the step graph
      RBF_CK(cudaMemcpyAsync(p->U[cur] + p->halo_recv_off[i], q->halo_sendbuf + q->halo_send_off[j],
                             sizeof(double) * p->halo_recv_count[i], cudaMemcpyDeviceToDevice, g->stream));
    }
  }
  return RBF_OK;
}

int group_reduce_decide(rbf_group* g, int64_t step, int flags) {
  if (g->nccl) {
    rbf_plan* p = g->parts[0];
    RBF_NCK(g_nccl.AllReduce(p->st->red, p->st->red, 2, ncclUint64, ncclMax, g->comm, g->stream));
  } else if (g->parts.size() > 1) {
    rbf::reduce_parts_kernel<<<1, 32, 0, g->stream>>>(g->d_status, static_cast<int>(g->parts.size()));
    RBF_CK(cudaGetLastError());
  }
  for (rbf_plan* p : g->parts) {
    rbf::decide_kernel<<<1, 32, 0, g->stream>>>(p->st, step, flags);
    RBF_CK(cudaGetLastError());
  }
  return RBF_OK;
}

// Field buffers a peer can write into: cudaMalloc'd (pool memory cannot be
// exported through CUDA IPC), plus the part's arrival counters.  The plan's
// captured graphs refer to the old buffers and are dropped.
int push_prepare_part(rbf_plan* p) {
  if (p->u_legacy) return RBF_OK;
  RBF_CK(cudaSetDevice(p->device));
  RBF_CK(cudaStreamSynchronize(p->stream));
  double* nu[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) {
    RBF_CK(cudaMalloc(&nu[b], sizeof(double) * std::max<int64_t>(p->N, 1)));
    RBF_CK(cudaMemcpy(nu[b], p->U[b], sizeof(double) * p->N, cudaMemcpyDeviceToDevice));
    pool_free(p->U[b], p->stream);
    p->U[b] = nu[b];
  }
  RBF_CK(cudaMalloc(&p->push_flags, sizeof(unsigned long long) * 64));
  RBF_CK(cudaMemset(p->push_flags, 0, sizeof(unsigned long long) * 64));
  for (auto& gr : p->graphs)
    if (gr) {
      cudaGraphExecDestroy(gr);
      gr = nullptr;
    }
  if (p->pair_graph) {
    cudaGraphExecDestroy(p->pair_graph);
    p->pair_graph = nullptr;
  }
  p->u_legacy = true;
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

int push_finish_part(rbf_group* g, rbf_plan* p, int id, rbf::PushArgs* pa) {
  if (p->halo_peers.size() > static_cast<size_t>(rbf::kMaxPushPeers))
    return fail(RBF_ERR_PARAM, "push mode supports at most 8 neighbour parts");
  if (id < 0 || id >= 64) return fail(RBF_ERR_PARAM, "push mode supports part ids 0..63");
  pa->u[0] = p->U[0];
  pa->u[1] = p->U[1];
  pa->send_idx = p->halo_send_idx;
  pa->total = p->halo_send_total;
  pa->my_id = id;
  pa->st = p->st;
  unsigned int* ticket = nullptr;
  RBF_CK(cudaMalloc(&ticket, sizeof(unsigned int)));
  RBF_CK(cudaMemset(ticket, 0, sizeof(unsigned int)));
  g->tickets.push_back(ticket);
  pa->ticket = ticket;
  p->wait_n = static_cast<int>(p->halo_peers.size());
  for (int i = 0; i < p->wait_n; ++i) p->wait_ids[i] = p->halo_peers[i];
  p->push = true;
  return RBF_OK;
}

int group_push(rbf_group* g, size_t a, int out) {
  const rbf::PushArgs& pa = g->push_args[a];
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((pa.total + 255) / 256, 148 * 2)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = g->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RBF_CK(cudaLaunchKernelEx(&cfg, rbf::push_halo_kernel, pa, out));
  ++g->parts[a]->launches;
  return RBF_OK;
}

int group_step_kernel(rbf_group* g, rbf_plan* p, int cur, int flags) {
  // the plan's own launch path, redirected to the group stream (PDL only in
  // push mode, where the previous kernel of the stream is the push kernel)
  cudaStream_t saved = p->stream;
  const bool pdl = p->pdl;
  p->stream = g->stream;
  p->pdl = pdl && g->push && p->push;
  const int rc = launch_step(p, cur, flags);
  p->stream = saved;
  p->pdl = pdl;
  return rc;
}

constexpr int kGroupGraph = 64;  // even: buffer parity is static inside the graph

// One fixed-mode step of every local part without a per-step reduction: each
// part's step kernel keeps its own first bad step and (on the last step) its
// residual max in its status, like a single-plan run.
int group_fast_step(rbf_group* g, int cur, int flags) {
  if (g->push) {  // step, then push this step's owned halo values into the peers
    for (size_t a = 0; a < g->parts.size(); ++a) {
      RBF_TRY(group_step_kernel(g, g->parts[a], cur, flags));
      RBF_TRY(group_push(g, a, 1 - cur));
    }
    return RBF_OK;
  }
  for (rbf_plan* p : g->parts) RBF_TRY(group_pack(g, p, cur));
  RBF_TRY(group_exchange(g, cur));
  for (rbf_plan* p : g->parts) RBF_TRY(group_step_kernel(g, p, cur, flags));
  return RBF_OK;
}

int group_fast_graph(rbf_group* g, cudaGraphExec_t* out) {
  if (g->fast_graph) {
    *out = g->fast_graph;
    return RBF_OK;
  }
  std::vector<int64_t> before;
  for (rbf_plan* p : g->parts) before.push_back(p->launches);
  RBF_CK(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
  int rc = RBF_OK;
  for (int i = 0; i < kGroupGraph && rc == RBF_OK; ++i) rc = group_fast_step(g, i & 1, 0);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(g->stream, &graph);
  // captured launches are counted when the graph runs
  g->graph_launches.assign(g->parts.size(), 0);
  for (size_t a = 0; a < g->parts.size(); ++a) {
    g->graph_launches[a] = g->parts[a]->launches - before[a];
    g->parts[a]->launches = before[a];
  }
  if (rc != RBF_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return fail(RBF_ERR_CUDA, std::string("group graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&g->fast_graph, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(RBF_ERR_CUDA, std::string("group graph instantiate: ") + cudaGetErrorString(e));
  *out = g->fast_graph;
  return RBF_OK;
}

void part_loop_release(rbf_group* g) {
  for (void* b : g->part_bufs) cudaFree(b);
  g->part_bufs.clear();
  if (g->d_parts) cudaFree(g->d_parts);
  if (g->d_bars) cudaFree(g->d_bars);
  g->d_parts = nullptr;
  g->d_bars = nullptr;
  g->h_parts.clear();
  g->part_loop_state = 0;
}

// Whether the fixed-step fast path can run as one part_loop_kernel launch
// (push mode, every part on the persistent streaming loop with the same
// kernel and ring geometry, identity numbering), and its descriptors.
int part_loop_prepare(rbf_group* g) {
  if (g->part_loop_state != 0) return RBF_OK;
  g->part_loop_state = -1;
  const char* env = std::getenv("RBFFD_PART_LOOP");
  if ((env && std::atoi(env) == 0) || g->step_barrier) return RBF_OK;
  bool any_peer = false;  // without push mode, only parts that exchange nothing
  for (rbf_plan* p : g->parts) any_peer = any_peer || !p->halo_peers.empty();
  if (!g->push && any_peer) return RBF_OK;
  rbf_plan* p0 = g->parts[0];
  for (rbf_plan* p : g->parts) {
    if (!p->loop_fn || p->renumbered || p->n != p0->n || p->index_bits != p0->index_bits ||
        p->loop_geom.sps != p0->loop_geom.sps || p->loop_geom.stages != p0->loop_geom.stages ||
        p->loop_smem != p0->loop_smem || p->tma_block != p0->tma_block || p->N_i < 1)
      return RBF_OK;
  }
  PartLoopFn fn = nullptr;
  switch (p0->n) {
#define RBF_PCASE(K) \
  case K:            \
    fn = KernelSet<K>::part_loop(p0->index_bits == 16); \
    break;
    RBF_SPECIALISED(RBF_PCASE)
#undef RBF_PCASE
    default:
      return RBF_OK;
  }
  if (set_max_smem(fn) != cudaSuccess) {
    cudaGetLastError();
    return RBF_OK;
  }
  int sms = 0, occ = 0;
  RBF_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, p0->tma_block, p0->loop_smem) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    return RBF_OK;
  }
  const int total = sms * occ, np = static_cast<int>(g->parts.size());
  if (np > total) return RBF_OK;
  // CTAs per part in proportion to its slices (>= 1, <= its chunks)
  const int sps = p0->loop_geom.sps;
  int64_t S_all = 0;
  for (rbf_plan* p : g->parts) S_all += p->S;
  std::vector<int> ncta(np);
  int used = 0;
  for (int a = 0; a < np; ++a) {
    const int64_t chunks = (g->parts[a]->S + sps - 1) / sps;
    const int64_t want = std::max<int64_t>(1, (total - np) * g->parts[a]->S / std::max<int64_t>(S_all, 1) + 1);
    ncta[a] = static_cast<int>(std::min<int64_t>(want, chunks));
    used += ncta[a];
  }
  if (used > total) return RBF_OK;
  g->h_parts.assign(np, rbf::PartLoop{});
  int cta0 = 0;
  for (int a = 0; a < np; ++a) {
    rbf_plan* p = g->parts[a];
    const rbf::PushArgs pa = g->push ? g->push_args[a] : rbf::PushArgs{};
    rbf::PartLoop& P = g->h_parts[a];
    const bool saved = p->push;
    p->push = false;  // plain streaming args (the part loop waits by itself)
    P.a = p->args();
    p->push = saved;
    P.U[0] = p->U[0];
    P.U[1] = p->U[1];
    P.cta0 = cta0;
    P.ncta = ncta[a];
    cta0 += ncta[a];
    // per-slice push lists from the part's send segments
    std::vector<int64_t> cnt(static_cast<size_t>(p->S) + 1, 0);
    std::vector<unsigned long long> ent;
    int64_t first_push_row = p->N_i;
    for (int i = 0; i < pa.n_peer; ++i) {
      for (int64_t k = pa.peer[i].src_off; k < pa.peer[i].src_off + pa.peer[i].count; ++k) {
        const int64_t row = static_cast<int64_t>(p->halo_send_idx_h[static_cast<size_t>(k)]) - p->B;
        if (row < 0 || row >= p->N_i) return fail(RBF_ERR_PARAM, "send list entry outside the part's rows");
        ++cnt[static_cast<size_t>(row >> 5) + 1];
        first_push_row = std::min(first_push_row, row);
      }
    }
    for (int64_t sl = 0; sl < p->S; ++sl) cnt[static_cast<size_t>(sl) + 1] += cnt[static_cast<size_t>(sl)];
    if (cnt.back() > 0) {
      if (cnt.back() >= (int64_t(1) << 31)) return RBF_OK;  // int32 per-slice offsets
      ent.assign(static_cast<size_t>(cnt.back()), 0ull);
      std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
      for (int i = 0; i < pa.n_peer; ++i) {
        for (int64_t k = pa.peer[i].src_off; k < pa.peer[i].src_off + pa.peer[i].count; ++k) {
          const int64_t row = static_cast<int64_t>(p->halo_send_idx_h[static_cast<size_t>(k)]) - p->B;
          const unsigned long long slot =
              static_cast<unsigned long long>(pa.peer[i].dst_off + (k - pa.peer[i].src_off));
          if (slot >= (1ull << 52)) return RBF_OK;
          ent[static_cast<size_t>(fill[static_cast<size_t>(row >> 5)]++)] =
              (static_cast<unsigned long long>(i) << 58) | (static_cast<unsigned long long>(row & 31) << 52) | slot;
        }
      }
      const std::vector<int> off(cnt.begin(), cnt.end());
      int* d_off = nullptr;
      unsigned long long* d_ent = nullptr;
      RBF_CK(cudaMalloc(&d_off, sizeof(int) * off.size()));
      g->part_bufs.push_back(d_off);
      RBF_CK(cudaMalloc(&d_ent, sizeof(unsigned long long) * ent.size()));
      g->part_bufs.push_back(d_ent);
      RBF_CK(cudaMemcpy(d_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
      RBF_CK(cudaMemcpy(d_ent, ent.data(), sizeof(unsigned long long) * ent.size(), cudaMemcpyHostToDevice));
      P.push_off = d_off;
      P.push_ent = d_ent;
    }
    for (int i = 0; i < pa.n_peer; ++i) {
      P.peer_u[i][0] = pa.peer[i].u[0];
      P.peer_u[i][1] = pa.peer[i].u[1];
    }
    for (int j = 0; j < pa.n_nbr; ++j) P.nbr_flags[j] = pa.nbr_flags[j];
    P.n_nbr = pa.n_nbr;
    P.my_id = pa.my_id;
    P.sys_scope = pa.sys_scope;
    P.my_flags = p->push_flags;
    P.wait_mask = 0;
    for (int i = 0; g->push && i < p->wait_n; ++i) P.wait_mask |= 1ull << p->wait_ids[i];
    P.sync_row0 = std::min<int64_t>(p->halo_row0, first_push_row);
  }
  // one 128-byte line per part: a part's spinning CTAs must not share the
  // line its neighbour's arrivals hit
  RBF_CK(cudaMalloc(&g->d_bars, sizeof(unsigned long long) * 16 * np));
  for (int a = 0; a < np; ++a) g->h_parts[a].bar = g->d_bars + 16 * a;
  RBF_CK(cudaMalloc(&g->d_parts, sizeof(rbf::PartLoop) * np));
  g->part_fn = fn;
  g->part_smem = p0->loop_smem;
  g->part_grid = cta0;
  g->part_block = p0->tma_block;
  g->part_geom = p0->loop_geom;
  g->part_loop_state = 1;
  return RBF_OK;
}

// Descriptors and barrier words of this run (before the timed region).
int part_loop_upload(rbf_group* g) {
  const int np = static_cast<int>(g->parts.size());
  for (int a = 0; a < np; ++a) g->h_parts[a].base = static_cast<unsigned long long>(g->parts[a]->push_base);
  RBF_CK(cudaMemcpyAsync(g->d_parts, g->h_parts.data(), sizeof(rbf::PartLoop) * np, cudaMemcpyHostToDevice,
                         g->stream));
  std::vector<unsigned long long> bars(static_cast<size_t>(16 * np), 0ull);
  for (int a = 0; a < np; ++a) bars[static_cast<size_t>(16 * a + 1)] = ~0ull;
  RBF_CK(cudaMemcpyAsync(g->d_bars, bars.data(), sizeof(unsigned long long) * bars.size(), cudaMemcpyHostToDevice,
                         g->stream));
  RBF_CK(cudaStreamSynchronize(g->stream));  // the host arrays above are pageable locals
  return RBF_OK;
}

int part_loop_launch(rbf_group* g, int64_t limit) {
  const int np = static_cast<int>(g->parts.size());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g->part_grid);
  cfg.blockDim = dim3(g->part_block);
  cfg.dynamicSmemBytes = g->part_smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every part's CTAs co-resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const rbf::PartLoop* dp = g->d_parts;
  RBF_CK(cudaLaunchKernelEx(&cfg, g->part_fn, dp, np, static_cast<long long>(limit), g->part_geom));
  for (rbf_plan* p : g->parts) ++p->launches;
  return RBF_OK;
}

// Fixed-mode run without per-step reductions.  On return *any_bad tells the
// caller to restore the start field and replay on the exact per-step path.
int group_run_fast(rbf_group* g, int64_t limit, bool* any_bad, unsigned long long* res_bits) {
  *any_bad = false;
  for (rbf_plan* p : g->parts) {
    if (!p->u_init) RBF_TRY(dev_alloc(p, &p->u_init, static_cast<size_t>(p->N)));
    RBF_CK(cudaMemcpyAsync(p->u_init, p->U[0], sizeof(double) * p->N, cudaMemcpyDeviceToDevice, g->stream));
  }
  cudaGraphExec_t graph = nullptr;
  const bool paced = g->step_barrier != nullptr;
  RBF_TRY(part_loop_prepare(g));
  const bool fused = g->part_loop_state == 1;
  if (limit > kGroupGraph && !paced && !fused) RBF_TRY(group_fast_graph(g, &graph));
  if (paced) {  // every rank finished its setup / previous run
    RBF_CK(cudaStreamSynchronize(g->stream));
    g->step_barrier(g->step_barrier_ctx);
  }
  if (fused) RBF_TRY(part_loop_upload(g));
  if (!g->d_red) RBF_CK(cudaMalloc(&g->d_red, 2 * sizeof(long long)));
  if (g->nccl && g->push) {
    // every rank has set its start field (rbf_set_field is synchronous)
    // before any rank's first push can land in its buffers: a one-element
    // all-reduce orders this launch after every rank's call
    RBF_NCK(g_nccl.AllReduce(g->d_red, g->d_red, 1, ncclInt64, ncclMax, g->comm, g->stream));
  }
  RBF_CK(cudaEventRecord(g->ev0, g->stream));
  if (fused) RBF_TRY(part_loop_launch(g, limit));
  const int64_t chunks = (paced || fused) ? 0 : (limit - 1) / kGroupGraph;
  for (int64_t c = 0; c < chunks; ++c) {
    RBF_CK(cudaGraphLaunch(graph, g->stream));
    for (size_t a = 0; a < g->parts.size(); ++a) g->parts[a]->launches += g->graph_launches[a];
  }
  for (int64_t s = fused ? limit : chunks * kGroupGraph; s < limit; ++s) {
    RBF_TRY(group_fast_step(g, static_cast<int>(s & 1), s == limit - 1 ? rbf::kNeedResidual : 0));
    if (paced) {  // this step and its pushes are complete on every rank before any rank steps on
      RBF_CK(cudaStreamSynchronize(g->stream));
      g->step_barrier(g->step_barrier_ctx);
    }
  }
  RBF_CK(cudaEventRecord(g->ev1, g->stream));
  for (rbf_plan* p : g->parts) {
    if (g->push) p->push_base += limit;  // every part ran all `limit` pushes
  }
  if (fused && std::getenv("RBFFD_TRACE")) {  // RBFFD_TRACE: {-ncta, steps, [steps][ncta][4]} per part
    RBF_CK(cudaStreamSynchronize(g->stream));
    for (size_t a = 0; a < g->parts.size(); ++a) {
      rbf_plan* p = g->parts[a];
      if (!p->trace) continue;
      const int64_t n_tr = std::min<int64_t>(limit, p->trace_cap), G = g->h_parts[a].ncta;
      std::vector<unsigned long long> h(static_cast<size_t>(n_tr * G * 4));
      RBF_CK(cudaMemcpy(h.data(), p->trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      if (std::FILE* f = std::fopen(std::getenv("RBFFD_TRACE"), "ab")) {
        const int64_t hdr[2] = {-G, n_tr};
        std::fwrite(hdr, sizeof(hdr), 1, f);
        std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
        std::fclose(f);
      }
    }
  }
  // end-of-run reduction over all parts: min first-bad-step, max residual bits
  long long key = std::numeric_limits<long long>::max();
  unsigned long long bits = 0;
  RBF_CK(cudaStreamSynchronize(g->stream));
  for (rbf_plan* p : g->parts) {
    RBF_TRY(read_status(p));
    if (p->h_st->bad_step >= 0) key = std::min<long long>(key, p->h_st->bad_step);
    if (p->h_st->last_res_step == limit - 1) bits = std::max<unsigned long long>(bits, p->h_st->last_res_bits);
  }
  if (g->nccl) {
    long long h[2] = {key, static_cast<long long>(bits)};
    RBF_CK(cudaMemcpyAsync(g->d_red, h, sizeof(h), cudaMemcpyHostToDevice, g->stream));
    RBF_NCK(g_nccl.GroupStart());
    RBF_NCK(g_nccl.AllReduce(g->d_red, g->d_red, 1, ncclInt64, ncclMin, g->comm, g->stream));
    RBF_NCK(g_nccl.AllReduce(g->d_red + 1, g->d_red + 1, 1, ncclUint64, ncclMax, g->comm, g->stream));
    RBF_NCK(g_nccl.GroupEnd());
    RBF_CK(cudaMemcpyAsync(h, g->d_red, sizeof(h), cudaMemcpyDeviceToHost, g->stream));
    RBF_CK(cudaStreamSynchronize(g->stream));
    key = h[0];
    bits = static_cast<unsigned long long>(h[1]);
  }
  *res_bits = bits;
  if (key != std::numeric_limits<long long>::max()) {
    *any_bad = true;
    for (rbf_plan* p : g->parts) {
      RBF_CK(cudaMemcpyAsync(p->U[0], p->u_init, sizeof(double) * p->N, cudaMemcpyDeviceToDevice, g->stream));
      RBF_CK(cudaMemcpyAsync(p->U[1], p->u_init, sizeof(double) * p->N, cudaMemcpyDeviceToDevice, g->stream));
    }
    RBF_CK(cudaStreamSynchronize(g->stream));
  }
  return RBF_OK;
}

}  // namespace

extern "C" {

int rbf_nccl_unique_id(char* out128) {
  if (!out128) return fail(RBF_ERR_PARAM, "NULL argument");
  RBF_TRY(load_nccl());
  ncclUniqueId id;
  RBF_NCK(g_nccl.GetUniqueId(&id));
  std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return RBF_OK;
}

int rbf_plan_set_halo(rbf_plan* p, int32_t n_peers, const int32_t* peers, const int64_t* send_counts,
                      const int64_t* send_idx, const int64_t* recv_counts, const int64_t* recv_offsets) {
  if (!p || n_peers < 0 || (n_peers > 0 && (!peers || !send_counts || !recv_counts || !recv_offsets)))
    return fail(RBF_ERR_PARAM, "bad halo arguments");
  RBF_CK(cudaSetDevice(p->device));
  p->halo_peers.assign(peers, peers + n_peers);
  p->halo_send_count.assign(send_counts, send_counts + n_peers);
  p->halo_recv_count.assign(recv_counts, recv_counts + n_peers);
  p->halo_recv_off.assign(recv_offsets, recv_offsets + n_peers);
  p->halo_send_off.assign(n_peers, 0);
  int64_t total = 0;
  for (int i = 0; i < n_peers; ++i) {
    if (send_counts[i] < 0 || recv_counts[i] < 0 || recv_offsets[i] < 0 ||
        recv_offsets[i] + recv_counts[i] > p->B)
      return fail(RBF_ERR_PARAM, "halo slice outside the non-owned range of the part");
    p->halo_send_off[i] = total;
    total += send_counts[i];
  }
  if (total > 0 && !send_idx) return fail(RBF_ERR_PARAM, "send_idx is NULL");
  std::vector<int32_t> idx(static_cast<size_t>(total));
  for (int64_t k = 0; k < total; ++k) {
    if (send_idx[k] < p->B || send_idx[k] >= p->N)
      return fail(RBF_ERR_PARAM, "a part can only send the values of rows it owns");
    idx[k] = static_cast<int32_t>(send_idx[k]);
  }
  pool_free(p->halo_send_idx, p->stream);
  pool_free(p->halo_sendbuf, p->stream);
  p->halo_send_total = total;
  RBF_TRY(dev_alloc(p, &p->halo_send_idx, static_cast<size_t>(total)));
  RBF_TRY(dev_alloc(p, &p->halo_sendbuf, static_cast<size_t>(total)));
  if (total > 0)
    RBF_CK(cudaMemcpyAsync(p->halo_send_idx, idx.data(), sizeof(int32_t) * total, cudaMemcpyHostToDevice,
                           p->stream));
  RBF_CK(cudaStreamSynchronize(p->stream));
  p->halo_send_idx_h = std::move(idx);
  // first row that reads a halo value: the TMA step overlaps the rows before
  // it with the neighbours' pushes (parts order their rows interior-first)
  int64_t h_lo = p->B, h_hi = 0;
  for (int i = 0; i < n_peers; ++i)
    if (recv_counts[i] > 0) {
      h_lo = std::min<int64_t>(h_lo, recv_offsets[i]);
      h_hi = std::max<int64_t>(h_hi, recv_offsets[i] + recv_counts[i]);
    }
  p->halo_row0 = p->N_i;
  if (h_hi > h_lo && p->N_i > 0) {
    unsigned long long* d_first = nullptr;
    RBF_TRY(pool_alloc(&d_first, 1, p->stream));
    RBF_CK(cudaMemsetAsync(d_first, 0xff, sizeof(unsigned long long), p->stream));
    const int blocks = static_cast<int>(std::min<int64_t>((p->S * 32 * p->n + 255) / 256, 148 * 16));
    rbf::first_row_reading_kernel<<<blocks, 256, 0, p->stream>>>(p->C, p->N_i, p->n, h_lo, h_hi, d_first);
    RBF_CK(cudaGetLastError());
    unsigned long long first = 0;
    RBF_CK(cudaMemcpyAsync(&first, d_first, sizeof(first), cudaMemcpyDeviceToHost, p->stream));
    RBF_CK(cudaStreamSynchronize(p->stream));
    pool_free(d_first, p->stream);
    if (first != ~0ull) p->halo_row0 = static_cast<int64_t>(first);
  }
  RBF_CK(cudaStreamSynchronize(p->stream));
  return RBF_OK;
}

int rbf_group_create(rbf_group** out, int32_t n_local, rbf_plan* const* plans, const int32_t* part_ids,
                     const char* nccl_uid, int32_t rank, int32_t nranks) {
  if (!out || n_local < 1 || !plans || !part_ids) return fail(RBF_ERR_PARAM, "bad group arguments");
  *out = nullptr;
  std::unique_ptr<rbf_group> g(new rbf_group());
  g->nccl = nccl_uid != nullptr;
  if (g->nccl && n_local != 1) return fail(RBF_ERR_PARAM, "an NCCL group holds one part per process");
  for (int i = 0; i < n_local; ++i) {
    if (!plans[i]) return fail(RBF_ERR_PARAM, "NULL plan");
    if (plans[i]->device != plans[0]->device)
      return fail(RBF_ERR_PARAM, "an in-process group keeps its parts on one device");
    g->parts.push_back(plans[i]);
    g->ids.push_back(part_ids[i]);
    g->local_of[part_ids[i]] = i;
  }
  g->device = plans[0]->device;
  g->rank = rank;
  g->nranks = nranks;
  RBF_CK(cudaSetDevice(g->device));
  RBF_CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  RBF_CK(cudaEventCreate(&g->ev0));
  RBF_CK(cudaEventCreate(&g->ev1));
  std::vector<rbf::DevStatus*> sts;
  for (rbf_plan* p : g->parts) sts.push_back(p->st);
  RBF_CK(cudaMalloc(&g->d_status, sizeof(rbf::DevStatus*) * sts.size()));
  RBF_CK(cudaMemcpy(g->d_status, sts.data(), sizeof(rbf::DevStatus*) * sts.size(), cudaMemcpyHostToDevice));
  if (g->nccl) {
    RBF_TRY(load_nccl());
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_uid, NCCL_UNIQUE_ID_BYTES);
    RBF_NCK(g_nccl.CommInitRank(&g->comm, nranks, id, rank));
  }
  *out = g.release();
  return RBF_OK;
}

int rbf_group_run(rbf_group* g, double dt, int64_t steps, int32_t mode, double tol, int64_t max_steps,
                  int64_t* steps_done, double* residual, int32_t* has_residual, int64_t* bad_step,
                  double* device_seconds) {
  if (!g) return fail(RBF_ERR_PARAM, "group is NULL");
  if (mode != RBF_MODE_FIXED && mode != RBF_MODE_STEADY) return fail(RBF_ERR_PARAM, "bad mode");
  const bool steady = mode == RBF_MODE_STEADY;
  const int64_t limit = steady ? max_steps : steps;
  if (limit < 0) return fail(RBF_ERR_PARAM, "steps/max_steps must be >= 0");
  RBF_CK(cudaSetDevice(g->device));
  for (rbf_plan* p : g->parts) {
    RBF_TRY(normalise_current(p));
    RBF_TRY(reset_status(p, dt, tol));
    RBF_CK(cudaStreamSynchronize(p->stream));
  }
  if (!steady && limit >= 2 && !std::getenv("RBFFD_GROUP_EXACT")) {
    bool any_bad = false;
    unsigned long long bits = 0;
    RBF_TRY(group_run_fast(g, limit, &any_bad, &bits));
    if (!any_bad) {
      float ms = 0.f;
      RBF_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
      for (rbf_plan* p : g->parts) p->cur = static_cast<int>(limit & 1);
      double m;
      std::memcpy(&m, &bits, sizeof(m));
      if (device_seconds) *device_seconds = ms * 1e-3;
      if (bad_step) *bad_step = -1;
      if (steps_done) *steps_done = limit;
      if (residual) *residual = m / dt;
      if (has_residual) *has_residual = 1;
      return RBF_OK;
    }
    // a non-finite value appeared: replay from the start field on the exact
    // per-step path, which stops at the reference's step (solver.py:200-206)
    for (rbf_plan* p : g->parts) {
      p->cur = 0;
      RBF_TRY(reset_status(p, dt, tol));
      RBF_CK(cudaStreamSynchronize(p->stream));
    }
  }
  // the exact per-step path exchanges by pack + copy / NCCL: no arrival waits
  struct PushOff {
    rbf_group* g;
    explicit PushOff(rbf_group* gg) : g(gg) {
      for (rbf_plan* p : g->parts) p->push = false;
    }
    ~PushOff() {
      for (rbf_plan* p : g->parts) p->push = g->push;
    }
  } push_off(g);
  RBF_CK(cudaEventRecord(g->ev0, g->stream));
  constexpr int64_t kPoll = 64;
  for (int64_t s = 0; s < limit; ++s) {
    const int cur = static_cast<int>(s & 1);
    const bool need_res = steady || s == limit - 1;
    const int flags = rbf::kDistributed | (need_res ? rbf::kNeedResidual : 0) | (steady ? rbf::kSteady : 0);
    for (rbf_plan* p : g->parts) RBF_TRY(group_pack(g, p, cur));
    RBF_TRY(group_exchange(g, cur));
    for (rbf_plan* p : g->parts) RBF_TRY(group_step_kernel(g, p, cur, flags));
    RBF_TRY(group_reduce_decide(g, s, flags));
    if (steady && (s + 1) % kPoll == 0) {
      rbf::DevStatus st;
      RBF_CK(cudaMemcpyAsync(&st, g->parts[0]->st, sizeof(st), cudaMemcpyDeviceToHost, g->stream));
      RBF_CK(cudaStreamSynchronize(g->stream));
      if (st.bad_step >= 0 || st.conv_step >= 0) break;
    }
  }
  RBF_CK(cudaEventRecord(g->ev1, g->stream));
  RBF_CK(cudaStreamSynchronize(g->stream));
  float ms = 0.f;
  RBF_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
  rbf_plan* p0 = g->parts[0];
  RBF_TRY(read_status(p0));
  const rbf::DevStatus s = *p0->h_st;
  const int64_t done = limit > 0 ? s.step : 0;
  bool have_res = false;
  double res = 0.0;
  if (s.last_res_step >= 0 && s.last_res_step == done - 1) {
    double m;
    std::memcpy(&m, &s.last_res_bits, sizeof(m));
    res = m / dt;
    have_res = true;
  }
  if (device_seconds) *device_seconds = ms * 1e-3;
  if (bad_step) *bad_step = s.bad_step;
  if (s.bad_step >= 0) {
    for (rbf_plan* p : g->parts) p->cur = static_cast<int>((s.bad_step + 1) & 1);
    if (steps_done) *steps_done = s.bad_step;
    if (has_residual) *has_residual = 0;
    return fail(RBF_ERR_INSTABILITY, "time loop unstable at step " + std::to_string(s.bad_step));
  }
  for (rbf_plan* p : g->parts) p->cur = static_cast<int>(done & 1);
  if (steps_done) *steps_done = done;
  if (residual) *residual = have_res ? res : 0.0;
  if (has_residual) *has_residual = have_res ? 1 : 0;
  if (steady && done == max_steps && (!have_res || !(res <= tol)))
    return fail(RBF_ERR_TIMEOUT, "no steady state after " + std::to_string(done) + " steps");
  return RBF_OK;
}

// Push mode for the parts of this process (one device): peers' buffers are
// plain device pointers.
int rbf_group_push_local(rbf_group* g) {
  if (!g) return fail(RBF_ERR_PARAM, "group is NULL");
  if (g->nccl) return fail(RBF_ERR_PARAM, "use rbf_group_push_export/import for NCCL groups");
  RBF_CK(cudaSetDevice(g->device));
  for (rbf_plan* p : g->parts) RBF_TRY(push_prepare_part(p));
  g->push_args.assign(g->parts.size(), rbf::PushArgs{});
  for (size_t a = 0; a < g->parts.size(); ++a) {
    rbf_plan* p = g->parts[a];
    rbf::PushArgs& pa = g->push_args[a];
    RBF_TRY(push_finish_part(g, p, g->ids[a], &pa));
    int np = 0, nn = 0;
    for (size_t i = 0; i < p->halo_peers.size(); ++i) {
      auto it = g->local_of.find(p->halo_peers[i]);
      if (it == g->local_of.end()) return fail(RBF_ERR_PARAM, "peer part not in this group");
      rbf_plan* q = g->parts[it->second];
      pa.nbr_flags[nn++] = q->push_flags;
      if (p->halo_send_count[i] == 0) continue;
      int j = -1;
      for (size_t k = 0; k < q->halo_peers.size(); ++k)
        if (q->halo_peers[k] == g->ids[a]) j = static_cast<int>(k);
      if (j < 0 || q->halo_recv_count[j] != p->halo_send_count[i])
        return fail(RBF_ERR_PARAM, "halo lists of two parts disagree");
      pa.peer[np].u[0] = q->U[0];
      pa.peer[np].u[1] = q->U[1];
      pa.peer[np].dst_off = q->halo_recv_off[j];
      pa.peer[np].src_off = p->halo_send_off[i];
      pa.peer[np].count = p->halo_send_count[i];
      ++np;
    }
    pa.n_peer = np;
    pa.n_nbr = nn;
    pa.sys_scope = 0;  // all parts on this device
  }
  if (g->fast_graph) {
    cudaGraphExecDestroy(g->fast_graph);
    g->fast_graph = nullptr;
  }
  part_loop_release(g);
  g->push = true;
  return RBF_OK;
}

// IPC mode (one part per process): the blob this part publishes.
int rbf_group_push_export(rbf_group* g, void* out, int64_t cap, int64_t* len) {
  if (!g || !out || !len) return fail(RBF_ERR_PARAM, "NULL argument");
  if (g->parts.size() != 1) return fail(RBF_ERR_PARAM, "IPC push mode holds one part per process");
  if (cap < static_cast<int64_t>(sizeof(PushBlob))) return fail(RBF_ERR_PARAM, "export buffer too small");
  RBF_CK(cudaSetDevice(g->device));
  rbf_plan* p = g->parts[0];
  if (p->halo_peers.size() > static_cast<size_t>(rbf::kMaxPushPeers))
    return fail(RBF_ERR_PARAM, "push mode supports at most 8 neighbour parts");
  RBF_TRY(push_prepare_part(p));
  PushBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = kPushMagic;
  b.part_id = g->ids[0];
  RBF_CK(cudaIpcGetMemHandle(&b.u0, p->U[0]));
  RBF_CK(cudaIpcGetMemHandle(&b.u1, p->U[1]));
  RBF_CK(cudaIpcGetMemHandle(&b.flags, p->push_flags));
  b.n_peers = static_cast<int>(p->halo_peers.size());
  for (int i = 0; i < b.n_peers; ++i) {
    b.peer_ids[i] = p->halo_peers[i];
    b.recv_off[i] = p->halo_recv_off[i];
    b.recv_count[i] = p->halo_recv_count[i];
  }
  std::memcpy(out, &b, sizeof(b));
  *len = static_cast<int64_t>(sizeof(b));
  return RBF_OK;
}

// IPC mode: map the neighbours' buffers from their blobs (all parts' blobs,
// `stride` bytes apart) and switch the fast path to push mode.  Every rank
// must import before any rank runs (the caller holds a barrier).
int rbf_group_push_import(rbf_group* g, int32_t n_blobs, const void* blobs, int64_t stride) {
  if (!g || !blobs || n_blobs < 1 || stride < static_cast<int64_t>(sizeof(PushBlob)))
    return fail(RBF_ERR_PARAM, "bad push import arguments");
  if (g->parts.size() != 1) return fail(RBF_ERR_PARAM, "IPC push mode holds one part per process");
  RBF_CK(cudaSetDevice(g->device));
  rbf_plan* p = g->parts[0];
  RBF_TRY(push_prepare_part(p));
  std::map<int, PushBlob> by_id;
  for (int k = 0; k < n_blobs; ++k) {
    PushBlob b;
    std::memcpy(&b, static_cast<const unsigned char*>(blobs) + k * stride, sizeof(b));
    if (b.magic != kPushMagic) return fail(RBF_ERR_PARAM, "not a push-mode blob");
    by_id[b.part_id] = b;
  }
  g->push_args.assign(1, rbf::PushArgs{});
  rbf::PushArgs& pa = g->push_args[0];
  RBF_TRY(push_finish_part(g, p, g->ids[0], &pa));
  int np = 0, nn = 0;
  for (size_t i = 0; i < p->halo_peers.size(); ++i) {
    const int q = p->halo_peers[i];
    auto it = by_id.find(q);
    if (it == by_id.end()) return fail(RBF_ERR_PARAM, "missing blob of a neighbour part");
    const PushBlob& b = it->second;
    void* fl = nullptr;
    RBF_CK(cudaIpcOpenMemHandle(&fl, b.flags, cudaIpcMemLazyEnablePeerAccess));
    g->ipc_opened.push_back(fl);
    pa.nbr_flags[nn++] = static_cast<unsigned long long*>(fl);
    if (p->halo_send_count[i] == 0) continue;
    int j = -1;
    for (int k = 0; k < b.n_peers; ++k)
      if (b.peer_ids[k] == g->ids[0]) j = k;
    if (j < 0 || b.recv_count[j] != p->halo_send_count[i])
      return fail(RBF_ERR_PARAM, "halo lists of two parts disagree");
    void *u0 = nullptr, *u1 = nullptr;
    RBF_CK(cudaIpcOpenMemHandle(&u0, b.u0, cudaIpcMemLazyEnablePeerAccess));
    g->ipc_opened.push_back(u0);
    RBF_CK(cudaIpcOpenMemHandle(&u1, b.u1, cudaIpcMemLazyEnablePeerAccess));
    g->ipc_opened.push_back(u1);
    pa.peer[np].u[0] = static_cast<double*>(u0);
    pa.peer[np].u[1] = static_cast<double*>(u1);
    pa.peer[np].dst_off = b.recv_off[j];
    pa.peer[np].src_off = p->halo_send_off[i];
    pa.peer[np].count = p->halo_send_count[i];
    ++np;
  }
  pa.n_peer = np;
  pa.n_nbr = nn;
  pa.sys_scope = 1;  // peers are other GPUs
  if (g->fast_graph) {
    cudaGraphExecDestroy(g->fast_graph);
    g->fast_graph = nullptr;
  }
  part_loop_release(g);
  g->push = true;
  return RBF_OK;
}

int rbf_group_push_mode(const rbf_group* g) { return g && g->push ? 1 : 0; }
int rbf_group_fused(const rbf_group* g) { return g && g->part_loop_state == 1 ? 1 : 0; }

int rbf_group_set_step_barrier(rbf_group* g, void (*fn)(void*), void* ctx) {
  if (!g) return fail(RBF_ERR_PARAM, "group is NULL");
  g->step_barrier = fn;
  g->step_barrier_ctx = ctx;
  part_loop_release(g);
  return RBF_OK;
}

// Back to the pack + NCCL / copy exchange (every rank must agree: used when
// some rank could not map its neighbours).
int rbf_group_push_off(rbf_group* g) {
  if (!g) return fail(RBF_ERR_PARAM, "group is NULL");
  g->push = false;
  for (rbf_plan* p : g->parts) p->push = false;
  if (g->fast_graph) {
    cudaGraphExecDestroy(g->fast_graph);
    g->fast_graph = nullptr;
  }
  part_loop_release(g);
  return RBF_OK;
}

void rbf_group_destroy(rbf_group* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  for (void* m : g->ipc_opened) cudaIpcCloseMemHandle(m);
  for (unsigned int* t : g->tickets) cudaFree(t);
  part_loop_release(g);
  for (rbf_plan* p : g->parts) p->push = false;
  if (g->fast_graph) cudaGraphExecDestroy(g->fast_graph);
  if (g->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(g->comm);
  cudaFree(g->d_status);
  cudaFree(g->d_red);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

}  // extern "C"
