// common.cuh -- shared state, layout and device helpers of the explicit
// RBF-FD pseudo-time step kernels (included by every kernel translation unit;
// only templates, inline functions and types, so it may be included twice).
//
// Reference semantics: rbffd.solver._step_kernel, pkg/src/rbffd/solver.py:294-311
//   acc = 0.0; for j: acc += weights[k,j]*u1[rows[k,j]]            (:304-306)
//   value = u1[interior[k]] + dt*(f_int[k] + acc); u2[interior[k]] = value   (:307-308)
//   flag if !isfinite(value)                                          (:309-311)
// plus the loop-level pieces of run_time_loop (solver.py:198-217): the per-step
// non-finite check, the residual max|u2-u1|/dt and the steady-state break, all
// fused into the step so the host never touches the field between steps.
//
// Bitwise parity: numba compiles the update to separate fmul/fadd with no
// contraction, so every product and sum here is an explicit
// __dmul_rn / __dadd_rn (ptxas cannot fuse those into DFMA), the accumulator
// starts at +0.0 and the j-order is serial.
//
// Device layout (SELL-32, "sliced transposed ELL"): rows are grouped in
// slices of 32; slice s stores its n weights as W[s*n*32 + j*32 + lane]
// (fp64) and node ids as C[...] (int32), so warp-wide loads of one j are one
// contiguous 256 B (W) / 128 B (C) segment.  Node ids are renumbered so that
// interior row r updates node (B + r), B = N - N_i (non-interior nodes first),
// which removes the `interior` array from the stream.  Per-row algorithmic
// bytes: 8n (W) + 4n (C) + 8 (F) + 8 (u_self) + 8 (u write) = 12n + 24.
#pragma once
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace rbf {

// Device-resident loop state.  Written only by the last CTA of each step
// (ticket pattern) or by CTAs that see a non-finite value.
struct DevStatus {
  unsigned long long res_bits;       // running max of |u2-u1| bits (>= 0 doubles order like uints)
  unsigned long long last_res_bits;  // residual numerator of the last residual step
  long long last_res_step;           // step index of last_res_bits (-1 none)
  long long bad_step;                // first step with a non-finite value (-1 none)
  long long conv_step;               // steady: step whose residual <= tol (-1 none)
  long long step;                    // global index of the next step to execute
  unsigned int ticket;               // CTAs finished in the current step
  unsigned int pad0;
  double dt;
  double tol;
  unsigned long long red[2];         // distributed mode: [residual bits max, non-finite any]
  long long push_base;               // push-mode groups: arrivals counted before this run
  long long push_count;              // push-mode groups: halo pushes completed in this run
};

struct StepArgs {
  const double* __restrict__ W;  // [S*n*32]
  const int* __restrict__ C;     // [S*n*32]
  const double* __restrict__ F;  // [S*32]
  const unsigned short* __restrict__ C16;  // [S*n*32] 16-bit ids (two-window), or null
  const int4* __restrict__ meta;           // [S] {base0, base1, ok, 0} of the 16-bit ids
  long long n_rows;
  long long dst_base;            // node id of row 0 (= N - N_i)
  int n;
  DevStatus* st;
  // push-mode partitioned runs (group.inc.cuh): before reading the field, wait
  // until every neighbour part has pushed the halo of this step into this
  // part's buffers (wait_flags[id] counts neighbour id's pushes), or null
  const unsigned long long* wait_flags;
  unsigned long long wait_mask;  // bit i: part i is a neighbour
  unsigned long long wait_ns;    // a wait longer than this traps (a peer died)
  long long halo_row0;           // rows >= this read halo values; the TMA step waits
                                 // for the peers only before those (interior rows first)
  unsigned long long* trace;     // RBFFD_TRACE diagnostics: per (step, CTA) globaltimer
                                 // {entry, dependency resolved, ring issued, exit}, or null
  int trace_cap;                 // steps the trace buffer holds
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kMaxPushPeers = 8;

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Push-mode wait: every neighbour's arrival count must reach this part's own
// push count, i.e. the neighbour finished the previous step (its halo values
// for this step are in place and it no longer reads the buffer this step
// writes into its peers).  One lane of the CTA's first consumer warp polls
// with acquire loads; the other consumer warps are released by a named
// barrier (nthreads = all consumer threads), which orders their field reads
// after the acquire.  A wait longer than wait_ns (20 s; RBFFD_WAIT_TIMEOUT_MS)
// means a peer died: trap instead of hanging the GPU.
__device__ __forceinline__ void wait_peers(const unsigned long long* flags, unsigned long long mask,
                                           DevStatus* st, bool first_warp, int nthreads,
                                           unsigned long long wait_ns = 20000000000ull) {
  if (!flags) return;
  if (first_warp && (threadIdx.x & 31) == 0) {
    const unsigned long long need = static_cast<unsigned long long>(
        *reinterpret_cast<volatile long long*>(&st->push_base) +
        *reinterpret_cast<volatile long long*>(&st->push_count));
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (unsigned long long m = mask; m; m &= m - 1) {
      const int j = __ffsll(static_cast<long long>(m)) - 1;
      while (ld_acquire_sys_u64(flags + j) < need) {
        __nanosleep(64);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > wait_ns) __trap();
      }
    }
  }
  asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
}

// Per-warp variant of wait_peers for the TMA step: lane 0 polls, the warp
// barrier orders the other lanes' field reads after its acquire loads.
__device__ __forceinline__ void wait_peers_warp(const unsigned long long* flags, unsigned long long mask,
                                                DevStatus* st, unsigned long long wait_ns) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long need = static_cast<unsigned long long>(
        *reinterpret_cast<volatile long long*>(&st->push_base) +
        *reinterpret_cast<volatile long long*>(&st->push_count));
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (unsigned long long m = mask; m; m &= m - 1) {
      const int j = __ffsll(static_cast<long long>(m)) - 1;
      while (ld_acquire_sys_u64(flags + j) < need) {
        __nanosleep(64);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > wait_ns) __trap();
      }
    }
  }
  __syncwarp();
}

enum StepFlags : int {
  kNeedResidual = 1,  // compute max|u2-u1| for this step
  kSteady = 2,        // compare residual with tol and set conv_step
  kDistributed = 4,   // partitioned run: only accumulate red[]; the group's
                      // all-reduce + decide_kernel finalise the step
  kPublish = 8,       // persistent loop: copy the final field into both buffers
};


// ---- load helpers --------------------------------------------------------
// Streamed, read-once data (weights, ids, forcing): bypass L1, L2 evict-first,
// so they do not push the gathered field out of L2.
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream_s32(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_unchanged() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Gathered field values: coherent load (the buffer is written by the previous
// step, which may still be draining under programmatic dependent launch).
__device__ __forceinline__ double ld_field(const double* p) { return *p; }

__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch_dependents() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.launch_dependents;");
#endif
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// One row: serial-j dot product, update, written in exactly the reference
// association.  `w`/`c` are the row's preloaded weights / node ids.
template <int NJ>
__device__ __forceinline__ double row_update(const double (&w)[NJ], const int (&c)[NJ],
                                             const double* u_in, double f, double u_self,
                                             double dt) {
  double g[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) g[j] = ld_field(u_in + c[j]);
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(w[j], g[j]));
  return __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(f, acc)));
}

// CTA epilogue shared by the streaming kernels: OR the non-finite flag, max the
// residual, and let the last CTA of the step finalise the step (ticket).
// span: time steps the launch advanced (1, or 2 for the two-step tile kernel,
// whose residual belongs to its second step and whose bad flag marks the pair)
__device__ __forceinline__ void step_epilogue(DevStatus* st, long long gstep, bool bad,
                                              unsigned long long dbits, int flags, int span = 1) {
  __shared__ unsigned long long s_max[32];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  const bool dist = (flags & kDistributed) != 0;
  const int any_bad = __syncthreads_or(bad ? 1 : 0);
  if (any_bad && threadIdx.x == 0) {
    if (dist) {
      atomicMax(&st->red[1], 1ull);
    } else {
      atomicCAS(reinterpret_cast<unsigned long long*>(&st->bad_step),
                static_cast<unsigned long long>(-1LL), static_cast<unsigned long long>(gstep));
    }
  }
  if (flags & kNeedResidual) {
    unsigned long long m = warp_max_u64(dbits);
    if (lane == 0) s_max[warp] = m;
    __syncthreads();
    if (warp == 0) {
      m = lane < nwarps ? s_max[lane] : 0ull;
      m = warp_max_u64(m);
      if (lane == 0 && m != 0ull) atomicMax(dist ? &st->red[0] : &st->res_bits, m);
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(&st->ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    if ((flags & kNeedResidual) && !dist) {
      const unsigned long long m = atomicExch(&st->res_bits, 0ull);
      st->last_res_bits = m;
      st->last_res_step = gstep + span - 1;
      if ((flags & kSteady) && st->bad_step < 0) {
        const double r = __ddiv_rn(__longlong_as_double(static_cast<long long>(m)), st->dt);
        if (r <= st->tol) st->conv_step = gstep + span - 1;
      }
    }
    st->ticket = 0u;
    st->step = gstep + span;
    __threadfence();
  }
}

// Streaming step: one thread per row, grid-stride over slices.  NJ > 0 is the
// compile-time support size (fully unrolled); the generic NJ == 0 variant
// loops over a runtime n.
template <int NJ>
__global__ void __launch_bounds__(256)
step_stream_kernel(StepArgs a, const double* u_in, double* u_out, int flags) {
  const uint64_t pol = policy_evict_first();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int n = NJ > 0 ? NJ : a.n;
  // Let the next step's CTAs get scheduled as ours retire (they still wait in
  // pdl_wait() before touching the field).
  pdl_launch_dependents();

  // Prefetch this thread's first row of weights / ids before waiting on the
  // previous step: they do not depend on it.
  constexpr int KW = NJ > 0 ? NJ : 1;
  double w[KW];
  int c[KW];
  double f = 0.0;
  if (NJ > 0 && r < a.n_rows) {
    const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      w[j] = ld_stream_f64(a.W + base + 32LL * j, pol);
      c[j] = ld_stream_s32(a.C + base + 32LL * j, pol);
    }
    f = ld_stream_f64(a.F + r, pol);
  }
  pdl_wait();

  DevStatus* st = a.st;
  const long long gstep = *reinterpret_cast<volatile long long*>(&st->step);
  const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
  const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
  // loop already stopped (push-mode groups keep stepping: the peers wait on us)
  if (!a.wait_flags && ((bs >= 0 && bs < gstep) || (cs >= 0 && cs < gstep))) return;
  wait_peers(a.wait_flags, a.wait_mask, a.st, threadIdx.x < 32, static_cast<int>(blockDim.x), a.wait_ns);
  const double dt = st->dt;

  bool bad = false;
  unsigned long long dmax = 0ull;
  bool first = true;
  for (; r < a.n_rows; r += stride) {
    const long long node = a.dst_base + r;
    double value, u_self;
    if constexpr (NJ > 0) {
      if (!first) {
        const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          w[j] = ld_stream_f64(a.W + base + 32LL * j, pol);
          c[j] = ld_stream_s32(a.C + base + 32LL * j, pol);
        }
        f = ld_stream_f64(a.F + r, pol);
      }
      u_self = ld_field(u_in + node);
      value = row_update<NJ>(w, c, u_in, f, u_self, dt);
    } else {
      const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
      double acc = 0.0;
      int j = 0;
      for (; j + 4 <= n; j += 4) {
        double wv[4], g[4];
        int cv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wv[q] = ld_stream_f64(a.W + base + 32LL * (j + q), pol);
          cv[q] = ld_stream_s32(a.C + base + 32LL * (j + q), pol);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q] = ld_field(u_in + cv[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = __dadd_rn(acc, __dmul_rn(wv[q], g[q]));
      }
      for (; j < n; ++j) {
        const double wv = ld_stream_f64(a.W + base + 32LL * j, pol);
        const int cv = ld_stream_s32(a.C + base + 32LL * j, pol);
        acc = __dadd_rn(acc, __dmul_rn(wv, ld_field(u_in + cv)));
      }
      f = ld_stream_f64(a.F + r, pol);
      u_self = ld_field(u_in + node);
      value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(f, acc)));
    }
    first = false;
    u_out[node] = value;
    if (!isfinite(value)) bad = true;
    if (flags & kNeedResidual) {
      const double d = fabs(__dsub_rn(value, u_self));
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
      dmax = b > dmax ? b : dmax;
    }
  }
  step_epilogue(st, gstep, bad, dmax, flags);
}

// ---------------------------------------------------------------------------
// TMA-pipelined streaming step (the default for specialised widths).
//
// Warp-specialised and persistent: warp 0 (one elected lane) streams chunks
// of `sps` SELL slices -- weights, ids and forcing, three contiguous ranges --
// into a `stages`-deep shared-memory ring with cp.async.bulk (the 1D TMA
// path) and mbarrier transaction counts; CW consumer warps each take one
// 32-row slice at a time from the ring, gather u through L1/L2 and write the
// update.  The copies do not depend on the previous step, so the producer
// issues the whole ring before griddepcontrol.wait: under programmatic
// dependent launch step s+1 is already streaming its weights while step s
// drains.  Arithmetic and j-order are those of row_update (bitwise parity).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_count(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

struct TmaGeom {
  int sps;     // slices per chunk (stage)
  int stages;  // ring depth
  int contig;  // pair kernel: log2(sps); unused by the step kernel
  // each CTA's first `res` chunks are streamed with L2::evict_last: the ring
  // fill (issued before griddepcontrol.wait while the previous step drains,
  // and right after it) then comes from L2 in every step but the first, which
  // shortens each step's start (C2: +4 % at res = 1.5 x stages,
  // profiles/README.md); the rest of the stream stays evict_first
  long long res;
};

template <int NJ, int IB>
__host__ __device__ constexpr int tma_slice_bytes() {
  return NJ * 32 * (8 + IB) + 32 * 8 + (IB == 2 ? 16 : 0);  // + the slice's window bases
}

// 16-bit ids (IB == 2): each SELL slice stores its ids as 15-bit offsets from
// one of two per-slice bases (bit 15 selects base1).  With Morton-ordered rows
// 99.4-99.6 % of slices fit (profiles/README.md); the rest keep ok == 0 and
// their consumers read the int32 ids from global memory instead.  Saves 2n of
// the 12n+24 bytes each row streams.
__device__ __forceinline__ int decode_id(unsigned int v, int4 m) {
  return (v & 0x8000u) ? m.y + static_cast<int>(v & 0x7fffu) : m.x + static_cast<int>(v);
}

}  // namespace rbf
