// step_kernels.cuh -- sm_100a kernels of the explicit RBF-FD pseudo-time step
// (single-step streaming, resident, cluster loops, packing/renumbering).
// Semantics, layout and parity rules: common.cuh.
#pragma once
#include <climits>

#include "common.cuh"

namespace rbf {

__global__ void compress_ids_kernel(const int* __restrict__ C, long long n_rows, int n,
                                    unsigned short* __restrict__ C16, int4* __restrict__ meta,
                                    unsigned long long* n_overflow) {
  const int lane = threadIdx.x & 31;
  const long long S = (n_rows + 31) >> 5;
  for (long long sl = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; sl < S;
       sl += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const bool live = sl * 32 + lane < n_rows;
    const int* c = C + sl * n * 32 + lane;
    int mn = 0x7fffffff;
    for (int j = 0; j < n && live; ++j) mn = min(mn, c[32 * j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    const long long lim = static_cast<long long>(mn) + 32767;
    int mn1 = 0x7fffffff, mx1 = -1;
    for (int j = 0; j < n && live; ++j) {
      const int v = c[32 * j];
      if (v > lim) {
        mn1 = min(mn1, v);
        mx1 = max(mx1, v);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn1 = min(mn1, __shfl_xor_sync(0xffffffffu, mn1, o));
      mx1 = max(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const bool ok = (mx1 < 0) || (mx1 - mn1 <= 32767);
    const int base1 = mx1 < 0 ? mn : mn1;
    unsigned short* d = C16 + sl * n * 32 + lane;
    for (int j = 0; j < n; ++j) {
      unsigned short e = 0;
      if (live && ok) {
        const int v = c[32 * j];
        e = (v <= lim) ? static_cast<unsigned short>(v - mn)
                       : static_cast<unsigned short>(0x8000 | (v - base1));
      }
      d[32 * j] = e;
    }
    if (lane == 0) {
      meta[sl] = make_int4(mn, base1, ok ? 1 : 0, 0);
      if (!ok) atomicAdd(n_overflow, 1ull);
    }
  }
}

// RPL: slices per consumer unit (each lane carries RPL independent rows, so a
// warp keeps RPL*NJ gathers in flight); sps must be a multiple of RPL.
template <int NJ, int CW, int RPL, int IB>
__global__ void __launch_bounds__(32 * (CW + 1), 1)
step_tma_kernel(StepArgs a, const double* u_in, double* u_out, int flags, TmaGeom g) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  constexpr int kMaxStages = 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(tma_smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* ring = tma_smem + 2 * kMaxStages * sizeof(uint64_t);
  // Chunks issued so far by the producer.  A consumer strides CW units ahead
  // per iteration and can lead the producer by more than one ring lap; an
  // mbarrier parity wait two phases ahead would alias the previous phase, so
  // consumers first wait until their chunk has been armed (expect_tx issued).
  __shared__ int s_issued;
  const int sps = g.sps, stages = g.stages;
  const int wbytes = sps * NJ * 32 * 8, cbytes = sps * NJ * 32 * IB;
  const int stage_bytes = sps * tma_slice_bytes<NJ, IB>();
  const long long S = (a.n_rows + 31) >> 5;
  const long long nchunks = (S + sps - 1) / sps;
  // CTA b streams chunks b, b + G, b + 2G, ... (G = gridDim.x).  Chunk,
  // ring-stage and phase indices are 32-bit (no 64-bit division on the
  // per-unit path: the SASS of a 64-bit div/mod is a subroutine call).
  const int my_n = blockIdx.x < nchunks ? static_cast<int>((nchunks - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    s_issued = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], static_cast<uint32_t>(sps / RPL));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_launch_dependents();

  DevStatus* st = a.st;
  bool bad = false;
  unsigned long long dmax = 0ull;
  long long gstep = 0;
#ifdef RBF_TRACE
  unsigned long long tr[4] = {0, 0, 0, 0};  // RBFFD_TRACE (thread 0; built with make TRACE=1)
  if (a.trace && threadIdx.x == 0) tr[0] = globaltimer();
#endif

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
      auto issue = [&](int i, int s) {
        const long long c = blockIdx.x + static_cast<long long>(i) * gridDim.x;
        const uint64_t pol = i < g.res ? pol_last : pol_first;
        const long long s0 = c * sps;
        const int ns = static_cast<int>(S - s0 < sps ? S - s0 : sps);
        unsigned char* dst = ring + static_cast<size_t>(s) * stage_bytes;
        const uint32_t wb = ns * NJ * 32 * 8, cb = ns * NJ * 32 * IB, fb = ns * 32 * 8;
        const uint32_t mb = IB == 2 ? ns * 16 : 0;
        mbar_expect_tx(&full[s], wb + cb + fb + mb);
        bulk_g2s(dst, a.W + s0 * NJ * 32, wb, &full[s], pol);
        if constexpr (IB == 2) {
          bulk_g2s(dst + wbytes, a.C16 + s0 * NJ * 32, cb, &full[s], pol);
          bulk_g2s(dst + wbytes + cbytes + sps * 32 * 8, a.meta + s0, mb, &full[s], pol);
        } else {
          bulk_g2s(dst + wbytes, a.C + s0 * NJ * 32, cb, &full[s], pol);
        }
        bulk_g2s(dst + wbytes + cbytes, a.F + s0 * 32, fb, &full[s], pol);
        __threadfence_block();  // order the arm before the publication below
        *reinterpret_cast<volatile int*>(&s_issued) = i + 1;
      };
      const int pre = my_n < stages ? my_n : stages;
      for (int i = 0; i < pre; ++i) issue(i, i);  // before the dependency wait
      pdl_wait();
#ifdef RBF_TRACE
      if (a.trace) tr[1] = globaltimer();
#endif
      const long long g0 = *reinterpret_cast<volatile long long*>(&st->step);
      const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
      const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
      if (!a.wait_flags && ((bs >= 0 && bs < g0) || (cs >= 0 && cs < g0))) {
        for (int i = 0; i < pre; ++i) mbar_wait(&full[i], 0);  // drain the ring
        return;
      }
      // chunk i reuses stage i % stages once its previous occupant (chunk
      // i - stages, empty-barrier phase (i / stages - 1) & 1) was consumed
      if constexpr (NJ > 32) {
        // wide stencils (1-slice chunks, consumer-bound): this form -- stage
        // and phase from a 64-bit index each chunk -- measured 5 % faster at
        // C4 (2.60 vs 2.74 ms per step, profiles/r02/ab_producer_c4.log) than
        // the incremental one below, which is 0.5 % faster at n = 15; the
        // mechanism was not isolated (same copies, same waits)
        for (long long i = pre; i < my_n; ++i) {
          const int s = static_cast<int>(i % stages);
          mbar_wait(&empty[s], static_cast<uint32_t>(((i / stages) - 1) & 1));
          issue(static_cast<int>(i), s);
        }
      } else {
        int s = 0;
        uint32_t ph = 0;
        for (int i = pre; i < my_n; ++i) {
          mbar_wait(&empty[s], ph);
          issue(i, s);
          if (++s == stages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
#ifdef RBF_TRACE
      if (a.trace) tr[2] = globaltimer();
#endif
    } else {
      pdl_wait();
      const long long g0 = *reinterpret_cast<volatile long long*>(&st->step);
      const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
      const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
      if (!a.wait_flags && ((bs >= 0 && bs < g0) || (cs >= 0 && cs < g0))) return;
    }
    gstep = *reinterpret_cast<volatile long long*>(&st->step);
  } else {
    pdl_wait();
    gstep = *reinterpret_cast<volatile long long*>(&st->step);
    const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
    const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
    if (!a.wait_flags && ((bs >= 0 && bs < gstep) || (cs >= 0 && cs < gstep))) return;
    // push-mode parts order their rows interior-first: a warp waits for the
    // neighbours' halo pushes only before its first unit with a row >=
    // halo_row0, so rows that read no halo value overlap the exchange
    bool waited = a.wait_flags == nullptr;
    const double dt = st->dt;
    const int upc = sps / RPL;  // consumer units per chunk
    // this warp's units q = warp-1, warp-1+CW, ... -> (chunk i, unit u),
    // ring stage s, phase ph (32-bit arithmetic)
    const int total = my_n * upc;
    for (int q = warp - 1; q < total; q += CW) {
      const int i = q / upc, u = q - i * upc;
      const int s = i % stages;
      const uint32_t ph = static_cast<uint32_t>((i / stages) & 1);
      const int slot0 = u * RPL;
      if (lane == 0) {
        while (*reinterpret_cast<volatile int*>(&s_issued) <= i) __nanosleep(64);
      }
      __syncwarp();
      mbar_wait(&full[s], ph);
      const unsigned char* base = ring + static_cast<size_t>(s) * stage_bytes;
      const long long slice0 = (blockIdx.x + static_cast<long long>(i) * gridDim.x) * sps + slot0;
      if (!waited && (slice0 + RPL) * 32 > a.halo_row0) {
        wait_peers_warp(a.wait_flags, a.wait_mask, a.st, a.wait_ns);
        waited = true;
      }
      {
        bool live[RPL];
        double g[RPL][NJ];
        double u_self[RPL];
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const long long r = (slice0 + t) * 32 + lane;
          live[t] = (slice0 + t) < S && r < a.n_rows;
          if (live[t]) {
            // ids from the ring -> gathers, all issued before the first use
            int c0;
            if constexpr (IB == 2) {
              const int4 m = reinterpret_cast<const int4*>(base + wbytes + cbytes + sps * 32 * 8)[slot0 + t];
              if (m.z) {
                const unsigned short* sC =
                    reinterpret_cast<const unsigned short*>(base + wbytes) + (slot0 + t) * NJ * 32;
                c0 = decode_id(sC[lane], m);
                g[t][0] = ld_field(u_in + c0);
#pragma unroll
                for (int j = 1; j < NJ; ++j) g[t][j] = ld_field(u_in + decode_id(sC[j * 32 + lane], m));
              } else {  // slice too spread for two 15-bit windows: int32 ids from HBM
                const int* gC = a.C + (slice0 + t) * NJ * 32 + lane;
                c0 = __ldg(gC);
                g[t][0] = ld_field(u_in + c0);
#pragma unroll
                for (int j = 1; j < NJ; ++j) g[t][j] = ld_field(u_in + __ldg(gC + 32 * j));
              }
            } else {
              const int* sC = reinterpret_cast<const int*>(base + wbytes) + (slot0 + t) * NJ * 32;
              c0 = sC[lane];
              g[t][0] = ld_field(u_in + c0);
#pragma unroll
              for (int j = 1; j < NJ; ++j) g[t][j] = ld_field(u_in + sC[j * 32 + lane]);
            }
            // stencils list the centre first (neighborhoods.py:29-32): reuse it
            const long long node = a.dst_base + r;
            u_self[t] = (c0 == node) ? g[t][0] : ld_field(u_in + node);
          }
        }
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          if (!live[t]) continue;
          const long long r = (slice0 + t) * 32 + lane;
          const double* sW = reinterpret_cast<const double*>(base) + (slot0 + t) * NJ * 32;
          const double* sF = reinterpret_cast<const double*>(base + wbytes + cbytes) + (slot0 + t) * 32;
          double acc = 0.0;  // weights read from the ring inside the serial chain
#pragma unroll
          for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(sW[j * 32 + lane], g[t][j]));
          const double value = __dadd_rn(u_self[t], __dmul_rn(dt, __dadd_rn(sF[lane], acc)));
          u_out[a.dst_base + r] = value;
          if (!isfinite(value)) bad = true;
          if (flags & kNeedResidual) {
            const unsigned long long b = static_cast<unsigned long long>(
                __double_as_longlong(fabs(__dsub_rn(value, u_self[t]))));
            dmax = b > dmax ? b : dmax;
          }
        }
      }
      // unit fully consumed: hand it back to the producer (the arrive has
      // release semantics; __syncwarp orders the other lanes' shared reads)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // every warp has waited before the step completes: the push that follows
    // this step must not overwrite a neighbour's buffer it still reads
    // (send-only neighbours, parts without halo rows)
    if (!waited) wait_peers_warp(a.wait_flags, a.wait_mask, a.st, a.wait_ns);
  }
  step_epilogue(st, gstep, bad, dmax, flags);
#ifdef RBF_TRACE
  if (a.trace && threadIdx.x == 0) {  // after the epilogue: the CTA's consumers are done
    tr[3] = globaltimer();
    unsigned long long* o = a.trace + (static_cast<long long>(gstep % a.trace_cap) * gridDim.x + blockIdx.x) * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = tr[k];
  }
#endif
}

// ---------------------------------------------------------------------------
// Persistent streaming loop: the whole run in one cooperative launch (1 CTA
// per SM), for problems the streaming step serves.  Per step, the launch
// boundary of the graph loop costs a ring drain (the last `stages` chunks of
// every CTA are consumed with no new stream traffic) and 4.9 us until
// griddepcontrol.wait returns (profiles/r02/trace_c2_pdl.txt).  Here the
// producer never stops: the chunk sequence of step k+1 is the same as step
// k's (the weights do not depend on the field), so it streams step k+1 into
// every stage the consumers free while they finish step k and wait at the
// grid barrier; the consumers resume on a full ring.  The grid barrier and
// the per-step decisions (first non-finite step, residual, steady stop) are
// grid_loop_kernel's: a monotonic arrival counter carrying the non-finite
// flag in its high bits (read only at the exact count), residual maxima in
// three rotating slots.  Same arithmetic and j-order as step_tma_kernel.
struct LoopArgs {
  double* U0;  // start field; the final field is published into both buffers
  double* U1;
  long long limit;             // steps to run (fixed: steps, steady: max_steps)
  int flags;                   // kSteady
  unsigned long long* red;     // [0..2] residual slots, [6] arrival counter
};

template <int NJ, int CW, int IB>
__global__ void __launch_bounds__(32 * (CW + 1), 1)
stream_loop_kernel(StepArgs a, LoopArgs L, TmaGeom g) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  constexpr int kMaxStages = 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(tma_smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* ring = tma_smem + 2 * kMaxStages * sizeof(uint64_t);
  __shared__ long long s_issued;   // chunks armed so far (all steps)
  __shared__ int s_stop;           // consumers -> producer: stop streaming
  __shared__ unsigned long long s_max[32];
  __shared__ unsigned int s_bad[32];
  __shared__ unsigned long long s_seen;
  const int sps = g.sps, stages = g.stages;
  const int wbytes = sps * NJ * 32 * 8, cbytes = sps * NJ * 32 * IB;
  const int stage_bytes = sps * tma_slice_bytes<NJ, IB>();
  const long long S = (a.n_rows + 31) >> 5;
  const long long nchunks = (S + sps - 1) / sps;
  const int my_n = blockIdx.x < nchunks ? static_cast<int>((nchunks - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long total_q = L.limit * my_n;  // chunks this CTA streams over the run
  constexpr unsigned long long kBad = 1ull << 40, kCount = kBad - 1;

  if (threadIdx.x == 0) {
    s_issued = 0;
    s_stop = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], static_cast<uint32_t>(sps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  DevStatus* st = a.st;

  if (warp == 0) {
    if (lane == 0) {
      // chunks i < g.res of every step are streamed with L2::evict_last and
      // stay L2-resident across steps; the rest with evict_first
      // g.contig (unused by this kernel's geometry) selects the stream's L2
      // policy for experiments: 0 evict_first (default), 1 evict_normal,
      // 2 evict_unchanged (RBFFD_LOOP_POLICY)
      const uint64_t pol_first = g.contig == 1 ? policy_evict_normal()
                                 : g.contig == 2 ? policy_evict_unchanged() : policy_evict_first();
      const uint64_t pol_last = policy_evict_last();
      int i = 0, s = 0;
      uint32_t ph = 1;  // empty-barrier parity of the stage's previous occupant
      long long q = 0;
      for (; q < total_q; ++q) {
        if (q >= stages) {  // wait for the stage's previous occupant, or a stop
          bool stopped = false;
          while (true) {
            uint32_t done;
            asm volatile(
                "{\n.reg .pred P;\n"
                "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
                "selp.u32 %0, 1, 0, P;\n}\n"
                : "=r"(done) : "r"(smem_u32(&empty[s])), "r"(ph) : "memory");
            if (done) break;
            if (*reinterpret_cast<volatile int*>(&s_stop)) {
              stopped = true;
              break;
            }
          }
          if (stopped) break;
        }
        const long long c = blockIdx.x + static_cast<long long>(i) * gridDim.x;
        const long long s0 = c * sps;
        const int ns = static_cast<int>(S - s0 < sps ? S - s0 : sps);
        unsigned char* dst = ring + static_cast<size_t>(s) * stage_bytes;
        const uint32_t wb = ns * NJ * 32 * 8, cb = ns * NJ * 32 * IB, fb = ns * 32 * 8;
        const uint32_t mb = IB == 2 ? ns * 16 : 0;
        const uint64_t pol = i < g.res ? pol_last : pol_first;
        mbar_expect_tx(&full[s], wb + cb + fb + mb);
        bulk_g2s(dst, a.W + s0 * NJ * 32, wb, &full[s], pol);
        if constexpr (IB == 2) {
          bulk_g2s(dst + wbytes, a.C16 + s0 * NJ * 32, cb, &full[s], pol);
          bulk_g2s(dst + wbytes + cbytes + sps * 32 * 8, a.meta + s0, mb, &full[s], pol);
        } else {
          bulk_g2s(dst + wbytes, a.C + s0 * NJ * 32, cb, &full[s], pol);
        }
        bulk_g2s(dst + wbytes + cbytes, a.F + s0 * 32, fb, &full[s], pol);
        __threadfence_block();
        *reinterpret_cast<volatile long long*>(&s_issued) = q + 1;
        if (++i == my_n) i = 0;
        if (++s == stages) {
          s = 0;
          ph ^= 1u;
        }
      }
      // leave no bulk copy in flight: wait for the last `stages` armed chunks
      // (a consumed one has completed its phase already)
      for (long long r = (q > stages ? q - stages : 0); r < q; ++r)
        mbar_wait(&full[r % stages], static_cast<uint32_t>((r / stages) & 1));
    }
    return;  // warp 0 takes no part in the consumers' barriers
  }

  // ---- consumer warps
  const int ctid = threadIdx.x - 32, nthreads = 32 * CW;
  const double dt = st->dt, tol = st->tol;
  const bool steady = (L.flags & kSteady) != 0;
  const int upc = sps;  // one slice per unit
  long long bad_step = -1, conv_step = -1, last_res_step = -1, step = 0;
  unsigned long long last_bits = 0;
  for (; step < L.limit; ++step) {
    const double* u_in = (step & 1) ? L.U1 : L.U0;
    double* u_out = (step & 1) ? L.U0 : L.U1;
    const bool need = steady || step == L.limit - 1;
    bool bad = false;
    unsigned long long dmax = 0ull;
#ifdef RBF_TRACE
    unsigned long long tr0 = 0;
    if (a.trace && ctid == 0) tr0 = globaltimer();
#endif
    // ring position of chunk q = step * my_n + i: one 64-bit division per
    // step, 32-bit arithmetic per unit (a 64-bit div/mod is a SASS subroutine)
    const long long qbase = step * my_n;
    const long long qdiv = qbase / stages;
    const int qmod = static_cast<int>(qbase - qdiv * stages);
    const uint32_t qpar = static_cast<uint32_t>(qdiv & 1);
    for (int uq = warp - 1; uq < my_n * upc; uq += CW) {
      const int i = uq / upc, slot = uq - i * upc;
      const long long q = qbase + i;
      const int t = qmod + i, tdiv = t / stages;
      const int s = t - tdiv * stages;
      const uint32_t ph = (qpar + static_cast<uint32_t>(tdiv)) & 1u;
      if (lane == 0) {
        while (*reinterpret_cast<volatile long long*>(&s_issued) <= q) __nanosleep(64);
      }
      __syncwarp();
      mbar_wait(&full[s], ph);
      const unsigned char* base = ring + static_cast<size_t>(s) * stage_bytes;
      const long long slice = (blockIdx.x + static_cast<long long>(i) * gridDim.x) * sps + slot;
      const long long r = slice * 32 + lane;
      if (slice < S && r < a.n_rows) {
        double gv[NJ];
        int c0;
        if constexpr (IB == 2) {
          const int4 m = reinterpret_cast<const int4*>(base + wbytes + cbytes + sps * 32 * 8)[slot];
          if (m.z) {
            const unsigned short* sC = reinterpret_cast<const unsigned short*>(base + wbytes) + slot * NJ * 32;
            c0 = decode_id(sC[lane], m);
            gv[0] = ld_field(u_in + c0);
#pragma unroll
            for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + decode_id(sC[j * 32 + lane], m));
          } else {
            const int* gC = a.C + slice * NJ * 32 + lane;
            c0 = __ldg(gC);
            gv[0] = ld_field(u_in + c0);
#pragma unroll
            for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + __ldg(gC + 32 * j));
          }
        } else {
          const int* sC = reinterpret_cast<const int*>(base + wbytes) + slot * NJ * 32;
          c0 = sC[lane];
          gv[0] = ld_field(u_in + c0);
#pragma unroll
          for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + sC[j * 32 + lane]);
        }
        const long long node = a.dst_base + r;
        const double u_self = (c0 == node) ? gv[0] : ld_field(u_in + node);
        const double* sW = reinterpret_cast<const double*>(base) + slot * NJ * 32;
        const double* sF = reinterpret_cast<const double*>(base + wbytes + cbytes) + slot * 32;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(sW[j * 32 + lane], gv[j]));
        const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(sF[lane], acc)));
        u_out[node] = value;
        if (!isfinite(value)) bad = true;
        if (need) {
          const unsigned long long b =
              static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
          dmax = b > dmax ? b : dmax;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // ---- CTA partials (consumer warps), then the grid barrier
    const unsigned int wb = __ballot_sync(0xffffffffu, bad) ? 1u : 0u;
    const unsigned long long wm = need ? warp_max_u64(dmax) : 0ull;
    if (lane == 0) {
      s_bad[warp] = wb;
      s_max[warp] = wm;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
    const int rs = static_cast<int>(step % 3);
#ifdef RBF_TRACE
    unsigned long long tr1 = 0;
    if (a.trace && ctid == 0) tr1 = globaltimer();
#endif
    if (ctid == 0) {
      unsigned int cbad = 0;
      unsigned long long cm = 0ull;
      for (int w = 1; w <= CW; ++w) {
        cbad |= s_bad[w];
        cm = s_max[w] > cm ? s_max[w] : cm;
      }
      if (need && cm) atomicMax(&L.red[rs], cm);
      if (blockIdx.x == 0) L.red[(step + 1) % 3] = 0ull;  // free two barriers ahead
      __threadfence();  // this CTA's field stores before its arrival
      atomicAdd(&L.red[6], 1ull + (cbad ? kBad : 0ull));
      const unsigned long long target = static_cast<unsigned long long>(step + 1) * gridDim.x;
      unsigned long long v;
      const unsigned long long t0 = globaltimer();
      for (int spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&L.red[6]) : "memory");
        if ((v & kCount) >= target) break;
        if ((spin & 1023) == 1023 && globaltimer() - t0 > 20000000000ull) __trap();
      }
      // flag bits are this barrier's only at the exact count (a CTA already
      // past it has passed a clean barrier: a flagged one stops every CTA)
      s_seen = ((v & kCount) == target) ? v : 0ull;
#ifdef RBF_TRACE
      if (a.trace) {  // per step and CTA: start, arrival, release, chunks armed at arrival
        unsigned long long* o = a.trace + ((step % a.trace_cap) * gridDim.x + blockIdx.x) * 4;
        o[0] = tr0;
        o[1] = tr1;
        o[2] = globaltimer();
        o[3] = static_cast<unsigned long long>(*reinterpret_cast<volatile long long*>(&s_issued) - (step + 1) * my_n);
      }
#endif
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
    // the reference checks every step's flag before its residual (solver.py:200-217)
    bool stop = false;
    if ((s_seen >> 40) != 0) {
      bad_step = step;
      stop = true;
    } else if (need) {
      const unsigned long long gm = *reinterpret_cast<volatile unsigned long long*>(&L.red[rs]);
      last_bits = gm;
      last_res_step = step;
      if (steady && __ddiv_rn(__longlong_as_double(static_cast<long long>(gm)), dt) <= tol) {
        conv_step = step;
        stop = true;
      }
    }
    if (stop) {
      ++step;  // the field of this step (its u2) is the result
      break;
    }
  }
  if (ctid == 0) *reinterpret_cast<volatile int*>(&s_stop) = 1;  // release the producer
  // with kPublish (copy-back runs): the final field (buffer step & 1) into
  // the other buffer too, every CTA copying the rows it wrote; otherwise the
  // host takes buffer st->step & 1 as the current one
  const double* uf = (step & 1) ? L.U1 : L.U0;
  double* uo = (step & 1) ? L.U0 : L.U1;
  for (int uq = warp - 1; (L.flags & kPublish) && uq < my_n * upc; uq += CW) {
    const int i = uq / upc, slot = uq - i * upc;
    const long long slice = (blockIdx.x + static_cast<long long>(i) * gridDim.x) * sps + slot;
    const long long r = slice * 32 + lane;
    if (slice < S && r < a.n_rows) uo[a.dst_base + r] = uf[a.dst_base + r];
  }
  if (blockIdx.x == 0 && ctid == 0) {
    st->bad_step = bad_step;
    st->conv_step = conv_step;
    st->last_res_bits = last_bits;
    st->last_res_step = last_res_step;
    st->step = (bad_step >= 0) ? bad_step + 1 : step;
  }
}

// ---------------------------------------------------------------------------
// Partitioned persistent loop (fixed-step fast path of a
// push-mode group): every local part of the group runs the streaming loop
// above on its own CTA range of ONE cooperative launch, and the halo exchange
// is fused into it.  A row whose value a neighbour part reads is stored
// straight into the neighbour's field buffer (its halo slot in the buffer the
// neighbour reads next step: P2P stores over NVLink when the neighbour is
// another GPU's part mapped through CUDA IPC) by the consumer lane that
// computed it.  Per step and part: part-local grid barrier (arrival counter);
// its last arriver publishes "steps done" to every neighbour's arrival array
// (release; system scope across GPUs).  A warp waits for its neighbours'
// previous step before its first unit at or after `sync_row0` -- the first
// row that reads a halo value or is pushed (parts order those rows last), so
// interior rows overlap the neighbours' step -- and every CTA that pushes has
// waited: no push overwrites a halo slot its neighbour still reads.
// No early stop: the group's end-of-run reduction decides (first non-finite
// step -> exact replay, solver.py:200-206), like the graph fast path.
struct PartLoop {
  StepArgs a;                 // W / C16 / C / meta / F / n_rows / dst_base / st of the part
  double* U[2];               // the part's field buffers (start field in U[0])
  int cta0, ncta;             // CTA range of the part in the launch
  long long sync_row0;        // first row that reads a halo value or is pushed
  unsigned long long* bar;    // [0] arrival counter, [1] first non-finite step (min), [2] residual bits (max)
  const int* push_off;        // [S+1] per-slice ranges of push_ent (nullptr: no pushes)
  const unsigned long long* push_ent;  // (peer << 58) | (lane << 52) | slot in the peer's numbering
  double* peer_u[kMaxPushPeers][2];
  unsigned long long* nbr_flags[kMaxPushPeers];  // neighbours' arrival arrays (this part writes [my_id])
  const unsigned long long* my_flags;            // this part's arrival array (neighbours write [their id])
  unsigned long long wait_mask;                  // neighbour ids to wait for
  unsigned long long base;    // arrival count before this run (steps pushed in earlier runs)
  int n_nbr, my_id, sys_scope;
};

// Acquire polls at the scope of the neighbours (gpu: parts of this launch;
// sys: parts on other GPUs).  A relaxed poll + one fence.acq_rel.sys was
// measured slower (two in-process parts at C2: 33.9 vs 28.7 us per step).
__device__ __forceinline__ void wait_arrivals(const unsigned long long* flags, unsigned long long mask,
                                              unsigned long long need, int sys, unsigned long long wait_ns) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long t0 = globaltimer();
    for (unsigned long long m = mask; m; m &= m - 1) {
      const int j = __ffsll(static_cast<long long>(m)) - 1;
      for (;;) {
        unsigned long long v;
        if (sys)
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + j) : "memory");
        else
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + j) : "memory");
        if (v >= need) break;
        __nanosleep(32);
        if (globaltimer() - t0 > wait_ns) __trap();  // RBFFD_WAIT_TIMEOUT_MS (default 20 s)
      }
    }
  }
  __syncwarp();
}

template <int NJ, int CW, int IB>
__global__ void __launch_bounds__(32 * (CW + 1), 1)
part_loop_kernel(const PartLoop* __restrict__ parts, int n_parts, long long limit, TmaGeom g) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  constexpr int kMaxStages = 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(tma_smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* ring = tma_smem + 2 * kMaxStages * sizeof(uint64_t);
  __shared__ long long s_issued;
  __shared__ unsigned long long s_max[32];
  __shared__ unsigned int s_bad[32];
#ifdef RBF_TRACE
  __shared__ unsigned long long s_wait;  // longest neighbour wait of a warp this step (ns)
#endif
  int q_part = 0;
  while (q_part + 1 < n_parts && static_cast<int>(blockIdx.x) >= parts[q_part + 1].cta0) ++q_part;
  const PartLoop& P = parts[q_part];  // rarely used fields stay in global memory
  const StepArgs a = P.a;
  double* const U0 = P.U[0];
  double* const U1 = P.U[1];
  const long long sync_row0 = P.sync_row0;
  const int* const push_off = P.push_off;
  const unsigned long long* const push_ent = P.push_ent;
  const unsigned long long* const my_flags = P.my_flags;
  const unsigned long long wait_mask = P.wait_mask, fbase = P.base;
  unsigned long long* const bar = P.bar;
  const int sys_scope = P.sys_scope;
  const int G = P.ncta, b = static_cast<int>(blockIdx.x) - P.cta0;
  const int sps = g.sps, stages = g.stages;
  const int wbytes = sps * NJ * 32 * 8, cbytes = sps * NJ * 32 * IB;
  const int stage_bytes = sps * tma_slice_bytes<NJ, IB>();
  const long long S = (a.n_rows + 31) >> 5;
  const long long nchunks = (S + sps - 1) / sps;
  const int my_n = b < nchunks ? static_cast<int>((nchunks - 1 - b) / G + 1) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long total_q = limit * my_n;

  if (threadIdx.x == 0) {
    s_issued = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], static_cast<uint32_t>(sps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // producer: the part's chunk sequence, step after step
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int i = 0, s = 0;
      uint32_t ph = 1;
      for (long long q = 0; q < total_q; ++q) {
        if (q >= stages) mbar_wait(&empty[s], ph);
        const long long c = b + static_cast<long long>(i) * G;
        const long long s0 = c * sps;
        const int ns = static_cast<int>(S - s0 < sps ? S - s0 : sps);
        unsigned char* dst = ring + static_cast<size_t>(s) * stage_bytes;
        const uint32_t wb = ns * NJ * 32 * 8, cb = ns * NJ * 32 * IB, fb = ns * 32 * 8;
        const uint32_t mb = IB == 2 ? ns * 16 : 0;
        mbar_expect_tx(&full[s], wb + cb + fb + mb);
        bulk_g2s(dst, a.W + s0 * NJ * 32, wb, &full[s], pol);
        if constexpr (IB == 2) {
          bulk_g2s(dst + wbytes, a.C16 + s0 * NJ * 32, cb, &full[s], pol);
          bulk_g2s(dst + wbytes + cbytes + sps * 32 * 8, a.meta + s0, mb, &full[s], pol);
        } else {
          bulk_g2s(dst + wbytes, a.C + s0 * NJ * 32, cb, &full[s], pol);
        }
        bulk_g2s(dst + wbytes + cbytes, a.F + s0 * 32, fb, &full[s], pol);
        __threadfence_block();
        *reinterpret_cast<volatile long long*>(&s_issued) = q + 1;
        if (++i == my_n) i = 0;
        if (++s == stages) {
          s = 0;
          ph ^= 1u;
        }
      }
      // every armed chunk is consumed before the consumers leave: no copy in flight
    }
    return;
  }

  // ---- consumer warps
  const int ctid = threadIdx.x - 32, nthreads = 32 * CW;
  const double dt = a.st->dt;
  const int upc = sps;
  for (long long step = 0; step < limit; ++step) {
    const double* u_in = (step & 1) ? U1 : U0;
    double* u_out = (step & 1) ? U0 : U1;
    const int ob = static_cast<int>((step & 1) ^ 1);  // the neighbours' buffer this step writes
    const bool need = step == limit - 1;
    bool bad = false, waited = wait_mask == 0ull;
    unsigned long long dmax = 0ull;
#ifdef RBF_TRACE
    unsigned long long tr0 = 0;
    if (a.trace && ctid == 0) {
      tr0 = globaltimer();
      s_wait = 0;
    }
#endif
    const long long qbase = step * my_n;
    const long long qdiv = qbase / stages;
    const int qmod = static_cast<int>(qbase - qdiv * stages);
    const uint32_t qpar = static_cast<uint32_t>(qdiv & 1);
    for (int uq = warp - 1; uq < my_n * upc; uq += CW) {
      const int i = uq / upc, slot = uq - i * upc;
      const long long q = qbase + i;
      const int t = qmod + i, tdiv = t / stages;
      const int s = t - tdiv * stages;
      const uint32_t ph = (qpar + static_cast<uint32_t>(tdiv)) & 1u;
      if (lane == 0) {
        while (*reinterpret_cast<volatile long long*>(&s_issued) <= q) __nanosleep(64);
      }
      __syncwarp();
      mbar_wait(&full[s], ph);
      const unsigned char* base = ring + static_cast<size_t>(s) * stage_bytes;
      const long long slice = (b + static_cast<long long>(i) * G) * sps + slot;
      if (!waited && (slice + 1) * 32 > sync_row0) {
#ifdef RBF_TRACE
        const unsigned long long tw = globaltimer();
#endif
        wait_arrivals(my_flags, wait_mask, fbase + static_cast<unsigned long long>(step), sys_scope, a.wait_ns);
        waited = true;
#ifdef RBF_TRACE
        if (a.trace && lane == 0) atomicMax(&s_wait, globaltimer() - tw);
#endif
      }
      const long long r = slice * 32 + lane;
      double value = 0.0;
      if (slice < S && r < a.n_rows) {
        double gv[NJ];
        int c0;
        if constexpr (IB == 2) {
          const int4 m = reinterpret_cast<const int4*>(base + wbytes + cbytes + sps * 32 * 8)[slot];
          if (m.z) {
            const unsigned short* sC = reinterpret_cast<const unsigned short*>(base + wbytes) + slot * NJ * 32;
            c0 = decode_id(sC[lane], m);
            gv[0] = ld_field(u_in + c0);
#pragma unroll
            for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + decode_id(sC[j * 32 + lane], m));
          } else {
            const int* gC = a.C + slice * NJ * 32 + lane;
            c0 = __ldg(gC);
            gv[0] = ld_field(u_in + c0);
#pragma unroll
            for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + __ldg(gC + 32 * j));
          }
        } else {
          const int* sC = reinterpret_cast<const int*>(base + wbytes) + slot * NJ * 32;
          c0 = sC[lane];
          gv[0] = ld_field(u_in + c0);
#pragma unroll
          for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + sC[j * 32 + lane]);
        }
        const long long node = a.dst_base + r;
        const double u_self = (c0 == node) ? gv[0] : ld_field(u_in + node);
        const double* sW = reinterpret_cast<const double*>(base) + slot * NJ * 32;
        const double* sF = reinterpret_cast<const double*>(base + wbytes + cbytes) + slot * 32;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(sW[j * 32 + lane], gv[j]));
        value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(sF[lane], acc)));
        u_out[node] = value;
        if (!isfinite(value)) bad = true;
        if (need) {
          const unsigned long long bb =
              static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
          dmax = bb > dmax ? bb : dmax;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      // fused halo push: this slice's rows the neighbours read, straight into
      // their next-step buffer (warp-uniform range; the matching lane stores)
      if (push_off && slice < S && (slice + 1) * 32 > sync_row0) {  // no sent row before sync_row0
        const int pb = __ldg(push_off + slice), pe = __ldg(push_off + slice + 1);
        for (int k = pb; k < pe; ++k) {
          const unsigned long long e = __ldg(push_ent + k);
          if (static_cast<int>((e >> 52) & 31) == lane)
            P.peer_u[e >> 58][ob][e & ((1ull << 52) - 1)] = value;
        }
      }
    }
    // (a warp that neither read a halo value nor pushed need not wait: the
    // part's arrival below certifies its own reads and pushes of this step)
    const unsigned int wb = __ballot_sync(0xffffffffu, bad) ? 1u : 0u;
    const unsigned long long wm = need ? warp_max_u64(dmax) : 0ull;
    if (lane == 0) {
      s_bad[warp] = wb;
      s_max[warp] = wm;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
#ifdef RBF_TRACE
    unsigned long long tr1 = 0;
    if (a.trace && ctid == 0) tr1 = globaltimer();
#endif
    if (ctid == 0) {
      unsigned int cbad = 0;
      unsigned long long cm = 0ull;
      for (int w = 1; w <= CW; ++w) {
        cbad |= s_bad[w];
        cm = s_max[w] > cm ? s_max[w] : cm;
      }
      if (cbad) atomicMin(&bar[1], static_cast<unsigned long long>(step));
      if (need && cm) atomicMax(&bar[2], cm);
      if (sys_scope) __threadfence_system();  // field stores and P2P pushes before the arrival
      else __threadfence();
      const unsigned long long target = static_cast<unsigned long long>(step + 1) * G;
      atomicAdd(&bar[0], 1ull);  // no return value: a fire-and-forget reduction
      unsigned long long v;
      const unsigned long long t0 = globaltimer();
      for (int spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&bar[0]) : "memory");
        if (v >= target) break;
        if ((spin & 1023) == 1023 && globaltimer() - t0 > 20000000000ull) __trap();
      }
      if (b == 0) {  // the part's step is complete: tell the neighbours
        const unsigned long long fv = fbase + static_cast<unsigned long long>(step + 1);
        if (sys_scope) __threadfence_system();
        for (int j = 0; j < P.n_nbr; ++j) {
          if (sys_scope)
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.nbr_flags[j] + P.my_id), "l"(fv) : "memory");
          else
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(P.nbr_flags[j] + P.my_id), "l"(fv) : "memory");
        }
      }
#ifdef RBF_TRACE
      if (a.trace) {  // per step and CTA of the part: start, arrival, release, longest halo wait
        unsigned long long* o = a.trace + ((step % a.trace_cap) * G + b) * 4;
        o[0] = tr0;
        o[1] = tr1;
        o[2] = globaltimer();
        o[3] = s_wait;
      }
#endif
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
  }
  if (b == 0 && ctid == 0) {  // the last barrier: every CTA of the part is done
    DevStatus* st = a.st;
    const unsigned long long fb = *reinterpret_cast<volatile unsigned long long*>(&bar[1]);
    st->bad_step = fb == ~0ull ? -1 : static_cast<long long>(fb);
    st->conv_step = -1;
    st->last_res_bits = *reinterpret_cast<volatile unsigned long long*>(&bar[2]);
    st->last_res_step = limit - 1;
    st->step = limit;
  }
}

// ---------------------------------------------------------------------------
// Resident loop: the whole problem (weights, ids, forcing, both field buffers)
// lives in one CTA's shared memory and the CTA runs every step of the loop
// on-chip.  Used when the working set fits (the paper's Fig. 1 case, N=1025,
// n=15: ~190 KB), where a launch per step would dominate (the
// N=1027 case is launch/latency bound).
struct ResidentArgs {
  const double* W;   // SELL-32 global copy (read once)
  const int* C;
  const double* F;
  double* U0;        // global field buffers; U0 holds the start field
  double* U1;
  long long n_rows;
  long long N;
  long long dst_base;
  long long limit;   // steps to run (fixed: steps, steady: max_steps)
  int n;
  int flags;         // kSteady
  int copy_back;
  DevStatus* st;
};

template <int NJ>
__global__ void __launch_bounds__(1024, 1) resident_loop_kernel(ResidentArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = NJ > 0 ? NJ : a.n;
  const int rows = static_cast<int>(a.n_rows);
  const int rows_pad = (rows + 31) & ~31;
  const int N = static_cast<int>(a.N);
  // smem: W[n][rows_pad] f64 | F[rows_pad] f64 | U[2][N] f64 | C[n][rows_pad] s32
  double* sW = reinterpret_cast<double*>(smem_raw);
  double* sF = sW + static_cast<size_t>(n) * rows_pad;
  double* sU0 = sF + rows_pad;
  double* sU1 = sU0 + N;
  int* sC = reinterpret_cast<int*>(sU1 + N);
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ unsigned long long s_red[32];
  __shared__ int s_stop;

  // Load: SELL-32 (slice-major) -> j-major across the whole CTA.
  for (int r = tid; r < rows; r += nt) {
    const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
    for (int j = 0; j < n; ++j) {
      sW[j * rows_pad + r] = a.W[base + 32LL * j];
      sC[j * rows_pad + r] = a.C[base + 32LL * j];
    }
    sF[r] = a.F[r];
  }
  for (int i = tid; i < N; i += nt) {
    const double v = a.U0[i];
    sU0[i] = v;
    sU1[i] = v;
  }
  __syncthreads();

  DevStatus* st = a.st;
  const double dt = st->dt, tol = st->tol;
  const bool steady = (a.flags & kSteady) != 0;
  double* cur = sU0;
  double* nxt = sU1;
  long long step = 0;
  long long bad_step = -1, conv_step = -1;
  unsigned long long last_bits = 0;
  long long last_res_step = -1;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  for (; step < a.limit; ++step) {
    const bool need_res = steady || (step == a.limit - 1);
    bool bad = false;
    unsigned long long dmax = 0ull;
    for (int r = tid; r < rows; r += nt) {
      double acc = 0.0;
      if constexpr (NJ > 0) {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          acc = __dadd_rn(acc, __dmul_rn(sW[j * rows_pad + r], cur[sC[j * rows_pad + r]]));
      } else {
        for (int j = 0; j < n; ++j)
          acc = __dadd_rn(acc, __dmul_rn(sW[j * rows_pad + r], cur[sC[j * rows_pad + r]]));
      }
      const int node = static_cast<int>(a.dst_base) + r;
      const double u_self = cur[node];
      const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(sF[r], acc)));
      nxt[node] = value;
      bad |= !isfinite(value);
      if (need_res) {
        const unsigned long long b =
            static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
        dmax = b > dmax ? b : dmax;
      }
    }
    const int any_bad = __syncthreads_or(bad ? 1 : 0);  // also orders the nxt writes
    if (any_bad) {
      bad_step = step;
      break;  // uniform
    }
    if (need_res) {
      unsigned long long m = warp_max_u64(dmax);
      if (lane == 0) s_red[warp] = m;
      __syncthreads();
      if (warp == 0) {
        m = lane < nwarps ? s_red[lane] : 0ull;
        m = warp_max_u64(m);
        if (lane == 0) {
          s_red[0] = m;
          s_stop = steady && (__ddiv_rn(__longlong_as_double(static_cast<long long>(m)), dt) <= tol);
        }
      }
      __syncthreads();
      last_bits = s_red[0];
      last_res_step = step;
      const int stop = s_stop;
      __syncthreads();  // s_red / s_stop reused next step
      if (a.copy_back) {
        for (int i = tid; i < N; i += nt) cur[i] = nxt[i];
        __syncthreads();
      } else {
        double* t = cur; cur = nxt; nxt = t;
      }
      if (stop) {
        conv_step = step;
        ++step;
        break;
      }
    } else {
      if (a.copy_back) {
        for (int i = tid; i < N; i += nt) cur[i] = nxt[i];
        __syncthreads();
      } else {
        double* t = cur; cur = nxt; nxt = t;
      }
    }
  }
  // Publish: the field the host must read.  After a bad step that is the
  // failing step's u2 (`nxt`, solver.py:201); otherwise the current buffer.
  const double* out = (bad_step >= 0) ? nxt : cur;
  for (int i = tid; i < N; i += nt) {
    const double v = out[i];
    a.U0[i] = v;
    a.U1[i] = v;
  }
  if (tid == 0) {
    st->bad_step = bad_step;
    st->conv_step = conv_step;
    st->last_res_bits = last_bits;
    st->last_res_step = last_res_step;
    st->step = (bad_step >= 0) ? bad_step + 1 : step;
  }
}

// ---------------------------------------------------------------------------
// Cluster-resident loop: the small-problem loop spread over a thread-block
// cluster of Q CTAs (Q <= 16, one SM each) instead of one SM.  Every CTA keeps
// the whole field (double-buffered) and its own rows' weights / ids / forcing
// in shared memory; per step it updates its rows and pushes each new value
// straight into the shared memory of the CTAs whose stencils read it (DSMEM
// stores, per-row destination masks built on the host), plus its partial
// residual max / non-finite flag into every CTA's reduction slots; one
// cluster barrier (release / acquire) then publishes the step.  All CTAs take
// the same stop decision from the same reduced values (solver.py:200-217).
struct ClusterArgs {
  const double* W;          // SELL-32 (plan layout), rows of all CTAs
  const int* C;
  const double* F;
  const unsigned int* dest;    // [N_i] bit q: CTA q (other than the owner) reads this row's node
  double* U0;               // global field buffers (start field in U0)
  double* U1;
  long long n_rows, N, dst_base, limit;
  int n, flags, rpc;        // rows per CTA (even)
  DevStatus* st;
  unsigned long long* phase_cycles;  // optional [4]: compute / partials / cluster barrier / decide (CTA 0)
};

template <int NJ, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) cluster_loop_kernel(ClusterArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char cl_smem[];
  // narrow stencils in <=256-thread CTAs keep their row's weights / ids in
  // registers (one row per thread); otherwise they are read from shared memory
  constexpr bool kReg = NJ > 0 && NJ <= 32 && MAXT <= 256;
  constexpr int KR = kReg ? NJ : 1;
  const int n = NJ > 0 ? NJ : a.n;
  const int q = static_cast<int>(cluster.block_rank());
  const int Q = static_cast<int>(cluster.num_blocks());
  const int B = static_cast<int>(a.dst_base);
  const int IB = (B + 1) & ~1;             // interior rows start 16-B aligned
  const int NU = IB + static_cast<int>(a.n_rows) + 2;
  const int r0 = q * a.rpc;
  const int r1 = min(static_cast<int>(a.n_rows), r0 + a.rpc);
  const int nr = max(0, r1 - r0);
  const int rp = (a.rpc + 1) & ~1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nt + 31) >> 5;
  // smem: U[2][NU] | red[2][16*32][2] u64 | W[n][rp] | F[rp] | C[n][rp] | mask[rp] (u32)
  double* U = reinterpret_cast<double*>(cl_smem);
  unsigned long long* red = reinterpret_cast<unsigned long long*>(U + 2 * NU);
  const int slots = Q * nwarps;  // partials: one slot per (CTA, warp)
  double* sW = reinterpret_cast<double*>(red + 2 * 16 * 32 * 2);
  double* sF = sW + static_cast<size_t>(n) * rp;
  int* sC = reinterpret_cast<int*>(sF + rp);
  unsigned int* sM = reinterpret_cast<unsigned int*>(sC + static_cast<size_t>(n) * rp);

  for (int i = tid; i < static_cast<int>(a.N); i += nt) {
    const int li = i < B ? i : i - B + IB;
    const double v = a.U0[i];
    U[li] = v;
    U[NU + li] = v;
  }
  for (int k = tid; k < nr; k += nt) {
    const int r = r0 + k;
    const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
    for (int j = 0; j < n; ++j) {
      sW[j * rp + k] = a.W[base + 32LL * j];
      const int c = a.C[base + 32LL * j];
      sC[j * rp + k] = c < B ? c : c - B + IB;
    }
    sF[k] = a.F[r];
    sM[k] = a.dest[r];
  }
  for (int i = tid; i < 2 * 16 * 32 * 2; i += nt) red[i] = 0ull;
  __syncthreads();
  // this thread's row in registers (kReg: requires nr <= blockDim, host-checked)
  double wr[KR];
  int cr[KR];
  double fr = 0.0;
  unsigned int mr = 0;
  const bool own = tid < nr;
  if (kReg && own) {
#pragma unroll
    for (int j = 0; j < KR; ++j) {
      wr[j] = sW[j * rp + tid];
      cr[j] = sC[j * rp + tid];
    }
    fr = sF[tid];
    mr = sM[tid];
  }
  cluster.sync();

  DevStatus* st = a.st;
  const double dt = st->dt, tol = st->tol;
  const bool steady = (a.flags & kSteady) != 0;
  long long step = 0, bad_step = -1, conv_step = -1, last_res_step = -1;
  unsigned long long last_bits = 0;
  int cur = 0;
  long long t_a = 0, t_b = 0, t_c = 0, t_d = 0;
  const bool timed = a.phase_cycles != nullptr && q == 0 && tid == 0;
  for (; step < a.limit; ++step) {
    const long long t0 = timed ? clock64() : 0;
    const int nxt = cur ^ 1;
    const bool need_res = steady || step == a.limit - 1;
    const double* uc = U + cur * NU;
    double* un = U + nxt * NU;
    bool bad = false;
    unsigned long long dmax = 0ull;
    if constexpr (kReg) {
      if (own) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < KR; ++j) acc = __dadd_rn(acc, __dmul_rn(wr[j], uc[cr[j]]));
        const int li = IB + r0 + tid;
        const double u_self = uc[li];
        const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(fr, acc)));
        un[li] = value;
        unsigned int m = mr;
        while (m) {  // push to the CTAs that read this node
          const int dq = __ffs(m) - 1;
          m &= m - 1;
          *cluster.map_shared_rank(un + li, dq) = value;
        }
        bad = !isfinite(value);
        if (need_res)
          dmax = static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
      }
    } else {
      for (int k = tid; k < nr; k += nt) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(sW[j * rp + k], uc[sC[j * rp + k]]));
        const int li = IB + r0 + k;
        const double u_self = uc[li];
        const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(sF[k], acc)));
        un[li] = value;
        unsigned int m = sM[k];
        while (m) {
          const int dq = __ffs(m) - 1;
          m &= m - 1;
          *cluster.map_shared_rank(un + li, dq) = value;
        }
        bad |= !isfinite(value);
        if (need_res) {
          const unsigned long long b =
              static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
          dmax = b > dmax ? b : dmax;
        }
      }
    }
    const long long t1 = timed ? clock64() : 0;
    // warp partials -> slot (q, warp) of every CTA, one lane per destination.
    // The residual max is only reduced on steps that need it (every step in
    // steady mode, the last one in fixed mode, solver.py:208-211); the
    // non-finite flag every step (solver.py:200).
    const unsigned int wb = __reduce_or_sync(0xffffffffu, bad ? 1u : 0u);
    const unsigned long long wm = need_res ? warp_max_u64(dmax) : 0ull;
    if (lane < Q) {
      unsigned long long* slot = cluster.map_shared_rank(red + (nxt * 16 * 32 + q * nwarps + warp) * 2, lane);
      slot[0] = wm;
      slot[1] = wb;
    }
    const long long t2 = timed ? clock64() : 0;
    cluster.sync();  // publishes the step: field values and partials
    const long long t3 = timed ? clock64() : 0;
    unsigned long long gmax = 0ull;
    unsigned int lb = 0;
    for (int e = lane; e < slots; e += 32) lb |= static_cast<unsigned int>(red[(nxt * 16 * 32 + e) * 2 + 1]);
    const unsigned int gbad = __reduce_or_sync(0xffffffffu, lb);
    if (need_res) {
      for (int e = lane; e < slots; e += 32) {
        const unsigned long long v = red[(nxt * 16 * 32 + e) * 2];
        gmax = v > gmax ? v : gmax;
      }
      gmax = warp_max_u64(gmax);
    }
    cur = nxt;
    if (timed) {
      t_a += t1 - t0;
      t_b += t2 - t1;
      t_c += t3 - t2;
      t_d += clock64() - t3;
    }
    if (gbad) {
      bad_step = step;
      break;
    }
    if (need_res) {
      last_bits = gmax;
      last_res_step = step;
      if (steady && __ddiv_rn(__longlong_as_double(static_cast<long long>(gmax)), dt) <= tol) {
        conv_step = step;
        ++step;
        break;
      }
    }
  }
  if (timed) {
    a.phase_cycles[0] = t_a;
    a.phase_cycles[1] = t_b;
    a.phase_cycles[2] = t_c;
    a.phase_cycles[3] = t_d;
  }
  // the field after the last executed step (after a failure: its u2) is U[cur]
  const double* uf = U + cur * NU;
  for (int k = tid; k < nr; k += nt) {
    const long long node = a.dst_base + r0 + k;
    const double v = uf[IB + r0 + k];
    a.U0[node] = v;
    a.U1[node] = v;
  }
  if (q == 0) {
    for (int i = tid; i < B; i += nt) {
      a.U0[i] = uf[i];
      a.U1[i] = uf[i];
    }
    if (tid == 0) {
      st->bad_step = bad_step;
      st->conv_step = conv_step;
      st->last_res_bits = last_bits;
      st->last_res_step = last_res_step;
      st->step = (bad_step >= 0) ? bad_step + 1 : step;
    }
  }
  cluster.sync();  // no CTA leaves while a peer may still address its shared memory
}

// ---------------------------------------------------------------------------
// Grid-resident loop for mid-size problems (too big for one cluster's shared
// memory, small enough that every SM can hold its share of the rows): one
// cooperative launch runs every step.  Each CTA copies its contiguous range
// of SELL slices (weights, ids, forcing) into shared memory once; the field
// stays in global memory (L2-resident at these sizes, double-buffered); one
// grid barrier per step publishes the new values and the per-step
// non-finite / residual partials (three rotating slots, so a slot is reset
// two barriers after it was read).  Removes the per-step launch, ring fill
// and weight stream of the streaming path.  Arithmetic and j-order are those
// of row_update (bitwise parity).
struct GridArgs {
  const double* W;
  const int* C;
  const double* F;
  double* U0;  // start field in U0; the final field is published into both
  double* U1;
  long long n_rows, dst_base, limit;
  int spc;     // slices per CTA
  int spr;     // of which held in shared memory; the rest is re-read every step
               // from global memory, kept L2-resident (evict_last)
  int flags;   // kSteady
  DevStatus* st;
  unsigned long long* red;  // [2s, 2s+1] residual bits max of barrier slot s (3 slots),
                            // [6] the grid barrier's arrival counter (+2^40 / +2^52 per
                            // CTA with a non-finite value in the first / second step)
  // two steps per barrier (pair_kernels.cu tables, one tile per CTA), or HW == null:
  // halo rows' W / ids / forcing / node, tile-local ids of every row, per-tile halo slices
  const double* HW;
  const int* HC;
  const double* HF;
  const int* HR;
  const unsigned short* L16;
  const int* hoff;
  const int* hsl;
  int u1_cap;
};

template <int NJ, bool TWO>
__global__ void __launch_bounds__(512, 1) grid_loop_kernel(GridArgs a) {
  extern __shared__ __align__(16) unsigned char gl_smem[];
  const long long S = (a.n_rows + 31) >> 5;
  const long long s0 = static_cast<long long>(blockIdx.x) * a.spc;
  const long long s1 = s0 + a.spc < S ? s0 + a.spc : S;
  const int ns = s1 > s0 ? static_cast<int>(s1 - s0) : 0;
  double* sW = reinterpret_cast<double*>(gl_smem);
  double* sF = sW + static_cast<size_t>(a.spr) * NJ * 32;
  int* sC = reinterpret_cast<int*>(sF + static_cast<size_t>(a.spr) * 32);
  double* sU1 = reinterpret_cast<double*>(sC + static_cast<size_t>(a.spr) * NJ * 32);  // two-step mode
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int nres = ns < a.spr ? ns : a.spr;  // slices held in shared memory
  const uint64_t pol_keep = policy_evict_last();
  {
    const long long e0 = s0 * NJ * 32, ne = static_cast<long long>(nres) * NJ * 32;
    for (long long e = tid; e < ne; e += blockDim.x) {
      sW[e] = a.W[e0 + e];
      sC[e] = a.C[e0 + e];
    }
    for (long long e = tid; e < static_cast<long long>(nres) * 32; e += blockDim.x) sF[e] = a.F[s0 * 32 + e];
  }
  __shared__ unsigned long long s_max[16], s_max2[16];
  __shared__ unsigned int s_bad[16];
  __shared__ unsigned long long s_seen;
  DevStatus* st = a.st;
  const double dt = st->dt, tol = st->tol;
  const bool steady = (a.flags & kSteady) != 0;
  const bool two_ok = TWO && a.HW != nullptr && nres == ns;  // two-step mode needs every row on chip
  const long long row_lo = s0 * 32;
  const long long nt = a.n_rows - row_lo < static_cast<long long>(a.spc) * 32
                           ? (a.n_rows > row_lo ? a.n_rows - row_lo : 0) : static_cast<long long>(a.spc) * 32;
  long long step = 0, bad_step = -1, conv_step = -1, last_res_step = -1;
  unsigned long long last_bits = 0;
  long long it = 0;  // barriers passed
  int cur = 0;
  constexpr unsigned long long kBad1 = 1ull << 40, kBad2 = 1ull << 52, kCount = kBad1 - 1;
  __syncthreads();
  while (step < a.limit) {
    const bool two = two_ok && step + 2 <= a.limit;
    const bool need1 = steady || (!two && step == a.limit - 1);
    const bool need2 = two && (steady || step + 2 == a.limit);
    const double* uc = cur ? a.U1 : a.U0;
    double* un = cur ? a.U0 : a.U1;
    bool bad1 = false, bad2 = false;
    unsigned long long dmax1 = 0ull, dmax2 = 0ull;
    // ---- step t -> t+1 for this CTA's rows (into shared memory in two-step mode)
    for (int k = warp; k < ns; k += nwarps) {
      const long long r = (s0 + k) * 32 + lane;
      if (r >= a.n_rows) continue;
      const long long node = a.dst_base + r;
      double acc = 0.0, u_self, fk;
      if (k < nres) {  // rows held in shared memory
        const double* w = sW + static_cast<size_t>(k) * NJ * 32 + lane;
        const int* c = sC + static_cast<size_t>(k) * NJ * 32 + lane;
        double g[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) g[j] = uc[c[32 * j]];
        u_self = (c[0] == node) ? g[0] : uc[node];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(w[32 * j], g[j]));
        fk = sF[k * 32 + lane];
      } else {  // rows re-read from L2 every step
        const long long e = (s0 + k) * NJ * 32 + lane;
        int c[NJ];
        double w[NJ], g[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          c[j] = ld_stream_s32(a.C + e + 32 * j, pol_keep);
          w[j] = ld_stream_f64(a.W + e + 32 * j, pol_keep);
        }
        fk = ld_stream_f64(a.F + r, pol_keep);
#pragma unroll
        for (int j = 0; j < NJ; ++j) g[j] = uc[c[j]];
        u_self = (c[0] == node) ? g[0] : uc[node];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(w[j], g[j]));
      }
      const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(fk, acc)));
      if (two) sU1[r - row_lo] = value;
      else un[node] = value;
      bad1 |= !isfinite(value);
      if (need1) {
        const unsigned long long b =
            static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
        dmax1 = b > dmax1 ? b : dmax1;
      }
    }
    if constexpr (TWO) if (two) {
      // halo rows of this CTA at step t+1 (recomputed exactly as their owners
      // do) and the Dirichlet nodes its rows read, after its own rows in sU1
      const long long h0 = a.hoff[blockIdx.x];
      const int hn = a.hsl[blockIdx.x];
      for (int h = warp; h < hn; h += nwarps) {
        const long long e = (h0 + h) * 32 + lane;
        const int hr = a.HR[e];
        const long long loc = nt + h * 32 + lane;
        if (hr >= 0) {
          const long long eb = (h0 + h) * NJ * 32 + lane;
          int c[NJ];
          double w[NJ], g[NJ];
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            c[j] = a.HC[eb + 32 * j];
            w[j] = a.HW[eb + 32 * j];
          }
#pragma unroll
          for (int j = 0; j < NJ; ++j) g[j] = uc[c[j]];
          const double u_self = (c[0] == hr) ? g[0] : uc[hr];
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(w[j], g[j]));
          sU1[loc] = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(a.HF[e], acc)));
        } else if (hr != INT_MIN) {
          sU1[loc] = uc[-(hr + 1)];
        }
      }
      __syncthreads();
      // ---- step t+1 -> t+2 for this CTA's rows, from shared memory
      for (int k = warp; k < ns; k += nwarps) {
        const long long r = (s0 + k) * 32 + lane;
        if (r >= a.n_rows) continue;
        const double* w = sW + static_cast<size_t>(k) * NJ * 32 + lane;
        const unsigned short* l = a.L16 + (s0 + k) * NJ * 32 + lane;
        double g[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) g[j] = sU1[l[32 * j]];
        const double u_self = sU1[r - row_lo];
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(w[32 * j], g[j]));
        const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(sF[k * 32 + lane], acc)));
        un[a.dst_base + r] = value;
        bad2 |= !isfinite(value);
        if (need2) {
          const unsigned long long b =
              static_cast<unsigned long long>(__double_as_longlong(fabs(__dsub_rn(value, u_self))));
          dmax2 = b > dmax2 ? b : dmax2;
        }
      }
    }
    // ---- CTA partials, then the grid barrier: the non-finite flags ride on
    // the arrival (high bits; the loop stops at the first, so any high bit
    // means this barrier), residual maxima go to this barrier's slot, the slot
    // two barriers ahead is reset by CTA 0
    const unsigned int wb = __reduce_or_sync(0xffffffffu, (bad1 ? 1u : 0u) | (bad2 ? 2u : 0u));
    const unsigned long long wm1 = need1 ? warp_max_u64(dmax1) : 0ull;
    const unsigned long long wm2 = need2 ? warp_max_u64(dmax2) : 0ull;
    if (lane == 0) {
      s_bad[warp] = wb;
      s_max[warp] = wm1;
      s_max2[warp] = wm2;
    }
    __syncthreads();
    const int slot = static_cast<int>(it % 3);
    if (tid == 0) {
      unsigned int cb = 0;
      unsigned long long cm1 = 0ull, cm2 = 0ull;
      for (int w = 0; w < nwarps; ++w) {
        cb |= s_bad[w];
        cm1 = s_max[w] > cm1 ? s_max[w] : cm1;
        cm2 = s_max2[w] > cm2 ? s_max2[w] : cm2;
      }
      if (need1 && cm1) atomicMax(&a.red[slot * 2], cm1);
      if (need2 && cm2) atomicMax(&a.red[slot * 2 + 1], cm2);
      if (blockIdx.x == 0) {
        const int nx = static_cast<int>((it + 1) % 3);
        a.red[nx * 2] = 0ull;
        a.red[nx * 2 + 1] = 0ull;
      }
      // grid barrier on a monotonic arrival counter: the fence publishes the
      // CTA's field stores (ordered after the CTA barrier above), the acquire
      // spin orders every CTA's reads of the new field after all arrivals
      __threadfence();
      atomicAdd(&a.red[6], 1ull + ((cb & 1u) ? kBad1 : 0ull) + ((cb & 2u) ? kBad2 : 0ull));
      const unsigned long long target = static_cast<unsigned long long>(it + 1) * gridDim.x;
      unsigned long long v, t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (int spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&a.red[6]) : "memory");
        if ((v & kCount) >= target) break;
        if ((spin & 1023) == 1023) {  // all CTAs are co-resident: a 20 s wait is a fault
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (t - t0 > 20000000000ull) __trap();
        }
      }
      // The flag bits belong to this barrier only when no CTA has arrived at
      // the next one yet (count == target).  A count past target means some
      // CTA already left this barrier, which it only does when this barrier
      // was clean (a flagged barrier stops every CTA): its own next-barrier
      // bits must not be read as this barrier's.
      s_seen = ((v & kCount) == target) ? v : 0ull;
    }
    __syncthreads();
    ++it;
    const bool gbad1 = ((s_seen >> 40) & 0xfffull) != 0;
    const bool gbad2 = (s_seen >> 52) != 0;
    // the reference checks every step's flag before its residual (solver.py:200-217)
    bool stop_at_first = false;  // two-step mode: stop with u^{t+1} (held in sU1)
    if (gbad1) {
      bad_step = step;
      stop_at_first = two;
    } else if (need1) {
      const unsigned long long gmax = *reinterpret_cast<volatile unsigned long long*>(&a.red[slot * 2]);
      last_bits = gmax;
      last_res_step = step;
      if (steady && __ddiv_rn(__longlong_as_double(static_cast<long long>(gmax)), dt) <= tol) {
        conv_step = step;
        stop_at_first = two;
      }
    }
    if (TWO && stop_at_first) {  // publish u^{t+1} of this CTA's rows in place of u^{t+2}
      for (int k = warp; k < ns; k += nwarps) {
        const long long r = (s0 + k) * 32 + lane;
        if (r < a.n_rows) un[a.dst_base + r] = sU1[r - row_lo];
      }
    }
    if (bad_step >= 0 || conv_step >= 0 || !two) {
      cur ^= 1;
      step += 1;
      if (bad_step >= 0 || conv_step >= 0) break;
      continue;
    }
    // second step of the pair
    cur ^= 1;
    if (gbad2) {
      bad_step = step + 1;
      step += 2;
      break;
    }
    if (need2) {
      const unsigned long long gmax = *reinterpret_cast<volatile unsigned long long*>(&a.red[slot * 2 + 1]);
      last_bits = gmax;
      last_res_step = step + 1;
      if (steady && __ddiv_rn(__longlong_as_double(static_cast<long long>(gmax)), dt) <= tol) {
        conv_step = step + 1;
        step += 2;
        break;
      }
    }
    step += 2;
  }
  // the field after the last executed step (after a failure: its u2) is in
  // buffer `cur`; publish it into both buffers
  __syncthreads();
  const double* uf = cur ? a.U1 : a.U0;
  double* uo = cur ? a.U0 : a.U1;
  for (int k = warp; k < ns; k += nwarps) {
    const long long r = (s0 + k) * 32 + lane;
    if (r < a.n_rows) uo[a.dst_base + r] = uf[a.dst_base + r];
  }
  if (blockIdx.x == 0 && tid == 0) {
    st->bad_step = bad_step;
    st->conv_step = conv_step;
    st->last_res_bits = last_bits;
    st->last_res_step = last_res_step;
    st->step = (bad_step >= 0) ? bad_step + 1 : step;
  }
}

// dest[row(c)] |= 1 << owner(r) for every stencil entry c of row r that is an
// interior node owned by another CTA of the cluster (owner(r) = r / rpc)
__global__ void cluster_dest_kernel(const int* __restrict__ C, long long n_rows, int n, long long B,
                                    int rpc, unsigned int* __restrict__ dest) {
  const long long total = n_rows * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / n;
    const int j = static_cast<int>(e - r * n);
    const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
    const long long c = C[base + 32LL * j];
    if (c < B) continue;
    const long long rc = c - B;
    const int qr = static_cast<int>(r / rpc), qc = static_cast<int>(rc / rpc);
    if (qr != qc) atomicOr(dest + rc, 1u << qr);
  }
}

// ---- plan construction kernels --------------------------------------------
// Scatter row-major (reference layout) rows [k0, k0+cnt) into SELL-32 at the
// renumbered row position; node ids renumbered through new_id.
__global__ void pack_rows_kernel(const double* __restrict__ w_raw, const int* __restrict__ c_raw,
                                 const double* __restrict__ f_raw, long long k0, long long cnt, int n,
                                 const long long* __restrict__ row_of_k,  // nullptr: identity
                                 const int* __restrict__ new_id, long long N,
                                 double* __restrict__ W, int* __restrict__ C, double* __restrict__ F,
                                 int* __restrict__ err) {
  const long long total = cnt * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long kk = e / n;
    const int j = static_cast<int>(e - kk * n);
    const long long k = k0 + kk;
    const long long r = row_of_k ? row_of_k[k] : k;
    const long long dst = (r >> 5) * static_cast<long long>(n) * 32 + 32LL * j + (r & 31);
    const long long col = c_raw[e];  // range-checked on the host while staging
    if (col < 0 || col >= N) {
      atomicExch(err, 1);
      continue;
    }
    W[dst] = w_raw[e];
    C[dst] = new_id ? new_id[col] : static_cast<int>(col);
    if (j == 0) F[r] = f_raw[kk];
  }
}

// u_dev[new_id[i]] = u_host_order[i]   (new_id == nullptr: identity)
__global__ void scatter_field_kernel(const double* __restrict__ src, const int* __restrict__ new_id,
                                     long long N, double* __restrict__ d0, double* __restrict__ d1) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = new_id[i];
    d0[t] = src[i];
    if (d1) d1[t] = src[i];
  }
}
// ---- partitioned (multi-GPU) loop helpers -----------------------------------
// sendbuf[k] = u[idx[k]]: the owned values the peers read (their halo)
__global__ void pack_halo_kernel(const double* __restrict__ u, const int* __restrict__ idx,
                                 long long count, double* __restrict__ sendbuf) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    sendbuf[k] = u[idx[k]];
}

// In-process all-reduce(max) of red[] over the parts of a local group.
__global__ void reduce_parts_kernel(DevStatus* const* st, int n_parts) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long m0 = 0, m1 = 0;
  for (int p = 0; p < n_parts; ++p) {
    m0 = st[p]->red[0] > m0 ? st[p]->red[0] : m0;
    m1 = st[p]->red[1] > m1 ? st[p]->red[1] : m1;
  }
  for (int p = 0; p < n_parts; ++p) {
    st[p]->red[0] = m0;
    st[p]->red[1] = m1;
  }
}

// After the all-reduce: the same decision on every part (solver.py:200-217).
__global__ void decide_kernel(DevStatus* st, long long step, int flags) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long bs = st->bad_step, cs = st->conv_step;
  if ((bs >= 0 && bs < step) || (cs >= 0 && cs < step)) return;  // already stopped
  if (st->red[1]) {
    st->bad_step = step;
  } else if (flags & kNeedResidual) {
    const unsigned long long m = st->red[0];
    st->last_res_bits = m;
    st->last_res_step = step;
    if ((flags & kSteady) &&
        __ddiv_rn(__longlong_as_double(static_cast<long long>(m)), st->dt) <= st->tol)
      st->conv_step = step;
  }
  st->red[0] = 0;
  st->red[1] = 0;
}

// max_r sum_j |w_rj| over the SELL rows (stability_bound, solver.py:249-254;
// each row summed in numpy's order (below), then an exact max over
// non-negative bit patterns): 2 / this has the reference's auto-dt bits.
// sum_j |w[j*32]| for j in [j0, j0+len) in numpy's pairwise order
// (np.abs(weights).sum(axis=1) reduces each row on its own: pairwise_sum of
// loops_utils.h.src, 8 accumulators up to 128 entries, halving above)
__device__ double pairwise_abs_row(const double* __restrict__ w, int j0, int len) {
  if (len < 8) {
    double res = 0.0;
    for (int i = 0; i < len; ++i) res = __dadd_rn(res, fabs(w[32LL * (j0 + i)]));
    return res;
  }
  if (len <= 128) {
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = fabs(w[32LL * (j0 + q)]);
    int i = 8;
    for (; i < len - (len % 8); i += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], fabs(w[32LL * (j0 + i + q)]));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < len; ++i) res = __dadd_rn(res, fabs(w[32LL * (j0 + i)]));
    return res;
  }
  int n2 = len / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_abs_row(w, j0, n2), pairwise_abs_row(w, j0 + n2, len - n2));
}

__global__ void row_abs_sum_max_kernel(const double* __restrict__ W, long long n_rows, int n,
                                       double* out) {
  unsigned long long m = 0ull;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
    const double s = pairwise_abs_row(W + base, 0, n);
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(s));
    m = b > m ? b : m;
  }
  m = warp_max_u64(m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(reinterpret_cast<unsigned long long*>(out), m);
}

// ---- renumbering (plan build) -----------------------------------------------
// 2-D bit interleave of a 21-bit coordinate: bit i -> bit 2i
__device__ __forceinline__ unsigned long long spread_bits21(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
// Bounding box of the node positions for the Morton quantisation, on the
// device (min / max are exact: the same values as a host pass).
// partial[4 * block] = {xmin, xmax, ymin, ymax}; finish with one block.
__global__ void __launch_bounds__(256) bounds_partial_kernel(const double* __restrict__ pos, long long n,
                                                             double* __restrict__ partial) {
  double a0 = 1e300, a1 = -1e300, b0 = 1e300, b1 = -1e300;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = pos[2 * i], y = pos[2 * i + 1];
    a0 = fmin(a0, x);
    a1 = fmax(a1, x);
    b0 = fmin(b0, y);
    b1 = fmax(b1, y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 = fmin(a0, __shfl_xor_sync(0xffffffffu, a0, o));
    a1 = fmax(a1, __shfl_xor_sync(0xffffffffu, a1, o));
    b0 = fmin(b0, __shfl_xor_sync(0xffffffffu, b0, o));
    b1 = fmax(b1, __shfl_xor_sync(0xffffffffu, b1, o));
  }
  __shared__ double s[8][4];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s[w][0] = a0;
    s[w][1] = a1;
    s[w][2] = b0;
    s[w][3] = b1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
      a0 = fmin(a0, s[k][0]);
      a1 = fmax(a1, s[k][1]);
      b0 = fmin(b0, s[k][2]);
      b1 = fmax(b1, s[k][3]);
    }
    partial[4 * blockIdx.x + 0] = a0;
    partial[4 * blockIdx.x + 1] = a1;
    partial[4 * blockIdx.x + 2] = b0;
    partial[4 * blockIdx.x + 3] = b1;
  }
}
// key[k] = Morton code of interior node k's position (21 bits per axis over
// the bounding box from bounds_partial_kernel's `nb` partials; the IEEE
// expression of multigpu.morton_codes), val[k] = k; a stable radix sort of
// (key, val) orders the rows by (code, k).
__global__ void morton_keys_dev_kernel(const double* __restrict__ pos, const long long* __restrict__ interior,
                                       long long n_rows, const double* __restrict__ partial, int nb,
                                       unsigned long long* __restrict__ key, long long* __restrict__ val) {
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (int k = 0; k < nb; ++k) {
    xmin = fmin(xmin, partial[4 * k + 0]);
    xmax = fmax(xmax, partial[4 * k + 1]);
    ymin = fmin(ymin, partial[4 * k + 2]);
    ymax = fmax(ymax, partial[4 * k + 3]);
  }
  const double sx = (xmax > xmin) ? __ddiv_rn(2097151.0, __dsub_rn(xmax, xmin)) : 0.0;
  const double sy = (ymax > ymin) ? __ddiv_rn(2097151.0, __dsub_rn(ymax, ymin)) : 0.0;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n_rows;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long v = interior[k];
    const unsigned long long qx = static_cast<unsigned int>(__dmul_rn(__dsub_rn(pos[2 * v], xmin), sx));
    const unsigned long long qy = static_cast<unsigned int>(__dmul_rn(__dsub_rn(pos[2 * v + 1], ymin), sy));
    key[k] = spread_bits21(qx) | (spread_bits21(qy) << 1);
    val[k] = k;
  }
}
__global__ void iota_kernel(long long* __restrict__ out, long long n) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    out[k] = k;
}
__global__ void invert_order_kernel(const long long* __restrict__ order, long long n, long long* __restrict__ row_of_k) {
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<long long>(gridDim.x) * blockDim.x)
    row_of_k[order[r]] = r;
}
__global__ void not_seen_kernel(const unsigned char* __restrict__ seen, long long n, int* __restrict__ flag) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    flag[i] = seen[i] ? 0 : 1;
}
__global__ void interior_ids_kernel(const long long* __restrict__ interior, const long long* __restrict__ row_of_k,
                                    long long n_rows, long long B, int* __restrict__ new_id) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n_rows;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    new_id[interior[k]] = static_cast<int>(B + row_of_k[k]);
}

// F[row_of_k[k]] = f[k]
__global__ void scatter_rows_kernel(const double* __restrict__ f, const long long* __restrict__ row_of_k,
                                    long long n_rows, double* __restrict__ F) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n_rows;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    F[row_of_k[k]] = f[k];
}
// First row whose stencil reads a node in [lo, hi) (a part's halo slice):
// atomicMin over the SELL entries.
__global__ void first_row_reading_kernel(const int* __restrict__ C, long long n_rows, int n, long long lo,
                                         long long hi, unsigned long long* first) {
  const long long total = ((n_rows + 31) >> 5) * 32LL * n;
  unsigned long long m = ~0ull;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = (e / (32LL * n)) * 32 + (e & 31);
    const int c = C[e];
    if (r < n_rows && c >= lo && c < hi && static_cast<unsigned long long>(r) < m) m = r;
  }
  if (m != ~0ull) atomicMin(first, m);
}

// Plan-file payload check (rbf_plan_load): every streamed node id in [0, N),
// every 16-bit id of a fitting slice decodes to its int32 id, the renumbering
// maps stay in range.  err bits: 1 C, 2 C16/meta, 4 new_id, 8 row_of_k.
__global__ void validate_plan_kernel(const int* __restrict__ C, const unsigned short* __restrict__ C16,
                                     const int4* __restrict__ meta, long long n_rows, int n, long long N,
                                     const int* __restrict__ new_id, const long long* __restrict__ row_of_k,
                                     unsigned int* err) {
  const long long S = (n_rows + 31) >> 5;
  const long long total = S * 32 * n;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  unsigned int e = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const long long sl = i / (32LL * n);
    const int lane = static_cast<int>(i & 31);
    if (sl * 32 + lane >= n_rows) continue;  // padding lanes are never read
    const int c = C[i];
    if (c < 0 || c >= N) e |= 1u;
    if (C16) {
      const int4 m = meta[sl];
      if (m.z && decode_id(C16[i], m) != c) e |= 2u;
    }
  }
  if (new_id)
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N; i += stride)
      if (new_id[i] < 0 || new_id[i] >= N) e |= 4u;
  if (row_of_k)
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_rows; i += stride)
      if (row_of_k[i] < 0 || row_of_k[i] >= n_rows) e |= 8u;
  if (e) atomicOr(err, e);
}

// error_norms (solver.py:239-246), numpy's bits.  norm_diff_kernel: in
// original node order d_i = u[new_id[i]] - exact[i]; sq[i] = d_i * d_i (in
// place of exact) and max|d| as non-negative bit patterns (NaN patterns order
// above every finite one, so a NaN wins like in np.max).
__global__ void norm_diff_kernel(const double* __restrict__ u, const int* __restrict__ new_id, double* ex_sq,
                                 long long N, unsigned long long* max_bits) {
  unsigned long long m = 0ull;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < N;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double d = __dsub_rn(u[new_id ? new_id[g] : g], ex_sq[g]);
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(fabs(d)));
    m = bits > m ? bits : m;
    ex_sq[g] = __dmul_rn(d, d);
  }
  m = warp_max_u64(m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(max_bits, m);
}

// Block sums of numpy's pairwise summation (loops_utils.h.src pairwise_sum)
// over [start[b], start[b+1]) (<= 128 elements): below 8 elements a serial
// sum from 0.0, else 8 accumulators, their fixed combination, then the tail.
__global__ void norm_blocks_kernel(const double* __restrict__ sq, const long long* __restrict__ start,
                                   long long n_blocks, double* __restrict__ block_sum) {
  for (long long b = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; b < n_blocks;
       b += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double* a = sq + start[b];
    const long long n = start[b + 1] - start[b];
    double res;
    if (n < 8) {
      res = 0.0;
      for (long long i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    } else {
      double r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = a[j];
      long long i = 8;
      for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
      }
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    }
    block_sum[b] = res;
  }
}

__global__ void gather_field_kernel(const double* __restrict__ src, const int* __restrict__ new_id,
                                    long long N, double* __restrict__ dst) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = src[new_id[i]];
}

// ---------------------------------------------------------------------------
// Push-mode halo exchange (group.inc.cuh): after a part's step, store the
// owned values its neighbours read straight into their field buffers (P2P
// stores over NVLink; plain device stores between the parts of one process),
// then publish the arrival with one system-scope release store per neighbour.
// Replaces pack + NCCL send/recv + their per-step launch latency.
struct PushPeer {
  double* u[2];        // the peer's field buffers (IPC-mapped or local)
  long long dst_off;   // first slot of this part's halo group in the peer's numbering
  long long src_off;   // first entry of the peer's segment in send_idx
  long long count;
};

struct PushArgs {
  const double* u[2];            // this part's field buffers
  const int* send_idx;           // [total] owned local ids, segmented per peer
  long long total;
  int n_peer;                    // peers this part sends to
  int n_nbr;                     // neighbours to notify (senders and receivers)
  int my_id;
  PushPeer peer[kMaxPushPeers];
  unsigned long long* nbr_flags[kMaxPushPeers];  // neighbours' arrival arrays
  DevStatus* st;
  unsigned int* ticket;
  int sys_scope;                 // 1: peers on other GPUs (fences at system scope)
};

__global__ void __launch_bounds__(256) push_halo_kernel(PushArgs a, int out) {
  pdl_wait();  // the step that produced u[out] is complete and visible
  pdl_launch_dependents();
  const double* u = a.u[out];
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < a.total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    int i = 0;
    while (i + 1 < a.n_peer && k >= a.peer[i + 1].src_off) ++i;
    a.peer[i].u[out][a.peer[i].dst_off + (k - a.peer[i].src_off)] = u[a.send_idx[k]];
  }
  // the CTA's stores -> (barrier) -> one fence by thread 0 -> ticket; the last
  // CTA's release store then publishes every CTA's stores (causality is
  // transitive through the barrier, the fences and the ticket's RMW chain)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (a.sys_scope) __threadfence_system();
    else __threadfence();
    const unsigned int t = atomicAdd(a.ticket, 1u);
    if (t == gridDim.x - 1) {
      *a.ticket = 0u;
      const long long v = a.st->push_base + (++a.st->push_count);
      if (a.sys_scope) __threadfence_system();
      else __threadfence();
      for (int j = 0; j < a.n_nbr; ++j) {
        if (a.sys_scope) {
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.nbr_flags[j] + a.my_id),
                       "l"(static_cast<unsigned long long>(v))
                       : "memory");
        } else {
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.nbr_flags[j] + a.my_id),
                       "l"(static_cast<unsigned long long>(v))
                       : "memory");
        }
      }
    }
  }
}

}  // namespace rbf
