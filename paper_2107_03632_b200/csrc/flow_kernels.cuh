// flow_kernels.cuh -- persistent "dataflow" time loop for fixed-step runs.
//
// The graph/PDL path ends every step with a grid-wide dependency (the next
// launch waits for the whole previous grid), so each step pays a fill/drain
// bubble (~2.6 us of a 32 us step at N=1e6, profiles/README.md).  Here one
// cooperative launch runs all K steps.  CTA b owns a contiguous range of SELL
// slices (contiguous in the Morton order, so spatially compact); before it
// starts step s+1 it waits only for the CTAs it shares stencil entries with
// (both directions: the ones whose rows it reads, and the ones that read its
// rows -- the latter protects the double-buffered field against overwrite)
// to have published step s.  The producer warp keeps streaming the (step
// independent) weights / ids into the TMA ring across step boundaries, so
// HBM never idles at a step edge.
//
// Arithmetic and j-order are exactly those of step_tma_kernel (bitwise
// parity).  Fixed mode only: the non-finite check records the first bad step
// (global atomicMin) and the host re-runs the prefix on the exact graph path
// to reproduce the reference's failure state (solver.py:200-206); the
// residual is reduced on the last step only (solver.py:210-211).
#pragma once

namespace rbf {

struct FlowArgs {
  StepArgs a;
  double* U0;
  double* U1;
  int* flags;            // [grid] steps published per CTA (zeroed before the launch)
  const int* dep_off;    // [grid+1] offsets into dep
  const int* dep;        // neighbour CTA ids
  long long steps;       // K
  int spc;               // slices per CTA
  int need_res_last;     // reduce the residual on the last step
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int NJ, int CW, int IB>
__global__ void __launch_bounds__(32 * (CW + 1), 1) step_flow_kernel(FlowArgs fa, TmaGeom g) {
  extern __shared__ __align__(128) unsigned char flow_smem[];
  constexpr int kMaxStages = 16;
  const StepArgs& a = fa.a;
  uint64_t* full = reinterpret_cast<uint64_t*>(flow_smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* ring = flow_smem + 2 * kMaxStages * sizeof(uint64_t);
  __shared__ int s_issued;
  __shared__ int s_dep[160];
  __shared__ int s_ndep;
  __shared__ unsigned long long s_max[32];
  const int sps = g.sps, stages = g.stages;
  const int wbytes = sps * NJ * 32 * 8, cbytes = sps * NJ * 32 * IB;
  const int stage_bytes = sps * tma_slice_bytes<NJ, IB>();
  const long long S = (a.n_rows + 31) >> 5;
  const int b = blockIdx.x;
  const long long sl_lo = static_cast<long long>(b) * fa.spc;
  const long long sl_hi = sl_lo + fa.spc < S ? sl_lo + fa.spc : S;
  const long long my_slices = sl_hi > sl_lo ? sl_hi - sl_lo : 0;
  const long long chunks_per_step = (my_slices + sps - 1) / sps;
  const long long total_chunks = chunks_per_step * fa.steps;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = 32 * CW;

  if (threadIdx.x == 0) {
    s_issued = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], static_cast<uint32_t>(sps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int d0 = fa.dep_off[b], d1 = fa.dep_off[b + 1];
    s_ndep = d1 - d0 < 160 ? d1 - d0 : 160;
    for (int k = 0; k < s_ndep; ++k) s_dep[k] = fa.dep[d0 + k];
  }
  __syncthreads();
  DevStatus* st = a.st;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (long long i = 0; i < total_chunks; ++i) {
        const int s = static_cast<int>(i % stages);
        if (i >= stages) mbar_wait(&empty[s], static_cast<uint32_t>(((i / stages) - 1) & 1));
        const long long lc = i % chunks_per_step;
        const long long s0 = sl_lo + lc * sps;
        const int ns = static_cast<int>(sl_hi - s0 < sps ? sl_hi - s0 : sps);
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
        *reinterpret_cast<volatile int*>(&s_issued) = static_cast<int>(i + 1);
      }
    }
    return;  // the producer warp takes no part in the consumer barriers
  }

  // ---- consumers --------------------------------------------------------
  const double dt = st->dt;
  const int cw = warp - 1;
  bool bad_any = false;
  long long first_bad = -1;
  unsigned long long dmax = 0ull;
  for (long long step = 0; step < fa.steps; ++step) {
    const double* u_in = (step & 1) ? fa.U1 : fa.U0;
    double* u_out = (step & 1) ? fa.U0 : fa.U1;
    const bool last = step == fa.steps - 1;
    bool bad = false;
    // units = slices of this CTA for this step, round robin over consumer warps
    for (long long q = cw; q < my_slices; q += CW) {
      const long long i = step * chunks_per_step + q / sps;
      const int slot = static_cast<int>(q % sps);
      const int s = static_cast<int>(i % stages);
      if (lane == 0) {
        while (*reinterpret_cast<volatile int*>(&s_issued) <= i) __nanosleep(64);
      }
      __syncwarp();
      mbar_wait(&full[s], static_cast<uint32_t>((i / stages) & 1));
      const unsigned char* base = ring + static_cast<size_t>(s) * stage_bytes;
      const long long slice = sl_lo + q;
      const long long r = slice * 32 + lane;
      if (r < a.n_rows) {
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
        if (last && fa.need_res_last) {
          const unsigned long long bits = static_cast<unsigned long long>(
              __double_as_longlong(fabs(__dsub_rn(value, u_self))));
          dmax = bits > dmax ? bits : dmax;
        }
      }
      __syncwarp();
      if (lane == 0) {
        // a CTA's last chunk of a step may hold fewer than sps slices: its
        // last real slot also arrives for the missing ones
        const long long lc = q / sps;
        const int ns = static_cast<int>(my_slices - lc * sps < sps ? my_slices - lc * sps : sps);
        if (slot == ns - 1 && ns < sps) mbar_arrive_count(&empty[s], static_cast<uint32_t>(sps - ns + 1));
        else mbar_arrive(&empty[s]);
      }
    }
    if (bad && first_bad < 0) first_bad = step;
    bad_any |= bad;
    if (last) break;
    // ---- step edge: publish step, wait for the neighbour CTAs ------------
    consumer_bar(ncons);  // every consumer of this CTA finished the step
    if (warp == 1) {
      if (lane == 0) {
        // bar.sync ordered every consumer's stores before this release (cumulative)
        st_release_gpu(fa.flags + b, static_cast<int>(step + 1));
      }
      // poll the neighbours in parallel (relaxed), then one acquire fence
      for (int k = lane; k < s_ndep; k += 32) {
        const volatile int* f = fa.flags + s_dep[k];
        while (*f < step + 1) __nanosleep(20);
      }
      __syncwarp();
      if (lane == 0) __threadfence();  // gpu-scope fence: acquire, and invalidates this SM's L1
      __syncwarp();
    }
    consumer_bar(ncons);
  }
  // ---- end: first bad step (min over all threads) and the last residual ----
  if (first_bad >= 0) atomicMin(reinterpret_cast<long long*>(&st->bad_step), first_bad);
  const unsigned long long wm = warp_max_u64(dmax);
  if (lane == 0) s_max[cw] = wm;
  consumer_bar(ncons);
  if (threadIdx.x == 32) {
    unsigned long long m = 0;
    for (int w = 0; w < CW; ++w) m = s_max[w] > m ? s_max[w] : m;
    if (m) atomicMax(&st->res_bits, m);
  }
  (void)bad_any;
}

// After a flow launch: translate the accumulated values into the status
// fields the host reads for the graph path (solver.py:207-211).
__global__ void flow_finalize_kernel(DevStatus* st, long long steps, int need_res) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st->bad_step == 0x7fffffffffffffffLL) st->bad_step = -1;
  if (st->bad_step < 0) {
    st->step = steps;
    if (need_res) {
      st->last_res_bits = st->res_bits;
      st->last_res_step = steps - 1;
    }
  }
  st->res_bits = 0;
}

// dep[b] |= cb for every stencil entry of CTA b's rows owned by CTA cb
// (symmetric), as a grid x grid bit matrix of 32-bit words.
__global__ void flow_dep_kernel(const int* __restrict__ C, long long n_rows, int n, long long B,
                                long long rows_per_cta, int words, unsigned int* __restrict__ mat) {
  const long long total = n_rows * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / n;
    const int j = static_cast<int>(e - r * n);
    const long long base = (r >> 5) * static_cast<long long>(n) * 32 + (r & 31);
    const long long c = C[base + 32LL * j];
    if (c < B) continue;
    const int br = static_cast<int>(r / rows_per_cta), bc = static_cast<int>((c - B) / rows_per_cta);
    if (br == bc) continue;
    atomicOr(mat + static_cast<long long>(br) * words + (bc >> 5), 1u << (bc & 31));
    atomicOr(mat + static_cast<long long>(bc) * words + (br >> 5), 1u << (br & 31));
  }
}

}  // namespace rbf
