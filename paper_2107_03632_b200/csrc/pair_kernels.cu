// pair_kernels.cu -- two time steps per launch by tile-local temporal blocking.
//
// Why: the single-step kernel streams every row's weights, ids and forcing
// from HBM once per step (~10n+24 bytes with 16-bit ids), which bounds it at
// the HBM roofline.  Two consecutive steps use the same weights, so a launch
// that advances the field by two steps can read them from HBM once:
//
//   phase 1 (step t -> t+1): for the rows of tile b AND the tile's halo (the
//     rows of other tiles its stencils reference) compute u^{t+1} from u^t in
//     global memory, exactly as the owning tile would, into a shared-memory
//     buffer U1 in tile-local numbering [tile rows | halo entries]; Dirichlet
//     nodes referenced by the tile are halo entries that copy u^t;
//   phase 2 (step t+1 -> t+2): for the tile's rows, gather u^{t+1} from U1
//     through 16-bit tile-local ids and write u^{t+2} to global memory.
//
// The halo rows are recomputed redundantly (same weights, same ids, same
// serial j-order, same u^t inputs), so every value is bitwise the single-step
// kernel's; u^{t+1} never reaches global memory.  HBM traffic per row per two
// steps: the main stream once (10n+24, weights and forcing kept L2-resident
// with evict_last for their phase-2 re-read), the halo rows' stream (int32
// ids), the 2n bytes of local ids and one field write.
//
// Pipeline: the TMA ring of step_tma_kernel (one producer lane, CW consumer
// warps, cp.async.bulk + mbarrier transaction counts) streams phase-1 data
// only, per tile [main rows | halo rows]; the producer also prefetches each
// tile's local ids into L2.  Consumers walk segments: segment k interleaves
// phase 1 of tile k (ring) with phase 2 of tile k-1 (direct loads of the
// L2-resident weights/forcing and the prefetched local ids), so HBM streams
// the next tile while the previous one finishes; the consumer warps meet at
// one named barrier per segment, and U1 is double-buffered (tile k writes
// buffer k&1 while tile k-1 is read from the other).
//
// Measured (profiles/README.md): HBM traffic per pair is as designed (268 MB
// read at C2 against 2 x 172 MB for two single steps), but the consumers are
// latency-bound (15 warps, ~2 us per 32-row unit), so the pair only wins
// where the per-launch grid dependency dominates -- 1.1-1.5x up to ~1e6
// stencil entries.  The driver builds it there, but at those sizes the
// grid-resident loop (step_kernels.cuh) is faster still and runs instead; the
// pair kernel runs when the on-chip loops are off (RBF_NO_RESIDENT), and its
// halo / local-id tables drive the grid loop's two-step mode.
//
// Failure semantics: the epilogue flags a non-finite value anywhere in the
// pair and the driver replays the run on the single-step path, which stops at
// the exact step with the reference's payload (rbffd_b200.cu run_pair).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rbffd_b200.h"
#include "pair.h"

namespace rbf_detail {
int fail_c(int code, const char* msg);
}

namespace rbf {

namespace {

struct TileInfo {
  long long s_lo, s_hi;  // slices [s_lo, s_hi)
  int n1;                // main chunks (phase 1 and phase 2 each)
  int nh;                // halo chunks
  long long h0;          // first halo slice
};

__device__ __forceinline__ TileInfo tile_info(const PairArgs& pa, long long S, int sps, int b) {
  TileInfo t;
  t.s_lo = static_cast<long long>(b) * pa.ts;
  t.s_hi = t.s_lo + pa.ts < S ? t.s_lo + pa.ts : S;
  t.n1 = static_cast<int>((t.s_hi - t.s_lo + sps - 1) / sps);
  t.nh = pa.hsl[b] / sps;
  t.h0 = pa.hoff[b];
  return t;
}

__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

}  // namespace

template <int NJ, int CW>
__global__ void __launch_bounds__(32 * (CW + 1), 1)
pair_tma_kernel(PairArgs pa, const double* u_in, double* u_out, int flags, TmaGeom g) {
  extern __shared__ __align__(128) unsigned char pair_smem[];
  constexpr int kMaxStages = 16;
  constexpr int kW = NJ * 32 * 8, kC16 = NJ * 32 * 2, kC32 = NJ * 32 * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(pair_smem);
  uint64_t* empty = full + kMaxStages;
  unsigned char* ring = pair_smem + 2 * kMaxStages * sizeof(uint64_t);
  __shared__ long long s_issued;  // chunks armed so far (parity-alias gate, see step_tma_kernel)
  const StepArgs& a = pa.a;
  const int sps = g.sps, lsps = g.contig, stages = g.stages;  // sps = 1 << lsps
  const int wbytes = sps * kW;
  const int stage_bytes = sps * (kW + kC32 + 32 * 12);  // the halo chunk is the largest kind
  double* U1base = reinterpret_cast<double*>(ring + static_cast<size_t>(stages) * stage_bytes);
  const long long S = (a.n_rows + 31) >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_my = pa.n_tiles > static_cast<int>(blockIdx.x)
                       ? (pa.n_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1 : 0;

  // ring chunks of this CTA: phase-1 data only, per tile n1 + nh
  long long total = 0;
  for (int k = 0; k < n_my; ++k) {
    const TileInfo t = tile_info(pa, S, sps, blockIdx.x + k * gridDim.x);
    total += t.n1 + t.nh;
  }

  if (threadIdx.x == 0) {
    s_issued = 0;
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], static_cast<uint32_t>(sps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_launch_dependents();

  DevStatus* st = a.st;
  bool bad = false;
  unsigned long long dmax = 0ull;
  long long gstep = 0;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
      int kt = 0, phase = 0, k = 0;
      TileInfo ti = {};
      if (n_my > 0) ti = tile_info(pa, S, sps, blockIdx.x);
      long long i = 0;
      auto issue = [&]() {
        const int s = static_cast<int>(i % stages);
        unsigned char* dst = ring + static_cast<size_t>(s) * stage_bytes;
        if (phase == 0) {  // main rows: W | C16 | F | meta (W, F re-read in phase 2: keep in L2)
          const long long s0 = ti.s_lo + static_cast<long long>(k) * sps;
          const int ns = static_cast<int>(ti.s_hi - s0 < sps ? ti.s_hi - s0 : sps);
          if (k == 0) {  // the tile's phase-2 local ids, into L2 ahead of their use
            const uint32_t lb = static_cast<uint32_t>((ti.s_hi - ti.s_lo) * kC16);
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(pa.L16 + ti.s_lo * NJ * 32),
                         "r"(lb), "l"(pol_last)
                         : "memory");
          }
          mbar_expect_tx(&full[s], ns * (kW + kC16 + 256 + 16));
          bulk_g2s(dst, a.W + s0 * NJ * 32, ns * kW, &full[s], pol_last);
          bulk_g2s(dst + wbytes, a.C16 + s0 * NJ * 32, ns * kC16, &full[s], pol_first);
          bulk_g2s(dst + wbytes + sps * kC16, a.F + s0 * 32, ns * 256, &full[s], pol_last);
          bulk_g2s(dst + wbytes + sps * kC16 + sps * 256, a.meta + s0, ns * 16, &full[s], pol_first);
          if (++k == ti.n1) {
            k = 0;
            phase = 1;
          }
        } else {  // halo rows: W | HC | HF | HR (full chunks)
          const long long h = ti.h0 + static_cast<long long>(k) * sps;
          mbar_expect_tx(&full[s], sps * (kW + kC32 + 256 + 128));
          bulk_g2s(dst, pa.HW + h * NJ * 32, sps * kW, &full[s], pol_first);
          bulk_g2s(dst + wbytes, pa.HC + h * NJ * 32, sps * kC32, &full[s], pol_first);
          bulk_g2s(dst + wbytes + sps * kC32, pa.HF + h * 32, sps * 256, &full[s], pol_first);
          bulk_g2s(dst + wbytes + sps * kC32 + sps * 256, pa.HR + h * 32, sps * 128, &full[s], pol_first);
          ++k;
        }
        if (phase == 1 && k == ti.nh) {
          k = 0;
          phase = 0;
          if (++kt < n_my) ti = tile_info(pa, S, sps, blockIdx.x + kt * gridDim.x);
        }
        __threadfence_block();
        ++i;
        *reinterpret_cast<volatile long long*>(&s_issued) = i;
      };
      const long long pre = total < stages ? total : stages;
      while (i < pre) issue();  // weights only: before the dependency wait
      pdl_wait();
      const long long g0 = *reinterpret_cast<volatile long long*>(&st->step);
      const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
      const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
      if ((bs >= 0 && bs < g0) || (cs >= 0 && cs < g0)) {
        for (long long q = 0; q < pre; ++q) mbar_wait(&full[q % stages], 0);  // drain the ring
        return;
      }
      while (i < total) {
        const int s = static_cast<int>(i % stages);
        mbar_wait(&empty[s], static_cast<uint32_t>(((i / stages) - 1) & 1));
        issue();
      }
    } else {
      pdl_wait();
      const long long g0 = *reinterpret_cast<volatile long long*>(&st->step);
      const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
      const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
      if ((bs >= 0 && bs < g0) || (cs >= 0 && cs < g0)) return;
    }
    gstep = *reinterpret_cast<volatile long long*>(&st->step);
  } else {
    pdl_wait();
    gstep = *reinterpret_cast<volatile long long*>(&st->step);
    const long long bs = *reinterpret_cast<volatile long long*>(&st->bad_step);
    const long long cs = *reinterpret_cast<volatile long long*>(&st->conv_step);
    if ((bs >= 0 && bs < gstep) || (cs >= 0 && cs < gstep)) return;
    const double dt = st->dt;
    const uint64_t pol_first = policy_evict_first();
    long long cbase = 0;  // first ring chunk of the current segment's phase-1 tile
    // Segment k: phase 1 of tile k (ring) interleaved with phase 2 of tile
    // k-1 (direct loads, L2-resident weights), so HBM streams the next tile
    // while the previous one finishes; one consumer barrier per segment.
    for (int kseg = 0; kseg <= n_my; ++kseg) {
      TileInfo t1 = {}, t2 = {};
      int A = 0, Bn = 0;
      if (kseg < n_my) {
        t1 = tile_info(pa, S, sps, blockIdx.x + kseg * gridDim.x);
        A = (t1.n1 + t1.nh) << lsps;
      }
      if (kseg > 0) {
        t2 = tile_info(pa, S, sps, blockIdx.x + (kseg - 1) * gridDim.x);
        Bn = static_cast<int>(t2.s_hi - t2.s_lo);
      }
      const long long lo1 = t1.s_lo * 32, lo2 = t2.s_lo * 32;
      const long long nt1 = (a.n_rows - lo1) < static_cast<long long>(pa.ts) * 32 ? a.n_rows - lo1
                                                                                     : static_cast<long long>(pa.ts) * 32;
      double* U1w = U1base + static_cast<size_t>(kseg & 1) * pa.u1_cap;              // phase 1 writes
      const double* U1r = U1base + static_cast<size_t>((kseg + 1) & 1) * pa.u1_cap;  // phase 2 reads
      const int both = 2 * (A < Bn ? A : Bn);
      const int main1 = t1.n1 << lsps;
      for (int q = warp - 1; q < A + Bn; q += CW) {
        int p1 = -1, p2 = -1;
        if (q < both) {
          if (q & 1) p2 = q >> 1;
          else p1 = q >> 1;
        } else if (A > Bn) {
          p1 = q - (both >> 1);
        } else {
          p2 = q - (both >> 1);
        }
        if (p1 >= 0) {
          // ---- phase 1: u^t (global) -> u^{t+1} (U1w), tile rows and halo
          const long long i = cbase + (p1 >> lsps);
          const int slot = p1 & (sps - 1);
          const int s = static_cast<int>(i % stages);
          if (lane == 0) {
            while (*reinterpret_cast<volatile long long*>(&s_issued) <= i) __nanosleep(32);
          }
          __syncwarp();
          mbar_wait(&full[s], static_cast<uint32_t>((i / stages) & 1));
          const unsigned char* base = ring + static_cast<size_t>(s) * stage_bytes;
          const double* sW = reinterpret_cast<const double*>(base) + slot * NJ * 32;
          if (p1 < main1) {
            const long long sl = t1.s_lo + p1;
            const long long r = sl * 32 + lane;
            if (sl < t1.s_hi && r < a.n_rows) {
              const int4 m = reinterpret_cast<const int4*>(base + wbytes + sps * kC16 + sps * 256)[slot];
              double gv[NJ];
              int c0;
              if (m.z) {
                const unsigned short* sC = reinterpret_cast<const unsigned short*>(base + wbytes) + slot * NJ * 32;
                c0 = decode_id(sC[lane], m);
                gv[0] = ld_field(u_in + c0);
#pragma unroll
                for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + decode_id(sC[j * 32 + lane], m));
              } else {  // slice outside the two 15-bit windows: int32 ids from HBM
                const int* gC = a.C + sl * NJ * 32 + lane;
                c0 = __ldg(gC);
                gv[0] = ld_field(u_in + c0);
#pragma unroll
                for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + __ldg(gC + 32 * j));
              }
              const long long node = a.dst_base + r;
              const double u_self = (c0 == node) ? gv[0] : ld_field(u_in + node);
              const double f = reinterpret_cast<const double*>(base + wbytes + sps * kC16)[slot * 32 + lane];
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(sW[j * 32 + lane], gv[j]));
              const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(f, acc)));
              U1w[r - lo1] = value;
              if (!isfinite(value)) bad = true;
            }
          } else {
            const int e = ((p1 - main1) << 5) + lane;  // halo entry of the tile
            const int hr = reinterpret_cast<const int*>(base + wbytes + sps * kC32 + sps * 256)[slot * 32 + lane];
            if (hr >= 0) {
              const int* sC = reinterpret_cast<const int*>(base + wbytes) + slot * NJ * 32;
              double gv[NJ];
              const int c0 = sC[lane];
              gv[0] = ld_field(u_in + c0);
#pragma unroll
              for (int j = 1; j < NJ; ++j) gv[j] = ld_field(u_in + sC[j * 32 + lane]);
              const double u_self = (c0 == hr) ? gv[0] : ld_field(u_in + hr);
              const double f = reinterpret_cast<const double*>(base + wbytes + sps * kC32)[slot * 32 + lane];
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(sW[j * 32 + lane], gv[j]));
              U1w[nt1 + e] = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(f, acc)));
            } else if (hr != INT_MIN) {
              U1w[nt1 + e] = ld_field(u_in + (-(hr + 1)));  // Dirichlet node: fixed
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        } else {
          // ---- phase 2 of the previous tile: u^{t+1} (U1r) -> u^{t+2} (global)
          const long long sl = t2.s_lo + p2;
          const long long r = sl * 32 + lane;
          if (r < a.n_rows) {
            const double* gW = a.W + sl * NJ * 32 + lane;
            const unsigned short* gL = pa.L16 + sl * NJ * 32 + lane;
            double w[NJ];
            unsigned short l[NJ];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              w[j] = ld_stream_f64(gW + 32 * j, pol_first);
              l[j] = __ldg(gL + 32 * j);
            }
            const double f = ld_stream_f64(a.F + sl * 32 + lane, pol_first);
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc = __dadd_rn(acc, __dmul_rn(w[j], U1r[l[j]]));
            const double u_self = U1r[r - lo2];
            const double value = __dadd_rn(u_self, __dmul_rn(dt, __dadd_rn(f, acc)));
            u_out[a.dst_base + r] = value;
            if (!isfinite(value)) bad = true;
            if (flags & kNeedResidual) {
              const unsigned long long bits = static_cast<unsigned long long>(
                  __double_as_longlong(fabs(__dsub_rn(value, u_self))));
              dmax = bits > dmax ? bits : dmax;
            }
          }
        }
      }
      cbase += t1.n1 + t1.nh;
      if (kseg < n_my) consumer_bar(CW * 32);  // phase 1 of tile kseg complete
    }
  }
  step_epilogue(st, gstep, bad, dmax, flags, 2);
}

// ---------------------------------------------------------------------------
// Table construction (plan build, stream-ordered).

namespace {

constexpr unsigned long long kNoKey = ~0ull;

// key (tile << 32 | node) for every stencil entry that leaves its row's tile
__global__ void pair_keys_kernel(const int* __restrict__ C, long long n_rows, int n, long long B, int ts,
                                 unsigned long long* __restrict__ keys) {
  const long long S = (n_rows + 31) >> 5;
  const long long total = S * n * 32;
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long sl = x / (static_cast<long long>(n) * 32);
    const int lane = static_cast<int>(x & 31);
    const long long r = sl * 32 + lane;
    unsigned long long key = kNoKey;
    if (r < n_rows) {
      const long long c = C[x];
      const long long b = sl / ts;
      const long long rl = b * ts * 32;
      const long long rh = rl + static_cast<long long>(ts) * 32 < n_rows ? rl + static_cast<long long>(ts) * 32 : n_rows;
      const bool inside = c >= B && c - B >= rl && c - B < rh;
      if (!inside) key = (static_cast<unsigned long long>(b) << 32) | static_cast<unsigned long long>(c);
    }
    keys[x] = key;
  }
}

struct NotNoKey {
  __host__ __device__ bool operator()(unsigned long long k) const { return k != kNoKey; }
};

__global__ void pair_count_kernel(const unsigned long long* __restrict__ uniq, long long m,
                                  int* __restrict__ cnt) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    atomicAdd(cnt + (uniq[e] >> 32), 1);
}

__global__ void pair_fill_hr_kernel(int* __restrict__ HR, long long count) {
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < count;
       x += static_cast<long long>(gridDim.x) * blockDim.x)
    HR[x] = INT_MIN;
}

// halo entry e of tile b -> halo slice hoff[b] + k/32, lane k%32 (k = e - eoff[b])
__global__ void pair_halo_kernel(const unsigned long long* __restrict__ uniq, long long m,
                                 const long long* __restrict__ eoff, const int* __restrict__ hoff,
                                 const double* __restrict__ W, const int* __restrict__ C,
                                 const double* __restrict__ F, long long B, int n,
                                 double* __restrict__ HW, int* __restrict__ HC, double* __restrict__ HF,
                                 int* __restrict__ HR) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(uniq[e] >> 32);
    const long long c = static_cast<long long>(uniq[e] & 0xffffffffull);
    const long long k = e - eoff[b];
    const long long hs = hoff[b] + k / 32;
    const int ln = static_cast<int>(k & 31);
    if (c >= B) {
      const long long row = c - B;
      const long long ss = row >> 5;
      const int sl = static_cast<int>(row & 31);
      for (int j = 0; j < n; ++j) {
        HW[(hs * n + j) * 32 + ln] = W[(ss * n + j) * 32 + sl];
        HC[(hs * n + j) * 32 + ln] = C[(ss * n + j) * 32 + sl];
      }
      HF[hs * 32 + ln] = F[ss * 32 + sl];
      HR[hs * 32 + ln] = static_cast<int>(c);
    } else {
      HR[hs * 32 + ln] = -static_cast<int>(c) - 1;
    }
  }
}

// tile-local id of every stencil entry: own rows first, then the halo entries
__global__ void pair_local_kernel(const int* __restrict__ C, long long n_rows, int n, long long B, int ts,
                                  const unsigned long long* __restrict__ uniq,
                                  const long long* __restrict__ eoff, const int* __restrict__ ecnt,
                                  unsigned short* __restrict__ L16, int* __restrict__ overflow) {
  const long long S = (n_rows + 31) >> 5;
  const long long total = S * n * 32;
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long sl = x / (static_cast<long long>(n) * 32);
    const int lane = static_cast<int>(x & 31);
    const long long r = sl * 32 + lane;
    long long loc = 0;
    if (r < n_rows) {
      const long long c = C[x];
      const long long b = sl / ts;
      const long long rl = b * ts * 32;
      const long long cap = static_cast<long long>(ts) * 32;
      const long long nt = n_rows - rl < cap ? n_rows - rl : cap;
      if (c >= B && c - B >= rl && c - B < rl + nt) {
        loc = c - B - rl;
      } else {
        const unsigned long long key = (static_cast<unsigned long long>(b) << 32) | static_cast<unsigned long long>(c);
        long long lo = eoff[b], hi = eoff[b] + ecnt[b];
        while (lo < hi) {
          const long long mid = (lo + hi) >> 1;
          if (uniq[mid] < key) lo = mid + 1;
          else hi = mid;
        }
        loc = nt + (lo - eoff[b]);
        if (lo >= eoff[b] + ecnt[b] || uniq[lo] != key) atomicExch(overflow, 2);  // cannot happen
      }
      if (loc > 0xffff) atomicExch(overflow, 1);
    }
    L16[x] = static_cast<unsigned short>(loc);
  }
}

template <int NJ>
struct PairSet {
  static constexpr int kCW = 15;  // + 1 producer warp = 512 threads
  static PairFn fn() { return pair_tma_kernel<NJ, kCW>; }
};

int ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RBF_OK;
  return rbf_detail::fail_c(RBF_ERR_CUDA, (std::string("pair build: ") + what + ": " + cudaGetErrorString(e)).c_str());
}

template <typename T>
int alloc(T** p, size_t count, cudaStream_t st, const char* what) {
  return ck(cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T), st), what);
}

}  // namespace

#define RBF_PAIR_WIDTHS(X) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(12) X(15) X(16) X(20) X(21) X(24) X(28) X(30) X(32)

PairFn pair_kernel_for(int n, int* cw) {
  switch (n) {
#define RBF_PCASE(K)           \
  case K:                      \
    *cw = PairSet<K>::kCW;     \
    return PairSet<K>::fn();
    RBF_PAIR_WIDTHS(RBF_PCASE)
#undef RBF_PCASE
    default:
      return nullptr;
  }
}

#define RBF_TRY_(x)              \
  do {                           \
    int rc_ = (x);               \
    if (rc_ != RBF_OK) return rc_; \
  } while (0)

int pair_build(const StepArgs& a, int sps, int tiles_per_cta, int sms, size_t smem_budget,
               cudaStream_t st, PairPlan* out, bool* ok, int ts_fixed, bool tables_only) {
  *ok = false;
  int cw = 0;
  PairFn fn = pair_kernel_for(a.n, &cw);
  if (!tables_only && (!fn || !a.C16 || !a.meta)) return RBF_OK;
  if (a.n_rows <= 0) return RBF_OK;
  const int n = a.n;
  const long long S = (a.n_rows + 31) >> 5;
  {  // the pair ring streams chunks of a power-of-two slice count
    int p2 = 1;
    while (p2 * 2 <= sps) p2 *= 2;
    sps = p2;
  }
  // tile size: `tiles_per_cta` tiles per SM-resident CTA, a multiple of sps,
  // at most 32 slices (1024 rows) so rows + halo stay within 16-bit local ids
  long long ts = (S + static_cast<long long>(sms) * tiles_per_cta - 1) / (static_cast<long long>(sms) * tiles_per_cta);
  ts = std::max<long long>(ts, sps);
  ts = (ts + sps - 1) / sps * sps;
  ts = std::min<long long>(ts, std::max<long long>(sps, 64 / sps * sps));
  if (ts_fixed > 0) ts = ts_fixed;  // tiles = the caller's CTA ranges (grid-resident loop)
  const int n_tiles = static_cast<int>((S + ts - 1) / ts);
  const long long total = S * n * 32;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 32));

  unsigned long long *keys = nullptr, *sel = nullptr, *sorted = nullptr, *uniq = nullptr;
  long long* d_num = nullptr;
  void* tmp = nullptr;
  RBF_TRY_(alloc(&keys, total, st, "keys"));
  RBF_TRY_(alloc(&sel, total, st, "selected"));
  RBF_TRY_(alloc(&d_num, 2, st, "count"));
  pair_keys_kernel<<<blocks, 256, 0, st>>>(a.C, a.n_rows, n, a.dst_base, static_cast<int>(ts), keys);
  RBF_TRY_(ck(cudaGetLastError(), "keys kernel"));
  size_t tb = 0;
  RBF_TRY_(ck(cub::DeviceSelect::If(nullptr, tb, keys, sel, d_num, total, NotNoKey(), st), "select size"));
  RBF_TRY_(alloc(reinterpret_cast<unsigned char**>(&tmp), tb, st, "select tmp"));
  RBF_TRY_(ck(cub::DeviceSelect::If(tmp, tb, keys, sel, d_num, total, NotNoKey(), st), "select"));
  long long m_sel = 0;
  RBF_TRY_(ck(cudaMemcpyAsync(&m_sel, d_num, sizeof(long long), cudaMemcpyDeviceToHost, st), "count d2h"));
  RBF_TRY_(ck(cudaStreamSynchronize(st), "sync"));
  cudaFreeAsync(tmp, st);
  tmp = nullptr;
  cudaFreeAsync(keys, st);
  keys = nullptr;
  int tile_bits = 1;
  while ((1LL << tile_bits) < n_tiles) ++tile_bits;
  RBF_TRY_(alloc(&sorted, m_sel, st, "sorted"));
  RBF_TRY_(alloc(&uniq, m_sel, st, "unique"));
  tb = 0;
  RBF_TRY_(ck(cub::DeviceRadixSort::SortKeys(nullptr, tb, sel, sorted, m_sel, 0, 32 + tile_bits, st), "sort size"));
  RBF_TRY_(alloc(reinterpret_cast<unsigned char**>(&tmp), tb, st, "sort tmp"));
  RBF_TRY_(ck(cub::DeviceRadixSort::SortKeys(tmp, tb, sel, sorted, m_sel, 0, 32 + tile_bits, st), "sort"));
  cudaFreeAsync(tmp, st);
  tmp = nullptr;
  tb = 0;
  RBF_TRY_(ck(cub::DeviceSelect::Unique(nullptr, tb, sorted, uniq, d_num + 1, m_sel, st), "unique size"));
  RBF_TRY_(alloc(reinterpret_cast<unsigned char**>(&tmp), tb, st, "unique tmp"));
  RBF_TRY_(ck(cub::DeviceSelect::Unique(tmp, tb, sorted, uniq, d_num + 1, m_sel, st), "unique"));
  cudaFreeAsync(tmp, st);
  tmp = nullptr;
  cudaFreeAsync(sel, st);
  cudaFreeAsync(sorted, st);
  int* d_cnt = nullptr;
  RBF_TRY_(alloc(&d_cnt, n_tiles, st, "tile counts"));
  RBF_TRY_(ck(cudaMemsetAsync(d_cnt, 0, sizeof(int) * n_tiles, st), "memset"));
  long long m = 0;
  RBF_TRY_(ck(cudaMemcpyAsync(&m, d_num + 1, sizeof(long long), cudaMemcpyDeviceToHost, st), "unique d2h"));
  RBF_TRY_(ck(cudaStreamSynchronize(st), "sync"));
  if (m > 0) {
    pair_count_kernel<<<static_cast<int>(std::min<long long>((m + 255) / 256, 4096)), 256, 0, st>>>(uniq, m, d_cnt);
    RBF_TRY_(ck(cudaGetLastError(), "count kernel"));
  }
  std::vector<int> cnt(n_tiles), hsl(n_tiles), hoff(n_tiles);
  std::vector<long long> eoff(n_tiles);
  RBF_TRY_(ck(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int) * n_tiles, cudaMemcpyDeviceToHost, st), "counts d2h"));
  RBF_TRY_(ck(cudaStreamSynchronize(st), "sync"));
  long long e_acc = 0, h_acc = 0;
  int u1_cap = 0;
  bool fits = true;
  for (int b = 0; b < n_tiles; ++b) {
    eoff[b] = e_acc;
    e_acc += cnt[b];
    const int slices = (cnt[b] + 31) / 32;
    hsl[b] = (slices + sps - 1) / sps * sps;
    hoff[b] = static_cast<int>(h_acc);
    h_acc += hsl[b];
    const long long rl = static_cast<long long>(b) * ts * 32;
    const long long nt = std::min<long long>(ts * 32, a.n_rows - rl);
    const long long cap = nt + static_cast<long long>(hsl[b]) * 32;
    if (nt + cnt[b] > 0xffff + 1) fits = false;
    u1_cap = static_cast<int>(std::max<long long>(u1_cap, cap));
  }
  const long long HS = h_acc;
  long long* d_eoff = nullptr;
  int *d_hoff = nullptr, *d_hsl = nullptr, *d_over = nullptr, *HC = nullptr, *HR = nullptr;
  double *HW = nullptr, *HF = nullptr;
  unsigned short* L16 = nullptr;
  RBF_TRY_(alloc(&d_eoff, n_tiles, st, "eoff"));
  RBF_TRY_(alloc(&d_hoff, n_tiles, st, "hoff"));
  RBF_TRY_(alloc(&d_hsl, n_tiles, st, "hsl"));
  RBF_TRY_(alloc(&d_over, 1, st, "overflow"));
  RBF_TRY_(ck(cudaMemcpyAsync(d_eoff, eoff.data(), sizeof(long long) * n_tiles, cudaMemcpyHostToDevice, st), "eoff h2d"));
  RBF_TRY_(ck(cudaMemcpyAsync(d_hoff, hoff.data(), sizeof(int) * n_tiles, cudaMemcpyHostToDevice, st), "hoff h2d"));
  RBF_TRY_(ck(cudaMemcpyAsync(d_hsl, hsl.data(), sizeof(int) * n_tiles, cudaMemcpyHostToDevice, st), "hsl h2d"));
  RBF_TRY_(ck(cudaMemsetAsync(d_over, 0, sizeof(int), st), "memset"));
  RBF_TRY_(alloc(&HW, HS * n * 32, st, "HW"));
  RBF_TRY_(alloc(&HC, HS * n * 32, st, "HC"));
  RBF_TRY_(alloc(&HF, HS * 32, st, "HF"));
  RBF_TRY_(alloc(&HR, HS * 32, st, "HR"));
  RBF_TRY_(alloc(&L16, total, st, "L16"));
  RBF_TRY_(ck(cudaMemsetAsync(HW, 0, sizeof(double) * std::max<long long>(HS * n * 32, 1), st), "memset"));
  RBF_TRY_(ck(cudaMemsetAsync(HC, 0, sizeof(int) * std::max<long long>(HS * n * 32, 1), st), "memset"));
  RBF_TRY_(ck(cudaMemsetAsync(HF, 0, sizeof(double) * std::max<long long>(HS * 32, 1), st), "memset"));
  if (HS > 0) {
    pair_fill_hr_kernel<<<static_cast<int>(std::min<long long>((HS * 32 + 255) / 256, 4096)), 256, 0, st>>>(HR, HS * 32);
    RBF_TRY_(ck(cudaGetLastError(), "fill kernel"));
  }
  if (m > 0) {
    pair_halo_kernel<<<static_cast<int>(std::min<long long>((m + 255) / 256, 8192)), 256, 0, st>>>(
        uniq, m, d_eoff, d_hoff, a.W, a.C, a.F, a.dst_base, n, HW, HC, HF, HR);
    RBF_TRY_(ck(cudaGetLastError(), "halo kernel"));
  }
  pair_local_kernel<<<blocks, 256, 0, st>>>(a.C, a.n_rows, n, a.dst_base, static_cast<int>(ts), uniq, d_eoff, d_cnt,
                                            L16, d_over);
  RBF_TRY_(ck(cudaGetLastError(), "local kernel"));
  int over = 0;
  RBF_TRY_(ck(cudaMemcpyAsync(&over, d_over, sizeof(int), cudaMemcpyDeviceToHost, st), "overflow d2h"));
  RBF_TRY_(ck(cudaStreamSynchronize(st), "sync"));
  cudaFreeAsync(uniq, st);
  cudaFreeAsync(d_num, st);
  cudaFreeAsync(d_over, st);
  cudaFreeAsync(d_eoff, st);

  PairPlan pp;
  pp.fn = fn;
  pp.args.a = a;
  pp.args.HW = HW;
  pp.args.HC = HC;
  pp.args.HF = HF;
  pp.args.HR = HR;
  pp.args.L16 = L16;
  pp.args.hoff = d_hoff;
  pp.args.hsl = d_hsl;
  pp.args.ts = static_cast<int>(ts);
  pp.args.n_tiles = n_tiles;
  pp.args.u1_cap = u1_cap;
  pp.halo_entries = m;
  pp.halo_slices = HS;
  void* bufs[8] = {HW, HC, HF, HR, L16, d_hoff, d_hsl, d_cnt};
  for (int k = 0; k < 8; ++k) pp.bufs[k] = bufs[k];
  // ring: halo-chunk sized stages in what the two U1 buffers leave
  const size_t stage = static_cast<size_t>(sps) * (static_cast<size_t>(n) * 32 * 12 + 32 * 12);
  const size_t fixed = 2 * 16 * sizeof(uint64_t) + 2 * static_cast<size_t>(u1_cap) * sizeof(double);
  const int stages = fixed + 2 * stage <= smem_budget
                         ? static_cast<int>(std::min<size_t>(16, (smem_budget - fixed) / stage)) : 0;
  int lsps = 0;
  while ((2 << lsps) <= sps) ++lsps;
  pp.geom = TmaGeom{sps, stages, lsps, 0};
  pp.smem = fixed + static_cast<size_t>(stages) * stage;
  pp.block = 32 * (cw + 1);
  pp.grid = std::min(sms, n_tiles);
  *out = pp;
  if (tables_only) {
    if (over != 0 || !fits) {
      pair_free(out, st);
      return RBF_OK;
    }
    *ok = true;
    return RBF_OK;
  }
  if (over != 0 || !fits || stages < 2) {
    pair_free(out, st);
    return RBF_OK;
  }
  *ok = true;
  return RBF_OK;
}

// HF[x] = F[row of HR[x]] for every computed halo entry: the halo rows'
// forcing follows the plan's forcing (rbf_set_forcing).
__global__ void pair_refresh_hf_kernel(const int* __restrict__ HR, long long count, const double* __restrict__ F,
                                       long long B, double* __restrict__ HF) {
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < count;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = HR[x];
    if (c >= 0) HF[x] = F[c - B];
  }
}

int pair_refresh_forcing(PairPlan* pp, cudaStream_t st) {
  if (!pp->bufs[2] || pp->halo_slices == 0) return 0;
  const long long count = pp->halo_slices * 32;
  pair_refresh_hf_kernel<<<static_cast<int>(std::min<long long>((count + 255) / 256, 4096)), 256, 0, st>>>(
      static_cast<const int*>(pp->bufs[3]), count, pp->args.a.F, pp->args.a.dst_base,
      static_cast<double*>(pp->bufs[2]));
  return ck(cudaGetLastError(), "refresh forcing");
}

void pair_free(PairPlan* pp, cudaStream_t st) {
  for (void*& b : pp->bufs) {
    if (b) cudaFreeAsync(b, st);
    b = nullptr;
  }
  pp->fn = nullptr;
}

}  // namespace rbf
