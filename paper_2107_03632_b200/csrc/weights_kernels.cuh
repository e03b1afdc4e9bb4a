// weights_kernels.cuh -- GPU assembly of the RBF-FD Laplacian weights
// (the "next" component after the time loop).
//
// Restates rbffd.weights._weights_batch (pkg/src/rbffd/weights.py:218-259):
// per interior row, shift the support to its first point, scale by the
// support radius, build the saddle system
//     [ A  P ] [w]   [ 9 r_i       ]     A_ij = |x_i - x_j|^3   (phs3, :89)
//     [ P' 0 ] [l] = [ lap0(monos) ]     P_ik = x_i^a_k y_i^b_k (graded lex, :35-68)
// solve it, and rescale w by 1 / radius^2.  One warp solves one system with
// Gaussian elimination with partial pivoting (LAPACK gesv's algorithm, not
// its blocking: the weights agree with the reference to rounding, not bit
// for bit -- the reference's own tests pin weights by polynomial
// reproduction, test_weights.py:51-104).  The condition-number guard of the
// reference (COND_LIMIT, weights.py:29, an SVD) is replaced by a zero-pivot /
// non-finite check that flags the first failing row.
#pragma once
#include <cstdint>

namespace rbf {

struct WeightArgs {
  const double* pos;       // [N*2] node positions
  const int* rows;         // [cnt*n] support node ids (row-major, entry 0 = centre)
  long long cnt;           // rows in this launch
  long long k0;            // global index of the first row (error reporting)
  int n;                   // support size
  int M;                   // monomials
  int ex[28], ey[28];      // exponents, degree <= 6
  double lap0[28];         // Laplacian of each monomial at the origin
  double* w_out;           // [cnt*n] row-major weights
  long long* bad_row;      // first degenerate row (atomicMin), LLONG_MAX if none
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void assemble_weights_kernel(WeightArgs a) {
  extern __shared__ __align__(16) unsigned char wsmem[];
  const int n = a.n, M = a.M, S = n + M, L = S + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const size_t per_warp = static_cast<size_t>(S) * L + 2 * n;  // doubles
  double* A = reinterpret_cast<double*>(wsmem) + per_warp * warp;
  double* sx = A + static_cast<size_t>(S) * L;
  double* sy = sx + n;
  for (long long k = static_cast<long long>(blockIdx.x) * nwarps + warp; k < a.cnt;
       k += static_cast<long long>(gridDim.x) * nwarps) {
    const int* rk = a.rows + k * n;
    const long long c = rk[0];
    const double cx = a.pos[2 * c], cy = a.pos[2 * c + 1];
    double r2max = 0.0;
    for (int i = lane; i < n; i += 32) {
      const long long g = rk[i];
      const double lx = a.pos[2 * g] - cx, ly = a.pos[2 * g + 1] - cy;
      sx[i] = lx;
      sy[i] = ly;
      r2max = fmax(r2max, lx * lx + ly * ly);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2max = fmax(r2max, __shfl_xor_sync(0xffffffffu, r2max, o));
    const double radius = sqrt(r2max);
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      sx[i] /= radius;
      sy[i] /= radius;
    }
    __syncwarp();
    // build [K | rhs]
    for (int e = lane; e < S * L; e += 32) {
      const int i = e / L, j = e - i * L;
      double v;
      if (j == S) {
        v = i < n ? 9.0 * sqrt(sx[i] * sx[i] + sy[i] * sy[i]) : a.lap0[i - n];
      } else if (i < n && j < n) {
        const double dx = sx[i] - sx[j], dy = sy[i] - sy[j];
        const double r = sqrt(dx * dx + dy * dy);
        v = r * r * r;
      } else if (i < n || j < n) {
        const int p = i < n ? i : j, mk = i < n ? j - n : i - n;
        double t = 1.0;
        for (int q = 0; q < a.ex[mk]; ++q) t *= sx[p];
        for (int q = 0; q < a.ey[mk]; ++q) t *= sy[p];
        v = t;
      } else {
        v = 0.0;
      }
      A[e] = v;
    }
    __syncwarp();
    bool singular = false;
    for (int kk = 0; kk < S; ++kk) {
      // partial pivoting: first index of the largest |a_ik| (idamax)
      double best = -1.0;
      int bi = S;
      for (int i = kk + lane; i < S; i += 32) {
        const double v = fabs(A[i * L + kk]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (!(best > 0.0)) {
        singular = true;
        break;
      }
      if (bi != kk) {
        for (int j = kk + lane; j <= S; j += 32) {
          const double t = A[kk * L + j];
          A[kk * L + j] = A[bi * L + j];
          A[bi * L + j] = t;
        }
      }
      __syncwarp();
      const double piv = A[kk * L + kk];
      for (int i = kk + 1 + lane; i < S; i += 32) {
        const double l = A[i * L + kk] / piv;
        for (int j = kk + 1; j <= S; ++j) A[i * L + j] -= l * A[kk * L + j];
      }
      __syncwarp();
    }
    if (!singular) {
      // back substitution, solution overwrites the rhs column
      for (int i = S - 1; i >= 0; --i) {
        double s = 0.0;
        for (int j = i + 1 + lane; j < S; j += 32) s += A[i * L + j] * A[j * L + S];
        s = warp_sum_d(s);
        if (lane == 0) A[i * L + S] = (A[i * L + S] - s) / A[i * L + i];
        __syncwarp();
      }
    }
    const double inv_r2 = 1.0 / (radius * radius);
    bool bad = singular;
    for (int j = lane; j < n; j += 32) {
      const double w = singular ? __longlong_as_double(0x7ff8000000000000LL) : A[j * L + S] * inv_r2;
      a.w_out[k * n + j] = w;
      bad |= !isfinite(w);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0)
      atomicMin(reinterpret_cast<long long*>(a.bad_row), a.k0 + k);
    __syncwarp();
  }
}

}  // namespace rbf
