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
// reproduction, test_weights.py:51-104).
//
// Condition guard (weights.py:29, :183-192, :250-258: reject a stencil when
// np.linalg.cond -- the 2-norm condition of the saddle matrix -- exceeds
// COND_LIMIT = 1e14).  The matrix is symmetric, so kappa_2 <= kappa_1 <=
// S * kappa_2 (S = n + M).  From the LU factors the kernel estimates
// ||K^-1||_1 (Hager / Higham: a lower bound from three solves, K^-T = K^-1)
// and classifies each row:
//   0  kappa_1 estimate <= 1e10: far below the limit (typical rows: 1e3-1e7)
//   1  estimate in (1e10, S * 1e14]: the caller re-checks the exact 2-norm
//      condition on the host (np.linalg.cond, the reference's own test)
//   2  zero pivot, non-finite value, or estimate > S * 1e14 (then
//      kappa_2 >= kappa_1 / S > 1e14 for certain): degenerate.
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
  long long* bad_row;      // first flagged row, status 1 or 2 (atomicMin), LLONG_MAX if none
  unsigned char* status;   // [k0 + cnt] per-row status (0 ok, 1 host check, 2 degenerate), or null
  unsigned long long* n_flagged;  // rows with status != 0 (atomicAdd)
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr double kCondLimit = 1e14;      // weights.py:29
constexpr double kCondHostCheck = 1e10;  // kappa_1 estimates above this go to the exact host check

// In-place solve K v = b with the warp's LU factors (row swaps applied step
// by step as in the elimination; multipliers below the diagonal).
__device__ __forceinline__ void lu_solve_warp(const double* A, int L, int S, const int* piv, double* v,
                                              int lane) {
  for (int kk = 0; kk < S; ++kk) {
    if (lane == 0 && piv[kk] != kk) {
      const double t = v[kk];
      v[kk] = v[piv[kk]];
      v[piv[kk]] = t;
    }
    __syncwarp();
    const double bk = v[kk];
    for (int i = kk + 1 + lane; i < S; i += 32) v[i] -= A[i * L + kk] * bk;
    __syncwarp();
  }
  for (int i = S - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = i + 1 + lane; j < S; j += 32) s += A[i * L + j] * v[j];
    s = warp_sum_d(s);
    if (lane == 0) v[i] = (v[i] - s) / A[i * L + i];
    __syncwarp();
  }
}

__device__ __forceinline__ double warp_sum_abs(const double* v, int S, int lane) {
  double s = 0.0;
  for (int i = lane; i < S; i += 32) s += fabs(v[i]);
  return warp_sum_d(s);
}

// Shared memory per warp (doubles): [K | rhs] S x (S+1), the support (2n),
// two estimator vectors (2S), the pivot indices (S ints).
__host__ __device__ inline size_t assemble_smem_doubles(int n, int M) {
  const size_t S = static_cast<size_t>(n + M);
  return S * (S + 1) + 2 * static_cast<size_t>(n) + 2 * S + (S + 1) / 2;
}

__global__ void assemble_weights_kernel(WeightArgs a) {
  extern __shared__ __align__(16) unsigned char wsmem[];
  const int n = a.n, M = a.M, S = n + M, L = S + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const size_t per_warp = assemble_smem_doubles(n, M);  // doubles
  double* A = reinterpret_cast<double*>(wsmem) + per_warp * warp;
  double* sx = A + static_cast<size_t>(S) * L;
  double* sy = sx + n;
  double* v1 = sy + n;  // estimator vectors
  double* v2 = v1 + S;
  int* piv = reinterpret_cast<int*>(v2 + S);
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
    // ||K||_1 (K symmetric: = ||K||_inf): largest absolute column sum
    double anorm = 0.0;
    for (int j = lane; j < S; j += 32) {
      double cs = 0.0;
      for (int i = 0; i < S; ++i) cs += fabs(A[i * L + j]);
      anorm = fmax(anorm, cs);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) anorm = fmax(anorm, __shfl_xor_sync(0xffffffffu, anorm, o));
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
      if (lane == 0) piv[kk] = bi;
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
        A[i * L + kk] = l;  // multiplier, for the estimator's solves
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
    // ||K^-1||_1 lower bound (Hager / Higham, K^-T = K^-1): y = K^-1 (1/S),
    // z = K^-1 sign(y) -> max(||y||_1, ||z||_inf), and Higham's alternating
    // vector x_i = (-1)^i (1 + i/(S-1)) -> 2 ||K^-1 x||_1 / (3 S)
    double est = 0.0;
    if (!singular) {
      for (int i = lane; i < S; i += 32) v1[i] = 1.0 / S;
      __syncwarp();
      lu_solve_warp(A, L, S, piv, v1, lane);
      est = warp_sum_abs(v1, S, lane);
      for (int i = lane; i < S; i += 32) v2[i] = v1[i] >= 0.0 ? 1.0 : -1.0;
      __syncwarp();
      lu_solve_warp(A, L, S, piv, v2, lane);
      double zmax = 0.0;
      for (int i = lane; i < S; i += 32) zmax = fmax(zmax, fabs(v2[i]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
      est = fmax(est, zmax);
      for (int i = lane; i < S; i += 32)
        v1[i] = ((i & 1) ? -1.0 : 1.0) * (1.0 + (S > 1 ? static_cast<double>(i) / (S - 1) : 0.0));
      __syncwarp();
      lu_solve_warp(A, L, S, piv, v1, lane);
      est = fmax(est, 2.0 * warp_sum_abs(v1, S, lane) / (3.0 * S));
    }
    const double kappa1 = anorm * est;
    const double inv_r2 = 1.0 / (radius * radius);
    bool nonfinite = false;
    for (int j = lane; j < n; j += 32) {
      const double w = singular ? __longlong_as_double(0x7ff8000000000000LL) : A[j * L + S] * inv_r2;
      a.w_out[k * n + j] = w;
      nonfinite |= !isfinite(w);
    }
    nonfinite = __any_sync(0xffffffffu, nonfinite);
    const int st = (singular || nonfinite || !(kappa1 <= kCondLimit * S)) ? 2
                   : (kappa1 > kCondHostCheck ? 1 : 0);
    if (lane == 0) {
      if (a.status) a.status[a.k0 + k] = static_cast<unsigned char>(st);
      if (st) {
        atomicMin(reinterpret_cast<long long*>(a.bad_row), a.k0 + k);
        atomicAdd(a.n_flagged, 1ull);
      }
    }
    __syncwarp();
  }
}

}  // namespace rbf
