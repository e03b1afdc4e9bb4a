// knn_kernels.cuh -- exact k-nearest-neighbour supports on the GPU
// (restates rbffd.neighborhoods.build_stencils,
// pkg/src/rbffd/neighborhoods.py:51-94).
//
// Result contract (the reference's, pinned by its brute-force oracle
// tests/oracles.py:16-24): row i lists the n nodes nearest to node i sorted
// by (distance, index), distance = sqrt((x_j - x_i)^2 + (y_j - y_i)^2) in
// IEEE double with separately rounded operations -- so exact distance ties
// are broken by the lower index, exactly like np.lexsort((idx, dist)).
//
// Method: points are counting-sorted into a uniform grid (~2 points per
// cell).  One thread per query scans square rings of cells around its own
// cell, keeping the n best (distance, index) pairs sorted in local memory;
// once the n-th best distance is strictly below the distance to the nearest
// unscanned cell, one more ring is scanned (guard against rounding in the
// bound) and the search stops.  Exact by construction, independent of ties.
#pragma once
#include <cstdint>

namespace rbf {

struct KnnGrid {
  double x0, y0, inv_c, c;
  int nx, ny;
};

__device__ __forceinline__ int knn_cell_x(const KnnGrid& g, double x) {
  int cx = static_cast<int>((x - g.x0) * g.inv_c);
  return cx < 0 ? 0 : (cx >= g.nx ? g.nx - 1 : cx);
}
__device__ __forceinline__ int knn_cell_y(const KnnGrid& g, double y) {
  int cy = static_cast<int>((y - g.y0) * g.inv_c);
  return cy < 0 ? 0 : (cy >= g.ny ? g.ny - 1 : cy);
}

__global__ void knn_count_kernel(const double* __restrict__ pos, long long N, KnnGrid g,
                                 int* __restrict__ cell_of, unsigned int* __restrict__ count) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = knn_cell_y(g, pos[2 * i + 1]) * g.nx + knn_cell_x(g, pos[2 * i]);
    cell_of[i] = c;
    atomicAdd(count + c, 1u);
  }
}

// scatter point ids into their cells (order inside a cell is irrelevant: the
// search sorts candidates by (distance, index))
__global__ void knn_fill_kernel(const int* __restrict__ cell_of, long long N,
                                unsigned int* __restrict__ cursor, int* __restrict__ sorted) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned int slot = atomicAdd(cursor + cell_of[i], 1u);
    sorted[slot] = static_cast<int>(i);
  }
}

template <int KMAX>
__global__ void __launch_bounds__(128) knn_query_kernel(const double* __restrict__ pos, long long N,
                                                         KnnGrid g, const unsigned int* __restrict__ start,
                                                         const int* __restrict__ sorted, int k,
                                                         long long q0, long long nq,
                                                         long long* __restrict__ out,
                                                         const long long* __restrict__ qids = nullptr) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < nq;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long qi = qids ? qids[q0 + t] : q0 + t;  // query node (all nodes, or a subset)
    const double qx = pos[2 * qi], qy = pos[2 * qi + 1];
    const int cx = knn_cell_x(g, qx), cy = knn_cell_y(g, qy);
    double bd[KMAX];
    int bi[KMAX];
    int cnt = 0;
    int extra = -1;  // rings still to scan after the stop test first passes
    const int rmax = max(g.nx, g.ny);
    for (int r = 0; r <= rmax; ++r) {
      // cells at Chebyshev ring distance r
      for (int yy = cy - r; yy <= cy + r; ++yy) {
        if (yy < 0 || yy >= g.ny) continue;
        const bool edge_row = (yy == cy - r) || (yy == cy + r);
        for (int xx = cx - r; xx <= cx + r; xx += (edge_row || r == 0) ? 1 : 2 * r) {
          if (xx < 0 || xx >= g.nx) continue;
          const int c = yy * g.nx + xx;
          for (unsigned int s = start[c]; s < start[c + 1]; ++s) {
            const int j = sorted[s];
            const double dx = __dsub_rn(pos[2 * j], qx), dy = __dsub_rn(pos[2 * j + 1], qy);
            const double d = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
            if (cnt == k && (d > bd[k - 1] || (d == bd[k - 1] && j > bi[k - 1]))) continue;
            int p = cnt < k ? cnt++ : k - 1;
            while (p > 0 && (bd[p - 1] > d || (bd[p - 1] == d && bi[p - 1] > j))) {
              bd[p] = bd[p - 1];
              bi[p] = bi[p - 1];
              --p;
            }
            bd[p] = d;
            bi[p] = j;
          }
        }
      }
      if (extra > 0) {
        if (--extra == 0) break;
        continue;
      }
      if (cnt == k) {
        // distance from the query to the nearest unscanned cell (sides that
        // reach the edge of the grid have none)
        constexpr double kInf = 1e300;
        const double lx = (cx - r > 0) ? qx - (g.x0 + (cx - r) * g.c) : kInf;
        const double hx = (cx + r < g.nx - 1) ? (g.x0 + (cx + r + 1) * g.c) - qx : kInf;
        const double ly = (cy - r > 0) ? qy - (g.y0 + (cy - r) * g.c) : kInf;
        const double hy = (cy + r < g.ny - 1) ? (g.y0 + (cy + r + 1) * g.c) - qy : kInf;
        const double bound = fmin(fmin(lx, hx), fmin(ly, hy));
        if (bound >= kInf) break;                   // the whole grid has been scanned
        if (bd[k - 1] < bound) extra = 1;           // one more ring guards the rounding of `bound`
      }
    }
    long long* o = out + t * k;
    for (int m = 0; m < k; ++m) o[m] = bi[m];
  }
}

}  // namespace rbf
