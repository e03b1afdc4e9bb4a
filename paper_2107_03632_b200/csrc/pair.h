// pair.h -- host interface of the two-step tile kernel (pair_kernels.cu) to
// the plan driver (rbffd_b200.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace rbf {

// Device tables of the two-step (temporal-blocking) layout of one plan.
// Rows are cut into tiles of `ts` SELL slices.  For tile b, the halo is the
// sorted set of nodes its rows' stencils reference outside the tile (interior
// rows of other tiles and Dirichlet nodes); the tile's local numbering is
// [its own rows | its halo entries], so its second step reads every value it
// needs from shared memory.
struct PairArgs {
  StepArgs a;
  const double* HW;           // [HS*n*32] halo rows' weights (SELL, halo slices)
  const int* HC;              // [HS*n*32] halo rows' node ids (int32)
  const double* HF;           // [HS*32]   halo rows' forcing
  const int* HR;              // [HS*32]   node of the entry: >= 0 row to compute,
                              //           -(c+1) Dirichlet node c (copied), INT_MIN padding
  const unsigned short* L16;  // [S*n*32]  tile-local ids of every row's stencil
  const int* hoff;            // [n_tiles] first halo slice of the tile (multiple of sps)
  const int* hsl;             // [n_tiles] halo slices of the tile (multiple of sps)
  int ts;                     // slices per tile (multiple of sps)
  int n_tiles;
  int u1_cap;                 // doubles per shared-memory value buffer (2 buffers)
};

using PairFn = void (*)(PairArgs, const double*, double*, int, TmaGeom);

struct PairPlan {
  PairFn fn = nullptr;
  PairArgs args = {};
  TmaGeom geom = {1, 2, 0, 0};
  size_t smem = 0;
  int block = 0;
  int grid = 0;
  int64_t halo_entries = 0;   // sum over tiles of the halo sizes
  int64_t halo_slices = 0;
  void* bufs[8] = {};         // device allocations owned by the plan (pool)
};

// Kernel for support size n (nullptr when not specialised); consumer warps.
PairFn pair_kernel_for(int n, int* cw);
// Builds the tables for a plan with n_rows rows in SELL slices (W, C, F),
// B Dirichlet nodes first, stream-ordered on `st`.  Returns 0 or an RBF_ERR_*
// code (message via rbf_detail::fail_c); *ok = false when the layout does not
// apply (local ids would not fit 16 bits).
// ts_fixed > 0: tiles of exactly ts_fixed slices; tables_only: build the halo /
// local-id tables without requiring the pair kernel (the grid-resident loop's
// two-step mode uses them).
int pair_build(const StepArgs& a, int sps, int tiles_per_cta, int sms, size_t smem_budget,
               cudaStream_t st, PairPlan* out, bool* ok, int ts_fixed = 0, bool tables_only = false);
void pair_free(PairPlan* pp, cudaStream_t st);
// Re-copy the halo rows' forcing from the plan's F (after rbf_set_forcing).
int pair_refresh_forcing(PairPlan* pp, cudaStream_t st);

}  // namespace rbf
