/*
 * rbffd_b200.h -- C ABI of the B200-native explicit RBF-FD time loop.
 *
 * This library replaces, for one NVIDIA B200 (sm_100a), the hot path of the
 * reference package `rbffd` (arXiv 2107.03632, /root/reference/pkg):
 *
 *   rbffd.solver._step_kernel   pkg/src/rbffd/solver.py:294-311  (numba, the update)
 *   rbffd.solver.run_time_loop  pkg/src/rbffd/solver.py:168-236  (the step loop,
 *                               flag check :200-206, residual :208-211,
 *                               swap/copy-back :212-215, steady break :216-217)
 *   rbffd.solver.explicit_step  pkg/src/rbffd/solver.py:141-165  (one step)
 *
 * The reference has no FFI: its boundary is the Python call
 *   _step_kernel(u1, u2, interior, rows, weights, f_int, dt, chunk, flags)
 * (solver.py:294-295).  The functions below are the entry points a ctypes
 * binding of that call binds.  Plain C types only.
 *
 * Arithmetic contract (bitwise parity with the reference): per interior row k,
 *     acc = 0.0;  for j in 0..n-1: acc = acc + w[k,j]*u1[rows[k,j]]   (serial j)
 *     u2[interior[k]] = u1[interior[k]] + dt*(f_int[k] + acc)
 * every product and sum separately rounded (no FMA), exactly as the numba
 * kernel compiles (solver.py:304-307).
 *
 * Status codes (int return of every call):
 *     RBF_OK 0, RBF_ERR_CUDA 1, RBF_ERR_PARAM 2, RBF_ERR_INSTABILITY 4,
 *     RBF_ERR_TIMEOUT 5, RBF_ERR_ILLCOND 6 (weight assembly only).
 * They map onto the reference exceptions (pkg/src/rbffd/errors.py):
 *     2 -> ParameterError (:4), 4 -> InstabilityError(step, max_abs) (:21-27),
 *     5 -> SteadyStateTimeout(steps, residual) (:30-36), 6 -> after the
 *     caller's exact condition check of the flagged rows,
 *     DegenerateStencilError(node_index, position) (:8-18).
 * rbf_last_error() returns a thread-local message for the last failure.
 *
 * Calls are synchronous.  A plan is not thread-safe: one plan per host thread.
 */
#ifndef RBFFD_B200_H
#define RBFFD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBF_OK 0
#define RBF_ERR_CUDA 1
#define RBF_ERR_PARAM 2
#define RBF_ERR_INSTABILITY 4
#define RBF_ERR_TIMEOUT 5
#define RBF_ERR_ILLCOND 6

/* plan flags */
#define RBF_RENUMBER_MORTON 0x1u  /* locality renumbering of interior rows (needs positions) */
#define RBF_NO_RESIDENT 0x2u      /* never use an on-chip loop (single-CTA, cluster or grid-resident):
                                     always the streaming step */
#define RBF_NO_PDL 0x4u           /* disable programmatic dependent launch between steps */
#define RBF_STREAM_LDG 0x8u       /* streaming step with plain loads instead of the TMA ring */
#define RBF_NO_CLUSTER 0x10u      /* small problems: single-CTA resident loop, not the cluster loop */
#define RBF_NO_IDX16 0x20u        /* keep int32 node ids in the streamed step (no 16-bit windows) */
/* 0x40u: reserved (was an opt-in dataflow loop, measured slower and removed) */
#define RBF_NO_PAIR 0x80u         /* fixed-step runs one step per launch (no two-step tile kernel) */
#define RBF_PAIR 0x100u           /* two-step tile kernel for fixed-step runs at any size (default:
                                     only up to N_i*n = 1e6, where it is measured faster) */
#define RBF_NO_PERSIST 0x400u     /* streaming runs: one graph-captured launch per step instead of
                                     the persistent loop (one cooperative launch per run) */
#define RBF_ACCEPT_ILLCOND 0x200u /* rbf_plan_create_assembled: accept row status 1 (the caller has
                                     checked those rows' exact condition); status 2 still fails */

/* run modes (SolveConfig.mode, solver.py:53) */
#define RBF_MODE_FIXED 0
#define RBF_MODE_STEADY 1

typedef struct rbf_plan rbf_plan;

/*
 * Build a plan on `device`: pack the reference's ShapeStore into the
 * sliced-transposed ELL layout (SELL-32, fp64 weights, int32 node ids) and
 * upload it.  Replaces the per-call array prep of run_time_loop
 * (solver.py:181-190) and the layout of ShapeStore (weights.py:71-86) +
 * StencilSet (neighborhoods.py:25-35).
 *
 *   N          total node count (NodeSet.n_total, geometry.py:53-55)
 *   N_i        interior row count (ShapeStore.n_rows, weights.py:84-86)
 *   n          support size (StencilSet.n)
 *   interior   [N_i]    ShapeStore.interior_nodes (distinct node ids)
 *   rows       [N_i*n]  stencils.neighbors[interior], row-major (solver.py:182)
 *   weights    [N_i*n]  ShapeStore.weights, row-major
 *   f_int      [N_i]    forcing at interior nodes (solver.py:184); may be NULL (zero forcing,
 *                       set later with rbf_set_forcing)
 *   positions  [N*2]    node coordinates, only read with RBF_RENUMBER_MORTON (may be NULL)
 * The caller keeps ownership of every host array.
 */
int rbf_plan_create(rbf_plan** out, int64_t N, int64_t N_i, int32_t n,
                    const int64_t* interior, const int64_t* rows,
                    const double* weights, const double* f_int,
                    const double* positions, int32_t device, uint32_t flags);

/*
 * Weight assembly on the device: restates
 * rbffd.weights._weights_batch (weights.py:218-259) -- PHS r^3 + monomials of
 * `degree` (<= 6), support shifted to rows[k*n] and scaled by its radius, one
 * saddle solve per row (Gaussian elimination with partial pivoting, one warp
 * per system), weights rescaled by 1/radius^2.  Agrees with the reference's
 * LAPACK solve to rounding (pinned by polynomial reproduction, like
 * test_weights.py:51-104), not bit for bit.
 *
 * Condition guard (weights.py:29, :183-192, :250-258 reject a stencil whose
 * np.linalg.cond, the 2-norm condition, exceeds COND_LIMIT = 1e14).  The
 * saddle matrix K is symmetric, so kappa_2 <= kappa_1 <= S kappa_2 (S = n+M);
 * from its LU factors the device estimates kappa_1 (Hager/Higham lower
 * bound) and writes row_status[k] (optional, N_i bytes):
 *     0  estimate <= 1e10 (typical stencils: 1e3-1e7): accepted;
 *     1  estimate in (1e10, S*1e14]: the caller must check the exact 2-norm
 *        condition of that row (np.linalg.cond) against 1e14;
 *     2  zero pivot, non-finite weights, or estimate > S*1e14 (then
 *        kappa_2 > 1e14 for certain): degenerate.
 * Returns RBF_OK when every row has status 0; RBF_ERR_ILLCOND with *bad_row
 * = the first flagged row otherwise (weights of status-0/1 rows are valid).
 */
int rbf_assemble_weights(const double* positions, int64_t N, const int64_t* rows, int64_t N_i,
                         int32_t n, int32_t degree, double* weights_out, int64_t* bad_row,
                         uint8_t* row_status, int32_t device);

/*
 * Exact k-nearest-neighbour supports on the device (
 * rbffd.neighborhoods.build_stencils, neighborhoods.py:51-94): row i of
 * neighbors_out[N*n] lists the n nodes nearest to node i sorted by
 * (distance, index) with distance = sqrt(dx*dx + dy*dy) in IEEE double --
 * the reference's tie rule (tests/oracles.py:16-24).  1 <= n <= min(N, 128).
 */
int rbf_knn(const double* positions, int64_t N, int32_t n, int64_t* neighbors_out, int32_t device);

/* rbf_knn for a subset of query nodes (a rank's own rows in a partitioned
 * setup): row q of neighbors_out[n_query*n] lists the n nearest of ALL N
 * nodes to node query_ids[q], same order and tie rule. */
int rbf_knn_subset(const double* positions, int64_t N, int32_t n, const int64_t* query_ids, int64_t n_query,
                   int64_t* neighbors_out, int32_t device);

/*
 * The reference's advancing-front node set on the unit disk (SURVEY.md §8f
 * row 4; rbffd.geometry.generate_unit_disk_nodes, geometry.py:105-198),
 * bit-identical: same MT19937 candidate-angle stream, same acceptance order,
 * same IEEE operations.  Host code (the algorithm is sequential by
 * construction; a parallel acceptance rule would change the node set).
 * seed_key[key_len] are the 32-bit little-endian words of |seed| as CPython's
 * random.seed(int) uses them (one zero word for seed 0).  On success
 * *positions_out is a malloc'd [N*2] array (boundary ring first, then the
 * interior in acceptance order) to be released with rbf_free_host.
 */
int rbf_generate_unit_disk_nodes(double h, const uint32_t* seed_key, int32_t key_len,
                                 double** positions_out, int64_t* n_total, int64_t* n_boundary);
void rbf_free_host(void* p);

/* rbf_plan_create with the weights assembled on the device straight into the
 * SELL layout (the host never holds them; positions are required).  Same
 * condition guard as rbf_assemble_weights: any flagged row fails the call
 * with RBF_ERR_ILLCOND and fills row_status (optional, N_i bytes); with
 * RBF_ACCEPT_ILLCOND in `flags` status-1 rows are accepted (the caller has
 * checked them exactly), status-2 rows still fail. */
int rbf_plan_create_assembled(rbf_plan** out, int64_t N, int64_t N_i, int32_t n, int32_t degree,
                              const int64_t* interior, const int64_t* rows,
                              const double* positions, const double* f_int, int32_t device,
                              uint32_t flags, uint8_t* row_status);

/* max_k sum_j |w_kj| of the plan's weights (stability_bound = 2 / this,
 * solver.py:249-254), for plans whose weights never left the device.  Each
 * row is summed in numpy's pairwise order (np.abs(w).sum(axis=1)), so the
 * result has the reference's bits. */
int rbf_plan_weight_row_sum_max(rbf_plan* plan, double* out);

/*
 * Plan files (replacing the reference's CSV shape /
 * stencil files, weights.py:209-215, neighborhoods.py:104-122, for the hot
 * path): the packed device layout -- SELL weights and ids, forcing, 16-bit id
 * windows, renumbering maps -- written once and loaded straight back into
 * HBM, skipping validation, renumbering, packing and id compression.  A
 * loaded plan runs bit-identically to the plan that was saved.  `path` must
 * be a regular (seekable) file: sections move through pinned staging chunks
 * with parallel positional reads / writes (RBF_ERR_PARAM otherwise).
 */
int rbf_plan_save(const rbf_plan* plan, const char* path);
int rbf_plan_load(rbf_plan** out, const char* path, int32_t device, uint32_t flags);

/* Page-locked host memory for the field-sized arrays of a call (forcing,
 * start field, exact solution, result field): transfers from / to it skip
 * the pinned staging copy every other host pointer goes through. */
int rbf_host_alloc(int64_t bytes, void** out);
void rbf_host_free_pinned(void* p);

/* Replace the per-row forcing (explicit_step's f[interior], solver.py:156). */
int rbf_set_forcing(rbf_plan* plan, const double* f_int);

/* Upload the full field u[N] (original node order) into both device buffers
 * (run_time_loop: u1 = apply_dirichlet(...); u2 = u1.copy(), solver.py:186-187). */
int rbf_set_field(rbf_plan* plan, const double* u_host);

/* Download the current field u[N] in original node order.  After
 * RBF_ERR_INSTABILITY this is the u2 of the failing step (solver.py:201). */
int rbf_get_field(rbf_plan* plan, double* u_host);

/*
 * error_norms (solver.py:239-246) of the current field against `exact`
 * (host [N], original node order, e.g. closed_form_solution(positions)):
 *   linf = max|u - exact|, l2 = sqrt(mean((u - exact)**2))
 * with numpy's bits: the differences and squares are elementwise IEEE, the
 * max is order-free, and the sum follows numpy's pairwise summation tree
 * (128-element blocks with 8 accumulators, splits at n/2 rounded down to a
 * multiple of 8; numpy/_core/src/umath/loops_utils.h.src) -- block sums on
 * the device, the tree above them on the host.
 */
int rbf_error_norms(rbf_plan* plan, const double* exact, double* linf, double* l2);

/*
 * The time loop of run_time_loop (solver.py:191-225), on the device.
 *   mode      RBF_MODE_FIXED: `steps` steps, residual of the last step only
 *             RBF_MODE_STEADY: up to `max_steps` steps, residual every step,
 *             stop when residual <= tol
 *   copy_back 0 swap buffers (solver.py:215), 1 copy u2 into u1 (solver.py:213)
 * Outputs: steps_done, residual (max|u2-u1|/dt, valid when *has_residual),
 *   bad_step (first step with a non-finite value, -1 if none), device_seconds
 *   (CUDA-event time of the loop).
 * Returns RBF_ERR_INSTABILITY (bad_step set) or RBF_ERR_TIMEOUT like the
 * reference raises InstabilityError / SteadyStateTimeout.
 */
int rbf_run(rbf_plan* plan, double dt, int64_t steps, int32_t mode, double tol,
            int64_t max_steps, int32_t copy_back, int64_t* steps_done,
            double* residual, int32_t* has_residual, int64_t* bad_step,
            double* device_seconds);

/* One explicit step on the resident field (explicit_step, solver.py:141-165);
 * RBF_ERR_INSTABILITY if any updated value is non-finite. */
int rbf_step(rbf_plan* plan, double dt);

/*
 * Literal drop-in for the numba kernel's call signature (solver.py:294-311):
 * host arrays in, u2[interior] and flags[ceil(N_i/chunk)] out.  Uploads,
 * runs one step and downloads every call (slow by construction; the plan API
 * above is the fast path).
 */
int rbf_step_kernel(const double* u1, double* u2, int64_t N,
                    const int64_t* interior, const int64_t* rows,
                    const double* weights, const double* f_int, int64_t N_i,
                    int32_t n, double dt, int64_t chunk, uint8_t* flags,
                    int32_t device);

/* Introspection for benchmarks / tests. */
typedef struct rbf_plan_info {
  int64_t N, N_i;
  int32_t n;
  int32_t device;
  int32_t resident;        /* 1: whole loop runs on-chip in one CTA */
  int32_t renumbered;      /* 1: rows/nodes permuted (field order restored on get/set) */
  int32_t kernel_n;        /* compile-time width of the chosen step kernel (0: generic) */
  int32_t grid, block;     /* streaming kernel launch geometry */
  int32_t variant;         /* 0 resident loop (1 CTA), 1 LDG streaming step, 2 TMA-ring
                              streaming step, 3 cluster-resident loop (DSMEM halo), 4 grid-resident
                              loop (rows in every SM's shared memory, one cooperative launch) */
  int32_t index_bits;      /* 32, or 16: two-window 16-bit ids streamed by the TMA step */
  int64_t device_bytes;    /* device memory held by the plan */
  int64_t bytes_per_step;  /* algorithmic HBM bytes per step: N_i*(12n+24) */
  int64_t launches;        /* kernel launches issued by this plan so far */
  int64_t stream_bytes_per_step; /* bytes the step actually streams (<= bytes_per_step with 16-bit ids) */
  int32_t pair;            /* 1: fixed-step runs advance two steps per launch (tile-local
                              temporal blocking, bitwise identical) */
  int32_t pair_tiles;      /* its row tiles */
  int64_t pair_halo_rows;  /* halo entries over all tiles (rows recomputed per launch) */
  int32_t persist;         /* 1: streaming runs (variant 2) go through the persistent loop, one
                              cooperative launch per run (RBF_NO_PERSIST: one launch per step) */
  int32_t persist_grid;    /* its CTAs */
} rbf_plan_info;

int rbf_plan_get_info(const rbf_plan* plan, rbf_plan_info* info);

/* Time `iters` bare step launches (fixed mode, no residual) with CUDA events
 * on the plan's stream; returns the mean per-launch duration in seconds.
 * Used by bench.py for the roofline of the dominant kernel. */
int rbf_time_step_kernel(rbf_plan* plan, double dt, int32_t iters,
                         double* seconds_per_launch);

/* ---- node-partitioned multi-GPU loop ---------------------
 * A part is an ordinary plan whose local numbering is
 *   [replicated boundary nodes | halo, grouped by owner | owned rows]
 * (paper_2107_03632_b200/multigpu.py:partition).  The reference has no
 * multi-device path; these entry points add it.
 *
 * rbf_plan_set_halo: exchange lists of one part.  For peer i: send
 * send_counts[i] owned values (local ids, concatenated in send_idx) and
 * receive recv_counts[i] values into u[recv_offsets[i] ...] (its halo slice).
 * rbf_group_create: nccl_uid != NULL -> one part per process, halos over NCCL
 * (uid from rbf_nccl_unique_id on rank 0, broadcast by the caller); NULL ->
 * all n_local parts live in this process and halos move by device copies.
 * rbf_group_run: the loop of rbf_run over all parts: pack, exchange, step,
 * all-reduce(max) of {residual bits, non-finite flag}, decide; bitwise equal
 * to a single plan's run.  Fields are read / written per part with
 * rbf_set_field / rbf_get_field (local numbering). */
typedef struct rbf_group rbf_group;
int rbf_nccl_unique_id(char* out128);
int rbf_plan_set_halo(rbf_plan* plan, int32_t n_peers, const int32_t* peers,
                      const int64_t* send_counts, const int64_t* send_idx,
                      const int64_t* recv_counts, const int64_t* recv_offsets);
int rbf_group_create(rbf_group** out, int32_t n_local, rbf_plan* const* plans,
                     const int32_t* part_ids, const char* nccl_uid, int32_t rank,
                     int32_t nranks);
int rbf_group_run(rbf_group* group, double dt, int64_t steps, int32_t mode, double tol,
                  int64_t max_steps, int64_t* steps_done, double* residual,
                  int32_t* has_residual, int64_t* bad_step, double* device_seconds);
void rbf_group_destroy(rbf_group* group);

/*
 * Push-mode halo exchange for fixed-step runs (BASELINE.json north star (4),
 * "NCCL or P2P"; replaces pack + NCCL send/recv): after each step a small
 * kernel stores the owned values the neighbours read straight into their field
 * buffers (P2P stores over NVLink, CUDA IPC mappings between processes) and
 * publishes the arrival with a system-scope release store; the next step's
 * consumers wait (acquire) for their neighbours' arrivals.  Bitwise identical
 * to the NCCL path.  Steady-mode runs and failure replays keep the exact
 * per-step NCCL / copy path.
 *   rbf_group_push_local   parts of one process (one device): plain pointers
 *   rbf_group_push_export  one part per process: the blob (<= 1024 bytes) its
 *                          peers need -- IPC handles of its field buffers and
 *                          arrival counters, its halo slices per owner
 *   rbf_group_push_import  all ranks' blobs, `stride` bytes apart; every rank
 *                          must import before any rank runs (hold a barrier)
 *   rbf_group_push_mode    1 when the group's fast path pushes
 *   rbf_group_fused        1 when the last fixed-step fast run was ONE
 *                          cooperative launch of the partitioned persistent
 *                          loop: every local part's streaming loop on its own
 *                          CTA range, the halo pushes fused into the lanes
 *                          that compute the sent rows, a per-part grid
 *                          barrier and release/acquire arrival counters
 *                          between neighbours (RBFFD_PART_LOOP=0: the step +
 *                          push kernels of the graph path instead)
 */
int rbf_group_push_local(rbf_group* group);
int rbf_group_push_export(rbf_group* group, void* blob_out, int64_t capacity, int64_t* length);
int rbf_group_push_import(rbf_group* group, int32_t n_blobs, const void* blobs, int64_t stride);
int rbf_group_push_mode(const rbf_group* group);
int rbf_group_fused(const rbf_group* group);

/* Host-paced push mode: after every fixed-mode step (and its halo pushes)
 * the group synchronises its stream and calls fn(ctx) -- a barrier across
 * the ranks -- so no step kernel waits on a kernel of another process.  For
 * ranks that share one GPU (time-sliced contexts give no co-scheduling
 * guarantee), e.g. the cross-process test of the IPC push path; NULL turns
 * it off.  Fixed-step runs of groups without NCCL return each rank's own
 * residual / first bad step; the caller reduces them across ranks. */
int rbf_group_set_step_barrier(rbf_group* g, void (*fn)(void*), void* ctx);
int rbf_group_push_off(rbf_group* group);  /* back to pack + NCCL / copy (all ranks must agree) */

void rbf_plan_destroy(rbf_plan* plan);
const char* rbf_last_error(void);
int rbf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RBFFD_B200_H */
