/*
 * gridse_b200.h -- C ABI of libgridse_b200.so, the B200-native (sm_100a) engine
 * behind the multi-area WLS Gauss-Newton solve path.
 *
 * The reference (pure Python, /root/reference/pkg/src/gridse) has no FFI; its
 * boundary for this path is a set of Python callables.  Each entry point below
 * names the reference callable it stands behind (file:line under
 * pkg/src/gridse); the Python shim in paper_2604_23175_b200/ keeps the
 * reference signatures and forwards to these symbols through ctypes.
 *
 * Conventions
 *   - plain C types only; every array argument is a host pointer unless its
 *     name ends in _dev (device pointer, e.g. torch tensor data_ptr()).
 *   - int return: 0 = ok, <0 = error code (GSE_E_*); details via gse_last_error.
 *   - one plan = one CUDA device = one host thread at a time; plans are
 *     independent (reentrant across plans).  No exceptions cross the ABI.
 *   - the plan owns every device buffer it allocates; the caller owns the
 *     state vectors va_dev / vm_dev (float64, length n_bus).
 */
#ifndef GRIDSE_B200_H
#define GRIDSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSE_OK 0
#define GSE_E_INVALID -1     /* bad argument / inconsistent description          */
#define GSE_E_CUDA -2        /* CUDA runtime failure (message in gse_last_error)  */
#define GSE_E_NOT_SPD_AREA -3     /* area interior block lost positive definiteness  */
#define GSE_E_NOT_SPD_BOUNDARY -4 /* reduced boundary system not positive definite   */
#define GSE_E_NO_DEVICE -5   /* no CUDA device: there is no CPU fallback           */

typedef struct gse_plan gse_plan;

/* Problem description: network model, measurement set, partition and variable maps.
 * Mirrors the inputs of solve_multiarea(net, ms, part, maps) -- solver.py:204-234,
 * with build_variable_maps' output (partition.py:478-538) passed as flat arrays. */
typedef struct {
    int32_t n_bus, n_branch, n_rows, n_areas, n_gamma, slack;
    /* Ybus CSR, sorted columns, structural diagonal (network.py:191-208) */
    const int32_t *y_ptr, *y_idx;
    const double *y_g, *y_b;
    /* branches: endpoints + two-port admittances [n_branch][8] =
     * (ff.re ff.im ft.re ft.im tf.re tf.im tt.re tt.im)  (network.py:65-78) */
    const int32_t *br_from, *br_to;
    const double *br_y;
    /* measurement rows in global row order (measurement.py:92-122) */
    const int32_t *m_type, *m_target;
    const double *m_z, *m_w;
    /* partition + maps: per area a, CSR-style slices (ptr arrays have n_areas+1 entries) */
    const int32_t *area_of_bus;
    const int32_t *ia_ptr, *ia_bus;   /* interior angle buses   (slot order of x_i[:na]) */
    const int32_t *im_ptr, *im_bus;   /* interior magnitude buses                         */
    const int32_t *ba_ptr, *ba_bus;   /* local boundary angle buses (slack excluded)      */
    const int32_t *bm_ptr, *bm_bus;   /* local boundary magnitude buses                   */
    const int32_t *sel_ptr, *sel;     /* boundary_selector: local boundary slot -> x_Gamma slot */
    /* x_Gamma layout (BoundaryOrdering, partition.py:35-62): bus and quantity (0=va,1=vm) per slot */
    const int32_t *gamma_bus, *gamma_quant;
} gse_problem_desc;

/* Build-time options. */
typedef struct {
    int32_t device;          /* CUDA device ordinal                                        */
    int32_t backend_dense;   /* 1: SolverConfig.backend == "dense" (solver.py:49,61-63)    */
    int32_t leaf_buses;      /* nested-dissection leaf size in buses (0 = default 48)       */
    int32_t max_pivots;      /* front pivot-block width, 32 or 64 (0 = default 64)          */
    int32_t rank, world;     /* area sharding: this process / number of processes           */
    const int32_t *area_rank;/* [n_areas] owner rank per area, NULL = all on rank 0          */
    int32_t persistent;      /* gse_solve scheduler: 0 auto (persistent dataflow kernel on single-rank plans),
                              * 1 persistent, 2 level launches captured in a CUDA graph             */
    int32_t tile_rows;       /* update-row chunk per task, multiple of 8, <= 96 (0 = default: 32 up to 30k buses, else 48) */
    int32_t boundary_mode;   /* boundary factorisation: 0 auto, 1 dense chain (dense_cholesky_solve), 2 block-sparse tree */
    void *stream;            /* cudaStream_t every kernel / copy of the plan is enqueued on; NULL = a stream of its own */
    int32_t max_ctas;        /* cap on the CTAs of the persistent kernel (0 = every resident slot of the device);
                              * rank plans that share one GPU must fit side by side                          */
} gse_options;

typedef struct {
    int32_t max_outer_iterations;  /* SolverConfig.max_outer_iterations (solver.py:45) */
    double convergence_tol;        /* SolverConfig.convergence_tol      (solver.py:47) */
    int32_t time_phases;           /* 1: fill gse_report.phase_s from CUDA events       */
} gse_config;

typedef struct {
    int32_t iterations, converged;
    double objective;              /* J(x) at the returned state (solver.py:100-103)   */
    double delta_inf[64];          /* per-iteration stacked update infinity norm        */
    /* seconds: assembly, local_condense, boundary_assemble, boundary_solve, recovery
     * (solver.py:36), then the whole GN loop */
    double phase_s[5];
    double loop_s;                 /* host wall clock around the loop                   */
    double gpu_s;                  /* CUDA-event time on the plan's stream, same region */
} gse_report;

typedef struct {
    int32_t code;      /* GSE_E_* */
    int32_t area;      /* failing area (GSE_E_NOT_SPD_AREA), else -1 */
    int32_t pivot;     /* area: original interior variable index; boundary: x_Gamma slot */
    char message[200];
} gse_error;

/* ---- plan lifetime --------------------------------------------------------------- */
/* Symbolic analysis (templates, slot map, ordering, fronts) + device upload; once.
 * Stands behind build_patterns (assembly.py:172-400) and symbolic_analyze
 * (linalg.py:395-398) for every area.  *out is valid even on error (for
 * gse_last_error) unless allocation itself failed. */
int gse_plan_create(const gse_problem_desc *desc, const gse_options *opt, gse_plan **out);
void gse_plan_destroy(gse_plan *plan);
const gse_error *gse_last_error(const gse_plan *plan);
/* Mask / unmask = weight refresh only (measurement.py:404-421); no re-analysis. */
int gse_set_weights(gse_plan *plan, const double *w);
int gse_set_measurements(gse_plan *plan, const double *z);
/* The same refresh from caller-owned pinned host memory: asynchronous copies on the plan's stream, no
 * staging; either pointer may be NULL (w_pinned == z_pinned + n_rows: one copy for both).  The buffers must stay
 * unchanged until the next solve returns. */
int gse_set_rows_pinned(gse_plan *plan, const double *z_pinned, const double *w_pinned);

/* ---- the solve (solve_multiarea, solver.py:204-346) -------------------------------- */
/* Runs the GN loop on the device from the state in va_dev / vm_dev (the shim writes
 * the flat start); per iteration only the convergence scalar + failure flag cross to
 * the host.  On GSE_E_NOT_SPD_* the report is partially filled. */
int gse_solve(gse_plan *plan, const gse_config *cfg, double *va_dev, double *vm_dev,
              gse_report *report);
/* The same solve with its transfers folded into the one enqueue: init_dev = start state (va | vm, 2 n_bus doubles on
 * the device, e.g. the flat start of solver.py:236 kept resident) copied into va_dev / vm_dev first, or NULL;
 * out_pinned = pinned host buffer that receives the final (va | vm), or NULL.  One host synchronisation per solve. */
int gse_solve_io(gse_plan *plan, const gse_config *cfg, const double *init_dev, double *va_dev, double *vm_dev,
                 double *out_pinned, gse_report *report);
/* One outer iteration (used when the caller wants on_iteration callbacks, solver.py:334). */
int gse_iterate(gse_plan *plan, double *va_dev, double *vm_dev, double *delta_inf);
/* One inner GN step of every owned area with the boundary state held fixed: SolverConfig.inner_gn_steps > 1
 * (solver.py:253-260: fused_accumulate, numeric_refactor, cache.solve(b_i), apply_interior_delta).
 * *delta_inf = max |delta x_i| of the step. */
int gse_inner_step(gse_plan *plan, double *va_dev, double *vm_dev, double *delta_inf);

/* ---- phase-level entry points (component parity + the multi-GPU driver) ------------ */
/* fused_accumulate for every owned area (assembly.py:486-524). */
int gse_phase_assemble(gse_plan *plan, const double *va_dev, const double *vm_dev);
/* numeric_refactor + schur_condense for every owned area (linalg.py:401-424):
 * leaves packed (S_b, b_hat) of each area in the exchange buffer. */
int gse_phase_condense(gse_plan *plan);
/* assemble_boundary in area order + dense_cholesky_solve (solver.py:106-119, linalg.py:46-61);
 * coordinator rank only. */
int gse_phase_boundary(gse_plan *plan);
/* interior_recover + apply_interior_delta + BoundaryOrdering.apply_delta + the
 * stacked infinity norm (linalg.py:427-434, partition.py:59-62,113-116, solver.py:328-333). */
int gse_phase_recover(gse_plan *plan, double *va_dev, double *vm_dev, double *delta_inf);
/* The same phases, enqueue-only (no host synchronisation, no failure check): with gse_options.stream set
 * to the caller's stream, collectives enqueued there between the calls are ordered by the stream.
 * gse_phase_recover_async leaves [max |dx|, failed ? 1 : 0] in gse_status_dev for one MAX all-reduce;
 * after a reduced failure flag, gse_check on the owning rank names the area / pivot. */
int gse_phase_local_async(gse_plan *plan, const double *va_dev, const double *vm_dev);
int gse_phase_boundary_async(gse_plan *plan);
int gse_phase_recover_async(gse_plan *plan, double *va_dev, double *vm_dev);
/* Poll the device failure flag after a phase: 0 or GSE_E_NOT_SPD_*. */
int gse_check(gse_plan *plan);
/* objective(ms, state) (solver.py:100-103). */
int gse_objective(gse_plan *plan, const double *va_dev, const double *vm_dev, double *j_out);

/* ---- result readback in the reference's layouts (component parity tests) ----------- */
/* sizes: out[0]=n_i out[1]=n_b out[2]=nnz(G_ii) out[3]=nnz(G_ib) out[4]=rows out[5]=slots
 *        out[6]=fronts out[7]=factor nnz (dense panels) */
int gse_area_dims(const gse_plan *plan, int32_t area, int32_t *out);
/* CSR patterns of G_ii / G_ib in the reference's layout (AssemblyPattern, assembly.py:133-137). */
int gse_area_pattern(const gse_plan *plan, int32_t area, int32_t *ii_ptr, int32_t *ii_idx,
                     int32_t *ib_ptr, int32_t *ib_idx);
/* AreaNormalBlocks values after gse_phase_assemble: data_ii[nnz_ii], data_ib[nnz_ib],
 * g_bb[n_b*n_b] row-major full, b_i[n_i], b_b[n_b] (assembly.py:32-53).  Host outputs. */
int gse_area_blocks(gse_plan *plan, int32_t area, double *data_ii, double *data_ib,
                    double *g_bb, double *b_i, double *b_b);
/* The materialised template layer of an area after gse_phase_assemble -- what the reference's explicit oracle path
 * builds its JacobianTriplets from (explicit_assemble, assembly.py:531-560): rows[n_rows] global row ids,
 * slot_ptr[n_rows + 1], slot_var[n_slots] local variable per slot (x_i slots, then n_i + local boundary slot),
 * g[n_slots] = dh/dx per slot, wr[n_rows] = w (z - h).  Sizes: gse_area_dims out[4], out[5].  Host outputs. */
int gse_area_templates(gse_plan *plan, int32_t area, int32_t *rows, int32_t *slot_ptr, int32_t *slot_var,
                       double *g, double *wr);
/* SchurResult after gse_phase_condense: s_b[n_b*n_b] full symmetric, b_hat[n_b] (linalg.py:38-43). */
int gse_area_schur(gse_plan *plan, int32_t area, double *s_b, double *b_hat);
/* Interior update of the last gse_phase_recover, in x_i slot order (solver.py:269). */
int gse_area_delta(gse_plan *plan, int32_t area, double *dx_i);
/* BoundarySystem after gse_phase_boundary: s_gamma[n_gamma^2], b_gamma, delta_x_gamma (solver.py:91-97). */
int gse_boundary_system(gse_plan *plan, double *s_gamma, double *b_gamma, double *dx_gamma);
/* Override the boundary increment before gse_phase_recover (interior_recover with a
 * caller-supplied delta_xb, linalg.py:427). */
int gse_set_boundary_delta(gse_plan *plan, const double *dx_gamma);

/* ---- standalone linear algebra on caller-supplied matrices (reference linalg.py) ------------------
 * A matrix plan is a one-area Schur-mode plan whose blocks come from the caller instead of from
 * measurement templates; it reuses the plan type (gse_plan_destroy, gse_last_error, gse_area_schur). */
/* symbolic_analyze (linalg.py:395-398) for G_ii [n_i x n_i, CSR, sorted columns, structurally
 * symmetric] with the coupling pattern of G_ib [n_i x n_b CSR] that schur_condense will be given.
 * opt->backend_dense = 1: one dense chain in natural order (dense_cholesky_solve, linalg.py:46-61). */
int gse_matrix_plan_create(int32_t n_i, int32_t n_b, const int32_t *ii_ptr, const int32_t *ii_idx,
                           const int32_t *ib_ptr, const int32_t *ib_idx, const gse_options *opt,
                           gse_plan **out);
/* Values in the reference's block layout (AreaNormalBlocks, assembly.py:32-53): data_ii / data_ib
 * aligned with the CSR patterns, g_bb row-major n_b x n_b, b_i, b_b.  NULL = zeros.  Host arrays. */
int gse_matrix_set_values(gse_plan *plan, const double *data_ii, const double *data_ib,
                          const double *g_bb, const double *b_i, const double *b_b);
/* numeric_refactor + schur_condense (linalg.py:401-424); then gse_area_schur(plan, 0, ...) returns
 * (S_b, b_hat).  GSE_E_NOT_SPD_AREA with the original pivot index on a non-positive pivot. */
int gse_matrix_condense(gse_plan *plan);
/* interior_recover (linalg.py:427-434): dx_i = G_ii^-1 (b_i - G_ib dx_b) with the factor and b_i of the
 * last gse_matrix_condense; dx_b NULL = zeros (a plain cache.solve(b_i)). */
int gse_matrix_recover(gse_plan *plan, const double *dx_b, double *dx_i);
/* SparseCholeskyCache.forward / .backward (linalg.py:340-383), in this factor's coordinates.  perm[e] =
 * original index of elimination position e (cache.perm).  gse_matrix_forward_get: y = L^-1 P b of the b_i given to
 * the last gse_matrix_set_values + gse_matrix_condense (the right-hand side rides through the factorisation as
 * one extra row of every front).  gse_matrix_backward: x = P^T L^-T y, x in original order.  Host arrays [n_i]. */
int gse_matrix_perm(const gse_plan *plan, int32_t *perm);
int gse_matrix_forward_get(gse_plan *plan, double *y);
int gse_matrix_backward(gse_plan *plan, const double *y, double *x);
/* assemble_boundary (solver.py:106-119) for caller-supplied Schur blocks: s_b = the areas' n_b x n_b
 * blocks concatenated, b_hat likewise, sel_ptr / sel the boundary selectors.  Host in, host out. */
int gse_assemble_boundary(int32_t n_gamma, int32_t n_areas, const int32_t *sel_ptr, const int32_t *sel,
                          const double *s_b, const double *b_hat, double *s_gamma, double *b_gamma);

/* ---- multi-GPU exchange buffers ---------------------------- */
/* Device pointer + length (doubles) of the packed per-area (S_b | b_hat) exchange buffer;
 * area a occupies [off[a], off[a+1]) with off = gse_exchange_offsets (n_areas+1 entries);
 * areas of one rank are contiguous. */
double *gse_exchange_buffer_dev(gse_plan *plan, int64_t *n_doubles);
int gse_exchange_offsets(const gse_plan *plan, int64_t *off);
/* Device pointer to delta_x_gamma (n_gamma doubles) -- broadcast from the coordinator. */
double *gse_boundary_delta_dev(gse_plan *plan);
/* Device pointer to [delta_inf, failure code] as two doubles for a MAX all-reduce. */
double *gse_status_dev(gse_plan *plan);

/* ---- peer-linked multi-rank solve: the exchanges INSIDE the persistent kernel, over peer memory -------
 * One process (or plan) per GPU; every rank runs the whole GN loop in one launch of its own.  The two
 * exchange points of the reference loop (solver.py:277-298 gather of the areas' Schur blocks, 318-326
 * broadcast of delta_x_Gamma) and the convergence scalar (solver.py:328-338) happen inside the kernels:
 * area roots of rank r store (S_b | b_hat) straight into the coordinator's update storage and bump its
 * completion counters; the coordinator's boundary back-substitution tasks store their pivots' share of
 * delta_x_Gamma into every rank's solution vector; every rank max-merges its norm / failure code into
 * every rank's copy.  No collective, no host round trip inside the loop; results are bit-identical to
 * the single-rank solve.  Setup: every rank fills a gse_peer_info, the records are exchanged by the host
 * layer (torch.distributed all_gather of the raw bytes), every rank links.  Ranks in other processes are
 * mapped with CUDA IPC, rank plans of the same process (tests; one process driving several GPUs) with
 * their device addresses + cudaDeviceEnablePeerAccess.  At most 8 ranks. */
typedef struct {
    int32_t rank, world, n_gamma_fronts, device;
    int64_t pid;                 /* exporting process                                                  */
    uint64_t ubuf, xsol, sync;   /* device addresses (exporting process) of the update storage, the
                                  * solution vector and the sync block                                  */
    uint8_t ipc[3][64];          /* cudaIpcMemHandle_t of the allocations that hold them                */
    int64_t ipc_off[3];          /* their byte offsets inside those allocations                         */
} gse_peer_info;
int gse_peer_info_get(gse_plan *plan, gse_peer_info *out);
/* all: world records ordered by rank (this rank's own included).  After a successful link gse_solve runs
 * the peer-linked persistent kernel; gse_report.objective is NaN (J needs the merged state: gse_objective). */
int gse_peer_link(gse_plan *plan, const gse_peer_info *all);
/* Before EVERY gse_solve of a linked plan: clears this rank's sync block and waits for it; then the host
 * layer barriers the ranks (no rank may launch before every block is clear), then gse_solve. */
int gse_peer_solve_prepare(gse_plan *plan);

/* ---- partitioner passes on the host (no device involved) ---------------------------------
 * One attempt of partition_network (reference partition.py:373-403; passes partition.py:198-365:
 * farthest-point seeds, multi-source growth, re-centring, balance moves, cascade, cut thinning) on the
 * bus graph given as the CSR of net.neighbors(u) (same neighbor order) and the branch end arrays.
 * first_seed is the bus numpy's default_rng(seed).integers(n) drew.  Returns 0 and area_out[n], or 1
 * with info = {starved area, its size, buses left unassigned} (the caller raises PartitionError). */
int gse_partition_attempt(int32_t n_bus, const int32_t *nbr_ptr, const int32_t *nbr_idx, int32_t n_branch,
                          const int32_t *br_from, const int32_t *br_to, int32_t k, int32_t first_seed,
                          int32_t *area_out, int32_t *info);
/* The cut-thinning pass alone, in place (merged variants of a finer attempt). */
int gse_partition_thin_cuts(int32_t n_bus, const int32_t *nbr_ptr, const int32_t *nbr_idx, int32_t n_branch,
                            const int32_t *br_from, const int32_t *br_to, int32_t k, int32_t *area_inout);

/* ---- introspection ------------------------------------------------------------------ */
/* stats[0]=kernel launches of the last gse_solve/gse_iterate, [1]=fronts, [2]=levels,
 * [3]=tasks, [4]=max front order, [5]=factor doubles, [6]=update doubles,
 * [7]=pair contributions, [8]=slots, [9]=algorithmic bytes of the assembly kernels per
 * iteration (SURVEY.md section 8(d) A_min), [10]=dense flops per iteration (fronts),
 * [11]=launches per iteration. */
int gse_plan_stats(const gse_plan *plan, double *stats, int32_t n);
/* Item layout of one iteration of the persistent kernel: out[0..4] = eval, accumulate, front, backward,
 * update items; out[5] = resident CTAs, out[6] = dynamic shared memory, out[7] = 1 if gse_solve uses it. */
int gse_solve_layout(const gse_plan *plan, int32_t *out);
/* Debug: per-item timeline of the persistent kernel (tools/persist_trace.py).  enable = 1 arms tracing for
 * the next solves; enable = 0 copies [items][32] words to out and disarms.  Returns items per iteration. */
int gse_debug_trace(gse_plan *plan, int enable, unsigned long long *out, int64_t max_words);
/* The CUDA stream (cudaStream_t) every kernel of the plan is launched on. */
void *gse_stream(gse_plan *plan);
const char *gse_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GRIDSE_B200_H */
