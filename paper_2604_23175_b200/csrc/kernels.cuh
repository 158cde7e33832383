// kernels.cuh -- device program layout shared by kernels.cu and api.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gse {

// Template evaluation units (SoA, one thread per unit).
struct EvalProg {
    // network (read-only)
    const int32_t *y_ptr, *y_idx;
    const double *y_g, *y_b, *br_y;
    const double *z, *w;
    int32_t slack;
    int32_t n_vm, n_fl, n_inj;
    int32_t has_current;          // any current-magnitude row (types 7 / 8) in the plan
    const int32_t *vm_bus, *vm_row, *vm_slot;
    const int32_t *fl_branch, *fl_from, *fl_to, *fl_row, *fl_slot;
    const int32_t *inj_bus, *inj_rowp, *inj_rowq, *inj_slotp, *inj_slotq, *inj_nth;
    // outputs = the unified value array val = [(g, w*g) per slot, interleaved | wr]: per slot the partial
    // and weight * partial, per measurement row weight * residual
    double *g, *wr;
};

// One (front, row-chunk, col-chunk) task: everything the CTA needs, read with one coalesced load.
struct TaskRec {                                      // 128 bytes
    int32_t front, ci, cj, p, u1, T, nchild, child_off;
    int32_t reg[8];                                   // original-entry ranges (relative to gval_off): PP, IP, JP, tile
    int64_t gval_off, l_off, u_off;
    int32_t flags, dinv_off;                          // flags bit 0: tile read directly from the single child's U;
                                                      //       bit 1: the front has original entries (waits for the accumulation)
                                                      //       bit 2: area root of a non-coordinator rank -- its update matrix (S_b | b_hat)
                                                      //              goes straight into the coordinator's exchange buffer (peer memory)
    int32_t phase, kind, nch, area, level, pad[3];    // phase: 1 local_condense, 2 boundary_assemble, 3 boundary_solve
                                                      // kind: 0 fused, 1 panel, 2 update (front_body.cuh); nch: row chunks of the front
                                                      // area: owning area of the front (-1: boundary front)
};
// One child of a task (children that do not reach the task's regions are pruned on the host).
// front / need: dataflow dependency -- the child is complete when its counter reaches need per iteration.
// front < 0: the root of area -(front + 1), owned by another rank -- its tiles arrive over peer memory and are
// counted per area (CTR_AREA0).
struct ChildRec { int64_t u_off; int32_t rel_off, eP, bI, eI, bJ, eJ; int32_t front, need, pad[2]; };   // 48 bytes
// dep: nearest ancestor front with pivots (-1: none); need: forward tasks of the own front
// dep2 / early: fronts with several splits whose later splits (update rows 64 ...) only read solution entries of
// ancestors ABOVE the nearest one (its pivots are the first update rows): those splits wait for front dep2 instead and
// finish a level early; split 0 -- the only one that needs the nearest ancestor -- combines (backward_body).
struct BwdTask { int32_t front, split, nsplit, pbase, p, u, rows_off, dinv_off; int64_t l_off; int32_t dep, need, phase, dep2, early, pad; };   // 64 bytes
static_assert(sizeof(TaskRec) == 128 && sizeof(ChildRec) == 48 && sizeof(BwdTask) == 64, "device record layout");


// Front tables (SoA over fronts).
struct FrontTab {
    const int32_t *p, *u1, *T, *nchild, *child_ptr, *children;
    const int32_t *rel_off, *rel;          // rel of a front as a child: update row -> parent local row
    const int32_t *cb_off, *cbounds;       // per (front, child): lower bounds of rel at p and at every chunk edge
    const int32_t *reg_off, *reg_ptr;      // original-entry region table
    const uint32_t *orig_pos;              // (local row << 16) | local col, aligned with gval
    const int64_t *gval_off, *l_off, *u_off;
    const int32_t *rows_off, *rows;        // global positions of [pivots | update rows]
    const ChildRec* crecs;          // per-task child records
    double* dinv;                          // reciprocal pivots per front (written forward, read backward)
    double* ubuf_root;                     // peer-linked multi-rank solve: the coordinator's update storage (tasks with flag bit 2
                                           // write there); nullptr = this rank's own
    long long* tbuf;                       // optional per-task phase clocks (debug), 8 per task
    const void* task0;                     // base of the task array (indexes tbuf)
};

constexpr int kFrontThreads = 256;
constexpr int kMaxTile = 96;

inline __host__ __device__ int pad_ld(int p) { return ((((p + 7) & ~7) + 11) / 16) * 16 + 4; }   // == 4 mod 16, >= round8(p)
inline __host__ __device__ int round8(int x) { return (x + 7) & ~7; }

// shared-memory doubles needed by one front task
inline __host__ __device__ size_t task_smem_doubles(int p, int ni, int nj, bool diag, bool direct = false, int kind = 0) {
    size_t ld = pad_ld(p);
    size_t rows = ((p && kind != 2) ? round8(p) : 0) + (p ? round8(ni) : 0) + ((p && !diag) ? round8(nj) : 0);
    size_t ldt = (size_t)(round8(nj) | 1);
    return rows * ld + ((direct || kind == 1) ? 0 : (size_t)round8(ni) * ldt) + 16;
}

void launch_eval(const EvalProg& ep, const double* va, const double* vm, cudaStream_t s);
// plain form (reference-layout program of the component-parity API): one thread per destination
void launch_accumulate(const int32_t* ptr, const int32_t* a, const int32_t* b, const double* val,
                       double* out, int64_t n, cudaStream_t s);
// staged form (solver layout): one CTA per item, operands in shared memory
struct AccProg {
    const int32_t *items, *uniq, *ptr;     // items: 8-int records (plan.hpp); ptr: item-local contribution pointers
    const uint32_t* pair;                  // per contribution: staged positions (b << 16 | a)
    const double* val;
    double* out;
    int32_t n_items;
};
void launch_accumulate_staged(const AccProg& ap, cudaStream_t s);
// pclass: 0 (assembly only), 32 or 64
void launch_front_tasks(int pclass, const FrontTab& ft, const TaskRec* tasks, int ntasks,
                        size_t smem_bytes, const double* gval, double* lbuf, double* ubuf,
                        unsigned long long* err, cudaStream_t s);
void launch_backward(const FrontTab& ft, const BwdTask* tasks, int ntasks, const double* lbuf,
                     double* xsol, double* bpart, int32_t* bcnt, cudaStream_t s);
void launch_update(const int32_t* bus, const int32_t* quant, const int32_t* pos, int n,
                   const double* xsol, double* va, double* vm, unsigned long long* delta_bits,
                   cudaStream_t s);
void launch_objective(const EvalProg& ep, const int32_t* m_type, const int32_t* m_target,
                      const int32_t* br_from, const int32_t* br_to, int n_rows, const double* va,
                      const double* vm, double* partial, double* out, cudaStream_t s);
int objective_blocks(int n_rows);
void launch_status(const unsigned long long* flags, double* status, cudaStream_t s);
void launch_assemble_boundary(int n_gamma, int n_areas, const int32_t* inv, const int64_t* off, const int32_t* sel_ptr,
                              const double* s_b, const double* b_hat, double* s_gamma, double* b_gamma, cudaStream_t s);
cudaError_t configure_kernels();
cudaError_t configure_unit_kernels();

// ---- persistent dataflow kernel (solve_kernel.cu): the whole Gauss-Newton loop in ONE launch ----
// Work items of one iteration, in dependency (topological) order:
//   [eval blocks | accumulate blocks | front tasks (level order) | backward tasks (top-down) | update blocks]
// CTAs pull item indices from a global counter and spin on per-front completion counters.
constexpr int kSolveThreads = 256;
#ifndef GSE_EVAL_PER_ITEM
#define GSE_EVAL_PER_ITEM 256
#endif
constexpr int kEvalPerItem = GSE_EVAL_PER_ITEM, kUpdPerItem = 1024;
enum { CTR_NEXT = 0, CTR_EVAL = 32, CTR_ACC = 64, CTR_FWD = 96, CTR_BWD = 128, CTR_UPD = 160, CTR_OBJ = 192,
       CTR_GAMMA = 224,      // peer-linked solve: boundary fronts whose share of delta_x_Gamma has arrived from the coordinator
       CTR_ITER = 256,       // peer-linked solve: ranks that have finished (and published the norm of) an iteration
       CTR_SM0 = 288,        // per SM (512 slots): CTAs of this launch seen on it -- the second one keeps off the chain tasks (solve_kernel.cu)
       CTR_AREA0 = 288 + 512 };    // peer-linked solve: per AREA, tasks of its root that have stored their tile of (S_b | b_hat) in the
                             // coordinator's buffer (fronts are numbered per rank, areas are not)
// per-front counters from SolveProg::front0 = CTR_AREA0 + n_areas rounded up to 32: fdone[n_fronts] (tasks that
// wrote U), pdone[n_fronts] (tasks that stored a factor panel), bdone[n_fronts] (backward solves)
inline __host__ __device__ int ctr_front0(int n_areas) { return CTR_AREA0 + ((n_areas + 31) / 32) * 32; }

// Peer-linked multi-rank solve (one process per GPU, areas sharded over the ranks; reference solver.py:277-298,
// 318-326 are the two exchange points).  Every rank runs gn_solve_kernel over its own items; the exchanges happen
// INSIDE the kernels over peer-mapped memory (NVLink): the area roots of a rank write (S_b | b_hat) straight into
// the coordinator's update storage and bump the coordinator's completion counters, the coordinator's boundary
// back-substitution tasks store their pivots' share of delta_x_Gamma into every rank's solution vector, and the
// per-iteration norm / failure code are max-merged into every rank's copy, so all ranks take the same decision.
constexpr int kMaxPeers = 8;
struct PeerLink {
    int32_t rank, world;               // world == 1: not linked (single-rank plan)
    int32_t n_gamma_fronts;            // boundary fronts with pivots (pieces delta_x_Gamma arrives in)
    int32_t pad;
    unsigned* root_ctr;                // the coordinator's counter block (fdone of the area roots lives there)
    double* xsol[kMaxPeers];           // every rank's solution vector
    unsigned* ctr[kMaxPeers];          // every rank's counter block (CTR_GAMMA, CTR_ITER)
    unsigned long long* gdelta[kMaxPeers];   // every rank's copy of the global per-iteration norm [64]
    unsigned long long* gerr[kMaxPeers];     // every rank's copy of the global failure code, stored inverted (0 = none)
};
struct SolveProg {
    int32_t n_eval_items, n_acc_items, n_tasks, n_btasks, n_upd_items, items_per_it;
    int32_t n_units, n_upd, n_bwd_fronts, n_fronts, n_rows, max_it;
    int32_t front0, n_chain;      // offset of the per-front counters inside ctr (ctr_front0(n_areas)); chain ranges in use
    int32_t bwd_poll, pad0;       // back-substitution hand-off through the solution entries themselves (front_body.cuh: kXUnset)
    int32_t chain_lo[4], chain_hi[4];   // task-index ranges [lo, hi) of runs of levels with at most one panel task per SM:
                                  // the latency chains (top of the areas, boundary tree), handed to one CTA per SM only
    int64_t n_gval;
    double tol;
    const TaskRec* tasks;
    const BwdTask* btasks;
    const int32_t *acc_items, *acc_uniq, *acc_ptr;
    const uint32_t* acc_pair;
    const double* val;
    const int32_t *upd_bus, *upd_quant, *upd_pos;
    const int32_t* pos_bq;        // elimination position -> 2 * bus + (0 angle | 1 magnitude): state update fused into the backward tasks
    const int32_t *m_type, *m_target, *br_from, *br_to;
    double *gval, *lbuf, *ubuf, *xsol, *bpart, *obj_partial;   // obj_partial[nblocks] then the total
    int32_t* bcnt;
    unsigned int* ctr;            // CTR_* globals, then fdone / pdone / bdone [n_fronts] each
    unsigned long long* delta;    // [64] per-iteration |dx| max as ordered bits
    unsigned long long* err;      // failure code (min), ~0 = none
    unsigned long long* stamps;   // optional [1 + 64 * 8] globaltimer stamps (nullptr: off)
    int32_t* result;              // [0] iterations, [1] converged
    unsigned long long* err_out;  // copy of *err for the single readback
    double* obj_out;              // J(x) at the final state
    unsigned long long* trace;    // optional per-item stamps [item][8]: pull, originals ready, children ready, end, smid (debug)
    PeerLink lk;                  // multi-rank exchange over peer memory (world == 1: unused)
};
size_t solve_kernel_static_smem();
cudaError_t solve_kernel_debug_watchdog(unsigned long long* host_mapped, unsigned long long ns);
// returns the number of co-resident CTAs (0 on failure)
int solve_kernel_max_ctas(size_t dyn_smem, int device);
cudaError_t launch_solve(const SolveProg& sp, const EvalProg& ep, const FrontTab& ft, double* va, double* vm,
                         int grid, size_t dyn_smem, cudaStream_t s, bool cooperative = true);

}  // namespace gse
