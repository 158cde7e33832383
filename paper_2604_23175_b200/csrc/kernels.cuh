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
    const int32_t *vm_bus, *vm_row, *vm_slot;
    const int32_t *fl_branch, *fl_from, *fl_to, *fl_row, *fl_slot;
    const int32_t *inj_bus, *inj_rowp, *inj_rowq, *inj_slotp, *inj_slotq;
    // per-slot outputs: gradient, weight*gradient, (weight*residual)*gradient
    double *g, *gw, *wrg;
};

// One (front, row-chunk, col-chunk) task: everything the CTA needs, read with one coalesced load.
struct TaskRec {                                      // 128 bytes
    int32_t front, ci, cj, p, u1, T, nchild, child_off;
    int32_t reg[8];                                   // original-entry ranges (relative to gval_off): PP, IP, JP, tile
    int64_t gval_off, l_off, u_off;
    int32_t flags, dinv_off, pad[8];                  // flags bit 0: tile read directly from the single child's U
};
// One child of a task (children that do not reach the task's regions are pruned on the host).
struct ChildRec { int64_t u_off; int32_t rel_off, eP, bI, eI, bJ, eJ; };   // 32 bytes
struct BwdTask { int32_t front, split, nsplit, pbase, p, u, rows_off, dinv_off; int64_t l_off, pad2; };   // 48 bytes


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
    long long* tbuf;                       // optional per-task phase clocks (debug), 8 per task
    const void* task0;                     // base of the task array (indexes tbuf)
};

constexpr int kFrontThreads = 256;
constexpr int kMaxTile = 96;

inline __host__ __device__ int pad_ld(int p) { return ((((p + 7) & ~7) + 11) / 16) * 16 + 4; }   // == 4 mod 16, >= round8(p)
inline __host__ __device__ int round8(int x) { return (x + 7) & ~7; }

// shared-memory doubles needed by one front task
inline __host__ __device__ size_t task_smem_doubles(int p, int ni, int nj, bool diag, bool direct = false) {
    size_t ld = pad_ld(p);
    size_t rows = (p ? round8(p) : 0) + (p ? round8(ni) : 0) + ((p && !diag) ? round8(nj) : 0);
    size_t ldt = (size_t)(round8(nj) | 1);
    return rows * ld + (direct ? 0 : (size_t)round8(ni) * ldt) + 16;
}

void launch_eval(const EvalProg& ep, const double* va, const double* vm, cudaStream_t s);
void launch_accumulate(const int32_t* ptr, const int32_t* a, const int32_t* b, const double* g,
                       const double* gw, const double* wrg, double* out, int64_t n, cudaStream_t s);
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
cudaError_t configure_kernels();

}  // namespace gse
