// front_kernels.cu -- the multifrontal Schur-mode factorisation and its back-substitution.
//
// front_task_kernel<HAS_PIVOTS>: one CTA = one (front, row-chunk I, col-chunk J) task.
//   0. one coalesced read brings the task header and its (pruned) child records into shared memory,
//      so no phase starts with a chain of dependent global loads;
//   1. assemble in shared memory: original entries (written by accumulate_kernel) + extend-add of
//      the children's packed update matrices in fixed child order (deterministic, no atomics);
//   2. factor the pivot block and solve the two row chunks against it: left-looking in blocks of
//      8 columns -- the rank-k update of each block column runs on the FP64 tensor pipe
//      (mma.sync m8n8k4 f64 from shared memory); warp 0 updates and factors the 8x8 diagonal
//      block while the other warps update the remaining rows (look-ahead), then every row thread
//      solves its row against the published block;
//   3. trailing / Schur update U_IJ = F_IJ - L_I L_J^T on the tensor pipe, written packed-lower;
//   4. diagonal tasks store their slice of the factor panel for the backward pass.
// Every task of a front recomputes the (small) pivot-block factor instead of exchanging it:
// redundancy is free while SMs idle, a second launch is not.
//
// Restates numeric_refactor + schur_condense (reference linalg.py:292-332,410-424), assemble_boundary
// (solver.py:106-119) and dense_cholesky_solve's factorisation (linalg.py:46-61) as one tree.
#include "front_body.cuh"

namespace gse {

template <int HAS_PIVOTS>
__global__ void __launch_bounds__(kFrontThreads, HAS_PIVOTS ? 1 : 2)
front_task_kernel(FrontTab ft, const TaskRec* __restrict__ tasks, const double* gval, double* lbuf, double* ubuf,
                  unsigned long long* err) {
    extern __shared__ __align__(16) double sm[];
    __shared__ FrontScratch S;
    long long* tb = ft.tbuf ? ft.tbuf + 32 * ((&tasks[blockIdx.x]) - (const TaskRec*)ft.task0) : nullptr;
    load_task_header(S, &tasks[blockIdx.x]);
    __syncthreads();
    front_task_body<HAS_PIVOTS>(S, sm, ft, gval, lbuf, ubuf, err, tb, NoWait{});
}

void launch_front_tasks(int pclass, const FrontTab& ft, const TaskRec* tasks, int ntasks,
                        size_t smem_bytes, const double* gval, double* lbuf, double* ubuf,
                        unsigned long long* err, cudaStream_t s) {
    if (ntasks == 0) return;
    if (pclass == 0) front_task_kernel<0><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
    else front_task_kernel<1><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
}

__global__ void __launch_bounds__(128) backward_kernel(FrontTab ft, const BwdTask* __restrict__ tasks, const double* lbuf,
                                                       double* xsol, double* bpart, int32_t* bcnt) {
    __shared__ BwdScratch B;
    const BwdTask tk = tasks[blockIdx.x];
    backward_body(B, tk, ft, lbuf, xsol, bpart, bcnt, NoWait{});
}

void launch_backward(const FrontTab& ft, const BwdTask* tasks, int ntasks, const double* lbuf,
                     double* xsol, double* bpart, int32_t* bcnt, cudaStream_t s) {
    if (ntasks == 0) return;
    backward_kernel<<<ntasks, 128, 0, s>>>(ft, tasks, lbuf, xsol, bpart, bcnt);
}

cudaError_t configure_kernels() {
    const int maxsm = 214 * 1024;   // static + dynamic must stay within the 227 KB opt-in limit
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    return cudaSuccess;
}

}  // namespace gse
