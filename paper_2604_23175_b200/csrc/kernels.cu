// kernels.cu -- sm_100a kernels of the multi-area Gauss-Newton iteration.
//
//  eval_templates_kernel   fixed-sparsity measurement templates (V, P/Q injection, P/Q flow):
//                          residual + analytic partials per template slot   [assembly.py:427-483]
//  accumulate_kernel       atomic-free, order-preserving gather-reduction of w*g_a*g_b and
//                          (w*r)*g_a into precomputed destination slots      [assembly.py:486-524]
//  (front_task_kernel / backward_kernel: front_kernels.cu)
//  update_state_kernel     va/vm += dx, stacked infinity norm               [partition.py:59-62,113-116;
//                                                                            solver.py:328-333]
//  objective_kernel        J(x) = sum w (z - h(x))^2                        [solver.py:100-103]
#include <cstdio>

#include "kernels.cuh"
#include "plan.hpp"
#include "unit_bodies.cuh"

namespace gse {

__global__ void __launch_bounds__(128) eval_templates_kernel(EvalProg ep, const double* va, const double* vm) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < ep.n_fl + ep.n_inj + ep.n_vm) eval_unit(ep, u, va, vm);
}

void launch_eval(const EvalProg& ep, const double* va, const double* vm, cudaStream_t s) {
    int n = ep.n_vm + ep.n_fl + ep.n_inj;
    if (n == 0) return;
    eval_templates_kernel<<<(n + 127) / 128, 128, 0, s>>>(ep, va, vm);
}

// Accumulation, plain form: one thread per destination (atomic-free gather, fixed summation order).
__global__ void __launch_bounds__(256) accumulate_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ a,
                                                         const int32_t* __restrict__ b, const double* val,
                                                         double* __restrict__ out, int64_t n) {
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d < n) out[d] = acc_dest(ptr, a, b, val, d);
}

void launch_accumulate(const int32_t* ptr, const int32_t* a, const int32_t* b, const double* val,
                       double* out, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    accumulate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ptr, a, b, val, out, n);
}

// Accumulation, staged form: one CTA per item of the solver-layout program.
__global__ void __launch_bounds__(256) accumulate_staged_kernel(AccProg ap) {
    extern __shared__ __align__(16) double stage[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned parity = 0;
    acc_item_staged(ap, blockIdx.x, stage, &bar, parity);
}

void launch_accumulate_staged(const AccProg& ap, cudaStream_t s) {
    if (ap.n_items == 0) return;
    accumulate_staged_kernel<<<ap.n_items, 256, kAccSmemBytes, s>>>(ap);
}

// State update + stacked infinity norm (max is order independent -> deterministic)
__global__ void __launch_bounds__(256) update_state_kernel(const int32_t* __restrict__ bus, const int32_t* __restrict__ quant,
                                                           const int32_t* __restrict__ pos, int n, const double* xsol,
                                                           double* va, double* vm, unsigned long long* delta_bits) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long bits = v < n ? update_var(bus, quant, pos, v, xsol, va, vm) : 0ull;
    for (int o = 16; o > 0; o >>= 1) { unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o); bits = other > bits ? other : bits; }
    if ((threadIdx.x & 31) == 0 && bits) atomicMax(delta_bits, bits);
}

void launch_update(const int32_t* bus, const int32_t* quant, const int32_t* pos, int n, const double* xsol,
                   double* va, double* vm, unsigned long long* delta_bits, cudaStream_t s) {
    if (n == 0) return;
    update_state_kernel<<<(n + 255) / 256, 256, 0, s>>>(bus, quant, pos, n, xsol, va, vm, delta_bits);
}

// Objective: per-block partial sums, then one block adds them in block order (fixed order).
__global__ void __launch_bounds__(256) objective_kernel(EvalProg ep, const int32_t* __restrict__ m_type,
                                                        const int32_t* __restrict__ m_target, const int32_t* __restrict__ br_from,
                                                        const int32_t* __restrict__ br_to, int n_rows, const double* va,
                                                        const double* vm, double* __restrict__ partial) {
    __shared__ double red[256];
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    red[threadIdx.x] = r < n_rows ? objective_row(ep, m_type, m_target, br_from, br_to, r, va, vm) : 0.0;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) objective_final_kernel(const double* __restrict__ partial, int n, double* out) {
    __shared__ double red[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) s += partial[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// assemble_boundary (reference solver.py:106-119) for caller-supplied Schur blocks: one thread per
// entry of S_Gamma (and one per entry of b_Gamma), areas added in ascending order -> the same sums
// in the same order as the reference's loop.  inv[a][slot] = local boundary index of x_Gamma slot.
__global__ void __launch_bounds__(256) assemble_boundary_kernel(int n_gamma, int n_areas, const int32_t* __restrict__ inv,
                                                                const int64_t* __restrict__ off, const int32_t* __restrict__ sel_ptr,
                                                                const double* __restrict__ s_b, const double* __restrict__ b_hat,
                                                                double* __restrict__ s_gamma, double* __restrict__ b_gamma) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nn = (int64_t)n_gamma * n_gamma;
    if (t < nn) {
        const int I = (int)(t / n_gamma), J = (int)(t % n_gamma);
        double s = 0.0;
        for (int a = 0; a < n_areas; ++a) {
            const int i = inv[(size_t)a * n_gamma + I], j = inv[(size_t)a * n_gamma + J];
            if (i >= 0 && j >= 0) s += s_b[off[a] + (int64_t)i * (sel_ptr[a + 1] - sel_ptr[a]) + j];
        }
        s_gamma[t] = s;
    } else if (t < nn + n_gamma) {
        const int I = (int)(t - nn);
        double s = 0.0;
        for (int a = 0; a < n_areas; ++a) { const int i = inv[(size_t)a * n_gamma + I]; if (i >= 0) s += b_hat[sel_ptr[a] + i]; }
        b_gamma[I] = s;
    }
}

void launch_assemble_boundary(int n_gamma, int n_areas, const int32_t* inv, const int64_t* off, const int32_t* sel_ptr,
                              const double* s_b, const double* b_hat, double* s_gamma, double* b_gamma, cudaStream_t s) {
    const int64_t n = (int64_t)n_gamma * n_gamma + n_gamma;
    assemble_boundary_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n_gamma, n_areas, inv, off, sel_ptr, s_b, b_hat, s_gamma, b_gamma);
}

// flags = [|dx| max as ordered bits, failure code (~0 = none)] -> status = [max |dx|, failed ? 1 : 0]
__global__ void status_kernel(const unsigned long long* __restrict__ flags, double* __restrict__ status) {
    status[0] = __longlong_as_double((long long)flags[0]);
    status[1] = flags[1] != ~0ull ? 1.0 : 0.0;
}
void launch_status(const unsigned long long* flags, double* status, cudaStream_t s) { status_kernel<<<1, 1, 0, s>>>(flags, status); }

cudaError_t configure_unit_kernels() {
    return cudaFuncSetAttribute(accumulate_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAccSmemBytes);
}

int objective_blocks(int n_rows) { return (n_rows + 255) / 256; }

void launch_objective(const EvalProg& ep, const int32_t* m_type, const int32_t* m_target, const int32_t* br_from,
                      const int32_t* br_to, int n_rows, const double* va, const double* vm, double* partial,
                      double* out, cudaStream_t s) {
    const int nb = objective_blocks(n_rows);
    if (nb) objective_kernel<<<nb, 256, 0, s>>>(ep, m_type, m_target, br_from, br_to, n_rows, va, vm, partial);
    objective_final_kernel<<<1, 256, 0, s>>>(partial, nb, out);
}

}  // namespace gse
