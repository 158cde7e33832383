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

namespace gse {

// ---------------------------------------------------------------------------------------------
// Templates
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void put_slot(const EvalProg& ep, int s, double gv, double w, double wr) {
    ep.g[s] = gv;
    ep.gw[s] = w * gv;
    ep.wrg[s] = wr * gv;
}

__device__ __forceinline__ void flow_row(const EvalProg& ep, int row, int slot, bool f_slack,
                                         bool t_slack, double h, double d_thf, double d_tht,
                                         double d_vf, double d_vt) {
    if (row < 0) return;
    const double w = ep.w[row];
    const double wr = w * (ep.z[row] - h);
    int s = slot;
    if (!f_slack) put_slot(ep, s++, d_thf, w, wr);
    if (!t_slack) put_slot(ep, s++, d_tht, w, wr);
    put_slot(ep, s++, d_vf, w, wr);
    put_slot(ep, s, d_vt, w, wr);
}

__global__ void __launch_bounds__(128) eval_templates_kernel(EvalProg ep, const double* __restrict__ va,
                                                             const double* __restrict__ vm) {
    int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < ep.n_fl) {
        // one unit per measured branch: PF, PT, QF, QT share one sincos of the angle difference
        const int e = ep.fl_branch[u], f = ep.fl_from[u], t = ep.fl_to[u];
        const double4* yy = reinterpret_cast<const double4*>(ep.br_y + 8 * (size_t)e);
        const double4 y0 = yy[0], y1 = yy[1];   // (ff.re ff.im ft.re ft.im) (tf.re tf.im tt.re tt.im)
        const double vf = vm[f], vt = vm[t];
        double sn, cs;
        sincos(va[f] - va[t], &sn, &cs);
        const bool fs = f == ep.slack, ts = t == ep.slack;
        const int4 rows = reinterpret_cast<const int4*>(ep.fl_row)[u];
        const int4 slots = reinterpret_cast<const int4*>(ep.fl_slot)[u];
        // from end: own = f, y_own = y_ff = a + jb, y_oth = y_ft = c + jd, delta = th_f - th_t
        {
            const double a = y0.x, b = y0.y, c = y0.z, d = y0.w;
            const double ec = c * cs + d * sn, es = c * sn - d * cs;
            const double vv = vf * vt;
            // P = Vf^2 a + Vf Vt ec ; Q = -Vf^2 b + Vf Vt es
            flow_row(ep, rows.x, slots.x, fs, ts, vf * (vf * a + vt * ec), -vv * es, vv * es,
                     2.0 * vf * a + vt * ec, vf * ec);
            flow_row(ep, rows.z, slots.z, fs, ts, vf * (-vf * b + vt * es), vv * ec, -vv * ec,
                     -2.0 * vf * b + vt * es, vf * es);
        }
        // to end: own = t, y_own = y_tt, y_oth = y_tf, delta = th_t - th_f  (cos same, sin negated)
        {
            const double a = y1.z, b = y1.w, c = y1.x, d = y1.y;
            const double ec = c * cs - d * sn, es = -c * sn - d * cs;
            const double vv = vf * vt;
            flow_row(ep, rows.y, slots.y, fs, ts, vt * (vt * a + vf * ec), vv * es, -vv * es,
                     vt * ec, 2.0 * vt * a + vf * ec);
            flow_row(ep, rows.w, slots.w, fs, ts, vt * (-vt * b + vf * es), -vv * ec, vv * ec,
                     vt * es, -2.0 * vt * b + vf * es);
        }
        return;
    }
    u -= ep.n_fl;
    if (u < ep.n_inj) {
        // one unit per measured bus: P and Q injection share the neighbor loop
        const int i = ep.inj_bus[u];
        const int rp = ep.inj_rowp[u], rq = ep.inj_rowq[u];
        const int sp = ep.inj_slotp[u], sq = ep.inj_slotq[u];
        const int p0 = ep.y_ptr[i], p1 = ep.y_ptr[i + 1];
        const double vi = vm[i], thi = va[i];
        int nth = 0;
        for (int p = p0; p < p1; ++p) nth += ep.y_idx[p] != ep.slack;
        double sum_p = 0.0, sum_q = 0.0, gd = 0.0, bd = 0.0;
        int dth = -1, dvm = -1, cth = 0;
        // pass 1: sums (ascending neighbor order, self excluded -- the bincount order)
        for (int p = p0; p < p1; ++p) {
            const int j = ep.y_idx[p];
            if (j == i) { gd = ep.y_g[p]; bd = ep.y_b[p]; continue; }
            double sn, cs;
            sincos(thi - va[j], &sn, &cs);
            const double g = ep.y_g[p], b = ep.y_b[p], vj = vm[j];
            sum_p += vj * (g * cs + b * sn);
            sum_q += vj * (g * sn - b * cs);
        }
        const double wp = rp >= 0 ? ep.w[rp] : 0.0, wq = rq >= 0 ? ep.w[rq] : 0.0;
        const double hp = vi * (vi * gd + sum_p), hq = vi * (-vi * bd + sum_q);
        const double wrp = rp >= 0 ? wp * (ep.z[rp] - hp) : 0.0, wrq = rq >= 0 ? wq * (ep.z[rq] - hq) : 0.0;
        // pass 2: partials per slot
        for (int p = p0, q = 0; p < p1; ++p, ++q) {
            const int j = ep.y_idx[p];
            const int thpos = (j != ep.slack) ? cth++ : -1;
            const int vmpos = nth + q;
            if (j == i) { dth = thpos; dvm = vmpos; continue; }
            double sn, cs;
            sincos(thi - va[j], &sn, &cs);
            const double g = ep.y_g[p], b = ep.y_b[p], vj = vm[j];
            const double uc = g * cs + b * sn, us = g * sn - b * cs;
            if (rp >= 0) { if (thpos >= 0) put_slot(ep, sp + thpos, vi * (vj * us), wp, wrp); put_slot(ep, sp + vmpos, vi * uc, wp, wrp); }
            if (rq >= 0) { if (thpos >= 0) put_slot(ep, sq + thpos, -vi * (vj * uc), wq, wrq); put_slot(ep, sq + vmpos, vi * us, wq, wrq); }
        }
        if (rp >= 0) { if (dth >= 0) put_slot(ep, sp + dth, -vi * sum_q, wp, wrp); put_slot(ep, sp + dvm, 2.0 * vi * gd + sum_p, wp, wrp); }
        if (rq >= 0) { if (dth >= 0) put_slot(ep, sq + dth, vi * sum_p, wq, wrq); put_slot(ep, sq + dvm, -2.0 * vi * bd + sum_q, wq, wrq); }
        return;
    }
    u -= ep.n_inj;
    if (u < ep.n_vm) {
        const int row = ep.vm_row[u];
        const double w = ep.w[row];
        put_slot(ep, ep.vm_slot[u], 1.0, w, w * (ep.z[row] - vm[ep.vm_bus[u]]));
    }
}

void launch_eval(const EvalProg& ep, const double* va, const double* vm, cudaStream_t s) {
    int n = ep.n_vm + ep.n_fl + ep.n_inj;
    if (n == 0) return;
    eval_templates_kernel<<<(n + 127) / 128, 128, 0, s>>>(ep, va, vm);
}

// ---------------------------------------------------------------------------------------------
// Accumulation: one thread per destination, contributions summed in ascending row order with
// separately rounded multiply / add (the reference's bincount arithmetic, assembly.py:502-520).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) accumulate_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ a,
                                                         const int32_t* __restrict__ b, const double* __restrict__ g,
                                                         const double* __restrict__ gw, const double* __restrict__ wrg,
                                                         double* __restrict__ out, int64_t n) {
    int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n) return;
    double s = 0.0;
    const int q1 = ptr[d + 1];
    for (int q = ptr[d]; q < q1; ++q) {
        const int ia = a[q], ib = b[q];
        const double term = ib < 0 ? wrg[ia] : __dmul_rn(g[ia], gw[ib]);
        s = __dadd_rn(s, term);
    }
    out[d] = s;
}

void launch_accumulate(const int32_t* ptr, const int32_t* a, const int32_t* b, const double* g,
                       const double* gw, const double* wrg, double* out, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    accumulate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ptr, a, b, g, gw, wrg, out, n);
}

// ---------------------------------------------------------------------------------------------
// State update + stacked infinity norm (max is order independent -> deterministic)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) update_state_kernel(const int32_t* __restrict__ bus, const int32_t* __restrict__ quant,
                                                           const int32_t* __restrict__ pos, int n, const double* __restrict__ xsol,
                                                           double* __restrict__ va, double* __restrict__ vm,
                                                           unsigned long long* delta_bits) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    double mag = 0.0;
    if (v < n) {
        const double dx = xsol[pos[v]];
        if (quant[v] == 0) va[bus[v]] += dx; else vm[bus[v]] += dx;
        mag = fabs(dx);
    }
    unsigned long long bits = (unsigned long long)__double_as_longlong(mag);   // NaN sorts above inf
    for (int o = 16; o > 0; o >>= 1) { unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o); bits = other > bits ? other : bits; }
    if ((threadIdx.x & 31) == 0 && bits) atomicMax(delta_bits, bits);
}

void launch_update(const int32_t* bus, const int32_t* quant, const int32_t* pos, int n, const double* xsol,
                   double* va, double* vm, unsigned long long* delta_bits, cudaStream_t s) {
    if (n == 0) return;
    update_state_kernel<<<(n + 255) / 256, 256, 0, s>>>(bus, quant, pos, n, xsol, va, vm, delta_bits);
}

// ---------------------------------------------------------------------------------------------
// Objective (eval_h_all arithmetic: the diagonal term sits inside the neighbor sum)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) objective_kernel(EvalProg ep, const int32_t* __restrict__ m_type,
                                                        const int32_t* __restrict__ m_target, const int32_t* __restrict__ br_from,
                                                        const int32_t* __restrict__ br_to, int n_rows, const double* __restrict__ va,
                                                        const double* __restrict__ vm, double* __restrict__ partial) {
    __shared__ double red[256];
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    double term = 0.0;
    if (r < n_rows) {
        const int t = m_type[r], tg = m_target[r];
        double h;
        if (t == 0) h = vm[tg];
        else if (t <= 2) {
            double acc = 0.0;
            for (int p = ep.y_ptr[tg]; p < ep.y_ptr[tg + 1]; ++p) {
                const int j = ep.y_idx[p];
                double sn, cs;
                sincos(va[tg] - va[j], &sn, &cs);
                acc += (t == 1) ? vm[j] * (ep.y_g[p] * cs + ep.y_b[p] * sn) : vm[j] * (ep.y_g[p] * sn - ep.y_b[p] * cs);
            }
            h = vm[tg] * acc;
        } else {
            const int f = br_from[tg], tt = br_to[tg];
            const double* y = ep.br_y + 8 * (size_t)tg;
            const bool fe = (t == 3 || t == 5);
            const int ob = fe ? f : tt, ub = fe ? tt : f;
            const double a = fe ? y[0] : y[6], b = fe ? y[1] : y[7], c = fe ? y[2] : y[4], d = fe ? y[3] : y[5];
            double sn, cs;
            sincos(va[ob] - va[ub], &sn, &cs);
            const double vo = vm[ob], vu = vm[ub];
            h = (t >= 5) ? vo * (-vo * b + vu * (c * sn - d * cs)) : vo * (vo * a + vu * (c * cs + d * sn));
        }
        const double res = ep.z[r] - h;
        term = ep.w[r] * res * res;
    }
    red[threadIdx.x] = term;
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

int objective_blocks(int n_rows) { return (n_rows + 255) / 256; }

void launch_objective(const EvalProg& ep, const int32_t* m_type, const int32_t* m_target, const int32_t* br_from,
                      const int32_t* br_to, int n_rows, const double* va, const double* vm, double* partial,
                      double* out, cudaStream_t s) {
    const int nb = objective_blocks(n_rows);
    if (nb) objective_kernel<<<nb, 256, 0, s>>>(ep, m_type, m_target, br_from, br_to, n_rows, va, vm, partial);
    objective_final_kernel<<<1, 256, 0, s>>>(partial, nb, out);
}

}  // namespace gse
