// kernels.cu -- sm_100a kernels of the multi-area Gauss-Newton iteration.
//
//  eval_templates_kernel   fixed-sparsity measurement templates (V, P/Q injection, P/Q flow):
//                          residual + analytic partials per template slot   [assembly.py:427-483]
//  accumulate_kernel       atomic-free, order-preserving gather-reduction of w*g_a*g_b and
//                          (w*r)*g_a into precomputed destination slots      [assembly.py:486-524]
//  front_task_kernel<P>    one (front, row-chunk, col-chunk) task of the multifrontal Schur-mode
//                          factorisation: extend-add assembly, register-resident panel Cholesky,
//                          FP64 tensor-core (DMMA m8n8k4) trailing / Schur update
//                                                      [linalg.py:292-332,410-424; solver.py:106-119;
//                                                       linalg.py:46-61 for the boundary chain]
//  backward_kernel         per-front back-substitution (top-down)          [linalg.py:366-383,427-434]
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
// Front tasks
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound_dev(const int32_t* __restrict__ a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (a[mid] < key) lo = mid + 1; else hi = mid; }
    return lo;
}

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// child update block rows [r0,r1) x cols [c0,c1) (lower part only) -> dst[(rel[i]-rs)*ld + rel[j]-cs]
__device__ __forceinline__ void add_child_block(const double* __restrict__ U, const int32_t* __restrict__ rel,
                                                int r0, int r1, int c0, int c1, double* dst, int ld,
                                                int rs, int cs, int tid, int nth) {
    const int w = c1 - c0, h = r1 - r0;
    if (w <= 0 || h <= 0) return;
    for (int t = tid; t < w * h; t += nth) {
        const int i = r0 + t / w, j = c0 + t % w;
        if (j <= i) dst[(rel[i] - rs) * ld + (rel[j] - cs)] += U[(size_t)i * (i + 1) / 2 + j];
    }
}

template <int P>
__global__ void __launch_bounds__(kFrontThreads, P == 64 ? 1 : 2)
front_task_kernel(FrontTab ft, const TaskRec* __restrict__ tasks, const double* __restrict__ gval,
                  double* __restrict__ lbuf, double* __restrict__ ubuf, unsigned long long* err) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int sb[8];
    const TaskRec tk = tasks[blockIdx.x];
    const int f = tk.front, ci = tk.ci, cj = tk.cj;
    const int p = P ? ft.p[f] : 0;
    const int u1 = ft.u1[f], T = ft.T[f];
    const int i0 = ci * T, ni = min(T, u1 - i0), j0 = cj * T, nj = min(T, u1 - j0);
    const bool diag = ci == cj;
    const int ld = pad_ld(p);
    const int rp = p ? round8(p) : 0, ri = p ? round8(ni) : 0, rj = (p && !diag) ? round8(nj) : 0;
    const int ldt = round8(nj) | 1;
    double* pan = sm;
    double* tile = sm + (size_t)(rp + ri + rj) * ld;
    const int tid = threadIdx.x, nth = blockDim.x;

    {
        const int total = (rp + ri + rj) * ld + round8(ni) * ldt;
        for (int t = tid; t < total; t += nth) sm[t] = 0.0;
    }
    __syncthreads();

    // ---- original entries (written by accumulate_kernel into gval) --------------------------
    {
        const int32_t* rptr = ft.reg_ptr + ft.reg_off[f];
        const int64_t goff = ft.gval_off[f];
        const uint32_t* opos = ft.orig_pos + goff;
        const double* gv = gval + goff;
        if (p) {
            for (int e = rptr[0] + tid; e < rptr[1]; e += nth) {       // region (0,0): pivot block
                const uint32_t q = opos[e];
                pan[(q >> 16) * ld + (q & 0xffffu)] = gv[e];
            }
            const int ridI = (ci + 1) * (ci + 2) / 2;
            for (int e = rptr[ridI] + tid; e < rptr[ridI + 1]; e += nth) {
                const uint32_t q = opos[e];
                pan[(rp + (int)(q >> 16) - p - i0) * ld + (q & 0xffffu)] = gv[e];
            }
            if (!diag) {
                const int ridJ = (cj + 1) * (cj + 2) / 2;
                for (int e = rptr[ridJ] + tid; e < rptr[ridJ + 1]; e += nth) {
                    const uint32_t q = opos[e];
                    pan[(rp + ri + (int)(q >> 16) - p - j0) * ld + (q & 0xffffu)] = gv[e];
                }
            }
        }
        const int ridT = (ci + 1) * (ci + 2) / 2 + cj + 1;
        for (int e = rptr[ridT] + tid; e < rptr[ridT + 1]; e += nth) {
            const uint32_t q = opos[e];
            tile[((int)(q >> 16) - p - i0) * ldt + ((int)(q & 0xffffu) - p - j0)] = gv[e];
        }
    }
    __syncthreads();

    // ---- extend-add of the children's update matrices, fixed child order --------------------
    {
        const int nchild = ft.nchild[f], cptr = ft.child_ptr[f];
        for (int c = 0; c < nchild; ++c) {
            const int ch = ft.children[cptr + c];
            const int cu1 = ft.u1[ch];
            const int32_t* rel = ft.rel + ft.rel_off[ch];
            const double* U = ubuf + ft.u_off[ch];
            if (tid < 5) {
                const int key = tid == 0 ? p : tid == 1 ? p + i0 : tid == 2 ? p + i0 + ni : tid == 3 ? p + j0 : p + j0 + nj;
                sb[tid] = lower_bound_dev(rel, cu1, key);
            }
            __syncthreads();
            const int eP = sb[0], bI = sb[1], eI = sb[2], bJ = sb[3], eJ = sb[4];
            if (p) {
                add_child_block(U, rel, 0, eP, 0, eP, pan, ld, 0, 0, tid, nth);
                add_child_block(U, rel, bI, eI, 0, eP, pan + (size_t)rp * ld, ld, p + i0, 0, tid, nth);
                if (!diag) add_child_block(U, rel, bJ, eJ, 0, eP, pan + (size_t)(rp + ri) * ld, ld, p + j0, 0, tid, nth);
            }
            add_child_block(U, rel, bI, eI, bJ, eJ, tile, ldt, p + i0, p + j0, tid, nth);
            __syncthreads();
        }
    }

    // ---- panel Cholesky: one thread per row, row in registers, one barrier per pivot --------
    if (P && p) {
        const int R = p + ni + (diag ? 0 : nj);
        const bool active = tid < R;
        const int prow = tid < p ? tid : tid < p + ni ? rp + (tid - p) : rp + ri + (tid - p - ni);
        double* myrow = pan + (size_t)(active ? prow : 0) * ld;
        double x[P ? P : 1];
#pragma unroll
        for (int k = 0; k < P; ++k) x[k] = (active && k < p) ? myrow[k] : 0.0;
        double ss = 0.0;
        if (tid == 0) {
            const double d = x[0];
            if (!(d > 0.0)) atomicMin(err, ((unsigned long long)f << 32) | 0ull);
            x[0] = sqrt(d);
            myrow[0] = x[0];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (k < p) {
                if (active && tid > k) {
                    const double* lk = pan + (size_t)k * ld;
                    double a0 = x[k], a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int j = 0; j < k; ++j) {
                        const double l = lk[j];
                        if ((j & 3) == 0) a0 = fma(-x[j], l, a0);
                        else if ((j & 3) == 1) a1 = fma(-x[j], l, a1);
                        else if ((j & 3) == 2) a2 = fma(-x[j], l, a2);
                        else a3 = fma(-x[j], l, a3);
                    }
                    x[k] = ((a0 + a1) + (a2 + a3)) / lk[k];
                    myrow[k] = x[k];
                    if (tid < p) {
                        ss = fma(x[k], x[k], ss);
                        if (k + 1 < P && tid == k + 1) {
                            const double d = x[k + 1 < P ? k + 1 : 0] - ss;
                            if (!(d > 0.0)) atomicMin(err, ((unsigned long long)f << 32) | (unsigned long long)(k + 1));
                            x[k + 1 < P ? k + 1 : 0] = sqrt(d);
                            myrow[k + 1] = x[k + 1 < P ? k + 1 : 0];
                        }
                    }
                }
                __syncthreads();
            }
        }
    }

    // ---- trailing update on the FP64 tensor pipe: U_IJ = F_IJ - L_I L_J^T -------------------
    {
        const double* Pi = pan + (size_t)rp * ld;
        const double* Pj = diag ? Pi : pan + (size_t)(rp + ri) * ld;
        const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
        const int nbi = round8(ni) >> 3, nbj = round8(nj) >> 3;
        const int kend = (p + 3) & ~3;
        double* U = ubuf + ft.u_off[f];
        for (int blk = warp; blk < nbi * nbj; blk += nwarps) {
            const int bi = blk / nbj, bj = blk % nbj;
            if (diag && bj > bi) continue;
            double c0 = 0.0, c1 = 0.0;
            if (p) {
                const double* ap = Pi + (size_t)(bi * 8 + (lane >> 2)) * ld + (lane & 3);
                const double* bp = Pj + (size_t)(bj * 8 + (lane >> 2)) * ld + (lane & 3);
#pragma unroll 4
                for (int kk = 0; kk < kend; kk += 4) dmma_m8n8k4(c0, c1, ap[kk], bp[kk]);
            }
            const int row = bi * 8 + (lane >> 2), col = bj * 8 + 2 * (lane & 3);
            if (row < ni) {
                const int I = i0 + row, J = j0 + col;
                double* urow = U + (size_t)I * (I + 1) / 2;
                if (col < nj && J <= I) urow[J] = tile[row * ldt + col] - c0;
                if (col + 1 < nj && J + 1 <= I) urow[J + 1] = tile[row * ldt + col + 1] - c1;
            }
        }
        // ---- factor panel to global (diagonal tasks own their row chunk) ----------------------
        if (p && diag) {
            double* L = lbuf + ft.l_off[f];
            if (ci == 0)
                for (int t = tid; t < p * p; t += nth) L[t] = pan[(t / p) * ld + (t % p)];
            double* Li = L + (size_t)(p + i0) * p;
            for (int t = tid; t < ni * p; t += nth) Li[t] = Pi[(t / p) * ld + (t % p)];
        }
    }
}

void launch_front_tasks(int pclass, const FrontTab& ft, const TaskRec* tasks, int ntasks,
                        size_t smem_bytes, const double* gval, double* lbuf, double* ubuf,
                        unsigned long long* err, cudaStream_t s) {
    if (ntasks == 0) return;
    if (pclass == 0) front_task_kernel<0><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
    else if (pclass == 32) front_task_kernel<32><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
    else front_task_kernel<64><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
}

// ---------------------------------------------------------------------------------------------
// Backward substitution: x_P = L11^{-T} (y_P - L21^T x_U), one CTA per front
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) backward_kernel(FrontTab ft, const int32_t* __restrict__ fronts,
                                                       const double* __restrict__ lbuf, double* __restrict__ xsol) {
    __shared__ double l11[64 * 65];
    __shared__ double part[4][64];
    __shared__ double tv[64];
    extern __shared__ double xu[];
    const int f = fronts[blockIdx.x];
    const int p = ft.p[f], u = ft.u1[f] - 1;
    const double* L = lbuf + ft.l_off[f];
    const int32_t* rows = ft.rows + ft.rows_off[f];
    const int tid = threadIdx.x;
    for (int i = tid; i < u; i += blockDim.x) xu[i] = xsol[rows[p + i]];
    for (int t = tid; t < p * p; t += blockDim.x) l11[(t / p) * 65 + (t % p)] = L[t];
    __syncthreads();
    const int k = tid & 63, grp = tid >> 6;
    {
        const int per = (u + 3) / 4, lo = grp * per, hi = min(u, lo + per);
        double s0 = 0.0, s1 = 0.0;
        if (k < p) {
            const double* col = L + (size_t)p * p + k;
            int i = lo;
            for (; i + 1 < hi; i += 2) { s0 = fma(col[(size_t)i * p], xu[i], s0); s1 = fma(col[(size_t)(i + 1) * p], xu[i + 1], s1); }
            if (i < hi) s0 = fma(col[(size_t)i * p], xu[i], s0);
        }
        part[grp][k] = s0 + s1;
    }
    __syncthreads();
    if (tid < p) tv[tid] = L[(size_t)(p + u) * p + tid] - ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]));
    __syncthreads();
    // warp 0+1 run the triangular solve with L11^T
    for (int c = p - 1; c >= 0; --c) {
        if (tid == c) tv[c] = tv[c] / l11[c * 65 + c];
        __syncthreads();
        if (tid < c) tv[tid] = fma(-l11[c * 65 + tid], tv[c], tv[tid]);
        __syncthreads();
    }
    if (tid < p) xsol[rows[tid]] = tv[tid];
}

void launch_backward(const FrontTab& ft, const int32_t* fronts, int nfronts, int max_u, const double* lbuf,
                     double* xsol, cudaStream_t s) {
    if (nfronts == 0) return;
    backward_kernel<<<nfronts, 256, sizeof(double) * (size_t)(max_u + 8), s>>>(ft, fronts, lbuf, xsol);
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

cudaError_t configure_kernels() {
    const int maxsm = 226 * 1024;   // static + dynamic must stay within the 227 KB opt-in limit
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024))) return e;
    return cudaSuccess;
}


}  // namespace gse
