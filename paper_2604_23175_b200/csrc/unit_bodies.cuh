// unit_bodies.cuh -- per-unit device bodies of the assembly / update / objective kernels, shared
// by the level-launch kernels (kernels.cu) and the persistent dataflow kernel (solve_kernel.cu).
//
// Every load of data that another CTA of the SAME launch may have produced (state vectors, slot
// values, solution vector) goes through ldc() = ld.global.cg: L1 is not coherent across SMs, and
// the persistent kernel re-reads the same addresses iteration after iteration.
#pragma once
#include "kernels.cuh"
#include "plan.hpp"

namespace gse {

__device__ __forceinline__ double ldc(const double* p) { return __ldcg(p); }

__device__ __forceinline__ void put_slot(const EvalProg& ep, int s, double gv, double w) {
    reinterpret_cast<double2*>(ep.g)[s] = make_double2(gv, w * gv);      // (g, w*g) interleaved: one 16-byte store
}

// (w, z of the row are passed in: the caller fetches them for all rows of the unit in one round of independent
// loads -- inside this function they would queue behind the stores of the previous row, one L2 round trip each)
__device__ __forceinline__ void flow_row(const EvalProg& ep, int row, int slot, bool f_slack,
                                         bool t_slack, double w, double z, double h, double d_thf, double d_tht,
                                         double d_vf, double d_vt) {
    if (row < 0) return;
    ep.wr[row] = w * (z - h);
    int s = slot;
    if (!f_slack) put_slot(ep, s++, d_thf, w);
    if (!t_slack) put_slot(ep, s++, d_tht, w);
    put_slot(ep, s++, d_vf, w);
    put_slot(ep, s, d_vt, w);
}

// One template evaluation unit u in [0, n_fl + n_inj + n_vm)   [assembly.py:427-483].
// Writes, per template slot, the partial g and w*g, and per row the weighted residual w*r.
__device__ __forceinline__ void eval_unit(const EvalProg& ep, int u, const double* va, const double* vm) {
    if (u < ep.n_fl) {
        // one unit per measured branch: PF, PT, QF, QT (and the current magnitudes IF, IT) share one sincos of the
        // angle difference
        const int e = ep.fl_branch[u], f = ep.fl_from[u], t = ep.fl_to[u];
        const int4 rows = reinterpret_cast<const int4*>(ep.fl_row)[2 * u];
        const int4 slots = reinterpret_cast<const int4*>(ep.fl_slot)[2 * u];
        // (plans without ammeter rows -- every reference-generated set -- skip the two loads)
        const int2 irows = ep.has_current ? reinterpret_cast<const int2*>(ep.fl_row)[4 * u + 2] : make_int2(-1, -1);
        const int2 islots = ep.has_current ? reinterpret_cast<const int2*>(ep.fl_slot)[4 * u + 2] : make_int2(-1, -1);
        const double4* yy = reinterpret_cast<const double4*>(ep.br_y + 8 * (size_t)e);
        const double4 y0 = yy[0], y1 = yy[1];   // (ff.re ff.im ft.re ft.im) (tf.re tf.im tt.re tt.im)
        const double vf = ldc(vm + f), vt = ldc(vm + t);
        const double thf = ldc(va + f), tht = ldc(va + t);
        // weights and measured values of the unit's rows: independent loads, issued with the state loads
        const int r6[6] = {rows.x, rows.y, rows.z, rows.w, irows.x, irows.y};
        double w6[6], z6[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) { w6[k] = r6[k] >= 0 ? ep.w[r6[k]] : 0.0; z6[k] = r6[k] >= 0 ? ep.z[r6[k]] : 0.0; }
        double sn, cs;
        sincos(thf - tht, &sn, &cs);
        const bool fs = f == ep.slack, ts = t == ep.slack;
        // from end: own = f, y_own = y_ff = a + jb, y_oth = y_ft = c + jd, delta = th_f - th_t
        {
            const double a = y0.x, b = y0.y, c = y0.z, d = y0.w;
            const double ec = c * cs + d * sn, es = c * sn - d * cs;
            const double vv = vf * vt;
            // P = Vf^2 a + Vf Vt ec ; Q = -Vf^2 b + Vf Vt es
            flow_row(ep, rows.x, slots.x, fs, ts, w6[0], z6[0], vf * (vf * a + vt * ec), -vv * es, vv * es,
                     2.0 * vf * a + vt * ec, vf * ec);
            flow_row(ep, rows.z, slots.z, fs, ts, w6[2], z6[2], vf * (-vf * b + vt * es), vv * ec, -vv * ec,
                     -2.0 * vf * b + vt * es, vf * es);
        }
        // to end: own = t, y_own = y_tt, y_oth = y_tf, delta = th_t - th_f  (cos same, sin negated)
        {
            const double a = y1.z, b = y1.w, c = y1.x, d = y1.y;
            const double ec = c * cs - d * sn, es = -c * sn - d * cs;
            const double vv = vf * vt;
            flow_row(ep, rows.y, slots.y, fs, ts, w6[1], z6[1], vt * (vt * a + vf * ec), vv * es, -vv * es,
                     vt * ec, 2.0 * vt * a + vf * ec);
            flow_row(ep, rows.w, slots.w, fs, ts, w6[3], z6[3], vt * (-vt * b + vf * es), -vv * ec, vv * ec,
                     vt * es, -2.0 * vt * b + vf * es);
        }
        // current magnitudes (north_star template; the reference has none, measurement.py:27-34): with i = y_own V_o +
        // y_oth V_u,  |i|^2 = |y_own|^2 Vo^2 + |y_oth|^2 Vu^2 + 2 Vo Vu (al cos d - be sin d),  al + j be = y_own conj(y_oth),
        // d = th_o - th_u;  h = |i| and dh/dx = d|i|^2/dx / (2 h).  A vanishing current (flat start on a branch without
        // charging) has no gradient: the row then contributes nothing to this iteration.
        if (irows.x >= 0) {
            const double a = y0.x, b = y0.y, c = y0.z, d = y0.w;
            const double al = a * c + b * d, be = b * c - a * d, A = a * a + b * b, C = c * c + d * d;
            const double E = al * cs - be * sn, vv = vf * vt;
            const double m2 = A * vf * vf + C * vt * vt + 2.0 * vv * E;
            const double h = sqrt(fmax(m2, 0.0)), ih = m2 > 1e-24 ? 1.0 / h : 0.0;
            const double dth = vv * (-al * sn - be * cs) * ih;
            flow_row(ep, irows.x, islots.x, fs, ts, w6[4], z6[4], h, dth, -dth, (A * vf + vt * E) * ih, (C * vt + vf * E) * ih);
        }
        if (irows.y >= 0) {
            const double a = y1.z, b = y1.w, c = y1.x, d = y1.y;       // own = t: y_tt, y_tf; d = th_t - th_f (sin negated)
            const double al = a * c + b * d, be = b * c - a * d, A = a * a + b * b, C = c * c + d * d;
            const double E = al * cs + be * sn, vv = vf * vt;
            const double m2 = A * vt * vt + C * vf * vf + 2.0 * vv * E;
            const double h = sqrt(fmax(m2, 0.0)), ih = m2 > 1e-24 ? 1.0 / h : 0.0;
            const double dtt = vv * (al * sn - be * cs) * ih;
            flow_row(ep, irows.y, islots.y, fs, ts, w6[5], z6[5], h, -dtt, dtt, (C * vf + vt * E) * ih, (A * vt + vf * E) * ih);
        }
        return;
    }
    u -= ep.n_fl;
    if (u < ep.n_inj) {
        // one unit per measured bus: P and Q injection share one pass over the Ybus row.  The
        // partials of the neighbor slots do not depend on the row sums, so they are written as the
        // row is walked (neighbors in batches of four: their indices, then their state and
        // admittances, are each fetched with independent loads); the self slots and the weighted
        // residuals follow once the sums are complete.
        const int i = ep.inj_bus[u];
        const int rp = ep.inj_rowp[u], rq = ep.inj_rowq[u];
        const int sp = ep.inj_slotp[u], sq = ep.inj_slotq[u];
        const int nth = ep.inj_nth[u];
        const int p0 = ep.y_ptr[i], p1 = ep.y_ptr[i + 1];
        const double vi = ldc(vm + i), thi = ldc(va + i);
        const double wp = rp >= 0 ? ep.w[rp] : 0.0, wq = rq >= 0 ? ep.w[rq] : 0.0;
        const double zp = rp >= 0 ? ep.z[rp] : 0.0, zq = rq >= 0 ? ep.z[rq] : 0.0;      // (fetched with the weights, not after the row walk)
        double sum_p = 0.0, sum_q = 0.0, gd = 0.0, bd = 0.0;
        int dth = -1, dvm = -1, cth = 0;
        for (int pb = p0; pb < p1; pb += 4) {
            int j[4];
            double thj[4], vj[4], gg[4], bb[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) j[k] = pb + k < p1 ? ep.y_idx[pb + k] : -1;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool ok = j[k] >= 0;
                thj[k] = ok ? ldc(va + j[k]) : 0.0; vj[k] = ok ? ldc(vm + j[k]) : 0.0;
                gg[k] = ok ? ep.y_g[pb + k] : 0.0; bb[k] = ok ? ep.y_b[pb + k] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (j[k] < 0) break;
                const int thpos = (j[k] != ep.slack) ? cth++ : -1;
                const int vmpos = nth + (pb + k - p0);
                if (j[k] == i) { gd = gg[k]; bd = bb[k]; dth = thpos; dvm = vmpos; continue; }
                double sn, cs;
                sincos(thi - thj[k], &sn, &cs);
                const double uc = gg[k] * cs + bb[k] * sn, us = gg[k] * sn - bb[k] * cs;
                sum_p += vj[k] * uc;     // ascending neighbor order, self excluded -- the bincount order
                sum_q += vj[k] * us;
                if (rp >= 0) { if (thpos >= 0) put_slot(ep, sp + thpos, vi * (vj[k] * us), wp); put_slot(ep, sp + vmpos, vi * uc, wp); }
                if (rq >= 0) { if (thpos >= 0) put_slot(ep, sq + thpos, -vi * (vj[k] * uc), wq); put_slot(ep, sq + vmpos, vi * us, wq); }
            }
        }
        if (rp >= 0) {
            ep.wr[rp] = wp * (zp - vi * (vi * gd + sum_p));
            if (dth >= 0) put_slot(ep, sp + dth, -vi * sum_q, wp);
            put_slot(ep, sp + dvm, 2.0 * vi * gd + sum_p, wp);
        }
        if (rq >= 0) {
            ep.wr[rq] = wq * (zq - vi * (-vi * bd + sum_q));
            if (dth >= 0) put_slot(ep, sq + dth, vi * sum_p, wq);
            put_slot(ep, sq + dvm, -2.0 * vi * bd + sum_q, wq);
        }
        return;
    }
    u -= ep.n_inj;
    if (u < ep.n_vm) {
        const int row = ep.vm_row[u];
        const double w = ep.w[row];
        ep.wr[row] = w * (ep.z[row] - ldc(vm + ep.vm_bus[u]));
        put_slot(ep, ep.vm_slot[u], 1.0, w);
    }
}

// One accumulation destination: contributions val[a] * val[b] summed in ascending row order with
// separately rounded multiply / add (the reference's bincount arithmetic, assembly.py:502-520).
__device__ __forceinline__ double acc_dest(const int32_t* __restrict__ ptr, const int32_t* __restrict__ a,
                                           const int32_t* __restrict__ b, const double* val, int64_t d) {
    double s = 0.0;
    const int q1 = ptr[d + 1];
    for (int q = ptr[d]; q < q1; ++q) s = __dadd_rn(s, __dmul_rn(ldc(val + a[q]), ldc(val + b[q])));
    return s;
}

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers ----------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy; bytes and both addresses are multiples of 16
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// shared -> global bulk copy (TMA store); bytes and both addresses are multiples of 16.  The issuing
// thread commits and, before the data may be signalled to other CTAs, waits for the group.
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// One staged accumulation item (symbolic.cpp: build_acc_items), entirely out of shared memory:
// one thread starts two TMA bulk copies (contribution pairs, item-local pointers) while all
// threads gather the item's distinct values (independent loads, eight in flight per thread);
// then every thread walks its destinations' contribution lists, four destinations interleaved.
// Same summation order and arithmetic as acc_dest.  stage: kAccSmemBytes of shared memory that
// no thread of the CTA touches concurrently; bar / parity: the CTA's mbarrier and its phase.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

// Rounds of K interleaved contribution lists, until list K - 1 (the shortest of them) is exhausted; every
// list sums in its own pair order with separately rounded multiply / add (the bincount arithmetic).
template <int K>
__device__ __forceinline__ void acc_rounds(const double* sv, const uint32_t* spair, int (&q)[4], const int (&qe)[4],
                                           uint32_t (&pr)[4], double (&s)[4]) {
    while (q[K - 1] < qe[K - 1]) {
        double x[K], y[K];
        uint32_t nx[K];
#pragma unroll
        for (int k = 0; k < K; ++k) { x[k] = sv[pr[k] & 0xffffu]; y[k] = sv[pr[k] >> 16]; }
#pragma unroll
        for (int k = 0; k < K; ++k) nx[k] = q[k] + 1 < qe[k] ? spair[q[k] + 1] : 0u;     // next round's pairs
#pragma unroll
        for (int k = 0; k < K; ++k) { s[k] = __dadd_rn(s[k], __dmul_rn(x[k], y[k])); ++q[k]; pr[k] = nx[k]; }
    }
}

__device__ __forceinline__ void acc_item_staged(const AccProg& ap, int item, double* stage, unsigned long long* bar,
                                                unsigned& parity, unsigned long long* tr = nullptr) {
    const int4 r0 = reinterpret_cast<const int4*>(ap.items)[2 * item];       // first dest, dests, value offset, values
    const int4 r1 = reinterpret_cast<const int4*>(ap.items)[2 * item + 1];   // pair offset, pairs, pointer offset
    const int tid = threadIdx.x, nth = blockDim.x;
    double* sv = stage;
    uint32_t* spair = reinterpret_cast<uint32_t*>(stage + kAccStageMax);
    int32_t* sptr = reinterpret_cast<int32_t*>(spair + kAccPairMax);
    if (tid == 0) {
        const unsigned pb = (unsigned)((r1.y + 3) & ~3) * 4u, qb = (unsigned)((2 * r0.y + 1 + 3) & ~3) * 4u;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // earlier generic accesses to the buffer
        mbar_expect_tx(bar, pb + qb);
        if (pb) tma_load_1d(spair, ap.pair + r1.x, pb, bar);
        tma_load_1d(sptr, ap.ptr + r1.z, qb, bar);
    }
    const int32_t* uq = ap.uniq + r0.z;
    for (int i = tid; i < r0.w; i += 8 * nth) {
        int idx[8];
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) idx[k] = i + k * nth < r0.w ? uq[i + k * nth] : -1;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = idx[k] >= 0 ? ldc(ap.val + idx[k]) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) if (idx[k] >= 0) sv[i + k * nth] = v[k];
    }
    __syncthreads();
    if (tr && tid == 0) tr[5] = gtimer();
    mbar_wait(bar, parity);
    parity ^= 1u;
    if (tr && tid == 0) tr[6] = gtimer();
    const int32_t* sord = sptr + r0.y + 1;      // processing order: longest contribution lists first
    for (int db = tid; db < r0.y; db += 4 * nth) {
        int q[4], qe[4], od[4];
        uint32_t pr[4];
        double s[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int d = db + k * nth;
            od[k] = d < r0.y ? sord[d] : -1;
            q[k] = od[k] >= 0 ? sptr[od[k]] : 0; qe[k] = od[k] >= 0 ? sptr[od[k] + 1] : 0; s[k] = 0.0;
            pr[k] = q[k] < qe[k] ? spair[q[k]] : 0u;
        }
        // ranks db, db + nth, ... are in decreasing length order: list 0 of the interleave is the longest, list 3
        // the shortest.  The interleave narrows as the short lists run out (4, 3, 2, then 1 list per round), so
        // the long tail of list 0 does not keep issuing the (predicated-off) shared-memory loads of the others.
        acc_rounds<4>(sv, spair, q, qe, pr, s);
        acc_rounds<3>(sv, spair, q, qe, pr, s);
        acc_rounds<2>(sv, spair, q, qe, pr, s);
        acc_rounds<1>(sv, spair, q, qe, pr, s);
#pragma unroll
        for (int k = 0; k < 4; ++k) if (od[k] >= 0) ap.out[r0.x + od[k]] = s[k];
    }
}

// State update of variable v; returns |dx| as ordered bits (NaN sorts above inf).
__device__ __forceinline__ unsigned long long update_var(const int32_t* __restrict__ bus, const int32_t* __restrict__ quant,
                                                         const int32_t* __restrict__ pos, int v, const double* xsol,
                                                         double* va, double* vm) {
    const double dx = ldc(xsol + pos[v]);
    double* dst = (quant[v] == 0 ? va : vm) + bus[v];
    *dst = ldc(dst) + dx;
    return (unsigned long long)__double_as_longlong(fabs(dx));
}

// w (z - h(x))^2 of measurement row r (eval_h_all arithmetic: the diagonal term sits inside the
// neighbor sum)   [solver.py:100-103, measurement.py:338-387]
__device__ __forceinline__ double objective_row(const EvalProg& ep, const int32_t* __restrict__ m_type,
                                                const int32_t* __restrict__ m_target, const int32_t* __restrict__ br_from,
                                                const int32_t* __restrict__ br_to, int r, const double* va, const double* vm) {
    const int t = m_type[r], tg = m_target[r];
    double h;
    if (t == 0) h = ldc(vm + tg);
    else if (t <= 2) {
        double acc = 0.0;
        for (int p = ep.y_ptr[tg]; p < ep.y_ptr[tg + 1]; ++p) {
            const int j = ep.y_idx[p];
            double sn, cs;
            sincos(ldc(va + tg) - ldc(va + j), &sn, &cs);
            acc += (t == 1) ? ldc(vm + j) * (ep.y_g[p] * cs + ep.y_b[p] * sn) : ldc(vm + j) * (ep.y_g[p] * sn - ep.y_b[p] * cs);
        }
        h = ldc(vm + tg) * acc;
    } else {
        const int f = br_from[tg], tt = br_to[tg];
        const double* y = ep.br_y + 8 * (size_t)tg;
        const bool fe = (t == 3 || t == 5 || t == 7);
        const int ob = fe ? f : tt, ub = fe ? tt : f;
        const double a = fe ? y[0] : y[6], b = fe ? y[1] : y[7], c = fe ? y[2] : y[4], d = fe ? y[3] : y[5];
        double sn, cs;
        sincos(ldc(va + ob) - ldc(va + ub), &sn, &cs);
        const double vo = ldc(vm + ob), vu = ldc(vm + ub);
        if (t >= 7) {
            const double m2 = (a * a + b * b) * vo * vo + (c * c + d * d) * vu * vu
                              + 2.0 * vo * vu * ((a * c + b * d) * cs - (b * c - a * d) * sn);
            h = sqrt(fmax(m2, 0.0));
        } else
        h = (t >= 5) ? vo * (-vo * b + vu * (c * sn - d * cs)) : vo * (vo * a + vu * (c * cs + d * sn));
    }
        const double res = ep.z[r] - h;
    return ep.w[r] * res * res;
}

}  // namespace gse
