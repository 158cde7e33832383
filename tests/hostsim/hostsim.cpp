// hostsim.cpp -- TEST-ONLY host interpreter of the device program (HostProgram).
//
// Not part of the product and never loaded by it: tests/test_symbolic_hostsim.py builds this
// file together with csrc/symbolic.cpp and walks the exact task lists, region tables, child
// index maps and contribution programs the CUDA kernels consume, in plain C++.  It lets the
// CPU-only test tier validate the plan-time analysis (ordering, fronts, extend-add maps,
// accumulation program) against the oracle without a GPU.  The arithmetic mirrors
// csrc/kernels.cu step for step.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2604_23175_b200/csrc/plan.hpp"

using namespace gse;

namespace {

struct Sim {
    HostProgram hp;
    gse_problem_desc d;
    std::vector<double> val, gval, lbuf, ubuf, xsol, w;   // val = [(g, w*g) per slot | w*r]
    long long fail_code = -1;
};

inline int pad_ld(int p) { return ((p + 11) / 16) * 16 + 4; }

void put(Sim& s, int slot, double gv, double w, double) { s.val[2 * slot] = gv; s.val[2 * slot + 1] = w * gv; }
void put_wr(Sim& s, int row, double wr) { if (row >= 0) s.val[2 * s.hp.n_slots + row] = wr; }

void flow_row(Sim& s, int row, int slot, bool fs, bool ts, double h, double a, double b, double c, double e) {
    if (row < 0) return;
    double w = s.w[row], wr = w * (s.d.m_z[row] - h);
    put_wr(s, row, wr);
    if (!fs) put(s, slot++, a, w, wr);
    if (!ts) put(s, slot++, b, w, wr);
    put(s, slot++, c, w, wr); put(s, slot, e, w, wr);
}

void eval(Sim& s, const double* va, const double* vm) {
    const HostProgram& hp = s.hp; const gse_problem_desc& d = s.d;
    for (size_t u = 0; u < hp.fl_branch.size(); ++u) {
        int e = hp.fl_branch[u], f = hp.fl_from[u], t = hp.fl_to[u];
        const double* y = d.br_y + 8 * (size_t)e;
        double vf = vm[f], vt = vm[t], sn = std::sin(va[f] - va[t]), cs = std::cos(va[f] - va[t]);
        bool fs = f == d.slack, ts = t == d.slack;
        const int32_t* rows = &hp.fl_row[8 * u]; const int32_t* sl = &hp.fl_slot[8 * u];
        { double a = y[0], b = y[1], c = y[2], dd = y[3], ec = c * cs + dd * sn, es = c * sn - dd * cs, vv = vf * vt;
          flow_row(s, rows[0], sl[0], fs, ts, vf * (vf * a + vt * ec), -vv * es, vv * es, 2.0 * vf * a + vt * ec, vf * ec);
          flow_row(s, rows[2], sl[2], fs, ts, vf * (-vf * b + vt * es), vv * ec, -vv * ec, -2.0 * vf * b + vt * es, vf * es); }
        { double a = y[6], b = y[7], c = y[4], dd = y[5], ec = c * cs - dd * sn, es = -c * sn - dd * cs, vv = vf * vt;
          flow_row(s, rows[1], sl[1], fs, ts, vt * (vt * a + vf * ec), vv * es, -vv * es, vt * ec, 2.0 * vt * a + vf * ec);
          flow_row(s, rows[3], sl[3], fs, ts, vt * (-vt * b + vf * es), -vv * ec, vv * ec, vt * es, -2.0 * vt * b + vf * es); }
        // current magnitudes at the from / to end (unit_bodies.cuh)
        if (rows[4] >= 0) { double a = y[0], b = y[1], c = y[2], dd = y[3], al = a * c + b * dd, be = b * c - a * dd, A = a * a + b * b, C = c * c + dd * dd;
          double E = al * cs - be * sn, vv = vf * vt, m2 = A * vf * vf + C * vt * vt + 2.0 * vv * E, h = std::sqrt(std::max(m2, 0.0)), ih = m2 > 1e-24 ? 1.0 / h : 0.0;
          double dth = vv * (-al * sn - be * cs) * ih;
          flow_row(s, rows[4], sl[4], fs, ts, h, dth, -dth, (A * vf + vt * E) * ih, (C * vt + vf * E) * ih); }
        if (rows[5] >= 0) { double a = y[6], b = y[7], c = y[4], dd = y[5], al = a * c + b * dd, be = b * c - a * dd, A = a * a + b * b, C = c * c + dd * dd;
          double E = al * cs + be * sn, vv = vf * vt, m2 = A * vt * vt + C * vf * vf + 2.0 * vv * E, h = std::sqrt(std::max(m2, 0.0)), ih = m2 > 1e-24 ? 1.0 / h : 0.0;
          double dtt = vv * (al * sn - be * cs) * ih;
          flow_row(s, rows[5], sl[5], fs, ts, h, -dtt, dtt, (C * vf + vt * E) * ih, (A * vt + vf * E) * ih); }
    }
    for (size_t u = 0; u < hp.inj_bus.size(); ++u) {
        int i = hp.inj_bus[u], rp = hp.inj_rowp[u], rq = hp.inj_rowq[u], sp = hp.inj_slotp[u], sq = hp.inj_slotq[u];
        int p0 = d.y_ptr[i], p1 = d.y_ptr[i + 1], nth = 0;
        for (int p = p0; p < p1; ++p) nth += d.y_idx[p] != d.slack;
        double vi = vm[i], sum_p = 0, sum_q = 0, gd = 0, bd = 0;
        for (int p = p0; p < p1; ++p) { int j = d.y_idx[p]; if (j == i) { gd = d.y_g[p]; bd = d.y_b[p]; continue; }
            double th = va[i] - va[j], sn = std::sin(th), cs = std::cos(th);
            sum_p += vm[j] * (d.y_g[p] * cs + d.y_b[p] * sn); sum_q += vm[j] * (d.y_g[p] * sn - d.y_b[p] * cs); }
        double wp = rp >= 0 ? s.w[rp] : 0, wq = rq >= 0 ? s.w[rq] : 0;
        double hpv = vi * (vi * gd + sum_p), hq = vi * (-vi * bd + sum_q);
        double wrp = rp >= 0 ? wp * (d.m_z[rp] - hpv) : 0, wrq = rq >= 0 ? wq * (d.m_z[rq] - hq) : 0;
        put_wr(s, rp, wrp); put_wr(s, rq, wrq);
        int cth = 0, dth = -1, dvm = -1;
        for (int p = p0, q = 0; p < p1; ++p, ++q) { int j = d.y_idx[p]; int thpos = j != d.slack ? cth++ : -1, vmpos = nth + q;
            if (j == i) { dth = thpos; dvm = vmpos; continue; }
            double th = va[i] - va[j], sn = std::sin(th), cs = std::cos(th), vj = vm[j];
            double uc = d.y_g[p] * cs + d.y_b[p] * sn, us = d.y_g[p] * sn - d.y_b[p] * cs;
            if (rp >= 0) { if (thpos >= 0) put(s, sp + thpos, vi * (vj * us), wp, wrp); put(s, sp + vmpos, vi * uc, wp, wrp); }
            if (rq >= 0) { if (thpos >= 0) put(s, sq + thpos, -vi * (vj * uc), wq, wrq); put(s, sq + vmpos, vi * us, wq, wrq); } }
        if (rp >= 0) { if (dth >= 0) put(s, sp + dth, -vi * sum_q, wp, wrp); put(s, sp + dvm, 2.0 * vi * gd + sum_p, wp, wrp); }
        if (rq >= 0) { if (dth >= 0) put(s, sq + dth, vi * sum_p, wq, wrq); put(s, sq + dvm, -2.0 * vi * bd + sum_q, wq, wrq); }
    }
    for (size_t u = 0; u < hp.vm_bus.size(); ++u) { int row = hp.vm_row[u]; double w = s.w[row];
        put_wr(s, row, w * (d.m_z[row] - vm[hp.vm_bus[u]]));
        put(s, hp.vm_slot[u], 1.0, w, 0.0); }
}

void accumulate(Sim& s, const std::vector<int32_t>& ptr, const std::vector<int32_t>& a, const std::vector<int32_t>& b, std::vector<double>& out) {
    for (size_t dd = 0; dd + 1 < ptr.size(); ++dd) { double acc = 0;
        for (int q = ptr[dd]; q < ptr[dd + 1]; ++q) acc += s.val[a[q]] * s.val[b[q]];
        out[dd] = acc; }
}

// the staged form of the solver-layout program, item by item as the CUDA kernel walks it
void accumulate_staged(Sim& s, std::vector<double>& out) {
    const HostProgram& hp = s.hp;
    std::vector<double> sv;
    for (size_t it = 0; it * 8 < hp.acc_items.size(); ++it) {
        const int32_t* r = &hp.acc_items[8 * it];
        const int d0 = r[0], nd = r[1], u0 = r[2], nu = r[3], p0 = r[4], l0 = r[6];
        sv.assign(nu, 0.0);
        for (int i = 0; i < nu; ++i) sv[i] = s.val[hp.acc_uniq[u0 + i]];
        for (int k = 0; k < nd; ++k) { double acc = 0;
            const int dd = hp.acc_lptr[l0 + nd + 1 + k];   // processing order (a permutation of the item's destinations)
            for (int q = hp.acc_lptr[l0 + dd]; q < hp.acc_lptr[l0 + dd + 1]; ++q) { uint32_t pr = hp.acc_pair[p0 + q]; acc += sv[pr & 0xffffu] * sv[pr >> 16]; }
            out[d0 + dd] = acc; }
    }
}

void run_task(Sim& s, const Task& tk, int fidx_unused = 0) {
    (void)fidx_unused;
    const HostProgram& hp = s.hp; const Front& f = hp.fronts[tk.front];
    const int p = f.p, u1 = f.u1, T = std::max(f.T, 1), ci = tk.ci, cj = tk.cj;
    const int i0 = ci * T, ni = std::min(T, u1 - i0), j0 = cj * T, nj = std::min(T, u1 - j0);
    const bool diag = ci == cj; const int ld = pad_ld(p);
    const int kind = tk.kind;   // 0 fused, 1 panel (factor + solve chunk I, store), 2 update (panels read back from lbuf)
    std::vector<double> PP((size_t)p * ld, 0.0), PI((size_t)ni * ld, 0.0), PJ((size_t)(diag ? 0 : nj) * ld, 0.0), tile((size_t)ni * nj, 0.0);
    const int32_t* rptr = &hp.reg_ptr[hp.front_reg_off[tk.front]];
    auto region = [&](int rid, auto&& fn) { for (int e = rptr[rid]; e < rptr[rid + 1]; ++e) { uint32_t q = hp.orig_pos[f.gval_off + e]; fn((int)(q >> 16), (int)(q & 0xffff), s.gval[f.gval_off + e]); } };
    if (p && kind != 2) {
        region(0, [&](int lr, int lc, double v) { PP[(size_t)lr * ld + lc] = v; });
        region((ci + 1) * (ci + 2) / 2, [&](int lr, int lc, double v) { PI[(size_t)(lr - p - i0) * ld + lc] = v; });
        if (!diag) region((cj + 1) * (cj + 2) / 2, [&](int lr, int lc, double v) { PJ[(size_t)(lr - p - j0) * ld + lc] = v; });
    }
    if (kind != 1) region((ci + 1) * (ci + 2) / 2 + cj + 1, [&](int lr, int lc, double v) { tile[(size_t)(lr - p - i0) * nj + (lc - p - j0)] = v; });
    for (size_t cx = 0; cx < f.children.size(); ++cx) {
        const int ch = f.children[cx];
        const Front& c = hp.fronts[ch];
        const std::vector<int>& rel = (cx < f.child_rel.size() && f.child_rel[cx] >= 0) ? hp.extra_rel[f.child_rel[cx]] : c.rel;
        const double* U = &s.ubuf[c.u_off];
        auto lb = [&](int key) { return (int)(std::lower_bound(rel.begin(), rel.end(), key) - rel.begin()); };
        int eP = lb(p), bI = lb(p + i0), eI = lb(p + i0 + ni), bJ = lb(p + j0), eJ = lb(p + j0 + nj);
        auto add = [&](int r0, int r1, int c0, int c1, double* dst, int ldd, int rs, int cs) {
            for (int i = r0; i < r1; ++i) for (int j = c0; j < c1 && j <= i; ++j) dst[(size_t)(rel[i] - rs) * ldd + (rel[j] - cs)] += U[(size_t)i * (i + 1) / 2 + j]; };
        if (p && kind != 2) { add(0, eP, 0, eP, PP.data(), ld, 0, 0); add(bI, eI, 0, eP, PI.data(), ld, p + i0, 0); if (!diag) add(bJ, eJ, 0, eP, PJ.data(), ld, p + j0, 0); }
        if (kind != 1) add(bI, eI, bJ, eJ, tile.data(), nj, p + i0, p + j0);
    }
    if (p && kind == 2) {   // the front's stored panels
        const double* L = &s.lbuf[f.l_off];
        for (int r = 0; r < ni; ++r) for (int k = 0; k < p; ++k) PI[(size_t)r * ld + k] = L[(size_t)(p + i0 + r) * p + k];
        if (!diag) for (int r = 0; r < nj; ++r) for (int k = 0; k < p; ++k) PJ[(size_t)r * ld + k] = L[(size_t)(p + j0 + r) * p + k];
    }
    if (p && kind != 2) {   // left-looking row Cholesky over [PP; PI; PJ]
        auto row = [&](int r) -> double* { return r < p ? &PP[(size_t)r * ld] : r < p + ni ? &PI[(size_t)(r - p) * ld] : &PJ[(size_t)(r - p - ni) * ld]; };
        const int R = p + ni + (diag ? 0 : nj);
        for (int k = 0; k < p; ++k) {
            double* lk = row(k); double dsum = lk[k];
            for (int j = 0; j < k; ++j) dsum -= lk[j] * lk[j];
            if (!(dsum > 0.0)) { long long code = ((long long)tk.front << 32) | k; if (s.fail_code < 0 || code < s.fail_code) s.fail_code = code; }
            lk[k] = std::sqrt(dsum);
            for (int r = k + 1; r < R; ++r) { double* x = row(r); double acc = x[k]; for (int j = 0; j < k; ++j) acc -= x[j] * lk[j]; x[k] = acc / lk[k]; }
        }
        for (int r = 0; r < p; ++r) for (int k = r + 1; k < p; ++k) PP[(size_t)r * ld + k] = 0.0;
    }
    double* U = &s.ubuf[f.u_off];
    const std::vector<double>& PJJ = diag ? PI : PJ;
    if (kind != 1) for (int i = 0; i < ni; ++i) for (int j = 0; j < nj; ++j) { int I = i0 + i, J = j0 + j; if (J > I) continue;
        double acc = 0; for (int k = 0; k < p; ++k) acc += PI[(size_t)i * ld + k] * PJJ[(size_t)j * ld + k];
        U[(size_t)I * (I + 1) / 2 + J] = tile[(size_t)i * nj + j] - acc; }
    if (p && diag && kind != 2) { double* L = &s.lbuf[f.l_off];
        if (ci == 0) for (int r = 0; r < p; ++r) for (int k = 0; k < p; ++k) L[(size_t)r * p + k] = PP[(size_t)r * ld + k];
        for (int r = 0; r < ni; ++r) for (int k = 0; k < p; ++k) L[(size_t)(p + i0 + r) * p + k] = PI[(size_t)r * ld + k]; }
}

void backward(Sim& s, int fi) {
    const Front& f = s.hp.fronts[fi]; const int p = f.p, u = f.u1 - 1; const double* L = &s.lbuf[f.l_off];
    std::vector<double> t(p);
    for (int k = 0; k < p; ++k) { double acc = 0; for (int i = 0; i < u; ++i) acc += L[(size_t)(p + i) * p + k] * s.xsol[f.rows[p + i]]; t[k] = L[(size_t)(p + u) * p + k] - acc; }
    for (int c = p - 1; c >= 0; --c) { t[c] /= L[(size_t)c * p + c]; for (int j = 0; j < c; ++j) t[j] -= L[(size_t)c * p + j] * t[c]; }
    for (int k = 0; k < p; ++k) s.xsol[f.rows[k]] = t[k];
}

}  // namespace

extern "C" {

void* hostsim_create(const gse_problem_desc* d, int dense, int leaf, int pmax, int rank, int world, const int32_t* area_rank, char* msg, int msglen, int boundary_mode) {
    Sim* s = new Sim(); s->d = *d;
    BuildOptions bo; bo.dense = dense != 0; if (leaf > 0) bo.leaf_buses = leaf; if (pmax == 32 || pmax == 64) bo.max_pivots = pmax;
    bo.rank = rank; bo.world = std::max(1, world); bo.boundary_mode = boundary_mode;
    if (const char* e = getenv("GSE_SEPW")) bo.sep_weight = atof(e);
    if (const char* e = getenv("GSE_GAMMA_SEPW")) bo.gamma_sep_weight = atof(e);
    if (const char* e = getenv("GSE_GAMMA_LEAF")) bo.gamma_leaf_buses = atoi(e);
    if (const char* e = getenv("GSE_LEAF_BUSES")) bo.leaf_buses = atoi(e);
    if (const char* e = getenv("GSE_INTERIOR_MERGE")) bo.interior_merge = atof(e);
    if (const char* e = getenv("GSE_GAMMA_MERGE")) bo.gamma_merge = atof(e);
    if (area_rank) bo.area_rank.assign(area_rank, area_rank + d->n_areas);
    std::string e = build_host_program(*d, bo, s->hp);
    if (!e.empty()) { snprintf(msg, msglen, "%s", e.c_str()); delete s; return nullptr; }
    const HostProgram& hp = s->hp;
    s->val.assign(hp.n_val, 0);
    s->gval.assign(hp.n_gval, 0); s->lbuf.assign(hp.n_lbuf, 0); s->ubuf.assign(hp.n_ubuf, 0); s->xsol.assign(hp.n_pos + 2, 0);
    s->w.assign(d->m_w, d->m_w + d->n_rows);
    return s;
}
void hostsim_destroy(void* h) { delete (Sim*)h; }
void hostsim_stats(void* h, double* out) { Sim* s = (Sim*)h; const HostProgram& hp = s->hp;
    out[0] = (double)hp.fronts.size(); out[1] = (double)hp.fwd_levels.size(); out[2] = hp.max_front; out[3] = (double)hp.n_lbuf;
    out[4] = (double)hp.n_ubuf; out[5] = (double)hp.n_pairs; out[6] = (double)hp.n_gval; out[7] = hp.dense_flops;
    size_t nt = 0; for (auto& l : hp.fwd_levels) nt += l.size(); out[8] = (double)nt; out[9] = (double)hp.bwd_levels.size();
    // sequential pivots on the longest leaf-to-root chain (total, and inside the boundary fronts)
    std::vector<double> path(hp.fronts.size(), 0.0), gpath(hp.fronts.size(), 0.0);
    double best = 0, gbest = 0;
    for (size_t f = 0; f < hp.fronts.size(); ++f) {     // children precede parents in front order? not guaranteed: iterate by level
    }
    std::vector<int> order(hp.fronts.size()); for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return hp.fronts[a].level < hp.fronts[b].level; });
    for (int f : order) { const Front& fr = hp.fronts[f];
        double c = 0, gc = 0; for (int ch : fr.children) { c = std::max(c, path[ch]); gc = std::max(gc, gpath[ch]); }
        path[f] = c + fr.p; gpath[f] = gc + (fr.kind == 3 ? fr.p : 0);
        best = std::max(best, path[f]); gbest = std::max(gbest, gpath[f]); }
    out[10] = best; out[11] = gbest; }
// one outer iteration; returns failure code or -1
long long hostsim_iterate(void* h, double* va, double* vm, double* delta_inf) {
    Sim* s = (Sim*)h; const HostProgram& hp = s->hp; s->fail_code = -1;
    eval(*s, va, vm);
    accumulate_staged(*s, s->gval);
    for (auto& lv : hp.fwd_levels) for (const Task& t : lv) run_task(*s, t);
    for (auto& lv : hp.bwd_levels) for (int f : lv) backward(*s, f);
    double dmax = 0;
    for (size_t v = 0; v < hp.upd_bus.size(); ++v) { double dx = s->xsol[hp.upd_pos[v]]; (hp.upd_quant[v] == 0 ? va : vm)[hp.upd_bus[v]] += dx; dmax = std::max(dmax, std::fabs(dx)); }
    *delta_inf = dmax;
    return s->fail_code;
}
// packed (S_b | b_hat) of an area after hostsim_iterate, unpacked to full
void hostsim_area_schur(void* h, int a, double* s_b, double* b_hat) {
    Sim* s = (Sim*)h; const Front& f = s->hp.fronts[s->hp.area_root[a]]; int n = s->hp.area_nb[a]; const double* U = &s->ubuf[f.u_off];
    const std::vector<int>& pos = s->hp.area_bpos[a];   // local boundary variable -> row of the root
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { int qi = std::max(pos[i], pos[j]), qj = std::min(pos[i], pos[j]); s_b[(size_t)i * n + j] = U[(size_t)qi * (qi + 1) / 2 + qj]; }
    for (int j = 0; j < n; ++j) b_hat[j] = U[(size_t)n * (n + 1) / 2 + pos[j]];
}
void hostsim_ref_blocks(void* h, double* out) {   // reference-layout values of all areas, concatenated
    Sim* s = (Sim*)h; std::vector<double> v(s->hp.n_ref_vals);
    build_reference_program(s->hp);
    accumulate(*s, s->hp.racc_ptr, s->hp.racc_a, s->hp.racc_b, v);
    memcpy(out, v.data(), v.size() * sizeof(double));
}
long long hostsim_n_ref(void* h) { return ((Sim*)h)->hp.n_ref_vals; }
void hostsim_ref_off(void* h, long long* off) { Sim* s = (Sim*)h; for (size_t i = 0; i < s->hp.ref_off.size(); ++i) off[i] = s->hp.ref_off[i]; }
}
