/*
 * mase_oracle.c -- CPU ORACLE for the multi-area WLS Gauss-Newton solve.
 *
 * TEST INFRASTRUCTURE ONLY.  This file restates, in plain C, the algorithm of
 * the reference package (/root/reference/pkg/src/gridse) for the hot path named
 * by BASELINE.json.  It is imported only by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs; the product
 * (paper_2604_23175_b200/) never links, loads or calls it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks this oracle against
 * fixtures produced by importing the unmodified reference
 * (tests/golden/make_golden.py) -- iteration counts, per-iteration update
 * norms, final states, objectives, per-area normal blocks, Schur blocks and
 * the boundary system -- and against the reference tests' hand values.
 *
 * Reference functions restated (file:line under pkg/src/gridse):
 *   build_variable_maps        partition.py:478-538   -> build_maps()
 *   area_row_ids/build_patterns assembly.py:166-400    -> build_rows(), build_pattern()
 *   _eval_blocks               assembly.py:427-483     -> eval_rows()
 *   fused_accumulate           assembly.py:486-524     -> accumulate()
 *   _min_degree_order          linalg.py:68-92         -> min_degree()
 *   _etree / _ereach           linalg.py:95-129        -> etree(), ereach()
 *   SparseCholeskyCache._analyze linalg.py:156-231     -> chol_analyze()
 *   refactor                   linalg.py:292-332       -> chol_refactor()
 *   forward / backward         linalg.py:340-383       -> chol_forward*(), chol_backward()
 *   schur_condense             linalg.py:410-424       -> condense()
 *   interior_recover           linalg.py:427-434       -> recover()
 *   assemble_boundary          solver.py:106-119       -> orc_boundary()
 *   dense_cholesky_solve       linalg.py:46-61         -> dense_chol(), dense_solve()
 *   solve_multiarea            solver.py:204-346       -> orc_solve()
 *   objective / eval_h_all     solver.py:100-103, measurement.py:338-387 -> orc_objective()
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (oracle/Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t n_bus, n_branch, n_rows, n_areas, slack, dense_threshold;
    double slack_va;
    const int32_t *y_ptr, *y_idx;
    const double *y_g, *y_b;
    const int32_t *br_from, *br_to;
    const double *br_y; /* [n_branch][8] ff.re ff.im ft.re ft.im tf.re tf.im tt.re tt.im */
    const int32_t *m_type, *m_target;
    const double *m_z, *m_w;
    const int32_t *area_of_bus;
} orc_desc;

typedef struct {
    int n, dense;
    int *pat_ptr, *pat_idx; /* analysed CSR pattern (borrowed) */
    int *perm, *c_ptr, *c_rows, *c_src, *parent;
    int *Lp, *Li, *row_ptr, *prog_col;
    int *fillcnt;
    double *Lx, *x, *dn; /* dn: dense lower factor n*n row-major */
} chol_t;

typedef struct {
    int n_i, n_b, n_ia, n_ba, n_int_bus, n_lb;
    int *int_bus, *ia_bus, *lb_bus, *ba_bus, *sel;
    int n_rows, *row_ids, *slot_ptr, *slot_var, n_slots;
    int *ii_ptr, *ii_idx, *ib_ptr, *ib_idx, nnz_ii, nnz_ib;
    double *data_ii, *data_ib, *g_bb, *b_i, *b_b, *g_flat, *resid;
    chol_t ch;
    double *s_b, *b_hat, *dxi, *zmat, *wvec;
    int fail_pivot;
} area_t;

typedef struct {
    orc_desc d;
    int n_gamma, n_ga;
    int *gamma_bus;   /* [n_gamma] bus of each slot */
    int *g_angle_slot, *g_mag_slot; /* per bus, -1 */
    area_t *areas;
    double *s_gamma, *b_gamma, *dx_gamma;
    int err_area, err_pivot, err_kind; /* kind 1 = area block, 2 = boundary */
} orc_t;

static void *xcalloc(size_t n, size_t s) { void *p = calloc(n ? n : 1, s); if (!p) abort(); return p; }

/* ------------------------------------------------------------------ maps */

static int cmp_int(const void *a, const void *b) { int x = *(const int *)a, y = *(const int *)b; return (x > y) - (x < y); }

static void build_maps(orc_t *o) {
    const orc_desc *d = &o->d;
    int nb = d->n_bus, K = d->n_areas;
    char *isb = xcalloc(nb, 1);
    for (int e = 0; e < d->n_branch; e++) {
        int f = d->br_from[e], t = d->br_to[e];
        if (d->area_of_bus[f] != d->area_of_bus[t]) isb[f] = isb[t] = 1;
    }
    o->g_angle_slot = xcalloc(nb, sizeof(int));
    o->g_mag_slot = xcalloc(nb, sizeof(int));
    int na = 0, nm = 0;
    for (int b = 0; b < nb; b++) { o->g_angle_slot[b] = o->g_mag_slot[b] = -1; }
    for (int b = 0; b < nb; b++) if (isb[b] && b != d->slack) o->g_angle_slot[b] = na++;
    for (int b = 0; b < nb; b++) if (isb[b]) o->g_mag_slot[b] = na + nm++;
    o->n_ga = na; o->n_gamma = na + nm;
    o->gamma_bus = xcalloc(o->n_gamma, sizeof(int));
    for (int b = 0; b < nb; b++) {
        if (o->g_angle_slot[b] >= 0) o->gamma_bus[o->g_angle_slot[b]] = b;
        if (o->g_mag_slot[b] >= 0) o->gamma_bus[o->g_mag_slot[b]] = b;
    }
    o->areas = xcalloc(K, sizeof(area_t));
    /* local boundary = own boundary buses + far ends of tie lines */
    int *cnt = xcalloc(K, sizeof(int));
    for (int b = 0; b < nb; b++) if (isb[b]) cnt[d->area_of_bus[b]]++;
    for (int e = 0; e < d->n_branch; e++) {
        int f = d->br_from[e], t = d->br_to[e];
        int af = d->area_of_bus[f], at = d->area_of_bus[t];
        if (af != at) { cnt[af]++; cnt[at]++; }
    }
    int **lists = xcalloc(K, sizeof(int *));
    int *fill = xcalloc(K, sizeof(int));
    for (int a = 0; a < K; a++) lists[a] = xcalloc(cnt[a], sizeof(int));
    for (int b = 0; b < nb; b++) if (isb[b]) { int a = d->area_of_bus[b]; lists[a][fill[a]++] = b; }
    for (int e = 0; e < d->n_branch; e++) {
        int f = d->br_from[e], t = d->br_to[e];
        int af = d->area_of_bus[f], at = d->area_of_bus[t];
        if (af != at) { lists[af][fill[af]++] = t; lists[at][fill[at]++] = f; }
    }
    for (int a = 0; a < K; a++) {
        area_t *A = &o->areas[a];
        qsort(lists[a], fill[a], sizeof(int), cmp_int);
        int m = 0;
        for (int i = 0; i < fill[a]; i++) if (i == 0 || lists[a][i] != lists[a][i - 1]) lists[a][m++] = lists[a][i];
        A->n_lb = m; A->lb_bus = lists[a];
        A->ba_bus = xcalloc(m, sizeof(int));
        for (int i = 0; i < m; i++) if (A->lb_bus[i] != d->slack) A->ba_bus[A->n_ba++] = A->lb_bus[i];
        A->n_b = A->n_ba + m;
        A->sel = xcalloc(A->n_b, sizeof(int));
        for (int i = 0; i < A->n_ba; i++) A->sel[i] = o->g_angle_slot[A->ba_bus[i]];
        for (int i = 0; i < m; i++) A->sel[A->n_ba + i] = o->g_mag_slot[A->lb_bus[i]];
        int ni = 0;
        for (int b = 0; b < nb; b++) if (d->area_of_bus[b] == a && !isb[b]) ni++;
        A->int_bus = xcalloc(ni, sizeof(int)); A->ia_bus = xcalloc(ni, sizeof(int));
        for (int b = 0; b < nb; b++) if (d->area_of_bus[b] == a && !isb[b]) {
            A->int_bus[A->n_int_bus++] = b;
            if (b != d->slack) A->ia_bus[A->n_ia++] = b;
        }
        A->n_i = A->n_ia + A->n_int_bus;
    }
    free(cnt); free(fill); free(lists); free(isb);
}

/* ------------------------------------------------- templates and patterns */

typedef struct { long code; } code_t;
static int cmp_long(const void *a, const void *b) { long x = *(const long *)a, y = *(const long *)b; return (x > y) - (x < y); }

static void build_pattern(orc_t *o, int a, int *loc_va, int *loc_vm) {
    const orc_desc *d = &o->d;
    area_t *A = &o->areas[a];
    int ni = A->n_i, nb = A->n_b;
    for (int i = 0; i < A->n_ia; i++) loc_va[A->ia_bus[i]] = i;
    for (int i = 0; i < A->n_int_bus; i++) loc_vm[A->int_bus[i]] = A->n_ia + i;
    for (int i = 0; i < A->n_ba; i++) loc_va[A->ba_bus[i]] = ni + i;
    for (int i = 0; i < A->n_lb; i++) loc_vm[A->lb_bus[i]] = ni + A->n_ba + i;

    int nr = 0;
    for (int r = 0; r < d->n_rows; r++) {
        int t = d->m_type[r], tg = d->m_target[r];
        int owner = t >= 3 ? d->br_from[tg] : tg;
        if (d->area_of_bus[owner] == a) nr++;
    }
    A->n_rows = nr; A->row_ids = xcalloc(nr, sizeof(int)); A->slot_ptr = xcalloc(nr + 1, sizeof(int));
    nr = 0; long ns = 0;
    for (int r = 0; r < d->n_rows; r++) {
        int t = d->m_type[r], tg = d->m_target[r];
        int owner = t >= 3 ? d->br_from[tg] : tg;
        if (d->area_of_bus[owner] != a) continue;
        A->row_ids[nr] = r;
        int s;
        if (t == 0) s = 1;
        else if (t <= 2) { int deg = d->y_ptr[tg + 1] - d->y_ptr[tg]; s = 2 * deg; for (int p = d->y_ptr[tg]; p < d->y_ptr[tg + 1]; p++) if (d->y_idx[p] == d->slack) s--; }
        else { s = 4; if (d->br_from[tg] == d->slack) s--; if (d->br_to[tg] == d->slack) s--; }
        ns += s; nr++; A->slot_ptr[nr] = (int)ns;
    }
    A->n_slots = (int)ns; A->slot_var = xcalloc(ns, sizeof(int));
    for (int k = 0; k < A->n_rows; k++) {
        int r = A->row_ids[k], t = d->m_type[r], tg = d->m_target[r];
        int *sv = A->slot_var + A->slot_ptr[k]; int c = 0;
        if (t == 0) sv[c++] = loc_vm[tg];
        else if (t <= 2) {
            for (int p = d->y_ptr[tg]; p < d->y_ptr[tg + 1]; p++) if (d->y_idx[p] != d->slack) sv[c++] = loc_va[d->y_idx[p]];
            for (int p = d->y_ptr[tg]; p < d->y_ptr[tg + 1]; p++) sv[c++] = loc_vm[d->y_idx[p]];
        } else {
            int f = d->br_from[tg], tt = d->br_to[tg];
            if (f != d->slack) sv[c++] = loc_va[f];
            if (tt != d->slack) sv[c++] = loc_va[tt];
            sv[c++] = loc_vm[f]; sv[c++] = loc_vm[tt];
        }
    }
    /* CSR patterns of g_ii and g_ib from the template pairs */
    long tot_ii = 0, tot_ib = 0;
    for (int k = 0; k < A->n_rows; k++) {
        int s0 = A->slot_ptr[k], s1 = A->slot_ptr[k + 1]; long ci = 0, cb = 0;
        for (int s = s0; s < s1; s++) { if (A->slot_var[s] < ni) ci++; else cb++; }
        tot_ii += ci * ci; tot_ib += ci * cb;
    }
    long *cii = xcalloc(tot_ii, sizeof(long)), *cib = xcalloc(tot_ib, sizeof(long));
    long pi = 0, pb = 0;
    for (int k = 0; k < A->n_rows; k++) {
        int s0 = A->slot_ptr[k], s1 = A->slot_ptr[k + 1];
        for (int x = s0; x < s1; x++) { int va = A->slot_var[x]; if (va >= ni) continue;
            for (int y = s0; y < s1; y++) { int vb = A->slot_var[y];
                if (vb < ni) cii[pi++] = (long)va * (ni > 0 ? ni : 1) + vb; else cib[pb++] = (long)va * (nb > 0 ? nb : 1) + (vb - ni); } }
    }
    qsort(cii, tot_ii, sizeof(long), cmp_long); qsort(cib, tot_ib, sizeof(long), cmp_long);
    long u = 0; for (long i = 0; i < tot_ii; i++) if (i == 0 || cii[i] != cii[i - 1]) cii[u++] = cii[i];
    A->nnz_ii = (int)u; A->ii_ptr = xcalloc(ni + 1, sizeof(int)); A->ii_idx = xcalloc(u, sizeof(int));
    for (long i = 0; i < u; i++) { int r = (int)(cii[i] / (ni > 0 ? ni : 1)); A->ii_ptr[r + 1]++; A->ii_idx[i] = (int)(cii[i] % (ni > 0 ? ni : 1)); }
    for (int i = 0; i < ni; i++) A->ii_ptr[i + 1] += A->ii_ptr[i];
    u = 0; for (long i = 0; i < tot_ib; i++) if (i == 0 || cib[i] != cib[i - 1]) cib[u++] = cib[i];
    A->nnz_ib = (int)u; A->ib_ptr = xcalloc(ni + 1, sizeof(int)); A->ib_idx = xcalloc(u, sizeof(int));
    for (long i = 0; i < u; i++) { int r = (int)(cib[i] / (nb > 0 ? nb : 1)); A->ib_ptr[r + 1]++; A->ib_idx[i] = (int)(cib[i] % (nb > 0 ? nb : 1)); }
    for (int i = 0; i < ni; i++) A->ib_ptr[i + 1] += A->ib_ptr[i];
    free(cii); free(cib);
    A->data_ii = xcalloc(A->nnz_ii, sizeof(double)); A->data_ib = xcalloc(A->nnz_ib, sizeof(double));
    A->g_bb = xcalloc((size_t)nb * nb, sizeof(double)); A->b_i = xcalloc(ni, sizeof(double)); A->b_b = xcalloc(nb, sizeof(double));
    A->g_flat = xcalloc(ns, sizeof(double)); A->resid = xcalloc(A->n_rows, sizeof(double));
    A->s_b = xcalloc((size_t)nb * nb, sizeof(double)); A->b_hat = xcalloc(nb, sizeof(double)); A->dxi = xcalloc(ni, sizeof(double));
    A->zmat = xcalloc((size_t)ni * nb, sizeof(double)); A->wvec = xcalloc(ni, sizeof(double));
}

/* row evaluation: residual + template gradient (assembly.py:427-483) */
static void eval_rows(const orc_t *o, area_t *A, const double *va, const double *vm) {
    const orc_desc *d = &o->d;
    for (int k = 0; k < A->n_rows; k++) {
        int r = A->row_ids[k], t = d->m_type[r], tg = d->m_target[r];
        double *g = A->g_flat + A->slot_ptr[k]; double h;
        if (t == 0) { h = vm[tg]; g[0] = 1.0; }
        else if (t <= 2) {
            int p0 = d->y_ptr[tg], p1 = d->y_ptr[tg + 1], deg = p1 - p0, nth = 0;
            for (int p = p0; p < p1; p++) if (d->y_idx[p] != d->slack) nth++;
            double vi = vm[tg], gd = 0, bd = 0, sum_p = 0.0, sum_q = 0.0;
            int c_th = 0, dth = -1, dvm = -1;
            for (int p = p0, q = 0; p < p1; p++, q++) {
                int j = d->y_idx[p]; int thpos = -1;
                if (j != d->slack) thpos = c_th++;
                int vmpos = nth + q;
                if (j == tg) { gd = d->y_g[p]; bd = d->y_b[p]; dth = thpos; dvm = vmpos; continue; }
                double th = va[tg] - va[j], vj = vm[j], cs = cos(th), sn = sin(th);
                double eg = d->y_g[p], eb = d->y_b[p];
                double tp = vj * (eg * cs + eb * sn), tq = vj * (eg * sn - eb * cs);
                sum_p += tp; sum_q += tq;
                if (t == 2) { if (thpos >= 0) g[thpos] = -vi * tp; g[vmpos] = vi * (eg * sn - eb * cs); }
                else { if (thpos >= 0) g[thpos] = vi * tq; g[vmpos] = vi * (eg * cs + eb * sn); }
            }
            (void)deg;
            if (t == 2) { h = vi * (-vi * bd + sum_q); if (dth >= 0) g[dth] = vi * sum_p; g[dvm] = -2.0 * vi * bd + sum_q; }
            else { h = vi * (vi * gd + sum_p); if (dth >= 0) g[dth] = -vi * sum_q; g[dvm] = 2.0 * vi * gd + sum_p; }
        } else {
            int f = d->br_from[tg], tt = d->br_to[tg]; const double *y = d->br_y + 8 * (size_t)tg;
            /* types 7 / 8: current magnitude |i_o| at the from / to end -- NOT in the reference (measurement.py:27-34
               stops at QT); a north_star template, restated here from the same two-port current i_o, parity unpinned
               (tests check it against finite differences and the device template against this) */
            int from_end = (t == 3 || t == 5 || t == 7), reactive = (t == 5 || t == 6), current = (t >= 7);
            int ob = from_end ? f : tt, ub = from_end ? tt : f;
            double yor = from_end ? y[0] : y[6], yoi = from_end ? y[1] : y[7];
            double yur = from_end ? y[2] : y[4], yui = from_end ? y[3] : y[5];
            double vmo = vm[ob], vmu = vm[ub];
            double co = cos(va[ob]), so = sin(va[ob]), cu = cos(va[ub]), su = sin(va[ub]);
            double vor = vmo * co, voi = vmo * so, vur = vmu * cu, vui = vmu * su;
            /* i_o = y_own v_o + y_oth v_u */
            double t1r = yor * vor - yoi * voi, t1i = yor * voi + yoi * vor;
            double t2r = yur * vur - yui * vui, t2i = yur * vui + yui * vur;
            double ir = t1r + t2r, ii = t1i + t2i;
            /* s = v_o conj(i_o) */
            double sr = vor * ir - voi * (-ii), si = vor * (-ii) + voi * ir;
            /* ds/dth_o = 1j (s - vmo^2 conj(y_own)) */
            double v2 = vmo * vmo; double ar = sr - v2 * yor, ai = si - v2 * (-yoi);
            double dthor = -ai, dthoi = ar;
            /* ds/dth_u = (-1j v_o) conj(y_oth v_u) */
            double mr = voi, mi = -vor; double cr = t2r, ci = -t2i;
            double dthur = mr * cr - mi * ci, dthui = mr * ci + mi * cr;
            /* ds/dvm_o = s / vmo + vmo conj(y_own) */
            double inv = 1.0 / vmo; double dvor = sr * inv + vmo * yor, dvoi = si * inv + vmo * (-yoi);
            /* ds/dvm_u = (v_o conj(y_oth)) exp(-1j th_u) */
            double pr = vor * yur - voi * (-yui), pi_ = vor * (-yui) + voi * yur;
            double dvur = pr * cu - pi_ * (-su), dvui = pr * (-su) + pi_ * cu;
            h = reactive ? si : sr;
            double g_tho = reactive ? dthoi : dthor, g_thu = reactive ? dthui : dthur;
            double g_vo = reactive ? dvoi : dvor, g_vu = reactive ? dvui : dvur;
            if (current) {
                /* h = |i_o|; dh/dx = Re(conj(i_o) di_o/dx) / h with di/dth_o = j y_own v_o, di/dth_u = j y_oth v_u,
                   di/dvm_o = y_own v_o / vm_o, di/dvm_u = y_oth v_u / vm_u; a vanishing current (flat start on a
                   branch without charging) has no gradient: the row then contributes nothing to this iteration */
                double m2 = ir * ir + ii * ii;
                h = sqrt(m2);
                double ih = m2 > 1e-24 ? 1.0 / h : 0.0;
                g_tho = (ir * (-t1i) + ii * t1r) * ih; g_thu = (ir * (-t2i) + ii * t2r) * ih;
                g_vo = (ir * t1r + ii * t1i) / vmo * ih; g_vu = (ir * t2r + ii * t2i) / vmu * ih;
            }
            int c = 0;
            if (f != d->slack) g[c++] = (f == ob) ? g_tho : g_thu;
            if (tt != d->slack) g[c++] = (tt == ob) ? g_tho : g_thu;
            g[c++] = (f == ob) ? g_vo : g_vu; g[c++] = (tt == ob) ? g_vo : g_vu;
        }
        A->resid[k] = d->m_z[r] - h;
    }
}

static int csr_find(const int *idx, int lo, int hi, int col) {
    while (lo < hi) { int mid = (lo + hi) >> 1; if (idx[mid] < col) lo = mid + 1; else hi = mid; }
    return lo;
}

/* fused accumulation in program order: ascending row, row-major (a, b) */
static void accumulate(const orc_t *o, area_t *A) {
    const orc_desc *d = &o->d; int ni = A->n_i, nb = A->n_b;
    memset(A->data_ii, 0, sizeof(double) * A->nnz_ii); memset(A->data_ib, 0, sizeof(double) * A->nnz_ib);
    memset(A->g_bb, 0, sizeof(double) * (size_t)nb * nb); memset(A->b_i, 0, sizeof(double) * ni); memset(A->b_b, 0, sizeof(double) * nb);
    for (int k = 0; k < A->n_rows; k++) {
        int s0 = A->slot_ptr[k], s1 = A->slot_ptr[k + 1]; double w = d->m_w[A->row_ids[k]];
        for (int x = s0; x < s1; x++) {
            int va = A->slot_var[x]; double ga = A->g_flat[x];
            for (int y = s0; y < s1; y++) {
                int vb = A->slot_var[y]; double v = ga * (w * A->g_flat[y]);
                if (va < ni) {
                    if (vb < ni) A->data_ii[csr_find(A->ii_idx, A->ii_ptr[va], A->ii_ptr[va + 1], vb)] += v;
                    else A->data_ib[csr_find(A->ib_idx, A->ib_ptr[va], A->ib_ptr[va + 1], vb - ni)] += v;
                } else if (vb >= ni) A->g_bb[(size_t)(va - ni) * nb + (vb - ni)] += v;
            }
        }
        double wr = w * A->resid[k];
        for (int x = s0; x < s1; x++) { int v = A->slot_var[x]; double c = wr * A->g_flat[x]; if (v < ni) A->b_i[v] += c; else A->b_b[v - ni] += c; }
    }
}

/* ------------------------------------------------------ sparse Cholesky */

static void min_degree(const int *ptr, const int *idx, int n, int *perm) {
    /* greedy exact minimum degree on the elimination graph, ties -> lowest id */
    int **adj = xcalloc(n, sizeof(int *)); int *deg = xcalloc(n, sizeof(int)); char *alive = xcalloc(n, 1);
    int *tmp = xcalloc(n + 1, sizeof(int));
    for (int i = 0; i < n; i++) {
        int c = 0; adj[i] = xcalloc(ptr[i + 1] - ptr[i], sizeof(int));
        for (int p = ptr[i]; p < ptr[i + 1]; p++) if (idx[p] != i) adj[i][c++] = idx[p]; /* sorted */
        deg[i] = c; alive[i] = 1;
    }
    for (int step = 0; step < n; step++) {
        int k = -1;
        for (int i = 0; i < n; i++) if (alive[i] && (k < 0 || deg[i] < deg[k])) k = i;
        perm[step] = k; alive[k] = 0;
        int nk = deg[k]; const int *N = adj[k];
        for (int q = 0; q < nk; q++) {
            int v = N[q]; int *av = adj[v]; int dv = deg[v], c = 0, x = 0, y = 0;
            while (x < dv || y < nk) { /* sorted union of adj[v] and adj[k], minus {k, v} */
                int pick;
                if (y >= nk) pick = av[x++];
                else if (x >= dv) pick = N[y++];
                else if (av[x] < N[y]) pick = av[x++];
                else if (N[y] < av[x]) pick = N[y++];
                else { pick = av[x]; x++; y++; }
                if (pick != k && pick != v) tmp[c++] = pick;
            }
            free(av); adj[v] = xcalloc(c, sizeof(int)); memcpy(adj[v], tmp, sizeof(int) * c); deg[v] = c;
        }
    }
    for (int i = 0; i < n; i++) free(adj[i]);
    free(adj); free(deg); free(alive); free(tmp);
}

static void chol_analyze(chol_t *c, int n, int *ptr, int *idx, int dense_threshold) {
    memset(c, 0, sizeof(*c));
    c->n = n; c->pat_ptr = ptr; c->pat_idx = idx; c->dense = n < dense_threshold;
    if (c->dense) { c->dn = xcalloc((size_t)n * n, sizeof(double)); return; }
    c->perm = xcalloc(n, sizeof(int)); min_degree(ptr, idx, n, c->perm);
    int *inv = xcalloc(n, sizeof(int)); for (int i = 0; i < n; i++) inv[c->perm[i]] = i;
    /* permuted upper triangle column-wise with source positions */
    c->c_ptr = xcalloc(n + 1, sizeof(int));
    for (int kn = 0; kn < n; kn++) { int ko = c->perm[kn], cnt = 0;
        for (int p = ptr[ko]; p < ptr[ko + 1]; p++) if (inv[idx[p]] <= kn) cnt++;
        c->c_ptr[kn + 1] = c->c_ptr[kn] + cnt; }
    c->c_rows = xcalloc(c->c_ptr[n], sizeof(int)); c->c_src = xcalloc(c->c_ptr[n], sizeof(int));
    for (int kn = 0; kn < n; kn++) { int ko = c->perm[kn], q = c->c_ptr[kn];
        for (int p = ptr[ko]; p < ptr[ko + 1]; p++) { int jn = inv[idx[p]]; if (jn <= kn) { c->c_rows[q] = jn; c->c_src[q] = p; q++; } } }
    /* elimination tree */
    c->parent = xcalloc(n, sizeof(int)); int *anc = xcalloc(n, sizeof(int));
    for (int k = 0; k < n; k++) { c->parent[k] = -1; anc[k] = -1; }
    for (int k = 0; k < n; k++)
        for (int p = c->c_ptr[k]; p < c->c_ptr[k + 1]; p++) {
            int i = c->c_rows[p];
            while (i != -1 && i < k) { int nxt = anc[i]; anc[i] = k; if (nxt == -1) c->parent[i] = k; i = nxt; }
        }
    /* row patterns via ereach, flattened */
    int *marked = xcalloc(n, sizeof(int)), *stack = xcalloc(n, sizeof(int));
    for (int k = 0; k < n; k++) marked[k] = -1;
    c->row_ptr = xcalloc(n + 1, sizeof(int));
    int cap = 4 * n + 16, len = 0; c->prog_col = xcalloc(cap, sizeof(int));
    int *counts = xcalloc(n, sizeof(int)); for (int k = 0; k < n; k++) counts[k] = 1;
    for (int k = 0; k < n; k++) {
        int top = n; marked[k] = k;
        for (int p = c->c_ptr[k]; p < c->c_ptr[k + 1]; p++) {
            int i = c->c_rows[p]; if (i > k) continue;
            int l = 0;
            while (marked[i] != k) { stack[l++] = i; marked[i] = k; i = c->parent[i]; }
            while (l > 0) stack[--top] = stack[--l];
        }
        for (int q = top; q < n; q++) {
            if (len == cap) { cap *= 2; c->prog_col = realloc(c->prog_col, sizeof(int) * cap); }
            c->prog_col[len++] = stack[q]; counts[stack[q]]++;
        }
        c->row_ptr[k + 1] = len;
    }
    c->Lp = xcalloc(n + 1, sizeof(int)); for (int k = 0; k < n; k++) c->Lp[k + 1] = c->Lp[k] + counts[k];
    c->Li = xcalloc(c->Lp[n], sizeof(int)); c->Lx = xcalloc(c->Lp[n], sizeof(double));
    c->fillcnt = xcalloc(n, sizeof(int)); c->x = xcalloc(n, sizeof(double));
    /* row indices are static: fill them once in program order */
    for (int k = 0; k < n; k++) c->Li[c->Lp[k]] = k;
    for (int k = 0; k < n; k++) for (int t = c->row_ptr[k]; t < c->row_ptr[k + 1]; t++) { int j = c->prog_col[t]; c->Li[c->Lp[j] + 1 + c->fillcnt[j]++] = k; }
    free(inv); free(anc); free(marked); free(stack); free(counts);
}

/* dense lower Cholesky in place (row-major n x n, lower triangle read); returns failing pivot or -1 */
static int dense_chol(double *a, int n) {
    for (int j = 0; j < n; j++) {
        double d = a[(size_t)j * n + j];
        for (int k = 0; k < j; k++) d -= a[(size_t)j * n + k] * a[(size_t)j * n + k];
        if (!(d > 0.0)) return j;
        d = sqrt(d); a[(size_t)j * n + j] = d;
        for (int i = j + 1; i < n; i++) {
            double s = a[(size_t)i * n + j]; const double *ri = a + (size_t)i * n, *rj = a + (size_t)j * n;
            for (int k = 0; k < j; k++) s -= ri[k] * rj[k];
            a[(size_t)i * n + j] = s / d;
        }
    }
    return -1;
}
static void dense_fwd(const double *l, int n, double *b, int nrhs) { /* b row-major n x nrhs */
    for (int i = 0; i < n; i++) {
        for (int k = 0; k < i; k++) { double lik = l[(size_t)i * n + k]; if (lik == 0.0) continue; for (int c = 0; c < nrhs; c++) b[(size_t)i * nrhs + c] -= lik * b[(size_t)k * nrhs + c]; }
        double d = l[(size_t)i * n + i]; for (int c = 0; c < nrhs; c++) b[(size_t)i * nrhs + c] /= d;
    }
}
static void dense_bwd(const double *l, int n, double *b) {
    for (int i = n - 1; i >= 0; i--) { double s = b[i]; for (int k = i + 1; k < n; k++) s -= l[(size_t)k * n + i] * b[k]; b[i] = s / l[(size_t)i * n + i]; }
}

static int chol_refactor(chol_t *c, const double *vals) {
    int n = c->n;
    if (c->dense) {
        memset(c->dn, 0, sizeof(double) * (size_t)n * n);
        for (int i = 0; i < n; i++) for (int p = c->pat_ptr[i]; p < c->pat_ptr[i + 1]; p++) c->dn[(size_t)i * n + c->pat_idx[p]] = vals[p];
        return dense_chol(c->dn, n);
    }
    double *x = c->x, *Lx = c->Lx; const int *Lp = c->Lp, *Li = c->Li;
    memset(x, 0, sizeof(double) * n); memset(c->fillcnt, 0, sizeof(int) * n);
    for (int k = 0; k < n; k++) {
        for (int p = c->c_ptr[k]; p < c->c_ptr[k + 1]; p++) x[c->c_rows[p]] = vals[c->c_src[p]];
        double d = x[k]; x[k] = 0.0;
        for (int t = c->row_ptr[k]; t < c->row_ptr[k + 1]; t++) {
            int j = c->prog_col[t]; double xj = x[j]; x[j] = 0.0;
            double lkj = xj / Lx[Lp[j]]; int m = c->fillcnt[j], s0 = Lp[j] + 1;
            for (int q = 0; q < m; q++) x[Li[s0 + q]] -= Lx[s0 + q] * lkj;
            d -= lkj * lkj; Lx[s0 + m] = lkj; c->fillcnt[j] = m + 1;
        }
        if (!(d > 0.0)) return c->perm[k];
        Lx[Lp[k]] = sqrt(d);
    }
    return -1;
}
/* y = L^{-1} P b for nrhs columns, b row-major n x nrhs (result overwrites out) */
static void chol_forward(const chol_t *c, const double *b, double *out, int nrhs) {
    int n = c->n;
    if (c->dense) { memcpy(out, b, sizeof(double) * (size_t)n * nrhs); dense_fwd(c->dn, n, out, nrhs); return; }
    for (int i = 0; i < n; i++) memcpy(out + (size_t)i * nrhs, b + (size_t)c->perm[i] * nrhs, sizeof(double) * nrhs);
    for (int j = 0; j < n; j++) {
        double dj = c->Lx[c->Lp[j]]; double *yj = out + (size_t)j * nrhs;
        for (int q = 0; q < nrhs; q++) yj[q] = yj[q] / dj;
        for (int p = c->Lp[j] + 1; p < c->Lp[j + 1]; p++) { double l = c->Lx[p]; double *yi = out + (size_t)c->Li[p] * nrhs; for (int q = 0; q < nrhs; q++) yi[q] -= l * yj[q]; }
    }
}
static void chol_backward(const chol_t *c, double *y, double *out) { /* y is destroyed */
    int n = c->n;
    if (c->dense) { dense_bwd(c->dn, n, y); memcpy(out, y, sizeof(double) * n); return; }
    for (int j = n - 1; j >= 0; j--) {
        double s = 0.0; int has = 0;
        for (int p = c->Lp[j] + 1; p < c->Lp[j + 1]; p++) { s += c->Lx[p] * y[c->Li[p]]; has = 1; }
        if (has) y[j] -= s;
        y[j] = y[j] / c->Lx[c->Lp[j]];
    }
    for (int i = 0; i < n; i++) out[c->perm[i]] = y[i];
}

/* ------------------------------------------------------- Schur / recovery */

static void condense(area_t *A) {
    int ni = A->n_i, nb = A->n_b;
    memcpy(A->s_b, A->g_bb, sizeof(double) * (size_t)nb * nb); memcpy(A->b_hat, A->b_b, sizeof(double) * nb);
    if (ni == 0 || nb == 0) return;
    double *gd = xcalloc((size_t)ni * nb, sizeof(double));
    for (int i = 0; i < ni; i++) for (int p = A->ib_ptr[i]; p < A->ib_ptr[i + 1]; p++) gd[(size_t)i * nb + A->ib_idx[p]] = A->data_ib[p];
    chol_forward(&A->ch, gd, A->zmat, nb); chol_forward(&A->ch, A->b_i, A->wvec, 1);
    free(gd);
    double *zz = xcalloc((size_t)nb * nb, sizeof(double)), *zw = xcalloc(nb, sizeof(double));
    for (int k = 0; k < ni; k++) { const double *zk = A->zmat + (size_t)k * nb; double wk = A->wvec[k];
        for (int i = 0; i < nb; i++) { double zi = zk[i]; if (zi == 0.0) continue; double *row = zz + (size_t)i * nb; for (int j = 0; j < nb; j++) row[j] += zi * zk[j]; zw[i] += zi * wk; } }
    for (size_t i = 0; i < (size_t)nb * nb; i++) A->s_b[i] = A->g_bb[i] - zz[i];
    for (int i = 0; i < nb; i++) A->b_hat[i] = A->b_b[i] - zw[i];
    free(zz); free(zw);
}
static void recover(area_t *A, const double *dx_gamma) {
    int ni = A->n_i; if (ni == 0) return;
    double *rhs = xcalloc(ni, sizeof(double)), *y = xcalloc(ni, sizeof(double));
    for (int i = 0; i < ni; i++) { double s = 0.0; for (int p = A->ib_ptr[i]; p < A->ib_ptr[i + 1]; p++) s += A->data_ib[p] * dx_gamma[A->sel[A->ib_idx[p]]]; rhs[i] = A->n_b ? A->b_i[i] - s : A->b_i[i]; }
    chol_forward(&A->ch, rhs, y, 1); chol_backward(&A->ch, y, A->dxi);
    free(rhs); free(y);
}

/* ------------------------------------------------------------ public API */

orc_t *orc_create(const orc_desc *desc) {
    orc_t *o = xcalloc(1, sizeof(orc_t)); o->d = *desc; o->err_area = -1; o->err_pivot = -1;
    build_maps(o);
    int nb = desc->n_bus;
    int *loc_va = xcalloc(nb, sizeof(int)), *loc_vm = xcalloc(nb, sizeof(int));
    for (int a = 0; a < desc->n_areas; a++) {
        for (int b = 0; b < nb; b++) loc_va[b] = loc_vm[b] = -1;
        build_pattern(o, a, loc_va, loc_vm);
    }
    free(loc_va); free(loc_vm);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int a = 0; a < desc->n_areas; a++) { area_t *A = &o->areas[a]; chol_analyze(&A->ch, A->n_i, A->ii_ptr, A->ii_idx, desc->dense_threshold); }
    int ng = o->n_gamma;
    o->s_gamma = xcalloc((size_t)ng * ng, sizeof(double)); o->b_gamma = xcalloc(ng, sizeof(double)); o->dx_gamma = xcalloc(ng, sizeof(double));
    return o;
}

void orc_destroy(orc_t *o) { /* test infrastructure: the process frees the arenas */ (void)o; }

int orc_n_gamma(const orc_t *o) { return o->n_gamma; }
void orc_area_dims(const orc_t *o, int a, int32_t *out) { const area_t *A = &o->areas[a];
    out[0] = A->n_i; out[1] = A->n_b; out[2] = A->n_rows; out[3] = A->n_slots; out[4] = A->nnz_ii; out[5] = A->nnz_ib; out[6] = A->ch.dense ? 0 : A->ch.Lp[A->ch.n]; out[7] = A->ch.dense; }
const int *orc_area_int(const orc_t *o, int a, int which) { const area_t *A = &o->areas[a];
    switch (which) { case 0: return A->ii_ptr; case 1: return A->ii_idx; case 2: return A->ib_ptr; case 3: return A->ib_idx; case 4: return A->sel; case 5: return A->row_ids; case 6: return A->slot_ptr; case 7: return A->slot_var; case 8: return A->ch.perm; } return 0; }
const double *orc_area_f64(const orc_t *o, int a, int which) { const area_t *A = &o->areas[a];
    switch (which) { case 0: return A->data_ii; case 1: return A->data_ib; case 2: return A->g_bb; case 3: return A->b_i; case 4: return A->b_b; case 5: return A->s_b; case 6: return A->b_hat; case 7: return A->dxi; case 8: return A->g_flat; case 9: return A->resid; } return 0; }
const double *orc_gamma_f64(const orc_t *o, int which) { return which == 0 ? o->s_gamma : which == 1 ? o->b_gamma : o->dx_gamma; }
void orc_last_error(const orc_t *o, int32_t *out) { out[0] = o->err_kind; out[1] = o->err_area; out[2] = o->err_pivot; }

/* assemble + refactor + condense every area at the state (va, vm); 0 or -1 */
int orc_local(orc_t *o, const double *va, const double *vm, int threads) {
    int K = o->d.n_areas; (void)threads;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (int a = 0; a < K; a++) {
        area_t *A = &o->areas[a];
        eval_rows(o, A, va, vm); accumulate(o, A);
        A->fail_pivot = chol_refactor(&A->ch, A->data_ii);
        if (A->fail_pivot < 0) condense(A);
    }
    for (int a = 0; a < K; a++) if (o->areas[a].fail_pivot >= 0) { o->err_kind = 1; o->err_area = a; o->err_pivot = o->areas[a].fail_pivot; return -1; }
    return 0;
}
int orc_assemble_only(orc_t *o, const double *va, const double *vm) {
    for (int a = 0; a < o->d.n_areas; a++) { eval_rows(o, &o->areas[a], va, vm); accumulate(o, &o->areas[a]); }
    return 0;
}
/* S_gamma[sel, sel] += S_b in area order; dense Cholesky solve; 0 or -1 */
int orc_boundary(orc_t *o) {
    int ng = o->n_gamma; if (ng == 0) return 0;
    memset(o->s_gamma, 0, sizeof(double) * (size_t)ng * ng); memset(o->b_gamma, 0, sizeof(double) * ng);
    for (int a = 0; a < o->d.n_areas; a++) { const area_t *A = &o->areas[a]; int nb = A->n_b;
        for (int i = 0; i < nb; i++) { double *row = o->s_gamma + (size_t)A->sel[i] * ng; const double *src = A->s_b + (size_t)i * nb;
            for (int j = 0; j < nb; j++) row[A->sel[j]] += src[j];
            o->b_gamma[A->sel[i]] += A->b_hat[i]; } }
    double *l = xcalloc((size_t)ng * ng, sizeof(double)); memcpy(l, o->s_gamma, sizeof(double) * (size_t)ng * ng);
    int piv = dense_chol(l, ng);
    if (piv >= 0) { free(l); o->err_kind = 2; o->err_area = -1; o->err_pivot = piv; return -1; }
    memcpy(o->dx_gamma, o->b_gamma, sizeof(double) * ng); dense_fwd(l, ng, o->dx_gamma, 1); dense_bwd(l, ng, o->dx_gamma);
    free(l); return 0;
}
/* interior recovery + state update; returns the stacked update's infinity norm */
double orc_recover(orc_t *o, double *va, double *vm, int threads) {
    int K = o->d.n_areas; double dmax = 0.0; (void)threads;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (int a = 0; a < K; a++) recover(&o->areas[a], o->dx_gamma);
    for (int a = 0; a < K; a++) { area_t *A = &o->areas[a];
        for (int i = 0; i < A->n_ia; i++) va[A->ia_bus[i]] += A->dxi[i];
        for (int i = 0; i < A->n_int_bus; i++) vm[A->int_bus[i]] += A->dxi[A->n_ia + i];
        for (int i = 0; i < A->n_i; i++) if (fabs(A->dxi[i]) > dmax) dmax = fabs(A->dxi[i]); }
    for (int s = 0; s < o->n_gamma; s++) { int b = o->gamma_bus[s]; if (s < o->n_ga) va[b] += o->dx_gamma[s]; else vm[b] += o->dx_gamma[s]; if (fabs(o->dx_gamma[s]) > dmax) dmax = fabs(o->dx_gamma[s]); }
    return dmax;
}
/* J(x) = sum w (z - h)^2 over all rows, h as in eval_h_all (diagonal inside the neighbor sum) */
double orc_objective(const orc_t *o, const double *va, const double *vm) {
    const orc_desc *d = &o->d; double sum = 0.0, comp = 0.0;
    for (int r = 0; r < d->n_rows; r++) {
        int t = d->m_type[r], tg = d->m_target[r]; double h;
        if (t == 0) h = vm[tg];
        else if (t <= 2) { double acc = 0.0;
            for (int p = d->y_ptr[tg]; p < d->y_ptr[tg + 1]; p++) { int j = d->y_idx[p]; double th = va[tg] - va[j];
                acc += (t == 1) ? vm[j] * (d->y_g[p] * cos(th) + d->y_b[p] * sin(th)) : vm[j] * (d->y_g[p] * sin(th) - d->y_b[p] * cos(th)); }
            h = vm[tg] * acc; }
        else { int f = d->br_from[tg], tt = d->br_to[tg]; const double *y = d->br_y + 8 * (size_t)tg; int fe = (t == 3 || t == 5 || t == 7);
            int ob = fe ? f : tt, ub = fe ? tt : f; double yor = fe ? y[0] : y[6], yoi = fe ? y[1] : y[7], yur = fe ? y[2] : y[4], yui = fe ? y[3] : y[5];
            double vor = vm[ob] * cos(va[ob]), voi = vm[ob] * sin(va[ob]), vur = vm[ub] * cos(va[ub]), vui = vm[ub] * sin(va[ub]);
            double ir = (yor * vor - yoi * voi) + (yur * vur - yui * vui), ii = (yor * voi + yoi * vor) + (yur * vui + yui * vur);
            h = (t >= 7) ? sqrt(ir * ir + ii * ii) : (t >= 5) ? (vor * (-ii) + voi * ir) : (vor * ir - voi * (-ii)); }
        double res = d->m_z[r] - h, term = d->m_w[r] * res * res;
        double tsum = sum + term; comp += (fabs(sum) >= fabs(term)) ? (sum - tsum) + term : (term - tsum) + sum; sum = tsum;
    }
    return sum + comp;
}
/* One inner GN step of every area with the boundary held fixed (reference solver.py:253-260):
   assemble, refactor, dx_i = G_ii^-1 b_i, apply to the interior state.  Returns max |dx_i| or -1. */
double orc_inner_step(orc_t *o, double *va, double *vm) {
    int K = o->d.n_areas; double dmax = 0.0;
    double *zero = xcalloc(o->n_gamma > 0 ? o->n_gamma : 1, sizeof(double));
    for (int a = 0; a < K; a++) {
        area_t *A = &o->areas[a];
        eval_rows(o, A, va, vm); accumulate(o, A);
        A->fail_pivot = chol_refactor(&A->ch, A->data_ii);
        if (A->fail_pivot >= 0) { o->err_kind = 1; o->err_area = a; o->err_pivot = A->fail_pivot; free(zero); return -1.0; }
        recover(A, zero);
        for (int i = 0; i < A->n_ia; i++) va[A->ia_bus[i]] += A->dxi[i];
        for (int i = 0; i < A->n_int_bus; i++) vm[A->int_bus[i]] += A->dxi[A->n_ia + i];
        for (int i = 0; i < A->n_i; i++) if (fabs(A->dxi[i]) > dmax) dmax = fabs(A->dxi[i]);
    }
    free(zero);
    return dmax;
}
/* Full GN loop.  trace_delta[max_iter]; trace_va/vm optional [max_iter][n_bus].
   Returns iterations (>0), or -1 on a non-SPD failure (see orc_last_error). */
int orc_solve_inner(orc_t *o, int max_iter, int inner_steps, double tol, double *va, double *vm, int threads,
                    double *trace_delta, double *trace_va, double *trace_vm, int32_t *converged) {
    int nb = o->d.n_bus; *converged = 0;
    for (int b = 0; b < nb; b++) { va[b] = 0.0; vm[b] = 1.0; }
    va[o->d.slack] = o->d.slack_va;
    for (int it = 1; it <= max_iter; it++) {
        double inner = 0.0;
        for (int s = 0; s + 1 < inner_steps; s++) { double d = orc_inner_step(o, va, vm); if (d < 0) return -1; if (d > inner) inner = d; }
        if (orc_local(o, va, vm, threads)) return -1;
        if (orc_boundary(o)) return -1;
        double dinf = orc_recover(o, va, vm, threads);
        if (inner > dinf) dinf = inner;
        if (trace_delta) trace_delta[it - 1] = dinf;
        if (trace_va) memcpy(trace_va + (size_t)(it - 1) * nb, va, sizeof(double) * nb);
        if (trace_vm) memcpy(trace_vm + (size_t)(it - 1) * nb, vm, sizeof(double) * nb);
        if (dinf < tol) { *converged = 1; return it; }
    }
    return max_iter;
}
int orc_solve(orc_t *o, int max_iter, double tol, double *va, double *vm, int threads,
              double *trace_delta, double *trace_va, double *trace_vm, int32_t *converged) {
    return orc_solve_inner(o, max_iter, 1, tol, va, vm, threads, trace_delta, trace_va, trace_vm, converged);
}
/* component-level helpers for tests: dense SPD solve and standalone Schur of user blocks */
int orc_dense_cholesky_solve(const double *a, const double *b, int n, double *x) {
    double *l = xcalloc((size_t)n * n, sizeof(double)); memcpy(l, a, sizeof(double) * (size_t)n * n);
    int piv = dense_chol(l, n); if (piv >= 0) { free(l); return piv + 1; }
    memcpy(x, b, sizeof(double) * n); dense_fwd(l, n, x, 1); dense_bwd(l, n, x); free(l); return 0;
}
int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- area-sharded variants (the multi-process driver tests shard areas over ranks) ---- */
int orc_local_masked(orc_t *o, const double *va, const double *vm, const int32_t *mine) {
    int K = o->d.n_areas;
    for (int a = 0; a < K; a++) {
        if (!mine[a]) continue;
        area_t *A = &o->areas[a];
        eval_rows(o, A, va, vm); accumulate(o, A);
        A->fail_pivot = chol_refactor(&A->ch, A->data_ii);
        if (A->fail_pivot < 0) condense(A);
        else { o->err_kind = 1; o->err_area = a; o->err_pivot = A->fail_pivot; return -1; }
    }
    return 0;
}
void orc_get_schur(const orc_t *o, int a, double *s_b, double *b_hat) { const area_t *A = &o->areas[a];
    memcpy(s_b, A->s_b, sizeof(double) * (size_t)A->n_b * A->n_b); memcpy(b_hat, A->b_hat, sizeof(double) * A->n_b); }
void orc_set_schur(orc_t *o, int a, const double *s_b, const double *b_hat) { area_t *A = &o->areas[a];
    memcpy(A->s_b, s_b, sizeof(double) * (size_t)A->n_b * A->n_b); memcpy(A->b_hat, b_hat, sizeof(double) * A->n_b); }
void orc_set_dx_gamma(orc_t *o, const double *dx) { memcpy(o->dx_gamma, dx, sizeof(double) * o->n_gamma); }
/* recovery of the owned areas + every rank's replica of the boundary state */
double orc_recover_masked(orc_t *o, double *va, double *vm, const int32_t *mine) {
    int K = o->d.n_areas; double dmax = 0.0;
    for (int a = 0; a < K; a++) { if (!mine[a]) continue; area_t *A = &o->areas[a];
        recover(A, o->dx_gamma);
        for (int i = 0; i < A->n_ia; i++) va[A->ia_bus[i]] += A->dxi[i];
        for (int i = 0; i < A->n_int_bus; i++) vm[A->int_bus[i]] += A->dxi[A->n_ia + i];
        for (int i = 0; i < A->n_i; i++) if (fabs(A->dxi[i]) > dmax) dmax = fabs(A->dxi[i]); }
    for (int s = 0; s < o->n_gamma; s++) { int b = o->gamma_bus[s]; if (s < o->n_ga) va[b] += o->dx_gamma[s]; else vm[b] += o->dx_gamma[s]; if (fabs(o->dx_gamma[s]) > dmax) dmax = fabs(o->dx_gamma[s]); }
    return dmax;
}
/* inner GN step of the owned areas only (multi-process driver with inner_gn_steps > 1) */
double orc_inner_step_masked(orc_t *o, double *va, double *vm, const int32_t *mine) {
    int K = o->d.n_areas; double dmax = 0.0;
    double *zero = xcalloc(o->n_gamma > 0 ? o->n_gamma : 1, sizeof(double));
    for (int a = 0; a < K; a++) {
        if (!mine[a]) continue;
        area_t *A = &o->areas[a];
        eval_rows(o, A, va, vm); accumulate(o, A);
        A->fail_pivot = chol_refactor(&A->ch, A->data_ii);
        if (A->fail_pivot >= 0) { o->err_kind = 1; o->err_area = a; o->err_pivot = A->fail_pivot; free(zero); return -1.0; }
        recover(A, zero);
        for (int i = 0; i < A->n_ia; i++) va[A->ia_bus[i]] += A->dxi[i];
        for (int i = 0; i < A->n_int_bus; i++) vm[A->int_bus[i]] += A->dxi[A->n_ia + i];
        for (int i = 0; i < A->n_i; i++) if (fabs(A->dxi[i]) > dmax) dmax = fabs(A->dxi[i]);
    }
    free(zero);
    return dmax;
}
/* buses whose state this rank owns: interiors of its areas (boundary buses are replicated) */
void orc_owned_interior_mask(const orc_t *o, const int32_t *mine, int32_t *bus_mask) {
    for (int b = 0; b < o->d.n_bus; b++) bus_mask[b] = 0;
    for (int a = 0; a < o->d.n_areas; a++) { if (!mine[a]) continue; const area_t *A = &o->areas[a];
        for (int i = 0; i < A->n_int_bus; i++) bus_mask[A->int_bus[i]] = 1; }
}
