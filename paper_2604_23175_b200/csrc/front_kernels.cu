// front_kernels.cu -- the multifrontal Schur-mode factorisation and its back-substitution.
//
// front_task_kernel<HAS_PIVOTS>: one CTA = one (front, row-chunk I, col-chunk J) task.
//   1. assemble in shared memory: original entries (written by accumulate_kernel) + extend-add of
//      the children's packed update matrices in fixed child order (deterministic, no atomics);
//   2. factor the pivot block and solve the two row chunks against it: left-looking in blocks of
//      8 columns -- the rank-k update of each block column runs on the FP64 tensor pipe
//      (mma.sync m8n8k4 f64 from shared memory), the 8x8 diagonal block is factored redundantly
//      in registers by every row thread (no communication), two barriers per 8 pivots;
//   3. trailing / Schur update U_IJ = F_IJ - L_I L_J^T on the tensor pipe, written packed-lower;
//   4. diagonal tasks store their slice of the factor panel for the backward pass.
// Every task of a front recomputes the (small) pivot-block factor instead of exchanging it:
// redundancy is free while SMs idle, a second launch is not.
//
// Restates numeric_refactor + schur_condense (reference linalg.py:292-332,410-424), assemble_boundary
// (solver.py:106-119) and dense_cholesky_solve's factorisation (linalg.py:46-61) as one tree.
#include "kernels.cuh"

namespace gse {

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// child update block rows [r0,r1) x cols [c0,c1) (lower part) -> dst[(srel[i-ro]-rs)*ld + srel[j-co]-cs]
// srow / scol: the child's rel map for these ranges, staged in shared memory.
__device__ __forceinline__ void add_child_block(const double* __restrict__ U, const int* __restrict__ srow,
                                                const int* __restrict__ scol, int r0, int r1, int c0, int c1,
                                                double* dst, int ld, int rs, int cs, int warp, int lane, int nwarps) {
    if (c1 <= c0 || r1 <= r0) return;
    for (int ib = r0 + warp; ib < r1; ib += 4 * nwarps) {
        for (int jb = c0; jb < c1; jb += 32) {
            const int j = jb + lane;
            double v[4];
            bool ok[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = ib + q * nwarps;
                ok[q] = i < r1 && j < c1 && j <= i;
                v[q] = ok[q] ? __ldg(U + (size_t)i * (i + 1) / 2 + j) : 0.0;
            }
            const int tc = j < c1 ? scol[j - c0] - cs : 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (ok[q]) dst[(srow[ib + q * nwarps - r0] - rs) * ld + tc] += v[q];
        }
    }
}

constexpr int kStage = kFrontThreads + 2 * kMaxTile + 16;   // staged rel entries: pivots + I + J ranges

template <int HAS_PIVOTS>
__global__ void __launch_bounds__(kFrontThreads, HAS_PIVOTS ? 1 : 2)
front_task_kernel(FrontTab ft, const TaskRec* __restrict__ tasks, const double* __restrict__ gval,
                  double* __restrict__ lbuf, double* __restrict__ ubuf, unsigned long long* err) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_rel[kStage];
    const TaskRec tk = tasks[blockIdx.x];
    const int f = tk.front, ci = tk.ci, cj = tk.cj;
    const int p = HAS_PIVOTS ? ft.p[f] : 0;
    const int u1 = ft.u1[f], T = ft.T[f];
    const int i0 = ci * T, ni = min(T, u1 - i0), j0 = cj * T, nj = min(T, u1 - j0);
    const bool diag = ci == cj;
    const int ld = pad_ld(p);
    const int rp = p ? round8(p) : 0, ri = p ? round8(ni) : 0, rj = (p && !diag) ? round8(nj) : 0;
    const int ldt = round8(nj) | 1;
    double* pan = sm;
    double* tile = sm + (size_t)(rp + ri + rj) * ld;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;

    {
        const int total = ((rp + ri + rj) * ld + round8(ni) * ldt + 1) >> 1;
        double2* z2 = reinterpret_cast<double2*>(sm);
        for (int t = tid; t < total; t += nth) z2[t] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (HAS_PIVOTS && tid < rp - p) pan[(p + tid) * ld + p + tid] = 1.0;   // identity on padded pivots

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
            const int32_t* rel = ft.rel + ft.rel_off[ch];
            const double* U = ubuf + ft.u_off[ch];
            const int32_t* cb = ft.cbounds + ft.cb_off[cptr + c];   // precomputed lower bounds of rel
            const int eP = cb[0], bI = cb[1 + ci], eI = cb[2 + ci], bJ = cb[1 + cj], eJ = cb[2 + cj];
            const int nI = eI - bI, nJ = eJ - bJ;
            if ((eP <= 0 || !p) && (nI <= 0 || nJ <= 0)) continue;   // nothing lands in this task (uniform)
            // stage the needed slices of rel: [0,eP) | [bI,eI) | [bJ,eJ)
            int* sP = s_rel; int* sI = s_rel + eP; int* sJ = sI + nI;
            for (int t = tid; t < eP + nI + nJ; t += nth)
                s_rel[t] = t < eP ? rel[t] : t < eP + nI ? rel[bI + t - eP] : rel[bJ + t - eP - nI];
            __syncthreads();
            if (p) {
                add_child_block(U, sP, sP, 0, eP, 0, eP, pan, ld, 0, 0, warp, lane, nwarps);
                add_child_block(U, sI, sP, bI, eI, 0, eP, pan + (size_t)rp * ld, ld, p + i0, 0, warp, lane, nwarps);
                if (!diag) add_child_block(U, sJ, sP, bJ, eJ, 0, eP, pan + (size_t)(rp + ri) * ld, ld, p + j0, 0, warp, lane, nwarps);
            }
            add_child_block(U, sI, sJ, bI, eI, bJ, eJ, tile, ldt, p + i0, p + j0, warp, lane, nwarps);
            __syncthreads();
        }
    }

    // ---- blocked panel factorisation (block = 8 columns) ---------------------------------------
    if (HAS_PIVOTS && p) {
        const int R = rp + ri + rj;                 // padded rows: [pivots | chunk I | chunk J]
        const int ntile = R >> 3;
        for (int kb = 0; kb < rp; kb += 8) {
            // A. rows >= kb: block column kb -= A[rows, 0:kb] * A[kb:kb+8, 0:kb]^T   (tensor pipe)
            if (kb) {
                const int t0 = kb >> 3;
                for (int tb = t0 + warp; tb < ntile; tb += 2 * nwarps) {
                    const int ta = tb, tc2 = tb + nwarps;
                    const bool two = tc2 < ntile;
                    const double* a0p = pan + (size_t)(ta * 8 + (lane >> 2)) * ld + (lane & 3);
                    const double* a1p = pan + (size_t)((two ? tc2 : ta) * 8 + (lane >> 2)) * ld + (lane & 3);
                    const double* bp = pan + (size_t)(kb + (lane >> 2)) * ld + (lane & 3);
                    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll 2
                    for (int kk = 0; kk < kb; kk += 4) {
                        const double b = bp[kk];
                        dmma_m8n8k4(c00, c01, a0p[kk], b);
                        dmma_m8n8k4(c10, c11, a1p[kk], b);
                    }
                    double* o0 = pan + (size_t)(ta * 8 + (lane >> 2)) * ld + kb + 2 * (lane & 3);
                    o0[0] -= c00; o0[1] -= c01;
                    if (two) {
                        double* o1 = pan + (size_t)(tc2 * 8 + (lane >> 2)) * ld + kb + 2 * (lane & 3);
                        o1[0] -= c10; o1[1] -= c11;
                    }
                }
                __syncthreads();
            }
            // B. every row thread factors the 8x8 diagonal block in registers (redundantly) and
            //    solves its own row against it
            const bool act = tid >= kb && tid < R;
            double d[36];   // lower triangle, row-major: d[i*(i+1)/2 + j]
            if (act) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j <= i; ++j) d[i * (i + 1) / 2 + j] = pan[(kb + i) * ld + kb + j];
            }
            __syncthreads();   // everyone holds the block before its owner rows overwrite it
            if (act) {
                double rinv[8];
                bool bad = false;
                int badk = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double dk = d[k * (k + 1) / 2 + k];
                    if (!(dk > 0.0) && !bad) { bad = true; badk = k; }
                    const double r = rsqrt(dk);
                    rinv[k] = r;
                    d[k * (k + 1) / 2 + k] = dk * r;
#pragma unroll
                    for (int i = k + 1; i < 8; ++i) d[i * (i + 1) / 2 + k] *= r;
#pragma unroll
                    for (int j = k + 1; j < 8; ++j)
#pragma unroll
                        for (int i = j; i < 8; ++i)
                            d[i * (i + 1) / 2 + j] = fma(-d[i * (i + 1) / 2 + k], d[j * (j + 1) / 2 + k], d[i * (i + 1) / 2 + j]);
                }
                double* myrow = pan + (size_t)tid * ld + kb;
                if (tid < kb + 8) {
                    if (tid == kb && bad && kb + badk < p) atomicMin(err, ((unsigned long long)f << 32) | (unsigned long long)(kb + badk));
                    const int i = tid - kb;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        double v = 0.0;
#pragma unroll
                        for (int ii = 0; ii < 8; ++ii) if (ii == i && j <= ii) v = d[ii * (ii + 1) / 2 + j];
                        myrow[j] = v;
                    }
                } else {
                    double y[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) y[j] = myrow[j];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        double acc = y[k];
#pragma unroll
                        for (int j = 0; j < k; ++j) acc = fma(-y[j], d[k * (k + 1) / 2 + j], acc);
                        y[k] = acc * rinv[k];
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) myrow[j] = y[j];
                }
            }
            __syncthreads();
        }
    }

    // ---- trailing update on the FP64 tensor pipe: U_IJ = F_IJ - L_I L_J^T -------------------
    {
        const double* Pi = pan + (size_t)rp * ld;
        const double* Pj = diag ? Pi : pan + (size_t)(rp + ri) * ld;
        const int nbi = round8(ni) >> 3, nbj = round8(nj) >> 3;
        const int ngj = (nbj + 3) >> 2;                 // groups of four 8-wide column blocks
        const int kend = (p + 3) & ~3;
        double* U = ubuf + ft.u_off[f];
        for (int w = warp; w < nbi * ngj; w += nwarps) {
            const int bi = w / ngj, gj = w % ngj;
            if (diag && gj * 4 > bi) continue;
            double c[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            if (p) {
                const double* ap = Pi + (size_t)(bi * 8 + (lane >> 2)) * ld + (lane & 3);
                const double* bp[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int bj = min(gj * 4 + q, nbj - 1);
                    bp[q] = Pj + (size_t)(bj * 8 + (lane >> 2)) * ld + (lane & 3);
                }
#pragma unroll 2
                for (int kk = 0; kk < kend; kk += 4) {
                    const double a = ap[kk];
#pragma unroll
                    for (int q = 0; q < 4; ++q) dmma_m8n8k4(c[2 * q], c[2 * q + 1], a, bp[q][kk]);
                }
            }
            const int row = bi * 8 + (lane >> 2);
            if (row < ni) {
                const int I = i0 + row;
                double* urow = U + (size_t)I * (I + 1) / 2;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int bj = gj * 4 + q;
                    if (bj >= nbj) break;
                    const int col = bj * 8 + 2 * (lane & 3), J = j0 + col;
                    if (col < nj && J <= I) urow[J] = tile[row * ldt + col] - c[2 * q];
                    if (col + 1 < nj && J + 1 <= I) urow[J + 1] = tile[row * ldt + col + 1] - c[2 * q + 1];
                }
            }
        }
        // ---- factor panel to global (diagonal tasks own their row chunk) ----------------------
        if (HAS_PIVOTS && p && diag) {
            double* L = lbuf + ft.l_off[f];
            if (ci == 0)
                for (int r = warp; r < p; r += nwarps)
                    for (int k = lane; k < p; k += 32) L[(size_t)r * p + k] = pan[r * ld + k];
            double* Li = L + (size_t)(p + i0) * p;
            for (int r = warp; r < ni; r += nwarps)
                for (int k = lane; k < p; k += 32) Li[(size_t)r * p + k] = Pi[r * ld + k];
        }
    }
}

void launch_front_tasks(int pclass, const FrontTab& ft, const TaskRec* tasks, int ntasks,
                        size_t smem_bytes, const double* gval, double* lbuf, double* ubuf,
                        unsigned long long* err, cudaStream_t s) {
    if (ntasks == 0) return;
    if (pclass == 0) front_task_kernel<0><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
    else front_task_kernel<1><<<ntasks, kFrontThreads, smem_bytes, s>>>(ft, tasks, gval, lbuf, ubuf, err);
}

// ---------------------------------------------------------------------------------------------
// Backward substitution: x_P = L11^{-T} (y_P - L21^T x_U).  The L21^T x_U product of a front is
// split over several CTAs (fixed row ranges, all loads issued up front); the last CTA to finish
// adds the partial sums in split order (deterministic) and runs the triangular solve in one warp.
// Restates backward / interior_recover (reference linalg.py:366-383,427-434) and dpotrs.
// ---------------------------------------------------------------------------------------------
constexpr int kBwdRows = 64;   // update rows per split

__global__ void __launch_bounds__(128) backward_kernel(FrontTab ft, const BwdTask* __restrict__ tasks,
                                                       const double* __restrict__ lbuf, double* __restrict__ xsol,
                                                       double* __restrict__ bpart, int32_t* __restrict__ bcnt) {
    __shared__ double l11[64 * 65];
    __shared__ double half[2][64];
    __shared__ double xs[kBwdRows];
    __shared__ double tv[64];
    __shared__ int s_last;
    const BwdTask tk = tasks[blockIdx.x];
    const int f = tk.front;
    const int p = ft.p[f], u = ft.u1[f] - 1;
    const double* L = lbuf + ft.l_off[f];
    const int32_t* rows = ft.rows + ft.rows_off[f];
    const int tid = threadIdx.x, k = tid & 63, h = tid >> 6;
    const int lo = tk.split * kBwdRows, n = min(kBwdRows, u - lo);
    if (tid < kBwdRows) xs[tid] = tid < n ? xsol[rows[p + lo + tid]] : 0.0;
    // the last split also prefetches L11 (needed only by whichever CTA finishes last, usually this one)
    __syncthreads();
    {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (k < p) {
            const double* col = L + (size_t)(p + lo) * p + k;
            const int a = h * (kBwdRows / 2), b = min(n, a + kBwdRows / 2);
            double v[kBwdRows / 2];
#pragma unroll
            for (int i = 0; i < kBwdRows / 2; ++i) v[i] = (a + i < b) ? __ldg(col + (size_t)(a + i) * p) : 0.0;
#pragma unroll
            for (int i = 0; i < kBwdRows / 2; i += 4) {
                s0 = fma(v[i], xs[min(a + i, kBwdRows - 1)], s0);
                s1 = fma(v[i + 1], xs[min(a + i + 1, kBwdRows - 1)], s1);
                s2 = fma(v[i + 2], xs[min(a + i + 2, kBwdRows - 1)], s2);
                s3 = fma(v[i + 3], xs[min(a + i + 3, kBwdRows - 1)], s3);
            }
        }
        half[h][k] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    if (tid < 64) bpart[(size_t)(tk.pbase + tk.split) * 64 + tid] = half[0][tid] + half[1][tid];
    if (tk.nsplit > 1) {
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&bcnt[f], 1) == tk.nsplit - 1;
        __syncthreads();
        if (!s_last) return;
        __threadfence();
    }
    // ---- last CTA of the front: combine, then solve L11^T x = t in warp 0 --------------------
    for (int r = tid >> 5; r < p; r += 4)
        for (int c = tid & 31; c < p; c += 32) l11[r * 65 + c] = L[(size_t)r * p + c];
    if (tid < 64) {
        double acc = 0.0;
        if (tid < p) {
            const volatile double* bp = bpart + (size_t)tk.pbase * 64 + tid;
            for (int s = 0; s < tk.nsplit; ++s) acc += bp[(size_t)s * 64];
            acc = L[(size_t)(p + u) * p + tid] - acc;
        }
        tv[tid] = acc;
    }
    if (tid == 0 && tk.nsplit > 1) bcnt[f] = 0;
    __syncthreads();
    if (tid < 32) {
        double t0 = tv[tid], t1 = tv[tid + 32];
        for (int c = p - 1; c >= 0; --c) {
            const double tc = __shfl_sync(0xffffffffu, c < 32 ? t0 : t1, c & 31);
            const double xc = tc / l11[c * 65 + c];
            if (tid == (c & 31)) { if (c < 32) t0 = xc; else t1 = xc; }
            if (tid < c) t0 = fma(-l11[c * 65 + tid], xc, t0);
            if (tid + 32 < c) t1 = fma(-l11[c * 65 + tid + 32], xc, t1);
        }
        if (tid < p) xsol[rows[tid]] = t0;
        if (tid + 32 < p) xsol[rows[tid + 32]] = t1;
    }
}

void launch_backward(const FrontTab& ft, const BwdTask* tasks, int ntasks, const double* lbuf,
                     double* xsol, double* bpart, int32_t* bcnt, cudaStream_t s) {
    if (ntasks == 0) return;
    backward_kernel<<<ntasks, 128, 0, s>>>(ft, tasks, lbuf, xsol, bpart, bcnt);
}

cudaError_t configure_kernels() {
    const int maxsm = 222 * 1024;   // static + dynamic must stay within the 227 KB opt-in limit
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    return cudaSuccess;
}

}  // namespace gse
