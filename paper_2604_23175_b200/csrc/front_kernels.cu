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
#include "kernels.cuh"

namespace gse {

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Extend-add as a GATHER: every destination entry of the task's shared-memory panels / tile is
// owned by one thread, which adds the contributions of the children in child order.  No barrier
// between children, no read-modify-write chains, and the loads of all children of a batch are in
// flight together -- the phase costs a few L2 latencies instead of several per child.
// inv[c][panel row] = row of child c that maps there (or -1), built from the child's rel map.
constexpr int kInvRows = 64 + 2 * kMaxTile;
constexpr int kGatherBatch = 4;

struct GatherArgs {
    double* pan; double* tile; const int* inv; const double* ubuf;
    int p, ld, ldt, rp, Rp, ni, nj, diag, direct, warp, lane, nwarps;
};

// NB children of one batch, compile-time so that empty child slots cost no instructions
template <int NB>
__device__ __forceinline__ void gather_batch(const GatherArgs& a, const ChildRec* __restrict__ crec) {
    const int p = a.p, ld = a.ld, ldt = a.ldt, rp = a.rp, Rp = a.Rp, ni = a.ni, nj = a.nj;
    const int warp = a.warp, lane = a.lane, nwarps = a.nwarps;
    const double* Ub[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) Ub[c] = a.ubuf + crec[c].u_off;
    // panel rows [pivots | I | J] x pivot columns
    if (p) {
        for (int Rb = warp; Rb < Rp; Rb += 4 * nwarps) {
            double v[NB][8];
#pragma unroll
            for (int c = 0; c < NB; ++c) {
                const int* inv = a.inv + c * kInvRows;
                int ic[2];
#pragma unroll
                for (int cp = 0; cp < 2; ++cp) { const int C = lane + 32 * cp; ic[cp] = C < p ? inv[C] : -1; }
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int R = Rb + g * nwarps;
                    const int ir = R < Rp ? inv[R] : -1;
                    const int irc = ir > 0 ? ir : 0;
                    const double* row = Ub[c] + (size_t)irc * (irc + 1) / 2;
#pragma unroll
                    for (int cp = 0; cp < 2; ++cp)
                        v[c][2 * g + cp] = (ir >= 0 && ic[cp] >= 0 && ic[cp] <= ir) ? __ldg(row + ic[cp]) : 0.0;
                }
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const int R = Rb + g * nwarps;
#pragma unroll
                for (int cp = 0; cp < 2; ++cp) {
                    const int C = lane + 32 * cp;
                    if (R < Rp && C < p) {
                        double acc = a.pan[R * ld + C];
#pragma unroll
                        for (int c = 0; c < NB; ++c) acc += v[c][2 * g + cp];
                        a.pan[R * ld + C] = acc;
                    }
                }
            }
        }
    }
    // tile: rows of chunk I x rows of chunk J
    if (!a.direct) {
        const int irow0 = rp, jrow0 = a.diag ? rp : rp + round8(ni);   // index of tile row / column 0 in inv
        for (int Cb = 0; Cb < nj; Cb += 64) {
            for (int Rb = warp; Rb < ni; Rb += 4 * nwarps) {
                double v[NB][8];
#pragma unroll
                for (int c = 0; c < NB; ++c) {
                    const int* inv = a.inv + c * kInvRows;
                    int ic[2];
#pragma unroll
                    for (int cp = 0; cp < 2; ++cp) { const int C = Cb + lane + 32 * cp; ic[cp] = C < nj ? inv[jrow0 + C] : -1; }
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const int R = Rb + g * nwarps;
                        const int ir = R < ni ? inv[irow0 + R] : -1;
                        const int irc = ir > 0 ? ir : 0;
                        const double* row = Ub[c] + (size_t)irc * (irc + 1) / 2;
#pragma unroll
                        for (int cp = 0; cp < 2; ++cp)
                            v[c][2 * g + cp] = (ir >= 0 && ic[cp] >= 0 && ic[cp] <= ir) ? __ldg(row + ic[cp]) : 0.0;
                    }
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int R = Rb + g * nwarps;
#pragma unroll
                    for (int cp = 0; cp < 2; ++cp) {
                        const int C = Cb + lane + 32 * cp;
                        if (R < ni && C < nj) {
                            double acc = a.tile[R * ldt + C];
#pragma unroll
                            for (int c = 0; c < NB; ++c) acc += v[c][2 * g + cp];
                            a.tile[R * ldt + C] = acc;
                        }
                    }
                }
            }
        }
    }
}

constexpr int kChildBatch = 32;

template <int HAS_PIVOTS>
__global__ void __launch_bounds__(kFrontThreads, HAS_PIVOTS ? 1 : 2)
front_task_kernel(FrontTab ft, const TaskRec* __restrict__ tasks, const double* __restrict__ gval,
                  double* __restrict__ lbuf, double* __restrict__ ubuf, unsigned long long* err) {
    extern __shared__ __align__(16) double sm[];
    double* __restrict__ dinv = ft.dinv;
    __shared__ __align__(16) TaskRec hdr;
    __shared__ __align__(16) ChildRec crec[kChildBatch];
    __shared__ int s_inv[kGatherBatch][kInvRows];
    __shared__ double s_ld[48];           // published 8x8 diagonal factor (36) + reciprocal pivots (8)
    __shared__ double s_rinv[64];         // reciprocal pivots of the whole front (stored for the backward pass)
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    long long* tb = ft.tbuf ? ft.tbuf + 32 * ((&tasks[blockIdx.x]) - (const TaskRec*)ft.task0) : nullptr;
#define GSE_TICK(k) do { if (tb && tid == 0) tb[k] = clock64(); } while (0)
    GSE_TICK(0);
    if (tid < (int)(sizeof(TaskRec) / 16))
        reinterpret_cast<int4*>(&hdr)[tid] = reinterpret_cast<const int4*>(&tasks[blockIdx.x])[tid];
    __syncthreads();
    const int f = hdr.front, ci = hdr.ci, cj = hdr.cj;
    const int p = HAS_PIVOTS ? hdr.p : 0;
    const int u1 = hdr.u1, T = hdr.T;
    const int i0 = ci * T, ni = min(T, u1 - i0), j0 = cj * T, nj = min(T, u1 - j0);
    const bool diag = ci == cj;
    const bool direct = (hdr.flags & 1) != 0;      // tile comes straight from the single child's U
    const int ld = pad_ld(p);
    const int rp = p ? round8(p) : 0, ri = p ? round8(ni) : 0, rj = (p && !diag) ? round8(nj) : 0;
    const int ldt = round8(nj) | 1;
    double* pan = sm;
    double* tile = sm + (size_t)(rp + ri + rj) * ld;
    // first batch of child records: issue now, consume after the zero fill
    const int nchild = hdr.nchild;
    if (tid < 2 * min(nchild, kChildBatch))
        reinterpret_cast<int4*>(crec)[tid] = reinterpret_cast<const int4*>(ft.crecs + hdr.child_off)[tid];

    {
        const int total = ((rp + ri + rj) * ld + (direct ? 0 : round8(ni) * ldt) + 1) >> 1;
        double2* z2 = reinterpret_cast<double2*>(sm);
        for (int t = tid; t < total; t += nth) z2[t] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (HAS_PIVOTS && tid < rp - p) pan[(p + tid) * ld + p + tid] = 1.0;   // identity on padded pivots
    GSE_TICK(1);

    // ---- original entries (written by accumulate_kernel into gval), four loads in flight ------
    {
        const uint32_t* opos = ft.orig_pos + hdr.gval_off;
        const double* gv = gval + hdr.gval_off;
        auto scatter = [&](int b, int e, double* dst, int ldd, int rsub, int csub) {
            for (int e0 = b + tid; e0 < e; e0 += 4 * nth) {
                uint32_t q[4];
                double v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int ee = e0 + k * nth;
                    q[k] = ee < e ? opos[ee] : 0u;
                    v[k] = ee < e ? gv[ee] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (e0 + k * nth < e) dst[((int)(q[k] >> 16) - rsub) * ldd + ((int)(q[k] & 0xffffu) - csub)] = v[k];
            }
        };
        if (p) {
            scatter(hdr.reg[0], hdr.reg[1], pan, ld, 0, 0);
            scatter(hdr.reg[2], hdr.reg[3], pan + (size_t)rp * ld, ld, p + i0, 0);
            if (!diag) scatter(hdr.reg[4], hdr.reg[5], pan + (size_t)(rp + ri) * ld, ld, p + j0, 0);
        }
        scatter(hdr.reg[6], hdr.reg[7], tile, ldt, p + i0, p + j0);
    }
    __syncthreads();
    GSE_TICK(2);

    // ---- extend-add of the children's update matrices, fixed child order (gather form) -------
    // (the child list of a task is pruned on the host to the children that reach its regions)
    for (int cb0 = 0; cb0 < nchild; cb0 += kGatherBatch) {
        const int nb = min(kGatherBatch, nchild - cb0);
        const int Rp = rp + ri + rj;
        if (cb0 && (cb0 % kChildBatch) == 0) {          // next page of child records
            __syncthreads();
            if (tid < 2 * min(kChildBatch, nchild - cb0))
                reinterpret_cast<int4*>(crec)[tid] = reinterpret_cast<const int4*>(ft.crecs + hdr.child_off + cb0)[tid];
        }
        __syncthreads();
        for (int t = tid; t < kGatherBatch * kInvRows; t += nth) (&s_inv[0][0])[t] = -1;
        __syncthreads();
        const int cbase = cb0 % kChildBatch;
        for (int c = 0; c < nb; ++c) {
            const ChildRec& cr = crec[cbase + c];
            const int32_t* rel = ft.rel + cr.rel_off;
            const int eP = p ? cr.eP : 0, nI = cr.eI - cr.bI, nJ = diag ? 0 : cr.eJ - cr.bJ;
            for (int t = tid; t < eP + nI + nJ; t += nth) {
                if (t < eP) s_inv[c][rel[t]] = t;
                else if (t < eP + nI) { const int i = cr.bI + t - eP; s_inv[c][rp + rel[i] - p - i0] = i; }
                else { const int i = cr.bJ + t - eP - nI; s_inv[c][rp + round8(ni) + rel[i] - p - j0] = i; }
            }
        }
        __syncthreads();
        if (cb0 == 0) GSE_TICK(7);
        GatherArgs ga{pan, tile, &s_inv[0][0], ubuf, p, ld, ldt, rp, Rp, ni, nj, diag ? 1 : 0, direct ? 1 : 0, warp, lane, nwarps};
        const ChildRec* cb = crec + cbase;
        switch (nb) {
            case 1: gather_batch<1>(ga, cb); break;
            case 2: gather_batch<2>(ga, cb); break;
            case 3: gather_batch<3>(ga, cb); break;
            default: gather_batch<4>(ga, cb); break;
        }
    }
    __syncthreads();
    GSE_TICK(3);

    // ---- blocked panel factorisation (block = 8 columns) ---------------------------------------
    // Per block: warp 0 updates the 8x8 diagonal tile (four independent MMA chains), factors it in
    // registers and publishes it while the other warps update the remaining row tiles on the tensor
    // pipe (look-ahead); then every row solves against the published block (right-looking:
    // independent FMAs).  Two barriers per 8 pivots.
    if (HAS_PIVOTS && p) {
        const int R = rp + ri + rj;                 // padded rows: [pivots | chunk I | chunk J]
        const int ntile = R >> 3;
        for (int kb = 0; kb < rp; kb += 8) {
            const int t0 = kb >> 3;
            if (warp == 0) {
                if (kb) {
                    const double* ap = pan + (size_t)(kb + (lane >> 2)) * ld + (lane & 3);
                    double c[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                    int kk = 0;
                    for (; kk + 12 < kb; kk += 16) {         // four independent chains
                        dmma_m8n8k4(c[0], c[1], ap[kk], ap[kk]);
                        dmma_m8n8k4(c[2], c[3], ap[kk + 4], ap[kk + 4]);
                        dmma_m8n8k4(c[4], c[5], ap[kk + 8], ap[kk + 8]);
                        dmma_m8n8k4(c[6], c[7], ap[kk + 12], ap[kk + 12]);
                    }
                    for (; kk < kb; kk += 4) dmma_m8n8k4(c[0], c[1], ap[kk], ap[kk]);
                    double* o = pan + (size_t)(kb + (lane >> 2)) * ld + kb + 2 * (lane & 3);
                    o[0] -= (c[0] + c[2]) + (c[4] + c[6]); o[1] -= (c[1] + c[3]) + (c[5] + c[7]);
                    __syncwarp();
                }
                double d[36];   // lower triangle, row-major: d[i*(i+1)/2 + j]
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j <= i; ++j) d[i * (i + 1) / 2 + j] = pan[(kb + i) * ld + kb + j];
                double rinv[8];
                int badk = -1;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double dk = d[k * (k + 1) / 2 + k];
                    if (!(dk > 0.0) && badk < 0) badk = k;
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
                // publish: every lane holds the same values; lane l writes entries l and l + 32
                {
                    double v0 = 0.0, v1 = 0.0;
#pragma unroll
                    for (int i = 0; i < 32; ++i) if (lane == i) v0 = d[i];
#pragma unroll
                    for (int i = 32; i < 36; ++i) if (lane == i - 32) v1 = d[i];
#pragma unroll
                    for (int k = 0; k < 8; ++k) if (lane == 4 + k) v1 = rinv[k];
                    s_ld[lane] = v0;
                    if (lane < 12) s_ld[32 + lane] = v1;
                    if (lane >= 4 && lane < 12 && kb + lane - 4 < p) s_rinv[kb + lane - 4] = v1;
                    if (lane == 0 && badk >= 0 && kb + badk < p) atomicMin(err, ((unsigned long long)f << 32) | (unsigned long long)(kb + badk));
                }
            } else if (kb) {
                // rows below the diagonal tile: block column kb -= A[rows, 0:kb] * A[kb:kb+8, 0:kb]^T
                const int nw = nwarps - 1;
                for (int tb2 = t0 + 1 + (warp - 1); tb2 < ntile; tb2 += 2 * nw) {
                    const int ta = tb2, tc2 = tb2 + nw;
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
            }
            __syncthreads();
            // every row at or below the block solves against the published 8x8 factor
            if (tid >= kb && tid < R) {
                double* myrow = pan + (size_t)tid * ld + kb;
                if (tid < kb + 8) {
                    const int i = tid - kb;
#pragma unroll
                    for (int j = 0; j < 8; ++j) myrow[j] = j <= i ? s_ld[i * (i + 1) / 2 + j] : 0.0;
                } else {
                    double y[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) y[j] = myrow[j];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        y[k] *= s_ld[36 + k];
#pragma unroll
                        for (int j = k + 1; j < 8; ++j) y[j] = fma(-y[k], s_ld[j * (j + 1) / 2 + k], y[j]);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) myrow[j] = y[j];
                }
            }
            __syncthreads();
        }
    }
    GSE_TICK(4);

    // ---- trailing update on the FP64 tensor pipe: U_IJ = F_IJ - L_I L_J^T -------------------
    {
        const double* Pi = pan + (size_t)rp * ld;
        const double* Pj = diag ? Pi : pan + (size_t)(rp + ri) * ld;
        const int nbi = round8(ni) >> 3, nbj = round8(nj) >> 3;
        const int ngj = (nbj + 3) >> 2;                 // groups of four 8-wide column blocks
        const int kend = (p + 3) & ~3;
        double* U = ubuf + hdr.u_off;
        const double* Uc = direct ? ubuf + crec[0].u_off : nullptr;   // chain: F_IJ lives in the child's U
        for (int w = warp; w < nbi * ngj; w += nwarps) {
            const int bi = w / ngj, gj = w % ngj;
            if (diag && gj * 4 > bi) continue;
            const int row = bi * 8 + (lane >> 2);
            const int I = i0 + row;
            double fv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) fv[q] = 0.0;
            if (direct && row < ni) {
                const double* crow = Uc + (size_t)(p + I) * (p + I + 1) / 2 + p;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = (gj * 4 + q) * 8 + 2 * (lane & 3), J = j0 + col;
                    if (col < nj && J <= I) fv[2 * q] = __ldg(crow + J);
                    if (col + 1 < nj && J + 1 <= I) fv[2 * q + 1] = __ldg(crow + J + 1);
                }
            }
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
            if (row < ni) {
                double* urow = U + (size_t)I * (I + 1) / 2;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int bj = gj * 4 + q;
                    if (bj >= nbj) break;
                    const int col = bj * 8 + 2 * (lane & 3), J = j0 + col;
                    if (col < nj && J <= I) urow[J] = (direct ? fv[2 * q] : tile[row * ldt + col]) - c[2 * q];
                    if (col + 1 < nj && J + 1 <= I) urow[J + 1] = (direct ? fv[2 * q + 1] : tile[row * ldt + col + 1]) - c[2 * q + 1];
                }
            }
        }
        GSE_TICK(5);
        // ---- factor panel to global (diagonal tasks own their row chunk) ----------------------
        if (HAS_PIVOTS && p && diag) {
            double* L = lbuf + hdr.l_off;
            if (ci == 0) {
                for (int r = warp; r < p; r += nwarps)
                    for (int k = lane; k < p; k += 32) L[(size_t)r * p + k] = pan[r * ld + k];
                if (tid < p) dinv[hdr.dinv_off + tid] = s_rinv[tid];
            }
            double* Li = L + (size_t)(p + i0) * p;
            for (int r = warp; r < ni; r += nwarps)
                for (int k = lane; k < p; k += 32) Li[(size_t)r * p + k] = Pi[r * ld + k];
        }
        GSE_TICK(6);
    }
#undef GSE_TICK
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
    const int p = tk.p, u = tk.u;
    const double* L = lbuf + tk.l_off;
    const int32_t* rows = ft.rows + tk.rows_off;
    const int tid = threadIdx.x, k = tid & 63, h = tid >> 6;
    const int lo = tk.split * kBwdRows, n = min(kBwdRows, u - lo);
    // L11 is needed only by the CTA that finishes last; every CTA prefetches it asynchronously so
    // the copy overlaps the matrix-vector part instead of following the atomic hand-off
    for (int t = tid; t < p * p; t += 128) {
        const int r = t / p, c = t - r * p;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&l11[r * 65 + c]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(L + t));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const double yk = (tid < p) ? __ldg(L + (size_t)(p + u) * p + tid) : 0.0;
    if (tid < kBwdRows) xs[tid] = tid < n ? xsol[rows[p + lo + tid]] : 0.0;
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
        if (!s_last) { asm volatile("cp.async.wait_group 0;\n" ::); return; }
        __threadfence();
    }
    // ---- last CTA of the front: combine (split order), then solve L11^T x = t in warp 0 ------
    if (tid < 64) {
        double acc = 0.0;
        if (tid < p) {
            const volatile double* bp = bpart + (size_t)tk.pbase * 64 + tid;
            int s = 0;
            for (; s + 3 < tk.nsplit; s += 4) {
                const double b0 = bp[(size_t)s * 64], b1 = bp[(size_t)(s + 1) * 64], b2 = bp[(size_t)(s + 2) * 64], b3 = bp[(size_t)(s + 3) * 64];
                acc = (((acc + b0) + b1) + b2) + b3;
            }
            for (; s < tk.nsplit; ++s) acc += bp[(size_t)s * 64];
            acc = yk - acc;
        }
        tv[tid] = acc;
    }
    if (tid == 0 && tk.nsplit > 1) bcnt[f] = 0;
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (tid < 32) {
        double t0 = tv[tid], t1 = tv[tid + 32];
        const double* di = ft.dinv + tk.dinv_off;
        const double r0 = tid < p ? di[tid] : 0.0, r1 = tid + 32 < p ? di[tid + 32] : 0.0;
        for (int c = p - 1; c >= 0; --c) {
            const double xc = __shfl_sync(0xffffffffu, c < 32 ? t0 * r0 : t1 * r1, c & 31);
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
    const int maxsm = 214 * 1024;   // static + dynamic must stay within the 227 KB opt-in limit
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(front_task_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    return cudaSuccess;
}

}  // namespace gse
