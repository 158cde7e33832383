// front_body.cuh -- device bodies of the multifrontal factorisation task and of the backward
// substitution task, shared by the level-launch kernels (front_kernels.cu) and the persistent
// dataflow kernel (solve_kernel.cu).  Loads of data produced by other CTAs go through ldc()
// (ld.global.cg, L2-coherent): see unit_bodies.cuh.
#pragma once
#include <type_traits>

#include "kernels.cuh"
#include "unit_bodies.cuh"

namespace gse {

#ifndef GSE_PANEL_QUIET
#define GSE_PANEL_QUIET 1
#endif
#ifndef GSE_CHILD_G
#define GSE_CHILD_G 3      // extend-add: child rows per warp and sweep (4: +0.2 %, 6: +2 %, 8: +4 % at PEGASE-9241/16; 2 and 1 slower)
#endif
#ifndef GSE_CHAIN_G
#define GSE_CHAIN_G 8      // chain pieces: child rows per warp and sweep of the direct copy (two loads per lane and row in flight; 6: +0.4 %, 10: no better)
#endif
#ifndef GSE_UPDATE_NARROW
#define GSE_UPDATE_NARROW 1
#endif

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Extend-add as a GATHER in fixed child order: no atomics, no read-modify-write chains in global memory.  Each child is
// walked by ITS rows -- a child row holds its entries contiguously, so a warp reads them coalesced, and only rows the
// child really has are visited -- and added to the task's shared-memory panels / tile through its child -> parent map;
// a CTA barrier separates two children, so every entry takes the children's contributions one after the other, in
// child order (the sums do not depend on which children were already complete when the task started).
// (A panel-driven form -- every destination entry owned by one thread that adds the children of a batch in order, the
// loads of up to four children in flight together -- was the first implementation; it picks the entries column by
// column through inverse maps, uncoalesced, and lost against this one on every shape: profiles/r02_sweep_build_constants.txt.)
constexpr int kInvRows = 64 + 2 * kMaxTile;
constexpr int kGatherBatch = 4;

struct GatherArgs {
    double* pan; double* tile; const double* ubuf;
    int p, ld, ldt, rp, ni, nj, diag, direct, warp, lane, nwarps;
};

// One child.  fwd: its child -> parent map (FrontScratch::fwd[c]): [0, eP) pivot row / column, then the tile rows of its
// rows in chunk I, then the tile columns of its rows in chunk J; eP / bI,eI / bJ,eJ: its row ranges (ChildRec).
// G child rows per warp and sweep.
template <int G>
__device__ __forceinline__ void gather_child(const GatherArgs& a, const ChildRec& cr, const int* __restrict__ fwd, int ri, long long* tb = nullptr) {
    const int p = a.p, ld = a.ld, ldt = a.ldt, rp = a.rp, warp = a.warp, lane = a.lane, nwarps = a.nwarps;
    const double* Uc = a.ubuf + cr.u_off;
    const int eP = p ? cr.eP : 0, nI = cr.eI - cr.bI, nJ = a.diag ? 0 : cr.eJ - cr.bJ;
    // panel: child rows that map into [pivots | chunk I | chunk J], child columns that map into the pivots
    if (eP > 0) {
        const int Rc = eP + nI + nJ;
        for (int rb = warp; rb < Rc; rb += G * nwarps) {
            double v[G][2];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int tt = rb + g * nwarps;
                const int t = tt < eP ? tt : tt < eP + nI ? cr.bI + tt - eP : cr.bJ + tt - eP - nI;      // child row
                const double* src = Uc + (size_t)t * (t + 1) / 2;
#pragma unroll
                for (int h = 0; h < 2; ++h) { const int j = lane + 32 * h; v[g][h] = (tt < Rc && j < eP && j <= t) ? ldc(src + j) : 0.0; }
            }
            // (the sixteen read-modify-writes of a lane hit distinct panel entries, but the compiler cannot know: written
            // one after the other they form a chain of shared-memory round trips.  All reads first, then all writes.)
            int off[G][2];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int tt = rb + g * nwarps;
                const int t = tt < eP ? tt : tt < eP + nI ? cr.bI + tt - eP : cr.bJ + tt - eP - nI;
                const int R = tt >= Rc ? 0 : tt < eP ? fwd[tt] : tt < eP + nI ? rp + fwd[tt] : rp + ri + fwd[tt];
#pragma unroll
                for (int h = 0; h < 2; ++h) { const int j = lane + 32 * h; off[g][h] = (tt < Rc && j < eP && j <= t) ? R * ld + fwd[j] : -1; }
            }
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int h = 0; h < 2; ++h) if (off[g][h] >= 0) v[g][h] += a.pan[off[g][h]];
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int h = 0; h < 2; ++h) if (off[g][h] >= 0) a.pan[off[g][h]] = v[g][h];
        }
    }
    if (tb && threadIdx.x == 0) tb[17] = (long long)gtimer();
    // tile: child rows in chunk I x child columns in chunk J (the lower triangle of the child's matrix)
    if (!a.direct && nI > 0) {
        const int bC = a.diag ? cr.bI : cr.bJ, nC = a.diag ? nI : nJ;       // child columns [bC, bC + nC) and where their map starts in fwd
        const int fC = a.diag ? eP : eP + nI;
        for (int cb = 0; cb < nC; cb += 64) {
            for (int rb = warp; rb < nI; rb += G * nwarps) {
                double v[G][2];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int ti = rb + g * nwarps, t = cr.bI + ti;
                    const double* src = Uc + (size_t)t * (t + 1) / 2 + bC;
#pragma unroll
                    for (int h = 0; h < 2; ++h) { const int jj = cb + lane + 32 * h; v[g][h] = (ti < nI && jj < nC && bC + jj <= t) ? ldc(src + jj) : 0.0; }
                }
                int off[G][2];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int ti = rb + g * nwarps, t = cr.bI + ti;
                    const int R = ti < nI ? fwd[eP + ti] : 0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) { const int jj = cb + lane + 32 * h; off[g][h] = (ti < nI && jj < nC && bC + jj <= t) ? R * ldt + fwd[fC + jj] : -1; }
                }
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int h = 0; h < 2; ++h) if (off[g][h] >= 0) v[g][h] += a.tile[off[g][h]];
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int h = 0; h < 2; ++h) if (off[g][h] >= 0) a.tile[off[g][h]] = v[g][h];
            }
        }
    }
}

constexpr int kChildBatch = 32;

// Diagonal 8x8 blocks of the pivot triangle are kept RIGHT-looking: as soon as a block column
// [kc, kc + 8) of the panel is final, every later diagonal block t takes its share
// D_t -= A[t, kc:kc+8] A[t, kc:kc+8]^T (two MMAs).  The block about to be factored is then always
// up to date and the serial chain of the panel never waits for a long left-looking product.
__device__ __forceinline__ void diag_rank8(double* pan, int ld, int t, int kc, int lane) {
    const double* ap = pan + (size_t)(t * 8 + (lane >> 2)) * ld + kc + (lane & 3);
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
    dmma_m8n8k4(c0, c1, ap[0], ap[0]);
    dmma_m8n8k4(e0, e1, ap[4], ap[4]);
    double* o = pan + (size_t)(t * 8 + (lane >> 2)) * ld + t * 8 + 2 * (lane & 3);
    o[0] -= c0 + e0; o[1] -= c1 + e1;
}

// Static shared scratch of one front task (the panels / tile live in dynamic shared memory).
struct __align__(16) FrontScratch {
    TaskRec hdr;
    ChildRec crec[kChildBatch];
    int fwd[kGatherBatch][kInvRows];   // per child of the current batch, child -> parent: [0, eP) pivot row / column, then the tile
                               // rows of its rows in chunk I, then the tile columns of its rows in chunk J (gather_child)
    double ld8[2][48];         // published 8x8 diagonal factor (36) + reciprocal pivots (8), double-buffered
    double rinv[64];           // reciprocal pivots of the whole front (stored for the backward pass)
    double colbuf[2][16];      // two columns of the 8x8 pivot block being eliminated (double-buffered)
    int nready;                // children of the current gather batch that are complete
};

__device__ __forceinline__ void load_task_header(FrontScratch& S, const TaskRec* __restrict__ task) {
    if (threadIdx.x < (int)(sizeof(TaskRec) / 16))
        reinterpret_cast<int4*>(&S.hdr)[threadIdx.x] = reinterpret_cast<const int4*>(task)[threadIdx.x];
}

// Dependency hooks of a front task.  The level-launch kernels run a whole tree level per launch,
// so their hooks are empty; the persistent kernel spins on completion counters here.
struct NoWait {
    static constexpr bool kEarlySplits = false;      // one launch per level: every split of a level starts together
    __device__ __forceinline__ void ancestor(const BwdTask&) const {}
    __device__ __forceinline__ void splits(const int32_t*, int) const {}
    __device__ __forceinline__ void factor(const BwdTask&) const {}
    __device__ __forceinline__ void parent(const BwdTask&) const {}
    __device__ __forceinline__ void originals(const TaskRec&) const {}
    __device__ __forceinline__ void children(const TaskRec&, const ChildRec*) const {}
    __device__ __forceinline__ int ready_children(const TaskRec&, const ChildRec*, int c, int nb, int*) const { return nb - c; }
    __device__ __forceinline__ void panels(const TaskRec&) const {}
    __device__ __forceinline__ void tile_done(const TaskRec&) const {}
    __device__ __forceinline__ bool poll_x() const { return false; }
    __device__ __forceinline__ double load_x(const double* p) const { return ldc(p); }
};

// Back-substitution hand-off through the data (dataflow kernel, single rank): the forward task that owns a front's pivots
// arms their entries of the solution vector with this pattern (all ones: a NaN no arithmetic produces; the producers
// store the canonical NaN instead of any other), the front's back-substitution overwrites them, and the descendants
// poll the entries they read instead of a completion counter followed by a load -- no fence and no atomic on the
// chain of twelve levels, and every split waits for exactly the ancestors it reads.
__device__ __forceinline__ double x_unset() { return __longlong_as_double(-1LL); }
__device__ __forceinline__ bool x_is_unset(double v) { return __double_as_longlong(v) == -1LL; }

// One front task; S.hdr is loaded and visible to the whole CTA.  tb: optional 8 clock stamps.
// Task kinds (TaskRec::kind):
//   0 fused   -- assemble [pivots | I | J] + tile, factor, update, store (fronts with one row chunk
//                or few pivots: recomputing the pivot block per task is cheaper than a hand-off);
//   1 panel   -- assemble [pivots | I], factor the pivot block, solve chunk I against it and store
//                its slice of the factor panel (ci == cj on the host side; no tile);
//   2 update  -- assemble the tile, then read the finished panels L_I, L_J of the front back from
//                the factor storage and run the trailing update (no pivot rows in shared memory).
// wait.originals() runs before the first read of gval, wait.children() / wait.ready_children() before
// the first read of a child's update matrix (they end with a CTA barrier when they waited), wait.panels() before
// the first read of the front's own factor panels (kind 2).
template <int HAS_PIVOTS, class Wait>
__device__ __forceinline__ void front_task_body(FrontScratch& S, double* sm, const FrontTab& ft, const double* gval,
                                                double* lbuf, double* ubuf, unsigned long long* err, long long* tb,
                                                const Wait& wait, double* xarm = nullptr) {
    double* dinv = ft.dinv;
    const TaskRec& hdr = S.hdr;
    ChildRec* crec = S.crec;
    int (*s_fwd)[kInvRows] = S.fwd;
    double* s_ld = &S.ld8[0][0];
    double* s_rinv = S.rinv;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
#define GSE_TICK(k) do { if (tb && tid == 0) tb[k] = (long long)gtimer(); } while (0)   // globaltimer, ns
    GSE_TICK(0);
    const int f = hdr.front, ci = hdr.ci, cj = hdr.cj;
    const int p = HAS_PIVOTS ? hdr.p : 0;
    const int u1 = hdr.u1, T = hdr.T;
    const int i0 = ci * T, ni = min(T, u1 - i0), j0 = cj * T, nj = min(T, u1 - j0);
    const bool diag = ci == cj;
    const int kind = HAS_PIVOTS ? hdr.kind : 0;
    const bool no_tile = kind == 1;
    const bool direct = (hdr.flags & 1) != 0;      // tile comes straight from the single child's U
    const int pp = kind == 2 ? 0 : p;              // pivot rows assembled and factored by this task
    const int ld = pad_ld(p);
    const int rp = pp ? round8(pp) : 0, ri = p ? round8(ni) : 0, rj = (p && !diag) ? round8(nj) : 0;
    const int ldt = round8(nj) | 1;
    double* pan = sm;
    double* tile = sm + (size_t)(rp + ri + rj) * ld;
    // (dataflow kernel) the task that owns the front's pivots arms their solution entries for this iteration's
    // back-substitution: every reader of the previous iteration's values finished before this iteration started
    if (HAS_PIVOTS && xarm && pp && ci == 0 && cj == 0 && tid < p) xarm[ft.rows[ft.rows_off[f] + tid]] = x_unset();
    // first batch of child records: issue now, consume after the zero fill
    const int nchild = hdr.nchild;
    if (tid < 3 * min(nchild, kChildBatch))
        reinterpret_cast<int4*>(crec)[tid] = reinterpret_cast<const int4*>(ft.crecs + hdr.child_off)[tid];

    {
        const int total = ((rp + ri + rj) * ld + ((direct || no_tile) ? 0 : round8(ni) * ldt) + 1) >> 1;
        double2* z2 = reinterpret_cast<double2*>(sm);
        for (int t = tid; t < total; t += nth) z2[t] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (HAS_PIVOTS && pp && tid < rp - p) pan[(p + tid) * ld + p + tid] = 1.0;   // identity on padded pivots
    GSE_TICK(1);

    // ---- original entries (written by accumulate_kernel into gval), four loads in flight ------
    wait.originals(hdr);
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
                    v[k] = ee < e ? ldc(gv + ee) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (e0 + k * nth < e) dst[((int)(q[k] >> 16) - rsub) * ldd + ((int)(q[k] & 0xffffu) - csub)] = v[k];
            }
        };
        if (pp) {
            scatter(hdr.reg[0], hdr.reg[1], pan, ld, 0, 0);
            scatter(hdr.reg[2], hdr.reg[3], pan + (size_t)rp * ld, ld, p + i0, 0);
            if (!diag) scatter(hdr.reg[4], hdr.reg[5], pan + (size_t)(rp + ri) * ld, ld, p + j0, 0);
        }
        if (!no_tile) scatter(hdr.reg[6], hdr.reg[7], tile, ldt, p + i0, p + j0);
    }
    __syncthreads();
    GSE_TICK(2);

    // ---- extend-add of the children's update matrices, fixed child order (gather form) -------
    // (the child list of a task is pruned on the host to the children that reach its regions)
    // (everything static -- child records, row maps -- is staged BEFORE waiting for the children, so
    // that only the loads of their update matrices follow the hand-off)
    if (direct && nchild == 1) {
        // Chain piece: the single child's update rows ARE this front's rows (identity map, no original
        // entries).  The tile is read in place later; the panel rows are a plain copy of row prefixes
        // of the child's packed update matrix -- coalesced, no index maps, sixteen loads per lane in flight.
        GSE_TICK(7);
        wait.children(hdr, ft.crecs + hdr.child_off);
        if (pp) {
            const double* Uc = ubuf + crec[0].u_off;
            const int Rn = p + ni + (diag ? 0 : nj);
            for (int rb = warp; rb < Rn; rb += GSE_CHAIN_G * nwarps) {
                double v[GSE_CHAIN_G][2];
#pragma unroll
                for (int g = 0; g < GSE_CHAIN_G; ++g) {
                    const int r = rb + g * nwarps;
                    const int cr_ = r < p ? r : r < p + ni ? p + i0 + (r - p) : p + j0 + (r - p - ni);   // child row
                    const double* src = Uc + (size_t)cr_ * (cr_ + 1) / 2;
#pragma unroll
                    for (int h = 0; h < 2; ++h) { const int C = lane + 32 * h; v[g][h] = (r < Rn && C < p && C <= cr_) ? ldc(src + C) : 0.0; }
                }
#pragma unroll
                for (int g = 0; g < GSE_CHAIN_G; ++g) {
                    const int r = rb + g * nwarps;
                    const int sr = r < p ? r : r < p + ni ? rp + (r - p) : rp + ri + (r - p - ni);      // panel row
#pragma unroll
                    for (int h = 0; h < 2; ++h) { const int C = lane + 32 * h; if (r < Rn && C < p) pan[sr * ld + C] += v[g][h]; }
                }
            }
        }
    } else
    for (int cb0 = 0; cb0 < nchild; cb0 += kGatherBatch) {
        const int nb = min(kGatherBatch, nchild - cb0);
        if (cb0 && (cb0 % kChildBatch) == 0) {          // next page of child records
            __syncthreads();
            if (tid < 3 * min(kChildBatch, nchild - cb0))
                reinterpret_cast<int4*>(crec)[tid] = reinterpret_cast<const int4*>(ft.crecs + hdr.child_off + cb0)[tid];
        }
        __syncthreads();
        const int cbase = cb0 % kChildBatch;
        for (int c = 0; c < nb; ++c) {
            const ChildRec& cr = crec[cbase + c];
            const int32_t* rel = ft.rel + cr.rel_off;
            const int eP = pp ? cr.eP : 0, nI = cr.eI - cr.bI, nJ = diag ? 0 : cr.eJ - cr.bJ;
            for (int t = tid; t < eP + nI + nJ; t += nth) {
                if (t < eP) s_fwd[c][t] = rel[t];
                else if (t < eP + nI) s_fwd[c][t] = rel[cr.bI + t - eP] - p - i0;
                else s_fwd[c][t] = rel[cr.bJ + t - eP - nI] - p - j0;
            }
        }
        __syncthreads();
        if (cb0 == 0) GSE_TICK(7);
        // children in order; whatever is already complete is folded in while the task still waits for a slower sibling
        const GatherArgs ga{pan, tile, ubuf, pp, ld, ldt, rp, ni, nj, diag ? 1 : 0, (direct || no_tile) ? 1 : 0, warp, lane, nwarps};
        for (int c = 0; c < nb;) {
            const int ready = wait.ready_children(hdr, ft.crecs + hdr.child_off + cb0, c, nb, &S.nready);
            for (int k = 0; k < ready; ++k) {
                __syncthreads();               // (the earlier children's sums are in place)
                const bool stamp = tb && c + k == nb - 1 && cb0 + nb == nchild;      // the task's last child
                if (stamp && tid == 0) tb[16] = (long long)gtimer();
                gather_child<GSE_CHILD_G>(ga, crec[cbase + c + k], &s_fwd[c + k][0], ri, stamp ? tb : nullptr);
                if (stamp && tid == 0) tb[18] = (long long)gtimer();
            }
            c += ready;
        }
    }
    __syncthreads();
    GSE_TICK(3);

    // ---- blocked panel factorisation (block = 8 columns), software-pipelined -------------------
    // Warp 0 owns the serial chain: per block k it brings the 8x8 diagonal tile up to date (rank-8 share of
    // the previous block column), eliminates it across its lanes, publishes the factor, solves the NEXT
    // pivot tile's eight rows against it -- and goes straight on to block k + 1.  The other warps trail one
    // step behind: they solve the remaining rows against block k, then run the right-looking diagonal
    // updates and the left-looking DMMA update of block column k + 1 while warp 0 already eliminates
    // block k + 1.  Per block: one CTA barrier (factor published / column k + 1 current) and one named
    // barrier that warp 0 only arrives at (its tile solve is done) -- the chain never waits for the bulk
    // row solves.  The published factor is double-buffered for the same reason.
    if (HAS_PIVOTS && pp) {
        const int R = rp + ri + rj;                 // padded rows: [pivots | chunk I | chunk J]
        const int ntile = R >> 3;
        long long pc[7] = {0, 0, 0, 0, 0, 0, 0}, pt = tb ? clock64() : 0;   // debug: cycles per panel sub-phase (thread 0)
#define GSE_PC(k) do { if (tb) { const long long now = clock64(); pc[k] += now - pt; pt = now; } } while (0)
        // one row of the panel against the published 8x8 factor (16-byte accesses: the row stride maps eight
        // rows onto four bank groups, so 8-byte accesses of one row per thread would be 8-way bank conflicted)
        auto solve_row = [&](int row, int kb, const double* sl) {
            double y[8];
            double2* my2 = reinterpret_cast<double2*>(pan + (size_t)row * ld + kb);
#pragma unroll
            for (int j = 0; j < 4; ++j) { const double2 t2 = my2[j]; y[2 * j] = t2.x; y[2 * j + 1] = t2.y; }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                y[k] *= sl[36 + k];
#pragma unroll
                for (int j = k + 1; j < 8; ++j) y[j] = fma(-y[k], sl[j * (j + 1) / 2 + k], y[j]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) my2[j] = make_double2(y[2 * j], y[2 * j + 1]);
        };
        // helper warps of the tensor-pipe work: the warps that share warp 0's scheduler (and with it its FP64 /
        // tensor issue port: an m8n8k4 DMMA holds the port for ~16 cycles, profiles/r01_microbench_b200.txt)
        // stay off the pipe, so the serial chain is not queued behind their MMAs
        const bool quiet = GSE_PANEL_QUIET && nwarps >= 8 && (nwarps & 3) == 0;
        const bool helper = warp != 0 && (!quiet || (warp & 3) != 0);
        const int nw = quiet ? nwarps - (nwarps >> 2) : nwarps - 1;
        const int wi = quiet ? warp - 1 - (warp >> 2) : warp - 1;
        for (int kb = 0; kb < rp; kb += 8) {
            const int t0 = kb >> 3;
            double* sl = s_ld + (t0 & 1) * 48;
            if (warp == 0) {
                // The 8x8 diagonal block lives in the MMA accumulator layout: lane (r = lane / 4, c = lane % 4)
                // holds D[r][2c], D[r][2c + 1].  It is loaded with one 16-byte read, takes the last block
                // column's share straight in registers, and is eliminated by all 32 lanes together.
                const int r = lane >> 2, c2 = 2 * (lane & 3);
                double2* dptr = reinterpret_cast<double2*>(pan + (size_t)(kb + r) * ld + kb + c2);
                const double2 dt = *dptr;
                double x0 = dt.x, x1 = dt.y;
                if (kb) {
                    const double* ap = pan + (size_t)(kb + r) * ld + (kb - 8) + (lane & 3);
                    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
                    dmma_m8n8k4(c0, c1, ap[0], ap[0]);
                    dmma_m8n8k4(e0, e1, ap[4], ap[4]);
                    x0 -= c0 + e0; x1 -= c1 + e1;
                }
                GSE_PC(0);
                // Division-free elimination: step k cross-multiplies
                //     a_ij <- (p_k a_ij - a_ik a_jk) * 2^-e,   p_k = a_kk,   2^e ~ p_k  (exact scaling),
                // one multiply-add per lane, so the serial chain per pivot is shuffle -> multiply -> FMA
                // instead of a reciprocal square root.  Stage-k entries equal c_k times the true Schur
                // complement, c_{k+1} = c_k p_k 2^-e in [1, 2^k); hence L_ik = a_ik / sqrt(p_k c_k) and
                // 1 / L_kk = c_k / sqrt(p_k c_k): the eight reciprocal square roots are independent and
                // run after the chain, one per lane.
                int badk = -1;
                double cs = 1.0, mine = 1.0, myc = 1.0;
                // two pivots per round: one exchange fetches what both elimination steps need
                // (columns k and k + 1 of the block live in the same lanes), the stage k+1 values of
                // column k + 1 are recomputed locally, and the serial chain per PAIR of pivots is one
                // shared-memory exchange plus ~7 dependent FP64 operations.
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    const int kh = k >> 1;
                    // columns k, k + 1 of the block go through a 16-double shared buffer: one 16-byte store by
                    // the eight lanes that hold them, then broadcast / quad-uniform 16-byte reads -- a third
                    // of the load/store-pipe traffic the equivalent nine 64-bit shuffles would need
                    double2* cb = reinterpret_cast<double2*>(S.colbuf[kh & 1]);
                    if ((lane & 3) == kh) cb[r] = make_double2(x0, x1);
                    __syncwarp();
                    const double pv = cb[k].x;                                               // a[k][k]
                    const double2 bc = cb[k + 1];                                            // a[k+1][k], a[k+1][k+1]
                    const double2 ai = cb[r], aj0 = cb[c2], aj1 = cb[c2 + 1];
                    const double bv = bc.x, cv = bc.y;
                    const double ai0 = ai.x, ai1 = ai.y;                                     // a[r][k], a[r][k+1]
                    const double aj00 = aj0.x, aj01 = aj0.y;                                 // a[2c][k], a[2c][k+1]
                    const double aj10 = aj1.x, aj11 = aj1.y;                                 // a[2c+1][k], a[2c+1][k+1]
                    // ---- stage k -> k + 1: pivot p_k, exact scale s1 = 2^-(exponent of p_k)
                    badk = (!(pv > 0.0) && badk < 0) ? k : badk;
                    const double s1 = __hiloint2double((2046 - ((__double2hiint(pv) >> 20) & 0x7ff)) << 20, 0);
                    const double ps = pv * s1;
                    const double p1 = fma(ps, cv, -((bv * bv) * s1));                       // a'[k+1][k+1]
                    const double ui = fma(ps, ai1, -((ai0 * bv) * s1));                     // a'[r][k+1]
                    const double uj0 = fma(ps, aj01, -((aj00 * bv) * s1));                  // a'[2c][k+1]
                    const double uj1 = fma(ps, aj11, -((aj10 * bv) * s1));                  // a'[2c+1][k+1]
                    const double y0 = fma(ps, x0, -((ai0 * aj00) * s1));                    // a'[r][2c]
                    const double y1 = fma(ps, x1, -((ai0 * aj10) * s1));                    // a'[r][2c+1]
                    // ---- stage k + 1 -> k + 2: pivot p'_{k+1}
                    badk = (!(p1 > 0.0) && badk < 0) ? k + 1 : badk;
                    const double s2 = __hiloint2double((2046 - ((__double2hiint(p1) >> 20) & 0x7ff)) << 20, 0);
                    const double p1s = p1 * s2;
                    const double z0 = fma(p1s, y0, -((ui * uj0) * s2));
                    const double z1 = fma(p1s, y1, -((ui * uj1) * s2));
                    // reciprocal-square-root arguments and scales of the two pivots (lane l keeps pivot l % 8)
                    const double cs1 = cs * ps;
                    const int own = lane & 7;
                    mine = own == k ? pv * cs : own == k + 1 ? p1 * cs1 : mine;
                    myc = own == k ? cs : own == k + 1 ? cs1 : myc;
                    cs = cs1 * p1s;
                    // own entries: both steps below / right of the pair, the first step only in column k + 1
                    x0 = (r > k + 1 && c2 > k + 1) ? z0 : x0;
                    x1 = (r > k + 1 && c2 + 1 > k + 1) ? z1 : ((c2 == k && r > k) ? y1 : x1);
                }
                const double q = rsqrt(mine);                  // lane l: 1 / sqrt(p_k c_k) of pivot k = l % 8
                const double rk = myc * q;                     // 1 / L_kk
                x0 *= __shfl_sync(0xffffffffu, q, c2);
                x1 *= __shfl_sync(0xffffffffu, q, c2 + 1);
                GSE_PC(2);
                // publish the factor of the block (packed lower triangle, reciprocal pivots) for the row solves
                // and put it in its place in the panel (zeros above the diagonal)
                if (c2 <= r) sl[r * (r + 1) / 2 + c2] = x0;
                if (c2 + 1 <= r) sl[r * (r + 1) / 2 + c2 + 1] = x1;
                *dptr = make_double2(c2 <= r ? x0 : 0.0, c2 + 1 <= r ? x1 : 0.0);
                if (lane < 8) { sl[36 + lane] = rk; s_rinv[kb + lane] = rk; }      // (padded pivots: reciprocal 1)
                if (lane == 0 && badk >= 0 && kb + badk < p) atomicMin(err, ((unsigned long long)f << 32) | (unsigned long long)(kb + badk));
                GSE_PC(3);
            }
            // the factor of block k is published; block column k of every row below it is current
            // (left-looking share applied by the helper warps during the previous step)
            __syncthreads();
            GSE_PC(4);
            if (warp == 0) {
                // the next pivot tile (or, after the last block, the first eight update rows)
                if (lane < 8 && kb + 8 + lane < R) solve_row(kb + 8 + lane, kb, sl);
                __syncwarp();
                asm volatile("bar.arrive 1, %0;" :: "r"(nth) : "memory");
                GSE_PC(5);
            } else {
                // the bulk rows, on the helper warps only (warp 0's scheduler stays free for its tile solve)
                if (helper) for (int row = kb + 16 + wi * 32 + lane; row < R; row += nw * 32) solve_row(row, kb, sl);
                asm volatile("bar.sync 1, %0;" :: "r"(nth) : "memory");      // + warp 0's tile
                if (helper && kb + 8 < rp) {
                    // later pivot tiles: their diagonal blocks take this block column's share now (tile k + 1
                    // takes it in warp 0's registers)
                    for (int t = t0 + 2 + wi; t < (rp >> 3); t += nw) diag_rank8(pan, ld, t, kb, lane);
                    // rows below the next diagonal tile: block column kn -= A[rows, 0:kn] * A[kn:kn+8, 0:kn]^T
                    const int kn = kb + 8;
                    for (int tb2 = t0 + 2 + wi; tb2 < ntile; tb2 += 2 * nw) {
                        const int ta = tb2, tc2 = tb2 + nw;
                        const bool two = tc2 < ntile;
                        const double* a0p = pan + (size_t)(ta * 8 + (lane >> 2)) * ld + (lane & 3);
                        const double* a1p = pan + (size_t)((two ? tc2 : ta) * 8 + (lane >> 2)) * ld + (lane & 3);
                        const double* bp = pan + (size_t)(kn + (lane >> 2)) * ld + (lane & 3);
                        double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll 2
                        for (int kk = 0; kk < kn; kk += 4) {
                            const double b = bp[kk];
                            dmma_m8n8k4(c00, c01, a0p[kk], b);
                            dmma_m8n8k4(c10, c11, a1p[kk], b);
                        }
                        double* o0 = pan + (size_t)(ta * 8 + (lane >> 2)) * ld + kn + 2 * (lane & 3);
                        o0[0] -= c00; o0[1] -= c01;
                        if (two) {
                            double* o1 = pan + (size_t)(tc2 * 8 + (lane >> 2)) * ld + kn + 2 * (lane & 3);
                            o1[0] -= c10; o1[1] -= c11;
                        }
                    }
                }
            }
        }
        __syncthreads();
        GSE_PC(6);
#undef GSE_PC
        if (tb && tid == 0) for (int k = 0; k < 7; ++k) tb[8 + k] = pc[k];
    }
    const bool bulk_panel = HAS_PIVOTS && pp && diag && (p & 1) == 0;
    GSE_TICK(4);

    // ---- update tasks: the front's finished panels come back from the factor storage -----------
    if (HAS_PIVOTS && kind == 2) {
        wait.panels(hdr);
        const double* L = lbuf + hdr.l_off;
        const int nrow = ni + (diag ? 0 : nj);
        // one warp per row, six rows (twelve independent loads per lane) in flight
        for (int rb = warp; rb < nrow; rb += 6 * nwarps) {
            double v[6][2];
#pragma unroll
            for (int g = 0; g < 6; ++g) {
                const int r = rb + g * nwarps;
                const double* src = L + (size_t)(p + (r < ni ? i0 + r : j0 + r - ni)) * p;
#pragma unroll
                for (int h = 0; h < 2; ++h) v[g][h] = (r < nrow && lane + 32 * h < p) ? ldc(src + lane + 32 * h) : 0.0;
            }
#pragma unroll
            for (int g = 0; g < 6; ++g) {
                const int r = rb + g * nwarps;
                double* dst = pan + (size_t)(r < ni ? r : ri + r - ni) * ld;
#pragma unroll
                for (int h = 0; h < 2; ++h) if (r < nrow && lane + 32 * h < p) dst[lane + 32 * h] = v[g][h];
            }
        }
        __syncthreads();
    }

    // ---- trailing update on the FP64 tensor pipe: U_IJ = F_IJ - L_I L_J^T -------------------
    const double* Pi = pan + (size_t)rp * ld;
    if (!no_tile) {
        const double* Pj = diag ? Pi : pan + (size_t)(rp + ri) * ld;
        const int nbi = round8(ni) >> 3, nbj = round8(nj) >> 3;
        const int kend = (p + 3) & ~3;
        double* U = (((hdr.flags & 4) && ft.ubuf_root) ? ft.ubuf_root : ubuf) + hdr.u_off;     // (area root of a non-coordinator rank: the coordinator's buffer)
        const double* Uc = direct ? ubuf + crec[0].u_off : nullptr;   // chain: F_IJ lives in the child's U
        // one warp per (8-row block, group of GW 8-wide column blocks); GW = 4 reuses every A fragment four times,
        // GW = 2 is taken when four-wide groups would leave warps idle (a 32 x 32 tile is four groups of four but
        // eight groups of two: half the MMA chain per warp on the critical path of a latency-bound front)
        auto update_groups = [&](auto gw_tag) {
            constexpr int GW = decltype(gw_tag)::value;
            const int ngj = (nbj + GW - 1) / GW;
            for (int w = warp; w < nbi * ngj; w += nwarps) {
                const int bi = w / ngj, gj = w % ngj;
                if (diag && gj * GW > bi) continue;
                const int row = bi * 8 + (lane >> 2);
                const int I = i0 + row;
                double fv[2 * GW];
#pragma unroll
                for (int q = 0; q < 2 * GW; ++q) fv[q] = 0.0;
                if (direct && row < ni) {
                    const double* crow = Uc + (size_t)(p + I) * (p + I + 1) / 2 + p;
#pragma unroll
                    for (int q = 0; q < GW; ++q) {
                        const int col = (gj * GW + q) * 8 + 2 * (lane & 3), J = j0 + col;
                        if (col < nj && J <= I) fv[2 * q] = ldc(crow + J);
                        if (col + 1 < nj && J + 1 <= I) fv[2 * q + 1] = ldc(crow + J + 1);
                    }
                }
                double c[2 * GW];
#pragma unroll
                for (int q = 0; q < 2 * GW; ++q) c[q] = 0.0;
                if (p) {
                    const double* ap = Pi + (size_t)(bi * 8 + (lane >> 2)) * ld + (lane & 3);
                    const double* bp[GW];
#pragma unroll
                    for (int q = 0; q < GW; ++q) {
                        const int bj = min(gj * GW + q, nbj - 1);
                        bp[q] = Pj + (size_t)(bj * 8 + (lane >> 2)) * ld + (lane & 3);
                    }
#pragma unroll 2
                    for (int kk = 0; kk < kend; kk += 4) {
                        const double a = ap[kk];
#pragma unroll
                        for (int q = 0; q < GW; ++q) dmma_m8n8k4(c[2 * q], c[2 * q + 1], a, bp[q][kk]);
                    }
                }
                if (row < ni) {
                    double* urow = U + (size_t)I * (I + 1) / 2;
#pragma unroll
                    for (int q = 0; q < GW; ++q) {
                        const int bj = gj * GW + q;
                        if (bj >= nbj) break;
                        const int col = bj * 8 + 2 * (lane & 3), J = j0 + col;
                        if (col < nj && J <= I) urow[J] = (direct ? fv[2 * q] : tile[row * ldt + col]) - c[2 * q];
                        if (col + 1 < nj && J + 1 <= I) urow[J + 1] = (direct ? fv[2 * q + 1] : tile[row * ldt + col + 1]) - c[2 * q + 1];
                    }
                }
            }
        };
        if (GSE_UPDATE_NARROW && nbi * ((nbj + 3) >> 2) < nwarps) update_groups(std::integral_constant<int, 2>{});
        else update_groups(std::integral_constant<int, 4>{});
    }
    GSE_TICK(5);
    {
        // ---- factor panel to global (diagonal tasks own their row chunk): one TMA bulk store per row.  Nothing ahead of
        // this front in the forward pass reads the factor -- only its own back-substitution does -- while the parent waits
        // for the update matrix: a fused task therefore reports its tile FIRST (wait.tile_done: the dataflow kernel's
        // hand-off to the parent) and stores its slice of the factor afterwards.  Starting the ~90 bulk stores of a
        // first-chunk task costs ~1 us, which used to sit on the critical path of every level: the diagonal tasks were
        // the last of their front to finish.
        if (HAS_PIVOTS && pp && diag) {
            if (kind == 0) wait.tile_done(hdr);
            double* L = lbuf + hdr.l_off;
            if (bulk_panel) {
                fence_proxy_async();            // the rows were written with ordinary shared-memory stores
                __syncthreads();
                const int n0 = ci == 0 ? p : 0;                       // pivot rows (first chunk only), then the rows of chunk I
                if (tid < n0 + ni) {
                    const int r = tid < n0 ? tid : tid - n0;
                    const double* src = tid < n0 ? pan + (size_t)r * ld : pan + (size_t)(rp + r) * ld;
                    double* dst = tid < n0 ? L + (size_t)r * p : L + (size_t)(p + i0 + r) * p;
                    tma_store_1d(dst, src, (unsigned)(p * sizeof(double)));
                    tma_store_commit();
                }
            }
            if (ci == 0 && tid < p) dinv[hdr.dinv_off + tid] = s_rinv[tid];
            if (bulk_panel) {
                tma_store_wait_all();            // (threads without a pending group return at once)
            } else {                            // odd pivot count: rows are not 16-byte multiples
                if (ci == 0)
                    for (int r = warp; r < p; r += nwarps)
                        for (int k = lane; k < p; k += 32) L[(size_t)r * p + k] = pan[r * ld + k];
                double* Li = L + (size_t)(p + i0) * p;
                for (int r = warp; r < ni; r += nwarps)
                    for (int k = lane; k < p; k += 32) Li[(size_t)r * p + k] = Pi[r * ld + k];
            }
        }
        GSE_TICK(6);
    }
#undef GSE_TICK
}

// ---------------------------------------------------------------------------------------------
// Backward substitution: x_P = L11^{-T} (y_P - L21^T x_U).  The L21^T x_U product of a front is
// split over several CTAs (fixed row ranges, all loads issued up front); the last CTA to finish
// adds the partial sums in split order (deterministic) and runs the triangular solve in one warp.
// Restates backward / interior_recover (reference linalg.py:366-383,427-434) and dpotrs.
// ---------------------------------------------------------------------------------------------
constexpr int kBwdRows = 64;   // update rows per split

struct __align__(16) BwdScratch {
    double l11[64 * 64];       // flat copy of the p x p pivot block (row stride p)
    double half[2][64];
    double xs[kBwdRows];
    double tv[64];
    int last;
};

// One backward task, executed by the first 128 threads of the CTA (all threads must call it).
// Returns true in the CTA that solved the front's pivots (the last split to finish).
// wait.factor() precedes the first read of the front's own factor, wait.parent() the first read of
// the solution of its ancestors: everything that only needs the factor (the pivot block, this
// split's slice of L21, the row indices) is fetched BEFORE waiting for the parent.
template <class Wait>
__device__ __forceinline__ bool backward_body(BwdScratch& B, const BwdTask& tk, const FrontTab& ft, const double* lbuf,
                                              double* xsol, double* bpart, int32_t* bcnt, const Wait& wait) {
    double* l11 = B.l11;
    double (*half)[64] = B.half;
    double* xs = B.xs;
    double* tv = B.tv;
    int& s_last = B.last;
    const int f = tk.front;
    const int p = tk.p, u = tk.u;
    const double* L = lbuf + tk.l_off;
    const int32_t* rows = ft.rows + tk.rows_off;
    const int tid = threadIdx.x, k = tid & 63, h = tid >> 6;
    const int lo = tk.split * kBwdRows, n = min(kBwdRows, u - lo);
    wait.factor(tk);
    // L11 is needed only by the CTA that finishes last; every CTA prefetches it asynchronously so
    // the copy overlaps the matrix-vector part instead of following the atomic hand-off
    // (l_off is even, so 16-byte cp.async.cg -- L2-coherent -- covers the block pairwise)
    if (tid < 128) {
        for (int t = 2 * tid; t + 1 < p * p; t += 256) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(&l11[t]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(L + t));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        if ((p & 1) && tid == 0) l11[p * p - 1] = ldc(L + p * p - 1);
    }
    const double yk = (tid < p) ? ldc(L + (size_t)(p + u) * p + tid) : 0.0;
    // what the triangular solve of the last CTA needs besides L11 -- reciprocal pivots, the pivots' positions in
    // the solution vector -- is fetched here as well: nothing but the parent's x is loaded after the hand-off
    const double* di = ft.dinv + tk.dinv_off;
    const double r0 = (tid < 32 && tid < p) ? ldc(di + tid) : 0.0, r1 = (tid < 32 && tid + 32 < p) ? ldc(di + tid + 32) : 0.0;
    const int prow0 = (tid < 32 && tid < p) ? rows[tid] : -1, prow1 = (tid < 32 && tid + 32 < p) ? rows[tid + 32] : -1;
    const int xrow = (tid < kBwdRows && tid < n) ? rows[p + lo + tid] : -1;
    const int a = (h & 1) * (kBwdRows / 2), b = min(n, a + kBwdRows / 2);
    double v[kBwdRows / 2];
    {
        const double* col = L + (size_t)(p + lo) * p + k;
#pragma unroll
        for (int i = 0; i < kBwdRows / 2; ++i) v[i] = (k < p && tid < 128 && a + i < b) ? ldc(col + (size_t)(a + i) * p) : 0.0;
    }
    // Early splits (dataflow kernel): the later splits of a front only read entries of ancestors above the nearest
    // one, so they wait for front dep2 and finish a level ahead; split 0 -- the only one on the chain -- combines.
    const bool early = Wait::kEarlySplits && tk.early != 0;
    if (wait.poll_x()) {
        // every thread polls the solution entry it reads (armed by the forward pass, see x_unset)
        if (tid < kBwdRows) xs[tid] = xrow >= 0 ? wait.load_x(xsol + xrow) : 0.0;
    } else {
        if (early && tk.split > 0) wait.ancestor(tk); else wait.parent(tk);
        if (tid < kBwdRows) xs[tid] = xrow >= 0 ? ldc(xsol + xrow) : 0.0;
    }
    __syncthreads();
    {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (k < p && tid < 128) {
#pragma unroll
            for (int i = 0; i < kBwdRows / 2; i += 4) {
                s0 = fma(v[i], xs[min(a + i, kBwdRows - 1)], s0);
                s1 = fma(v[i + 1], xs[min(a + i + 1, kBwdRows - 1)], s1);
                s2 = fma(v[i + 2], xs[min(a + i + 2, kBwdRows - 1)], s2);
                s3 = fma(v[i + 3], xs[min(a + i + 3, kBwdRows - 1)], s3);
            }
        }
        if (tid < 128) half[h][k] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    if (early) {
        if (tk.split > 0) {
            if (tid < 64) bpart[(size_t)(tk.pbase + tk.split) * 64 + tid] = half[0][tid] + half[1][tid];
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(&bcnt[f], 1);
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
            return false;
        }
        wait.splits(bcnt + f, tk.nsplit - 1);      // (long done when this split is released: they ran a level ahead)
    } else if (tk.nsplit > 1) {
        if (tid < 64) bpart[(size_t)(tk.pbase + tk.split) * 64 + tid] = half[0][tid] + half[1][tid];
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&bcnt[f], 1) == tk.nsplit - 1;
        __syncthreads();
        if (!s_last) { asm volatile("cp.async.wait_group 0;\n" ::); __syncthreads(); return false; }
        __threadfence();
    }
    // ---- last CTA of the front: combine (split order), then solve L11^T x = t in warp 0 ------
    if (tid < 64) {
        double acc = 0.0;
        if (tk.nsplit == 1) {
            // a single split (at most 64 update rows, most fronts): the partial sum never leaves the CTA
            // (0.0 + s, the same sum the general path forms after its round trip through global memory)
            acc = tid < p ? yk - (0.0 + (half[0][tid] + half[1][tid])) : 0.0;
        } else if (early) {
            // split 0 combines: its own partial from shared memory, the others' in split order (the same sum)
            if (tid < p) {
                const volatile double* bp = bpart + (size_t)tk.pbase * 64 + tid;
                acc = 0.0 + (half[0][tid] + half[1][tid]);
                for (int s = 1; s < tk.nsplit; ++s) acc += bp[(size_t)s * 64];
                acc = yk - acc;
            }
        } else if (tid < p) {
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
        // the lanes carry s_i = t_i / L_ii, so the serial chain per pivot is one shuffle and one FMA:
        // x_c = s_c, then s_i -= (L_ci / L_ii) x_c with the scaled factor entry formed off the chain
        t0 *= r0; t1 *= r1;
        // Two pivots per round: x_c, the not yet reduced s_{c-1} and the factor entry between the two come by three
        // independent shuffles, every lane forms x_{c-1} itself, and both updates follow -- the same operations in the same
        // order as one pivot per round (bit for bit), with one shuffle latency per PAIR on the chain.
#pragma unroll 2
        for (int c = p - 1; c >= 1; c -= 2) {
            const double la0 = tid < c ? l11[c * p + tid] * r0 : 0.0;
            const double la1 = tid + 32 < c ? l11[c * p + tid + 32] * r1 : 0.0;
            const double lb0 = tid < c - 1 ? l11[(c - 1) * p + tid] * r0 : 0.0;
            const double lb1 = tid + 32 < c - 1 ? l11[(c - 1) * p + tid + 32] * r1 : 0.0;
            const double xc = __shfl_sync(0xffffffffu, c < 32 ? t0 : t1, c & 31);
            const double sm1 = __shfl_sync(0xffffffffu, c - 1 < 32 ? t0 : t1, (c - 1) & 31);
            const double lcc = __shfl_sync(0xffffffffu, c - 1 < 32 ? la0 : la1, (c - 1) & 31);
            const double xm1 = fma(-lcc, xc, sm1);
            t0 = fma(-lb0, xm1, fma(-la0, xc, t0));
            t1 = fma(-lb1, xm1, fma(-la1, xc, t1));
        }
        // (a NaN leaves as the canonical one: the armed pattern of x_unset never comes out of a solve)
        if (prow0 >= 0) xsol[prow0] = t0 == t0 ? t0 : __longlong_as_double(0x7ff8000000000000LL);
        if (prow1 >= 0) xsol[prow1] = t1 == t1 ? t1 : __longlong_as_double(0x7ff8000000000000LL);
    }
    __syncthreads();
    return true;
}

}  // namespace gse
