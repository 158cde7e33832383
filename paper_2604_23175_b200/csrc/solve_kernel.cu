// solve_kernel.cu -- the whole multi-area Gauss-Newton solve as ONE persistent kernel.
//
// solve_multiarea's loop (reference solver.py:275-338) -- template evaluation, fused accumulation,
// per-area Schur-mode factorisation, boundary assembly + factorisation, back-substitution, state
// update, convergence test -- and the final objective (solver.py:100-103) run inside a single
// cooperative launch.  One CTA slot per SM-resident block; CTAs pull work items from a global
// counter in topological order
//     [eval blocks | accumulate blocks | front tasks (level order) | backward tasks | update blocks]
// (latency-bound plans have no update blocks: the state update and the norm of a front's pivots ride
// on its backward task) and spin on per-front completion counters instead of waiting for a kernel boundary: a front
// starts the moment its own children are done, areas progress independently, and nothing returns
// to the host until the loop has converged (the host then reads iterations, the per-iteration
// norms, the failure code and J in one copy).
//
// Deadlock freedom: an item only waits on items with a smaller index; indices are handed out in
// increasing order and every CTA of the (cooperative) grid is resident, so the smallest unfinished
// item is always held by a running CTA whose dependencies are complete.
// Determinism: no floating-point atomics; every reduction order is fixed by the program, so the
// result is bit-identical to the level-launch path whatever the CTA interleaving.
#include "front_body.cuh"

#ifndef GSE_POLL_NS
#define GSE_POLL_NS 40
#endif
#ifndef GSE_XPOLL_NS
#define GSE_XPOLL_NS 40     // back-substitution: interval between two looks at an armed solution entry
#endif

namespace gse {

namespace {

// Release fence of a hand-off (writes -> fence -> counter bump, observed with ld.acquire): acq_rel is all the
// pattern needs; __threadfence() is the sequentially consistent fence (MEMBAR.SC.GPU), which costs more.
__device__ __forceinline__ void fence_release() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Spin until *p >= target.  Called by ONE thread per dependency (the rest of the CTA parks on a
// barrier, which costs no issue slots); the back-off keeps a waiting CTA from stealing load/store
// bandwidth from the CTA it shares the SM with -- often the very producer it is waiting for.
// Debug record of a wait that ran into the watchdog: [cta][4] = {counter address, target, value seen, 1} in
// host-mapped memory (it outlives the aborted context); armed by gse_debug_watchdog, nullptr otherwise.
__device__ unsigned long long* g_stuck = nullptr;
__device__ unsigned long long g_watchdog_ns = 10000000000ull;
// sys: the counter is bumped by another GPU over peer memory (peer-linked multi-rank solve).
__device__ __forceinline__ void wait_ge(const unsigned* p, unsigned target, bool sys = false) {
    unsigned polls = 0;
    unsigned long long t0 = 0;
    unsigned v;
    while ((v = (sys ? ld_acquire_sys(p) : ld_acquire(p))) < target) {
        __nanosleep(GSE_POLL_NS);
        // watchdog: a dependency that never completes would hang the device; after ~10 s of waiting
        // the kernel aborts instead (the launch then fails with an error the host reports)
        if ((++polls & 0xffffu) == 0) {
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(now));
            if (t0 == 0) t0 = now;
            else if (now - t0 > g_watchdog_ns) {
                if (g_stuck) {
                    unsigned long long* d = g_stuck + 4 * (size_t)((blockIdx.x + 97u * gridDim.x) & 1023u);   // (rank plans sharing a device differ in grid size)
                    d[0] = (unsigned long long)(size_t)p; d[1] = target; d[2] = v; d[3] = 1ull;
                    __threadfence_system();
                    if (now - t0 < 2 * g_watchdog_ns) continue;      // let the other waiters leave their records too
                }
                __trap();
            }
        }
    }
}
// called by one thread after a CTA barrier that follows the item's last global write
__device__ __forceinline__ void signal(unsigned* p) {
    fence_release();
    atomicAdd(p, 1u);
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

struct SpinWait {
    const unsigned* ctr;
    unsigned epoch;          // iteration + 1
    unsigned acc_target;
    unsigned long long* tr;  // trace slots of this item (debug) or nullptr
    int n_fronts, front0;
    bool sys;                // peer-linked solve: child counters may be bumped by other GPUs
    unsigned gamma_need;     // non-coordinator ranks: pieces of delta_x_Gamma to wait for (0: none)
    bool early_tile = false; // latency-bound plans: fused diagonal tasks report their tile before they store the factor
    bool poll = false;       // back-substitution: the solution entries are the hand-off (x_unset, front_body.cuh)
    __device__ __forceinline__ bool poll_x() const { return poll; }
    __device__ __forceinline__ double load_x(const double* p) const {
        unsigned polls = 0;
        unsigned long long t0 = 0;
        double v;
        while (x_is_unset(v = __ldcg(p))) {
            __nanosleep(GSE_XPOLL_NS);
            if ((++polls & 0xffffu) == 0) {          // watchdog, as in wait_ge
                const unsigned long long now = globaltimer();
                if (t0 == 0) t0 = now;
                else if (now - t0 > g_watchdog_ns) __trap();
            }
        }
        if (tr && threadIdx.x == 0) tr[2] = globaltimer();
        return v;
    }
    // early splits of the back-substitution (front_body.cuh): later splits wait for front dep2; split 0 for the others
    static constexpr bool kEarlySplits = true;
    __device__ __forceinline__ void ancestor(const BwdTask& tk) const {
        if (threadIdx.x == 0) { wait_ge(ctr + front0 + 2 * n_fronts + tk.dep2, epoch); if (tr) tr[2] = globaltimer(); }
        __syncthreads();
    }
    __device__ __forceinline__ void splits(const int32_t* cnt, int need) const {
        if (threadIdx.x == 0) wait_ge(reinterpret_cast<const unsigned*>(cnt), (unsigned)need);
        __syncthreads();
    }
    // completion counter of a child: its front's, or -- root of an area another rank owns -- the area's
    __device__ __forceinline__ const unsigned* child_ctr(int cf) const { return cf >= 0 ? ctr + front0 + cf : ctr + CTR_AREA0 + (-cf - 1); }
    // backward tasks: own factor complete (all its panel-storing tasks), then the nearest ancestor solved
    __device__ __forceinline__ void factor(const BwdTask& tk) const {
        if (threadIdx.x == 0) wait_ge(ctr + front0 + n_fronts + tk.front, (unsigned)tk.need * epoch);
        __syncthreads();
    }
    __device__ __forceinline__ void parent(const BwdTask& tk) const {
        if (tk.dep < 0) {
            // no ancestor with pivots on this rank: on a non-coordinator rank the boundary values come from the
            // coordinator's back-substitution tasks, piece by piece, over peer memory
            if (gamma_need) {
                if (threadIdx.x == 0) { wait_ge(ctr + CTR_GAMMA, gamma_need * epoch, true); if (tr) tr[2] = globaltimer(); }
                __syncthreads();
            }
            return;
        }
        if (threadIdx.x == 0) { wait_ge(ctr + front0 + 2 * n_fronts + tk.dep, epoch); if (tr) tr[2] = globaltimer(); }
        __syncthreads();
    }
    __device__ __forceinline__ void originals(const TaskRec& hdr) const {
        if (!(hdr.flags & 2)) return;
        if (threadIdx.x == 0) { wait_ge(ctr + CTR_ACC, acc_target); if (tr) tr[1] = globaltimer(); }
        __syncthreads();
    }
    // a fused diagonal task has stored its tile of the update matrix: the parent may go on while the task stores its
    // slice of the factor (counted again, under pdone, when the task ends)
    __device__ __forceinline__ void tile_done(const TaskRec& hdr) const {
        if (!early_tile) return;      // (throughput-bound plans: one hand-off per task -- a second fence costs more CTA time than the parent gains)
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_release();
            atomicAdd(const_cast<unsigned*>(ctr) + front0 + hdr.front, 1u);
            if (tr) tr[30] = globaltimer();
        }
    }
    __device__ __forceinline__ void panels(const TaskRec& hdr) const {
        if (threadIdx.x == 0) {
            wait_ge(ctr + front0 + n_fronts + hdr.front, (unsigned)hdr.nch * epoch);
            if (tr) tr[5] = globaltimer();
        }
        __syncthreads();
    }
    __device__ __forceinline__ void children(const TaskRec& hdr, const ChildRec* cr) const {
        for (int c = threadIdx.x; c < hdr.nchild; c += blockDim.x) {
            wait_ge(child_ctr(cr[c].front), (unsigned)cr[c].need * epoch, sys);
            if (tr) atomicMax(tr + 2, globaltimer());
        }
        __syncthreads();
    }
    // Blocks until child c of the batch is complete, then counts how many of the following children
    // of the batch are complete as well (without waiting for them).  cr = records of the batch.
    __device__ __forceinline__ int ready_children(const TaskRec&, const ChildRec* cr, int c, int nb, int* s_n) const {
        if (threadIdx.x == 0) {
            wait_ge(child_ctr(cr[c].front), (unsigned)cr[c].need * epoch, sys);
            int n = 1;
            while (c + n < nb && (sys ? ld_acquire_sys(child_ctr(cr[c + n].front)) : ld_acquire(child_ctr(cr[c + n].front)))
                                     >= (unsigned)cr[c + n].need * epoch) ++n;
            *s_n = n;
            if (tr) tr[2] = globaltimer();
        }
        __syncthreads();
        const int n = *s_n;
        __syncthreads();
        return n;
    }
};

}  // namespace

// LINKED: the peer-linked multi-rank variant (exchanges over peer memory, sp.lk).  A separate instantiation: the
// single-rank kernel runs at the 128-register cap of two CTAs per SM and must not carry the other's live values.
template <bool LINKED>
__device__ __forceinline__ void gn_solve_body(const SolveProg& sp, const EvalProg& ep, const FrontTab& ft, double* va, double* vm) {
    extern __shared__ __align__(16) double sm[];
    __shared__ FrontScratch S;
    __shared__ int s_item, s_stop;
    __shared__ unsigned long long s_red[kSolveThreads / 32];
    __shared__ __align__(8) unsigned long long s_bar;      // mbarrier of the TMA bulk copies (accumulation items)
    const int tid = threadIdx.x;
    unsigned bar_parity = 0;
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
    unsigned* ctr = sp.ctr;
    unsigned* fdone = ctr + sp.front0;
    unsigned* pdone = fdone + sp.n_fronts;
    unsigned* bdone = pdone + sp.n_fronts;
    const int o_acc = sp.n_eval_items, o_front = o_acc + sp.n_acc_items, o_bwd = o_front + sp.n_tasks,
              o_upd = o_bwd + sp.n_btasks;
    const bool fused_update = sp.n_upd_items == 0;      // latency-bound plans: the update rides on the backward tasks
    const PeerLink& lk = sp.lk;
    constexpr bool linked = LINKED;                     // areas sharded over several GPUs, exchanges over peer memory
    const unsigned gamma_need = (linked && lk.rank != 0) ? (unsigned)lk.n_gamma_fronts : 0u;
    if (sp.stamps && blockIdx.x == 0 && tid == 0) sp.stamps[0] = globaltimer();
#define GSE_STAMP(it, k) do { if (sp.stamps) atomicMax(sp.stamps + 1 + 8 * (it) + (k), globaltimer()); } while (0)

    int known = 0;          // iterations [0, known) are complete and did not stop the loop
    int final_it = 0;       // iterations performed when the loop stopped
    int converged = 0, failed = 0;
    // Two panel factorisations on one SM slow each other by a quarter (shared FP64 port and shared-memory pipes: panel
    // 8.4 -> 10.5-12.5 us, tools/persist_trace.py GSE_TRACE_FRONT), and on the boundary chain the slowest task of a front
    // sets the pace.  The chain ranges of the task list (SolveProg::chain_lo / chain_hi: runs of levels with at most one panel
    // task per SM) are therefore handed out to ONE CTA per SM: the second CTA of an SM does not pull while the head of
    // the queue is inside such a range.  Items are still handed out in increasing order and the first CTAs never hold back, so the
    // smallest unfinished item is always held by a running CTA, as before.
    bool second_on_sm = false;
    if (tid == 0 && sp.n_chain > 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
        second_on_sm = (atomicAdd(ctr + CTR_SM0 + (smid & 511u), 1u) & 1u) != 0u;
    }
    for (;;) {
        if (tid == 0) {
            if (second_on_sm) {
                // (bounded patience: a head that has not moved for ~60 us means the others have left the loop -- the
                // solve has stopped -- or hold everything they can; pull then, like any CTA)
                unsigned last = ~0u, still = 0;
                for (;;) {
                    const unsigned head = *reinterpret_cast<volatile unsigned*>(ctr + CTR_NEXT);
                    const int l = (int)(head % (unsigned)sp.items_per_it);
                    const int t = l - o_front;
                    bool in_chain = false;
#pragma unroll
                    for (int k = 0; k < 4; ++k) in_chain = in_chain || (k < sp.n_chain && t >= sp.chain_lo[k] && t < sp.chain_hi[k]);
                    if (!in_chain || head / (unsigned)sp.items_per_it >= (unsigned)sp.max_it) break;
                    still = head == last ? still + 1 : 0;
                    last = head;
                    if (still > 200) break;
                    __nanosleep(300);
                }
            }
            s_item = (int)atomicAdd(ctr + CTR_NEXT, 1u);
        }
        __syncthreads();
        const int item = s_item;
        const int it = min(item / sp.items_per_it, sp.max_it);
        const int loc = item - it * sp.items_per_it;
        // ---- iteration boundaries between `known` and `it`: has the loop stopped? ---------------
        if (it > known) {
            if (tid == 0) {
                int stop = 0;
                for (int j = known + 1; j <= it && !stop; ++j) {
                    if (linked) {
                        // every rank has finished iteration j and max-merged its norm / failure code into this
                        // rank's copy: all ranks read the same values and take the same decision
                        wait_ge(ctr + CTR_ITER, (unsigned)lk.world * (unsigned)j, true);
                        const unsigned long long ge = ld_acquire64_sys(lk.gerr[lk.rank]);
                        const double gd = __longlong_as_double((long long)ld_acquire64_sys(lk.gdelta[lk.rank] + (j - 1)));
                        if (ge != 0ull) stop = 2 * 65536 + j;
                        else if (gd < sp.tol) stop = 1 * 65536 + j;
                        else if (j == sp.max_it) stop = 3 * 65536 + j;
                        continue;
                    }
                    if (fused_update) {
                        wait_ge(ctr + CTR_BWD, (unsigned)sp.n_bwd_fronts * (unsigned)j);     // every front solved, state updated
                        wait_ge(ctr + CTR_FWD, (unsigned)sp.n_tasks * (unsigned)j);
                    } else wait_ge(ctr + CTR_UPD, (unsigned)sp.n_upd_items * (unsigned)j);
                    const unsigned long long e = ld_acquire64(sp.err);
                    const double dv = __longlong_as_double((long long)ld_acquire64(sp.delta + (j - 1)));
                    if (e != ~0ull) stop = 2 * 65536 + j;
                    else if (dv < sp.tol) stop = 1 * 65536 + j;
                    else if (j == sp.max_it) stop = 3 * 65536 + j;
                }
                s_stop = stop;
            }
            __syncthreads();
            const int stop = s_stop;
            if (stop) { final_it = stop & 65535; converged = (stop >> 16) == 1; failed = (stop >> 16) == 2; break; }
            known = it;
        }
        const unsigned epoch = (unsigned)it + 1u;
        unsigned long long* tr = sp.trace ? sp.trace + 32 * (size_t)item : nullptr;
        if (tr && tid == 0) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
            tr[0] = globaltimer(); tr[4] = smid | ((unsigned long long)blockIdx.x << 32);
        }

        if (loc < o_acc) {
            // ---- template evaluation: one unit per thread ----------------------------------------
            const int u = loc * kEvalPerItem + tid;
            if (u < sp.n_units) eval_unit(ep, u, va, vm);
            __syncthreads();
            if (tid == 0) { signal(ctr + CTR_EVAL); GSE_STAMP(it, 0); }
        } else if (loc < o_front) {
            // ---- fused accumulation: one staged item (operands gathered to shared memory once) ----
            if (tid == 0) { wait_ge(ctr + CTR_EVAL, (unsigned)sp.n_eval_items * epoch); if (tr) tr[2] = globaltimer(); }
            __syncthreads();
            const AccProg ap{sp.acc_items, sp.acc_uniq, sp.acc_ptr, sp.acc_pair, sp.val, sp.gval, sp.n_acc_items};
            acc_item_staged(ap, loc - o_acc, sm, &s_bar, bar_parity, tr);
            __syncthreads();
            if (tr && tid == 0) tr[7] = globaltimer();
            if (tid == 0) { signal(ctr + CTR_ACC); GSE_STAMP(it, 1); }
        } else if (loc < o_bwd) {
            // ---- multifrontal task -----------------------------------------------------------------
            load_task_header(S, sp.tasks + (loc - o_front));
            __syncthreads();
            if (tr && tid == 0) {
                tr[6] = (unsigned long long)S.hdr.kind | ((unsigned long long)S.hdr.front << 8) | ((unsigned long long)S.hdr.ci << 32) | ((unsigned long long)S.hdr.cj << 48);
                tr[7] = (unsigned long long)S.hdr.p | ((unsigned long long)S.hdr.u1 << 16) | ((unsigned long long)S.hdr.nchild << 32) | ((unsigned long long)S.hdr.phase << 48);
            }
            const SpinWait w{ctr, epoch, (unsigned)sp.n_acc_items * epoch, tr, sp.n_fronts, sp.front0, linked, 0u, fused_update};
            if (S.hdr.p) front_task_body<1>(S, sm, ft, sp.gval, sp.lbuf, sp.ubuf, sp.err, tr ? (long long*)(tr + 8) : nullptr, w,
                                             (!linked && sp.bwd_poll) ? sp.xsol : nullptr);
            else front_task_body<0>(S, sm, ft, sp.gval, sp.lbuf, sp.ubuf, sp.err, tr ? (long long*)(tr + 8) : nullptr, w);
            __syncthreads();
            if (tid == 0 && linked && (S.hdr.flags & 4)) {
                // area root of a non-coordinator rank: its tile of (S_b | b_hat) sits in the coordinator's
                // memory; the coordinator's boundary fronts wait on THEIR counter of this front
                __threadfence_system();
                atomicAdd_system(lk.root_ctr + CTR_AREA0 + S.hdr.area, 1u);
                atomicAdd(ctr + CTR_FWD, 1u);
                GSE_STAMP(it, 1 + S.hdr.phase);
            } else if (tid == 0) {
                fence_release();
                const int kind = S.hdr.p ? S.hdr.kind : 0;
                if (kind != 2 && S.hdr.p && S.hdr.ci == S.hdr.cj) atomicAdd(pdone + S.hdr.front, 1u);
                const bool reported = fused_update && S.hdr.p && kind == 0 && S.hdr.ci == S.hdr.cj;     // (SpinWait::tile_done, before the factor stores)
                if (kind != 1 && !reported) atomicAdd(fdone + S.hdr.front, 1u);
                atomicAdd(ctr + CTR_FWD, 1u);
                GSE_STAMP(it, 1 + S.hdr.phase);
            }
        } else if (loc < o_upd) {
            // ---- backward substitution task ---------------------------------------------------------
            const BwdTask tk = sp.btasks[loc - o_bwd];
            const SpinWait w{ctr, epoch, 0u, tr, sp.n_fronts, sp.front0, linked, gamma_need, false, !linked && sp.bwd_poll != 0};
            const bool solved = backward_body(*reinterpret_cast<BwdScratch*>(sm), tk, ft, sp.lbuf, sp.xsol, sp.bpart, sp.bcnt, w);
            if (solved && linked && lk.rank == 0 && tk.phase == 3) {
                // coordinator, boundary front: this front's pivots are a piece of delta_x_Gamma -- store it into every
                // rank's solution vector (peer memory) and count the piece there (reference solver.py:318-326: the
                // broadcast of delta_x_Gamma, here tile by tile as the back-substitution produces it)
                if (tid < tk.p) {
                    const int pos = ft.rows[tk.rows_off + tid];
                    const double x = ldc(sp.xsol + pos);
                    for (int q = 1; q < lk.world; ++q) lk.xsol[q][pos] = x;
                }
                __syncthreads();
                if (tid == 0) {
                    __threadfence_system();
                    for (int q = 1; q < lk.world; ++q) atomicAdd_system(lk.ctr[q] + CTR_GAMMA, 1u);
                }
            }
            if (solved && !fused_update) {
                if (tid == 0) {
                    fence_release();
                    atomicAdd(bdone + tk.front, 1u);
                    atomicAdd(ctr + CTR_BWD, 1u);
                    GSE_STAMP(it, tk.phase == 3 ? 5 : 6);
                }
            } else if (solved) {
                // the children only need x: release them first, then fold the state update and the stacked
                // infinity norm of this front's pivots in (reference partition.py:59-62,113-116, solver.py:328-333)
                if (tid == 0) { fence_release(); atomicAdd(bdone + tk.front, 1u); }
                unsigned long long bits = 0ull;
                if (tid < tk.p) {
                    const int pos = ft.rows[tk.rows_off + tid];
                    const int bq = sp.pos_bq[pos];
                    if (bq >= 0) {
                        const double dx = ldc(sp.xsol + pos);
                        double* dst = ((bq & 1) ? vm : va) + (bq >> 1);
                        *dst = ldc(dst) + dx;
                        bits = (unsigned long long)__double_as_longlong(fabs(dx));
                    }
                }
                if (tid < 64) {
                    for (int o = 16; o > 0; o >>= 1) { const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o); bits = other > bits ? other : bits; }
                    if ((tid & 31) == 0) s_red[tid >> 5] = bits;
                }
                __syncthreads();
                if (tid == 0) {
                    bits = s_red[1] > bits ? s_red[1] : bits;
                    if (bits) atomicMax(sp.delta + it, bits);
                    fence_release();
                    atomicAdd(ctr + CTR_BWD, 1u);
                    GSE_STAMP(it, tk.phase == 3 ? 5 : 6);
                    GSE_STAMP(it, 7);
                }
            }
        } else {
            // ---- state update + stacked infinity norm (throughput-bound plans: separate items) --------
            if (tid == 0) {
                wait_ge(ctr + CTR_BWD, (unsigned)sp.n_bwd_fronts * epoch);
                wait_ge(ctr + CTR_FWD, (unsigned)sp.n_tasks * epoch);
                if (gamma_need) wait_ge(ctr + CTR_GAMMA, gamma_need * epoch, true);     // this rank's replica of x_Gamma is updated here too
                if (tr) tr[2] = globaltimer();
            }
            __syncthreads();
            unsigned long long bits = 0ull;
#pragma unroll
            for (int k = 0; k < kUpdPerItem / kSolveThreads; ++k) {
                const int v = (loc - o_upd) * kUpdPerItem + k * kSolveThreads + tid;
                if (v < sp.n_upd) {
                    const unsigned long long b = update_var(sp.upd_bus, sp.upd_quant, sp.upd_pos, v, sp.xsol, va, vm);
                    bits = b > bits ? b : bits;
                }
            }
            for (int o = 16; o > 0; o >>= 1) { const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o); bits = other > bits ? other : bits; }
            if ((tid & 31) == 0) s_red[tid >> 5] = bits;
            __syncthreads();
            if (tid == 0) {
                for (int k = 1; k < kSolveThreads / 32; ++k) bits = s_red[k] > bits ? s_red[k] : bits;
                if (bits) atomicMax(sp.delta + it, bits);
                fence_release();
                const unsigned before = atomicAdd(ctr + CTR_UPD, 1u);
                if (linked && before + 1u == (unsigned)sp.n_upd_items * epoch) {
                    // last update item of this rank's iteration: max-merge the rank's norm and failure code into every
                    // rank's copy, then count this rank as done there (the convergence scalar of solver.py:328-338;
                    // one 8-byte atomic per peer instead of a collective)
                    fence_release();
                    const unsigned long long d = ld_acquire64(sp.delta + it), e = ld_acquire64(sp.err);
                    for (int q = 0; q < lk.world; ++q) {
                        if (d) atomicMax_system(lk.gdelta[q] + it, d);
                        if (e != ~0ull) atomicMax_system(lk.gerr[q], ~e);
                    }
                    __threadfence_system();
                    for (int q = 0; q < lk.world; ++q) atomicAdd_system(lk.ctr[q] + CTR_ITER, 1u);
                }
                GSE_STAMP(it, 7);
            }
        }
        if (tr && tid == 0) tr[3] = globaltimer();
        __syncthreads();   // s_item / scratch are reused by the next item
    }
#undef GSE_STAMP

    if (blockIdx.x == 0 && tid == 0) {
        sp.result[0] = final_it; sp.result[1] = converged;
        *sp.err_out = linked ? ~ld_acquire64_sys(lk.gerr[lk.rank]) : ld_acquire64(sp.err);
    }
    // (peer-linked ranks hold only their own interiors: J is evaluated by the host layer on the merged state)
    if (failed || linked) return;

    // ---- objective J(x) at the final state: per-block partials, last CTA adds them in block order ----
    double* red = sm;
    const int nblk = (sp.n_rows + kSolveThreads - 1) / kSolveThreads;
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        const int r = b * kSolveThreads + tid;
        red[tid] = r < sp.n_rows ? objective_row(ep, sp.m_type, sp.m_target, sp.br_from, sp.br_to, r, va, vm) : 0.0;
        __syncthreads();
        for (int o = kSolveThreads / 2; o > 0; o >>= 1) {
            if (tid < o) red[tid] += red[tid + o];
            __syncthreads();
        }
        if (tid == 0) sp.obj_partial[b] = red[0];
        __syncthreads();
    }
    if (tid == 0) { __threadfence(); s_item = atomicAdd(ctr + CTR_OBJ, 1u) == gridDim.x - 1; }
    __syncthreads();
    if (!s_item) return;
    __threadfence();
    double s = 0.0;
    for (int i = tid; i < nblk; i += kSolveThreads) s += ldc(sp.obj_partial + i);
    red[tid] = s;
    __syncthreads();
    for (int o = kSolveThreads / 2; o > 0; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        __syncthreads();
    }
    if (tid == 0) *sp.obj_out = red[0];
}

cudaError_t solve_kernel_debug_watchdog(unsigned long long* host_mapped, unsigned long long ns) {
    cudaError_t e = cudaMemcpyToSymbol(g_stuck, &host_mapped, sizeof host_mapped);
    return e == cudaSuccess ? cudaMemcpyToSymbol(g_watchdog_ns, &ns, sizeof ns) : e;
}

__global__ void __launch_bounds__(kSolveThreads, 2)
gn_solve_kernel(SolveProg sp, EvalProg ep, FrontTab ft, double* va, double* vm) { gn_solve_body<false>(sp, ep, ft, va, vm); }
__global__ void __launch_bounds__(kSolveThreads, 2)
gn_solve_linked_kernel(SolveProg sp, EvalProg ep, FrontTab ft, double* va, double* vm) { gn_solve_body<true>(sp, ep, ft, va, vm); }

size_t solve_kernel_static_smem() {
    cudaFuncAttributes a{};
    if (cudaFuncGetAttributes(&a, gn_solve_kernel) != cudaSuccess) return 0;
    return a.sharedSizeBytes;
}

int solve_kernel_max_ctas(size_t dyn_smem, int device) {
    if (cudaFuncSetAttribute(gn_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem) != cudaSuccess) return 0;
    if (cudaFuncSetAttribute(gn_solve_linked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem) != cudaSuccess) return 0;
    int per_sm = 0, sms = 0, per_sm_l = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gn_solve_kernel, kSolveThreads, dyn_smem) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_l, gn_solve_linked_kernel, kSolveThreads, dyn_smem) != cudaSuccess) return 0;
    per_sm = per_sm < per_sm_l ? per_sm : per_sm_l;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    return per_sm * sms;
}

// cooperative: the launch itself guarantees that the whole grid is resident.  Rank plans that SHARE one device
// (peer-linked plans of one process on one GPU: tests, emulation) are launched plainly instead -- cooperative
// launches do not overlap with each other, and those kernels wait for one another; their grids are capped by the
// caller (gse_options.max_ctas) so that all of them fit side by side.
cudaError_t launch_solve(const SolveProg& sp, const EvalProg& ep, const FrontTab& ft, double* va, double* vm,
                         int grid, size_t dyn_smem, cudaStream_t s, bool cooperative) {
    void* args[] = {(void*)&sp, (void*)&ep, (void*)&ft, (void*)&va, (void*)&vm};
    const void* fn = sp.lk.world > 1 ? (const void*)gn_solve_linked_kernel : (const void*)gn_solve_kernel;
    if (cooperative) return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSolveThreads), args, dyn_smem, s);
    return cudaLaunchKernel(fn, dim3(grid), dim3(kSolveThreads), args, dyn_smem, s);
}

}  // namespace gse
