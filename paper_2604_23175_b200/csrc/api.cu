// api.cu -- C ABI of libgridse_b200.so (include/gridse_b200.h): plan lifetime, the
// device-resident Gauss-Newton loop (CUDA-graph captured), phase-level entry points and
// readback in the reference's layouts.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <unistd.h>

#include "kernels.cuh"
#include "plan.hpp"

using namespace gse;

namespace {

template <class T>
struct DevBuf {
    T* ptr = nullptr;
    size_t n = 0;
    cudaError_t upload(const std::vector<T>& h) {
        n = h.size();
        cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T));
        if (e != cudaSuccess) return e;
        if (n) e = cudaMemcpy(ptr, h.data(), n * sizeof(T), cudaMemcpyHostToDevice);
        return e;
    }
    cudaError_t alloc(size_t count, bool zero = true) {
        n = count;
        cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T));
        if (e == cudaSuccess && zero) e = cudaMemset(ptr, 0, std::max<size_t>(n, 1) * sizeof(T));
        return e;
    }
    void release() { if (ptr) cudaFree(ptr); ptr = nullptr; }
};

struct LevelLaunch { int pclass; int first, count; size_t smem; int phase; };
// (kBlkGDelta / kBlkGErr: this rank's copy of the GLOBAL per-iteration norms and of the inverted global failure
// code of a peer-linked solve -- every rank max-merges its own values into every copy)
constexpr int kBlkDelta = 0, kBlkResult = 64, kBlkErr = 65, kBlkObj = 66, kBlkStamps = 68, kBlkGDelta = 68 + 1 + 64 * 8,
              kBlkGErr = kBlkGDelta + 64, kBlkWords = kBlkGErr + 2;
struct BwdLaunch { int first, count, phase; };

}  // namespace

struct gse_plan {
    HostProgram hp;
    gse_error err{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;                   // false: the caller's stream (gse_options.stream)
    bool coordinator = true;

    // network + measurements
    DevBuf<int32_t> y_ptr, y_idx, br_from, br_to, m_type, m_target;
    DevBuf<double> y_g, y_b, br_y, z, w;
    // evaluation units
    DevBuf<int32_t> vm_bus, vm_row, vm_slot, fl_branch, fl_from, fl_to, fl_row, fl_slot;
    DevBuf<int32_t> inj_bus, inj_rowp, inj_rowq, inj_slotp, inj_slotq, inj_nth;
    DevBuf<double> val;                       // [(g, w*g) per slot | w*r per row]: template partials, weighted residuals
    // accumulation programs
    DevBuf<int32_t> acc_ptr, acc_items, acc_uniq, racc_ptr, racc_a, racc_b;
    DevBuf<uint32_t> acc_pair;
    AccProg ap{};
    DevBuf<double> gval, refval;
    // fronts
    DevBuf<int32_t> f_p, f_u1, f_T, f_nchild, f_child_ptr, f_children, f_rel_off, f_rel, f_reg_off, f_reg_ptr;
    DevBuf<int32_t> f_rows_off, f_rows, f_cb_off, f_cbounds, bcnt;
    DevBuf<BwdTask> btasks;
    DevBuf<double> bpart, dinv;
    DevBuf<long long> tbuf;
    DevBuf<uint32_t> orig_pos;
    DevBuf<int64_t> f_gval_off, f_l_off, f_u_off;
    DevBuf<TaskRec> tasks;
    DevBuf<ChildRec> crecs;
    DevBuf<int32_t> bwd_fronts;
    DevBuf<double> lbuf, ubuf, xsol;
    DevBuf<int32_t> upd_bus, upd_quant, upd_pos, pos_bq;
    DevBuf<double> obj_partial, status;       // status: [delta bits as double slot, err as double] (MAX-reducible)
    DevBuf<unsigned long long> flags;         // [0] delta_inf bits, [1] failure code (min)
    double* h_stage[2] = {nullptr, nullptr};  // pinned staging of new z / w
    cudaEvent_t stage_done[2] = {nullptr, nullptr};
    unsigned long long* h_flags = nullptr;    // pinned
    double* h_obj = nullptr;                  // pinned
    std::vector<LevelLaunch> fwd;
    std::vector<BwdLaunch> bwd;
    EvalProg ep{};
    FrontTab ft{};

    // persistent dataflow kernel (solve_kernel.cu)
    SolveProg sp{};
    DevBuf<unsigned long long> syncblk;       // [delta 64 | result | err copy | J | pad | stamps 1+512 | counters...]
    unsigned long long* h_blk = nullptr;      // pinned mirror of the first kBlkWords words
    DevBuf<unsigned long long> trace;         // per-item stamps of the persistent kernel (debug)
    int solve_grid = 0, max_ctas = 0;
    size_t solve_smem = 0, sync_bytes = 0;
    bool persistent = false, stamps = true;
    // peer-linked multi-rank solve (gse_peer_link): exchanges inside the persistent kernel over peer memory
    bool linked = false, prepared = false, shares_device = false;
    // gse_solve_io: start state (device) copied in and final state copied out (pinned host) on the plan's stream,
    // inside the same enqueue as the launch -- one host synchronisation per solve
    const double* io_init = nullptr;
    double* io_out = nullptr;
    int n_gamma_fronts = 0;
    std::vector<void*> ipc_opened;            // allocations of other processes mapped with cudaIpcOpenMemHandle

    cudaGraphExec_t graph = nullptr;
    const double* graph_va = nullptr;
    const double* graph_vm = nullptr;
    cudaEvent_t ev[8] = {};
    int launches_per_iter = 0;
    long long launches_last = 0;

    ~gse_plan();
};

namespace {

int fail(gse_plan* p, int code, const std::string& msg, int area = -1, int pivot = -1) {
    p->err.code = code; p->err.area = area; p->err.pivot = pivot;
    snprintf(p->err.message, sizeof(p->err.message), "%s", msg.c_str());
    return code;
}
#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(plan, GSE_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Host <-> device traffic of the C ABI is ordered on the PLAN's stream (a non-blocking stream, or the
// caller's): a copy on the legacy default stream would not be ordered with the plan's kernels, and a
// pageable host-to-device cudaMemcpy may return before the data has landed.  The copy is enqueued on
// the plan's stream and the host waits for it (the source / destination is caller memory).
cudaError_t copy_sync(gse_plan* plan, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    if (bytes == 0) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, plan->stream);
    return e == cudaSuccess ? cudaStreamSynchronize(plan->stream) : e;
}
// failure flag back to "none": stream-ordered, so it cannot race with the reads / atomicMin of the next solve
cudaError_t reset_failure_flag(gse_plan* plan) {
    return cudaMemsetAsync(plan->flags.ptr + 1, 0xff, sizeof(unsigned long long), plan->stream);
}

// all kernels of one outer iteration on plan->stream; phase boundaries marked with events if timed
int enqueue_phase_assemble(gse_plan* plan, const double* va, const double* vm) {
    launch_eval(plan->ep, va, vm, plan->stream);
    launch_accumulate_staged(plan->ap, plan->stream);
    return 2;
}
int enqueue_fwd(gse_plan* plan, int phase) {
    int n = 0;
    for (auto& L : plan->fwd) {
        if (L.phase != phase) continue;
        launch_front_tasks(L.pclass, plan->ft, plan->tasks.ptr + L.first, L.count, L.smem, plan->gval.ptr, plan->lbuf.ptr,
                           plan->ubuf.ptr, plan->flags.ptr + 1, plan->stream);
        ++n;
    }
    return n;
}
int enqueue_bwd(gse_plan* plan, int phase) {
    int n = 0;
    for (auto& B : plan->bwd) {
        if (B.phase != phase) continue;
        launch_backward(plan->ft, plan->btasks.ptr + B.first, B.count, plan->lbuf.ptr, plan->xsol.ptr, plan->bpart.ptr, plan->bcnt.ptr,
                        plan->stream);
        ++n;
    }
    return n;
}
int enqueue_update(gse_plan* plan, double* va, double* vm) {
    launch_update(plan->upd_bus.ptr, plan->upd_quant.ptr, plan->upd_pos.ptr, (int)plan->upd_bus.n, plan->xsol.ptr, va, vm,
                  plan->flags.ptr, plan->stream);
    return 1;
}

int enqueue_iteration(gse_plan* plan, double* va, double* vm, bool events) {
    cudaStream_t s = plan->stream;
    int n = 0;
    cudaMemsetAsync(plan->flags.ptr, 0, sizeof(unsigned long long), s);
    if (events) cudaEventRecord(plan->ev[0], s);
    n += enqueue_phase_assemble(plan, va, vm);
    if (events) cudaEventRecord(plan->ev[1], s);
    n += enqueue_fwd(plan, 1);
    if (events) cudaEventRecord(plan->ev[2], s);
    n += enqueue_fwd(plan, 2);
    if (events) cudaEventRecord(plan->ev[3], s);
    n += enqueue_fwd(plan, 3);
    n += enqueue_bwd(plan, 3);
    if (events) cudaEventRecord(plan->ev[4], s);
    n += enqueue_bwd(plan, 4);
    n += enqueue_update(plan, va, vm);
    if (events) cudaEventRecord(plan->ev[5], s);
    cudaMemcpyAsync(plan->h_flags, plan->flags.ptr, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    return n;
}

int decode_failure(gse_plan* plan, unsigned long long code) {
    const int f = (int)(code >> 32), k = (int)(code & 0xffffffffull);
    if (f < 0 || f >= (int)plan->hp.fronts.size())      // peer-linked solve: a boundary front, which only the coordinator's plan holds
        return fail(plan, GSE_E_NOT_SPD_BOUNDARY, "boundary system not positive definite (reported by the coordinator rank)", -1, -1);
    const Front& fr = plan->hp.fronts[f];
    const int pos = fr.rows[k];
    const int orig = plan->hp.perm_orig[pos];
    char buf[160];
    if (fr.kind == 3) {
        snprintf(buf, sizeof buf, "boundary system not positive definite at pivot %d", orig);
        return fail(plan, GSE_E_NOT_SPD_BOUNDARY, buf, -1, orig);
    }
    snprintf(buf, sizeof buf, "area %d interior block not positive definite at pivot %d", fr.area, orig);
    return fail(plan, GSE_E_NOT_SPD_AREA, buf, fr.area, orig);
}

int ensure_graph(gse_plan* plan, double* va, double* vm) {
    if (plan->graph && plan->graph_va == va && plan->graph_vm == vm) return GSE_OK;
    if (plan->graph) { cudaGraphExecDestroy(plan->graph); plan->graph = nullptr; }
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(plan->stream, cudaStreamCaptureModeThreadLocal));
    plan->launches_per_iter = enqueue_iteration(plan, va, vm, false);
    CU(cudaStreamEndCapture(plan->stream, &g));
    CU(cudaGraphInstantiate(&plan->graph, g, 0));
    cudaGraphDestroy(g);
    plan->graph_va = va; plan->graph_vm = vm;
    return GSE_OK;
}

}  // namespace

gse_plan::~gse_plan() {
    cudaSetDevice(device);
    if (graph) cudaGraphExecDestroy(graph);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (stream && own_stream) cudaStreamDestroy(stream);
    if (h_flags) cudaFreeHost(h_flags);
    if (h_obj) cudaFreeHost(h_obj);
    if (h_blk) cudaFreeHost(h_blk);
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    for (int i = 0; i < 2; ++i) { if (h_stage[i]) cudaFreeHost(h_stage[i]); if (stage_done[i]) cudaEventDestroy(stage_done[i]); }
    syncblk.release(); trace.release();
    DevBuf<int32_t>* ib[] = {&y_ptr, &y_idx, &br_from, &br_to, &m_type, &m_target, &vm_bus, &vm_row, &vm_slot, &fl_branch,
                             &fl_from, &fl_to, &fl_row, &fl_slot, &inj_bus, &inj_rowp, &inj_rowq, &inj_slotp, &inj_slotq, &inj_nth,
                             &acc_ptr, &acc_items, &acc_uniq, &racc_ptr, &racc_a, &racc_b, &f_p, &f_u1, &f_T, &f_nchild,
                             &f_child_ptr, &f_children, &f_rel_off, &f_rel, &f_reg_off, &f_reg_ptr, &f_rows_off, &f_rows, &f_cb_off, &f_cbounds, &bcnt,
                             &bwd_fronts, &upd_bus, &upd_quant, &upd_pos};
    for (auto* b : ib) b->release();
    DevBuf<double>* db[] = {&y_g, &y_b, &br_y, &z, &w, &val, &gval, &refval, &lbuf, &ubuf, &xsol, &obj_partial, &status};
    for (auto* b : db) b->release();
    dinv.release(); acc_pair.release();
    btasks.release(); bpart.release(); tbuf.release(); crecs.release();
    orig_pos.release(); f_gval_off.release(); f_l_off.release(); f_u_off.release(); tasks.release(); flags.release();
}

extern "C" {

const char* gse_version(void) { return "gridse-b200 0.1.0 (sm_100a)"; }

const gse_error* gse_last_error(const gse_plan* plan) { return &plan->err; }

static int create_plan(const gse_problem_desc* d, const gse_options* opt, BuildOptions bo, gse_plan** out);

int gse_plan_create(const gse_problem_desc* d, const gse_options* opt, gse_plan** out) {
    return create_plan(d, opt, BuildOptions{}, out);
}

static int create_plan(const gse_problem_desc* d, const gse_options* opt, BuildOptions bo, gse_plan** out) {
    if (!d || !out) return GSE_E_INVALID;
    gse_plan* plan = new gse_plan();
    *out = plan;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(plan, GSE_E_NO_DEVICE, "no CUDA device visible: gridse-b200 has no CPU fallback");
    plan->device = opt ? opt->device : 0;
    CU(cudaSetDevice(plan->device));
    // Update-row chunk of a task: latency-bound plans (every <= ~30k-bus shape: fewer tasks than ~4 per resident
    // CTA) run best with 32-row tiles -- shorter panels and gathers on the critical chain (PEGASE-9241: 1.49 vs
    // 1.51 ms, PEGASE-2869: 0.81 vs 0.85 ms per solve); throughput-bound plans with 48 (the ~100k-bus grid:
    // 5.60 vs 7.54 ms).  gse_options.tile_rows / GSE_TILE_ROWS override.
    bo.tile_rows = d->n_bus <= 30000 ? 32 : 48;
    bo.interior_merge = d->n_bus <= 30000 ? 0.0 : 1.0;       // relaxed amalgamation of the interiors: throughput-bound plans only (plan.hpp)
    if (d->n_bus > 30000) bo.leaf_buses = 32;                 // ... on finer leaves: the merges then fill the fronts up to the pivot cap
                                                              // (5.39 -> 5.29 ms at ~100k / 128, tools/gpu_sweep5.sh)
    if (opt) {
        bo.dense = opt->backend_dense != 0;
        if (opt->leaf_buses > 0) bo.leaf_buses = opt->leaf_buses;
        if (opt->max_pivots == 32 || opt->max_pivots == 64) bo.max_pivots = opt->max_pivots;
        if (opt->tile_rows >= 8 && opt->tile_rows <= kMaxTile) bo.tile_rows = opt->tile_rows / 8 * 8;
        if (opt->boundary_mode >= 0 && opt->boundary_mode <= 2) bo.boundary_mode = opt->boundary_mode;
        bo.rank = opt->rank; bo.world = std::max(1, opt->world);
        plan->max_ctas = std::max(0, opt->max_ctas);
        if (opt->area_rank) bo.area_rank.assign(opt->area_rank, opt->area_rank + d->n_areas);
    }
    if (const char* e = getenv("GSE_TILE_ROWS")) { int v = atoi(e); if (v >= 8 && v <= kMaxTile) bo.tile_rows = v / 8 * 8; }
    if (const char* e = getenv("GSE_GAMMA_TILE_ROWS")) { int v = atoi(e); if (v >= 8 && v <= kMaxTile) bo.gamma_tile_rows = v / 8 * 8; }
    if (const char* e = getenv("GSE_BOUNDARY")) { int v = atoi(e); if (v >= 0 && v <= 2) bo.boundary_mode = v; }
    if (const char* e = getenv("GSE_GAMMA_LEAF")) { int v = atoi(e); if (v >= 1) bo.gamma_leaf_buses = v; }
    if (const char* e = getenv("GSE_MAX_PIVOTS")) { int v = atoi(e); if (v == 32 || v == 64) bo.max_pivots = v; }
    if (const char* e = getenv("GSE_LEAF_BUSES")) { int v = atoi(e); if (v >= 1) bo.leaf_buses = v; }
    if (const char* e = getenv("GSE_SEPW")) bo.sep_weight = atof(e);
    if (const char* e = getenv("GSE_GAMMA_SEPW")) bo.gamma_sep_weight = atof(e);
    if (const char* e = getenv("GSE_SPLIT_MIN")) { int v = atoi(e); if (v >= 1) bo.split_min_pivots = v; }
    if (const char* e = getenv("GSE_SPLIT_TASKS")) { int v = atoi(e); if (v >= 1) bo.split_min_tasks = v; }
    if (const char* e = getenv("GSE_INTERIOR_MERGE")) bo.interior_merge = atof(e);
    if (const char* e = getenv("GSE_GAMMA_MERGE")) bo.gamma_merge = atof(e);
    if (const char* e = getenv("GSE_MAX_CTAS")) { int v = atoi(e); if (v >= 1) plan->max_ctas = v; }
    plan->coordinator = bo.rank == 0;
    HostProgram& hp = plan->hp;
    std::string msg = build_host_program(*d, bo, hp);
    if (!msg.empty()) return fail(plan, GSE_E_INVALID, msg);
    if (hp.max_front >= 65535) return fail(plan, GSE_E_INVALID, "front order exceeds 65534");

    if (opt && opt->stream) { plan->stream = (cudaStream_t)opt->stream; plan->own_stream = false; }
    else CU(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
    CU(configure_kernels());
    CU(configure_unit_kernels());
    for (auto& e : plan->ev) CU(cudaEventCreate(&e));
    CU(cudaMallocHost(&plan->h_flags, 2 * sizeof(unsigned long long)));
    CU(cudaMallocHost(&plan->h_obj, sizeof(double)));

    // ---- network / measurements ----
    const int nb = d->n_bus, nnz = d->y_ptr[nb];
    CU(plan->y_ptr.upload(std::vector<int32_t>(d->y_ptr, d->y_ptr + nb + 1)));
    CU(plan->y_idx.upload(std::vector<int32_t>(d->y_idx, d->y_idx + nnz)));
    CU(plan->y_g.upload(std::vector<double>(d->y_g, d->y_g + nnz)));
    CU(plan->y_b.upload(std::vector<double>(d->y_b, d->y_b + nnz)));
    CU(plan->br_from.upload(std::vector<int32_t>(d->br_from, d->br_from + d->n_branch)));
    CU(plan->br_to.upload(std::vector<int32_t>(d->br_to, d->br_to + d->n_branch)));
    CU(plan->br_y.upload(std::vector<double>(d->br_y, d->br_y + 8 * (size_t)d->n_branch)));
    CU(plan->m_type.upload(std::vector<int32_t>(d->m_type, d->m_type + d->n_rows)));
    CU(plan->m_target.upload(std::vector<int32_t>(d->m_target, d->m_target + d->n_rows)));
    {   // measured values and weights in ONE block [z | w]: a scan's refresh from a contiguous pinned block is one copy
        std::vector<double> zw(d->m_z, d->m_z + d->n_rows);
        zw.insert(zw.end(), d->m_w, d->m_w + d->n_rows);
        CU(plan->z.upload(zw));
    }
    // ---- evaluation units ----
    CU(plan->vm_bus.upload(hp.vm_bus)); CU(plan->vm_row.upload(hp.vm_row)); CU(plan->vm_slot.upload(hp.vm_slot));
    CU(plan->fl_branch.upload(hp.fl_branch)); CU(plan->fl_from.upload(hp.fl_from)); CU(plan->fl_to.upload(hp.fl_to));
    CU(plan->fl_row.upload(hp.fl_row)); CU(plan->fl_slot.upload(hp.fl_slot));
    CU(plan->inj_bus.upload(hp.inj_bus)); CU(plan->inj_rowp.upload(hp.inj_rowp)); CU(plan->inj_rowq.upload(hp.inj_rowq));
    CU(plan->inj_slotp.upload(hp.inj_slotp)); CU(plan->inj_slotq.upload(hp.inj_slotq)); CU(plan->inj_nth.upload(hp.inj_nth));
    CU(plan->val.alloc(hp.n_val));
    if (hp.acc_stage_max > kAccStageMax || hp.acc_pair_max > kAccPairMax) return fail(plan, GSE_E_INVALID, "a normal-equation entry has too many contributions for the staged accumulation");
    CU(plan->acc_ptr.upload(hp.acc_lptr)); CU(plan->acc_items.upload(hp.acc_items)); CU(plan->acc_uniq.upload(hp.acc_uniq));
    CU(plan->acc_pair.upload(hp.acc_pair));
    CU(plan->gval.alloc(hp.n_gval));
    plan->ap = AccProg{plan->acc_items.ptr, plan->acc_uniq.ptr, plan->acc_ptr.ptr, plan->acc_pair.ptr, plan->val.ptr,
                       plan->gval.ptr, (int32_t)(hp.acc_items.size() / 8)};
    EvalProg& ep = plan->ep;
    ep.y_ptr = plan->y_ptr.ptr; ep.y_idx = plan->y_idx.ptr; ep.y_g = plan->y_g.ptr; ep.y_b = plan->y_b.ptr;
    ep.br_y = plan->br_y.ptr; ep.z = plan->z.ptr; ep.w = plan->z.ptr + d->n_rows; ep.slack = d->slack;
    ep.n_vm = (int)hp.vm_bus.size(); ep.n_fl = (int)hp.fl_branch.size(); ep.n_inj = (int)hp.inj_bus.size();
    ep.has_current = 0;
    for (int r = 0; r < d->n_rows; ++r) if (d->m_type[r] >= 7) { ep.has_current = 1; break; }
    ep.vm_bus = plan->vm_bus.ptr; ep.vm_row = plan->vm_row.ptr; ep.vm_slot = plan->vm_slot.ptr;
    ep.fl_branch = plan->fl_branch.ptr; ep.fl_from = plan->fl_from.ptr; ep.fl_to = plan->fl_to.ptr;
    ep.fl_row = plan->fl_row.ptr; ep.fl_slot = plan->fl_slot.ptr;
    ep.inj_bus = plan->inj_bus.ptr; ep.inj_rowp = plan->inj_rowp.ptr; ep.inj_rowq = plan->inj_rowq.ptr;
    ep.inj_slotp = plan->inj_slotp.ptr; ep.inj_slotq = plan->inj_slotq.ptr; ep.inj_nth = plan->inj_nth.ptr;
    ep.g = plan->val.ptr; ep.wr = plan->val.ptr + 2 * hp.n_slots;

    // ---- front tables ----
    const size_t nf = hp.fronts.size();
    std::vector<int32_t> fp(nf), fu(nf), fT(nf), fnc(nf), fcp(nf), frel_off(nf), frows_off(nf), children, rel, rows;
    std::vector<int64_t> fg(nf), fl(nf), fuo(nf);
    for (size_t i = 0; i < nf; ++i) {
        const Front& f = hp.fronts[i];
        fp[i] = f.p; fu[i] = f.u1; fT[i] = std::max(f.T, 1); fnc[i] = (int)f.children.size(); fcp[i] = (int)children.size();
        children.insert(children.end(), f.children.begin(), f.children.end());
        frel_off[i] = (int)rel.size(); rel.insert(rel.end(), f.rel.begin(), f.rel.end());
        frows_off[i] = (int)rows.size(); rows.insert(rows.end(), f.rows.begin(), f.rows.end());
        fg[i] = f.gval_off; fl[i] = f.l_off; fuo[i] = f.u_off;
    }
    std::vector<int32_t> extra_rel_off(hp.extra_rel.size(), 0);
    for (size_t i = 0; i < hp.extra_rel.size(); ++i) { extra_rel_off[i] = (int32_t)rel.size(); rel.insert(rel.end(), hp.extra_rel[i].begin(), hp.extra_rel[i].end()); }
    std::vector<int32_t> cb_off(1, 0), cbounds(1, 0);   // (kept for the table layout; bounds now live in ChildRec)
    CU(plan->f_cb_off.upload(cb_off)); CU(plan->f_cbounds.upload(cbounds));
    CU(plan->f_p.upload(fp)); CU(plan->f_u1.upload(fu)); CU(plan->f_T.upload(fT)); CU(plan->f_nchild.upload(fnc));
    CU(plan->f_child_ptr.upload(fcp)); CU(plan->f_children.upload(children)); CU(plan->f_rel_off.upload(frel_off));
    CU(plan->f_rel.upload(rel)); CU(plan->f_reg_off.upload(hp.front_reg_off)); CU(plan->f_reg_ptr.upload(hp.reg_ptr));
    CU(plan->f_rows_off.upload(frows_off)); CU(plan->f_rows.upload(rows)); CU(plan->orig_pos.upload(hp.orig_pos));
    CU(plan->f_gval_off.upload(fg)); CU(plan->f_l_off.upload(fl)); CU(plan->f_u_off.upload(fuo));
    CU(plan->lbuf.alloc(hp.n_lbuf)); CU(plan->ubuf.alloc(hp.n_ubuf)); CU(plan->xsol.alloc(hp.n_pos + 2));
    FrontTab& ft = plan->ft;
    ft.p = plan->f_p.ptr; ft.u1 = plan->f_u1.ptr; ft.T = plan->f_T.ptr; ft.nchild = plan->f_nchild.ptr;
    ft.child_ptr = plan->f_child_ptr.ptr; ft.children = plan->f_children.ptr; ft.rel_off = plan->f_rel_off.ptr;
    ft.cb_off = plan->f_cb_off.ptr; ft.cbounds = plan->f_cbounds.ptr;
    ft.rel = plan->f_rel.ptr; ft.reg_off = plan->f_reg_off.ptr; ft.reg_ptr = plan->f_reg_ptr.ptr;
    ft.orig_pos = plan->orig_pos.ptr; ft.gval_off = plan->f_gval_off.ptr; ft.l_off = plan->f_l_off.ptr;
    ft.u_off = plan->f_u_off.ptr; ft.rows_off = plan->f_rows_off.ptr; ft.rows = plan->f_rows.ptr;

    // ---- level launches: tasks grouped by (level, pivot class) ----
    std::vector<int32_t> dinv_off(nf, 0);
    { int32_t c = 0; for (size_t i = 0; i < nf; ++i) { dinv_off[i] = c; c += (hp.fronts[i].p + 7) / 8 * 8; }
      CU(plan->dinv.alloc(c + 8)); plan->ft.dinv = plan->dinv.ptr; }
    std::vector<TaskRec> trecs;
    std::vector<ChildRec> crecs;
    auto ntasks_of = [&](int fr) { const int n = hp.fronts[fr].nch; return n * (n + 1) / 2; };
    int n_solve_tasks = 0;
    size_t solve_task_smem = 0;
    // two passes: the tasks of the solve in level order first (the persistent kernel walks exactly
    // this prefix), then the readback-only boundary root of the block-sparse mode (phase 5)
    // within a level: stage 0 = fused + panel tasks, stage 1 = update tasks (a separate launch on the
    // level path: they read the panels stage 0 stored)
    for (int pass = 0; pass < 2; ++pass)
    for (size_t lv = 0; lv < hp.fwd_levels.size(); ++lv) {
        for (int skey : {11, 10, 21, 20, 31, 30, 51, 50, 111, 121, 131, 151}) {      // (stage, phase, pivot class)
            const int key = skey % 100, stage = skey / 100;
            if ((key / 10 == 5) != (pass == 1)) continue;
            const int phase = key / 10, pclass = key % 10;
            LevelLaunch L{pclass, (int)trecs.size(), 0, 0, phase};
            for (const Task& t : hp.fwd_levels[lv]) {
                const Front& f = hp.fronts[t.front];
                const int cls = f.p == 0 ? 0 : 1;
                if (cls != pclass || t.phase != phase || (t.kind == 2) != (stage == 1)) continue;
                const int T = std::max(f.T, 1);
                const int ni = std::min(T, f.u1 - t.ci * T), nj = std::min(T, f.u1 - t.cj * T);
                const bool diag = t.ci == t.cj;
                const int kind = t.kind;
                // chain fronts: single child, identity map, no original entries -> tile read in place
                bool direct = f.kind == 3 && f.children.size() == 1 && f.n_orig == 0;
                if (direct) {
                    const std::vector<int>& rel_c = hp.fronts[f.children[0]].rel;
                    for (size_t q = 0; q < rel_c.size() && direct; ++q) direct = rel_c[q] == (int)q;
                }
                L.smem = std::max(L.smem, sizeof(double) * task_smem_doubles(f.p, ni, nj, diag, direct, kind));
                TaskRec r{};
                r.front = t.front; r.ci = t.ci; r.cj = t.cj; r.p = f.p; r.u1 = f.u1; r.T = T;
                r.gval_off = f.gval_off; r.l_off = f.l_off; r.u_off = f.u_off; r.flags = (direct ? 1 : 0) | (f.n_orig > 0 ? 2 : 0) | ((f.kind == 1 && bo.world > 1 && bo.rank != 0) ? 4 : 0);
                r.phase = phase; r.kind = kind; r.nch = f.nch; r.area = f.area; r.level = f.level;
                r.dinv_off = dinv_off[t.front];
                const int32_t* rp = &hp.reg_ptr[hp.front_reg_off[t.front]];
                const int ridI = (t.ci + 1) * (t.ci + 2) / 2, ridJ = (t.cj + 1) * (t.cj + 2) / 2;
                r.reg[0] = rp[0]; r.reg[1] = rp[1];
                r.reg[2] = rp[ridI]; r.reg[3] = rp[ridI + 1];
                r.reg[4] = rp[ridJ]; r.reg[5] = rp[ridJ + 1];
                r.reg[6] = rp[ridI + t.cj + 1]; r.reg[7] = rp[ridI + t.cj + 2];
                r.child_off = (int32_t)crecs.size();
                for (size_t cx = 0; cx < f.children.size(); ++cx) {
                    const int ch = f.children[cx];
                    const Front& c = hp.fronts[ch];
                    const bool over = cx < f.child_rel.size() && f.child_rel[cx] >= 0;
                    const std::vector<int>& relv = over ? hp.extra_rel[f.child_rel[cx]] : c.rel;
                    auto lb = [&](int key2) { return (int32_t)(std::lower_bound(relv.begin(), relv.end(), key2) - relv.begin()); };
                    ChildRec cr{};
                    cr.u_off = c.u_off; cr.rel_off = over ? extra_rel_off[f.child_rel[cx]] : frel_off[ch];
                    cr.eP = f.p ? lb(f.p) : 0;
                    cr.bI = lb(f.p + t.ci * T); cr.eI = lb(f.p + t.ci * T + ni);
                    cr.bJ = lb(f.p + t.cj * T); cr.eJ = lb(f.p + t.cj * T + nj);
                    cr.front = (c.kind == 1 && c.area >= 0 && !hp.owned[c.area]) ? -(c.area + 1) : ch; cr.need = ntasks_of(ch);
                    const bool hits_panel = f.p && kind != 2 && cr.eP > 0;
                    const bool hits_tile = !direct && kind != 1 && cr.eI > cr.bI && cr.eJ > cr.bJ;
                    if (!hits_panel && !hits_tile && !direct) continue;   // pruned (order of the rest is kept)
                    crecs.push_back(cr);
                    ++r.nchild;
                }
                trecs.push_back(r);
                ++L.count;
            }
            if (pass == 0) { n_solve_tasks = (int)trecs.size(); solve_task_smem = std::max(solve_task_smem, L.smem); }
            if (L.count) {
                if (L.smem > 214 * 1024) return fail(plan, GSE_E_INVALID, "front task exceeds shared memory");
                plan->fwd.push_back(L);
            }
        }
    }
    CU(plan->tasks.upload(trecs));
    CU(plan->crecs.upload(crecs));
    plan->ft.task0 = plan->tasks.ptr; plan->ft.tbuf = nullptr; plan->ft.crecs = plan->crecs.ptr;
    std::vector<BwdTask> btasks;
    int pbase = 0;
    std::vector<int> pivot_owner((size_t)hp.n_pos + 2, -1);       // solution position -> front that eliminates it (on this rank)
    for (size_t f = 0; f < nf; ++f) for (int k = 0; k < hp.fronts[f].p; ++k) pivot_owner[hp.fronts[f].rows[k]] = (int)f;
    for (size_t i = 0; i < hp.bwd_levels.size(); ++i) {
        BwdLaunch B{(int)btasks.size(), 0, hp.bwd_phase[i]};
        for (int f : hp.bwd_levels[i]) {
            const int u = hp.fronts[f].u1 - 1;
            const int ns = std::max(1, (u + 63) / 64);
            const Front& fr = hp.fronts[f];
            int dep = fr.parent;
            while (dep >= 0 && hp.fronts[dep].p == 0) dep = hp.fronts[dep].parent;
            for (int sp = 0; sp < ns; ++sp) {
                BwdTask bt{};
                bt.front = f; bt.split = sp; bt.nsplit = ns; bt.pbase = pbase; bt.p = fr.p; bt.u = u;
                bt.rows_off = frows_off[f]; bt.dinv_off = dinv_off[f]; bt.l_off = fr.l_off;
                bt.dep = dep; bt.need = fr.nch; bt.phase = hp.bwd_phase[i];   // need: tasks that store a factor panel
                // update rows are in elimination order, so the nearest ancestor's pivots come first (at most 64 of
                // them: all inside split 0); rows 64 ... belong to the front that eliminates row 64 or to its ancestors
                bt.dep2 = dep; bt.early = 0;
                if (ns > 1 && dep >= 0) {
                    const int o = pivot_owner[fr.rows[fr.p + 64]];
                    if (o >= 0 && o != dep) { bt.dep2 = o; bt.early = 1; }
                }
                btasks.push_back(bt);
            }
            pbase += ns; B.count += ns;
        }
        plan->bwd.push_back(B);
    }
    CU(plan->btasks.upload(btasks));
    CU(plan->bpart.alloc((size_t)pbase * 64 + 64));
    CU(plan->bcnt.alloc(nf + 1));
    CU(plan->upd_bus.upload(hp.upd_bus)); CU(plan->upd_quant.upload(hp.upd_quant)); CU(plan->upd_pos.upload(hp.upd_pos));
    CU(plan->obj_partial.alloc(objective_blocks(d->n_rows) + 1));
    CU(plan->status.alloc(2));
    CU(plan->flags.alloc(2));
    CU(cudaMemset(plan->flags.ptr + 1, 0xff, sizeof(unsigned long long)));

    // ---- persistent dataflow kernel: one launch per solve (single-rank plans) ----
    {
        int mode = opt ? opt->persistent : 0;                       // 0 auto, 1 on, 2 off
        if (const char* e = getenv("GSE_PERSISTENT")) mode = atoi(e) ? 1 : 2;
        if (const char* e = getenv("GSE_STAMPS")) plan->stamps = atoi(e) != 0;
        SolveProg& sp = plan->sp;
        sp.n_units = ep.n_fl + ep.n_inj + ep.n_vm;
        sp.n_eval_items = (sp.n_units + kEvalPerItem - 1) / kEvalPerItem;
        sp.n_gval = hp.n_gval;
        sp.n_acc_items = plan->ap.n_items;
        sp.n_tasks = n_solve_tasks;
        sp.n_btasks = (int)btasks.size();
        sp.n_upd = (int)hp.upd_bus.size();
        sp.n_upd_items = (sp.n_upd + kUpdPerItem - 1) / kUpdPerItem;
        {
            std::vector<int32_t> bq((size_t)hp.n_pos, -1);
            for (size_t v = 0; v < hp.upd_bus.size(); ++v) bq[hp.upd_pos[v]] = 2 * hp.upd_bus[v] + hp.upd_quant[v];
            CU(plan->pos_bq.upload(bq));
            sp.pos_bq = plan->pos_bq.ptr;
        }
        sp.items_per_it = sp.n_eval_items + sp.n_acc_items + sp.n_tasks + sp.n_btasks + sp.n_upd_items;
        sp.n_bwd_fronts = 0;
        for (auto& lv : hp.bwd_levels) sp.n_bwd_fronts += (int)lv.size();
        sp.n_fronts = (int)nf; sp.n_rows = d->n_rows;
        sp.tasks = plan->tasks.ptr; sp.btasks = plan->btasks.ptr;
        sp.acc_items = plan->acc_items.ptr; sp.acc_uniq = plan->acc_uniq.ptr; sp.acc_ptr = plan->acc_ptr.ptr;
        sp.acc_pair = plan->acc_pair.ptr; sp.val = plan->val.ptr;
        sp.upd_bus = plan->upd_bus.ptr; sp.upd_quant = plan->upd_quant.ptr; sp.upd_pos = plan->upd_pos.ptr;
        sp.m_type = plan->m_type.ptr; sp.m_target = plan->m_target.ptr; sp.br_from = plan->br_from.ptr; sp.br_to = plan->br_to.ptr;
        sp.gval = plan->gval.ptr; sp.lbuf = plan->lbuf.ptr; sp.ubuf = plan->ubuf.ptr; sp.xsol = plan->xsol.ptr;
        sp.bpart = plan->bpart.ptr; sp.obj_partial = plan->obj_partial.ptr; sp.bcnt = plan->bcnt.ptr;
        sp.front0 = ctr_front0(hp.n_areas);
        sp.bwd_poll = 1; sp.pad0 = 0;
        if (const char* e = getenv("GSE_BWD_POLL")) sp.bwd_poll = atoi(e) != 0;
        // chain ranges of the task list: runs of levels with at most ~one panel task per SM (the top of the areas, the
        // boundary tree).  Those tasks are the latency chains; the persistent kernel hands them to one CTA per SM only
        // (two panel factorisations on one SM slow each other by a quarter).
        sp.n_chain = 0;
        {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plan->device);
            std::vector<int> panels(hp.fwd_levels.size() + 1, 0), total(hp.fwd_levels.size() + 1, 0);
            for (int t = 0; t < n_solve_tasks; ++t) { total[trecs[t].level]++; panels[trecs[t].level] += trecs[t].p > 0; }
            int min_items = 4 * 2 * sms;                        // small plans: a grid's worth of pulls spans iterations
            if (const char* e = getenv("GSE_CHAIN_MIN_ITEMS")) min_items = atoi(e);
            bool on = sp.items_per_it >= min_items;
            if (const char* e = getenv("GSE_CHAIN_SM")) on = on && atoi(e) != 0;
            int mode = 1;                                       // 1: the boundary suffix (measured best), 2: every sparse run (the top interior levels too: 0.5 % slower)
            if (const char* e = getenv("GSE_CHAIN_MODE")) mode = atoi(e);
            auto sparse = [&](int t) {
                const int lv = trecs[t].level;
                if (mode == 1) return trecs[t].phase == 3 && total[lv] <= sms - 8;
                return panels[lv] > 0 && panels[lv] <= sms - 8 && total[lv] <= 2 * sms;
            };
            for (int t = 0; on && t < n_solve_tasks;) {
                if (!sparse(t)) { ++t; continue; }
                int e = t;
                while (e < n_solve_tasks && sparse(e)) ++e;
                if (e - t >= 8) {
                    if (sp.n_chain == 4) { sp.chain_hi[3] = e; }       // (more runs than slots: the last slot absorbs the rest)
                    else { sp.chain_lo[sp.n_chain] = t; sp.chain_hi[sp.n_chain] = e; ++sp.n_chain; }
                }
                t = e;
            }
            if (mode == 1 && sp.n_chain) {                      // the suffix form: only a run that reaches the end of the list
                if (sp.chain_hi[sp.n_chain - 1] == n_solve_tasks) { sp.chain_lo[0] = sp.chain_lo[sp.n_chain - 1]; sp.chain_hi[0] = n_solve_tasks; sp.n_chain = 1; }
                else sp.n_chain = 0;
            }
        }
        const size_t nctr = sp.front0 + 3 * nf;
        plan->sync_bytes = sizeof(unsigned long long) * kBlkWords + sizeof(unsigned) * nctr;
        CU(plan->syncblk.alloc(kBlkWords + (nctr + 1) / 2));
        CU(cudaMallocHost(&plan->h_blk, sizeof(unsigned long long) * kBlkWords));
        unsigned long long* blk = plan->syncblk.ptr;
        sp.delta = blk + kBlkDelta; sp.result = reinterpret_cast<int32_t*>(blk + kBlkResult);
        sp.err_out = blk + kBlkErr; sp.obj_out = reinterpret_cast<double*>(blk + kBlkObj);
        sp.stamps = plan->stamps ? blk + kBlkStamps : nullptr;
        sp.ctr = reinterpret_cast<unsigned*>(blk + kBlkWords);
        sp.err = plan->flags.ptr + 1;
        plan->solve_smem = std::max<size_t>(solve_task_smem, kAccSmemBytes);   // >= BwdScratch too
        plan->persistent = false;
        if (mode != 2 && bo.world == 1 && sp.items_per_it > 0) {
            const int cap = solve_kernel_max_ctas(plan->solve_smem, plan->device);
            if (cap <= 0) return fail(plan, GSE_E_CUDA, "persistent solve kernel does not fit this device");
            // Latency-bound plans (a few backward tasks per resident CTA): the state update and the norm ride on
            // the backward tasks (every variable is the pivot of exactly one front) and the update items go.
            // Throughput-bound plans keep them: ~1.5 us more per backward task would cost more than the hop saves.
            bool fuse = sp.n_btasks < 4 * cap;
            if (const char* e = getenv("GSE_FUSED_UPDATE")) fuse = atoi(e) != 0;
            if (fuse) { sp.items_per_it -= sp.n_upd_items; sp.n_upd_items = 0; }
            plan->solve_grid = std::min(cap, sp.items_per_it);
            if (plan->max_ctas > 0) plan->solve_grid = std::min(plan->solve_grid, plan->max_ctas);
            plan->persistent = true;
        }
        for (auto& f : hp.fronts) if (f.kind == 3 && f.p > 0) ++plan->n_gamma_fronts;
    }
    CU(cudaDeviceSynchronize());
    plan->err.code = GSE_OK; plan->err.area = -1; plan->err.pivot = -1; plan->err.message[0] = 0;
    return GSE_OK;
}

void gse_plan_destroy(gse_plan* plan) { delete plan; }

// New weights / values on the same rows: staged through plan-owned pinned memory and copied on the
// plan's stream, so the call returns without waiting for the device and the next solve (same stream)
// sees the data.  which: 0 = z, 1 = w.
static int stage_rows(gse_plan* plan, int which, const double* src, double* dst_dev) {
    CU(cudaSetDevice(plan->device));
    const size_t bytes = sizeof(double) * plan->hp.n_rows;
    if (bytes == 0) return GSE_OK;
    if (!plan->h_stage[which]) {
        CU(cudaMallocHost(&plan->h_stage[which], bytes));
        CU(cudaEventCreateWithFlags(&plan->stage_done[which], cudaEventDisableTiming));
    } else {
        CU(cudaEventSynchronize(plan->stage_done[which]));      // the previous copy out of this buffer
    }
    memcpy(plan->h_stage[which], src, bytes);
    CU(cudaMemcpyAsync(dst_dev, plan->h_stage[which], bytes, cudaMemcpyHostToDevice, plan->stream));
    CU(cudaEventRecord(plan->stage_done[which], plan->stream));
    return GSE_OK;
}
// Same refresh straight from caller-owned PINNED host memory (cudaHostAlloc / torch pin_memory): one
// asynchronous copy per array on the plan's stream, no staging.  The buffers must stay unchanged until
// the next solve / iterate call has returned.
int gse_set_rows_pinned(gse_plan* plan, const double* z_pinned, const double* w_pinned) {
    CU(cudaSetDevice(plan->device));
    const size_t bytes = sizeof(double) * plan->hp.n_rows;
    double* w_dev = plan->z.ptr + plan->hp.n_rows;
    if (z_pinned && w_pinned == z_pinned + plan->hp.n_rows && bytes) {
        CU(cudaMemcpyAsync(plan->z.ptr, z_pinned, 2 * bytes, cudaMemcpyHostToDevice, plan->stream));
        return GSE_OK;
    }
    if (z_pinned && bytes) CU(cudaMemcpyAsync(plan->z.ptr, z_pinned, bytes, cudaMemcpyHostToDevice, plan->stream));
    if (w_pinned && bytes) CU(cudaMemcpyAsync(w_dev, w_pinned, bytes, cudaMemcpyHostToDevice, plan->stream));
    return GSE_OK;
}
int gse_set_weights(gse_plan* plan, const double* w) { return stage_rows(plan, 1, w, plan->z.ptr + plan->hp.n_rows); }
int gse_set_measurements(gse_plan* plan, const double* z) { return stage_rows(plan, 0, z, plan->z.ptr); }

int gse_check(gse_plan* plan) {
    CU(cudaSetDevice(plan->device));
    unsigned long long code = 0;
    CU(copy_sync(plan, &code, plan->flags.ptr + 1, sizeof code, cudaMemcpyDeviceToHost));
    if (code == ~0ull) return GSE_OK;
    CU(reset_failure_flag(plan));
    return decode_failure(plan, code);
}

int gse_iterate(gse_plan* plan, double* va, double* vm, double* delta_inf) {
    CU(cudaSetDevice(plan->device));
    int rc = ensure_graph(plan, va, vm);
    if (rc) return rc;
    CU(cudaGraphLaunch(plan->graph, plan->stream));
    CU(cudaStreamSynchronize(plan->stream));
    plan->launches_last = plan->launches_per_iter;
    if (plan->h_flags[1] != ~0ull) {
        unsigned long long code = plan->h_flags[1];
        reset_failure_flag(plan);
        return decode_failure(plan, code);
    }
    double dv; memcpy(&dv, &plan->h_flags[0], sizeof dv);
    if (delta_inf) *delta_inf = dv;
    return GSE_OK;
}

// One inner Gauss-Newton step of every owned area with the boundary state held fixed
// (reference solver.py:253-260: fused_accumulate -> numeric_refactor -> cache.solve(b_i) ->
// apply_interior_delta).  On the device: assembly, the interior fronts of the forward pass, the
// interior back-substitution with delta_x_Gamma = 0, and the state update of the interior
// variables only.  *delta_inf = max |delta x_i| of this step.
int gse_inner_step(gse_plan* plan, double* va, double* vm, double* delta_inf) {
    CU(cudaSetDevice(plan->device));
    cudaStream_t s = plan->stream;
    const HostProgram& hp = plan->hp;
    CU(cudaMemsetAsync(plan->flags.ptr, 0, sizeof(unsigned long long), s));
    enqueue_phase_assemble(plan, va, vm);
    enqueue_fwd(plan, 1);
    if (hp.n_gamma) CU(cudaMemsetAsync(plan->xsol.ptr + hp.gamma_base, 0, sizeof(double) * hp.n_gamma, s));
    enqueue_bwd(plan, 4);
    const int n_interior = (int)plan->upd_bus.n - hp.n_gamma;      // update list = interiors of every area, then x_Gamma
    launch_update(plan->upd_bus.ptr, plan->upd_quant.ptr, plan->upd_pos.ptr, n_interior, plan->xsol.ptr, va, vm, plan->flags.ptr, s);
    CU(cudaMemcpyAsync(plan->h_flags, plan->flags.ptr, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (plan->h_flags[1] != ~0ull) {
        unsigned long long code = plan->h_flags[1];
        reset_failure_flag(plan);
        return decode_failure(plan, code);
    }
    double dv; memcpy(&dv, &plan->h_flags[0], sizeof dv);
    if (delta_inf) *delta_inf = dv;
    return GSE_OK;
}

int gse_objective(gse_plan* plan, const double* va, const double* vm, double* j_out) {
    CU(cudaSetDevice(plan->device));
    launch_objective(plan->ep, plan->m_type.ptr, plan->m_target.ptr, plan->br_from.ptr, plan->br_to.ptr, plan->hp.n_rows, va, vm,
                     plan->obj_partial.ptr, plan->obj_partial.ptr + objective_blocks(plan->hp.n_rows), plan->stream);
    CU(cudaMemcpyAsync(plan->h_obj, plan->obj_partial.ptr + objective_blocks(plan->hp.n_rows), sizeof(double),
                       cudaMemcpyDeviceToHost, plan->stream));
    CU(cudaStreamSynchronize(plan->stream));
    *j_out = *plan->h_obj;
    return GSE_OK;
}

// The whole GN loop + objective in one cooperative launch; one 4.6 KB readback at the end.
static int solve_persistent(gse_plan* plan, const gse_config* cfg, int max_it, double* va, double* vm, gse_report* rep) {
    cudaStream_t s = plan->stream;
    SolveProg sp = plan->sp;
    sp.max_it = max_it; sp.tol = cfg->convergence_tol;
    if (sp.trace) CU(cudaMemsetAsync(sp.trace, 0, sizeof(unsigned long long) * 32 * (size_t)sp.items_per_it * 16, s));
    auto t0 = std::chrono::steady_clock::now();
    const size_t nb2 = sizeof(double) * (size_t)plan->hp.n_bus;
    const bool one_block = vm == va + plan->hp.n_bus;      // (va | vm) contiguous like the start state and the host block: one copy each way
    if (plan->io_init) {
        if (one_block) CU(cudaMemcpyAsync(va, plan->io_init, 2 * nb2, cudaMemcpyDeviceToDevice, s));
        else {
            CU(cudaMemcpyAsync(va, plan->io_init, nb2, cudaMemcpyDeviceToDevice, s));
            CU(cudaMemcpyAsync(vm, plan->io_init + plan->hp.n_bus, nb2, cudaMemcpyDeviceToDevice, s));
        }
    }
    cudaEventRecord(plan->ev[6], s);      // gpu_s: the loop itself (counter reset, launch, report readback), as gse_solve times it
    if (plan->linked) {
        // the sync block was cleared by gse_peer_solve_prepare BEFORE the ranks' barrier: a peer that starts
        // first may already be counting its area roots into it
        if (!plan->prepared) return fail(plan, GSE_E_INVALID, "peer-linked plan: call gse_peer_solve_prepare (then barrier the ranks) before gse_solve");
        plan->prepared = false;
    } else {
        CU(cudaMemsetAsync(plan->syncblk.ptr, 0, plan->sync_bytes, s));
    }
    CU(launch_solve(sp, plan->ep, plan->ft, va, vm, plan->solve_grid, plan->solve_smem, s, !plan->shares_device));
    CU(cudaMemcpyAsync(plan->h_blk, plan->syncblk.ptr, sizeof(unsigned long long) * kBlkWords, cudaMemcpyDeviceToHost, s));
    cudaEventRecord(plan->ev[7], s);
    if (plan->io_out) {
        if (one_block) CU(cudaMemcpyAsync(plan->io_out, va, 2 * nb2, cudaMemcpyDeviceToHost, s));
        else {
            CU(cudaMemcpyAsync(plan->io_out, va, nb2, cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(plan->io_out + plan->hp.n_bus, vm, nb2, cudaMemcpyDeviceToHost, s));
        }
    }
    CU(cudaStreamSynchronize(s));
    rep->loop_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    { float ms = 0; cudaEventElapsedTime(&ms, plan->ev[6], plan->ev[7]); rep->gpu_s = ms * 1e-3; }
    const unsigned long long* blk = plan->h_blk;
    const int32_t* res = reinterpret_cast<const int32_t*>(blk + kBlkResult);
    rep->iterations = res[0]; rep->converged = res[1];
    plan->launches_last = 1;
    for (int it = 0; it < rep->iterations && it < 64; ++it)
        memcpy(&rep->delta_inf[it], &blk[(plan->linked ? kBlkGDelta : kBlkDelta) + it], sizeof(double));
    if (plan->stamps) {
        // phase end stamps (globaltimer ns) per iteration: 0 eval, 1 accumulate, 2 local condense,
        // 3 boundary assemble, 4 boundary factor, 5 boundary back-substitution, 6 recovery, 7 update.
        // Phases overlap in the dataflow schedule; each is charged from the previous phase's end.
        unsigned long long start = blk[kBlkStamps];
        for (int it = 0; it < rep->iterations && it < 64; ++it) {
            const unsigned long long* st = blk + kBlkStamps + 1 + 8 * it;
            unsigned long long cur = start;
            auto take = [&](unsigned long long end) { double dt = end > cur ? (end - cur) * 1e-9 : 0.0; if (end > cur) cur = end; return dt; };
            rep->phase_s[0] += take(std::max(st[0], st[1]));
            rep->phase_s[1] += take(st[2]);
            rep->phase_s[2] += take(st[3]);
            rep->phase_s[3] += take(std::max(st[4], st[5]));
            rep->phase_s[4] += take(std::max(st[6], st[7]));
            start = std::max(cur, st[7]);
        }
    }
    if (blk[kBlkErr] != ~0ull) {
        reset_failure_flag(plan);
        return decode_failure(plan, blk[kBlkErr]);
    }
    memcpy(&rep->objective, &blk[kBlkObj], sizeof(double));
    if (plan->linked) rep->objective = std::nan("");      // J needs the merged state of all ranks: gse_objective afterwards
    return GSE_OK;
}

int gse_solve(gse_plan* plan, const gse_config* cfg, double* va, double* vm, gse_report* rep) {
    CU(cudaSetDevice(plan->device));
    memset(rep, 0, sizeof *rep);
    // the report carries 64 per-iteration norms / stamp blocks: longer loops go through gse_iterate (the
    // reference has no cap; the Python layer switches to that loop by itself)
    if (cfg->max_outer_iterations < 1 || cfg->max_outer_iterations > 64)
        return fail(plan, GSE_E_INVALID, "gse_solve: max_outer_iterations must be in [1, 64]; drive longer loops with gse_iterate");
    const int max_it = cfg->max_outer_iterations;
    const bool timed = cfg->time_phases != 0;
    // rank-sharded plans: the loop needs the exchanges -- inside the kernels once the ranks are linked, else the
    // caller's (gse_phase_*_async + collectives); a plain gse_solve would silently skip them
    if (plan->hp.world > 1 && !(plan->linked && !timed))
        return fail(plan, GSE_E_INVALID, plan->linked ? "gse_solve on a peer-linked plan: time_phases is not available (phases overlap across ranks)"
                                                      : "gse_solve on a rank-sharded plan: link the ranks first (gse_peer_link) or drive the phases (gse_phase_*_async)");
    if (!timed && plan->persistent) return solve_persistent(plan, cfg, max_it, va, vm, rep);
    if (!timed) { int rc = ensure_graph(plan, va, vm); if (rc) return rc; }
    plan->launches_last = 0;
    auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(plan->ev[6], plan->stream);
    int status = GSE_OK;
    for (int it = 1; it <= max_it; ++it) {
        if (timed) plan->launches_last += enqueue_iteration(plan, va, vm, true);
        else { CU(cudaGraphLaunch(plan->graph, plan->stream)); plan->launches_last += plan->launches_per_iter; }
        CU(cudaStreamSynchronize(plan->stream));
        if (timed)
            for (int ph = 0; ph < 5; ++ph) { float ms = 0; cudaEventElapsedTime(&ms, plan->ev[ph], plan->ev[ph + 1]); rep->phase_s[ph] += ms * 1e-3; }
        rep->iterations = it;
        if (plan->h_flags[1] != ~0ull) {
            unsigned long long code = plan->h_flags[1];
            reset_failure_flag(plan);
            status = decode_failure(plan, code);
            break;
        }
        double dv; memcpy(&dv, &plan->h_flags[0], sizeof dv);
        rep->delta_inf[it - 1] = dv;
        if (dv < cfg->convergence_tol) { rep->converged = 1; break; }
    }
    cudaEventRecord(plan->ev[7], plan->stream);
    cudaEventSynchronize(plan->ev[7]);
    rep->loop_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    { float ms = 0; cudaEventElapsedTime(&ms, plan->ev[6], plan->ev[7]); rep->gpu_s = ms * 1e-3; }
    if (status != GSE_OK) return status;
    return gse_objective(plan, va, vm, &rep->objective);
}

// gse_solve with the start state and the result transfer folded into the same enqueue: init_dev = (va | vm) start
// state on the device (2 n_bus doubles, e.g. the flat start kept resident) or NULL, out_pinned = pinned host buffer
// for the final (va | vm) or NULL.  One host synchronisation per solve on the persistent path; the other paths
// order the copies around the loop.
int gse_solve_io(gse_plan* plan, const gse_config* cfg, const double* init_dev, double* va, double* vm, double* out_pinned,
                 gse_report* rep) {
    CU(cudaSetDevice(plan->device));
    const bool fused = plan->persistent && !cfg->time_phases && cfg->max_outer_iterations >= 1 && cfg->max_outer_iterations <= 64
                       && (plan->hp.world == 1 || plan->linked);
    const size_t nb2 = sizeof(double) * (size_t)plan->hp.n_bus;
    if (fused) {
        plan->io_init = init_dev; plan->io_out = out_pinned;
        const int rc = gse_solve(plan, cfg, va, vm, rep);
        plan->io_init = nullptr; plan->io_out = nullptr;
        return rc;
    }
    if (init_dev) {
        CU(cudaMemcpyAsync(va, init_dev, nb2, cudaMemcpyDeviceToDevice, plan->stream));
        CU(cudaMemcpyAsync(vm, init_dev + plan->hp.n_bus, nb2, cudaMemcpyDeviceToDevice, plan->stream));
    }
    const int rc = gse_solve(plan, cfg, va, vm, rep);
    if (rc == GSE_OK && out_pinned) {
        CU(cudaMemcpyAsync(out_pinned, va, nb2, cudaMemcpyDeviceToHost, plan->stream));
        CU(cudaMemcpyAsync(out_pinned + plan->hp.n_bus, vm, nb2, cudaMemcpyDeviceToHost, plan->stream));
        CU(cudaStreamSynchronize(plan->stream));
    }
    return rc;
}

// ---- generic Schur-mode matrix plans (standalone linear algebra of reference linalg.py) ---------
// One "area" whose interior block G_ii and coupling G_ib are given by pattern; the forward pass of
// the multifrontal tree is numeric_refactor + schur_condense, the interior back-substitution is
// interior_recover / cache.solve.  Built from a synthetic one-area problem without measurement rows
// (every variable is the magnitude of its own bus), as a non-coordinator rank so that the tree stops
// at the area root (= S_b | b_hat).
int gse_matrix_plan_create(int32_t n_i, int32_t n_b, const int32_t* ii_ptr, const int32_t* ii_idx, const int32_t* ib_ptr,
                           const int32_t* ib_idx, const gse_options* opt, gse_plan** out) {
    if (n_i < 0 || n_b < 0 || n_i + n_b == 0 || !out || (n_i && (!ii_ptr || !ii_idx))) return GSE_E_INVALID;
    const int n = n_i + n_b;
    std::vector<int32_t> zero1{0, 0}, y_ptr(n + 1, 0), aob(n, 0), im_ptr{0, n_i}, bm_ptr{0, n_b}, sel_ptr{0, n_b};
    std::vector<int32_t> im_bus(n_i), bm_bus(n_b), sel(n_b), gbus(n_b), gq(n_b, 1);
    for (int i = 0; i < n_i; ++i) im_bus[i] = i;
    for (int j = 0; j < n_b; ++j) { bm_bus[j] = n_i + j; sel[j] = j; gbus[j] = n_i + j; }
    int32_t none = 0; double nonef = 0.0;
    gse_problem_desc d{};
    d.n_bus = n; d.n_branch = 0; d.n_rows = 0; d.n_areas = 1; d.n_gamma = n_b; d.slack = -1;
    d.y_ptr = y_ptr.data(); d.y_idx = &none; d.y_g = &nonef; d.y_b = &nonef;
    d.br_from = &none; d.br_to = &none; d.br_y = &nonef;
    d.m_type = &none; d.m_target = &none; d.m_z = &nonef; d.m_w = &nonef;
    d.area_of_bus = aob.data();
    d.ia_ptr = zero1.data(); d.ia_bus = &none; d.im_ptr = im_ptr.data(); d.im_bus = im_bus.data();
    d.ba_ptr = zero1.data(); d.ba_bus = &none; d.bm_ptr = bm_ptr.data(); d.bm_bus = bm_bus.data();
    d.sel_ptr = sel_ptr.data(); d.sel = sel.data(); d.gamma_bus = gbus.data(); d.gamma_quant = gq.data();
    BuildOptions bo;
    bo.ext_pattern = true;
    bo.ext_ii_ptr.assign(ii_ptr ? ii_ptr : zero1.data(), (ii_ptr ? ii_ptr : zero1.data()) + n_i + 1);
    bo.ext_ii_idx.assign(ii_idx, ii_idx + bo.ext_ii_ptr[n_i]);
    if (ib_ptr) { bo.ext_ib_ptr.assign(ib_ptr, ib_ptr + n_i + 1); bo.ext_ib_idx.assign(ib_idx, ib_idx + ib_ptr[n_i]); }
    else bo.ext_ib_ptr.assign(n_i + 1, 0);
    for (int u = 0; u < n_i; ++u) {
        for (int p = bo.ext_ii_ptr[u]; p < bo.ext_ii_ptr[u + 1]; ++p)
            if (bo.ext_ii_idx[p] < 0 || bo.ext_ii_idx[p] >= n_i || (p > bo.ext_ii_ptr[u] && bo.ext_ii_idx[p] <= bo.ext_ii_idx[p - 1])) return GSE_E_INVALID;
        for (int p = bo.ext_ib_ptr[u]; p < bo.ext_ib_ptr[u + 1]; ++p)
            if (bo.ext_ib_idx[p] < 0 || bo.ext_ib_idx[p] >= n_b || (p > bo.ext_ib_ptr[u] && bo.ext_ib_idx[p] <= bo.ext_ib_idx[p - 1])) return GSE_E_INVALID;
    }
    gse_options o{};
    if (opt) o = *opt;
    o.rank = 1; o.world = 2;                  // not the coordinator: no boundary factorisation
    const int32_t owner = 1;
    o.area_rank = &owner;
    o.persistent = 2;
    return create_plan(&d, &o, bo, out);
}

// values in the reference's block layout (AreaNormalBlocks); nullptr = zeros
int gse_matrix_set_values(gse_plan* plan, const double* data_ii, const double* data_ib, const double* g_bb, const double* b_i,
                          const double* b_b) {
    const HostProgram& hp = plan->hp;
    if (hp.gval_src.size() != (size_t)hp.n_gval) return fail(plan, GSE_E_INVALID, "not a matrix plan");
    CU(cudaSetDevice(plan->device));
    const int64_t nii = (int64_t)hp.ii_idx[0].size(), nib = (int64_t)hp.ib_idx[0].size(), nb = hp.area_nb[0], ni = hp.area_ni[0];
    const int64_t o_ib = nii, o_bb = o_ib + nib, o_bi = o_bb + nb * nb, o_bbv = o_bi + ni;
    std::vector<double> g((size_t)hp.n_gval, 0.0);
    for (size_t e = 0; e < g.size(); ++e) {
        const int64_t s = hp.gval_src[e];
        if (s < 0) continue;
        const double* src = s < o_ib ? data_ii : s < o_bb ? data_ib : s < o_bi ? g_bb : s < o_bbv ? b_i : b_b;
        const int64_t off = s < o_ib ? 0 : s < o_bb ? o_ib : s < o_bi ? o_bb : s < o_bbv ? o_bi : o_bbv;
        if (src) g[e] = src[s - off];
    }
    CU(copy_sync(plan, plan->gval.ptr, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice));
    return GSE_OK;
}

// numeric_refactor + schur_condense: the forward pass over the interior fronts and the area root
int gse_matrix_condense(gse_plan* plan) {
    CU(cudaSetDevice(plan->device));
    enqueue_fwd(plan, 1);
    return gse_check(plan);
}

// interior_recover: dx_i = G_ii^-1 (b_i - G_ib dx_b) from the factor of the last gse_matrix_condense
int gse_matrix_recover(gse_plan* plan, const double* dx_b, double* dx_i) {
    const HostProgram& hp = plan->hp;
    CU(cudaSetDevice(plan->device));
    if (hp.n_gamma) {
        if (dx_b) CU(copy_sync(plan, plan->xsol.ptr + hp.gamma_base, dx_b, sizeof(double) * hp.n_gamma, cudaMemcpyHostToDevice));
        else CU(cudaMemsetAsync(plan->xsol.ptr + hp.gamma_base, 0, sizeof(double) * hp.n_gamma, plan->stream));
    }
    enqueue_bwd(plan, 4);
    CU(cudaStreamSynchronize(plan->stream));
    return gse_area_delta(plan, 0, dx_i);
}

// SparseCholeskyCache.forward / .backward (linalg.py:340-383) in THIS factor's coordinates: perm[e] = original
// index of elimination position e (the reference's cache.perm).  forward: y = L^-1 P b is the right-hand-side row
// every front carries through the factorisation (read after gse_matrix_set_values(b_i = b) + gse_matrix_condense).
int gse_matrix_perm(const gse_plan* plan, int32_t* perm) {
    const HostProgram& hp = plan->hp;
    if (hp.gval_src.size() != (size_t)hp.n_gval) return GSE_E_INVALID;
    for (int e = 0; e < hp.area_ni[0]; ++e) perm[e] = hp.perm_orig[hp.area_base[0] + e];
    return GSE_OK;
}
int gse_matrix_forward_get(gse_plan* plan, double* y) {
    const HostProgram& hp = plan->hp;
    if (hp.gval_src.size() != (size_t)hp.n_gval) return fail(plan, GSE_E_INVALID, "not a matrix plan");
    CU(cudaSetDevice(plan->device));
    for (const Front& f : hp.fronts) {
        if (f.kind != 0 || f.p == 0) continue;
        // pivots of a front are consecutive elimination positions; its solved right-hand side is row p + u of the panel
        CU(cudaMemcpyAsync(y + (f.rows[0] - hp.area_base[0]), plan->lbuf.ptr + f.l_off + (size_t)(f.p + f.u1 - 1) * f.p,
                           sizeof(double) * f.p, cudaMemcpyDeviceToHost, plan->stream));
    }
    CU(cudaStreamSynchronize(plan->stream));
    return GSE_OK;
}
// backward: x = P^T L^-T y with the factor of the last gse_matrix_condense (the boundary increment held at zero)
int gse_matrix_backward(gse_plan* plan, const double* y, double* x) {
    const HostProgram& hp = plan->hp;
    if (hp.gval_src.size() != (size_t)hp.n_gval) return fail(plan, GSE_E_INVALID, "not a matrix plan");
    CU(cudaSetDevice(plan->device));
    for (const Front& f : hp.fronts) {
        if (f.kind != 0 || f.p == 0) continue;
        CU(cudaMemcpyAsync(plan->lbuf.ptr + f.l_off + (size_t)(f.p + f.u1 - 1) * f.p, y + (f.rows[0] - hp.area_base[0]),
                           sizeof(double) * f.p, cudaMemcpyHostToDevice, plan->stream));
    }
    CU(cudaStreamSynchronize(plan->stream));      // (y is pageable caller memory)
    return gse_matrix_recover(plan, nullptr, x);
}

// assemble_boundary (solver.py:106-119): S_Gamma[sel, sel] += S_b, b_Gamma[sel] += b_hat, areas in
// ascending order.  Host in / host out; the sums run on the device in area order per entry.
int gse_assemble_boundary(int32_t n_gamma, int32_t n_areas, const int32_t* sel_ptr, const int32_t* sel, const double* s_b,
                          const double* b_hat, double* s_gamma, double* b_gamma) {
    if (n_gamma < 0 || n_areas < 0) return GSE_E_INVALID;
    if (n_gamma == 0) return GSE_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return GSE_E_NO_DEVICE;
    std::vector<int32_t> inv((size_t)n_areas * n_gamma, -1);
    std::vector<int64_t> off(n_areas + 1, 0);
    for (int a = 0; a < n_areas; ++a) {
        const int nb = sel_ptr[a + 1] - sel_ptr[a];
        off[a + 1] = off[a] + (int64_t)nb * nb;
        for (int i = 0; i < nb; ++i) {
            const int s = sel[sel_ptr[a] + i];
            if (s < 0 || s >= n_gamma) return GSE_E_INVALID;
            inv[(size_t)a * n_gamma + s] = i;
        }
    }
    DevBuf<int32_t> d_inv, d_selptr; DevBuf<int64_t> d_off; DevBuf<double> d_sb, d_bh, d_sg, d_bg;
    cudaError_t e = cudaSuccess;
    auto ok = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
    ok(d_inv.upload(inv)); ok(d_off.upload(off)); ok(d_selptr.upload(std::vector<int32_t>(sel_ptr, sel_ptr + n_areas + 1)));
    ok(d_sb.upload(std::vector<double>(s_b, s_b + off[n_areas]))); ok(d_bh.upload(std::vector<double>(b_hat, b_hat + sel_ptr[n_areas])));
    ok(d_sg.alloc((size_t)n_gamma * n_gamma)); ok(d_bg.alloc(n_gamma));
    if (e == cudaSuccess) {
        launch_assemble_boundary(n_gamma, n_areas, d_inv.ptr, d_off.ptr, d_selptr.ptr, d_sb.ptr, d_bh.ptr, d_sg.ptr, d_bg.ptr, nullptr);
        ok(cudaMemcpy(s_gamma, d_sg.ptr, sizeof(double) * (size_t)n_gamma * n_gamma, cudaMemcpyDeviceToHost));
        ok(cudaMemcpy(b_gamma, d_bg.ptr, sizeof(double) * n_gamma, cudaMemcpyDeviceToHost));
    }
    d_inv.release(); d_off.release(); d_selptr.release(); d_sb.release(); d_bh.release(); d_sg.release(); d_bg.release();
    return e == cudaSuccess ? GSE_OK : GSE_E_CUDA;
}

// ---- phase-level entry points ------------------------------------------------------------------
int gse_phase_assemble(gse_plan* plan, const double* va, const double* vm) {
    CU(cudaSetDevice(plan->device));
    if (!plan->hp.ref_program_built) {      // the reference-layout program is only needed here: built on first use
        build_reference_program(plan->hp);
        CU(plan->racc_ptr.upload(plan->hp.racc_ptr)); CU(plan->racc_a.upload(plan->hp.racc_a)); CU(plan->racc_b.upload(plan->hp.racc_b));
        CU(plan->refval.alloc(plan->hp.n_ref_vals));
        CU(cudaDeviceSynchronize());          // the uploads ran on the legacy stream, the kernels below on the plan's
    }
    enqueue_phase_assemble(plan, va, vm);
    // reference-layout blocks for component parity (same slot values, second destination map)
    launch_accumulate(plan->racc_ptr.ptr, plan->racc_a.ptr, plan->racc_b.ptr, plan->val.ptr, plan->refval.ptr,
                      (int64_t)plan->hp.n_ref_vals, plan->stream);
    CU(cudaStreamSynchronize(plan->stream));
    return GSE_OK;
}
int gse_phase_condense(gse_plan* plan) {
    CU(cudaSetDevice(plan->device));
    enqueue_fwd(plan, 1);
    return gse_check(plan);
}
int gse_phase_boundary(gse_plan* plan) {
    CU(cudaSetDevice(plan->device));
    if (!plan->coordinator) return GSE_OK;
    enqueue_fwd(plan, 2); enqueue_fwd(plan, 5); enqueue_fwd(plan, 3); enqueue_bwd(plan, 3);
    return gse_check(plan);
}
int gse_phase_recover(gse_plan* plan, double* va, double* vm, double* delta_inf) {
    CU(cudaSetDevice(plan->device));
    CU(cudaMemsetAsync(plan->flags.ptr, 0, sizeof(unsigned long long), plan->stream));
    enqueue_bwd(plan, 4);
    enqueue_update(plan, va, vm);
    CU(cudaMemcpyAsync(plan->h_flags, plan->flags.ptr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, plan->stream));
    CU(cudaStreamSynchronize(plan->stream));
    double dv; memcpy(&dv, &plan->h_flags[0], sizeof dv);
    if (delta_inf) *delta_inf = dv;
    CU(copy_sync(plan, plan->status.ptr, &dv, sizeof dv, cudaMemcpyHostToDevice));
    return GSE_OK;
}

// ---- asynchronous phases (multi-GPU driver): enqueue only, no host synchronisation ----------------
// With gse_options.stream = the caller's stream, the collectives the caller enqueues on that stream
// (NCCL send/recv of the exchange segments, broadcast of delta_x_Gamma, MAX all-reduce of the status)
// are ordered with the phases by the stream itself; the host synchronises once per iteration, when it
// reads the reduced status.
int gse_phase_local_async(gse_plan* plan, const double* va, const double* vm) {
    CU(cudaSetDevice(plan->device));
    plan->launches_last = enqueue_phase_assemble(plan, va, vm);      // launches of this iteration (gse_plan_stats[0])
    plan->launches_last += enqueue_fwd(plan, 1);
    return GSE_OK;
}
int gse_phase_boundary_async(gse_plan* plan) {
    CU(cudaSetDevice(plan->device));
    if (!plan->coordinator) return GSE_OK;
    plan->launches_last += enqueue_fwd(plan, 2) + enqueue_fwd(plan, 3) + enqueue_bwd(plan, 3);
    return GSE_OK;
}
// interiors + state update; then status[0] = max |dx| of this rank, status[1] = 1 if any factorisation of
// this rank failed since the last gse_check (else 0) -- two doubles for one MAX all-reduce
int gse_phase_recover_async(gse_plan* plan, double* va, double* vm) {
    CU(cudaSetDevice(plan->device));
    CU(cudaMemsetAsync(plan->flags.ptr, 0, sizeof(unsigned long long), plan->stream));
    plan->launches_last += enqueue_bwd(plan, 4) + enqueue_update(plan, va, vm) + 1;
    launch_status(plan->flags.ptr, plan->status.ptr, plan->stream);
    return GSE_OK;
}

// ---- readback ------------------------------------------------------------------------------------
int gse_area_dims(const gse_plan* plan, int32_t a, int32_t* out) {
    const HostProgram& hp = plan->hp;
    if (a < 0 || a >= hp.n_areas) return GSE_E_INVALID;
    out[0] = hp.area_ni[a]; out[1] = hp.area_nb[a];
    out[2] = (int)hp.ii_idx[a].size(); out[3] = (int)hp.ib_idx[a].size();
    int nfr = 0; int64_t lnz = 0;
    for (auto& f : hp.fronts) if (f.area == a && f.kind == 0) { ++nfr; lnz += (int64_t)(f.p + f.u1 - 1) * f.p; }
    out[4] = (int32_t)hp.tmpl_rows[a].size(); out[5] = (int32_t)hp.tmpl_slot_var[a].size(); out[6] = nfr; out[7] = (int32_t)std::min<int64_t>(lnz, 2147483647);
    return GSE_OK;
}
int gse_area_pattern(const gse_plan* plan, int32_t a, int32_t* ii_ptr, int32_t* ii_idx, int32_t* ib_ptr, int32_t* ib_idx) {
    const HostProgram& hp = plan->hp;
    if (a < 0 || a >= hp.n_areas) return GSE_E_INVALID;
    memcpy(ii_ptr, hp.ii_ptr[a].data(), hp.ii_ptr[a].size() * 4); memcpy(ii_idx, hp.ii_idx[a].data(), hp.ii_idx[a].size() * 4);
    memcpy(ib_ptr, hp.ib_ptr[a].data(), hp.ib_ptr[a].size() * 4); memcpy(ib_idx, hp.ib_idx[a].data(), hp.ib_idx[a].size() * 4);
    return GSE_OK;
}
int gse_area_blocks(gse_plan* plan, int32_t a, double* data_ii, double* data_ib, double* g_bb, double* b_i, double* b_b) {
    const HostProgram& hp = plan->hp;
    if (a < 0 || a >= hp.n_areas || !hp.owned[a]) return fail(plan, GSE_E_INVALID, "area not owned by this plan");
    if (!plan->refval.ptr) return fail(plan, GSE_E_INVALID, "gse_area_blocks needs a preceding gse_phase_assemble");
    CU(cudaSetDevice(plan->device));
    const size_t nii = hp.ii_idx[a].size(), nib = hp.ib_idx[a].size(), nb = hp.area_nb[a], ni = hp.area_ni[a];
    const double* base = plan->refval.ptr + hp.ref_off[a];
    CU(copy_sync(plan, data_ii, base, nii * 8, cudaMemcpyDeviceToHost));
    CU(copy_sync(plan, data_ib, base + nii, nib * 8, cudaMemcpyDeviceToHost));
    CU(copy_sync(plan, g_bb, base + nii + nib, nb * nb * 8, cudaMemcpyDeviceToHost));
    CU(copy_sync(plan, b_i, base + nii + nib + nb * nb, ni * 8, cudaMemcpyDeviceToHost));
    CU(copy_sync(plan, b_b, base + nii + nib + nb * nb + ni, nb * 8, cudaMemcpyDeviceToHost));
    return GSE_OK;
}
// The area's materialised template layer after gse_phase_assemble (the reference's explicit oracle path,
// assembly.py:531-560: JacobianTriplets): per owned row k its global row id, slot range and local variable per slot
// (reference numbering: interior x_i slots, then n_i + local boundary slot), the partial dh/dx per slot as the
// template kernel wrote it, and the weighted residual w (z - h) per row.
int gse_area_templates(gse_plan* plan, int32_t a, int32_t* rows, int32_t* slot_ptr, int32_t* slot_var, double* g, double* wr) {
    const HostProgram& hp = plan->hp;
    if (a < 0 || a >= hp.n_areas || !hp.owned[a]) return fail(plan, GSE_E_INVALID, "area not owned by this plan");
    CU(cudaSetDevice(plan->device));
    const size_t nr = hp.tmpl_rows[a].size(), ns = hp.tmpl_slot_var[a].size();
    for (size_t k = 0; k < nr; ++k) rows[k] = hp.tmpl_rows[a][k];
    for (size_t k = 0; k <= nr; ++k) slot_ptr[k] = hp.tmpl_slot_ptr[a][k];
    for (size_t s = 0; s < ns; ++s) slot_var[s] = hp.tmpl_slot_var[a][s];
    std::vector<double> pairs(2 * ns), allwr((size_t)hp.n_rows);
    CU(copy_sync(plan, pairs.data(), plan->val.ptr + 2 * hp.tmpl_slot_base[a], pairs.size() * 8, cudaMemcpyDeviceToHost));
    CU(copy_sync(plan, allwr.data(), plan->val.ptr + 2 * hp.n_slots, allwr.size() * 8, cudaMemcpyDeviceToHost));
    for (size_t s = 0; s < ns; ++s) g[s] = pairs[2 * s];
    for (size_t k = 0; k < nr; ++k) wr[k] = allwr[(size_t)hp.tmpl_rows[a][k]];
    return GSE_OK;
}
// packed lower (rows in front order) -> full symmetric in the caller's order; pos[i] = front row of item i
static int unpack_lower(gse_plan* plan, const Front& f, int n, const std::vector<int>& pos, double* full, double* rhs) {
    std::vector<double> packed((size_t)f.u1 * (f.u1 + 1) / 2);
    cudaError_t e = copy_sync(plan, packed.data(), plan->ubuf.ptr + f.u_off, packed.size() * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(plan, GSE_E_CUDA, cudaGetErrorString(e));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int qi = std::max(pos[i], pos[j]), qj = std::min(pos[i], pos[j]);
            full[(size_t)i * n + j] = packed[(size_t)qi * (qi + 1) / 2 + qj];
        }
    for (int j = 0; j < n; ++j) rhs[j] = packed[(size_t)n * (n + 1) / 2 + pos[j]];
    return GSE_OK;
}
int gse_area_schur(gse_plan* plan, int32_t a, double* s_b, double* b_hat) {
    const HostProgram& hp = plan->hp;
    if (a < 0 || a >= hp.n_areas) return GSE_E_INVALID;
    CU(cudaSetDevice(plan->device));
    return unpack_lower(plan, hp.fronts[hp.area_root[a]], hp.area_nb[a], hp.area_bpos[a], s_b, b_hat);
}
int gse_boundary_system(gse_plan* plan, double* s_gamma, double* b_gamma, double* dx_gamma) {
    const HostProgram& hp = plan->hp;
    CU(cudaSetDevice(plan->device));
    if (hp.n_gamma == 0) return GSE_OK;
    if (hp.gamma_root < 0) return fail(plan, GSE_E_INVALID, "boundary system lives on the coordinator rank");
    int rc = unpack_lower(plan, hp.fronts[hp.gamma_root], hp.n_gamma, hp.gamma_sparse ? hp.gamma_epos : std::vector<int>(hp.gamma_epos), s_gamma, b_gamma);
    if (rc) return rc;
    CU(copy_sync(plan, dx_gamma, plan->xsol.ptr + hp.gamma_base, hp.n_gamma * 8, cudaMemcpyDeviceToHost));
    return GSE_OK;
}
int gse_area_delta(gse_plan* plan, int32_t a, double* dx_i) {
    const HostProgram& hp = plan->hp;
    if (a < 0 || a >= hp.n_areas || !hp.owned[a]) return fail(plan, GSE_E_INVALID, "area not owned by this plan");
    CU(cudaSetDevice(plan->device));
    const int ni = hp.area_ni[a];
    std::vector<double> x(ni);
    CU(copy_sync(plan, x.data(), plan->xsol.ptr + hp.area_base[a], ni * 8, cudaMemcpyDeviceToHost));
    for (int e = 0; e < ni; ++e) dx_i[hp.perm_orig[hp.area_base[a] + e]] = x[e];
    return GSE_OK;
}
int gse_set_boundary_delta(gse_plan* plan, const double* dx_gamma) {
    CU(cudaSetDevice(plan->device));
    CU(copy_sync(plan, plan->xsol.ptr + plan->hp.gamma_base, dx_gamma, plan->hp.n_gamma * 8, cudaMemcpyHostToDevice));
    return GSE_OK;
}

// ---- peer-linked multi-rank solve: the exchanges inside the persistent kernel, over peer memory --------------
// (reference solver.py:277-298 gather of the Schur blocks, 318-326 broadcast of delta_x_Gamma, 328-338 the
// convergence scalar)
static cudaError_t allocation_base(const void* p, unsigned long long* base) {
    typedef int (*range_fn)(unsigned long long*, size_t*, unsigned long long);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &qr);
    if (e != cudaSuccess) return e;
    if (!fn || qr != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
    size_t size = 0;
    return reinterpret_cast<range_fn>(fn)(base, &size, (unsigned long long)(uintptr_t)p) == 0 ? cudaSuccess : cudaErrorInvalidValue;
}

int gse_peer_info_get(gse_plan* plan, gse_peer_info* out) {
    CU(cudaSetDevice(plan->device));
    memset(out, 0, sizeof *out);
    const HostProgram& hp = plan->hp;
    out->rank = hp.rank; out->world = hp.world; out->device = plan->device;
    out->n_gamma_fronts = plan->n_gamma_fronts;
    out->pid = (int64_t)getpid();
    unsigned long long* blk = plan->syncblk.ptr;
    const void* ptrs[3] = {plan->ubuf.ptr, plan->xsol.ptr, blk};
    out->ubuf = (uint64_t)(uintptr_t)plan->ubuf.ptr; out->xsol = (uint64_t)(uintptr_t)plan->xsol.ptr;
    out->sync = (uint64_t)(uintptr_t)blk;
    for (int k = 0; k < 3; ++k) {
        unsigned long long base = 0;
        CU(allocation_base(ptrs[k], &base));
        out->ipc_off[k] = (int64_t)((unsigned long long)(uintptr_t)ptrs[k] - base);
        cudaIpcMemHandle_t h;
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        CU(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
        memcpy(out->ipc[k], &h, 64);
    }
    return GSE_OK;
}

int gse_peer_link(gse_plan* plan, const gse_peer_info* all) {
    CU(cudaSetDevice(plan->device));
    const HostProgram& hp = plan->hp;
    const int world = hp.world, rank = hp.rank;
    if (world < 2) return fail(plan, GSE_E_INVALID, "gse_peer_link: the plan is not rank-sharded (world < 2)");
    if (world > kMaxPeers) return fail(plan, GSE_E_INVALID, "gse_peer_link: at most 8 ranks (one node); larger worlds use the collective driver");
    SolveProg& sp = plan->sp;
    if (sp.items_per_it <= 0 || sp.n_upd_items <= 0) return fail(plan, GSE_E_INVALID, "gse_peer_link: this rank has no work items");
    PeerLink lk{};
    lk.rank = rank; lk.world = world;
    const int64_t pid = (int64_t)getpid();
    for (int q = 0; q < world; ++q) {
        const gse_peer_info& pi = all[q];
        if (pi.rank != q || pi.world != world) return fail(plan, GSE_E_INVALID, "gse_peer_link: peer records must be ordered by rank and share the world size");
        unsigned char* base[3];
        if (q == rank || pi.pid == pid) {
            // same address space (this rank, or rank plans that share a process): the device addresses as they are
            base[0] = (unsigned char*)(uintptr_t)pi.ubuf; base[1] = (unsigned char*)(uintptr_t)pi.xsol; base[2] = (unsigned char*)(uintptr_t)pi.sync;
            if (q != rank && pi.device == plan->device) plan->shares_device = true;
            if (pi.device != plan->device) {
                cudaError_t e = cudaDeviceEnablePeerAccess(pi.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) return fail(plan, GSE_E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
            }
        } else {
            for (int k = 0; k < 3; ++k) {
                cudaIpcMemHandle_t h;
                memcpy(&h, pi.ipc[k], 64);
                void* mapped = nullptr;
                CU(cudaIpcOpenMemHandle(&mapped, h, cudaIpcMemLazyEnablePeerAccess));
                plan->ipc_opened.push_back(mapped);
                base[k] = (unsigned char*)mapped + pi.ipc_off[k];
            }
        }
        unsigned long long* blk = reinterpret_cast<unsigned long long*>(base[2]);
        lk.xsol[q] = reinterpret_cast<double*>(base[1]);
        lk.ctr[q] = reinterpret_cast<unsigned*>(blk + kBlkWords);
        lk.gdelta[q] = blk + kBlkGDelta;
        lk.gerr[q] = blk + kBlkGErr;
        if (q == 0) {
            lk.root_ctr = lk.ctr[0];
            lk.n_gamma_fronts = pi.n_gamma_fronts;
            plan->ft.ubuf_root = rank == 0 ? nullptr : reinterpret_cast<double*>(base[0]);
        }
    }
    sp.lk = lk;
    // all ranks run the persistent kernel; the state update stays in its own items (they also refresh this
    // rank's replica of the boundary state, and the last one publishes the rank's norm)
    const int cap = solve_kernel_max_ctas(plan->solve_smem, plan->device);
    if (cap <= 0) return fail(plan, GSE_E_CUDA, "persistent solve kernel does not fit this device");
    plan->solve_grid = std::min(cap, sp.items_per_it);
    if (plan->max_ctas > 0) plan->solve_grid = std::min(plan->solve_grid, plan->max_ctas);
    plan->persistent = true; plan->linked = true; plan->prepared = false;
    return GSE_OK;
}

int gse_peer_solve_prepare(gse_plan* plan) {
    CU(cudaSetDevice(plan->device));
    if (!plan->linked) return fail(plan, GSE_E_INVALID, "gse_peer_solve_prepare: the plan is not peer-linked");
    CU(cudaMemsetAsync(plan->syncblk.ptr, 0, plan->sync_bytes, plan->stream));
    CU(cudaStreamSynchronize(plan->stream));
    plan->prepared = true;
    return GSE_OK;
}

double* gse_exchange_buffer_dev(gse_plan* plan, int64_t* n) { if (n) *n = plan->hp.xchg_len; return plan->ubuf.ptr + plan->hp.xchg_off; }
int gse_exchange_offsets(const gse_plan* plan, int64_t* off) {
    for (size_t i = 0; i < plan->hp.xchg_area_off.size(); ++i) off[i] = plan->hp.xchg_area_off[i];
    return GSE_OK;
}
double* gse_boundary_delta_dev(gse_plan* plan) { return plan->xsol.ptr + plan->hp.gamma_base; }
double* gse_status_dev(gse_plan* plan) { return plan->status.ptr; }

void* gse_stream(gse_plan* plan) { return (void*)plan->stream; }

// Debug: per-task phase clocks of the front kernel (8 clock64 stamps per task) of the next launches.
int gse_debug_task_clocks(gse_plan* plan, int enable, long long* out, int64_t max_n) {
    CU(cudaSetDevice(plan->device));
    if (enable) {
        if (!plan->tbuf.ptr) CU(plan->tbuf.alloc(plan->tasks.n * 32 + 32));
        plan->ft.tbuf = plan->tbuf.ptr;
        if (plan->graph) { cudaGraphExecDestroy(plan->graph); plan->graph = nullptr; }
        return (int)plan->tasks.n;
    }
    if (out && plan->tbuf.ptr) CU(cudaMemcpy(out, plan->tbuf.ptr, sizeof(long long) * std::min<int64_t>(max_n, plan->tasks.n * 32), cudaMemcpyDeviceToHost));
    plan->ft.tbuf = nullptr;
    if (plan->graph) { cudaGraphExecDestroy(plan->graph); plan->graph = nullptr; }
    return (int)plan->tasks.n;
}

// One outer iteration with a CUDA event around every launch (warm, ungraphed): per-launch device
// time in microseconds.  kind: 0 eval, 1 accumulate, 2 front tasks, 3 backward, 4 state update.
int gse_profile_iteration(gse_plan* plan, double* va, double* vm, int32_t max_n, int32_t* kind, int32_t* phase,
                          int32_t* ctas, double* usec) {
    CU(cudaSetDevice(plan->device));
    std::vector<cudaEvent_t> evs;
    std::vector<int> k, ph, ct;
    auto mark = [&]() { cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, plan->stream); evs.push_back(e); };
    cudaMemsetAsync(plan->flags.ptr, 0, sizeof(unsigned long long), plan->stream);
    mark();
    launch_eval(plan->ep, va, vm, plan->stream); mark(); k.push_back(0); ph.push_back(0); ct.push_back((plan->ep.n_vm + plan->ep.n_fl + plan->ep.n_inj + 127) / 128);
    launch_accumulate_staged(plan->ap, plan->stream);
    mark(); k.push_back(1); ph.push_back(0); ct.push_back(plan->ap.n_items);
    for (int phs : {1, 2, 3})
        for (auto& L : plan->fwd) {
            if (L.phase != phs) continue;
            launch_front_tasks(L.pclass, plan->ft, plan->tasks.ptr + L.first, L.count, L.smem, plan->gval.ptr, plan->lbuf.ptr, plan->ubuf.ptr,
                               plan->flags.ptr + 1, plan->stream);
            mark(); k.push_back(2); ph.push_back(phs); ct.push_back(L.count);
        }
    for (int phs : {3, 4})
        for (auto& B : plan->bwd) {
            if (B.phase != phs) continue;
            launch_backward(plan->ft, plan->btasks.ptr + B.first, B.count, plan->lbuf.ptr, plan->xsol.ptr, plan->bpart.ptr, plan->bcnt.ptr, plan->stream);
            mark(); k.push_back(3); ph.push_back(phs); ct.push_back(B.count);
        }
    enqueue_update(plan, va, vm); mark(); k.push_back(4); ph.push_back(4); ct.push_back((int)(plan->upd_bus.n + 255) / 256);
    CU(cudaStreamSynchronize(plan->stream));
    int n = (int)k.size();
    for (int i = 0; i < n && i < max_n; ++i) {
        float ms = 0; cudaEventElapsedTime(&ms, evs[i], evs[i + 1]);
        kind[i] = k[i]; phase[i] = ph[i]; ctas[i] = ct[i]; usec[i] = ms * 1e3;
    }
    for (auto e : evs) cudaEventDestroy(e);
    return n;
}

// Debug: per-item stamps of the persistent kernel.  enable=1 arms tracing for the next solves (first
// 16 iterations); enable=0 copies [items][16] words (pull, originals ready, children ready, end,
// smid | cta << 32, ..., then the 8 phase stamps of a front task) to out and disarms.  Returns the items per iteration.
int gse_debug_trace(gse_plan* plan, int enable, unsigned long long* out, int64_t max_words) {
    CU(cudaSetDevice(plan->device));
    const size_t words = 32 * (size_t)plan->sp.items_per_it * 16;
    if (enable) {
        if (!plan->trace.ptr) CU(plan->trace.alloc(words));
        plan->sp.trace = plan->trace.ptr;
        return plan->sp.items_per_it;
    }
    if (out && plan->trace.ptr) CU(cudaMemcpy(out, plan->trace.ptr, sizeof(unsigned long long) * std::min<size_t>(max_words, words), cudaMemcpyDeviceToHost));
    plan->sp.trace = nullptr;
    return plan->sp.items_per_it;
}
// Debug: arm the watchdog record of the persistent kernel.  buf = host memory from cudaHostAlloc(mapped) with
// 4 words per CTA ({counter address, target, value seen, 1} of a wait that timed out), ms = watchdog period.
// out[0..2] = device addresses of this plan's counter block, update storage, solution vector (to decode records).
int gse_debug_watchdog(gse_plan* plan, unsigned long long** buf, int32_t ms, uint64_t* out) {
    CU(cudaSetDevice(plan->device));
    static unsigned long long* host = nullptr;
    if (!host) { CU(cudaHostAlloc(&host, sizeof(unsigned long long) * 4 * 1024, cudaHostAllocMapped)); memset(host, 0, sizeof(unsigned long long) * 4 * 1024); }
    unsigned long long* dev = nullptr;
    CU(cudaHostGetDevicePointer(&dev, host, 0));
    CU(solve_kernel_debug_watchdog(dev, (unsigned long long)ms * 1000000ull));
    if (buf) *buf = host;
    if (out) { out[0] = (uint64_t)(uintptr_t)plan->sp.ctr; out[1] = (uint64_t)(uintptr_t)plan->ubuf.ptr; out[2] = (uint64_t)(uintptr_t)plan->xsol.ptr; }
    return GSE_OK;
}
// Item layout of one iteration of the persistent kernel: eval, accumulate, front, backward, update counts.
int gse_solve_layout(const gse_plan* plan, int32_t* out) {
    const SolveProg& sp = plan->sp;
    out[0] = sp.n_eval_items; out[1] = sp.n_acc_items; out[2] = sp.n_tasks; out[3] = sp.n_btasks; out[4] = sp.n_upd_items;
    out[5] = plan->solve_grid; out[6] = (int32_t)plan->solve_smem; out[7] = plan->persistent ? 1 : 0;
    return GSE_OK;
}

int gse_plan_stats(const gse_plan* plan, double* s, int32_t n) {
    const HostProgram& hp = plan->hp;
    double v[16] = {(double)plan->launches_last, (double)hp.fronts.size(), (double)hp.fwd_levels.size(), (double)plan->tasks.n,
                    (double)hp.max_front, (double)hp.n_lbuf, (double)hp.n_ubuf, (double)hp.n_pairs, (double)hp.n_slots,
                    hp.alg_bytes, hp.dense_flops, (double)plan->launches_per_iter,
                    plan->persistent ? 1.0 : 0.0, (double)plan->solve_grid, (double)plan->solve_smem, (double)plan->sp.items_per_it};
    for (int i = 0; i < n && i < 16; ++i) s[i] = v[i];
    return GSE_OK;
}

}  // extern "C"
