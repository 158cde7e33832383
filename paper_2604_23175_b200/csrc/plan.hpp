// plan.hpp -- host-side symbolic structures and the device program layout.
//
// One plan = one (network, measurement set, partition) triple analysed once
// (the reference re-runs build_patterns + symbolic_analyze inside every solve,
// solver.py:221-229; here both are plan-time).  Everything the GN loop touches
// lives in flat int32 / float64 device arrays described by DevProgram.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/gridse_b200.h"

namespace gse {

// ---------------------------------------------------------------------------
// Fronts.  The whole hierarchy -- area interiors (nested dissection), one
// assembly-only root per area (its update matrix IS the Schur block S_b with
// b_hat as the extra row), the boundary assembly root (S_Gamma, b_Gamma) and the
// dense boundary factorisation (a chain of fronts) -- is ONE multifrontal tree.
// ---------------------------------------------------------------------------
struct Front {
    int area = -1;          // owning area, -1 for coordinator fronts
    int kind = 0;           // 0 interior, 1 area root (S_b), 2 gamma root (S_Gamma), 3 chain
    int p = 0;              // pivots eliminated here
    int u1 = 0;             // update rows including the trailing RHS row
    int parent = -1;
    int level = 0;
    int T = 0, nch = 0;     // update-row chunking
    std::vector<int> rows;  // global positions of [pivots | update rows] (RHS row not listed)
    std::vector<int> children;
    std::vector<int> child_rel;   // optional, parallel to children: index into HostProgram::extra_rel (else the child's own rel)
    std::vector<int> rel;   // as a child: update row i -> local row of the parent
    int64_t l_off = 0, u_off = 0, gval_off = 0;
    int n_orig = 0;
};

struct Task { int front, ci, cj, phase, kind; };   // kind: 0 fused, 1 panel, 2 update (front_body.cuh)

struct HostProgram {
    // sizes
    int n_bus = 0, n_rows = 0, n_areas = 0, n_gamma = 0, slack = 0;
    int64_t n_slots = 0, n_pairs = 0;
    int n_pos = 0;                       // length of the global solution vector
    int gamma_base = 0;                  // first position of x_Gamma in it
    std::vector<int> area_base;          // first interior position of each area
    std::vector<int> area_ni, area_nb;
    std::vector<int> owned;              // 1 if this rank assembles / factors the area
    bool gamma_sparse = false;           // boundary system factored as a tree (block sparsity) instead of a dense chain
    std::vector<int> gamma_epos;         // x_Gamma slot -> elimination rank (identity in dense mode)
    std::vector<std::vector<int>> area_bpos;   // per area: local boundary variable -> row of the area root
    std::vector<std::vector<int>> extra_rel;   // rel maps that are not a front's own (boundary-root readback)
    int rank = 0, world = 1;

    // template evaluation units
    std::vector<int32_t> vm_bus, vm_row, vm_slot;
    std::vector<int32_t> fl_branch, fl_from, fl_to, fl_row /*8 per unit: PF PT QF QT IF IT - -*/, fl_slot /*8 per unit*/;
    std::vector<int32_t> inj_bus, inj_rowp, inj_rowq, inj_slotp, inj_slotq, inj_nth /*angle slots of the row*/;

    // accumulation: destination-sorted contribution lists (solver layout -> gval)
    // every contribution is val[a] * val[b], val = [g | w*g | w*r per row] (n_val entries)
    std::vector<int32_t> acc_ptr, acc_a, acc_b;
    int64_t n_val = 0;
    // staged form of the same program.  Item record (8 ints): first destination, destinations,
    // value-list offset, values, pair offset, pairs, local-pointer offset, 0.  The pointer segment holds
    // the item-local contribution pointers (destinations + 1) followed by the processing order
    // (destinations by decreasing contribution count).  Segments are padded to multiples of 4
    // entries (16 bytes) for TMA bulk copies.
    std::vector<int32_t> acc_items, acc_uniq, acc_lptr;
    std::vector<uint32_t> acc_pair;                 // per contribution: staged positions (b << 16 | a)
    int acc_stage_max = 0, acc_pair_max = 0;        // longest value list / pair list of an item
    // reference layout (component parity): per area CSR patterns + a second program
    std::vector<std::vector<int32_t>> ii_ptr, ii_idx, ib_ptr, ib_idx;
    std::vector<int64_t> ref_off;        // per area offset into the ref-layout value array
    std::vector<int32_t> racc_ptr, racc_a, racc_b;   // built on demand: build_reference_program
    int64_t n_ref_vals = 0;
    bool ref_program_built = false;
    // per area template layout (rows, slot pointers, slot variables, first global slot)
    std::vector<std::vector<int>> tmpl_rows, tmpl_slot_ptr, tmpl_slot_var;
    std::vector<int64_t> tmpl_slot_base;
    std::vector<int32_t> perm_orig;      // per position: original local variable (error reports)

    // fronts / tasks / levels
    std::vector<Front> fronts;
    std::vector<int> area_root;          // front id of each area's root
    int gamma_root = -1;
    std::vector<std::vector<Task>> fwd_levels;      // factor tasks per level
    std::vector<std::vector<int>> bwd_levels;       // fronts per backward level (top-down)
    std::vector<int> level_phase;        // 1 local_condense, 2 boundary_assemble, 3 boundary_solve
    std::vector<int> bwd_phase;          // 3 boundary_solve, 4 recovery
    // original entries per front: (row_local << 16 | col_local), region table
    std::vector<uint32_t> orig_pos;
    std::vector<int32_t> reg_ptr;        // flattened per-front region pointers
    std::vector<int32_t> front_reg_off;  // per front offset into reg_ptr
    int64_t n_gval = 0, n_lbuf = 0, n_ubuf = 0;
    std::vector<int64_t> gval_src;       // generic matrix plan: source of every original entry in the caller's layout
    // exchange buffer = U storage of the area roots, contiguous in area order
    int64_t xchg_off = 0, xchg_len = 0;
    std::vector<int64_t> xchg_area_off;  // n_areas + 1 (relative to xchg_off)

    // state update: one entry per solved variable
    std::vector<int32_t> upd_bus, upd_quant, upd_pos;

    // stats
    double alg_bytes = 0, dense_flops = 0;
    int max_front = 0;
};

// staging limits of one accumulation item: 48 KB of values + 44 KB of pairs + 12 KB of pointers / order
constexpr int kAccStageMax = 6144;     // distinct values
constexpr int kAccPairMax = 11264;     // contributions
constexpr int kAccItemDestMax = 1532;  // destinations (pointers + order: at most 3072 entries)
constexpr size_t kAccSmemBytes = 8 * (size_t)kAccStageMax + 4 * (size_t)kAccPairMax + 4 * 3072;

struct BuildOptions {
    bool dense = false;
    int leaf_buses = 48;   // measured best on the PEGASE-9241 shape (tools/gpu_leaf.sh: 12 -> 4.2 ms, 48 -> 3.25 ms per solve)
    int max_pivots = 64;
    int boundary_mode = 0;     // 0 auto (tree when n_Gamma > 192), 1 dense chain, 2 tree
    int gamma_leaf_buses = 16; // nested-dissection leaf of the boundary tree, in boundary buses
    // nested dissection picks the BFS level minimising |left - right| + w * |separator|: a larger w trades
    // balance for shorter chains of sequential pivots (the solve is latency-bound on that chain)
    double sep_weight = 2.0, gamma_sep_weight = 2.0;
    // fronts with several row chunks and at least this many pivots run as panel + update tasks.  Measured on the
    // PEGASE-9241 shape (tools/gpu_sweep2.sh): the panel is bound by its serial 8x8 chain, not by its row count,
    // so the split only adds a hand-off (2.06 ms vs 2.03 ms per solve) -- off by default, kept for wide fronts.
    int split_min_pivots = 1 << 20;
    int split_min_tasks = 0;   // ... and at least this many tile tasks (GSE_SPLIT_TASKS)
    // relaxed amalgamation of the area interiors' nested-dissection nodes: a node joins its parent's front when both fit
    // one front and the node's columns grow by at most this fraction of explicit zeros (0: off).  Throughput-bound plans
    // (the ~100k-bus grid) gain 8-11 % with 1.0 (fewer, fuller fronts: 6770 -> 4730); latency-bound ones lose (more
    // pivots per front on the chains), measured on every BASELINE shape (profiles/r02_sweep_interior_merge.txt).
    double interior_merge = 0.0;
    double gamma_merge = 0.0;  // the same for the boundary tree on top of its fill-free amalgamation (0: fill-free only)
    int tile_rows = 48;   // update-row chunk (task tile) size (48: best measured on PEGASE-9241 shape)
    int gamma_tile_rows = 0;   // the same for the fronts of the boundary tree (0: tile_rows); GSE_GAMMA_TILE_ROWS
    int rank = 0, world = 1;
    std::vector<int> area_rank;
    // generic matrix plan (gse_matrix_plan_create): one area whose G_ii / G_ib patterns come from the
    // caller instead of from measurement templates
    bool ext_pattern = false;
    std::vector<int32_t> ext_ii_ptr, ext_ii_idx, ext_ib_ptr, ext_ib_idx;
};

// symbolic.cpp
std::string build_host_program(const gse_problem_desc& d, const BuildOptions& opt, HostProgram& hp);
void build_reference_program(HostProgram& hp);

}  // namespace gse
