// symbolic.cpp -- plan-time analysis on the host (runs once per plan).
//
// Replaces, for every area at once, the reference's build_patterns /
// _build_pair_programs (assembly.py:172-400) and SparseCholeskyCache._analyze
// (linalg.py:156-231):
//   * template slots in the reference's slot order + SoA evaluation units
//     (VM rows, one unit per measured branch, one unit per measured bus);
//   * CSR patterns of G_ii / G_ib in the reference layout (component parity);
//   * a nested-dissection ordering of each area's interior on the bus graph
//     (the ordering is free: SPEC.md "ordering is an implementation choice"),
//     relaxed supernodes ("fronts") of at most max_pivots columns, their update
//     sets and the assembly tree;
//   * one assembly-only root front per area (Schur mode: boundary variables are
//     never eliminated locally), the boundary assembly root and the dense
//     boundary factorisation as a chain of fronts;
//   * destination-sorted contribution lists: for every stored entry of every
//     front (and of the right-hand-side row) the template slot pairs that add
//     into it, in ascending row order -- the deterministic, atomic-free
//     replacement of the five bincount scatters (assembly.py:502-520).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>

#include "plan.hpp"

namespace gse {
namespace {

// Plan-time work that splits by area / by item runs on a few host threads (GSE_BUILD_THREADS
// overrides the count; 1 = serial).  Every piece writes its own output, merged in index order:
// the program does not depend on the thread count.
int build_threads() {
    if (const char* e = getenv("GSE_BUILD_THREADS")) return std::max(1, atoi(e));
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::min(16u, std::max(1u, hw));
}
template <class F>
void parallel_for(int n, int nthreads, F&& fn) {
    nthreads = std::min(nthreads, n);
    if (nthreads <= 1) { for (int i = 0; i < n; ++i) fn(i); return; }
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t] { for (int i = t; i < n; i += nthreads) fn(i); });
    for (auto& th : pool) th.join();
}

struct AreaSym {
    int ni = 0, nb = 0;
    std::vector<int> var_bus;            // interior variable -> index into im_bus
    std::vector<int> th_var, vm_var;     // per interior bus index: variable ids (-1 none)
    std::vector<int> epos, order;        // variable -> elimination position and inverse
    std::vector<int> rows;               // global row ids owned, ascending
    std::vector<int> slot_ptr, slot_var; // reference template layout
    int64_t slot_base = 0;
    // lower-triangular pattern in position space incl. boundary (pos >= ni) and RHS row (pos == ni+nb)
    std::vector<int> col_ptr, col_row;
    std::vector<int64_t> col_dest;
    std::vector<int> front_of_pos;       // interior position -> front id (global)
    int first_front = 0, n_fronts = 0, root = -1;
};

// ---- nested dissection on the interior bus graph ---------------------------------
struct NDGraph {
    std::vector<int> xadj, adj;
    std::vector<int> stamp, level;
    int cur = 0;
    double sep_weight = 2.0;   // level-set choice: |left - right| + sep_weight * |separator|
};

void nd_recurse(NDGraph& g, std::vector<int>& verts, int leaf, std::vector<std::vector<int>>& out) {
    const int n = (int)verts.size();
    if (n == 0) return;
    if (n <= leaf) { out.push_back(verts); return; }
    // connected components of the induced subgraph
    int tag = ++g.cur;
    for (int v : verts) g.stamp[v] = tag;
    std::vector<int> comp_tag_start;
    {
        std::vector<std::vector<int>> comps;
        int seen_tag = ++g.cur;
        for (int s : verts) {
            if (g.stamp[s] != tag) continue;
            std::vector<int> comp{s};
            g.stamp[s] = seen_tag;
            for (size_t h = 0; h < comp.size(); ++h) {
                int u = comp[h];
                for (int p = g.xadj[u]; p < g.xadj[u + 1]; ++p) {
                    int w = g.adj[p];
                    if (g.stamp[w] == tag) { g.stamp[w] = seen_tag; comp.push_back(w); }
                }
            }
            comps.push_back(std::move(comp));
        }
        if (comps.size() > 1) {
            for (auto& c : comps) { std::sort(c.begin(), c.end()); nd_recurse(g, c, leaf, out); }
            return;
        }
    }
    // level structure from a pseudo-peripheral vertex
    tag = ++g.cur;
    for (int v : verts) g.stamp[v] = tag;
    int start = verts[0];
    std::vector<int> bfs;
    int depth = 0;
    for (int sweep = 0; sweep < 3; ++sweep) {
        int vis = ++g.cur;
        bfs.assign(1, start);
        g.stamp[start] = vis; g.level[start] = 0;
        for (size_t h = 0; h < bfs.size(); ++h) {
            int u = bfs[h];
            for (int p = g.xadj[u]; p < g.xadj[u + 1]; ++p) {
                int w = g.adj[p];
                if (g.stamp[w] == tag) { g.stamp[w] = vis; g.level[w] = g.level[u] + 1; bfs.push_back(w); }
            }
        }
        int d = g.level[bfs.back()];
        // restore membership tag for the next sweep
        for (int v : verts) g.stamp[v] = tag;
        if (sweep > 0 && d <= depth) { depth = std::max(depth, d); break; }
        depth = d;
        // farthest vertex of smallest degree (ties: lowest id)
        int best = -1, bdeg = 1 << 30;
        for (int v : bfs) if (g.level[v] == d) {
            int deg = g.xadj[v + 1] - g.xadj[v];
            if (deg < bdeg || (deg == bdeg && v < best)) { best = v; bdeg = deg; }
        }
        if (sweep < 2) start = best;
    }
    // final BFS from `start` (levels valid for it)
    {
        int vis = ++g.cur;
        bfs.assign(1, start);
        g.stamp[start] = vis; g.level[start] = 0;
        for (size_t h = 0; h < bfs.size(); ++h) {
            int u = bfs[h];
            for (int p = g.xadj[u]; p < g.xadj[u + 1]; ++p) {
                int w = g.adj[p];
                if (g.stamp[w] == tag) { g.stamp[w] = vis; g.level[w] = g.level[u] + 1; bfs.push_back(w); }
            }
        }
        depth = g.level[bfs.back()];
    }
    if (depth < 2) { out.push_back(verts); return; }
    std::vector<int> cnt(depth + 1, 0);
    for (int v : verts) cnt[g.level[v]]++;
    int best_j = 1; double best_cost = 1e300; int below = cnt[0];
    for (int j = 1; j <= depth - 1; ++j) {
        int above = n - below - cnt[j];
        double cost = std::abs(below - above) + g.sep_weight * cnt[j];
        if (cost < best_cost) { best_cost = cost; best_j = j; }
        below += cnt[j];
    }
    std::vector<int> A, B, S;
    for (int v : verts) {
        int l = g.level[v];
        if (l < best_j) A.push_back(v);
        else if (l > best_j) B.push_back(v);
        else {
            bool touches_b = false;
            for (int p = g.xadj[v]; p < g.xadj[v + 1] && !touches_b; ++p) {
                int w = g.adj[p];
                touches_b = (g.stamp[w] == g.cur) && g.level[w] == best_j + 1;
            }
            (touches_b ? S : A).push_back(v);
        }
    }
    std::sort(A.begin(), A.end()); std::sort(B.begin(), B.end()); std::sort(S.begin(), S.end());
    nd_recurse(g, A, leaf, out);
    nd_recurse(g, B, leaf, out);
    out.push_back(S);
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

void choose_chunks(Front& f, int TMAX) {
    if (f.u1 <= TMAX) { f.T = f.u1; f.nch = f.u1 > 0 ? 1 : 0; return; }
    int nch = (f.u1 + TMAX - 1) / TMAX;
    int T = round_up((f.u1 + nch - 1) / nch, 8);
    f.T = T; f.nch = (f.u1 + T - 1) / T;
}

// Staged accumulation program: the destination range is cut into items that one CTA processes
// entirely out of shared memory.  Per item: the sorted list of distinct value indices (gathered
// once), the item-local contribution pointers and, per contribution, the two positions in the
// value list packed as (b << 16 | a).  The pointer and pair segments of an item are contiguous and
// 16-byte aligned so that one TMA bulk copy each brings them on chip.  Items are sized so that
// about one wave of CTAs covers the whole program (the persistent kernel keeps ~2 CTAs per SM
// resident) within the staging limits kAccStageMax / kAccPairMax / kAccItemDestMax.
void build_acc_items(HostProgram& hp) {
    const int64_t n = hp.n_gval;
    hp.acc_items.clear(); hp.acc_uniq.clear(); hp.acc_pair.clear(); hp.acc_lptr.clear();
    hp.acc_stage_max = 0;
    if (n == 0) return;
    const int64_t target_items = 280;
    int64_t dmax = (n + target_items - 1) / target_items;
    dmax = std::min<int64_t>(std::max<int64_t>((dmax + 255) / 256 * 256, 256), kAccItemDestMax);
    auto pad4 = [](auto& v) { while (v.size() % 4) v.push_back(0); };
    // The destination range is cut into kSeg fixed segments (multiples of dmax; the count does not
    // depend on the machine), each cut greedily into items on its own thread with private scratch;
    // the pieces are concatenated in segment order.
    constexpr int kSeg = 8;
    struct Piece { std::vector<int32_t> items, uniq, lptr; std::vector<uint32_t> pair; int stage_max = 0, pair_max = 0; };
    const int64_t chunks = (n + dmax - 1) / dmax;
    const int nseg = (int)std::min<int64_t>(kSeg, chunks);
    std::vector<Piece> pieces(nseg);
    int nthreads = build_threads();
    nthreads = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads, (1024LL << 20) / (8 * std::max<int64_t>(hp.n_val, 1))));
    nthreads = std::min(nthreads, nseg);
    std::vector<std::vector<int32_t>> stamps(nthreads), locals(nthreads);
    auto cut_segment = [&](int sg, std::vector<int32_t>& stamp, std::vector<int32_t>& local) {
        Piece& P = pieces[sg];
        const int64_t lo = chunks * sg / nseg * dmax, hi = std::min<int64_t>(n, chunks * (sg + 1) / nseg * dmax);
        std::vector<int32_t> uniq;
        int64_t d0 = lo;
        while (d0 < hi) {
            const int item = (int)(P.items.size() / 8) + sg * (1 << 24);      // stamp value: unique per (segment, item)
            uniq.clear();
            int64_t d1 = d0;
            while (d1 < hi && d1 - d0 < dmax) {
                // distinct values / pairs the next destination would add
                const size_t before = uniq.size();
                for (int q = hp.acc_ptr[d1]; q < hp.acc_ptr[d1 + 1]; ++q)
                    for (int32_t v : {hp.acc_a[q], hp.acc_b[q]})
                        if (stamp[v] != item) { stamp[v] = item; uniq.push_back(v); }
                if (((int)uniq.size() > kAccStageMax || hp.acc_ptr[d1 + 1] - hp.acc_ptr[d0] > kAccPairMax) && d1 > d0) {
                    for (size_t i = before; i < uniq.size(); ++i) stamp[uniq[i]] = -1;
                    uniq.resize(before);
                    break;
                }
                ++d1;
            }
            std::sort(uniq.begin(), uniq.end());
            for (size_t i = 0; i < uniq.size(); ++i) local[uniq[i]] = (int32_t)i;
            const int32_t q0 = hp.acc_ptr[d0], np = hp.acc_ptr[d1] - q0;
            const int32_t pair_off = (int32_t)P.pair.size(), ptr_off = (int32_t)P.lptr.size(), uniq_off = (int32_t)P.uniq.size();
            for (int q = q0; q < q0 + np; ++q) P.pair.push_back(((uint32_t)local[hp.acc_b[q]] << 16) | (uint32_t)local[hp.acc_a[q]]);
            pad4(P.pair);
            for (int64_t dd = d0; dd <= d1; ++dd) P.lptr.push_back(hp.acc_ptr[dd] - q0);
            // processing order: destinations by decreasing contribution count, so that the threads of a
            // warp (consecutive ranks) walk lists of similar length
            {
                std::vector<int32_t> ord((size_t)(d1 - d0));
                std::iota(ord.begin(), ord.end(), 0);
                std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
                    return hp.acc_ptr[d0 + x + 1] - hp.acc_ptr[d0 + x] > hp.acc_ptr[d0 + y + 1] - hp.acc_ptr[d0 + y]; });
                P.lptr.insert(P.lptr.end(), ord.begin(), ord.end());
            }
            pad4(P.lptr);
            P.uniq.insert(P.uniq.end(), uniq.begin(), uniq.end());
            pad4(P.uniq);
            const int32_t rec[8] = {(int32_t)d0, (int32_t)(d1 - d0), uniq_off, (int32_t)uniq.size(), pair_off, np, ptr_off, 0};
            P.items.insert(P.items.end(), rec, rec + 8);
            P.stage_max = std::max(P.stage_max, (int)uniq.size());
            P.pair_max = std::max(P.pair_max, (int)np);
            d0 = d1;
        }
    };
    const bool dbg_time = getenv("GSE_DEBUG_TIME") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* w) { if (!dbg_time) return; auto now = std::chrono::steady_clock::now(); fprintf(stderr, "    acc items: %-22s %.3f s\n", w, std::chrono::duration<double>(now - t0).count()); t0 = now; };
    {
        std::vector<std::thread> pool;
        auto work = [&](int t) {
            stamps[t].assign((size_t)hp.n_val, -1); locals[t].assign((size_t)hp.n_val, 0);
            for (int sg = t; sg < nseg; sg += nthreads) cut_segment(sg, stamps[t], locals[t]);
        };
        for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
    }
    lap("segments (threads)");
    {
        size_t ni = 0, nu = 0, npr = 0, nl = 0;
        for (const Piece& P : pieces) { ni += P.items.size(); nu += P.uniq.size(); npr += P.pair.size(); nl += P.lptr.size(); }
        hp.acc_items.reserve(ni); hp.acc_uniq.reserve(nu); hp.acc_pair.reserve(npr); hp.acc_lptr.reserve(nl);
    }
    for (const Piece& P : pieces) {
        const int32_t uo = (int32_t)hp.acc_uniq.size(), po = (int32_t)hp.acc_pair.size(), lo = (int32_t)hp.acc_lptr.size();
        for (size_t i = 0; i < P.items.size(); i += 8) {
            int32_t rec[8]; std::copy(P.items.begin() + i, P.items.begin() + i + 8, rec);
            rec[2] += uo; rec[4] += po; rec[6] += lo;
            hp.acc_items.insert(hp.acc_items.end(), rec, rec + 8);
        }
        hp.acc_uniq.insert(hp.acc_uniq.end(), P.uniq.begin(), P.uniq.end());
        hp.acc_pair.insert(hp.acc_pair.end(), P.pair.begin(), P.pair.end());
        hp.acc_lptr.insert(hp.acc_lptr.end(), P.lptr.begin(), P.lptr.end());
        hp.acc_stage_max = std::max(hp.acc_stage_max, P.stage_max);
        hp.acc_pair_max = std::max(hp.acc_pair_max, P.pair_max);
    }
    lap("merge");
    if (getenv("GSE_DEBUG_ACC")) {
        auto fnv = [](const void* p, size_t bytes) { uint64_t h = 1469598103934665603ull; const unsigned char* c = (const unsigned char*)p; for (size_t i = 0; i < bytes; ++i) { h ^= c[i]; h *= 1099511628211ull; } return h; };
        fprintf(stderr, "acc program checksums: items %016llx pair %016llx lptr %016llx uniq %016llx a %016llx b %016llx ptr %016llx\n",
                (unsigned long long)fnv(hp.acc_items.data(), hp.acc_items.size() * 4), (unsigned long long)fnv(hp.acc_pair.data(), hp.acc_pair.size() * 4),
                (unsigned long long)fnv(hp.acc_lptr.data(), hp.acc_lptr.size() * 4), (unsigned long long)fnv(hp.acc_uniq.data(), hp.acc_uniq.size() * 4),
                (unsigned long long)fnv(hp.acc_a.data(), hp.acc_a.size() * 4), (unsigned long long)fnv(hp.acc_b.data(), hp.acc_b.size() * 4),
                (unsigned long long)fnv(hp.acc_ptr.data(), hp.acc_ptr.size() * sizeof(hp.acc_ptr[0])));
        int n_items = (int)(hp.acc_items.size() / 8), max_nd = 0, max_np = hp.acc_pair_max; double sum_nu = 0;
        for (int i = 0; i < n_items; ++i) { max_nd = std::max(max_nd, hp.acc_items[8 * i + 1]); sum_nu += hp.acc_items[8 * i + 3]; }
        {   // contribution-list lengths: the longest list of an item bounds its sequential rounds
            int64_t sum_max = 0, sum_w0 = 0; int gmax = 0;
            for (int i = 0; i < n_items; ++i) {
                const int l0 = hp.acc_items[8 * i + 6], nd = hp.acc_items[8 * i + 1];
                const int32_t* ord = &hp.acc_lptr[l0 + nd + 1];
                auto len = [&](int d) { return hp.acc_lptr[l0 + d + 1] - hp.acc_lptr[l0 + d]; };
                const int mx = nd ? len(ord[0]) : 0; gmax = std::max(gmax, mx); sum_max += mx;
                int w0 = 0; for (int g = 0; g * 256 < nd; ++g) w0 += len(ord[g * 256]);   // rounds of thread 0 over its groups
                sum_w0 += w0;
            }
            fprintf(stderr, "acc lists: longest %d, mean longest per item %.1f, mean rounds of the slowest thread %.1f\n",
                    gmax, (double)sum_max / std::max(n_items, 1), (double)sum_w0 / std::max(n_items, 1));
        }
        fprintf(stderr, "acc items %d (dmax %lld): max dests %d, max pairs %d, max values %d, mean values %.0f, n_val %lld, n_gval %lld, pairs %zu\n",
                n_items, (long long)dmax, max_nd, max_np, hp.acc_stage_max, sum_nu / std::max(n_items, 1), (long long)hp.n_val, (long long)n, hp.acc_a.size());
    }
}

}  // namespace


// Fill-free amalgamation of nested-dissection nodes: a node whose update structure is exactly its parent's whole front
// (pivots + update rows) is eliminated WITH the parent -- the same factor entries, one front and one dependency hop
// less -- when that saves a front (nodes are cut into fronts of <= pmax pivots) and the node either fits the parent's
// last front or is tiny (otherwise every task of the parent's fronts factors a taller pivot block: measured slower).
// Moving the node's elimination to just before its parent is a valid reordering: everything in between belongs to
// other subtrees.  nodes: vertex lists in elimination order; xadj / adj: the graph; ext: per vertex, ids of variables
// that are never eliminated here (an area's boundary variables) and belong to every structure that reaches them.
template <class SlotsOf>
static void amalgamate_nodes(std::vector<std::vector<int>>& nodes, int nn, const std::vector<int>& xadj, const std::vector<int>& adj,
                             const std::vector<std::vector<int>>* ext, SlotsOf slots_of, int pmax, double fill_tol = 0.0) {
    int n_ext = 0;
    if (ext) for (auto& e : *ext) for (int x : e) n_ext = std::max(n_ext, x + 1);
    for (bool merged = true; merged;) {
        merged = false;
        const int nn_nodes = (int)nodes.size();
        std::vector<int> node_of(nn, -1), pos_of(nn, -1);
        { int q = 0; for (int i = 0; i < nn_nodes; ++i) for (int b : nodes[i]) { node_of[b] = i; pos_of[b] = q++; } }
        // structure of every node (vertices eliminated later that its front reaches), children before parents
        std::vector<std::vector<int>> st(nn_nodes), se(nn_nodes), kids(nn_nodes);
        std::vector<int> parent(nn_nodes, -1), mark(nn, -1), emark(n_ext, -1);
        for (int i = 0; i < nn_nodes; ++i) {
            const int last = pos_of[nodes[i].back()];
            auto add = [&](int b) { if (pos_of[b] > last && mark[b] != i) { mark[b] = i; st[i].push_back(b); } };
            auto add_ext = [&](int x) { if (emark[x] != i) { emark[x] = i; se[i].push_back(x); } };
            for (int b : nodes[i]) {
                for (int e = xadj[b]; e < xadj[b + 1]; ++e) add(adj[e]);
                if (ext) for (int x : (*ext)[b]) add_ext(x);
            }
            for (int c : kids[i]) { for (int b : st[c]) add(b); for (int x : se[c]) add_ext(x); }
            if (st[i].empty()) continue;
            int first = st[i][0];
            for (int b : st[i]) if (pos_of[b] < pos_of[first]) first = b;
            parent[i] = node_of[first];
            kids[parent[i]].push_back(i);
        }
        auto pieces = [&](int v) { return (v + pmax - 1) / pmax; };
        for (int i = 0; i < nn_nodes && !merged; ++i) {
            const int q = parent[i];
            if (q < 0) continue;
            const int pi = slots_of(nodes[i]), pq = slots_of(nodes[q]);
            if (pieces(pi + pq) >= pieces(pi) + pieces(pq)) continue;                 // must save a front
            if (pi + pq > pmax && pi > 8) continue;
            // (fill_tol > 0: relaxed amalgamation -- the node's columns may grow by that fraction of explicit zeros,
            // only into a single front)
            const size_t have = st[i].size() + se[i].size(), want = nodes[q].size() + st[q].size() + se[q].size();
            if (have != want && !(fill_tol > 0.0 && pi + pq <= pmax && (double)(want - have) <= fill_tol * (double)want)) continue;
            std::vector<int> both = nodes[i];
            both.insert(both.end(), nodes[q].begin(), nodes[q].end());
            nodes[q] = std::move(both);
            nodes.erase(nodes.begin() + i);
            merged = true;
        }
    }
}

// Cut point q of a node of nv pivots split into `pieces` fronts: even shares, moved up to the next multiple of 8 when
// every piece still fits pmax -- the panel factorisation runs in 8-pivot blocks, so 116 pivots cost 8 + 7 blocks as
// 64 + 52 but 8 + 8 as 58 + 58.
static inline int piece_cut(int nv, int pieces, int q, int pmax) {
    if (q <= 0) return 0;
    if (q >= pieces) return nv;
    const int even = (int)((int64_t)nv * q / pieces);
    const int up = (even + 7) & ~7;
    // the pieces before the cut get at most `up - previous cut` <= pmax when up <= q * pmax; the rest must fit too
    if (up < nv && up <= q * pmax && nv - up <= (pieces - q) * pmax && up - (int)((int64_t)nv * (q - 1) / pieces) <= pmax + 7) return up;
    return even;
}
std::string build_host_program(const gse_problem_desc& d, const BuildOptions& opt, HostProgram& hp) {
    const int nbus = d.n_bus, K = d.n_areas, m = d.n_rows, ng = d.n_gamma;
    if (nbus <= 0 || K <= 0 || m < 0) return "empty problem";
    const bool dbg_time = getenv("GSE_DEBUG_TIME") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    double t_sec[6] = {0, 0, 0, 0, 0, 0};
    auto t_mark = std::chrono::steady_clock::now();
    auto sec = [&](int k) { if (!dbg_time) return; auto now = std::chrono::steady_clock::now(); t_sec[k] += std::chrono::duration<double>(now - t_mark).count(); t_mark = now; };
    auto lap = [&](const char* what) {
        if (!dbg_time) return;
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "  plan build: %-28s %.3f s\n", what, std::chrono::duration<double>(now - t_prev).count());
        t_prev = now;
    };
    const int PMAX = opt.max_pivots;
    hp.n_bus = nbus; hp.n_rows = m; hp.n_areas = K; hp.n_gamma = ng; hp.slack = d.slack;
    hp.rank = opt.rank; hp.world = opt.world;
    hp.owned.assign(K, 1);
    if (!opt.area_rank.empty()) for (int a = 0; a < K; ++a) hp.owned[a] = opt.area_rank[a] == opt.rank;
    const bool coordinator = opt.rank == 0;

    std::vector<AreaSym> as(K);
    hp.area_ni.resize(K); hp.area_nb.resize(K); hp.area_base.resize(K);
    int pos_cursor = 0;
    for (int a = 0; a < K; ++a) {
        AreaSym& A = as[a];
        int n_ia = d.ia_ptr[a + 1] - d.ia_ptr[a], n_im = d.im_ptr[a + 1] - d.im_ptr[a];
        int n_ba = d.ba_ptr[a + 1] - d.ba_ptr[a], n_bm = d.bm_ptr[a + 1] - d.bm_ptr[a];
        A.ni = n_ia + n_im; A.nb = n_ba + n_bm;
        if (d.sel_ptr[a + 1] - d.sel_ptr[a] != A.nb) return "boundary selector length mismatch";
        for (int j = 1; j < A.nb; ++j)
            if (d.sel[d.sel_ptr[a] + j] <= d.sel[d.sel_ptr[a] + j - 1]) return "boundary selector must be increasing";
        hp.area_ni[a] = A.ni; hp.area_nb[a] = A.nb; hp.area_base[a] = pos_cursor;
        pos_cursor += A.ni;
    }
    hp.gamma_base = pos_cursor;
    hp.n_pos = pos_cursor + ng;
    hp.perm_orig.assign(hp.n_pos, -1);

    // ---- elimination order of the boundary system -----------------------------------------
    // dense mode: natural slot order, factored as a chain of dense fronts (the reference's
    // dense_cholesky_solve).  sparse mode: nested dissection on the graph whose cliques are the
    // areas' local boundary sets -- the same Cholesky factorisation of the same S_Gamma, but
    // the structural zeros between non-adjacent areas are never touched.
    const bool sparse_gamma = ng > 0 && (opt.boundary_mode == 2 || (opt.boundary_mode == 0 && ng > 192));
    hp.gamma_sparse = sparse_gamma;
    hp.gamma_epos.resize(ng);
    std::iota(hp.gamma_epos.begin(), hp.gamma_epos.end(), 0);
    std::vector<std::vector<int>> gamma_nodes;     // per ND node: the x_Gamma slots it eliminates
    if (sparse_gamma) {
        std::vector<int> node_of_bus(nbus, -1), ang_slot, mag_slot, node_bus;
        for (int s = 0; s < ng; ++s) if (d.gamma_quant[s] == 1) {
            node_of_bus[d.gamma_bus[s]] = (int)node_bus.size(); node_bus.push_back(d.gamma_bus[s]);
            mag_slot.push_back(s); ang_slot.push_back(-1);
        }
        for (int s = 0; s < ng; ++s) if (d.gamma_quant[s] == 0) ang_slot[node_of_bus[d.gamma_bus[s]]] = s;
        const int nn = (int)node_bus.size();
        std::vector<int64_t> edges;
        for (int a = 0; a < K; ++a)
            for (int i = d.bm_ptr[a]; i < d.bm_ptr[a + 1]; ++i)
                for (int j = d.bm_ptr[a]; j < d.bm_ptr[a + 1]; ++j)
                    if (i != j) edges.push_back((int64_t)node_of_bus[d.bm_bus[i]] * nn + node_of_bus[d.bm_bus[j]]);
        std::sort(edges.begin(), edges.end()); edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
        NDGraph g;
        g.xadj.assign(nn + 1, 0); g.adj.resize(edges.size());
        for (size_t i = 0; i < edges.size(); ++i) { g.xadj[edges[i] / nn + 1]++; g.adj[i] = (int)(edges[i] % nn); }
        for (int i = 0; i < nn; ++i) g.xadj[i + 1] += g.xadj[i];
        g.stamp.assign(nn, 0); g.level.assign(nn, 0);
        g.sep_weight = opt.gamma_sep_weight;
        std::vector<int> all(nn); std::iota(all.begin(), all.end(), 0);
        std::vector<std::vector<int>> nodes;
        nd_recurse(g, all, std::max(1, opt.gamma_leaf_buses), nodes);
        if (!getenv("GSE_NO_GAMMA_MERGE"))
            amalgamate_nodes(nodes, nn, g.xadj, g.adj, nullptr,
                             [&](const std::vector<int>& node) { int c = 0; for (int b : node) c += 1 + (ang_slot[b] >= 0); return c; }, PMAX,
                             opt.gamma_merge);
        int rank = 0;
        for (auto& node : nodes) {
            std::vector<int> slots;
            for (int b : node) { if (ang_slot[b] >= 0) slots.push_back(ang_slot[b]); slots.push_back(mag_slot[b]); }
            for (int s : slots) hp.gamma_epos[s] = rank++;
            gamma_nodes.push_back(std::move(slots));
        }
        if (rank != ng) return "boundary ordering did not cover x_Gamma";
    }
    std::vector<int> gamma_slot_of_rank(ng);
    for (int s = 0; s < ng; ++s) gamma_slot_of_rank[hp.gamma_epos[s]] = s;
    // per area: local boundary variables in boundary elimination order (identity in dense mode)
    hp.area_bpos.assign(K, {});
    std::vector<std::vector<int>> bvar_of_pos(K);
    for (int a = 0; a < K; ++a) {
        const int nb = as[a].nb;
        bvar_of_pos[a].resize(nb);
        std::iota(bvar_of_pos[a].begin(), bvar_of_pos[a].end(), 0);
        std::sort(bvar_of_pos[a].begin(), bvar_of_pos[a].end(), [&](int x, int y) {
            return hp.gamma_epos[d.sel[d.sel_ptr[a] + x]] < hp.gamma_epos[d.sel[d.sel_ptr[a] + y]]; });
        hp.area_bpos[a].resize(nb);
        for (int q = 0; q < nb; ++q) hp.area_bpos[a][bvar_of_pos[a][q]] = q;
    }

    // ---- rows per area -----------------------------------------------------------
    for (int r = 0; r < m; ++r) {
        int t = d.m_type[r], tg = d.m_target[r];
        if (t < 0 || t > 8) return "unknown measurement type";      // 0 VM, 1-2 P/Q injection, 3-6 P/Q flow, 7-8 current magnitude
        if (tg < 0 || tg >= (t >= 3 ? d.n_branch : nbus)) return "measurement target out of range";
        int owner = t >= 3 ? d.br_from[tg] : tg;
        as[d.area_of_bus[owner]].rows.push_back(r);
    }

    lap("boundary ordering, rows");
    // ---- template slots + evaluation units ------------------------------------------
    std::vector<int> loc_va(nbus, -1), loc_vm(nbus, -1);
    std::vector<int> unit_of_branch(d.n_branch, -1), unit_of_bus(nbus, -1);
    int64_t slot_cursor = 0;
    hp.ii_ptr.resize(K); hp.ii_idx.resize(K); hp.ib_ptr.resize(K); hp.ib_idx.resize(K);
    hp.ref_off.assign(K + 1, 0);
    double nnz_total = 0, rhs_total = 0;

    // reference-layout program pieces are collected per area then concatenated

    t_mark = std::chrono::steady_clock::now();
    for (int a = 0; a < K; ++a) {
        AreaSym& A = as[a];
        const int ni = A.ni, nb = A.nb;
        const int n_ia = d.ia_ptr[a + 1] - d.ia_ptr[a];
        const int n_ba = d.ba_ptr[a + 1] - d.ba_ptr[a];
        // local variable ids of this area (closure: only these buses may be referenced)
        std::vector<int> touched;
        auto setv = [&](std::vector<int>& arr, int bus, int v) { arr[bus] = v; touched.push_back(bus); };
        for (int i = 0; i < n_ia; ++i) setv(loc_va, d.ia_bus[d.ia_ptr[a] + i], i);
        for (int i = d.im_ptr[a]; i < d.im_ptr[a + 1]; ++i) setv(loc_vm, d.im_bus[i], n_ia + (i - d.im_ptr[a]));
        for (int i = 0; i < n_ba; ++i) setv(loc_va, d.ba_bus[d.ba_ptr[a] + i], ni + i);
        for (int i = d.bm_ptr[a]; i < d.bm_ptr[a + 1]; ++i) setv(loc_vm, d.bm_bus[i], ni + n_ba + (i - d.bm_ptr[a]));
        // interior bus index <-> variables
        const int nib = d.im_ptr[a + 1] - d.im_ptr[a];
        A.var_bus.assign(ni, -1); A.th_var.assign(nib, -1); A.vm_var.assign(nib, -1);
        for (int i = 0; i < nib; ++i) {
            int bus = d.im_bus[d.im_ptr[a] + i];
            A.vm_var[i] = n_ia + i; A.var_bus[n_ia + i] = i;
            if (loc_va[bus] >= 0 && loc_va[bus] < ni) { A.th_var[i] = loc_va[bus]; A.var_bus[loc_va[bus]] = i; }
        }

        A.slot_base = slot_cursor;
        A.slot_ptr.assign(A.rows.size() + 1, 0);
        bool closure_ok = true;
        auto need = [&](int v) { if (v < 0) closure_ok = false; return v; };
        for (size_t k = 0; k < A.rows.size(); ++k) {
            int r = A.rows[k], t = d.m_type[r], tg = d.m_target[r];
            int32_t gslot = (int32_t)(A.slot_base + A.slot_var.size());
            if (t == 0) {
                A.slot_var.push_back(need(loc_vm[tg]));
                if (hp.owned[a]) { hp.vm_bus.push_back(tg); hp.vm_row.push_back(r); hp.vm_slot.push_back(gslot); }
            } else if (t <= 2) {
                for (int p = d.y_ptr[tg]; p < d.y_ptr[tg + 1]; ++p) if (d.y_idx[p] != d.slack) A.slot_var.push_back(need(loc_va[d.y_idx[p]]));
                for (int p = d.y_ptr[tg]; p < d.y_ptr[tg + 1]; ++p) A.slot_var.push_back(need(loc_vm[d.y_idx[p]]));
                if (hp.owned[a]) {
                    int u = unit_of_bus[tg];
                    if (u < 0) {
                        u = unit_of_bus[tg] = (int)hp.inj_bus.size();
                        hp.inj_bus.push_back(tg); hp.inj_rowp.push_back(-1); hp.inj_rowq.push_back(-1);
                        hp.inj_slotp.push_back(-1); hp.inj_slotq.push_back(-1);
                        int nth = 0;
                        for (int p = d.y_ptr[tg]; p < d.y_ptr[tg + 1]; ++p) nth += d.y_idx[p] != d.slack;
                        hp.inj_nth.push_back(nth);
                    }
                    if (t == 1) { if (hp.inj_rowp[u] >= 0) return "duplicate injection row"; hp.inj_rowp[u] = r; hp.inj_slotp[u] = gslot; }
                    else { if (hp.inj_rowq[u] >= 0) return "duplicate injection row"; hp.inj_rowq[u] = r; hp.inj_slotq[u] = gslot; }
                }
            } else {
                int f = d.br_from[tg], tt = d.br_to[tg];
                if (f != d.slack) A.slot_var.push_back(need(loc_va[f]));
                if (tt != d.slack) A.slot_var.push_back(need(loc_va[tt]));
                A.slot_var.push_back(need(loc_vm[f])); A.slot_var.push_back(need(loc_vm[tt]));
                if (hp.owned[a]) {
                    int u = unit_of_branch[tg];
                    if (u < 0) {
                        u = unit_of_branch[tg] = (int)hp.fl_branch.size();
                        hp.fl_branch.push_back(tg); hp.fl_from.push_back(f); hp.fl_to.push_back(tt);
                        for (int q = 0; q < 8; ++q) { hp.fl_row.push_back(-1); hp.fl_slot.push_back(-1); }   // PF PT QF QT IF IT - -
                    }
                    if (hp.fl_row[8 * u + (t - 3)] >= 0) return "duplicate flow row";
                    hp.fl_row[8 * u + (t - 3)] = r; hp.fl_slot[8 * u + (t - 3)] = gslot;
                }
            }
            A.slot_ptr[k + 1] = (int)A.slot_var.size();
        }
        if (!closure_ok) return "measurement row references a bus outside its area's variable map";
        slot_cursor += (int64_t)A.slot_var.size();
        for (int b : touched) { loc_va[b] = -1; loc_vm[b] = -1; }
        sec(0);
    }

    // ---- per area, on a few threads: reference-layout patterns and the nested dissection ----
    // (both read only the area's own template layout and write only the area's own outputs)
    std::vector<std::vector<std::vector<int>>> nodes_of(K);   // per area: tree nodes, each a list of interior bus indices
    parallel_for(K, build_threads(), [&](int a) {
        AreaSym& A = as[a];
        const int ni = A.ni, nb = A.nb;
        const int nib = d.im_ptr[a + 1] - d.im_ptr[a];
        // ---- reference-layout CSR patterns of G_ii, G_ib ------------------------------
        // (per interior variable: the sorted, de-duplicated columns its rows reach)
        if (opt.ext_pattern) {      // generic matrix plan: the caller supplies the patterns
            hp.ii_ptr[a] = opt.ext_ii_ptr; hp.ii_idx[a] = opt.ext_ii_idx;
            hp.ib_ptr[a] = opt.ext_ib_ptr; hp.ib_idx[a] = opt.ext_ib_idx;
        } else {
            // rows of every interior variable (CSR), then per variable one stamped sweep over the
            // slots of its rows: each distinct column is collected once, and only those are sorted
            std::vector<int> vr_ptr(ni + 1, 0), vr_row;
            for (int x : A.slot_var) if (x < ni) vr_ptr[x + 1]++;
            for (int v = 0; v < ni; ++v) vr_ptr[v + 1] += vr_ptr[v];
            vr_row.resize(vr_ptr[ni]);
            {
                std::vector<int> cur(vr_ptr.begin(), vr_ptr.end() - 1);
                for (size_t k = 0; k < A.rows.size(); ++k)
                    for (int x = A.slot_ptr[k]; x < A.slot_ptr[k + 1]; ++x)
                        if (A.slot_var[x] < ni) vr_row[cur[A.slot_var[x]]++] = (int)k;
            }
            std::vector<int> mark(ni + nb, -1), cols;
            hp.ii_ptr[a].assign(ni + 1, 0); hp.ib_ptr[a].assign(ni + 1, 0);
            for (int v = 0; v < ni; ++v) {
                cols.clear();
                for (int q = vr_ptr[v]; q < vr_ptr[v + 1]; ++q) {
                    const int k = vr_row[q];
                    for (int y = A.slot_ptr[k]; y < A.slot_ptr[k + 1]; ++y) {
                        const int vb = A.slot_var[y];
                        if (mark[vb] != v) { mark[vb] = v; cols.push_back(vb); }
                    }
                }
                std::sort(cols.begin(), cols.end());
                const auto mid = std::lower_bound(cols.begin(), cols.end(), ni);
                hp.ii_idx[a].insert(hp.ii_idx[a].end(), cols.begin(), mid);
                for (auto it = mid; it != cols.end(); ++it) hp.ib_idx[a].push_back(*it - ni);
                hp.ii_ptr[a][v + 1] = (int32_t)hp.ii_idx[a].size();
                hp.ib_ptr[a][v + 1] = (int32_t)hp.ib_idx[a].size();
            }
        }
        // ---- ordering of the interior: nested dissection on the bus graph ----------------
        std::vector<std::vector<int>>& nodes = nodes_of[a];   // each: interior bus indices, in elimination order
        if (!hp.owned[a]) return;
        if (opt.dense || ni <= PMAX) {
            std::vector<int> all(nib); std::iota(all.begin(), all.end(), 0);
            if (nib) nodes.push_back(all);
        } else {
            NDGraph g;
            // bus graph from the G_ii pattern
            std::vector<int64_t> edges;
            for (int u = 0; u < ni; ++u)
                for (int p = hp.ii_ptr[a][u]; p < hp.ii_ptr[a][u + 1]; ++p) {
                    int bu = A.var_bus[u], bv = A.var_bus[hp.ii_idx[a][p]];
                    if (bu != bv) edges.push_back((int64_t)bu * nib + bv);
                }
            std::sort(edges.begin(), edges.end()); edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
            g.xadj.assign(nib + 1, 0); g.adj.resize(edges.size());
            for (size_t i = 0; i < edges.size(); ++i) { g.xadj[edges[i] / nib + 1]++; g.adj[i] = (int)(edges[i] % nib); }
            for (int i = 0; i < nib; ++i) g.xadj[i + 1] += g.xadj[i];
            g.stamp.assign(nib, 0); g.level.assign(nib, 0);
            g.sep_weight = opt.sep_weight;
            std::vector<int> all(nib); std::iota(all.begin(), all.end(), 0);
            nd_recurse(g, all, std::max(1, opt.leaf_buses), nodes);
            if (opt.interior_merge > 0.0) {
                // boundary variables coupled to each interior bus (they belong to the update structure of its front)
                std::vector<std::vector<int>> ext(nib);
                for (int u = 0; u < ni; ++u)
                    for (int p = hp.ib_ptr[a][u]; p < hp.ib_ptr[a][u + 1]; ++p) ext[A.var_bus[u]].push_back(hp.ib_idx[a][p]);
                for (auto& e : ext) { std::sort(e.begin(), e.end()); e.erase(std::unique(e.begin(), e.end()), e.end()); }
                amalgamate_nodes(nodes, nib, g.xadj, g.adj, &ext,
                                 [&](const std::vector<int>& node) { int c = 0; for (int b : node) c += 1 + (A.th_var[b] >= 0); return c; }, PMAX,
                                 opt.interior_merge);
            }
        }
    });
    sec(1);

    for (int a = 0; a < K; ++a) {
        AreaSym& A = as[a];
        const int ni = A.ni, nb = A.nb;
        const int n_ia = d.ia_ptr[a + 1] - d.ia_ptr[a];
        const int n_ba = d.ba_ptr[a + 1] - d.ba_ptr[a];
        const int nib = d.im_ptr[a + 1] - d.im_ptr[a];
        (void)n_ia; (void)n_ba; (void)nib;
        // ref value layout of the area: [data_ii | data_ib | g_bb | b_i | b_b]
        hp.ref_off[a + 1] = hp.ref_off[a] + (int64_t)hp.ii_idx[a].size() + (int64_t)hp.ib_idx[a].size() + (int64_t)nb * nb + ni + nb;
        nnz_total += (double)hp.ii_idx[a].size() + (double)hp.ib_idx[a].size() + (double)nb * nb; rhs_total += ni + nb;
        // template layout kept for the (lazily built) reference-layout program
        hp.tmpl_rows.push_back(A.rows); hp.tmpl_slot_ptr.push_back(A.slot_ptr); hp.tmpl_slot_var.push_back(A.slot_var);
        hp.tmpl_slot_base.push_back(A.slot_base);

        // ---- fronts of the interior, in the order found above ----------------------------
        A.epos.assign(ni, -1); A.order.assign(ni, -1);
        int ep = 0;
        A.first_front = (int)hp.fronts.size();
        A.front_of_pos.assign(ni, -1);
        if (!hp.owned[a]) {
            for (int v = 0; v < ni; ++v) { A.epos[v] = v; A.order[v] = v; }
            ep = ni;
        } else {
        std::vector<std::vector<int>>& nodes = nodes_of[a];
        // nodes -> fronts of at most PMAX pivots
        for (auto& node : nodes) {
            std::vector<int> vars;
            for (int b : node) { if (A.th_var[b] >= 0) vars.push_back(A.th_var[b]); vars.push_back(A.vm_var[b]); }
            int nv = (int)vars.size();
            int pieces = (nv + PMAX - 1) / PMAX;
            for (int q = 0; q < pieces; ++q) {
                int lo = piece_cut(nv, pieces, q, PMAX), hi = piece_cut(nv, pieces, q + 1, PMAX);
                Front f; f.area = a; f.kind = 0; f.p = hi - lo;
                for (int i = lo; i < hi; ++i) {
                    A.epos[vars[i]] = ep; A.order[ep] = vars[i];
                    A.front_of_pos[ep] = (int)hp.fronts.size();
                    f.rows.push_back(hp.area_base[a] + ep);
                    hp.perm_orig[hp.area_base[a] + ep] = vars[i];
                    ++ep;
                }
                hp.fronts.push_back(std::move(f));
            }
        }
        }
        if (ep != ni) return "ordering did not cover the interior";
        A.n_fronts = (int)hp.fronts.size() - A.first_front;

        sec(2);
        // ---- lower-triangular pattern in position space ------------------------------
        const int nloc = ni + nb;
        auto lpos = [&](int v) { return v < ni ? A.epos[v] : v; };
        std::vector<std::vector<int>> colrows(nloc);
        if (hp.owned[a]) {
            for (int u = 0; u < ni; ++u) {
                for (int p = hp.ii_ptr[a][u]; p < hp.ii_ptr[a][u + 1]; ++p) {
                    int v = hp.ii_idx[a][p];
                    if (A.epos[u] >= A.epos[v]) colrows[A.epos[v]].push_back(A.epos[u]);
                }
                for (int p = hp.ib_ptr[a][u]; p < hp.ib_ptr[a][u + 1]; ++p) colrows[A.epos[u]].push_back(ni + hp.area_bpos[a][hp.ib_idx[a][p]]);
            }
            if (opt.dense) for (int c = 0; c < ni; ++c) { colrows[c].clear(); for (int r = c; r < nloc; ++r) colrows[c].push_back(r); }
            for (int c = ni; c < nloc; ++c) for (int r = c; r < nloc; ++r) colrows[c].push_back(r);
            A.col_ptr.assign(nloc + 1, 0);
            for (int c = 0; c < nloc; ++c) {
                std::sort(colrows[c].begin(), colrows[c].end());
                colrows[c].push_back(nloc);   // RHS row
                A.col_ptr[c + 1] = A.col_ptr[c] + (int)colrows[c].size();
            }
            A.col_row.reserve(A.col_ptr[nloc]);
            for (int c = 0; c < nloc; ++c) A.col_row.insert(A.col_row.end(), colrows[c].begin(), colrows[c].end());
            A.col_dest.assign(A.col_row.size(), -1);
        }
        (void)lpos;

        sec(3);
        // ---- update sets + assembly tree of the interior fronts ---------------------
        std::vector<std::vector<int>> structs(A.n_fronts);   // local positions (>= pivots' end), sorted
        std::vector<int> mark(nloc, -1);
        // area root
        Front root; root.area = a; root.kind = 1; root.p = 0; root.u1 = nb + 1;
        for (int q = 0; q < nb; ++q) root.rows.push_back(hp.gamma_base + d.sel[d.sel_ptr[a] + bvar_of_pos[a][q]]);
        const int root_id = A.first_front + A.n_fronts;
        A.root = root_id;
        std::vector<std::vector<int>> kids(A.n_fronts + 1);
        int e0 = 0;
        for (int fi = 0; fi < A.n_fronts; ++fi) {
            Front& f = hp.fronts[A.first_front + fi];
            const int e1 = e0 + f.p;
            std::vector<int>& st = structs[fi];
            for (int c = e0; c < e1; ++c)
                for (int q = A.col_ptr[c]; q < A.col_ptr[c + 1] - 1; ++q) {
                    int r = A.col_row[q];
                    if (r >= e1 && mark[r] != fi) { mark[r] = fi; st.push_back(r); }
                }
            for (int ch : kids[fi])
                for (int r : structs[ch]) if (r >= e1 && mark[r] != fi) { mark[r] = fi; st.push_back(r); }
            std::sort(st.begin(), st.end());
            f.u1 = (int)st.size() + 1;
            for (int r : st) f.rows.push_back(r < ni ? hp.area_base[a] + r : hp.gamma_base + d.sel[d.sel_ptr[a] + bvar_of_pos[a][r - ni]]);
            int par = A.n_fronts;   // area root by default
            if (!st.empty() && st[0] < ni) par = A.front_of_pos[st[0]] - A.first_front;
            kids[par].push_back(fi);
            f.parent = A.first_front + par;
            e0 = e1;
        }
        if (hp.owned[a]) {
            // rel maps child -> parent
            e0 = 0;
            std::vector<int> e_start(A.n_fronts + 1, 0);
            for (int fi = 0; fi < A.n_fronts; ++fi) e_start[fi + 1] = e_start[fi] + hp.fronts[A.first_front + fi].p;
            for (int fi = 0; fi < A.n_fronts; ++fi) {
                Front& f = hp.fronts[A.first_front + fi];
                int par = f.parent - A.first_front;
                const std::vector<int>& st = structs[fi];
                f.rel.resize(f.u1);
                if (par == A.n_fronts) {
                    for (size_t i = 0; i < st.size(); ++i) f.rel[i] = st[i] - ni;
                    f.rel[f.u1 - 1] = nb;
                } else {
                    Front& P = hp.fronts[A.first_front + par];
                    const std::vector<int>& ps = structs[par];
                    int pe0 = e_start[par], pe1 = e_start[par + 1];
                    for (size_t i = 0; i < st.size(); ++i) {
                        int r = st[i];
                        if (r < pe1) { if (r < pe0) return "internal: child row precedes parent pivots"; f.rel[i] = r - pe0; }
                        else {
                            auto it = std::lower_bound(ps.begin(), ps.end(), r);
                            if (it == ps.end() || *it != r) return "internal: update row missing in parent front";
                            f.rel[i] = P.p + (int)(it - ps.begin());
                        }
                    }
                    f.rel[f.u1 - 1] = P.p + P.u1 - 1;
                }
            }
            for (int fi = 0; fi < A.n_fronts; ++fi) {
                Front& f = hp.fronts[A.first_front + fi];
                for (int ch : kids[fi]) f.children.push_back(A.first_front + ch);
            }
            for (int ch : kids[A.n_fronts]) root.children.push_back(A.first_front + ch);
        }
        hp.fronts.push_back(std::move(root));
        hp.area_root.push_back(root_id);

        // stash structs for the entry layout below
        if (hp.owned[a]) {
            // ---- front-major, region-sorted layout of the original entries -------------
            std::vector<int> e_start(A.n_fronts + 1, 0);
            for (int fi = 0; fi < A.n_fronts; ++fi) e_start[fi + 1] = e_start[fi] + hp.fronts[A.first_front + fi].p;
            for (int fi = 0; fi <= A.n_fronts; ++fi) {
                Front& f = hp.fronts[A.first_front + fi];
                choose_chunks(f, opt.tile_rows);
                const bool is_root = fi == A.n_fronts;
                const int c0 = is_root ? ni : e_start[fi], c1 = is_root ? nloc : e_start[fi + 1];
                const std::vector<int>* st = is_root ? nullptr : &structs[fi];
                auto local_row = [&](int r) -> int {
                    if (r == nloc) return f.p + f.u1 - 1;
                    if (is_root) return r - ni;
                    if (r < c1) return r - c0;
                    return f.p + (int)(std::lower_bound(st->begin(), st->end(), r) - st->begin());
                };
                auto chunk_of = [&](int lr) { return lr < f.p ? 0 : 1 + (lr - f.p) / f.T; };
                struct Ent { int reg; uint32_t pos; int q; };
                std::vector<Ent> ents;
                for (int c = c0; c < c1; ++c)
                    for (int q = A.col_ptr[c]; q < A.col_ptr[c + 1]; ++q) {
                        int lr = local_row(A.col_row[q]), lc = is_root ? c - ni : c - c0;
                        int rc = chunk_of(lr), cc = is_root ? 1 + lc / f.T : 0;
                        if (is_root && rc < cc) return "internal: upper entry in root";
                        ents.push_back({rc * (rc + 1) / 2 + cc, ((uint32_t)lr << 16) | (uint32_t)lc, q});
                    }
                std::stable_sort(ents.begin(), ents.end(), [](const Ent& x, const Ent& y) { return x.reg < y.reg; });
                const int nreg = (f.nch + 1) * (f.nch + 2) / 2;
                hp.front_reg_off.resize(hp.fronts.size(), 0);
                hp.front_reg_off[A.first_front + fi] = (int32_t)hp.reg_ptr.size();
                f.gval_off = hp.n_gval; f.n_orig = (int)ents.size();
                std::vector<int32_t> rp(nreg + 1, 0);
                for (auto& e : ents) rp[e.reg + 1]++;
                for (int i = 0; i < nreg; ++i) rp[i + 1] += rp[i];
                hp.reg_ptr.insert(hp.reg_ptr.end(), rp.begin(), rp.end());
                for (size_t i = 0; i < ents.size(); ++i) { hp.orig_pos.push_back(ents[i].pos); A.col_dest[ents[i].q] = hp.n_gval + (int64_t)i; }
                hp.n_gval += (int64_t)ents.size();
            }
            if (opt.ext_pattern) {
                // where every original entry comes from, as an index into the caller's value layout
                // [data_ii | data_ib | g_bb (row-major) | b_i | b_b]  (AreaNormalBlocks, assembly.py:32-53)
                const int64_t o_ib = (int64_t)hp.ii_idx[a].size(), o_bb = o_ib + (int64_t)hp.ib_idx[a].size();
                const int64_t o_bi = o_bb + (int64_t)nb * nb, o_bbv = o_bi + ni;
                hp.gval_src.assign((size_t)hp.n_gval, -1);
                auto find = [](const std::vector<int32_t>& ptr, const std::vector<int32_t>& idx, int r, int c) -> int64_t {
                    auto b = idx.begin() + ptr[r], e = idx.begin() + ptr[r + 1];
                    auto it = std::lower_bound(b, e, c);
                    return (it == e || *it != c) ? -1 : (int64_t)(it - idx.begin());
                };
                for (int c = 0; c < nloc; ++c)
                    for (int q = A.col_ptr[c]; q < A.col_ptr[c + 1]; ++q) {
                        const int r = A.col_row[q];
                        const int64_t dst = A.col_dest[q];
                        if (dst < 0) continue;
                        int64_t src;
                        if (c < ni) {
                            const int uc = A.order[c];
                            if (r == nloc) src = o_bi + uc;
                            else if (r < ni) src = find(hp.ii_ptr[a], hp.ii_idx[a], A.order[r], uc);
                            else { const int64_t f = find(hp.ib_ptr[a], hp.ib_idx[a], uc, bvar_of_pos[a][r - ni]); src = f < 0 ? -1 : o_ib + f; }
                        } else {
                            const int bc = bvar_of_pos[a][c - ni];
                            if (r == nloc) src = o_bbv + bc;
                            else src = o_bb + (int64_t)bvar_of_pos[a][r - ni] * nb + bc;
                        }
                        hp.gval_src[(size_t)dst] = src;
                    }
            }
        } else {
            choose_chunks(hp.fronts[root_id], opt.tile_rows);
        }
        sec(4);
    }
    hp.n_slots = slot_cursor;
    if (dbg_time) fprintf(stderr, "  plan build (areas): slots/units %.3f  patterns+dissection (threads) %.3f  fronts %.3f  lower pattern %.3f  update sets+entries %.3f\n",
                          t_sec[0], t_sec[1], t_sec[2], t_sec[3], t_sec[4]);

    lap("areas: slots, patterns, fronts");
    // ---- coordinator fronts: boundary assembly root + dense factorisation chain -----
    const int first_coord = (int)hp.fronts.size();
    if (ng > 0 && sparse_gamma) {
        // rel of every area root into the boundary root (rows in boundary elimination order)
        std::vector<std::vector<int>> root_rel(K);
        for (int a = 0; a < K; ++a) {
            root_rel[a].resize(as[a].nb + 1);
            for (int q = 0; q < as[a].nb; ++q) root_rel[a][q] = hp.gamma_epos[d.sel[d.sel_ptr[a] + bvar_of_pos[a][q]]];
            root_rel[a][as[a].nb] = ng;
            hp.fronts[hp.area_root[a]].parent = -1;
        }
        if (coordinator) {
            // boundary root: S_Gamma / b_Gamma for readback only (not part of the solve in this mode)
            Front g; g.kind = 2; g.p = 0; g.u1 = ng + 1;
            for (int q = 0; q < ng; ++q) g.rows.push_back(hp.gamma_base + gamma_slot_of_rank[q]);
            for (int a = 0; a < K; ++a) { g.children.push_back(hp.area_root[a]); g.child_rel.push_back((int)hp.extra_rel.size()); hp.extra_rel.push_back(root_rel[a]); }
            choose_chunks(g, opt.tile_rows);
            hp.gamma_root = first_coord;
            hp.fronts.push_back(std::move(g));
            // fronts of the boundary tree: ND nodes cut into pieces of at most PMAX pivots
            const int first_gf = (int)hp.fronts.size();
            std::vector<int> front_of_rank(ng, -1), e_lo, e_hi;
            for (auto& slots : gamma_nodes) {
                const int nv = (int)slots.size(), pieces = (nv + PMAX - 1) / PMAX;
                for (int q = 0; q < pieces; ++q) {
                    const int lo = piece_cut(nv, pieces, q, PMAX), hi = piece_cut(nv, pieces, q + 1, PMAX);
                    Front f; f.kind = 3; f.p = hi - lo;
                    e_lo.push_back(hp.gamma_epos[slots[lo]]); e_hi.push_back(hp.gamma_epos[slots[lo]] + (hi - lo));
                    for (int i = lo; i < hi; ++i) { front_of_rank[hp.gamma_epos[slots[i]]] = (int)hp.fronts.size(); f.rows.push_back(hp.gamma_base + slots[i]); }
                    hp.fronts.push_back(std::move(f));
                }
            }
            const int ngf = (int)hp.fronts.size() - first_gf;
            // cliques (areas) containing each rank
            std::vector<std::vector<int>> areas_of_rank(ng);
            for (int a = 0; a < K; ++a) for (int q = 0; q < as[a].nb; ++q) areas_of_rank[root_rel[a][q]].push_back(a);
            std::vector<std::vector<int>> gstruct(ngf), gkids(ngf);
            std::vector<int> gmark(ng, -1);
            for (int fi = 0; fi < ngf; ++fi) {
                Front& f = hp.fronts[first_gf + fi];
                std::vector<int>& st = gstruct[fi];
                for (int e = e_lo[fi]; e < e_hi[fi]; ++e)
                    for (int a : areas_of_rank[e])
                        for (int q = 0; q < as[a].nb; ++q) { int r = root_rel[a][q]; if (r >= e_hi[fi] && gmark[r] != fi) { gmark[r] = fi; st.push_back(r); } }
                for (int ch : gkids[fi]) for (int r : gstruct[ch]) if (r >= e_hi[fi] && gmark[r] != fi) { gmark[r] = fi; st.push_back(r); }
                std::sort(st.begin(), st.end());
                f.u1 = (int)st.size() + 1;
                for (int r : st) f.rows.push_back(hp.gamma_base + gamma_slot_of_rank[r]);
                if (!st.empty()) { int par = front_of_rank[st[0]] - first_gf; gkids[par].push_back(fi); f.parent = first_gf + par; }
                choose_chunks(f, opt.gamma_tile_rows > 0 ? opt.gamma_tile_rows : opt.tile_rows);
            }
            auto local_index = [&](int fi, int r) -> int {   // rank r inside front fi: pivots then update rows
                if (r < e_hi[fi]) return r - e_lo[fi];
                const std::vector<int>& st = gstruct[fi];
                return hp.fronts[first_gf + fi].p + (int)(std::lower_bound(st.begin(), st.end(), r) - st.begin());
            };
            for (int fi = 0; fi < ngf; ++fi) {
                Front& f = hp.fronts[first_gf + fi];
                for (int ch : gkids[fi]) f.children.push_back(first_gf + ch);
                if (f.parent >= 0) {
                    const int par = f.parent - first_gf;
                    f.rel.resize(f.u1);
                    for (size_t i = 0; i < gstruct[fi].size(); ++i) f.rel[i] = local_index(par, gstruct[fi][i]);
                    f.rel[f.u1 - 1] = hp.fronts[f.parent].p + hp.fronts[f.parent].u1 - 1;
                }
            }
            // every area root enters the front of its first-eliminated boundary variable
            for (int a = 0; a < K; ++a) {
                Front& r = hp.fronts[hp.area_root[a]];
                if (as[a].nb == 0) continue;
                const int fi = front_of_rank[root_rel[a][0]] - first_gf;
                r.parent = first_gf + fi;
                r.rel.resize(r.u1);
                for (int q = 0; q < as[a].nb; ++q) r.rel[q] = local_index(fi, root_rel[a][q]);
                r.rel[r.u1 - 1] = hp.fronts[r.parent].p + hp.fronts[r.parent].u1 - 1;
                // children stay in area order: the reference's summation order of assemble_boundary
                hp.fronts[r.parent].children.push_back(hp.area_root[a]);
            }
            for (int fi = 0; fi < ngf; ++fi) {   // area roots first (area order), then boundary-tree children
                Front& f = hp.fronts[first_gf + fi];
                std::stable_sort(f.children.begin(), f.children.end(), [&](int x, int y) {
                    return (hp.fronts[x].kind == 1) > (hp.fronts[y].kind == 1); });
            }
        }
    } else if (ng > 0) {
        for (int a = 0; a < K; ++a) {
            Front& r = hp.fronts[hp.area_root[a]];
            r.parent = first_coord;
            r.rel.resize(r.u1);
            for (int j = 0; j < as[a].nb; ++j) r.rel[j] = d.sel[d.sel_ptr[a] + j];
            r.rel[r.u1 - 1] = ng;
        }
        if (coordinator) {
            Front g; g.kind = 2; g.p = 0; g.u1 = ng + 1;
            for (int s = 0; s < ng; ++s) g.rows.push_back(hp.gamma_base + s);
            for (int a = 0; a < K; ++a) g.children.push_back(hp.area_root[a]);
            g.parent = first_coord + 1;
            g.rel.resize(g.u1); std::iota(g.rel.begin(), g.rel.end(), 0);
            choose_chunks(g, opt.tile_rows);
            hp.gamma_root = first_coord;
            hp.fronts.push_back(std::move(g));
            int nchain = (ng + PMAX - 1) / PMAX;
            for (int k = 0; k < nchain; ++k) {
                int lo = (int)((int64_t)ng * k / nchain), hi = (int)((int64_t)ng * (k + 1) / nchain);
                Front c; c.kind = 3; c.p = hi - lo; c.u1 = ng - hi + 1;
                for (int s = lo; s < ng; ++s) c.rows.push_back(hp.gamma_base + s);
                c.children.push_back((int)hp.fronts.size() - 1);
                c.parent = k + 1 < nchain ? (int)hp.fronts.size() + 1 : -1;
                c.rel.resize(c.u1); std::iota(c.rel.begin(), c.rel.end(), 0);
                choose_chunks(c, opt.tile_rows);
                hp.fronts.push_back(std::move(c));
            }
        } else {
            for (int a = 0; a < K; ++a) hp.fronts[hp.area_root[a]].parent = -1;
        }
    }
    for (int s = 0; s < ng; ++s) hp.perm_orig[hp.gamma_base + s] = s;
    hp.front_reg_off.resize(hp.fronts.size(), 0);
    for (size_t f = 0; f < hp.fronts.size(); ++f)
        if (hp.fronts[f].kind >= 2) {   // no original entries: an all-empty region table
            hp.front_reg_off[f] = (int32_t)hp.reg_ptr.size();
            int nreg = (hp.fronts[f].nch + 1) * (hp.fronts[f].nch + 2) / 2;
            hp.reg_ptr.insert(hp.reg_ptr.end(), nreg + 1, 0);
        }

    lap("coordinator fronts");
    // ---- storage offsets ----------------------------------------------------------------
    // update matrices: area roots first, contiguous in area order (the exchange buffer)
    hp.xchg_off = 0; hp.xchg_area_off.assign(K + 1, 0);
    int64_t ucur = 0;
    for (int a = 0; a < K; ++a) {
        Front& r = hp.fronts[hp.area_root[a]];
        r.u_off = ucur; hp.xchg_area_off[a] = ucur;
        ucur += (int64_t)r.u1 * (r.u1 + 1) / 2;
    }
    hp.xchg_area_off[K] = ucur; hp.xchg_len = ucur;
    int64_t lcur = 0;
    for (auto& f : hp.fronts) {
        if (f.kind != 1) { f.u_off = ucur; ucur += (int64_t)f.u1 * (f.u1 + 1) / 2; }
        f.l_off = lcur; lcur += ((int64_t)(f.p + f.u1) * f.p + 1) & ~(int64_t)1;   // even: 16-byte cp.async of the pivot block
        hp.max_front = std::max(hp.max_front, f.p + f.u1);
        double p = f.p, u = f.u1;
        hp.dense_flops += p * p * p / 3.0 + p * p * u + p * u * u;
    }
    hp.n_ubuf = ucur; hp.n_lbuf = lcur;

    // ---- levels + tasks -------------------------------------------------------------------
    int max_interior = -1;
    for (auto& f : hp.fronts) if (f.kind == 0) {
        int lv = 0;
        for (int c : f.children) lv = std::max(lv, hp.fronts[c].level + 1);
        f.level = lv; max_interior = std::max(max_interior, lv);
    }
    const int root_level = max_interior + 1;
    int n_levels = root_level + 1;
    for (auto& f : hp.fronts) {
        if (f.kind == 1) f.level = root_level;
        else if (f.kind == 2) { f.level = root_level + 1; n_levels = std::max(n_levels, f.level + 1); }
    }
    // boundary fronts (chain or tree): one level above their deepest child
    for (auto& f : hp.fronts) if (f.kind == 3) {
        int lv = root_level + 1;
        for (int c : f.children) lv = std::max(lv, hp.fronts[c].level + 1);
        f.level = lv; n_levels = std::max(n_levels, lv + 1);
    }
    // Child order = summation order of the extend-add.  The dataflow kernel folds a child's update
    // matrix in as soon as that child is complete while it still waits for the next one, so children
    // are ordered by the length of the pivot chain below them (the proxy for when they finish): the
    // slowest subtree comes last.  Area roots stay first and in area order (assemble_boundary's order).
    {
        std::vector<int> by_level(hp.fronts.size());
        std::iota(by_level.begin(), by_level.end(), 0);
        std::stable_sort(by_level.begin(), by_level.end(), [&](int a, int b) { return hp.fronts[a].level < hp.fronts[b].level; });
        std::vector<int64_t> chain(hp.fronts.size(), 0);
        for (int fi : by_level) {
            Front& f = hp.fronts[fi];
            if ((f.kind == 0 || f.kind == 3) && f.child_rel.empty())
                std::stable_sort(f.children.begin(), f.children.end(), [&](int a, int b) {
                    const int64_t ka = hp.fronts[a].kind == 1 ? -1 : chain[a], kb = hp.fronts[b].kind == 1 ? -1 : chain[b];
                    return ka < kb; });
            int64_t c = 0;
            for (int ch : f.children) c = std::max(c, chain[ch]);
            chain[fi] = c + f.p + 8;       // + a per-front overhead (hand-off, gather) in pivot units
        }
    }
    hp.fwd_levels.assign(n_levels, {}); hp.level_phase.assign(n_levels, 1);
    for (size_t fi = 0; fi < hp.fronts.size(); ++fi) {
        Front& f = hp.fronts[fi];
        if (f.area >= 0 && !hp.owned[f.area]) continue;
        // phase 1 local_condense, 2 boundary_assemble, 3 boundary_solve, 5 readback-only boundary root
        const int phase = f.kind <= 1 ? 1 : f.kind == 2 ? (sparse_gamma ? 5 : 2) : 3;
        // wide fronts: one panel task per row chunk (factor + solve, stored) and one update task per
        // tile (reads the stored panels) instead of tasks that each redo the pivot block
        const bool split = f.p > 0 && f.nch >= 2 && f.p >= opt.split_min_pivots && f.nch * (f.nch + 1) / 2 >= opt.split_min_tasks;
        if (split) for (int ci = 0; ci < f.nch; ++ci) hp.fwd_levels[f.level].push_back({(int)fi, ci, ci, phase, 1});
        for (int ci = 0; ci < f.nch; ++ci) for (int cj = 0; cj <= ci; ++cj) hp.fwd_levels[f.level].push_back({(int)fi, ci, cj, phase, split ? 2 : 0});
        hp.level_phase[f.level] = phase;
    }
    // within a level: panel and fused tasks, then the update tasks.  Most critical first: when a level has more tasks
    // than resident CTAs (the leaf levels), the ones left for the second wave should be the ones with the shortest way
    // to the root -- remaining chain = estimated time from the front's start to the end of the factorisation along
    // its ancestors (per front ~6 us of hand-off, gather and update plus 1 us per 8-pivot block of the panel).
    // GSE_TASK_ORDER=size restores largest-first.
    std::vector<double> remaining(hp.fronts.size(), 0.0);
    {
        std::vector<int> by_level(hp.fronts.size());
        std::iota(by_level.begin(), by_level.end(), 0);
        std::stable_sort(by_level.begin(), by_level.end(), [&](int a, int b) { return hp.fronts[a].level > hp.fronts[b].level; });
        for (int fi : by_level) {
            const Front& f = hp.fronts[fi];
            const double cost = f.p > 0 ? 6.0 + (f.p + 7) / 8 : 3.0;
            remaining[fi] = cost + (f.parent >= 0 ? remaining[f.parent] : 0.0);
        }
    }
    const char* order_env = getenv("GSE_TASK_ORDER");
    const bool by_size = order_env && !strcmp(order_env, "size");
    for (auto& lv : hp.fwd_levels)
        std::stable_sort(lv.begin(), lv.end(), [&](const Task& x, const Task& y) {
            if ((x.kind == 2) != (y.kind == 2)) return y.kind == 2;
            const Front& a = hp.fronts[x.front]; const Front& b = hp.fronts[y.front];
            if (!by_size && remaining[x.front] != remaining[y.front]) return remaining[x.front] > remaining[y.front];
            return (int64_t)a.p * (a.p + a.u1) > (int64_t)b.p * (b.p + b.u1); });
    // back-substitution, top-down; within a level the fronts with the longest chain of fronts BELOW them first (the
    // mirror of the forward order: what is left for a second wave should be what finishes the iteration soonest)
    std::vector<double> below(hp.fronts.size(), 0.0);
    {
        std::vector<int> by_level(hp.fronts.size());
        std::iota(by_level.begin(), by_level.end(), 0);
        std::stable_sort(by_level.begin(), by_level.end(), [&](int a, int b) { return hp.fronts[a].level < hp.fronts[b].level; });
        for (int fi : by_level) {
            const Front& f = hp.fronts[fi];
            double c = 0.0;
            for (int ch : f.children) c = std::max(c, below[ch]);
            below[fi] = c + (f.p > 0 ? 3.0 + f.p / 40.0 : 0.0);
        }
    }
    for (int lv = n_levels - 1; lv >= 0; --lv) {
        std::vector<int> fs; int phase = 4;
        for (size_t fi = 0; fi < hp.fronts.size(); ++fi) {
            const Front& f = hp.fronts[fi];
            if (f.level != lv || f.p == 0) continue;
            if (f.area >= 0 && !hp.owned[f.area]) continue;
            fs.push_back((int)fi); if (f.kind == 3) phase = 3;
        }
        if (!by_size) std::stable_sort(fs.begin(), fs.end(), [&](int a, int b) { return below[a] > below[b]; });
        if (!fs.empty()) { hp.bwd_levels.push_back(fs); hp.bwd_phase.push_back(phase); }
    }

    lap("offsets, levels, tasks");
    // ---- solver-layout accumulation program ---------------------------------------------
    // Every contribution is a product val[a] * val[b] of the unified value array
    // val = [(g, w*g) per slot, interleaved | w*r (n_rows)]: a indexes g, b indexes w*g (matrix
    // entries) or w*r of the row (right-hand sides, collected above as -(row + 1)).
    hp.n_val = 2 * hp.n_slots + m;
    if (hp.n_val > 2147483647LL) return "value array exceeds int32 indexing";
    auto val_index = [&](int32_t b) { return b >= 0 ? (int32_t)(2 * b + 1) : (int32_t)(2 * hp.n_slots + (-b - 1)); };
    {
        // pairs of every area on its own thread (read-only plan data, private output), in area order below
        struct AreaPairs { std::vector<int64_t> dest; std::vector<int32_t> pa, pb; bool bad = false; int64_t lo = INT64_MAX, hi = -1; };
        std::vector<AreaPairs> ap(K);
        const int nthreads = build_threads();
        parallel_for(K, nthreads, [&](int a) {
            if (!hp.owned[a]) return;
            const AreaSym& A = as[a];
            AreaPairs& out = ap[a];
            const int ni = A.ni, nloc = A.ni + A.nb;
            auto lp = [&](int v) { return v < ni ? A.epos[v] : ni + hp.area_bpos[a][v - ni]; };
            auto find = [&](int c, int r) -> int64_t {
                auto b = A.col_row.begin() + A.col_ptr[c], e = A.col_row.begin() + A.col_ptr[c + 1];
                auto it = std::lower_bound(b, e, r);
                return (it == e || *it != r) ? -1 : A.col_dest[it - A.col_row.begin()];
            };
            size_t np = 0;
            for (size_t k = 0; k < A.rows.size(); ++k) { const size_t sl = A.slot_ptr[k + 1] - A.slot_ptr[k]; np += sl * (sl + 1) / 2 + sl; }
            out.dest.reserve(np); out.pa.reserve(np); out.pb.reserve(np);
            std::vector<int> pos;
            for (size_t k = 0; k < A.rows.size(); ++k) {
                int s0 = A.slot_ptr[k], s1 = A.slot_ptr[k + 1];
                pos.resize(s1 - s0);
                for (int x = s0; x < s1; ++x) pos[x - s0] = lp(A.slot_var[x]);
                for (int x = s0; x < s1; ++x) {
                    int ra_ = pos[x - s0];
                    for (int y = s0; y < s1; ++y) {
                        int cb = pos[y - s0];
                        if (ra_ < cb) continue;
                        int64_t dd = find(cb, ra_);
                        if (dd < 0) { out.bad = true; return; }
                        out.dest.push_back(dd); out.pa.push_back((int32_t)(A.slot_base + x)); out.pb.push_back((int32_t)(A.slot_base + y));
                    }
                }
                for (int x = s0; x < s1; ++x) {
                    int64_t dd = find(pos[x - s0], nloc);
                    if (dd < 0) { out.bad = true; return; }
                    out.dest.push_back(dd); out.pa.push_back((int32_t)(A.slot_base + x)); out.pb.push_back(-(A.rows[k] + 1));
                }
            }
            for (int64_t dd : out.dest) { out.lo = std::min(out.lo, dd); out.hi = std::max(out.hi, dd); }
        });
        lap("  acc program: pairs per area (threads)");
        int64_t n_pairs = 0;
        for (int a = 0; a < K; ++a) { if (ap[a].bad) return "internal: pair without a destination"; n_pairs += (int64_t)ap[a].dest.size(); }
        if (n_pairs > 2147483647LL) return "contribution program exceeds int32 indexing";
        hp.n_pairs = n_pairs;
        // stable counting sort by destination keeps ascending-row order per slot (areas in order)
        hp.acc_ptr.assign(hp.n_gval + 1, 0);
        for (int a = 0; a < K; ++a) for (int64_t dd : ap[a].dest) hp.acc_ptr[dd + 1]++;
        for (int64_t i = 0; i < hp.n_gval; ++i) hp.acc_ptr[i + 1] += hp.acc_ptr[i];
        hp.acc_a.resize((size_t)n_pairs); hp.acc_b.resize((size_t)n_pairs);
        std::vector<int32_t> cur(hp.acc_ptr.begin(), hp.acc_ptr.end() - 1);
        // the destination ranges of distinct areas are disjoint (every entry lives in a front of its
        // area), so the scatter of an area touches only its own cursors; checked, serial otherwise
        lap("  acc program: count + prefix");
        bool disjoint = true;
        {
            std::vector<std::pair<int64_t, int64_t>> rg;
            for (int a = 0; a < K; ++a) if (ap[a].hi >= 0) rg.push_back({ap[a].lo, ap[a].hi});
            std::sort(rg.begin(), rg.end());
            for (size_t i = 1; i < rg.size(); ++i) if (rg[i].first <= rg[i - 1].second) disjoint = false;
        }
        parallel_for(K, disjoint ? nthreads : 1, [&](int a) {
            const AreaPairs& in = ap[a];
            for (size_t i = 0; i < in.dest.size(); ++i) { int32_t q = cur[in.dest[i]]++; hp.acc_a[q] = 2 * in.pa[i]; hp.acc_b[q] = val_index(in.pb[i]); }
        });
    }
    lap("accumulation program (sort)");
    build_acc_items(hp);
    lap("accumulation items");
    hp.n_ref_vals = hp.ref_off[K];
    lap("reference-layout program");
    // ---- state update list ----------------------------------------------------------------
    for (int a = 0; a < K; ++a) {
        if (!hp.owned[a]) continue;
        AreaSym& A = as[a];
        int n_ia = d.ia_ptr[a + 1] - d.ia_ptr[a];
        for (int v = 0; v < A.ni; ++v) {
            int bus = v < n_ia ? d.ia_bus[d.ia_ptr[a] + v] : d.im_bus[d.im_ptr[a] + (v - n_ia)];
            hp.upd_bus.push_back(bus); hp.upd_quant.push_back(v < n_ia ? 0 : 1); hp.upd_pos.push_back(hp.area_base[a] + A.epos[v]);
        }
    }
    for (int s = 0; s < ng; ++s) { hp.upd_bus.push_back(d.gamma_bus[s]); hp.upd_quant.push_back(d.gamma_quant[s]); hp.upd_pos.push_back(hp.gamma_base + s); }

    hp.alg_bytes = 16.0 * m + 32.0 * nbus + 96.0 * d.n_branch + 8.0 * nnz_total + 8.0 * rhs_total;
    return "";
}

// Second accumulation program with the reference's block layout (AreaNormalBlocks: CSR G_ii / G_ib
// values, dense G_bb, b_i, b_b -- assembly.py:32-53), used only by the component-parity entry
// point gse_phase_assemble; built on first use so that a plain solve does not pay for it.
void build_reference_program(HostProgram& hp) {
    if (hp.ref_program_built) return;
    hp.ref_program_built = true;
    const int K = hp.n_areas;
    std::vector<int64_t> rdest; std::vector<int32_t> ra, rb;   // (dest, a, b) in program order
    for (int a = 0; a < K; ++a) {
        if (!hp.owned[a]) continue;
        const int ni = hp.area_ni[a], nb = hp.area_nb[a];
        const std::vector<int>& rows = hp.tmpl_rows[a]; const std::vector<int>& slot_ptr = hp.tmpl_slot_ptr[a];
        const std::vector<int>& slot_var = hp.tmpl_slot_var[a];
        const int64_t slot_base = hp.tmpl_slot_base[a];
        const int64_t base = hp.ref_off[a];
        const int64_t o_ib = base + (int64_t)hp.ii_idx[a].size(), o_bb = o_ib + (int64_t)hp.ib_idx[a].size();
        const int64_t o_bi = o_bb + (int64_t)nb * nb, o_bbv = o_bi + ni;
        auto find = [](const std::vector<int32_t>& ptr, const std::vector<int32_t>& idx, int r, int c) {
            return (int64_t)(std::lower_bound(idx.begin() + ptr[r], idx.begin() + ptr[r + 1], c) - idx.begin());
        };
        for (size_t k = 0; k < rows.size(); ++k) {
            const int s0 = slot_ptr[k], s1 = slot_ptr[k + 1];
            for (int x = s0; x < s1; ++x) {
                const int va = slot_var[x];
                for (int y = s0; y < s1; ++y) {
                    const int vb = slot_var[y]; int64_t dest;
                    if (va < ni && vb < ni) dest = base + find(hp.ii_ptr[a], hp.ii_idx[a], va, vb);
                    else if (va < ni) dest = o_ib + find(hp.ib_ptr[a], hp.ib_idx[a], va, vb - ni);
                    else if (vb >= ni) dest = o_bb + (int64_t)(va - ni) * nb + (vb - ni);
                    else continue;
                    rdest.push_back(dest); ra.push_back((int32_t)(slot_base + x)); rb.push_back((int32_t)(slot_base + y));
                }
            }
            for (int x = s0; x < s1; ++x) {
                const int v = slot_var[x];
                rdest.push_back(v < ni ? o_bi + v : o_bbv + (v - ni)); ra.push_back((int32_t)(slot_base + x)); rb.push_back(-(rows[k] + 1));
            }
        }
    }
    auto val_index = [&](int32_t b) { return b >= 0 ? (int32_t)(2 * b + 1) : (int32_t)(2 * hp.n_slots + (-b - 1)); };
    hp.racc_ptr.assign(hp.n_ref_vals + 1, 0);
    for (int64_t dd : rdest) hp.racc_ptr[dd + 1]++;
    for (int64_t i = 0; i < hp.n_ref_vals; ++i) hp.racc_ptr[i + 1] += hp.racc_ptr[i];
    hp.racc_a.resize(rdest.size()); hp.racc_b.resize(rdest.size());
    std::vector<int32_t> cur(hp.racc_ptr.begin(), hp.racc_ptr.end() - 1);
    for (size_t i = 0; i < rdest.size(); ++i) { int32_t q = cur[rdest[i]]++; hp.racc_a[q] = 2 * ra[i]; hp.racc_b[q] = val_index(rb[i]); }
}

}  // namespace gse
