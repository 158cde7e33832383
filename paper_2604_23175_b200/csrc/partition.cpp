// partition.cpp -- the graph passes of partition_network on the host, in C++.
//
// partition_network (reference partition.py:373-403) is outside the solve path but it is what a user
// waits for before the first solve: 24 s / 182 s in the reference at the PEGASE-2869 / 9241 shapes.
// The passes of one attempt -- farthest-point seeds, multi-source growth, re-centring on the
// minimum-eccentricity bus, balance moves, cascade along the area graph, cut thinning
// (partition.py:198-365) -- are pure integer graph walks; they are restated here with the same visiting
// orders and tie-breaks (lowest index / (size, index) keys / FIFO growth fronts), so the result equals
// the Python passes of paper_2604_23175_b200/partition.py bus for bus (tests/test_host_api.py compares
// the two on random grids and against the partitions the reference itself produced).  The random
// draw of the first seed stays in Python (numpy's generator) and comes in as an argument.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <vector>

namespace {

struct Grid {
    int n = 0;
    const int32_t* ptr = nullptr;   // neighbors of u: idx[ptr[u] .. ptr[u + 1]) in net.neighbors(u) order
    const int32_t* idx = nullptr;
    int nbr = 0;
    const int32_t* f = nullptr;     // branch ends
    const int32_t* t = nullptr;
    mutable std::vector<int> mark;  // scratch stamps of the connectivity walks
    mutable int stamp = 0;
};

std::vector<int> hop_distance(const Grid& g, const std::vector<int>& sources) {
    std::vector<int> dist(g.n, -1);
    std::deque<int> q(sources.begin(), sources.end());
    for (int s : sources) dist[s] = 0;
    while (!q.empty()) {
        const int u = q.front(); q.pop_front();
        for (int p = g.ptr[u]; p < g.ptr[u + 1]; ++p) {
            const int v = g.idx[p];
            if (dist[v] < 0) { dist[v] = dist[u] + 1; q.push_back(v); }
        }
    }
    return dist;
}

std::vector<int> seed_buses(const Grid& g, int k, int first) {
    std::vector<int> seeds{first};
    while ((int)seeds.size() < k) {
        const std::vector<int> dist = hop_distance(g, seeds);
        const int mx = *std::max_element(dist.begin(), dist.end());
        seeds.push_back((int)(std::find(dist.begin(), dist.end(), mx) - dist.begin()));   // lowest index at the maximum
    }
    return seeds;
}

// Multi-source growth: the currently smallest area claims one bus per turn.  Returns the number of buses
// left unclaimed (0 = success); starved / starved_size describe the failure.
int grow(const Grid& g, const std::vector<int>& seeds, std::vector<int>& area, int& starved, int& starved_size) {
    const int k = (int)seeds.size();
    area.assign(g.n, -1);
    std::vector<int> size(k, 1);
    for (int a = 0; a < k; ++a) area[seeds[a]] = a;
    std::vector<std::deque<int>> fronts(k);
    for (int a = 0; a < k; ++a)
        for (int p = g.ptr[seeds[a]]; p < g.ptr[seeds[a] + 1]; ++p)
            if (area[g.idx[p]] == -1) fronts[a].push_back(g.idx[p]);
    int unclaimed = g.n - k;
    std::vector<char> live(k, 1);
    int n_live = k;
    while (unclaimed && n_live) {
        int a = -1;
        for (int i = 0; i < k; ++i) if (live[i] && (a < 0 || size[i] < size[a])) a = i;     // min by (size, index)
        std::deque<int>& q = fronts[a];
        bool claimed = false;
        while (!q.empty()) {
            const int u = q.front(); q.pop_front();
            if (area[u] != -1) continue;
            area[u] = a; ++size[a]; --unclaimed;
            for (int p = g.ptr[u]; p < g.ptr[u + 1]; ++p) if (area[g.idx[p]] == -1) q.push_back(g.idx[p]);
            claimed = true;
            break;
        }
        if (!claimed) { live[a] = 0; --n_live; }
    }
    if (unclaimed) {
        starved = (int)(std::min_element(size.begin(), size.end()) - size.begin());
        starved_size = size[starved];
    }
    return unclaimed;
}

// Minimum-eccentricity bus of the induced subgraph (ties: lowest index); distances to unreachable members
// do not count (the reference maps them to -1 before the row maximum).
int center_of(const Grid& g, const std::vector<int>& area, int a) {
    std::vector<int> members;
    for (int u = 0; u < g.n; ++u) if (area[u] == a) members.push_back(u);
    if (members.size() == 1) return members[0];
    std::vector<int> dist(g.n, -1), q;
    int best = -1, best_ecc = 0;
    for (int s : members) {
        q.clear(); q.push_back(s); dist[s] = 0;
        int ecc = 0;
        for (size_t h = 0; h < q.size(); ++h) {
            const int u = q[h];
            ecc = dist[u];                                  // BFS order: the last one popped is the farthest
            for (int p = g.ptr[u]; p < g.ptr[u + 1]; ++p) {
                const int v = g.idx[p];
                if (area[v] == a && dist[v] < 0) { dist[v] = dist[u] + 1; q.push_back(v); }
            }
        }
        for (int u : q) dist[u] = -1;
        if (best < 0 || ecc < best_ecc) { best = s; best_ecc = ecc; }
    }
    return best;
}

// Is area a minus bus `without` (-1: nothing removed) non-empty and connected?
bool stays_connected(const Grid& g, const std::vector<int>& area, const std::vector<int>& size, int a, int without) {
    const int members = size[a] - ((without >= 0 && area[without] == a) ? 1 : 0);
    if (members <= 0) return false;
    // (the answer does not depend on where the walk starts: a neighbor of the removed bus saves the scan)
    int start = -1;
    if (without >= 0)
        for (int p = g.ptr[without]; p < g.ptr[without + 1] && start < 0; ++p)
            if (area[g.idx[p]] == a && g.idx[p] != without) start = g.idx[p];
    if (start < 0)
        for (int u = 0; u < g.n; ++u) if (area[u] == a && u != without) { start = u; break; }
    if ((int)g.mark.size() != g.n) { g.mark.assign(g.n, 0); g.stamp = 0; }
    const int st = ++g.stamp;
    std::vector<int> todo{start};
    g.mark[start] = st;
    int seen = 1;
    while (!todo.empty()) {
        const int u = todo.back(); todo.pop_back();
        for (int p = g.ptr[u]; p < g.ptr[u + 1]; ++p) {
            const int v = g.idx[p];
            if (v != without && area[v] == a && g.mark[v] != st) { g.mark[v] = st; ++seen; todo.push_back(v); }
        }
    }
    return seen == members;
}

std::vector<int> sizes_of(const std::vector<int>& area, int k) {
    std::vector<int> size(k, 0);
    for (int a : area) ++size[a];
    return size;
}

void balance_pass(const Grid& g, std::vector<int>& area, int k, int max_passes = 12) {
    std::vector<int> size = sizes_of(area, k), opts;
    for (int pass = 0; pass < max_passes; ++pass) {
        bool moved = false;
        for (int u = 0; u < g.n; ++u) {
            const int a = area[u];
            if (size[a] <= 1) continue;
            int b = -1;                                       // min by (size, index) over the neighbor areas that are smaller by 2+
            for (int p = g.ptr[u]; p < g.ptr[u + 1]; ++p) {
                const int c = area[g.idx[p]];
                if (c == a || !(size[a] > size[c] + 1)) continue;
                if (b < 0 || size[c] < size[b] || (size[c] == size[b] && c < b)) b = c;
            }
            if (b < 0) continue;
            if (!stays_connected(g, area, size, a, u)) continue;
            area[u] = b; --size[a]; ++size[b];
            moved = true;
        }
        if (!moved) break;
    }
}

bool push_one(const Grid& g, std::vector<int>& area, int a, int b, std::vector<int>& size) {
    for (int u = 0; u < g.n; ++u) {
        if (area[u] != a || size[a] <= 1) continue;
        bool touches = false;
        for (int p = g.ptr[u]; p < g.ptr[u + 1] && !touches; ++p) touches = area[g.idx[p]] == b;
        if (!touches) continue;
        if (stays_connected(g, area, size, a, u)) { area[u] = b; --size[a]; ++size[b]; return true; }
    }
    return false;
}

// Drain the largest area toward the smallest along the area graph.
void cascade(const Grid& g, std::vector<int>& area, int k, double target_ratio = 2.0) {
    std::vector<int> size = sizes_of(area, k);
    for (int round = 0; round < 2 * g.n; ++round) {
        const int mx = *std::max_element(size.begin(), size.end()), mn = *std::min_element(size.begin(), size.end());
        if ((double)mx <= target_ratio * (double)mn && mx - mn <= std::max(2, mn)) break;
        const int big = (int)(std::max_element(size.begin(), size.end()) - size.begin());
        const int small = (int)(std::min_element(size.begin(), size.end()) - size.begin());
        std::vector<std::vector<int>> link(k);
        for (int e = 0; e < g.nbr; ++e) {
            const int x = area[g.f[e]], y = area[g.t[e]];
            if (x != y) { link[x].push_back(y); link[y].push_back(x); }
        }
        for (auto& l : link) { std::sort(l.begin(), l.end()); l.erase(std::unique(l.begin(), l.end()), l.end()); }
        std::vector<int> came_from(k, -2);                    // -2 unseen, -1 root
        came_from[big] = -1;
        std::deque<int> q{big};
        while (!q.empty() && came_from[small] == -2) {
            const int u = q.front(); q.pop_front();
            for (int v : link[u]) if (came_from[v] == -2) { came_from[v] = u; q.push_back(v); }
        }
        if (came_from[small] == -2) break;
        std::vector<int> route;
        for (int node = small; node != -1; node = came_from[node]) route.push_back(node);
        std::reverse(route.begin(), route.end());
        bool ok = true;
        for (size_t i = 0; i + 1 < route.size() && ok; ++i) ok = push_one(g, area, route[i], route[i + 1], size);
        if (!ok) break;
    }
}

void thin_cuts(const Grid& g, std::vector<int>& area, int k, int max_passes = 6) {
    std::vector<int> size = sizes_of(area, k), nb;
    int cap = 2 * *std::min_element(size.begin(), size.end());
    for (int pass = 0; pass < max_passes; ++pass) {
        bool moved = false;
        for (int u = 0; u < g.n; ++u) {
            const int a = area[u];
            if (size[a] <= 1) continue;
            nb.clear();
            for (int p = g.ptr[u]; p < g.ptr[u + 1]; ++p) nb.push_back(area[g.idx[p]]);
            const int here = (int)std::count(nb.begin(), nb.end(), a);
            std::vector<int> cand(nb);
            std::sort(cand.begin(), cand.end()); cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
            int pick = -1, pick_gain = 0;
            for (int b : cand) {
                if (b == a) continue;
                const int gain = (int)std::count(nb.begin(), nb.end(), b) - here;
                if (gain > pick_gain && size[b] + 1 <= cap && size[a] - 1 >= 1) { pick = b; pick_gain = gain; }
            }
            if (pick < 0 || !stays_connected(g, area, size, a, u)) continue;
            area[u] = pick; --size[a]; ++size[pick];
            cap = 2 * *std::min_element(size.begin(), size.end());
            moved = true;
        }
        if (!moved) break;
    }
}

Grid make_grid(int n, const int32_t* ptr, const int32_t* idx, int nbr, const int32_t* f, const int32_t* t) {
    Grid g; g.n = n; g.ptr = ptr; g.idx = idx; g.nbr = nbr; g.f = f; g.t = t;
    return g;
}

}  // namespace

extern "C" {

// One attempt of partition_network (partition.py:353-365 of this package, reference partition.py `_attempt`).
// first_seed: the bus numpy's generator drew.  area_out[n].  Returns 0, or 1 when the growth starves
// (info = {starved area, its size, buses left unassigned}; the caller raises PartitionError).
int gse_partition_attempt(int32_t n, const int32_t* nbr_ptr, const int32_t* nbr_idx, int32_t n_branch, const int32_t* br_from,
                          const int32_t* br_to, int32_t k, int32_t first_seed, int32_t* area_out, int32_t* info) {
    const Grid g = make_grid(n, nbr_ptr, nbr_idx, n_branch, br_from, br_to);
    std::vector<int> seeds = seed_buses(g, k, first_seed), area;
    int starved = 0, starved_size = 0;
    int left = grow(g, seeds, area, starved, starved_size);
    for (int round = 0; round < 3 && !left; ++round) {
        std::vector<int> centers(k);
        for (int a = 0; a < k; ++a) centers[a] = center_of(g, area, a);
        if (centers == seeds) break;
        seeds = centers;
        left = grow(g, seeds, area, starved, starved_size);
    }
    if (left) { info[0] = starved; info[1] = starved_size; info[2] = left; return 1; }
    balance_pass(g, area, k);
    cascade(g, area, k);
    balance_pass(g, area, k);
    thin_cuts(g, area, k);
    for (int u = 0; u < n; ++u) area_out[u] = area[u];
    return 0;
}

// The cut-thinning pass alone (merged variants of a finer attempt, partition.py `_merged_variants`).
int gse_partition_thin_cuts(int32_t n, const int32_t* nbr_ptr, const int32_t* nbr_idx, int32_t n_branch, const int32_t* br_from,
                            const int32_t* br_to, int32_t k, int32_t* area_inout) {
    const Grid g = make_grid(n, nbr_ptr, nbr_idx, n_branch, br_from, br_to);
    std::vector<int> area(area_inout, area_inout + n);
    thin_cuts(g, area, k);
    for (int u = 0; u < n; ++u) area_inout[u] = area[u];
    return 0;
}

}  // extern "C"
