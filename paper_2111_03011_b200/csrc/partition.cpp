// partition.cpp -- multilevel hypergraph bisection for the contraction-order search (setup).
//
// The planner builds contraction trees by recursive min-cut bisection of the tensor network: the bonds
// cut by a bisection are the legs of the two halves' results, so small balanced cuts keep every
// intermediate small (the graph-partitioning view of contraction ordering).  The sparse output adds one
// net: all tensors that carry sparse rows (fixed output legs) share a "rows" net whose weight is the
// number of index bits the rows cost once they are split across both halves (log2 L at saturation), so
// the partitioner prefers to keep the output boundary together in one half -- the big-head / tail split of
// P:L89-L91 emerges from the cut objective instead of being hand-designed.
//
// Algorithm (standard multilevel scheme): heavy-edge coarsening until ~24 nodes, greedy-growing initial
// bisections + Fiduccia-Mattheyses refinement at the coarsest level, then projection and FM refinement
// on every finer level.  Deterministic for a given rng state.
#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <map>
#include <numeric>

#include "tnb.h"

namespace tnb {

namespace {

struct Level {
    HyperGraph g;
    std::vector<int> up;  // fine node -> node of the next coarser level
};

// weighted cut of a bisection
int64_t cut_of(const HyperGraph& g, const std::vector<char>& side) {
    int64_t c = 0;
    for (size_t e = 0; e < g.nets.size(); e++) {
        bool s0 = false, s1 = false;
        for (int v : g.nets[e]) (side[v] ? s1 : s0) = true;
        if (s0 && s1) c += g.net_w[e];
    }
    return c;
}

// node -> incident nets
std::vector<std::vector<int>> incidence(const HyperGraph& g) {
    std::vector<std::vector<int>> inc(g.n);
    for (size_t e = 0; e < g.nets.size(); e++)
        for (int v : g.nets[e]) inc[v].push_back((int)e);
    return inc;
}

// Contract a matching: nodes with the same `up` id merge; nets are re-pinned, single-pin nets dropped,
// parallel 2-pin nets merged (weights summed).
HyperGraph coarsen_graph(const HyperGraph& g, const std::vector<int>& up, int nc) {
    HyperGraph h;
    h.n = nc;
    h.node_w.assign(nc, 0);
    for (int v = 0; v < g.n; v++) h.node_w[up[v]] += g.node_w[v];
    if (!g.fixed.empty()) {
        h.fixed.assign(nc, -1);
        for (int v = 0; v < g.n; v++)
            if (g.fixed[v] >= 0) h.fixed[up[v]] = g.fixed[v];
    }
    std::map<std::pair<int, int>, int> two;
    for (size_t e = 0; e < g.nets.size(); e++) {
        std::vector<int> p;
        for (int v : g.nets[e]) p.push_back(up[v]);
        std::sort(p.begin(), p.end());
        p.erase(std::unique(p.begin(), p.end()), p.end());
        if (p.size() < 2) continue;
        if (p.size() == 2) {
            auto it = two.find({p[0], p[1]});
            if (it != two.end()) {
                h.net_w[it->second] += g.net_w[e];
                continue;
            }
            two[{p[0], p[1]}] = (int)h.nets.size();
        }
        h.nets.push_back(p);
        h.net_w.push_back(g.net_w[e]);
    }
    return h;
}

// FM refinement: passes of single-node moves (best gain first, balance kept), each pass rolled back to
// its best prefix; stops when a pass does not improve the cut.
void fm_refine(const HyperGraph& g, const std::vector<std::vector<int>>& inc, std::vector<char>& side, int64_t lo,
               int64_t hi, std::mt19937_64& rng, int max_passes) {
    const int n = g.n;
    const int ne = (int)g.nets.size();
    std::vector<std::array<int, 2>> cnt(ne);
    auto recount = [&]() {
        for (int e = 0; e < ne; e++) {
            cnt[e] = {0, 0};
            for (int v : g.nets[e]) cnt[e][side[v]]++;
        }
    };
    auto gain_of = [&](int v) {
        int64_t gsum = 0;
        const int s = side[v];
        for (int e : inc[v]) {
            if (cnt[e][s] == 1 && cnt[e][1 - s] > 0) gsum += g.net_w[e];
            if (cnt[e][1 - s] == 0) gsum -= g.net_w[e];
        }
        return gsum;
    };
    int64_t w0 = 0;
    for (int v = 0; v < n; v++)
        if (side[v] == 0) w0 += g.node_w[v];
    recount();
    int64_t cut = cut_of(g, side);
    std::vector<int64_t> gain(n);
    std::vector<char> locked(n);
    for (int pass = 0; pass < max_passes; pass++) {
        for (int v = 0; v < n; v++) gain[v] = gain_of(v);
        std::fill(locked.begin(), locked.end(), 0);
        std::vector<int> moves;
        int64_t cur = cut, best = cut, cw0 = w0, best_w0 = w0;
        size_t best_len = 0;
        // a balanced prefix is preferred over an unbalanced start
        bool start_ok = (w0 >= lo && w0 <= hi);
        bool best_ok = start_ok;
        for (int step = 0; step < n; step++) {
            int bv = -1;
            int64_t bg = LLONG_MIN;
            for (int v = 0; v < n; v++) {
                if (locked[v] || (!g.fixed.empty() && g.fixed[v] >= 0)) continue;
                const int64_t nw0 = cw0 + (side[v] == 0 ? -g.node_w[v] : g.node_w[v]);
                // moves that leave the balance window are allowed only toward it
                const bool ok = (nw0 >= lo && nw0 <= hi) || std::llabs(nw0 - (lo + hi) / 2) < std::llabs(cw0 - (lo + hi) / 2);
                if (!ok) continue;
                if (gain[v] > bg || (gain[v] == bg && (rng() & 1))) {
                    bg = gain[v];
                    bv = v;
                }
            }
            if (bv < 0) break;
            locked[bv] = 1;
            const int s = side[bv];
            cw0 += (s == 0 ? -g.node_w[bv] : g.node_w[bv]);
            for (int e : inc[bv]) {
                cnt[e][s]--;
                cnt[e][1 - s]++;
            }
            side[bv] = (char)(1 - s);
            cur -= bg;
            moves.push_back(bv);
            for (int e : inc[bv])
                for (int u : g.nets[e])
                    if (!locked[u]) gain[u] = gain_of(u);
            const bool ok = (cw0 >= lo && cw0 <= hi);
            if ((ok && !best_ok) || (ok == best_ok && cur < best)) {
                best = cur;
                best_len = moves.size();
                best_w0 = cw0;
                best_ok = ok;
            }
        }
        for (size_t i = moves.size(); i > best_len; i--) {
            const int v = moves[i - 1];
            side[v] = (char)(1 - side[v]);
        }
        recount();
        w0 = best_w0;
        const bool improved = best < cut;
        cut = best;
        if (!improved) break;
    }
}

// greedy growing from a random seed node: repeatedly add the outside node with the largest connection
// weight to the growing side until it holds `target` node weight
std::vector<char> grow(const HyperGraph& g, const std::vector<std::vector<int>>& inc, int64_t target,
                       std::mt19937_64& rng) {
    std::vector<char> side(g.n, 1);
    std::vector<double> conn(g.n, 0.0);
    int64_t w = 0;
    auto add = [&](int v) {
        side[v] = 0;
        w += g.node_w[v];
        for (int e : inc[v]) {
            const double c = (double)g.net_w[e] / (double)(g.nets[e].size() - 1);
            for (int u : g.nets[e]) conn[u] += c;
        }
    };
    bool any_fixed0 = false;
    for (int v = 0; v < (int)g.fixed.size(); v++)
        if (g.fixed[v] == 0) {
            add(v);
            any_fixed0 = true;
        }
    if (!any_fixed0) {
        int seed = (int)(rng() % (uint64_t)g.n);
        for (int tries = 0; tries < 64 && !g.fixed.empty() && g.fixed[seed] == 1; tries++)
            seed = (int)(rng() % (uint64_t)g.n);
        add(seed);
    }
    while (w < target) {
        int bv = -1;
        double bc = -1;
        for (int v = 0; v < g.n; v++)
            if (side[v] == 1 && (g.fixed.empty() || g.fixed[v] < 0) && (conn[v] > bc || (conn[v] == bc && (rng() & 1)))) {
                bc = conn[v];
                bv = v;
            }
        if (bv < 0) break;
        add(bv);
    }
    return side;
}

}  // namespace

std::vector<char> ml_bisect(const HyperGraph& g0, double eps, std::mt19937_64& rng, int init_tries) {
    const int64_t total = std::accumulate(g0.node_w.begin(), g0.node_w.end(), (int64_t)0);
    const int64_t lo = (int64_t)std::floor(total * (0.5 - eps / 2)), hi = (int64_t)std::ceil(total * (0.5 + eps / 2));
    std::vector<Level> lv;
    lv.push_back({g0, {}});
    // ---------------- coarsening (heavy-edge matching, bounded node weight)
    const int64_t wmax = std::max<int64_t>(1, (int64_t)std::ceil(total * std::max(0.02, eps / 4 + 0.04)));
    while (lv.back().g.n > 24) {
        const HyperGraph& g = lv.back().g;
        auto inc = incidence(g);
        std::vector<int> order(g.n);
        std::iota(order.begin(), order.end(), 0);
        std::shuffle(order.begin(), order.end(), rng);
        std::vector<int> mate(g.n, -1);
        std::vector<double> rate(g.n, 0.0);
        for (int u : order) {
            if (mate[u] >= 0) continue;
            std::vector<int> touched;
            for (int e : inc[u]) {
                if (g.nets[e].size() > 64) continue;
                const double r = (double)g.net_w[e] / (double)(g.nets[e].size() - 1);
                for (int v : g.nets[e]) {
                    if (v == u || mate[v] >= 0) continue;
                    if (rate[v] == 0.0) touched.push_back(v);
                    rate[v] += r;
                }
            }
            int bv = -1;
            double br = 0;
            for (int v : touched) {
                // prefer light partners (heavy-edge rating normalised by the merged weight)
                const double r = rate[v] / std::sqrt((double)(g.node_w[u] + g.node_w[v]));
                const bool clash = !g.fixed.empty() && g.fixed[u] >= 0 && g.fixed[v] >= 0 && g.fixed[u] != g.fixed[v];
                if (!clash && g.node_w[u] + g.node_w[v] <= wmax && (r > br || (r == br && (rng() & 1)))) {
                    br = r;
                    bv = v;
                }
            }
            for (int v : touched) rate[v] = 0.0;
            if (bv >= 0) {
                mate[u] = bv;
                mate[bv] = u;
            }
        }
        std::vector<int> up(g.n, -1);
        int nc = 0;
        for (int u = 0; u < g.n; u++) {
            if (up[u] >= 0) continue;
            up[u] = nc;
            if (mate[u] >= 0) up[mate[u]] = nc;
            nc++;
        }
        if (nc > 0.92 * g.n) break;  // no longer shrinking
        lv.back().up = up;
        HyperGraph h = coarsen_graph(g, up, nc);
        lv.push_back({std::move(h), {}});
    }
    // ---------------- initial bisection at the coarsest level
    const HyperGraph& gc = lv.back().g;
    auto incc = incidence(gc);
    std::vector<char> best;
    int64_t best_cut = LLONG_MAX;
    bool best_bal = false;
    for (int r = 0; r < init_tries; r++) {
        const int64_t target = lo + (int64_t)((hi - lo) * ((rng() % 1000) / 1000.0));
        std::vector<char> side = grow(gc, incc, std::max<int64_t>(1, (target + lo) / 2), rng);
        fm_refine(gc, incc, side, lo, hi, rng, 16);
        int64_t w0 = 0;
        for (int v = 0; v < gc.n; v++)
            if (!side[v]) w0 += gc.node_w[v];
        const bool bal = w0 >= lo && w0 <= hi && w0 > 0 && w0 < total;
        const int64_t c = cut_of(gc, side);
        if ((bal && !best_bal) || (bal == best_bal && c < best_cut)) {
            best = side;
            best_cut = c;
            best_bal = bal;
        }
    }
    // ---------------- uncoarsening with FM refinement
    std::vector<char> side = best;
    for (int i = (int)lv.size() - 2; i >= 0; i--) {
        const HyperGraph& g = lv[i].g;
        std::vector<char> fine(g.n);
        for (int v = 0; v < g.n; v++) fine[v] = side[lv[i].up[v]];
        auto inc = incidence(g);
        fm_refine(g, inc, fine, lo, hi, rng, 8);
        side.swap(fine);
    }
    return side;
}

}  // namespace tnb
