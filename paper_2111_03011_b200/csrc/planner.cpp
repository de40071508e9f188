// planner.cpp -- contraction order ("contracting neighboring tensors in a complexity-greedy
// manner") and slicing ("select some indices ... and fix them ... in order to decrease the
// overall space complexity").  Setup, not the hot path.
//
// 1. randomised greedy trees (two criteria x Gumbel temperatures), best few kept;
// 2. subtree reconfiguration: every subtree cut at <= KMAX frontier tensors is replaced by the optimal
//    order of its frontier (exact DP over subsets), repeated to a fixed point;
// 3. slicing interleaved with reconfiguration: slice the edge that minimises 2^s x (time per slice),
//    re-optimise the tree with that edge removed, until every tensor fits max_tensor_size.
// All plans are ranked by one roofline-time model of a slice ("the planner objective
// should be roofline time, not flops").
#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <set>
#include <sstream>
#include <functional>
#include <climits>
#include <map>
#include <unordered_map>

#include "tnb.h"

namespace tnb {

// ------------------------------------------------------------------------------ row model

double RowModel::rows(uint64_t qmask) {
    if (qmask == 0) return 1.0;
    for (auto& kv : memo)
        if (kv.first == qmask) return kv.second;
    double r;
    const double L = (double)req->fixed.size();
    if (req->fixed.size() <= (1u << 16)) {
        r = (double)rows_of(*req, qmask).size();
    } else {  // expected distinct count of L uniform keys over 2^q values
        const int q = __builtin_popcountll(qmask);
        const double V = std::ldexp(1.0, q);
        r = V * (1.0 - std::exp(L * std::log1p(-1.0 / V)));
        r = std::max(1.0, std::min(r, L));
    }
    memo.push_back({qmask, r});
    return r;
}

namespace {

constexpr int W = 24;  // bitset words: up to 1536 edges
struct Bits {
    uint64_t w[W] = {0};
    void set(int e) { w[e >> 6] |= 1ull << (e & 63); }
    bool get(int e) const { return (w[e >> 6] >> (e & 63)) & 1; }
    int count() const {
        int c = 0;
        for (int i = 0; i < W; i++) c += __builtin_popcountll(w[i]);
        return c;
    }
};
inline Bits operator|(const Bits& a, const Bits& b) { Bits r; for (int i = 0; i < W; i++) r.w[i] = a.w[i] | b.w[i]; return r; }
inline Bits operator&(const Bits& a, const Bits& b) { Bits r; for (int i = 0; i < W; i++) r.w[i] = a.w[i] & b.w[i]; return r; }
inline Bits operator^(const Bits& a, const Bits& b) { Bits r; for (int i = 0; i < W; i++) r.w[i] = a.w[i] ^ b.w[i]; return r; }
inline Bits andnot(const Bits& a, const Bits& b) { Bits r; for (int i = 0; i < W; i++) r.w[i] = a.w[i] & ~b.w[i]; return r; }
inline int popc_andnot(const Bits& a, const Bits& b) {
    int c = 0;
    for (int i = 0; i < W; i++) c += __builtin_popcountll(a.w[i] & ~b.w[i]);
    return c;
}

// roofline constants of the model (B200): HBM ~5.5 TB/s achievable, 3xTF32 complex
// ~25e12 CMAC/s on the tensor-core path, ~5e12 CMAC/s for the SIMT path, ~3 us per launch.
constexpr double BW = 5.5e12, C_TC = 25e12, C_SIMT = 5e12, T_LAUNCH = 3e-6;

// Time of one pairwise step given dense leg counts (after slicing) and row counts.
struct StepCost {
    double time, cmac, bytes, sC;
    bool gemm;
};
inline StepCost step_cost(int a, int b, int c, int u, double rA, double rB, double rC, bool rowsA, bool rowsB) {
    StepCost s;
    const double sA = rA * std::ldexp(1.0, a), sB = rB * std::ldexp(1.0, b);
    s.sC = rC * std::ldexp(1.0, c);
    s.cmac = rC * std::ldexp(1.0, u);
    s.bytes = 8.0 * (sA + sB + s.sC);
    const int kk = (a + b - c) / 2;
    s.gemm = false;
    if (!(rowsA && rowsB)) {
        const bool a_is_m = rowsA || (!rowsB && sA >= sB);
        const double sM = a_is_m ? sA : sB, sN = a_is_m ? sB : sA;
        const double m = sM / std::ldexp(1.0, kk), n = sN / std::ldexp(1.0, kk);
        s.gemm = ((m >= 128 && n >= 64) || (m >= 64 && n >= 128) || (m >= 128 && n >= 16 && kk >= 6)) && kk >= 4;
    }
    if (s.gemm) {
        // pre-passes read both operands and write hi + lo (the smaller one embedded, 2x), the GEMM reads
        // them back
        const double ops_bytes = s.bytes + 8.0 * (4.0 * (sA + sB) + 4.0 * std::min(sA, sB));
        s.time = std::max(s.cmac / C_TC, ops_bytes / BW) + 3 * T_LAUNCH;
    } else if (rowsA && rowsB) {
        // gather-contract: every output row re-reads its parents' rows (mostly from L2, ~3x HBM)
        const double reread = 8.0 * rC * (std::ldexp(1.0, a) + std::ldexp(1.0, b));
        s.time = std::max(std::max(s.cmac / C_SIMT, s.bytes / BW), reread / (3.0 * BW)) + T_LAUNCH;
    } else {
        s.time = std::max(s.cmac / C_SIMT, s.bytes / BW) + T_LAUNCH;
    }
    return s;
}

// ------------------------------------------------------------------------------ contraction tree

struct Node {
    int left = -1, right = -1, leaf = -1, parent = -1;
    Bits legs;           // dense legs of the result (unsliced)
    uint64_t q = 0;      // fixed final qubits
    double rows = 1;
};

struct Tree {
    std::vector<Node> nodes;  // leaves are nodes[0..NL)
    int root = -1;
};

struct Ctx {
    RowModel* rm;
    Bits sliced;
    double max_elems;
};

// companion edges (tn_slicing.companions): slicing an edge also cuts its companion, so every cost below is
// evaluated on the closure of the planner's sliced set (companions of companions are not cut)
thread_local const std::vector<std::pair<int, int>>* g_companions = nullptr;
inline Bits closure(const Bits& S) {
    if (!g_companions || g_companions->empty()) return S;
    Bits r = S;
    for (const auto& p : *g_companions)
        if (S.get(p.first)) r.set(p.second);
    return r;
}

double node_size_raw(const Node& n, const Bits& C) { return n.rows * std::ldexp(1.0, popc_andnot(n.legs, C)); }
double node_size(const Node& n, const Bits& S) { return node_size_raw(n, closure(S)); }

StepCost node_step_raw(const Tree& t, int v, const Bits& S) {
    const Node& N = t.nodes[v];
    const Node& A = t.nodes[N.left];
    const Node& B = t.nodes[N.right];
    const int a = popc_andnot(A.legs, S), b = popc_andnot(B.legs, S), c = popc_andnot(N.legs, S);
    const int u = popc_andnot(A.legs | B.legs, S);
    return step_cost(a, b, c, u, A.rows, B.rows, N.rows, A.q != 0, B.q != 0);
}
StepCost node_step(const Tree& t, int v, const Bits& S) { return node_step_raw(t, v, closure(S)); }

struct TreeEval {
    double time = 0, cmac = 0, bytes = 0, peak = 0;
};

TreeEval eval_tree(const Tree& t, const Bits& S) {
    TreeEval e;
    const Bits C = closure(S);
    for (int v = 0; v < (int)t.nodes.size(); v++) {
        const Node& N = t.nodes[v];
        e.peak = std::max(e.peak, node_size_raw(N, C));
        if (N.leaf >= 0) continue;
        StepCost s = node_step_raw(t, v, C);
        e.time += s.time;
        e.cmac += s.cmac;
        e.bytes += s.bytes;
    }
    return e;
}

// ------------------------------------------------------------------------------ subtree reconfiguration

constexpr int KMAX = 9;
constexpr int LW = 4;  // local bitset words (<= 256 local edges)
struct LBits {
    uint64_t w[LW] = {0};
};
inline LBits lxor(const LBits& a, const LBits& b) { LBits r; for (int i = 0; i < LW; i++) r.w[i] = a.w[i] ^ b.w[i]; return r; }
inline LBits lor(const LBits& a, const LBits& b) { LBits r; for (int i = 0; i < LW; i++) r.w[i] = a.w[i] | b.w[i]; return r; }
inline int lpop(const LBits& a) { int c = 0; for (int i = 0; i < LW; i++) c += __builtin_popcountll(a.w[i]); return c; }

// Try to improve the subtree rooted at v; returns true if the tree changed.
bool reconf_node(Tree& t, int v, Ctx& cx) {
    if (t.nodes[v].leaf >= 0) return false;
    // frontier: expand the largest internal node until KMAX inputs
    std::vector<int> front = {v}, internal;
    while ((int)front.size() < KMAX) {
        int bi = -1;
        double bs = -1;
        for (int i = 0; i < (int)front.size(); i++) {
            const Node& N = t.nodes[front[i]];
            if (N.leaf >= 0) continue;
            double s = node_size(N, cx.sliced);
            if (s > bs) { bs = s; bi = i; }
        }
        if (bi < 0) break;
        int x = front[bi];
        internal.push_back(x);
        front[bi] = t.nodes[x].left;
        front.push_back(t.nodes[x].right);
    }
    const int K = (int)front.size();
    if (K < 3) return false;
    // old cost
    double old = 0;
    for (int x : internal) old += node_step(t, x, cx.sliced).time;
    // local edge index
    std::unordered_map<int, int> loc;
    std::vector<LBits> fl(K);
    for (int i = 0; i < K; i++) {
        Bits eff = andnot(t.nodes[front[i]].legs, closure(cx.sliced));
        for (int wd = 0; wd < W; wd++) {
            uint64_t m = eff.w[wd];
            while (m) {
                int b = __builtin_ctzll(m);
                m &= m - 1;
                int e = wd * 64 + b;
                auto it = loc.find(e);
                int id;
                if (it == loc.end()) {
                    id = (int)loc.size();
                    if (id >= LW * 64) return false;
                    loc[e] = id;
                } else id = it->second;
                fl[i].w[id >> 6] |= 1ull << (id & 63);
            }
        }
    }
    const int NS = 1 << K;
    std::vector<LBits> legs(NS);
    std::vector<uint64_t> q(NS, 0);
    std::vector<double> rows(NS, 1), cost(NS, 0);
    std::vector<int> split(NS, 0), nleg(NS, 0);
    for (int m = 1; m < NS; m++) {
        int low = __builtin_ctz(m);
        int rest = m & (m - 1);
        legs[m] = rest ? lxor(legs[rest], fl[low]) : fl[low];
        q[m] = rest ? (q[rest] | t.nodes[front[low]].q) : t.nodes[front[low]].q;
        rows[m] = (rest == 0) ? t.nodes[front[low]].rows : cx.rm->rows(q[m]);
        nleg[m] = lpop(legs[m]);
    }
    for (int m = 1; m < NS; m++) {
        if (__builtin_popcount(m) < 2) continue;
        double best = 1e300;
        int bsub = 0;
        // enumerate splits with the lowest member in `sub` to visit each pair once
        const int low = m & (-m);
        for (int sub = (m - 1) & m; sub; sub = (sub - 1) & m) {
            if (!(sub & low)) continue;
            const int oth = m ^ sub;
            const double base = cost[sub] + cost[oth];
            if (base >= best) continue;
            const int u = lpop(lor(legs[sub], legs[oth]));
            StepCost s = step_cost(nleg[sub], nleg[oth], nleg[m], u, rows[sub], rows[oth], rows[m], q[sub] != 0,
                                   q[oth] != 0);
            double c = base + s.time;
            // hard bound: intermediates larger than max_elems are heavily penalised
            if (s.sC > cx.max_elems) c += 1e3 * s.time * (s.sC / cx.max_elems);
            if (c < best) { best = c; bsub = sub; }
        }
        cost[m] = best;
        split[m] = bsub;
    }
    // compare against the old cost under the same penalty
    double old_pen = old;
    for (int x : internal) {
        StepCost s = node_step(t, x, cx.sliced);
        if (s.sC > cx.max_elems) old_pen += 1e3 * s.time * (s.sC / cx.max_elems);
    }
    if (cost[NS - 1] >= old_pen * (1 - 1e-9) - 1e-15) return false;
    // rebuild: reuse the internal node ids, v stays the root
    std::vector<int> pool(internal.begin() + 1, internal.end());  // internal[0] == v
    std::function<int(int, int)> build;
    build = [&](int m, int id) -> int {
        if (__builtin_popcount(m) == 1) {
            int f = front[__builtin_ctz(m)];
            return f;
        }
        int node = id;
        if (node < 0) {
            node = pool.back();
            pool.pop_back();
        }
        int a = build(split[m], -1);
        int b = build(m ^ split[m], -1);
        Node& N = t.nodes[node];
        N.left = a;
        N.right = b;
        N.leaf = -1;
        t.nodes[a].parent = node;
        t.nodes[b].parent = node;
        N.legs = t.nodes[a].legs ^ t.nodes[b].legs;
        N.q = t.nodes[a].q | t.nodes[b].q;
        N.rows = cx.rm->rows(N.q);
        return node;
    };
    build(NS - 1, v);
    return true;
}

void reconfigure(Tree& t, Ctx& cx, double budget_s, std::chrono::steady_clock::time_point t0) {
    for (int pass = 0; pass < 20; pass++) {
        bool any = false;
        // bottom-up order
        std::vector<int> order;
        std::vector<int> st = {t.root};
        while (!st.empty()) {
            int x = st.back();
            st.pop_back();
            order.push_back(x);
            if (t.nodes[x].leaf < 0) {
                st.push_back(t.nodes[x].left);
                st.push_back(t.nodes[x].right);
            }
        }
        std::reverse(order.begin(), order.end());
        for (int x : order) {
            if (reconf_node(t, x, cx)) any = true;
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > budget_s) return;
        }
        if (!any) break;
    }
}

// ------------------------------------------------------------------------------ greedy tree

Tree greedy_tree(const Network& net, const std::vector<Leaf>& leaves, RowModel& rm, const std::vector<int>& internal,
                 const std::vector<int>& slot_of_tensor, int crit, double tau, double alpha, std::mt19937_64& rng) {
    const int NL = (int)leaves.size();
    Tree t;
    t.nodes.resize(NL);
    for (int i = 0; i < NL; i++) {
        Node& N = t.nodes[i];
        N.leaf = i;
        for (int e : leaves[i].legs) N.legs.set(e);
        N.q = leaves[i].qmask;
        N.rows = (double)leaves[i].rows.size();
    }
    std::vector<int> cur(NL);  // slot -> node id
    for (int i = 0; i < NL; i++) cur[i] = i;
    std::vector<char> alive(NL, 1);
    std::extreme_value_distribution<double> gumbel(0.0, 1.0);
    std::vector<std::pair<int, int>> ends(net.edges.size(), {-1, -1});
    for (int e : internal) ends[e] = {slot_of_tensor[net.edges[e].t0], slot_of_tensor[net.edges[e].t1]};
    int n_alive = NL;
    while (n_alive > 1) {
        std::set<std::pair<int, int>> cand;
        for (int e : internal) {
            int a = ends[e].first, b = ends[e].second;
            if (a < 0 || b < 0 || a == b) continue;
            cand.insert({std::min(a, b), std::max(a, b)});
        }
        int ba = -1, bb = -1;
        auto sz = [&](int slot) { const Node& N = t.nodes[cur[slot]]; return N.rows * std::ldexp(1.0, N.legs.count()); };
        if (cand.empty()) {
            std::vector<std::pair<double, int>> v;
            for (int i = 0; i < NL; i++)
                if (alive[i]) v.push_back({sz(i), i});
            std::sort(v.begin(), v.end());
            ba = v[0].second;
            bb = v[1].second;
        } else {
            double bs = 1e300;
            for (auto& pr : cand) {
                int a = pr.first, b = pr.second;
                const Node& A = t.nodes[cur[a]];
                const Node& B = t.nodes[cur[b]];
                Bits C = A.legs ^ B.legs;
                double rC = rm.rows(A.q | B.q);
                double sC = rC * std::ldexp(1.0, C.count());
                double sA = sz(a), sB = sz(b);
                double sc = (crit == 0) ? sC - alpha * (sA + sB) : std::log2(sC) - alpha * std::log2(sA + sB);
                if (tau > 0) {
                    double g = gumbel(rng);
                    sc = (crit == 0) ? sc - tau * g * (sA + sB) : sc - tau * g;
                }
                if (sc < bs) { bs = sc; ba = a; bb = b; }
            }
        }
        Node N;
        N.left = cur[ba];
        N.right = cur[bb];
        N.legs = t.nodes[N.left].legs ^ t.nodes[N.right].legs;
        N.q = t.nodes[N.left].q | t.nodes[N.right].q;
        N.rows = rm.rows(N.q);
        int id = (int)t.nodes.size();
        t.nodes[N.left].parent = id;
        t.nodes[N.right].parent = id;
        t.nodes.push_back(N);
        cur[ba] = id;
        alive[bb] = 0;
        n_alive--;
        for (int e : internal) {
            if (ends[e].first == bb) ends[e].first = ba;
            if (ends[e].second == bb) ends[e].second = ba;
            if (ends[e].first == ba && ends[e].second == ba) ends[e] = {-1, -1};
        }
    }
    for (int i = 0; i < NL; i++)
        if (alive[i]) t.root = cur[i];
    return t;
}


// ------------------------------------------------------------------------------ recursive bisection
// Min-cut bisection of the tensor graph (Fiduccia-Mattheyses with random restarts, balance +-eps),
// applied recursively; small parts are finished greedily.  The cut bonds of a part are the legs of
// its result, so balanced min-cuts keep every intermediate small (the graph-partitioning view of
// contraction ordering).
struct Graph {
    std::vector<std::vector<std::pair<int, int>>> adj;  // leaf -> (neighbour leaf, #shared bonds)
};

std::vector<char> fm_bisect(const std::vector<int>& V, const Graph& g, double eps, std::mt19937_64& rng, int restarts) {
    const int n = (int)V.size();
    std::unordered_map<int, int> loc;
    for (int i = 0; i < n; i++) loc[V[i]] = i;
    std::vector<std::vector<std::pair<int, int>>> adj(n);
    for (int i = 0; i < n; i++)
        for (auto& pr : g.adj[V[i]]) {
            auto it = loc.find(pr.first);
            if (it != loc.end()) adj[i].push_back({it->second, pr.second});
        }
    const int lo = std::max(1, (int)std::floor(n * (0.5 - eps / 2))), hi = std::min(n - 1, (int)std::ceil(n * (0.5 + eps / 2)));
    std::vector<char> best(n, 0);
    long best_cut = -1;
    std::uniform_int_distribution<int> pick(0, n - 1);
    for (int r = 0; r < restarts; r++) {
        // initial: BFS growing from a random seed to n/2
        std::vector<char> side(n, 1);
        int cnt0 = 0, target = n / 2;
        std::vector<int> conn(n, 0);
        int seed = pick(rng);
        side[seed] = 0;
        cnt0 = 1;
        for (auto& e : adj[seed]) conn[e.first] += e.second;
        while (cnt0 < target) {
            int bv = -1, bc = -1;
            for (int v = 0; v < n; v++)
                if (side[v] == 1 && (conn[v] > bc || (conn[v] == bc && (rng() & 1)))) { bc = conn[v]; bv = v; }
            side[bv] = 0;
            cnt0++;
            for (auto& e : adj[bv]) conn[e.first] += e.second;
        }
        // FM passes
        auto cut_of = [&](const std::vector<char>& sd) {
            long c = 0;
            for (int v = 0; v < n; v++)
                for (auto& e : adj[v])
                    if (sd[v] != sd[e.first]) c += e.second;
            return c / 2;
        };
        long cut = cut_of(side);
        for (int pass = 0; pass < 8; pass++) {
            std::vector<int> gain(n, 0);
            for (int v = 0; v < n; v++)
                for (auto& e : adj[v]) gain[v] += (side[v] != side[e.first]) ? e.second : -e.second;
            std::vector<char> locked(n, 0);
            std::vector<int> moves;
            long cur = cut, bestc = cut;
            int best_len = 0;
            int c0 = cnt0;
            for (int step = 0; step < n; step++) {
                int bv = -1, bg = INT32_MIN;
                for (int v = 0; v < n; v++) {
                    if (locked[v]) continue;
                    int nc0 = c0 + (side[v] == 0 ? -1 : 1);
                    if (nc0 < lo || nc0 > hi) continue;
                    if (gain[v] > bg || (gain[v] == bg && (rng() & 3) == 0)) { bg = gain[v]; bv = v; }
                }
                if (bv < 0) break;
                locked[bv] = 1;
                c0 += (side[bv] == 0 ? -1 : 1);
                side[bv] ^= 1;
                cur -= bg;
                moves.push_back(bv);
                for (auto& e : adj[bv]) gain[e.first] += (side[e.first] == side[bv]) ? -2 * e.second : 2 * e.second;
                gain[bv] = -gain[bv];
                if (cur < bestc) { bestc = cur; best_len = (int)moves.size(); }
            }
            for (int i = (int)moves.size() - 1; i >= best_len; i--) side[moves[i]] ^= 1;
            cnt0 = 0;
            for (int v = 0; v < n; v++) cnt0 += side[v] == 0;
            if (bestc >= cut) { cut = bestc; break; }
            cut = bestc;
        }
        if (best_cut < 0 || cut < best_cut) { best_cut = cut; best = side; }
    }
    return best;
}

// greedy subtree over the leaves in V (appends nodes to t, returns the root node id)
int greedy_sub(Tree& t, const std::vector<int>& V, RowModel& rm) {
    std::vector<int> cur(V.begin(), V.end());  // node ids
    while (cur.size() > 1) {
        int ba = -1, bb = -1;
        double bs = 1e300;
        for (size_t i = 0; i < cur.size(); i++)
            for (size_t j = i + 1; j < cur.size(); j++) {
                const Node& A = t.nodes[cur[i]];
                const Node& B = t.nodes[cur[j]];
                Bits sh = A.legs & B.legs;
                bool share = false;
                for (int w = 0; w < W && !share; w++) share = sh.w[w] != 0;
                Bits C = A.legs ^ B.legs;
                double sC = rm.rows(A.q | B.q) * std::ldexp(1.0, C.count());
                double sA = A.rows * std::ldexp(1.0, A.legs.count()), sB = B.rows * std::ldexp(1.0, B.legs.count());
                double sc = sC - (sA + sB) + (share ? 0.0 : 1e200);
                if (sc < bs) { bs = sc; ba = (int)i; bb = (int)j; }
            }
        Node N;
        N.left = cur[ba];
        N.right = cur[bb];
        N.legs = t.nodes[N.left].legs ^ t.nodes[N.right].legs;
        N.q = t.nodes[N.left].q | t.nodes[N.right].q;
        N.rows = rm.rows(N.q);
        int id = (int)t.nodes.size();
        t.nodes[N.left].parent = id;
        t.nodes[N.right].parent = id;
        t.nodes.push_back(N);
        cur[ba] = id;
        cur.erase(cur.begin() + bb);
    }
    return cur[0];
}

int rb_rec(Tree& t, const std::vector<int>& V, const Graph& g, RowModel& rm, double eps, std::mt19937_64& rng,
           int cutoff) {
    if ((int)V.size() <= cutoff) return greedy_sub(t, V, rm);
    std::vector<char> side = fm_bisect(V, g, eps, rng, 6);
    std::vector<int> A, B;
    for (size_t i = 0; i < V.size(); i++) (side[i] ? B : A).push_back(V[i]);
    if (A.empty() || B.empty()) return greedy_sub(t, V, rm);
    int a = rb_rec(t, A, g, rm, eps, rng, cutoff);
    int b = rb_rec(t, B, g, rm, eps, rng, cutoff);
    Node N;
    N.left = a;
    N.right = b;
    N.legs = t.nodes[a].legs ^ t.nodes[b].legs;
    N.q = t.nodes[a].q | t.nodes[b].q;
    N.rows = rm.rows(N.q);
    int id = (int)t.nodes.size();
    t.nodes[a].parent = id;
    t.nodes[b].parent = id;
    t.nodes.push_back(N);
    return id;
}

Tree rb_tree(const std::vector<Leaf>& leaves, const Graph& g, RowModel& rm, double eps, int cutoff,
             std::mt19937_64& rng) {
    const int NL = (int)leaves.size();
    Tree t;
    t.nodes.resize(NL);
    for (int i = 0; i < NL; i++) {
        Node& N = t.nodes[i];
        N.leaf = i;
        for (int e : leaves[i].legs) N.legs.set(e);
        N.q = leaves[i].qmask;
        N.rows = (double)leaves[i].rows.size();
    }
    std::vector<int> V(NL);
    for (int i = 0; i < NL; i++) V[i] = i;
    t.root = rb_rec(t, V, g, rm, eps, rng, cutoff);
    return t;
}

// emit (i, j) pairs with the result stored at i (SPEC.md S:L252 convention)
std::vector<std::pair<int, int>> tree_order(const Tree& t) {
    std::vector<std::pair<int, int>> out;
    std::vector<int> rep(t.nodes.size(), -1);
    std::vector<std::pair<int, int>> st = {{t.root, 0}};
    while (!st.empty()) {
        auto [x, s] = st.back();
        st.pop_back();
        const Node& N = t.nodes[x];
        if (N.leaf >= 0) {
            rep[x] = N.leaf;
            continue;
        }
        if (s == 0) {
            st.push_back({x, 1});
            st.push_back({N.right, 0});
            st.push_back({N.left, 0});
        } else {
            out.push_back({rep[N.left], rep[N.right]});
            rep[x] = rep[N.left];
        }
    }
    return out;
}

}  // namespace

std::string find_plan(const Network& net, const std::vector<Leaf>& leaves, const Request& req,
                      const PlanOptions& opt, Plan& out) {
    const int NL = (int)leaves.size();
    if ((int)net.edges.size() > W * 64) return "network too large for the planner bitsets";
    RowModel rm;
    rm.req = &req;
    std::vector<int> slot_of_tensor(net.tensors.size(), -1);
    for (int i = 0; i < NL; i++) slot_of_tensor[leaves[i].tensor_id] = i;
    std::vector<int> internal;
    Bits internal_bits;
    for (int e = 0; e < (int)net.edges.size(); e++) {
        const Edge& E = net.edges[e];
        if (!E.output && E.t0 >= 0 && E.t1 >= 0 && net.tensors[E.t0].alive && net.tensors[E.t1].alive) {
            internal.push_back(e);
            internal_bits.set(e);
        }
    }
    for (int e : opt.forced)
        if (e < 0 || !internal_bits.get(e)) return "forced wire is not an internal edge of the simplified network";
    if (NL == 1) {
        out = Plan();
        for (int e : opt.forced) out.sliced.push_back(e);
        if (opt.n_sliced > (int)out.sliced.size()) return "nothing to slice in a single-tensor network";
        return "";
    }

    struct CompGuard {
        explicit CompGuard(const std::vector<std::pair<int, int>>* c) { g_companions = c; }
        ~CompGuard() { g_companions = nullptr; }
    } comp_guard(&opt.companions);
    std::mt19937_64 rng(opt.seed ? opt.seed : 1);
    const int trials = opt.trials > 0 ? opt.trials : 24;
    const double budget = opt.time_budget_s > 0 ? opt.time_budget_s : 30.0;
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };

    // ---------------- 1. greedy trees; keep the best few by unsliced modelled time
    std::vector<std::pair<double, Tree>> pool;
    Bits none;
    for (int trial = 0; trial < trials; trial++) {
        if (trial >= 2 && elapsed() > 0.25 * budget) break;
        const int crit = trial % 2;
        const double tau = (trial < 2) ? 0.0 : std::vector<double>{0.05, 0.1, 0.2, 0.4, 0.8}[(trial / 2) % 5];
        const double alpha = (trial < 2) ? 1.0 : std::vector<double>{1.0, 0.75, 1.25, 0.5}[(trial / 10) % 4];
        Tree t = greedy_tree(net, leaves, rm, internal, slot_of_tensor, crit, tau, alpha, rng);
        double tt = eval_tree(t, none).time;
        pool.push_back({tt, std::move(t)});
    }
    // recursive-bisection trees
    Graph g;
    g.adj.resize(NL);
    {
        std::map<std::pair<int, int>, int> w;
        for (int e : internal) {
            int a = slot_of_tensor[net.edges[e].t0], b = slot_of_tensor[net.edges[e].t1];
            if (a == b) continue;
            w[{std::min(a, b), std::max(a, b)}]++;
        }
        for (auto& kv : w) {
            g.adj[kv.first.first].push_back({kv.first.second, kv.second});
            g.adj[kv.first.second].push_back({kv.first.first, kv.second});
        }
    }
    const int rb_trials = NL > 24 ? std::max(8, trials) : 0;
    for (int trial = 0; trial < rb_trials; trial++) {
        if (trial >= 2 && elapsed() > 0.45 * budget) break;
        const double eps = std::vector<double>{0.1, 0.3, 0.5, 0.2, 0.05, 0.4}[trial % 6];
        const int cutoff = std::vector<int>{8, 12, 6, 10}[(trial / 6) % 4];
        Tree t = rb_tree(leaves, g, rm, eps, cutoff, rng);
        pool.push_back({0.0, std::move(t)});
    }
    // rank by a quick sliced estimate (greedy slicing to max_elems, no reconfiguration)
    for (auto& pt : pool) {
        Bits S;
        for (int e : opt.forced) S.set(e);
        int s = (int)opt.forced.size();
        for (int it = 0; it < 62; it++) {
            TreeEval ev = eval_tree(pt.second, S);
            if (ev.peak <= opt.max_elems && (opt.n_sliced < 0 || s >= opt.n_sliced)) break;
            Bits cand;
            const double thr = ev.peak > opt.max_elems ? opt.max_elems : ev.peak * 0.999;
            for (const Node& N : pt.second.nodes)
                if (node_size(N, S) > thr) cand = cand | N.legs;
            cand = andnot(cand & internal_bits, closure(S));
            if (ev.peak <= opt.max_elems) cand = andnot(internal_bits, closure(S));
            int be = -1;
            double bt = 1e300;
            for (int e : internal) {
                if (!cand.get(e)) continue;
                Bits S2 = S;
                S2.set(e);
                double tt = eval_tree(pt.second, S2).time;
                if (tt < bt) { bt = tt; be = e; }
            }
            if (be < 0) break;
            S.set(be);
            s++;
        }
        pt.first = std::ldexp(eval_tree(pt.second, S).time, s);
    }
    std::sort(pool.begin(), pool.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    const int keep = std::min<int>((int)pool.size(), 3);

    bool have = false;
    Plan best;
    double best_time = 1e300;
    std::string last_err = "no plan found";
    for (int c = 0; c < keep; c++) {
        Tree t = pool[c].second;
        const double cbudget = budget * (0.25 + 0.75 * (c + 1) / keep);
        Ctx cx{&rm, Bits(), opt.max_elems};
        std::vector<int> sliced;
        for (int e : opt.forced) {
            cx.sliced.set(e);
            sliced.push_back(e);
        }
        reconfigure(t, cx, cbudget, t0);
        bool ok = true;
        // ---------------- 2. slice + reconfigure
        while (true) {
            TreeEval ev = eval_tree(t, cx.sliced);
            const int s = (int)sliced.size();
            const bool need_peak = ev.peak > opt.max_elems;
            const bool need_count = opt.n_sliced >= 0 && s < opt.n_sliced;
            if (!need_peak && !need_count) break;
            if (opt.n_sliced >= 0 && s >= opt.n_sliced && need_peak) {
                ok = false;
                last_err = "max_tensor_size not reachable with the requested number of sliced edges";
                break;
            }
            if (s >= 62) { ok = false; last_err = "more than 62 sliced edges"; break; }
            const double thr = need_peak ? opt.max_elems : ev.peak * 0.999;
            Bits cand;
            for (const Node& N : t.nodes)
                if (node_size(N, cx.sliced) > thr) cand = cand | N.legs;
            cand = andnot(cand & internal_bits, closure(cx.sliced));
            if (!need_peak) cand = andnot(internal_bits, closure(cx.sliced));  // only the count is missing
            int be = -1;
            double bt = 1e300, bpeak = 1e300;
            for (int e : internal) {
                if (!cand.get(e)) continue;
                Bits S2 = cx.sliced;
                S2.set(e);
                TreeEval e2 = eval_tree(t, S2);
                double tt = std::ldexp(e2.time, s + 1);
                if (tt < bt * 0.999 || (tt < bt * 1.001 && e2.peak < bpeak)) {
                    bt = tt;
                    bpeak = e2.peak;
                    be = e;
                }
            }
            if (be < 0) {
                ok = false;
                last_err = "max_tensor_size is unreachable even with every edge sliced";
                break;
            }
            cx.sliced.set(be);
            sliced.push_back(be);
            if (elapsed() < cbudget) reconfigure(t, cx, cbudget, t0);
        }
        if (!ok) continue;
        TreeEval ev = eval_tree(t, cx.sliced);
        double tt = std::ldexp(ev.time, (int)sliced.size());
        if (!have || tt < best_time) {
            have = true;
            best_time = tt;
            best.order = tree_order(t);
            best.sliced = sliced;
            best.cmac = ev.cmac;
            best.bytes = ev.bytes;
            best.time_s = ev.time;
            best.peak = ev.peak;
        }
    }
    if (!have) return last_err;
    out = best;
    return "";
}

}  // namespace tnb
