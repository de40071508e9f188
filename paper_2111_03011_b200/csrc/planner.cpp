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
#include <cstdio>
#include <cstdlib>
#include <map>
#include <unordered_map>

#include "tnb.h"

namespace tnb {

// ------------------------------------------------------------------------------ row model

double RowModel::rows(uint64_t qmask) {
    if (qmask == 0) return 1.0;
    auto it = memo.find(qmask);
    if (it != memo.end()) return it->second;
    double r;
    if (req->fixed.size() <= (1u << 16)) {
        r = (double)rows_of(*req, qmask).size();
    } else {
        r = estimate(qmask);
    }
    memo[qmask] = r;
    return r;
}

// expected number of distinct keys when L uniform fixed parts are projected onto 2^|q| values
double RowModel::estimate(uint64_t qmask) const {
    if (qmask == 0) return 1.0;
    const double L = (double)req->fixed.size();
    const int q = __builtin_popcountll(qmask);
    const double V = std::ldexp(1.0, q);
    double r = V * (1.0 - std::exp(L * std::log1p(-1.0 / V)));
    return std::max(1.0, std::min(r, L));
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
    } else if (!(rowsA && rowsB) && [&]() {
                   // big stem x small rowless tensor: the fused tensor-core gate kernel (lower.cpp / gate_tc.cuh)
                   const bool a_small = !rowsA && (rowsB || sA < sB);
                   const int dsmall = a_small ? a : b, dbig = a_small ? b : a;
                   const double rbig = a_small ? rB : rA;
                   const int fb = dsmall - kk, fa = dbig - kk;
                   return kk >= 3 && kk <= 5 && fb >= 1 && fb <= 7 && fa <= 32 && (kk >= 4 || fb >= 4) &&
                          rbig * std::ldexp(1.0, fa) >= 1048576.0 && s.cmac >= 4.0 * 1048576.0 * 16;
               }()) {
        s.time = std::max(s.cmac / C_TC, s.bytes / BW) + T_LAUNCH;
    } else if (rowsA && rowsB && [&]() {
                   // gather-contract on the gate kernel (modes 1 / 2, lower.cpp): the bigger-per-row operand's free
                   // legs fill whole tiles, k fits the resident gate
                   const int fa = std::max(a, b) - kk;
                   return kk >= 3 && kk <= 5 && fa >= 7 && fa <= 32 && s.cmac >= 4.0 * 1048576.0 * 16;
               }()) {
        s.time = std::max(s.cmac / C_TC, s.bytes / BW) + T_LAUNCH;
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
    int seg = -1;        // loop-program segment of an internal node (-1: none); reconfiguration stays inside one
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
            if (N.leaf >= 0 || N.seg != t.nodes[v].seg) continue;
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
        N.seg = t.nodes[v].seg;
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

// ------------------------------------------------------------------------------ multilevel bisection trees
// Recursive multilevel hypergraph bisection (partition.cpp).  Nets: one per internal bond (weight 1 = one
// index bit), plus the "rows" net over the row-carrying leaves of the part (weight rows_w bits: splitting the
// sparse output boundary across both halves makes both carry rows).  Parts of <= cutoff leaves are finished
// greedily; subtree reconfiguration later re-optimises the small subtrees exactly.
struct RB2 {
    const std::vector<Leaf>* leaves;
    const Network* net;
    const std::vector<int>* slot_of_tensor;
    const std::vector<int>* internal;
    RowModel* rm;
    double eps_lo, eps_hi;
    int cutoff, rows_w;
    double fix_ext;  // probability that a bisection pins the part's external legs to one side
};

int rb2_rec(Tree& t, const std::vector<int>& V, const RB2& P, std::mt19937_64& rng, int depth) {
    if ((int)V.size() <= P.cutoff) return greedy_sub(t, V, *P.rm);
    std::unordered_map<int, int> loc;
    for (int i = 0; i < (int)V.size(); i++) loc[V[i]] = i;
    HyperGraph g;
    g.n = (int)V.size();
    g.node_w.assign(g.n, 1);
    for (int e : *P.internal) {
        auto a = loc.find((*P.slot_of_tensor)[P.net->edges[e].t0]);
        auto b = loc.find((*P.slot_of_tensor)[P.net->edges[e].t1]);
        if (a == loc.end() || b == loc.end() || a->second == b->second) continue;
        g.nets.push_back({a->second, b->second});
        g.net_w.push_back(1);
    }
    if (P.rows_w > 0) {
        std::vector<int> rp;
        for (int i = 0; i < g.n; i++)
            if ((*P.leaves)[V[i]].qmask) rp.push_back(i);
        if (rp.size() >= 2) {
            g.nets.push_back(rp);
            g.net_w.push_back(P.rows_w);
        }
    }
    // external legs (bonds to tensors outside V, open output legs): with probability fix_ext they are
    // pinned to one side through a weightless fixed node, so that one half takes the part's boundary and
    // the other is a compact branch with a small cut (stem-and-branch trees)
    if (depth > 0 && (rng() % 1000) < P.fix_ext * 1000) {
        const int X = g.n++;
        g.node_w.push_back(0);
        g.fixed.assign(g.n, -1);
        g.fixed[X] = 0;
        for (int i = 0; i < X; i++) {
            int ext = 0;
            for (int e : (*P.leaves)[V[i]].legs) {
                const Edge& E = P.net->edges[e];
                if (E.t1 < 0) { ext++; continue; }
                const int o = (*P.slot_of_tensor)[E.t0] == V[i] ? E.t1 : E.t0;
                if (!loc.count((*P.slot_of_tensor)[o])) ext++;
            }
            if (ext) {
                g.nets.push_back({i, X});
                g.net_w.push_back(ext);
            }
        }
    }
    // imbalance drawn per bisection from [eps_lo, eps_hi]
    const double eps = P.eps_lo + (P.eps_hi - P.eps_lo) * ((rng() % 10000) / 10000.0);
    std::vector<char> side = ml_bisect(g, eps, rng, 8);
    static const int vb = getenv("TNB_PLAN_VERBOSE") ? atoi(getenv("TNB_PLAN_VERBOSE")) : 0;
    if (vb >= 2 && depth <= 3) {
        int64_t c = 0;
        for (size_t e = 0; e < g.nets.size(); e++) {
            bool s0 = false, s1 = false;
            for (int v : g.nets[e]) (side[v] ? s1 : s0) = true;
            if (s0 && s1) c += g.net_w[e];
        }
        int n0 = 0;
        for (int i = 0; i < (int)V.size(); i++) n0 += !side[i];
        fprintf(stderr, "%*s[rb2] depth %d |V| %zu eps %.2f -> %d / %zu cut %lld\n", 2 * depth, "", depth, V.size(), eps, n0,
                V.size() - n0, (long long)c);
    }
    std::vector<int> A, B;
    for (int i = 0; i < (int)V.size(); i++) (side[i] ? B : A).push_back(V[i]);
    if (A.empty() || B.empty()) return greedy_sub(t, V, *P.rm);
    int a = rb2_rec(t, A, P, rng, depth + 1);
    int b = rb2_rec(t, B, P, rng, depth + 1);
    Node N;
    N.left = a;
    N.right = b;
    N.legs = t.nodes[a].legs ^ t.nodes[b].legs;
    N.q = t.nodes[a].q | t.nodes[b].q;
    N.rows = P.rm->rows(N.q);
    int id = (int)t.nodes.size();
    t.nodes[a].parent = id;
    t.nodes[b].parent = id;
    t.nodes.push_back(N);
    return id;
}

Tree rb2_tree(const RB2& P, std::mt19937_64& rng) {
    const std::vector<Leaf>& leaves = *P.leaves;
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
    t.root = rb2_rec(t, V, P, rng, 0);
    return t;
}

// ------------------------------------------------------------------------------ sweep (stem) orders
// A linear order pi of the leaves defines a stem tree: the stem absorbs pi[1], pi[2], ... one at a time
// (P:L429's head and tail are stems absorbing branches).  Step k costs rows(Q_k) * 2^|dV_{k-1} u legs(pi_k)|,
// dV = the boundary (dense legs) of the absorbed set.  Simulated annealing over single-leaf moves minimises
// the total; subtree reconfiguration later turns stem segments into small branches where that is cheaper.
struct Sweep {
    int NL = 0;
    std::vector<std::vector<std::pair<int, int>>> nbr;  // per leaf: (other endpoint leaf, edge) per internal leg
    std::vector<int> deg;                // dense legs per leaf (internal + open)
    std::vector<uint64_t> q;
    std::vector<char> sliced;            // per edge: 1 = sliced (own loop bit), 2 = companion tied to a sliced edge
    std::vector<int> tie;                // per edge: the sliced partner of a tied companion edge, else -1
    const std::vector<std::pair<int, int>>* comps = nullptr;  // (sliced edge, companion edge), add_companions order
    double tmax = 1e300;                 // soft bound on every stem size (per slice)
    int local = 1;                       // sum each sliced edge right after the step that closes it
    RowModel* rm = nullptr;
};

struct SweepState {
    std::vector<int> pi, pos;
    std::vector<int> B;        // boundary size after position k (sliced legs excluded)
    std::vector<int> Sk;       // sliced edges touched up to position k (the prefix of the slice order)
    std::vector<uint64_t> Q;   // fixed-qubit mask after position k
    std::vector<double> C;     // modelled cost at position k (0 for k = 0), including the peak penalty
    double total = 0;
};

// Cost of stem step k over all slices with prefix caching: the step depends on the sliced edges touched so
// far (S_k of them, the first S_k of the slice order), so it runs 2^S_k times; per run it costs
// rows * 2^|union| with the sliced legs removed.  Stems above tmax pay a steep penalty.
inline double sweep_cost(double rows, int uni, int b, int sk, double tmax) {
    double c = rows * std::ldexp(1.0, uni + sk);
    const double sz = rows * std::ldexp(1.0, b);
    if (sz > tmax) c *= 1e6 * (sz / tmax) * (sz / tmax);
    return c;
}

// recompute positions lo..hi (inclusive) from the state at lo-1; returns the new sum of C over lo..hi
// companion edges ("rank one approximation to companion edges"): every sliced edge's companion
// that add_companions would cut is tied to the partner's bit; the tie removes its dense leg but adds no loop
void sweep_retie(Sweep& S) {
    for (size_t e = 0; e < S.sliced.size(); e++)
        if (S.sliced[e] == 2) S.sliced[e] = 0;
    std::fill(S.tie.begin(), S.tie.end(), -1);
    if (!S.comps) return;
    for (const auto& pc : *S.comps)
        if (S.sliced[pc.first] == 1 && S.sliced[pc.second] == 0) {
            S.sliced[pc.second] = 2;
            S.tie[pc.second] = pc.first;
        }
}

inline double sweep_range(const Sweep& S, SweepState& st, int lo, int hi) {
    int b = lo > 0 ? st.B[lo - 1] : 0;
    int sk = lo > 0 ? st.Sk[lo - 1] : 0;
    uint64_t Q = lo > 0 ? st.Q[lo - 1] : 0;
    double sum = 0;
    for (int k = lo; k <= hi; k++) {
        const int v = st.pi[k];
        int shared = 0, sl_new = 0, sl_deg = 0, sl_close = 0;
        for (const auto& ue : S.nbr[v]) {
            if (S.sliced[ue.second]) {
                sl_deg++;
                if (S.sliced[ue.second] == 2) continue;
                if (st.pos[ue.first] > k) sl_new++;
                else sl_close++;
            } else {
                shared += st.pos[ue.first] < k;
            }
        }
        const int dv = S.deg[v] - sl_deg;
        const int uni = b + dv - shared;
        Q |= S.q[v];
        b = b + dv - 2 * shared;
        // the step depends on every sliced edge open at it (opened before or at k, closed at or after k); a
        // sliced edge is summed right after the step that closes it (local slicing), so later steps do not
        // depend on it.  S.local == 0: flat slicing with prefix caching (touched edges stay)
        const int dk = sk + sl_new;
        sk = S.local ? sk + sl_new - sl_close : sk + sl_new;
        st.B[k] = b;
        st.Sk[k] = sk;
        st.Q[k] = Q;
        st.C[k] = k == 0 ? 0.0 : sweep_cost(S.rm->estimate(Q), uni, b, dk, S.tmax);
        sum += st.C[k];
    }
    return sum;
}

void sweep_init(const Sweep& S, SweepState& st, const std::vector<int>& pi) {
    st.pi = pi;
    st.pos.assign(S.NL, 0);
    for (int k = 0; k < S.NL; k++) st.pos[pi[k]] = k;
    st.B.assign(S.NL, 0);
    st.Sk.assign(S.NL, 0);
    st.Q.assign(S.NL, 0);
    st.C.assign(S.NL, 0.0);
    st.total = sweep_range(S, st, 0, S.NL - 1);
}

// move the leaf at position i to position j (shifting the ones between)
inline void sweep_move(SweepState& st, int i, int j) {
    const int v = st.pi[i];
    if (i < j)
        for (int k = i; k < j; k++) { st.pi[k] = st.pi[k + 1]; st.pos[st.pi[k]] = k; }
    else
        for (int k = i; k > j; k--) { st.pi[k] = st.pi[k - 1]; st.pos[st.pi[k]] = k; }
    st.pi[j] = v;
    st.pos[v] = j;
}

void sweep_anneal(const Sweep& S, SweepState& st, std::mt19937_64& rng, int64_t iters, double T0, double T1) {
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<int> saveB, saveS;
    std::vector<uint64_t> saveQ;
    std::vector<double> saveC;
    double best_total = st.total;
    SweepState best = st;
    for (int64_t it = 0; it < iters; it++) {
        const double T = T0 * std::pow(T1 / T0, (double)it / (double)iters);
        const int i = (int)(rng() % (uint64_t)S.NL);
        const int w = (rng() % 8 == 0) ? S.NL : 12;
        int j = i + (int)(rng() % (uint64_t)(2 * w + 1)) - w;
        j = std::max(0, std::min(S.NL - 1, j));
        if (j == i) continue;
        const int lo = std::min(i, j), hi = std::max(i, j);
        double old = 0;
        for (int k = lo; k <= hi; k++) old += st.C[k];
        saveB.assign(st.B.begin() + lo, st.B.begin() + hi + 1);
        saveS.assign(st.Sk.begin() + lo, st.Sk.begin() + hi + 1);
        saveQ.assign(st.Q.begin() + lo, st.Q.begin() + hi + 1);
        saveC.assign(st.C.begin() + lo, st.C.begin() + hi + 1);
        sweep_move(st, i, j);
        const double nw = sweep_range(S, st, lo, hi);
        const double newtot = st.total - old + nw;
        const double d = std::log2(std::max(newtot, 1e-300)) - std::log2(std::max(st.total, 1e-300));
        if (d <= 0 || U(rng) < std::exp(-d / T)) {
            st.total = newtot;
            if (st.total < best_total) {
                best_total = st.total;
                best = st;
            }
        } else {
            sweep_move(st, j, i);
            std::copy(saveB.begin(), saveB.end(), st.B.begin() + lo);
            std::copy(saveS.begin(), saveS.end(), st.Sk.begin() + lo);
            std::copy(saveQ.begin(), saveQ.end(), st.Q.begin() + lo);
            std::copy(saveC.begin(), saveC.end(), st.C.begin() + lo);
        }
        if ((it & 0xffff) == 0xffff) st.total = sweep_range(S, st, 0, S.NL - 1);  // drift control
    }
    st = best;
    st.total = sweep_range(S, st, 0, S.NL - 1);
}

// Checkpointed loop program of a sliced stem (the head/tail "local slices" of P:L131-L136 generalised):
// checkpoints 0 = p_0 < p_1 < ... < p_J = NL-1 split the stem into segments (p_{j-1}, p_j].  A sliced edge
// opened at a_e and closed at b_e is looped over by every segment that overlaps [a_e, b_e] and summed at the
// end of the segment that contains b_e; edges still open in the last segment are the global slices (summed
// by the readout, split across pipelines and GPUs).  Segment (p, q] runs 2^#{e: a_e <= q, b_e > p} times;
// the stem at every checkpoint persists across loop iterations (the accumulator at summation points).
struct Checkpoints {
    std::vector<int> cp;      // checkpoint positions, cp.back() = NL-1
    double cost = 0;          // modelled CMAC over all global slices
    double persist = 0;       // elements persisted at internal checkpoints (one slice iteration)
};

struct StemEvents {
    std::vector<double> c;         // per position: rows * 2^|union| of one iteration (sliced legs fixed)
    std::vector<double> size;      // per position: stem size of one iteration
    std::vector<std::pair<int, int>> ab;  // per sliced edge: (open position, close position)
    std::vector<int> edge;         // sliced edge ids (same order)
};

StemEvents stem_events(const Sweep& S, const SweepState& st, const Network& net, const std::vector<int>& slot_of_tensor) {
    StemEvents ev;
    const int NL = S.NL;
    ev.c.assign(NL, 0.0);
    ev.size.assign(NL, 0.0);
    int b = 0;
    uint64_t Q = 0;
    for (int k = 0; k < NL; k++) {
        const int v = st.pi[k];
        int shared = 0, sl_deg = 0;
        for (const auto& ue : S.nbr[v]) {
            if (S.sliced[ue.second]) sl_deg++;
            else shared += st.pos[ue.first] < k;
        }
        const int dv = S.deg[v] - sl_deg;
        const int uni = b + dv - shared;
        Q |= S.q[v];
        b = b + dv - 2 * shared;
        const double r = S.rm->estimate(Q);
        ev.c[k] = k == 0 ? 0.0 : r * std::ldexp(1.0, uni);
        ev.size[k] = r * std::ldexp(1.0, b);
    }
    for (int e = 0; e < (int)S.sliced.size(); e++) {
        if (S.sliced[e] != 1) continue;
        int lo = std::min(st.pos[slot_of_tensor[net.edges[e].t0]], st.pos[slot_of_tensor[net.edges[e].t1]]);
        int hi = std::max(st.pos[slot_of_tensor[net.edges[e].t0]], st.pos[slot_of_tensor[net.edges[e].t1]]);
        // a tied companion reads the same bit: the loop spans its endpoints too
        for (int c = 0; c < (int)S.tie.size(); c++)
            if (S.tie[c] == e)
                for (int t : {net.edges[c].t0, net.edges[c].t1}) {
                    lo = std::min(lo, st.pos[slot_of_tensor[t]]);
                    hi = std::max(hi, st.pos[slot_of_tensor[t]]);
                }
        ev.ab.push_back({lo, hi});
        ev.edge.push_back(e);
    }
    return ev;
}

// exact DP over checkpoint sets with at most J segments; persisted memory is charged lambda CMAC per element
Checkpoints checkpoint_dp(const StemEvents& ev, int J, double lambda) {
    const int K = (int)ev.c.size();
    std::vector<double> pre(K + 1, 0.0);
    for (int k = 0; k < K; k++) pre[k + 1] = pre[k] + ev.c[k];
    auto seg = [&](int p, int q) {  // steps p+1..q; edges with a <= q and b > p
        int n = 0;
        double acc = 0;
        for (const auto& x : ev.ab) {
            if (x.first <= q && x.second > p) {
                n++;
                if (x.second <= q && q < K - 1) acc = 1;  // a summation at q (an accumulate pass)
            }
        }
        return (pre[q + 1] - pre[p + 1] + acc * 3 * ev.size[q]) * std::ldexp(1.0, n);
    };
    const double INF = 1e308;
    std::vector<std::vector<double>> D(J + 1, std::vector<double>(K, INF));
    std::vector<std::vector<int>> arg(J + 1, std::vector<int>(K, -1));
    D[0][0] = 0;
    for (int j = 1; j <= J; j++)
        for (int q = 1; q < K; q++)
            for (int p = 0; p < q; p++) {
                if (D[j - 1][p] >= INF) continue;
                const double v = D[j - 1][p] + seg(p, q) + (p > 0 ? lambda * ev.size[p] : 0.0);
                if (v < D[j][q]) {
                    D[j][q] = v;
                    arg[j][q] = p;
                }
            }
    Checkpoints best;
    best.cost = INF;
    int bj = -1;
    for (int j = 1; j <= J; j++)
        if (D[j][K - 1] < best.cost) {
            best.cost = D[j][K - 1];
            bj = j;
        }
    for (int q = K - 1, j = bj; j > 0; q = arg[j][q], j--) best.cp.push_back(q);
    std::reverse(best.cp.begin(), best.cp.end());
    best.cost = 0;
    best.persist = 0;
    int p = 0;
    for (int q : best.cp) {
        best.cost += seg(p, q);
        if (q < K - 1) best.persist += ev.size[q];
        p = q;
    }
    return best;
}

// Loop nest of a checkpointed stem.  Every sliced edge gets the segment interval [a, b] over which it is looped
// (opened at segment a, summed at the end of segment b; b = J-1: a global slice, summed by the readout).  The
// intervals are made laminar (nested or disjoint) by extending crossing ones -- the cheaper of "sum the earlier
// one later" and "open the later one earlier" -- so that the loops form a proper nest: each segment then runs
// exactly 2^|D_j| times, D_j = the intervals containing j.  Bit significance = preorder of the interval forest
// (outer loops and earlier sequential loops more significant): with it, no segment re-runs because of a loop
// it does not depend on, and every summation completes before its consumers run.
struct LoopNest {
    std::vector<int> a, b;        // per sliced edge (StemEvents order)
    std::vector<int> order;       // edge indices, most significant first
    std::vector<double> segc;     // per segment: modelled CMAC of one run (steps + accumulate pass)
    double cost = 0;              // sum_j segc[j] * 2^|D_j|
};

double nest_cost(const std::vector<double>& segc, const std::vector<int>& a, const std::vector<int>& b) {
    double c = 0;
    for (int j = 0; j < (int)segc.size(); j++) {
        int d = 0;
        for (size_t e = 0; e < a.size(); e++) d += a[e] <= j && j <= b[e];
        c += segc[j] * std::ldexp(1.0, d);
    }
    return c;
}

LoopNest loop_nest(const StemEvents& ev, const std::vector<int>& cp, int min_global) {
    const int J = (int)cp.size(), ns = (int)ev.edge.size(), K = (int)ev.c.size();
    auto seg_of_pos = [&](int pos) {
        int j = 0;
        while (cp[j] < pos) j++;
        return j;
    };
    LoopNest L;
    L.a.resize(ns);
    L.b.resize(ns);
    for (int e = 0; e < ns; e++) {
        L.a[e] = seg_of_pos(std::max(1, ev.ab[e].first));
        L.b[e] = seg_of_pos(ev.ab[e].second);
    }
    std::vector<double> base(J, 0.0);
    for (int k = 1; k < K; k++) base[seg_of_pos(k)] += ev.c[k];
    auto costs = [&]() {  // segment costs incl. one accumulate pass where a local loop ends
        std::vector<double> sc = base;
        for (int j = 0; j + 1 < J; j++) {
            bool acc = false;
            for (int e = 0; e < ns; e++) acc = acc || L.b[e] == j;
            if (acc) sc[j] += 3 * ev.size[cp[j]];
        }
        return sc;
    };
    auto laminarize = [&]() {
        for (int guard = 0; guard < 100000; guard++) {
            int x = -1, y = -1;
            for (int i = 0; i < ns && x < 0; i++)
                for (int k = 0; k < ns; k++)
                    if (L.a[i] < L.a[k] && L.a[k] <= L.b[i] && L.b[i] < L.b[k]) {
                        x = i;
                        y = k;
                        break;
                    }
            if (x < 0) return;
            const std::vector<double> sc = costs();
            std::vector<int> b1 = L.b, a2 = L.a;
            b1[x] = L.b[y];      // sum x later
            a2[y] = L.a[x];      // open y earlier
            if (nest_cost(sc, L.a, b1) <= nest_cost(sc, a2, L.b)) L.b = b1;
            else L.a = a2;
        }
    };
    laminarize();
    for (;;) {  // at least min_global global slices: promote the cheapest local loops
        int ng = 0;
        for (int e = 0; e < ns; e++) ng += L.b[e] == J - 1;
        if (ng >= std::min(min_global, ns)) break;
        int be = -1;
        double bc = 1e308;
        const std::vector<double> sc = costs();
        for (int e = 0; e < ns; e++) {
            if (L.b[e] == J - 1) continue;
            std::vector<int> b1 = L.b;
            b1[e] = J - 1;
            const double c = nest_cost(sc, L.a, b1);
            if (c < bc) { bc = c; be = e; }
        }
        L.b[be] = J - 1;
        laminarize();
    }
    L.segc = costs();
    L.cost = nest_cost(L.segc, L.a, L.b);
    // preorder of the laminar forest: start ascending, end descending (parents before children)
    L.order.resize(ns);
    for (int e = 0; e < ns; e++) L.order[e] = e;
    std::stable_sort(L.order.begin(), L.order.end(), [&](int x, int y) {
        if (L.a[x] != L.a[y]) return L.a[x] < L.a[y];
        return L.b[x] > L.b[y];
    });
    return L;
}

Tree sweep_tree(const std::vector<Leaf>& leaves, const std::vector<int>& pi, RowModel& rm) {
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
    int cur = pi[0];
    for (int k = 1; k < NL; k++) {
        Node N;
        N.left = cur;
        N.right = pi[k];
        N.legs = t.nodes[cur].legs ^ t.nodes[pi[k]].legs;
        N.q = t.nodes[cur].q | t.nodes[pi[k]].q;
        N.rows = rm.rows(N.q);
        const int id = (int)t.nodes.size();
        t.nodes[cur].parent = id;
        t.nodes[pi[k]].parent = id;
        t.nodes.push_back(N);
        cur = id;
    }
    t.root = cur;
    return t;
}

// leaves of a tree in depth-first order (a nested-dissection linear order for rb2 trees)
std::vector<int> leaf_order(const Tree& t) {
    std::vector<int> out, st = {t.root};
    while (!st.empty()) {
        const int x = st.back();
        st.pop_back();
        const Node& N = t.nodes[x];
        if (N.leaf >= 0) { out.push_back(N.leaf); continue; }
        st.push_back(N.right);
        st.push_back(N.left);
    }
    return out;
}

// loop programs: (i, j) pairs plus the segment of each step, children visited stem-first (the child whose
// subtree holds the lowest segment first), so that segments are nondecreasing in program order
std::vector<std::pair<int, int>> tree_order_seg(const Tree& t, std::vector<int>& step_seg) {
    std::vector<int> minseg(t.nodes.size(), INT_MAX);
    std::function<int(int)> ms = [&](int x) -> int {
        const Node& N = t.nodes[x];
        if (N.leaf >= 0) return minseg[x] = INT_MAX;
        return minseg[x] = std::min(N.seg, std::min(ms(N.left), ms(N.right)));
    };
    ms(t.root);
    std::vector<std::pair<int, int>> out;
    step_seg.clear();
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
        const bool swap = minseg[N.right] < minseg[N.left];
        const int first = swap ? N.right : N.left, second = swap ? N.left : N.right;
        if (s == 0) {
            st.push_back({x, 1});
            st.push_back({second, 0});
            st.push_back({first, 0});
        } else {
            out.push_back({rep[first], rep[second]});
            step_seg.push_back(N.seg);
            rep[x] = rep[first];
        }
    }
    return out;
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

// The loop-program planner (method 2): stem sweeps with local slicing and checkpointed segments.
//   1. multilevel-bisection trees give nested-dissection leaf orders;
//   2. each order is annealed as a stem (sweep_anneal), then sliced edge by edge under max_elems with the
//      local-summation cost model, re-annealing after every slice;
//   3. checkpoint_dp picks <= max_segments segments under the persistence budget;
//   4. the best program by modelled CMAC becomes the plan (order = the stem, segments, global/local bits).
std::string sweep_plan(const Network& net, const std::vector<Leaf>& leaves, const Request& req, const PlanOptions& opt,
                       const std::vector<int>& internal, const std::vector<int>& slot_of_tensor, RowModel& rm,
                       std::mt19937_64& rng, double budget, Plan& out) {
    static const bool verbose = getenv("TNB_PLAN_VERBOSE") != nullptr;
    const int NL = (int)leaves.size();
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    Bits none;
    // ---------------- 1. bisection trees (their leaf orders seed the sweeps)
    RB2 P{&leaves, &net, &slot_of_tensor, &internal, &rm, 0.0, 0.0, 0, 0, 0.0};
    std::vector<std::pair<double, Tree>> hp;
    const double L2 = std::log2(std::max<double>(1.0, (double)req.fixed.size()));
    const int rb_trials = std::max(4, opt.trials > 0 ? opt.trials : 64);
    for (int trial = 0; trial < rb_trials && (trial < 4 || elapsed() < 0.25 * budget); trial++) {
        P.eps_lo = std::vector<double>{0.01, 0.05, 0.1, 0.2}[rng() % 4];
        P.eps_hi = P.eps_lo + std::vector<double>{0.0, 0.1, 0.3, 0.6}[rng() % 4];
        P.cutoff = 2 + (int)(rng() % 12);
        P.rows_w = (int)std::lround(L2 * std::vector<double>{0.0, 0.25, 0.5, 1.0, 2.0}[rng() % 5]);
        P.fix_ext = 0.0;
        Tree t = rb2_tree(P, rng);
        TreeEval ev = eval_tree(t, none);
        hp.push_back({ev.cmac, std::move(t)});
    }
    std::sort(hp.begin(), hp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    if (verbose)
        for (int k = 0; k < std::min<int>(5, (int)hp.size()); k++)
            fprintf(stderr, "[plan] bisection tree %d: unsliced %.3e CMAC, peak 2^%.1f (%zu trees, %.1f s)\n", k,
                    hp[k].first, std::log2(eval_tree(hp[k].second, none).peak), hp.size(), elapsed());
    // ---------------- 2. sweeps
    Sweep S;
    S.NL = NL;
    S.rm = &rm;
    S.nbr.resize(NL);
    S.deg.resize(NL);
    S.q.resize(NL);
    S.sliced.assign(net.edges.size(), 0);
    S.tie.assign(net.edges.size(), -1);
    if (!opt.companions.empty()) S.comps = &opt.companions;
    for (int i = 0; i < NL; i++) {
        S.deg[i] = (int)leaves[i].legs.size();
        S.q[i] = leaves[i].qmask;
    }
    for (int e : internal) {
        const int a = slot_of_tensor[net.edges[e].t0], b = slot_of_tensor[net.edges[e].t1];
        S.nbr[a].push_back({b, e});
        S.nbr[b].push_back({a, e});
    }
    // sweep objective: TNB_SWEEP_LOCAL=0 anneals under prefix caching only (every touched sliced edge stays open),
    // which is what the laminar loop nest mostly reduces to when the stem keeps its sliced legs to the end
    if (getenv("TNB_SWEEP_LOCAL")) S.local = atoi(getenv("TNB_SWEEP_LOCAL"));
    int64_t iters = opt.sweep_iters > 0 ? opt.sweep_iters : std::max<int64_t>(20000, (int64_t)NL * 4000);
    if (getenv("TNB_SWEEP_ITERS")) iters = atoll(getenv("TNB_SWEEP_ITERS"));
    const double pbudget = opt.persist_budget > 0 ? opt.persist_budget : 8.0 * opt.max_elems;
    auto peak_of = [&](const SweepState& x) {
        double pk = 0;
        for (int i = 0; i < NL; i++) pk = std::max(pk, rm.estimate(x.Q[i]) * std::ldexp(1.0, x.B[i]));
        return pk;
    };
    bool have = false;
    double best_cost = 1e308;
    SweepState best_st;
    std::vector<char> best_sliced;
    Checkpoints best_cp;
    StemEvents best_ev;
    for (int k = 0; k < (int)hp.size() && (k < 2 || elapsed() < budget); k++) {
        std::fill(S.sliced.begin(), S.sliced.end(), 0);
        for (int e : opt.forced) S.sliced[e] = 1;
        sweep_retie(S);
        S.tmax = 1e300;
        SweepState st;
        sweep_init(S, st, leaf_order(hp[k].second));
        sweep_anneal(S, st, rng, iters, 0.5, 0.01);
        S.tmax = opt.max_elems;
        bool ok = true;
        for (int ns = 0;; ns++) {
            st.total = sweep_range(S, st, 0, NL - 1);
            if (peak_of(st) <= opt.max_elems) break;
            if (ns >= 62) { ok = false; break; }
            std::vector<char> cand(net.edges.size(), 0);
            for (int i = 0; i < NL; i++) {
                if (rm.estimate(st.Q[i]) * std::ldexp(1.0, st.B[i]) <= opt.max_elems) continue;
                for (int j = 0; j <= i; j++)
                    for (const auto& ue : S.nbr[st.pi[j]])
                        if (!S.sliced[ue.second] && st.pos[ue.first] > i) cand[ue.second] = 1;
            }
            int be = -1;
            double bt = 1e308;
            SweepState tmp = st;
            for (int e : internal) {
                if (!cand[e]) continue;
                const char was = S.sliced[e];
                S.sliced[e] = 1;
                if (S.comps) sweep_retie(S);
                const double tt = sweep_range(S, tmp, 0, NL - 1);
                S.sliced[e] = was;
                if (S.comps) sweep_retie(S);
                if (tt < bt) { bt = tt; be = e; }
            }
            if (be < 0) { ok = false; break; }
            S.sliced[be] = 1;
            sweep_retie(S);
            st.total = sweep_range(S, st, 0, NL - 1);
            sweep_anneal(S, st, rng, iters / 8, 0.2, 0.01);
        }
        if (!ok) continue;
        // leaves larger than the bound cannot be sliced further by this planner
        StemEvents sev = stem_events(S, st, net, slot_of_tensor);
        // checkpoints: the DP's candidates for every segment count, scored by the laminar loop nest's cost
        Checkpoints c;
        c.cost = 1e308;
        for (int Jc = 1; Jc <= std::max(1, opt.max_segments); Jc++) {
            Checkpoints cj;
            for (double lambda = 0.0;; lambda = lambda > 0 ? lambda * 4 : 1e-3) {
                cj = checkpoint_dp(sev, Jc, lambda);
                if (cj.persist <= pbudget || lambda > 1e12) break;
            }
            if (cj.persist > pbudget) continue;
            cj.cost = loop_nest(sev, cj.cp, std::max(0, opt.n_sliced)).cost;
            if (cj.cost < c.cost) c = cj;
        }
        if (c.cp.empty()) continue;
        if (verbose)
            fprintf(stderr, "[plan] sweep %d: s %zu, %zu segments, cost %.3e, persist 2^%.1f, peak 2^%.1f (%.1f s)\n", k,
                    sev.edge.size(), c.cp.size(), c.cost, std::log2(std::max(1.0, c.persist)), std::log2(peak_of(st)),
                    elapsed());
        if (!have || c.cost < best_cost) {
            have = true;
            best_cost = c.cost;
            best_st = st;
            best_sliced = S.sliced;
            best_cp = c;
            best_ev = sev;
        }
    }
    if (!have) return "the loop-program planner found no plan within max_tensor_size and the persistence budget";
    // ---------------- 3. the plan: stem order, bits, segments
    Plan pl;
    Tree t = sweep_tree(leaves, best_st.pi, rm);
    const std::vector<int>& cp = best_cp.cp;
    const int J = (int)cp.size();
    auto seg_of_pos = [&](int pos) {
        int j = 0;
        while (cp[j] < pos) j++;
        return j;
    };
    for (int k = 1; k < NL; k++) t.nodes[NL + k - 1].seg = seg_of_pos(k);
    // branch merging inside each segment: subtree reconfiguration under the
    // roofline-time model turns runs of small absorptions into branches contracted first and absorbed by
    // one tensor-core-sized step; it never moves work across a checkpoint
    Bits Sall;
    for (int e = 0; e < (int)best_sliced.size(); e++)
        if (best_sliced[e] == 1) Sall.set(e);
    const double t_before = eval_tree(t, Sall).time;
    if (!(getenv("TNB_NO_MERGE") && atoi(getenv("TNB_NO_MERGE")) != 0)) {
        Ctx cx{&rm, Sall, opt.max_elems};
        reconfigure(t, cx, elapsed() + std::max(2.0, 0.25 * budget), t0);
    }
    const double t_after = eval_tree(t, Sall).time;
    pl.order = tree_order_seg(t, pl.step_seg);
    // loop nest: laminar intervals, at least opt.n_sliced global slices, bit order = interval-forest preorder
    const int ns = (int)best_ev.edge.size();
    LoopNest LN = loop_nest(best_ev, cp, std::max(0, opt.n_sliced));
    pl.n_global = 0;
    for (int r = 0; r < ns; r++) {
        const int e = LN.order[r];
        pl.sliced.push_back(best_ev.edge[e]);
        pl.is_global.push_back(LN.b[e] == J - 1 ? 1 : 0);
        pl.n_global += LN.b[e] == J - 1;
    }
    auto bit = [&](int rank) { return 1ull << (ns - 1 - rank); };
    pl.segs.resize(J);
    for (int j = 0; j < J; j++) {
        for (int r = 0; r < ns; r++) {
            const int e = LN.order[r];
            if (LN.a[e] <= j && j <= LN.b[e]) pl.segs[j].D |= bit(r);
            if (LN.b[e] == j && j < J - 1) pl.segs[j].E |= bit(r);
            if (LN.b[e] < j) pl.segs[j].Sum |= bit(r);
        }
    }
    pl.total_cmac = LN.cost;
    pl.persist_elems = best_cp.persist;
    TreeEval ev = eval_tree(t, Bits());
    (void)ev;
    // per-iteration figures of the sliced network (cmac of one pass over every step)
    {
        double c = 0, pk = 0;
        for (int k = 0; k < NL; k++) {
            c += best_ev.c[k];
            pk = std::max(pk, best_ev.size[k]);
        }
        pl.cmac = c;
        pl.peak = pk;
    }
    // modelled time over all slices: per segment, the tree's step times of one iteration x its runs
    {
        std::vector<double> segt(J, 0.0);
        for (int x = NL; x < (int)t.nodes.size(); x++)
            if (t.nodes[x].seg >= 0) segt[t.nodes[x].seg] += node_step(t, x, Sall).time;
        pl.time_s = 0;
        for (int j = 0; j < J; j++) pl.time_s += segt[j] * std::ldexp(1.0, __builtin_popcountll(pl.segs[j].D));
    }
    if (verbose) {
        fprintf(stderr, "[plan] branch merge: one-iteration model time %.3e -> %.3e s; whole program %.3e s\n", t_before,
                t_after, pl.time_s);
        fprintf(stderr, "[plan] loop program: %d global + %d local bits, %d segments, total %.3e CMAC, persist 2^%.1f\n",
                pl.n_global, ns - pl.n_global, J, pl.total_cmac, std::log2(std::max(1.0, pl.persist_elems)));
        for (int j = 0; j < J; j++)
            fprintf(stderr, "[plan]   seg %d: steps ..%d  |D| %d  |Sum| %d  |E| %d  run %.3e CMAC x 2^%d = %.3e  stem 2^%.1f rows 2^%.1f\n",
                    j, cp[j], __builtin_popcountll(pl.segs[j].D), __builtin_popcountll(pl.segs[j].Sum),
                    __builtin_popcountll(pl.segs[j].E), LN.segc[j], __builtin_popcountll(pl.segs[j].D),
                    LN.segc[j] * std::ldexp(1.0, __builtin_popcountll(pl.segs[j].D)), std::log2(best_ev.size[cp[j]]),
                    std::log2(rm.estimate(best_st.Q[cp[j]])));
    }
    out = pl;
    return "";
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

    const int method = opt.method != 0 ? opt.method : (NL > 160 ? 2 : 1);
    if (method == 2) {
        return sweep_plan(net, leaves, req, opt, internal, slot_of_tensor, rm, rng, budget, out);
    }
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
    const bool hyper = false;
    static const bool verbose = getenv("TNB_PLAN_VERBOSE") != nullptr;
    const int rb_trials = (NL > 24 && !hyper) ? std::max(8, trials) : 0;
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
        if (verbose) {
            TreeEval e0 = eval_tree(pt.second, none), e1 = eval_tree(pt.second, S);
            fprintf(stderr, "[plan] pool: unsliced cmac %.3e peak 2^%.1f -> s %d total cmac %.3e time %.3e s\n", e0.cmac,
                    std::log2(e0.peak), s, std::ldexp(e1.cmac, s), pt.first);
        }
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
