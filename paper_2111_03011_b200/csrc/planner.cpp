// planner.cpp -- contraction order ("contracting neighboring tensors in a complexity-greedy
// manner") and slicing ("select some indices ... and fix them ... in order to decrease the
// overall space complexity").  Setup, not the hot path.
//
// Randomised greedy (several criteria x temperatures, best of `trials`) followed by greedy
// slicing; plans are ranked by a roofline-time model of one slice times 2^s (SURVEY §7.3 H2:
// "the planner objective should be roofline time, not flops").
#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <set>
#include <sstream>

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

struct PStep {
    Bits A, B, C;     // dense legs of operands and result
    double rA, rB, rC;
    bool rowsA, rowsB;
};

// roofline constants of the model (B200): HBM copy 6.5 TB/s, 3xTF32 complex
// ~30e12 CMAC/s on the tensor-core path, ~6e12 CMAC/s for the SIMT path, ~3 us per launch.
constexpr double BW = 5.5e12, C_TC = 25e12, C_SIMT = 5e12, T_LAUNCH = 3e-6;

struct Eval {
    double cmac = 0, bytes = 0, time = 0, peak = 0, gemm_cmac = 0;
};

Eval evaluate(const std::vector<PStep>& steps, const std::vector<Bits>& leaves, const std::vector<double>& leaf_rows,
              const Bits& S) {
    Eval e;
    for (size_t i = 0; i < leaves.size(); i++)
        e.peak = std::max(e.peak, leaf_rows[i] * std::ldexp(1.0, popc_andnot(leaves[i], S)));
    for (const PStep& p : steps) {
        const int a = popc_andnot(p.A, S), b = popc_andnot(p.B, S), c = popc_andnot(p.C, S);
        const int u = popc_andnot(p.A | p.B, S);
        const double sA = p.rA * std::ldexp(1.0, a), sB = p.rB * std::ldexp(1.0, b), sC = p.rC * std::ldexp(1.0, c);
        const double cmac = p.rC * std::ldexp(1.0, u);
        const int k = a + b - c;  // shared (each shared leg counted in a and b, absent from c)
        const int kk = k / 2;
        double bytes = 8.0 * (sA + sB + sC);
        double t;
        // tensor-core path: exactly one side carries rows (or none), m >= 128, n >= 64, k >= 16
        bool both_rows = p.rowsA && p.rowsB;
        double m = 0, n = 0;
        if (!both_rows) {
            bool a_is_m = p.rowsA || (!p.rowsB && sA >= sB);
            double sM = a_is_m ? sA : sB, sN = a_is_m ? sB : sA;
            double rM = a_is_m ? p.rA : p.rB;
            (void)rM;
            m = sM / std::ldexp(1.0, kk);
            n = sN / std::ldexp(1.0, kk);
            // N operand has no rows here
        }
        if (!both_rows && m >= 128 && n >= 64 && kk >= 4) {
            double ops_bytes = bytes + 8.0 * (4.0 * (sA + sB));  // pre-pass split + reread
            t = std::max(cmac / C_TC, ops_bytes / BW) + 3 * T_LAUNCH;
            e.gemm_cmac += cmac;
        } else {
            t = std::max(cmac / C_SIMT, bytes / BW) + T_LAUNCH;
        }
        e.cmac += cmac;
        e.bytes += bytes;
        e.time += t;
        e.peak = std::max(e.peak, sC);
    }
    return e;
}

}  // namespace

std::string find_plan(const Network& net, const std::vector<Leaf>& leaves, const Request& req,
                      const PlanOptions& opt, Plan& out) {
    const int NL = (int)leaves.size();
    if ((int)net.edges.size() > W * 64) return "network too large for the planner bitsets";
    RowModel rm;
    rm.req = &req;

    std::vector<Bits> lb(NL);
    std::vector<double> lrows(NL);
    std::vector<uint64_t> lq(NL);
    std::vector<int> slot_of_tensor(net.tensors.size(), -1);
    for (int i = 0; i < NL; i++) {
        for (int e : leaves[i].legs) lb[i].set(e);
        lrows[i] = (double)leaves[i].rows.size();
        lq[i] = leaves[i].qmask;
        slot_of_tensor[leaves[i].tensor_id] = i;
    }
    // internal edges (sliceable): both endpoints are tensors
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

    std::mt19937_64 rng(opt.seed ? opt.seed : 1);
    const int trials = opt.trials > 0 ? opt.trials : 48;
    const double budget = opt.time_budget_s > 0 ? opt.time_budget_s : 20.0;
    auto t0 = std::chrono::steady_clock::now();

    bool have = false;
    Plan best;
    double best_time = 1e300;
    std::string last_err = "no plan found";

    for (int trial = 0; trial < trials; trial++) {
        double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (have && elapsed > budget) break;
        // criterion / temperature schedule
        const int crit = trial % 2;               // 0: absolute size reduction, 1: relative growth
        const double tau = (trial < 2) ? 0.0 : std::vector<double>{0.05, 0.1, 0.2, 0.4, 0.8}[(trial / 2) % 5];
        const double alpha = (trial < 2) ? 1.0 : std::vector<double>{1.0, 0.75, 1.25, 0.5}[(trial / 10) % 4];
        std::extreme_value_distribution<double> gumbel(0.0, 1.0);  // Gumbel

        // ---------------- greedy order
        std::vector<Bits> cur = lb;
        std::vector<uint64_t> cq = lq;
        std::vector<double> cr = lrows;
        std::vector<char> alive(NL, 1);
        std::vector<std::pair<int, int>> order;
        std::vector<PStep> steps;
        // edge endpoints in slot space
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
            if (cand.empty()) {  // disconnected components: outer product of the two smallest
                std::vector<std::pair<double, int>> sz;
                for (int i = 0; i < NL; i++)
                    if (alive[i]) sz.push_back({cr[i] * std::ldexp(1.0, cur[i].count()), i});
                std::sort(sz.begin(), sz.end());
                ba = sz[0].second;
                bb = sz[1].second;
            } else {
                double bs = 1e300;
                for (auto& pr : cand) {
                    int a = pr.first, b = pr.second;
                    Bits C = cur[a] ^ cur[b];
                    double rC = rm.rows(cq[a] | cq[b]);
                    double sC = rC * std::ldexp(1.0, C.count());
                    double sA = cr[a] * std::ldexp(1.0, cur[a].count()), sB = cr[b] * std::ldexp(1.0, cur[b].count());
                    double sc;
                    if (crit == 0) sc = sC - alpha * (sA + sB);
                    else sc = std::log2(sC) - alpha * std::log2(sA + sB);
                    if (tau > 0) {
                        double g = gumbel(rng);
                        sc = (crit == 0) ? sc - tau * g * (sA + sB) : sc - tau * g;
                    }
                    if (sc < bs) { bs = sc; ba = a; bb = b; }
                }
            }
            // keep the larger operand's slot for the result (i in (i, j))
            PStep ps;
            ps.A = cur[ba];
            ps.B = cur[bb];
            ps.rA = cr[ba];
            ps.rB = cr[bb];
            ps.rowsA = cq[ba] != 0;
            ps.rowsB = cq[bb] != 0;
            Bits C = cur[ba] ^ cur[bb];
            double rC = rm.rows(cq[ba] | cq[bb]);
            ps.C = C;
            ps.rC = rC;
            steps.push_back(ps);
            order.push_back({ba, bb});
            cur[ba] = C;
            cq[ba] = cq[ba] | cq[bb];
            cr[ba] = rC;
            alive[bb] = 0;
            n_alive--;
            for (int e : internal) {
                if (ends[e].first == bb) ends[e].first = ba;
                if (ends[e].second == bb) ends[e].second = ba;
                if (ends[e].first == ba && ends[e].second == ba) ends[e] = {-1, -1};
            }
        }

        // ---------------- slicing
        Bits S;
        std::vector<int> sliced;
        for (int e : opt.forced) {
            S.set(e);
            sliced.push_back(e);
        }
        Eval ev = evaluate(steps, lb, lrows, S);
        auto total_time = [&](const Eval& x, int s) { return std::ldexp(x.time, s); };
        bool ok = true;
        while (true) {
            int s = (int)sliced.size();
            bool need_peak = ev.peak > opt.max_elems;
            bool need_count = opt.n_sliced >= 0 && s < opt.n_sliced;
            if (!need_peak && !need_count) break;
            if (opt.n_sliced >= 0 && s >= opt.n_sliced && need_peak) { ok = false; last_err = "max_tensor_size not reachable with the requested number of sliced edges"; break; }
            // candidate edges: internal, unsliced, present in some tensor larger than the bound
            // (or in the largest tensor when only the count is missing)
            Bits cand_bits;
            double thr = need_peak ? opt.max_elems : ev.peak * 0.999;
            for (size_t i = 0; i < lb.size(); i++)
                if (lrows[i] * std::ldexp(1.0, popc_andnot(lb[i], S)) > thr) cand_bits = cand_bits | lb[i];
            for (const PStep& p : steps)
                if (p.rC * std::ldexp(1.0, popc_andnot(p.C, S)) > thr) cand_bits = cand_bits | p.C;
            cand_bits = andnot(cand_bits & internal_bits, S);
            int be = -1;
            double bt = 1e300, bpeak = 1e300;
            for (int e : internal) {
                if (!cand_bits.get(e)) continue;
                Bits S2 = S;
                S2.set(e);
                Eval e2 = evaluate(steps, lb, lrows, S2);
                double tt = total_time(e2, s + 1);
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
            S.set(be);
            sliced.push_back(be);
            ev = evaluate(steps, lb, lrows, S);
            if (sliced.size() > 62) { ok = false; last_err = "more than 62 sliced edges"; break; }
        }
        if (!ok) continue;
        double tt = total_time(ev, (int)sliced.size());
        if (!have || tt < best_time) {
            have = true;
            best_time = tt;
            best.order = order;
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
