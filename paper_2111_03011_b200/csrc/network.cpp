// network.cpp -- circuit -> tensor network G, simplification, and the
// sparse-state boundary in row form.
#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <sstream>

#include "tnb.h"

namespace tnb {

namespace {

// PAPER.md Eq. (1), L96-L102.  Index: row = output 2*o_a + o_b, column = input 2*i_a + i_b.
void fsim_matrix(double theta, double phi, cd F[4][4]) {
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) F[r][c] = 0.0;
    const cd mi(0.0, -1.0);
    F[0][0] = 1.0;
    F[1][1] = std::cos(theta);
    F[1][2] = mi * std::sin(theta);
    F[2][1] = mi * std::sin(theta);
    F[2][2] = std::cos(theta);
    F[3][3] = std::exp(cd(0.0, -phi));
}

struct Mat2 {
    cd m[2][2] = {{1.0, 0.0}, {0.0, 1.0}};
};

Mat2 mul(const Mat2& a, const Mat2& b) {  // a * b
    Mat2 r;
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++) r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j];
    return r;
}

// apply a 2x2 matrix to leg position `pos` (0 = MSB) of tensor t: t'[..o..] = sum_i P[o][i] t[..i..]
void apply_on_leg(HTensor& t, int pos, const Mat2& P) {
    const int d = (int)t.legs.size();
    const int64_t N = (int64_t)1 << d;
    const int64_t m = (int64_t)1 << (d - 1 - pos);
    for (int64_t i = 0; i < N; i++) {
        if (i & m) continue;
        cd a0 = t.data[i], a1 = t.data[i | m];
        t.data[i] = P.m[0][0] * a0 + P.m[0][1] * a1;
        t.data[i | m] = P.m[1][0] * a0 + P.m[1][1] * a1;
    }
}

// fix leg position `pos` to value v (drops the leg)
HTensor fix_leg(const HTensor& t, int pos, int v) {
    HTensor r;
    const int d = (int)t.legs.size();
    for (int i = 0; i < d; i++)
        if (i != pos) r.legs.push_back(t.legs[i]);
    const int64_t N = (int64_t)1 << (d - 1);
    r.data.resize(N);
    const int lo = d - 1 - pos;  // bit index of the leg
    for (int64_t o = 0; o < N; o++) {
        int64_t hi = (o >> lo) << (lo + 1), low = o & (((int64_t)1 << lo) - 1);
        r.data[o] = t.data[hi | ((int64_t)v << lo) | low];
    }
    return r;
}

}  // namespace

HTensor contract_host(const HTensor& A, const HTensor& B) {
    std::vector<int> shared, fa, fb;
    for (int e : A.legs)
        if (std::find(B.legs.begin(), B.legs.end(), e) != B.legs.end()) shared.push_back(e);
        else fa.push_back(e);
    for (int e : B.legs)
        if (std::find(shared.begin(), shared.end(), e) == shared.end()) fb.push_back(e);
    HTensor C;
    C.legs = fa;
    C.legs.insert(C.legs.end(), fb.begin(), fb.end());
    const int dA = (int)A.legs.size(), dB = (int)B.legs.size(), dC = (int)C.legs.size();
    const int ns = (int)shared.size();
    auto pos = [](const std::vector<int>& legs, int e) {
        return (int)(std::find(legs.begin(), legs.end(), e) - legs.begin());
    };
    C.data.assign((size_t)1 << dC, cd(0.0));
    for (int64_t c = 0; c < ((int64_t)1 << dC); c++) {
        int64_t ia = 0, ib = 0;
        for (int i = 0; i < dC; i++) {
            int bit = (c >> (dC - 1 - i)) & 1;
            if (!bit) continue;
            int e = C.legs[i];
            if (i < (int)fa.size()) ia |= (int64_t)1 << (dA - 1 - pos(A.legs, e));
            else ib |= (int64_t)1 << (dB - 1 - pos(B.legs, e));
        }
        cd s = 0.0;
        for (int64_t kk = 0; kk < ((int64_t)1 << ns); kk++) {
            int64_t ja = ia, jb = ib;
            for (int i = 0; i < ns; i++)
                if ((kk >> (ns - 1 - i)) & 1) {
                    ja |= (int64_t)1 << (dA - 1 - pos(A.legs, shared[i]));
                    jb |= (int64_t)1 << (dB - 1 - pos(B.legs, shared[i]));
                }
            s += A.data[ja] * B.data[jb];
        }
        C.data[c] = s;
    }
    return C;
}

std::string build_network(const tn_circuit* c, Network& net, const std::vector<int32_t>& holes) {
    const int n = c->n_qubits;
    std::set<int> hole_set;
    for (int32_t h : holes) {
        const int ng = c->n_moments > 0 ? c->moment_offsets[c->n_moments] : 0;
        if (h < 0 || h >= ng) return "hole index out of range";
        if (c->gates[h].kind != 1) return "a hole must be an fSim gate";
        if (!hole_set.insert(h).second) return "hole listed twice";
    }
    if (n < 1 || n > 63) return "n_qubits must be in [1, 63]";
    if (c->n_moments < 0 || (c->n_moments > 0 && (!c->moment_offsets || !c->gates)))
        return "bad moment arrays";
    net = Network();
    net.n = n;
    std::vector<int> cur_t(n, -1), cur_e(n, -1), gcount(n, 0);
    std::vector<Mat2> P(n);
    for (int mo = 0; mo < c->n_moments; mo++) {
        int g0 = c->moment_offsets[mo], g1 = c->moment_offsets[mo + 1];
        if (g0 < 0 || g1 < g0) return "bad moment_offsets";
        std::set<int> used;
        for (int g = g0; g < g1; g++) {
            const tn_gate& G = c->gates[g];
            std::vector<int> qs;
            if (G.kind == 0) qs = {G.q0};
            else if (G.kind == 1) qs = {G.q0, G.q1};
            else return "gate kind must be 0 (single) or 1 (fSim)";
            for (int q : qs) {
                if (q < 0 || q >= n) return "gate qubit out of range";
                if (!used.insert(q).second) {
                    std::ostringstream o;
                    o << "qubit " << q << " appears twice in moment " << mo;
                    return o.str();
                }
            }
            if (G.kind == 1 && c->qubit_rc) {
                int dr = std::abs(c->qubit_rc[2 * G.q0] - c->qubit_rc[2 * G.q1]);
                int dc = std::abs(c->qubit_rc[2 * G.q0 + 1] - c->qubit_rc[2 * G.q1 + 1]);
                if (dr + dc != 1) {
                    std::ostringstream o;
                    o << "fSim targets " << G.q0 << "," << G.q1 << " are not grid neighbours";
                    return o.str();
                }
            }
            if (G.kind == 0) {
                Mat2 U;
                for (int i = 0; i < 4; i++) U.m[i / 2][i % 2] = cd(G.u[2 * i], G.u[2 * i + 1]);
                P[G.q0] = mul(U, P[G.q0]);  // absorbed into the next tensor on the wire
                gcount[G.q0]++;
                continue;
            }
            // fSim tensor T[oa, ob, ia, ib]
            const int a = G.q0, b = G.q1;
            gcount[a]++;
            gcount[b]++;
            if (hole_set.count(g)) {
                // drilled hole (case (i) P:L106-L109): both input edges broken by
                // E = (1,0)x(1,0) right before the gate; fSim|00> = |00>, so the gate drops out exactly and
                // each wire carries |0><0| U (its pending single-qubit gates, then the break)
                for (int q : {a, b}) {
                    Mat2 pin;
                    pin.m[0][0] = 1.0;
                    pin.m[0][1] = 0.0;
                    pin.m[1][0] = 0.0;
                    pin.m[1][1] = 0.0;
                    P[q] = mul(pin, P[q]);
                }
                continue;
            }
            cd F[4][4];
            fsim_matrix(G.theta, G.phi, F);
            HTensor T;
            int ea = (int)net.edges.size();
            net.edges.push_back(Edge{a, gcount[a], -1, -1, false, false});
            int eb = (int)net.edges.size();
            net.edges.push_back(Edge{b, gcount[b], -1, -1, false, false});
            T.legs = {ea, eb, -2, -3};  // placeholders for the inputs
            T.data.resize(16);
            for (int o = 0; o < 4; o++)
                for (int i = 0; i < 4; i++) T.data[4 * o + i] = F[o][i];
            // pending single-qubit gates act before the fSim: T' = F (P_a (x) P_b)
            apply_on_leg(T, 2, Mat2{{{P[a].m[0][0], P[a].m[1][0]}, {P[a].m[0][1], P[a].m[1][1]}}});
            apply_on_leg(T, 3, Mat2{{{P[b].m[0][0], P[b].m[1][0]}, {P[b].m[0][1], P[b].m[1][1]}}});
            const int tid = (int)net.tensors.size();
            // inputs: |0> (no previous tensor on the wire) or the open edge of the previous tensor
            int pos_b = 3;
            if (cur_t[a] < 0) {
                T = fix_leg(T, 2, 0);
                pos_b = 2;
            } else {
                T.legs[2] = cur_e[a];
                net.edges[cur_e[a]].t1 = tid;
            }
            if (cur_t[b] < 0) {
                T = fix_leg(T, pos_b, 0);
            } else {
                T.legs[pos_b] = cur_e[b];
                net.edges[cur_e[b]].t1 = tid;
            }
            net.edges[ea].t0 = tid;
            net.edges[eb].t0 = tid;
            {
                FsimRec R;
                R.q[0] = a;
                R.q[1] = b;
                R.in[0] = cur_t[a] < 0 ? -1 : cur_e[a];
                R.in[1] = cur_t[b] < 0 ? -1 : cur_e[b];
                R.out[0] = ea;
                R.out[1] = eb;
                R.kin[0] = gcount[a] - 1;
                R.kin[1] = gcount[b] - 1;
                for (int r = 0; r < 2; r++)
                    for (int cc = 0; cc < 2; cc++) {
                        R.P[0][r][cc] = P[a].m[r][cc];
                        R.P[1][r][cc] = P[b].m[r][cc];
                    }
                R.theta = G.theta;
                net.fsims.push_back(R);
            }
            net.tensors.push_back(T);
            cur_t[a] = tid;
            cur_e[a] = ea;
            cur_t[b] = tid;
            cur_e[b] = eb;
            P[a] = Mat2();
            P[b] = Mat2();
        }
    }
    // final single-qubit layer absorbed into the previous tensor; output legs
    for (int q = 0; q < n; q++) {
        if (cur_t[q] < 0) {
            // no fSim on this wire: the tensor is P|0> with the output leg only
            int e = (int)net.edges.size();
            int tid = (int)net.tensors.size();
            net.edges.push_back(Edge{q, gcount[q], tid, -1, true, false});
            HTensor T;
            T.legs = {e};
            T.data = {P[q].m[0][0], P[q].m[1][0]};
            net.tensors.push_back(T);
            continue;
        }
        HTensor& T = net.tensors[cur_t[q]];
        int pos = (int)(std::find(T.legs.begin(), T.legs.end(), cur_e[q]) - T.legs.begin());
        apply_on_leg(T, pos, P[q]);
        Edge& E = net.edges[cur_e[q]];
        E.output = true;
        E.k = gcount[q];
    }
    return "";
}

namespace {
int leg_pos(const HTensor& t, int e) { return (int)(std::find(t.legs.begin(), t.legs.end(), e) - t.legs.begin()); }

bool unitary(const cd P[2][2]) {
    double dev = 0;
    for (int r = 0; r < 2; r++)
        for (int cc = 0; cc < 2; cc++) {
            cd x = 0;
            for (int k = 0; k < 2; k++) x += std::conj(P[k][r]) * P[k][cc];
            dev += std::abs(x - (r == cc ? 1.0 : 0.0));
        }
    return dev <= 1e-9;
}
}  // namespace

std::vector<CompanionPair> companion_pairs(const Network& net) {
    std::vector<CompanionPair> out;
    for (int f = 0; f < (int)net.fsims.size(); f++) {
        const FsimRec& R = net.fsims[f];
        for (int side = 0; side < 2; side++) {
            const int w = R.in[1 - side];  // companion: the other qubit's input edge of the same gate
            if (w < 0 || R.out[side] < 0) continue;
            const Edge& E = net.edges[w];
            if (E.output || E.t0 < 0 || E.t1 < 0 || !net.tensors[E.t0].alive || !net.tensors[E.t1].alive) continue;
            if (E.t0 == E.t1) continue;
            if (leg_pos(net.tensors[E.t0], w) >= (int)net.tensors[E.t0].legs.size() ||
                leg_pos(net.tensors[E.t1], w) >= (int)net.tensors[E.t1].legs.size())
                continue;
            // only a unitary P moves across the edge exactly (a drilled hole upstream makes it singular)
            if (!unitary(R.P[1 - side])) continue;
            out.push_back({R.out[side], w, f, 1 - side});
        }
    }
    return out;
}

void add_companions(Network& net, Plan& plan) {
    plan.tied.clear();
    plan.tied_factor.clear();
    plan.tied_wire.clear();
    std::map<int, int> sliced_bit;
    for (int i = 0; i < (int)plan.sliced.size(); i++) sliced_bit[plan.sliced[i]] = i;
    std::set<int> taken(plan.sliced.begin(), plan.sliced.end());
    for (const CompanionPair& cp : companion_pairs(net)) {
        auto it = sliced_bit.find(cp.sliced_edge);
        if (it == sliced_bit.end() || taken.count(cp.companion_edge)) continue;
        const FsimRec& R = net.fsims[cp.fsim];
        const int w = cp.companion_edge, side = cp.side;
        Edge& E = net.edges[w];
        HTensor& up = net.tensors[E.t0];
        HTensor& down = net.tensors[E.t1];
        Mat2 U, Uc;
        for (int r = 0; r < 2; r++)
            for (int cc = 0; cc < 2; cc++) {
                U.m[r][cc] = R.P[side][r][cc];
                Uc.m[r][cc] = std::conj(R.P[side][r][cc]);
            }
        // edge index y := fSim input: up'[y] = sum_i P[y][i] up[i], down'[y] = sum_i conj(P[y][i]) down[i]
        apply_on_leg(up, leg_pos(up, w), U);
        apply_on_leg(down, leg_pos(down, w), Uc);
        taken.insert(w);
        plan.tied.push_back({w, it->second});
        plan.tied_wire.push_back({R.q[side], R.kin[side]});
        const double s2 = std::sin(R.theta) * std::sin(R.theta);
        plan.tied_factor.push_back((1.0 + s2) / 2.0);
    }
}

void simplify(Network& net) {
    // P:L130 "contracting order-one and order-two tensors into their neighbors"
    bool changed = true;
    while (changed) {
        changed = false;
        for (int t = 0; t < (int)net.tensors.size(); t++) {
            HTensor& T = net.tensors[t];
            if (!T.alive || T.legs.size() > 2) continue;
            // neighbour sharing the most internal edges
            std::map<int, int> cnt;
            for (int e : T.legs) {
                const Edge& E = net.edges[e];
                if (E.output) continue;
                int o = (E.t0 == t) ? E.t1 : E.t0;
                if (o >= 0) cnt[o]++;
            }
            if (cnt.empty()) continue;
            int best = -1, bc = -1;
            for (auto& kv : cnt)
                if (kv.second > bc) { best = kv.first; bc = kv.second; }
            HTensor C = contract_host(net.tensors[best], T);
            // edges of T that survive now end at `best`
            for (int e : C.legs) {
                Edge& E = net.edges[e];
                if (E.t0 == t) E.t0 = best;
                if (E.t1 == t) E.t1 = best;
            }
            net.tensors[best].legs = C.legs;
            net.tensors[best].data = std::move(C.data);
            T.alive = false;
            T.legs.clear();
            T.data.clear();
            changed = true;
        }
    }
}

std::vector<uint64_t> rows_of(const Request& req, uint64_t qmask) {
    std::vector<uint64_t> r;
    r.reserve(req.fixed.size());
    for (uint64_t f : req.fixed) r.push_back(f & qmask);
    std::sort(r.begin(), r.end());
    r.erase(std::unique(r.begin(), r.end()), r.end());
    return r;
}

std::vector<Leaf> make_leaves(const Network& net, const Request& req) {
    std::vector<Leaf> out;
    const int n = net.n;
    for (int t = 0; t < (int)net.tensors.size(); t++) {
        const HTensor& T = net.tensors[t];
        if (!T.alive) continue;
        Leaf L;
        L.tensor_id = t;
        std::vector<int> fixed_pos;
        for (int i = 0; i < (int)T.legs.size(); i++) {
            const Edge& E = net.edges[T.legs[i]];
            if (E.output && !E.open) {
                L.qmask |= (uint64_t)1 << (n - 1 - E.q);
                fixed_pos.push_back(i);
            } else {
                L.legs.push_back(T.legs[i]);
            }
        }
        L.rows = rows_of(req, L.qmask);
        const int d = (int)T.legs.size(), dd = (int)L.legs.size();
        L.data.resize(L.rows.size() << dd);
        for (size_t r = 0; r < L.rows.size(); r++) {
            int64_t base = 0;
            for (int p : fixed_pos) {
                int q = net.edges[T.legs[p]].q;
                if ((L.rows[r] >> (n - 1 - q)) & 1) base |= (int64_t)1 << (d - 1 - p);
            }
            for (int64_t i = 0; i < ((int64_t)1 << dd); i++) {
                int64_t full = base;
                int j = 0;
                for (int p = 0; p < d; p++) {
                    if (std::find(fixed_pos.begin(), fixed_pos.end(), p) != fixed_pos.end()) continue;
                    if ((i >> (dd - 1 - j)) & 1) full |= (int64_t)1 << (d - 1 - p);
                    j++;
                }
                L.data[(r << dd) + i] = T.data[full];
            }
        }
        out.push_back(std::move(L));
    }
    return out;
}

}  // namespace tnb
