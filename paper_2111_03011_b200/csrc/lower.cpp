// lower.cpp -- lowers a plan to the per-slice step program executed on the device.
//
// Every tensor of one slice is [rows][2^d] complex64: rows = sparse-state rows (the sorted distinct
// projections of the requested bitstrings onto the tensor's fixed final qubits), d =
// dense legs (internal bonds and open output legs) with sliced legs removed.  A pairwise
// contraction becomes either
//   K_APPLY  : the SIMT sparse-row contraction (gate-application style, any bit positions, row
//              gathers through parent maps) -- SURVEY §8(a) rows a5, a6;
//   K_PREP_A, K_PREP_B, K_GEMM : permute+3xTF32-split pre-passes and the tcgen05 GEMM -- row a4.
// K_INSTANTIATE (row a2) fills the sliced leaves for slice sigma; K_READOUT (rows a6 iii + a7) gathers
// the M amplitudes and accumulates them.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <sstream>
#include <string>

#include "tnb.h"

namespace tnb {

namespace {

struct Alloc {
    std::vector<std::pair<int64_t, int64_t>> fl;  // free blocks (offset, size), sorted by offset
    int64_t top = 0, peak = 0;
    static int64_t rnd(int64_t b) { return (b + 1023) & ~(int64_t)1023; }
    int64_t alloc(int64_t bytes) {
        bytes = rnd(std::max<int64_t>(bytes, 1));
        for (size_t i = 0; i < fl.size(); i++) {
            if (fl[i].second >= bytes) {
                int64_t off = fl[i].first;
                fl[i].first += bytes;
                fl[i].second -= bytes;
                if (fl[i].second == 0) fl.erase(fl.begin() + i);
                return off;
            }
        }
        int64_t off = top;
        top += bytes;
        peak = std::max(peak, top);
        return off;
    }
    void release(int64_t off, int64_t bytes) {
        bytes = rnd(std::max<int64_t>(bytes, 1));
        fl.push_back({off, bytes});
        std::sort(fl.begin(), fl.end());
        std::vector<std::pair<int64_t, int64_t>> m;
        for (auto& b : fl) {
            if (!m.empty() && m.back().first + m.back().second == b.first) m.back().second += b.second;
            else m.push_back(b);
        }
        fl = m;
        if (!fl.empty() && fl.back().first + fl.back().second == top) {
            top = fl.back().first;
            fl.pop_back();
        }
    }
};

struct LT {
    std::vector<int> legs;           // MSB first, sliced legs removed
    uint64_t qmask = 0;
    std::vector<uint64_t> rows;
    BufRef buf;
    int64_t bytes = 0;               // allocation size if in the workspace / persistent region
    bool variant = false;            // depends on a sliced edge (else computed once per tn_contract)
};

inline int bitpos(const std::vector<int>& legs, int e) {
    int i = (int)(std::find(legs.begin(), legs.end(), e) - legs.begin());
    return (int)legs.size() - 1 - i;
}
inline bool has(const std::vector<int>& v, int e) { return std::find(v.begin(), v.end(), e) != v.end(); }

int64_t push_blob(std::vector<uint8_t>& blob, const void* p, size_t bytes) {
    size_t off = (blob.size() + 255) & ~(size_t)255;
    blob.resize(off + bytes);
    if (bytes) std::memcpy(blob.data() + off, p, bytes);
    return (int64_t)off;
}

std::string wire_str(const Network& net, int e) {
    std::ostringstream o;
    o << "[" << net.edges[e].q << "," << net.edges[e].k << "]";
    return o.str();
}

}  // namespace


std::string lower_plan(const Network& net, const std::vector<Leaf>& leaves, const Request& req,
                       const Plan& plan, Program& prog) {
    prog = Program();
    const int s = (int)plan.sliced.size();
    prog.s = s;
    std::map<int, int> slice_index;
    for (int i = 0; i < s; i++) slice_index[plan.sliced[i]] = i;
    for (const auto& t : plan.tied) slice_index[t.first] = t.second;  // companion edges share the bit
    Alloc wa;  // per-slice workspace (reused between steps)
    Alloc pa;  // persistent region for slice-invariant results (read by every slice)
    Alloc la;  // loop program: tensors kept across loop iterations (checkpoint stems, accumulators)
    const bool segmented = !plan.segs.empty();
    const int n_seg = segmented ? (int)plan.segs.size() : 0;
    if (segmented) {
        if (plan.step_seg.size() != plan.order.size()) return "loop program: step_seg length differs from the order";
        if (plan.n_global < 0 || plan.n_global > s) return "loop program: bad n_global";
        prog.segs.resize(n_seg);
        for (int j = 0; j < n_seg; j++) {
            prog.segs[j].D = plan.segs[j].D;
            prog.segs[j].Sum = plan.segs[j].Sum;
            prog.segs[j].E = plan.segs[j].E;
            if (plan.segs[j].E & ~plan.segs[j].D) return "loop program: a segment sums a bit it does not loop over";
        }
        if ((int)plan.is_global.size() != s) return "loop program: is_global length differs from the sliced list";
        uint64_t local = 0;
        int ng = 0;
        prog.bit_global.assign(plan.is_global.begin(), plan.is_global.end());
        for (int i = 0; i < s; i++) {
            if (!plan.is_global[i]) local |= 1ull << (s - 1 - i);
            ng += plan.is_global[i] != 0;
        }
        if (ng != plan.n_global) return "loop program: n_global differs from the global flags";
        if (plan.segs.back().E != 0) return "loop program: the last segment cannot sum local bits";
        if (plan.segs.back().Sum != local) return "loop program: the last segment must follow every local summation";
        for (const Plan::Seg& g : plan.segs)
            if (g.E & ~local) return "loop program: a segment sums a global bit";
        prog.s_global = plan.n_global;
    } else {
        prog.s_global = s;
    }
    // tau-bit mask of every sliced edge (natural dependencies, checked against the segments)
    auto tau_bit = [&](int e) -> uint64_t {
        auto it = slice_index.find(e);
        return it == slice_index.end() ? 0ull : (1ull << (s - 1 - it->second));
    };
    std::vector<uint64_t> nat(leaves.size(), 0);
    std::vector<InstLeafDesc> leaf_desc(leaves.size());
    std::vector<char> leaf_pending(leaves.size(), 0);     // segmented: instantiated when first consumed
    std::vector<std::vector<InstLeafDesc>> seg_inst(n_seg);
    std::vector<int64_t> seg_items(n_seg, 0);
    std::vector<LT> slot(leaves.size());
    std::ostringstream js;
    js.precision(17);
    js << "{\"n\":" << req.n << ",\"s\":" << s << ",\"sliced_wires\":[";
    for (int i = 0; i < s; i++) js << (i ? "," : "") << wire_str(net, plan.sliced[i]);
    js << "],\"leaves\":[";

    auto acc = [](Step& st, const BufRef& b, int64_t bytes, bool write) {
        if (b.region != REG_WORK && b.region != REG_PERS && b.region != REG_LVL) return;
        MemAcc m;
        m.region = b.region;
        m.write = write ? 1 : 0;
        m.offset = b.offset;
        m.bytes = bytes;
        st.mem.push_back(m);
    };

    // ---------------------------------------------------------------- leaves: bank + instantiation
    std::vector<InstLeafDesc> inst;
    int64_t inst_items = 0;
    for (size_t li = 0; li < leaves.size(); li++) {
        const Leaf& L = leaves[li];
        LT& t = slot[li];
        t.qmask = L.qmask;
        t.rows = L.rows;
        int64_t bank_off = (int64_t)prog.bank.size() / 2;  // complex elements
        for (const cd& v : L.data) {
            prog.bank.push_back((float)v.real());
            prog.bank.push_back((float)v.imag());
        }
        std::vector<int> keep, sl;
        for (int e : L.legs) (slice_index.count(e) ? sl : keep).push_back(e);
        t.legs = keep;
        t.variant = !sl.empty();
        if (sl.empty()) {
            t.buf = BufRef{REG_BANK, bank_off * 8};
        } else {
            InstLeafDesc d;
            std::memset(&d, 0, sizeof(d));
            d.bank_off = bank_off;
            d.d_full = (int)L.legs.size();
            d.d_out = (int)keep.size();
            d.n_sl = (int)sl.size();
            d.items = (int64_t)L.rows.size() << d.d_out;
            d.item_begin = inst_items;
            inst_items += d.items;
            for (int b = 0; b < d.d_out; b++) {
                int e = keep[d.d_out - 1 - b];
                d.out_src[b] = (int8_t)bitpos(L.legs, e);
            }
            for (int j = 0; j < d.n_sl; j++) {
                d.sl_pos[j] = (int8_t)bitpos(L.legs, sl[j]);
                d.sl_idx[j] = (int8_t)slice_index[sl[j]];
                nat[li] |= tau_bit(sl[j]);
            }
            t.bytes = d.items * 8;
            if (segmented) {
                inst_items -= d.items;
                leaf_desc[li] = d;
                leaf_pending[li] = 1;
            } else {
                int64_t off = wa.alloc(t.bytes);
                d.out_off = off;
                t.buf = BufRef{REG_WORK, off};
                inst.push_back(d);
            }
        }
        js << (li ? "," : "") << "{\"tensor\":" << L.tensor_id << ",\"qmask\":" << L.qmask << ",\"rows\":" << L.rows.size()
           << ",\"legs\":[";
        for (size_t i = 0; i < L.legs.size(); i++) js << (i ? "," : "") << wire_str(net, L.legs[i]);
        js << "]}";
    }
    js << "],\"steps\":[";
    if (!inst.empty()) {
        Step st;
        st.kind = K_INSTANTIATE;
        st.ip.n_items = inst_items;
        st.ip.n_leaves = (int32_t)inst.size();
        st.ip.table = BufRef{REG_MAPS, push_blob(prog.maps, inst.data(), inst.size() * sizeof(InstLeafDesc))};
        st.bytes = 16.0 * inst_items;
        for (const InstLeafDesc& d : inst) acc(st, BufRef{REG_WORK, d.out_off}, d.items * 8, true);
        prog.steps.push_back(st);
    }

    // ---------------------------------------------------------------- pairwise steps
    int final_slot = plan.order.empty() ? 0 : plan.order.back().first;
    // consumer step of each step's result (segmented: results consumed in another segment persist)
    std::vector<int> consumer(plan.order.size(), -1);
    {
        std::vector<int> last_writer(leaves.size(), -1);
        for (size_t p = 0; p < plan.order.size(); p++) {
            const int i = plan.order[p].first, j = plan.order[p].second;
            if (last_writer[i] >= 0) consumer[last_writer[i]] = (int)p;
            if (last_writer[j] >= 0) consumer[last_writer[j]] = (int)p;
            last_writer[i] = (int)p;
        }
    }
    // segmented: the segment that first consumes each sliced leaf instantiates it (in every run)
    std::vector<int> leaf_seg(leaves.size(), -1);
    if (segmented)
        for (size_t p = 0; p < plan.order.size(); p++)
            for (int li : {plan.order[p].first, plan.order[p].second})
                if (leaf_pending[li] && leaf_seg[li] < 0) leaf_seg[li] = plan.step_seg[p];
    for (size_t p = 0; p < plan.order.size(); p++) {
        int i = plan.order[p].first, j = plan.order[p].second;
        const int sg = segmented ? plan.step_seg[p] : -1;
        if (segmented && (p == 0 || plan.step_seg[p - 1] != sg)) {
            // K_INSTANTIATE runs first in the segment: all of its leaves get their buffers now, before any
            // step of the segment allocates a temporary (no overlap with the segment's other tensors)
            for (size_t li = 0; li < leaves.size(); li++) {
                if (!leaf_pending[li] || leaf_seg[li] != sg) continue;
                InstLeafDesc d = leaf_desc[li];
                d.item_begin = seg_items[sg];
                seg_items[sg] += d.items;
                d.out_off = wa.alloc(slot[li].bytes);
                slot[li].buf = BufRef{REG_WORK, d.out_off};
                seg_inst[sg].push_back(d);
                leaf_pending[li] = 0;
            }
        }
        LT X = slot[i], Y = slot[j];
        const uint64_t natC = nat[i] | nat[j];
        if (segmented && (natC & ~plan.segs[sg].D))
            return "loop program: step " + std::to_string(p) + " depends on a sliced bit its segment does not loop over";
        std::vector<int> K;
        for (int e : X.legs)
            if (has(Y.legs, e)) K.push_back(e);
        const uint64_t qC = X.qmask | Y.qmask;
        std::vector<uint64_t> rowsC = rows_of(req, qC);
        const int64_t RC = (int64_t)rowsC.size();
        const bool rx = X.qmask != 0, ry = Y.qmask != 0;
        auto per_row = [](const LT& t) { return (int64_t)1 << t.legs.size(); };

        // roles
        bool use_gemm = false;
        LT *A = &X, *B = &Y;
        bool grouped = false;
        if (rx && ry) {
            // gather-contract: the operand with FEWER rows is reused by many output rows -> M side
            if (Y.rows.size() < X.rows.size() || (Y.rows.size() == X.rows.size() && per_row(Y) > per_row(X)))
                std::swap(A, B);
            // gather-contract on the tensor cores when the per-row GEMMs are big enough and many output
            // rows share an A parent (grouped GEMM, see GemmParams::grouped)
            const int64_t fa = (int64_t)A->legs.size() - (int64_t)K.size();
            const int64_t fb = (int64_t)B->legs.size() - (int64_t)K.size();
            const double cm = (double)RC * std::ldexp(1.0, (int)(fa + fb + K.size()));
            const int64_t RA = (int64_t)A->rows.size();
            // (short k, <= 32, goes to the gate kernel's modes 1 / 2 below, which read A once without a pre-pass)
            // (either operand may be the gate kernel's stem: the one with the longer rows, whose free legs must
            // fill whole tiles)
            const int64_t fbig = per_row(*A) >= per_row(*B) ? fa : fb;
            grouped = K.size() >= 4 && fa >= 5 && cm >= 16.0 * 1024 * 1024 &&
                      (RC >= 16 * RA || (fa >= 7 && RC >= 2 * RA)) && !(K.size() <= 5 && fbig >= 7);
            if (!grouped && per_row(*B) > per_row(*A)) std::swap(A, B);  // SIMT: stream the larger rows
            use_gemm = grouped;
        } else {
            if (ry || (!rx && per_row(Y) > per_row(X))) std::swap(A, B);
            int64_t fa = (int64_t)A->legs.size() - (int64_t)K.size();
            int64_t fb = (int64_t)B->legs.size() - (int64_t)K.size();
            int64_t m = RC << fa, n = (int64_t)1 << fb, k = (int64_t)1 << K.size();
            use_gemm = (m >= 128 && n >= 64 && k >= 16) || (m >= 64 && n >= 128 && k >= 16) ||
                       (m >= 128 && n >= 16 && k >= 64);  // tall-skinny, long K: N tile 32 / 64
            if (!use_gemm && per_row(*B) > per_row(*A)) std::swap(A, B);
        }
        // parent maps
        std::vector<int32_t> ma(RC), mb(RC);
        bool ma_id = (int64_t)A->rows.size() == RC;
        for (int64_t r = 0; r < RC; r++) {
            ma[r] = (int32_t)(std::lower_bound(A->rows.begin(), A->rows.end(), rowsC[r] & A->qmask) - A->rows.begin());
            mb[r] = (int32_t)(std::lower_bound(B->rows.begin(), B->rows.end(), rowsC[r] & B->qmask) - B->rows.begin());
            if (ma[r] != r) ma_id = false;
        }
        BufRef maRef, mbRef;
        if (!ma_id) maRef = BufRef{REG_MAPS, push_blob(prog.maps, ma.data(), ma.size() * 4)};
        if (B->qmask != 0) mbRef = BufRef{REG_MAPS, push_blob(prog.maps, mb.data(), mb.size() * 4)};
        std::vector<int> fb;
        for (int e : B->legs)
            if (!has(K, e)) fb.push_back(e);
        std::vector<int> fa;
        for (int e : A->legs)
            if (!has(K, e)) fa.push_back(e);
        // slice-invariant steps (no sliced edge below them) run once per tn_contract, before the slices
        // (the sliced-network analogue of the paper's head-result reuse)
        const bool var = X.variant || Y.variant;
        std::string apply_json, gemm_json;
        // segmented: a variant result consumed by another segment is kept across loop iterations
        // (REG_LVL), unless the segment ends with a summation (then the accumulator is the kept copy)
        const bool seg_last = segmented && (p + 1 == plan.order.size() || plan.step_seg[p + 1] != sg);
        const bool accum = segmented && var && seg_last && plan.segs[sg].E != 0;
        const bool keep = segmented && var && !accum && consumer[p] >= 0 && plan.step_seg[consumer[p]] != sg;
        Alloc& al0 = var ? wa : pa;
        const int32_t reg0 = var ? REG_WORK : REG_PERS;
        std::vector<Step>& out = var ? (segmented ? prog.segs[sg].steps : prog.steps) : prog.pre_steps;
        // the result's allocator; operands' temporaries (prep buffers) always come from al0
        Alloc& alC = keep ? la : al0;
        const int32_t regC = keep ? REG_LVL : reg0;
        Alloc& al = al0;
        const int32_t reg = reg0;
        LT Cn;
        Cn.qmask = qC;
        Cn.rows = rowsC;
        Cn.variant = var;
        const double cmac = (double)RC * std::ldexp(1.0, (int)(fa.size() + fb.size() + K.size()));
        const int64_t sizeA = (int64_t)A->rows.size() << A->legs.size();
        const int64_t sizeB = (int64_t)B->rows.size() << B->legs.size();

        if (!use_gemm) {
            // C legs.  Default: A's free legs keep their relative order in the low bits and the B-free legs go on
            // top, so that consecutive orbits (A's low free bits) are consecutive in C (coalesced stores) and the
            // new legs, usually contracted soon after, are high bits of the next step's A (coalesced gathers).
            // TNB_C_LAYOUT=inplace: A's layout with the K legs replaced by the B-free legs (extra ones on top).
            static const bool inplace = getenv("TNB_C_LAYOUT") && std::string(getenv("TNB_C_LAYOUT")) == "inplace";
            if (inplace) {
                size_t nfb = fb.size(), used = 0;
                size_t extra = nfb > K.size() ? nfb - K.size() : 0;
                for (size_t t = 0; t < extra; t++) Cn.legs.push_back(fb[used++]);
                for (int e : A->legs) {
                    if (has(K, e)) {
                        if (used < nfb) Cn.legs.push_back(fb[used++]);
                    } else {
                        Cn.legs.push_back(e);
                    }
                }
            } else {
                for (int e : fb) Cn.legs.push_back(e);
                for (int e : A->legs)
                    if (!has(K, e)) Cn.legs.push_back(e);
            }
            Step st;
            st.kind = K_APPLY;
            st.pair = (int)p;
            ApplyParams& ap = st.ap;
            ap.A = A->buf;
            ap.B = B->buf;
            ap.ma = maRef;
            ap.mb = mbRef;
            ap.R = RC;
            // several output rows read the same big A row: process them consecutively so that the re-reads hit
            // L2 (gather-contract steps whose output rows are sorted by key, not by A parent)
            if (maRef.region && ((int64_t)1 << A->legs.size()) >= 4096 && RC > (int64_t)A->rows.size()) {
                bool mono = true;
                for (int64_t r = 1; r < RC && mono; r++) mono = ma[r] >= ma[r - 1];
                if (!mono) {
                    std::vector<int32_t> perm(RC);
                    for (int64_t r = 0; r < RC; r++) perm[r] = (int32_t)r;
                    std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return ma[x] < ma[y]; });
                    ap.rperm = BufRef{REG_MAPS, push_blob(prog.maps, perm.data(), perm.size() * 4)};
                }
            }
            ap.dA = (int)A->legs.size();
            ap.dB = (int)B->legs.size();
            ap.dC = (int)Cn.legs.size();
            ap.a_row = (int64_t)1 << ap.dA;
            ap.b_row = (int64_t)1 << ap.dB;
            ap.c_row = (int64_t)1 << ap.dC;
            ap.cA.n = 0;
            for (int e : fa) {
                ap.cA.dst[ap.cA.n] = (int8_t)bitpos(Cn.legs, e);
                ap.cA.src[ap.cA.n] = (int8_t)bitpos(A->legs, e);
                ap.cA.n++;
            }
            ap.cB.n = 0;
            for (int e : fb) {
                ap.cB.dst[ap.cB.n] = (int8_t)bitpos(Cn.legs, e);
                ap.cB.src[ap.cB.n] = (int8_t)bitpos(B->legs, e);
                ap.cB.n++;
            }
            ap.nk = (int)K.size();
            for (int t = 0; t < ap.nk; t++) {
                ap.kA[t] = (int8_t)bitpos(A->legs, K[t]);
                ap.kB[t] = (int8_t)bitpos(B->legs, K[t]);
            }
            // inner (per-thread) C bits: up to 4 B-free legs with the lowest C bit positions
            std::vector<int> fbpos;
            for (int e : fb) fbpos.push_back(bitpos(Cn.legs, e));
            std::sort(fbpos.begin(), fbpos.end());
            ap.n_inner = (int)std::min<size_t>(4, fbpos.size());
            for (int t = 0; t < ap.n_inner; t++) ap.inner_c[t] = (int8_t)fbpos[t];
            Cn.bytes = RC * ap.c_row * 8;
            int64_t off = alC.alloc(Cn.bytes);
            Cn.buf = BufRef{regC, off};
            ap.C = Cn.buf;
            ap.a_elems = sizeA;
            ap.b_elems = sizeB;
            acc(st, A->buf, sizeA * 8, false);
            acc(st, B->buf, sizeB * 8, false);
            acc(st, Cn.buf, Cn.bytes, true);
            st.cmac = cmac;
            st.bytes = 8.0 * (double)(sizeA + sizeB + RC * ap.c_row) + (maRef.region ? 4.0 * RC : 0) + (mbRef.region ? 4.0 * RC : 0);
            // big stem x small rowless tensor: the fused tensor-core gate kernel (gate_tc.cuh) reads the stem once
            // and writes the result once; SIMT would be FMA-bound (4 * 2^nk FFMA per element)
            {
                const int nk = ap.nk, nb = ap.cB.n;
                // measured on config 4: 16x16 gates 3.5 ms (TC) vs 5.8 ms (SIMT) on a 2^30 stem; 8x8 gates are
                // faster on SIMT (4.7 vs 5.6 ms), so small k needs a wide output to go to the tensor cores
                // TNB_GATE_ANY=1 (test hook): every structurally eligible step goes to the gate kernel, whatever its
                // size, so that small networks exercise all three modes against the oracle
                const char* gany_env = getenv("TNB_GATE_ANY");
                const bool gany = gany_env && atoi(gany_env) != 0;
                const bool fits = nk >= 3 && nk <= 5 && nb >= 1 && nb <= 7 && ap.cA.n <= 32 &&
                                  (gany || nk >= 4 || nb >= 4);
                const bool big = gany ||
                                 ((double)RC * std::ldexp(1.0, ap.cA.n) >= 1048576.0 && cmac >= 4.0 * 1048576.0 * 16);
                static const bool gate_off = getenv("TNB_NO_GATE_TC") != nullptr;
                if (!gate_off && fits && big && B->qmask == 0 && !mbRef.region) st.kind = K_GATE;
                // gather-contract (both operands carry rows) on the gate kernel: A's orbits fill whole tiles
                // (>= 128 per row).  Mode 2 when several output rows share an A row (A read once, the gate's
                // columns are the group's B rows); mode 1 when few B rows serve many output rows (rows processed
                // grouped by B parent, the resident gate reloaded at group boundaries)
                const int64_t RA = (int64_t)A->rows.size(), RB = (int64_t)B->rows.size();
                const bool gfit = nk >= 3 && nk <= 5 && ap.cA.n >= 7 && ap.cA.n <= 32 && B->qmask != 0 && mbRef.region;
                if (!gate_off && gfit && big) {
                    std::vector<int32_t> cnt(RA, 0);
                    for (int64_t r = 0; r < RC; r++) cnt[ma[r]]++;
                    const int gmax = *std::max_element(cnt.begin(), cnt.end());
                    int gm = 1;
                    while (gm < gmax) gm *= 2;
                    const int ncols2 = gm << nb;  // complex gate columns in mode 2
                    const int cap2 = nk <= 4 ? 128 : 64;
                    // mode 2 also when fewer output rows share an A row (RC >= 1.25 RA) if an A row spans >= 16
                    // tiles: mode 1 would read A once per output row (config 4 step 198: 16.8 GB of DRAM traffic
                    // for 10.8 GB of algorithmic bytes), mode 2 pays a gate reload per A row instead
                    const bool share = RC >= 2 * RA || (4 * RC >= 5 * RA && ap.cA.n >= 11);
                    if (share && gm <= 16 && ncols2 <= cap2 && (gany || nk >= 4 || ncols2 >= 16 || RC >= 3 * RA)) {
                        std::vector<int32_t> perm(RC), gs(RA, 0);
                        for (int64_t r = 0; r < RC; r++) perm[r] = (int32_t)r;
                        std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return ma[x] < ma[y]; });
                        for (int64_t a = 1; a < RA; a++) gs[a] = gs[a - 1] + cnt[a - 1];
                        st.kind = K_GATE;
                        st.ap.gate_mode = 2;
                        st.ap.gm = gm;
                        st.ap.a_rows = RA;
                        st.ap.gperm = BufRef{REG_MAPS, push_blob(prog.maps, perm.data(), perm.size() * 4)};
                        st.ap.gstart = BufRef{REG_MAPS, push_blob(prog.maps, gs.data(), gs.size() * 4)};
                        st.ap.gcnt = BufRef{REG_MAPS, push_blob(prog.maps, cnt.data(), cnt.size() * 4)};
                    } else if (nb <= 7 && (gany || (RB * 8 <= RC && (nk >= 4 || nb >= 4)))) {
                        std::vector<int32_t> perm(RC);
                        for (int64_t r = 0; r < RC; r++) perm[r] = (int32_t)r;
                        std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return mb[x] < mb[y]; });
                        st.kind = K_GATE;
                        st.ap.gate_mode = 1;
                        st.ap.a_rows = RA;
                        st.ap.gperm = BufRef{REG_MAPS, push_blob(prog.maps, perm.data(), perm.size() * 4)};
                    }
                }
            }
            {
                std::ostringstream o;
                o << ",\"apply\":{\"dA\":" << ap.dA << ",\"dB\":" << ap.dB << ",\"dC\":" << ap.dC << ",\"kA\":[";
                for (int t = 0; t < ap.nk; t++) o << (t ? "," : "") << (int)ap.kA[t];
                o << "],\"kB\":[";
                for (int t = 0; t < ap.nk; t++) o << (t ? "," : "") << (int)ap.kB[t];
                o << "],\"cA\":[";
                for (int t = 0; t < ap.cA.n; t++) o << (t ? "," : "") << "[" << (int)ap.cA.dst[t] << "," << (int)ap.cA.src[t] << "]";
                o << "],\"cB\":[";
                for (int t = 0; t < ap.cB.n; t++) o << (t ? "," : "") << "[" << (int)ap.cB.dst[t] << "," << (int)ap.cB.src[t] << "]";
                o << "],\"inner\":[";
                for (int t = 0; t < ap.n_inner; t++) o << (t ? "," : "") << (int)ap.inner_c[t];
                o << "],\"ma\":" << (maRef.region ? 1 : 0) << ",\"mb\":" << (mbRef.region ? 1 : 0) << "}";
                apply_json = o.str();
            }
            if (st.kind == K_GATE) apply_json += ",\"gate_tc\":" + std::to_string(st.ap.gate_mode);
            out.push_back(st);
        } else {
            Cn.legs = fa;
            Cn.legs.insert(Cn.legs.end(), fb.begin(), fb.end());
            const int64_t m = (int64_t)1 << fa.size(), n = (int64_t)1 << fb.size(), k = (int64_t)1 << K.size();
            const int64_t RA = (int64_t)A->rows.size();
            const int64_t Mp = grouped ? RA * m : RC * m;  // rows of the prepped A
            GemmParams gp;
            gp.A = A->buf;
            gp.B = B->buf;
            gp.ma = grouped ? BufRef() : maRef;
            gp.R = grouped ? RA : RC;
            gp.m = m;
            gp.n = n;
            gp.k = k;
            gp.dA = (int)A->legs.size();
            gp.dB = (int)B->legs.size();
            gp.a_row = (int64_t)1 << gp.dA;
            gp.aM.n = (int)fa.size();
            for (int t = 0; t < gp.aM.n; t++) {
                gp.aM.dst[t] = (int8_t)(gp.aM.n - 1 - t);             // m-index bit
                gp.aM.src[t] = (int8_t)bitpos(A->legs, fa[t]);        // A bit
            }
            // can an operand be TMA-loaded raw (split to hi/lo inside the GEMM)?  Its contracted legs must
            // be its lowest bits and its rows contiguous (no row map).
            auto low_is_K = [&](const LT* T) {
                for (int e : K)
                    if (bitpos(T->legs, e) >= (int)K.size()) return false;
                return true;
            };
            const bool a_low = low_is_K(A) && (grouped || !maRef.region);
            const bool b_low = low_is_K(B);
            gemm_json = std::string(",\"a_lowK\":") + (a_low ? "1" : "0") + ",\"b_lowK\":" + (b_low ? "1" : "0");
            {
                auto ids = [](const std::vector<int>& v) {
                    std::string o = "[";
                    for (size_t t = 0; t < v.size(); t++) o += (t ? "," : "") + std::to_string(v[t]);
                    return o + "]";
                };
                // leg ids (MSB first) of both operands, the contracted legs and the free legs, in GEMM order
                gemm_json += ",\"legs_a\":" + ids(A->legs) + ",\"legs_b\":" + ids(B->legs) + ",\"legs_k\":" +
                             ids(K) + ",\"legs_fa\":" + ids(fa) + ",\"legs_fb\":" + ids(fb);
            }
            gp.aK.n = (int)K.size();
            gp.bK.n = (int)K.size();
            for (int t = 0; t < gp.aK.n; t++) {
                gp.aK.dst[t] = (int8_t)(gp.aK.n - 1 - t);
                gp.aK.src[t] = (int8_t)bitpos(A->legs, K[t]);
                gp.bK.dst[t] = (int8_t)(gp.bK.n - 1 - t);
                gp.bK.src[t] = (int8_t)bitpos(B->legs, K[t]);
            }
            gp.bN.n = (int)fb.size();
            for (int t = 0; t < gp.bN.n; t++) {
                gp.bN.dst[t] = (int8_t)(gp.bN.n - 1 - t);
                gp.bN.src[t] = (int8_t)bitpos(B->legs, fb[t]);
            }
            int64_t NBcols = n;  // complex columns of the prepped B
            if (grouped) {
                gp.grouped = 1;
                gp.RC = RC;
                gp.NB = RC;
                gp.b_row = (int64_t)1 << B->legs.size();
                NBcols = RC * n;
                // group output rows by their A parent (stable), gathered B blocks in that order
                std::vector<int32_t> perm(RC), rowsel(RC);
                for (int64_t r = 0; r < RC; r++) perm[r] = (int32_t)r;
                std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return ma[x] < ma[y]; });
                for (int64_t q = 0; q < RC; q++) rowsel[q] = mb[perm[q]];
                gp.perm = BufRef{REG_MAPS, push_blob(prog.maps, perm.data(), perm.size() * 4)};
                gp.rowsel = BufRef{REG_MAPS, push_blob(prog.maps, rowsel.data(), rowsel.size() * 4)};
                gp.embed_a = (RA * m < RC * n) ? 1 : 0;
                const int xs = gp.embed_a ? 2 : 1, ys = gp.embed_a ? 1 : 2;
                // tiles never straddle two groups (a tile's A rows are one group's); one table per tile
                // size: 128 x 128 for single-CTA tiles, 256 x 256 for CTA pairs
                auto group_tiles = [&](int64_t TX, int64_t TY) {
                    std::vector<GemmTile> tiles;
                    int64_t q = 0;
                    while (q < RC) {
                        const int32_t a = ma[perm[q]];
                        int64_t e = q;
                        while (e < RC && ma[perm[e]] == a) e++;
                        const int64_t xb = (int64_t)a * m * xs, xr = m * xs;
                        const int64_t yb = q * n * ys, yr = (e - q) * n * ys;
                        for (int64_t x0 = xb; x0 < xb + xr; x0 += TX)
                            for (int64_t y0 = yb; y0 < yb + yr; y0 += TY) {
                                GemmTile t;
                                t.x0 = (int32_t)x0;
                                t.xvalid = (int32_t)std::min<int64_t>(TX, xb + xr - x0);
                                t.xbase = (int32_t)xb;
                                t.y0 = (int32_t)y0;
                                t.yvalid = (int32_t)std::min<int64_t>(TY, yb + yr - y0);
                                t.ybase = (int32_t)yb;
                                t.off = (int32_t)q;
                                t.pad = 0;
                                tiles.push_back(t);
                            }
                        q = e;
                    }
                    return tiles;
                };
                const std::vector<GemmTile> t1 = group_tiles(128, 128), t2 = group_tiles(256, 256);
                gp.n_tiles = (int64_t)t1.size();
                gp.tiles = BufRef{REG_MAPS, push_blob(prog.maps, t1.data(), t1.size() * sizeof(GemmTile))};
                gp.n_tiles2 = (int64_t)t2.size();
                gp.tiles2 = BufRef{REG_MAPS, push_blob(prog.maps, t2.data(), t2.size() * sizeof(GemmTile))};
            } else {
                // embed the smaller operand in the complex-as-real GEMM (its rows double); EA needs n >= 32
                gp.embed_a = ((Mp < n && n >= 128) || Mp < 128) && n >= 32 ? 1 : 0;
                // plain GEMM, opt-in TNB_GEMM_CMAJ=1: store C column-major within each row (B-free legs on top,
                // A-free legs low), so that the epilogue's lanes (consecutive m) write consecutive addresses.
                // Measured (same box): config-4 k=64 n=256 GEMM 4.06 -> 3.50 ms but the step total unchanged,
                // config 3 -3 % (its consumers prefer the row-major result), so the default stays row-major
                static const bool cmaj_on = getenv("TNB_GEMM_CMAJ") && atoi(getenv("TNB_GEMM_CMAJ")) != 0;
                if (!gp.embed_a && cmaj_on && m >= 32) {
                    gp.c_colmajor = 1;
                    Cn.legs = fb;
                    Cn.legs.insert(Cn.legs.end(), fa.begin(), fa.end());
                }
            }
            const int64_t abytes = (gp.embed_a ? 2 : 1) * Mp * 2 * k * 4,
                          bbytes = (gp.embed_a ? 1 : 2) * NBcols * 2 * k * 4;
            // fused A pre-pass (plain GEMMs with A on the plain side): the GEMM gathers and splits A itself.
            // Opt-in (TNB_GATHER_A=1): measured on config 4 it is neutral to +1 % (the pair GEMMs then wait on the
            // gather producers), and one config-3 run with 16 concurrent pipelines did not finish (not reproduced
            // with either fused kernel alone; under investigation), so the default keeps the pre-pass
            static const bool ga_on = getenv("TNB_GATHER_A") != nullptr && atoi(getenv("TNB_GATHER_A")) != 0;
            gp.gather_a = (ga_on && !grouped && !gp.embed_a && k <= 1024 && fa.size() <= 32) ? 1 : 0;
            if (!gp.gather_a) {
                gp.Ahi = BufRef{reg, al.alloc(abytes)};
                gp.Alo = BufRef{reg, al.alloc(abytes)};
            }
            gp.Bhi = BufRef{reg, al.alloc(bbytes)};
            gp.Blo = BufRef{reg, al.alloc(bbytes)};
            Cn.bytes = RC * m * n * 8;
            Cn.buf = BufRef{regC, alC.alloc(Cn.bytes)};
            gp.C = Cn.buf;
            Step sa;
            sa.kind = K_PREP_A;
            sa.pair = (int)p;
            sa.gp = gp;
            sa.bytes = 8.0 * Mp * k + 2.0 * abytes;  // read A once, write hi + lo
            Step sb;
            sb.kind = K_PREP_B;
            sb.pair = (int)p;
            sb.gp = gp;
            sb.bytes = 8.0 * NBcols * k + 2.0 * bbytes;
            Step sg;
            sg.kind = K_GEMM;
            sg.pair = (int)p;
            sg.gp = gp;
            sg.cmac = cmac;
            sg.bytes = 2.0 * abytes + 2.0 * bbytes + 8.0 * RC * m * n;
            acc(sb, B->buf, sizeB * 8, false);
            acc(sb, gp.Bhi, bbytes, true);
            acc(sb, gp.Blo, bbytes, true);
            acc(sg, gp.Bhi, bbytes, false);
            acc(sg, gp.Blo, bbytes, false);
            acc(sg, Cn.buf, Cn.bytes, true);
            if (gp.gather_a) {
                sg.gp = gp;
                sg.bytes = 8.0 * Mp * k + 2.0 * bbytes + 8.0 * RC * m * n;
                acc(sg, A->buf, sizeA * 8, false);
            } else {
                acc(sa, A->buf, sizeA * 8, false);
                acc(sa, gp.Ahi, abytes, true);
                acc(sa, gp.Alo, abytes, true);
                acc(sg, gp.Ahi, abytes, false);
                acc(sg, gp.Alo, abytes, false);
                out.push_back(sa);
            }
            out.push_back(sb);
            out.push_back(sg);
            if (!gp.gather_a) {
                al.release(gp.Ahi.offset, abytes);
                al.release(gp.Alo.offset, abytes);
            }
            al.release(gp.Bhi.offset, bbytes);
            al.release(gp.Blo.offset, bbytes);
            if (var) prog.gemm_cmac += cmac;
        }
        if (var) prog.cmac += cmac;
        else prog.pre_cmac += cmac;
        if (segmented && var) prog.total_cmac += cmac * std::ldexp(1.0, __builtin_popcountll(plan.segs[sg].D));
        nat[i] = natC;
        if (accum) {
            // local-slice summation: acc = (first value of the E bits ? 0 : acc) + C, kept across iterations
            if ((natC & plan.segs[sg].E) != plan.segs[sg].E)
                return "loop program: segment " + std::to_string(sg) + " sums bits its last step does not depend on";
            const int64_t n_el = RC << Cn.legs.size();
            Step sa;
            sa.kind = K_ACCUM;
            sa.pair = (int)p;
            sa.cp.src = Cn.buf;
            sa.cp.n = n_el;
            sa.cp.E = plan.segs[sg].E;
            const BufRef accb{REG_LVL, la.alloc(n_el * 8)};
            sa.cp.dst = accb;
            sa.bytes = 24.0 * n_el;
            acc(sa, Cn.buf, n_el * 8, false);
            prog.segs[sg].steps.push_back(sa);
            prog.total_cmac += 0.0;
            wa.release(Cn.buf.offset, Cn.bytes);
            Cn.buf = accb;
            nat[i] = natC & ~plan.segs[sg].E;
        } else if (segmented && var && keep && consumer[p] >= 0) {
            // only the stem may carry the summed bits out of a segment
            (void)0;
        }
        prog.peak_elems = std::max<int64_t>(prog.peak_elems, RC << Cn.legs.size());
        // release operands held in the workspace (REG_LVL tensors stay for the whole loop program)
        if (X.buf.region == REG_WORK) wa.release(X.buf.offset, X.bytes);
        if (Y.buf.region == REG_WORK) wa.release(Y.buf.offset, Y.bytes);
        // persistent results consumed by another invariant step can be recycled inside the prologue;
        // those consumed by a per-slice step must stay valid for every slice
        if (!var && X.buf.region == REG_PERS) pa.release(X.buf.offset, X.bytes);
        if (!var && Y.buf.region == REG_PERS) pa.release(Y.buf.offset, Y.bytes);
        js << (p ? "," : "") << "{\"pair\":[" << i << "," << j << "],\"gemm\":" << (use_gemm ? 1 : 0)
           << ",\"invariant\":" << (var ? 0 : 1) << ",\"grouped\":" << (grouped ? 1 : 0) << ",\"qmask\":" << qC << ",\"rows\":" << RC << ",\"m_rows\":" << A->rows.size() << ",\"n_rows\":" << B->rows.size()
           << ",\"fa\":" << fa.size() << ",\"fb\":" << fb.size() << ",\"k\":" << K.size() << ",\"cmac\":" << cmac
           << apply_json << gemm_json;
        if (RC <= 4096 && qC != 0) {
            js << ",\"row_keys\":[";
            for (int64_t r = 0; r < RC; r++) js << (r ? "," : "") << rowsC[r];
            js << "],\"qmask_a\":" << A->qmask << ",\"qmask_b\":" << B->qmask << ",\"map_a\":[";
            for (int64_t r = 0; r < RC; r++) js << (r ? "," : "") << ma[r];
            js << "],\"map_b\":[";
            for (int64_t r = 0; r < RC; r++) js << (r ? "," : "") << mb[r];
            js << "]";
        }
        js << "}";
        slot[i] = Cn;
        slot[j] = LT();
    }

    // ---------------------------------------------------------------- readout + accumulate
    const LT& F = slot[final_slot];
    for (int e : F.legs)
        if (!(net.edges[e].output && net.edges[e].open)) return "internal error: final tensor has a non-open leg";
    std::vector<int64_t> idx(req.M);
    const int dF = (int)F.legs.size();
    for (int64_t jj = 0; jj < req.M; jj++) {
        uint64_t x = req.bits[jj];
        int64_t r = std::lower_bound(F.rows.begin(), F.rows.end(), x & F.qmask) - F.rows.begin();
        if (r >= (int64_t)F.rows.size() || F.rows[r] != (x & F.qmask)) return "internal error: readout row missing";
        int64_t off = 0;
        for (int t = 0; t < dF; t++) {
            int q = net.edges[F.legs[t]].q;
            if ((x >> (req.n - 1 - q)) & 1) off |= (int64_t)1 << (dF - 1 - t);
        }
        idx[jj] = (r << dF) + off;
    }
    Step st;
    st.kind = K_READOUT;
    st.rp.F = F.buf;
    st.rp.M = req.M;
    st.rp.idx = BufRef{REG_MAPS, push_blob(prog.maps, idx.data(), idx.size() * 8)};
    st.bytes = (8.0 + 8.0 + 32.0) * (double)req.M;
    acc(st, F.buf, ((int64_t)F.rows.size() << dF) * 8, false);
    if (segmented) {
        uint64_t glob = 0;
        for (int i = 0; i < s; i++)
            if (plan.is_global[i]) glob |= 1ull << (s - 1 - i);
        if (nat[final_slot] & ~glob) return "loop program: the final tensor still depends on a local bit";
        prog.segs.back().steps.push_back(st);
        // K_INSTANTIATE first in every segment that instantiates sliced leaves
        for (int j = 0; j < n_seg; j++) {
            if (seg_inst[j].empty()) continue;
            Step si;
            si.kind = K_INSTANTIATE;
            si.ip.n_items = seg_items[j];
            si.ip.n_leaves = (int32_t)seg_inst[j].size();
            si.ip.table = BufRef{REG_MAPS, push_blob(prog.maps, seg_inst[j].data(), seg_inst[j].size() * sizeof(InstLeafDesc))};
            si.bytes = 16.0 * seg_items[j];
            for (const InstLeafDesc& d : seg_inst[j]) acc(si, BufRef{REG_WORK, d.out_off}, d.items * 8, true);
            prog.segs[j].steps.insert(prog.segs[j].steps.begin(), si);
        }
        prog.lvl_bytes = la.peak;
    } else {
        prog.steps.push_back(st);
        prog.lvl_bytes = 0;
    }

    js << "],\"final\":{\"qmask\":" << F.qmask << ",\"rows\":" << F.rows.size() << ",\"legs\":[";
    for (int t = 0; t < dF; t++) js << (t ? "," : "") << wire_str(net, F.legs[t]);
    js << "]";
    if (F.rows.size() <= 65536) {
        js << ",\"row_keys\":[";
        for (size_t r = 0; r < F.rows.size(); r++) js << (r ? "," : "") << F.rows[r];
        js << "]";
    }
    js << "}}";
    prog.dump_json = js.str();
    prog.n_pairs = (int64_t)plan.order.size();
    prog.work_bytes = std::max<int64_t>(wa.peak, 1024);
    prog.pers_bytes = std::max<int64_t>(pa.peak, 1024);
    for (const Step& x : prog.steps) prog.bytes += x.bytes;
    for (const auto& sg : prog.segs)
        for (const Step& x : sg.steps) prog.bytes += x.bytes;
    if (!segmented) prog.total_cmac = std::ldexp(prog.cmac, s) + prog.pre_cmac;
    else prog.total_cmac += prog.pre_cmac;
    // largest leaf counts toward the peak as well
    for (const LT& t : slot) (void)t;
    return "";
}

}  // namespace tnb
