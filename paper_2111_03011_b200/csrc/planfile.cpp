// planfile.cpp -- replayable plan files ("plan file is an explicit, replayable artifact",
// S:L324 JSON).  A plan is setup data: the contraction order, the sliced wires and the loop program; saving
// it lets another process (a rank of a multi-GPU run, a later benchmark) reuse a plan found by a long
// search, and lets a plan produced by any other tool be imported.
//
// Format (one JSON object):
//   {"format": "tnb200-plan/1",
//    "leaves":  [tensor id of leaf slot 0, 1, ...],          // the network's leaves, for validation
//    "order":   [[i, j], ...],                             // leaf slots; result stored at i
//    "sliced":  [[q, k], ...],                             // sliced wires in loop-bit order (MSB first)
//    "n_global": g,                                        // -1: flat slicing (all bits are slice ids)
//    "global":  [1 if sliced[i] is a slice-id bit, ...],
//    "step_seg": [segment of step p, ...],
//    "segs":    [[D, Sum, E], ...],                        // tau-bit masks (decimal)
//    "companions": 0 | 1}                                  // 1: tie the sliced wires' companion edges
#include <cctype>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>

#include "tnb.h"

namespace tnb {

namespace {

// minimal JSON value: numbers are kept as their decimal text (uint64 masks must stay exact)
struct JV {
    enum Kind { NUL, NUM, STR, ARR, OBJ } kind = NUL;
    std::string text;
    std::vector<JV> arr;
    std::map<std::string, JV> obj;
    int64_t i64() const { return std::strtoll(text.c_str(), nullptr, 10); }
    uint64_t u64() const { return std::strtoull(text.c_str(), nullptr, 10); }
};

struct Parser {
    const std::string& s;
    size_t p = 0;
    std::string err;
    explicit Parser(const std::string& x) : s(x) {}
    void ws() {
        while (p < s.size() && std::isspace((unsigned char)s[p])) p++;
    }
    bool value(JV& v) {
        ws();
        if (p >= s.size()) return fail("unexpected end");
        const char c = s[p];
        if (c == '[') {
            v.kind = JV::ARR;
            p++;
            ws();
            if (p < s.size() && s[p] == ']') { p++; return true; }
            while (true) {
                JV x;
                if (!value(x)) return false;
                v.arr.push_back(std::move(x));
                ws();
                if (p < s.size() && s[p] == ',') { p++; continue; }
                if (p < s.size() && s[p] == ']') { p++; return true; }
                return fail("expected , or ]");
            }
        }
        if (c == '{') {
            v.kind = JV::OBJ;
            p++;
            ws();
            if (p < s.size() && s[p] == '}') { p++; return true; }
            while (true) {
                JV k;
                ws();
                if (!value(k) || k.kind != JV::STR) return fail("expected a key");
                ws();
                if (p >= s.size() || s[p] != ':') return fail("expected :");
                p++;
                JV x;
                if (!value(x)) return false;
                v.obj[k.text] = std::move(x);
                ws();
                if (p < s.size() && s[p] == ',') { p++; continue; }
                if (p < s.size() && s[p] == '}') { p++; return true; }
                return fail("expected , or }");
            }
        }
        if (c == '"') {
            v.kind = JV::STR;
            p++;
            while (p < s.size() && s[p] != '"') v.text += s[p++];
            if (p >= s.size()) return fail("unterminated string");
            p++;
            return true;
        }
        if (c == '-' || std::isdigit((unsigned char)c)) {
            v.kind = JV::NUM;
            while (p < s.size() && (s[p] == '-' || s[p] == '+' || s[p] == '.' || s[p] == 'e' || s[p] == 'E' ||
                                    std::isdigit((unsigned char)s[p])))
                v.text += s[p++];
            return true;
        }
        if (s.compare(p, 4, "null") == 0) {
            p += 4;
            return true;
        }
        return fail("unexpected character");
    }
    bool fail(const std::string& m) {
        std::ostringstream o;
        o << m << " at offset " << p;
        err = o.str();
        return false;
    }
};

int find_edge(const Network& net, int q, int k) {
    for (int e = 0; e < (int)net.edges.size(); e++) {
        const Edge& E = net.edges[e];
        if (E.q == q && E.k == k && !E.output && E.t1 >= 0 && net.tensors[E.t0].alive && net.tensors[E.t1].alive)
            return e;
    }
    return -1;
}

}  // namespace

std::string save_plan(const Network& net, const std::vector<Leaf>& leaves, const Plan& plan, const std::string& path) {
    std::ofstream f(path);
    if (!f) return "cannot open " + path;
    f << "{\"format\": \"tnb200-plan/1\",\n \"leaves\": [";
    for (size_t i = 0; i < leaves.size(); i++) f << (i ? "," : "") << leaves[i].tensor_id;
    f << "],\n \"order\": [";
    for (size_t p = 0; p < plan.order.size(); p++)
        f << (p ? "," : "") << "[" << plan.order[p].first << "," << plan.order[p].second << "]";
    f << "],\n \"sliced\": [";
    for (size_t i = 0; i < plan.sliced.size(); i++)
        f << (i ? "," : "") << "[" << net.edges[plan.sliced[i]].q << "," << net.edges[plan.sliced[i]].k << "]";
    f << "],\n \"n_global\": " << (plan.segs.empty() ? -1 : plan.n_global) << ",\n \"global\": [";
    for (size_t i = 0; i < plan.is_global.size(); i++) f << (i ? "," : "") << (int)plan.is_global[i];
    f << "],\n \"step_seg\": [";
    for (size_t p = 0; p < plan.step_seg.size(); p++) f << (p ? "," : "") << plan.step_seg[p];
    f << "],\n \"segs\": [";
    for (size_t j = 0; j < plan.segs.size(); j++)
        f << (j ? "," : "") << "[" << plan.segs[j].D << "," << plan.segs[j].Sum << "," << plan.segs[j].E << "]";
    f << "],\n \"companions\": " << (plan.companions ? 1 : 0) << "}\n";
    return f ? "" : "write failed: " + path;
}

std::string load_plan(const Network& net, const std::vector<Leaf>& leaves, const std::string& path, Plan& plan) {
    std::ifstream f(path);
    if (!f) return "cannot open plan file " + path;
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    Parser P(text);
    JV root;
    if (!P.value(root) || root.kind != JV::OBJ) return "plan file " + path + ": " + (P.err.empty() ? "not an object" : P.err);
    auto get = [&](const char* k) -> const JV* {
        auto it = root.obj.find(k);
        return it == root.obj.end() ? nullptr : &it->second;
    };
    const JV* fmt = get("format");
    if (!fmt || fmt->text != "tnb200-plan/1") return "plan file: unknown format";
    const JV* jl = get("leaves");
    const JV* jo = get("order");
    const JV* js = get("sliced");
    if (!jl || !jo || !js || jl->kind != JV::ARR || jo->kind != JV::ARR || js->kind != JV::ARR)
        return "plan file: missing leaves / order / sliced";
    const int NL = (int)leaves.size();
    if ((int)jl->arr.size() != NL) return "plan file: leaf count differs from the network";
    for (int i = 0; i < NL; i++)
        if (jl->arr[i].i64() != leaves[i].tensor_id) return "plan file: leaf tensor ids differ from the network";
    Plan pl;
    std::vector<char> alive(NL, 1);
    for (const JV& pr : jo->arr) {
        if (pr.kind != JV::ARR || pr.arr.size() != 2) return "plan file: bad order entry";
        const int i = (int)pr.arr[0].i64(), j = (int)pr.arr[1].i64();
        if (i < 0 || j < 0 || i >= NL || j >= NL || i == j || !alive[i] || !alive[j])
            return "plan file: order entry refers to a consumed or unknown slot";
        alive[j] = 0;
        pl.order.push_back({i, j});
    }
    if ((int)pl.order.size() != NL - 1) return "plan file: the order does not contract the whole network";
    for (const JV& w : js->arr) {
        if (w.kind != JV::ARR || w.arr.size() != 2) return "plan file: bad sliced wire";
        const int e = find_edge(net, (int)w.arr[0].i64(), (int)w.arr[1].i64());
        if (e < 0) return "plan file: sliced wire is not an internal edge of the network";
        for (int x : pl.sliced)
            if (x == e) return "plan file: duplicate sliced wire";
        pl.sliced.push_back(e);
    }
    const JV* jg = get("n_global");
    const int ng = jg ? (int)jg->i64() : -1;
    const int s = (int)pl.sliced.size();
    if (ng >= 0) {
        const JV* jss = get("step_seg");
        const JV* jsg = get("segs");
        if (!jss || !jsg || jss->kind != JV::ARR || jsg->kind != JV::ARR) return "plan file: missing segments";
        if (ng > s) return "plan file: n_global > number of sliced wires";
        pl.n_global = ng;
        const JV* jgl = get("global");
        if (!jgl || jgl->kind != JV::ARR || (int)jgl->arr.size() != s) return "plan file: missing global flags";
        int cnt = 0;
        for (const JV& x : jgl->arr) {
            pl.is_global.push_back(x.i64() ? 1 : 0);
            cnt += x.i64() ? 1 : 0;
        }
        if (cnt != ng) return "plan file: n_global differs from the global flags";
        for (const JV& x : jsg->arr) {
            if (x.kind != JV::ARR || x.arr.size() != 3) return "plan file: bad segment";
            Plan::Seg g;
            g.D = x.arr[0].u64();
            g.Sum = x.arr[1].u64();
            g.E = x.arr[2].u64();
            const uint64_t all = s >= 64 ? ~0ull : ((1ull << s) - 1);
            if ((g.D | g.Sum | g.E) & ~all) return "plan file: segment mask outside the sliced bits";
            pl.segs.push_back(g);
        }
        if (pl.segs.empty()) return "plan file: a loop program needs at least one segment";
        if ((int)jss->arr.size() != NL - 1) return "plan file: step_seg length differs from the order";
        int last = 0;
        for (const JV& x : jss->arr) {
            const int j = (int)x.i64();
            if (j < last || j >= (int)pl.segs.size()) return "plan file: step segments must be nondecreasing and valid";
            last = j;
            pl.step_seg.push_back(j);
        }
        // the local bits must each be summed exactly once
        uint64_t summed = 0, local = 0;
        for (int i = 0; i < s; i++)
            if (!pl.is_global[i]) local |= 1ull << (s - 1 - i);
        for (const Plan::Seg& g : pl.segs) {
            if (g.E & summed) return "plan file: a local bit is summed twice";
            summed |= g.E;
        }
        if (summed != local) return "plan file: the summed bits must be exactly the local bits";
    }
    const JV* jc = get("companions");
    pl.companions = jc && jc->i64() != 0;
    plan = pl;
    return "";
}

}  // namespace tnb
