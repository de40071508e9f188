// api.cpp -- the extern "C" boundary declared in include/tn.h and include/tn_debug.h.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>

#include "../../include/tn_debug.h"
#include "exec.h"
#include "tnb.h"

struct tn_ctx {
    std::string err;
    tnb::Network net;
    tnb::Request req;
    std::vector<tnb::Leaf> leaves;
    bool planned = false;
    tnb::Plan plan;
    tnb::Program prog;
    std::vector<int32_t> sliced_wires;
    std::vector<int32_t> local_wires;
    std::vector<int32_t> companion_wires;
    tn_plan_info info{};
    tnb::Device* dev = nullptr;
};

namespace {

tn_status fail(tn_ctx* c, tn_status s, const std::string& m) {
    if (c) c->err = m;
    return s;
}

// splitmix64 counter-based stream (identical definition in tn_inputs/rng.py)
inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline uint64_t rng_key(uint64_t seed, uint64_t tag) { return mix64(seed ^ (tag * 0xD1B54A32D192ED03ull)); }
inline uint64_t rng_word(uint64_t key, uint64_t i) { return mix64(key + (i + 1) * 0x9E3779B97F4A7C15ull); }
constexpr uint64_t TAG_SAMPLER = 4;
constexpr uint64_t TAG_METROPOLIS = 5;

}  // namespace

extern "C" {

const char* tn_version(void) { return "tnb200 0.1 (sm_100a)"; }

const char* tn_last_error(const tn_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

void tn_destroy(tn_ctx* ctx) {
    if (!ctx) return;
    if (ctx->dev) tnb::dev_destroy(ctx->dev);
    delete ctx;
}

tn_status tn_build(const tn_circuit* circuit, const uint64_t* bitstrings, int64_t M, uint64_t open_mask,
                   tn_ctx** out) {
    return tn_build_drilled(circuit, bitstrings, M, open_mask, nullptr, 0, out);
}

tn_status tn_build_drilled(const tn_circuit* circuit, const uint64_t* bitstrings, int64_t M, uint64_t open_mask,
                           const int32_t* holes, int32_t n_holes, tn_ctx** out) {
    if (!out) return TN_EINVAL;
    *out = nullptr;
    tn_ctx* c = new tn_ctx();
    *out = c;  // returned even on failure so that tn_last_error works; caller must tn_destroy
    if (!circuit || !bitstrings || M < 1) return fail(c, TN_EINVAL, "null circuit/bitstrings or M < 1");
    const int n = circuit->n_qubits;
    if (n < 1 || n > 63) return fail(c, TN_EINVAL, "n_qubits must be in [1, 63]");
    const uint64_t full = (n == 64) ? ~0ull : ((1ull << n) - 1);
    if (open_mask & ~full) return fail(c, TN_EINVAL, "open_mask has bits outside the n qubits");
    tnb::Request& r = c->req;
    r.n = n;
    r.open_mask = open_mask;
    r.M = M;
    r.bits.assign(bitstrings, bitstrings + M);
    for (int64_t j = 0; j < M; j++)
        if (r.bits[j] & ~full) {
            std::ostringstream o;
            o << "bitstring " << j << " has bits beyond the " << n << " qubits";
            return fail(c, TN_EINVAL, o.str());
        }
    const int nopen = __builtin_popcountll(open_mask);
    r.l = (int64_t)1 << nopen;
    if (M % r.l) return fail(c, TN_EINVAL, "M is not a multiple of l = 2^popcount(open_mask)");
    r.L = M / r.l;
    if (open_mask) {
        // open configuration mu -> its bits, lowest open qubit id = MSB of mu
        std::vector<int> oq;
        for (int q = 0; q < n; q++)
            if ((open_mask >> (n - 1 - q)) & 1) oq.push_back(q);
        for (int64_t g = 0; g < r.L; g++) {
            const uint64_t f = r.bits[g * r.l] & ~open_mask;
            for (int64_t mu = 0; mu < r.l; mu++) {
                uint64_t want = f;
                for (int i = 0; i < nopen; i++)
                    if ((mu >> (nopen - 1 - i)) & 1) want |= 1ull << (n - 1 - oq[i]);
                if (r.bits[g * r.l + mu] != want) {
                    std::ostringstream o;
                    o << "group " << g << " entry " << mu << " breaks the group structure (shared fixed bits, "
                      << "open bits ascending)";
                    return fail(c, TN_EINVAL, o.str());
                }
            }
        }
    }
    r.fixed.resize(M);
    for (int64_t j = 0; j < M; j++) r.fixed[j] = r.bits[j] & ~open_mask;
    std::sort(r.fixed.begin(), r.fixed.end());
    r.fixed.erase(std::unique(r.fixed.begin(), r.fixed.end()), r.fixed.end());

    if (n_holes < 0 || (n_holes > 0 && !holes)) return fail(c, TN_EINVAL, "bad hole list");
    std::string e = tnb::build_network(circuit, c->net, std::vector<int32_t>(holes, holes + n_holes));
    if (!e.empty()) return fail(c, TN_EINVAL, e);
    for (auto& E : c->net.edges)
        if (E.output && ((open_mask >> (n - 1 - E.q)) & 1)) E.open = true;
    tnb::simplify(c->net);
    c->leaves = tnb::make_leaves(c->net, r);
    return TN_OK;
}

tn_status tn_plan(tn_ctx* ctx, const tn_slicing* slicing, int64_t max_tensor_size, tn_plan_info* info) {
    if (!ctx) return TN_EINVAL;
    if (ctx->leaves.empty()) return fail(ctx, TN_EINVAL, "tn_plan before a successful tn_build");
    if (max_tensor_size < 1) return fail(ctx, TN_EINVAL, "max_tensor_size must be >= 1");
    if (max_tensor_size > (1ll << 60)) return fail(ctx, TN_EINVAL, "max_tensor_size must be <= 2^60");
    if (ctx->dev) {
        tnb::dev_destroy(ctx->dev);
        ctx->dev = nullptr;
    }
    tnb::PlanOptions opt;
    opt.max_elems = (double)max_tensor_size;
    if (slicing) {
        opt.n_sliced = slicing->n_sliced;
        opt.seed = slicing->seed;
        opt.trials = slicing->trials;
        opt.time_budget_s = slicing->time_budget_s;
        if (slicing->n_forced < 0 || (slicing->n_forced > 0 && !slicing->forced_wires))
            return fail(ctx, TN_EINVAL, "bad forced wires");
        for (int i = 0; i < slicing->n_forced; i++) {
            int q = slicing->forced_wires[2 * i], k = slicing->forced_wires[2 * i + 1];
            int found = -1;
            for (int e = 0; e < (int)ctx->net.edges.size(); e++) {
                const tnb::Edge& E = ctx->net.edges[e];
                if (E.q == q && E.k == k && !E.output && E.t1 >= 0 && ctx->net.tensors[E.t0].alive &&
                    ctx->net.tensors[E.t1].alive)
                    found = e;
            }
            if (found < 0) {
                std::ostringstream o;
                o << "forced wire (" << q << "," << k << ") is not a sliceable edge of the simplified network";
                return fail(ctx, TN_EINVAL, o.str());
            }
            if (std::find(opt.forced.begin(), opt.forced.end(), found) != opt.forced.end())
                return fail(ctx, TN_EINVAL, "duplicate forced wire");
            opt.forced.push_back(found);
        }
        if (opt.n_sliced >= 0 && opt.n_sliced < (int)opt.forced.size())
            return fail(ctx, TN_EINVAL, "n_sliced smaller than the number of forced wires");
        if (opt.n_sliced > 62) return fail(ctx, TN_EINVAL, "n_sliced must be <= 62");
    }
    if (slicing && slicing->companions)
        for (const tnb::CompanionPair& cp : tnb::companion_pairs(ctx->net))
            opt.companions.push_back({cp.sliced_edge, cp.companion_edge});
    if (slicing) {
        opt.method = slicing->method;
        if (slicing->max_segments > 0) opt.max_segments = slicing->max_segments;
        opt.persist_budget = slicing->persist_budget;
    }
    tnb::Plan plan;
    std::string e;
    if (slicing && slicing->plan_path) {
        e = tnb::load_plan(ctx->net, ctx->leaves, slicing->plan_path, plan);
        if (!e.empty()) return fail(ctx, TN_EINVAL, e);
        if ((slicing->companions != 0) != plan.companions)
            return fail(ctx, TN_EINVAL, "tn_slicing.companions differs from the plan file's companions flag");
    } else {
        e = tnb::find_plan(ctx->net, ctx->leaves, ctx->req, opt, plan);
        if (!e.empty()) return fail(ctx, TN_EINFEASIBLE, e);
    }
    if (slicing && slicing->companions) {
        plan.companions = true;
        // the companion edges change the network (exact basis changes) and the leaves: plan on a copy
        tnb::Network net2 = ctx->net;
        tnb::add_companions(net2, plan);
        std::vector<tnb::Leaf> leaves2 = tnb::make_leaves(net2, ctx->req);
        e = tnb::lower_plan(net2, leaves2, ctx->req, plan, ctx->prog);
    } else {
        e = tnb::lower_plan(ctx->net, ctx->leaves, ctx->req, plan, ctx->prog);
    }
    if (!e.empty()) return fail(ctx, TN_EINVAL, e);
    ctx->plan = plan;
    ctx->planned = true;
    ctx->sliced_wires.clear();
    ctx->local_wires.clear();
    const int s_all = (int)plan.sliced.size();
    const int s_glob = plan.segs.empty() ? s_all : plan.n_global;
    for (int i = 0; i < s_all; i++) {
        const int eid = plan.sliced[i];
        const bool g = plan.segs.empty() || plan.is_global[i];
        auto& v = g ? ctx->sliced_wires : ctx->local_wires;
        v.push_back(ctx->net.edges[eid].q);
        v.push_back(ctx->net.edges[eid].k);
    }
    tn_plan_info& I = ctx->info;
    I = tn_plan_info{};
    I.s = (int32_t)s_glob;
    I.s_local = (int32_t)(s_all - s_glob);
    I.local_wires = ctx->local_wires.data();
    I.n_segments = plan.segs.empty() ? 1 : (int32_t)plan.segs.size();
    I.total_cmac = plan.segs.empty() ? std::ldexp(ctx->prog.cmac, s_all) + ctx->prog.pre_cmac : ctx->prog.total_cmac;
    I.persist_bytes = ctx->prog.lvl_bytes;
    I.sliced_wires = ctx->sliced_wires.data();
    I.n_tensors = (int64_t)ctx->leaves.size();
    I.n_steps = ctx->prog.n_pairs;
    I.n_launches = (int64_t)ctx->prog.steps.size();
    for (const auto& sg : ctx->prog.segs) I.n_launches += (int64_t)sg.steps.size();
    I.peak_elems = std::max<int64_t>(ctx->prog.peak_elems, 1);
    // per pipeline: step workspace + the loop program's kept region (executor.cu dev_bind)
    I.workspace_bytes = ((ctx->prog.work_bytes + 4095) & ~(int64_t)4095) +
                        (ctx->prog.segs.empty() ? 0 : ((ctx->prog.lvl_bytes + 4095) & ~(int64_t)4095));
    I.cmac_per_slice = ctx->prog.cmac;
    I.bytes_per_slice = ctx->prog.bytes;
    I.gemm_cmac_per_slice = ctx->prog.gemm_cmac;
    I.n_invariant_steps = 0;
    for (const auto& st : ctx->prog.pre_steps)
        if (st.kind == tnb::K_APPLY || st.kind == tnb::K_GEMM) I.n_invariant_steps++;
    I.invariant_cmac = ctx->prog.pre_cmac;
    ctx->companion_wires.clear();
    I.companion_fidelity = 1.0;
    // a companion's partner index counts in sliced_wires, then local_wires (loop programs)
    std::vector<int> pub(s_all, 0);
    for (int i = 0, ng = 0, nl = 0; i < s_all; i++)
        pub[i] = (plan.segs.empty() || plan.is_global[i]) ? ng++ : s_glob + nl++;
    for (size_t t = 0; t < plan.tied.size(); t++) {
        ctx->companion_wires.push_back(plan.tied_wire[t].first);
        ctx->companion_wires.push_back(plan.tied_wire[t].second);
        ctx->companion_wires.push_back(pub[plan.tied[t].second]);
        I.companion_fidelity *= plan.tied_factor[t];
    }
    I.n_companions = (int32_t)plan.tied.size();
    I.companion_wires = ctx->companion_wires.data();
    if (info) *info = I;
    return TN_OK;
}

tn_status tn_plan_dump(const tn_ctx* ctx, const char* path) {
    if (!ctx || !path) return TN_EINVAL;
    if (!ctx->planned) return TN_EINVAL;
    std::ofstream f(path);
    if (!f) return TN_EINVAL;
    f << ctx->prog.dump_json;
    return TN_OK;
}

tn_status tn_plan_save(const tn_ctx* ctx, const char* path) {
    if (!ctx || !path) return TN_EINVAL;
    if (!ctx->planned) return TN_EINVAL;
    std::string e = tnb::save_plan(ctx->net, ctx->leaves, ctx->plan, path);
    if (!e.empty()) return TN_EINVAL;
    return TN_OK;
}

tn_status tn_bind_device(tn_ctx* ctx, int device, void* workspace, size_t bytes, void* cuda_stream) {
    if (!ctx) return TN_EINVAL;
    if (!ctx->planned) return fail(ctx, TN_EINVAL, "tn_bind_device before tn_plan");
    if (ctx->prog.peak_elems > (1ll << 32))
        return fail(ctx, TN_EINVAL, "plan has a tensor above 2^32 elements (executor index range); re-plan with a "
                                    "smaller max_tensor_size");
    if (ctx->dev) {
        tnb::dev_destroy(ctx->dev);
        ctx->dev = nullptr;
    }
    std::string e;
    int rc = tnb::dev_bind(&ctx->dev, ctx->prog, device, workspace, bytes, cuda_stream, ctx->req.M, 32, e);
    if (rc) return fail(ctx, (tn_status)rc, e);
    return TN_OK;
}

tn_status tn_contract(tn_ctx* ctx, const uint64_t* slice_ids, int64_t n_ids, void* amps_out, int32_t out_on_device,
                      double* seconds_out) {
    if (!ctx) return TN_EINVAL;
    if (!ctx->dev) return fail(ctx, TN_EINVAL, "tn_contract before tn_bind_device");
    if (!slice_ids || n_ids < 1) return fail(ctx, TN_EINVAL, "empty slice subset");
    if (!amps_out) return fail(ctx, TN_EINVAL, "null amps_out");
    const int s = ctx->plan.segs.empty() ? (int)ctx->plan.sliced.size() : ctx->plan.n_global;
    std::vector<uint64_t> ids(slice_ids, slice_ids + n_ids);
    std::sort(ids.begin(), ids.end());
    for (int64_t i = 0; i < n_ids; i++) {
        if (s < 64 && ids[i] >= (1ull << s)) return fail(ctx, TN_EINVAL, "slice id out of range [0, 2^s)");
        if (i && ids[i] == ids[i - 1]) return fail(ctx, TN_EINVAL, "duplicate slice id");
    }
    std::string e;
    int rc = tnb::dev_contract(ctx->dev, ids.data(), n_ids, amps_out, out_on_device != 0, seconds_out, e);
    if (rc) return fail(ctx, (tn_status)rc, e);
    return TN_OK;
}

tn_status tn_segment_runs(tn_ctx* ctx, const uint64_t* slice_ids, int64_t n_ids, int64_t* runs) {
    if (!ctx || !runs) return TN_EINVAL;
    if (!ctx->dev) return fail(ctx, TN_EINVAL, "tn_segment_runs before tn_bind_device");
    if (!slice_ids || n_ids < 1) return fail(ctx, TN_EINVAL, "empty slice subset");
    const int s = ctx->plan.segs.empty() ? (int)ctx->plan.sliced.size() : ctx->plan.n_global;
    std::vector<uint64_t> ids(slice_ids, slice_ids + n_ids);
    std::sort(ids.begin(), ids.end());
    for (int64_t i = 0; i < n_ids; i++) {
        if (s < 64 && ids[i] >= (1ull << s)) return fail(ctx, TN_EINVAL, "slice id out of range [0, 2^s)");
        if (i && ids[i] == ids[i - 1]) return fail(ctx, TN_EINVAL, "duplicate slice id");
    }
    return (tn_status)tnb::dev_segment_runs(ctx->dev, ids.data(), n_ids, runs);
}

tn_status tn_profile_slice(tn_ctx* ctx, uint64_t slice_id, tn_launch_stat* stats, int32_t max_stats,
                           int32_t* n_stats) {
    if (!ctx || !stats || !n_stats) return TN_EINVAL;
    if (!ctx->dev) return fail(ctx, TN_EINVAL, "tn_profile_slice before tn_bind_device");
    const int s = (int)ctx->plan.sliced.size();
    if (s < 64 && slice_id >= (1ull << s)) return fail(ctx, TN_EINVAL, "slice id out of range");
    std::string e;
    int n = 0;
    int rc = tnb::dev_profile(ctx->dev, slice_id, stats, max_stats, &n, e);
    *n_stats = n;
    if (rc) return fail(ctx, (tn_status)rc, e);
    return TN_OK;
}

tn_status tn_sample_report(const tn_ctx* cctx, const float* amps, const float* ideal_amps, int64_t n_slices_summed,
                           uint64_t seed, int32_t sampler, int32_t steps, uint64_t* samples_out, int64_t* index_out,
                           tn_report* rep) {
    tn_ctx* ctx = const_cast<tn_ctx*>(cctx);
    if (!ctx || !amps || !samples_out || !rep) return TN_EINVAL;
    const tnb::Request& r = ctx->req;
    if (r.M < 1) return fail(ctx, TN_EINVAL, "tn_sample before tn_build");
    const int s = ctx->planned ? (int)ctx->plan.sliced.size() : 0;
    if (n_slices_summed < 1 || (s < 63 && n_slices_summed > (1ll << s)))
        return fail(ctx, TN_EINVAL, "n_slices_summed must be in [1, 2^s]");
    if (sampler != 0 && sampler != 1) return fail(ctx, TN_EINVAL, "sampler must be 0 (categorical) or 1 (Metropolis)");
    if (sampler == 1 && steps < 1) return fail(ctx, TN_EINVAL, "Metropolis needs steps >= 1");
    auto w_of = [&](const float* a, int64_t mu) {
        const double re = (double)a[2 * mu], im = (double)a[2 * mu + 1];
        return re * re + im * im;
    };
    auto u53 = [](uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); };
    const uint64_t key = rng_key(seed, TAG_SAMPLER);
    const uint64_t mkey = rng_key(seed, TAG_METROPOLIS);
    const uint64_t stride = 2 * (uint64_t)std::max(steps, 0) + 1;
    std::vector<int64_t> pick_j(r.L);
    double norm2 = 0.0;
    for (int64_t g = 0; g < r.L; g++) {
        const float* a = amps + 2 * g * r.l;
        // weights |a|^2 = re*re + im*im in fp64, cumulated in ascending mu
        double tot = 0.0;
        for (int64_t mu = 0; mu < r.l; mu++) tot += w_of(a, mu);
        if (!(tot > 0.0)) {
            std::ostringstream o;
            o << "all-zero group " << g;
            return fail(ctx, TN_ENUMERIC, o.str());
        }
        norm2 += tot;
        int64_t pick = r.l - 1;
        if (sampler == 0) {
            const double thr = u53(rng_word(key, (uint64_t)g)) * tot;
            double cum = 0.0;
            for (int64_t mu = 0; mu < r.l; mu++) {
                cum += w_of(a, mu);
                if (cum > thr) {
                    pick = mu;
                    break;
                }
            }
        } else {
            const uint64_t c0 = (uint64_t)g * stride;
            auto idx = [&](uint64_t c) { return std::min<int64_t>(r.l - 1, (int64_t)(u53(rng_word(mkey, c)) * (double)r.l)); };
            int64_t x = idx(c0);
            double wx = w_of(a, x);
            for (int t = 1; t <= steps; t++) {
                const int64_t y = idx(c0 + 2 * (uint64_t)t - 1);
                const double wy = w_of(a, y);
                if (u53(rng_word(mkey, c0 + 2 * (uint64_t)t)) * wx < wy) {
                    x = y;
                    wx = wy;
                }
            }
            pick = x;
        }
        pick_j[g] = g * r.l + pick;
    }
    const double N = std::ldexp(1.0, r.n);
    const double nan = std::nan("");
    rep->f = (double)n_slices_summed / std::ldexp(1.0, s);
    rep->F_norm = N / (double)r.M * norm2;
    // phat_j = |a_j|^2 / F_norm (a distribution over all 2^n bitstrings, estimated from the M requested)
    const double Z = rep->F_norm;
    double hs = 0.0, xs = 0.0, ls = 0.0;
    for (int64_t g = 0; g < r.L; g++) {
        const int64_t j = pick_j[g];
        samples_out[g] = r.bits[j];
        if (index_out) index_out[g] = j;
        hs -= std::log(w_of(amps, j) / Z);
        if (ideal_amps) {
            const double P = w_of(ideal_amps, j);
            xs += P;
            ls += std::log(N * P);
        }
    }
    constexpr double kEulerGamma = 0.57721566490153286061;
    rep->entropy_samples = hs / (double)r.L;
    rep->xeb = ideal_amps ? N / (double)r.L * xs - 1.0 : nan;
    rep->log_xeb = ideal_amps ? ls / (double)r.L + kEulerGamma : nan;
    double hst = 0.0;
    std::vector<double> x(r.M);
    for (int64_t j = 0; j < r.M; j++) {
        const double p = w_of(amps, j) / Z;
        if (p > 0) hst -= p * std::log(p);
        x[j] = N * p;
    }
    rep->entropy_state = N / (double)r.M * hst;
    std::sort(x.begin(), x.end());
    double ks = 0.0;
    for (int64_t j = 0; j < r.M; j++) {
        const double F = -std::expm1(-x[j]);  // 1 - e^-x
        ks = std::max(ks, std::max((double)(j + 1) / (double)r.M - F, F - (double)j / (double)r.M));
    }
    rep->pt_ks = ks;
    return TN_OK;
}

tn_status tn_sample(const tn_ctx* ctx, const float* amps, const float* ideal_amps, int64_t n_slices_summed,
                    uint64_t seed, uint64_t* samples_out, double est[3]) {
    if (!est) return TN_EINVAL;
    tn_report rep;
    const tn_status st = tn_sample_report(ctx, amps, ideal_amps, n_slices_summed, seed, 0, 0, samples_out, nullptr, &rep);
    if (st != TN_OK) return st;
    est[0] = rep.f;
    est[1] = rep.F_norm;
    est[2] = rep.xeb;
    return TN_OK;
}

// ---------------------------------------------------------------------------- debug entries

tn_status tn_debug_gemm_tf32x3(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                               int32_t embed_a, void* cuda_stream) {
    std::string e;
    int rc = tnb::debug_gemm(A, B, C, M, N, K, embed_a, cuda_stream, e);
    return (tn_status)rc;
}

tn_status tn_debug_network(const tn_ctx* ctx, int64_t* n_tensors, int64_t* n_edges, int64_t* n_internal) {
    if (!ctx || ctx->leaves.empty()) return TN_EINVAL;
    int64_t alive = 0, internal = 0;
    for (auto& t : ctx->net.tensors) alive += t.alive;
    for (auto& E : ctx->net.edges)
        if (!E.output && E.t1 >= 0 && ctx->net.tensors[E.t0].alive && ctx->net.tensors[E.t1].alive) internal++;
    if (n_tensors) *n_tensors = alive;
    if (n_edges) *n_edges = (int64_t)ctx->net.edges.size();
    if (n_internal) *n_internal = internal;
    return TN_OK;
}

tn_status tn_debug_launch_counts(const tn_ctx* ctx, int64_t* per_slice, int64_t* per_contract) {
    if (!ctx || !ctx->dev) return TN_EINVAL;
    int64_t a = 0, b = 0;
    tnb::dev_launch_counts(ctx->dev, &a, &b);
    if (per_slice) *per_slice = a;
    if (per_contract) *per_contract = b;
    return TN_OK;
}

}  // extern "C"
