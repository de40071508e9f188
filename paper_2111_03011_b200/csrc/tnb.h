// tnb.h -- internal host-side data structures of the B200 sliced sparse-state contraction.
// Citations: P:Lnnn = PAPER.md line; SURVEY §x = repo blueprint.
#pragma once

#include <complex>
#include <cstdint>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tn.h"

namespace tnb {

using cd = std::complex<double>;

// ---------------------------------------------------------------------------- network

struct Edge {
    int q = -1, k = -1;     // wire id (q, k): segment of qubit q after its k-th gate
    int t0 = -1, t1 = -1;   // endpoint tensors; t1 = -1 for an output leg
    bool output = false;    // output leg of qubit q (final-state boundary)
    bool open = false;      // output leg of an open qubit (kept dense)
};

struct HTensor {
    std::vector<int> legs;  // edge ids; legs[0] is the most significant bit of the dense index
    std::vector<cd> data;   // 2^legs.size() values (fp64 on the host)
    bool alive = true;
};

// One (undrilled) fSim gate of the circuit, for the companion-edge rank-one truncation:
// its input / output edges per qubit (in = -1: the |0> input) and the single-qubit products absorbed
// into its tensor on each input (T = fSim (P_a x P_b)).
struct FsimRec {
    int q[2] = {-1, -1};
    int in[2] = {-1, -1}, out[2] = {-1, -1};
    int kin[2] = {0, 0};  // gates on each qubit before this one: wire (q, kin) = right before the gate
    cd P[2][2][2];  // P[i][row][col]
    double theta = 0;
};

struct Network {
    int n = 0;
    std::vector<Edge> edges;
    std::vector<HTensor> tensors;
    std::vector<FsimRec> fsims;
};

// A leaf of the contraction in row form: the fixed output legs of the tensor are absorbed as
// sparse rows = sorted distinct projections of the requested bitstrings onto those qubits
// (SURVEY App. A.3).  Row keys are the bitstring masked to the fixed qubits, so
// ascending keys = ascending packed projections with the lowest qubit id as MSB.
struct Leaf {
    int tensor_id = -1;
    uint64_t qmask = 0;            // fixed qubits (bitstring-convention mask)
    std::vector<uint64_t> rows;    // sorted distinct (fixed & qmask); {0} when qmask == 0
    std::vector<int> legs;         // dense legs (edge ids), MSB first
    std::vector<cd> data;          // rows.size() * 2^legs.size()
};

struct Request {
    int n = 0;
    uint64_t open_mask = 0;
    int64_t M = 0, l = 1, L = 0;
    std::vector<uint64_t> bits;    // the M requested bitstrings (caller order)
    std::vector<uint64_t> fixed;   // distinct fixed parts, sorted (bits & ~open_mask)
};

// Build the network of a circuit (one tensor per fSim; single-qubit gates and |0> inputs
// absorbed into the next tensor on the wire, the final layer into the previous one) and
// simplify it (order-1 and order-2 tensors contracted into neighbours).
// Returns an empty string on success, else an error message.

// holes: indices into c->gates of fSim gates drilled out (both input edges broken)
std::string build_network(const tn_circuit* c, Network& net, const std::vector<int32_t>& holes = {});
void simplify(Network& net);
std::vector<Leaf> make_leaves(const Network& net, const Request& req);

// generic host contraction of two dense tensors (fp64); result legs = A\B then B\A
HTensor contract_host(const HTensor& A, const HTensor& B);

// rows of the fixed set qmask: sorted distinct (fixed & qmask)
std::vector<uint64_t> rows_of(const Request& req, uint64_t qmask);

// ---------------------------------------------------------------------------- plan

struct PlanTensor {
    std::vector<int> legs;   // sorted dense edge ids
    uint64_t qmask = 0;
    double rows = 1;
};

struct Plan {
    std::vector<std::pair<int, int>> order;  // (i, j): contract leaves/intermediates, result at i
    std::vector<int> sliced;                 // edge ids, MSB-first slice order
    // companion edges: edge, slice bit of its partner sliced edge, fidelity factor
    std::vector<std::pair<int, int>> tied;
    std::vector<double> tied_factor;
    std::vector<std::pair<int, int>> tied_wire;  // (q, k): the projector's wire, right before the gate
    double cmac = 0, bytes = 0, time_s = 0;  // per slice
    double peak = 0;                         // elements, per slice
    // Loop program (head/tail local slices; planner.cpp loop_nest).  Empty `segs`: flat
    // slicing, every sliced edge is a slice-id bit.  Otherwise `sliced` lists every looped edge by loop
    // significance (outermost first); is_global marks the slice-id bits (global slices, summed by the readout;
    // slice id sigma's bits are the global entries in list order), the rest are local loop bits summed inside
    // the program.  Loop index tau has s = sliced.size() bits, sliced[i] <-> tau bit (s-1-i).  Pairwise step p
    // belongs to segment step_seg[p] (nondecreasing); the executor enumerates tau in increasing order (global
    // bits restricted to the caller's slice ids) and runs a segment when all its Sum bits are 1 and its D bits
    // differ from its previous run; E = local bits summed (accumulated) at the end of the segment.
    int n_global = -1;
    bool companions = false;  // plan file flag: the companion edges of the sliced wires are tied (add_companions)
    std::vector<char> is_global;   // loop program: per entry of `sliced`, 1 = a slice-id bit (any position)
    std::vector<int> step_seg;
    struct Seg {
        uint64_t D = 0, Sum = 0, E = 0;
    };
    std::vector<Seg> segs;
    double total_cmac = 0;   // modelled CMAC of the whole loop program over all global slices
    double persist_elems = 0;
};

// Companion-edge rank-one truncation (supplement "singular values of the sliced fSim gate"):
// for every sliced edge that is an output of an fSim gate G on qubit a, the input edge of G on the other
// qubit b is re-expressed in G's own input basis (the single-qubit product P_b absorbed into G's tensor
// moves across the edge into the upstream tensor: exact for unitary P_b) and tied to the sliced edge's
// slice bit, i.e. projected onto the dominant right singular vector e_v of the pinned gate.  Modifies
// `net` (pass a copy) and fills plan.tied / plan.tied_factor ((1 + sin^2 theta)/2 each).
void add_companions(Network& net, Plan& plan);

// (sliced edge -> companion edge) pairs that add_companions would cut, for the planner's cost model
struct CompanionPair {
    int sliced_edge, companion_edge, fsim, side;  // side: which input of net.fsims[fsim] is the companion
};
std::vector<CompanionPair> companion_pairs(const Network& net);

struct PlanOptions {
    int n_sliced = -1;
    std::vector<std::pair<int, int>> companions;  // (edge, companion): slicing edge also cuts companion
    std::vector<int> forced;   // edge ids
    uint64_t seed = 1;
    int trials = 0;
    double time_budget_s = 0;
    double max_elems = 0;
    int hyper = -1;
    int64_t sweep_iters = 0;   // annealing moves per sweep order (0: default)
    int method = 0;            // 0 auto, 1 flat slicing (greedy/bisection pool), 2 sweep loop program
    int max_segments = 8;      // loop program: at most this many segments
    double persist_budget = 0; // loop program: elements persisted across iterations (0: 8 x max_elems)            // multilevel-bisection tree search: 1 on, 0 off, -1 auto (> 160 leaves)
};

// row-count oracle used by the planner (exact with memo for small L, estimate otherwise)
struct RowModel {
    const Request* req = nullptr;
    double rows(uint64_t qmask);
    double estimate(uint64_t qmask) const;
    std::unordered_map<uint64_t, double> memo;
};

// A hypergraph for the partitioner (partition.cpp): nodes with weights, nets (pin lists) with weights.
struct HyperGraph {
    int n = 0;
    std::vector<int> node_w;
    std::vector<std::vector<int>> nets;
    std::vector<int> net_w;
    std::vector<int8_t> fixed;  // empty, or per node: -1 free, 0 / 1 fixed to that side
};
// Multilevel min-cut bisection: side[v] in {0, 1}, each side's node weight within (1/2 +- eps/2) * total
// when reachable.  init_tries greedy-growing starts at the coarsest level.
std::vector<char> ml_bisect(const HyperGraph& g, double eps, std::mt19937_64& rng, int init_tries);

std::string find_plan(const Network& net, const std::vector<Leaf>& leaves, const Request& req,
                      const PlanOptions& opt, Plan& out);

// Plan files (planfile.cpp): the order by tensor id, sliced wires (q, k) in bit
// order, n_global, step segments and the segment masks.  load_plan validates the file against the network.
std::string save_plan(const Network& net, const std::vector<Leaf>& leaves, const Plan& plan, const std::string& path);
std::string load_plan(const Network& net, const std::vector<Leaf>& leaves, const std::string& path, Plan& plan);

// ---------------------------------------------------------------------------- lowered program

// Bit mapping: destination bit dst[i] takes source bit src[i].
struct BitMap {
    int n = 0;
    int8_t src[40];
    int8_t dst[40];
};

enum BufRegion : int32_t { REG_NONE = 0, REG_WORK = 1, REG_BANK = 2, REG_MAPS = 3, REG_PERS = 4, REG_LVL = 5 };
struct BufRef {
    int32_t region = REG_NONE;
    int64_t offset = 0;   // bytes
};

enum StepKind : int32_t {
    K_INSTANTIATE = 0,
    K_APPLY = 1,
    K_PREP_A = 2,
    K_PREP_B = 3,
    K_GEMM = 4,
    K_READOUT = 5,
    K_PERMUTE = 6,
    K_MULTI = 7,
    K_ACCUM = 8,      // loop program: dst = ((tau & E) == 0 ? 0 : dst) + src (local-slice summation)
    K_SETTAU = 9,     // (executor-internal)
    K_GATE = 10       // stem x small rowless tensor on the tensor cores (gate_tc.cuh), ApplyParams
};

// General sparse-row pairwise contraction (SIMT path):
//   C[r][c] = sum_kk A[ma[r]][addrA(c, kk)] * B[mb[r]][addrB(c, kk)]
struct ApplyParams {
    BufRef A, B, C;
    BufRef ma, mb;            // int32 maps (REG_MAPS); region NONE: A identity, B row 0
    BufRef rperm;             // int32 processing order of the output rows (grouped by A parent), or NONE
    int64_t R = 1;            // output rows
    int64_t a_row = 0, b_row = 0, c_row = 0;   // row strides in complex elements
    int dA = 0, dB = 0, dC = 0;
    BitMap cA;                // C bit -> A bit (A-free legs)
    BitMap cB;                // C bit -> B bit (B-free legs)
    int nk = 0;
    int8_t kA[40], kB[40];    // contracted leg i at A bit kA[i], B bit kB[i]
    int n_inner = 0;          // number of B-free C bits computed per thread (<= 4)
    int8_t inner_c[4];        // their C bit positions
    int64_t a_elems = 0, b_elems = 0;  // operand extents (complex elements), for hazard analysis
    // K_GATE variants (gate_tc.cuh GateDev::mode): 1 = gate per B row (rows in gperm order), 2 = tiles over A rows
    // with the gate columns = the B rows of the A row's output rows (gstart / gcnt per A row, <= gm members)
    int gate_mode = 0;
    BufRef gperm, gstart, gcnt;
    int gm = 1;
    int64_t a_rows = 0;
};

// Tensor-core path: TTGT with 3xTF32.
//   PREP_A: Ahi/Alo [Mp][2K] fp32 (K-major, complex interleaved along K) from A (rows via ma)
//   PREP_B: Bhi/Blo [2N][2K] fp32 (K-major), the real embedding [[br, -bi], [bi, br]]^T
//   GEMM  : C[Mp][2N] fp32 (= complex [Mp][N]) = Ahi*Bhi + Ahi*Blo + Alo*Bhi
struct GemmParams {
    BufRef A, B, C, ma;
    BufRef Ahi, Alo, Bhi, Blo;
    int64_t R = 1, m = 1, n = 1, k = 1;  // per-row m (A-free), n (B-free), k; Mp = R * m
    int64_t a_row = 0;
    int dA = 0, dB = 0;
    BitMap aM, aK;            // A index bits from (m index bit -> A bit), (k index bit -> A bit)
    BitMap bN, bK;            // B index bits from (n index bit -> B bit), (k index bit -> B bit)
    int gather_a = 0;         // 1: no A pre-pass; the GEMM's producer warps gather + split A (gemm_tc.cuh GatherA)
    int c_colmajor = 0;       // plain GEMM: C legs = B-free legs on top, A-free legs low (coalesced epilogue stores)
    int embed_a = 0;          // 1: embed A ([2Mp][2K] rows (ar,-ai),(ai,ar)), B plain [N][2K] ("EA");
                              // 0: A plain [Mp][2K], embed B ([2N][2K] rows (br,-bi),(bi,br)) ("EB")
    // grouped mode (both operands carry rows, SURVEY a6 GATHER-CONTRACT on the tensor cores): output
    // rows are grouped by their A parent; group a is the GEMM A_a [m x k] x [B_{mb[r]} for r in group]
    // [k x n|G_a|].  A is prepped as-is (R = A's rows, no map), B is gathered in group order through
    // `rowsel` (B row of gathered block p), and the epilogue scatters block p to output row perm[p].
    int grouped = 0;
    int64_t RC = 0;           // output rows (grouped)
    int64_t NB = 0;           // gathered B blocks (= RC)
    int64_t b_row = 0;
    BufRef perm, rowsel, tiles;   // tiles: 128 x 128 (single-CTA tiles)
    int64_t n_tiles = 0;
    BufRef tiles2;                 // 256 x 256 tiles for CTA pairs (same format)
    int64_t n_tiles2 = 0;
};

// one output tile of the grouped tensor-core GEMM (D-row / D-col units, see GemmParams::grouped)
struct GemmTile {
    int32_t x0, xvalid, xbase, y0, yvalid, ybase, off, pad;
};

struct InstParams {
    int64_t n_items = 0;      // total elements written across all sliced leaves
    BufRef table;             // REG_MAPS: per-leaf descriptors (see executor)
    int32_t n_leaves = 0;
};

struct AccumParams {
    BufRef src, dst;
    int64_t n = 0;            // complex elements
    uint64_t E = 0;           // tau bits summed here: the first value (all zero) overwrites
};

struct ReadoutParams {
    BufRef F;                 // final tensor
    BufRef idx;               // REG_MAPS: int64 index per amplitude
    int64_t M = 0;
};

// one workspace / persistent-region range a step reads or writes (the executor derives the graph's
// dependency edges from these: RAW / WAR / WAW overlaps)
struct MemAcc {
    int32_t region = REG_NONE;
    int32_t write = 0;
    int64_t offset = 0, bytes = 0;
};

struct Step {
    int32_t kind = 0;
    int32_t pair = -1;        // pairwise step index
    double cmac = 0, bytes = 0;
    std::vector<MemAcc> mem;  // REG_WORK / REG_PERS accesses (bank and maps are read-only)
    ApplyParams ap;
    GemmParams gp;
    InstParams ip;
    ReadoutParams rp;
    AccumParams cp;
};

// device-side descriptor of one sliced leaf for K_INSTANTIATE (slice instantiate, row a2)
struct InstLeafDesc {
    int64_t bank_off;     // complex elements into the leaf bank
    int64_t out_off;      // bytes into the workspace
    int64_t item_begin;   // first global item of this leaf
    int64_t items;        // rows * 2^d_out
    int32_t d_full, d_out, n_sl, pad;
    int8_t out_src[40];   // output bit b (LSB = 0) comes from full bit out_src[b]
    int8_t sl_pos[24];    // sliced leg j sits at full bit sl_pos[j] ...
    int8_t sl_idx[24];    // ... and takes slice bit sl_idx[j]: value (sigma >> (s-1-idx)) & 1
};

struct Program {
    std::vector<Step> steps;       // per slice
    std::vector<Step> pre_steps;   // slice-invariant steps, once per tn_contract (outputs in REG_PERS)
    int64_t pers_bytes = 0;
    std::vector<float> bank;       // complex64 leaf bank (interleaved)
    std::vector<uint8_t> maps;     // int32/int64 maps and tables
    int64_t work_bytes = 0;
    int64_t peak_elems = 0;
    double cmac = 0, bytes = 0, gemm_cmac = 0;  // per slice (slice-dependent steps)
    double pre_cmac = 0;                          // once per tn_contract (slice-invariant steps)
    int64_t n_pairs = 0;
    // per-leaf slicing info for K_INSTANTIATE (also in `maps`)
    int s = 0;
    // loop program (Plan::segs): per segment the run condition and its steps; empty = flat (`steps`)
    struct Seg {
        uint64_t D = 0, Sum = 0, E = 0;
        std::vector<Step> steps;
    };
    std::vector<Seg> segs;
    int s_global = 0;          // slice-id bits
    std::vector<char> bit_global;  // per sliced index (MSB first): 1 = slice-id bit
    int64_t lvl_bytes = 0;     // REG_LVL: tensors kept across loop iterations (checkpoints, accumulators)
    double total_cmac = 0;     // over all 2^s_global slices, counting each segment's runs
    // plan dump support
    std::string dump_json;
};

std::string lower_plan(const Network& net, const std::vector<Leaf>& leaves, const Request& req,
                       const Plan& plan, Program& prog);

}  // namespace tnb
