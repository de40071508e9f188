/*
 * tn.h -- C ABI of the B200-native sliced sparse-state contraction of arXiv:2111.03011
 * (F. Pan, K. Chen, P. Zhang, "Solving the Sampling Problem of the Sycamore Quantum
 * Circuits").  Citations "P:Lnnn" are lines of the paper text; "SURVEY §x" is the
 * repo's blueprint.
 *
 * The call sequence follows the paper's statement of the problem (BASELINE.json north_star):
 *     tn_build(circuit, bitstrings)        -> the network G with a sparse output boundary
 *     tn_plan(slicing, max_tensor_size)    -> contraction order + sliced edges
 *     tn_bind_device(...)                  -> program, leaf bank and row maps on the GPU
 *     tn_contract(slice_subset)            -> the M amplitudes summed over the subset
 *     tn_sample(amplitudes)                -> one bitstring per group + fidelity / XEB estimates
 *
 * Conventions:
 *   - bitstring: uint64, bit (n-1-q) = value of qubit q (qubit 0 = MSB), so the value equals the
 *     state-vector index.
 *   - wire (q, k): the segment of qubit q after its k-th gate, counting EVERY gate on q (single-
 *     and two-qubit), k >= 1.  Only internal segments between two fSim gates can be sliced.
 *   - slice id sigma in [0, 2^s): sliced wire e_i takes value (sigma >> (s-1-i)) & 1 (MSB-first),
 *     so the prefix [0, 2^(s-j)) pins e_0..e_(j-1) to 0 -- the paper's edge breaking with
 *     F ~ 2^-j.
 *   - complex numbers are interleaved (re, im); amplitudes are complex64.
 *
 * Errors: every call returns a tn_status; nothing throws or aborts across the ABI.  The message
 * of the last failure is available from tn_last_error(ctx).  A ctx is single-threaded; separate
 * ctxs (one per GPU / rank) are independent.
 *
 * Ownership: the caller owns every buffer it passes in; the library copies what it keeps.
 * The ctx owns the host network, the plan, and every device allocation the library makes
 * (leaf bank, maps, program; the workspace only when the caller passed none).  tn_destroy frees
 * exactly those, never caller memory.
 */
#ifndef TN_B200_H
#define TN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tn_ctx tn_ctx;

/* Status codes; 2/3/4 mirror SPEC.md's CLI exit codes. */
typedef enum {
    TN_OK = 0,
    TN_EINVAL = 2,       /* invalid argument or call out of order                      */
    TN_EINFEASIBLE = 3,  /* max_tensor_size unreachable even with every edge sliced      */
    TN_ENUMERIC = 4,     /* all-zero group / zero norm in tn_sample     */
    TN_ECUDA = 5,        /* a CUDA runtime / driver call failed                          */
    TN_ENOMEM = 6        /* workspace too small or allocation failed                     */
} tn_status;

/* One gate.  kind 0: single-qubit gate on q0 with matrix u = U[out][in] row-major as (re, im)
 * pairs: u = {U00.re, U00.im, U01.re, U01.im, U10.re, U10.im, U11.re, U11.im}.
 * kind 1: fSim(theta, phi) of P:L96-L102 (Eq. (1)) on (q0, q1), acting on the local index
 * 2*x_q0 + x_q1.  Unused fields are ignored. */
typedef struct {
    int32_t kind;
    int32_t q0, q1;
    double theta, phi;
    double u[8];
} tn_gate;

/* A circuit: gates of moment m are gates[moment_offsets[m] .. moment_offsets[m+1]).
 * qubit_rc (nullable): n_qubits (row, col) pairs; when given, fSim targets must be grid
 * neighbours.  No qubit may appear twice in a moment. */
typedef struct {
    int32_t n_qubits;            /* 1..63 */
    int32_t n_moments;
    const int32_t* moment_offsets;
    const tn_gate* gates;
    const int32_t* qubit_rc;
} tn_circuit;

/* tn_build -- P:L57-L60 (circuit -> tensor network G, |0> inputs and the final state as the two
 * boundaries), P:L130 (order-1/2 tensors contracted into neighbours)
 * (the sparse-state boundary: only the requested bitstrings' configurations are computed).
 *   bitstrings: M requested bitstrings (uint64, see conventions), M >= 1.
 *   open_mask : bitstring-convention mask of the open qubits O.  0 means every
 *               qubit is fixed (l = 1).  Otherwise the entries must come in groups of
 *               l = 2^popcount(open_mask) consecutive bitstrings that share their fixed bits,
 *               with the open bits running through all l values in ascending order.
 * Copies the circuit and the bitstrings.  EINVAL on: n out of range, bad gate, non-adjacent fSim
 * (when qubit_rc given), qubit repeated in a moment, bitstring >= 2^n, broken group structure. */
tn_status tn_build(const tn_circuit* circuit, const uint64_t* bitstrings, int64_t M,
                   uint64_t open_mask, tn_ctx** out);

/* tn_build_drilled -- tn_build on the network with K/2 holes drilled (Fig. 1 "each hole is
 * created by breaking two edges"; case (i) P:L106-L109).  holes[h] indexes circuit->gates and must be
 * an fSim gate; both of its input edges are broken, E = (1,0)x(1,0) inserted on each qubit right before
 * the gate (after its pending single-qubit gates).  Because fSim|00> = |00>, the gate then drops out of the
 * network exactly: each of its wires carries |0><0| U and the two qubits decouple at that gate.  Wire ids
 * are unchanged (the drilled gate still counts on both wires).  The estimated fidelity of the result is
 * 2^-2 per hole times the slice fraction.  EINVAL on a hole that is out of range, not an fSim, or
 * repeated; otherwise as tn_build. */
tn_status tn_build_drilled(const tn_circuit* circuit, const uint64_t* bitstrings, int64_t M, uint64_t open_mask,
                           const int32_t* holes, int32_t n_holes, tn_ctx** out);

typedef struct {
    int32_t n_sliced;            /* -1: the minimal s meeting max_tensor_size; else exactly s  */
    int32_t n_forced;            /* sliced wires forced first (in this order)                 */
    const int32_t* forced_wires; /* 2*n_forced ints: (q, k) pairs                             */
    uint64_t seed;               /* planner randomisation seed                                */
    int32_t trials;              /* randomized greedy restarts (<= 0: default)                */
    double time_budget_s;        /* planner wall-clock budget (<= 0: default)                 */
    int32_t companions;          /* 1: companion-edge rank-one truncation: for each
                                    sliced wire that is an output of an fSim G, the input edge of G
                                    on the other qubit is projected onto the dominant singular vector
                                    of the pinned gate, i.e. onto |v> in G's input basis with v the
                                    sliced wire's value (cutting that companion edge too); fidelity
                                    factor (1 + sin^2 theta)/2 each.  Flat plans and loop
                                    programs (the interface's companion edges); with
                                    plan_path it must equal the plan file's "companions" flag       */
    int32_t method;              /* 0 auto (loop program above 160 tensors), 1 flat slicing (every
                                    sliced wire is a slice-id bit), 2 loop program: a stem sweep with
                                    local slices summed inside the program and checkpointed segments
                                    that reuse the head across slices (the
                                    head result shared by the tail's local slices).  With 2, n_sliced
                                    is the minimum number of slice-id (global) bits.               */
    int32_t max_segments;        /* loop program: at most this many segments (<= 0: 8)             */
    double persist_budget;       /* loop program: complex elements kept across loop iterations
                                    (checkpointed stems and accumulators; <= 0: 8 x max_tensor_size) */
    const char* plan_path;       /* nullable: import the plan saved by tn_plan_save at this path
                                    instead of searching ("plan file is an explicit,
                                    replayable artifact"); the search options above are ignored    */
} tn_slicing;

typedef struct {
    int32_t s;                   /* number of sliced wires                                    */
    const int32_t* sliced_wires; /* 2*s ints, (q, k) pairs, MSB-first order (owned by ctx)    */
    int64_t n_tensors;           /* tensors after simplification                              */
    int64_t n_steps;             /* pairwise contractions per slice                           */
    int64_t n_launches;          /* kernel launches per slice                                 */
    int64_t peak_elems;          /* largest tensor of one slice, complex elements             */
    int64_t workspace_bytes;     /* device workspace tn_bind_device needs                     */
    double cmac_per_slice;       /* complex multiply-adds per slice (P:L294 T_c convention)   */
    double bytes_per_slice;      /* algorithmic HBM bytes per slice            */
    double gemm_cmac_per_slice;  /* part of cmac_per_slice on the tensor-core GEMM path       */
    int64_t n_invariant_steps;   /* steps with no sliced edge below them: run once per        */
    double invariant_cmac;       /* tn_contract, before the slices (their CMACs)              */
    int32_t n_companions;        /* companion edges cut (tn_slicing.companions)               */
    const int32_t* companion_wires; /* 3*n ints: (q, k, b): Pi_v on wire (q, k) -- right before
                                    the fSim, after its single-qubit gates -- with v = the value of
                                    sliced wire b, counted in sliced_wires and then local_wires
                                    (owned by ctx)                                             */
    double companion_fidelity;   /* prod (1 + sin^2 theta_i)/2 over the companions   */
    int32_t s_local;             /* loop program: local sliced wires, summed inside tn_contract    */
    const int32_t* local_wires;  /* 2*s_local ints, (q, k) pairs, loop-bit order (owned by ctx)   */
    int32_t n_segments;          /* loop program segments (1 for flat slicing)                     */
    double total_cmac;           /* modelled CMAC of a tn_contract over all 2^s slices, with the
                                    loop program's reuse (flat: 2^s * cmac_per_slice + invariant)  */
    int64_t persist_bytes;       /* device bytes kept across loop iterations (per pipeline)        */
} tn_plan_info;

/* tn_plan -- P:L91 (complexity-greedy contraction order), P:L246 (slicing: fix index values so
 * that the space fits the device; the sum over sub-tasks returns the original contraction).
 * info.s / info.sliced_wires are the slice-id (global) wires that tn_contract's slice ids enumerate;
 * a loop program's local wires (info.local_wires) are summed inside every slice, so a slice id of a loop
 * program denotes the sum over all local values (Sigma_v Pi_v = I on those wires).
 * max_tensor_size: bound on every intermediate of one slice, in complex elements (<= 2^60 for planning;
 * tn_bind_device accepts plans whose tensors are <= 2^32 elements).
 * Fills *info (pointers owned by the ctx, valid until the next tn_plan or tn_destroy).
 * EINFEASIBLE if the bound cannot be met; EINVAL if called before tn_build or with bad forced
 * wires. */
tn_status tn_plan(tn_ctx* ctx, const tn_slicing* slicing, int64_t max_tensor_size, tn_plan_info* info);

/* Write the plan (order, sliced wires, per-step shapes, row tables of sparse tensors) as JSON. */
tn_status tn_plan_dump(const tn_ctx* ctx, const char* path);

/* tn_plan_save -- write the current plan as a replayable plan file: the
 * contraction order by tensor id, the sliced wires (q, k) in loop-bit order, the number of global bits
 * and the loop program's segments.  tn_plan with tn_slicing.plan_path = this file reproduces the plan on
 * the same circuit and request (a ctx on another rank or process).  EINVAL before tn_plan or when the
 * file cannot be written. */
tn_status tn_plan_save(const tn_ctx* ctx, const char* path);

/* tn_bind_device -- uploads leaf bank, row maps and the step program, captures the per-slice
 * CUDA graph.  workspace: device pointer of >= info.workspace_bytes (from the caller's allocator,
 * e.g. torch) or NULL to let the library allocate it.  cuda_stream: a cudaStream_t (NULL = the
 * legacy default stream).  EINVAL before tn_plan; ENOMEM if bytes is too small; ECUDA on a CUDA
 * failure. */
tn_status tn_bind_device(tn_ctx* ctx, int device, void* workspace, size_t bytes, void* cuda_stream);

/* tn_contract -- the hot path.  Sums the slices in slice_ids (host array, unique, each < 2^s,
 * any order, executed ascending; "by summing over paths") and writes the M amplitudes, in
 * the caller's bitstring order, to amps_out (M complex64: device pointer if out_on_device, else
 * host).  Multi-GPU: each rank passes its own block and the caller all-reduces the outputs.
 * seconds_out (nullable): device time of the call (CUDA events).  EINVAL on empty / duplicate /
 * out-of-range ids or before tn_bind_device. */
tn_status tn_contract(tn_ctx* ctx, const uint64_t* slice_ids, int64_t n_ids, void* amps_out,
                      int32_t out_on_device, double* seconds_out);

/* Per-launch device times of one slice, for roofline accounting (CUDA events around every
 * launch on the bound stream, no graph).  Loop programs: one pass through every segment at the slice's
 * first local value (a segment's share of a full run is its time x its runs, tn_segment_runs).  Fills up
 * to max_stats entries. */
typedef struct {
    int32_t kind;        /* 0 instantiate, 1 apply (SIMT contraction), 2 gemm pre-pass A,
                            3 gemm pre-pass B, 4 tcgen05 gemm, 5 readout+accumulate, 6 permute,
                            7 fused run of small steps (one persistent launch) */
    int32_t step;        /* pairwise step index (-1 for non-step launches)                    */
    double cmac;         /* complex MACs of the launch                                         */
    double bytes;        /* algorithmic bytes of the launch                                    */
    double ms;           /* measured device time                                               */
    int64_t m, n, k, rows;
    int32_t seg;         /* loop program: segment of the launch (-1: flat program)                */
    int32_t pad;
} tn_launch_stat;
tn_status tn_profile_slice(tn_ctx* ctx, uint64_t slice_id, tn_launch_stat* stats, int32_t max_stats,
                           int32_t* n_stats);

/* tn_segment_runs -- loop programs: how often each segment runs when tn_contract is called with the given
 * slice ids on this ctx's bound pipelines (the executor's own enumeration, without launching anything).
 * runs[j] for j < n_segments (tn_plan_info.n_segments; flat programs: 1 segment = one run per slice).
 * EINVAL before tn_bind_device or on bad ids. */
tn_status tn_segment_runs(tn_ctx* ctx, const uint64_t* slice_ids, int64_t n_ids, int64_t* runs);

/* tn_sample -- host.  One sample per group of l bitstrings: exact categorical
 * draw with weights |a|^2 (frugal within the group), u = top 53 bits of a
 * splitmix64 stream keyed by (seed, group).
 *   amps       : M complex64 from tn_contract (host).
 *   ideal_amps : nullable, M complex64 of the exact state at the same bitstrings (for XEB).
 *   samples_out: L = M / l bitstrings.
 *   est[0] = f = n_slices_summed / 2^s, est[1] = F_norm = (2^n/M) sum |a|^2
 *   (P:L152-L153), est[2] = linear XEB (2^n/L) sum |ideal(s_i)|^2 - 1 or NaN.
 * ENUMERIC on an all-zero group. */
tn_status tn_sample(const tn_ctx* ctx, const float* amps, const float* ideal_amps, int64_t n_slices_summed,
                    uint64_t seed, uint64_t* samples_out, double est[3]);

/* tn_sample_report -- host.  The sampler with a choice of within-group method plus the validation
 * estimators of the paper's supplement.
 *   sampler 0: the categorical draw of tn_sample (frugal within a group).
 *   sampler 1: uniform-proposal Metropolis chain over the group's l indices ("a Markov chain ...
 *              using the Metropolis algorithm"): splitmix64 stream keyed by
 *              (seed, TAG 5), words c = g*(2*steps+1) + t, u_c = top 53 bits * 2^-53; start
 *              x = floor(u_c0 * l); step t proposes y = floor(u_{c0+2t-1} * l) and moves when
 *              u_{c0+2t} * w(x) < w(y), w = |a|^2 in fp64; the sample is the state after `steps` steps
 *              (only the final state is returned, so a burn-in is implicit).  steps >= 1.
 *   index_out (nullable): L indices j into the M requested bitstrings (samples_out[g] = bits[j]).
 *   rep: the estimators below; phat_j = |a_j|^2 / F_norm is the approximate distribution normalised by
 *   the paper's estimate F_norm = (2^n/M) sum |a|^2.  Fields that need ideal_amps are NaN
 *   without them; a zero probability yields +-inf.
 * EINVAL on bad arguments; ENUMERIC on an all-zero group. */
typedef struct {
    double f;                /* n_slices_summed / 2^s                                          */
    double F_norm;           /* (2^n/M) sum_j |a_j|^2                                     */
    double xeb;              /* (2^n/L) sum_i P(s_i) - 1, P = |ideal|^2                    */
    double log_xeb;          /* <ln(2^n P(s_i))> + Euler's gamma ("logarithmic XEB")     */
    double entropy_samples;  /* -<ln phat(s_i)> over the L samples                      */
    double entropy_state;    /* -(2^n/M) sum_j phat_j ln phat_j: the sparse state's distribution        */
    double pt_ks;            /* KS distance of {2^n phat_j} to Exp(1) (Porter-Thomas)          */
} tn_report;
tn_status tn_sample_report(const tn_ctx* ctx, const float* amps, const float* ideal_amps, int64_t n_slices_summed,
                           uint64_t seed, int32_t sampler, int32_t steps, uint64_t* samples_out, int64_t* index_out,
                           tn_report* rep);

void tn_destroy(tn_ctx* ctx);
const char* tn_last_error(const tn_ctx* ctx);
const char* tn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TN_B200_H */
