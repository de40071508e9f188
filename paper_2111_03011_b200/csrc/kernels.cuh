// kernels.cuh -- the bandwidth-bound kernels of one slice.
//
// Index arithmetic: every tensor is [rows][2^d] complex64 with its legs as the bits of the dense
// index.  Bit permutations are evaluated with byte-sliced lookup tables staged in shared memory:
// offset(x) = sum_t tab[t][(x >> 8t) & 255], i.e. a pdep/pext of up to 40 bits in <= 5 LDS + adds.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tnb.h"

namespace tnb {
namespace kern {

__device__ __forceinline__ float2 cmac(float2 acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, acc.x);
    acc.x = fmaf(-a.y, b.y, acc.x);
    acc.y = fmaf(a.x, b.y, acc.y);
    acc.y = fmaf(a.y, b.x, acc.y);
    return acc;
}

// ---------------------------------------------------------------------------- K1: slice instantiate
// (row a2) sigma -> v_j = (sigma >> (s-1-j)) & 1; copies the v-part of every sliced leaf from the bank.
__global__ void k_instantiate(const InstLeafDesc* __restrict__ tab, int n_leaves, int64_t n_items,
                              const float2* __restrict__ bank, char* __restrict__ work,
                              const uint64_t* __restrict__ slice_ids, const int64_t* __restrict__ counter, int s) {
    const uint64_t sigma = slice_ids[*counter];
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        int l = 0;
        while (l + 1 < n_leaves && tab[l + 1].item_begin <= it) l++;
        const InstLeafDesc& d = tab[l];
        const int64_t local = it - d.item_begin;
        const int64_t r = local >> d.d_out;
        const int64_t o = local & (((int64_t)1 << d.d_out) - 1);
        int64_t src = 0;
        for (int b = 0; b < d.d_out; b++)
            if ((o >> b) & 1) src |= (int64_t)1 << d.out_src[b];
        for (int j = 0; j < d.n_sl; j++)
            if ((sigma >> (s - 1 - d.sl_idx[j])) & 1) src |= (int64_t)1 << d.sl_pos[j];
        float2* out = (float2*)(work + d.out_off);
        out[local] = bank[d.bank_off + (r << d.d_full) + src];
    }
}

// ---------------------------------------------------------------------------- K3b/K4: sparse-row apply
// (rows a5, a6) C[r][c] = sum_kk A[ma[r]][offA(c,kk)] * B[mb[r]][offB(c,kk)].
// A "team" of TEAM threads owns one orbit (a C index with its NI inner bits free): each member sums a
// strided share of kk for the 2^NI outputs, then the team reduces with warp shuffles (deterministic).
struct ApplyDev {
    const float2* A;
    const float2* B;
    float2* C;
    const int32_t* ma;
    const int32_t* mb;
    int64_t R, a_row, b_row, c_row, n_orbits;
    const uint32_t* tab;   // [ntab][256][4] = (c_off, a_off, b_off, 0) of the orbit index bytes
    const uint32_t* ktab;  // [2^nk][2] = (a_off, b_off) of kk, when nk <= KTAB_MAX_BITS
    int ntab, nk;
    int8_t kA[40], kB[40];
    uint32_t inner_c[16], inner_b[16];
    int stage_b;           // 1: a 256-thread chunk lies in one output row; B's row is staged in smem
    int kparts;            // k_apply_rows: lanes sharing one orbit (power of two <= 32)
    uint32_t a_extra[4], c_extra[4];  // k_apply_na: offsets of the per-thread A-free C bits
    const int32_t* rperm;  // output rows in processing order (grouped by A parent, so that re-reads of a shared
                           // A row hit L2); null = ascending
};
constexpr int KTAB_MAX_BITS = 12;
constexpr int STAGE_B_MAX = 4096;  // complex elements of B per row staged in shared memory
constexpr int RG_SMEM_MAX = 100 * 1024;   // k_apply_rg: B row (<= 8192 complex) + tables + reduction buffer
constexpr int ROWS_SMEM_MAX = 112 * 1024;  // k_apply_rows: tables + both parent rows in shared memory (>= 2 CTAs/SM)

#ifndef TNB_APPLY_MINB
#define TNB_APPLY_MINB 3  // 3 CTAs per SM (<= 80 registers): measured 2544 vs 2385 slices/s with 2
#endif
// the 16-output warp-team variant needs more than 80 registers (it spilled 108 B at 3 CTAs/SM): 2 CTAs/SM
template <int NI, int TEAM>
__global__ void __launch_bounds__(256, (NI == 4 && TEAM == 32) ? 2 : TNB_APPLY_MINB) k_apply(const ApplyDev p) {
    extern __shared__ uint32_t sm[];
    const int tabn = p.ntab * 256 * 4;
    for (int i = threadIdx.x; i < tabn; i += blockDim.x) sm[i] = p.tab[i];
    uint32_t* sk = sm + tabn;
    const bool has_ktab = p.ktab != nullptr;
    if (has_ktab) {
        const int kn = 2 << p.nk;
        for (int i = threadIdx.x; i < kn; i += blockDim.x) sk[i] = p.ktab[i];
    }
    __syncthreads();
    const int64_t K = (int64_t)1 << p.nk;
    const int lane = (TEAM == 1) ? 0 : (threadIdx.x & (TEAM - 1));
    const int64_t total = p.R * p.n_orbits;
    if (p.stage_b) {
        // chunked loop: chunk c covers teams [c*256/TEAM, (c+1)*256/TEAM), all in one output row
        float2* sB = (float2*)(sk + (has_ktab ? (2 << p.nk) : 0));
        const int64_t per = 256 / TEAM;
        const int64_t nchunks = total / per;
        const int64_t span = (nchunks + gridDim.x - 1) / gridDim.x;  // contiguous chunks per block
        const int64_t ch0 = blockIdx.x * span, ch1 = ch0 + span < nchunks ? ch0 + span : nchunks;
        int64_t cached = -1;
        for (int64_t ch = ch0; ch < ch1; ch++) {
            const int64_t w = ch * per + threadIdx.x / TEAM;
            const int64_t r0 = w / p.n_orbits;
            const int64_t r = p.rperm ? (int64_t)p.rperm[r0] : r0;
            const int64_t rb = p.mb ? (int64_t)p.mb[r] : 0;
            if (rb != cached) {
                __syncthreads();
                const float2* src = p.B + rb * p.b_row;
                for (int i = threadIdx.x; i < p.b_row; i += blockDim.x) sB[i] = src[i];
                __syncthreads();
                cached = rb;
            }
            const int64_t o = w - r0 * p.n_orbits;
            uint32_t coff = 0, aoff = 0, boff = 0;
            for (int t = 0; t < p.ntab; t++) {
                const uint32_t* e = sm + ((t << 8) + (int)((o >> (8 * t)) & 255)) * 4;
                coff += e[0];
                aoff += e[1];
                boff += e[2];
            }
            const int64_t ra = p.ma ? (int64_t)p.ma[r] : r;
            const float2* __restrict__ Ar = p.A + ra * p.a_row + aoff;
            const float2* Br = sB + boff;
            float2 acc[1 << NI];
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) acc[ii] = make_float2(0.f, 0.f);
            // unrolled so several iterations' A loads are in flight (the loop is long-scoreboard bound)
#pragma unroll 4
            for (int64_t kk = lane; kk < K; kk += TEAM) {
                const uint32_t ka = sk[2 * kk], kb = sk[2 * kk + 1];
                const float2 a = Ar[ka];
#pragma unroll
                for (int ii = 0; ii < (1 << NI); ii++) acc[ii] = cmac(acc[ii], a, Br[kb + p.inner_b[ii]]);
            }
            if (TEAM > 1) {
#pragma unroll
                for (int ii = 0; ii < (1 << NI); ii++) {
#pragma unroll
                    for (int sh = TEAM / 2; sh >= 1; sh >>= 1) {
                        acc[ii].x += __shfl_xor_sync(0xffffffffu, acc[ii].x, sh);
                        acc[ii].y += __shfl_xor_sync(0xffffffffu, acc[ii].y, sh);
                    }
                }
            }
            if (lane == 0) {
                float2* Cr = p.C + r * p.c_row + coff;
#pragma unroll
                for (int ii = 0; ii < (1 << NI); ii++) Cr[p.inner_c[ii]] = acc[ii];
            }
        }
        return;
    }
    const int64_t team0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TEAM;
    const int64_t nteams = ((int64_t)gridDim.x * blockDim.x) / TEAM;
    for (int64_t w = team0; w < total; w += nteams) {
        const int64_t r0 = w / p.n_orbits;
        const int64_t o = w - r0 * p.n_orbits;
        const int64_t r = p.rperm ? (int64_t)p.rperm[r0] : r0;
        uint32_t coff = 0, aoff = 0, boff = 0;
        for (int t = 0; t < p.ntab; t++) {
            const uint32_t* e = sm + ((t << 8) + (int)((o >> (8 * t)) & 255)) * 4;
            coff += e[0];
            aoff += e[1];
            boff += e[2];
        }
        const int64_t ra = p.ma ? (int64_t)p.ma[r] : r;
        const int64_t rb = p.mb ? (int64_t)p.mb[r] : 0;
        const float2* __restrict__ Ar = p.A + ra * p.a_row + aoff;
        const float2* __restrict__ Br = p.B + rb * p.b_row + boff;
        float2 acc[1 << NI];
#pragma unroll
        for (int ii = 0; ii < (1 << NI); ii++) acc[ii] = make_float2(0.f, 0.f);
        for (int64_t kk = lane; kk < K; kk += TEAM) {
            uint32_t ka, kb;
            if (has_ktab) {
                ka = sk[2 * kk];
                kb = sk[2 * kk + 1];
            } else {
                ka = 0;
                kb = 0;
                for (int t = 0; t < p.nk; t++)
                    if ((kk >> t) & 1) {
                        ka += 1u << p.kA[t];
                        kb += 1u << p.kB[t];
                    }
            }
            const float2 a = Ar[ka];
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) acc[ii] = cmac(acc[ii], a, Br[kb + p.inner_b[ii]]);
        }
        if (TEAM > 1) {
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) {
#pragma unroll
                for (int sh = TEAM / 2; sh >= 1; sh >>= 1) {
                    acc[ii].x += __shfl_xor_sync(0xffffffffu, acc[ii].x, sh);
                    acc[ii].y += __shfl_xor_sync(0xffffffffu, acc[ii].y, sh);
                }
            }
        }
        if (lane == 0) {
            float2* Cr = p.C + r * p.c_row + coff;
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) Cr[p.inner_c[ii]] = acc[ii];
        }
    }
}

// ---------------------------------------------------------------------------- register-blocked apply
// (row a5) as k_apply with TEAM = 1, but every thread owns 2^NA orbits that differ only in A-free bits
// (above the lane bits, so loads stay coalesced): each B value loaded feeds 2^NA x more FMAs.
template <int NI, int NA>
__global__ void __launch_bounds__(256) k_apply_na(const ApplyDev p) {
    extern __shared__ uint32_t sm[];
    const int tabn = p.ntab * 256 * 4;
    for (int i = threadIdx.x; i < tabn; i += blockDim.x) sm[i] = p.tab[i];
    uint32_t* sk = sm + tabn;
    const int kn = 2 << p.nk;
    for (int i = threadIdx.x; i < kn; i += blockDim.x) sk[i] = p.ktab[i];
    __syncthreads();
    const int64_t K = (int64_t)1 << p.nk;
    const int64_t total = p.R * p.n_orbits;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r0 = w / p.n_orbits;
        const int64_t o = w - r0 * p.n_orbits;
        const int64_t r = p.rperm ? (int64_t)p.rperm[r0] : r0;
        uint32_t coff = 0, aoff = 0, boff = 0;
        for (int t = 0; t < p.ntab; t++) {
            const uint32_t* e = sm + ((t << 8) + (int)((o >> (8 * t)) & 255)) * 4;
            coff += e[0];
            aoff += e[1];
            boff += e[2];
        }
        const int64_t ra = p.ma ? (int64_t)p.ma[r] : r;
        const int64_t rb = p.mb ? (int64_t)p.mb[r] : 0;
        const float2* __restrict__ Ar = p.A + ra * p.a_row + aoff;
        const float2* __restrict__ Br = p.B + rb * p.b_row + boff;
        float2 acc[1 << NA][1 << NI];
#pragma unroll
        for (int j = 0; j < (1 << NA); j++)
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) acc[j][ii] = make_float2(0.f, 0.f);
        for (int64_t kk = 0; kk < K; kk++) {
            const uint32_t ka = sk[2 * kk], kb = sk[2 * kk + 1];
            float2 a[1 << NA];
#pragma unroll
            for (int j = 0; j < (1 << NA); j++) a[j] = Ar[ka + p.a_extra[j]];
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) {
                const float2 b = Br[kb + p.inner_b[ii]];
#pragma unroll
                for (int j = 0; j < (1 << NA); j++) acc[j][ii] = cmac(acc[j][ii], a[j], b);
            }
        }
        float2* Cr = p.C + r * p.c_row + coff;
#pragma unroll
        for (int j = 0; j < (1 << NA); j++)
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) Cr[p.c_extra[j] + p.inner_c[ii]] = acc[j][ii];
    }
}

// ---------------------------------------------------------------------------- row-staged gather-contract
// (row a6, GATHER-CONTRACT with small rows) one block per output row r: both parent rows A[ma[r]] and
// B[mb[r]] are copied to shared memory with coalesced loads, then every output of the row is computed from
// shared memory (any bit layout); `kparts` lanes split k for one orbit and reduce with shuffles.
template <int NI>
__global__ void __launch_bounds__(256) k_apply_rows(const ApplyDev p) {
    extern __shared__ uint32_t sm[];
    const int tabn = p.ntab * 256 * 4;
    for (int i = threadIdx.x; i < tabn; i += blockDim.x) sm[i] = p.tab[i];
    uint32_t* sk = sm + tabn;
    const int kn = 2 << p.nk;
    for (int i = threadIdx.x; i < kn; i += blockDim.x) sk[i] = p.ktab[i];
    float2* sA = (float2*)(sk + kn);
    float2* sB = sA + p.a_row;
    const int64_t K = (int64_t)1 << p.nk;
    const int kparts = p.kparts;
    const int64_t total_w = p.n_orbits * kparts;
    for (int64_t r0 = blockIdx.x; r0 < p.R; r0 += gridDim.x) {
        const int64_t r = p.rperm ? (int64_t)p.rperm[r0] : r0;
        __syncthreads();
        const float2* Ag = p.A + (p.ma ? (int64_t)p.ma[r] : r) * p.a_row;
        const float2* Bg = p.B + (p.mb ? (int64_t)p.mb[r] : 0) * p.b_row;
        for (int64_t i = threadIdx.x; i < p.a_row; i += blockDim.x) sA[i] = Ag[i];
        for (int64_t i = threadIdx.x; i < p.b_row; i += blockDim.x) sB[i] = Bg[i];
        __syncthreads();
        float2* Cr = p.C + r * p.c_row;
        for (int64_t base = 0; base < total_w; base += blockDim.x) {
            const int64_t w = base + threadIdx.x;
            const bool valid = w < total_w;
            const int64_t o = valid ? w / kparts : 0;
            const int kp = (int)(w % kparts);
            uint32_t coff = 0, aoff = 0, boff = 0;
            for (int t = 0; t < p.ntab; t++) {
                const uint32_t* e = sm + ((t << 8) + (int)((o >> (8 * t)) & 255)) * 4;
                coff += e[0];
                aoff += e[1];
                boff += e[2];
            }
            float2 acc[1 << NI];
#pragma unroll
            for (int ii = 0; ii < (1 << NI); ii++) acc[ii] = make_float2(0.f, 0.f);
            if (valid) {
                for (int64_t kk = kp; kk < K; kk += kparts) {
                    const float2 a = sA[aoff + sk[2 * kk]];
                    const uint32_t kb = boff + sk[2 * kk + 1];
#pragma unroll
                    for (int ii = 0; ii < (1 << NI); ii++) acc[ii] = cmac(acc[ii], a, sB[kb + p.inner_b[ii]]);
                }
            }
            for (int sh = kparts >> 1; sh >= 1; sh >>= 1) {
#pragma unroll
                for (int ii = 0; ii < (1 << NI); ii++) {
                    acc[ii].x += __shfl_xor_sync(0xffffffffu, acc[ii].x, sh);
                    acc[ii].y += __shfl_xor_sync(0xffffffffu, acc[ii].y, sh);
                }
            }
            if (valid && kp == 0) {
#pragma unroll
                for (int ii = 0; ii < (1 << NI); ii++) Cr[coff + p.inner_c[ii]] = acc[ii];
            }
        }
    }
}

// ---------------------------------------------------------------------------- tiny-step chains
// A run of consecutive tiny contraction steps (<= 256 work items each: leaf cones absorbing gates one at a
// time) executed by ONE CTA in program order.  Dependencies (RAW / WAR / WAW on workspace buffers) become
// __syncthreads before the dependent step; operands are read with ld.global.cg (L2) and written with
// st.global.cg because the run reuses workspace buffers.
constexpr int MULTI_MAX_DEPS = 8;
constexpr int CHAIN_MAX_STEPS = 64;    // steps per k_chain launch (descriptors staged in smem)
constexpr int CHAIN_SMEM_MAX = 160 * 1024;  // run-internal intermediates kept in k_chain's shared memory
struct MStep {
    const float2* A;
    const float2* B;
    float2* C;
    const int32_t* ma;
    const int32_t* mb;
    int64_t a_row, b_row, c_row, n_orbits, total;
    int nk, ni, ndep, barrier, nob;  // barrier: k_chain syncs the CTA before this step
    int a_sm, b_sm, c_sm;            // >= 0: the operand lives in the chain's shared memory at this float2 offset
    int a_pre, b_pre;                // > 0: preload this many elements of A / B from global at kernel start
    int dep[MULTI_MAX_DEPS];
    uint32_t inner_c[16], inner_b[16];
    // per-bit offsets (no table lookups on the chain's critical path): orbit bit t -> (C, A, B) offsets,
    // contracted bit t -> (A, B) offsets
    uint32_t ob_c[8], ob_a[8], ob_b[8];
    uint32_t kb_a[12], kb_b[12];
};

// one work item (output orbit w) of a fused tiny step: offsets from per-bit sums (XOR of disjoint bits)
// instead of table lookups on the chain's critical path
__device__ __forceinline__ void multi_item(const MStep& S, int64_t w, float2* sm) {
    const int64_t r = w >> S.nob;
    const uint32_t o = (uint32_t)(w & ((1 << S.nob) - 1));
    const int64_t ra = S.ma ? (int64_t)__ldg(S.ma + r) : r;
    const int64_t rb = S.mb ? (int64_t)__ldg(S.mb + r) : 0;
    uint32_t coff = 0, aoff = 0, boff = 0;
    for (int t = 0; t < S.nob; t++)
        if ((o >> t) & 1) {
            coff ^= S.ob_c[t];
            aoff ^= S.ob_a[t];
            boff ^= S.ob_b[t];
        }
    const bool a_sm = S.a_sm >= 0, b_sm = S.b_sm >= 0;  // uniform per step
    const float2* Ar = (a_sm ? sm + S.a_sm : S.A) + ra * S.a_row + aoff;
    const float2* Br = (b_sm ? sm + S.b_sm : S.B) + rb * S.b_row + boff;
    const int nout = 1 << S.ni;
    const int64_t K = (int64_t)1 << S.nk;
    float2 acc[16];
#pragma unroll
    for (int ii = 0; ii < 16; ii++) acc[ii] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int64_t i = 0; i < K; i++) {
        // offsets of contraction index i from its bits: independent across iterations, so the unrolled
        // loads of several iterations are in flight together
        uint32_t ka = 0, kb = 0;
        for (int t = 0; t < S.nk; t++)
            if ((i >> t) & 1) {
                ka ^= S.kb_a[t];
                kb ^= S.kb_b[t];
            }
        const float2 a = a_sm ? Ar[ka] : __ldcg(Ar + ka);
#pragma unroll
        for (int ii = 0; ii < 16; ii++)
            if (ii < nout) {
                const float2* bp = Br + kb + S.inner_b[ii];
                acc[ii] = cmac(acc[ii], a, b_sm ? *bp : __ldcg(bp));
            }
    }
    const bool c_sm = S.c_sm >= 0;
    float2* Cr = (c_sm ? sm + S.c_sm : S.C) + r * S.c_row + coff;
#pragma unroll
    for (int ii = 0; ii < 16; ii++)
        if (ii < nout) {
            if (c_sm)
                Cr[S.inner_c[ii]] = acc[ii];
            else
                __stcg(Cr + S.inner_c[ii], acc[ii]);
        }
}

// A run of tiny steps (<= 256 work items each) executed by ONE CTA in program order: no cross-CTA
// synchronisation; a __syncthreads only before a step that depends on a step issued since the previous
// barrier (S.barrier, host-computed from the run's hazards), so independent neighbours overlap.
__global__ void __launch_bounds__(256) k_chain(const MStep* __restrict__ steps, int nsteps) {
    // the run's descriptors live in smem: the item loop reads table pointers / offsets with LDS, not with a
    // chain of dependent global loads per output
    __shared__ MStep sS[CHAIN_MAX_STEPS];
    extern __shared__ float2 chain_sm[];  // run-internal intermediates (host-assigned offsets)
    {
        const int words = nsteps * (int)(sizeof(MStep) / 4);
        const uint32_t* src = (const uint32_t*)steps;
        uint32_t* dst = (uint32_t*)sS;
        for (int i = threadIdx.x; i < words; i += 256) dst[i] = src[i];
    }
    __syncthreads();
#ifdef TNB_CHAIN_CLOCK
    long long t_prev = clock64();
    if (threadIdx.x == 0) printf("[chain] start nsteps %d\n", nsteps);
#endif
    // preload the run's external operands (one memory latency for the whole run)
    for (int s = 0; s < nsteps; s++) {
        const MStep& S = sS[s];
        for (int e = threadIdx.x; e < S.a_pre; e += 256) chain_sm[S.a_sm + e] = __ldcg(S.A + e);
        for (int e = threadIdx.x; e < S.b_pre; e += 256) chain_sm[S.b_sm + e] = __ldcg(S.B + e);
    }
    __syncthreads();
#ifdef TNB_CHAIN_CLOCK
    if (threadIdx.x == 0) {
        const long long t = clock64();
        printf("[chain] descriptors+preload %lld cycles\n", t - t_prev);
        t_prev = t;
    }
#endif
    for (int s = 0; s < nsteps; s++) {
        const MStep& S = sS[s];
        if (S.barrier) __syncthreads();
#ifdef TNB_CHAIN_CLOCK
        if (threadIdx.x == 0) {
            const long long t = clock64();
            printf("[chain] step %d items %lld nk %d ni %d a_sm %d b_sm %d c_sm %d barrier %d: %lld cycles since last\n", s,
                   (long long)S.total, S.nk, S.ni, S.a_sm, S.b_sm, S.c_sm, S.barrier, t - t_prev);
            t_prev = t;
        }
#endif
        for (int64_t w = threadIdx.x; w < S.total; w += 256) multi_item(S, w, chain_sm);
    }
}

// ---------------------------------------------------------------------------- row GEMM (rows a5/a6)
// Gather-contract with long k and few outputs per row:
//   C[r][cA(i) + cB(j)] = sum_kk A[ma[r]][aK(kk) + aF(i)] * B[mb[r]][bK(kk) + bF(j)]
// One CTA per output row: B's row is staged in shared memory (XOR-swizzled so that the lanes' B
// addresses hit distinct banks), A's row is streamed once from HBM with lanes walking A's lowest
// contracted bits (full sectors).  Thread group g (2^G groups of 256/2^G threads) owns the A-free
// combos [g*2^FAT, (g+1)*2^FAT); every thread accumulates its 2^FAT x 2^FB outputs over its share
// of k, then a recursive-halving warp reduction and a shared-memory sum over the group's warps.
struct RowGemmDev {
    const float2* A;
    const float2* B;
    float2* C;
    const int32_t* ma;
    const int32_t* mb;
    int64_t R, a_row, b_row, c_row;
    const uint32_t* ktab;  // [2^nk][2] = (A offset, swizzled B offset), kk bit t = t-th lowest A k-bit
    const uint32_t* ftab;  // [2^fa][2] = (A offset, C offset) of the A-free combos, then [2^FB][2] = (swz B, C)
    int nk, fa, g;
    int nswz;
    int swz_src[4], swz_dst[4];  // B staging swizzle: bit dst of the smem index ^= bit src
    const int32_t* rperm;        // output rows in processing order (null = ascending)
};

template <int FAT, int FB>
__global__ void __launch_bounds__(256, 2) k_apply_rg(const RowGemmDev p) {
    constexpr int NA = 1 << FAT, NB = 1 << FB, NV = NA * NB;
    static_assert(NV <= 32, "at most 32 complex accumulators per thread");
    extern __shared__ __align__(16) float2 smf[];
    float2* sB = smf;
    uint32_t* sK = (uint32_t*)(sB + p.b_row);
    const int kn = 2 << p.nk;
    uint32_t* sF = sK + kn;
    const int fn = (2 << p.fa) + 2 * NB;
    float2* red = (float2*)(sF + fn);  // [8 warps][NV]
    for (int i = threadIdx.x; i < kn; i += 256) sK[i] = p.ktab[i];
    for (int i = threadIdx.x; i < fn; i += 256) sF[i] = p.ftab[i];
    const int tpg = 256 >> p.g;
    const int grp = threadIdx.x / tpg, tg = threadIdx.x % tpg;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int K = 1 << p.nk;
    for (int64_t r0 = blockIdx.x; r0 < p.R; r0 += gridDim.x) {
        const int64_t r = p.rperm ? (int64_t)p.rperm[r0] : r0;
        const int64_t ra = p.ma ? (int64_t)p.ma[r] : r;
        const int64_t rb = p.mb ? (int64_t)p.mb[r] : 0;
        __syncthreads();  // the previous row is done with sB / red (and the tables are loaded)
        {
            const float4* src = (const float4*)(p.B + rb * p.b_row);
            for (int i = threadIdx.x; i < (int)(p.b_row >> 1); i += 256) {
                const float4 v = __ldg(src + i);
                int e = 2 * i, x = 0;
                for (int t = 0; t < p.nswz; t++) x |= ((e >> p.swz_src[t]) & 1) << p.swz_dst[t];
                // swizzle sources are bits >= 4, so e and e + 1 share x
                sB[e ^ x] = make_float2(v.x, v.y);
                sB[(e + 1) ^ x] = make_float2(v.z, v.w);
            }
        }
        __syncthreads();
        uint32_t aoff[NA], boff[NB];
#pragma unroll
        for (int i = 0; i < NA; i++) aoff[i] = sF[2 * ((grp << FAT) + i)];
#pragma unroll
        for (int j = 0; j < NB; j++) boff[j] = sF[(2 << p.fa) + 2 * j];
        const float2* __restrict__ Ar = p.A + ra * p.a_row;
        float2 acc[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int kk = tg; kk < K; kk += tpg) {
            const uint32_t ka = sK[2 * kk], kb = sK[2 * kk + 1];
            float2 a[NA], b[NB];
#pragma unroll
            for (int i = 0; i < NA; i++) a[i] = __ldg(Ar + ka + aoff[i]);
#pragma unroll
            for (int j = 0; j < NB; j++) b[j] = sB[kb ^ boff[j]];
#pragma unroll
            for (int i = 0; i < NA; i++)
#pragma unroll
                for (int j = 0; j < NB; j++) acc[i * NB + j] = cmac(acc[i * NB + j], a[i], b[j]);
        }
        // recursive halving over the lanes: after level l the lane keeps half of its values
        int base = 0;
#pragma unroll
        for (int l = 0; l < 5; l++) {
            const int o = 16 >> l;
            const int H = NV >> (l + 1);
            if (H >= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < (NV >> 1); i++) {
                    if (i < H) {
                        const float2 lo = acc[i], hi = acc[i + H];
                        float2 snd = up ? lo : hi;
                        const float2 keep = up ? hi : lo;
                        snd.x = __shfl_xor_sync(0xffffffffu, snd.x, o);
                        snd.y = __shfl_xor_sync(0xffffffffu, snd.y, o);
                        acc[i] = make_float2(keep.x + snd.x, keep.y + snd.y);
                    }
                }
                if (up) base += H;
            } else {
                acc[0].x += __shfl_xor_sync(0xffffffffu, acc[0].x, o);
                acc[0].y += __shfl_xor_sync(0xffffffffu, acc[0].y, o);
            }
        }
        constexpr int VPL = NV >= 32 ? NV / 32 : 1;  // values per lane after the halving
        const bool writer = NV >= 32 || (lane & ((32 / NV) - 1)) == 0;
        if (writer) {
#pragma unroll
            for (int i = 0; i < VPL; i++) red[warp * NV + base + i] = acc[i];
        }
        __syncthreads();
        const int wpg = tpg >> 5;
        for (int t = threadIdx.x; t < (NV << p.g); t += 256) {
            const int gg = t / NV, o = t % NV;
            float2 sum = make_float2(0.f, 0.f);
            for (int u = 0; u < wpg; u++) {
                const float2 x = red[(gg * wpg + u) * NV + o];
                sum.x += x.x;
                sum.y += x.y;
            }
            const int ia = (gg << FAT) + o / NB, jb = o % NB;
            p.C[r * p.c_row + sF[2 * ia + 1] + sF[(2 << p.fa) + 2 * jb + 1]] = sum;
        }
    }
}

// ---------------------------------------------------------------------------- GEMM pre-passes (row a3)
// permute to K-major + 3xTF32 split: hi = cvt.rna.tf32(x), lo = x - hi
__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

struct PrepADev {
    const float2* A;
    const int32_t* ma;
    float2* hi;            // [Mp][K] float2 (plain) or [2Mp][K] float2 (embedded)
    float2* lo;
    int64_t Mp, K, a_row;
    int log2m, log2k;
    const uint32_t* tab;   // [ntm + ntk][256]: A offsets of m-index bytes, then of k-index bytes
    int ntm, ntk;
    int embed;
};

struct PrepBDev {
    const float2* B;
    float2* hi;   // [2N][K] float2 = [2N][2K] fp32 (embedded) or [N][K] float2 (plain)
    float2* lo;
    int64_t N, K;
    int log2k;
    const uint32_t* tab;  // [ntn + ntk][256]
    int ntn, ntk;
    int embed;
    const int32_t* rowsel;  // grouped GEMM: B row of gathered block p = nn >> log2n (else null)
    int64_t b_row;
    int log2n;
};

// Tiled pre-pass (both GEMM operands): out[r][x][k] (K-major, hi/lo split, optionally embedded) =
// src[rowmap(r)][pi(x, k)] for a bit permutation pi.  One CTA per tile: the tile spans the source's and the
// output's lowest bits (<= 2^10 elements), read coalesced from the source into a swizzled smem tile,
// written coalesced in output order.  Embedding (the operand on the embedded side of the complex-as-real
// GEMM): rows 2x = (re, -im), 2x+1 = (im, re) along K.
struct PrepTDev {
    const float2* src;
    const int32_t* rowmap;   // source row of output row r (null: r)
    float2* hi;
    float2* lo;
    int64_t R, src_row;      // output rows, source row stride (elements)
    int log2_row, log2k;     // output bits per row (x and k bits), k bits
    int n_tile;              // tile bits |S|
    const uint2* tin;        // [2^n_tile]: (smem slot, source offset), source order
    const uint32_t* tout;    // [2^n_tile]: output offset, output order (slot = index)
    const uint2* outer;      // [nto][256]: outer index byte -> (source offset, output offset)
    int nto;
    int embed;
    int pairs;               // 16-byte loads / stores of element pairs (tile >= 2 elements, K >= 2)
};

__device__ __forceinline__ int prep_swz(int slot) { return slot ^ (((slot >> 4) ^ (slot >> 8)) & 15); }

__global__ void __launch_bounds__(256) k_prep_t(const PrepTDev p) {
    __shared__ float2 tile[1024];
    const int tn = 1 << p.n_tile;
    const int64_t n_outer = (int64_t)1 << (p.log2_row - p.n_tile);
    const int64_t K = (int64_t)1 << p.log2k;
    for (int64_t blk = blockIdx.x; blk < p.R * n_outer; blk += gridDim.x) {
        const int64_t r = blk >> (p.log2_row - p.n_tile);
        const int64_t o = blk & (n_outer - 1);
        uint32_t so = 0, oo = 0;
        for (int t = 0; t < p.nto; t++) {
            const uint2 e = __ldg(p.outer + (t << 8) + (int)((o >> (8 * t)) & 255));
            so += e.x;
            oo += e.y;
        }
        const int64_t sr = p.rowmap ? (int64_t)__ldg(p.rowmap + r) : r;
        const float2* __restrict__ src = p.src + sr * p.src_row + so;
        if (p.pairs) {
            // source-order pairs (2e, 2e+1) differ in source bit 0, output-order pairs in output bit 0:
            // 16-byte loads and stores
            for (int e = 2 * threadIdx.x; e < tn; e += 512) {
                const uint2 t = __ldg(p.tin + e);
                const float4 v = __ldg((const float4*)(src + t.y));
                const uint2 t1 = __ldg(p.tin + e + 1);
                tile[prep_swz((int)t.x)] = make_float2(v.x, v.y);
                tile[prep_swz((int)t1.x)] = make_float2(v.z, v.w);
            }
        } else {
            for (int e = threadIdx.x; e < tn; e += 256) {
                const uint2 t = __ldg(p.tin + e);
                tile[prep_swz((int)t.x)] = __ldg(src + t.y);
            }
        }
        __syncthreads();
        const int64_t obase = (r << p.log2_row) + oo;
        if (p.pairs) {
            for (int e = 2 * threadIdx.x; e < tn; e += 512) {
                const float2 v0 = tile[prep_swz(e)], v1 = tile[prep_swz(e + 1)];
                const int64_t it = obase + __ldg(p.tout + e);
                const float4 h = make_float4(tf32_hi(v0.x), tf32_hi(v0.y), tf32_hi(v1.x), tf32_hi(v1.y));
                const float4 l = make_float4(v0.x - h.x, v0.y - h.y, v1.x - h.z, v1.y - h.w);
                if (!p.embed) {
                    *(float4*)(p.hi + it) = h;
                    *(float4*)(p.lo + it) = l;
                } else {
                    const int64_t x = it >> p.log2k, kk = it & (K - 1);
                    const int64_t i0 = (2 * x) * K + kk, i1 = i0 + K;
                    *(float4*)(p.hi + i0) = make_float4(h.x, -h.y, h.z, -h.w);
                    *(float4*)(p.lo + i0) = make_float4(l.x, -l.y, l.z, -l.w);
                    *(float4*)(p.hi + i1) = make_float4(h.y, h.x, h.w, h.z);
                    *(float4*)(p.lo + i1) = make_float4(l.y, l.x, l.w, l.z);
                }
            }
        } else {
            for (int e = threadIdx.x; e < tn; e += 256) {
                const float2 v = tile[prep_swz(e)];
                const int64_t it = obase + __ldg(p.tout + e);
                const float2 h = make_float2(tf32_hi(v.x), tf32_hi(v.y));
                const float2 l = make_float2(v.x - h.x, v.y - h.y);
                if (!p.embed) {
                    p.hi[it] = h;
                    p.lo[it] = l;
                } else {
                    const int64_t x = it >> p.log2k, kk = it & (K - 1);
                    const int64_t i0 = (2 * x) * K + kk, i1 = i0 + K;
                    p.hi[i0] = make_float2(h.x, -h.y);
                    p.lo[i0] = make_float2(l.x, -l.y);
                    p.hi[i1] = make_float2(h.y, h.x);
                    p.lo[i1] = make_float2(l.y, l.x);
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------- K4 readout + K5 accumulate
// (rows a6 iii, a7) acc[j] += F[idx[j]] in fp64, ascending slice order per GPU; the last slice kernel
// advances the device slice counter.
__global__ void k_readout(const float2* __restrict__ F, const int64_t* __restrict__ idx, double2* __restrict__ acc,
                          int64_t M, int64_t* __restrict__ counter) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = F[idx[j]];
        double2 a = acc[j];
        a.x += (double)v.x;
        a.y += (double)v.y;
        acc[j] = a;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *counter += 1;
}

// Loop program (local slices): dst = src on the first value of the summed bits E of tau, else
// dst + src.  Elementwise over n complex64 values (float4 = two complex values per thread step).
__global__ void k_accum(const float2* __restrict__ src, float2* __restrict__ dst, int64_t n,
                        const uint64_t* __restrict__ tau, uint64_t E) {
    const bool first = (*tau & E) == 0;
    const int64_t n2 = n >> 1;
    const float4* s4 = (const float4*)src;
    float4* d4 = (float4*)dst;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        float4 v = s4[i];
        if (!first) {
            const float4 a = d4[i];
            v.x += a.x;
            v.y += a.y;
            v.z += a.z;
            v.w += a.w;
        }
        d4[i] = v;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        float2 v = src[n - 1];
        if (!first) {
            v.x += dst[n - 1].x;
            v.y += dst[n - 1].y;
        }
        dst[n - 1] = v;
    }
}

__global__ void k_set_tau(uint64_t* __restrict__ tau, uint64_t v) { *tau = v; }

__global__ void k_finalize(const double2* __restrict__ acc, float2* __restrict__ out, int64_t M) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = make_float2((float)acc[j].x, (float)acc[j].y);
}

}  // namespace kern
}  // namespace tnb
