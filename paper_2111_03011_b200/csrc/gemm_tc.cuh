// gemm_tc.cuh -- complex64 pairwise contraction on the 5th-gen tensor cores.
//
// The complex GEMM C = A B (complex64, C[m][n] = sum_k A[m][k] B[k][n]) is run as one real GEMM via
// the complex-as-real embedding:
//   A_real [Mp][2K] = A interleaved (re, im) along K         (K-major as stored)
//   Bt     [2N][2K] : row 2n = (br, -bi) pairs, row 2n+1 = (bi, br) pairs along K   (K-major)
//   C_real [Mp][2N] = A_real Bt^T  = complex C interleaved.
// 3xTF32 keeps fp32-level accuracy on the TF32 tensor cores:
//   x = hi + lo, hi = cvt.rna.tf32(x), lo = x - hi;  C = Ahi Bhi + Ahi Blo + Alo Bhi  (lo*lo dropped),
// all three products accumulated in one fp32 TMEM accumulator.
//
// Kernel anatomy (sm_100a): persistent, one CTA per SM, 192 threads, 128x128 output tiles.
//   warp 0 / lane 0 : TMA producer (cp.async.bulk.tensor, SWIZZLE_128B) into a 3-stage smem ring,
//                     four 128x32 fp32 tiles per stage (Ahi, Alo, Bhi, Blo), mbarrier full/empty.
//   warp 1 / lane 0 : MMA issuer, tcgen05.mma.cta_group::1.kind::tf32 M=128 N=128 K=8, 12 per stage,
//                     tcgen05.commit -> smem empty barrier; after a tile -> TMEM-full barrier.
//   warps 2-5       : epilogue, tcgen05.ld 32x32b (TMEM lane quarter = warp % 4) -> registers -> global,
//                     then arrive on the TMEM-empty barrier.  The accumulator is double-buffered in TMEM
//                     (2 x 128 columns), so the epilogue of tile i overlaps the MMAs of tile i+1.
// CTA-pair variant (CG = 2, clusters of 2 CTAs on one TPC): the pair computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (M = 256) issued by the leader CTA.  Each CTA TMA-loads its own 128 A rows and
// half of the B tile (BN/2 rows), completing on the leader's full barrier; the leader's MMA commits are
// multicast to both CTAs' empty / TMEM-full barriers, and both CTAs' epilogue warps arrive on the leader's
// TMEM-empty barrier.  Per SM this halves the operand bytes per output at BN = 256 (the GEMMs here are
// L2->SMEM bandwidth bound); BN = 256 uses one accumulator per TMEM buffer (KSPLIT 1) to fit 512 columns.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tnb {
namespace tc {

constexpr int BM = 128;          // rows of A per tile (MMA M)
constexpr int BK = 32;           // fp32 elements per k-block = 128 B = one swizzle atom row
constexpr int TILE_BYTES = BM * BK * 4;              // 16 KB A tile
constexpr int THREADS = 192;
constexpr int KSPLIT = 2;       // k-blocks alternate between KSPLIT accumulators (summed in fp32 RN):
                                // the tensor-core accumulator truncates, so shorter chains = less bias
// BN (MMA N = rows of the B tile = real output columns per tile) is a template parameter: 128 for wide
// contractions, 64 / 32 for tall-skinny ones (long K, few output columns).
// Fused pre-pass for the plain (non-grouped, A-not-embedded) GEMM: 8 extra producer warps gather the A tile
// straight from the stem in its own bit layout, split it into tf32 hi / lo and store it into the SWIZZLE_128B
// layout (no K-major hi / lo copy of A through HBM); B keeps its TMA path.
struct GatherA {
    const float2* A;
    const int32_t* ma;      // A row of output row r (null: r)
    int64_t a_row, Mp;      // A row stride; D rows = R * 2^log2m
    int log2m, ntab, K;     // m-index bits, byte tables, complex k
    const uint32_t* tabm;   // [ntab][256]: A offsets of the m-index bytes
    const uint32_t* koff;   // [K]: A offsets of k
};
constexpr int GA_PROD = 256;    // gather producer threads (2 groups of 128 rows, alternating stages)
constexpr int GA_KMAX = 1024;   // koff table entries in shared memory

template <int BN, int CG = 1>
struct Cfg {
    static constexpr int BH = BN / CG;                              // B rows (MMA N) held by one CTA
    static constexpr int BTILE = BH * BK * 4;                       // B tile bytes per CTA
    static constexpr int STAGE = 2 * TILE_BYTES + 2 * BTILE;        // Ahi, Alo, Bhi, Blo
    static constexpr int STAGES = (200 * 1024) / STAGE < 5 ? (200 * 1024) / STAGE : 5;
    static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int SMEM_GA = SMEM + 4 * 256 * 4 + GA_KMAX * 4;  // + gather tables
    static constexpr int KS = BN == 256 ? 1 : KSPLIT;               // accumulators per tile buffer
    static constexpr int TMEM_COLS = 2 * KS * BN;                   // 2 tile buffers x KS x BN columns
    static_assert(TMEM_COLS <= 512, "TMEM has 512 columns");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: start>>4, LBO = 1 (16 B, unused for
// swizzled K-major), SBO = 1024 B (8 rows x 128 B), version 1 (sm_100), layout type 2 (SW128).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// instruction descriptor: D fp32 (bit 4), A/B tf32 (format 2 at bits 7, 10), K-major both,
// N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// ---- CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {  // shared::cluster address
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {  // arrive on the barrier in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

template <int BN, int CG = 1, bool GA = false>
__global__ void __launch_bounds__(GA ? THREADS + GA_PROD : THREADS, 1)
    k_gemm_tf32x3(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                  const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                  float* __restrict__ C, int64_t Mp, int64_t N2, int64_t K2, int ea_flags,
                  const int4* __restrict__ tiles, const int32_t* __restrict__ perm, int64_t cm, int64_t cn,
                  int n_tiles, int tiles_n, const GatherA ga) {
    using CF = Cfg<BN, CG>;
    constexpr int STAGES = CF::STAGES;
    constexpr int STAGE_BYTES = CF::STAGE;
    constexpr int TMEM_COLS = CF::TMEM_COLS;
    constexpr int KS = CF::KS;
    constexpr int BH = CF::BH;
    constexpr int B0 = 2 * TILE_BYTES, B1 = 2 * TILE_BYTES + CF::BTILE;  // Bhi / Blo offsets
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;   // [2]
    uint64_t* tempty = tfull + 2;       // [2]
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    uint32_t* s_tabm = (uint32_t*)((uint8_t*)full + 256);   // GA: gather tables after the barriers
    uint32_t* s_koff = s_tabm + 4 * 256;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if constexpr (GA) {
        for (int i = threadIdx.x; i < ga.ntab * 256; i += blockDim.x) s_tabm[i] = ga.tabm[i];
        for (int i = threadIdx.x; i < ga.K; i += blockDim.x) s_koff[i] = ga.koff[i];
    }
    const int nkb = (int)(K2 / BK);
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;       // CTA rank in the pair (0 = MMA leader)
    const int tile0 = (int)blockIdx.x / CG, tstride = (int)gridDim.x / CG;
    // grouped scatter: cm (rows per output row-block) and cn (columns) are powers of two
    const int lcm = 63 - __clzll(cm > 0 ? cm : 1), lcn = 63 - __clzll(cn > 0 ? cn : 1);
    const int ea = ea_flags & 1;            // embedded A
    const bool cmaj = (ea_flags & 2) != 0;  // plain C stored column-major within a row: (r, n, m) with m lowest

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            // GA: the TMA thread's expect_tx arrive + one arrive per gather producer (of both CTAs of a pair)
            mbar_init(&full[s], GA ? 1 + CG * (GA_PROD / 2) : 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4 * CG);  // one arrive per epilogue warp (of both CTAs of a pair)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if constexpr (CG == 2)
        cluster_sync_all();  // both CTAs' barriers are initialised before any remote arrive / TMA
    else
        __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    // tile -> (m0, n0) in D-row / D-col units, plus grouped-mode extents
    auto tile_coords = [&](int t, int& m0, int& n0, int& xvalid, int& xbase, int& yvalid, int& ybase, int& goff) {
        if (tiles) {
            const int4 t0 = tiles[2 * t], t1 = tiles[2 * t + 1];
            m0 = t0.x;
            xvalid = t0.y;
            xbase = t0.z;
            n0 = t0.w;
            yvalid = t1.x;
            ybase = t1.y;
            goff = t1.z;
        } else if (tiles_n > 0) {  // N fastest: neighbouring CTAs share the A (M-side) tile
            m0 = (t / tiles_n) * BM * CG;
            n0 = (t % tiles_n) * BN;
            xvalid = BM * CG;
            xbase = 0;
            yvalid = BN;
            ybase = 0;
            goff = 0;
        } else {  // tiles_n < 0 encodes M fastest over -tiles_n M-tiles: CTAs share the B tile
            m0 = (t % (-tiles_n)) * BM * CG;
            n0 = (t / (-tiles_n)) * BN;
            xvalid = BM * CG;
            xbase = 0;
            yvalid = BN;
            ybase = 0;
            goff = 0;
        }
        // this CTA's half of a pair tile: D rows [m0 + rank * BM, +BM)
        m0 += (int)rank * BM;
        xvalid -= (int)rank * BM;
    };

    if (warp == 0) {
        if (lane == 0) {
            // -------------------------------------------------------- TMA producer
            int it = 0;
            for (int t = tile0; t < n_tiles; t += tstride) {
                int m0, n0, xv, xb, yv, yb, go;
                tile_coords(t, m0, n0, xv, xb, yv, yb, go);
                for (int kb = 0; kb < nkb; kb++, it++) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * STAGE_BYTES;
                    const int kc = kb * BK;
                    if constexpr (CG == 2) {
                        // both CTAs' bytes complete on the leader's barrier; the leader arms it for both
                        const uint32_t fb = map_to_rank(&full[s], 0);
                        if (rank == 0) mbar_expect_tx(&full[s], GA ? 2 * 2 * CF::BTILE : 2 * STAGE_BYTES);
                        // grouped tiles run MMA N = the group's columns (rounded to 16): CTA r holds
                        // D columns [r * N/2, (r + 1) * N/2) of the tile
                        const int ntile = tiles ? min(BN, (yv + 15) & ~15) : BN;
                        const int nb = n0 + (int)rank * (ntile >> 1);
                        if constexpr (!GA) {
                            tma_load_2d_pair(st + 0 * TILE_BYTES, &mAhi, fb, kc, m0);
                            tma_load_2d_pair(st + 1 * TILE_BYTES, &mAlo, fb, kc, m0);
                        }
                        tma_load_2d_pair(st + B0, &mBhi, fb, kc, nb);
                        tma_load_2d_pair(st + B1, &mBlo, fb, kc, nb);
                    } else {
                        mbar_expect_tx(&full[s], GA ? 2 * CF::BTILE : STAGE_BYTES);
                        if constexpr (!GA) {
                            tma_load_2d(st + 0 * TILE_BYTES, &mAhi, &full[s], kc, m0);
                            tma_load_2d(st + 1 * TILE_BYTES, &mAlo, &full[s], kc, m0);
                        }
                        tma_load_2d(st + B0, &mBhi, &full[s], kc, n0);
                        tma_load_2d(st + B1, &mBlo, &full[s], kc, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // -------------------------------------------------------- MMA issuer (the pair's leader)
            int it = 0, lt = 0;
            for (int t = tile0; t < n_tiles; t += tstride, lt++) {
                int ntile = BN;
                if (CG == 2 && tiles) ntile = min(BN, (tiles[2 * t + 1].x + 15) & ~15);
                const uint32_t idesc = idesc_tf32(BM * CG, ntile);
                const int buf = lt & 1;
                const uint32_t tph = (lt >> 1) & 1;
                if (lt >= 2) mbar_wait(&tempty[buf], tph ^ 1);  // epilogue drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t acc0 = tmem + (uint32_t)(buf * BN * KS);
                for (int kb = 0; kb < nkb; kb++, it++) {
                    const uint32_t acc = acc0 + (uint32_t)((kb % KS) * BN);
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 8; k++) {
                        const uint32_t koff = k * 32;  // 8 tf32 = 32 B along the swizzled 128 B row
                        const uint64_t dAhi = sdesc_sw128(st + 0 * TILE_BYTES + koff);
                        const uint64_t dAlo = sdesc_sw128(st + 1 * TILE_BYTES + koff);
                        const uint64_t dBhi = sdesc_sw128(st + B0 + koff);
                        const uint64_t dBlo = sdesc_sw128(st + B1 + koff);
                        const uint32_t first = (kb < KS && k == 0) ? 0u : 1u;
                        if constexpr (CG == 2) {
                            mma_tf32_pair(acc, dAlo, dBhi, idesc, first);  // small terms first
                            mma_tf32_pair(acc, dAhi, dBlo, idesc, 1u);
                            mma_tf32_pair(acc, dAhi, dBhi, idesc, 1u);
                        } else {
                            mma_tf32(acc, dAlo, dBhi, idesc, first);
                            mma_tf32(acc, dAhi, dBlo, idesc, 1u);
                            mma_tf32(acc, dAhi, dBhi, idesc, 1u);
                        }
                    }
                    // frees the smem stage (in both CTAs of a pair) once these MMAs have read it
                    if constexpr (CG == 2)
                        mma_commit_pair(&empty[s]);
                    else
                        mma_commit(&empty[s]);
                }
                if constexpr (CG == 2)
                    mma_commit_pair(&tfull[buf]);  // accumulator halves ready for both epilogues
                else
                    mma_commit(&tfull[buf]);
            }
        }
    } else if (GA && warp >= THREADS / 32) {
        if constexpr (GA) {
            // -------------------------------------------------------- gather producers (fused A pre-pass)
            const int pt = threadIdx.x - THREADS, g = pt >> 7, row = pt & 127;
            const uint32_t fb0 = CG == 2 ? map_to_rank(&full[0], 0) : 0u;
            int it = 0;
            for (int t = tile0; t < n_tiles; t += tstride) {
                int m0, n0, xv, xb, yv, yb, go;
                tile_coords(t, m0, n0, xv, xb, yv, yb, go);
                const int64_t x = (int64_t)m0 + row;
                const float2* __restrict__ base = nullptr;
                if (x < ga.Mp) {
                    const int64_t r = x >> ga.log2m, mi = x & (((int64_t)1 << ga.log2m) - 1);
                    uint32_t aoff = 0;
                    for (int b = 0; b < ga.ntab; b++) aoff += s_tabm[b * 256 + (int)((mi >> (8 * b)) & 255)];
                    base = ga.A + (ga.ma ? (int64_t)ga.ma[r] : r) * ga.a_row + aoff;
                }
                for (int kb = 0; kb < nkb; kb++, it++) {
                    if ((it & 1) != g) continue;
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * STAGE_BYTES;
                    float2 v[16];
#pragma unroll
                    for (int kk = 0; kk < 16; kk++) {
                        const int k = kb * 16 + kk;
                        v[kk] = (base && k < ga.K) ? __ldg(base + s_koff[k]) : make_float2(0.f, 0.f);
                    }
#pragma unroll
                    for (int kk = 0; kk < 16; kk += 2) {
                        float4 h, l;
                        uint32_t r0;
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r0) : "f"(v[kk].x));
                        h.x = __uint_as_float(r0);
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r0) : "f"(v[kk].y));
                        h.y = __uint_as_float(r0);
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r0) : "f"(v[kk + 1].x));
                        h.z = __uint_as_float(r0);
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r0) : "f"(v[kk + 1].y));
                        h.w = __uint_as_float(r0);
                        l = make_float4(v[kk].x - h.x, v[kk].y - h.y, v[kk + 1].x - h.z, v[kk + 1].y - h.w);
                        const int c = 2 * kk;  // float column of this 16-byte chunk
                        const uint32_t o = (uint32_t)(row * 128 + (((c >> 2) ^ (row & 7)) << 4));
                        *(float4*)(st + o) = h;
                        *(float4*)(st + TILE_BYTES + o) = l;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if constexpr (CG == 2)
                        mbar_arrive_cluster(fb0 + (uint32_t)(s * sizeof(uint64_t)));
                    else
                        mbar_arrive(&full[s]);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue warps 2..5
        const int quarter = warp & 3;         // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;  // TMEM lane = tile row
        int lt = 0;
        const uint32_t tempty_leader = CG == 2 ? map_to_rank(&tempty[0], 0) : 0u;
        for (int t = tile0; t < n_tiles; t += tstride, lt++) {
            int m0, n0, xvalid, xbase, yvalid, ybase, goff;
            tile_coords(t, m0, n0, xvalid, xbase, yvalid, ybase, goff);
            const int buf = lt & 1;
            const uint32_t tph = (lt >> 1) & 1;
            mbar_wait(&tfull[buf], tph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t gm = (int64_t)m0 + row;
#pragma unroll 1
            const int ncol = (CG == 2 && tiles) ? min(BN, (yvalid + 15) & ~15) : BN;  // MMA N of this tile
            for (int c0 = 0; c0 < ncol; c0 += 32) {
                uint32_t v[32];
                {
                    float f[32];
#pragma unroll
                    for (int q = 0; q < 32; q++) f[q] = 0.f;
                    const int nsplit = nkb < KS ? nkb : KS;
                    for (int sp = 0; sp < nsplit; sp++) {
                        uint32_t u[32];
                        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) +
                                               (uint32_t)((buf * KS + sp) * BN + c0);
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                            : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                              "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                              "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
                              "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
                              "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                            : "r"(taddr));
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int q = 0; q < 32; q++) f[q] += __uint_as_float(u[q]);
                    }
#pragma unroll
                    for (int q = 0; q < 32; q++) v[q] = __float_as_uint(f[q]);
                }
                if (tiles) {
                    // grouped scatter: D column -> gathered block p = goff + j / cn, fb = j % cn; C row perm[p]
                    if (!ea && cn >= 2) {
                        // tile columns start group-aligned (cn | 16), so complex pairs (q, q+1) share a block
                        // and are adjacent in C: one 16-byte store per pair; C has < 2^32 elements (bind)
                        if (row < xvalid) {
                            const uint32_t fa = (uint32_t)(m0 - xbase + row);
                            const uint32_t j0 = (uint32_t)(n0 - ybase + c0) >> 1;
                            float2* C2 = (float2*)C;
#pragma unroll
                            for (int q = 0; q < 16; q += 2) {
                                if (c0 + 2 * q >= yvalid) break;
                                const uint32_t j = j0 + (uint32_t)q;
                                const uint32_t r = (uint32_t)__ldg(perm + goff + (int)(j >> lcn));
                                const uint32_t idx = ((((r << lcm) + fa) << lcn) + (j & (uint32_t)(cn - 1)));
                                *(float4*)(C2 + idx) = make_float4(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]),
                                                                   __uint_as_float(v[2 * q + 2]),
                                                                   __uint_as_float(v[2 * q + 3]));
                            }
                        }
                    } else if (!ea) {
                        if (row < xvalid) {
                            const int64_t fa = (int64_t)(m0 - xbase) + row;
#pragma unroll
                            for (int q = 0; q < 16; q++) {
                                const int c = c0 + 2 * q;
                                if (c >= yvalid) break;
                                const int64_t j = (int64_t)(n0 - ybase + c) >> 1;
                                const int64_t pblk = goff + (j >> lcn), fb = j & (cn - 1);
                                const int64_t r = perm[pblk];
                                *(float2*)(C + 2 * ((((r << lcm) + fa) << lcn) + fb)) =
                                    make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
                            }
                        }
                    } else {
                        const bool odd = lane & 1;
                        float y[16];
#pragma unroll
                        for (int j = 0; j < 16; j++) {
                            const float x = __uint_as_float(odd ? v[j] : v[16 + j]);
                            y[j] = __shfl_xor_sync(0xffffffffu, x, 1);
                        }
                        const int rloc = row & ~1;
                        if (rloc < xvalid) {
                            const int64_t fa = ((int64_t)(m0 - xbase) + rloc) >> 1;
#pragma unroll
                            for (int q = 0; q < 16; q++) {
                                const int c = c0 + (odd ? 16 : 0) + q;
                                if (c >= yvalid) break;
                                const int64_t j = (int64_t)(n0 - ybase + c);
                                const int64_t pblk = goff + (j >> lcn), fb = j & (cn - 1);
                                const int64_t r = perm[pblk];
                                const float re = odd ? y[q] : __uint_as_float(v[q]);
                                const float im = odd ? __uint_as_float(v[16 + q]) : y[q];
                                *(float2*)(C + 2 * ((((r << lcm) + fa) << lcn) + fb)) = make_float2(re, im);
                            }
                        }
                    }
                } else if (!ea && cmaj) {
                    // column-major C (lower.cpp): complex (m = gm, n) at ((r << lcn) + n) << lcm | orbit, r = gm >> lcm;
                    // the 32 lanes hold consecutive m, so each store is 256 contiguous bytes
                    if (gm < Mp) {
                        float2* C2 = (float2*)C;
                        const int64_t rb = ((gm >> lcm) << (lcm + lcn)) + (gm & (cm - 1));
                        const int64_t nf = (int64_t)(n0 + c0) >> 1;
#pragma unroll
                        for (int q = 0; q < 16; q++)
                            if (nf + q < cn)
                                C2[rb + ((nf + q) << lcm)] = make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
                    }
                } else if (!ea) {
                    // D = C interleaved: row gm of D is row gm of C (real columns 2n, 2n+1 = re, im)
                    if (gm < Mp) {
                        float4* dst = (float4*)(C + gm * N2 + n0 + c0);
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                                 __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                    }
                } else {
                    // embedded A: D row 2m = Re C[m][:], row 2m+1 = Im C[m][:] (lanes 2i, 2i+1 of this warp);
                    // exchange halves so that each lane writes 16 interleaved complex values
                    const bool odd = lane & 1;
                    float y[16];
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        const float x = __uint_as_float(odd ? v[j] : v[16 + j]);
                        y[j] = __shfl_xor_sync(0xffffffffu, x, 1);
                    }
                    const int64_t mc = gm >> 1;
                    if (gm < Mp) {  // here Mp counts D rows (= 2 x complex rows)
                        float4* dst = (float4*)(C + (mc * N2 + n0 + c0 + (odd ? 16 : 0)) * 2);
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const int j0 = 2 * q, j1 = 2 * q + 1;
                            if (!odd)
                                dst[q] = make_float4(__uint_as_float(v[j0]), y[j0], __uint_as_float(v[j1]), y[j1]);
                            else
                                dst[q] = make_float4(y[j0], __uint_as_float(v[16 + j0]), y[j1],
                                                     __uint_as_float(v[16 + j1]));
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2)
                    mbar_arrive_cluster(tempty_leader + (uint32_t)(buf * sizeof(uint64_t)));
                else
                    mbar_arrive(&tempty[buf]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if constexpr (CG == 2) {
        cluster_sync_all();  // neither CTA frees TMEM / exits while its peer's MMAs or arrivals are in flight
        if (warp == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    } else {
        __syncthreads();
        if (warp == 2)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

}  // namespace tc
}  // namespace tnb
