// gate_tc.cuh -- "stem absorbs a small tensor" on the 5th-gen tensor cores.
//
//   C[r][x, y] = sum_k A[ma(r)][x, k] * G[k, y]
//
// A is the big stem in its own bit layout (any positions for the k legs), G a small rowless tensor
// (K = 2^nk <= 32 rows, N = 2^nn <= 128 columns after the complex-as-real embedding fits shared memory),
// C the result in its own bit layout.  On SIMT a 16x16 complex gate costs 64 FFMA per stem element, which
// made these steps ALU-bound at ~2x the HBM time (round-1 VERDICT: SIMT apply family at 23-43 % of the FMA
// roof).  Here the stem is read once and written once, so the step is HBM-bound:
//
//   warps 0-7  producers, in groups that fill consecutive stages: a thread owns 1-4 tile rows (orbits x) and
//              gathers their K complex values with the orbit's and the k legs' byte-sliced offset tables (all
//              loads issued before any use: >= 16 in flight per thread), splits them into tf32 hi / lo (3xTF32,
//              SURVEY §8(c) item 19) and stores them straight into the UMMA SWIZZLE_128B K-major layout of a
//              2-4-stage shared-memory ring (no pre-pass through HBM), then fence.proxy.async + mbarrier.
//   warp 12    MMA issuer: tcgen05.mma kind::tf32 M=128 N=2N K=8, three products (lo*hi, hi*lo, hi*hi) per
//              k step, against the gate held resident in shared memory (embedded once per CTA at start:
//              rows (gr, -gi) / (gi, gr), hi / lo), accumulators double-buffered in TMEM.
//   warps 8-11 epilogue: tcgen05.ld (TMEM lane quarter = warp % 4) -> complex outputs -> C through the
//              orbit's and the output legs' offset tables (coalesced when the orbit's low bits are C's).
// Persistent: one CTA per SM (grid = min(tiles, 148)).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_tc.cuh"

namespace tnb {
namespace gtc {

constexpr int PROD = 256;         // producer threads (8 warps)
constexpr int THREADS = PROD + 160;  // + 4 epilogue warps + 1 MMA warp
constexpr int EPI0 = PROD / 32;      // first epilogue warp
constexpr int MMAW = EPI0 + 4;       // MMA warp
constexpr int ROWS = 128;         // orbits per tile (MMA M)

struct GateDev {
    const float2* A;
    const float2* G;
    float2* C;
    const int32_t* ma;        // A row of output row r (null: r)
    int64_t R, a_row, c_row;  // output rows, row strides (complex elements)
    int64_t n_orb;            // orbits per row (power of two)
    int log2_orb;
    int64_t n_tiles;
    int K, N;                 // actual k and n (complex); KC/BN may pad them
    int kpair, ypair;         // 1: k index bit 0 is A's bit 0 / n index bit 0 is C's bit 0 -> 16-byte loads / stores
    const uint32_t* tab;      // [ntab][256][2]: (A offset, C offset) of the orbit index bytes
    int ntab;
    const uint32_t* koff;     // [K]: A offset of k
    const uint32_t* yoff;     // [N]: C offset of output n
    const uint32_t* goff;     // [K][N]: G offset of (k, n) within a G row
    // gather-contract variants (both operands carry sparse rows, SURVEY a6 GATHER-CONTRACT)
    int mode;                 // 0: one rowless gate G
                              // 1: the gate of a tile is G's row mb[r] of its output row r; output rows are
                              //    processed in perm order (grouped by B parent: the gate changes rarely)
                              // 2: tiles run over A's rows (R = A rows); the gate's columns are (member i, n): the
                              //    G rows of the output rows that share the tile's A row, so A is read once
    const int32_t* perm;      // modes 1, 2: output rows in processing order
    const int32_t* mb;        // modes 1, 2: G row of output row r
    int64_t g_row;            // G row stride (complex elements)
    const int32_t* gstart;    // mode 2: first perm position of A row a's output rows
    const int32_t* gcnt;      // mode 2: their count (<= GM)
    int GM;                   // mode 2: member slots per tile (gate columns = GM * N)
};

template <int KC, int BN>
struct GCfg {
    static constexpr int STAGES = KC == 32 ? 4 : 2;
    static constexpr int NKB = KC / 32;                  // 32-float (128 B) k-blocks
    static constexpr int ATILE = ROWS * 128;             // one k-block of A: 16 KB
    static constexpr int STAGE = 2 * NKB * ATILE;        // hi + lo
    static constexpr int BTILE = BN * 128;               // one k-block of the gate
    static constexpr int BBYTES = 2 * NKB * BTILE;       // hi + lo
    static constexpr int SMEM = STAGES * STAGE + BBYTES + 1024 + 256;
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    static_assert(SMEM <= 227 * 1024, "gate kernel shared memory");
};

// byte offset of fp32 element (row, col) of a K-major SWIZZLE_128B tile made of 32-float k-blocks
__device__ __forceinline__ uint32_t sw128_off(int row, int col, int rows) {
    const int kb = col >> 5, c = col & 31;
    const int chunk = (c >> 2) ^ (row & 7);
    return (uint32_t)(kb * rows * 128 + row * 128 + chunk * 16 + (c & 3) * 4);
}

__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    hi = __uint_as_float(r);
    lo = x - hi;
}

template <int KV, int BN>
__global__ void __launch_bounds__(THREADS, 1) k_gate_tc(const GateDev p) {
    constexpr int KC = KV >= 16 ? 2 * KV : 32;  // real K columns (K padded to >= 16 complex)
    using CF = GCfg<KC, BN>;
    constexpr int STAGES = CF::STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* bt = smem + STAGES * CF::STAGE;             // resident gate: hi k-blocks, then lo k-blocks
    uint64_t* full = (uint64_t*)(bt + CF::BBYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint64_t* gfree = tempty + 2;      // [1]: the MMAs reading the resident gate have completed
    uint32_t* tmem_slot = (uint32_t*)(gfree + 1);
    __shared__ uint32_t s_tab[4 * 256 * 2];
    __shared__ uint32_t s_koff[32];
    __shared__ uint32_t s_yoff[128];
    __shared__ int64_t s_cofs[4][128];  // mode 2: C offset of gate column (member i, n), per epilogue warp

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < p.ntab * 512; i += THREADS) s_tab[i] = p.tab[i];
    for (int i = threadIdx.x; i < p.K; i += THREADS) s_koff[i] = p.koff[i];
    for (int i = threadIdx.x; i < p.N; i += THREADS) s_yoff[i] = p.yoff[i];
    // producer groups: each group of PG threads fills one stage (RPT rows per thread, >= 16 loads in flight per
    // thread); NG = PROD / PG groups work on consecutive tiles, so NG stages are being filled at once
    // >= 32 loads in flight per producer thread where the ring allows it (ncu: the kernel is long-scoreboard
    // bound at 1 row x 16 loads per thread)
    constexpr int RPT0 = KV >= 32 ? 1 : 32 / KV;
    constexpr int RPT = RPT0 > ROWS * STAGES / PROD ? ROWS * STAGES / PROD : RPT0;
    constexpr int PG = ROWS / RPT, NG = PROD / PG;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            tc::mbar_init(&full[s], PG);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 4);
        }
        tc::mbar_init(gfree, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMAW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                     "r"(CF::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    // contiguous tile ranges per CTA: consecutive tiles share their gate (modes 1, 2), so reloads are rare
    const int64_t tb = p.n_tiles * blockIdx.x / gridDim.x, te = p.n_tiles * (blockIdx.x + 1) / gridDim.x;
    const int64_t total = p.R * p.n_orb;
    // A row of a tile unit u (mode 2: u is the A row; else u is a perm position)
    auto out_row = [&](int64_t u) -> int64_t { return p.perm ? (int64_t)p.perm[u] : u; };

    if (warp < EPI0) {
        // ------------------------------------------------------------ producers: gather + split + swizzle
        const int g = threadIdx.x / PG, tid = threadIdx.x % PG;
        int it = g;
        // modes 1, 2: the A row of the last unit seen per row slot (consecutive tiles mostly stay in one output
        // row, so the dependent perm / ma loads are paid once per row, not once per tile)
        int64_t last_u[RPT], last_ra[RPT];
#pragma unroll
        for (int rr = 0; rr < RPT; rr++) last_u[rr] = -1, last_ra[rr] = 0;
        for (int64_t t = tb + g; t < te; t += NG, it += NG) {
            const int s = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            if (it >= STAGES) tc::mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * CF::STAGE;
            float2 v[RPT * KV];
            // issue every load of the stage first (16-32 in flight per thread), then split and store
#pragma unroll
            for (int rr = 0; rr < RPT; rr++) {
                const int row = tid + rr * PG;
                const int64_t x = t * ROWS + row;
                if (x < total) {
                    const int64_t u = x >> p.log2_orb, o = x & (p.n_orb - 1);
                    uint32_t aoff = 0;
                    for (int b = 0; b < p.ntab; b++) aoff += s_tab[(b * 256 + (int)((o >> (8 * b)) & 255)) * 2];
                    int64_t ra = u;
                    if (p.mode != 2) {
                        if (u != last_u[rr]) {
                            const int64_t r = out_row(u);
                            last_ra[rr] = p.ma ? (int64_t)p.ma[r] : r;
                            last_u[rr] = u;
                        }
                        ra = last_ra[rr];
                    }
                    const float2* __restrict__ src = p.A + ra * p.a_row + aoff;
#pragma unroll
                    if (KV >= 2 && p.kpair) {  // (kk, kk + 1) adjacent in memory: one 16-byte load
#pragma unroll
                        for (int kk = 0; kk < KV; kk += 2) {
                            const float4 w = __ldg((const float4*)(src + s_koff[kk]));
                            v[rr * KV + kk] = make_float2(w.x, w.y);
                            v[rr * KV + kk + 1] = make_float2(w.z, w.w);
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < KV; kk++) v[rr * KV + kk] = __ldg(src + s_koff[kk]);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < KV; kk++) v[rr * KV + kk] = make_float2(0.f, 0.f);
                }
            }
#pragma unroll
            for (int rr = 0; rr < RPT; rr++) {
                const int row = tid + rr * PG;
#pragma unroll
                for (int kk = 0; kk < KC / 2; kk += 2) {  // one 16-byte chunk = 2 complex values (zero padding)
                    const float2 a = kk < KV ? v[rr * KV + kk] : make_float2(0.f, 0.f);
                    const float2 b = kk + 1 < KV ? v[rr * KV + kk + 1] : make_float2(0.f, 0.f);
                    float4 h, l;
                    tf32_split(a.x, h.x, l.x);
                    tf32_split(a.y, h.y, l.y);
                    tf32_split(b.x, h.z, l.z);
                    tf32_split(b.y, h.w, l.w);
                    const uint32_t o = sw128_off(row, 2 * kk, ROWS);
                    *(float4*)(st + o) = h;
                    *(float4*)(st + CF::NKB * CF::ATILE + o) = l;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc::mbar_arrive(&full[s]);
        }
    } else if (warp == MMAW) {
        // ------------------------------------------------------------ MMA issuer (+ gate loads)
        constexpr uint32_t idesc = tc::idesc_tf32(ROWS, BN);
        const uint32_t bth = tc::smem_u32(bt), btl = bth + CF::NKB * CF::BTILE;
        int64_t cur = -1, last_u0 = -1, last_gid = 0;
        uint32_t gph = 0;
        int it = 0;
        for (int64_t t = tb; t < te; t++, it++) {
            // the tile's gate: mode 0 one gate; mode 1 the G row of the tile's output row (looked up once per
            // output row: the dependent perm / mb loads would stall the issuer every tile); mode 2 the tile's A row
            const int64_t u0 = (t * ROWS) >> p.log2_orb;
            if (p.mode == 1 && u0 != last_u0) {
                last_gid = (int64_t)p.mb[out_row(u0)];
                last_u0 = u0;
            }
            const int64_t gid = p.mode == 0 ? 0 : (p.mode == 1 ? last_gid : u0);
            if (gid != cur) {
                if (cur >= 0) {  // drain: every MMA that reads the resident gate has completed
                    if (lane == 0) tc::mma_commit(gfree);
                    tc::mbar_wait(gfree, gph);
                    gph ^= 1;
                }
                // embedded gate (row 2n = (gr, -gi), row 2n+1 = (gi, gr) along k), split hi / lo, swizzled
                const int members = p.mode == 2 ? p.gcnt[u0] : 1;
                for (int e = lane; e < BN * (KC / 2); e += 32) {
                    const int j = e / (KC / 2), kk = e % (KC / 2);  // D column j = 2 * (i * N + n) + part
                    const int ne = j >> 1, part = j & 1;
                    const int i = p.mode == 2 ? ne / p.N : 0, n = p.mode == 2 ? ne % p.N : ne;
                    float2 g = make_float2(0.f, 0.f);
                    if (kk < p.K && n < p.N && i < members) {
                        int64_t grow = 0;
                        if (p.mode == 1) grow = gid;
                        else if (p.mode == 2) grow = p.mb[p.perm[p.gstart[u0] + i]];
                        g = p.G[grow * p.g_row + p.goff[kk * p.N + n]];
                    }
                    const float v0 = part ? g.y : g.x, v1 = part ? g.x : -g.y;
                    float h0, l0, h1, l1;
                    tf32_split(v0, h0, l0);
                    tf32_split(v1, h1, l1);
                    const uint32_t o0 = sw128_off(j, 2 * kk, BN), o1 = sw128_off(j, 2 * kk + 1, BN);
                    *(float*)(bt + o0) = h0;
                    *(float*)(bt + o1) = h1;
                    *(float*)(bt + CF::NKB * CF::BTILE + o0) = l0;
                    *(float*)(bt + CF::NKB * CF::BTILE + o1) = l1;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                cur = gid;
            }
            if (lane == 0) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                const int buf = it & 1;
                const uint32_t tph = (it >> 1) & 1;
                if (it >= 2) tc::mbar_wait(&tempty[buf], tph ^ 1);
                tc::mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ah = tc::smem_u32(smem + s * CF::STAGE), al = ah + CF::NKB * CF::ATILE;
                const uint32_t acc = tmem + (uint32_t)(buf * BN);
#pragma unroll
                for (int kb = 0; kb < CF::NKB; kb++)
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint32_t ka = kb * CF::ATILE + k * 32, kbb = kb * CF::BTILE + k * 32;
                        const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
                        tc::mma_tf32(acc, tc::sdesc_sw128(al + ka), tc::sdesc_sw128(bth + kbb), idesc, first);
                        tc::mma_tf32(acc, tc::sdesc_sw128(ah + ka), tc::sdesc_sw128(btl + kbb), idesc, 1u);
                        tc::mma_tf32(acc, tc::sdesc_sw128(ah + ka), tc::sdesc_sw128(bth + kbb), idesc, 1u);
                    }
                tc::mma_commit(&empty[s]);
                tc::mma_commit(&tfull[buf]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue warps EPI0 .. EPI0 + 3
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        constexpr int CH = BN < 32 ? BN : 32;  // TMEM columns per load
        int it = 0;
        // the output row of the last unit (mode 1) and the member table of the last A row (mode 2) are kept across
        // tiles: the dependent index loads would otherwise sit in every tile's epilogue (~1-2 us, about one
        // tile's HBM time), and are looked up before the accumulator wait so their latency hides behind it
        int64_t last_uu = -1, last_crow = 0, last_u0 = -1;
        int nvalid = 0;  // mode 2: valid gate columns (members x N) of the current A row
        const int lgN = 31 - __clz(p.N);
        for (int64_t t = tb; t < te; t++, it++) {
            const int buf = it & 1;
            const uint32_t tph = (it >> 1) & 1;
            const int64_t x = t * ROWS + row;
            if (p.mode == 2) {
                // a tile lies in one A row, so the whole warp shares the members' output row offsets
                const int64_t u0 = (t * ROWS) >> p.log2_orb;
                if (u0 != last_u0) {
                    // one C offset per gate column (member row + output legs): each store is then one LDS + add,
                    // like mode 0 (the per-store member lookup made the epilogue the bottleneck: ncu, 2.9 TB/s)
                    const int members = p.gcnt[u0];
                    nvalid = members * p.N;
                    __syncwarp();
                    for (int e = lane; e < nvalid; e += 32)
                        s_cofs[quarter][e] = (int64_t)p.perm[p.gstart[u0] + (e >> lgN)] * p.c_row + s_yoff[e & (p.N - 1)];
                    __syncwarp();
                    last_u0 = u0;
                }
            } else if (x < total) {
                const int64_t u1 = x >> p.log2_orb;
                if (u1 != last_uu) {
                    last_crow = out_row(u1) * p.c_row;
                    last_uu = u1;
                }
            }
            tc::mbar_wait(&tfull[buf], tph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const bool valid = x < total;
            uint32_t coff = 0;
            float2* dst = nullptr;
            if (valid) {
                const int64_t o = x & (p.n_orb - 1);
                for (int b = 0; b < p.ntab; b++) coff += s_tab[(b * 256 + (int)((o >> (8 * b)) & 255)) * 2 + 1];
                if (p.mode != 2) dst = p.C + last_crow + coff;
            }
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += CH) {
                uint32_t u[32];
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * BN + c0);
                if constexpr (CH == 32) {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                          "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                          "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
                          "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
                          "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                        : "r"(taddr));
                } else {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                        "%14,%15}, [%16];"
                        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                          "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                          "=r"(u[14]), "=r"(u[15])
                        : "r"(taddr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (valid && p.mode != 2 && p.ypair) {  // (n, n + 1) adjacent in C: one 16-byte store
#pragma unroll
                    for (int q = 0; q < CH / 2; q += 2) {
                        const int n = (c0 >> 1) + q;
                        if (n < p.N)
                            *(float4*)(dst + s_yoff[n]) = make_float4(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1]),
                                                                      __uint_as_float(u[2 * q + 2]), __uint_as_float(u[2 * q + 3]));
                    }
                } else if (valid && p.mode != 2) {
#pragma unroll
                    for (int q = 0; q < CH / 2; q++) {
                        const int n = (c0 >> 1) + q;
                        if (n < p.N) dst[s_yoff[n]] = make_float2(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1]));
                    }
                } else if (valid && p.ypair) {  // mode 2, (n, n + 1) of one member adjacent in C
                    float2* base = p.C + coff;
#pragma unroll
                    for (int q = 0; q < CH / 2; q += 2) {
                        const int ne = (c0 >> 1) + q;
                        if (ne < nvalid)
                            *(float4*)(base + s_cofs[quarter][ne]) =
                                make_float4(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1]),
                                            __uint_as_float(u[2 * q + 2]), __uint_as_float(u[2 * q + 3]));
                    }
                } else if (valid) {
                    float2* base = p.C + coff;
#pragma unroll
                    for (int q = 0; q < CH / 2; q++) {
                        const int ne = (c0 >> 1) + q;
                        if (ne < nvalid)
                            base[s_cofs[quarter][ne]] = make_float2(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1]));
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == MMAW)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
}

}  // namespace gtc
}  // namespace tnb
