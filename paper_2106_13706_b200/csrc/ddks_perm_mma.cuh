// ddks_perm_mma.cuh — the label-invariant permutation null as a tensor-core
// contraction on the 5th-generation tensor cores (tcgen05, accumulators in TMEM).
//
// For a fixed pooled set the orthant code(o, x) does not depend on the labels (P:L371 repeats the statistic per
// permutation). Write it as two 0/1 matrices:
//     A[(o, q)][x] = [code(o, x) == q]              (2^d N rows x N points: the one-hot classification)
//     L[x][j]      = [x in P' of permutation j]      (N points x n_perm permutations)
// then C = A L holds every permutation's P'-count c_P'[o][q][j] at once, T[o][q] = sum_x A[(o, q)][x], and
//     num_j = g * max_{o, q} |(a + b) C[(o, q)][j] - b T[o][q]|          (a = n_Q / g, b = n_P / g)
// exactly as the SMEM-counter kernel k_perm_count computes it. The contraction is dense (a GEMM of M = 2^d N,
// K = N, N_gemm = n_perm) and exact: fp16 0/1 operands, fp32 accumulation of at most N <= 65535 < 2^24 ones.
//
// One CTA computes a 128 x 256 tile of C (128 (origin, orthant) rows, 256 permutations) over all points:
//   * warp 4 (one lane) streams the label tile B[j][x] (prepared by k_labels_mma in the UMMA canonical K-major layout,
//     so a whole tile is one cp.async.bulk) and the k-block's 64 packed points into a 3-stage ring (mbarriers);
//   * warps 0-3 classify: the 2^d-code of every (origin of the tile, point of the k-block) pair with d FP32 >=
//     compares (the pair classification of the hot path), then expand each code into its one-hot fp16 row of A
//     directly in SMEM (thread t owns row t = (origin t / 2^d, orthant t % 2^d) and counts T in a register);
//   * warp 5 (one lane) issues tcgen05.mma.kind::f16 (M = 128, N = 256, K = 16) x 4 per k-block into a TMEM
//     accumulator of 256 columns and commits each stage back to the ring;
//   * epilogue: warps 0-3 read their 128 TMEM lanes (tcgen05.ld 32x32b.x32), form |(a + b) C - b T| per column,
//     reduce it over the 128 rows (redux.sync max + SMEM atomicMax) and atomicMax g * that into num[j].
#pragma once
#include <cstdint>

#include "ddks_kernels.cuh"

namespace ddks {
namespace {

constexpr int PM_M = 128, PM_N = 256, PM_KB = 64, PM_S = 3;          // tile rows, permutations, points per k-block
constexpr int PM_A_BYTES = PM_M * PM_KB * 2, PM_B_BYTES = PM_N * PM_KB * 2;  // 16 KB, 32 KB fp16 tiles
constexpr int PM_THREADS = 192;                                       // warps 0-3 classify + epilogue, 4 TMA, 5 MMA

// Byte offset of element (row, k) of a [rows][PM_KB] fp16 tile in the canonical K-major, no-swizzle UMMA layout:
// core matrices of 8 rows x 8 elements (128 contiguous bytes), the 8 K-chunks of an 8-row group adjacent (LBO = 128 B),
// 8-row groups 1024 B apart (SBO).
__host__ __device__ constexpr uint32_t pm_off(int row, int k) {
    return (uint32_t)((row >> 3) * 1024 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

template <int D> struct PermMmaGeo {
    static constexpr int NQ = 1 << D, OPT = PM_M / NQ;  // origins per tile (D <= 7)
    static constexpr int DP = padded_dim<D>();
    static constexpr int PTS_BYTES = PM_KB * DP * 4;
    static constexpr int STAGE_BYTES = PM_B_BYTES + PM_A_BYTES + PTS_BYTES;
    static constexpr int CODE_BYTES = OPT * PM_KB;  // one byte per (origin, point) of a k-block
    static constexpr int SMEM_BYTES = PM_S * STAGE_BYTES + PM_S * CODE_BYTES + OPT * DP * 4 + PM_N * 4 + 128;
    static_assert(D >= 1 && D <= 7, "tensor-core null: d <= 7 (128-row tiles of whole origins)");
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

struct PermMmaArgs {
    const float* pts;        // pooled packed [N][DP], rows >= N never read as origins; k-block rows past N are ignored
    const uint8_t* bimg;     // label images [n_tiles][k_blocks][PM_B_BYTES] (k_labels_mma)
    int32_t N, n_perm, k_blocks;
    uint32_t a, b;           // DIFF weights (a + b) C - b T
    uint64_t g;
    uint64_t* num;           // [n_perm] atomicMax targets
    unsigned long long* clk; // profiling (or nullptr): [2] += FP32 compares executed
};

// ---------------------------------------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor (SM100 UMMA): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48),
// base offset 0, layout SWIZZLE_NONE (0) [61,64)
__device__ __forceinline__ uint64_t pm_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46);
}
// instruction descriptor, kind::f16: D f32 (bits 4-5 = 1), A = B = f16 (0), both K-major, N >> 3 at [17,23), M >> 4 at [24,29)
constexpr uint32_t PM_IDESC = (1u << 4) | ((uint32_t)(PM_N >> 3) << 17) | ((uint32_t)(PM_M >> 4) << 24);

__device__ __forceinline__ void pm_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(PM_IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void pm_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void pm_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------------------------- label images
// B[j][x] = 1.0h iff point x is in P' of permutation j (perms[j][0 .. n_P)), in the canonical layout of the tile
// (n_tile = j / 256, k_block = x / 64); the buffer is zeroed first. Validates every perms row as in k_labels.
__global__ void k_labels_mma(const int32_t* __restrict__ perms, int64_t n_perm, int64_t N, int64_t n_P, int k_blocks,
                             uint8_t* __restrict__ bimg, uint32_t* __restrict__ bitmap, uint32_t* flag) {
    const int64_t words = (N + 31) / 32;
    const int64_t total = n_perm * N;
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / N, pos = i - j * N;
        const int32_t src = perms[i];
        if (src < 0 || src >= N) { bad = true; continue; }
        const uint32_t bit = 1u << (src & 31);
        if (atomicOr(&bitmap[j * words + (src >> 5)], bit) & bit) bad = true;
        if (pos < n_P) {
            const int64_t tile = (j / PM_N) * k_blocks + src / PM_KB;
            *reinterpret_cast<uint16_t*>(bimg + tile * PM_B_BYTES + pm_off((int)(j % PM_N), (int)(src % PM_KB))) =
                (uint16_t)0x3C00u;  // fp16 1.0
        }
    }
    if (bad) atomicOr(flag, 2u);
}

// ---------------------------------------------------------------------------------------------- the null kernel
template <int D, bool GT>
__global__ void __launch_bounds__(PM_THREADS, 1) k_perm_mma(const PermMmaArgs a) {
    using G = PermMmaGeo<D>;
    constexpr int NQ = G::NQ, OPT = G::OPT, DP = G::DP;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;                                                       // [S][B | A | points]
    uint8_t* codes = smem + PM_S * G::STAGE_BYTES;                                // [S][OPT][PM_KB]
    float* ocoord = reinterpret_cast<float*>(codes + PM_S * G::CODE_BYTES);       // [OPT][DP]
    uint32_t* colmax = reinterpret_cast<uint32_t*>(ocoord + OPT * DP);            // [PM_N]
    uint64_t* bars = reinterpret_cast<uint64_t*>(colmax + PM_N);                  // full[S], aready[S], empty[S], done
    uint64_t* full = bars;
    uint64_t* aready = bars + PM_S;
    uint64_t* empty = bars + 2 * PM_S;
    uint64_t* done = bars + 3 * PM_S;
    __shared__ uint32_t tmem_base;

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int m_tile = blockIdx.x, n_tile = blockIdx.y;
    const int o0 = m_tile * OPT;
    const int KB = a.k_blocks;

    if (t == 0) {
        for (int s = 0; s < PM_S; ++s) mbar_init(&full[s], 1), mbar_init(&aready[s], 128), mbar_init(&empty[s], 1);
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) {  // TMEM: 256 fp32 columns x 128 lanes for the accumulator
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "n"(PM_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = t; i < PM_N; i += PM_THREADS) colmax[i] = 0u;
    for (int i = t; i < OPT * DP; i += PM_THREADS) {
        const int o = o0 + i / DP;
        ocoord[i] = o < a.N ? a.pts[(int64_t)o * DP + i % DP] : 0.0f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 4) {
        if (lane == 0) {  // producer: label tile + the k-block's points per stage (codes[s] is rewritten only S
                          // k-blocks later, after S - 1 further classify barriers)
            const uint8_t* bsrc = a.bimg + (int64_t)n_tile * KB * PM_B_BYTES;
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % PM_S;
                if (kb >= PM_S) mbar_wait(&empty[s], (uint32_t)(((kb / PM_S) - 1) & 1));
                uint8_t* st = stages + s * G::STAGE_BYTES;
                mbar_expect_tx(&full[s], (uint32_t)(PM_B_BYTES + G::PTS_BYTES));
                bulk_g2s(st, bsrc + (int64_t)kb * PM_B_BYTES, PM_B_BYTES, &full[s]);
                bulk_g2s(st + PM_B_BYTES + PM_A_BYTES, a.pts + (int64_t)kb * PM_KB * DP, G::PTS_BYTES, &full[s]);
            }
        }
        __syncwarp();
    } else if (warp == 5) {
        if (lane == 0) {  // MMA issuer
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % PM_S;
                const uint32_t ph = (uint32_t)((kb / PM_S) & 1);
                mbar_wait(&full[s], ph);
                mbar_wait(&aready[s], ph);
                tc_fence_after();
                const uint32_t bsa = smem_u32(stages + s * G::STAGE_BYTES);
                const uint32_t asa = bsa + PM_B_BYTES;
#pragma unroll
                for (int k = 0; k < PM_KB / 16; ++k)
                    pm_mma(tmem, pm_desc(asa + k * 256), pm_desc(bsa + k * 256), (kb | k) ? 1u : 0u);
                pm_commit(&empty[s]);  // the stage is free once these MMAs have read it
            }
            pm_commit(done);
        }
        __syncwarp();
    } else {
        // classify (warps 0-3): codes of every (origin, point) pair of the k-block, then the one-hot A row of thread t
        const int orow = t / NQ, qrow = t % NQ;
        uint32_t Tcnt = 0;
        unsigned long long exec_cmp = 0;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % PM_S;
            mbar_wait(&full[s], (uint32_t)((kb / PM_S) & 1));  // points landed (and the stage's MMAs of kb - S done)
            uint8_t* st = stages + s * G::STAGE_BYTES;
            const float* pts = reinterpret_cast<const float*>(st + PM_B_BYTES + PM_A_BYTES);
            uint8_t* cd = codes + s * G::CODE_BYTES;
            for (int i = t; i < OPT * PM_KB; i += 128) {
                const int o = i / PM_KB, x = i % PM_KB;
                uint32_t c = 0;
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const float xv = pts[x * DP + k], ov = ocoord[o * DP + k];
                    c |= (GT ? (xv > ov) : (xv >= ov)) ? (1u << k) : 0u;
                }
                cd[i] = (uint8_t)c;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int xvalid = min(PM_KB, a.N - kb * PM_KB);  // points past N are zero columns of A
            const bool rvalid = o0 + orow < a.N;
            uint8_t* A = st + PM_B_BYTES;
            const uint32_t* crow = reinterpret_cast<const uint32_t*>(cd + orow * PM_KB);
#pragma unroll
            for (int kc = 0; kc < PM_KB / 8; ++kc) {
                uint32_t h[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int x0 = kc * 8 + 2 * e;
                    const uint32_t cw = crow[x0 >> 2] >> (8 * (x0 & 3));
                    const bool m0 = rvalid && x0 < xvalid && (cw & 0xffu) == (uint32_t)qrow;
                    const bool m1 = rvalid && x0 + 1 < xvalid && ((cw >> 8) & 0xffu) == (uint32_t)qrow;
                    h[e] = (m0 ? 0x3C00u : 0u) | (m1 ? 0x3C000000u : 0u);
                    Tcnt += (uint32_t)m0 + (uint32_t)m1;
                }
                *reinterpret_cast<uint4*>(A + pm_off(t, kc * 8)) = make_uint4(h[0], h[1], h[2], h[3]);
            }
            exec_cmp += (unsigned long long)D * OPT * PM_KB / 128;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
            mbar_arrive(&aready[s]);
        }
        if (a.clk && t == 0) atomicAdd(&a.clk[2], exec_cmp * 128ull);

        // epilogue: this thread's row (TMEM lane t) against every permutation column of the tile
        mbar_wait(done, 0);
        tc_fence_after();
        const bool rvalid = o0 + orow < a.N;
        const int64_t bT = (int64_t)a.b * Tcnt;
#pragma unroll 1
        for (int c0 = 0; c0 < PM_N; c0 += 32) {
            uint32_t v[32];
            pm_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int64_t cP = (int64_t)__uint_as_float(v[j]);  // an exact integer count (< 2^24)
                const int64_t df = (int64_t)(a.a + a.b) * cP - bT;
                uint32_t val = rvalid ? (uint32_t)(df < 0 ? -df : df) : 0u;
                val = __reduce_max_sync(0xffffffffu, val);
                if (lane == 0) atomicMax(&colmax[c0 + j], val);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(PM_N));
    }
    for (int j = t; j < PM_N; j += PM_THREADS) {
        const int jj = n_tile * PM_N + j;
        if (jj < a.n_perm) atomicMax(reinterpret_cast<unsigned long long*>(&a.num[jj]), (unsigned long long)colmax[j] * a.g);
    }
}

}  // namespace
}  // namespace ddks
