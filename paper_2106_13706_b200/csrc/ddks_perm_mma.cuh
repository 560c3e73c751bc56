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
// K = N, N_gemm = n_perm) and exact: FP8 E4M3 0/1 operands (1.0 = 0x38), fp32 accumulation of at most
// N <= 65535 < 2^24 ones (tcgen05.mma kind::f8f6f4: half the operand bytes and twice the rate of fp16).
//
// One CTA computes a 128 x 256 tile of C (128 (origin, orthant) rows, 256 permutations) over all points:
//   * warp 8 (one lane) streams the label tile B[j][x] (prepared by k_labels_mma in the UMMA canonical K-major layout,
//     so a whole tile is one cp.async.bulk) and the k-block's 128 packed points into a 3-stage ring (mbarriers);
//   * warps 0-7 classify: the 2^d-code of every (origin of the tile, point of the k-block) pair with d FP32 >=
//     compares (the pair classification of the hot path), then expand the codes into the one-hot fp8 rows of A
//     directly in SMEM (byte-SIMD: 4 codes compared with the row's orthant per instruction; two threads per row,
//     each counting its half of T in a register);
//   * warp 9 (one lane) issues tcgen05.mma.kind::f8f6f4 (M = 128, N = 256, K = 32) x 4 per k-block into a TMEM
//     accumulator of 256 columns and commits each stage back to the ring;
//   * epilogue: warps 0-7 read the 128 TMEM lanes (two warps per lane quadrant, half the columns each) (tcgen05.ld 32x32b.x32), form |(a + b) C - b T| per column,
//     reduce it over the 128 rows (redux.sync max + SMEM atomicMax) and atomicMax g * that into num[j].
#pragma once
#include <cstdint>

#include "ddks_kernels.cuh"

namespace ddks {
namespace {

#ifndef DDKS_PM_S  // pipeline stages: 2 (two CTAs per SM, one's epilogue under the other's MMAs; C4b null 120 -> 99 us vs 3)
#define DDKS_PM_S 2
#endif
constexpr int PM_M = 128, PM_N = 256, PM_KB = 128, PM_S = DDKS_PM_S;  // tile rows, permutations, points per k-block
constexpr int PM_A_BYTES = PM_M * PM_KB, PM_B_BYTES = PM_N * PM_KB;   // 16 KB, 32 KB fp8 tiles
constexpr uint8_t PM_ONE = 0x38;                                      // FP8 E4M3 1.0
constexpr int PM_GEN = 256;                                           // classify + epilogue threads (warps 0-7)
constexpr int PM_THREADS = PM_GEN + 64;                               // + warp 8 (TMA producer) + warp 9 (MMA issuer)
constexpr int PM_WTMA = PM_GEN / 32, PM_WMMA = PM_WTMA + 1;

// Byte offset of element (row, k) of a [rows][PM_KB] fp8 tile in the canonical K-major, no-swizzle UMMA layout:
// core matrices of 8 rows x 16 elements (128 contiguous bytes), the 8 K-chunks of an 8-row group adjacent
// (LBO = 128 B), 8-row groups 1024 B apart (SBO).
__host__ __device__ constexpr uint32_t pm_off(int row, int k) {
    return (uint32_t)((row >> 3) * 1024 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

template <int D> struct PermMmaGeo {
    static constexpr int NQ = 1 << D, OPT = PM_M / NQ;  // origins per tile (D <= 7)
    static constexpr int DP = padded_dim<D>();
    static constexpr int PTS_BYTES = PM_KB * DP * 4;
    static constexpr int STAGE_BYTES = PM_B_BYTES + PM_A_BYTES + PTS_BYTES;
    static constexpr int CODE_BYTES = OPT * PM_KB;  // one byte per (origin, point) of a k-block
    static constexpr int SMEM_BYTES = PM_S * STAGE_BYTES + PM_S * CODE_BYTES + OPT * DP * 4 + PM_N * 4 + 2 * PM_M * 4 + 128;
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

// ---------------------------------------------------------------------------------------------- PTX wrappers (tcgen05: alloc / mma / commit / ld)
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
// instruction descriptor, kind::f8f6f4: D f32 (bits 4-5 = 1), A = B = E4M3 (0), both K-major, N >> 3 at [17,23),
// M >> 4 at [24,29)
constexpr uint32_t PM_IDESC = (1u << 4) | ((uint32_t)(PM_N >> 3) << 17) | ((uint32_t)(PM_M >> 4) << 24);

__device__ __forceinline__ void pm_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
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
// B[j][x] = 1.0 (E4M3) iff point x is in P' of permutation j (perms[j][0 .. n_P)), in the canonical layout of the tile
// (n_tile = j / 256, k_block = x / 128); the buffer is zeroed first. Validates every perms row as in k_labels.
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
            bimg[tile * PM_B_BYTES + pm_off((int)(j % PM_N), (int)(src % PM_KB))] = PM_ONE;
        }
    }
    if (bad) atomicOr(flag, 2u);
}

// ---------------------------------------------------------------------------------------------- the null kernel
template <int D, bool GT>
__global__ void __launch_bounds__(PM_THREADS, PM_S <= 2 ? 2 : 1) k_perm_mma(const PermMmaArgs a) {
    using G = PermMmaGeo<D>;
    constexpr int NQ = G::NQ, OPT = G::OPT, DP = G::DP;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;                                                       // [S][B | A | points]
    uint8_t* codes = smem + PM_S * G::STAGE_BYTES;                                // [S][OPT][PM_KB]
    float* ocoord = reinterpret_cast<float*>(codes + PM_S * G::CODE_BYTES);       // [OPT][DP]
    uint32_t* colmax = reinterpret_cast<uint32_t*>(ocoord + OPT * DP);            // [PM_N]
    uint32_t* tsh = colmax + PM_N;                                                // [2][PM_M] half-row T counts
    uint64_t* bars = reinterpret_cast<uint64_t*>(tsh + 2 * PM_M);                 // full[S], aready[S], empty[S], done
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
        for (int s = 0; s < PM_S; ++s) mbar_init(&full[s], 1), mbar_init(&aready[s], PM_GEN), mbar_init(&empty[s], 1);
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == PM_WMMA) {  // TMEM: 256 fp32 columns x 128 lanes for the accumulator
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

    if (warp == PM_WTMA) {
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
    } else if (warp == PM_WMMA) {
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
                for (int k = 0; k < PM_KB / 32; ++k)  // K = 32 fp8 per MMA: two 16-byte chunks, 256 bytes apart
                    pm_mma(tmem, pm_desc(asa + k * 256), pm_desc(bsa + k * 256), (kb | k) ? 1u : 0u);
                pm_commit(&empty[s]);  // the stage is free once these MMAs have read it
            }
            pm_commit(done);
        }
        __syncwarp();
    } else {
        // classify (warps 0-7): the code of every (origin, point) pair of the k-block (invalid origins / points get
        // code 0xFF, which no orthant matches), then thread t writes half h = t / 128 of A row r = t % 128 =
        // (origin r / 2^d, orthant r % 2^d): four 16-byte chunks of 16 fp8, built 4 codes at a time with byte SIMD
        const int r = t & (PM_M - 1), h = t >> 7;
        const int orow = r / NQ, qrow = r % NQ;
        const uint32_t qrep = (uint32_t)qrow * 0x01010101u;
        uint32_t Tcnt = 0;
        unsigned long long exec_cmp = 0;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % PM_S;
            mbar_wait(&full[s], (uint32_t)((kb / PM_S) & 1));  // points landed (and the stage's MMAs of kb - S done)
            uint8_t* st = stages + s * G::STAGE_BYTES;
            const float* pts = reinterpret_cast<const float*>(st + PM_B_BYTES + PM_A_BYTES);
            uint8_t* cd = codes + s * G::CODE_BYTES;
            const int xvalid = min(PM_KB, a.N - kb * PM_KB);
            for (int i = t; i < OPT * PM_KB; i += PM_GEN) {
                const int o = i / PM_KB, x = i % PM_KB;
                uint32_t c = 0;
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const float xv = pts[x * DP + k], ov = ocoord[o * DP + k];
                    c |= (GT ? (xv > ov) : (xv >= ov)) ? (1u << k) : 0u;
                }
                cd[i] = (x < xvalid && o0 + o < a.N) ? (uint8_t)c : (uint8_t)0xFF;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(PM_GEN) : "memory");
            uint8_t* A = st + PM_B_BYTES;
            const uint4* crow = reinterpret_cast<const uint4*>(cd + orow * PM_KB);
#pragma unroll
            for (int c4 = 0; c4 < PM_KB / 32; ++c4) {
                const int kc = h * (PM_KB / 32) + c4;  // this thread's 16-point chunks
                const uint4 cw = crow[kc];
                uint32_t w[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
                for (int wi = 0; wi < 4; ++wi) {
                    const uint32_t y = w[wi] ^ qrep;                                        // zero byte <=> code == q
                    const uint32_t z = ~(((y & 0x7f7f7f7fu) + 0x7f7f7f7fu) | y) & 0x80808080u;  // 0x80 per match
                    Tcnt += __popc(z);
                    w[wi] = (z >> 7) * (uint32_t)PM_ONE;                                      // E4M3 1.0 per match
                }
                *reinterpret_cast<uint4*>(A + pm_off(r, kc * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
            exec_cmp += (unsigned long long)D * OPT * PM_KB / PM_GEN;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
            mbar_arrive(&aready[s]);
        }
        if (a.clk && t == 0) atomicAdd(&a.clk[2], exec_cmp * (unsigned long long)PM_GEN);
        tsh[h * PM_M + r] = Tcnt;
        asm volatile("bar.sync 1, %0;" ::"n"(PM_GEN) : "memory");

        // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (its 32 rows) for the columns [128 (w / 4), + 128)
        mbar_wait(done, 0);
        tc_fence_after();
        const int er = (warp & 3) * 32 + lane;
        const int64_t bT = (int64_t)a.b * (tsh[er] + tsh[PM_M + er]);
#pragma unroll 1
        for (int c0 = (warp >> 2) * (PM_N / 2); c0 < (warp >> 2) * (PM_N / 2) + PM_N / 2; c0 += 32) {
            uint32_t v[32];
            pm_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int64_t cP = (int64_t)__uint_as_float(v[j]);  // an exact integer count (< 2^24)
                const int64_t df = (int64_t)(a.a + a.b) * cP - bT;
                uint32_t val = (uint32_t)(df < 0 ? -df : df);  // invalid rows: C = T = 0
                val = __reduce_max_sync(0xffffffffu, val);
                if (lane == 0) atomicMax(&colmax[c0 + j], val);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == PM_WMMA) {
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
