// ddks_kernels.cuh — sm_100a kernels of the exact ddKS hot path (SURVEY.md §8a rows a1–a9).
//
// The statistic (Eq. 1-2, Eq. 3, Eq. 6):
//   for every pooled origin o (P rows, then Q rows) and every pooled point x:
//       code(o, x) = sum_k [x_k >= o_k] 2^k          (FP32 ordered compare, no FTZ)
//       c_P[o][code]++ if x in P else c_Q[o][code]++
//   num(o) = max_q |c_P[o][q] n_Q - c_Q[o][q] n_P|, num = max_o num(o), den = n_P n_Q.
//
// B200 design:
//   * one thread owns R origins (coordinates in registers); a CTA of T threads owns R*T origins;
//   * point tiles are streamed HBM/L2 -> SMEM with cp.async.bulk (TMA bulk engine, UBLKCP) into an
//     S-stage ring guarded by mbarriers; every thread reads each point as a broadcast LDS.128;
//   * each pair costs d FSET.BF (ALU pipe, the compare roofline) + d FFMA-immediate (FMA pipe) that build
//     the histogram *byte address* inside a float whose bit pattern is 0x4B000000 + offset, + one
//     fire-and-forget ATOMS.ADD to a thread-private, bank-conflict-free SMEM counter;
//   * DIFF mode keeps one signed counter per orthant: c_P*a - c_Q*b with a = n_Q/g, b = n_P/g
//     (g = gcd(n_P, n_Q)), so |counter| * g is exactly |c_P n_Q - c_Q n_P| (P:L238 cross-multiplied);
//     SPLIT mode (when DIFF would overflow, and for the significance, which needs c_Q) keeps c_P and c_Q apart;
//   * kd ordering (N >= 40 000): rows pre-sorted label-major and hierarchically by x_0 .. x_{KX-1}, so for most tiles
//     the bits of those dims are decided once per tile and only the other dims are compared (DESIGN.md §7 "kd
//     ordering"); a tile left with ONE compared dim sums its compare bits in registers (count_points, one-dim path);
//   * finalisation is exact integer arithmetic; the max (and the packed argmax key: red(o) << 31 | ~origin) is a
//     warp-shuffle + CTA + atomicMax(u64) reduction, or k_finalize after segmented counts;
//   * the label-invariant permutation null (k_labels / k_perm_count) classifies each pair once per chunk of
//     permutations (the tensor-core version is ddks_perm_mma.cuh; the fused small-N statistic ddks_small.cuh).
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "ddks_common.cuh"

namespace ddks {
namespace {  // internal linkage: several translation units include these kernels

// ----------------------------------------------------------------------------------------------- config
// Counters are 16-bit halves of 32-bit SMEM words. A CTA owns R*T origins; origin j = r*T + t (slot r of thread t)
// lives in word (bin, j mod WPB), low half if j < WPB else high half, WPB = R*T/2 words per bin. For R >= 2 that is
// word (bin, r mod R/2, t): a thread's two origins r and r + R/2 share a word; for R == 1 threads t and t + T/2
// share one. Either way the 32 lanes of a warp hit 32 consecutive words (conflict-free). A CTA processes at most W
// points per launch segment (W chosen by the host so no half can leave int16), then flushes its counters to int32
// global accumulators; if the whole point set fits one segment it finalises in-kernel instead.
template <int D> struct Cfg;
#ifndef DDKS_UNROLL  // experiments: points per unrolled step of the R > 2 inner loop
#define DDKS_UNROLL 8
#endif
constexpr int kUnrollPts = DDKS_UNROLL;
#ifndef DDKS_TWODIM  // experiment, measured slower (C5 651 vs 627 ms, profiles/r2b_twodim_rejected.txt): kd tiles with two
                     // compared dims left accumulate sum a, sum b, sum ab in registers
#define DDKS_TWODIM 0
#endif
#ifndef DDKS_R1_PTS  // points per step of the R == 1 inner loop (d = 8)
#define DDKS_R1_PTS 2
#endif
#ifndef DDKS_UNROLL_PARTIAL  // the same for the kd variants that compare some of the first KX dims (colder code)
#define DDKS_UNROLL_PARTIAL DDKS_UNROLL
#endif
// R origins per thread (1 or even), T threads per CTA (multiple of 64 when R == 1), TILE points per SMEM stage,
// S stages (DIFF mode). T is a multiple of 128 so every SMSP gets the same number of warps.
template <> struct Cfg<1> { static constexpr int R = 8, T = 256, TILE = 512, S = 3; };
template <> struct Cfg<2> { static constexpr int R = 8, T = 256, TILE = 512, S = 3; };
#ifndef DDKS_C3R  // geometry experiments (d = 3), as for d = 5 below
#define DDKS_C3R 8
#define DDKS_C3T 256
#define DDKS_C3TILE 512
#endif
template <> struct Cfg<3> { static constexpr int R = DDKS_C3R, T = DDKS_C3T, TILE = DDKS_C3TILE, S = 3; };
#ifndef DDKS_C4R  // geometry experiments (d = 4; the C4 batch: one 1024-origin item per CTA)
#define DDKS_C4R 4
#define DDKS_C4T 256
#endif
template <> struct Cfg<4> { static constexpr int R = DDKS_C4R, T = DDKS_C4T, TILE = 512, S = 3; };
#ifndef DDKS_C5R  // geometry experiments: -DDDKS_C5R=.. -DDDKS_C5T=.. -DDDKS_C5TILE=.. -DDDKS_C5S=..
// d = 5: R = 4 x 16 warps, 2048 origins per CTA (round 2, with the one-dim register path: C5 count 636.6 -> 630.7 ms
// vs R = 6 x 16 warps; R = 8 x 12 643, R = 6 x 12 653, R = 4 x 24 721, R = 12 x 8 684, R = 2 x 32 782 ms --
// profiles/r2_c5_geometry.txt). Round 1 (no one-dim path): R = 6 x 16 812 vs R = 12 x 8 830 ms.
#define DDKS_C5R 4
#define DDKS_C5T 512
#define DDKS_C5TILE 256
#define DDKS_C5S 3
#endif
template <> struct Cfg<5> { static constexpr int R = DDKS_C5R, T = DDKS_C5T, TILE = DDKS_C5TILE, S = DDKS_C5S; };
template <> struct Cfg<6> { static constexpr int R = 4, T = 384, TILE = 256, S = 3; };
template <> struct Cfg<7> { static constexpr int R = 2, T = 384, TILE = 256, S = 3; };
#ifndef DDKS_C8R  // geometry experiments (d = 8): -DDDKS_C8R=.. -DDDKS_C8T=..
#define DDKS_C8R 1
#define DDKS_C8T 384
#endif
#ifndef DDKS_C8TILE
#define DDKS_C8TILE 256
#endif
template <> struct Cfg<8> { static constexpr int R = DDKS_C8R, T = DDKS_C8T, TILE = DDKS_C8TILE, S = 3; };


// SPLIT (c_P and c_Q kept apart) doubles the bins: halve R (keeping it even or 1), or T when R is already <= 2
template <int D> struct CfgSplit {
    static constexpr int R = Cfg<D>::R > 2 ? Cfg<D>::R / 2 : Cfg<D>::R;
    static constexpr int T = Cfg<D>::R <= 2 ? Cfg<D>::T / 2 : Cfg<D>::T;
};
#ifndef DDKS_S5R  // experiments: SPLIT geometry at d = 5 (the significance's count)
#define DDKS_S5R 4
#define DDKS_S5T 384
#endif
template <> struct CfgSplit<5> { static constexpr int R = DDKS_S5R, T = DDKS_S5T; };  // A/B: 12 warps beat R=6 x 8 warps
template <> struct CfgSplit<7> { static constexpr int R = 1, T = 384; };  // 12 balanced warps: -9% vs R=2 x 6

// SMALL: the geometry of single statistics with few points (N <= kSmallN, SURVEY §7 hard part 4): 256 origins per
// CTA (R = 2, T = 128) and 256-point tiles in a 2-stage ring, so N = 400 (C1) runs 2 CTAs of 128 threads instead of
// one CTA of 2048 origin slots of which 80 % would repeat the last origin.
constexpr int kSmallN = 8192;
template <int D, bool SPLIT, bool SMALL = false> struct Geo {
    static constexpr int R = SMALL ? 2 : (SPLIT ? CfgSplit<D>::R : Cfg<D>::R);
    static constexpr int T = SMALL ? ((SPLIT && D == 8) ? 64 : 128) : (SPLIT ? CfgSplit<D>::T : Cfg<D>::T);
    static constexpr int RP = R / 2;                            // counter words per (bin, thread) when R >= 2
    static constexpr int NBASE = R >= 2 ? RP : 1;               // distinct counter base addresses per thread
    static constexpr int WPB = R * T / 2;                       // counter words per bin
    static constexpr int TILE = SMALL ? 256 : Cfg<D>::TILE;
    static constexpr int S = SMALL ? 2 : Cfg<D>::S;
    static constexpr int DP = padded_dim<D>();
    static constexpr int NQ = 1 << D;
    static constexpr int NB = NQ * (SPLIT ? 2 : 1);            // counters per origin
    static constexpr int HIST_WORDS = NB * WPB;
    static constexpr int TILE_BYTES = TILE * DP * 4;
    static constexpr int SMEM_BYTES = S * TILE_BYTES + HIST_WORDS * 4 + 64;
    static constexpr int ORIGINS = R * T;
    static_assert(R == 1 || R % 2 == 0, "R must be 1 or even");
    static_assert(R >= 2 || T % 64 == 0, "R == 1 pairs thread t with t + T/2: T/2 must be whole warps");
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
    __host__ __device__ static constexpr int slot(int r, int t) { return (r * T + t) % WPB; }
    __host__ __device__ static constexpr bool high(int r, int t) { return r * T + t >= WPB; }
};

template <int D> __device__ __forceinline__ void load_point(const float* sp, float (&x)[D]) {
    const float4 a = *reinterpret_cast<const float4*>(sp);
    if constexpr (D >= 1) x[0] = a.x;
    if constexpr (D >= 2) x[1] = a.y;
    if constexpr (D >= 3) x[2] = a.z;
    if constexpr (D >= 4) x[3] = a.w;
    if constexpr (D >= 5) {
        if constexpr (D == 5) {
            x[4] = sp[4];
        } else {
            const float4 b = *reinterpret_cast<const float4*>(sp + 4);
            x[4] = b.x;
            if constexpr (D >= 6) x[5] = b.y;
            if constexpr (D >= 7) x[6] = b.z;
            if constexpr (D >= 8) x[7] = b.w;
        }
    }
}

// ----------------------------------------------------------------------------------------------- a1: validate + pack
// P: [B][n_P][d], Q: [B][n_Q][d] row-major f32 -> dst: [B][n_P + n_Q][DP] (P rows, then Q rows).
// -0 -> +0, pad dims = 0. Non-finite -> *flag |= 1 (SPEC core-types NonFiniteValue). One launch for both samples.
__global__ void k_pack(const float* __restrict__ P, int64_t n_P, const float* __restrict__ Q, int64_t n_Q, int d,
                       int64_t B, float* __restrict__ dst, int DP, int validate, uint32_t* flag) {
    const int64_t N = n_P + n_Q;
    const int64_t total = B * N;
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / N, r = i - b * N;
        const float* s = r < n_P ? P + (b * n_P + r) * d : Q + (b * n_Q + (r - n_P)) * d;
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float t = (k < d) ? s[k] : 0.0f;
            if (k < d && validate && !isfinite(t)) bad = true;
            v[k] = (t == 0.0f) ? 0.0f : t;
        }
        float4* o = reinterpret_cast<float4*>(dst + i * DP);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        if (DP == 8) o[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (bad) atomicOr(flag, 1u);
}

// a1 for batches of small items, rows of every (item, label) run ordered by x_0 (for k_count<WX>): one CTA of KPS_T
// threads per run of n <= KPS_T KPS_R rows. The order only has to be close to sorted (it changes speed, never counts):
// a one-pass bucket sort into 256 equal-width x_0 buckets between the run's min and max (SMEM histogram, scan,
// atomic slots), then the rows are written in bucket order (validated, -0 -> +0, pad dims = 0). Row order inside a
// label run does not change the statistic.
// Small CTAs (KPS_T threads, up to KPS_R rows each) so that ~16 runs are resident per SM: the kernel is a chain of
// block barriers per run, latency-bound with one row per thread of 512-thread CTAs (C4: 54 us for 8192 runs).
#ifndef DDKS_KPS_T  // experiments: threads per run (KPS_T * KPS_R must stay 1024)
#define DDKS_KPS_T 128
#endif
constexpr int KPS_T = DDKS_KPS_T, KPS_R = 1024 / KPS_T;  // n <= KPS_T * KPS_R = 1024 rows per run
__global__ void __launch_bounds__(KPS_T) k_pack_sorted(const float* __restrict__ P, int64_t n_P,
                                                       const float* __restrict__ Q, int64_t n_Q, int d,
                                                       float* __restrict__ dst, int DP, int validate, uint32_t* flag) {
    constexpr int NBK = 256;
    __shared__ uint32_t cnt[NBK];
    __shared__ float red[2][KPS_T / 32];
    const int64_t b = blockIdx.x;
    const bool lab = blockIdx.y != 0;
    const int n = (int)(lab ? n_Q : n_P);
    const float* src = lab ? Q + b * n_Q * d : P + b * n_P * d;
    float* out = dst + (b * (n_P + n_Q) + (lab ? n_P : 0)) * DP;
    const int t = threadIdx.x;
    for (int i = t; i < NBK; i += KPS_T) cnt[i] = 0u;
    // x_0 of this thread's rows (all loads in flight) and the run's min / max (non-finite values are flagged below and
    // excluded from the range so the bucket arithmetic stays finite)
    float x[KPS_R];
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int k = 0; k < KPS_R; ++k) {
        const int i = t + k * KPS_T;
        x[k] = i < n ? src[(int64_t)i * d] : 0.0f;
    }
#pragma unroll
    for (int k = 0; k < KPS_R; ++k)
        if (t + k * KPS_T < n && isfinite(x[k])) lo = fminf(lo, x[k]), hi = fmaxf(hi, x[k]);
#pragma unroll
    for (int sh = 16; sh; sh >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
    }
    if ((t & 31) == 0) red[0][t >> 5] = lo, red[1][t >> 5] = hi;
    __syncthreads();
    lo = red[0][0], hi = red[1][0];
#pragma unroll
    for (int w = 1; w < KPS_T / 32; ++w) lo = fminf(lo, red[0][w]), hi = fmaxf(hi, red[1][w]);
    const float scale = hi > lo ? (float)NBK / (hi - lo) : 0.0f;
    uint32_t slot[KPS_R];  // bucket << 16 | rank inside the bucket
#pragma unroll
    for (int k = 0; k < KPS_R; ++k) {
        if (t + k * KPS_T < n) {
            const float v = isfinite(x[k]) ? (x[k] - lo) * scale : 0.0f;
            const int bk = v >= (float)(NBK - 1) ? NBK - 1 : (v > 0.0f ? (int)v : 0);
            slot[k] = ((uint32_t)bk << 16) | atomicAdd(&cnt[bk], 1u);
        }
    }
    __syncthreads();
    if (t < 32) {  // exclusive scan of the 256 bucket counts by one warp (8 per lane)
        uint32_t v[NBK / 32], run = 0;
#pragma unroll
        for (int j = 0; j < NBK / 32; ++j) v[j] = cnt[t * (NBK / 32) + j], run += v[j];
        uint32_t inc = run;
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, sh);
            if (t >= sh) inc += y;
        }
        uint32_t off = inc - run;
#pragma unroll
        for (int j = 0; j < NBK / 32; ++j) cnt[t * (NBK / 32) + j] = off, off += v[j];
    }
    __syncthreads();
    // whole rows (re-read: L1 / L2 hits; one 16-byte load when d == 4 and aligned) -> validated, -0 -> +0, pad = 0
    const bool vec4 = d == 4 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < KPS_R; ++k) {
        const int i = t + k * KPS_T;
        if (i >= n) continue;
        const float* s = src + (int64_t)i * d;
        float v[8];
        if (vec4) {
            const float4 q = *reinterpret_cast<const float4*>(s);
            v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w, v[4] = v[5] = v[6] = v[7] = 0.0f;
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) v[m] = (m < d) ? s[m] : 0.0f;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m < d && validate && !isfinite(v[m])) bad = true;
            v[m] = (v[m] == 0.0f) ? 0.0f : v[m];
        }
        const int dstrow = (int)cnt[slot[k] >> 16] + (int)(slot[k] & 0xffffu);
        DDKS_ASSERT(dstrow < n);
        float4* o = reinterpret_cast<float4*>(out + (int64_t)dstrow * DP);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        if (DP == 8) o[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (bad) atomicOr(flag, 1u);
}

// Permutation gather (a9): dst[j][i] = pooled[perm[j][i]]; checks every row is a permutation of 0..N-1
// (range + no duplicates via a per-row bitmap), else *flag |= 2.
template <int DP>
__global__ void k_gather(const float* __restrict__ pooled, const int32_t* __restrict__ perms, int64_t n_perm,
                         int64_t N, float* __restrict__ dst, uint32_t* __restrict__ bitmap, uint32_t* flag) {
    const int64_t words = (N + 31) / 32;
    const int64_t total = n_perm * N;
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / N;
        const int32_t src = perms[i];
        if (src < 0 || src >= N) { bad = true; continue; }
        const uint32_t bit = 1u << (src & 31);
        const uint32_t old = atomicOr(&bitmap[j * words + (src >> 5)], bit);
        if (old & bit) bad = true;
        const float4* s = reinterpret_cast<const float4*>(pooled + (int64_t)src * DP);
        float4* o = reinterpret_cast<float4*>(dst + i * DP);
        o[0] = s[0];
        if (DP == 8) o[1] = s[1];
    }
    if (bad) atomicOr(flag, 2u);
}

// ----------------------------------------------------------------------------------------------- a3-a6: count
struct CountArgs {
    const float* pts;        // packed [B][N][DP]
    int64_t item_stride;     // floats per item = N * DP
    int32_t N, n_P;          // pooled points per item; the first n_P are P
    int32_t o_begin, o_end;  // origin range (pooled indices) this launch owns, per item
    // origin blocks of R*T: CTA y takes block y * blk_stride + blk_off of [o_begin, o_end) (kd-ordered shards stride
    // over the blocks so every rank gets the same mix of cells); accumulator slot li = y * R*T + r*T + t, acc_stride
    // slots per item (stride 1: li = o - o_begin)
    int32_t blk_stride = 1, blk_off = 0, acc_stride = 0;
    // slot (r, t) of a block holds origin r*T + t, or (warp_major: kd / WX counts) warp*32R + r*32 + lane
    int32_t warp_major = 0;
    int32_t seg_points;      // points per grid.z segment (multiple of TILE, <= the int16 flush window)
    uint32_t incP, incQ;     // DIFF: +aQ and -bP (two's complement); SPLIT: 1 and 1
    uint64_t* item_num;      // [B] atomicMax target
    uint64_t* per_origin;    // [o_end - o_begin] or nullptr (B == 1)
    int32_t* accum;          // accumulate mode: [B][NB][acc_stride] int32 counters (zeroed before the launch),
                             // else nullptr (direct mode: the whole point set is one segment)
    int32_t blk_base = 0;    // this launch's first origin block (grid.y is chunked at 65535)
    // packed argmax (B == 1, or nullptr): atomicMax of red(o) << 31 | (2^31 - 1 - pooled index) over the
    // origins, i.e. the max num and, among origins attaining it, the smallest pooled index (R7); the host
    // uses it only when n_P n_Q / gcd < 2^33, so the key fits 64 bits
    unsigned long long* best_key;
    uint64_t gg;             // gcd(n_P, n_Q): num(o) = gg * red(o), red = |c_P aQ - c_Q bP| (DIFF: |counter|)
    int64_t aQ, bP;          // n_Q / gg, n_P / gg
    const float* boxes;      // kd-ordered mode: [n_tiles][KX][2] min / max of dims < KX per TILE rows, else nullptr
    const int32_t* perm;     // kd-ordered mode: perm[j] = pooled index of sorted origin j; per_origin is then a
                             // full [N] array in pooled order (else nullptr: per_origin indexed o - o_begin)
    unsigned long long* hist;  // SPLIT only, or nullptr: hist[item * hist_stride + c_Q] += 1 for every (origin,
                               // orthant) cell (the M_T histogram of the analytic significance, ddks_significance.cuh)
    int64_t hist_stride;       // n_Q + 1 (one histogram per batch item)
    // profiling (or nullptr): [0] += SM cycles and [1] += globaltimer ns of every CTA's count loop, [2] += FP32
    // compares executed (every lane of every warp, decided kd / WX bits excluded: the work the ALU pipe really did)
    unsigned long long* clk = nullptr;
};

// decode the two signed 16-bit halves of a counter word (value = lo + 65536 * hi, both in int16 range)
__device__ __forceinline__ void split16(uint32_t w, int32_t& lo, int32_t& hi) {
    lo = (int32_t)(int16_t)(w & 0xffffu);
    hi = ((int32_t)w - lo) >> 16;
}

// hist[v] += 1 for every active lane, one atomic per distinct v in the warp (the popular small counts of the
// significance histogram would otherwise serialise on a few addresses)
__device__ __forceinline__ void hist_add_aggregated(unsigned long long* hist, int64_t v) {
    const uint32_t mask = __activemask();
    const uint32_t peers = __match_any_sync(mask, (unsigned long long)v);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[v], (unsigned long long)__popc(peers));
}

// red(o) = num(o) / gcd(n_P, n_Q) of origin r of thread t from the SMEM counters (direct mode)
template <int D, bool SPLIT, bool SMALL>
__device__ __forceinline__ uint64_t origin_red(const uint32_t* hist, int r, int t, const CountArgs& a, int64_t item) {
    using G = Geo<D, SPLIT, SMALL>;
    constexpr int NQ = G::NQ;
    const int sl = G::slot(r, t);
    const bool high = G::high(r, t);
    uint64_t best = 0;
    for (int q = 0; q < NQ; ++q) {
        int32_t lo, hi;
        split16(hist[q * G::WPB + sl], lo, hi);
        const int32_t v = high ? hi : lo;
        if constexpr (!SPLIT) {
            const uint64_t av = (uint64_t)(v < 0 ? -v : v);
            best = av > best ? av : best;
        } else {
            int32_t lo2, hi2;
            split16(hist[(NQ + q) * G::WPB + sl], lo2, hi2);
            const int64_t cQ = high ? hi2 : lo2;
            if (a.hist) hist_add_aggregated(a.hist, item * a.hist_stride + cQ);
            const int64_t df = (int64_t)v * a.aQ - cQ * a.bP;
            const uint64_t av = (uint64_t)(df < 0 ? -df : df);
            best = av > best ? av : best;
        }
    }
    return best;
}

// Float-encoded counter address of the pair (origin o, point x): base + sum_k [x_k >= o_k] * 4 * 2^k * WPB, as d
// FSET.BF (ALU pipe) + d FFMA-immediate (FMA pipe); exact, every partial sum is an integer < 2^24.
// kd ordering (KX > 0): dims k < KX whose bit was decided for the whole tile (bit k of UM clear) are not compared;
// their weight is folded into base by the caller. Dims k >= KX are always compared.
template <int KX, int UM> __host__ __device__ constexpr bool cmp_dim(int k) { return k >= KX || ((UM >> k) & 1); }
template <int D, int KX, int UM> __host__ __device__ constexpr int n_cmp() {
    int c = 0;
    for (int k = 0; k < D; ++k) c += cmp_dim<KX, UM>(k) ? 1 : 0;
    return c;
}

// the i-th compared dim (ascending), -1 if fewer
template <int D, int KX, int UM> __host__ __device__ constexpr int cmp_dim_idx(int i) {
    for (int k = 0; k < D; ++k)
        if (cmp_dim<KX, UM>(k)) {
            if (i == 0) return k;
            --i;
        }
    return -1;
}

template <int D, bool GT, int WPB, int KX = 0, int UM = 0, bool SPLIT_CHAIN = (D >= 6)>
__device__ __forceinline__ float code_addr(const float (&x)[D], const float (&o)[D], float base) {
    constexpr int NC = n_cmp<D, KX, UM>();
    if constexpr (SPLIT_CHAIN && NC >= 4) {
        // two half-length FFMA chains shorten the dependency chain when few warps are resident (d >= 6 keeps 256+
        // counters per origin in SMEM)
        float f0 = base, f1 = 0.0f;
        int c = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (!cmp_dim<KX, UM>(k)) continue;
            const float w = (float)(4 * (1 << k) * WPB);
            if (c < NC / 2) f0 = fmaf(cmp_bit<GT>(x[k], o[k]), w, f0);
            else            f1 = fmaf(cmp_bit<GT>(x[k], o[k]), w, f1);
            ++c;
        }
        return f0 + f1;
    } else {
        float f = base;
#pragma unroll
        for (int k = 0; k < D; ++k)
            if (cmp_dim<KX, UM>(k)) f = fmaf(cmp_bit<GT>(x[k], o[k]), (float)(4 * (1 << k) * WPB), f);
        return f;
    }
}

// Classify + count the points [lo, hi) of one SMEM tile for the R origins of this thread.
// Per pair: D x FSET.BF (ALU) + D x FFMA-immediate (FMA) + 1 x ATOMS.ADD; the next point(s) are prefetched.
// base[r % NB_] is the float-encoded address of origin slot r's bin-0 word; weights 4 * 2^k * WPB. inc_lo / inc_hi:
// the increment for low-half / high-half origins (R == 1: the caller passes this thread's increment in both).
// With R <= 2 origins per thread two points are classified per step, so a warp has 2R independent chains in flight.
// SMEM counter increment at the float-encoded byte offset f (debug builds check it lies inside the counters)
__device__ __forceinline__ void red_counter(float f, uint32_t ubase, uint32_t inc, uint32_t hbytes) {
    DDKS_ASSERT(__float_as_uint(f) - 0x4B000000u < hbytes);
    (void)hbytes;
    red_add_shared(__float_as_uint(f) + ubase, inc);
}

template <int D, bool GT, int R, int RP, int NB_, int WPB, int DP, int KX = 0, int UM = 0>
__device__ __forceinline__ void count_points(const float* tile, int lo, int hi, const float (&o)[R][D],
                                             const float (&base)[NB_], uint32_t ubase, uint32_t inc_lo,
                                             uint32_t inc_hi, uint32_t hbytes) {
    if (lo >= hi) return;
    int p = lo;
    // prefetches read at most PPS (<= 4) points past hi <= TILE: still inside the SMEM allocation (the next stage or the
    // counters), and the values are never used
#ifndef DDKS_NO_ONEDIM
    if constexpr (KX > 0 && UM == 0 && n_cmp<D, KX, UM>() == 1 && R >= 2) {
        // kd tile with every sorted bit decided and ONE compared dim left (d = 5 at K = 4: x_4): every pair is still
        // classified by its own compare, and its increment goes to one of two counters of the origin; the compare bit
        // (FSET.BF, 1.0 / 0.0) is accumulated in a float register (FADD: exact, <= TILE) and the two counters are
        // updated once per origin and tile part with the exact totals -- per pair 1 FSET + 1 FADD instead of
        // FSET + FFMA + ATOMS, on the ALU and FMA pipes in balance.
        constexpr int K1 = KX;  // the compared dim (D == KX + 1)
        constexpr float W1 = (float)(4 * (1 << K1) * WPB);
        float sacc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) sacc[r] = 0.0f;
        float xn = tile[p * DP + K1];
#pragma unroll 8
        for (; p < hi; ++p) {
            const float x = xn;
            xn = tile[(p + 1) * DP + K1];
#pragma unroll
            for (int r = 0; r < R; ++r) sacc[r] += cmp_bit<GT>(x, o[r][K1]);
        }
        const uint32_t n = (uint32_t)(hi - lo);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t inc = (r < RP) ? inc_lo : inc_hi;
            const uint32_t n1 = (uint32_t)sacc[r];
            if (n1) red_counter(base[r % NB_] + W1, ubase, inc * n1, hbytes);
            if (n1 != n) red_counter(base[r % NB_], ubase, inc * (n - n1), hbytes);
        }
        return;
    }
#endif
#if DDKS_TWODIM
    if constexpr (KX > 0 && n_cmp<D, KX, UM>() == 2 && R >= 2) {
        // kd tile with TWO compared dims left (one open sorted dim + the unsorted last dim at d = K + 1): every pair
        // is still classified by its own two compares, and its increment goes to one of four counters of the
        // origin; the compare bits a, b (FSET.BF, 1.0 / 0.0) are accumulated as sum a, sum b and sum ab (FADD, FADD,
        // FFMA; exact, <= TILE) and the four counters receive the exact totals once per origin and tile part:
        // n11 = sum ab, n10 = sum a - sum ab, n01 = sum b - sum ab, n00 = n - sum a - sum b + sum ab.
        constexpr int C0 = cmp_dim_idx<D, KX, UM>(0), C1 = cmp_dim_idx<D, KX, UM>(1);
        constexpr float W0 = (float)(4 * (1 << C0) * WPB), W1 = (float)(4 * (1 << C1) * WPB);
        float sa[R], sb[R], sab[R];
#pragma unroll
        for (int r = 0; r < R; ++r) sa[r] = 0.0f, sb[r] = 0.0f, sab[r] = 0.0f;
        float xa = tile[p * DP + C0], xb = tile[p * DP + C1];
#pragma unroll 8
        for (; p < hi; ++p) {
            const float x0 = xa, x1 = xb;
            xa = tile[(p + 1) * DP + C0];
            xb = tile[(p + 1) * DP + C1];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float ba = cmp_bit<GT>(x0, o[r][C0]), bb = cmp_bit<GT>(x1, o[r][C1]);
                sa[r] += ba;
                sb[r] += bb;
                sab[r] = fmaf(ba, bb, sab[r]);
            }
        }
        const uint32_t n = (uint32_t)(hi - lo);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t inc = (r < RP) ? inc_lo : inc_hi;
            const uint32_t n11 = (uint32_t)sab[r], na = (uint32_t)sa[r], nb = (uint32_t)sb[r];
            const uint32_t n10 = na - n11, n01 = nb - n11, n00 = n - na - nb + n11;
            const float b0 = base[r % NB_];
            if (n00) red_counter(b0, ubase, inc * n00, hbytes);
            if (n10) red_counter(b0 + W0, ubase, inc * n10, hbytes);
            if (n01) red_counter(b0 + W1, ubase, inc * n01, hbytes);
            if (n11) red_counter(b0 + W0 + W1, ubase, inc * n11, hbytes);
        }
        return;
    }
#endif
    if constexpr (R <= 2) {
        // PPS points per step (R == 1: DDKS_R1_PTS), the next PPS loaded before this step's compares: a warp has
        // PPS * R independent address chains in flight
        constexpr int PPS = R == 1 ? DDKS_R1_PTS : 2;
        float nx[PPS][D];
#pragma unroll
        for (int j = 0; j < PPS; ++j) load_point<D>(tile + (p + j) * DP, nx[j]);
#pragma unroll 4
        for (; p + PPS - 1 < hi; p += PPS) {
            float x[PPS][D];
#pragma unroll
            for (int j = 0; j < PPS; ++j)
#pragma unroll
                for (int k = 0; k < D; ++k) x[j][k] = nx[j][k];
#pragma unroll
            for (int j = 0; j < PPS; ++j) load_point<D>(tile + (p + PPS + j) * DP, nx[j]);
            float f[PPS][R];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int j = 0; j < PPS; ++j)  // PPS points in flight already give independent chains: no split
                    f[j][r] = code_addr<D, GT, WPB, KX, UM, false>(x[j], o[r], base[r % NB_]);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t inc = (R >= 2 && r < RP) ? inc_lo : inc_hi;
#pragma unroll
                for (int j = 0; j < PPS; ++j) red_counter(f[j][r], ubase, inc, hbytes);
            }
        }
#pragma unroll
        for (int j = 0; j < PPS - 1; ++j) {
            if (p + j < hi) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    red_counter(code_addr<D, GT, WPB, KX, UM>(nx[j], o[r], base[r % NB_]), ubase,
                                (R >= 2 && r < RP) ? inc_lo : inc_hi, hbytes);
            }
        }
        return;
    }
    float xn[D];
    load_point<D>(tile + p * DP, xn);
    // K = 4 has 16 loop variants: with R >= 8 origins per thread (large bodies) the ones with undecided dims are
    // unrolled 4 deep to relieve the instruction cache (C5: 840 -> 827 ms; K = 3, or R = 4 at d = 6, do better with
    // the full unroll)
    constexpr int UNR = (KX > 0 && UM != 0) ? ((KX >= 4 && R >= 8) ? 4 : DDKS_UNROLL_PARTIAL) : kUnrollPts;
#pragma unroll UNR
    for (; p < hi; ++p) {
        float x[D];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = xn[k];
        load_point<D>(tile + (p + 1) * DP, xn);
#pragma unroll
        for (int r = 0; r < R; ++r)
            red_counter(code_addr<D, GT, WPB, KX, UM>(x, o[r], base[r % NB_]), ubase,
                        (R >= 2 && r < RP) ? inc_lo : inc_hi, hbytes);
    }
}

// Loop variants instantiated for KX levels: every undecided-dims mask for KX <= 4 (restricting K = 4 to <= 2 open dims
// measured 1 % slower); for KX = 5 only the masks with at most 2 undecided dims (plus "all undecided"), 17 variants
// instead of 32; a tile with more open dims is counted by the all-undecided variant (the caller drops its decided
// weights).
#ifndef DDKS_KD_OPEN4  // experiments: open dims instantiated for K = 4
#define DDKS_KD_OPEN4 4
#endif
__host__ __device__ constexpr int kd_max_open(int KX) { return KX >= 5 ? 2 : (KX == 4 ? DDKS_KD_OPEN4 : KX); }
__host__ __device__ constexpr int popc_c(int v) { return v ? (v & 1) + popc_c(v >> 1) : 0; }

// count_points for the undecided-dims mask um (one instantiation per instantiated mask; um is warp-uniform)
template <int D, bool GT, int R, int RP, int NB_, int WPB, int DP, int KX, int UM = (1 << KX) - 1>
__device__ __forceinline__ void count_points_um(int um, const float* tile, int lo, int hi, const float (&o)[R][D],
                                                const float (&base)[NB_], uint32_t ubase, uint32_t inc_lo,
                                                uint32_t inc_hi, uint32_t hbytes) {
    if constexpr (UM == 0) {
        count_points<D, GT, R, RP, NB_, WPB, DP, KX, 0>(tile, lo, hi, o, base, ubase, inc_lo, inc_hi, hbytes);
    } else {
        if constexpr (popc_c(UM) <= kd_max_open(KX) || UM == (1 << KX) - 1) {
            if (um == UM) {
                count_points<D, GT, R, RP, NB_, WPB, DP, KX, UM>(tile, lo, hi, o, base, ubase, inc_lo, inc_hi, hbytes);
                return;
            }
        }
        count_points_um<D, GT, R, RP, NB_, WPB, DP, KX, UM - 1>(um, tile, lo, hi, o, base, ubase, inc_lo, inc_hi, hbytes);
    }
}

// KX > 0 (kd ordering): the rows are in kd order (label-major, hierarchically sorted by x_0 .. x_{KX-1}, see k_kd_keys;
// a.perm maps a row back to its pooled index) and a.boxes holds every tile's [min, max] of dims < KX. Bit k < KX is
// decided for a whole tile when the tile's x_k range does not interleave with the CTA's origins' (DESIGN.md §7
// "kd ordering"); only the undecided dims are compared.
//
// WX (batches of small items, rows of every label run pre-sorted by x_0, see k_pack_sorted): each warp owns 32 R
// consecutive origins of the sorted order, and bit 0 is decided per (warp, 32-point sub-tile) when the sub-tile's
// x_0 range does not interleave with the warp's -- the kd idea at warp granularity inside one item.
// Resident CTAs per SM the register budget must allow: 3 for the position-ordered d <= 4 counts (their SMEM -- tiles +
// 32 KB of counters -- fits 3; measured C2: 117 us at 3 CTAs/SM vs 150 us when the registers allowed only 2), else 1.
template <int D, int KX, bool SMALL> __host__ __device__ constexpr int count_min_blocks() {
    return SMALL ? 4 : ((D <= 4 && KX == 0) ? 3 : 1);
}

template <int D, bool SPLIT, bool GT, int KX = 0, bool WX = false, bool SMALL = false>
__global__ void __launch_bounds__(Geo<D, SPLIT, SMALL>::T, count_min_blocks<D, KX, SMALL>()) k_count(const CountArgs a) {
    static_assert(!(WX && KX > 0), "WX and KX are exclusive");
    static_assert(KX <= 5 && KX <= D, "at most 5 kd levels");
    using G = Geo<D, SPLIT, SMALL>;
    constexpr int R = G::R, RP = G::RP, T = G::T, DP = G::DP, TILE = G::TILE, S = G::S, NBASE = G::NBASE,
                  WPB = G::WPB;
    extern __shared__ __align__(128) uint8_t smem[];
    float* tiles = reinterpret_cast<float*>(smem);                                  // [S][TILE][DP]
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + S * G::TILE_BYTES);          // [NB][WPB]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * G::TILE_BYTES + G::HIST_WORDS * 4);

    // grid: x = point segment (fastest, so the CTAs in flight share origin blocks and their accumulators stay
    // L2-resident), y = origin block, z = item
    const int t = threadIdx.x;
    const int64_t item = blockIdx.z;
    const float* pts = a.pts + item * a.item_stride;
    const int32_t by = a.blk_base + (int32_t)blockIdx.y;  // origin block of this launch
    const int32_t blk_o0 = a.o_begin + (by * a.blk_stride + a.blk_off) * G::ORIGINS;
    const int32_t li0 = by * G::ORIGINS;  // this CTA's first accumulator slot
    const int32_t seg0 = (int32_t)blockIdx.x * a.seg_points;
    const int32_t seg1 = min(a.N, seg0 + a.seg_points);
    const int n_tiles = (seg1 - seg0 + TILE - 1) / TILE;

    __shared__ uint32_t done_cnt[S];  // warps done with each stage (monotone over the rounds)
    __shared__ unsigned long long s_exec;  // profiling: this CTA's executed compares
    if (t == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1), done_cnt[s] = 0u;
        s_exec = 0ull;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = t; i < G::HIST_WORDS; i += T) hist[i] = 0u;
    __syncthreads();

    if (t == 0) {  // prologue: fill the ring
        for (int s = 0; s < S && s < n_tiles; ++s) {
            const int32_t p0 = seg0 + s * TILE;
            const uint32_t bytes = (uint32_t)(min(TILE, seg1 - p0) * DP * 4);
            mbar_expect_tx(&bars[s], bytes);
            bulk_g2s(tiles + s * TILE * DP, pts + (int64_t)p0 * DP, bytes, &bars[s]);
        }
    }

    // origins of this thread: slot r -> o = blk_o0 + r*T + t (WX: blk_o0 + warp*32R + r*32 + lane, so a warp's
    // origins are consecutive), clamped to a valid origin (ignored at the end); counters stay in slot (r, t)
    const int lane = t & 31, warp = t >> 5;
    auto origin_of = [&](int r) -> int32_t {
        return (WX || KX > 0) ? blk_o0 + warp * (32 * R) + r * 32 + lane : blk_o0 + r * T + t;
    };
    float o[R][D];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int32_t oi = origin_of(r);
        oi = oi < a.o_end ? oi : a.o_end - 1;
        const float* op = pts + (int64_t)oi * DP;
#pragma unroll
        for (int k = 0; k < D; ++k) o[r][k] = __ldg(op + k);
    }

    // the counter byte address lives in the mantissa of a float in [2^23, 2^24): bits = 0x4B000000 + offset
    const uint32_t ubase = smem_u32(hist) - 0x4B000000u;
    float baseP[NBASE], baseQ[NBASE];
#pragma unroll
    for (int b = 0; b < NBASE; ++b) {
        const uint32_t sl = (uint32_t)G::slot(b, t);
        baseP[b] = __uint_as_float(0x4B000000u + 4u * sl);
        baseQ[b] = SPLIT ? __uint_as_float(0x4B000000u + 4u * (uint32_t)(G::NQ * WPB + sl)) : baseP[b];
    }
    const uint32_t incP_hi = a.incP << 16, incQ_hi = a.incQ << 16;
    // R == 1: this thread's single origin is a low or a high half for its whole life
    const uint32_t incP_lo = (R == 1 && G::high(0, t)) ? incP_hi : a.incP;
    const uint32_t incQ_lo = (R == 1 && G::high(0, t)) ? incQ_hi : a.incQ;
    // KX > 0: the box [cmin, cmax] of dims < KX over this CTA's origins (clamped slots repeat o_end - 1, which is in
    // the last block), block-reduced once
    constexpr int KB = KX > 0 ? KX : 1;
    float cmin[KB], cmax[KB];
    if constexpr (KX > 0) {
        __shared__ float sbox[32][2 * KB];
#pragma unroll
        for (int k = 0; k < KX; ++k) {
            float lo = o[0][k], hi = o[0][k];
#pragma unroll
            for (int r = 1; r < R; ++r) lo = fminf(lo, o[r][k]), hi = fmaxf(hi, o[r][k]);
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
                hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
            }
            if ((t & 31) == 0) sbox[t >> 5][2 * k] = lo, sbox[t >> 5][2 * k + 1] = hi;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < KX; ++k) {
            cmin[k] = sbox[0][2 * k], cmax[k] = sbox[0][2 * k + 1];
            for (int w = 1; w < T / 32; ++w) cmin[k] = fminf(cmin[k], sbox[w][2 * k]), cmax[k] = fmaxf(cmax[k], sbox[w][2 * k + 1]);
        }
    }
    // WX: the x_0 range of this warp's origins; KX > 0: the range of the last sorted dim x_{KX-1}, in which a warp's
    // 32 R consecutive origins are far narrower than the CTA's (the bit is then decided per warp and tile)
    constexpr int WD = KX > 0 ? KX - 1 : 0;
    float xw_lo = 0.0f, xw_hi = 0.0f;
    if constexpr (WX || KX > 0) {
        xw_lo = o[0][WD], xw_hi = o[0][WD];
#pragma unroll
        for (int r = 1; r < R; ++r) xw_lo = fminf(xw_lo, o[r][WD]), xw_hi = fmaxf(xw_hi, o[r][WD]);
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) {
            xw_lo = fminf(xw_lo, __shfl_xor_sync(0xffffffffu, xw_lo, sh));
            xw_hi = fmaxf(xw_hi, __shfl_xor_sync(0xffffffffu, xw_hi, sh));
        }
    }
    // the tile box of the next tile is loaded one iteration ahead (tiles are TILE-aligned from row 0)
    float bnext[2 * KB];
    if constexpr (KX > 0) {
#pragma unroll
        for (int k = 0; k < 2 * KX; ++k) bnext[k] = __ldg(a.boxes + (int64_t)(seg0 / TILE) * 2 * KX + k);
    }

    // in-kernel clock probe (profiling only; one lane of every 8th CTA -- the clk / ns ratio needs a sample, and
    // thousands of same-address atomics at the kernel tail cost ~8 us at C2): the SM clock this launch ran at
    const bool probe = a.clk && t == 0 && ((blockIdx.x + blockIdx.y) & 7) == 0;
    unsigned long long clk0 = 0, ns0 = 0;
    if (probe) clk0 = clock64(), ns0 = globaltimer_ns();
    unsigned long long exec_cmp = 0;  // profiling: compares this warp executed / (32 R)

    for (int it = 0; it < n_tiles; ++it) {
        const int s = it % S;
        mbar_wait(&bars[s], (uint32_t)((it / S) & 1));
        const float* tile = tiles + s * TILE * DP;
        const int32_t p0 = seg0 + it * TILE;
        const int32_t cnt = min(TILE, seg1 - p0);
        // sample-homogeneous sub-ranges: [p0, n_P) are P points, [n_P, ...) are Q points
        int32_t split = a.n_P - p0;
        split = split < 0 ? 0 : (split > cnt ? cnt : split);
        // undecided dims among the first KX (bit k of um) and the weight of the bits decided as 1
        int um = (1 << KX) - 1;
        float add = 0.0f;
        if constexpr (KX > 0) {
            float bx[2 * KX];
#pragma unroll
            for (int k = 0; k < 2 * KX; ++k) bx[k] = bnext[k];
            if (it + 1 < n_tiles) {
#pragma unroll
                for (int k = 0; k < 2 * KX; ++k) bnext[k] = __ldg(a.boxes + (int64_t)(p0 / TILE + 1) * 2 * KX + k);
            }
#pragma unroll
            for (int k = 0; k < KX; ++k) {
                // bit k = [x_k >= o_k] (GT: >) is uniform over tile x origins when the ranges do not interleave
                if (GT ? (bx[2 * k + 1] <= cmin[k]) : (bx[2 * k + 1] < cmin[k])) {
                    um &= ~(1 << k);
                } else if (GT ? (bx[2 * k] > cmax[k]) : (bx[2 * k] >= cmax[k])) {
                    um &= ~(1 << k);
                    add += (float)(4 * (1 << k) * WPB);  // exact: integers < 2^24
                }
            }
            // still open at CTA level: the last sorted dim against this warp's own (narrow) origin range
            if ((um >> WD) & 1) {
                if (GT ? (bx[2 * WD + 1] <= xw_lo) : (bx[2 * WD + 1] < xw_lo)) {
                    um &= ~(1 << WD);
                } else if (GT ? (bx[2 * WD] > xw_hi) : (bx[2 * WD] >= xw_hi)) {
                    um &= ~(1 << WD);
                    add += (float)(4 * (1 << WD) * WPB);
                }
            }
            // more open dims than any instantiated variant: compare them all (and drop the decided weights)
            if constexpr (kd_max_open(KX) < KX) {
                if (__popc(um) > kd_max_open(KX)) um = (1 << KX) - 1, add = 0.0f;
            }
        }
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
            const int lo = part ? split : 0, hi = part ? cnt : split;
            if (lo >= hi) continue;
            float bb[NBASE];
#pragma unroll
            for (int b = 0; b < NBASE; ++b) bb[b] = (part ? baseQ[b] : baseP[b]) + add;
            const uint32_t il = part ? incQ_lo : incP_lo;
            const uint32_t ih = R == 1 ? il : (part ? incQ_hi : incP_hi);
            if constexpr (WX) {
                // 32-point sub-tiles (x_0-sorted within the run): bit 0 decided per warp when the ranges do not meet
                for (int sb = lo; sb < hi; sb += 32) {
                    const int se = min(hi, sb + 32);
                    float mn = tile[min(sb + lane, se - 1) * DP], mx = mn;
#pragma unroll
                    for (int sh = 16; sh; sh >>= 1) {
                        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, sh));
                        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, sh));
                    }
                    int wm = 1;
                    float wadd = 0.0f;
                    if (GT ? (mx <= xw_lo) : (mx < xw_lo)) {
                        wm = 0;
                    } else if (GT ? (mn > xw_hi) : (mn >= xw_hi)) {
                        wm = 0;
                        wadd = (float)(4 * WPB);
                    }
                    float wb[NBASE];
#pragma unroll
                    for (int b = 0; b < NBASE; ++b) wb[b] = bb[b] + wadd;
                    if (a.clk) exec_cmp += (unsigned long long)((D - 1 + wm) * (se - sb));
                    count_points_um<D, GT, R, RP, NBASE, WPB, DP, 1>(wm, tile, sb, se, o, wb, ubase, il, ih,
                                                                    G::HIST_WORDS * 4u);
                }
            } else {
                if (a.clk) exec_cmp += (unsigned long long)((D - KX + __popc(um)) * (hi - lo));
                count_points_um<D, GT, R, RP, NBASE, WPB, DP, KX>(um, tile, lo, hi, o, bb, ubase, il, ih,
                                                                 G::HIST_WORDS * 4u);
            }
        }
        // kd counts (per-warp loop variants): release stage s without a CTA barrier -- the last warp done with it
        // refills it, so warps may drift up to S - 1 tiles apart instead of waiting at every tile. Measured (count
        // kernel): C5 724 -> 711 ms, d = 7 / 8 at N = 4e5 -3 %, d = 6 +9 % and the position-ordered C2 / C3 +4 %
        // (lockstep warps keep the full S - 1 tiles of TMA slack), so those keep the barrier.
        constexpr bool WREL = KX > 0 && D != 6;
        if constexpr (!WREL) {
            __syncthreads();  // every thread is done with stage s
            if (t == 0 && it + S < n_tiles) {
                fence_proxy_async();
                const int32_t q0 = seg0 + (it + S) * TILE;
                const uint32_t bytes = (uint32_t)(min(TILE, seg1 - q0) * DP * 4);
                mbar_expect_tx(&bars[s], bytes);
                bulk_g2s(tiles + s * TILE * DP, pts + (int64_t)q0 * DP, bytes, &bars[s]);
            }
            continue;
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            const uint32_t prev = atomicAdd(&done_cnt[s], 1u);  // monotone: round it / S ends at (round + 1) * warps
            if (prev == (uint32_t)((it / S + 1) * (T / 32) - 1) && it + S < n_tiles) {
                __threadfence_block();
                fence_proxy_async();
                const int32_t q0 = seg0 + (it + S) * TILE;
                const uint32_t bytes = (uint32_t)(min(TILE, seg1 - q0) * DP * 4);
                mbar_expect_tx(&bars[s], bytes);
                bulk_g2s(tiles + s * TILE * DP, pts + (int64_t)q0 * DP, bytes, &bars[s]);
            }
        }
    }
    if (a.clk && lane == 0) atomicAdd(&s_exec, exec_cmp * (unsigned long long)(32 * R));
    __syncthreads();  // all red.shared retired before reading the counters
    if (a.clk && t == 0) {
        atomicAdd(&a.clk[2], s_exec);  // one global atomic per CTA
        if (probe) {
            atomicAdd(&a.clk[0], (unsigned long long)(clock64() - clk0));
            atomicAdd(&a.clk[1], globaltimer_ns() - ns0);
        }
    }

    // per-origin epilogue shared by both modes: num(o) -> per-origin export, the CTA max, the packed argmax key
    uint64_t best = 0;
    unsigned long long bkey = 0;
    auto take = [&](int32_t oi, uint64_t red) {
        const int32_t pooled = a.perm ? a.perm[oi] : oi;
        const uint64_t m = red * a.gg;
        if (a.per_origin) a.per_origin[a.perm ? pooled : oi - a.o_begin] = m;
        best = m > best ? m : best;
        if (a.best_key) {
            const unsigned long long k = ((unsigned long long)red << 31) | (unsigned long long)(0x7fffffff - pooled);
            bkey = k > bkey ? k : bkey;
        }
    };

    if (a.accum != nullptr) {
        // flush: exact int32 partial counters -> global (red.global.add, fire-and-forget: the CTA exits while they
        // drain; measured: a last-CTA-finalises variant that fences here made C3 +14 % and C5 +14 % slower)
        int32_t* acc = a.accum + item * (int64_t)G::NB * a.acc_stride;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
            const int32_t oi = origin_of(r);
            if (oi >= a.o_end) continue;
            const int sl = G::slot(r, t);
            const bool hiw = G::high(r, t);
#pragma unroll 4
            for (int q = 0; q < G::NB; ++q) {
                int32_t lo, hi;
                split16(hist[q * WPB + sl], lo, hi);
                const int32_t v = hiw ? hi : lo;
                DDKS_ASSERT(li0 + r * T + t < a.acc_stride && oi >= a.o_begin);
                if (v) atomicAdd(&acc[(int64_t)q * a.acc_stride + (li0 + r * T + t)], v);
            }
        }
        return;  // k_finalize reads the partials once every segment has flushed
    }
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
        const int32_t oi = origin_of(r);
        if (oi >= a.o_end) continue;
        take(oi, origin_red<D, SPLIT, SMALL>(hist, r, t, a, item));
    }
    best = warp_max_u64(best);
    bkey = warp_max_u64(bkey);
    __shared__ uint64_t wmax[32], wkey[32];
    if ((t & 31) == 0) wmax[t >> 5] = best, wkey[t >> 5] = bkey;
    __syncthreads();
    if (t == 0) {
        uint64_t m = 0, k = 0;
        for (int w = 0; w < T / 32; ++w) m = wmax[w] > m ? wmax[w] : m, k = wkey[w] > k ? wkey[w] : k;
        atomicMax(reinterpret_cast<unsigned long long*>(&a.item_num[item]), (unsigned long long)m);
        if (a.best_key) atomicMax(a.best_key, (unsigned long long)k);
    }
}

// ----------------------------------------------------------------------------------------------- kd ordering
// Bit elision (DESIGN.md §7 "kd ordering"). The pooled rows are reordered label-major (P rows, then Q rows, so tiles
// stay sample-homogeneous) and, within each label run, hierarchically: level 0 sorts the run by x_0 and cuts it into
// G0 slabs, level 1 sorts every slab by x_1 and cuts it into G1 cells, level 2 sorts every cell by x_2 (KX levels in
// all). Cut points are rounded to multiples of A = lcm(origins per CTA, TILE), so a CTA's origins and a tile lie in one
// cell. A CTA's origins then span a narrow range of the last sorted dim and one slab / cell range of the others,
// and k_count<KX> decides bit k for a whole tile whenever the tile's x_k range does not interleave with it.
// The order only affects speed: every decision is taken from the actual per-tile and per-CTA min / max.

// cut point i of the run [s, e) into G parts, rounded to a multiple of A (monotone in i; cut 0 = s, cut G = e)
__device__ __forceinline__ int64_t kd_cut(int64_t s, int64_t e, int64_t G, int64_t i, int64_t A) {
    if (i <= 0) return s;
    if (i >= G) return e;
    const int64_t x = s + (e - s) * i / G;
    const int64_t r = (x + A / 2) / A * A;
    return r < s ? s : (r > e ? e : r);
}
// the part of [s, e) holding row j: the largest i < G with kd_cut(i) <= j
__device__ __forceinline__ int64_t kd_part(int64_t j, int64_t s, int64_t e, int64_t G, int64_t A) {
    int64_t i = e > s ? (j - s) * G / (e - s) : 0;
    i = i < 0 ? 0 : (i >= G ? G - 1 : i);
    while (i + 1 < G && kd_cut(s, e, G, i + 1, A) <= j) ++i;
    while (i > 0 && kd_cut(s, e, G, i, A) > j) --i;
    return i;
}

// keys of level `level` (0 <= level < 5) for rows already in the order of the previous level:
// key = label (1 bit) | cell of the previous levels (cb bits) | the top kb bits of f32_key(x_level) | ... | row index
// (low ib bits; kb <= 63 - cb - ib). A stable LSD sort of the top 1 + cb + kb bits gives the level's order (ties keep
// the previous order); kb < 32 only coarsens the order inside a cell, which changes speed, never counts.
__global__ void k_kd_keys(const float* __restrict__ pts, int DP, int64_t N, int64_t n_P, int level, int64_t G0,
                          int64_t G1, int64_t G2, int64_t G3, int64_t A, int ib, int cb, int kb,
                          uint64_t* __restrict__ keys) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        const bool lab = j >= n_P;
        const int64_t s = lab ? n_P : 0, e = lab ? N : n_P;
        uint64_t cell = 0;
        if (level >= 1) {
            const int64_t i0 = kd_part(j, s, e, G0, A);
            cell = (uint64_t)i0;
            if (level >= 2) {
                const int64_t s1 = kd_cut(s, e, G0, i0, A), e1 = kd_cut(s, e, G0, i0 + 1, A);
                const int64_t i1 = kd_part(j, s1, e1, G1, A);
                cell = (uint64_t)(i0 * G1 + i1);
                if (level >= 3) {
                    const int64_t s2 = kd_cut(s1, e1, G1, i1, A), e2 = kd_cut(s1, e1, G1, i1 + 1, A);
                    const int64_t i2 = kd_part(j, s2, e2, G2, A);
                    cell = cell * (uint64_t)G2 + (uint64_t)i2;
                    if (level >= 4) {
                        const int64_t s3 = kd_cut(s2, e2, G2, i2, A), e3 = kd_cut(s2, e2, G2, i2 + 1, A);
                        cell = cell * (uint64_t)G3 + (uint64_t)kd_part(j, s3, e3, G3, A);
                    }
                }
            }
        }
        uint64_t k = f32_key(pts[j * DP + level]);
        if (kb < 32) k >>= (32 - kb);
        keys[j] = ((uint64_t)lab << 63) | (cb ? cell << (63 - cb) : 0ull) | (k << (63 - cb - kb)) | (uint64_t)j;
    }
}

// ---- mid-N kd ordering by bucket counting sorts (N < 80000; DESIGN.md §7 "kd ordering, mid N") -------------------
// Level l reorders every (label, cell of the previous levels) run by x_l quantised to KB_NBK equal-width buckets of the
// label's [min, max] of x_l: one histogram, one scan, one scatter instead of the radix sort's ~17 launches per level.
// Rows of a bucket keep an arbitrary order (atomic slots) -- the order only changes speed, never counts.
constexpr int KB_NBK = 1024;

__global__ void k_kdb_range_init(unsigned int* rng, int pairs) {
    for (int i = threadIdx.x; i < pairs; i += blockDim.x) rng[2 * i] = ~0u, rng[2 * i + 1] = 0u;
}

// rng[(lab * K + k) * 2 + {0, 1}] = order-preserving keys of min / max of x_k over the label's rows (init ~0 / 0)
__global__ void k_kdb_range(const float* __restrict__ pts, int DP, int64_t N, int64_t n_P, int K,
                            unsigned int* __restrict__ rng) {
    for (int k = 0; k < K; ++k) {
        unsigned int lo[2] = {~0u, ~0u}, hi[2] = {0u, 0u};
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
            const unsigned int v = f32_key(pts[j * DP + k]);
            const int lab = j >= n_P;
            lo[lab] = v < lo[lab] ? v : lo[lab];
            hi[lab] = v > hi[lab] ? v : hi[lab];
        }
#pragma unroll
        for (int lab = 0; lab < 2; ++lab) {
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                lo[lab] = min(lo[lab], __shfl_xor_sync(0xffffffffu, lo[lab], sh));
                hi[lab] = max(hi[lab], __shfl_xor_sync(0xffffffffu, hi[lab], sh));
            }
            if ((threadIdx.x & 31) == 0) {
                atomicMin(&rng[(lab * K + k) * 2], lo[lab]);
                atomicMax(&rng[(lab * K + k) * 2 + 1], hi[lab]);
            }
        }
    }
}

// the (label, cell, bucket) key of row j at level `level` (cells: position cuts of the previous levels, as k_kd_keys)
__device__ __forceinline__ uint32_t kdb_key(const float* pts, int DP, int64_t j, int64_t N, int64_t n_P, int level,
                                            int K, int64_t G0, int64_t G1, int64_t G2, int64_t A, int64_t cells,
                                            const unsigned int* rng) {
    const bool lab = j >= n_P;
    const int64_t s = lab ? n_P : 0, e = lab ? N : n_P;
    int64_t cell = 0;
    if (level >= 1) {
        const int64_t i0 = kd_part(j, s, e, G0, A);
        cell = i0;
        if (level >= 2) {
            const int64_t s1 = kd_cut(s, e, G0, i0, A), e1 = kd_cut(s, e, G0, i0 + 1, A);
            const int64_t i1 = kd_part(j, s1, e1, G1, A);
            cell = i0 * G1 + i1;
            if (level >= 3) {
                const int64_t s2 = kd_cut(s1, e1, G1, i1, A), e2 = kd_cut(s1, e1, G1, i1 + 1, A);
                cell = cell * G2 + kd_part(j, s2, e2, G2, A);
            }
        }
    }
    const float lo = key_f32(rng[((int)lab * K + level) * 2]), hi = key_f32(rng[((int)lab * K + level) * 2 + 1]);
    const float x = pts[j * DP + level];
    const float scale = hi > lo ? (float)KB_NBK / (hi - lo) : 0.0f;
    const float v = (x - lo) * scale;
    const int b = v >= (float)(KB_NBK - 1) ? KB_NBK - 1 : (v > 0.0f ? (int)v : 0);
    return (uint32_t)((((int64_t)lab * cells + cell) * KB_NBK) + b);
}

__global__ void k_kdb_hist(const float* __restrict__ pts, int DP, int64_t N, int64_t n_P, int level, int K,
                           int64_t G0, int64_t G1, int64_t G2, int64_t A, int64_t cells,
                           const unsigned int* __restrict__ rng, uint32_t* __restrict__ keys,
                           unsigned int* __restrict__ hist) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t key = kdb_key(pts, DP, j, N, n_P, level, K, G0, G1, G2, A, cells, rng);
        keys[j] = key;
        atomicAdd(&hist[key], 1u);
    }
}

// exclusive scan of n bucket counts in place, one CTA of 1024 threads (n <= a few 10^5)
__global__ void __launch_bounds__(1024) k_kdb_scan(unsigned int* __restrict__ hist, int64_t n) {
    __shared__ unsigned int wsum[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t per = (n + 1023) / 1024;
    const int64_t b0 = t * per, b1 = min(n, b0 + per);
    unsigned int sum = 0;
    for (int64_t i = b0; i < b1; ++i) sum += hist[i];
    unsigned int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned int v = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    unsigned int run = x - sum + (w ? wsum[w - 1] : 0u);
    for (int64_t i = b0; i < b1; ++i) {
        const unsigned int c = hist[i];
        hist[i] = run;
        run += c;
    }
}

// row j goes to the next free slot of its key: out[pos] = pts[j], perm_out[pos] = perm_in[j] (perm_in null: j)
__global__ void k_kdb_scatter(const float* __restrict__ pts, int DP, int64_t N, const uint32_t* __restrict__ keys,
                              unsigned int* __restrict__ offs, const int32_t* __restrict__ perm_in,
                              float* __restrict__ out, int32_t* __restrict__ perm_out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pos = atomicAdd(&offs[keys[j]], 1u);
        DDKS_ASSERT(pos < N);
        const float4* src = reinterpret_cast<const float4*>(pts + j * DP);
        float4* dst = reinterpret_cast<float4*>(out + pos * DP);
        dst[0] = src[0];
        if (DP == 8) dst[1] = src[1];
        perm_out[pos] = perm_in ? perm_in[j] : (int32_t)j;
    }
}

// ---- the whole mid-N kd ordering in ONE cooperative launch (k_kdb_fused) -------------------------------------------
// The same bucket counting sorts as k_kdb_range / k_kdb_hist / k_kdb_scan / k_kdb_scatter / k_tile_boxes (identical
// keys, cells and boxes), phase after phase inside one persistent grid separated by grid barriers, instead of ~10
// dependent launches and memsets. The scan of a level's histogram is spread over all CTAs (each scans its chunk;
// the scatter adds the exclusive prefix of the chunk totals, which every CTA forms in SMEM), and the histograms and
// ranges are left zeroed / reset at the end of the launch for the next one (the buffer is zeroed when allocated).
// Launched with the cooperative attribute (every CTA resident, so the barriers cannot deadlock).
constexpr int KDF_T = 512, KDF_MAXB = 1024;  // threads per CTA, CTAs at most (chunk totals in SMEM)
struct KdbFusedArgs {
    const float* pts;              // packed rows [N][DP] (P rows, then Q rows)
    int DP, K;
    int64_t N, n_P, G0, G1, G2, A;
    float* out[2];                 // ping-pong row buffers; level l writes out[(K - 1 - l) & 1] (the last: out[0])
    int32_t* perm[2];              // the same for the permutations (sorted position -> pooled index)
    uint32_t* keys;                // [N] this level's key of every row
    uint32_t* hist;                // levels' histograms back to back: 2 cells_l KB_NBK words each (zero at entry)
    uint32_t* rng;                 // [2 labels][K][2] order-preserving min / max keys (~0 / 0 at entry)
    uint32_t* tot;                 // [gridDim.x] chunk totals of the current level's histogram
    uint32_t* bar;                 // grid barrier {arrived, generation} (arrived 0 between launches)
    float* boxes;                  // [n_tiles][K][2] tile min / max of x_0..x_{K-1}
    int TILE;
};

// sense-reversing grid barrier (all CTAs resident: cooperative launch)
__device__ __forceinline__ void kdf_grid_sync(uint32_t* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t* vb = bar;
        const uint32_t gen = vb[1];
        __threadfence();
        if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
            bar[0] = 0u;
            __threadfence();
            atomicAdd(&bar[1], 1u);
        } else {
            while (vb[1] == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// exclusive scan of h[0, n) in place by one CTA of KDF_T threads (contiguous sub-chunks per thread); returns the total
__device__ __forceinline__ uint32_t kdf_block_scan(uint32_t* h, int64_t n, uint32_t* wsum) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t per = (n + KDF_T - 1) / KDF_T;
    const int64_t b0 = min(n, t * per), b1 = min(n, b0 + per);
    uint32_t sum = 0;
    for (int64_t i = b0; i < b1; ++i) sum += __ldcg(h + i);
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < KDF_T / 32 ? wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < KDF_T / 32) wsum[lane] = v;
    }
    __syncthreads();
    uint32_t run = x - sum + (w ? wsum[w - 1] : 0u);
    const uint32_t total = wsum[KDF_T / 32 - 1];
    for (int64_t i = b0; i < b1; ++i) {
        const uint32_t c = __ldcg(h + i);
        h[i] = run;
        run += c;
    }
    __syncthreads();  // wsum is reused
    return total;
}

__global__ void __launch_bounds__(KDF_T) k_kdb_fused(const KdbFusedArgs a) {
    __shared__ uint32_t wsum[KDF_T / 32];
    __shared__ uint32_t toff[KDF_MAXB];  // exclusive prefix of the chunk totals
    const int64_t gt = blockIdx.x * (int64_t)KDF_T + threadIdx.x, gs = (int64_t)gridDim.x * KDF_T;
    const int K = a.K, DP = a.DP, nb = gridDim.x;
    const int64_t N = a.N, n_P = a.n_P;
    const int64_t gl[3] = {a.G0, a.G1, a.G2};
    // phase 1: per-label min / max of x_0..x_{K-1} (as k_kdb_range)
    for (int k = 0; k < K; ++k) {
        uint32_t lo[2] = {~0u, ~0u}, hi[2] = {0u, 0u};
        for (int64_t j = gt; j < N; j += gs) {
            const uint32_t v = f32_key(a.pts[j * DP + k]);
            const int lab = j >= n_P;
            lo[lab] = v < lo[lab] ? v : lo[lab];
            hi[lab] = v > hi[lab] ? v : hi[lab];
        }
#pragma unroll
        for (int lab = 0; lab < 2; ++lab) {
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                lo[lab] = min(lo[lab], __shfl_xor_sync(0xffffffffu, lo[lab], sh));
                hi[lab] = max(hi[lab], __shfl_xor_sync(0xffffffffu, hi[lab], sh));
            }
            if ((threadIdx.x & 31) == 0) {
                atomicMin(&a.rng[(lab * K + k) * 2], lo[lab]);
                atomicMax(&a.rng[(lab * K + k) * 2 + 1], hi[lab]);
            }
        }
    }
    kdf_grid_sync(a.bar);
    // levels: histogram of the (label, cell, bucket) keys, distributed scan, scatter (as k_kdb_hist / _scan / _scatter)
    const float* src = a.pts;
    const int32_t* src_perm = nullptr;
    int64_t cells = 1, hoff = 0;
    for (int level = 0; level < K; ++level) {
        uint32_t* h = a.hist + hoff;
        const int64_t nk = 2 * cells * KB_NBK;
        const int64_t chunk = (nk + nb - 1) / nb;
        for (int64_t j = gt; j < N; j += gs) {
            const uint32_t key = kdb_key(src, DP, j, N, n_P, level, K, a.G0, a.G1, a.G2, a.A, cells, a.rng);
            a.keys[j] = key;
            atomicAdd(&h[key], 1u);
        }
        kdf_grid_sync(a.bar);
        {
            const int64_t c0 = min(nk, blockIdx.x * chunk), c1 = min(nk, c0 + chunk);
            const uint32_t t = kdf_block_scan(h + c0, c1 - c0, wsum);
            if (threadIdx.x == 0) a.tot[blockIdx.x] = t;
        }
        kdf_grid_sync(a.bar);
        // every CTA: exclusive prefix of the chunk totals in SMEM (nb <= KDF_MAXB)
        for (int i = threadIdx.x; i < nb; i += KDF_T) toff[i] = __ldcg(a.tot + i);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (int i = 0; i < nb; ++i) {
                const uint32_t c = toff[i];
                toff[i] = run;
                run += c;
            }
        }
        __syncthreads();
        const int o = (K - 1 - level) & 1;
        float* dst = a.out[o];
        int32_t* dperm = a.perm[o];
        for (int64_t j = gt; j < N; j += gs) {
            const uint32_t key = a.keys[j];
            const int64_t pos = (int64_t)toff[key / chunk] + atomicAdd(&h[key], 1u);
            DDKS_ASSERT(pos < N);
            const float4* sp = reinterpret_cast<const float4*>(src + j * DP);
            float4* dp = reinterpret_cast<float4*>(dst + pos * DP);
            dp[0] = __ldcg(sp);  // rows written by other CTAs before the barrier: read through L2
            if (DP == 8) dp[1] = __ldcg(sp + 1);
            dperm[pos] = src_perm ? __ldcg(src_perm + j) : (int32_t)j;
        }
        kdf_grid_sync(a.bar);
        src = dst;
        src_perm = dperm;
        hoff += nk;
        cells *= (level < 3 ? gl[level] : 1);
    }
    // tail: 4 zero rows after the last one (the count's prefetch reads them), tile boxes (as k_tile_boxes), and the
    // histograms / ranges reset for the next launch
    for (int64_t i = gt; i < hoff; i += gs) a.hist[i] = 0u;
    if (gt < 2 * K) a.rng[2 * gt] = ~0u, a.rng[2 * gt + 1] = 0u;
    float* fin = a.out[0];
    if (gt < 4 * DP) fin[N * DP + gt] = 0.0f;
    const int64_t n_tiles = (N + a.TILE - 1) / a.TILE;
    const int lane = threadIdx.x & 31;
    for (int64_t w = gt >> 5; w < n_tiles; w += gs >> 5) {
        const int64_t r0 = w * a.TILE, r1 = min(N, r0 + a.TILE);
        for (int k = 0; k < K; ++k) {
            float lo = INFINITY, hi = -INFINITY;
            for (int64_t r = r0 + lane; r < r1; r += 32) {
                const float v = __ldcg(fin + r * DP + k);
                lo = fminf(lo, v), hi = fmaxf(hi, v);
            }
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
                hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
            }
            if (lane == 0) a.boxes[(w * K + k) * 2] = lo, a.boxes[(w * K + k) * 2 + 1] = hi;
        }
    }
}

// out[j] = pts[idx_j] (whole padded rows), perm_out[j] = perm_in[idx_j] (perm_in == nullptr: idx_j), idx_j = the low
// ib bits of the sorted key j (pooled indices < 2^31)
__global__ void k_permute_rows(const float* __restrict__ pts, int DP, int64_t N, const uint64_t* __restrict__ keys,
                               int ib, const int32_t* __restrict__ perm_in, float* __restrict__ out,
                               int32_t* __restrict__ perm_out) {
    const uint64_t mask = (ib >= 64) ? ~0ull : ((1ull << ib) - 1);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = (int64_t)(keys[j] & mask);
        DDKS_ASSERT(idx < N);
        const float4* src = reinterpret_cast<const float4*>(pts + idx * DP);
        float4* dst = reinterpret_cast<float4*>(out + j * DP);
        dst[0] = src[0];
        if (DP == 8) dst[1] = src[1];
        perm_out[j] = perm_in ? perm_in[idx] : (int32_t)idx;
    }
}

// TEST ONLY: row p of each label run [s, s + n) goes to s + (p * m mod n'), with m made coprime to the run length by
// stepping it up (a bijection), rows and permutation together
__device__ __forceinline__ int64_t gcd_i64(int64_t a, int64_t b) {
    while (b) { const int64_t t = a % b; a = b; b = t; }
    return a;
}
__global__ void k_shuffle_runs(const float* __restrict__ pts, const int32_t* __restrict__ perm_in, int DP, int64_t N,
                               int64_t n_P, int64_t m, float* __restrict__ out, int32_t* __restrict__ perm_out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        const bool lab = j >= n_P;
        const int64_t s = lab ? n_P : 0, n = lab ? N - n_P : n_P;
        int64_t mm = m % n;
        if (mm == 0) mm = 1;
        while (gcd_i64(mm, n) != 1) ++mm;
        const int64_t dst = s + (int64_t)(((unsigned __int128)(j - s) * (unsigned __int128)mm) % (unsigned __int128)n);
        const float4* src = reinterpret_cast<const float4*>(pts + j * DP);
        float4* o = reinterpret_cast<float4*>(out + dst * DP);
        o[0] = src[0];
        if (DP == 8) o[1] = src[1];
        perm_out[dst] = perm_in[j];
    }
}

// boxes[t][k] = {min, max} of x_k over rows [t*TILE, min(N, (t+1)*TILE)), k < KX: one warp per tile
__global__ void k_tile_boxes(const float* __restrict__ pts, int DP, int64_t N, int TILE, int KX,
                             float* __restrict__ boxes) {
    const int64_t n_tiles = (N + TILE - 1) / TILE;
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n_tiles;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r0 = w * TILE, r1 = min(N, r0 + TILE);
        for (int k = 0; k < KX; ++k) {
            float lo = INFINITY, hi = -INFINITY;
            for (int64_t r = r0 + lane; r < r1; r += 32) {
                const float v = pts[r * DP + k];
                lo = fminf(lo, v), hi = fmaxf(hi, v);
            }
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
                hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
            }
            if (lane == 0) boxes[(w * KX + k) * 2] = lo, boxes[(w * KX + k) * 2 + 1] = hi;
        }
    }
}

// Finaliser of the accumulate mode: num(o) from the int32 partials of every segment (streaming loads). Per-origin export, the item max and the
// packed argmax key as in k_count's direct epilogue. SPLIT with a.hist (significance): M_T values below HS are
// histogrammed in a block-private SMEM histogram and flushed once per block; larger values (rare) go straight to global.
// A slot's 2^d bins are split over TPS threads (TPS warps of a CTA share 32 consecutive slots, so every load and store
// is coalesced) -- d = 8 has 256 bins per slot and only N slots: one thread per slot left C3's finaliser latency-bound.
constexpr int HS = 2048;

template <int D, bool SPLIT, bool SMALL = false>
__global__ void __launch_bounds__(256) k_finalize(const CountArgs a, int64_t B) {
    using G = Geo<D, SPLIT, SMALL>;
    constexpr int NQ = 1 << D;
    constexpr int NB = G::NB;
    constexpr int TPS = NQ >= 256 ? 8 : (NQ >= 128 ? 4 : (NQ >= 64 ? 2 : 1));  // threads per slot
    constexpr int QPT = NQ / TPS;                                                // bins per thread
    constexpr int SPI = 256 / TPS;                                               // slots per CTA iteration
    const int32_t n_orig = a.o_end - a.o_begin;
    __shared__ uint32_t sh_hist[SPLIT ? HS : 1];
    __shared__ uint64_t sh_red[TPS > 1 ? TPS : 1][TPS > 1 ? SPI : 1];
    const bool priv = SPLIT && a.hist && B == 1;  // a block-private histogram only when every cell is one item's
    if constexpr (SPLIT) {
        if (priv) {
            for (int i = threadIdx.x; i < HS; i += blockDim.x) sh_hist[i] = 0u;
            __syncthreads();
        }
    }
    constexpr int ORIG = G::ORIGINS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int part = warp % TPS, grp = warp / TPS;
    const int64_t ns = a.acc_stride;  // accumulator slots per item
    const int64_t total = B * ns;
    uint64_t best = 0;
    unsigned long long bkey = 0;
    for (int64_t base = blockIdx.x * (int64_t)SPI; base < total; base += (int64_t)gridDim.x * SPI) {  // CTA-uniform
        const int64_t i = base + grp * 32 + lane;
        const int64_t item = i / ns, li = i - item * ns;
        // slot li -> origin offset oi in [0, n_orig) (block li / ORIG of this launch is block
        // (li / ORIG) * blk_stride + blk_off of the range); slots past the range hold no origin (and stay zero)
        const int64_t sl = li % ORIG;  // slot r*T + t inside the block
        int64_t off = sl;
        if (a.warp_major) {
            constexpr int TT = G::T, RR = G::R;
            const int64_t r = sl / TT, tt = sl % TT;
            off = (tt >> 5) * (32 * RR) + r * 32 + (tt & 31);
        }
        const int64_t oi = ((li / ORIG) * a.blk_stride + a.blk_off) * ORIG + off;
        const bool valid = i < total && oi < n_orig;
        uint64_t red = 0;
        if (valid) {
            const int32_t* acc = a.accum + item * (int64_t)NB * ns + li;
            constexpr int CH = QPT < 8 ? QPT : 8;
            if constexpr (!SPLIT) {
                uint32_t mm = 0;
#pragma unroll 1
                for (int q0 = part * QPT; q0 < (part + 1) * QPT; q0 += CH) {
                    int32_t v[CH];
#pragma unroll
                    for (int j = 0; j < CH; ++j) v[j] = __ldcs(acc + (int64_t)(q0 + j) * ns);
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const uint32_t av = (uint32_t)(v[j] < 0 ? -v[j] : v[j]);
                        mm = av > mm ? av : mm;
                    }
                }
                red = mm;
            } else {
#pragma unroll 1
                for (int q0 = part * QPT; q0 < (part + 1) * QPT; q0 += CH) {
                    int32_t vp[CH], vq[CH];
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        vp[j] = __ldcs(acc + (int64_t)(q0 + j) * ns), vq[j] = __ldcs(acc + (int64_t)(NQ + q0 + j) * ns);
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const int64_t cP = vp[j], cQ = vq[j];
                        if (a.hist) {
                            if (priv && cQ < HS) atomicAdd(&sh_hist[cQ], 1u);
                            else hist_add_aggregated(a.hist, item * a.hist_stride + cQ);
                        }
                        const int64_t df = cP * a.aQ - cQ * a.bP;
                        const uint64_t av = (uint64_t)(df < 0 ? -df : df);
                        red = av > red ? av : red;
                    }
                }
            }
        }
        if constexpr (TPS > 1) {  // max over the TPS parts of each slot
            sh_red[part][grp * 32 + lane] = red;
            __syncthreads();
            if (part == 0)
                for (int p = 1; p < TPS; ++p) red = sh_red[p][grp * 32 + lane] > red ? sh_red[p][grp * 32 + lane] : red;
            __syncthreads();
        }
        if (!valid || part != 0) continue;
        const uint64_t m = red * a.gg;
        if (B == 1) {
            const int64_t pooled = a.perm ? a.perm[a.o_begin + oi] : a.o_begin + oi;
            if (a.per_origin) a.per_origin[a.perm ? pooled : oi] = m;
            best = m > best ? m : best;
            if (a.best_key) {
                const unsigned long long k = ((unsigned long long)red << 31) | (unsigned long long)(0x7fffffff - pooled);
                bkey = k > bkey ? k : bkey;
            }
        } else {
            atomicMax(reinterpret_cast<unsigned long long*>(&a.item_num[item]), (unsigned long long)m);
        }
    }
    if (B == 1) {
        best = warp_max_u64(best);
        bkey = warp_max_u64(bkey);
        if (lane == 0) {
            atomicMax(reinterpret_cast<unsigned long long*>(&a.item_num[0]), (unsigned long long)best);
            if (a.best_key) atomicMax(a.best_key, bkey);
        }
    }
    if constexpr (SPLIT) {
        if (priv) {
            __syncthreads();
            for (int i = threadIdx.x; i < HS; i += blockDim.x)
                if (sh_hist[i]) atomicAdd(&a.hist[i], (unsigned long long)sh_hist[i]);
        }
    }
}

// ----------------------------------------------------------------------------------------------- a9: label-invariant permutation null
// SURVEY.md §8f NEXT-2. code(o, x) does not depend on the labels, so one classification of a pair serves J
// permutations at once: for permutation j only the P'-count is needed, because with T[q] = all points in orthant q,
//     c_P' a - c_Q' b = (a + b) c_P' - b T[q]          (a = n_Q/g, b = n_P/g, exact integers).
// Counters are unsigned F-bit fields, PPW = 32 / F permutations per 32-bit word: F = 10 (three per word) when
// c_P' <= n_P <= 1023, else F = 16 (two per word; the host guarantees N <= 65535); T[q] has a word of its own. The
// labels arrive pre-spread: for point x and label word i the increment word has bit F*m set iff x is in P' of
// permutation PPW*i + m, so per pair the kernel does d FSET + d FFMA (address, once) + one ATOMS for T + JW ATOMS with
// the label word as the increment (no predicates, no branches). F = 10 gives 1.5x the permutations per classification
// and per ATOMS at the same shared memory (the SMEM-instruction queue is what bounds this kernel).
template <int D> struct PermCfg;  // JW label words per point, T origins (threads) per CTA
template <> struct PermCfg<1> { static constexpr int JW = 8, T = 256; };
template <> struct PermCfg<2> { static constexpr int JW = 8, T = 256; };
template <> struct PermCfg<3> { static constexpr int JW = 8, T = 256; };
#ifndef DDKS_P4T
#define DDKS_P4T 128  // C4b: 128 -> 116 us, 64 -> 117 us, 256 -> 138 us (wave tail of 336 CTAs on 296 slots)
#endif
template <> struct PermCfg<4> { static constexpr int JW = 4, T = DDKS_P4T; };
template <> struct PermCfg<5> { static constexpr int JW = 8, T = 160; };
template <> struct PermCfg<6> { static constexpr int JW = 4, T = 128; };
template <> struct PermCfg<7> { static constexpr int JW = 2, T = 128; };
template <> struct PermCfg<8> { static constexpr int JW = 1, T = 96; };

template <int D, int F> struct PermGeo {
    static_assert(F == 10 || F == 16, "label field width");
    static constexpr int PPW = 32 / F, JW = PermCfg<D>::JW, J = JW * PPW, T = PermCfg<D>::T;
    static constexpr uint32_t MASK = (1u << F) - 1u;
    static constexpr int NQ = 1 << D, DP = padded_dim<D>(), TILE = 256, S = 2;
    static constexpr int CNT_WORDS = NQ * (JW + 1) * T;   // [q][JW + 1][T]; slot JW holds T[q]
    static constexpr int STAGE_BYTES = TILE * DP * 4 + TILE * JW * 4;
    static constexpr int SMEM_BYTES = CNT_WORDS * 4 + S * STAGE_BYTES + 64;
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

struct PermArgs {
    const float* pts;         // pooled packed [N][DP]
    const uint32_t* labels;   // [n_chunks][chunk_words] spread increment words [N][JW] (see above)
    int64_t chunk_words;      // N*JW rounded up to 4 (16-byte aligned chunk rows for the bulk copies)
    int32_t N, n_perm;
    uint32_t a, b;            // DIFF weights
    uint64_t g;
    uint64_t* num;            // [n_perm] atomicMax targets
    unsigned long long* clk;  // profiling (or nullptr): [2] += FP32 compares executed (as CountArgs::clk)
};

// labels + validation: for row j of perms, check it is a permutation of 0..N-1 (range + no duplicate via bitmap,
// else *flag |= 2) and, for i < n_P, set the P' bit of permutation j in the increment word of point perms[j][i]
// (chunk j / J, word (j % J) / PPW, bit F * ((j % J) % PPW)).
__global__ void k_labels(const int32_t* __restrict__ perms, int64_t n_perm, int64_t N, int64_t n_P, int J, int JW,
                         int F, int64_t chunk_words, uint32_t* __restrict__ labels, uint32_t* __restrict__ bitmap,
                         uint32_t* flag) {
    const int64_t words = (N + 31) / 32;
    const int64_t total = n_perm * N;
    const int PPW = 32 / F;
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / N, pos = i - j * N;
        const int32_t src = perms[i];
        if (src < 0 || src >= N) { bad = true; continue; }
        const uint32_t bit = 1u << (src & 31);
        if (atomicOr(&bitmap[j * words + (src >> 5)], bit) & bit) bad = true;
        if (pos < n_P) {
            const int jj = (int)(j % J);
            atomicOr(&labels[(j / J) * chunk_words + (int64_t)src * JW + jj / PPW], 1u << (F * (jj % PPW)));
        }
    }
    if (bad) atomicOr(flag, 2u);
}

template <int D, bool GT, int F>
__global__ void __launch_bounds__(PermGeo<D, F>::T, 1) k_perm_count(const PermArgs a) {
    using G = PermGeo<D, F>;
    constexpr int J = G::J, JP = G::JW, T = G::T, DP = G::DP, TILE = G::TILE, S = G::S, NQ = G::NQ;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);                                 // [NQ][JP+1][T]
    uint8_t* stages = smem + G::CNT_WORDS * 4;                                          // S x (points, labels)
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + S * G::STAGE_BYTES);

    const int t = threadIdx.x;
    const int chunk = blockIdx.x;
    const int j0 = chunk * J;
    const int nj = min(J, a.n_perm - j0);
    const uint32_t* lab = a.labels + (int64_t)chunk * a.chunk_words;
    int32_t oi = (int32_t)blockIdx.y * T + t;
    const bool valid = oi < a.N;
    oi = valid ? oi : a.N - 1;
    const int n_tiles = (a.N + TILE - 1) / TILE;

    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = t; i < G::CNT_WORDS; i += T) cnt[i] = 0u;
    __syncthreads();
    auto issue = [&](int it, int s) {
        const int32_t p0 = it * TILE;
        const int n = min(TILE, a.N - p0);
        float* sp = reinterpret_cast<float*>(stages + s * G::STAGE_BYTES);
        uint32_t* sl = reinterpret_cast<uint32_t*>(stages + s * G::STAGE_BYTES + TILE * DP * 4);
        const uint32_t pb = (uint32_t)(n * DP * 4), lb = (uint32_t)((n * JP * 4 + 15) & ~15);
        mbar_expect_tx(&bars[s], pb + lb);
        bulk_g2s(sp, a.pts + (int64_t)p0 * DP, pb, &bars[s]);
        bulk_g2s(sl, lab + (int64_t)p0 * JP, lb, &bars[s]);
    };
    if (t == 0)
        for (int s = 0; s < S && s < n_tiles; ++s) issue(s, s);

    float o[D];
#pragma unroll
    for (int k = 0; k < D; ++k) o[k] = __ldg(a.pts + (int64_t)oi * DP + k);
    const uint32_t ubase = smem_u32(cnt) - 0x4B000000u;
    const float base = __uint_as_float(0x4B000000u + 4u * (uint32_t)t);
    constexpr uint32_t SLOT = 4u * T;  // bytes between permutation-pair slots of one bin

    for (int it = 0; it < n_tiles; ++it) {
        const int s = it % S;
        mbar_wait(&bars[s], (uint32_t)((it / S) & 1));
        const float* sp = reinterpret_cast<const float*>(stages + s * G::STAGE_BYTES);
        const uint32_t* sl = reinterpret_cast<const uint32_t*>(stages + s * G::STAGE_BYTES + TILE * DP * 4);
        const int n = min(TILE, a.N - it * TILE);
        // software-pipelined: the point and label words of the next point are loaded before this point's REDs are
        // issued (program order would otherwise put every LDS behind the previous point's fire-and-forget REDs and
        // expose the full SMEM latency per point; C4b measured 30 % issue-active that way). Prefetches read at most
        // one point past n: inside the stage (or the next stage / the barriers), values unused.
        float xn[D];
        uint32_t ln[JP];
        auto load_pt = [&](int p, float (&x)[D], uint32_t (&l)[JP]) {
            load_point<D>(sp + p * DP, x);
            const uint32_t* lw = sl + p * JP;
            if constexpr (JP % 4 == 0) {
#pragma unroll
                for (int i = 0; i < JP; i += 4) {
                    const uint4 w = *reinterpret_cast<const uint4*>(lw + i);
                    l[i] = w.x, l[i + 1] = w.y, l[i + 2] = w.z, l[i + 3] = w.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < JP; ++i) l[i] = lw[i];
            }
        };
        load_pt(0, xn, ln);
#pragma unroll 4
        for (int p = 0; p < n; ++p) {
            float x[D];
            uint32_t lw[JP];
#pragma unroll
            for (int k = 0; k < D; ++k) x[k] = xn[k];
#pragma unroll
            for (int i = 0; i < JP; ++i) lw[i] = ln[i];
            load_pt(p + 1, xn, ln);
            float f = base;
#pragma unroll
            for (int k = 0; k < D; ++k) f = fmaf(cmp_bit<GT>(x[k], o[k]), (float)(4 * (1 << k) * (JP + 1) * T), f);
            const uint32_t addr = __float_as_uint(f) + ubase;
            DDKS_ASSERT(__float_as_uint(f) - 0x4B000000u + JP * SLOT < (uint32_t)G::CNT_WORDS * 4u);
            red_add_shared(addr + JP * SLOT, 1u);  // T[q]
#pragma unroll
            for (int i = 0; i < JP; ++i) red_add_shared(addr + i * SLOT, lw[i]);
        }
        __syncthreads();
        if (t == 0 && it + S < n_tiles) {
            fence_proxy_async();
            issue(it + S, s);
        }
    }
    __syncthreads();
    if (a.clk && t == 0) atomicAdd(&a.clk[2], (unsigned long long)D * (unsigned long long)a.N * (unsigned long long)T);

    // finalise: num_j(o) = g * max_q |(a+b) c_P'[q] - b T[q]|, then max over this warp's origins per permutation
    __shared__ uint64_t wmax[T / 32][J];
    for (int j = 0; j < nj; ++j) {
        uint64_t m = 0;
        if (valid) {
            for (int q = 0; q < NQ; ++q) {
                const uint32_t w = cnt[(q * (JP + 1) + j / G::PPW) * T + t];
                const int64_t cP = (w >> (F * (j % G::PPW))) & G::MASK;
                const int64_t Tq = cnt[(q * (JP + 1) + JP) * T + t];
                const int64_t v = (int64_t)(a.a + a.b) * cP - (int64_t)a.b * Tq;
                const uint64_t av = (uint64_t)(v < 0 ? -v : v);
                m = av > m ? av : m;
            }
            m *= a.g;
        }
        m = warp_max_u64(m);
        if ((t & 31) == 0) wmax[t >> 5][j] = m;
    }
    __syncthreads();
    if (t < nj) {
        uint64_t m = 0;
        for (int w = 0; w < T / 32; ++w) m = wmax[w][t] > m ? wmax[w][t] : m;
        atomicMax(reinterpret_cast<unsigned long long*>(&a.num[j0 + t]), (unsigned long long)m);
    }
}

// argmax (reading R7): smallest pooled origin index whose num(o) equals the global num.
__global__ void k_argmax(const uint64_t* __restrict__ per_origin, int64_t n, int64_t o_begin,
                         const uint64_t* __restrict__ num, unsigned long long* __restrict__ arg) {
    const uint64_t target = *num;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (per_origin[i] == target) atomicMin(arg, (unsigned long long)(o_begin + i));
}

}  // namespace
}  // namespace ddks
