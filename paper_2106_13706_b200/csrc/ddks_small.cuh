// ddks_small.cuh — the fused small-N statistic (SURVEY.md §7 hard part 4; config C1: N = 400): one launch does
// a1 (validate + pack), a3/a4 (classify + count) and a5/a6 (per-origin statistic, block max, packed argmax).
//
// Why a separate kernel: for N of a few hundred to a few thousand points the position-ordered path is launch- and
// latency-bound (pack, memset, count, finalise, argmax: five dependent launches around a count of a few us). Here
//   * the CTA reads its origins and point rows straight from the caller's row-major P / Q (no packed copy; the FP32
//     compares treat -0 == +0, so no canonicalisation is needed) and flags non-finite values while loading;
//   * the point axis is split over the CTAs of a thread-block CLUSTER (grid.x = segment = cluster rank): after
//     counting, every non-leader CTA adds its counter words into the leader's shared memory through DSMEM
//     (red.shared::cluster via a mapped pointer), so no global partials, no memset and no finaliser launch.
//     Word-wise adds of the packed int16 halves are exact because the whole point set fits one int16 window
//     (the host checks N * max(a, b) <= 32767: every partial and the total stay inside int16);
//   * the leader writes one 32-byte record per origin block {num, packed argmax key, flags} with plain stores straight
//     into the context's pinned host buffer (zero-copy); the host reduces the records (ddks_combine_records
//     semantics) after the stream sync -- no result initialisation, no atomics, no copy: the call is ONE graph node.
// The counting itself is k_count's: FSET.BF + FFMA build the float-encoded SMEM counter address, one red.shared per
// pair, thread-private counters (two origins per thread, 16-bit halves).
#pragma once
#include <cooperative_groups.h>

#include "ddks_kernels.cuh"

namespace ddks {
namespace {

constexpr int SM_R = 2, SM_T = 128, SM_TILE = 256, SM_MAX_CLUSTER = 8;

template <int D> struct SmallGeo {
    static constexpr int R = SM_R, T = SM_T, RP = R / 2, NBASE = RP, WPB = R * T / 2, TILE = SM_TILE;
    static constexpr int DP = padded_dim<D>(), NQ = 1 << D, NB = NQ, HIST_WORDS = NB * WPB, ORIGINS = R * T;
    static constexpr int SMEM_BYTES = TILE * DP * 4 + HIST_WORDS * 4 + 16;
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
    __host__ __device__ static constexpr int slot(int r, int t) { return (r * T + t) % WPB; }
    __host__ __device__ static constexpr bool high(int r, int t) { return r * T + t >= WPB; }
};

struct SmallArgs {
    const float* P;           // [n_P][d] row-major (caller's buffer)
    const float* Q;           // [n_Q][d]
    int32_t n_P, N;           // pooled points (P rows, then Q rows)
    int32_t seg_points;       // points per cluster rank
    uint32_t incP, incQ;      // DIFF increments +aQ, -bP (two's complement)
    uint64_t gg;              // gcd(n_P, n_Q): num(o) = gg * |counter|
    int validate;
    unsigned long long* out;  // [blocks][4]: {num, key, flags, 0} per origin block, written by the cluster leader
                              // (device view of pinned host memory)
    unsigned long long* clk;  // profiling (or nullptr): [2] += executed compares
};

__device__ __forceinline__ const float* small_row(const SmallArgs& a, int32_t j, int d) {
    return j < a.n_P ? a.P + (int64_t)j * d : a.Q + (int64_t)(j - a.n_P) * d;
}

template <int D, bool GT>
__global__ void __launch_bounds__(SM_T) k_count_small(const SmallArgs a) {
    using G = SmallGeo<D>;
    constexpr int R = G::R, RP = G::RP, T = G::T, DP = G::DP, TILE = G::TILE, WPB = G::WPB;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t smem[];
    float* tile = reinterpret_cast<float*>(smem);                                   // [TILE][DP]
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + TILE * DP * 4);            // [NB][WPB]
    uint32_t* sflag = hist + G::HIST_WORDS;                                         // this CTA's flags

    const int t = threadIdx.x;
    const int32_t seg0 = (int32_t)blockIdx.x * a.seg_points;
    const int32_t seg1 = min(a.N, seg0 + a.seg_points);
    const int32_t blk_o0 = (int32_t)blockIdx.y * G::ORIGINS;
    for (int i = t; i < G::HIST_WORDS; i += T) hist[i] = 0u;
    if (t == 0) *sflag = 0u;

    // origins of this thread: slot r -> blk_o0 + r*T + t (clamped to the last origin; ignored at the end)
    float o[R][D];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int32_t oi = min(blk_o0 + r * T + t, a.N - 1);
        const float* src = small_row(a, oi, D);
#pragma unroll
        for (int k = 0; k < D; ++k) o[r][k] = __ldg(src + k);
    }
    const uint32_t ubase = smem_u32(hist) - 0x4B000000u;
    float base[1];
    base[0] = __uint_as_float(0x4B000000u + 4u * (uint32_t)G::slot(0, t));
    const uint32_t incP_hi = a.incP << 16, incQ_hi = a.incQ << 16;
    bool bad = false;
    unsigned long long exec_cmp = 0;

    for (int32_t p0 = seg0; p0 < seg1; p0 += TILE) {
        const int cnt = min(TILE, seg1 - p0);
        __syncthreads();  // the previous tile is consumed (and the counters are zeroed, first time)
        for (int i = t; i < cnt; i += T) {  // rows -> padded SMEM rows, validated on the way
            const float* src = small_row(a, p0 + i, D);
            float v[DP];
#pragma unroll
            for (int k = 0; k < DP; ++k) {
                v[k] = k < D ? __ldg(src + k) : 0.0f;
                if (k < D && a.validate && !isfinite(v[k])) bad = true;
            }
            float4* dst = reinterpret_cast<float4*>(tile + i * DP);
            dst[0] = make_float4(v[0], v[1], v[2], v[3]);
            if constexpr (DP == 8) dst[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
        __syncthreads();
        int32_t split = a.n_P - p0;
        split = split < 0 ? 0 : (split > cnt ? cnt : split);
        // prefetches of count_points read up to two rows past cnt: inside the counters region, values unused
        if (split > 0)
            count_points<D, GT, R, RP, 1, WPB, DP>(tile, 0, split, o, base, ubase, a.incP, incP_hi,
                                                  G::HIST_WORDS * 4u);
        if (split < cnt)
            count_points<D, GT, R, RP, 1, WPB, DP>(tile, split, cnt, o, base, ubase, a.incQ, incQ_hi,
                                                  G::HIST_WORDS * 4u);
        exec_cmp += (unsigned long long)D * cnt;
    }
    if (bad) atomicOr(sflag, 1u);
    // every thread executed the same compares: one global atomic per CTA
    if (a.clk && t == 0) atomicAdd(&a.clk[2], exec_cmp * (unsigned long long)(T * R));

    // cluster reduction: every rank's counts into the leader's counters (DSMEM), then the leader finalises
    __syncthreads();
    cluster.sync();
    const unsigned rank = cluster.block_rank();
    if (rank != 0) {
        uint32_t* lead = cluster.map_shared_rank(hist, 0);
        for (int i = t; i < G::HIST_WORDS; i += T) {
            const uint32_t w = hist[i];
            if (w) atomicAdd(lead + i, w);
        }
        if (t == 0 && *sflag) atomicOr(cluster.map_shared_rank(sflag, 0), *sflag);
    }
    cluster.sync();
    if (rank != 0) return;

    uint64_t best = 0;
    unsigned long long bkey = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int32_t oi = blk_o0 + r * T + t;
        if (oi >= a.N) continue;
        const int sl = G::slot(r, t);
        const bool hiw = G::high(r, t);
        uint32_t mm = 0;
        for (int q = 0; q < G::NQ; ++q) {
            int32_t lo, hi;
            split16(hist[q * WPB + sl], lo, hi);
            const int32_t v = hiw ? hi : lo;
            const uint32_t av = (uint32_t)(v < 0 ? -v : v);
            mm = av > mm ? av : mm;
        }
        const uint64_t m = (uint64_t)mm * a.gg;
        best = m > best ? m : best;
        const unsigned long long k = ((unsigned long long)mm << 31) | (unsigned long long)(0x7fffffff - oi);
        bkey = k > bkey ? k : bkey;
    }
    best = warp_max_u64(best);
    bkey = warp_max_u64(bkey);
    __shared__ uint64_t wb[SM_T / 32], wk[SM_T / 32];
    if ((t & 31) == 0) wb[t >> 5] = best, wk[t >> 5] = bkey;
    __syncthreads();
    if (t == 0) {
        uint64_t m = 0, k = 0;
        for (int w = 0; w < T / 32; ++w) m = wb[w] > m ? wb[w] : m, k = wk[w] > k ? wk[w] : k;
        unsigned long long* rec = a.out + (int64_t)blockIdx.y * 4;
        rec[0] = m;
        rec[1] = k;
        rec[2] = *sflag;
        rec[3] = 0ull;
    }
}

}  // namespace
}  // namespace ddks
