// ddks_kd_cluster.cuh — the mid-N kd ordering (DESIGN.md §7 "kd ordering at mid N") with one thread-block cluster per
// label run: the same hierarchy as k_kdb_fused (per (cell of the previous levels) bucket counting sort by x_level,
// equal-width buckets of the run's [min, max]; cells cut by position, rounded to A), computed by the KDC_CS CTAs of
// one cluster with histograms in shared memory and hardware cluster barriers instead of grid barriers:
//   ranges:  each CTA reduces its slice of rows; every CTA reads the others' partials through DSMEM;
//   level l: local SMEM histogram of the (cell, bucket) keys (the atomicAdd return is the row's rank in its
//            (CTA, key) group); the owner CTA of each key range reads that key's 8 local counts through DSMEM,
//            forms the key totals and the cross-CTA prefixes, scans its range, and after one more barrier writes
//            every CTA's final offset of the key back into that CTA's SMEM; every row then lands at
//            run start + offset(key) + rank, with no global atomics.
// The two label runs are independent (keys are label-major), so the two clusters never wait on each other. The order
// only changes speed -- every kd decision is taken from actual min / max values -- so counts are exact whatever
// the bucketing (buckets per cell here: about a quarter of the rows per cell, at most 1024).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "ddks_common.cuh"
#include "ddks_kernels.cuh"

namespace ddks {
namespace {

constexpr int KDC_T = 1024, KDC_CS = 8;  // threads per CTA, CTAs per cluster (one cluster per label run)
constexpr int KDC_RPT = 8;               // rows per thread at most: a run of <= KDC_CS * KDC_T * KDC_RPT = 65536 rows
constexpr int KDC_HW = 16384;            // histogram / offset words per CTA (dynamic SMEM 2 x 64 KB)
constexpr int KDC_SMEM = 2 * KDC_HW * 4;

struct KdcArgs {
    const float* pts;    // packed rows [N][DP] (P rows, then Q rows)
    int DP, K;
    int64_t N, n_P, G0, G1, G2, A;
    float* out[2];       // ping-pong row buffers; level l writes out[(K - 1 - l) & 1] (the last: out[0])
    int32_t* perm[2];    // the same for the permutations (sorted position -> pooled index)
};

// buckets per cell at a level with `cells` cells over a run of n rows: a power of two, about a quarter of the rows per
// cell (finer buckets only cost offset work: the owner phase touches every key in every CTA), at most 1024, and
// cells x buckets <= KDC_HW
__host__ __device__ inline int kdc_nbk(int64_t cells, int64_t n) {
    int b = 1024;
    while (b > 16 && (int64_t)b * 4 * cells > n) b >>= 1;
    while (b > 1 && (int64_t)b * cells > KDC_HW) b >>= 1;
    return b;
}

// start position of cell c (0 <= c <= cells) of the run [s, e) at `level`: cells are contiguous position ranges, the
// nested cuts of the previous levels (kd_cut, rounded to A); bounds[cells] = e
__device__ __forceinline__ int64_t kdc_bound(int64_t c, int64_t s, int64_t e, int level, int64_t G0, int64_t G1,
                                             int64_t G2, int64_t A) {
    if (level == 0) return c ? e : s;
    if (level == 1) return kd_cut(s, e, G0, c, A);
    if (level == 2) {
        const int64_t i0 = c / G1, i1 = c % G1;
        if (i0 >= G0) return e;
        return kd_cut(kd_cut(s, e, G0, i0, A), kd_cut(s, e, G0, i0 + 1, A), G1, i1, A);
    }
    const int64_t i0 = c / (G1 * G2), i1 = (c / G2) % G1, i2 = c % G2;
    if (i0 >= G0) return e;
    const int64_t s1 = kd_cut(s, e, G0, i0, A), e1 = kd_cut(s, e, G0, i0 + 1, A);
    return kd_cut(kd_cut(s1, e1, G1, i1, A), kd_cut(s1, e1, G1, i1 + 1, A), G2, i2, A);
}

__global__ void __cluster_dims__(KDC_CS, 1, 1) __launch_bounds__(KDC_T) k_kdb_cluster(const KdcArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ uint32_t kdc_sm[];
    uint32_t* hist = kdc_sm;            // [KDC_HW] local counts of this level's keys (owner: key totals, then scan)
    uint32_t* off = kdc_sm + KDC_HW;    // [KDC_HW] this CTA's final offset of every key
    __shared__ uint32_t part[4][2];     // this CTA's min / max keys of x_0..x_{K-1}
    __shared__ float rlo[4], rhi[4];    // the run's ranges
    __shared__ uint32_t wsum[KDC_T / 32];
    __shared__ uint32_t range_total;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int cr = (int)cluster.block_rank();
    const int lab = blockIdx.x / KDC_CS;
    const int64_t s = lab ? a.n_P : 0, e = lab ? a.N : a.n_P, n = e - s;
    const int64_t r0 = s + n * cr / KDC_CS, r1 = s + n * (cr + 1) / KDC_CS;  // this CTA's rows (positions)
    const int K = a.K, DP = a.DP;
    const int64_t gl[3] = {a.G0, a.G1, a.G2};

    // ranges of x_0..x_{K-1} over the run
    if (t < 4) part[t][0] = ~0u, part[t][1] = 0u;
    __syncthreads();
    for (int k = 0; k < K; ++k) {
        uint32_t lo = ~0u, hi = 0u;
        for (int64_t j = r0 + t; j < r1; j += KDC_T) {
            const uint32_t v = f32_key(__ldcg(a.pts + j * DP + k));
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
        }
        if (lane == 0) atomicMin(&part[k][0], lo), atomicMax(&part[k][1], hi);
    }
    cluster.sync();
    if (t < K) {
        uint32_t lo = ~0u, hi = 0u;
        for (int r = 0; r < KDC_CS; ++r) {
            const uint32_t* rp = cluster.map_shared_rank(&part[0][0], r);
            lo = min(lo, rp[2 * t]);
            hi = max(hi, rp[2 * t + 1]);
        }
        rlo[t] = key_f32(lo), rhi[t] = key_f32(hi);
    }
    __syncthreads();

    const float* src = a.pts;
    const int32_t* src_perm = nullptr;
    int64_t cells = 1;
    for (int level = 0; level < K; ++level) {
        const int nbk = kdc_nbk(cells, n);
        const int nk = (int)(cells * nbk);
        for (int i = t; i < nk; i += KDC_T) hist[i] = 0u;
        // the cells' start positions (relative to s; cells + 1 <= KDC_HW words) in `off`, free until the offsets
        uint32_t* bnd = off;
        for (int64_t c = t; c <= cells; c += KDC_T)
            bnd[c] = (uint32_t)(kdc_bound(c, s, e, level, a.G0, a.G1, a.G2, a.A) - s);
        __syncthreads();
        // local histogram; the atomic's return value is the row's rank among this CTA's rows of the same key
        const float lo = rlo[level], hi = rhi[level];
        const float scale = hi > lo ? (float)nbk / (hi - lo) : 0.0f;
        uint32_t key[KDC_RPT], rank[KDC_RPT];
#pragma unroll
        for (int i = 0; i < KDC_RPT; ++i) {
            const int64_t j = r0 + t + (int64_t)i * KDC_T;
            if (j < r1) {
                // cell: the last start <= j - s (binary search over the sorted starts)
                const uint32_t jr = (uint32_t)(j - s);
                int lo_c = 0, hi_c = (int)cells;  // bnd[lo_c] <= jr < bnd[hi_c] (empty cells share starts)
                while (hi_c - lo_c > 1) {
                    const int mid = (lo_c + hi_c) >> 1;
                    if (bnd[mid] <= jr) lo_c = mid; else hi_c = mid;
                }
                const float v = (__ldcg(src + j * DP + level) - lo) * scale;
                const int b = v >= (float)(nbk - 1) ? nbk - 1 : (v > 0.0f ? (int)v : 0);
                key[i] = (uint32_t)(lo_c * nbk + b);
                rank[i] = atomicAdd(&hist[key[i]], 1u);
            }
        }
        cluster.sync();  // every CTA's local counts complete
        // owner of keys [k0, k1): the cross-CTA prefixes (kept in registers) and the key totals (into its own hist)
        const int k0 = nk * cr / KDC_CS, k1 = nk * (cr + 1) / KDC_CS;
        const int per = (k1 - k0 + KDC_T - 1) / KDC_T;  // <= KDC_HW / KDC_CS / KDC_T = 2
        uint32_t pre[2][KDC_CS];
        uint32_t mysum = 0;
        for (int q = 0; q < per && q < 2; ++q) {
            const int k = k0 + t * per + q;
            if (k < k1) {
                uint32_t run = 0;
#pragma unroll
                for (int r = 0; r < KDC_CS; ++r) {
                    pre[q][r] = run;
                    run += cluster.map_shared_rank(hist, r)[k];
                }
                mysum += run;
                hist[k] = run;          // total of key k (read back after the barrier)
            }
        }
        // block-exclusive scan of the owned totals (each thread owns `per` consecutive keys)
        uint32_t x = mysum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t v = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            wsum[lane] = v;
            if (lane == 31) range_total = v;
        }
        __syncthreads();
        const uint32_t my_excl = x - mysum + (w ? wsum[w - 1] : 0u);
        cluster.sync();  // every owner's range total is published
        uint32_t base = 0;
        for (int r = 0; r < cr; ++r) base += *cluster.map_shared_rank(&range_total, r);
        {
            uint32_t run = base + my_excl;
            for (int q = 0; q < per && q < 2; ++q) {
                const int k = k0 + t * per + q;
                if (k < k1) {
                    const uint32_t tot = hist[k];
#pragma unroll
                    for (int r = 0; r < KDC_CS; ++r) cluster.map_shared_rank(off, r)[k] = run + pre[q][r];
                    run += tot;
                }
            }
        }
        cluster.sync();  // every CTA's offsets written
        const int o = (K - 1 - level) & 1;
        float* dst = a.out[o];
        int32_t* dperm = a.perm[o];
#pragma unroll
        for (int i = 0; i < KDC_RPT; ++i) {
            const int64_t j = r0 + t + (int64_t)i * KDC_T;
            if (j < r1) {
                const int64_t pos = s + (int64_t)off[key[i]] + rank[i];
                DDKS_ASSERT(pos >= s && pos < e);
                const float4* sp = reinterpret_cast<const float4*>(src + j * DP);
                float4* dp = reinterpret_cast<float4*>(dst + pos * DP);
                dp[0] = __ldcg(sp);
                if (DP == 8) dp[1] = __ldcg(sp + 1);
                dperm[pos] = src_perm ? __ldcg(src_perm + j) : (int32_t)j;
            }
        }
        cluster.sync();  // this level's rows written (cluster-scope release / acquire) before the next level reads them
        src = dst;
        src_perm = dperm;
        cells *= (level < 3 ? gl[level] : 1);
    }
}

}  // namespace
}  // namespace ddks
