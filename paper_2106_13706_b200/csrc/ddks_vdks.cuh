// ddks_vdks.cuh — vdKS, the voxel approximation of ddKS (§2.2.2, Alg. 1).
//
//   NormalizeData: x' = (x - min_m) / (max_m - min_m) per dimension over the pooled points (constant dim -> 0.5);
//   IndexFromPoint: c_m = min(floor(x'_m k), k - 1), flat = sum_m c_m k^m;
//   Diff = VoxelList[T]/n_T - VoxelList[P]/n_P, kept exact as diff[v] = cQ[v] n_P - cP[v] n_Q (R16);
//   for each filled voxel v: the 2^d orthant sums of Diff split at v's lower corner (v itself in the all->= orthant),
//   D = max over filled voxels and orthants of |sum| / (n_P n_Q).
//
// B200 design (DESIGN.md §7 "vdKS"): HBM/L2-bound, no pair loop at all.
//   * k_minmax: per-dimension min/max as order-preserving uint32 keys (one atomic per warp);
//   * k_vox_hist: one thread per point; the voxel decision is taken in f64 with explicit _rn intrinsics (no FMA
//     contraction), the same arithmetic as the oracle, so cells are bit-identical; counts by global atomics;
//   * k_prefix_line (d passes, the first one reading the counts): the inclusive d-dimensional prefix sum S of
//     diff (int64, exact);
//   * k_vox_orthants: one thread per filled voxel gathers the 2^d box sums G[b] = S[corner(b)] with corner_m = k-1
//     (bit m set) or c_m - 1, and a subset Moebius transform (d x 2^(d-1) subtractions) turns them into the 2^d
//     orthant sums: O[q] = sum_{b subset of q} (-1)^{|q|-|b|} G[b]. Cost O(k^d d + F 2^d d) instead of the
//     literal O(F k^d) of Alg. 1's SumOrthants.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ddks_common.cuh"
#include "ddks_minmax.cuh"

namespace ddks {

// Row i of the pooled set, read in place from the caller's arrays (P rows, then Q rows; row-major [n][d] f32).
__device__ __forceinline__ const float* pooled_row(const float* P, const float* Q, int64_t n_P, int d, int64_t i) {
    return i < n_P ? P + i * d : Q + (i - n_P) * d;
}

// keys[0..d) = min keys (init 0xffffffff), keys[8..8+d) = max keys (init 0) over pooled rows [i_begin, i_end), read
// in place (no pack); -0 counts as +0. validate: a non-finite coordinate sets *flag |= 1 (SPEC NonFiniteValue).
// Grid-stride per thread, block reduction in SMEM, one atomic pair per (block, dimension).
__global__ void __launch_bounds__(256) k_minmax(const float* __restrict__ P, const float* __restrict__ Q, int64_t n_P,
                                                int64_t i_begin, int64_t i_end, int d, uint32_t* keys, int validate,
                                                uint32_t* flag) {
    __shared__ uint32_t sa[8][8], sb[8][8];
    uint32_t mn[8], mx[8];
    bool bad = false;
#pragma unroll
    for (int m = 0; m < 8; ++m) mn[m] = 0xffffffffu, mx[m] = 0u;
    for (int64_t i = i_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < i_end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float* x = pooled_row(P, Q, n_P, d, i);
#pragma unroll
        for (int m = 0; m < 8; ++m)
            if (m < d) {
                const float v = x[m];
                if (validate && !isfinite(v)) bad = true;
                const uint32_t k = f32_key(v == 0.0f ? 0.0f : v);
                mn[m] = k < mn[m] ? k : mn[m];
                mx[m] = k > mx[m] ? k : mx[m];
            }
    }
    if (bad) atomicOr(flag, 1u);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        uint32_t a = mn[m], b = mx[m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 31) == 0) sa[threadIdx.x >> 5][m] = a, sb[threadIdx.x >> 5][m] = b;
    }
    __syncthreads();
    if (threadIdx.x < d) {
        const int m = threadIdx.x;
        uint32_t a = 0xffffffffu, b = 0u;
        for (int w = 0; w < 8; ++w) a = min(a, sa[w][m]), b = max(b, sb[w][m]);
        atomicMin(&keys[m], a);
        atomicMax(&keys[8 + m], b);
    }
}

// NormalizeData + IndexFromPoint in f64, round-to-nearest everywhere, no contraction (matches the oracle bit for bit).
__device__ __forceinline__ int64_t voxel_of(const float* x, int d, const double* mn, const double* rng, int64_t k) {
    int64_t flat = 0, stride = 1;
    for (int m = 0; m < d; ++m) {
        const double xn = rng[m] > 0.0 ? __ddiv_rn(__dsub_rn((double)x[m], mn[m]), rng[m]) : 0.5;
        int64_t c = (int64_t)floor(__dmul_rn(xn, (double)k));
        c = c > k - 1 ? k - 1 : (c < 0 ? 0 : c);
        flat += c * stride;
        stride *= k;
    }
    return flat;
}

// cnt[2 v] = # P points in voxel v, cnt[2 v + 1] = # Q points. Pooled rows [p_begin, p_end), read in place.
__global__ void k_vox_hist(const float* __restrict__ P, const float* __restrict__ Q, int64_t p_begin, int64_t p_end,
                           int64_t n_P, int d, const uint32_t* __restrict__ keys, int64_t k, uint32_t* __restrict__ cnt) {
    double mn[8], rng[8];
    for (int m = 0; m < d; ++m) {
        mn[m] = (double)key_f32(keys[m]);
        rng[m] = __dsub_rn((double)key_f32(keys[8 + m]), mn[m]);
    }
    for (int64_t i = p_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p_end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = voxel_of(pooled_row(P, Q, n_P, d, i), d, mn, rng, k);
        atomicAdd(&cnt[2 * v + (i < n_P ? 0 : 1)], 1u);
    }
}

// Inclusive scan of S along dimension j (stride k^j), one thread per line of k cells. Loads of a 16-cell chunk are
// issued before its adds and stores, so they overlap (the stores may alias later loads of the same line only).
// from_cnt (dimension 0 only): the line's values are first computed from the voxel counts, S = cQ n_P - cP n_Q.
__global__ void k_prefix_line(int64_t* __restrict__ S, int64_t V, int64_t k, int64_t stride,
                              const uint32_t* __restrict__ cnt, int64_t n_P, int64_t n_Q) {
    constexpr int C = 16;
    const int64_t lines = V / k;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < lines; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = l % stride, hi = l / stride;
        const int64_t base = hi * stride * k + lo;
        int64_t run = 0;
        for (int64_t c0 = 0; c0 < k; c0 += C) {
            int64_t v[C];
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const int64_t idx = base + (c0 + j) * stride;
                if (c0 + j < k) v[j] = cnt ? (int64_t)cnt[2 * idx + 1] * n_P - (int64_t)cnt[2 * idx] * n_Q : S[idx];
            }
#pragma unroll
            for (int j = 0; j < C; ++j)
                if (c0 + j < k) {
                    run += v[j];
                    S[base + (c0 + j) * stride] = run;
                }
        }
    }
}

// Dimension-0 pass for k in {2, 4, 8, 16, 32}: one thread per voxel (coalesced), S = cQ n_P - cP n_Q scanned along
// each line of k consecutive voxels by a segmented warp scan (a line is k consecutive lanes; V is a multiple of k).
__global__ void k_prefix_first(int64_t* __restrict__ S, int64_t V, int k, const uint32_t* __restrict__ cnt,
                               int64_t n_P, int64_t n_Q) {
    const int lane = threadIdx.x & 31, pos = lane & (k - 1);
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < V;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = base + lane;
        int64_t x = 0;
        if (v < V) {
            const uint2 c = *reinterpret_cast<const uint2*>(cnt + 2 * v);
            x = (int64_t)c.y * n_P - (int64_t)c.x * n_Q;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (off < k && pos >= off) x += y;
        }
        if (v < V) S[v] = x;
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_vox_orthants(const uint32_t* __restrict__ cnt, const int64_t* __restrict__ S,
                                                      int64_t v_begin, int64_t v_end, int64_t k,
                                                      unsigned long long* num) {
    constexpr int NQ = 1 << D;
    uint64_t best = 0;
    for (int64_t v = v_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < v_end;
         v += (int64_t)gridDim.x * blockDim.x) {
        if ((cnt[2 * v] | cnt[2 * v + 1]) == 0) continue;  // FilledVoxels only
        int64_t c[D], stride[D];
        int64_t r = v, s = 1;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            c[m] = r % k;
            r /= k;
            stride[m] = s;
            s *= k;
        }
        int64_t G[NQ];
#pragma unroll
        for (int b = 0; b < NQ; ++b) {
            // box [0, corner]: corner_m = k - 1 if bit m of b is set, else c_m - 1 (empty box if that is -1)
            int64_t idx = 0;
            bool empty = false;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const int64_t cm = ((b >> m) & 1) ? k - 1 : c[m] - 1;
                DDKS_ASSERT(cm < k);
                empty |= cm < 0;
                idx += cm * stride[m];
            }
            G[b] = empty ? 0 : S[idx];
        }
        // subset Moebius transform: O[q] = sum_{b subset of q} (-1)^{|q \ b|} G[b]
#pragma unroll
        for (int m = 0; m < D; ++m)
#pragma unroll
            for (int b = 0; b < NQ; ++b)
                if ((b >> m) & 1) G[b] -= G[b ^ (1 << m)];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const uint64_t a = (uint64_t)(G[q] < 0 ? -G[q] : G[q]);
            best = a > best ? a : best;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, best, o);
        best = w > best ? w : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(num, (unsigned long long)best);
}

}  // namespace ddks
