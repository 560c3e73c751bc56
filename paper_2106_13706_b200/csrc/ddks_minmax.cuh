// ddks_minmax.cuh — vectorised per-dimension min / max (NormalizeData of vdKS and rdKS, Alg. 1-2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ddks_common.cuh"

namespace ddks {

#ifndef DDKS_MINMAX_BLOCKS
#define DDKS_MINMAX_BLOCKS (148 * 2)
#endif
// grid cap of k_minmax_vec: every block ends in 2 D same-address atomics, so fewer, longer blocks (two groups of
// rows in flight per thread keep the loads overlapped)
constexpr int MINMAX_BLOCKS = DDKS_MINMAX_BLOCKS;

// Per-dimension min / max of all pooled points as order-preserving keys (-0 as +0): keys[m] = min (init 0xffffffff),
// keys[max_off + m] = max (init 0); validate: a non-finite coordinate sets *flag |= 1. For 16-byte aligned row-major
// [n][D] inputs: 4 rows = D float4 per step (dims fixed at compile time), the < 4 leftover rows of each sample scalar.
// Used by vdKS (max_off 8) and rdKS (max_off D).
template <int D>
__global__ void __launch_bounds__(256) k_minmax_vec(const float* __restrict__ P, int64_t n_P,
                                                    const float* __restrict__ Q, int64_t n_Q, uint32_t* keys,
                                                    int max_off, int validate, uint32_t* flag) {
    __shared__ uint32_t sa[8][8], sb[8][8];
    // per-thread extremes as floats (FMNMX; -0 + 0 = +0 canonicalises the zero), keys formed once per thread. A NaN
    // is skipped by fminf / fmaxf; it is flagged when validating (and is undefined input otherwise)
    float fmn[D], fmx[D];
    bool bad = false;
#pragma unroll
    for (int m = 0; m < D; ++m) fmn[m] = INFINITY, fmx[m] = -INFINITY;
    auto take = [&](float v, int m) {
        if (validate && !(fabsf(v) < INFINITY)) bad = true;
        v += 0.0f;
        fmn[m] = fminf(fmn[m], v);
        fmx[m] = fmaxf(fmx[m], v);
    };
    const int64_t gP = n_P / 4, gQ = n_Q / 4, gs = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 2;  // groups of 4 rows in flight per thread
    for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < gP + gQ; g0 += U * gs) {
        float4 v[U][D];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t g = g0 + u * gs;
            if (g < gP + gQ) {
                const float4* src = reinterpret_cast<const float4*>(g < gP ? P + g * 4 * D : Q + (g - gP) * 4 * D);
#pragma unroll
                for (int j = 0; j < D; ++j) v[u][j] = __ldg(src + j);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (g0 + u * gs >= gP + gQ) break;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                take(v[u][j].x, (4 * j + 0) % D);
                take(v[u][j].y, (4 * j + 1) % D);
                take(v[u][j].z, (4 * j + 2) % D);
                take(v[u][j].w, (4 * j + 3) % D);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) {  // leftover rows
        const int r = threadIdx.x;
        const float* row = r < 4 ? (4 * gP + r < n_P ? P + (4 * gP + r) * D : nullptr)
                                 : (4 * gQ + (r - 4) < n_Q ? Q + (4 * gQ + (r - 4)) * D : nullptr);
        if (row) {
#pragma unroll
            for (int m = 0; m < D; ++m) take(row[m], m);
        }
    }
    if (bad) atomicOr(flag, 1u);
#pragma unroll
    for (int m = 0; m < D; ++m) {
        // no row seen: the identity keys (an all-infinite dimension is non-finite input: flagged when validating,
        // undefined otherwise)
        uint32_t a = fmn[m] == INFINITY ? 0xffffffffu : f32_key(fmn[m]);
        uint32_t b = fmx[m] == -INFINITY ? 0u : f32_key(fmx[m]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 31) == 0) sa[threadIdx.x >> 5][m] = a, sb[threadIdx.x >> 5][m] = b;
    }
    __syncthreads();
    if (threadIdx.x < D) {
        const int m = threadIdx.x;
        uint32_t a = 0xffffffffu, b = 0u;
        for (int w = 0; w < 8; ++w) a = min(a, sa[w][m]), b = max(b, sb[w][m]);
        atomicMin(&keys[m], a);
        atomicMax(&keys[max_off + m], b);
    }
}

}  // namespace ddks
