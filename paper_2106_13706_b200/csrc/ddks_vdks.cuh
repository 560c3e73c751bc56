// ddks_vdks.cuh — vdKS, the voxel approximation of ddKS (§2.2.2, Alg. 1).
//
//   NormalizeData: x' = (x - min_m) / (max_m - min_m) per dimension over the pooled points (constant dim -> 0.5);
//   IndexFromPoint: c_m = min(floor(x'_m k), k - 1), flat = sum_m c_m k^m;
//   Diff = VoxelList[T]/n_T - VoxelList[P]/n_P, kept exact as diff[v] = cQ[v] n_P - cP[v] n_Q (R16);
//   for each filled voxel v: the 2^d orthant sums of Diff split at v's lower corner (v itself in the all->= orthant),
//   D = max over filled voxels and orthants of |sum| / (n_P n_Q).
//
// B200 design (DESIGN.md §7 "vdKS"): HBM/L2-bound, no pair loop at all.
//   * k_minmax / k_minmax_vec: per-dimension min/max as order-preserving uint32 keys;
//   * voxel decision (voxel_of): f64 with explicit _rn intrinsics (no FMA contraction), the same arithmetic as the
//     oracle, so cells are bit-identical;
//   * k_vox_hist (one thread per point) / k_vox_hist_vec (aligned inputs on one rank: 4 rows per D float4 loads):
//     global atomics into [k^d][2] u32 counts (all-reduced across ranks);
//   * k_vox_prefix_slab: the grid is cut into slabs of L = k^J consecutive voxels (the first J dimensions, L <= 4096);
//     one CTA per slab forms diff = cQ n_P - cP n_Q, the filled-voxel byte map and list, and scans the J inner
//     dimensions in SHARED memory; k_vox_outer scans the d - J outer ones for a column chunk held in SMEM (2 launches
//     instead of d line passes; k_prefix_line remains for > 512 slabs and k > 4096);
//   * k_vox_orthants: one thread per filled voxel (list; one rank) or per voxel of a shard (fill bytes), gathers the 2^d box sums G[b] = S[corner(b)] with
//     corner_m = k-1 (bit m set) or c_m - 1, and a subset Moebius transform (d x 2^(d-1) subtractions) turns them
//     into the 2^d orthant sums: O[q] = sum_{b subset of q} (-1)^{|q|-|b|} G[b]. Cost O(k^d d + F 2^d d) instead of
//     the literal O(F k^d) of Alg. 1's SumOrthants.
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
                              const uint32_t* __restrict__ cnt, int64_t n_P, int64_t n_Q, uint8_t* __restrict__ fill) {
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
                if (c0 + j < k) {
                    if (cnt) {
                        const uint32_t cp = cnt[2 * idx], cq = cnt[2 * idx + 1];
                        v[j] = (int64_t)cq * n_P - (int64_t)cp * n_Q;
                        fill[idx] = (cp | cq) != 0u;
                    } else {
                        v[j] = S[idx];
                    }
                }
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

// The max |orthant sum| over the filled voxels: list != nullptr -- one thread per entry of the filled-voxel list
// (list[0 .. *n_list)); else one thread per voxel of [v_begin, v_end), filled ones (fill byte) only. 32-bit index
// math (V <= 2^30); lg = log2 k for a power-of-two k, else -1.
template <int D>
__global__ void __launch_bounds__(256) k_vox_orthants(const uint8_t* __restrict__ fill, const uint32_t* __restrict__ list,
                                                      const uint32_t* __restrict__ n_list,
                                                      const int64_t* __restrict__ S, int64_t v_begin, int64_t v_end,
                                                      int k, int lg, unsigned long long* num) {
    constexpr int NQ = 1 << D;
    uint64_t best = 0;
    const int64_t n_it = list ? (int64_t)*n_list : v_end - v_begin;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_it; it += (int64_t)gridDim.x * blockDim.x) {
        int64_t v;
        if (list) {
            v = list[it];
        } else {
            v = v_begin + it;
            if (!fill[v]) continue;  // FilledVoxels only
        }
        int c[D], stride[D];
        uint32_t r = (uint32_t)v;
        int s = 1;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            if (lg >= 0) {
                c[m] = (int)(r & (uint32_t)(k - 1));
                r >>= lg;
            } else {
                c[m] = (int)(r % (uint32_t)k);
                r /= (uint32_t)k;
            }
            stride[m] = s;
            s *= k;
        }
        int64_t G[NQ];
#pragma unroll
        for (int b = 0; b < NQ; ++b) {
            // box [0, corner]: corner_m = k - 1 if bit m of b is set, else c_m - 1 (empty box if that is -1)
            int idx = 0;
            bool empty = false;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const int cm = ((b >> m) & 1) ? k - 1 : c[m] - 1;
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

// Per-call initialisation in one launch: min / max keys, the result record {num 0, arg ~0, key 0, flag 0}, the list
// length.
__global__ void k_vox_init(uint32_t* keys, unsigned long long* res, uint32_t* n_list) {
    const int t = threadIdx.x;
    if (t < 16) keys[t] = t < 8 ? 0xffffffffu : 0u;
    if (t == 0) res[0] = 0ull, res[1] = ~0ull, res[2] = 0ull, res[3] = 0ull;
    if (t == 0 && n_list) *n_list = 0u;
}

// ----------------------------------------------------------------------------------------------------- slab scans
// Slab geometry: L = k^J consecutive voxels (the first J dimensions, L <= VS_MAX_L), NS = V / L slabs.
constexpr int VS_MAX_L = 4096, VS_OUTER_MAX_NS = 512, VS_OUTER_CW = 16, VS_SLAB_T = 512;

// Voxel of a pooled row: same f64 arithmetic as voxel_of (32-bit flat index, V <= 2^30).
template <int D>
__device__ __forceinline__ uint32_t voxel_flat(const float* x, const double* mn, const double* rng, int k) {
    uint32_t flat = 0, stride = 1;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        const double xn = rng[m] > 0.0 ? __ddiv_rn(__dsub_rn((double)x[m], mn[m]), rng[m]) : 0.5;
        int64_t c = (int64_t)floor(__dmul_rn(xn, (double)k));
        c = c > k - 1 ? k - 1 : (c < 0 ? 0 : c);
        flat += (uint32_t)c * stride;
        stride *= (uint32_t)k;
    }
    return flat;
}

// k_vox_hist for 16-byte aligned inputs held whole by one rank: a thread takes groups of 4 rows (D float4 loads, two
// groups in flight -- the scalar version is load-latency bound), the < 4 leftover rows of each sample go to block 0.
template <int D>
__global__ void __launch_bounds__(256) k_vox_hist_vec(const float* __restrict__ P, int64_t n_P,
                                                      const float* __restrict__ Q, int64_t n_Q,
                                                      const uint32_t* __restrict__ keys, int k,
                                                      uint32_t* __restrict__ cnt) {
    double mn[D], rng[D];
#pragma unroll
    for (int m = 0; m < D; ++m) {
        mn[m] = (double)key_f32(keys[m]);
        rng[m] = __dsub_rn((double)key_f32(keys[8 + m]), mn[m]);
    }
    constexpr int U = 2;
    const int64_t gP = n_P / 4, G = gP + n_Q / 4, gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < G; g0 += U * gs) {
        float4 v[U][D];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t g = g0 + u * gs;
            if (g < G) {
                const float4* src = reinterpret_cast<const float4*>(g < gP ? P + g * 4 * D : Q + (g - gP) * 4 * D);
#pragma unroll
                for (int j = 0; j < D; ++j) v[u][j] = __ldg(src + j);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t g = g0 + u * gs;
            if (g >= G) break;
            const float* f = reinterpret_cast<const float*>(v[u]);
            const uint32_t q = g < gP ? 0u : 1u;
#pragma unroll
            for (int r = 0; r < 4; ++r) atomicAdd(&cnt[2 * voxel_flat<D>(f + r * D, mn, rng, k) + q], 1u);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) {  // leftover rows
        const int r = threadIdx.x;
        const int64_t gQ = n_Q / 4;
        const float* row = r < 4 ? (4 * gP + r < n_P ? P + (4 * gP + r) * D : nullptr)
                                 : (4 * gQ + (r - 4) < n_Q ? Q + (4 * gQ + (r - 4)) * D : nullptr);
        if (row) atomicAdd(&cnt[2 * voxel_flat<D>(row, mn, rng, k) + (r < 4 ? 0u : 1u)], 1u);
    }
}

// One CTA per slab s (voxels [s L, s L + L)): diff = cQ n_P - cP n_Q from the (all-reduced) counts, the fill bytes,
// the inclusive scan along the J inner dimensions in SMEM (dimension 0 by segmented warp shuffles when k is a power of
// two <= 32; the others one thread per line, 16 values loaded before their adds), S written. list != nullptr: the
// slab's filled voxels are appended to list (one global atomic per CTA; order across CTAs arbitrary). clean: the
// non-zero counts are reset to zero once read. Dynamic SMEM: L int64 + L bytes.
__global__ void __launch_bounds__(VS_SLAB_T) k_vox_prefix_slab(uint32_t* __restrict__ cnt, int clean, int k, int lg,
                                                               int J, int L, int64_t n_P, int64_t n_Q,
                                                               int64_t* __restrict__ S, uint8_t* __restrict__ fill,
                                                               uint32_t* __restrict__ list,
                                                               uint32_t* __restrict__ n_list) {
    extern __shared__ __align__(16) int64_t sv[];  // [L] then [L] fill bytes
    uint8_t* sf = reinterpret_cast<uint8_t*>(sv + L);
    __shared__ uint32_t wsum[VS_SLAB_T / 32 + 1];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const uint32_t lo = blockIdx.x * (uint32_t)L;
    const bool wscan = lg >= 0 && k <= 32;
    uint32_t nfill = 0;
    constexpr int U = VS_MAX_L / VS_SLAB_T;  // all of the slab's count loads in flight at once
    uint2 c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = u * VS_SLAB_T + t;
        c[u] = i < L ? *reinterpret_cast<const uint2*>(cnt + 2 * ((int64_t)lo + i)) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = u * VS_SLAB_T + t;
        if (u * VS_SLAB_T >= L) break;  // uniform: every thread runs the same iterations (shuffles)
        int64_t x = 0;
        if (i < L) {
            x = (int64_t)c[u].y * n_P - (int64_t)c[u].x * n_Q;
            const uint8_t f = (c[u].x | c[u].y) != 0u;
            fill[lo + i] = f;
            sf[i] = f;
            nfill += f;
            // leave the counts zeroed for the next call (the host zeroes them only when a call did not get here)
            if (clean && f) *reinterpret_cast<uint2*>(cnt + 2 * ((int64_t)lo + i)) = make_uint2(0u, 0u);
        }
        if (wscan) {
            const int pos = lane & (k - 1);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
                if (off < k && pos >= off) x += y;
            }
        }
        if (i < L) sv[i] = x;
    }
    int stride = wscan ? k : 1;
    for (int m = wscan ? 1 : 0; m < J; ++m, stride *= k) {
        __syncthreads();
        for (int l = t; l < L / k; l += VS_SLAB_T) {
            const int base = (l / stride) * stride * k + l % stride;
            int64_t run = 0;
            for (int c0 = 0; c0 < k; c0 += 16) {
                int64_t v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < k) v[j] = sv[base + (c0 + j) * stride];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < k) {
                        run += v[j];
                        sv[base + (c0 + j) * stride] = run;
                    }
            }
        }
    }
    __syncthreads();
    for (int i = t; i < L; i += VS_SLAB_T) S[lo + i] = sv[i];
    if (list == nullptr) return;
    // filled-voxel list: block-exclusive scan of the per-thread counts, one atomic for the block's range
    uint32_t inc = nfill;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (t == 0) {
        uint32_t tot = 0;
        for (int j = 0; j < VS_SLAB_T / 32; ++j) {
            const uint32_t x = wsum[j];
            wsum[j] = tot;
            tot += x;
        }
        wsum[VS_SLAB_T / 32] = tot ? atomicAdd(n_list, tot) : 0u;
    }
    __syncthreads();
    uint32_t pos = wsum[VS_SLAB_T / 32] + wsum[w] + inc - nfill;
    for (int i = t; i < L; i += VS_SLAB_T)
        if (sf[i]) list[pos++] = lo + i;
}

// The d - J outer dimensions (NS = k^(d-J) <= VS_OUTER_MAX_NS slabs): a CTA holds the column chunk
// [c0, c0 + VS_OUTER_CW) of the in-slab offset for every slab in SMEM ([NS][CW] int64) and scans it along each outer
// dimension (stride k^m in slab index), 16 values loaded before their adds.
__global__ void __launch_bounds__(256) k_vox_outer(int64_t* __restrict__ S, int k, int L, int NS, int n_outer) {
    extern __shared__ __align__(16) int64_t so[];  // [NS][CW]
    constexpr int CW = VS_OUTER_CW, T = 256, U = 16;
    const int t = threadIdx.x;
    const int c0 = blockIdx.x * CW, cw = min(CW, L - c0);
    for (int i0 = 0; i0 < NS * CW; i0 += U * T) {
        int64_t x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * T + t, sl = i / CW, c = i % CW;
            x[u] = (i < NS * CW && c < cw) ? S[(int64_t)sl * L + c0 + c] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * T + t;
            if (i < NS * CW) so[i] = x[u];
        }
    }
    int stride = 1;
    for (int m = 0; m < n_outer; ++m, stride *= k) {
        __syncthreads();
        for (int it = t; it < (NS / k) * CW; it += T) {
            const int l = it / CW, c = it % CW;
            if (c >= cw) continue;
            const int base = (l / stride) * stride * k + l % stride;
            int64_t run = 0;
            for (int j0 = 0; j0 < k; j0 += 16) {
                int64_t v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j0 + j < k) v[j] = so[(base + (j0 + j) * stride) * CW + c];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j0 + j < k) {
                        run += v[j];
                        so[(base + (j0 + j) * stride) * CW + c] = run;
                    }
            }
        }
    }
    __syncthreads();
    for (int i = t; i < NS * CW; i += T) {
        const int sl = i / CW, c = i % CW;
        if (c < cw) S[(int64_t)sl * L + c0 + c] = so[i];
    }
}

}  // namespace ddks
