// ddks_rdks.cuh — rdKS, the radial approximation of ddKS (§2.2.3, Alg. 2).
//
//   NormalizeData (as vdKS), corners C = {0} U {e_m} (d + 1 of them), for every corner c the Euclidean
//   distances |x' - c| of both samples, sorted, and GetDFromCornerLists = the two-sample KS of the two distance lists
//   (evaluated once every value <= the current one is consumed, R17); D = max over corners.
//
// B200 design (DESIGN.md §7 "rdKS"), O((d+1) N log N) as the paper states, no pair loop:
//   * k_rd_minmax / k_rd_normalize: x' in f64 with _rn intrinsics (bit-identical to the oracle);
//   * k_rd_keys: one thread per (point, corner), the literal sequential sum of (x'_m - c_m)^2 (no FMA) and a
//     correctly rounded sqrt; key = dist bits << 1 | label (label 0 = P, 1 = Q), segment = corner;
//   * a segmented LSD radix sort, 8 passes of 8-bit digits: per 4096-key tile histogram -> per-segment offsets ->
//     stable scatter (warp __match_any_sync ranks + per-warp digit counters);
//   * k_rd_sweep: per tile, the P-count prefix (earlier tiles' counts + a block scan) gives the two ECDFs at every
//     sorted position; |i_P n_Q - i_Q n_P| is taken only at the last position of each distinct distance.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ddks_common.cuh"

namespace ddks {

// keys[0..d) = min keys (init 0xffffffff), keys[d..2d) = max keys (init 0), as order-preserving uint32.
// grid.y strides over dimensions, grid.x over point chunks (so d = 1000 with 200 points is 1000 CTAs, and d = 5 with
// 2M points is 5 x 60); block reduction, one atomic pair per (block, dimension); non-finite -> *flag |= 1.
__global__ void __launch_bounds__(256) k_rd_minmax(const float* __restrict__ P, int64_t n_P,
                                                   const float* __restrict__ Q, int64_t n_Q, int d, uint32_t* keys,
                                                   uint32_t* flag) {
    __shared__ uint32_t sa[8], sb[8];
    const int64_t N = n_P + n_Q;
    bool bad = false;
    for (int m = blockIdx.y; m < d; m += gridDim.y) {
        uint32_t a = 0xffffffffu, b = 0u;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
            float x = i < n_P ? P[i * d + m] : Q[(i - n_P) * d + m];
            bad |= !isfinite(x);
            x = x == 0.0f ? 0.0f : x;  // -0 -> +0
            const uint32_t k = f32_key(x);
            a = min(a, k);
            b = max(b, k);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 31) == 0) sa[threadIdx.x >> 5] = a, sb[threadIdx.x >> 5] = b;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) a = min(a, sa[w]), b = max(b, sb[w]);
            atomicMin(&keys[m], a);
            atomicMax(&keys[d + m], b);
        }
        __syncthreads();
    }
    if (bad) atomicOr(flag, 1u);
}

// x'_m = (x_m - min_m) / (max_m - min_m) in f64 (0.5 for a constant dimension; NormalizeData), read in place
__device__ __forceinline__ double rd_norm(const float* row, int m, const uint32_t* __restrict__ keys, int d) {
    const double mn = (double)key_f32(keys[m]);
    const double rng = __dsub_rn((double)key_f32(keys[d + m]), mn);
    return rng > 0.0 ? __ddiv_rn(__dsub_rn((double)row[m], mn), rng) : 0.5;
}

__device__ __forceinline__ int rdb_bucket(uint64_t key, double scale, int nbk);

// xn[i][m] = x'_im for every pooled row (large d: normalise once instead of once per corner)
__global__ void k_rd_normalize(const float* __restrict__ P, int64_t n_P, const float* __restrict__ Q, int64_t n_Q,
                               int d, const uint32_t* __restrict__ keys, double* __restrict__ xn) {
    const int64_t total = (n_P + n_Q) * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / d;
        const int m = (int)(e - i * d);
        xn[e] = rd_norm(i < n_P ? P + i * d : Q + (i - n_P) * d, m, keys, d);
    }
}

// key[c][i] = bits(|x'_i - corner_c|) << 1 | (i >= n_P) for corners c in [c_begin, c_end); corner 0 = origin,
// corner c >= 1 = unit vector e_{c-1}. x' comes from xn when given (large d), else it is formed on the fly from the
// caller's rows (same f64 _rn arithmetic as the oracle either way, so the keys are bit-identical). Threads: corner
// fastest, so the threads of one point share its row.
// cnt != nullptr (bucket-pruned sweep): also counts the key into its distance bucket, cnt[(c * nbk + b) * 2 + label].
__global__ void k_rd_keys(const float* __restrict__ P, const float* __restrict__ Q, const double* __restrict__ xn,
                          int64_t N, int64_t n_P, int d,
                          const uint32_t* __restrict__ keys, int c_begin, int c_end, uint64_t* __restrict__ key,
                          uint32_t* __restrict__ cnt, int nbk, double scale) {
    const int nc = c_end - c_begin;
    const int64_t total = N * nc;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / nc;
        const int c = (int)(e - i * nc) + c_begin;
        const float* row = i < n_P ? P + i * d : Q + (i - n_P) * d;
        double s = 0.0;
#pragma unroll 4
        for (int m = 0; m < d; ++m) {
            const double xm = xn ? xn[i * d + m] : rd_norm(row, m, keys, d);
            const double t = __dsub_rn(xm, (c >= 1 && m == c - 1) ? 1.0 : 0.0);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        const double dist = __dsqrt_rn(s);
        const uint64_t k = ((uint64_t)__double_as_longlong(dist) << 1) | (uint64_t)(i >= n_P);
        key[(int64_t)(c - c_begin) * N + i] = k;
        if (cnt) atomicAdd(&cnt[2 * ((int64_t)(c - c_begin) * nbk + rdb_bucket(k, scale, nbk)) + (k & 1ull)], 1u);
    }
}

// d <= 8: one thread per point computes x' once (d divisions instead of d per corner) and every corner's key in
// the same literal sequential f64 order as k_rd_keys (bit-identical keys); keys of corner c stay coalesced.
template <int D>
__global__ void k_rd_keys_pt(const float* __restrict__ P, const float* __restrict__ Q, int64_t N, int64_t n_P,
                             const uint32_t* __restrict__ keys, int c_begin, int c_end, uint64_t* __restrict__ key,
                             uint32_t* __restrict__ cnt, int nbk, double scale) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const float* row = i < n_P ? P + i * D : Q + (i - n_P) * D;
        double x[D];
#pragma unroll
        for (int m = 0; m < D; ++m) x[m] = rd_norm(row, m, keys, D);
        const uint64_t lab = (uint64_t)(i >= n_P);
        for (int c = c_begin; c < c_end; ++c) {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const double t = __dsub_rn(x[m], (c >= 1 && m == c - 1) ? 1.0 : 0.0);
                s = __dadd_rn(s, __dmul_rn(t, t));
            }
            const uint64_t k = ((uint64_t)__double_as_longlong(__dsqrt_rn(s)) << 1) | lab;
            key[(int64_t)(c - c_begin) * N + i] = k;
            if (cnt) atomicAdd(&cnt[2 * ((int64_t)(c - c_begin) * nbk + rdb_bucket(k, scale, nbk)) + lab], 1u);
        }
    }
}

// ------------------------------------------------------------------------------------ GetDFromCornerLists sweep
// tcnt[seg * tiles + tile] = # P keys (label 0) in the tile
__global__ void __launch_bounds__(RS_T) k_rd_count(const uint64_t* __restrict__ key, int64_t N, int tiles,
                                                   uint32_t* __restrict__ tcnt) {
    __shared__ uint32_t red[RS_WARPS];
    const int seg = blockIdx.x / tiles, tile = blockIdx.x - seg * tiles;
    const int64_t base = (int64_t)seg * N + (int64_t)tile * RS_TILE;
    const int n = (int)min((int64_t)RS_TILE, N - (int64_t)tile * RS_TILE);
    uint32_t c = 0;
    for (int i = threadIdx.x; i < n; i += RS_T) c += (uint32_t)((key[base + i] & 1ull) == 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int i = 0; i < RS_WARPS; ++i) s += red[i];
        tcnt[blockIdx.x] = s;
    }
}

// cnum[seg] = max over the tie-complete positions of |i_P n_Q - i_Q n_P| (atomicMax; init 0)
__global__ void __launch_bounds__(RS_T) k_rd_sweep(const uint64_t* __restrict__ key, int64_t N, int tiles,
                                                   int64_t n_P, int64_t n_Q, const uint32_t* __restrict__ tcnt,
                                                   unsigned long long* __restrict__ cnum) {
    const int seg = blockIdx.x / tiles, tile = blockIdx.x - seg * tiles;
    const int64_t sbase = (int64_t)seg * N;
    const int64_t p0 = (int64_t)tile * RS_TILE;
    const int n = (int)min((int64_t)RS_TILE, N - p0);
    // P keys in earlier tiles of this segment
    uint32_t c = 0;
    for (int t = threadIdx.x; t < tile; t += RS_T) c += tcnt[(int64_t)seg * tiles + t];
    uint32_t before = 0;
    block_excl_scan256(c, &before);
    // blocked arrangement: thread t owns positions [t * ITEMS, t * ITEMS + ITEMS) of the tile
    uint64_t k[RS_ITEMS];
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const int idx = threadIdx.x * RS_ITEMS + j;
        k[j] = idx < n ? key[sbase + p0 + idx] : ~0ull;
        mine += (uint32_t)(idx < n && (k[j] & 1ull) == 0);
    }
    const uint32_t mine_before = block_excl_scan256(mine);
    int64_t iP = (int64_t)before + mine_before;
    uint64_t best = 0;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const int idx = threadIdx.x * RS_ITEMS + j;
        if (idx >= n) break;
        iP += (int64_t)((k[j] & 1ull) == 0);
        const int64_t pos = p0 + idx;  // 0-based position in the merged list; pos + 1 keys consumed
        bool last = pos == N - 1;
        if (!last) {
            const uint64_t nk = (j + 1 < RS_ITEMS && idx + 1 < n) ? k[j + 1] : key[sbase + pos + 1];
            last = (nk >> 1) != (k[j] >> 1);
        }
        if (last) {
            const int64_t iQ = pos + 1 - iP;
            const int64_t t = iP * n_Q - iQ * n_P;
            const uint64_t a = (uint64_t)(t < 0 ? -t : t);
            best = a > best ? a : best;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t v = __shfl_xor_sync(0xffffffffu, best, o);
        best = v > best ? v : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(&cnum[seg], (unsigned long long)best);
}

}  // namespace ddks

namespace ddks {

// ------------------------------------------------------------------------------------ bucket-pruned sweep
// GetDFromCornerLists without sorting every key (DESIGN.md §7 "rdKS"). Distances are bucketed by a monotone map
// b = min(NBK - 1, floor(dist * scale)) (equal distances share a bucket, so every bucket end is a tie-group end).
// Per bucket: counts (cP, cQ) and the min / max distance bits. A prefix over the buckets gives the exact ECDF pair at
// every bucket end; inside bucket b the statistic t = i_P n_Q - i_Q n_P stays within
// [t_start - cQ n_P, t_start + cP n_Q], so only buckets whose bound beats the best bucket-end value and that hold two
// distinct distances can hide a larger value: their keys are compacted and sorted in SMEM (bitonic) and swept exactly.
// A candidate bucket with more than RDB_CAPK keys and two distinct distances sets *flag bit 8 (as does a candidate
// set larger than N/2), and the caller falls back to the full radix sort.
constexpr int RDB_CAPK = 4096;

__device__ __forceinline__ int rdb_bucket(uint64_t key, double scale, int nbk) {
    const double dist = __longlong_as_double((long long)(key >> 1));
    const double v = __dmul_rn(dist, scale);
    const int b = v >= (double)(nbk - 1) ? nbk - 1 : (int)v;
    return b < 0 ? 0 : b;
}

// Bucket prefix sums, many CTAs: a chunk is RDB_CH consecutive buckets of one segment (256 threads x 4 buckets).
// (cP, cQ) travel packed as cP << 32 | cQ (each < 2^31, so the halves never carry into each other).
constexpr int RDB_CH = 1024;

__device__ __forceinline__ uint64_t rdb_pair(const uint32_t* cnt, int64_t i) {
    return ((uint64_t)cnt[2 * i] << 32) | cnt[2 * i + 1];
}

// csum[s * nch + c] = packed (cP, cQ) total of chunk c of segment s. grid (nch, nseg), 256 threads.
__global__ void __launch_bounds__(256) k_rdb_reduce(const uint32_t* __restrict__ cnt, int nbk,
                                                    uint64_t* __restrict__ csum) {
    const int s = blockIdx.y, c = blockIdx.x, nch = gridDim.x;
    uint64_t v = 0;
#pragma unroll
    for (int j = 0; j < RDB_CH / 256; ++j) {
        const int b = c * RDB_CH + threadIdx.x * (RDB_CH / 256) + j;
        if (b < nbk) v += rdb_pair(cnt, (int64_t)s * nbk + b);
    }
    uint64_t tot;
    block_excl_scan256_u64(v, &tot);
    if (threadIdx.x == 0) csum[(int64_t)s * nch + c] = tot;
}

// exclusive scan of the chunk totals of each segment (one CTA per segment; nch <= 1024 * 4)
__global__ void __launch_bounds__(256) k_rdb_chunk_scan(uint64_t* __restrict__ csum, int nch) {
    uint64_t* c = csum + (int64_t)blockIdx.x * nch;
    const int per = (nch + 255) / 256;
    uint64_t v = 0;
    for (int j = 0; j < per; ++j) {
        const int k = threadIdx.x * per + j;
        if (k < nch) v += c[k];
    }
    uint64_t run = block_excl_scan256_u64(v);
    for (int j = 0; j < per; ++j) {
        const int k = threadIdx.x * per + j;
        if (k < nch) {
            const uint64_t x = c[k];
            c[k] = run;
            run += x;
        }
    }
}

// pst[b] = (P, Q) keys before bucket b; cnum[s] = max over bucket ends of |i_P n_Q - i_Q n_P| (atomicMax; init 0)
__global__ void __launch_bounds__(256) k_rdb_down(const uint32_t* __restrict__ cnt, int nbk,
                                                  const uint64_t* __restrict__ csum, int64_t n_P, int64_t n_Q,
                                                  uint2* __restrict__ pst, unsigned long long* __restrict__ cnum) {
    const int s = blockIdx.y, c = blockIdx.x, nch = gridDim.x;
    constexpr int J = RDB_CH / 256;
    uint64_t v[J], sum = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int b = c * RDB_CH + threadIdx.x * J + j;
        v[j] = b < nbk ? rdb_pair(cnt, (int64_t)s * nbk + b) : 0ull;
        sum += v[j];
    }
    uint64_t run = csum[(int64_t)s * nch + c] + block_excl_scan256_u64(sum);
    uint64_t best = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int b = c * RDB_CH + threadIdx.x * J + j;
        if (b >= nbk) break;
        pst[(int64_t)s * nbk + b] = make_uint2((uint32_t)(run >> 32), (uint32_t)run);
        run += v[j];
        const int64_t t = (int64_t)(run >> 32) * n_Q - (int64_t)(uint32_t)run * n_P;
        const uint64_t a = (uint64_t)(t < 0 ? -t : t);
        best = a > best ? a : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, best, o);
        best = w > best ? w : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(&cnum[s], (unsigned long long)best);
}

// Candidates: at least two keys inside, and the reachable extreme beats the best bucket end (cnum[s] after
// k_rdb_down). Each gets a slot in the segment's candidate buffer (coff) and list (clist) by atomics on the
// segment's counters seg[2 * s] (keys) and seg[2 * s + 1] (buckets), a zeroed fill counter, and its bit in the
// candidate bitmap cbits (one ballot word per 32 buckets; nbk is a power of two >= 256, so a warp's 32 consecutive
// buckets are one word). Non-candidate buckets' counts are re-zeroed here (the candidates' in k_rdb_finish), so the
// next call needs no memset of the count array.
__global__ void k_rdb_cand(uint32_t* __restrict__ cnt, const uint2* __restrict__ pst, int nseg,
                           int nbk, int64_t n_P, int64_t n_Q, const unsigned long long* __restrict__ cnum,
                           uint32_t* __restrict__ coff, uint32_t* __restrict__ fill, uint32_t* __restrict__ cbits,
                           int32_t* __restrict__ clist, uint32_t* __restrict__ seg) {
    const int64_t total = (int64_t)nseg * nbk;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;  // a multiple of 32: every warp stays word-aligned
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - (threadIdx.x & 31) < total; i += step) {
        bool cand = false;
        if (i < total) {
            const int s = (int)(i / nbk);
            const uint2 c2 = reinterpret_cast<const uint2*>(cnt)[i];
            const int64_t cp = c2.x, cq = c2.y;
            const uint2 st = pst[i];
            const int64_t t0 = (int64_t)st.x * n_Q - (int64_t)st.y * n_P;
            const int64_t hi = t0 + cp * n_Q, lo = t0 - cq * n_P;
            const uint64_t bound = (uint64_t)max(hi < 0 ? -hi : hi, lo < 0 ? -lo : lo);
            cand = cp + cq >= 2 && bound > cnum[s];
            if (cand) {
                coff[i] = atomicAdd(&seg[2 * s], (uint32_t)(cp + cq));
                fill[i] = 0u;
                clist[(int64_t)s * nbk + atomicAdd(&seg[2 * s + 1], 1u)] = (int32_t)(i - (int64_t)s * nbk);
            } else if (cp + cq) {
                reinterpret_cast<uint2*>(cnt)[i] = make_uint2(0u, 0u);
            }
        }
        const uint32_t w = __ballot_sync(0xffffffffu, cand);
        if ((threadIdx.x & 31) == 0 && i < total) cbits[i >> 5] = w;
    }
}

// candidate keys, grouped by bucket (order inside a bucket arbitrary): ck[s * N + coff[b] + k]. grid (chunks, nseg):
// the CTA holds segment s's candidate bitmap in SMEM (nbk / 8 bytes), so a non-candidate key costs its coalesced
// load, its bucket and one shared-memory bit test; only candidate keys touch coff / fill (global).
constexpr int RDB_CT = 512;
#ifndef DDKS_RDB_U  // experiments: keys in flight per compaction thread, compaction CTAs per SM
#define DDKS_RDB_U 4
#endif
#ifndef DDKS_RDB_CPS
#define DDKS_RDB_CPS 3
#endif
__global__ void __launch_bounds__(RDB_CT) k_rdb_compact(const uint64_t* __restrict__ key, int64_t N, int nbk,
                                                        double scale, const uint32_t* __restrict__ cbits,
                                                        const uint32_t* __restrict__ coff, uint32_t* __restrict__ fill,
                                                        uint64_t* __restrict__ ck) {
    extern __shared__ uint4 sbits4[];
    const int s = blockIdx.y;
    const uint4* src = reinterpret_cast<const uint4*>(cbits + (int64_t)s * (nbk / 32));
    for (int i = threadIdx.x; i < nbk / 128; i += RDB_CT) sbits4[i] = src[i];
    __syncthreads();
    const uint32_t* sbits = reinterpret_cast<const uint32_t*>(sbits4);
    const uint64_t* ks = key + (int64_t)s * N;
    constexpr int U = DDKS_RDB_U;  // keys in flight per thread
    const int64_t gs = (int64_t)gridDim.x * RDB_CT;
    for (int64_t e0 = blockIdx.x * (int64_t)RDB_CT + threadIdx.x; e0 < N; e0 += U * gs) {
        uint64_t k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) k[u] = e0 + u * gs < N ? __ldcs(ks + e0 + u * gs) : 0ull;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (e0 + u * gs >= N) break;
            const int b = rdb_bucket(k[u], scale, nbk);
            if ((sbits[b >> 5] >> (b & 31)) & 1u) {
                const int64_t bi = (int64_t)s * nbk + b;
                const uint32_t pos = coff[bi] + atomicAdd(&fill[bi], 1u);
                DDKS_ASSERT(pos < N);
                ck[(int64_t)s * N + pos] = k[u];
            }
        }
    }
}

// One CTA per candidate bucket (grid-stride over the segment's list): bitonic sort of its <= RDB_CAPK keys in SMEM,
// then the exact sweep from the bucket's start counts; atomicMax into cnum[s].
__global__ void __launch_bounds__(256) k_rdb_finish(const uint64_t* __restrict__ ck, int64_t N, int nbk,
                                                    uint32_t* __restrict__ cnt, const uint2* __restrict__ pst,
                                                    const uint32_t* __restrict__ coff,
                                                    const int32_t* __restrict__ clist,
                                                    const uint32_t* __restrict__ seg, int64_t n_P, int64_t n_Q,
                                                    unsigned long long* __restrict__ cnum, uint32_t* flag) {
    __shared__ uint64_t sk[RDB_CAPK];
    const int s = blockIdx.y;
    // too many candidate keys (e.g. nearly identical samples): cheaper to sort everything, the caller falls back
    if (seg[2 * s] > (uint32_t)(N / 2)) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(flag, 256u);
        return;
    }
    for (int k = blockIdx.x; k < (int)seg[2 * s + 1]; k += gridDim.x) {
        const int b = clist[(int64_t)s * nbk + k];
        const int64_t i = (int64_t)s * nbk + b;
        const int n = (int)(cnt[2 * i] + cnt[2 * i + 1]);
        if (n > RDB_CAPK) {
            // too large for SMEM: harmless if every key has the same distance (no tie-group end inside), else the
            // caller re-runs the full sort
            const uint64_t* src = ck + (int64_t)s * N + coff[i];
            uint64_t mn = ~0ull, mx = 0;
            for (int j = threadIdx.x; j < n; j += blockDim.x) mn = min(mn, src[j] >> 1), mx = max(mx, src[j] >> 1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mn = min(mn, (uint64_t)__shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, (uint64_t)__shfl_xor_sync(0xffffffffu, mx, o));
            }
            if ((threadIdx.x & 31) == 0 && mn != mx) atomicOr(flag, 256u);
            __syncthreads();  // every thread has read the counts
            if (threadIdx.x == 0) reinterpret_cast<uint2*>(cnt)[i] = make_uint2(0u, 0u);
            continue;
        }
        int np2 = 1;
        while (np2 < n) np2 <<= 1;
        const uint64_t* src = ck + (int64_t)s * N + coff[i];
        DDKS_ASSERT(coff[i] + (int64_t)n <= N && np2 <= RDB_CAPK);
        for (int j = threadIdx.x; j < np2; j += blockDim.x) sk[j] = j < n ? src[j] : ~0ull;
        __syncthreads();
        for (int size = 2; size <= np2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int j = threadIdx.x; j < np2; j += blockDim.x) {
                    const int p = j ^ stride;
                    if (p > j) {
                        const bool up = (j & size) == 0;
                        const uint64_t a = sk[j], c = sk[p];
                        if ((a > c) == up) sk[j] = c, sk[p] = a;
                    }
                }
                __syncthreads();
            }
        // sweep: blocked arrangement, 16 keys per thread (256 x 16 = RDB_CAPK)
        const uint2 st = pst[i];
        uint32_t mine = 0;
        const int j0 = threadIdx.x * (RDB_CAPK / 256);
        for (int j = j0; j < j0 + RDB_CAPK / 256 && j < n; ++j) mine += (uint32_t)((sk[j] & 1ull) == 0);
        uint32_t before = block_excl_scan256(mine);
        int64_t iP = (int64_t)st.x + before;
        uint64_t best = 0;
        for (int j = j0; j < j0 + RDB_CAPK / 256 && j < n; ++j) {
            iP += (int64_t)((sk[j] & 1ull) == 0);
            if (j + 1 < n && (sk[j + 1] >> 1) == (sk[j] >> 1)) continue;  // not a tie-group end
            const int64_t iQ = (int64_t)st.x + st.y + j + 1 - iP;
            const int64_t t = iP * n_Q - iQ * n_P;
            const uint64_t a = (uint64_t)(t < 0 ? -t : t);
            best = a > best ? a : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t v = __shfl_xor_sync(0xffffffffu, best, o);
            best = v > best ? v : best;
        }
        if ((threadIdx.x & 31) == 0 && best) atomicMax(&cnum[s], (unsigned long long)best);
        __syncthreads();  // sk is reused by the next bucket; every thread has read the counts
        if (threadIdx.x == 0) reinterpret_cast<uint2*>(cnt)[i] = make_uint2(0u, 0u);  // clean for the next call
    }
}

}  // namespace ddks
