// ddks_rank.cuh — the rank-lane count: rows a3 + a4 (orthant classification + per-orthant counting)
// for single statistics in position order, with ceil(d / 3) integer adds per pair instead of d FP32 compares +
// d FFMAs (default at d = 3 and d = 5..8 in the measured N ranges of rank_applicable, ddks_api.cu). DIFF counters in
// one launch; SPLIT counters as two launches over the P rows and the Q rows (RankArgs::pt_rows with a.N / a.n_P set per launch).
//
// What it computes is unchanged (Eq. 3: bit k of the orthant code = [x_k >= o_k], P:L46 loop
// method, P:L238 normalised difference): every (origin, point) pair of the CTA's 384 origins and the segment's points
// is classified by its own d comparisons and increments exactly one counter of its origin.
//
// How the comparisons are done (DESIGN.md §7 "rank lanes"): a CTA owns 384 origins. For each dim k let V_k be the
// multiset of its origins' x_k values. For any real x and any o in V_k
//     x >= o   <=>   #{v in V_k : v <= x}  >=  #{v in V_k : v <= o}
// (if x >= o every v <= o is <= x; if x < o, o itself is counted on the right and not on the left, and nothing counted
// on the left is missing on the right). Both counts lie in [0, 511] (V_k is padded to 511 entries with +inf), so the
// compare of two floats becomes the compare of two small integers rx = rank(x), ro = rank(o), and three of those fit
// one 32-bit word: 10-bit lanes holding rx + (512 - ro) in [1, 1023] — no borrow, no carry between lanes — whose top
// bit is exactly [x_k >= o_k]. A point has NW = ceil(d / 3) rank words (1 for d <= 3, 2 for d = 4..6, 3 for d = 7, 8):
// dim k lives in word j = k % NW, lane i = k / NW, at bit offset j + 10 i, so the d result bits of the OR of the masked
// words sit at bits 9 + j + 10 i — three groups of NW adjacent bits — and one multiply (RankGeo::MUL: a sum of three
// powers of two whose partial products never overlap, so no carries) moves group i next to group i - 1 at the top of
// the word, leaving the orthant code sum_k [x_k >= o_k] 2^k after one shift. Per pair: NW IADD, NW LOP3, IMAD, SHF,
// IMAD (counter address), ATOMS and 1 / PPL of a broadcast LDS.128 (PPL = 4, 2, 1 points per load): ~6.3
// instructions at d = 3 and ~11 at d = 8, against d FSET + d FFMA + ATOMS + LDS for the FP32 path.
//
// The ranks of the points are taken per CTA and tile: each thread maps one point of the 384-point tile (d branch-free
// searches of V_k, stored in Eytzinger order so the nine probe levels spread over the SMEM banks), the rank words go to
// a double-buffered SMEM tile, and all threads then classify the tile against their origin. V_k is sorted once per
// origin block by k_rank_sort (a bitonic network in SMEM, one CTA per (block, dim)).
#pragma once
#include "ddks_kernels.cuh"

namespace ddks {
namespace {

#ifndef DDKS_RK_PTS  // points per step of the rank-lane count loop
#define DDKS_RK_PTS 24
#endif
constexpr int RK_PTS = DDKS_RK_PTS;
#ifndef DDKS_RK_PTS1  // the same for one rank word per point (d <= 3: four points per LDS.128)
#define DDKS_RK_PTS1 16
#endif
#ifndef DDKS_RK_CTAS1  // resident CTAs per SM the d <= 3 kernels are register-capped for (16 x 4 measured best at C2:
                       // count 0.107 ms against 0.109 - 0.111 for 24 x 3, 32 x 3, 16 x 3, 24 x 4)
#define DDKS_RK_CTAS1 4
#endif
#ifndef DDKS_RK_R  // origins per thread of the rank-lane count (1: 384 threads, 2: 192 threads)
#define DDKS_RK_R 1
#endif

template <int D> struct RankGeo {
    static_assert(D >= 1 && D <= 9, "three 10-bit lanes per word, up to three words");
    static constexpr int NW = (D + 2) / 3;     // rank words per point / origin: dim k in word k % NW, lane k / NW
    static constexpr int NWS = NW == 3 ? 4 : NW;  // words stored per point in the SMEM tile (16 B holds 4 / NWS points)
    static constexpr int PPL = 4 / NWS;        // points per LDS.128
    // the gather multiply: result bits 9 + j + 10 i (word j, lane i) -> orthant code in the product's top bits
    //   NW = 1: bits 9, 19, 29           x (1 + 2^9 + 2^18) -> bits 27..29 (others land on 9, 18, 19)
    //   NW = 2: bits {9,10} + 10 i       x (2 + 2^9 + 2^17) -> bits 26..31 (others on 10, 11, 18..21)
    //   NW = 3: bits {9,10,11} + 10 i    x (1 + 2^7 + 2^14) -> bits 23..31 (others on 9..11, 16..21)
    // every partial product occupies its own bits, so the sum has no carries
    static constexpr uint32_t MUL = NW == 1 ? 0x40201u : (NW == 2 ? 0x20202u : 0x4081u);
    static constexpr int SH = NW == 1 ? 27 : (NW == 2 ? 26 : 23);
    static constexpr int ORIGINS = 384;        // origins per CTA (384 / RR threads, RR origins each)
    static constexpr int TILE = ORIGINS;       // points per tile: RR per thread to rank
    static constexpr int WPB = ORIGINS / 2;    // counter words per bin (two signed 16-bit halves per word)
    static constexpr int NQ = 1 << D, NB = NQ; // DIFF counters only
    static constexpr int VN = 511;             // Eytzinger tree of 9 levels: 384 origin values + 127 x +inf
    static constexpr int VW = 512;             // floats per (block, dim) in the workspace and in SMEM
    static constexpr int HIST_WORDS = NB * WPB;
    static constexpr int SMEM_BYTES = HIST_WORDS * 4 + D * VW * 4 + 2 * TILE * NWS * 4 + 64;
    static constexpr int MIN_CTAS = D >= 8 ? 1 : (D >= 6 ? 2 : (D >= 4 ? 3 : DDKS_RK_CTAS1));
    static constexpr int PTS = NW == 1 ? DDKS_RK_PTS1 : RK_PTS;  // points per step of the count loop
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
    __host__ __device__ static constexpr int slot(int t) { return t % WPB; }
    __host__ __device__ static constexpr bool high(int t) { return t >= WPB; }
};

// result-bit mask of word j: bits 9 + j + 10 i for the dims k = NW i + j < D
__host__ __device__ constexpr uint32_t rank_mask(int j, int D) {
    const int NW = (D + 2) / 3;
    uint32_t m = 0;
    if (j >= NW) return 0u;
    for (int i = 0; NW * i + j < D; ++i) m |= 1u << (9 + j + 10 * i);
    return m;
}

// 16-byte SMEM load kept in program order with the counter REDs (asm volatile): a step's RK_PTS loads all issue
// before its first RED (the compiler otherwise interleaves them with the classification and exposes their latency)
__device__ __forceinline__ uint4 lds_v4(const uint4* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}

// #{v in V : v <= x} for the 511-node Eytzinger tree E (node i's children 2i+1, 2i+2): nine probes, branch-free
__device__ __forceinline__ uint32_t eyt_rank(const float* E, float x) {
    uint32_t i = 0;
#pragma unroll
    for (int l = 0; l < 9; ++l) i = 2u * i + 1u + (E[i] <= x ? 1u : 0u);
    return i - 511u;
}

// V_k of every origin block, sorted and laid out as an Eytzinger tree: one CTA of 256 threads per (block, dim).
// out[(blk * D + k) * 512 + i] = node i (i < 511). Origin slots past o_end repeat origin o_end - 1 (as k_count's
// clamped slots), which only duplicates a value of V_k.
template <int D>
__global__ void __launch_bounds__(256) k_rank_sort(const float* __restrict__ pts, int DP, int32_t o_begin,
                                                   int32_t o_end, float* __restrict__ out) {
    __shared__ float s[512];
    const int blk = blockIdx.x, k = blockIdx.y, t = threadIdx.x;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = t + 256 * h;
        float v = INFINITY;
        if (i < RankGeo<D>::ORIGINS) {
            int32_t oi = o_begin + blk * RankGeo<D>::ORIGINS + i;
            oi = oi < o_end ? oi : o_end - 1;
            v = pts[(int64_t)oi * DP + k];
        }
        s[i] = v;
    }
    __syncthreads();
    // bitonic sort of 512 values, ascending (one compare-exchange per thread and step)
    for (int kk = 2; kk <= 512; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const int i = 2 * t - (t & (j - 1)), l = i + j;
            const float a = s[i], b = s[l];
            const bool up = (i & kk) == 0;
            if ((a > b) == up) s[i] = b, s[l] = a;
            __syncthreads();
        }
    }
    // node i at level L (i in [2^L - 1, 2^(L+1) - 1)), position q in its level: in-order index (2q + 1) 2^(8-L) - 1
    float* o = out + ((int64_t)blk * D + k) * RankGeo<D>::VW;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = t + 256 * h;
        if (i >= RankGeo<D>::VN) continue;
        const int L = 31 - __clz(i + 1), q = i + 1 - (1 << L);
        o[i] = s[(2 * q + 1) * (1 << (8 - L)) - 1];
    }
}

// the three rank words of a point (or, with neg, of an origin: 512 - rank in each lane)
template <int D, bool NEG>
__device__ __forceinline__ void rank_words(const float* V, const float (&x)[D], uint32_t (&w)[3]) {
    constexpr int NW = RankGeo<D>::NW;
    w[0] = w[1] = w[2] = 0u;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const uint32_t r = eyt_rank(V + k * RankGeo<D>::VW, x[k]);
        w[k % NW] |= (NEG ? 512u - r : r) << ((k % NW) + 10 * (k / NW));
    }
}

// Work: units = (origin block, 384-point tile) pairs, linearised block-major; CTA c owns units
// [c U / grid, (c + 1) U / grid) (stream-K: every SM gets the same number of tiles, and a CTA visits at most a few
// blocks). Per visited block the CTA loads V_k and its origin's rank words, classifies its tile range in chunks of at
// most chunk_tiles (the int16 window) and flushes exact int32 partials to a.accum after each chunk (k_finalize sums
// them), or -- a.accum == nullptr, one CTA per whole block -- finalises in-kernel.
struct RankArgs {
    const float* vsorted;  // [blocks][D][VW] Eytzinger trees (k_rank_sort)
    const float* pt_rows;  // the rows counted by this launch, a.N of them, the first a.n_P with inc P: all packed rows for
                           //   DIFF counters; SPLIT counters (c_P and c_Q kept apart) take the P rows and the Q rows in
                           //   two launches (the origins always come from a.pts)
    int32_t n_tiles;       // tiles per block (the rows of the launch in 384-point tiles)
    int32_t chunk_tiles;   // tiles per flush window
    int64_t units;         // blocks * n_tiles
};

// RR origins per thread (T = 384 / RR threads): thread t owns origins t + r T of the block, i.e. with RR = 2 both
// 16-bit halves of counter column t, and every point's rank words (one LDS.128) serve RR classifications.
template <int D, int RR>
__global__ void __launch_bounds__(RankGeo<D>::ORIGINS / RR, RankGeo<D>::MIN_CTAS) k_count_rank(const CountArgs a, const RankArgs ra) {
    using G = RankGeo<D>;
    constexpr int OB = G::ORIGINS, T = OB / RR, TILE = G::TILE, WPB = G::WPB, DP = padded_dim<D>();
    constexpr int NW = G::NW, NWS = G::NWS, PPL = G::PPL;
    constexpr int PTS = G::PTS;
    static_assert(PTS % 4 == 0, "whole LDS.128 groups per step");
    static_assert(RR == 1 || RR == 2, "one or two origins per thread");
    constexpr uint32_t M0 = rank_mask(0, D), M1 = rank_mask(1, D), M2 = rank_mask(2, D);
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem);                                   // [NB][WPB]
    float* V = reinterpret_cast<float*>(smem + G::HIST_WORDS * 4);                      // [D][VW] Eytzinger
    uint32_t* W = reinterpret_cast<uint32_t*>(smem + G::HIST_WORDS * 4 + D * G::VW * 4);  // [2][TILE][NWS] rank words

    const int t = threadIdx.x;
    const float* pts = a.pts;
    const float* ppts = ra.pt_rows;
    uint32_t ubase[RR], incP[RR], incQ[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        const int oo = t + r * T;  // origin offset in the block
        ubase[r] = smem_u32(hist) + 4u * (uint32_t)G::slot(oo);
        incP[r] = G::high(oo) ? a.incP << 16 : a.incP;
        incQ[r] = G::high(oo) ? a.incQ << 16 : a.incQ;
    }
    const int64_t u_begin = (int64_t)blockIdx.x * ra.units / gridDim.x;
    const int64_t u_end = (int64_t)(blockIdx.x + 1) * ra.units / gridDim.x;

    const bool probe = a.clk && t == 0 && (blockIdx.x & 7) == 0;
    unsigned long long clk0 = 0, ns0 = 0;
    if (probe) clk0 = clock64(), ns0 = globaltimer_ns();
    unsigned long long pts_done = 0, visits = 0;

    for (int i = t; i < G::HIST_WORDS; i += T) hist[i] = 0u;
    for (int64_t u = u_begin; u < u_end;) {
        const int32_t by = (int32_t)(u / ra.n_tiles);
        const int32_t tb = (int32_t)(u - (int64_t)by * ra.n_tiles);
        const int32_t te = (int32_t)min((int64_t)min(ra.n_tiles, tb + ra.chunk_tiles), (int64_t)tb + (u_end - u));
        u += te - tb;
        const int32_t blk_o0 = a.o_begin + by * OB;
        const int32_t seg0 = tb * TILE, seg1 = min(a.N, te * TILE);
        const int n_tiles = te - tb;
        ++visits;
        pts_done += (unsigned long long)(seg1 - seg0);
        __syncthreads();  // the previous chunk's V, W and counters are no longer read
        {
            const float4* src = reinterpret_cast<const float4*>(ra.vsorted + (int64_t)by * D * G::VW);
            float4* dst = reinterpret_cast<float4*>(V);
            for (int i = t; i < D * G::VW / 4; i += T) dst[i] = __ldg(src + i);
        }
        // this thread's origins (clamped slots repeat o_end - 1 and are ignored at the end) and its first points
        float o[RR][D], xn[RR][D];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            int32_t oi = blk_o0 + t + r * T;
            oi = oi < a.o_end ? oi : a.o_end - 1;
            load_point<D>(pts + (int64_t)oi * DP, o[r]);
            if (seg0 + t + r * T < seg1) load_point<D>(ppts + (int64_t)(seg0 + t + r * T) * DP, xn[r]);
        }
        __syncthreads();  // V visible
        uint32_t ow[RR][3];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            rank_words<D, true>(V, o[r], ow[r]);
            if (seg0 + t + r * T < seg1) {
                uint32_t xw[3];
                rank_words<D, false>(V, xn[r], xw);
#pragma unroll
                for (int j = 0; j < NW; ++j) W[(t + r * T) * NWS + j] = xw[j];
            }
        }
        for (int it = 0; it < n_tiles; ++it) {
            // the next tile's points of this thread (global / L2 loads in flight during the count)
            const int32_t pn = seg0 + (it + 1) * TILE + t;
#pragma unroll
            for (int r = 0; r < RR; ++r)
                if (it + 1 < n_tiles && pn + r * T < seg1) load_point<D>(ppts + (int64_t)(pn + r * T) * DP, xn[r]);
            __syncthreads();  // tile it's words written; tile it - 1's words no longer read
            const uint32_t* Wt = W + (it & 1) * (TILE * NWS);
            const int32_t p0 = seg0 + it * TILE;
            const int32_t cnt = min(TILE, seg1 - p0);
            int32_t split = a.n_P - p0;
            split = split < 0 ? 0 : (split > cnt ? cnt : split);
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {
                const int lo = part ? split : 0, hi = part ? cnt : split;
                uint32_t inc[RR];
#pragma unroll
                for (int r = 0; r < RR; ++r) inc[r] = part ? incQ[r] : incP[r];
                auto count = [&](uint32_t x0, uint32_t x1, uint32_t x2) {
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        uint32_t w = (x0 + ow[r][0]) & M0;
                        if (NW > 1) w |= (x1 + ow[r][1]) & M1;
                        if (NW > 2) w |= (x2 + ow[r][2]) & M2;
                        const uint32_t code = (w * G::MUL) >> G::SH;  // sum_k [x_k >= o_k] 2^k
                        DDKS_ASSERT(code < (uint32_t)G::NQ);
                        red_add_shared(ubase[r] + code * (4u * WPB), inc[r]);
                    }
                };
                auto count_one = [&](int q) {
                    const uint32_t* wq = Wt + q * NWS;
                    count(wq[0], NW > 1 ? wq[1] : 0u, NW > 2 ? wq[2] : 0u);
                };
                auto count_v4 = [&](const uint4& v) {  // one LDS.128 = PPL points
                    if (PPL == 1) count(v.x, v.y, v.z);
                    if (PPL == 2) count(v.x, v.y, 0u), count(v.z, v.w, 0u);
                    if (PPL == 4) count(v.x, 0u, 0u), count(v.y, 0u, 0u), count(v.z, 0u, 0u), count(v.w, 0u, 0u);
                };
                int p = lo;
                for (; p < hi && (p % PPL) != 0; ++p) count_one(p);  // up to a 16-byte boundary of the tile
                // PTS points per step, all loads issued first: PTS x RR independent chains per warp
#pragma unroll 1
                for (; p + PTS <= hi; p += PTS) {
                    uint4 xv[PTS / PPL];
#pragma unroll
                    for (int j = 0; j < PTS / PPL; ++j) xv[j] = lds_v4(reinterpret_cast<const uint4*>(Wt + p * NWS) + j);
#pragma unroll
                    for (int j = 0; j < PTS / PPL; ++j) count_v4(xv[j]);
                }
                for (; p < hi; ++p) count_one(p);
            }
            // the next tile's rank words into the other buffer (read by nobody until the barrier above)
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                if (it + 1 < n_tiles && pn + r * T < seg1) {
                    uint32_t xw[3];
                    rank_words<D, false>(V, xn[r], xw);
#pragma unroll
                    for (int j = 0; j < NW; ++j) W[(((it + 1) & 1) * TILE + t + r * T) * NWS + j] = xw[j];
                }
            }
        }
        __syncthreads();  // all red.shared retired before reading the counters
        if (a.accum != nullptr) {
            // exact int32 partials -> global (fire-and-forget REDs); each counter word (two origins' halves) is read
            // and re-zeroed by one thread, coalesced over consecutive slots
            int32_t* acc = a.accum + (int64_t)by * OB;
            for (int wi = t; wi < G::HIST_WORDS; wi += T) {
                const int q = wi / WPB, s2 = wi - q * WPB;
                const uint32_t wv = hist[wi];
                if (wv == 0u) continue;
                hist[wi] = 0u;
                int32_t lo, hi;
                split16(wv, lo, hi);
                DDKS_ASSERT((int64_t)by * OB + s2 + WPB < a.acc_stride + OB);
                if (lo && blk_o0 + s2 < a.o_end) atomicAdd(&acc[(int64_t)q * a.acc_stride + s2], lo);
                if (hi && blk_o0 + s2 + WPB < a.o_end) atomicAdd(&acc[(int64_t)q * a.acc_stride + s2 + WPB], hi);
            }
            continue;
        }
        // direct mode (this CTA owns the whole block): num(o), the per-origin export, the CTA max, the argmax key
        uint64_t best = 0;
        unsigned long long bkey = 0;
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            const int oo = t + r * T;
            const int32_t myo = blk_o0 + oo;
            if (myo >= a.o_end) continue;
            uint32_t mm = 0;
            for (int q = 0; q < G::NQ; ++q) {
                int32_t lo, hi;
                split16(hist[q * WPB + G::slot(oo)], lo, hi);
                const int32_t v = G::high(oo) ? hi : lo;
                const uint32_t av = (uint32_t)(v < 0 ? -v : v);
                mm = av > mm ? av : mm;
            }
            const uint64_t red = mm;
            const uint64_t m = red * a.gg;
            if (a.per_origin) a.per_origin[myo - a.o_begin] = m;
            best = m > best ? m : best;
            if (a.best_key) {
                const unsigned long long k = ((unsigned long long)red << 31) | (unsigned long long)(0x7fffffff - myo);
                bkey = k > bkey ? k : bkey;
            }
        }
        best = warp_max_u64(best);
        bkey = warp_max_u64(bkey);
        __shared__ uint64_t wmax[T / 32], wkey[T / 32];
        if ((t & 31) == 0) wmax[t >> 5] = best, wkey[t >> 5] = bkey;
        __syncthreads();
        if (t == 0) {
            uint64_t m = 0, k = 0;
            for (int w = 0; w < T / 32; ++w) m = wmax[w] > m ? wmax[w] : m, k = wkey[w] > k ? wkey[w] : k;
            atomicMax(reinterpret_cast<unsigned long long*>(&a.item_num[0]), (unsigned long long)m);
            if (a.best_key) atomicMax(a.best_key, (unsigned long long)k);
        }
        __syncthreads();
        for (int i = t; i < G::HIST_WORDS; i += T) hist[i] = 0u;
    }
    if (a.clk && t == 0) {
        // executed compares: the d of every pair (done as three 32-bit adds on 10-bit lanes) and the rank searches'
        // FP32 compares (9 per point, dim and visit)
        atomicAdd(&a.clk[2], (unsigned long long)D * pts_done * OB + 9ull * D * (pts_done + visits * OB));
        if (probe) {
            atomicAdd(&a.clk[0], (unsigned long long)(clock64() - clk0));
            atomicAdd(&a.clk[1], globaltimer_ns() - ns0);
        }
    }
}

}  // namespace
}  // namespace ddks
